for k in 16 64; do
  echo "keep=$k"
  CURVKIT_POOL_KEEP_GB=$k CURVKIT_HOST_TIMING=1 timeout 900 python bench.py --no-extra --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 5 2>&1 | grep -o '"ms_per_step": [0-9.]*, "path"\|\[curvkit\] assemble_opg [a-z+]* [0-9.]* ms' | tr '\n' ' ' | sed 's/\[curvkit\] assemble_opg upload/\n  upload/g'
  echo
done
