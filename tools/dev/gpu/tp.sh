timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_f32" 2>&1 | tail -5
for e in 0 1; do
  if [ $e = 1 ]; then export CURVKIT_SERIAL_DOWNLOAD=1; fi
  echo "serial=$e"
  CURVKIT_HOST_TIMING=1 timeout 900 python bench.py --no-extra --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 5 2>&1 | grep -o '"ms_per_step": [0-9.]*, "path"\|"result_symmetric": [a-z]*\|\[curvkit\] assemble_opg [a-z+]* [0-9.]* ms' | tr '\n' ' ' | sed 's/\[curvkit\] assemble_opg upload/\n  upload/g'
  echo
done
