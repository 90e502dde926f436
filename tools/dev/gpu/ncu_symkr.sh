# full ncu captures of the c2 layer-0 symmetric-kernel launch, tf32 and f16s
for prec in tf32 f16s; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:symkr -c 1 -o gpurun_out/c2_symkr_$prec \
  python bench.py --config c2 --precision $prec --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ncu_c2_$prec.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c2_$prec.log
done
ls -la gpurun_out/*.ncu-rep
