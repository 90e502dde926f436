# fp64 tensor-core peak; c3 per-launch DRAM traffic of the step's kernels (tf32 headline)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_rate tools/dmma_rate.cu && ./tools/dmma_rate > gpurun_out/dmma_rate.txt 2>&1
cat gpurun_out/dmma_rate.txt
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/c3_traffic.csv \
  python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/c3_traffic.log 2>&1
echo "ncu rc=$?"
grep -c symkr gpurun_out/c3_traffic.csv
