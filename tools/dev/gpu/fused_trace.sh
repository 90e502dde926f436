mkdir -p gpurun_out/tr0 gpurun_out/tr3
CURVKIT_TRACE=1 timeout 300 python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/tr.log 2>&1
mv gpurun_out/trace_*.bin gpurun_out/tr0/ 2>/dev/null
CURVKIT_DEV_FUSED=3 CURVKIT_TRACE=1 timeout 300 python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/tr.log 2>&1
mv gpurun_out/trace_*.bin gpurun_out/tr3/ 2>/dev/null
python tools/dev/trace_fused.py gpurun_out/tr0/trace_0.bin gpurun_out/tr3/trace_0.bin
