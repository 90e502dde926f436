timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_shards.py -x -q -m gpu -k "hessian or config1 or config2 or union" 2>&1 | tail -2
for d in 0 2 3; do echo "== dev=$d"; CURVKIT_DEV_SYMKR=$d timeout 120 python tools/hess_c1_once.py c1 5 2>&1 | tail -1; done
rm -f gpurun_out/symkr_trace_*.bin; CURVKIT_TRACE=1 timeout 120 python tools/hess_c1_once.py c1 2 2>&1 | tail -1; python tools/trace_fused.py gpurun_out/symkr_trace_0.bin 2>&1 | grep -v "transform:"
