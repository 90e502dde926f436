timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_shards.py -x -q -m gpu -k "hessian or config1 or config2 or union or opg" 2>&1 | tail -2
for d in 0 128; do echo "== dev=$d"; CURVKIT_DEV_SYMKR=$d timeout 60 python tools/hess_c1_once.py c1 5 2>&1 | tail -1 | grep -o "'hess_symkr': ([^)]*)"; done
rm -f gpurun_out/symkr_epi_*.bin; CURVKIT_TRACE=1 timeout 60 python tools/hess_c1_once.py c1 2 2>&1 | tail -1 | grep -o "'hess_symkr': ([^)]*)"; python tools/symkr_epi_trace.py gpurun_out/symkr_epi_0.bin
