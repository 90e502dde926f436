timeout 120 python tools/hess_c1_once.py c1 5 2>&1 | tail -1 | grep -o "'hess_symkr': ([^)]*)" || echo "c1 run failed/hung"
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_shards.py -x -q -m gpu -k "hessian or config1 or config2 or union or opg" 2>&1 | tail -2
timeout 300 python tools/run_configs.py c2 2>&1 | grep -o "'hess_symkr': ([^)]*)"
