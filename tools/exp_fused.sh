timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config1_hessian" 2>&1 | grep -E "Error|assert|rel|passed|failed" | head -20
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "hessian or config2" 2>&1 | tail -2
for d in 0 1 2; do echo "== dev=$d"; CURVKIT_DEV_SYMKR=$d timeout 120 python tools/hess_c1_once.py c1 5 2>&1 | tail -1; done
