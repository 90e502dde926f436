timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_shards.py -x -q -m gpu -k "hessian or config1 or config2 or config3 or union or opg" 2>&1 | tail -2
for ss in 0 1; do echo "== SS=$ss"; if [ $ss = 1 ]; then export CURVKIT_SYMKR_SS=1; fi
timeout 60 python tools/hess_c1_once.py c1 5 2>&1 | tail -1 | grep -o "'hess_symkr': ([^)]*)"
CURVKIT_DEV_SYMKR=3 timeout 60 python tools/hess_c1_once.py c1 5 2>&1 | tail -1 | grep -o "'hess_symkr': ([^)]*)"
timeout 300 python tools/run_configs.py c2 c3 2>&1 | grep -o "'[a-z_]*symkr': ([^)]*)\|c3 opg 1.*\|c2 hessian 1.*"; done
