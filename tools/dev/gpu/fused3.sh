for ts in 0 1; do
  if [ $ts = 1 ]; then export CURVKIT_HESS_TS=1; else unset CURVKIT_HESS_TS; fi
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py -m gpu -q -x -k "hessian" > gpurun_out/fc_tests_$ts.log 2>&1; echo "rc=$?" >> gpurun_out/fc_tests_$ts.log
  for cfg in c2 c1; do for d in 0 3; do
  CURVKIT_DEV_FUSED=$d timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('ts $ts $cfg dev $d', round(d['ms_per_step'],3), round(k['hess_fused']['ms_per_step'],3), round(k['hess_fused']['tflops'],1), d['clocks']['sm_mhz'])
" >> gpurun_out/fused3.txt
  done; done
done
tail -n 2 gpurun_out/fc_tests_*.log; cat gpurun_out/fused3.txt
