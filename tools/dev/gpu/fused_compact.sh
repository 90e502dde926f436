timeout 900 python -m pytest tests/test_gpu_sketch_pins.py tests/test_gpu_parity.py tests/test_bands.py -m gpu -q -x -k "hessian or band" > gpurun_out/fc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fc_tests.log
for nc in 1 0; do for cfg in c2 c1; do
  if [ $nc = 1 ]; then export CURVKIT_FUSED_NOCOMPACT=1; else unset CURVKIT_FUSED_NOCOMPACT; fi
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('nocompact $nc $cfg', round(d['ms_per_step'],3), round(k['hess_fused']['ms_per_step'],3), round(k['hess_fused']['tflops'],1), d['clocks']['sm_mhz'])
" >> gpurun_out/fc_ab.txt
done; done
tail -n 3 gpurun_out/fc_tests.log; cat gpurun_out/fc_ab.txt
