timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py tests/test_bands.py -m gpu -q -x -k "hessian or band" > gpurun_out/f6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f6_tests.log
for d in 0 16 3 19 11 27; do
  CURVKIT_DEV_FUSED=$d timeout 300 python bench.py --config c2 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('c2 dev $d', round(d['ms_per_step'],3), round(k['hess_fused']['ms_per_step'],3), round(k['hess_fused']['tflops'],1), d['clocks']['sm_mhz'])
" >> gpurun_out/f6.txt
done
tail -n 2 gpurun_out/f6_tests.log; cat gpurun_out/f6.txt
