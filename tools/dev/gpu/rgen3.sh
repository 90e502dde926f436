timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py tests/test_bands.py -m gpu -q -x -k "hessian or hvp or band" > gpurun_out/rgen_tests0.log 2>&1; echo "rc=$?" >> gpurun_out/rgen_tests0.log
CURVKIT_HESS_RGEN=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py -m gpu -q -x -k "hessian" > gpurun_out/rgen_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rgen_tests.log
for r in 0 1; do for cfg in c2 c1; do
  if [ $r = 1 ]; then export CURVKIT_HESS_RGEN=1; else unset CURVKIT_HESS_RGEN; fi
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('rgen $r $cfg', round(d['ms_per_step'],3), {a:round(b['ms_per_step'],3) for a,b in k.items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/rgen3.txt
done; done
unset CURVKIT_HESS_RGEN
timeout 300 python bench.py --config c1 --precision f64 --steps 3 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('c1 f64', round(d['ms_per_step'],3), {a:round(b['ms_per_step'],3) for a,b in d['kernels'].items()})
" >> gpurun_out/rgen3.txt
tail -n 2 gpurun_out/rgen_tests0.log gpurun_out/rgen_tests.log; cat gpurun_out/rgen3.txt
