timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py tests/test_bands.py tests/test_acceptance.py -m gpu -q -x -k "hessian or hvp or band or acceptance" > gpurun_out/rgen_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rgen_tests.log
for prec in tf32 f16s; do for cfg in c2 c1; do
  timeout 300 python bench.py --config $cfg --precision $prec --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$prec $cfg', round(d['ms_per_step'],3), {a:(round(b['ms_per_step'],3), round(b['tflops'] or 0,1)) for a,b in k.items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/rgen4.txt
done; done
tail -n 2 gpurun_out/rgen_tests.log; cat gpurun_out/rgen4.txt
