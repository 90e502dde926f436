timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py -m gpu -q -x -k "hessian_matches or opg_and or c1" > gpurun_out/w16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w16_tests.log
for w in 0 1; do
  CURVKIT_SYMKR_W16=$w timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('w16 $w c1', round(d['ms_per_step'],3), {a:(round(b['ms_per_step'],3), round(b['tflops'] or 0,1)) for a,b in k.items() if 'symkr' in a}, d['clocks']['sm_mhz'])
" >> gpurun_out/w16.txt
  tail -2 gpurun_out/ab.log | cut -c1-300 >> gpurun_out/w16.txt
done
tail -n 4 gpurun_out/w16_tests.log; cat gpurun_out/w16.txt
