timeout 900 python -m pytest tests/test_gpu_sketch_pins.py tests/test_gpu_parity.py tests/test_bands.py -m gpu -q -x -k "sketch or f16s or hessian_matches or opg_and or band" > gpurun_out/zr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zr_tests.log
for prec in tf32 f16s; do for cfg in c2 c3 c1; do for d in 0 3; do
  CURVKIT_DEV_SYMKR=$d timeout 300 python bench.py --config $cfg --precision $prec --steps 6 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$prec $cfg dev $d', round(d['ms_per_step'],3), {a:(round(b['ms_per_step'],3), round(b['tflops'] or 0,1)) for a,b in k.items() if 'symkr' in a}, d['clocks']['sm_mhz'])
" >> gpurun_out/zr.txt
done; done; done
tail -n 2 gpurun_out/zr_tests.log; cat gpurun_out/zr.txt
