# A/B: orbit types 2,3 by LSU stores; f64 DMMA GEMM (cp.async); parity under both
CURVKIT_SYMKR_LSU23=1 timeout 900 python -m pytest tests/test_gpu_sketch_pins.py tests/test_gpu_parity.py tests/test_bands.py -m gpu -q -x -k "c1 or hessian_matches or opg_and or band" > gpurun_out/lsu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lsu_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py -m gpu -q -x -k "f64" > gpurun_out/f64_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f64_tests.log
for l in 0 1; do for cfg in c1 c2 c3; do
  CURVKIT_SYMKR_LSU23=$l timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('lsu23 $l $cfg', round(d['ms_per_step'],3), {a:round(b['ms_per_step'],3) for a,b in k.items() if 'symkr' in a}, d['clocks']['sm_mhz'])
" >> gpurun_out/lsu_ab.txt
done; done
timeout 300 python bench.py --config c1 --precision f64 --steps 3 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('c1 f64', round(d['ms_per_step'],3), {a:(round(b['ms_per_step'],3), b['tflops'] and round(b['tflops'],1)) for a,b in d['kernels'].items()})
" >> gpurun_out/lsu_ab.txt
tail -3 gpurun_out/lsu_tests.log gpurun_out/f64_tests.log; cat gpurun_out/lsu_ab.txt
