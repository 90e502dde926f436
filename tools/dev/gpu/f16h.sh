timeout 900 python -m pytest tests/test_gpu_sketch_pins.py tests/test_gpu_parity.py -m gpu -q -s -x -k "f16s" > gpurun_out/f16h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f16h_tests.log
for prec in tf32 f16s; do for cfg in c2 c1; do
  timeout 300 python bench.py --config $cfg --precision $prec --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$prec $cfg', round(d['ms_per_step'],3), {a:(round(b['ms_per_step'],3), round(b['tflops'] or 0,1)) for a,b in k.items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/f16h.txt
done; done
grep -h "rel-Fro\|passed\|failed\|Error" gpurun_out/f16h_tests.log | tail -12; cat gpurun_out/f16h.txt
for prec in tf32 f16s; do
  timeout 300 python bench.py --config c3 --precision $prec --steps 12 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$prec c3', round(d['ms_per_step'],3), {a:(round(b['ms_per_step'],3), round(b['tflops'] or 0,1)) for a,b in k.items()}, d['clocks']['sm_mhz'])
" >> gpurun_out/f16h.txt
done
cat gpurun_out/f16h.txt
