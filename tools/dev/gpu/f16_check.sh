# symkr transform change: parity (goldens, sketches, bands) then c3/c2/c1 timings of tf32 and f16s
timeout 1200 python -m pytest tests/test_gpu_sketch_pins.py tests/test_gpu_parity.py tests/test_bands.py -m gpu -q -s -x -k "sketch or f16s or hessian_matches or opg_and or band" > gpurun_out/f16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f16_tests.log
for prec in tf32 f16s; do
  for cfg in c3 c2 c1; do
  timeout 600 python bench.py --config $cfg --precision $prec --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/f16_${cfg}_$prec.log 2>&1
  done
done
grep -h "passed\|failed\|rel-Fro\|Error" gpurun_out/f16_tests.log | tail -40
for f in gpurun_out/f16_c*.log; do echo "== $f"; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks']['reasons']); print({k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})
"; tail -1 $f | cut -c1-300; done
