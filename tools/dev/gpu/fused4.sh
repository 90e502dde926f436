timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py tests/test_bands.py -m gpu -q -x -k "hessian or band" > gpurun_out/f4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f4_tests.log
for cfg in c2 c1; do for d in 0 3; do
  CURVKIT_DEV_FUSED=$d timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$cfg dev $d', round(d['ms_per_step'],3), round(k['hess_fused']['ms_per_step'],3), round(k['hess_fused']['tflops'],1), d['clocks']['sm_mhz'])
" >> gpurun_out/f4.txt
done; done
mkdir -p gpurun_out/tr4; CURVKIT_TRACE=1 timeout 300 python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/tr.log 2>&1; mv gpurun_out/trace_*.bin gpurun_out/tr4/
python tools/dev/trace_fused.py gpurun_out/tr4/trace_0.bin >> gpurun_out/f4.txt
tail -n 2 gpurun_out/f4_tests.log; cat gpurun_out/f4.txt
