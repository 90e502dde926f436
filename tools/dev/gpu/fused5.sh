for d in 3 11; do
  CURVKIT_DEV_FUSED=$d timeout 300 python bench.py --config c2 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('c2 dev $d', round(k['hess_fused']['ms_per_step'],3), round(k['hess_fused']['tflops'],1), d['clocks']['sm_mhz'])
" >> gpurun_out/f5.txt
done
cat gpurun_out/f5.txt
