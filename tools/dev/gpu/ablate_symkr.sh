# symkr ablations at c2 (timings only; dev modes produce wrong values)
for prec in tf32 f16s; do for dev in 0 1 2 3 32; do
  CURVKIT_DEV_SYMKR=$dev timeout 300 python bench.py --config c2 --precision $prec --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/abl.log 2>&1
  python -c "
import json
for l in open('gpurun_out/abl.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$prec dev $dev', round(d['kernels']['hess_symkr']['ms_per_step'],3), d['clocks']['sm_mhz'])
" >> gpurun_out/ablate.txt
done; done
cat gpurun_out/ablate.txt
