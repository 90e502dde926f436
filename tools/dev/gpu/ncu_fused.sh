timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_hess_fused -c 1 -o gpurun_out/c2_fused \
  python bench.py --config c2 --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ncu_c2_fused.log 2>&1
echo "rc=$?"
for d in 0 1 2 3; do
  CURVKIT_DEV_FUSED=$d timeout 300 python bench.py --config c2 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('fused dev $d', round(k['hess_fused']['ms_per_step'],3), d['clocks']['sm_mhz'])
" >> gpurun_out/fused_ab.txt
done
cat gpurun_out/fused_ab.txt
