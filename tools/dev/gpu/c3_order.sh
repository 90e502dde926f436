# c3 tile-order knobs: symkr square size and rectangle GEMM rasterisation group
for sb in 5 10 25; do for gm in 16 8 4; do
  CURVKIT_SYMKR_SB=$sb CURVKIT_GROUP_M=$gm timeout 300 python bench.py --config c3 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ord.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ord.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('sb $sb gm $gm', round(d['ms_per_step'],2), round(k['opg_symkr']['ms_per_step'],2), round(k['opg_gemm']['ms_per_step'],2), d['clocks']['sm_mhz'])
" >> gpurun_out/c3_order.txt
done; done
cat gpurun_out/c3_order.txt
