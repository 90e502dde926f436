for prec in tf32 f16s; do for sb in 5 0 2; do for d in 0 3; do
  CURVKIT_SYMKR_SB=$sb CURVKIT_DEV_SYMKR=$d timeout 300 python bench.py --config c2 --precision $prec --steps 6 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$prec c2 sb $sb dev $d', {a:(round(b['ms_per_step'],3), round(b['tflops'] or 0,1)) for a,b in k.items() if 'symkr' in a}, d['clocks']['sm_mhz'])
" >> gpurun_out/sb.txt
done; done; done
cat gpurun_out/sb.txt
