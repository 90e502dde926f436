for d in 0 4096 2; do echo "DEV_SYMKR=$d"; CURVKIT_DEV_SYMKR=$d timeout 600 python bench.py --config c1 --no-extra --no-e2e --no-cpu-baseline --steps 20 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if 'symkr' in k})
"; done
