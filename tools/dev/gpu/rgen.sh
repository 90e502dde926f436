timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py tests/test_bands.py -m gpu -x -q 2>&1 | tail -3
for c in c2 c1; do timeout 600 python bench.py --config $c --no-extra --no-e2e --no-cpu-baseline --steps 20 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})
"; done
