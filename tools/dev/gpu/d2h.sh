for one in 1 0; do
  if [ $one = 1 ]; then export CURVKIT_D2H_ONE=1; else unset CURVKIT_D2H_ONE; fi
  timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-extra --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('one_engine $one', round(d['ms_per_step'],2), d['e2e'])
" >> gpurun_out/d2h.txt
done
cat gpurun_out/d2h.txt
