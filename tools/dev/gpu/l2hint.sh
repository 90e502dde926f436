timeout 600 python -m pytest tests/test_gpu_sketch_pins.py tests/test_gpu_parity.py -m gpu -q -x -k "c1 or c3 or hessian_matches or opg_and" > gpurun_out/l2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l2_tests.log
for cfg in c3 c2 c1; do
  timeout 300 python bench.py --config $cfg --steps 12 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$cfg', round(d['ms_per_step'],3), {a:(round(b['ms_per_step'],3), round(b['tflops'] or 0,1)) for a,b in k.items() if 'symkr' in a or 'gemm' in a}, d['clocks']['sm_mhz'])
" >> gpurun_out/l2.txt
done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"symkr|pair" -c 3 --csv --log-file gpurun_out/l2_dram.csv python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline > /dev/null 2>&1
tail -n 2 gpurun_out/l2_tests.log; cat gpurun_out/l2.txt; grep -h "dram__bytes\|gpu__time" gpurun_out/l2_dram.csv | cut -d, -f13-15
