timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py tests/test_gpu_gemm.py tests/test_incremental.py -m gpu -q -x -k "f64 or incremental or streaming or single_block or contract or device_blocks" > gpurun_out/f64e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f64e_tests.log
timeout 300 python bench.py --config c1 --precision f64 --steps 3 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('c1 f64', round(d['ms_per_step'],3), {a:(round(b['ms_per_step'],3), round(b['tflops'] or 0,1)) for a,b in d['kernels'].items()})
" > gpurun_out/f64e.txt
tail -n 2 gpurun_out/f64e_tests.log; cat gpurun_out/f64e.txt
