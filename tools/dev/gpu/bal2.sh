timeout 900 python -m pytest tests/test_bands.py tests/test_gpu_gemm.py -m gpu -q -x > gpurun_out/bal_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bal_tests.log
python tools/band_profile.py 8 > gpurun_out/bandprof.txt 2>&1
bash tools/dev/gpu/bal.sh > /dev/null 2>&1
tail -n 2 gpurun_out/bal_tests.log; cat gpurun_out/bandprof.txt; python -c "
import json; d=json.load(open('gpurun_out/bal.txt')); print(d['one_gpu_ms'], {k:(round(v['max_band_ms'],2), round(v['projected_speedup'],2)) for k,v in d.items() if k.startswith('W')})"
