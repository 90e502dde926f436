timeout 1500 python -m pytest tests/test_gpu_kr_f16.py tests/test_gpu_parity.py -m gpu -q -s -x -k "topk or f16s_products or shard_rows" > gpurun_out/krf16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/krf16_tests.log
python tools/c4_profile.py f16s > gpurun_out/c4prof_f16s.txt 2>&1
grep -h "passed\|failed\|Error\|c4 max" gpurun_out/krf16_tests.log | tail -5; head -5 gpurun_out/c4prof_f16s.txt; grep -A4 "auto" gpurun_out/c4prof_f16s.txt
