set -x
timeout 900 python -m pytest tests/test_eigops.py -m gpu -x -q > gpurun_out/eigops_tests.log 2>&1; echo "rc=$?" >> gpurun_out/eigops_tests.log
tail -30 gpurun_out/eigops_tests.log
timeout 600 python tools/dev/eigops_time.py > gpurun_out/eigops_time.log 2>&1; echo "rc=$?" >> gpurun_out/eigops_time.log
cat gpurun_out/eigops_time.log
