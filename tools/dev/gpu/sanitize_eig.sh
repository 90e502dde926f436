set -x
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_eigops.py -m gpu -x -q -k "not config4_size" > gpurun_out/eig_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/eig_memcheck.log
tail -8 gpurun_out/eig_memcheck.log
CURVKIT_POISON=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5_poison.log 2>&1; echo "poison rc=$?" >> gpurun_out/s5_poison.log
tail -4 gpurun_out/s5_poison.log
