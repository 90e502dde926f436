set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5b_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5b_gputests.log
tail -n 4 gpurun_out/s5b_gputests.log
timeout 900 python bench.py > gpurun_out/s5b_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s5b_bench.log
tail -c 1800 gpurun_out/s5b_bench.log
