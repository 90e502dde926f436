set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench1.log 2>&1; echo "bench rc=$?" >> gpurun_out/r02_bench1.log
tail -3 gpurun_out/r02_gputests.log; tail -c 3000 gpurun_out/r02_bench1.log
