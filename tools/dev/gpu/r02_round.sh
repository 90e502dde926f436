# round-2 GPU pass: suite, default bench (c3 headline + extras), reference arm, launch list of the headline
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r02_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputests.log
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r02_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/r02_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r02_ncu.log
tail -15 gpurun_out/r02_gputests.log; tail -c 4000 gpurun_out/r02_bench.log; tail -c 1500 gpurun_out/r02_bench_ref.log; tail -3 gpurun_out/r02_ncu.log
