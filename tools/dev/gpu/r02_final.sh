# round-2 validation: suite, default bench (c3 headline + extras), reference arm, launch list, full capture of the headline kernel
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02f_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02f_gputests.log
timeout 900 python bench.py > gpurun_out/r02f_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r02f_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/r02f_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r02f_ncu.log
timeout 2400 ncu --set full --replay-mode application --import-source on --clock-control none -k regex:symkr -c 1 -o gpurun_out/r02f_c3_symkr_full python bench.py --config c3 --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/r02f_ncu_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/r02f_ncu_full.log
tail -3 gpurun_out/r02f_gputests.log; tail -c 600 gpurun_out/r02f_bench.log; tail -2 gpurun_out/r02f_bench_ref.log gpurun_out/r02f_ncu.log gpurun_out/r02f_ncu_full.log
