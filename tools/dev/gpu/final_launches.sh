timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/fl_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/fl_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/r02_final_launches.csv | head -30
