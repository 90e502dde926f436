set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5f_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5f_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s5f_smoke.log
timeout 900 python bench.py > gpurun_out/s5f_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s5f_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s5f_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/s5f_bench_ref.log
tail -n 3 gpurun_out/s5f_gputests.log; tail -n 3 gpurun_out/s5f_smoke.log; tail -c 400 gpurun_out/s5f_bench.log; tail -c 400 gpurun_out/s5f_bench_ref.log
