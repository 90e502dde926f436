timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02g_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02g_gputests.log
timeout 900 python bench.py > gpurun_out/r02g_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r02g_bench.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02g_smoke.log
tail -n 3 gpurun_out/r02g_gputests.log; tail -n 3 gpurun_out/r02g_smoke.log; tail -c 300 gpurun_out/r02g_bench.log
