set -x
timeout 900 python -m pytest tests/test_eigops.py tests/test_gpu_gemm.py -m gpu -x -q 2>&1 | tail -5
timeout 600 python tools/dev/eigops_time.py 2>&1 | grep -v "f32 full\|quadform\|nvec=16"
timeout 600 python bench.py --no-extra --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/eig2_bench.log 2>&1; tail -c 1500 gpurun_out/eig2_bench.log | head -c 1200
