# bench code paths on one GPU: N=1 c1 alone, the reference arm, 2 ranks over the host transport
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/r02_bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_c1.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_ref.log
CURVKIT_BENCH_COMM=host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c1 --steps 3 --warmup 1 > gpurun_out/r02_bench_2rank_host.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_2rank_host.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "topk or eigs" > gpurun_out/r02_eig_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_eig_tests.log
for f in r02_bench_c1 r02_bench_ref r02_bench_2rank_host r02_eig_tests; do echo "== $f"; tail -c 1500 gpurun_out/$f.log; done
