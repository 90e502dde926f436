# bench code paths: 2 ranks over the host transport on one GPU (c1, c3), then the default N = 1 run with its extras
CURVKIT_BENCH_COMM=host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c1 --steps 3 --warmup 1 > gpurun_out/n2_c1.log 2>&1; echo "rc=$?" >> gpurun_out/n2_c1.log
CURVKIT_BENCH_COMM=host timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config c3 --steps 3 --warmup 1 --no-e2e > gpurun_out/n2_c3.log 2>&1; echo "rc=$?" >> gpurun_out/n2_c3.log
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/n1_default.log 2>&1; echo "rc=$? wall $(( $(date +%s) - t0 )) s" >> gpurun_out/n1_default.log
tail -c 800 gpurun_out/n2_c1.log; tail -c 800 gpurun_out/n2_c3.log; tail -c 400 gpurun_out/n1_default.log
