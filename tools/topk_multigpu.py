"""Multi-GPU top-k eigenpairs of G (config 4 by default), parameter rows
sharded over ranks; the library all-reduces J X and the Grams over NCCL.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port 29533 tools/topk_multigpu.py [cfg] [reps]

Rank 0 prints one JSON line: time per solve (max over ranks, CUDA events),
the eigenvalues' head and the orthonormality of the gathered eigenvectors."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1905_05559_b200 import curv  # noqa: E402
from paper_1905_05559_b200.workloads import CONFIGS  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def bcast(b):
        obj = [b]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    comm = curv.Comm.create(rank, world, bcast)
    wl = CONFIGS[cfg]
    params, x, y, lab = wl.draw()
    dev = torch.device("cuda", local)
    p = torch.tensor(params, dtype=torch.float32, device=dev)
    xx = torch.tensor(x, dtype=torch.float32, device=dev)
    ll = torch.tensor(lab, dtype=torch.int32, device=dev)
    spec = curv.ModelSpec(wl.widths, wl.activation)
    k = getattr(wl, "eig_k", 100)
    os_ = getattr(wl, "oversample", 20)
    pi = getattr(wl, "power_iters", 2)
    b, e = curv.topk_shard_rows(spec, world, rank)
    q = torch.empty((max(e - b, 1), k), device=dev)
    lam = torch.empty(k, device=dev)
    times = []
    for it in range(reps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        curv.dev_opg_topk_sharded(spec, p, xx, ll, wl.n, k, os_, pi, 7, q, lam, comm)
        s1.record()
        torch.cuda.synchronize()
        t = torch.tensor([s0.elapsed_time(s1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if it > 0:
            times.append(float(t.item()))
    # gather the eigenvector rows and check orthonormality on rank 0
    qs = [None] * world
    dist.all_gather_object(qs, q[: e - b].cpu())
    if rank == 0:
        Q = torch.cat(qs).double()
        err = (Q.T @ Q - torch.eye(k, dtype=torch.float64)).abs().max().item()
        print(json.dumps({"config": cfg, "n_gpus": world, "P": wl.P, "k": k, "ms_per_solve": min(times),
                          "ms_all": times, "lambda_head": lam[:5].tolist(), "orthonormality_err": err}))
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
