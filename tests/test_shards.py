"""Row-shard partition for multi-GPU assembly (no data-path collective):
area balance and coverage on the host, a world_size-2 gloo run of the
per-rank shard selection, and (GPU) union-of-shards == full matrix."""
import os

import numpy as np
import pytest

from paper_1905_05559_b200 import curv


@pytest.mark.parametrize("P", [67, 2080, 25450, 55050, 109386])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_rows_cover_and_balance(P, world):
    bounds = [curv.shard_rows(P, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == P
    for (b0, e0), (b1, e1) in zip(bounds, bounds[1:]):
        assert e0 == b1 and b1 % 32 == 0
    if P >= 25450 and world > 1:  # lower-triangle area per shard within 5% of the mean
        area = [(e * (e + 1) - b * (b + 1)) / 2 for b, e in bounds]
        assert max(area) / (sum(area) / world) < 1.05


def _gloo_worker(rank, world, port, P, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = curv.shard_rows(P, world, rank)
    t = torch.tensor([b, e], dtype=torch.int64)
    out = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, t)
    # the bench's timing reduction: max over ranks
    ms = torch.tensor([1.0 + rank])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put(([tuple(o.tolist()) for o in out], float(ms.item())))
    dist.destroy_process_group()


def test_gloo_two_ranks_partition():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, 25450, q)) for r in range(2)]
    for p in procs:
        p.start()
    shards, ms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert shards[0][0] == 0 and shards[0][1] == shards[1][0] and shards[1][1] == 25450
    assert ms == 2.0


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["tf32", "f64"])
def test_union_of_shards_is_full_matrix(prec):
    torch = pytest.importorskip("torch")
    from paper_1905_05559_b200.workloads import CONFIGS
    wl = CONFIGS["c1"] if prec == "tf32" else CONFIGS["c0"]
    params, x, y, lab = wl.draw()
    dt = torch.float64 if prec == "f64" else torch.float32
    dev = "cuda:0"
    p = torch.tensor(params, dtype=dt, device=dev)
    xx = torch.tensor(x, dtype=dt, device=dev)
    ll = torch.tensor(lab, dtype=torch.int32, device=dev)
    spec = curv.ModelSpec(wl.widths, wl.activation)
    P = wl.P
    ld = (P + 31) // 32 * 32
    for full_fn, shard_fn in ((curv.dev_assemble_hessian, curv.dev_hessian_shard),
                              (curv.dev_assemble_opg, curv.dev_opg_shard)):
        full = torch.zeros((P, ld), dtype=dt, device=dev)
        full_fn(spec, p, xx, ll, wl.n, full, ld, precision=prec)
        parts = torch.zeros((P, ld), dtype=dt, device=dev)
        for r in range(4):
            b, e = curv.shard_rows(P, 4, r)
            shard_fn(spec, p, xx, ll, wl.n, b, e, parts, ld, precision=prec)
        torch.cuda.synchronize()
        assert torch.equal(full[:, :P], parts[:, :P])
