"""Parameter-row-sharded top-k (multi-GPU, NCCL all-reduce of J X and of the
CholeskyQR Grams).

CPU:
- the shard partition covers P contiguously, cuts only at output-unit weight
  blocks or 4-aligned bias blocks, and balances parameter counts;
- a world_size-2 gloo run of the sharded range finder, with the oracle
  Jacobian as J, reproduces the single-process eigenvalues.  This checks the
  exchange pattern (what is summed, and where) that the CUDA path uses.

GPU:
- the matrix-free operators J[:, range] X and J[:, range]^T T (the sharded
  Khatri-Rao kernels) agree with the dense fp64 products, and the shard sum
  is the full product;
- the sharded entry point over a 1-rank communicator equals the unsharded
  solver."""
import os

import numpy as np
import pytest

from conftest import rel_fro
from paper_1905_05559_b200 import curv

MODELS = [([4, 8, 3], "sigmoid"), ([784, 32, 10], "sigmoid"), ([7, 5, 6, 3], "tanh"),
          ([1024, 512, 512, 512, 10], "tanh")]


def _cuts(widths):
    """Legal shard boundaries: weight blocks of each output unit, 4-aligned biases."""
    cuts, at = {0}, 0
    for k in range(len(widths) - 1):
        tk, to = widths[k], widths[k + 1]
        cuts.update(at + o * tk for o in range(to))
        boff = at + to * tk
        cuts.update(boff + b for b in range(0, to, 4))
        cuts.add(boff + to)
        at = boff + to
    return cuts, at


@pytest.mark.parametrize("widths,act", MODELS)
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_topk_shard_partition(widths, act, world):
    spec = curv.ModelSpec(widths, act)
    cuts, P = _cuts(widths)
    assert P == curv.param_count(spec)
    bounds = [curv.topk_shard_rows(spec, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == P
    for (b0, e0), (b1, e1) in zip(bounds, bounds[1:]):
        assert e0 == b1
    for b, e in bounds:
        assert b in cuts and e in cuts and b <= e
    if P >= 100000:  # balanced to within one unit block of the mean
        sizes = [e - b for b, e in bounds]
        assert max(sizes) - P / world <= max(widths) + 4


def _sharded_range_finder(J, rows, k, l, iters, seed, allreduce):
    """The CUDA solver's exchange pattern, on a row block of J (numpy)."""
    n, P = J.shape
    b, e = rows
    om = np.random.default_rng(seed).standard_normal((P, l))[b:e]
    Jr = J[:, b:e]
    x = om
    for _ in range(iters + 1):
        t = allreduce(Jr @ x)          # J X: partials over row blocks
        y = Jr.T @ t                   # local rows of J^T J X
        for _ in range(2):             # CholeskyQR2: Gram all-reduced, rows local
            w = allreduce(y.T @ y)
            r = np.linalg.cholesky(w).T
            y = np.linalg.solve(r.T, y.T).T
        x = y
    t = allreduce(Jr @ x)
    lam = np.linalg.eigvalsh(t.T @ t / n)[::-1][:k]
    return lam


def _cholqr2(y, allreduce):
    for _ in range(2):                 # CholeskyQR2: Gram all-reduced, rows local
        w = allreduce(y.T @ y)
        r = np.linalg.cholesky(w).T
        y = np.linalg.solve(r.T, y.T).T
    return y


def _sharded_filtered(J, rows, k, l, steps, degree, seed, allreduce):
    """The Chebyshev-filtered solver's exchange pattern (eigen.cuh topk_core,
    cheb_degree > 0): sketch, then rounds of Ritz values (all-reduced J X),
    a row-local three-term recurrence on [0, theta_l], CholeskyQR2."""
    n, P = J.shape
    b, e = rows
    Jr = J[:, b:e]
    x = _cholqr2(Jr.T @ allreduce(Jr @ np.random.default_rng(seed).standard_normal((P, l))[b:e]), allreduce)
    used = 0
    while used < steps * degree:
        t = allreduce(Jr @ x)
        th = np.linalg.eigvalsh(t.T @ t / n)
        lo, top = th.min(), th.max()
        deg = degree
        if 2 * top / lo - 1 > 1:
            deg = int(np.clip(np.floor(9.9 / np.arccosh(2 * top / lo - 1)), 1, degree))
        deg = min(deg, steps * degree - used)
        used += deg
        c = e_ = lo / 2
        a, bb = None, x
        for d in range(1, deg + 1):
            cc = Jr.T @ allreduce(Jr @ bb)          # N G B, local rows
            f = 1.0 if d == 1 else 2.0
            nxt = f / (e_ * n) * cc - f * c / e_ * bb - (a if d > 1 else 0.0)
            a, bb = bb, nxt
        x = _cholqr2(bb, allreduce)
    t = allreduce(Jr @ x)
    return np.linalg.eigvalsh(t.T @ t / n)[::-1][:k]


def _gloo_topk_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle
    from paper_1905_05559_b200.workloads import glorot_params, splitmix64, uniform
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    widths = [7, 5, 6, 3]
    spec = curv.ModelSpec(widths, "tanh")
    n = 40
    params = glorot_params(widths, 3, 0.1)
    x = uniform(4, n * widths[0]).reshape(n, widths[0])
    lab = (splitmix64(5, n) % np.uint64(widths[-1])).astype(int)
    y = np.zeros((n, widths[-1]))
    y[np.arange(n), lab] = 1.0
    J = Oracle().jacobian({"widths": widths, "activation": "tanh"}, params, x, y)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    rows = curv.topk_shard_rows(spec, world, rank)
    lam = _sharded_range_finder(J, rows, 4, 10, 2, 11, allreduce)
    full = _sharded_range_finder(J, (0, J.shape[1]), 4, 10, 2, 11, lambda a: a)
    flam = _sharded_filtered(J, rows, 4, 10, 2, 3, 11, allreduce)
    ffull = _sharded_filtered(J, (0, J.shape[1]), 4, 10, 2, 3, 11, lambda a: a)
    if rank == 0:
        exact = np.linalg.eigvalsh(J.T @ J / n)[::-1][:4]
        q.put((lam.tolist(), full.tolist(), rows, flam.tolist(), ffull.tolist(), exact.tolist()))
    dist.destroy_process_group()


def test_gloo_two_ranks_sharded_range_finder():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_topk_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    lam, full, rows, flam, ffull, exact = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert 0 < rows[1]
    np.testing.assert_allclose(lam, full, rtol=1e-10)
    np.testing.assert_allclose(flam, ffull, rtol=1e-10)     # filtered: sharded == unsharded
    np.testing.assert_allclose(ffull, exact, rtol=1e-6)     # and converged (6 applications)


# ---- GPU -------------------------------------------------------------------

def _c1(torch):
    from paper_1905_05559_b200.workloads import CONFIGS
    wl = CONFIGS["c1"]
    params, x, y, lab = wl.draw()
    dev = "cuda:0"
    spec = curv.ModelSpec(wl.widths, wl.activation)
    return wl, spec, [torch.tensor(a, dtype=torch.float64, device=dev) for a in (params, x)], \
        torch.tensor(lab, dtype=torch.int32, device=dev)


@pytest.mark.gpu
def test_jacobian_apply_shards_match_dense():
    torch = pytest.importorskip("torch")
    wl, spec, (p64, x64), lab = _c1(torch)
    P, n, l = wl.P, wl.n, 40
    J = torch.empty((n, P), dtype=torch.float64, device="cuda:0")
    curv.dev_assemble_jacobian(spec, p64, x64, lab, n, J, P, precision="f64")
    p32, x32 = p64.float(), x64.float()
    g = torch.Generator(device="cuda:0").manual_seed(5)
    X = torch.zeros((P, 64), device="cuda:0")
    X[:, :l] = torch.randn((P, l), device="cuda:0", generator=g)
    T = torch.zeros((n, 64), device="cuda:0")
    curv.dev_jacobian_apply(spec, p32, x32, lab, n, 0, P, X, 64, l, T, 64)
    Tref = J @ X[:, :l].double()
    assert rel_fro(T[:, :l].double().cpu().numpy(), Tref.cpu().numpy()) <= 1e-3
    # shards of the top-k partition sum to the full product
    acc = torch.zeros((n, l), dtype=torch.float64, device="cuda:0")
    for r in range(3):
        b, e = curv.topk_shard_rows(spec, 3, r)
        Tr = torch.zeros((n, 64), device="cuda:0")
        curv.dev_jacobian_apply(spec, p32, x32, lab, n, b, e, X[b:e].contiguous(), 64, l, Tr, 64)
        acc += Tr[:, :l].double()
    assert rel_fro(acc.cpu().numpy(), T[:, :l].double().cpu().numpy()) <= 1e-6
    # transpose: full rows and shard rows
    U = torch.zeros((n, 64), device="cuda:0")
    U[:, :l] = torch.randn((n, l), device="cuda:0", generator=g)
    Y = torch.zeros((P, 64), device="cuda:0")
    curv.dev_jacobian_apply(spec, p32, x32, lab, n, 0, P, U, 64, l, Y, 64, transpose=True)
    Yref = J.T @ U[:, :l].double()
    assert rel_fro(Y[:, :l].double().cpu().numpy(), Yref.cpu().numpy()) <= 1e-3
    for r in range(3):
        b, e = curv.topk_shard_rows(spec, 3, r)
        Yr = torch.zeros((e - b, 64), device="cuda:0")
        curv.dev_jacobian_apply(spec, p32, x32, lab, n, b, e, U, 64, l, Yr, 64, transpose=True)
        assert rel_fro(Yr[:, :l].double().cpu().numpy(), Y[b:e, :l].double().cpu().numpy()) <= 1e-6


@pytest.mark.gpu
def test_sharded_entry_one_rank_equals_unsharded():
    torch = pytest.importorskip("torch")
    wl, spec, (p64, x64), lab = _c1(torch)
    p32, x32 = p64.float(), x64.float()
    k = 12
    q0 = torch.empty((wl.P, k), device="cuda:0")
    l0 = torch.empty(k, device="cuda:0")
    curv.dev_opg_topk(spec, p32, x32, lab, wl.n, k, 10, 2, 3, q0, l0)
    comm = curv.Comm.create(0, 1, lambda b: b)
    try:
        q1 = torch.empty((wl.P, k), device="cuda:0")
        l1 = torch.empty(k, device="cuda:0")
        curv.dev_opg_topk_sharded(spec, p32, x32, lab, wl.n, k, 10, 2, 3, q1, l1, comm)
    finally:
        comm.close()
    torch.cuda.synchronize()
    assert torch.equal(l0, l1) and torch.equal(q0, q1)


@pytest.mark.gpu
def test_sharded_filtered_one_rank_equals_unsharded():
    torch = pytest.importorskip("torch")
    wl, spec, (p64, x64), lab = _c1(torch)
    p32, x32 = p64.float(), x64.float()
    k = 12
    q0 = torch.empty((wl.P, k), device="cuda:0")
    l0 = torch.empty(k, device="cuda:0")
    curv.dev_opg_topk_filtered(spec, p32, x32, lab, wl.n, k, 10, 2, 3, 3, q0, l0)
    comm = curv.Comm.create(0, 1, lambda b: b)
    try:
        q1 = torch.empty((wl.P, k), device="cuda:0")
        l1 = torch.empty(k, device="cuda:0")
        curv.dev_opg_topk_sharded_filtered(spec, p32, x32, lab, wl.n, k, 10, 2, 3, 3, q1, l1, comm)
    finally:
        comm.close()
    torch.cuda.synchronize()
    assert torch.equal(l0, l1) and torch.equal(q0, q1)


@pytest.mark.gpu
def test_nccl_loopback_one_rank(monkeypatch):
    """The NCCL calls themselves on a one-GPU box: under CURVKIT_COMM_LOOPBACK=1 a
    one-rank NCCL communicator issues its all-reduces (sharded top-k) and the
    send/recv pair of the final band gather instead of short-cutting them; the
    results equal the communication-free ones bitwise (a one-rank sum and a
    self send are copies)."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("CURVKIT_COMM_LOOPBACK", "1")
    wl, spec, (p64, x64), lab = _c1(torch)
    p32, x32 = p64.float(), x64.float()
    k = 12
    q0 = torch.empty((wl.P, k), device="cuda:0")
    l0 = torch.empty(k, device="cuda:0")
    curv.dev_opg_topk_filtered(spec, p32, x32, lab, wl.n, k, 10, 2, 3, 3, q0, l0)
    P = wl.P
    ld = (P + 31) // 32 * 32
    comm = curv.Comm.create(0, 1, lambda b: b)
    try:
        n0 = curv.launch_count()
        q1 = torch.empty((wl.P, k), device="cuda:0")
        l1 = torch.empty(k, device="cuda:0")
        curv.dev_opg_topk_sharded_filtered(spec, p32, x32, lab, wl.n, k, 10, 2, 3, 3, q1, l1, comm)
        band = torch.full((curv.shard_units_rows(spec, 1, 0), ld), float("nan"), device="cuda:0")
        curv.dev_assemble_band(spec, "opg", p32, x32, lab, wl.n, 1, 0, band, ld)
        full = torch.full((P, ld), float("nan"), device="cuda:0")
        curv.dev_gather_bands(spec, band, ld, full, ld, comm)
        assert curv.launch_count() > n0
    finally:
        comm.close()
    torch.cuda.synchronize()
    assert torch.equal(l0, l1) and torch.equal(q0, q1)
    local = torch.full((P, ld), float("nan"), device="cuda:0")
    curv.dev_band_scatter(spec, 1, 0, band, ld, local, ld)
    curv.dev_symmetrize_units(spec, local, ld)
    torch.cuda.synchronize()
    assert not torch.isnan(full[:, :P]).any() and torch.equal(full[:, :P], local[:, :P])
