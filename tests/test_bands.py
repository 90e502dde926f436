"""Unit bands: the multi-GPU layout of H and G (bands.cuh).

Shard r of W owns the output units curvkit_shard_units(W, r) of every layer
and assembles the rows of those units whose column unit is <= the row's unit
in the unit-major order; the final gather scatters the bands' rows into place
and mirrors the upper unit-major triangle.

CPU (no GPU needed):
- the partition covers every unit of every layer once, its band rows are a
  permutation of [0, P), and the per-layer work is balanced;
- the band contract, restated in numpy on the reference's own H and G
  (tests/golden): masked bands -> scatter -> mirror rebuilds the matrix
  exactly, for 1..5 shards;
- a world_size-2 gloo run of the same assembly through torch.distributed
  gather (the exchange the library's host transport performs).

GPU:
- bands from curvkit_dev_assemble_band, assembled on one device, equal the
  single-call matrix (no entry left unwritten: NaN-filled target) and the
  reference, for 1..8 shards, H and G;
- configs 2 and 3 at full size assembled from 4 / 8 bands against the
  reference sketches;
- two processes sharing the GPU run the real multi-rank entry points over the
  host transport (gloo): the band gather, and the sharded top-k solvers.
"""
import os

import numpy as np
import pytest

from conftest import SMALL_CASES, load_golden, rel_fro
from paper_1905_05559_b200 import curv

MODELS = [([4, 8, 3], "sigmoid"), ([3, 5, 2], "tanh"), ([784, 32, 10], "sigmoid"), ([784, 64, 64, 10], "tanh"),
          ([784, 128, 64, 10], "sigmoid"), ([1024, 512, 512, 512, 10], "tanh"), ([5, 4, 6, 5, 3], "tanh")]


def _layer_cost(widths, k, u0, u1):
    w = widths
    woff = sum(w[j] * w[j + 1] + w[j + 1] for j in range(k))
    orb = (w[k] + 1) * (w[k] + 2) / 2.0
    c = lambda u: u * (u + 1) / 2.0 * orb + u * (w[k] + 1) * woff  # noqa: E731
    return c(u1) - c(u0), c(1) - c(0) + orb * (w[k + 1])  # share, an upper bound of one unit's cost


@pytest.mark.parametrize("widths,act", MODELS)
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_units_partition(widths, act, world):
    spec = curv.ModelSpec(widths, act)
    P = curv.param_count(spec)
    L = len(widths) - 1
    parts = [curv.shard_units(spec, world, r) for r in range(world)]
    total = sum(_layer_cost(widths, k, 0, widths[k + 1])[0] for k in range(L))
    # cut quantum: 1 unit in the first layer (no rectangle rows), 4 elsewhere
    slack = 2 * sum((1 if k == 0 else 4) * _layer_cost(widths, k, 0, widths[k + 1])[1] for k in range(L))
    for k in range(L):
        U = widths[k + 1]
        assert parts[0][0][k] == 0 and parts[-1][1][k] == U
        for a, b in zip(parts, parts[1:]):
            assert a[1][k] == b[0][k]
        for u0, u1, _ in parts:
            assert u0[k] <= u1[k]
            if k > 0:
                assert u0[k] % 4 == 0 or u0[k] == U  # band row ranges start 16-byte aligned (or are empty)
    for u0, u1, _ in parts:  # every shard's total work within the cut quanta of 1/W
        share = sum(_layer_cost(widths, k, u0[k], u1[k])[0] for k in range(L))
        assert share <= total / world + slack + 1e-9
    rows = np.concatenate([curv.band_rows_index(spec, world, r) for r in range(world)])
    assert sorted(rows.tolist()) == list(range(P))
    assert sum(p[2] for p in parts) == P


def _bands_from(M, spec, world):
    """The band contract on a known matrix: rows of the shard's units, entries
    with column unit <= row unit (others NaN: unspecified)."""
    g = curv.unit_ids(spec)
    out = []
    for r in range(world):
        idx = curv.band_rows_index(spec, world, r)
        B = M[idx].copy()
        B[g[None, :] > g[idx][:, None]] = np.nan
        out.append(B)
    return out


def _assemble(spec, bands, world):
    g = curv.unit_ids(spec)
    P = len(g)
    F = np.full((P, P), np.nan)
    for r, B in enumerate(bands):
        F[curv.band_rows_index(spec, world, r)] = B
    up = g[None, :] > g[:, None]
    F[up] = F.T[up]
    return F


@pytest.mark.parametrize("name", SMALL_CASES + ["config0"])
@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_band_contract_restated_on_reference(name, world):
    gd = load_golden(name)
    spec = curv.ModelSpec(gd["spec"]["widths"], gd["spec"]["activation"], gd["spec"]["output_mode"])
    for M in (gd["H"], gd["G"]):
        F = _assemble(spec, _bands_from(M, spec, world), world)
        assert not np.isnan(F).any()
        assert np.array_equal(F, M)


def _gloo_band_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gd = load_golden("config0")
    spec = curv.ModelSpec(gd["spec"]["widths"], gd["spec"]["activation"])
    mine = _bands_from(gd["G"], spec, world)[rank]
    rows = [curv.shard_units_rows(spec, world, r) for r in range(world)]
    P = gd["G"].shape[0]
    t = torch.zeros((max(rows), P), dtype=torch.float64)
    t[:rows[rank]] = torch.from_numpy(mine)
    lst = [torch.zeros_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, lst, dst=0)
    ms = torch.tensor([1.0 + rank])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)   # bench.py's timing reduction
    if rank == 0:
        F = _assemble(spec, [lst[r][:rows[r]].numpy() for r in range(world)], world)
        q.put((bool(np.array_equal(F, gd["G"])), float(ms.item())))
    dist.destroy_process_group()


def test_gloo_two_ranks_band_gather():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_band_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, ms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok and ms == 2.0


# ---- GPU -------------------------------------------------------------------

def _device_case(torch, name):
    from paper_1905_05559_b200.workloads import CONFIGS
    if name in CONFIGS:
        wl = CONFIGS[name]
        params, x, y, lab = wl.draw()
        spec = curv.ModelSpec(wl.widths, wl.activation)
        ref = None
    else:
        gd = load_golden(name)
        params, x, y = gd["params"], gd["x"], gd["y"]
        lab = np.argmax(y, axis=1)
        spec = curv.ModelSpec(gd["spec"]["widths"], gd["spec"]["activation"], gd["spec"]["output_mode"])
        ref = gd
    dev = "cuda:0"
    t = lambda a: torch.tensor(a, dtype=torch.float32, device=dev)  # noqa: E731
    return spec, t(params), t(x), torch.tensor(lab, dtype=torch.int32, device=dev), x.shape[0], ref


def _assemble_on_device(torch, spec, product, p, x, lab, n, world, ld):
    P = curv.param_count(spec)
    full = torch.full((P, ld), float("nan"), device="cuda:0")
    for r in range(world):
        rows = curv.shard_units_rows(spec, world, r)
        band = torch.full((max(rows, 1), ld), float("nan"), device="cuda:0")
        curv.dev_assemble_band(spec, product, p, x, lab, n, world, r, band, ld)
        curv.dev_band_scatter(spec, world, r, band, ld, full, ld)
        del band
    curv.dev_symmetrize_units(spec, full, ld)
    torch.cuda.synchronize()
    return full


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "tanh352", "sigmoid654", "deep4653", "config0"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_bands_assemble_to_full_matrix(name, world):
    torch = pytest.importorskip("torch")
    spec, p, x, lab, n, ref = _device_case(torch, name)
    P = curv.param_count(spec)
    ld = (P + 31) // 32 * 32
    for product, single in (("hessian", curv.dev_assemble_hessian), ("opg", curv.dev_assemble_opg)):
        full = _assemble_on_device(torch, spec, product, p, x, lab, n, world, ld)
        F = full[:, :P]
        assert not torch.isnan(F).any(), (product, world)
        assert torch.equal(F, F.T)
        one = torch.empty((P, ld), device="cuda:0")
        single(spec, p, x, lab, n, one, ld, precision="tf32")
        torch.cuda.synchronize()
        # the same kernels except where a band's bias rows are not 16-byte aligned
        # (the fused block kernel instead of the J GEMM: another TF32 rounding)
        err = rel_fro(F.double().cpu().numpy(), one[:, :P].double().cpu().numpy())
        assert err <= 3e-4, (product, world, err)
        if ref is not None:
            want = ref["H"] if product == "hessian" else ref["G"]
            if np.abs(want).max() > 0:
                assert rel_fro(F.double().cpu().numpy(), want) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("name,product,world", [("c2", "hessian", 4), ("c3", "opg", 8)])
def test_full_size_bands_match_reference_sketch(name, product, world):
    torch = pytest.importorskip("torch")
    from paper_1905_05559_b200.workloads import CONFIGS, normal
    wl = CONFIGS[name]
    spec, p, x, lab, n, _ = _device_case(torch, name)
    P = wl.P
    ld = (P + 31) // 32 * 32
    full = _assemble_on_device(torch, spec, product, p, x, lab, n, world, ld)
    pins = load_golden(f"{name}_sketch")
    om = torch.tensor(normal(0x5EED0000 + int(name[1:]), P * int(pins["k"])).reshape(P, -1), dtype=torch.float64,
                      device="cuda:0")
    got = torch.empty((P, om.shape[1]), dtype=torch.float64, device="cuda:0")
    for r0 in range(0, P, 4096):
        got[r0:r0 + 4096] = full[r0:r0 + 4096, :P].double() @ om
    want = pins["h_omega" if product == "hessian" else "g_omega"].astype(np.float64)
    err = rel_fro(got.cpu().numpy(), want)
    assert err <= 1e-3, err
    band = full[:4096, :P]
    assert torch.equal(band, full[:P, :4096].T)


def _two_rank_worker(rank, world, port, q):
    """Two processes on cuda:0: the real multi-rank entry points over the host
    transport (gloo collectives on host memory)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        from paper_1905_05559_b200.workloads import CONFIGS
        torch.cuda.set_device(0)
        wl = CONFIGS["c1"]
        params, x, y, lab = wl.draw()
        spec = curv.ModelSpec(wl.widths, wl.activation)
        dev = "cuda:0"
        p = torch.tensor(params, dtype=torch.float32, device=dev)
        xx = torch.tensor(x, dtype=torch.float32, device=dev)
        ll = torch.tensor(lab, dtype=torch.int32, device=dev)
        P, n = wl.P, wl.n
        ld = (P + 31) // 32 * 32
        comm = curv.Comm.create_host(rank, world)
        for product, single in (("hessian", curv.dev_assemble_hessian), ("opg", curv.dev_assemble_opg)):
            band = torch.empty((curv.shard_units_rows(spec, world, rank), ld), device=dev)
            curv.dev_assemble_band(spec, product, p, xx, ll, n, world, rank, band, ld)
            full = torch.full((P, ld), float("nan"), device=dev) if rank == 0 else None
            curv.dev_gather_bands(spec, band, ld, full, ld, comm)
            torch.cuda.synchronize()
            if rank == 0:
                one = torch.empty((P, ld), device=dev)
                single(spec, p, xx, ll, n, one, ld, precision="tf32")
                torch.cuda.synchronize()
                F = full[:, :P]
                out[product] = (bool(torch.isnan(F).any()), bool(torch.equal(F, F.T)),
                                rel_fro(F.double().cpu().numpy(), one[:, :P].double().cpu().numpy()))
        # sharded top-k over the same communicator: power iterations and the converged solver
        k = 12
        b, e = curv.topk_shard_rows(spec, world, rank)
        for tag in ("power", "auto"):
            qs = torch.empty((e - b, k), device=dev)
            ls = torch.empty(k, device=dev)
            if tag == "power":
                curv.dev_opg_topk_sharded(spec, p, xx, ll, n, k, 10, 2, 3, qs, ls, comm)
            else:
                curv.dev_opg_topk_sharded_auto(spec, p, xx, ll, n, k, 10, 3, qs, ls, comm)
            torch.cuda.synchronize()
            allq = [torch.zeros(0) for _ in range(world)]
            dist.all_gather_object(allq, qs.cpu())
            alll = [torch.zeros(0) for _ in range(world)]
            dist.all_gather_object(alll, ls.cpu())
            if rank == 0:
                q1 = torch.empty((P, k), device=dev)
                l1 = torch.empty(k, device=dev)
                if tag == "power":
                    curv.dev_opg_topk(spec, p, xx, ll, n, k, 10, 2, 3, q1, l1)
                else:
                    curv.dev_opg_topk_auto(spec, p, xx, ll, n, k, 10, 3, q1, l1)
                torch.cuda.synchronize()
                Q = torch.cat(allq, 0).double().numpy()
                out[tag] = (bool(torch.equal(alll[0], alll[1])),
                            float(np.max(np.abs(alll[0].double().numpy() - l1.double().cpu().numpy())
                                         / np.abs(l1.double().cpu().numpy()))),
                            float(np.abs(Q.T @ Q - np.eye(k)).max()))
        comm.close()
    except Exception as ex:  # noqa: BLE001
        out["error"] = repr(ex)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_processes_host_transport():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert "error" not in out, out
    for product in ("hessian", "opg"):
        has_nan, sym, err = out[product]
        assert not has_nan and sym and err <= 3e-4, (product, out[product])
    for tag in ("power", "auto"):
        same, lerr, orth = out[tag]
        assert same, tag                        # every rank holds the same eigenvalues
        assert lerr <= 1e-4 and orth <= 1e-4, (tag, out[tag])
