"""The consumers of eigenpairs (curv::validate_eigen_pairs, low_rank_* and
full_rank_*, eigensolve.cpp:11-30 and 278-358) against vectors the reference
itself produced (tests/golden/eigops.npz, tests/golden/make_eigops_golden.py).

CPU: the numpy restatement in oracle/ against the golden vectors, and the
contract / shape errors of the C-ABI (raised before any device work, with the
reference's text).  GPU: every operator through the C-ABI in f64 / f32 / tf32 /
f16s, batched vectors, the device entry points at config-1 and config-4 size.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_fro
from oracle import oracle as orc
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.errors import ContractError, ShapeError

CASES = ["c0_opg", "ortho300", "k1", "full_k", "thin2000"]
ROWS = (0, 7, 1023, 1999)  # make_eigops_golden.py keeps these matrix rows when P > 400
# relative Frobenius tolerance per precision mode (north_star: 1e-5 fp64, 1e-3 fp32 / TF32)
TOL = {"f64": 1e-12, "f32": 1e-5, "tf32x3": 1e-5, "tf32": 1e-3, "f16s": 1e-3}


def case(name):
    d = np.load(os.path.join(GOLDEN, "eigops.npz"))
    return {k.split("/", 1)[1]: d[k] for k in d.files if k.startswith(name + "/")}


def rows_of(m, p):
    return m[list(ROWS)] if p > 400 else m


# ---- CPU: the oracle restatement against the reference's vectors ----------------

@pytest.mark.parametrize("name", CASES)
def test_port_matches_reference_vectors(name):
    c = case(name)
    q, lam, lt = c["q"], c["lam"], float(c["lt"])
    p = q.shape[0]
    assert rel_fro(rows_of(orc.eig_materialize_port(q, lam), p), c["low"]) <= 1e-13
    assert rel_fro(rows_of(orc.eig_materialize_port(q, lam, lt), p), c["full"]) <= 1e-13
    for i, x in enumerate(c["x"]):
        y, qf = orc.eig_apply_port(q, lam, x)
        assert rel_fro(y, c["low_y"][i]) <= 1e-12 and abs(qf - c["low_quad"][i]) <= 1e-12 * max(1, abs(qf))
        y, qf = orc.eig_apply_port(q, lam, x, lt)
        assert rel_fro(y, c["full_y"][i]) <= 1e-12 and abs(qf - c["full_quad"][i]) <= 1e-12 * max(1, abs(qf))


def test_golden_default_lambda_tilde_is_smallest_eigenvalue():
    for name in ("c0_opg", "thin2000"):  # generated with curv::default_lambda_tilde
        c = case(name)
        assert float(c["lt"]) == c["lam"][-1] == curv.default_lambda_tilde(curv.EigenPairs(c["q"], c["lam"]))
    with pytest.raises(ContractError, match="not positive"):
        curv.default_lambda_tilde(curv.EigenPairs(np.eye(3)[:, :2], np.array([1.0, -0.5])))
    with pytest.raises(ContractError, match="no eigenvalues"):
        curv.default_lambda_tilde(curv.EigenPairs(np.zeros((3, 0)), np.zeros(0)))


def test_contract_errors_before_device_work():
    """The refusals of eigensolve.cpp:11-30 and 255-275, with the reference's text;
    none of them needs a GPU (they are raised before any device call)."""
    c = case("k1")
    pairs = curv.EigenPairs(c["q"], c["lam"])
    p = c["q"].shape[0]
    with pytest.raises(ContractError, match=r"low_rank_materialize: P = 50 exceeds the dense memory cap 8; use the "
                                            r"implicit quadform/apply forms instead"):
        curv.low_rank_materialize(pairs, memory_cap=8)
    with pytest.raises(ContractError, match="full_rank_materialize: P = 50 exceeds the dense memory cap 49"):
        curv.full_rank_materialize(pairs, 0.5, memory_cap=49)
    for bad in (0.0, -1.0, float("nan")):
        with pytest.raises(ContractError, match="full-rank approximation requires lambda_tilde > 0, got"):
            curv.full_rank_materialize(pairs, bad)  # checked before the memory cap, as in the reference
        with pytest.raises(ContractError, match="full-rank approximation requires lambda_tilde > 0"):
            curv.full_rank_quadform(pairs, bad, np.zeros(p))
        with pytest.raises(ContractError, match="full-rank approximation requires lambda_tilde > 0"):
            curv.full_rank_apply(pairs, bad, np.zeros(p))
    with pytest.raises(ShapeError, match="eigen operator: vector length 49 does not match P = 50"):
        curv.low_rank_apply(pairs, np.zeros(p - 1))
    with pytest.raises(ShapeError, match="eigen operator: vector length 51 does not match P = 50"):
        curv.full_rank_quadform(pairs, 0.5, np.zeros(p + 1))
    with pytest.raises(ShapeError, match="lambda length does not match column count"):
        curv.validate_eigen_pairs(curv.EigenPairs(c["q"], np.array([2.0, 1.0])))
    with pytest.raises(ShapeError, match="more columns than rows"):
        curv.validate_eigen_pairs(curv.EigenPairs(np.zeros((2, 3)), np.array([3.0, 2.0, 1.0])))
    q2 = case("c0_opg")["q"]
    with pytest.raises(ContractError, match="eigenvalues not sorted descending"):
        curv.validate_eigen_pairs(curv.EigenPairs(q2, np.array([1.0, 3.0, 2.0, 1.0, 0.5, 0.1])))
    with pytest.raises(ContractError, match="unknown precision"):
        curv.low_rank_apply(pairs, np.zeros(p), precision="bf16")


@pytest.mark.skipif(not orc.Ref.available(), reason="oracle/_ref not built")
def test_reference_raises_the_same_refusals():
    ref = orc.Ref()
    c = case("k1")
    with pytest.raises(orc.OracleError, match="exceeds the dense memory cap 8; use the implicit"):
        ref.eig_ops(c["q"], c["lam"], materialize=True, memory_cap=8)
    with pytest.raises(orc.OracleError, match="requires lambda_tilde > 0"):
        ref.eig_ops(c["q"], c["lam"], lambda_tilde=0.0, materialize=True, memory_cap=8)
    with pytest.raises(orc.OracleError, match="vector length 49 does not match P = 50"):
        ref.eig_ops(c["q"], c["lam"], x=np.zeros(49))


# ---- GPU: the operators through the C-ABI ---------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32", "tf32", "tf32x3", "f16s"])
@pytest.mark.parametrize("name", CASES)
def test_materialize_matches_reference(name, prec):
    c = case(name)
    pairs = curv.EigenPairs(c["q"], c["lam"])
    p = c["q"].shape[0]
    low = curv.low_rank_materialize(pairs, precision=prec)
    full = curv.full_rank_materialize(pairs, float(c["lt"]), precision=prec)
    assert low.shape == full.shape == (p, p)
    assert np.array_equal(low, low.T) and np.array_equal(full, full.T)  # mirrored lower tiles: exactly symmetric
    assert rel_fro(rows_of(low, p), c["low"]) <= TOL[prec]
    assert rel_fro(rows_of(full, p), c["full"]) <= TOL[prec]


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32", "tf32"])
@pytest.mark.parametrize("name", CASES)
def test_apply_and_quadform_match_reference(name, prec):
    c = case(name)
    pairs = curv.EigenPairs(c["q"], c["lam"])
    lt = float(c["lt"])
    tol = 1e-12 if prec == "f64" else 2e-5  # the implicit forms run exact FMAs in every fp32 mode
    for i, x in enumerate(c["x"]):
        assert rel_fro(curv.low_rank_apply(pairs, x, precision=prec), c["low_y"][i]) <= tol
        assert rel_fro(curv.full_rank_apply(pairs, lt, x, precision=prec), c["full_y"][i]) <= tol
        scale = max(1.0, float(np.sum(c["lam"][0] * x * x)))
        assert abs(curv.low_rank_quadform(pairs, x, precision=prec) - c["low_quad"][i]) <= tol * scale
        assert abs(curv.full_rank_quadform(pairs, lt, x, precision=prec) - c["full_quad"][i]) <= tol * scale


@pytest.mark.gpu
def test_batched_vectors_equal_single_calls():
    c = case("ortho300")
    pairs = curv.EigenPairs(c["q"], c["lam"])
    lt = float(c["lt"])
    xs = np.concatenate([c["x"], c["x"][::-1] * 0.5, c["x"][:1] - c["x"][1:2]])  # 7 vectors: two passes of four
    for ltv in (None, lt):
        y, quad = curv.eig_apply(pairs, xs, ltv)
        for i, x in enumerate(xs):
            y1, q1 = curv.eig_apply(pairs, x, ltv)
            assert np.array_equal(y[i], y1) and quad[i] == q1  # fixed-order reductions: bitwise
    ref_y = np.array([orc.eig_apply_port(c["q"], c["lam"], x, lt)[0] for x in xs])
    assert rel_fro(y, ref_y) <= 1e-12


@pytest.mark.gpu
def test_validate_eigen_pairs_on_device():
    for name in CASES:
        c = case(name)
        curv.validate_eigen_pairs(curv.EigenPairs(c["q"], c["lam"]))
    c = case("ortho300")
    q = c["q"].copy()
    q[:, 5] += 1e-6 * q[:, 6]  # |q5.q6| = 1e-6 > 1e-8
    with pytest.raises(ContractError, match="columns are not orthonormal"):
        curv.validate_eigen_pairs(curv.EigenPairs(q, c["lam"]))
    curv.validate_eigen_pairs(curv.EigenPairs(q, c["lam"]), ortho_tol=1e-5)
    q = c["q"].copy()
    q[:, 36] *= 1.0 + 1e-6  # the last column's norm
    with pytest.raises(ContractError, match="columns are not orthonormal"):
        curv.validate_eigen_pairs(curv.EigenPairs(q, c["lam"]))


@pytest.mark.gpu
def test_empty_basis():
    """k = 0: the low-rank operator is zero, the full-rank one lambda_tilde I."""
    pairs = curv.EigenPairs(np.zeros((9, 0)), np.zeros(0))
    x = np.arange(9.0)
    assert np.array_equal(curv.low_rank_materialize(pairs), np.zeros((9, 9)))
    assert np.array_equal(curv.full_rank_materialize(pairs, 0.5), 0.5 * np.eye(9))
    assert np.array_equal(curv.low_rank_apply(pairs, x), np.zeros(9))
    assert np.allclose(curv.full_rank_apply(pairs, 0.5, x), 0.5 * x, rtol=1e-15)
    assert curv.full_rank_quadform(pairs, 0.5, x) == pytest.approx(0.5 * x @ x, rel=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("prec,dt", [("tf32", "float32"), ("f16s", "float32"), ("f64", "float64")])
def test_device_entry_points_config1_size(prec, dt):
    """P = 25 450 (config 1), k = 100: the materialised matrix against its own
    implicit forms and against fp64 torch products of the same eigenpairs."""
    import torch
    tdt = getattr(torch, dt)
    dev = torch.device("cuda", 0)
    p, k, lt = 25450, 100, 0.02
    g = torch.Generator(device="cpu").manual_seed(11)
    q64, _ = torch.linalg.qr(torch.randn(p, k, generator=g, dtype=torch.float64))
    lam64 = (2.0 * 0.93 ** torch.arange(k, dtype=torch.float64))
    ldq, ldh = 104, (p + 3) // 4 * 4
    q = torch.zeros((p, ldq), dtype=tdt, device=dev)
    q[:, :k] = q64.to(dev).to(tdt)
    lam = lam64.to(dev).to(tdt)
    h = torch.empty((p, ldh), dtype=tdt, device=dev)
    xs = torch.randn(5, p, generator=g, dtype=torch.float64).to(dev).to(tdt)
    y = torch.empty_like(xs)
    quad = torch.empty(5, dtype=torch.float64, device=dev)
    qd, ld_ = q[:, :k].double(), lam.double()
    for ltv in (None, lt):
        curv.dev_eig_materialize(p, k, q, ldq, lam, h, ldh, lambda_tilde=ltv, precision=prec)
        curv.dev_eig_apply(p, k, q, ldq, lam, 5, xs, p, y, p, quad, lambda_tilde=ltv, precision=prec)
        torch.cuda.synchronize()
        hm = h[:, :p]
        assert torch.equal(hm, hm.T)
        shift = 0.0 if ltv is None else ltv
        xd = xs.double()
        t = xd @ qd
        y_ref = (t * (ld_ - shift)) @ qd.T + shift * xd
        quad_ref = (t * t * (ld_ - shift)).sum(1) + shift * (xd * xd).sum(1)
        tol = 1e-12 if prec == "f64" else 2e-5
        assert float(torch.linalg.norm(y.double() - y_ref) / torch.linalg.norm(y_ref)) <= tol
        assert float(((quad - quad_ref).abs() / quad_ref.abs().clamp_min(1.0)).max()) <= tol
        # whole matrix: H X against the fp64 products (every entry of H enters)
        hx = (hm.double() @ xd.T).T
        assert float(torch.linalg.norm(hx - y_ref) / torch.linalg.norm(y_ref)) <= TOL[prec]


@pytest.mark.gpu
def test_device_apply_config4_size():
    """P = 1 055 242 (config 4), k = 100, fp32 storage: two passes over the 422 MB basis."""
    import torch
    dev = torch.device("cuda", 0)
    p, k, lt = 1055242, 100, 0.38
    g = torch.Generator(device=dev).manual_seed(5)
    q, _ = torch.linalg.qr(torch.randn(p, k, generator=g, dtype=torch.float32, device=dev))
    q = q.contiguous()
    lam = torch.linspace(0.5, 0.38, k, device=dev)
    xs = torch.randn(4, p, generator=g, dtype=torch.float32, device=dev)
    y = torch.empty_like(xs)
    quad = torch.empty(4, dtype=torch.float64, device=dev)
    curv.dev_eig_apply(p, k, q, k, lam, 4, xs, p, y, p, quad, lambda_tilde=lt, precision="f32")
    torch.cuda.synchronize()
    qd, xd, ld_ = q.double(), xs.double(), lam.double()
    t = xd @ qd
    y_ref = (t * (ld_ - lt)) @ qd.T + lt * xd
    quad_ref = (t * t * (ld_ - lt)).sum(1) + lt * (xd * xd).sum(1)
    assert float(torch.linalg.norm(y.double() - y_ref) / torch.linalg.norm(y_ref)) <= 2e-6
    assert float(((quad - quad_ref).abs() / quad_ref.abs()).max()) <= 2e-6


@pytest.mark.gpu
@pytest.mark.parametrize("prec,dt", [("f32", "float32"), ("tf32", "float32"), ("f64", "float64")])
@pytest.mark.parametrize("name", ["c0_opg", "ortho300", "k1"])
def test_device_entry_points_unpadded_operands(name, prec, dt):
    """Dense device operands as a caller may hold them: ldq = k and ldh = P (odd, or not a
    multiple of 4: rows that are not 16-byte aligned take the scalar-load and
    scalar-store forms of the kernels)."""
    import torch
    tdt = getattr(torch, dt)
    dev = torch.device("cuda", 0)
    c = case(name)
    p, k = c["q"].shape
    lt = float(c["lt"])
    q = torch.tensor(c["q"], dtype=tdt, device=dev).contiguous()
    lam = torch.tensor(c["lam"], dtype=tdt, device=dev)
    xs = torch.tensor(c["x"], dtype=tdt, device=dev).contiguous()
    h = torch.empty((p, p), dtype=tdt, device=dev)
    y = torch.empty_like(xs)
    quad = torch.empty(xs.shape[0], dtype=torch.float64, device=dev)
    tol = {"f64": 1e-12, "f32": 1e-5, "tf32": 1e-3}[prec]
    atol = 1e-12 if prec == "f64" else 2e-5
    for ltv, hk, yk, qk in ((None, "low", "low_y", "low_quad"), (lt, "full", "full_y", "full_quad")):
        curv.dev_eig_materialize(p, k, q, k, lam, h, p, lambda_tilde=ltv, precision=prec)
        curv.dev_eig_apply(p, k, q, k, lam, xs.shape[0], xs, p, y, p, quad, lambda_tilde=ltv, precision=prec)
        torch.cuda.synchronize()
        hh = h.double().cpu().numpy()
        assert np.array_equal(hh, hh.T)
        assert rel_fro(rows_of(hh, p), c[hk]) <= tol
        assert rel_fro(y.double().cpu().numpy(), c[yk]) <= atol
        scale = np.maximum(1.0, np.abs(c[qk]))
        assert np.max(np.abs(quad.cpu().numpy() - c[qk]) / scale) <= atol


# ---- row-sharded apply (the consumer of the sharded top-k solvers' output) ------

def _shard_apply_worker(rank, world, port, q):
    """Two processes on cuda:0 over the host transport: each holds its rows of Q, x, y."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        torch.cuda.set_device(0)
        dev = "cuda:0"
        c = case("ortho300")
        p, k = c["q"].shape
        lt = float(c["lt"])
        cut = [0, 113, p]  # an uneven row partition
        r0, r1 = cut[rank], cut[rank + 1]
        comm = curv.Comm.create_host(rank, world)
        for prec, tdt in (("f64", torch.float64), ("f32", torch.float32)):
            ql = torch.tensor(c["q"][r0:r1], dtype=tdt, device=dev).contiguous()
            lam = torch.tensor(c["lam"], dtype=tdt, device=dev)
            xl = torch.tensor(c["x"][:, r0:r1], dtype=tdt, device=dev).contiguous()
            yl = torch.empty_like(xl)
            quad = torch.empty(xl.shape[0], dtype=torch.float64, device=dev)
            for key, ltv in (("low", None), ("full", lt)):
                curv.dev_eig_apply_sharded(r1 - r0, k, ql, k, lam, xl.shape[0], xl, r1 - r0, comm, yl, r1 - r0, quad,
                                           lambda_tilde=ltv, precision=prec)
                torch.cuda.synchronize()
                ref_y = c[key + "_y"][:, r0:r1]
                out[(prec, key)] = (float(np.linalg.norm(yl.double().cpu().numpy() - ref_y) / np.linalg.norm(ref_y)),
                                    quad.cpu().numpy().tolist())
        comm.close()
    except Exception as ex:  # noqa: BLE001
        out = {"error": repr(ex)}
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_apply_two_processes_host_transport():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_shard_apply_worker, args=(r, 2, port, qq)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = dict(qq.get(timeout=600) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    c = case("ortho300")
    for rank in (0, 1):
        assert "error" not in outs[rank], outs[rank]
    for prec, tol in (("f64", 1e-12), ("f32", 2e-5)):
        for key in ("low", "full"):
            e0, q0 = outs[0][(prec, key)]
            e1, q1 = outs[1][(prec, key)]
            assert e0 <= tol and e1 <= tol, (prec, key, e0, e1)
            assert q0 == q1  # the all-reduced projections are the same bytes on every rank
            ref = c[key + "_quad"]
            assert np.max(np.abs(np.array(q0) - ref) / np.maximum(1.0, np.abs(ref))) <= tol


@pytest.mark.gpu
def test_sharded_apply_nccl_loopback_equals_unsharded(monkeypatch):
    """One rank holding every row: the NCCL all-reduce of the projections runs
    (CURVKIT_COMM_LOOPBACK=1) and the result equals the unsharded call bitwise."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("CURVKIT_COMM_LOOPBACK", "1")
    dev = "cuda:0"
    c = case("thin2000")
    p, k = c["q"].shape
    q = torch.tensor(c["q"], dtype=torch.float32, device=dev).contiguous()
    lam = torch.tensor(c["lam"], dtype=torch.float32, device=dev)
    xs = torch.tensor(c["x"], dtype=torch.float32, device=dev).contiguous()
    y0, y1 = torch.empty_like(xs), torch.empty_like(xs)
    q0 = torch.empty(3, dtype=torch.float64, device=dev)
    q1 = torch.empty(3, dtype=torch.float64, device=dev)
    curv.dev_eig_apply(p, k, q, k, lam, 3, xs, p, y0, p, q0, lambda_tilde=float(c["lt"]), precision="f32")
    comm = curv.Comm.create(0, 1, lambda b: b)
    try:
        curv.dev_eig_apply_sharded(p, k, q, k, lam, 3, xs, p, comm, y1, p, q1, lambda_tilde=float(c["lt"]),
                                   precision="f32")
    finally:
        comm.close()
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(q0, q1)


def _gloo_apply_worker(rank, world, port, q):
    """The exchange of curvkit_dev_eig_apply_sharded restated in numpy over gloo:
    partial projections of this rank's rows, one all-reduce of k + 1 doubles,
    local expansion."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = case("ortho300")
    p, k = c["q"].shape
    lt = float(c["lt"])
    cut = [0, 113, p]
    r0, r1 = cut[rank], cut[rank + 1]
    ql, lam = c["q"][r0:r1], c["lam"]
    res = []
    for v in range(c["x"].shape[0]):
        xl = c["x"][v, r0:r1]
        t = torch.tensor(np.concatenate([ql.T @ xl, [xl @ xl]]))  # (Q^T x)_local, (x.x)_local
        dist.all_reduce(t)
        t = t.numpy()
        yl = ql @ ((lam - lt) * t[:k]) + lt * xl
        quad = float(np.sum(lam * t[:k] ** 2) + lt * t[k] - lt * np.sum(t[:k] ** 2))
        res.append((yl, quad))
    q.put((rank, res))
    dist.destroy_process_group()


def test_gloo_two_ranks_sharded_apply():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    port = 29800 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_apply_worker, args=(r, 2, port, qq)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = dict(qq.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    c = case("ortho300")
    for v in range(c["x"].shape[0]):
        y = np.concatenate([outs[0][v][0], outs[1][v][0]])
        assert rel_fro(y, c["full_y"][v]) <= 1e-12
        assert outs[0][v][1] == outs[1][v][1]
        assert abs(outs[0][v][1] - c["full_quad"][v]) <= 1e-12 * max(1.0, abs(c["full_quad"][v]))


@pytest.mark.gpu
@pytest.mark.parametrize("dt,prec,tol", [("float32", "f32", 2e-5), ("float64", "f64", 1e-12)])
def test_device_apply_wide_basis(dt, prec, tol):
    """k = 300 > the 256 (fp32) / 128 (fp64) columns of one expansion chunk and the 128 / 64
    columns of one projection pass: the accumulators persist across the chunks."""
    import torch
    tdt = getattr(torch, dt)
    dev = torch.device("cuda", 0)
    p, k, lt = 1500, 300, 0.05
    g = torch.Generator(device="cpu").manual_seed(21)
    q64, _ = torch.linalg.qr(torch.randn(p, k, generator=g, dtype=torch.float64))
    lam64 = torch.linspace(3.0, 0.1, k, dtype=torch.float64)
    x64 = torch.randn(5, p, generator=g, dtype=torch.float64)
    q, lam, xs = q64.to(dev).to(tdt).contiguous(), lam64.to(dev).to(tdt), x64.to(dev).to(tdt).contiguous()
    y = torch.empty_like(xs)
    quad = torch.empty(5, dtype=torch.float64, device=dev)
    curv.dev_eig_apply(p, k, q, k, lam, 5, xs, p, y, p, quad, lambda_tilde=lt, precision=prec)
    torch.cuda.synchronize()
    qd, xd, ld_ = q.double(), xs.double(), lam.double()
    t = xd @ qd
    y_ref = (t * (ld_ - lt)) @ qd.T + lt * xd
    quad_ref = (t * t * (ld_ - lt)).sum(1) + lt * (xd * xd).sum(1)
    assert float(torch.linalg.norm(y.double() - y_ref) / torch.linalg.norm(y_ref)) <= tol
    assert float(((quad - quad_ref).abs() / quad_ref.abs().clamp_min(1.0)).max()) <= tol


@pytest.mark.gpu
def test_random_shapes_against_the_port():
    """Forty seeded shapes (P from 1 to 700, k from 0 to P, 1 to 6 vectors, padded and
    unpadded leading dimensions, fp64 and fp32) through the device entry points
    against the numpy port: ragged tiles, single rows, k = P."""
    import torch
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(2024)
    for trial in range(40):
        p = int(rng.choice([1, 2, 3, 7, 31, 32, 33, 64, 65, 129, 255, 300, 511, 700]))
        k = int(rng.integers(0, min(p, 140) + 1))
        nvec = int(rng.integers(1, 7))
        f64 = bool(trial % 2)
        tdt, prec, tol = (torch.float64, "f64", 1e-11) if f64 else (torch.float32, "f32", 5e-5)
        qn = np.linalg.qr(rng.standard_normal((p, max(k, 1))))[0][:, :k] if k else np.zeros((p, 0))
        lam = np.sort(rng.uniform(0.1, 3.0, k))[::-1].copy()
        lt = float(rng.uniform(0.01, 0.5)) if trial % 3 else None
        xs = rng.standard_normal((nvec, p))
        ldq = k + int(rng.integers(0, 6)) if k else 4
        ldx = p + int(rng.integers(0, 5))
        ldh = p + int(rng.integers(0, 9))
        q = torch.zeros((p, ldq), dtype=tdt, device=dev)
        q[:, :k] = torch.tensor(qn, dtype=tdt, device=dev)
        lamd = torch.tensor(lam, dtype=tdt, device=dev) if k else torch.zeros(1, dtype=tdt, device=dev)
        xd = torch.zeros((nvec, ldx), dtype=tdt, device=dev)
        xd[:, :p] = torch.tensor(xs, dtype=tdt, device=dev)
        y = torch.full((nvec, ldx), float("nan"), dtype=tdt, device=dev)
        quad = torch.empty(nvec, dtype=torch.float64, device=dev)
        h = torch.full((p, ldh), float("nan"), dtype=tdt, device=dev)
        curv.dev_eig_apply(p, k, q, ldq, lamd, nvec, xd, ldx, y, ldx, quad, lambda_tilde=lt, precision=prec)
        curv.dev_eig_materialize(p, k, q, ldq, lamd, h, ldh, lambda_tilde=lt, precision=prec)
        torch.cuda.synchronize()
        tag = (trial, p, k, nvec, prec, lt, ldq, ldx, ldh)
        qr_, xr = q[:, :k].double().cpu().numpy(), xd[:, :p].double().cpu().numpy()  # the operands as stored
        lr = lamd[:k].double().cpu().numpy()
        href = orc.eig_materialize_port(qr_, lr, lt) if k else (np.eye(p) * lt if lt else np.zeros((p, p)))
        hh = h[:, :p].double().cpu().numpy()
        assert np.array_equal(hh, hh.T), tag
        assert np.abs(hh - href).max() <= tol * max(1.0, np.abs(href).max()), tag
        for v in range(nvec):
            yr, qf = (orc.eig_apply_port(qr_, lr, xr[v], lt) if k else
                      ((lt or 0.0) * xr[v], (lt or 0.0) * float(xr[v] @ xr[v])))
            assert np.abs(y[v, :p].double().cpu().numpy() - yr).max() <= tol * max(1.0, np.abs(yr).max()), tag
            assert abs(float(quad[v]) - qf) <= tol * max(1.0, abs(qf)), tag
        if ldx > p:
            assert torch.isnan(y[:, p:]).all(), tag  # nothing written past the vectors
