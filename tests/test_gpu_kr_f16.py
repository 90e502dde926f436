"""F16S Khatri-Rao products (J X and J^T T, J never formed) against the TF32
ones and against the dense Jacobian.

F16S stores every operand as an fp16 significand under an exact power-of-two
scale (a_k per example row for J X, per input column for J^T T; X per column;
delta_o T per (unit, column)), i.e. the same 11-bit round-to-nearest operands
as TF32, so the two precisions differ only in the fp32 accumulation order:
bound 2e-5 between them, 1e-3 (the TF32 class) against J from
curvkit_dev_assemble_jacobian in fp64.  Shapes cover the per-layer fallback
(T_k % 8 != 0 takes the TF32 J X kernel), K-split J^T T (narrow layers), two
128-column tiles, and shard ranges.
"""
import numpy as np
import pytest

from conftest import rel_fro
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS, Workload

CASES = {
    "c0": CONFIGS["c0"],
    "c1": CONFIGS["c1"],
    "c2": CONFIGS["c2"],
    "odd": Workload("odd", [13, 40, 24, 7], "tanh", 333, "normal", "normal", 91),
    "wide": Workload("wide", [96, 200, 5], "sigmoid", 700, "uniform", "zero", 92),
}


def _setup(torch, wl):
    params, x, _, lab = wl.draw()
    dev = "cuda:0"
    spec = curv.ModelSpec(wl.widths, wl.activation)
    p64 = torch.tensor(params, dtype=torch.float64, device=dev)
    x64 = torch.tensor(x, dtype=torch.float64, device=dev)
    labels = torch.tensor(lab, dtype=torch.int32, device=dev)
    J = torch.empty((wl.n, wl.P), dtype=torch.float64, device=dev)
    curv.dev_assemble_jacobian(spec, p64, x64, labels, wl.n, J, wl.P, precision="f64")
    return spec, p64.float(), x64.float(), labels, J


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("l", [40, 150])
def test_f16s_products_match_tf32_and_dense(name, l):
    torch = pytest.importorskip("torch")
    wl = CASES[name]
    spec, p32, x32, lab, J = _setup(torch, wl)
    n, P = wl.n, wl.P
    ld = ((l + 31) // 32) * 32
    g = torch.Generator(device="cuda:0").manual_seed(17 + l)
    X = torch.zeros((P, ld), device="cuda:0")
    X[:, :l] = torch.randn((P, l), device="cuda:0", generator=g)
    U = torch.zeros((n, ld), device="cuda:0")
    U[:, :l] = torch.randn((n, l), device="cuda:0", generator=g)
    out = {}
    for prec in ("tf32", "f16s"):
        T = torch.zeros((n, ld), device="cuda:0")
        curv.dev_jacobian_apply(spec, p32, x32, lab, n, 0, P, X, ld, l, T, ld, precision=prec)
        Y = torch.zeros((P, ld), device="cuda:0")
        curv.dev_jacobian_apply(spec, p32, x32, lab, n, 0, P, U, ld, l, Y, ld, transpose=True, precision=prec)
        out[prec] = (T[:, :l].double().cpu().numpy(), Y[:, :l].double().cpu().numpy())
    Tref = (J @ X[:, :l].double()).cpu().numpy()
    Yref = (J.T @ U[:, :l].double()).cpu().numpy()
    for prec, (T, Y) in out.items():
        assert rel_fro(T, Tref) <= 1e-3, (prec, "J X", rel_fro(T, Tref))
        assert rel_fro(Y, Yref) <= 1e-3, (prec, "J^T T", rel_fro(Y, Yref))
    assert rel_fro(out["f16s"][0], out["tf32"][0]) <= 2e-5
    assert rel_fro(out["f16s"][1], out["tf32"][1]) <= 2e-5


@pytest.mark.gpu
def test_f16s_shard_rows_sum_to_full():
    torch = pytest.importorskip("torch")
    wl = CASES["odd"]
    spec, p32, x32, lab, _ = _setup(torch, wl)
    n, P, l = wl.n, wl.P, 40
    g = torch.Generator(device="cuda:0").manual_seed(3)
    X = torch.zeros((P, 64), device="cuda:0")
    X[:, :l] = torch.randn((P, l), device="cuda:0", generator=g)
    U = torch.zeros((n, 64), device="cuda:0")
    U[:, :l] = torch.randn((n, l), device="cuda:0", generator=g)
    T = torch.zeros((n, 64), device="cuda:0")
    curv.dev_jacobian_apply(spec, p32, x32, lab, n, 0, P, X, 64, l, T, 64, precision="f16s")
    Y = torch.zeros((P, 64), device="cuda:0")
    curv.dev_jacobian_apply(spec, p32, x32, lab, n, 0, P, U, 64, l, Y, 64, transpose=True, precision="f16s")
    acc = np.zeros((n, l))
    for r in range(3):
        b, e = curv.topk_shard_rows(spec, 3, r)
        Tr = torch.zeros((n, 64), device="cuda:0")
        curv.dev_jacobian_apply(spec, p32, x32, lab, n, b, e, X[b:e].contiguous(), 64, l, Tr, 64, precision="f16s")
        acc += Tr[:, :l].double().cpu().numpy()
        Yr = torch.zeros((e - b, 64), device="cuda:0")
        curv.dev_jacobian_apply(spec, p32, x32, lab, n, b, e, U, 64, l, Yr, 64, transpose=True, precision="f16s")
        assert rel_fro(Yr[:, :l].double().cpu().numpy(), Y[b:e, :l].double().cpu().numpy()) <= 1e-6
    assert rel_fro(acc, T[:, :l].double().cpu().numpy()) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("extra", [0, 1, 3])
def test_dev_jacobian_any_pitch(prec, extra):
    """curvkit_dev_assemble_jacobian at pitches that break 16-byte row
    alignment (P = 67 and 4-input layers): scalar stores, same entries as the
    host entry point; the padding columns are left untouched."""
    torch = pytest.importorskip("torch")
    wl = CONFIGS["c0"]
    params, x, y, lab = wl.draw()
    spec = curv.ModelSpec(wl.widths, wl.activation)
    ref = curv.assemble_jacobian(spec, params, curv.Batch(x, y), precision="f64")
    dt = torch.float64 if prec == "f64" else torch.float32
    ld = wl.P + extra
    J = torch.full((wl.n, ld), 7.0, dtype=dt, device="cuda:0")
    curv.dev_assemble_jacobian(spec, torch.tensor(params, dtype=dt, device="cuda:0"),
                               torch.tensor(x, dtype=dt, device="cuda:0"),
                               torch.tensor(lab, dtype=torch.int32, device="cuda:0"), wl.n, J, ld, precision=prec)
    got = J.double().cpu().numpy()
    assert rel_fro(got[:, :wl.P], ref) <= (1e-12 if prec == "f64" else 1e-5)
    assert np.all(got[:, wl.P:] == 7.0)
