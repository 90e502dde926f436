"""Parity of the CUDA product (through the C-ABI) against the reference's own
outputs (tests/golden, produced by the unmodified reference library) and the
C oracle.  Tolerances (north_star, BASELINE.json): relative Frobenius error
<= 1e-5 in fp64 mode (we hold 1e-10), <= 1e-3 in fp32 / TF32 modes; top-k
eigenvalues within 1e-3 relative."""
import numpy as np
import pytest

from conftest import SMALL_CASES, load_golden, rel_fro
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-5, "tf32": 1e-3, "tf32x3": 1e-5, "f16s": 1e-3}
PRECS = list(TOL)


def spec_of(g):
    s = g["spec"]
    return curv.ModelSpec(s["widths"], s["activation"], s["output_mode"])


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", SMALL_CASES + ["config0", "linear_diag"])
def test_hessian_matches_reference(name, prec):
    g = load_golden(name)
    spec = spec_of(g)
    b = int(g["batch"]) if "batch" in g else g["x"].shape[0]
    cfg = curv.CurvatureConfig(batch_size_h=b)
    hr = curv.assemble_hessian(spec, g["params"], curv.Batch(g["x"], g["y"]), cfg, precision=prec, verify=True)
    if np.abs(g["H"]).max() == 0.0:
        assert np.abs(hr.h).max() <= 1e-12
        return
    assert rel_fro(hr.h, g["H"]) <= TOL[prec]
    assert np.array_equal(hr.h, hr.h.T)
    if prec == "f64":
        assert hr.asymmetry <= 1e-8 * max(1.0, np.abs(hr.h).max())
    # mirrored (fast) assembly equals the verified one
    fast = curv.assemble_hessian(spec, g["params"], curv.Batch(g["x"], g["y"]), cfg, precision=prec, verify=False)
    assert rel_fro(fast.h, g["H"]) <= TOL[prec]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", SMALL_CASES + ["config0", "linear_diag"])
def test_opg_and_jacobian_match_reference(name, prec):
    g = load_golden(name)
    spec = spec_of(g)
    b = int(g["batch"]) if "batch" in g else g["x"].shape[0]
    G = curv.assemble_opg(spec, g["params"], curv.Batch(g["x"], g["y"]), curv.CurvatureConfig(batch_size_g=b),
                          precision=prec)
    assert rel_fro(G, g["G"]) <= TOL[prec]
    assert np.array_equal(G, G.T)
    J = curv.assemble_jacobian(spec, g["params"], curv.Batch(g["x"], g["y"]), precision=prec)
    assert rel_fro(J, g["J"]) <= (1e-13 if prec == "f64" else 1e-6)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("name", SMALL_CASES)
def test_hvp_grad_match_reference(name, prec):
    g = load_golden(name)
    spec = spec_of(g)
    batch = curv.Batch(g["x"], g["y"])
    tol = 1e-12 if prec == "f64" else 1e-5
    HV = curv.hvp(spec, g["params"], batch, g["V"], precision=prec)
    for a, b in zip(HV, g["HV"]):
        assert rel_fro(a, b) <= tol
    op = curv.HvpOperator(spec, g["params"], batch, int(g["batch"]), precision=prec)
    assert rel_fro(op.apply(g["V"]), g["HVop"]) <= tol
    assert rel_fro(curv.grad_batch(spec, g["params"], batch, precision=prec).grad_total, g["grad"]) <= tol


def test_paper_listings_on_gpu():
    g = load_golden("linear_diag")
    spec = spec_of(g)
    batch = curv.Batch(g["x"], g["y"])
    J = curv.assemble_jacobian(spec, g["params"], batch)
    assert list(J[0, :4]) == [1, 2, 3, 4] and list(J[1, :4]) == [2, 3, 4, 5]   # Out [2], [3]
    assert list(curv.grad_batch(spec, g["params"], batch).grad_total[:4]) == [3, 5, 7, 9]  # Out [4]
    G = curv.assemble_opg(spec, g["params"], batch, curv.CurvatureConfig(batch_size_g=2))
    gbar = curv.grad_batch(spec, g["params"], batch).grad_total / 2
    assert np.abs(G - np.outer(gbar, gbar)).max() > 1e-3                    # Eq. 11
    assert np.abs(G - g["G"]).max() <= 1e-14


def test_hvp_symmetry_linearity():
    # acceptance criterion 9 on the (6,5,4) sigmoid model
    g = load_golden("sigmoid654")
    spec = spec_of(g)
    batch = curv.Batch(g["x"], g["y"])
    rng = np.random.default_rng(107)
    P = g["params"].shape[0]
    U = rng.normal(size=(20, P))
    V = rng.normal(size=(20, P))
    HU = curv.hvp(spec, g["params"], batch, U)
    HV = curv.hvp(spec, g["params"], batch, V)
    for u, v, hu, hv in zip(U, V, HU, HV):
        assert abs(u @ hv - v @ hu) <= 1e-9 * max(1.0, abs(u @ hv))
    a, b = 0.7, -1.3
    HC = curv.hvp(spec, g["params"], batch, a * U + b * V)
    assert rel_fro(HC, a * HU + b * HV) <= 1e-9


@pytest.mark.parametrize("prec", ["f64", "tf32", "f16s"])
def test_opg_topk_matches_dense_eig(prec):
    g = load_golden("config0")
    spec = spec_of(g)
    k = 5
    pairs = curv.opg_eigs(spec, g["params"], curv.Batch(g["x"], g["y"]), k, oversample=10, power_iters=2,
                          seed=3, precision=prec)
    w = np.linalg.eigvalsh(g["G"])[::-1]
    assert np.all(np.abs(pairs.lam - w[:k]) <= 1e-3 * np.abs(w[:k]))
    assert np.all(np.diff(pairs.lam) <= 0)
    qtq = pairs.q.T @ pairs.q
    assert np.abs(qtq - np.eye(k)).max() <= (1e-8 if prec == "f64" else 1e-4)
    r = g["G"] @ pairs.q - pairs.q * pairs.lam
    assert np.linalg.norm(r) <= 1e-3 * np.linalg.norm(g["G"])


# ---- full-size pins: configs 1 and 2 against reference columns / rows ---------

def _device_inputs(wl, torch, dtype):
    params, x, y, labels = wl.draw()
    dev = torch.device("cuda:0")
    return (torch.tensor(params, dtype=dtype, device=dev), torch.tensor(x, dtype=dtype, device=dev),
            torch.tensor(labels, dtype=torch.int32, device=dev))


@pytest.mark.parametrize("prec", ["tf32", "f64"])
def test_config1_hessian_and_opg_pins(prec):
    torch = pytest.importorskip("torch")
    wl = CONFIGS["c1"]
    pins = load_golden("c1_pins")
    dtype = torch.float64 if prec == "f64" else torch.float32
    p, x, lab = _device_inputs(wl, torch, dtype)
    spec = curv.ModelSpec(wl.widths, wl.activation)
    P = wl.P
    ld = (P + 3) // 4 * 4
    H = torch.empty((P, ld), dtype=dtype, device="cuda:0")
    curv.dev_assemble_hessian(spec, p, x, lab, wl.n, H, ld, precision=prec)
    torch.cuda.synchronize()
    cols = torch.tensor(pins["cols"], device="cuda:0")
    got = H[:, :P][:, cols].double().cpu().numpy()
    tol = 1e-9 if prec == "f64" else 1e-3
    for j in range(got.shape[1]):
        assert rel_fro(got[:, j], pins["hcols"][:, j]) <= tol, (j, rel_fro(got[:, j], pins["hcols"][:, j]))
    # symmetry by construction
    sub = H[:2000, :2000]
    assert torch.equal(sub, sub.T)
    del H
    G = torch.empty((P, ld), dtype=dtype, device="cuda:0")
    curv.dev_assemble_opg(spec, p, x, lab, wl.n, G, ld, precision=prec)
    torch.cuda.synchronize()
    rows = torch.tensor(pins["rows"], device="cuda:0")
    gr = G[rows, :P].double().cpu().numpy()
    for j in range(gr.shape[0]):
        assert rel_fro(gr[j], pins["grows"][j]) <= tol


def test_config3_opg_pins_tf32():
    """BASELINE config 3 at full size (P = 109 386, N = 10 000, G = 48 GB):
    six reference OPG rows (tests/golden/make_c3_pins.py) -- layer-0 weights
    (symmetric Khatri-Rao kernel), its bias, layer-1 weights and the output
    bias (rectangular J GEMM) -- and exact symmetry."""
    torch = pytest.importorskip("torch")
    wl = CONFIGS["c3"]
    pins = load_golden("c3_pins")
    p, x, lab = _device_inputs(wl, torch, torch.float32)
    spec = curv.ModelSpec(wl.widths, wl.activation)
    P = wl.P
    ld = (P + 3) // 4 * 4
    G = torch.empty((P, ld), dtype=torch.float32, device="cuda:0")
    curv.dev_assemble_opg(spec, p, x, lab, wl.n, G, ld, precision="tf32")
    torch.cuda.synchronize()
    rows = torch.tensor(pins["rows"], device="cuda:0")
    gr = G[rows, :P].double().cpu().numpy()
    for j in range(gr.shape[0]):
        assert rel_fro(gr[j], pins["grows"][j].astype(np.float64)) <= 1e-3, (int(pins["rows"][j]), rel_fro(gr[j], pins["grows"][j]))
    cols = G[:, rows].T.double().cpu().numpy()  # columns = rows by symmetry
    assert np.array_equal(cols, gr)
    del G
    torch.cuda.empty_cache()


def test_config2_hessian_pins_tf32():
    torch = pytest.importorskip("torch")
    wl = CONFIGS["c2"]
    pins = load_golden("c2_pins")
    p, x, lab = _device_inputs(wl, torch, torch.float32)
    spec = curv.ModelSpec(wl.widths, wl.activation)
    P = wl.P
    ld = (P + 3) // 4 * 4
    H = torch.empty((P, ld), dtype=torch.float32, device="cuda:0")
    curv.dev_assemble_hessian(spec, p, x, lab, wl.n, H, ld, precision="tf32")
    torch.cuda.synchronize()
    cols = torch.tensor(pins["cols"], device="cuda:0")
    got = H[:, :P][:, cols].double().cpu().numpy()
    for j in range(got.shape[1]):
        assert rel_fro(got[:, j], pins["hcols"][:, j]) <= 1e-3, j


@pytest.mark.parametrize("prec", ["tf32", "f32", "f16s"])
def test_config1_topk_against_dual_gram(prec):
    """Top-k of G at config-1 size (P = 23860, N = 4096): the K-split J X
    product and the device CholeskyQR2 path.  The nonzero spectrum of
    G = (1/N) J^T J equals that of the dual Gram (1/N) J J^T (N x N), formed
    here in fp64 from the fp64 Jacobian."""
    torch = pytest.importorskip("torch")
    wl = CONFIGS["c1"]
    spec = curv.ModelSpec(wl.widths, wl.activation)
    P, n = wl.P, wl.n
    p64, x64, lab = _device_inputs(wl, torch, torch.float64)
    J = torch.empty((n, P), dtype=torch.float64, device="cuda:0")
    curv.dev_assemble_jacobian(spec, p64, x64, lab, n, J, P, precision="f64")
    w = torch.linalg.eigvalsh(J @ J.T / n).flip(0)[:10].cpu().numpy()
    del J
    k = 20
    q = torch.empty((P, k), dtype=torch.float32, device="cuda:0")
    lam = torch.empty(k, dtype=torch.float32, device="cuda:0")
    curv.dev_opg_topk(spec, p64.float(), x64.float(), lab, n, k, 20, 2, 7, q, lam, precision=prec)
    torch.cuda.synchronize()
    lam = lam.double().cpu().numpy()
    assert np.all(np.diff(lam) <= 0)
    # the C - 1 = 9 separated eigenvalues (softmax: one direction per free
    # logit) within 1e-3; the first bulk eigenvalue is a range-finder
    # accuracy question (20 + 20 columns, 2 power iterations), not precision
    assert np.all(np.abs(lam[:9] - w[:9]) <= 1e-3 * np.abs(w[:9])), (lam[:10], w)
    assert lam[9] <= w[9] * (1 + 1e-3) and lam[9] >= 0.9 * w[9]
    qtq = (q.T.double() @ q.double()).cpu().numpy()
    assert np.abs(qtq - np.eye(k)).max() <= 1e-4
    # the default converged solver: all ten within 1e-3
    qa = torch.empty((P, 10), dtype=torch.float32, device="cuda:0")
    la = torch.empty(10, dtype=torch.float32, device="cuda:0")
    curv.dev_opg_topk_auto(spec, p64.float(), x64.float(), lab, n, 10, 20, 7, qa, la, precision=prec)
    torch.cuda.synchronize()
    la = la.double().cpu().numpy()
    assert np.all(np.abs(la - w[:10]) <= 1e-3 * np.abs(w[:10])), (la, w)


def test_config1_hessian_tmem_a_variant():
    """The opt-in fused Hessian variant with the R operand in TMEM
    (CURVKIT_HESS_TS=1, read once per process: run in a subprocess) against
    the reference's config-1 Hessian columns."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import load_golden, rel_fro
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS["c1"]; pins = load_golden("c1_pins")
params, x, y, lab = wl.draw()
d = "cuda:0"
p = torch.tensor(params, dtype=torch.float32, device=d); xx = torch.tensor(x, dtype=torch.float32, device=d)
ll = torch.tensor(lab, dtype=torch.int32, device=d)
spec = curv.ModelSpec(wl.widths, wl.activation); P = wl.P; ld = (P + 3) // 4 * 4
H = torch.empty((P, ld), dtype=torch.float32, device=d)
curv.dev_assemble_hessian(spec, p, xx, ll, wl.n, H, ld, precision="tf32"); torch.cuda.synchronize()
cols = torch.tensor(pins["cols"], device=d)
got = H[:, :P][:, cols].double().cpu().numpy()
err = max(rel_fro(got[:, j], pins["hcols"][:, j]) for j in range(got.shape[1]))
sub = H[:2000, :2000]
print("ERR", err, bool(torch.equal(sub, sub.T)))
'''
    import os
    env = dict(os.environ, CURVKIT_HESS_TS="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("ERR")][-1].split()
    assert float(line[1]) <= 1e-3 and line[2] == "True", line


@pytest.mark.parametrize("prec", ["f64", "tf32"])
def test_opg_eigs_from_jacobian_blocks(prec):
    """opg_eigs_incremental's input contract: the caller's row blocks of J.
    Against the reference's own streaming SVD (tests/golden/incremental_svd)
    and, for stacked config-0 blocks, the reference's G."""
    import os
    from conftest import GOLDEN
    g = np.load(os.path.join(GOLDEN, "incremental_svd.npz"))
    J = g["J"]
    pairs = curv.opg_eigs_incremental([J[:20], J[20:50], J[50:]], J.shape[0], 4, oversample=8, power_iters=2,
                                      precision=prec)
    tol = 1e-10 if prec == "f64" else 1e-3
    np.testing.assert_allclose(pairs.lam, g["lam"], rtol=tol)
    overlap = np.abs(np.sum(pairs.q * g["q"], axis=0))
    assert np.all(overlap >= 1 - (1e-9 if prec == "f64" else 1e-3)), overlap
    c0 = load_golden("config0")
    Jc = c0["J"]
    p2 = curv.opg_eigs_incremental([Jc[:50], Jc[50:100], Jc[100:]], Jc.shape[0], 5, oversample=10, power_iters=3,
                                   precision=prec)
    w = np.linalg.eigvalsh(c0["G"])[::-1][:5]
    assert np.all(np.abs(p2.lam - w) <= (1e-9 if prec == "f64" else 1e-3) * np.abs(w))
    with pytest.raises(curv.ContractError):
        curv.opg_eigs_incremental([Jc[:50]], Jc.shape[0], 5)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("name", SMALL_CASES + ["config0", "linear_diag"])
def test_forward_and_cost_match_oracle(name, prec):
    """curv::forward and curv::cost (model.cpp:178-256) against the C oracle."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import Oracle
    g = load_golden(name)
    spec = spec_of(g)
    orc = Oracle()
    tol = 1e-12 if prec == "f64" else 1e-5
    c_ref = orc.cost(g["spec"], g["params"], g["x"], g["y"])
    c = curv.cost(spec, g["params"], curv.Batch(g["x"], g["y"]), precision=prec)
    assert abs(c - c_ref) <= tol * max(1.0, abs(c_ref))
    out = curv.forward(spec, g["params"], g["x"], precision=prec)
    one = curv.forward(spec, g["params"], g["x"][0], precision=prec)
    np.testing.assert_allclose(one, out[0], rtol=tol, atol=tol)
    if spec.output_mode == curv.OutputMode.softmax_cross_entropy:
        np.testing.assert_allclose(out.sum(axis=1), 1.0, atol=tol * 10)


def test_opg_odd_pitch_device_buffer():
    """dev_assemble_opg (config 1: the CTA-pair SYRK with its TMA-box
    epilogue) into a buffer whose pitch is not a multiple of 4, where no TMA
    tensor is possible: the scalar epilogue must give the same G."""
    torch = pytest.importorskip("torch")
    wl = CONFIGS["c1"]
    p, x, lab = _device_inputs(wl, torch, torch.float32)
    spec = curv.ModelSpec(wl.widths, wl.activation)
    P = wl.P
    G1 = torch.zeros((P, P + 2), device="cuda:0")  # P + 2 = 25452: TMA-addressable
    curv.dev_assemble_opg(spec, p, x, lab, wl.n, G1, P + 2, precision="tf32")
    G2 = torch.zeros((P, P + 1), device="cuda:0")  # odd pitch
    curv.dev_assemble_opg(spec, p, x, lab, wl.n, G2, P + 1, precision="tf32")
    torch.cuda.synchronize()
    assert torch.equal(G1[:, :P], G2[:, :P])


def test_config4_topk_against_exact_spectrum():
    """BASELINE config 4 at full size (P = 1 055 242, N = 20 000): the device
    randomized range finder against the exact nonzero spectrum of G, from the
    dual Gram (1/N) J J^T (20 000 x 20 000, fp32 products accumulated in fp64,
    fp64 eigvalsh; J is 84 GB and formed only for this check).  Rayleigh-Ritz values are lower
    bounds of the true eigenvalues; the spectrum is flat (lambda_1/lambda_100 =
    1.3), so with the BASELINE's 2 power iterations they sit ~10% low and
    converge with more iterations: at 64 all 100 are within 1e-3 (DESIGN.md
    section 5)."""
    torch = pytest.importorskip("torch")
    wl = CONFIGS["c4"]
    p, x, lab = _device_inputs(wl, torch, torch.float32)
    spec = curv.ModelSpec(wl.widths, wl.activation)
    P, n, k = wl.P, wl.n, wl.eig_k
    lams = {}
    for it in (wl.power_iters, 64):
        q = torch.empty((P, k), dtype=torch.float32, device="cuda:0")
        lam = torch.empty(k, dtype=torch.float32, device="cuda:0")
        curv.dev_opg_topk(spec, p, x, lab, n, k, wl.oversample, it, 7, q, lam, precision="tf32")
        torch.cuda.synchronize()
        lams[it] = lam.double().cpu().numpy()
        del q
    # Chebyshev-filtered subspace iteration: 3 rounds of degree 6 (18 operator
    # applications instead of 64 power iterations), and the default converged
    # solver (Ritz-convergence stop rule, tol 1e-4)
    for tag in ("cheb3x6", "auto", "auto_f16s"):
        q = torch.empty((P, k), dtype=torch.float32, device="cuda:0")
        lam = torch.empty(k, dtype=torch.float32, device="cuda:0")
        if tag.startswith("auto"):
            curv.dev_opg_topk_auto(spec, p, x, lab, n, k, wl.oversample, 7, q, lam,
                                   precision="f16s" if tag == "auto_f16s" else "tf32")
        else:
            curv.dev_opg_topk_filtered(spec, p, x, lab, n, k, wl.oversample, 3, 6, 7, q, lam, precision="tf32")
        torch.cuda.synchronize()
        lams[tag] = lam.double().cpu().numpy()
        qtq = (q.T @ q).double().cpu().numpy()
        assert np.abs(qtq - np.eye(k)).max() <= 1e-4
        del q
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        ldj = (P + 31) // 32 * 32
        J = torch.empty((n, ldj), dtype=torch.float32, device="cuda:0")
        curv.dev_assemble_jacobian(spec, p, x, lab, n, J, ldj, precision="f32")
        # fp32 products accumulated in fp64 over column chunks of J: one
        # 20000 x 20000 x 1.05M SGEMM loses ~1e-3 of its entries on this GPU
        # (tools/gpu/dual_gram_check.py), chunks of 16384 keep them to ~2e-7
        K = torch.zeros((n, n), dtype=torch.float64, device="cuda:0")
        for c0 in range(0, P, 16384):
            Jc = J[:, c0:min(P, c0 + 16384)]
            K += (Jc @ Jc.T).double()
        del J, Jc
        torch.cuda.empty_cache()
        K = (K + K.T) / (2.0 * n)
        # the dual Gram rests on reference data: its block at 16 sampled examples
        # equals (1/N) J_s J_s^T of the reference's per-example gradient rows
        # (tests/golden/c4_sketch.npz, make_sketch_pins.py)
        pins = load_golden("c4_sketch")
        rows = torch.tensor(pins["rows"], device="cuda:0")
        blk = K[rows][:, rows].cpu().numpy()
        assert rel_fro(blk, pins["gram"] / n) <= 1e-5, rel_fro(blk, pins["gram"] / n)
        ev = torch.linalg.eigvalsh(K).flip(0)[:k].cpu().numpy()
        del K
        torch.cuda.empty_cache()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
    for it, lam in lams.items():
        assert np.all(np.diff(lam) <= 1e-6 * lam[0])            # descending
        assert np.all(lam <= ev * (1 + 1e-4)), it                  # Ritz values bound from below
    e2 = np.abs(lams[wl.power_iters] - ev) / ev
    e64 = np.abs(lams[64] - ev) / ev
    assert np.all(e64 <= e2 + 1e-4)                                # more iterations, closer
    assert e64.max() <= 1e-3, (e64.max(), int(e64.argmax()))       # the north_star's bar, all 100
    ec = np.abs(lams["cheb3x6"] - ev) / ev
    assert ec.max() <= 1e-3, (ec.max(), int(ec.argmax()))         # the same bar from 18 applications
    ea = np.abs(lams["auto"] - ev) / ev
    assert ea.max() <= 1e-3, (ea.max(), int(ea.argmax()))         # the default solver: stops converged
    ef = np.abs(lams["auto_f16s"] - ev) / ev
    assert ef.max() <= 1e-3, (ef.max(), int(ef.argmax()))         # the same in the F16S mode
    print(f"c4 max rel. eigenvalue error: power-2 {e2.max():.3e}, power-64 {e64.max():.3e}, "
          f"cheb 3x6 {ec.max():.3e}, auto {ea.max():.3e}, auto f16s {ef.max():.3e}")


@pytest.mark.parametrize("prec", ["f64", "tf32"])
def test_opg_eigs_default_is_converged(prec):
    """curv.opg_eigs with no solver arguments: the Chebyshev filter with the
    Ritz-convergence stop rule (curvkit_opg_topk_auto) against the dense
    eigendecomposition of the reference's G."""
    g = load_golden("config0")
    spec = spec_of(g)
    k = 5
    pairs = curv.opg_eigs(spec, g["params"], curv.Batch(g["x"], g["y"]), k, oversample=10, seed=3, precision=prec)
    w = np.linalg.eigvalsh(g["G"])[::-1]
    assert np.all(np.abs(pairs.lam - w[:k]) <= 1e-3 * np.abs(w[:k])), (pairs.lam, w[:k])
    assert np.abs(pairs.q.T @ pairs.q - np.eye(k)).max() <= (1e-8 if prec == "f64" else 1e-4)
    with pytest.raises(curv.ContractError):
        curv.opg_eigs(spec, g["params"], curv.Batch(g["x"], g["y"]), k, tol=0.0)


@pytest.mark.parametrize("prec", ["f64", "tf32"])
def test_opg_eigs_filtered_host_mirror(prec):
    g = load_golden("config0")
    spec = spec_of(g)
    k = 5
    pairs = curv.opg_eigs(spec, g["params"], curv.Batch(g["x"], g["y"]), k, oversample=10, seed=3, precision=prec,
                          filter_steps=2, filter_degree=4)
    w = np.linalg.eigvalsh(g["G"])[::-1]
    assert np.all(np.abs(pairs.lam - w[:k]) <= 1e-3 * np.abs(w[:k]))
    assert np.abs(pairs.q.T @ pairs.q - np.eye(k)).max() <= (1e-8 if prec == "f64" else 1e-4)


@pytest.mark.parametrize("prec", ["f64", "tf32"])
def test_filtered_topk_matches_dense_eig(prec):
    """Chebyshev-filtered top-k (curvkit_dev_opg_topk_filtered) against the
    dense eigendecomposition of the reference's config-0 G."""
    torch = pytest.importorskip("torch")
    g = load_golden("config0")
    spec = spec_of(g)
    dt = torch.float64 if prec == "f64" else torch.float32
    dev = "cuda:0"
    P, n, k = g["G"].shape[0], g["x"].shape[0], 5
    p = torch.tensor(g["params"], dtype=dt, device=dev)
    x = torch.tensor(g["x"], dtype=dt, device=dev)
    lab = torch.tensor(np.argmax(g["y"], axis=1), dtype=torch.int32, device=dev)
    qd = torch.empty((P, k), dtype=dt, device=dev)
    lamd = torch.empty(k, dtype=dt, device=dev)
    curv.dev_opg_topk_filtered(spec, p, x, lab, n, k, 10, 2, 4, 3, qd, lamd, precision=prec)
    torch.cuda.synchronize()
    lam = lamd.double().cpu().numpy()
    q = qd.double().cpu().numpy()
    w = np.linalg.eigvalsh(g["G"])[::-1]
    assert np.all(np.abs(lam - w[:k]) <= 1e-3 * np.abs(w[:k])), (lam, w[:k])
    assert np.all(np.diff(lam) <= 0)
    assert np.abs(q.T @ q - np.eye(k)).max() <= (1e-8 if prec == "f64" else 1e-4)
    r = g["G"] @ q - q * lam
    assert np.linalg.norm(r) <= 1e-3 * np.linalg.norm(g["G"])
    with pytest.raises(curv.ContractError):
        curv.dev_opg_topk_filtered(spec, p, x, lab, n, k, 10, 2, 0, 3, qd, lamd, precision=prec)


@pytest.mark.parametrize("prec", ["tf32", "f64"])
def test_wide_layer_orbits_against_oracle(prec):
    """A 400-unit layer: 80 200 packed (o, o'') columns (more than one grid
    dimension holds) through the symmetric-orbit kernels, against the C oracle
    for H and G; inputs in [4, 400, 3] make the first layer's T_k = 4."""
    from oracle.oracle import Oracle
    from paper_1905_05559_b200.workloads import normal, splitmix64
    widths, n = [4, 400, 3], 16
    P = sum(widths[k] * widths[k + 1] + widths[k + 1] for k in range(len(widths) - 1))
    params = 0.3 * normal(901, P)
    x = normal(907, n * widths[0]).reshape(n, widths[0])
    y = np.zeros((n, widths[-1]))
    y[np.arange(n), (splitmix64(913, n) % np.uint64(widths[-1])).astype(np.int64)] = 1.0
    ospec = dict(widths=widths, activation="sigmoid")
    orc = Oracle()
    H_ref, _ = orc.hessian(ospec, params, x, y, batch=n)
    G_ref = orc.opg(ospec, params, x, y)
    spec = curv.ModelSpec(widths, "sigmoid")
    hr = curv.assemble_hessian(spec, params, curv.Batch(x, y), curv.CurvatureConfig(batch_size_h=n), precision=prec)
    G = curv.assemble_opg(spec, params, curv.Batch(x, y), curv.CurvatureConfig(batch_size_g=n), precision=prec)
    tol = TOL[prec]
    assert rel_fro(hr.h, H_ref) <= tol, rel_fro(hr.h, H_ref)
    assert rel_fro(G, G_ref) <= tol, rel_fro(G, G_ref)
    assert np.array_equal(hr.h, hr.h.T) and np.array_equal(G, G.T)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["c1", "wide_upper"])
def test_host_f32_entry_points_equal_device_results(shape):
    """curvkit_assemble_opg_f32 / _hessian_f32 (fp32 host output; for G above 1 GiB the
    two-phase form: the upper layers' rows travel to the host while the first
    layer's block is computed) against the device entry points on the same inputs:
    the same kernels, so the same bytes."""
    import ctypes as C

    import torch
    from paper_1905_05559_b200 import _lib
    lib = _lib.load()
    if shape == "c1":  # first layer of 32 units: its block in four unit ranges
        wl = CONFIGS["c1"]
        params, x, y, lab = wl.draw()
        spec = curv.ModelSpec(wl.widths, wl.activation)
        P, n = wl.P, wl.n
    else:  # 12 units in the first layer (one range) and 39% of the rows in the layers above it
        rng = np.random.default_rng(17)
        widths, n = [1200, 12, 400, 10], 256
        spec = curv.ModelSpec(widths, "tanh")
        P = curv.param_count(spec)
        params = rng.normal(0.0, 0.05, P)
        x = rng.normal(0.0, 1.0, (n, widths[0]))
        lab = rng.integers(0, widths[-1], n)
        y = np.eye(widths[-1])[lab]
    dev = "cuda:0"
    p_d = torch.tensor(params, dtype=torch.float32, device=dev)
    x_d = torch.tensor(x, dtype=torch.float32, device=dev)
    l_d = torch.tensor(lab, dtype=torch.int32, device=dev)
    ld = (P + 31) // 32 * 32
    cfg = curv.CurvatureConfig(batch_size_h=n, batch_size_g=n, memory_cap=1 << 40)._c()
    m = spec._c()
    dp = lambda a: np.ascontiguousarray(a).ctypes.data_as(_lib.dptr)  # noqa: E731
    pp, xp, yp = (np.ascontiguousarray(a, dtype=np.float64) for a in (params, x, y))
    for host_fn, dev_fn, prec in ((lib.curvkit_assemble_opg_f32, curv.dev_assemble_opg, "tf32"),
                                  (lib.curvkit_assemble_opg_f32, curv.dev_assemble_opg, "f16s"),
                                  (lib.curvkit_assemble_hessian_f32, curv.dev_assemble_hessian, "tf32")):
        h = torch.full((P, P), float("nan"), dtype=torch.float32).pin_memory()
        _lib.check(host_fn(C.byref(m), dp(pp), dp(xp), dp(yp), n, C.byref(cfg), curv.PRECISION[prec],
                           C.cast(h.data_ptr(), _lib.fptr)))
        d = torch.empty((P, ld), dtype=torch.float32, device=dev)
        dev_fn(spec, p_d, x_d, l_d, n, d, ld, precision=prec)
        torch.cuda.synchronize()
        hd = d[:, :P].cpu()
        assert not torch.isnan(h).any()
        assert torch.equal(h, hd)
        assert torch.equal(h, h.T)
        del h, d, hd
