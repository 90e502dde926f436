"""curv::lanczos_topk on the Hessian operator (curvkit_hessian_topk_lanczos)
against the reference's own Lanczos run on the same HvpOperator
(tests/golden/lanczos_*.npz, made by tests/golden/make_lanczos_golden.py):
eigenvalues, eigenvectors up to sign, true residuals, iteration count, the
ConvergenceError path, and the reference's contract errors (CPU)."""
import numpy as np
import pytest

from conftest import load_golden
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.errors import ContractError, ConvergenceError

CONVERGED = ["lanczos_tanh", "lanczos_sigmoid_batched", "lanczos_deep"]


def _spec(g):
    s = g["spec"]
    return curv.ModelSpec(s["widths"], s["activation"], s["output_mode"])


def _cfg(g, **kw):
    c = dict(k=int(g["k"]), max_iterations=int(g["max_iterations"]), residual_tol=float(g["tol"]),
             seed=int(g["seed"]))
    c.update(kw)
    return curv.LanczosConfig(**c)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CONVERGED)
def test_lanczos_matches_reference(name):
    g = load_golden(name)
    r = curv.hessian_lanczos_topk(_spec(g), g["params"], curv.Batch(g["x"], g["y"]), int(g["batch"]), _cfg(g))
    lam, q = r.pairs.lam, r.pairs.q
    k = int(g["k"])
    np.testing.assert_allclose(lam, g["lam"], rtol=1e-9, atol=1e-12)
    assert np.all(np.diff(lam) <= 0)
    # orthonormal columns (validate_eigen_pairs, eigensolve.cpp:11-30) and the
    # reference's vectors up to sign
    assert np.abs(q.T @ q - np.eye(k)).max() <= 1e-8
    overlap = np.abs(np.sum(q * g["q"], axis=0))
    assert np.all(overlap >= 1 - 1e-7), overlap
    tol = float(g["tol"])
    assert np.all(r.residuals <= tol * np.maximum(1.0, np.abs(lam)))
    # the Krylov sequence starts from the reference's own start vector
    assert abs(r.iterations - int(g["iterations"])) <= 2, (r.iterations, int(g["iterations"]))


@pytest.mark.gpu
def test_lanczos_f32_mode():
    g = load_golden("lanczos_deep")
    r = curv.hessian_lanczos_topk(_spec(g), g["params"], curv.Batch(g["x"], g["y"]), int(g["batch"]),
                                  _cfg(g, residual_tol=1e-4), precision="f32")
    np.testing.assert_allclose(r.pairs.lam, g["lam"], rtol=1e-4, atol=1e-6)


@pytest.mark.gpu
def test_lanczos_convergence_error_carries_residuals():
    g = load_golden("lanczos_capped")
    with pytest.raises(ConvergenceError) as ei:
        curv.hessian_lanczos_topk(_spec(g), g["params"], curv.Batch(g["x"], g["y"]), int(g["batch"]), _cfg(g))
    assert len(ei.value.best_residuals) == int(g["k"])
    assert all(v > 0 for v in ei.value.best_residuals)


@pytest.mark.gpu
def test_lanczos_config1_rayleigh_quotients():
    """Top-5 of the config-1 Hessian (P = 25450): each Ritz value equals the
    Rayleigh quotient of its vector on the assembled fp64 H."""
    torch = pytest.importorskip("torch")
    from paper_1905_05559_b200.workloads import CONFIGS
    wl = CONFIGS["c1"]
    params, x, y, lab = wl.draw()
    spec = curv.ModelSpec(wl.widths, wl.activation)
    r = curv.hessian_lanczos_topk(spec, params, curv.Batch(x, y), wl.n,
                                  curv.LanczosConfig(k=5, max_iterations=300, residual_tol=1e-7, seed=1))
    d = "cuda:0"
    P = wl.P
    H = torch.empty((P, P), dtype=torch.float64, device=d)
    curv.dev_assemble_hessian(spec, torch.tensor(params, device=d), torch.tensor(x, device=d),
                              torch.tensor(lab, dtype=torch.int32, device=d), wl.n, H, P, precision="f64")
    Q = torch.tensor(r.pairs.q, device=d)
    rq = torch.sum(Q * (H @ Q), dim=0).cpu().numpy()
    np.testing.assert_allclose(rq, r.pairs.lam, rtol=1e-8, atol=1e-12)
    assert np.all(r.residuals <= 1e-7 * np.maximum(1.0, np.abs(r.pairs.lam)))


@pytest.mark.parametrize("kw,msg", [
    (dict(k=0), "need 1 <= k < p"),
    (dict(k=53), "need 1 <= k < p"),
    (dict(max_iterations=3), "max_iterations must be >= k"),
    (dict(residual_tol=0.0), "residual_tol must be > 0"),
])
def test_lanczos_contract_errors(kw, msg):
    g = load_golden("lanczos_tanh")
    with pytest.raises(ContractError, match=msg):
        curv.hessian_lanczos_topk(_spec(g), g["params"], curv.Batch(g["x"], g["y"]), int(g["batch"]), _cfg(g, **kw))


def test_lanczos_batch_divisibility():
    g = load_golden("lanczos_tanh")
    with pytest.raises(ContractError, match="not divisible"):
        curv.hessian_lanczos_topk(_spec(g), g["params"], curv.Batch(g["x"], g["y"]), 7, _cfg(g))
