"""The C restatement (oracle/curv_oracle.c) pinned against the reference's
own outputs (tests/golden, produced by oracle/_ref from the unmodified
reference sources) and, where the reference library is built here, live."""
import numpy as np
import pytest

from conftest import SMALL_CASES, load_golden, rel_fro
from oracle.oracle import Oracle, Ref

orc = Oracle()


@pytest.mark.parametrize("name", SMALL_CASES + ["config0"])
def test_oracle_matches_reference_golden(name):
    g = load_golden(name)
    spec, p, x, y = g["spec"], g["params"], g["x"], g["y"]
    b = int(g["batch"]) if "batch" in g else x.shape[0]
    H, asym = orc.hessian(spec, p, x, y, batch=b)
    assert np.max(np.abs(H - g["H"])) <= 1e-12 * max(1.0, np.abs(g["H"]).max())
    assert asym <= 1e-8 * max(1.0, np.abs(H).max())
    G = orc.opg(spec, p, x, y, batch=b)
    assert np.max(np.abs(G - g["G"])) <= 1e-12 * max(1.0, np.abs(g["G"]).max())
    J = orc.jacobian(spec, p, x, y)
    assert np.array_equal(J, g["J"])  # same arithmetic, same order: bit-exact
    if "HV" in g:
        for v, hv in zip(g["V"], g["HV"]):
            assert rel_fro(orc.hvp(spec, p, x, y, v), hv) <= 1e-12
        assert np.array_equal(orc.grad_batch(spec, p, x, y), g["grad"])
        assert abs(orc.cost(spec, p, x, y) - float(g["cost"])) <= 1e-13


def test_paper_listing_values_in_golden():
    g = load_golden("linear_diag")
    assert list(g["forward"]) == [34.0, 48.0]                      # Out [1]
    assert list(g["J"][0, :4]) == [1, 2, 3, 4]                      # Out [2]
    assert list(g["J"][1, :4]) == [2, 3, 4, 5]                      # Out [3]
    assert list(g["grad"][:4]) == [3, 5, 7, 9]                      # Out [4]
    assert np.all(g["H"] == 0.0)                                     # affine cost
    spec, p, x, y = g["spec"], g["params"], g["x"], g["y"]
    assert np.array_equal(orc.jacobian(spec, p, x, y), g["J"])
    assert orc.param_count([64, 32]) == 2080                         # Out [9]


def test_oracle_sym_eig_matches_reference():
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    ref = Ref()
    a = load_golden("config0")["G"]
    vo, qo = orc.sym_eig(a)
    vr, qr = ref.sym_eig(a)
    assert np.max(np.abs(vo - vr)) <= 1e-13
    assert np.max(np.abs(np.abs(qo) - np.abs(qr))) <= 1e-8


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_oracle_matches_reference_live_random():
    ref = Ref()
    rng = np.random.default_rng(0)
    for widths, act in (([4, 7, 3], "sigmoid"), ([5, 3, 4, 2], "tanh"), ([3, 6, 2], "relu")):
        P = sum(widths[k] * widths[k + 1] + widths[k + 1] for k in range(len(widths) - 1))
        n = 6
        p = rng.normal(size=P) * 0.7
        x = rng.normal(size=(n, widths[0]))
        y = np.eye(widths[-1])[rng.integers(0, widths[-1], n)]
        spec = dict(widths=widths, activation=act)
        Ho, _ = orc.hessian(spec, p, x, y, batch=3)
        Hr, _ = ref.hessian(spec, p, x, y, batch=3)
        assert np.max(np.abs(Ho - Hr)) <= 1e-12 * max(1, np.abs(Hr).max())
