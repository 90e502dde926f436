"""Generate tests/golden/*.npz from the REFERENCE library itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/libcurv_ref.so from the unmodified reference sources
(oracle/Makefile), draws seeded inputs with paper_1905_05559_b200.workloads,
and stores inputs + reference outputs.  The GPU box never needs
/root/reference: the tests read only these fixtures.

Paper listing values (Out[1]-[4], Out[9]) are asserted here before saving.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref, build  # noqa: E402
from paper_1905_05559_b200.workloads import CONFIGS, normal, splitmix64  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rand_case(widths, act, n, seed, scl=0.8, mode="softmax_cross_entropy"):
    P = sum(widths[k] * widths[k + 1] + widths[k + 1] for k in range(len(widths) - 1))
    params = scl * normal(seed, P)
    x = normal(seed + 7, n * widths[0]).reshape(n, widths[0])
    y = np.zeros((n, widths[-1]))
    if mode == "softmax_cross_entropy":
        lab = (splitmix64(seed + 13, n) % np.uint64(widths[-1])).astype(np.int64)
        y[np.arange(n), lab] = 1.0
    spec = dict(widths=widths, activation=act, output_mode=mode)
    return spec, params, x, y


def save(name, spec, **arrays):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), widths=np.array(spec["widths"]),
                        activation=spec["activation"], output_mode=spec.get("output_mode", "softmax_cross_entropy"),
                        **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items()})


def main():
    build()
    ref = Ref()

    # Paper listings (SPEC acceptance 1-2): linear diagnostic model
    spec = dict(widths=[4, 1], activation="identity", output_mode="raw_mean_output")
    params = np.array([3.0, 4.0, 5.0, 2.0, 0.0])
    x = np.array([[1.0, 2, 3, 4], [2.0, 3, 4, 5]])
    y = np.zeros((2, 1))
    f1 = ref.forward(spec, params, x[0])
    f2 = ref.forward(spec, params, x[1])
    assert f1[0] == 34.0 and f2[0] == 48.0  # Out [1]
    J = ref.jacobian(spec, params, x, y)
    assert list(J[0, :4]) == [1, 2, 3, 4] and list(J[1, :4]) == [2, 3, 4, 5]  # Out [2], [3]
    g = ref.grad_batch(spec, params, x, y)
    assert list(g[:4]) == [3, 5, 7, 9]  # Out [4]
    H, asym = ref.hessian(spec, params, x, y, batch=2)
    G = ref.opg(spec, params, x, y, batch=2)
    save("linear_diag", spec, params=params, x=x, y=y, forward=np.array([f1[0], f2[0]]), J=J, grad=g, H=H, G=G)
    assert ref.param_count([64, 32]) == 2080  # Out [9]

    small = [
        ("tanh352", [3, 5, 2], "tanh", 8, 101, 4),
        ("logistic32", [3, 2], "tanh", 8, 103, 8),
        ("sigmoid654", [6, 5, 4], "sigmoid", 8, 107, 8),
        ("relu543", [5, 4, 3], "relu", 6, 109, 3),
        ("deep4653", [4, 6, 5, 3], "tanh", 10, 111, 5),
        ("deep5_identity", [3, 4, 4, 3, 2], "identity", 6, 113, 6),
    ]
    for name, widths, act, n, seed, bh in small:
        spec, params, x, y = rand_case(widths, act, n, seed)
        P = len(params)
        H, asym = ref.hessian(spec, params, x, y, batch=bh)
        G = ref.opg(spec, params, x, y, batch=bh)
        J = ref.jacobian(spec, params, x, y)
        g = ref.grad_batch(spec, params, x, y)
        V = normal(seed + 99, 3 * P).reshape(3, P)
        HV = np.stack([ref.hvp(spec, params, x, y, v) for v in V])
        HVop = np.stack([ref.hvp_operator_apply(spec, params, x, y, bh, v) for v in V])
        cost = ref.cost(spec, params, x, y)
        save(name, spec, params=params, x=x, y=y, H=H, asym=asym, G=G, J=J, grad=g, V=V, HV=HV, HVop=HVop,
             batch=bh, cost=cost)

    # BASELINE config 0 (CPU-runnable oracle case), fp64
    wl = CONFIGS["c0"]
    params, x, y, _ = wl.draw()
    spec = dict(widths=wl.widths, activation=wl.activation)
    H, asym = ref.hessian(spec, params, x, y, batch=wl.n)
    G = ref.opg(spec, params, x, y, batch=wl.n)
    J = ref.jacobian(spec, params, x, y)
    save("config0", spec, params=params, x=x, y=y, H=H, asym=asym, G=G, J=J)

    # streaming-SVD single block is exact (acceptance 7): OPG eigen oracle
    rng_j = normal(105, 64 * 12).reshape(64, 12) * (0.5 ** np.arange(12))
    lam, q = ref.opg_eigs_incremental(rng_j, 64, 4)
    np.savez_compressed(os.path.join(OUT, "incremental_svd.npz"), J=rng_j, lam=lam, q=q)

    # Full-size pins for configs 1 and 2: Hessian columns / OPG rows computed
    # by the reference's own inner loops on the full datasets.
    for cname, cols, rows in (("c1", [0, 1, 783, 784, 12345, 25087, 25088, 25100, 25119, 25120, 25300, 25449],
                               [0, 5000, 25119, 25449]),
                              ("c2", [0, 30000, 50239, 50240, 52000, 54399, 54400, 55049], [])):
        wl = CONFIGS[cname]
        params, x, y, _ = wl.draw()
        spec = dict(widths=wl.widths, activation=wl.activation)
        hcols = np.concatenate([ref.hessian_columns_sample(spec, params, x, y, c, c + 1, 1) for c in cols], axis=1)
        arrays = dict(hcols=hcols, cols=np.array(cols))
        if rows:
            grows = np.concatenate([ref.opg_rows_sample(spec, params, x, y, r, r + 1, 8) for r in rows], axis=0)
            arrays.update(grows=grows, rows=np.array(rows))
        save(cname + "_pins", spec, **arrays)


if __name__ == "__main__":
    main()
