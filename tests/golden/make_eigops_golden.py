"""Golden vectors for the consumers of eigenpairs (curv::low_rank_* /
full_rank_* / validate_eigen_pairs / default_lambda_tilde,
eigensolve.cpp:11-30 and 278-358), produced by the reference library itself
(oracle/_ref) on seeded inputs.  Run here, where /root/reference exists:

    python tests/golden/make_eigops_golden.py

Cases (each: q, lambda, lambda_tilde, x (nx x P), and the reference's low /
full matrices, A x and x^T A x for both operators):
  c0_opg     the top-6 eigenpairs of config 0's G (reference assemble_opg +
             its own sym_eig), P = 67
  ortho300   an exactly orthonormalised seeded Gaussian basis, P = 300, k = 37
             (k not a multiple of 4 or 32: ragged column tiles), geometric spectrum
  k1         P = 50, k = 1
  full_k     P = 24, k = 24 (Q square: I - Q Q^T = 0)
  thin2000   P = 2000, k = 130 (more than one 128-column pass of the projection);
             of its matrices only the rows ROWS are kept (fixture size)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402
from paper_1905_05559_b200.workloads import CONFIGS, normal  # noqa: E402


ROWS = (0, 7, 1023, 1999)


def basis(seed, p, k):
    q, _ = np.linalg.qr(normal(seed, p * k).reshape(p, k))
    return np.ascontiguousarray(q)


def main():
    ref = Ref()
    cases = {}
    wl = CONFIGS["c0"]
    params, x, y, _ = wl.draw()
    G = ref.opg(dict(widths=wl.widths, activation=wl.activation), params, x, y)
    vals, vecs = ref.sym_eig(G)
    order = np.argsort(-vals)[:6]
    cases["c0_opg"] = (np.ascontiguousarray(vecs[:, order]), vals[order], None)
    cases["ortho300"] = (basis(301, 300, 37), 3.0 * 0.85 ** np.arange(37), 0.004)
    cases["k1"] = (basis(302, 50, 1), np.array([2.5]), 0.75)
    cases["full_k"] = (basis(303, 24, 24), np.linspace(4.0, 0.5, 24), 0.25)
    cases["thin2000"] = (basis(304, 2000, 130), 1.0 / (1.0 + np.arange(130)), None)
    out = {}
    for name, (q, lam, lt) in cases.items():
        p, k = q.shape
        ref.validate_eigen_pairs(q, lam, 1e-8)
        lt = ref.default_lambda_tilde(lam) if lt is None else lt
        xs = normal(310 + len(out), 3 * p).reshape(3, p)
        xs[2] = q[:, 0] * 2.0  # inside the retained subspace
        low, _, _ = ref.eig_ops(q, lam, materialize=True)
        full, _, _ = ref.eig_ops(q, lam, lambda_tilde=lt, materialize=True)
        ly, lq, fy, fq = [], [], [], []
        for v in xs:
            _, yv, qv = ref.eig_ops(q, lam, x=v)
            ly.append(yv), lq.append(qv)
            _, yv, qv = ref.eig_ops(q, lam, x=v, lambda_tilde=lt)
            fy.append(yv), fq.append(qv)
        if p > 400:
            low, full = low[list(ROWS)], full[list(ROWS)]
        for key, val in (("q", q), ("lam", lam), ("lt", np.array(lt)), ("x", xs), ("low", low), ("full", full),
                         ("low_y", np.array(ly)), ("low_quad", np.array(lq)), ("full_y", np.array(fy)),
                         ("full_quad", np.array(fq))):
            out[f"{name}/{key}"] = val
        print(name, p, k, "lambda_tilde", lt, "|low|", np.linalg.norm(low), "|full|", np.linalg.norm(full))
    np.savez_compressed(os.path.join(HERE, "eigops.npz"), **out)


if __name__ == "__main__":
    main()
