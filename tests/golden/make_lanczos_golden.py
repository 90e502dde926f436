"""Generate tests/golden/lanczos_*.npz from the REFERENCE library's own
curv::lanczos_topk on its HvpOperator (oracle/_ref).  Run here, where
/root/reference exists:  python tests/golden/make_lanczos_golden.py

Cases: converged top-k of H for three models (incl. a ragged width and a
mini-batched operator), and one capped run that raises ConvergenceError (the
best residuals it carries are stored)."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from make_golden import rand_case, save  # noqa: E402
from oracle.oracle import OracleError, Ref, build  # noqa: E402

CASES = [
    # name, widths, act, n, seed, batch, k, max_iterations, tol, lanczos seed
    ("lanczos_tanh", [6, 5, 3], "tanh", 40, 21, 40, 4, 200, 1e-9, 7),
    ("lanczos_sigmoid_batched", [9, 7, 4], "sigmoid", 48, 22, 12, 5, 300, 1e-9, 11),
    ("lanczos_deep", [10, 8, 6, 3], "tanh", 60, 23, 30, 6, 400, 1e-9, 3),
]


def main():
    build()
    ref = Ref()
    for name, widths, act, n, seed, batch, k, maxit, tol, lseed in CASES:
        spec, params, x, y = rand_case(widths, act, n, seed)
        q, lam, res, it = ref.hessian_lanczos(spec, params, x, y, batch, k, maxit, tol, lseed)
        save(name, spec, params=params, x=x, y=y, batch=batch, k=k, max_iterations=maxit, tol=tol, seed=lseed,
             q=q, lam=lam, residuals=res, iterations=it, converged=1)
    # a capped run: max_iterations = k cannot reach 1e-12 -> ConvergenceError
    spec, params, x, y = rand_case([9, 7, 4], "sigmoid", 48, 22)
    try:
        ref.hessian_lanczos(spec, params, x, y, 48, 4, 4, 1e-12, 5)
        raise SystemExit("expected ConvergenceError")
    except OracleError as e:
        assert e.code == 4, e
    save("lanczos_capped", spec, params=params, x=x, y=y, batch=48, k=4, max_iterations=4, tol=1e-12, seed=5,
         converged=0)


if __name__ == "__main__":
    main()
