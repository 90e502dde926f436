"""TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU checkers.

  Oracle -- oracle/liboracle.so, the plain-C restatement (curv_oracle.c)
  Ref    -- oracle/_ref/libcurv_ref.so, the unmodified reference sources
            compiled by oracle/Makefile (absent unless built)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.  The product (paper_1905_05559_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ACT = {"identity": 0, "sigmoid": 1, "tanh": 2, "relu": 3}
MODE = {"softmax_cross_entropy": 0, "raw_mean_output": 1}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
i64 = C.c_int64


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class _Lib:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        p = self.prefix
        model = [_ip, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, i64]
        sigs = {
            "jacobian": model + [_dp],
            "grad_batch": model + [_dp],
            "hvp": model + [_dp, _dp],
            "cost": model + [C.POINTER(C.c_double)],
        }
        for name, args in sigs.items():
            f = getattr(self.lib, p + name)
            f.argtypes = args
            f.restype = C.c_int
        getattr(self.lib, p + "param_count").argtypes = [_ip, C.c_int]
        getattr(self.lib, p + "param_count").restype = i64
        getattr(self.lib, p + "sym_eig").argtypes = [_dp, i64, _dp, _dp]
        getattr(self.lib, p + "sym_eig").restype = C.c_int

    def _err(self, rc):
        raise OracleError(rc)

    def _call(self, name, *args):
        rc = getattr(self.lib, self.prefix + name)(*args)
        if rc != 0:
            self._err(rc)

    @staticmethod
    def _m(spec):
        w = np.ascontiguousarray(spec["widths"], dtype=np.int64)
        return w, len(w), ACT[spec.get("activation", "tanh")], MODE[spec.get("output_mode", "softmax_cross_entropy")]

    def param_count(self, widths):
        w = np.ascontiguousarray(widths, dtype=np.int64)
        return int(getattr(self.lib, self.prefix + "param_count")(w, len(w)))

    def jacobian(self, spec, params, x, y):
        w, L, a, m = self._m(spec)
        n = x.shape[0]
        out = np.zeros((n, self.param_count(w)))
        self._call("jacobian", w, L, a, m, _f64(params), _f64(x), _f64(y), n, out)
        return out

    def grad_batch(self, spec, params, x, y):
        w, L, a, m = self._m(spec)
        out = np.zeros(self.param_count(w))
        self._call("grad_batch", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0], out)
        return out

    def hvp(self, spec, params, x, y, v):
        w, L, a, m = self._m(spec)
        out = np.zeros(self.param_count(w))
        self._call("hvp", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0], _f64(v), out)
        return out

    def cost(self, spec, params, x, y):
        w, L, a, m = self._m(spec)
        out = C.c_double()
        self._call("cost", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0], C.byref(out))
        return out.value

    def sym_eig(self, a):
        a = _f64(a)
        n = a.shape[0]
        vals = np.zeros(n)
        vecs = np.zeros((n, n))
        self._call("sym_eig", a, n, vals, vecs)
        return vals, vecs


class Oracle(_Lib):
    prefix = "orc_"

    def __init__(self):
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        super().__init__(path)
        self.lib.orc_hessian.argtypes = [_ip, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, i64, i64, _dp,
                                         C.POINTER(C.c_double)]
        self.lib.orc_opg.argtypes = [_ip, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, i64, i64, _dp]

    def hessian(self, spec, params, x, y, batch=None):
        w, L, a, m = self._m(spec)
        n = x.shape[0]
        P = self.param_count(w)
        H = np.zeros((P, P))
        asym = C.c_double()
        self._call("hessian", w, L, a, m, _f64(params), _f64(x), _f64(y), n, batch or n, H, C.byref(asym))
        return H, asym.value

    def opg(self, spec, params, x, y, batch=None):
        w, L, a, m = self._m(spec)
        n = x.shape[0]
        P = self.param_count(w)
        G = np.zeros((P, P))
        self._call("opg", w, L, a, m, _f64(params), _f64(x), _f64(y), n, batch or n, G)
        return G


class Ref(_Lib):
    """The reference library itself (oracle/_ref)."""
    prefix = "ref_"
    path = os.path.join(HERE, "_ref", "libcurv_ref.so")

    @classmethod
    def available(cls):
        return os.path.exists(cls.path)

    def __init__(self):
        super().__init__(self.path)
        lib = self.lib
        lib.ref_last_error.restype = C.c_char_p
        mdl = [_ip, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, i64]
        lib.ref_hessian.argtypes = mdl + [i64, i64, i64, _dp, C.POINTER(C.c_double)]
        lib.ref_opg.argtypes = mdl + [i64, i64, _dp]
        lib.ref_hessian_columns_sample.argtypes = mdl + [i64, i64, i64, _dp]
        lib.ref_opg_rows_sample.argtypes = mdl + [i64, i64, i64, _dp]
        lib.ref_hvp_operator_apply.argtypes = mdl + [i64, _dp, _dp]
        lib.ref_forward.argtypes = [_ip, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        lib.ref_opg_eigs_incremental.argtypes = [_dp, i64, i64, i64, i64, _dp, _dp]
        lib.ref_hessian_lanczos.argtypes = mdl + [i64, i64, i64, C.c_double, C.c_uint64, _dp, _dp, _dp,
                                                  C.POINTER(i64)]
        lib.ref_opg_rows_from_jacobian.argtypes = [_dp, i64, i64, i64, i64, i64, _dp]
        lib.ref_hessian_sketch.argtypes = mdl + [_dp, i64, i64, _dp]
        lib.ref_opg_sketch.argtypes = mdl + [_dp, i64, i64, _dp]
        lib.ref_eig_ops.argtypes = [_dp, _dp, i64, i64, C.c_int, C.c_double, i64, C.c_void_p, i64, C.c_void_p,
                                    C.c_void_p, C.c_void_p]
        lib.ref_validate_eigen_pairs.argtypes = [_dp, i64, i64, _dp, i64, C.c_double]
        lib.ref_default_lambda_tilde.argtypes = [_dp, i64, C.POINTER(C.c_double)]
        for f in ("ref_eig_ops", "ref_validate_eigen_pairs", "ref_default_lambda_tilde"):
            getattr(lib, f).restype = C.c_int
        for f in ("ref_hessian", "ref_opg", "ref_hessian_columns_sample", "ref_opg_rows_sample",
                  "ref_hvp_operator_apply", "ref_forward", "ref_opg_eigs_incremental", "ref_hessian_lanczos",
                  "ref_opg_rows_from_jacobian", "ref_hessian_sketch", "ref_opg_sketch"):
            getattr(lib, f).restype = C.c_int

    def _err(self, rc):
        raise OracleError(rc, self.lib.ref_last_error().decode())

    def forward(self, spec, params, x):
        w, L, a, m = self._m(spec)
        out = np.zeros(w[-1])
        self._call("forward", w, L, a, m, _f64(params), _f64(x), out)
        return out

    def hessian(self, spec, params, x, y, batch=None, lanes=1, memory_cap=1 << 40):
        w, L, a, m = self._m(spec)
        n = x.shape[0]
        P = self.param_count(w)
        H = np.zeros((P, P))
        asym = C.c_double()
        self._call("hessian", w, L, a, m, _f64(params), _f64(x), _f64(y), n, batch or n, lanes,
                   memory_cap, H, C.byref(asym))
        return H, asym.value

    def opg(self, spec, params, x, y, batch=None, memory_cap=1 << 40):
        w, L, a, m = self._m(spec)
        n = x.shape[0]
        P = self.param_count(w)
        G = np.zeros((P, P))
        self._call("opg", w, L, a, m, _f64(params), _f64(x), _f64(y), n, batch or n, memory_cap, G)
        return G

    def hvp_operator_apply(self, spec, params, x, y, batch, v):
        w, L, a, m = self._m(spec)
        out = np.zeros(self.param_count(w))
        self._call("hvp_operator_apply", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0],
                   batch, _f64(v), out)
        return out

    def hessian_lanczos(self, spec, params, x, y, batch, k, max_iterations, residual_tol, seed):
        """lanczos_topk on the reference HvpOperator: (q P x k, lambda, residuals, iterations)."""
        w, L, a, m = self._m(spec)
        P = self.param_count(w)
        q = np.zeros((P, k))
        lam = np.zeros(k)
        res = np.zeros(k)
        it = i64(0)
        self._call("hessian_lanczos", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0], batch, k,
                   max_iterations, residual_tol, seed, q, lam, res, C.byref(it))
        return q, lam, res, int(it.value)

    def hessian_columns_sample(self, spec, params, x, y, c0, c1, lanes):
        w, L, a, m = self._m(spec)
        P = self.param_count(w)
        out = np.zeros((P, c1 - c0))
        self._call("hessian_columns_sample", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0],
                   c0, c1, lanes, out)
        return out

    def opg_rows_sample(self, spec, params, x, y, r0, r1, lanes):
        w, L, a, m = self._m(spec)
        P = self.param_count(w)
        out = np.zeros((r1 - r0, P))
        self._call("opg_rows_sample", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0],
                   r0, r1, lanes, out)
        return out

    def opg_rows_from_jacobian(self, J, r0, r1, lanes):
        """Rows [r0, r1) of G by the reference's rank-1 loop on a held Jacobian."""
        n, p = J.shape
        out = np.zeros((r1 - r0, p))
        self._call("opg_rows_from_jacobian", J, n, p, r0, r1, lanes, out)
        return out

    def hessian_sketch(self, spec, params, x, y, omega, lanes):
        """H @ omega (P x k) by k reference HVPs of the dataset-averaged cost."""
        w, L, a, m = self._m(spec)
        omega = _f64(omega)
        out = np.zeros_like(omega)
        self._call("hessian_sketch", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0], omega,
                   omega.shape[1], lanes, out)
        return out

    def opg_sketch(self, spec, params, x, y, omega, block=256):
        """G @ omega (P x k) = (1/N) J^T (J omega), J from the reference, streamed in row blocks."""
        w, L, a, m = self._m(spec)
        omega = _f64(omega)
        out = np.zeros_like(omega)
        self._call("opg_sketch", w, L, a, m, _f64(params), _f64(x), _f64(y), x.shape[0], omega,
                   omega.shape[1], block, out)
        return out

    def opg_eigs_incremental(self, J, block, k):
        J = _f64(J)
        n, p = J.shape
        q = np.zeros((p, k))
        lam = np.zeros(k)
        self._call("opg_eigs_incremental", J, n, p, block, k, q, lam)
        return lam, q

    def eig_ops(self, q, lam, x=None, lambda_tilde=None, materialize=False, memory_cap=4096):
        """The reference's low-rank (lambda_tilde None) or full-rank operators
        (eigensolve.cpp:278-348): returns (H or None, A x or None, x^T A x or None)."""
        q, lam = _f64(q), _f64(lam)
        p, k = q.shape
        full = lambda_tilde is not None
        h = np.zeros((p, p)) if materialize else None
        xv = _f64(x) if x is not None else None
        y = np.zeros(xv.shape[0]) if xv is not None else None
        quad = C.c_double() if xv is not None else None
        vp = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None  # noqa: E731
        self._call("eig_ops", q, lam, p, k, 1 if full else 0, float(lambda_tilde) if full else 0.0, memory_cap,
                   vp(xv), xv.shape[0] if xv is not None else 0, vp(h), vp(y),
                   C.cast(C.byref(quad), C.c_void_p) if quad is not None else None)
        return h, y, (quad.value if quad is not None else None)

    def validate_eigen_pairs(self, q, lam, ortho_tol=1e-8):
        q, lam = _f64(q), _f64(lam)
        self._call("validate_eigen_pairs", q, q.shape[0], q.shape[1], lam, lam.shape[0], ortho_tol)

    def default_lambda_tilde(self, lam):
        lam = _f64(lam)
        out = C.c_double()
        self._call("default_lambda_tilde", lam, lam.shape[0], C.byref(out))
        return out.value


# ---- numpy restatement of the eigenpair operators (the "port") -----------------
# Pinned against the reference by tests/golden/eigops.npz (tests/test_oracle_pins.py).

def eig_materialize_port(q, lam, lambda_tilde=None):
    """eigensolve.cpp:278-292 (sum_c lambda_c q_c q_c^T) and :309-327
    (minus lambda_tilde q_c q_c^T per column, plus lambda_tilde on the diagonal)."""
    q, lam = _f64(q), _f64(lam)
    h = np.zeros((q.shape[0], q.shape[0]))
    for c in range(q.shape[1]):
        h += lam[c] * np.outer(q[:, c], q[:, c])
    if lambda_tilde is not None:
        for c in range(q.shape[1]):
            h -= lambda_tilde * np.outer(q[:, c], q[:, c])
        h[np.diag_indices_from(h)] += lambda_tilde
    return h


def eig_apply_port(q, lam, x, lambda_tilde=None):
    """(A x, x^T A x): eigensolve.cpp:294-305 (low rank), :329-350 (full rank)."""
    q, lam, x = _f64(q), _f64(lam), _f64(x)
    t = q.T @ x  # project(): eigensolve.cpp:263-269
    y = q @ (lam * t)
    quad = float(np.sum(lam * t * t))
    if lambda_tilde is not None:
        y = y + lambda_tilde * (x - q @ t)
        quad = quad + lambda_tilde * float(x @ x) - lambda_tilde * float(t @ t)
    return y, quad
