"""Host-side mirror of the reference curvkit API for the curvature hot path.

Names, argument meaning and error behaviour follow the reference C++
headers (/root/reference/proj/include/curv/{model,autodiff,curvature,
eigensolve}.hpp) so that code and tests written against the reference read
the same.  Every compute call goes through the C-ABI of
libcurvkit_b200.so; there is no CPU path.

Matrices are numpy float64 arrays (row-major), like the reference's
DenseMatrix.  `precision` selects the device arithmetic: "f64" (default,
the reference's), "f32", "tf32" (tcgen05 tensor cores) or "tf32x3".
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _lib
from .errors import ContractError, ShapeError

PRECISION = {"f64": 0, "f32": 1, "tf32": 2, "tf32x3": 3, "f16s": 4}


class Activation(IntEnum):  # model.hpp:11
    identity = 0
    sigmoid = 1
    tanh = 2
    relu = 3


class OutputMode(IntEnum):  # model.hpp:20
    softmax_cross_entropy = 0
    raw_mean_output = 1


def _enum(e, v):
    if isinstance(v, str):
        try:
            return e[v]
        except KeyError:
            raise ContractError(f"unknown {e.__name__.lower()}: {v}") from None
    return e(v)


@dataclass
class ModelSpec:  # model.hpp:27-42
    layer_widths: list
    hidden_activation: Activation = Activation.tanh
    output_mode: OutputMode = OutputMode.softmax_cross_entropy

    def __post_init__(self):
        self.layer_widths = [int(w) for w in self.layer_widths]
        self.hidden_activation = _enum(Activation, self.hidden_activation)
        self.output_mode = _enum(OutputMode, self.output_mode)

    def num_layers(self):
        return len(self.layer_widths)

    def input_width(self):
        return self.layer_widths[0]

    def output_width(self):
        return self.layer_widths[-1]

    def validate(self):  # model.cpp:80-87
        if len(self.layer_widths) < 2:
            raise ContractError("model needs at least an input and an output layer")
        if any(w < 1 for w in self.layer_widths):
            raise ContractError("layer widths must be >= 1")
        if self.output_mode == OutputMode.raw_mean_output and self.output_width() != 1:
            raise ContractError("raw_mean_output requires an output width of 1")

    def _c(self):
        self.validate()
        w = (C.c_int64 * len(self.layer_widths))(*self.layer_widths)
        m = _lib.Model(len(self.layer_widths), w, int(self.hidden_activation), int(self.output_mode))
        m._keep = w
        return m


@dataclass
class Batch:  # model.hpp:58-64
    x: np.ndarray
    y: np.ndarray = None

    def size(self):
        return self.x.shape[0]


@dataclass
class CurvatureConfig:  # curvature.hpp:11-18
    batch_size_h: int = 1
    batch_size_g: int = 1
    parallelism: int = 1
    memory_cap: int = 4096

    def _c(self):
        return _lib.CurvatureConfig(self.batch_size_h, self.batch_size_g, self.parallelism, self.memory_cap)


@dataclass
class HessianResult:  # curvature.hpp:20-23
    h: np.ndarray
    asymmetry: float = 0.0


@dataclass
class GradResult:  # autodiff.hpp:14-17
    grad_total: np.ndarray
    n: int = 0


@dataclass
class EigenPairs:  # eigensolve.hpp:14-17
    q: np.ndarray
    lam: np.ndarray = field(default=None)

    @property
    def lambda_(self):
        return self.lam


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise ShapeError(f"expected shape {shape}, got {a.shape}")
    return a


def _p(a):
    return a.ctypes.data_as(_lib.dptr) if a is not None else None


def _prec(p):
    if p not in PRECISION:
        raise ContractError(f"unknown precision {p!r}; use one of {sorted(PRECISION)}")
    return PRECISION[p]


def param_count(spec: ModelSpec) -> int:  # model.cpp:89-95
    out = C.c_int64()
    _lib.check(_lib.load().curvkit_param_count(C.byref(spec._c()), C.byref(out)))
    return out.value


def weight_block_offset(spec: ModelSpec, k: int) -> int:  # model.cpp:142-147
    w = spec.layer_widths
    return sum(w[i] * w[i + 1] + w[i + 1] for i in range(k))


def bias_block_offset(spec: ModelSpec, k: int) -> int:  # model.cpp:149-151
    w = spec.layer_widths
    return weight_block_offset(spec, k) + w[k] * w[k + 1]


def flatten_params(weights, biases) -> np.ndarray:  # model.cpp:97-119
    if len(weights) != len(biases) or not weights:
        raise ShapeError("flatten_params: need one bias per weight matrix")
    parts = []
    for k, (w, b) in enumerate(zip(weights, biases)):
        w = np.asarray(w, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64).reshape(-1)
        if w.shape[0] != b.shape[0]:
            raise ShapeError("flatten_params: bias length does not match weight rows")
        if k + 1 < len(weights) and np.asarray(weights[k + 1]).shape[1] != w.shape[0]:
            raise ShapeError("flatten_params: consecutive layer shapes do not chain")
        parts += [w.reshape(-1), b]
    return np.concatenate(parts)


def unflatten_params(spec: ModelSpec, params):  # model.cpp:121-140
    p = param_count(spec)
    params = np.asarray(params, dtype=np.float64).reshape(-1)
    if params.shape[0] != p:
        raise ShapeError(f"unflatten_params: parameter vector has length {params.shape[0]}, model needs {p}")
    w = spec.layer_widths
    weights, biases, at = [], [], 0
    for k in range(len(w) - 1):
        weights.append(params[at:at + w[k] * w[k + 1]].reshape(w[k + 1], w[k]).copy())
        at += w[k] * w[k + 1]
        biases.append(params[at:at + w[k + 1]].copy())
        at += w[k + 1]
    return weights, biases


def _inputs(spec: ModelSpec, params, batch: Batch):
    spec.validate()
    P = param_count(spec)
    params = _f64(params).reshape(-1)
    if params.shape[0] != P:
        raise ShapeError(f"parameter vector has length {params.shape[0]}, model needs {P}")
    x = _f64(batch.x)
    if x.ndim != 2 or x.shape[1] != spec.input_width():
        raise ShapeError(f"input width {x.shape[-1]} does not match model input {spec.input_width()}")
    n = x.shape[0]
    y = None
    if spec.output_mode == OutputMode.softmax_cross_entropy:
        y = _f64(batch.y)
        if y.shape != (n, spec.output_width()):
            raise ShapeError("target shape does not match model output")
    return P, params, x, y, n


def forward(spec: ModelSpec, params, x, precision: str = "f64") -> np.ndarray:
    """curv::forward (model.hpp:80): the network output (softmax
    probabilities, or the raw output).  x: one example (T_1,) as in the
    reference, or a batch (n, T_1) -> (n, T_L)."""
    spec.validate()
    params = _f64(params).reshape(-1)
    if params.shape[0] != param_count(spec):
        raise ShapeError(f"parameter vector has length {params.shape[0]}, model needs {param_count(spec)}")
    x = _f64(x)
    single = x.ndim == 1
    xb = x.reshape(1, -1) if single else x
    if xb.ndim != 2 or xb.shape[1] != spec.input_width():
        raise ShapeError(f"forward: input has length {xb.shape[-1]}, model expects {spec.input_width()}")
    out = np.empty((xb.shape[0], spec.output_width()))
    _lib.check(_lib.load().curvkit_forward(C.byref(spec._c()), _p(params), _p(xb), xb.shape[0], _prec(precision),
                                            _p(out)))
    return out[0] if single else out


def cost(spec: ModelSpec, params, batch: Batch, precision: str = "f64") -> float:
    """curv::cost (model.hpp:84): mean cross-entropy (fused log-softmax) or
    mean raw output over the batch."""
    P, params, x, y, n = _inputs(spec, params, batch)
    out = C.c_double()
    _lib.check(_lib.load().curvkit_cost(C.byref(spec._c()), _p(params), _p(x), None if y is None else _p(y), n,
                                         _prec(precision), C.byref(out)))
    return out.value


def assemble_jacobian(spec: ModelSpec, params, batch: Batch, precision: str = "f64") -> np.ndarray:
    """curvature.hpp:35-36: N x P, row n = gradient of C_n."""
    P, params, x, y, n = _inputs(spec, params, batch)
    out = np.empty((n, P))
    _lib.check(_lib.load().curvkit_assemble_jacobian(C.byref(spec._c()), _p(params), _p(x), _p(y), n,
                                                      _prec(precision), _p(out)))
    return out


def grad_batch(spec: ModelSpec, params, batch: Batch, precision: str = "f64") -> GradResult:
    """autodiff.hpp:54: sum of per-example gradients in one batched pass."""
    P, params, x, y, n = _inputs(spec, params, batch)
    out = np.empty(P)
    _lib.check(_lib.load().curvkit_grad_batch(C.byref(spec._c()), _p(params), _p(x), _p(y), n,
                                               _prec(precision), _p(out)))
    return GradResult(out, n)


def per_example_grad(spec: ModelSpec, params, x, y=None, precision: str = "f64") -> np.ndarray:
    """autodiff.hpp:49-50."""
    x = _f64(x).reshape(1, -1)
    y = None if y is None else _f64(y).reshape(1, -1)
    return grad_batch(spec, params, Batch(x, y), precision).grad_total


def hvp(spec: ModelSpec, params, batch: Batch, v, precision: str = "f64") -> np.ndarray:
    """autodiff.hpp:60-65: H_batch v (v may be P or nvec x P)."""
    P, params, x, y, n = _inputs(spec, params, batch)
    v = _f64(v)
    single = v.ndim == 1
    V = v.reshape(1, -1) if single else v
    if V.shape[1] != P:
        raise ShapeError(f"hvp: direction has length {V.shape[1]}, model has {P} parameters")
    out = np.empty_like(V)
    _lib.check(_lib.load().curvkit_hvp(C.byref(spec._c()), _p(params), _p(x), _p(y), n, _p(V), V.shape[0],
                                        _prec(precision), _p(out)))
    return out[0] if single else out


class HvpOperator:
    """autodiff.hpp:70-84: v -> Hv over a fixed dataset with equal mini-batches."""

    def __init__(self, spec: ModelSpec, params, data: Batch, batch_size: int, precision: str = "f64"):
        self.spec, self.data, self.batch_size, self.precision = spec, data, int(batch_size), precision
        self.p, self.params, self.x, self.y, self.n = _inputs(spec, params, data)
        if self.batch_size < 1:
            raise ContractError("HvpOperator: batch size must be >= 1")
        if self.n == 0:
            raise ContractError("HvpOperator: empty dataset")
        if self.n % self.batch_size != 0:
            raise ContractError(f"HvpOperator: dataset size {self.n} is not divisible by batch size "
                                f"{self.batch_size}; refusing to drop the remainder")

    def dim(self):
        return self.p

    def num_batches(self):
        return self.n // self.batch_size

    def apply(self, v):
        v = _f64(v)
        single = v.ndim == 1
        V = v.reshape(1, -1) if single else v
        if V.shape[1] != self.p:
            raise ShapeError(f"hvp: direction has length {V.shape[1]}, model has {self.p} parameters")
        out = np.empty_like(V)
        _lib.check(_lib.load().curvkit_hvp_operator_apply(
            C.byref(self.spec._c()), _p(self.params), _p(self.x), _p(self.y), self.n, self.batch_size, _p(V),
            V.shape[0], _prec(self.precision), _p(out)))
        return out[0] if single else out


def assemble_hessian(spec: ModelSpec, params, dataset: Batch, config: CurvatureConfig = None,
                     precision: str = "f64", verify: bool = True) -> HessianResult:
    """curvature.hpp:25-32.  verify=True assembles each diagonal layer block
    from both triangles and reports the pre-symmetrization asymmetry like the
    reference; verify=False fills the lower triangle and mirrors it."""
    config = config or CurvatureConfig(batch_size_h=max(1, Batch(dataset.x).size()))
    P, params, x, y, n = _inputs(spec, params, dataset)
    h = np.empty((P, P))
    asym = C.c_double(0.0)
    cfg = config._c()
    _lib.check(_lib.load().curvkit_assemble_hessian(C.byref(spec._c()), _p(params), _p(x), _p(y), n, C.byref(cfg),
                                                     _prec(precision), int(verify), _p(h), C.byref(asym)))
    return HessianResult(h, asym.value)


def assemble_opg(spec: ModelSpec, params, dataset: Batch, config: CurvatureConfig = None,
                 precision: str = "f64") -> np.ndarray:
    """curvature.hpp:37-42: (1/N) J^T J, symmetric PSD."""
    config = config or CurvatureConfig(batch_size_g=max(1, Batch(dataset.x).size()))
    P, params, x, y, n = _inputs(spec, params, dataset)
    g = np.empty((P, P))
    cfg = config._c()
    _lib.check(_lib.load().curvkit_assemble_opg(C.byref(spec._c()), _p(params), _p(x), _p(y), n, C.byref(cfg),
                                                 _prec(precision), _p(g)))
    return g


def opg_eigs(spec: ModelSpec, params, dataset: Batch, k: int, oversample: int = 20, power_iters: int = None,
             seed: int = 0, precision: str = "f64", filter_steps: int = 0, filter_degree: int = 0,
             tol: float = 1e-4, max_applications: int = 96) -> EigenPairs:
    """Top-k eigenpairs of G = (1/N) J^T J without forming G (replaces
    eigensolve.hpp:80-81 opg_eigs_incremental).  Eigenvalues descending,
    columns of q orthonormal eigenvectors.

    Default: Chebyshev-filtered subspace iteration stopped once every Ritz
    value has converged to `tol` (curvkit_opg_topk_auto; tol = 1e-4 holds the
    1e-3 eigenvalue bar).  power_iters = p runs the plain randomized range
    finder with p power iterations instead (BASELINE config 4 quotes p = 2,
    which on a flat spectrum leaves the Ritz values ~10% low: DESIGN.md
    section 5); filter_degree > 0 runs filter_steps fixed rounds."""
    P, params, x, y, n = _inputs(spec, params, dataset)
    q = np.empty((P, k))
    lam = np.empty(k)
    lib = _lib.load()
    if filter_degree > 0:
        _lib.check(lib.curvkit_opg_topk_filtered(C.byref(spec._c()), _p(params), _p(x), _p(y), n, int(k),
                                                 int(oversample), int(filter_steps), int(filter_degree),
                                                 int(seed), _prec(precision), _p(q), _p(lam)))
    elif power_iters is not None:
        _lib.check(lib.curvkit_opg_topk(C.byref(spec._c()), _p(params), _p(x), _p(y), n, int(k),
                                        int(oversample), int(power_iters), int(seed), _prec(precision),
                                        _p(q), _p(lam)))
    else:
        _lib.check(lib.curvkit_opg_topk_auto(C.byref(spec._c()), _p(params), _p(x), _p(y), n, int(k),
                                             int(oversample), float(tol), int(max_applications), int(seed),
                                             _prec(precision), _p(q), _p(lam)))
    return EigenPairs(q, lam)


@dataclass
class LanczosConfig:  # eigensolve.hpp:22-27
    k: int = 1
    max_iterations: int = 0
    residual_tol: float = 1e-6
    seed: int = 0


@dataclass
class LanczosResult:  # eigensolve.hpp:29-33
    pairs: EigenPairs
    residuals: np.ndarray
    iterations: int


def hessian_lanczos_topk(spec: ModelSpec, params, dataset: Batch, batch_size: int, cfg: LanczosConfig,
                         precision: str = "f64") -> LanczosResult:
    """curv::lanczos_topk (eigensolve.hpp:36-45) applied to HvpOperator(spec,
    params, dataset, batch_size): the k algebraically largest eigenpairs of
    the Hessian, full reorthogonalisation, Krylov basis on the device.
    Raises ConvergenceError (best residual estimates attached) when the
    tolerance is not met within cfg.max_iterations."""
    from .errors import ConvergenceError
    P, params, x, y, n = _inputs(spec, params, dataset)
    k = int(cfg.k)
    q = np.empty((P, max(k, 1)))
    lam = np.empty(max(k, 1))
    res = np.zeros(max(k, 1))
    it = C.c_int64(0)
    rc = _lib.load().curvkit_hessian_topk_lanczos(C.byref(spec._c()), _p(params), _p(x), _p(y), n, int(batch_size), k,
                                                   int(cfg.max_iterations), float(cfg.residual_tol), int(cfg.seed),
                                                   _prec(precision), _p(q), _p(lam), _p(res), C.byref(it))
    if rc == 4:
        raise ConvergenceError(_lib.load().curvkit_last_error().decode(), res[:k].tolist())
    _lib.check(rc)
    return LanczosResult(EigenPairs(q, lam), res, int(it.value))


def opg_eigs_incremental(j_blocks, n_total: int, k: int, oversample: int = 20, power_iters: int = 2, seed: int = 0,
                         precision: str = "f64") -> EigenPairs:
    """Top-k eigenpairs of G = (1/n) J^T J from the caller's row blocks of J --
    the input contract of curv::opg_eigs_incremental (eigensolve.hpp:80-81,
    eigensolve.cpp:245-251) -- by the device randomized range finder."""
    blocks = [np.ascontiguousarray(b, dtype=np.float64) for b in j_blocks]
    if not blocks:
        raise ContractError("opg_eigs_incremental: no row blocks")
    p = blocks[0].shape[1]
    if any(b.ndim != 2 or b.shape[1] != p or b.shape[0] < 1 for b in blocks):
        raise ShapeError("opg_eigs_incremental: blocks must be b x P with b >= 1")
    J = np.concatenate(blocks, axis=0)
    if J.shape[0] != int(n_total):
        raise ContractError("opg_eigs_incremental: n_total does not match the rows pushed")
    q = np.empty((p, k))
    lam = np.empty(k)
    _lib.check(_lib.load().curvkit_opg_topk_from_jacobian(_p(J), J.shape[0], p, int(k), int(oversample),
                                                           int(power_iters), int(seed), _prec(precision), _p(q),
                                                           _p(lam)))
    return EigenPairs(q, lam)


class IncrementalOpgEigs:
    """curv::IncrementalOpgEigs (eigensolve.hpp:52-78): streaming eigenpairs of
    G = (1/N) J^T J from row blocks of J, with the reference's algorithm and
    update windows; the factorisations run on the device in fp64
    (curvkit_incr_opg_*).  push_block takes b x P float64 rows (numpy, or a
    CUDA torch tensor); finalize(n_total) returns EigenPairs."""

    def __init__(self, p: int, k: int):
        self.p, self.k = int(p), int(k)
        h = C.c_void_p()
        _lib.check(_lib.load().curvkit_incr_opg_create(self.p, self.k, C.byref(h)))
        self._h = h

    def push_block(self, block) -> None:
        if hasattr(block, "data_ptr") and getattr(block, "is_cuda", False):
            if block.dim() != 2 or block.shape[1] != self.p or block.dtype.itemsize != 8 or block.stride(1) != 1:
                raise ShapeError(f"IncrementalOpgEigs: block must be b x {self.p} float64 with unit column stride")
            _lib.check(_lib.load().curvkit_incr_opg_dev_push_block(self._h, block.data_ptr(), block.shape[0],
                                                                   block.stride(0), None))
            return
        b = np.ascontiguousarray(block, dtype=np.float64)
        if b.ndim != 2 or b.shape[1] != self.p:
            raise ShapeError(f"IncrementalOpgEigs: block has {b.shape[-1] if b.ndim else 0} columns, "
                             f"expected {self.p}")
        _lib.check(_lib.load().curvkit_incr_opg_push_block(self._h, _p(b), b.shape[0]))

    def _counts(self):
        r, u = C.c_int64(0), C.c_int64(0)
        _lib.check(_lib.load().curvkit_incr_opg_counts(self._h, C.byref(r), C.byref(u)))
        return int(r.value), int(u.value)

    def rows_seen(self) -> int:
        return self._counts()[0]

    def updates(self) -> int:
        return self._counts()[1]

    def finalize(self, n_total: int) -> EigenPairs:
        q = np.empty((self.p, self.k))
        lam = np.empty(self.k)
        _lib.check(_lib.load().curvkit_incr_opg_finalize(self._h, int(n_total), _p(q), _p(lam)))
        return EigenPairs(q, lam)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().curvkit_incr_opg_destroy(h)
            except Exception:  # noqa: BLE001 -- interpreter teardown
                pass
            self._h = None


def dev_opg_topk_from_jacobian(J, ldj, n, p, k, oversample, power_iters, seed, q, lam, precision="tf32",
                               stream=None):
    _lib.check(_lib.load().curvkit_dev_opg_topk_from_jacobian(_ptr(J), ldj, n, p, k, oversample, power_iters, seed,
                                                               _prec(precision), _ptr(q), _ptr(lam),
                                                               _stream(stream)))


# ---- low/full-rank operators from eigenpairs (eigensolve.hpp:83-101) -----------
# All of them run on the device through the C-ABI (curvkit_eig_*): the Gram of
# validate, the symmetric GEMM of materialize, the two passes over Q of
# apply / quadform.  Shape and contract errors are raised by the library with the
# reference's text (eigensolve.cpp:11-30, 255-275).

def _pairs(pairs: EigenPairs):
    q = np.ascontiguousarray(pairs.q, dtype=np.float64)
    lam = np.ascontiguousarray(pairs.lam, dtype=np.float64).reshape(-1)
    if q.ndim != 2:
        raise ShapeError("EigenPairs: q must be a P x K matrix")
    return q, lam


def validate_eigen_pairs(pairs: EigenPairs, ortho_tol: float = 1e-8) -> None:
    """curv::validate_eigen_pairs (eigensolve.cpp:11-30): lambda length,
    descending order and column orthonormality within ortho_tol."""
    q, lam = _pairs(pairs)
    p, k = q.shape
    _lib.check(_lib.load().curvkit_eig_validate(p, k, _p(q), _p(lam), lam.shape[0], float(ortho_tol)))


def _materialize(pairs, full, lambda_tilde, memory_cap, precision):
    q, lam = _pairs(pairs)
    p, k = q.shape
    if lam.shape[0] != k:
        raise ShapeError("EigenPairs: lambda length does not match column count")
    # the dense-cap refusal comes first in the library; allocate only when it will pass
    out = np.empty((p, p) if p <= memory_cap and (not full or lambda_tilde > 0.0) else (0, 0), dtype=np.float64)
    _lib.check(_lib.load().curvkit_eig_materialize(p, k, _p(q), _p(lam), 1 if full else 0, float(lambda_tilde),
                                                   int(memory_cap), _prec(precision), _p(out)))
    return out


def low_rank_materialize(pairs: EigenPairs, memory_cap: int = 4096, precision: str = "f64") -> np.ndarray:
    """curv::low_rank_materialize (eigensolve.cpp:278-292): Q diag(lambda) Q^T."""
    return _materialize(pairs, False, 0.0, memory_cap, precision)


def full_rank_materialize(pairs: EigenPairs, lambda_tilde: float, memory_cap: int = 4096,
                          precision: str = "f64") -> np.ndarray:
    """curv::full_rank_materialize (eigensolve.cpp:309-327):
    Q diag(lambda) Q^T + lambda_tilde (I - Q Q^T)."""
    return _materialize(pairs, True, lambda_tilde, memory_cap, precision)


def eig_apply(pairs: EigenPairs, x, lambda_tilde: float = None, want_y: bool = True, want_quad: bool = True,
              precision: str = "f64"):
    """Batched form of the four implicit operators: x is one vector (P) or a
    stack (nvec x P); returns (A x, x^T A x) with A the low-rank operator
    (lambda_tilde None) or its full-rank extension."""
    q, lam = _pairs(pairs)
    p, k = q.shape
    if lam.shape[0] != k:
        raise ShapeError("EigenPairs: lambda length does not match column count")
    xs = np.ascontiguousarray(x, dtype=np.float64)
    single = xs.ndim == 1
    xs = xs.reshape(1, -1) if single else xs
    nvec, xlen = xs.shape
    full = lambda_tilde is not None
    ok = xlen == p and (not full or lambda_tilde > 0.0)
    y = np.empty((nvec, p), dtype=np.float64) if want_y and ok else None
    quad = np.empty(nvec, dtype=np.float64) if want_quad and ok else None
    _lib.check(_lib.load().curvkit_eig_apply(p, k, _p(q), _p(lam), 1 if full else 0,
                                             float(lambda_tilde) if full else 0.0, nvec, _p(xs), xlen,
                                             _prec(precision), _p(y), _p(quad)))
    if single:
        return (y[0] if y is not None else None), (float(quad[0]) if quad is not None else None)
    return y, quad


def low_rank_quadform(pairs: EigenPairs, x, precision: str = "f64") -> float:
    """curv::low_rank_quadform (eigensolve.cpp:294-299)."""
    return eig_apply(pairs, x, None, want_y=False, precision=precision)[1]


def low_rank_apply(pairs: EigenPairs, x, precision: str = "f64") -> np.ndarray:
    """curv::low_rank_apply (eigensolve.cpp:301-305)."""
    return eig_apply(pairs, x, None, want_quad=False, precision=precision)[0]


def default_lambda_tilde(pairs: EigenPairs) -> float:  # eigensolve.cpp:350-358
    if len(pairs.lam) == 0:
        raise ContractError("default_lambda_tilde: no eigenvalues")
    lk = float(pairs.lam[-1])
    if not lk > 0.0:
        raise ContractError(f"default_lambda_tilde: smallest retained eigenvalue {lk} is not positive; "
                            "pass an explicit lambda_tilde")
    return lk


def full_rank_quadform(pairs: EigenPairs, lambda_tilde: float, x, precision: str = "f64") -> float:
    """curv::full_rank_quadform (eigensolve.cpp:329-339)."""
    return eig_apply(pairs, x, float(lambda_tilde), want_y=False, precision=precision)[1]


def full_rank_apply(pairs: EigenPairs, lambda_tilde: float, x, precision: str = "f64") -> np.ndarray:
    """curv::full_rank_apply (eigensolve.cpp:341-350)."""
    return eig_apply(pairs, x, float(lambda_tilde), want_quad=False, precision=precision)[0]


# ---- device-resident entry points (torch tensors or raw pointers) -------------

def _ptr(t):
    return C.c_void_p(t if isinstance(t, int) else t.data_ptr())


def _stream(stream):
    if stream is None:
        return C.c_void_p(0)
    return C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)


def dev_assemble_hessian(spec, params, x, labels, n, out, ldh, precision="tf32", stream=None):
    _lib.check(_lib.load().curvkit_dev_assemble_hessian(C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n,
                                                         _prec(precision), _ptr(out), ldh, _stream(stream)))


def dev_assemble_opg(spec, params, x, labels, n, out, ldg, precision="tf32", stream=None):
    _lib.check(_lib.load().curvkit_dev_assemble_opg(C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n,
                                                     _prec(precision), _ptr(out), ldg, _stream(stream)))


def dev_assemble_jacobian(spec, params, x, labels, n, out, ldj, precision="tf32", stream=None):
    _lib.check(_lib.load().curvkit_dev_assemble_jacobian(C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels),
                                                          n, _prec(precision), _ptr(out), ldj, _stream(stream)))


def dev_opg_topk(spec, params, x, labels, n, k, oversample, power_iters, seed, q, lam, precision="tf32",
                 stream=None):
    _lib.check(_lib.load().curvkit_dev_opg_topk(C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n, k,
                                                 oversample, power_iters, seed, _prec(precision), _ptr(q), _ptr(lam),
                                                 _stream(stream)))


def dev_opg_topk_filtered(spec, params, x, labels, n, k, oversample, filter_steps, filter_degree, seed, q, lam,
                          precision="tf32", stream=None):
    """Top-k of G by Chebyshev-filtered subspace iteration (curvkit_dev_opg_topk_filtered):
    filter_steps rounds of a degree-filter_degree filter instead of power iterations."""
    _lib.check(_lib.load().curvkit_dev_opg_topk_filtered(C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n,
                                                          k, oversample, filter_steps, filter_degree, seed,
                                                          _prec(precision), _ptr(q), _ptr(lam), _stream(stream)))


def launch_count() -> int:
    return int(_lib.load().curvkit_launch_count())


def profile_begin():
    """Start CUDA-event timing of the library's hot kernels."""
    _lib.check(_lib.load().curvkit_profile_begin())


def profile_end() -> dict:
    """Stop timing; {region: {ms, launches, flops, bytes}} summed over the window."""
    import json
    buf = C.create_string_buffer(1 << 16)
    _lib.check(_lib.load().curvkit_profile_end(buf, len(buf)))
    return json.loads(buf.value.decode())


def dev_gemm(m, n, k, a, lda, a_kmajor, b, ldb, b_kmajor, c, ldc, alpha=1.0, precision="tf32", stream=None):
    """The curvature GEMM engine on device fp32 buffers (C = alpha A B^T)."""
    _lib.check(_lib.load().curvkit_dev_gemm(m, n, k, _ptr(a), lda, int(a_kmajor), _ptr(b), ldb, int(b_kmajor),
                                             _ptr(c), ldc, float(alpha), _prec(precision), _stream(stream)))


# ---- unit bands: multi-GPU H and G (bands.cuh) ------------

PRODUCT = {"hessian": 0, "opg": 1}


def shard_units(spec: ModelSpec, nshards: int, shard: int):
    """(unit_begin, unit_end, band_rows): the output units [unit_begin[k],
    unit_end[k]) of every layer k owned by `shard`, and its band's row count."""
    S = len(spec.layer_widths) - 1
    u0, u1, rows = (C.c_int64 * S)(), (C.c_int64 * S)(), C.c_int64()
    _lib.check(_lib.load().curvkit_shard_units(C.byref(spec._c()), nshards, shard, u0, u1, C.byref(rows)))
    return list(u0), list(u1), rows.value


def shard_units_rows(spec: ModelSpec, nshards: int, shard: int) -> int:
    return shard_units(spec, nshards, shard)[2]


def band_rows_index(spec: ModelSpec, nshards: int, shard: int) -> np.ndarray:
    """Global row of every band row (weights of the units, then their biases, per layer)."""
    u0, u1, _ = shard_units(spec, nshards, shard)
    w = spec.layer_widths
    out = []
    for k in range(len(w) - 1):
        wo, bo = weight_block_offset(spec, k), bias_block_offset(spec, k)
        out.append(np.arange(wo + u0[k] * w[k], wo + u1[k] * w[k]))
        out.append(np.arange(bo + u0[k], bo + u1[k]))
    return np.concatenate(out).astype(np.int64)


def unit_ids(spec: ModelSpec) -> np.ndarray:
    """Unit of every parameter row in the unit-major order (layers, then units)."""
    w = spec.layer_widths
    out, base = [], 0
    for k in range(len(w) - 1):
        out.append(base + np.repeat(np.arange(w[k + 1]), w[k]))
        out.append(base + np.arange(w[k + 1]))
        base += w[k + 1]
    return np.concatenate(out)


def dev_assemble_band(spec, product, params, x, labels, n, nshards, shard, band, ld, precision="tf32", stream=None):
    """This shard's unit band of H (product "hessian") or G ("opg")."""
    p = PRODUCT[product] if isinstance(product, str) else int(product)
    _lib.check(_lib.load().curvkit_dev_assemble_band(C.byref(spec._c()), p, _ptr(params), _ptr(x), _ptr(labels), n,
                                                      _prec(precision), nshards, shard, _ptr(band), ld,
                                                      _stream(stream)))


def dev_band_scatter(spec, nshards, shard, band, ld, full, ldf, precision="tf32", stream=None):
    _lib.check(_lib.load().curvkit_dev_band_scatter(C.byref(spec._c()), _prec(precision), nshards, shard, _ptr(band),
                                                     ld, _ptr(full), ldf, _stream(stream)))


def dev_symmetrize_units(spec, full, ldf, precision="tf32", stream=None):
    _lib.check(_lib.load().curvkit_dev_symmetrize_units(C.byref(spec._c()), _prec(precision), _ptr(full), ldf,
                                                         _stream(stream)))


def dev_gather_bands(spec, band, ld, full, ldf, comm, precision="tf32", stream=None):
    """Final gather: every rank's band to rank 0, assembled into the full
    symmetric matrix there (full may be None on other ranks)."""
    _lib.check(_lib.load().curvkit_dev_gather_bands(C.byref(spec._c()), _prec(precision), _ptr(band), ld,
                                                     C.c_void_p(0) if full is None else _ptr(full), ldf,
                                                     _stream(stream), comm.handle))


# ---- multi-GPU top-k (parameter-row shards, NCCL all-reduce of J X) --------

def topk_shard_rows(spec: ModelSpec, nshards: int, shard: int):
    """Parameter rows [begin, end) owned by `shard` in the sharded top-k solver
    (whole output-unit weight blocks and 4-aligned bias blocks, balanced by
    parameter count)."""
    b, e = C.c_int64(), C.c_int64()
    _lib.check(_lib.load().curvkit_topk_shard_rows(C.byref(spec._c()), nshards, shard, C.byref(b), C.byref(e)))
    return b.value, e.value


class Comm:
    """One rank of an NCCL communicator owned by the library.  Build it with
    `Comm.create(rank, world, broadcast)` where `broadcast(bytes) -> bytes`
    ships rank 0's 128-byte id to every rank (e.g. over torch.distributed)."""

    def __init__(self, handle, rank: int, world: int):
        self.handle, self.rank, self.world = handle, rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _lib.check(_lib.load().curvkit_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def create(cls, rank: int, world: int, broadcast):
        uid = broadcast(cls.unique_id() if rank == 0 else None)
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _lib.check(_lib.load().curvkit_comm_init(buf, world, rank, C.byref(h)))
        return cls(h, rank, world)

    @classmethod
    def create_host(cls, rank: int, world: int, group=None):
        """A communicator whose exchanges run over torch.distributed on host
        memory (e.g. the gloo backend) -- for ranks NCCL cannot serve, such as
        several processes sharing one GPU."""
        import torch
        import torch.distributed as dist

        def allreduce(buf, count, dtype, user):
            try:
                npt = np.float64 if dtype == 1 else np.float32
                a = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_double if dtype == 1 else C.c_float)),
                                          shape=(count,))
                t = torch.from_numpy(a)
                dist.all_reduce(t, group=group)
                del npt
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def gather(send, send_bytes, recv, recv_bytes, root, user):
            try:
                sizes = [int(recv_bytes[r]) for r in range(world)]
                mx = max(max(sizes), 1)
                t = torch.zeros(mx, dtype=torch.uint8)
                if send_bytes > 0:  # a view of the library's host buffer (no bytes copy)
                    t[:send_bytes] = torch.from_numpy(
                        np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(int(send_bytes),)))
                lst = [torch.empty(mx, dtype=torch.uint8) for _ in range(world)] if rank == root else None
                dist.gather(t, lst, dst=root, group=group)
                if rank == root:
                    off = 0
                    for r in range(world):
                        if sizes[r] > 0:
                            C.memmove(recv + off, lst[r].numpy().ctypes.data, sizes[r])
                        off += sizes[r]
                return 0
            except Exception:  # noqa: BLE001
                return 1

        ar = _lib.HOST_ALLREDUCE(allreduce)
        ga = _lib.HOST_GATHER(gather)
        h = C.c_void_p()
        _lib.check(_lib.load().curvkit_comm_init_host(world, rank, C.cast(ar, C.c_void_p), C.cast(ga, C.c_void_p),
                                                       None, C.byref(h)))
        c = cls(h, rank, world)
        c._keep = (ar, ga)  # the callbacks live as long as the communicator
        return c

    def close(self):
        if self.handle is not None:
            _lib.check(_lib.load().curvkit_comm_destroy(self.handle))
            self.handle = None


def dev_opg_topk_sharded(spec, params, x, labels, n, k, oversample, power_iters, seed, q, lam, comm: Comm,
                         precision="tf32", stream=None):
    """Top-k eigenpairs of G with the parameter rows sharded over comm's ranks:
    q receives this rank's rows (topk_shard_rows) x k, lam all k values."""
    _lib.check(_lib.load().curvkit_dev_opg_topk_sharded(C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n, k,
                                                         oversample, power_iters, seed, _prec(precision), _ptr(q),
                                                         _ptr(lam), _stream(stream), comm.handle))


def dev_opg_topk_sharded_filtered(spec, params, x, labels, n, k, oversample, filter_steps, filter_degree, seed, q, lam,
                                  comm: Comm, precision="tf32", stream=None):
    """dev_opg_topk_sharded with the Chebyshev filter of dev_opg_topk_filtered."""
    _lib.check(_lib.load().curvkit_dev_opg_topk_sharded_filtered(
        C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n, k, oversample, filter_steps, filter_degree, seed,
        _prec(precision), _ptr(q), _ptr(lam), _stream(stream), comm.handle))


def dev_opg_topk_auto(spec, params, x, labels, n, k, oversample, seed, q, lam, tol=1e-4, max_applications=96,
                      precision="tf32", stream=None):
    """Top-k of G to `tol` (curvkit_dev_opg_topk_auto): Chebyshev-filtered
    subspace iteration with the Ritz-convergence stop rule."""
    _lib.check(_lib.load().curvkit_dev_opg_topk_auto(C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n, k,
                                                      oversample, float(tol), int(max_applications), seed,
                                                      _prec(precision), _ptr(q), _ptr(lam), _stream(stream)))


def dev_opg_topk_sharded_auto(spec, params, x, labels, n, k, oversample, seed, q, lam, comm, tol=1e-4,
                              max_applications=96, precision="tf32", stream=None):
    _lib.check(_lib.load().curvkit_dev_opg_topk_sharded_auto(
        C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n, k, oversample, float(tol), int(max_applications),
        seed, _prec(precision), _ptr(q), _ptr(lam), _stream(stream), comm.handle))


def dev_jacobian_apply(spec, params, x, labels, n, p_begin, p_end, inp, ld_in, l, out, ld_out, transpose=False,
                       precision="tf32", stream=None):
    """Matrix-free J[:, p_begin:p_end] @ inp (transpose=False) or its
    transpose, with J never formed (tcgen05 Khatri-Rao kernels; precision
    "tf32" or "f16s")."""
    _lib.check(_lib.load().curvkit_dev_jacobian_apply(C.byref(spec._c()), _ptr(params), _ptr(x), _ptr(labels), n,
                                                       _prec(precision), p_begin, p_end, 1 if transpose else 0,
                                                       _ptr(inp), ld_in, l, _ptr(out), ld_out, _stream(stream)))


def dev_eig_materialize(p, k, q, ldq, lam, out, ldh, lambda_tilde=None, precision="tf32", stream=None):
    """Q diag(lambda) Q^T (lambda_tilde None) or its full-rank extension into the
    device matrix out (p x p, ldh); q, lam, out in the precision's storage type."""
    full = lambda_tilde is not None
    _lib.check(_lib.load().curvkit_dev_eig_materialize(p, k, _ptr(q), ldq, _ptr(lam), 1 if full else 0,
                                                       float(lambda_tilde) if full else 0.0, _prec(precision),
                                                       _ptr(out), ldh, _stream(stream)))


def dev_eig_apply(p, k, q, ldq, lam, nvec, x, ldx, y=None, ldy=0, quad=None, lambda_tilde=None, precision="tf32",
                  stream=None):
    """y[v] = A x[v] and quad[v] = x[v]^T A x[v] (fp64) for nvec device vectors."""
    full = lambda_tilde is not None
    null = C.c_void_p(0)
    _lib.check(_lib.load().curvkit_dev_eig_apply(p, k, _ptr(q), ldq, _ptr(lam), 1 if full else 0,
                                                 float(lambda_tilde) if full else 0.0, nvec, _ptr(x), ldx,
                                                 _ptr(y) if y is not None else null, ldy,
                                                 C.cast(_ptr(quad), _lib.dptr) if quad is not None else None,
                                                 _prec(precision), _stream(stream)))


def dev_eig_apply_sharded(p_local, k, q, ldq, lam, nvec, x, ldx, comm, y=None, ldy=0, quad=None, lambda_tilde=None,
                          precision="tf32", stream=None):
    """dev_eig_apply on this rank's parameter rows (the row shards of the sharded
    top-k solvers): one all-reduce of nvec (k + 1) doubles over comm; quad is the
    whole vector's quadratic form on every rank."""
    full = lambda_tilde is not None
    null = C.c_void_p(0)
    _lib.check(_lib.load().curvkit_dev_eig_apply_sharded(
        p_local, k, _ptr(q) if q is not None else null, ldq, _ptr(lam), 1 if full else 0,
        float(lambda_tilde) if full else 0.0, nvec, _ptr(x) if x is not None else null, ldx,
        _ptr(y) if y is not None else null, ldy, C.cast(_ptr(quad), _lib.dptr) if quad is not None else None,
        _prec(precision), _stream(stream), comm.handle))
