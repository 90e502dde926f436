// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libcurv_ref.so).  Used to pin oracle/curv_oracle.c, to
// generate tests/golden/, and as bench.py's reference CPU arm.  Every entry
// point forwards to the reference's own public API; the two *_sample
// functions replay the reference's own inner loops (curvature.cpp:49-57 and
// curvature.cpp:116-123) over a bounded slice so a CPU baseline can be
// timed on configurations whose full run would take hours.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "curv/autodiff.hpp"
#include "curv/curvature.hpp"
#include "curv/eigensolve.hpp"
#include "curv/errors.hpp"
#include "curv/linalg.hpp"
#include "curv/model.hpp"

using namespace curv;

namespace {
thread_local std::string g_err;

ModelSpec make_spec(const int64_t* w, int L, int act, int mode) {
    ModelSpec s;
    s.layer_widths.assign(w, w + L);
    s.hidden_activation = static_cast<Activation>(act);
    s.output_mode = static_cast<OutputMode>(mode);
    return s;
}

Batch make_batch(const ModelSpec& s, const double* x, const double* y, int64_t n) {
    const std::size_t t1 = s.input_width(), tl = s.output_width();
    Batch b{DenseMatrix(n, t1, std::vector<double>(x, x + n * t1)),
            DenseMatrix(n, tl, y ? std::vector<double>(y, y + n * tl)
                                 : std::vector<double>(n * tl, 0.0))};
    return b;
}

ParamVector make_params(const ModelSpec& s, const double* p) {
    const std::size_t np = param_count(s);
    return ParamVector{DenseVector(std::vector<double>(p, p + np))};
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 1;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 2;
    } catch (const ConvergenceError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int64_t ref_param_count(const int64_t* w, int L) {
    int64_t out = -1;
    guard([&] { out = (int64_t)param_count(make_spec(w, L, 2, 0)); });
    return out;
}

int ref_cost(const int64_t* w, int L, int act, int mode, const double* params, const double* x,
             const double* y, int64_t n, double* out) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        *out = cost(s, make_params(s, params), make_batch(s, x, y, n));
    });
}

int ref_forward(const int64_t* w, int L, int act, int mode, const double* params, const double* x,
                double* out) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        DenseVector xv(std::vector<double>(x, x + s.input_width()));
        DenseVector r = forward(s, make_params(s, params), xv);
        std::memcpy(out, r.data(), sizeof(double) * r.len());
    });
}

int ref_jacobian(const int64_t* w, int L, int act, int mode, const double* params,
                 const double* x, const double* y, int64_t n, double* J) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        DenseMatrix j = assemble_jacobian(s, make_params(s, params), make_batch(s, x, y, n));
        std::memcpy(J, j.data(), sizeof(double) * j.rows() * j.cols());
    });
}

int ref_grad_batch(const int64_t* w, int L, int act, int mode, const double* params,
                   const double* x, const double* y, int64_t n, double* g) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        GradResult r = grad_batch(s, make_params(s, params), make_batch(s, x, y, n));
        std::memcpy(g, r.grad_total.data(), sizeof(double) * r.grad_total.len());
    });
}

int ref_hvp(const int64_t* w, int L, int act, int mode, const double* params, const double* x,
            const double* y, int64_t n, const double* v, double* hv) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        const std::size_t p = param_count(s);
        DenseVector vv(std::vector<double>(v, v + p));
        DenseVector r = hvp(s, make_params(s, params), make_batch(s, x, y, n), vv);
        std::memcpy(hv, r.data(), sizeof(double) * r.len());
    });
}

int ref_hvp_operator_apply(const int64_t* w, int L, int act, int mode, const double* params,
                           const double* x, const double* y, int64_t n, int64_t batch,
                           const double* v, double* hv) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        const std::size_t p = param_count(s);
        HvpOperator op(s, make_params(s, params), make_batch(s, x, y, n), batch);
        DenseVector r = op.apply(DenseVector(std::vector<double>(v, v + p)));
        std::memcpy(hv, r.data(), sizeof(double) * r.len());
    });
}

int ref_hessian(const int64_t* w, int L, int act, int mode, const double* params,
                const double* x, const double* y, int64_t n, int64_t batch, int64_t lanes,
                int64_t memory_cap, double* H, double* asym) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        CurvatureConfig c;
        c.batch_size_h = batch;
        c.parallelism = lanes;
        c.memory_cap = memory_cap;
        HessianResult r = assemble_hessian(s, make_params(s, params), make_batch(s, x, y, n), c);
        std::memcpy(H, r.h.data(), sizeof(double) * r.h.rows() * r.h.cols());
        if (asym) *asym = r.asymmetry;
    });
}

int ref_opg(const int64_t* w, int L, int act, int mode, const double* params, const double* x,
            const double* y, int64_t n, int64_t batch, int64_t memory_cap, double* G) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        CurvatureConfig c;
        c.batch_size_g = batch;
        c.memory_cap = memory_cap;
        DenseMatrix g = assemble_opg(s, make_params(s, params), make_batch(s, x, y, n), c);
        std::memcpy(G, g.data(), sizeof(double) * g.rows() * g.cols());
    });
}

// Bounded sample of assemble_hessian (curvature.cpp:43-72): one mini-batch
// of `n` examples, columns [c0, c1) only, sharded over `lanes` threads the
// same way the reference shards them.  Out is P x (c1 - c0), row-major.
int ref_hessian_columns_sample(const int64_t* w, int L, int act, int mode, const double* params,
                               const double* x, const double* y, int64_t n, int64_t c0,
                               int64_t c1, int64_t lanes, double* out) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        const std::size_t p = param_count(s);
        const LayerParams lp = unflatten_params(s, make_params(s, params));
        const ForwardBackward fb = forward_backward(s, lp, make_batch(s, x, y, n));
        const std::size_t ncols = c1 - c0;
        lanes = std::max<int64_t>(1, lanes);
        std::exception_ptr err;
        std::mutex m;
        auto work = [&](std::size_t lane) {
            try {
                DenseVector e(p, 0.0);
                for (std::size_t col = c0 + lane; col < (std::size_t)c1; col += lanes) {
                    e[col] = 1.0;
                    const DenseVector hv = hvp_from_cache(s, lp, fb, e);
                    e[col] = 0.0;
                    for (std::size_t row = 0; row < p; ++row) out[row * ncols + (col - c0)] = hv[row];
                }
            } catch (...) {
                std::lock_guard<std::mutex> g(m);
                if (!err) err = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (int64_t l = 0; l < lanes; ++l) th.emplace_back(work, l);
        for (auto& t : th) t.join();
        if (err) std::rethrow_exception(err);
    });
}

// Bounded sample of assemble_opg (curvature.cpp:109-124): the Jacobian of
// `n` examples from the reference, then the reference's rank-1 update loop
// restricted to rows [r0, r1) of G, split over `lanes` threads by row.
int ref_opg_rows_sample(const int64_t* w, int L, int act, int mode, const double* params,
                        const double* x, const double* y, int64_t n, int64_t r0, int64_t r1,
                        int64_t lanes, double* out) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        const std::size_t p = param_count(s);
        const DenseMatrix jb = assemble_jacobian(s, make_params(s, params), make_batch(s, x, y, n));
        const double inv_rows = 1.0 / static_cast<double>(jb.rows());
        const std::size_t nr = r1 - r0;
        std::memset(out, 0, sizeof(double) * nr * p);
        lanes = std::max<int64_t>(1, lanes);
        auto work = [&](std::size_t lane) {
            for (std::size_t ex = 0; ex < jb.rows(); ++ex) {
                const double* row = jb.row(ex);
                for (std::size_t i = r0 + lane; i < (std::size_t)r1; i += lanes) {
                    if (row[i] == 0.0) continue;
                    double* grow = out + (i - r0) * p;
                    for (std::size_t j = 0; j < p; ++j) grow[j] += (row[i] * row[j]) * inv_rows;
                }
            }
        };
        std::vector<std::thread> th;
        for (int64_t l = 0; l < lanes; ++l) th.emplace_back(work, l);
        for (auto& t : th) t.join();
    });
}

// The reference's rank-1 update loop of assemble_opg (curvature.cpp:116-123)
// restricted to rows [r0, r1) of G, on a Jacobian the caller already holds
// (n x p, e.g. from ref_jacobian), split over `lanes` threads by row.  The
// CPU arm times this on a bounded row sample; the Jacobian is timed once.
int ref_opg_rows_from_jacobian(const double* J, int64_t n, int64_t p, int64_t r0, int64_t r1, int64_t lanes,
                               double* out) {
    return guard([&] {
        const double inv_rows = 1.0 / static_cast<double>(n);
        const std::size_t nr = r1 - r0;
        std::memset(out, 0, sizeof(double) * nr * p);
        lanes = std::max<int64_t>(1, lanes);
        auto work = [&](std::size_t lane) {
            for (int64_t ex = 0; ex < n; ++ex) {
                const double* row = J + ex * p;
                for (std::size_t i = r0 + lane; i < (std::size_t)r1; i += lanes) {
                    if (row[i] == 0.0) continue;
                    double* grow = out + (i - r0) * p;
                    for (int64_t j = 0; j < p; ++j) grow[j] += (row[i] * row[j]) * inv_rows;
                }
            }
        };
        std::vector<std::thread> th;
        for (int64_t l = 0; l < lanes; ++l) th.emplace_back(work, l);
        for (auto& t : th) t.join();
    });
}

// Sketches of the reference's full matrices without forming them, for
// whole-matrix parity pins at full BASELINE sizes (tests/golden/make_sketch_pins.py):
//   H Omega: column j is the reference HVP of the dataset-averaged cost on
//            omega[:, j] (autodiff.cpp:158-244 through HvpOperator, one
//            mini-batch = the dataset), columns over `lanes` threads;
//   G Omega: (1/N) J^T (J Omega) with J from the reference's assemble_jacobian
//            (curvature.cpp:94-100) on consecutive example blocks of `block`
//            rows, i.e. G = (1/N) J^T J of assemble_opg for equal batches.
// omega and out are P x k row-major.
int ref_hessian_sketch(const int64_t* w, int L, int act, int mode, const double* params, const double* x,
                       const double* y, int64_t n, const double* omega, int64_t k, int64_t lanes, double* out) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        const std::size_t p = param_count(s);
        const HvpOperator op(s, make_params(s, params), make_batch(s, x, y, n), (std::size_t)n);
        lanes = std::max<int64_t>(1, lanes);
        std::exception_ptr err;
        std::mutex m;
        auto work = [&](std::size_t lane) {
            try {
                for (int64_t j = lane; j < k; j += lanes) {
                    DenseVector v(p, 0.0);
                    for (std::size_t r = 0; r < p; ++r) v[r] = omega[r * k + j];
                    const DenseVector hv = op.apply(v);
                    for (std::size_t r = 0; r < p; ++r) out[r * k + j] = hv[r];
                }
            } catch (...) {
                std::lock_guard<std::mutex> g(m);
                if (!err) err = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (int64_t l = 0; l < lanes; ++l) th.emplace_back(work, l);
        for (auto& t : th) t.join();
        if (err) std::rethrow_exception(err);
    });
}

int ref_opg_sketch(const int64_t* w, int L, int act, int mode, const double* params, const double* x,
                   const double* y, int64_t n, const double* omega, int64_t k, int64_t block, double* out) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        const std::size_t p = param_count(s);
        const ParamVector pv = make_params(s, params);
        const Batch data = make_batch(s, x, y, n);
        std::memset(out, 0, sizeof(double) * p * k);
        std::vector<double> t;
        for (int64_t b0 = 0; b0 < n; b0 += block) {
            const int64_t nb = std::min(block, n - b0);
            const DenseMatrix jb = assemble_jacobian(s, pv, slice_batch(data, b0, nb));
            t.assign((std::size_t)nb * k, 0.0);
            for (int64_t e = 0; e < nb; ++e) {  // T = J_b Omega
                const double* row = jb.row(e);
                double* tr = t.data() + e * k;
                for (std::size_t r = 0; r < p; ++r) {
                    if (row[r] == 0.0) continue;
                    const double* om = omega + r * k;
                    for (int64_t j = 0; j < k; ++j) tr[j] += row[r] * om[j];
                }
            }
            for (int64_t e = 0; e < nb; ++e) {  // out += J_b^T T
                const double* row = jb.row(e);
                const double* tr = t.data() + e * k;
                for (std::size_t r = 0; r < p; ++r) {
                    if (row[r] == 0.0) continue;
                    double* o = out + r * k;
                    for (int64_t j = 0; j < k; ++j) o[j] += row[r] * tr[j];
                }
            }
        }
        const double inv = 1.0 / static_cast<double>(n);
        for (std::size_t i = 0; i < p * (std::size_t)k; ++i) out[i] *= inv;
    });
}

int ref_sym_eig(const double* a, int64_t n, double* vals, double* vecs) {
    return guard([&] {
        SymEig e = sym_eig(DenseMatrix(n, n, std::vector<double>(a, a + n * n)));
        std::memcpy(vals, e.values.data(), sizeof(double) * n);
        std::memcpy(vecs, e.vectors.data(), sizeof(double) * n * n);
    });
}

// opg_eigs_incremental over row blocks of J (eigensolve.cpp:245-251).
int ref_opg_eigs_incremental(const double* J, int64_t n, int64_t p, int64_t block, int64_t k,
                             double* q, double* lambda) {
    return guard([&] {
        std::vector<DenseMatrix> blocks;
        for (int64_t r = 0; r < n; r += block) {
            const int64_t b = std::min(block, n - r);
            blocks.emplace_back(b, p, std::vector<double>(J + r * p, J + (r + b) * p));
        }
        EigenPairs e = opg_eigs_incremental(blocks, n, k);
        std::memcpy(q, e.q.data(), sizeof(double) * e.q.rows() * e.q.cols());
        std::memcpy(lambda, e.lambda.data(), sizeof(double) * e.lambda.len());
    });
}

// lanczos_topk (eigensolve.cpp:46-156) on the HvpOperator of the data
// (autodiff.hpp:70-84).  rc 4 (ConvergenceError): residuals receive the
// best residuals the reference attaches.
int ref_hessian_lanczos(const int64_t* w, int L, int act, int mode, const double* params, const double* x,
                        const double* y, int64_t n, int64_t batch, int64_t k, int64_t max_iterations,
                        double residual_tol, uint64_t seed, double* q, double* lambda, double* residuals,
                        int64_t* iterations) {
    return guard([&] {
        ModelSpec s = make_spec(w, L, act, mode);
        const std::size_t p = param_count(s);
        HvpOperator op(s, make_params(s, params), make_batch(s, x, y, n), batch);
        LanczosConfig cfg;
        cfg.k = (std::size_t)k;
        cfg.max_iterations = (std::size_t)max_iterations;
        cfg.residual_tol = residual_tol;
        cfg.seed = seed;
        try {
            LanczosResult r = lanczos_topk([&](const DenseVector& v) { return op.apply(v); }, p, cfg);
            std::memcpy(q, r.pairs.q.data(), sizeof(double) * p * (std::size_t)k);
            std::memcpy(lambda, r.pairs.lambda.data(), sizeof(double) * (std::size_t)k);
            std::memcpy(residuals, r.residuals.data(), sizeof(double) * (std::size_t)k);
            *iterations = (int64_t)r.iterations;
        } catch (const ConvergenceError& e) {
            for (std::size_t i = 0; i < e.best_residuals.size() && i < (std::size_t)k; ++i)
                residuals[i] = e.best_residuals[i];
            throw;
        }
    });
}

// The consumers of eigenpairs on the reference itself (eigensolve.cpp:11-30,
// 278-358).  full = 0: low_rank_*; 1: full_rank_* with lambda_tilde.  h (p x p),
// y (xlen) and quad are each skipped when null; x may be null when only h is
// wanted.  The reference's own ShapeError / ContractError come back as rc 1 / 2.
int ref_eig_ops(const double* q, const double* lambda, int64_t p, int64_t k, int full, double lambda_tilde,
                int64_t memory_cap, const double* x, int64_t xlen, double* h, double* y, double* quad) {
    return guard([&] {
        EigenPairs e{DenseMatrix(p, k, std::vector<double>(q, q + p * k)),
                     DenseVector(std::vector<double>(lambda, lambda + k))};
        if (h) {
            const DenseMatrix m = full ? full_rank_materialize(e, lambda_tilde, (std::size_t)memory_cap)
                                       : low_rank_materialize(e, (std::size_t)memory_cap);
            std::memcpy(h, m.data(), sizeof(double) * p * p);
        }
        if (!x) return;
        const DenseVector xv(std::vector<double>(x, x + xlen));
        if (quad) *quad = full ? full_rank_quadform(e, lambda_tilde, xv) : low_rank_quadform(e, xv);
        if (y) {
            const DenseVector r = full ? full_rank_apply(e, lambda_tilde, xv) : low_rank_apply(e, xv);
            std::memcpy(y, r.data(), sizeof(double) * r.len());
        }
    });
}

int ref_validate_eigen_pairs(const double* q, int64_t p, int64_t k, const double* lambda, int64_t lambda_len,
                             double ortho_tol) {
    return guard([&] {
        EigenPairs e{DenseMatrix(p, k, std::vector<double>(q, q + p * k)),
                     DenseVector(std::vector<double>(lambda, lambda + lambda_len))};
        validate_eigen_pairs(e, ortho_tol);
    });
}

int ref_default_lambda_tilde(const double* lambda, int64_t k, double* out) {
    return guard([&] {
        EigenPairs e{DenseMatrix(std::max<int64_t>(k, 1), k, 0.0), DenseVector(std::vector<double>(lambda, lambda + k))};
        *out = default_lambda_tilde(e);
    });
}

}  // extern "C"
