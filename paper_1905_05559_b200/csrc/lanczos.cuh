// lanczos.cuh -- curv::lanczos_topk (eigensolve.cpp:46-156) on the Hessian
// operator, with the Krylov basis resident in HBM.
//
// Each step applies H by the device R-op engine (Engine::hvp: one batched
// forward/backward R-pass), then alpha, the three-term recurrence and two
// classical Gram-Schmidt passes against the whole basis (the reference's full
// reorthogonalisation, eigensolve.cpp:70-73) as fp64-accumulating kernels.
// The tridiagonal Ritz problem is small and sequential: it is solved on the
// host by implicit QL, rotating only the last row of the identity for the
// convergence estimates beta * |y_{m,i}| (eigensolve.cpp:78-94), and fully
// once the estimates pass, when the Ritz vectors are formed by one GEMM and
// confirmed against true residuals from a k-direction batched HVP
// (eigensolve.cpp:95-129).  Start vectors and restarts use the reference's
// splitmix64 + Box-Muller stream (rng.hpp), so the Krylov sequence starts
// where the reference's does.
#pragma once

#include <cmath>
#include <vector>

#include "common.cuh"
#include "curvature.cuh"
#include "gemm_simt.cuh"
#include "model.cuh"

namespace ck {

// ---- host: the reference's Rng (rng.hpp:10-31, rng.cpp:8-20 Box-Muller) ---
struct HostRng {
    uint64_t state;
    bool has_spare = false;
    double spare = 0.0;
    uint64_t next_u64() {
        uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double next_uniform() { return (double)(next_u64() >> 11) * 0x1.0p-53; }
    double next_normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        const double u1 = 1.0 - next_uniform();  // (0, 1]
        const double u2 = next_uniform();
        const double r = std::sqrt(-2.0 * std::log(u1)), th = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(th);
        has_spare = true;
        return r * std::cos(th);
    }
};

// ---- host: symmetric tridiagonal eigensolver (implicit QL, Wilkinson shift)
// The textbook routine (Numerical Recipes `tqli`; the reference uses the same
// algorithm in linalg.cpp:262-315 for its Lanczos Ritz solve).
// d (m) diagonal, e (m-1) off-diagonal.  z: nz x m rows that receive every
// rotation (identity -> eigenvectors; the last row of the identity -> the
// last components of the eigenvectors).  On return d holds the eigenvalues;
// order() gives them descending.
inline void tridiag_ql(std::vector<double>& d, std::vector<double> e, std::vector<double>& z, int64_t nz) {
    const int64_t m = (int64_t)d.size();
    e.resize(m, 0.0);
    for (int64_t l = 0; l < m; ++l) {
        int iter = 0;
        for (;;) {
            int64_t mm = l;
            for (; mm < m - 1; ++mm) {
                const double dd = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
                if (std::fabs(e[mm]) <= 1e-15 * dd) break;
            }
            if (mm == l) break;
            if (++iter > 60) throw CurvError(kConvergenceError, "lanczos_topk: tridiagonal QL did not converge");
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = std::hypot(g, 1.0);
            g = d[mm] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
            double s = 1.0, c = 1.0, p = 0.0;
            int64_t i = mm - 1;
            for (; i >= l; --i) {
                double f = s * e[i];
                const double b = c * e[i];
                r = std::hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {
                    d[i + 1] -= p;
                    e[mm] = 0.0;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[i + 1] - p;
                r = (d[i] - g) * s + 2.0 * c * b;
                p = s * r;
                d[i + 1] = g + p;
                g = c * r - b;
                for (int64_t k = 0; k < nz; ++k) {
                    f = z[k * m + i + 1];
                    z[k * m + i + 1] = s * z[k * m + i] + c * f;
                    z[k * m + i] = c * z[k * m + i] - s * f;
                }
            }
            if (r == 0.0 && i >= l) continue;
            d[l] -= p;
            e[l] = g;
            e[mm] = 0.0;
        }
    }
}

inline std::vector<int64_t> order_desc(const std::vector<double>& d) {
    std::vector<int64_t> o(d.size());
    for (size_t i = 0; i < o.size(); ++i) o[i] = (int64_t)i;
    std::stable_sort(o.begin(), o.end(), [&](int64_t a, int64_t b) { return d[a] > d[b]; });
    return o;
}

// ---- device helpers ----------------------------------------------------------
// out[c] = <V_c, w> for the m basis vectors V_c = V + c * P (fp64 accumulation)
template <class T>
__global__ void __launch_bounds__(256) lz_dots_kernel(const T* __restrict__ V, int64_t P, const T* __restrict__ w,
                                                      double* __restrict__ out) {
    __shared__ double red[8];
    const T* v = V + (int64_t)blockIdx.x * P;
    double s = 0.0;
    for (int64_t r = threadIdx.x; r < P; r += blockDim.x) s += (double)v[r] * (double)w[r];
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < 8; ++i) t += red[i];
        out[blockIdx.x] = t;
    }
}

// w -= sum_c coef[c] V_c  (a Gram-Schmidt pass; also the three-term recurrence)
template <class T>
__global__ void lz_sub_kernel(const T* __restrict__ V, int64_t P, int64_t m, const double* __restrict__ coef,
                              T* __restrict__ w) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= P) return;
    double acc = (double)w[r];
    for (int64_t c = 0; c < m; ++c) acc -= coef[c] * (double)V[c * P + r];
    w[r] = (T)acc;
}

// out = in * (1 / *nrm)
template <class T>
__global__ void lz_scale_kernel(const T* __restrict__ in, const double* __restrict__ nrm2, T* __restrict__ out,
                                int64_t P) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < P) out[r] = (T)((double)in[r] / std::sqrt(*nrm2));
}

// res[i] = || HQ_i - lambda_i Q_i ||^2 (fp64), one block per pair
template <class T>
__global__ void __launch_bounds__(256) lz_residual_kernel(const T* __restrict__ HQ, const T* __restrict__ Q,
                                                          const double* __restrict__ lam, int64_t P,
                                                          double* __restrict__ res) {
    __shared__ double red[8];
    const int64_t i = blockIdx.x;
    double s = 0.0;
    for (int64_t r = threadIdx.x; r < P; r += blockDim.x) {
        const double d = (double)HQ[i * P + r] - lam[i] * (double)Q[i * P + r];
        s += d * d;
    }
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        res[i] = t;
    }
}

struct LanczosOut {
    std::vector<double> q;          // P x k row-major (reference EigenPairs::q)
    std::vector<double> lambda;     // k, descending
    std::vector<double> residuals;  // k (true residuals on success, best estimates on failure)
    int64_t iterations = 0;
    bool converged = false;
};

// Top-k algebraically largest eigenpairs of H (batch-averaged Hessian of the
// cached dataset) -- eigensolve.cpp:46-156 restated.
template <class T>
LanczosOut lanczos_topk(const ModelDesc& md, const T* params, const Cache<T>& c, int64_t k, int64_t max_iterations,
                        double tol, uint64_t seed, int prec, cudaStream_t s) {
    const int64_t P = md.P;
    if (P < 2) throw CurvError(kContractError, "lanczos_topk: operator dimension must be >= 2");
    if (k < 1 || k >= P)
        throw CurvError(kContractError, "lanczos_topk: need 1 <= k < p, got k = " + std::to_string(k) +
                                            ", p = " + std::to_string(P));
    if (max_iterations < k) throw CurvError(kContractError, "lanczos_topk: max_iterations must be >= k");
    if (!(tol > 0.0)) throw CurvError(kContractError, "lanczos_topk: residual_tol must be > 0");
    const int64_t max_steps = std::min(max_iterations, P);
    Engine<T> eng{md, s, prec};
    const T alpha_h = T(1) / T(c.n);
    DevMem Vb((size_t)(max_steps + 1) * P * sizeof(T), s), W((size_t)P * sizeof(T), s);
    DevMem coef((size_t)(max_steps + 2) * sizeof(double), s), scal(4 * sizeof(double), s);
    T* V = dptr<T>(Vb);
    T* w = dptr<T>(W);
    double* cf = dptr<double>(coef);
    double* sc = dptr<double>(scal);
    const unsigned gb = (unsigned)ceil_div(P, 256);
    HostRng rng{seed};
    // random_unit_vector (eigensolve.cpp:32-38), then for a restart one
    // Gram-Schmidt pass against the basis and the 0.5 norm test (:131-141)
    auto unit_random = [&](T* dst, bool against_basis, int64_t m) -> bool {
        std::vector<double> h(P);
        double hn = 0.0;
        for (auto& v : h) {
            v = rng.next_normal();
            hn += v * v;
        }
        hn = std::sqrt(hn);
        std::vector<T> ht(P);
        for (int64_t i = 0; i < P; ++i) ht[i] = (T)(h[i] / hn);
        CK_CUDA(cudaMemcpyAsync(w, ht.data(), P * sizeof(T), cudaMemcpyHostToDevice, s));
        if (against_basis && m > 0) {
            lz_dots_kernel<T><<<(unsigned)m, 256, 0, s>>>(V, P, w, cf);
            CK_LAUNCH();
            lz_sub_kernel<T><<<gb, 256, 0, s>>>(V, P, m, cf, w);
            CK_LAUNCH();
        }
        lz_dots_kernel<T><<<1, 256, 0, s>>>(w, P, w, sc);
        CK_LAUNCH();
        double n2 = 0.0;
        CK_CUDA(cudaMemcpyAsync(&n2, sc, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK_CUDA(cudaStreamSynchronize(s));
        // the reference normalises its fresh vector when its norm exceeds 0.5
        if (against_basis && std::sqrt(n2) <= 0.5) return false;
        lz_scale_kernel<T><<<gb, 256, 0, s>>>(w, sc, dst, P);
        CK_LAUNCH();
        return true;
    };
    unit_random(V, false, 0);

    std::vector<double> alphas, betas, best;
    double opnorm = 0.0;
    LanczosOut out;
    for (int64_t j = 0; j < max_steps; ++j) {
        T* vj = V + j * P;
        eng.hvp(params, c, vj, 1, P, w, P, alpha_h);
        // alpha_j and the recurrence, then two full Gram-Schmidt passes.  alpha_j stays on
        // the device (sc[1] -> the recurrence coefficients) and comes to the host with
        // ||w||^2 in the step's one synchronisation
        lz_dots_kernel<T><<<1, 256, 0, s>>>(vj, P, w, sc + 1);
        CK_LAUNCH();
        if (j > 0) {  // w -= alpha v_j + beta_{j-1} v_{j-1}: V_{j-1}, V_j with coefficients (beta, alpha)
            CK_CUDA(cudaMemcpyAsync(cf, &betas[j - 1], sizeof(double), cudaMemcpyHostToDevice, s));
            CK_CUDA(cudaMemcpyAsync(cf + 1, sc + 1, sizeof(double), cudaMemcpyDeviceToDevice, s));
            lz_sub_kernel<T><<<gb, 256, 0, s>>>(V + (j - 1) * P, P, 2, cf, w);
        } else {
            CK_CUDA(cudaMemcpyAsync(cf, sc + 1, sizeof(double), cudaMemcpyDeviceToDevice, s));
            lz_sub_kernel<T><<<gb, 256, 0, s>>>(vj, P, 1, cf, w);
        }
        CK_LAUNCH();
        for (int pass = 0; pass < 2; ++pass) {
            lz_dots_kernel<T><<<(unsigned)(j + 1), 256, 0, s>>>(V, P, w, cf);
            CK_LAUNCH();
            lz_sub_kernel<T><<<gb, 256, 0, s>>>(V, P, j + 1, cf, w);
            CK_LAUNCH();
        }
        lz_dots_kernel<T><<<1, 256, 0, s>>>(w, P, w, sc);
        CK_LAUNCH();
        double hs[2] = {0.0, 0.0};  // ||w||^2, alpha_j
        CK_CUDA(cudaMemcpyAsync(hs, sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK_CUDA(cudaStreamSynchronize(s));
        const double b2 = hs[0], alpha = hs[1];
        alphas.push_back(alpha);
        const double beta = std::sqrt(b2);
        opnorm = std::max(opnorm, std::fabs(alpha) + beta + (j > 0 ? betas[j - 1] : 0.0));

        const int64_t m = j + 1;
        if (m >= k) {
            // Ritz values and the last components of their vectors
            std::vector<double> d = alphas, zl(m, 0.0);
            zl[m - 1] = 1.0;
            tridiag_ql(d, betas, zl, 1);
            const auto ord = order_desc(d);
            std::vector<double> est(k);
            bool small = true;
            double est_max = 0.0;
            for (int64_t i = 0; i < k; ++i) {
                est[i] = std::fabs(beta * zl[ord[i]]);
                est_max = std::max(est_max, est[i]);
                if (est[i] > tol * std::max(1.0, std::fabs(d[ord[i]]))) small = false;
            }
            if (best.empty() || est_max < *std::max_element(best.begin(), best.end())) best = est;
            if (small || m == P) {
                // full Ritz vectors: Qt (k x P) = Y^T V, Y = the top-k eigenvectors (m x k)
                std::vector<double> dv = alphas, z(m * m, 0.0);
                for (int64_t i = 0; i < m; ++i) z[i * m + i] = 1.0;
                tridiag_ql(dv, betas, z, m);
                const auto o2 = order_desc(dv);
                // z rows are the identity's rows rotated: z[r][i] = component r of eigenvector i
                std::vector<T> y((size_t)m * k);
                std::vector<double> lam(k);
                for (int64_t i = 0; i < k; ++i) {
                    lam[i] = dv[o2[i]];
                    for (int64_t r = 0; r < m; ++r) y[r * k + i] = (T)z[r * m + o2[i]];
                }
                DevMem Yd((size_t)m * k * sizeof(T), s), Qt((size_t)k * P * sizeof(T), s),
                    HQ((size_t)k * P * sizeof(T), s), nrm((size_t)k * sizeof(double), s),
                    lamd((size_t)k * sizeof(double), s), resd((size_t)k * sizeof(double), s);
                CK_CUDA(cudaMemcpyAsync(Yd.p, y.data(), y.size() * sizeof(T), cudaMemcpyHostToDevice, s));
                // Qt[i][r] = sum_c Y[c][i] V[c][r]
                EpiStore<T> e{dptr<T>(Qt), P, 0, T(1), T(0)};
                gemm_simt<T>(s, k, P, m, 1, mnmaj(dptr<T>(Yd), k), mnmaj(V, P), e);
                // normalise away the rounding drift of the basis product (eigensolve.cpp:107-112)
                for (int64_t i = 0; i < k; ++i) {
                    T* qi = dptr<T>(Qt) + i * P;
                    lz_dots_kernel<T><<<1, 256, 0, s>>>(qi, P, qi, dptr<double>(nrm) + i);
                    CK_LAUNCH();
                    lz_scale_kernel<T><<<gb, 256, 0, s>>>(qi, dptr<double>(nrm) + i, qi, P);
                    CK_LAUNCH();
                }
                eng.hvp(params, c, dptr<T>(Qt), k, P, dptr<T>(HQ), P, alpha_h);
                CK_CUDA(cudaMemcpyAsync(lamd.p, lam.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
                lz_residual_kernel<T><<<(unsigned)k, 256, 0, s>>>(dptr<T>(HQ), dptr<T>(Qt), dptr<double>(lamd), P,
                                                                  dptr<double>(resd));
                CK_LAUNCH();
                std::vector<double> res(k);
                std::vector<T> hq((size_t)k * P);
                CK_CUDA(cudaMemcpyAsync(res.data(), resd.p, k * sizeof(double), cudaMemcpyDeviceToHost, s));
                CK_CUDA(cudaMemcpyAsync(hq.data(), Qt.p, hq.size() * sizeof(T), cudaMemcpyDeviceToHost, s));
                CK_CUDA(cudaStreamSynchronize(s));
                bool confirmed = true;
                for (int64_t i = 0; i < k; ++i) {
                    res[i] = std::sqrt(res[i]);
                    if (res[i] > tol * std::max(1.0, std::fabs(lam[i]))) confirmed = false;
                }
                if (confirmed) {
                    out.q.assign((size_t)P * k, 0.0);
                    for (int64_t i = 0; i < k; ++i)
                        for (int64_t r = 0; r < P; ++r) out.q[r * k + i] = (double)hq[i * P + r];
                    out.lambda = lam;
                    out.residuals = res;
                    out.iterations = m;
                    out.converged = true;
                    return out;
                }
                if (m == P) break;
            }
        }
        if (m == max_steps) break;
        if (beta <= 1e-13 * std::max(opnorm, 1.0)) {
            // invariant subspace: continue in a fresh random direction (eigensolve.cpp:134-143)
            while (!unit_random(V + (j + 1) * P, true, m)) {
            }
            betas.push_back(0.0);
        } else {
            lz_scale_kernel<T><<<gb, 256, 0, s>>>(w, sc, V + (j + 1) * P, P);
            CK_LAUNCH();
            betas.push_back(beta);
        }
    }
    out.residuals = best;
    out.iterations = (int64_t)alphas.size();
    out.converged = false;
    return out;
}

}  // namespace ck
