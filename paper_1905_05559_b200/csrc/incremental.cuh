// incremental.cuh -- the streaming OPG eigensolver (curv::IncrementalOpgEigs,
// eigensolve.hpp:52-78, eigensolve.cpp:158-243) on the device.
//
// Same algorithm and update windows as the reference: row blocks of J are
// buffered until at least k rows are waiting; the compressed matrix
// M^T = [basis diag(sigma) | buffered rows^T] (P x m, m = k + buffered) is
// re-factorised and truncated back to rank k; eigenvalues are sigma^2 / N.
// The reference factorises M^T by one-sided Jacobi on the host.  Here the
// m x m Gram W = M M^T is accumulated in fp64 on the device (gram_kernel),
// diagonalised by the one-CTA Jacobi kernel (W = V diag(sigma^2) V^T), and
// the new basis M^T V / sigma is one fp64 GEMM (DMMA) -- the P-length work
// never leaves HBM; only the m eigenvalues and the m x k selection cross to
// the host.  Rank-deficient tails are completed with canonical directions
// orthogonal to the accepted columns, as the reference does (host, rare).
#pragma once

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "eigen.cuh"
#include "gemm_dmma.cuh"

namespace ck {

// MT[r][c0 + c] = basis[r][c] * sigma[c]   (r < p, c < sc)
__global__ void incr_scaled_basis_kernel(const double* __restrict__ basis, int64_t ldb, const double* __restrict__ sig,
                                         int64_t p, int64_t sc, double* __restrict__ mt, int64_t ldm) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= p * sc) return;
    const int64_t r = idx / sc, c = idx - r * sc;
    mt[r * ldm + c] = basis[r * ldb + c] * sig[c];
}

// MT[r][c0 + n] = block[n][r]   (n < b rows of the block, r < p): a 32 x 32 tiled transpose
__global__ void incr_rows_to_cols_kernel(const double* __restrict__ blk, int64_t ldk, int64_t b, int64_t p,
                                         double* __restrict__ mt, int64_t ldm, int64_t c0) {
    __shared__ double t[32][33];
    const int64_t n0 = (int64_t)blockIdx.y * 32, r0 = (int64_t)blockIdx.x * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t n = n0 + y, r = r0 + threadIdx.x;
        t[y][threadIdx.x] = (n < b && r < p) ? blk[n * ldk + r] : 0.0;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t r = r0 + y, n = n0 + threadIdx.x;
        if (r < p && n < b) mt[r * ldm + c0 + n] = t[threadIdx.x][y];
    }
}

// sig[c] = || U[:, c] ||_2 over the p rows of U (p x k, ld), one CTA per column
// (fixed-order block reduction: deterministic)
__global__ void incr_colnorm_kernel(const double* __restrict__ u, int64_t ld, int64_t p, double* __restrict__ sig) {
    __shared__ double red[32];
    const int64_t c = blockIdx.x;
    double acc = 0.0;
    for (int64_t r = threadIdx.x; r < p; r += blockDim.x) {
        const double x = u[r * ld + c];
        acc += x * x;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) sig[c] = sqrt(acc);
    }
}

// U[r][c] *= inv[c]
__global__ void incr_scale_cols_kernel(double* __restrict__ u, int64_t ld, int64_t p, int64_t k,
                                       const double* __restrict__ inv) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= p * k) return;
    const int64_t r = idx / k, c = idx - r * k;
    u[r * ld + c] *= inv[c];
}

struct IncrOpg {
    int64_t p = 0, k = 0;
    int64_t rows_seen = 0, updates = 0, buffered = 0;
    bool has_state = false;
    std::vector<double> sigma;  // singular values of the rows seen, descending
    DevMem basis;               // p x k, row-major (ld k), fp64
    std::vector<DevMem> buf;    // buffered row blocks, each b x p (ld p), fp64
    std::vector<int64_t> buf_rows;

    IncrOpg(int64_t p_, int64_t k_) : p(p_), k(k_) {
        if (k < 1 || k > p)
            throw CurvError(kContractError, "IncrementalOpgEigs: need 1 <= k <= p, got k = " + std::to_string(k) +
                                                ", p = " + std::to_string(p));
    }

    // push_block (eigensolve.cpp:165-174): rows x p fp64 at `src` (device,
    // leading dimension ld >= p) copied into the buffer
    void push(const double* src, int64_t rows, int64_t ld, cudaMemcpyKind kind, cudaStream_t s) {
        if (rows < 1) throw CurvError(kContractError, "IncrementalOpgEigs: empty block");
        if (ld < p) throw CurvError(kShapeError, "IncrementalOpgEigs: block has fewer than p columns");
        DevMem b((size_t)rows * p * sizeof(double), s);
        CK_CUDA(cudaMemcpy2DAsync(b.p, p * sizeof(double), src, ld * sizeof(double), p * sizeof(double), rows, kind, s));
        buf.push_back(std::move(b));
        buf_rows.push_back(rows);
        buffered += rows;
        rows_seen += rows;
        if (buffered >= k) update(s);
    }

    // update_from_buffer (eigensolve.cpp:176-224)
    void update(cudaStream_t s) {
        const int64_t sc = has_state ? (int64_t)sigma.size() : 0;
        const int64_t m = sc + buffered;
        DevMem mt((size_t)p * m * sizeof(double), s);
        if (sc > 0) {
            DevMem sig(sc * sizeof(double), s);
            CK_CUDA(cudaMemcpyAsync(sig.p, sigma.data(), sc * sizeof(double), cudaMemcpyHostToDevice, s));
            incr_scaled_basis_kernel<<<blocks_for(p * sc), 256, 0, s>>>(dptr<double>(basis), k, dptr<double>(sig), p,
                                                                        sc, dptr<double>(mt), m);
            CK_LAUNCH();
            CK_CUDA(cudaStreamSynchronize(s));  // sig is released at scope end
        }
        int64_t at = sc;
        for (size_t bi = 0; bi < buf.size(); ++bi) {
            const int64_t b = buf_rows[bi];
            dim3 g((unsigned)ceil_div(p, 32), (unsigned)ceil_div(b, 32));
            incr_rows_to_cols_kernel<<<g, dim3(32, 8), 0, s>>>(dptr<double>(buf[bi]), p, b, p, dptr<double>(mt), m, at);
            CK_LAUNCH();
            at += b;
        }
        buf.clear();
        buf_rows.clear();
        buffered = 0;

        // W = (M^T)^T M^T (m x m, fp64), then W = V diag(lambda) V^T
        DevMem w((size_t)m * m * sizeof(double), s), v((size_t)m * m * sizeof(double), s), sw(sizeof(int), s);
        CK_CUDA(cudaMemsetAsync(w.p, 0, (size_t)m * m * sizeof(double), s));
        {
            const int64_t ksplit = std::min<int64_t>(256, std::max<int64_t>(1, p / 2048));
            dim3 g((unsigned)ceil_div(m, 32), (unsigned)ceil_div(m, 32), (unsigned)ksplit);
            gram_kernel<double><<<g, 256, 0, s>>>(dptr<double>(mt), m, p, m, ceil_div(p, ksplit), dptr<double>(w));
            CK_LAUNCH();
        }
        jacobi_eig(dptr<double>(w), dptr<double>(v), m, dptr<int>(sw), s);
        std::vector<double> lam(m), vh((size_t)m * m);
        CK_CUDA(cudaMemcpy2DAsync(lam.data(), sizeof(double), w.p, (m + 1) * sizeof(double), sizeof(double), m,
                                  cudaMemcpyDeviceToHost, s));
        CK_CUDA(cudaMemcpyAsync(vh.data(), v.p, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> ord(m);
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return lam[a] > lam[b]; });
        const int64_t keep = std::min(k, m);
        // U = M^T V[:, top keep] (fp64 tensor cores); sigma_c = ||U_c|| (a direction in
        // the numerical null space of M^T gives ~eps ||M^T||, as the reference's
        // one-sided Jacobi does -- the Gram eigenvalue alone would say ~sqrt(eps))
        std::vector<double> bsel((size_t)keep * m);
        for (int64_t c = 0; c < keep; ++c)
            for (int64_t j = 0; j < m; ++j) bsel[(size_t)c * m + j] = vh[(size_t)j * m + ord[c]];
        DevMem bs((size_t)keep * m * sizeof(double), s), sd((size_t)keep * sizeof(double), s);
        CK_CUDA(cudaMemcpyAsync(bs.p, bsel.data(), bsel.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        DevMem nb((size_t)p * k * sizeof(double), s);
        if (keep < k) CK_CUDA(cudaMemsetAsync(nb.p, 0, (size_t)p * k * sizeof(double), s));
        EpiStore<double> e{dptr<double>(nb), k, 0, 1.0, 0.0};
        gemm_dmma(s, p, keep, m, 1, kmaj(dptr<double>(mt), m), kmaj(dptr<double>(bs), m), e);
        incr_colnorm_kernel<<<(unsigned)keep, 256, 0, s>>>(dptr<double>(nb), k, p, dptr<double>(sd));
        CK_LAUNCH();
        std::vector<double> sig(keep);
        CK_CUDA(cudaMemcpyAsync(sig.data(), sd.p, keep * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK_CUDA(cudaStreamSynchronize(s));
        // descending by the accurate norms (the Gram order can swap near-ties)
        std::vector<int64_t> perm(keep);
        std::iota(perm.begin(), perm.end(), 0);
        std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return sig[a] > sig[b]; });
        bool permuted = false;
        for (int64_t c = 0; c < keep; ++c) permuted |= perm[c] != c;
        if (permuted) {  // reorder the columns of U by a second pass of the small GEMM
            std::vector<double> b2((size_t)keep * m), s2(keep);
            for (int64_t c = 0; c < keep; ++c) {
                std::copy(bsel.begin() + (size_t)perm[c] * m, bsel.begin() + (size_t)(perm[c] + 1) * m,
                          b2.begin() + (size_t)c * m);
                s2[c] = sig[perm[c]];
            }
            CK_CUDA(cudaMemcpyAsync(bs.p, b2.data(), b2.size() * sizeof(double), cudaMemcpyHostToDevice, s));
            gemm_dmma(s, p, keep, m, 1, kmaj(dptr<double>(mt), m), kmaj(dptr<double>(bs), m), e);
            sig = s2;
        }
        const double rank_tol = 1e-12 * std::max(sig[0], 1e-300);
        std::vector<double> inv(keep);
        int64_t first_def = keep;
        for (int64_t c = 0; c < keep; ++c) {
            if (sig[c] > rank_tol) {
                inv[c] = 1.0 / sig[c];
            } else {
                inv[c] = 0.0;
                sig[c] = 0.0;
                first_def = std::min(first_def, c);
            }
        }
        CK_CUDA(cudaMemcpyAsync(sd.p, inv.data(), keep * sizeof(double), cudaMemcpyHostToDevice, s));
        incr_scale_cols_kernel<<<blocks_for(p * keep), 256, 0, s>>>(dptr<double>(nb), k, p, keep, dptr<double>(sd));
        CK_LAUNCH();
        basis = std::move(nb);
        if (first_def < keep) complete_rank_deficient(first_def, keep, s);  // host, rare
        sigma = sig;
        has_state = true;
        ++updates;
        CK_CUDA(cudaStreamSynchronize(s));  // the scratch above is released at scope end
    }

    // Columns c >= the first rank-deficient one: canonical directions e_cand
    // orthogonalised against the accepted columns, first with norm > 0.5
    // (eigensolve.cpp:203-218).
    void complete_rank_deficient(int64_t first, int64_t keep, cudaStream_t s) {
        std::vector<double> h((size_t)p * k);
        CK_CUDA(cudaMemcpyAsync(h.data(), basis.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK_CUDA(cudaStreamSynchronize(s));
        for (int64_t c = first; c < keep; ++c) {
            for (int64_t cand = 0; cand < p; ++cand) {
                std::vector<double> v(p, 0.0);
                v[cand] = 1.0;
                for (int64_t prev = 0; prev < c; ++prev) {
                    double d = 0.0;
                    for (int64_t r = 0; r < p; ++r) d += h[(size_t)r * k + prev] * v[r];
                    for (int64_t r = 0; r < p; ++r) v[r] -= d * h[(size_t)r * k + prev];
                }
                double nrm = 0.0;
                for (double x : v) nrm += x * x;
                nrm = std::sqrt(nrm);
                if (nrm > 0.5) {
                    for (int64_t r = 0; r < p; ++r) h[(size_t)r * k + c] = v[r] / nrm;
                    break;
                }
            }
        }
        CK_CUDA(cudaMemcpyAsync(basis.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        CK_CUDA(cudaStreamSynchronize(s));
    }

    // finalize (eigensolve.cpp:226-243): q (p x k row-major) and lambda (k)
    void finalize(int64_t n_total, double* q, double* lambda, cudaMemcpyKind kind, cudaStream_t s) const {
        if (rows_seen != n_total)
            throw CurvError(kContractError, "IncrementalOpgEigs: saw " + std::to_string(rows_seen) +
                                                " rows, n_total says " + std::to_string(n_total));
        if (buffered > 0)
            throw CurvError(kContractError, "IncrementalOpgEigs: " + std::to_string(buffered) +
                                                " leftover rows are fewer than k = " + std::to_string(k) +
                                                " in the final update window");
        if (!has_state) throw CurvError(kContractError, "IncrementalOpgEigs: no update performed; need at least k rows");
        const int64_t kk = (int64_t)sigma.size();
        if (q) CK_CUDA(cudaMemcpyAsync(q, basis.p, (size_t)p * k * sizeof(double), kind, s));
        std::vector<double> lam(kk);
        const double inv_n = 1.0 / (double)n_total;
        for (int64_t i = 0; i < kk; ++i) lam[i] = sigma[i] * sigma[i] * inv_n;
        if (lambda) {
            const cudaMemcpyKind lk = kind == cudaMemcpyDeviceToHost ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice;
            CK_CUDA(cudaMemcpyAsync(lambda, lam.data(), kk * sizeof(double), lk, s));
        }
        CK_CUDA(cudaStreamSynchronize(s));
    }
};

}  // namespace ck
