// eigen.cuh -- top-k eigenpairs of the OPG G = (1/N) J^T J without forming G.
//
// Randomized range finder (Halko-Martinsson-Tropp, Alg. 4.3/4.4):
//   Y = G Omega, Omega ~ N(0,1)^{P x l}, l = k + oversample
//   q power iterations Y <- G orth(Y)
//   Q = orth(Y);  B = Q^T G Q = (1/N) (J Q)^T (J Q)   (l x l)
//   B = V diag(lambda) V^T  (parallel cyclic Jacobi in one CTA)
//   eigenvectors Q V[:, :k], eigenvalues lambda[:k] (descending)
// G is only ever applied as J^T (J X): two passes over the per-example
// gradient matrix J, which stays in HBM.  orth() is CholeskyQR2 with the
// l x l Gram matrices accumulated in fp64.
//
// Replaces the reference's streaming SVD (eigensolve.cpp:158-251); its
// eigenvalue scaling sigma^2 / N (eigensolve.cpp:236-242) is the same
// quantity as lambda(B) here.
#pragma once

#include <algorithm>
#include <memory>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "curvature.cuh"
#include "gemm_tc.cuh"
#include "comm.cuh"
#include "kr.cuh"
#include "gemm_simt.cuh"
#include "model.cuh"

namespace ck {

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Omega[p][c] ~ N(0, 1): Box-Muller on the counter-based splitmix64 stream
template <class T>
__global__ void gaussian_kernel(T* out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, int64_t row0) {
    const int64_t loc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (loc >= rows * cols) return;
    // entry (row0 + r, c) of the global sketch: a shard draws exactly its rows
    const int64_t idx = row0 * cols + loc;
    const uint64_t pair = (uint64_t)idx >> 1;
    const double u1 = 1.0 - (double)(splitmix_at(seed, 2 * pair) >> 11) * 0x1.0p-53;
    const double u2 = (double)(splitmix_at(seed, 2 * pair + 1) >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double th = 6.283185307179586476925286766559 * u2;
    out[(loc / cols) * ld + loc % cols] = (T)((idx & 1) ? r * sin(th) : r * cos(th));
}

// W[c][d] += sum_{p in chunk} Y[p][c] * Y[p][d]   (fp64 accumulation)
template <class T>
__global__ void __launch_bounds__(256) gram_kernel(const T* __restrict__ Y, int64_t ld, int64_t rows, int64_t l,
                                                   int64_t chunk, double* __restrict__ W) {
    __shared__ double a[32][33], b[32][33];
    const int64_t c0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
    if (d0 > c0 + 31) return;  // lower triangle tiles only; mirrored below
    const int64_t p0 = blockIdx.z * chunk, p1 = min(rows, p0 + chunk);
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 8 row-groups
    double acc[4] = {0, 0, 0, 0};
    for (int64_t p = p0; p < p1; p += 32) {
        for (int r = ty; r < 32; r += 8) {
            const int64_t pp = p + r;
            a[r][tx] = (pp < p1 && c0 + tx < l) ? (double)Y[pp * ld + c0 + tx] : 0.0;
            b[r][tx] = (pp < p1 && d0 + tx < l) ? (double)Y[pp * ld + d0 + tx] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int r = 0; r < 32; ++r) {
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] += a[r][ty + 8 * u] * b[r][tx];
        }
        __syncthreads();
    }
    for (int u = 0; u < 4; ++u) {
        const int64_t c = c0 + ty + 8 * u, d = d0 + tx;
        if (c < l && d < l && d <= c) {
            atomicAdd(&W[c * l + d], acc[u]);
            if (d != c) atomicAdd(&W[d * l + c], acc[u]);
        }
    }
}

// W += Y^T Y over a chunk of rows (fp64): 64 x 64 output tiles of the lower
// triangle (blockIdx.x: tile, blockIdx.y: row chunk), 4 x 4 register
// micro-tiles per thread (rows tr + 16u, columns tc + 16v), the row panels
// staged in shared memory as fp64.
template <class T>
__global__ void __launch_bounds__(256) gram64_kernel(const T* __restrict__ Y, int64_t ld, int64_t rows, int64_t l,
                                                     int64_t chunk, double* __restrict__ W) {
    __shared__ double As[32][64], Bs[32][64];
    // lower tile (ci, di), di <= ci, from the triangular index
    int ci = 0;
    while ((ci + 1) * (ci + 2) / 2 <= (int)blockIdx.x) ++ci;
    const int di = (int)blockIdx.x - ci * (ci + 1) / 2;
    const int64_t c0 = ci * 64, d0 = di * 64;
    const int64_t p0 = blockIdx.y * chunk, p1 = min(rows, p0 + chunk);
    const int t = threadIdx.x, tr = t / 16, tc = t % 16;
    double acc[4][4] = {};
    // the next 32-row panel is fetched into registers while this one is used
    T ra[8], rb[8];
    auto fetch = [&](int64_t p) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = t + 256 * j, r = e / 64, cc = e % 64;
            const int64_t pp = p + r;
            ra[j] = (pp < p1 && c0 + cc < l) ? Y[pp * ld + c0 + cc] : T(0);
            rb[j] = (pp < p1 && d0 + cc < l) ? Y[pp * ld + d0 + cc] : T(0);
        }
    };
    if (p0 < p1) fetch(p0);
    for (int64_t p = p0; p < p1; p += 32) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = t + 256 * j, r = e / 64, cc = e % 64;
            As[r][cc] = (double)ra[j];
            Bs[r][cc] = (double)rb[j];
        }
        __syncthreads();
        if (p + 32 < p1) fetch(p + 32);
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
            double a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // interleaved micro-tile: conflict-free rows of Bs
                a[u] = As[r][tr + 16 * u];
                b[u] = Bs[r][tc + 16 * u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t c = c0 + tr + 16 * u, d = d0 + tc + 16 * v;
            if (c >= l || d >= l) continue;
            if (ci == di) {
                atomicAdd(&W[c * l + d], acc[u][v]);  // diagonal tile: both halves computed
            } else {
                atomicAdd(&W[c * l + d], acc[u][v]);
                atomicAdd(&W[d * l + c], acc[u][v]);
            }
        }
}

// W += Y^T Y (fp64) on the FP64 tensor cores: mma.sync m8n8k4 f64.  A block
// owns a 64 x 64 lower tile (blockIdx.x) over a row chunk (blockIdx.y); four
// warps each accumulate a 32 x 32 quarter as 4 x 4 fragments of 8 x 8.  Both
// MMA operands are plain elements of Y: A(c, p) = Y[p][c], B(p, d) = Y[p][d],
// staged per 32-row panel in shared memory (fp64, odd pitch).
__device__ __forceinline__ void dmma_8x8x4(double* c, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <class T>
__global__ void __launch_bounds__(128) gram_dmma_kernel(const T* __restrict__ Y, int64_t ld, int64_t rows, int64_t l,
                                                        int64_t chunk, double* __restrict__ W) {
    constexpr int LD = 65;  // odd pitch (doubles): the 4 k-rows of a fragment hit different banks
    __shared__ double As[32 * LD], Bs[32 * LD];
    int ci = 0;
    while ((ci + 1) * (ci + 2) / 2 <= (int)blockIdx.x) ++ci;
    const int di = (int)blockIdx.x - ci * (ci + 1) / 2;
    const int64_t c0 = ci * 64, d0 = di * 64;
    const int64_t p0 = blockIdx.y * chunk, p1 = min(rows, p0 + chunk);
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const int wc = (warp >> 1) * 32, wd = (warp & 1) * 32;  // warp quarter of the 64 x 64 tile
    const int fr = lane >> 2, fk = lane & 3;                  // fragment row / k of this lane
    double acc[4][4][2] = {};
    T ra[16], rb[16];
    auto fetch = [&](int64_t p) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int e = t + 128 * j, r = e / 64, cc = e % 64;
            const int64_t pp = p + r;
            ra[j] = (pp < p1 && c0 + cc < l) ? Y[pp * ld + c0 + cc] : T(0);
            rb[j] = (pp < p1 && d0 + cc < l) ? Y[pp * ld + d0 + cc] : T(0);
        }
    };
    if (p0 < p1) fetch(p0);
    for (int64_t p = p0; p < p1; p += 32) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int e = t + 128 * j, r = e / 64, cc = e % 64;
            As[r * LD + cc] = (double)ra[j];
            Bs[r * LD + cc] = (double)rb[j];
        }
        __syncthreads();
        if (p + 32 < p1) fetch(p + 32);
#pragma unroll
        for (int k4 = 0; k4 < 32; k4 += 4) {
            double a[4], b[4];
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                a[f] = As[(k4 + fk) * LD + wc + 8 * f + fr];  // A(c = wc + 8f + fr, k)
                b[f] = Bs[(k4 + fk) * LD + wd + 8 * f + fr];  // B(k, d = wd + 8f + fr)
            }
#pragma unroll
            for (int fa = 0; fa < 4; ++fa)
#pragma unroll
                for (int fb = 0; fb < 4; ++fb) dmma_8x8x4(acc[fa][fb], a[fa], b[fb]);
        }
        __syncthreads();
    }
    // D fragment: row fr, columns 2 fk + {0, 1}
#pragma unroll
    for (int fa = 0; fa < 4; ++fa)
#pragma unroll
        for (int fb = 0; fb < 4; ++fb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t c = c0 + wc + 8 * fa + fr, d = d0 + wd + 8 * fb + 2 * fk + h;
                if (c >= l || d >= l) continue;
                atomicAdd(&W[c * l + d], acc[fa][fb][h]);
                if (ci != di) atomicAdd(&W[d * l + c], acc[fa][fb][h]);
            }
}

// Shifted Cholesky W + shift I = R^T R and Rinv = R^{-1} in one CTA with the
// l x l matrix in shared memory (l <= 160): right-looking factorisation, then
// the in-place column-by-column inverse of the upper triangle.  The shift is
// rel * trace(W) / l (shifted CholeskyQR keeps rank-deficient Grams defined).
__global__ void __launch_bounds__(1024) chol_inv_smem_kernel(const double* __restrict__ Wg, int l, double rel,
                                                             double* __restrict__ Rinv) {
    extern __shared__ double R[];  // l x l, row-major
    __shared__ double shift_s;
    __shared__ double red[32];
    const int t = threadIdx.x, nt = blockDim.x;
    double part = 0.0;
    for (int i = t; i < l * l; i += nt) {
        const double v = Wg[i];
        R[i] = v;
        if (i / l == i % l) part += v;
    }
    for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if ((t & 31) == 0) red[t >> 5] = part;
    __syncthreads();
    if (t == 0) {
        double tr = 0.0;
        for (int w = 0; w < nt / 32; ++w) tr += red[w];
        shift_s = rel * tr / (double)l;
    }
    __syncthreads();
    for (int i = t; i < l; i += nt) R[i * l + i] += shift_s;
    __syncthreads();
    // upper Cholesky: row j of R, then the trailing upper triangle
    for (int j = 0; j < l; ++j) {
        const double d = R[j * l + j];
        const double rjj = sqrt(d > 0.0 ? d : 1e-300);
        __syncthreads();
        for (int c = j + 1 + t; c < l; c += nt) R[j * l + c] /= rjj;
        if (t == 0) R[j * l + j] = rjj;
        __syncthreads();
        const int m = l - j - 1;
        for (int idx = t; idx < m * m; idx += nt) {
            const int r = j + 1 + idx / m, c = j + 1 + idx % m;
            if (c >= r) R[r * l + c] -= R[j * l + r] * R[j * l + c];
        }
        __syncthreads();
    }
    // in-place inverse of the upper triangle, one column at a time:
    // X[j][j] = 1 / R[j][j];  X[i][j] = -X[j][j] * sum_{i<=m<j} X[i][m] R[m][j]
    for (int j = 0; j < l; ++j) {
        const double xjj = 1.0 / R[j * l + j];
        double v = 0.0;
        if (t < j) {
            for (int m = t; m < j; ++m) v += R[t * l + m] * R[m * l + j];
            v *= -xjj;
        }
        __syncthreads();
        if (t < j) R[t * l + j] = v;
        if (t == 0) R[j * l + j] = xjj;
        __syncthreads();
    }
    for (int i = t; i < l * l; i += nt) Rinv[i] = (i % l >= i / l) ? R[i] : 0.0;
}

// In-place upper Cholesky W = R^T R and Rinv = R^{-1}, one CTA (l <= 1024).
// A diagonal shift rel * trace(W) / l keeps rank-deficient Grams
// factorisable (shifted CholeskyQR); it is formed here, not on the host.
__global__ void chol_inv_kernel(double* W, int64_t l, double rel, double* Rinv) {
    __shared__ double shift_s;
    const int t = threadIdx.x;
    if (t == 0) {
        double tr = 0.0;
        for (int64_t i = 0; i < l; ++i) tr += W[i * l + i];
        shift_s = rel * tr / (double)l;
    }
    __syncthreads();
    const double shift = shift_s;
    for (int64_t i = t; i < l; i += blockDim.x) W[i * l + i] += shift;
    __syncthreads();
    // right-looking Cholesky on the upper triangle (row-major W)
    for (int64_t j = 0; j < l; ++j) {
        if (t == 0) {
            double d = W[j * l + j];
            W[j * l + j] = sqrt(d > 0.0 ? d : 1e-300);
        }
        __syncthreads();
        const double rjj = W[j * l + j];
        for (int64_t c = j + 1 + t; c < l; c += blockDim.x) W[j * l + c] /= rjj;
        __syncthreads();
        for (int64_t idx = t; idx < (l - j - 1) * (l - j - 1); idx += blockDim.x) {
            const int64_t r = j + 1 + idx / (l - j - 1), c = j + 1 + idx % (l - j - 1);
            if (c >= r) W[r * l + c] -= W[j * l + r] * W[j * l + c];
        }
        __syncthreads();
    }
    // Rinv: solve R X = I column by column (back substitution), upper triangular
    for (int64_t c = t; c < l; c += blockDim.x) {
        for (int64_t r = l - 1; r >= 0; --r) {
            double s = (r == c) ? 1.0 : 0.0;
            for (int64_t m = r + 1; m <= c; ++m) s -= W[r * l + m] * Rinv[m * l + c];
            Rinv[r * l + c] = r <= c ? s / W[r * l + r] : 0.0;
        }
    }
}

// Parallel cyclic Jacobi on a symmetric l x l matrix in one CTA (blockDim
// 128 x 8): each round rotates the l/2 disjoint (p, q) pairs of a round-robin
// tournament; a thread per pair computes the rotation, all threads apply it
// (threadIdx.x walks the matrix index, threadIdx.y the pairs).  A lives in
// shared memory at an odd pitch when it fits (conflict-free column access);
// the eigenvectors are kept transposed (Vt row p = eigenvector p) so every
// rotation update is a pair of contiguous rows.  A rotation is skipped once
// |a_pq| is at fp64 roundoff of its diagonal pair (|a_pq| <= 1e-15
// sqrt|a_pp a_qq|, or below 1e-18 ||A||_F); a sweep without rotations ends
// the iteration (the threshold Jacobi method).  Out: A's diagonal holds the
// eigenvalues, V (l x l, row-major) the eigenvectors by columns.
template <class VT, bool SMEM>
__global__ void __launch_bounds__(1024) jacobi_kernel(double* Ag, double* V, int l, int max_sweeps,
                                                      int* sweeps_out, int a_in_smem_rt) {
    // SMEM: A (and for fp32 vectors Vt) statically in shared memory, so every
    // rotation is LDS/STS, never a generic access
    const int a_in_smem = SMEM ? 1 : a_in_smem_rt;
    extern __shared__ double sh[];
    const int m = l + (l & 1);  // pad to even with a dummy index
    const int np = m / 2;
    double* cs = sh;            // cos per pair
    double* sn = sh + np;       // sin per pair
    int* pp = reinterpret_cast<int*>(sh + m);
    int* qq = pp + np;
    const int lda = a_in_smem ? l + ((l + 1) & 1) : l;  // odd pitch in shared memory
    double* A = SMEM ? sh + m + np + 1 : (a_in_smem ? sh + m + np + 1 : Ag);
    // transposed eigenvectors: fp64 in place in V, or fp32 in shared memory
    // after A (the eigenvalues come from A's fp64 rotations either way)
    VT* Vt;
    if constexpr (sizeof(VT) == 8) Vt = reinterpret_cast<VT*>(V);
    else Vt = reinterpret_cast<VT*>(A + l * lda);
    __shared__ int nrot;
    __shared__ double red[32];
    const int tx = threadIdx.x, ty = threadIdx.y, t = ty * blockDim.x + tx, nt = blockDim.x * blockDim.y;
    double part = 0.0;
    for (int r = ty; r < l; r += blockDim.y)
        for (int c = tx; c < l; c += blockDim.x) {
            const double v = Ag[r * l + c];
            part += v * v;
            if (a_in_smem) A[r * lda + c] = v;
            Vt[r * l + c] = r == c ? VT(1) : VT(0);
        }
    for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if ((t & 31) == 0) red[t >> 5] = part;
    __syncthreads();
    if (t == 0) {
        double f = 0.0;
        for (int w = 0; w < nt / 32; ++w) f += red[w];
        red[0] = sqrt(f);
    }
    __syncthreads();
    const double tiny = 1e-18 * red[0];
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        if (t == 0) nrot = 0;
        __syncthreads();
        for (int round = 0; round < m - 1; ++round) {
            for (int k = t; k < np; k += nt) {
                // circle method: index 0 fixed, others rotate
                const int x0 = k, x1 = m - 1 - k;
                int a = x0 == 0 ? 0 : 1 + (x0 - 1 + round) % (m - 1);
                int b = x1 == 0 ? 0 : 1 + (x1 - 1 + round) % (m - 1);
                if (a > b) { const int tmp = a; a = b; b = tmp; }
                pp[k] = a;
                qq[k] = b;
                double c = 1.0, s = 0.0;
                if (b < l) {
                    const double apq = A[a * lda + b], app = A[a * lda + a], aqq = A[b * lda + b];
                    if (fabs(apq) > fmax(1e-15 * sqrt(fabs(app * aqq)), tiny)) {
                        const double th = 0.5 * (aqq - app) / apq;
                        double tt = 1.0 / (fabs(th) + sqrt(1.0 + th * th));
                        if (th < 0.0) tt = -tt;
                        c = rsqrt(1.0 + tt * tt);
                        s = tt * c;
                        nrot = 1;  // any rotation this sweep (a plain store: no atomic serialisation)
                    }
                }
                cs[k] = c;
                sn[k] = s;
            }
            __syncthreads();
            // A <- J^T A J in one pass: for pair-indices (k, g), k <= g, the 2 x 2
            // block A[{a_k, b_k}, {a_g, b_g}] becomes J_k^T B J_g (J = [[c, s], [-s, c]]),
            // written with its mirror; the eigenvector rows a_k, b_k of Vt rotate
            // in the same phase (rows and blocks are disjoint within a round)
            {
                const int nb = np * (np + 1) / 2;
                for (int idx = t; idx < nb; idx += nt) {
                    // triangular index -> (k, g), k <= g
                    int k = (int)((sqrtf(8.f * idx + 1.f) - 1.f) * 0.5f);
                    while ((k + 1) * (k + 2) / 2 <= idx) ++k;
                    while (k * (k + 1) / 2 > idx) --k;
                    const int g = idx - k * (k + 1) / 2;  // g <= k: block (g, k)
                    const int ak = pp[g], bk = qq[g], ag = pp[k], bg = qq[k];
                    const double ck = cs[g], sk = sn[g], cg = cs[k], sg = sn[k];
                    if ((sk == 0.0 && sg == 0.0)) continue;
                    const bool vk = bk < l, vg = bg < l;  // the padded dummy index is never stored
                    double b00 = A[ak * lda + ag], b01 = vg ? A[ak * lda + bg] : 0.0;
                    double b10 = vk ? A[bk * lda + ag] : 0.0, b11 = (vk && vg) ? A[bk * lda + bg] : 0.0;
                    // right: columns (a_g, b_g) by J_g
                    double t00 = cg * b00 - sg * b01, t01 = sg * b00 + cg * b01;
                    double t10 = cg * b10 - sg * b11, t11 = sg * b10 + cg * b11;
                    // left: rows (a_k, b_k) by J_k^T
                    b00 = ck * t00 - sk * t10; b10 = sk * t00 + ck * t10;
                    b01 = ck * t01 - sk * t11; b11 = sk * t01 + ck * t11;
                    A[ak * lda + ag] = b00;
                    if (vg) A[ak * lda + bg] = b01;
                    if (vk) A[bk * lda + ag] = b10;
                    if (vk && vg) A[bk * lda + bg] = b11;
                    if (g != k) {  // mirror
                        A[ag * lda + ak] = b00;
                        if (vg) A[bg * lda + ak] = b01;
                        if (vk) A[ag * lda + bk] = b10;
                        if (vk && vg) A[bg * lda + bk] = b11;
                    }
                }
                for (int k = ty; k < np; k += blockDim.y) {
                    const double s = sn[k];
                    if (s == 0.0) continue;
                    const int a = pp[k], b = qq[k];
                    if (b >= l) continue;
                    const double c = cs[k];
                    for (int i = tx; i < l; i += blockDim.x) {
                        const VT vx = Vt[a * l + i], vy = Vt[b * l + i];
                        Vt[a * l + i] = (VT)c * vx - (VT)s * vy;
                        Vt[b * l + i] = (VT)s * vx + (VT)c * vy;
                    }
                }
            }
            __syncthreads();
        }
        if (nrot == 0) break;
        __syncthreads();
    }
    if (a_in_smem)
        for (int r = ty; r < l; r += blockDim.y)
            for (int c = tx; c < l; c += blockDim.x) Ag[r * l + c] = A[r * lda + c];
    __syncthreads();
    if constexpr (sizeof(VT) == 8) {  // Vt -> V in place (swap across the diagonal)
        for (int r = ty; r < l; r += blockDim.y)
            for (int c = tx; c < r; c += blockDim.x) {
                const double x = Vt[r * l + c];
                Vt[r * l + c] = Vt[c * l + r];
                Vt[c * l + r] = x;
            }
    } else {
        for (int r = ty; r < l; r += blockDim.y)
            for (int c = tx; c < l; c += blockDim.x) V[r * l + c] = (double)Vt[c * l + r];
    }
    if (t == 0) *sweeps_out = sweep;
}

// one-CTA symmetric eigensolve of the l x l matrix A (in place: diagonal =
// eigenvalues, V = eigenvectors by columns)
inline unsigned jacobi_ty() {  // dev knob: rows of 128 threads in the Jacobi CTA
    static const unsigned ty = getenv("CURVKIT_JACOBI_TY") ? (unsigned)atoi(getenv("CURVKIT_JACOBI_TY")) : 8;
    return ty;
}

// fp32_vectors: accumulate the rotations of the eigenvectors in fp32 shared
// memory (enough for fp32 outputs), so no rotation touches global memory.
inline void jacobi_eig(double* A, double* V, int64_t l, int* sweeps, cudaStream_t s, bool fp32_vectors = false) {
    const int64_t m = l + (l & 1);
    const size_t base = (size_t)(m + m / 2 + 1) * sizeof(double);
    const size_t with_a = base + (size_t)l * (l + 1 + ((l + 1) & 1)) * sizeof(double);
    const size_t with_v = with_a + (size_t)l * l * sizeof(float);
    func_attr_once((const void*)jacobi_kernel<double, false>, [] {
        CK_CUDA(cudaFuncSetAttribute(jacobi_kernel<double, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
        CK_CUDA(cudaFuncSetAttribute(jacobi_kernel<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
    });
    if (fp32_vectors && with_v <= 200 * 1024) {
        jacobi_kernel<float, true><<<1, dim3(128, jacobi_ty()), with_v, s>>>(A, V, (int)l, 60, sweeps, 1);
    } else {
        const bool smem_a = with_a <= 200 * 1024;
        jacobi_kernel<double, false><<<1, dim3(128, 8), smem_a ? with_a : base, s>>>(A, V, (int)l, 60, sweeps,
                                                                                  smem_a ? 1 : 0);
    }
    CK_LAUNCH();
}

template <class U>
__global__ void convert_d_kernel(const double* in, U* out, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (U)in[i];
}

// dst (rows x cols, ldd; padding zeroed) = src rounded to nearest TF32
template <class T>
__global__ void copy_rn_kernel(const T* __restrict__ src, int64_t lds, T* __restrict__ dst, int64_t ldd, int64_t rows,
                               int64_t cols) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * ldd;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / ldd, c = i - r * ldd;
        if constexpr (sizeof(T) == 4) dst[i] = c < cols ? round_tf32(src[r * lds + c]) : T(0);
        else dst[i] = c < cols ? src[r * lds + c] : T(0);
    }
}

template <class T>
void convert_rows_rn(const T* src, int64_t lds, T* dst, int64_t ldd, int64_t rows, int64_t cols, cudaStream_t s) {
    copy_rn_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(rows * ldd, 256), 148 * 64), 256, 0, s>>>(src, lds, dst,
                                                                                                       ldd, rows, cols);
    CK_LAUNCH();
}

template <class T>
struct EigenWork {
    const ModelDesc& md;
    cudaStream_t s;
    int prec;
    const Cache<T>* c = nullptr;
    const KrOperands* kr = nullptr;  // set: J X / J^T T from the activations (J never formed)
    TopkShard sh{};                  // parameter rows of this rank (all of them unsharded)
    const Comm* comm = nullptr;      // sums J X partials and Grams across ranks

    // Y <- orth(Y) (CholeskyQR2, fp64 Gram): pass 1 writes Y Rinv into the
    // scratch Y2, pass 2 writes back into Y; no host round trip
    // passes = 1 (between power iterations: the fp64 Gram keeps the basis
    // well conditioned) or 2 (CholeskyQR2, the final basis); returns the
    // buffer holding the result (Y after 2 passes, Y2 after 1)
    T* orth(T* Y, T* Y2, int64_t rows, int64_t l, int64_t ld, int passes = 2) {
        ProfScope ps("eig_orth", s, 2.0 * 2.0 * 2.0 * (double)rows * l * l, 2.0 * 2.0 * 2.0 * sizeof(T) * rows * ld);
        DevMem W((size_t)l * l * sizeof(double), s), Rinv((size_t)l * l * sizeof(double), s);
        DevMem Rt((size_t)l * l * sizeof(T), s);
        T* src = Y;
        T* dst = Y2;
        for (int pass = 0; pass < passes; ++pass) {
            ProfScope p1("orth_gram", s, 0.0, 0.0);
            CK_CUDA(cudaMemsetAsync(W.p, 0, l * l * sizeof(double), s));
            {
                const int64_t lt = ceil_div(l, 64), tiles = lt * (lt + 1) / 2;
                const int64_t ksplit = std::min<int64_t>(ceil_div(4 * 148, tiles), std::max<int64_t>(1, rows / 2048));
                gram_dmma_kernel<T><<<dim3((unsigned)tiles, (unsigned)ksplit), 128, 0, s>>>(src, ld, rows, l,
                                                                                        ceil_div(rows, ksplit),
                                                                                        dptr<double>(W));
                CK_LAUNCH();
            }
            if (comm) comm->sum(dptr<double>(W), (size_t)(l * l), s);  // Gram of all ranks' rows
            p1.end();
            ProfScope p2("orth_chol", s, 0.0, 0.0);
            chol_inv(dptr<double>(W), l, sizeof(T) == 4 ? 1e-7 : 1e-14, dptr<double>(Rinv));
            convert_to<T>(dptr<double>(Rinv), dptr<T>(Rt), l * l);
            p2.end();
            ProfScope p3("orth_apply", s, 0.0, 0.0);
            EpiStore<T> e{dst, ld, 0, T(1), T(0)};
            bool done = false;
            if constexpr (std::is_same_v<T, float>) {
                if (tf32_class(prec) && rows >= 512 && l % 4 == 0) {  // fp32-grade products on the tensor cores
                    gemm_tf32(k3xTF32, s, rows, l, l, kmaj(src, ld), mnmaj(dptr<T>(Rt), l), e);
                    done = true;
                }
            }
            if (!done) gemm_simt<T>(s, rows, l, l, 1, kmaj(src, ld), mnmaj(dptr<T>(Rt), l), e);
            p3.end();
            std::swap(src, dst);
        }
        return src;
    }

    // shifted Cholesky + inverse of the l x l Gram (shared memory when it fits)
    void chol_inv(double* W, int64_t l, double rel, double* Rinv) {
        const size_t bytes = (size_t)l * l * sizeof(double);
        if (bytes <= 200 * 1024) {
            func_attr_once((const void*)chol_inv_smem_kernel, [] {
                CK_CUDA(cudaFuncSetAttribute(chol_inv_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024));
            });
            chol_inv_smem_kernel<<<1, 1024, bytes, s>>>(W, (int)l, rel, Rinv);
        } else {
            chol_inv_kernel<<<1, 256, 0, s>>>(W, l, rel, Rinv);
        }
        CK_LAUNCH();
    }

    template <class U>
    void convert_to(const double* in, U* out, int64_t n) {
        convert_d_kernel<U><<<blocks_for(n), 256, 0, s>>>(in, out, n);
        CK_LAUNCH();
    }

    // T_out (n x l) = J X ; X is P x l (ld lx)
    void apply_j(const T* J, int64_t ldj, int64_t n, const T* X, int64_t ldx, int64_t l, T* Tout, int64_t ldt) {
        ProfScope ps("eig_apply_j", s, 2.0 * (double)n * md.P * l, kr ? 0.0 : (double)sizeof(T) * n * md.P);
        if constexpr (std::is_same_v<T, float>) {
            if (kr) {
                kr_apply_j(md, *c, *kr, sh, X, ldx, l, Tout, ldt, s);
                if (comm) comm->sum(Tout, (size_t)(n * ldt), s);  // J X = sum over ranks' rows
                return;
            }
            if (tf32_class(prec) || prec == k3xTF32) {  // split-K: only ceil(N/256) row tiles
                gemm_tf32_store(prec, s, n, l, md.P, read_once(pre_rounded(kmaj(J, ldj))), mnmaj(X, ldx), Tout,
                                ldt);
                return;
            }
        }
        EpiStore<T> e{Tout, ldt, 0, T(1), T(0)};
        CurvGemm<T, EpiStore<T>>::run(prec, s, n, l, md.P, pre_rounded(kmaj(J, ldj)), mnmaj(X, ldx), e);
    }
    // Y (P x l) = J^T Tn ; Tn is n x l
    void apply_jt(const T* J, int64_t ldj, int64_t n, const T* Tn, int64_t ldt, int64_t l, T* Y, int64_t ldy) {
        ProfScope ps("eig_apply_jt", s, 2.0 * (double)n * md.P * l, kr ? 0.0 : (double)sizeof(T) * n * md.P);
        if constexpr (std::is_same_v<T, float>) {
            if (kr) {
                kr_apply_jt(md, *c, *kr, sh, Tn, ldt, l, Y, ldy, s);
                return;
            }
        }
        EpiStore<T> e{Y, ldy, 0, T(1), T(0)};
        CurvGemm<T, EpiStore<T>>::run(prec, s, md.P, l, n, read_once(pre_rounded(mnmaj(J, ldj))), mnmaj(Tn, ldt), e);
    }
};

// Core driver: leaves eigenvectors (rows of this rank's shard x k, row-major,
// ld k) in q_dev and eigenvalues (k, descending) in lam_host.  With a
// communicator of nranks > 1 each rank holds the parameter rows of
// TopkShard::make(md, nranks, rank); the only exchanges are all-reduces of
// the N x l product J X and of the l x l Grams.
__global__ void scale_kernel(double* __restrict__ a, int64_t n, double f) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] *= f;
}

// out (l x k, row-major) = V[:, sel] (V l x l, eigenvectors by columns)
template <class T>
__global__ void select_columns_kernel(const double* __restrict__ V, int64_t l, const int32_t* __restrict__ sel,
                                      int64_t k, T* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < l * k) out[i] = (T)V[(i / k) * l + sel[i % k]];
}

// C <- sc C + sb B + sa A on the first l columns of R rows (one Chebyshev
// three-term step; A may be null)
template <class T>
__global__ void cheb_combine_kernel(T* __restrict__ C, const T* __restrict__ B, const T* __restrict__ A, int64_t rows,
                                    int64_t ld, int64_t l, T sc, T sb, T sa) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * l; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / l, j = r * ld + (i - r * l);
        T v = sc * C[j] + sb * B[j];
        if (A) v += sa * A[j];
        C[j] = v;
    }
}

// Filter: cheb_degree > 0 replaces the power iterations by cheb_steps rounds of
// Chebyshev-filtered subspace iteration (power_iters is then unused).  Each
// round takes the smallest Ritz value theta_l of the current basis as the
// upper end b of the damped interval [0, b] (G is PSD) and applies
// T_d((2 G - b) / b) by the three-term recurrence, d = cheb_degree operator
// applications; eigenvalues above b grow like cosh(d acosh(2 lambda / b - 1)),
// against (lambda / lambda')^d for d power iterations.
template <class T>
void topk_core(const ModelDesc& md, const Cache<T>& c, int64_t k, int64_t oversample, int64_t power_iters,
               uint64_t seed, int prec, T* q_dev, std::vector<double>& lam_host, cudaStream_t s,
               const Comm* comm = nullptr, const T* Jext = nullptr, int64_t ldj_ext = 0, int64_t cheb_steps = 0,
               int64_t cheb_degree = 0, double cheb_tol = 0.0) {
    const int64_t n = c.n, P = md.P;
    const bool sharded = comm && comm->nranks > 1;
    const TopkShard sh = TopkShard::make(md, sharded ? comm->nranks : 1, sharded ? comm->rank : 0);
    const int64_t R = sh.rows();
    if (k < 1 || k > std::min(n, P))
        throw CurvError(kContractError, "opg_topk: need 1 <= k <= min(N, P), got k = " + std::to_string(k));
    if (oversample < 0 || power_iters < 0) throw CurvError(kContractError, "opg_topk: negative oversample/power_iters");
    if (cheb_steps < 0 || cheb_degree < 0) throw CurvError(kContractError, "opg_topk: negative filter steps/degree");
    const int64_t l = std::min(k + oversample, P);
    const int64_t ldl = round_up(l, 32);
    // TF32: J X and J^T T straight from the activations and deltas (kr.cuh);
    // otherwise the per-example gradients are formed once and stay in HBM
    // a caller's J (opg_eigs_incremental's input): used as is, or -- TF32 --
    // through one copy rounded to nearest TF32 (the products take it pre-rounded)
    const bool ext = Jext != nullptr;
    std::unique_ptr<KrOperands> krop;
    if constexpr (std::is_same_v<T, float>)
        if (!ext && tf32_class(prec) && kr_supported(md, c))
            krop = std::make_unique<KrOperands>(md, c, s, prec == kF16S);
    if (sharded && !krop) throw CurvError(kContractError, "sharded opg_topk needs TF32 precision");
    const bool ext_copy = ext && tf32_class(prec);
    const int64_t ldj = ext && !ext_copy ? ldj_ext : (krop ? 0 : round_up(P, 32));
    DevMem J((size_t)((ext && !ext_copy) ? 0 : n * ldj) * sizeof(T), s);
    if (ext_copy) {
        convert_rows_rn<T>(Jext, ldj_ext, dptr<T>(J), ldj, n, P, s);
    } else if (!ext && !krop) {
        jacobian<T>(md, c, 0, n, dptr<T>(J), ldj, s, tf32_class(prec));  // TF32: stored pre-rounded
    }
    const T* Jp = (ext && !ext_copy) ? Jext : dptr<T>(J);
    const size_t rbytes = (size_t)std::max<int64_t>(R, 1) * ldl * sizeof(T);
    DevMem Y(rbytes, s), Om(rbytes, s), Y2(rbytes, s);
    DevMem Tn((size_t)n * ldl * sizeof(T), s);
    CK_CUDA(cudaMemsetAsync(Tn.p, 0, (size_t)n * ldl * sizeof(T), s));
    {
        ProfScope ps("eig_sketch", s, 0.0, (double)sizeof(T) * R * ldl);
        CK_CUDA(cudaMemsetAsync(Om.p, 0, rbytes, s));
        if (R > 0) {
            gaussian_kernel<T><<<blocks_for(R * l), 256, 0, s>>>(dptr<T>(Om), R, l, ldl, seed, sh.p0);
            CK_LAUNCH();
        }
    }
    EigenWork<T> ew{md, s, prec, &c, krop.get(), sh, sharded ? comm : nullptr};
    // Rayleigh-Ritz on the orthonormal basis X: B = (1/N) (J X)^T (J X) with
    // round-to-nearest TF32 operands (J stored rounded, X rounded per GEMM):
    // unbiased products.  B is scaled and diagonalised on the device (Bm ->
    // Ritz values on its diagonal, V the vectors); only the l Ritz values come
    // back to the host, for the stop rule and the filter bounds.  Sharded: the
    // ranks' Grams of the identical all-reduced J X are summed, so every rank
    // diagonalises the same bytes and takes the same decisions.
    DevMem Bm((size_t)l * l * sizeof(double), s), V((size_t)l * l * sizeof(double), s);
    std::vector<double> theta(l);
    const double nr = sharded ? (double)comm->nranks : 1.0;
    auto ritz = [&](const T* X) {
        ew.apply_j(Jp, ldj, n, X, ldl, l, dptr<T>(Tn), ldl);
        ProfScope rr("eig_ritz", s, 2.0 * (double)n * l * l, 0.0);
        CK_CUDA(cudaMemsetAsync(Bm.p, 0, l * l * sizeof(double), s));
        {
            const int64_t ksplit = std::min<int64_t>(256, std::max<int64_t>(1, n / 2048));
            dim3 g((unsigned)ceil_div(l, 32), (unsigned)ceil_div(l, 32), (unsigned)ksplit);
            gram_kernel<T><<<g, 256, 0, s>>>(dptr<T>(Tn), ldl, n, l, ceil_div(n, ksplit), dptr<double>(Bm));
            CK_LAUNCH();
        }
        if (sharded) comm->sum(dptr<double>(Bm), (size_t)(l * l), s);
        scale_kernel<<<blocks_for(l * l), 256, 0, s>>>(dptr<double>(Bm), l * l, 1.0 / ((double)n * nr));
        CK_LAUNCH();
        ProfScope pj("eig_ritz_eig", s, 0.0, 0.0);
        DevMem sw(sizeof(int), s);
        jacobi_eig(dptr<double>(Bm), dptr<double>(V), l, dptr<int>(sw), s, std::is_same_v<T, float>);
        CK_CUDA(cudaMemcpy2DAsync(theta.data(), sizeof(double), Bm.p, (l + 1) * sizeof(double), sizeof(double), l,
                                  cudaMemcpyDeviceToHost, s));
        int sweeps = 0;
        CK_CUDA(cudaMemcpyAsync(&sweeps, sw.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK_CUDA(cudaStreamSynchronize(s));
        if (getenv("CURVKIT_TRACE"))
            fprintf(stderr, "[curvkit] Rayleigh-Ritz Jacobi: l = %lld, %d sweeps\n", (long long)l, sweeps);
    };
    auto top_k = [&]() {  // the k largest Ritz values, descending
        std::vector<double> t(theta);
        std::sort(t.begin(), t.end(), std::greater<double>());
        t.resize(k);
        return t;
    };
    T* X = dptr<T>(Om);
    bool have_ritz = false;  // theta / V belong to the final X
    if (cheb_degree == 0) {
        for (int64_t it = 0; it <= power_iters; ++it) {
            ew.apply_j(Jp, ldj, n, X, ldl, l, dptr<T>(Tn), ldl);
            ew.apply_jt(Jp, ldj, n, dptr<T>(Tn), ldl, l, dptr<T>(Y), ldl);
            X = ew.orth(dptr<T>(Y), dptr<T>(Y2), R, l, ldl, it < power_iters ? 1 : 2);
        }
    } else {
        ew.apply_j(Jp, ldj, n, X, ldl, l, dptr<T>(Tn), ldl);
        ew.apply_jt(Jp, ldj, n, dptr<T>(Tn), ldl, l, dptr<T>(Y), ldl);
        X = ew.orth(dptr<T>(Y), dptr<T>(Y2), R, l, ldl, 2);  // -> Y
        T* bufs[3] = {dptr<T>(Y), dptr<T>(Om), dptr<T>(Y2)};
        const int64_t budget = cheb_steps * cheb_degree;  // operator applications
        // stop rule (cheb_tol > 0): Ritz values rise monotonically to the
        // eigenvalues; with the change d_t of round t and the contraction
        // rho = d_t / d_{t-1}, the remaining error is ~ d_t rho / (1 - rho).  A
        // value has converged when that is <= cheb_tol (relative), or when its
        // change is at the arithmetic's noise floor.
        const double floor_rel = sizeof(T) == 8 ? 1e-13 : 2e-5;
        std::vector<double> prev, prevd;
        for (int64_t used = 0; used < budget;) {
            ritz(X);  // Tn = J X: also the first operator application of the filter below
            have_ritz = true;
            if (cheb_tol > 0.0) {
                const std::vector<double> t = top_k();
                bool done = !prev.empty();
                std::vector<double> d(k, 0.0);
                for (int64_t j = 0; j < k && !prev.empty(); ++j) {
                    d[j] = t[j] - prev[j];
                    const double c = std::fabs(d[j]) / std::max(std::fabs(t[j]), 1e-300);
                    bool ok = c <= floor_rel;
                    if (!ok && !prevd.empty() && prevd[j] > 0.0 && d[j] >= 0.0) {
                        const double rho = d[j] / prevd[j];
                        ok = rho < 0.9 && c * rho / (1.0 - rho) <= cheb_tol;
                    }
                    done = done && ok;
                }
                if (getenv("CURVKIT_TRACE"))
                    fprintf(stderr, "[curvkit] filter round after %lld applications: theta_k %.8e%s\n", (long long)used,
                            t[k - 1], done ? " (converged)" : "");
                if (done) break;
                if (!prev.empty()) prevd = d;
                prev = t;
            }
            double b = INFINITY, top = 0.0;
            for (int64_t j = 0; j < l; ++j) {
                b = std::min(b, theta[j]);
                top = std::max(top, theta[j]);
            }
            if (!(b > 0.0)) break;  // basis already spans G's range (rank < l)
            // the filter grows the top Ritz direction by T_d(2 top / b - 1) against <= 1
            // on [0, b]: keep that range within ~2e4 (fp32 basis, CholeskyQR2) by
            // lowering this round's degree on steep spectra (degree 1 = a shifted
            // power step); the application budget stays steps x degree
            int64_t deg = cheb_degree;
            const double x1 = 2.0 * top / b - 1.0;
            if (x1 > 1.0) deg = std::clamp<int64_t>((int64_t)std::floor(9.9 / std::acosh(x1)), 1, cheb_degree);
            deg = std::min(deg, budget - used);
            used += deg;
            const double e = b / 2.0, cc = b / 2.0;  // [0, b] -> [-1, 1]
            ProfScope pf("eig_cheb_filter", s, 0.0, 0.0);
            T* Bp = X;
            T* Ap = nullptr;
            int free_idx[2], nf = 0;
            for (T* q : bufs)
                if (q != X) free_idx[nf++] = (int)(std::find(bufs, bufs + 3, q) - bufs);
            T* Cp = bufs[free_idx[0]];
            T* Dp = bufs[free_idx[1]];  // the third buffer
            for (int64_t d = 1; d <= deg; ++d) {
                if (d > 1) ew.apply_j(Jp, ldj, n, Bp, ldl, l, dptr<T>(Tn), ldl);  // d = 1: Tn = J X from ritz()
                ew.apply_jt(Jp, ldj, n, dptr<T>(Tn), ldl, l, Cp, ldl);  // C = J^T J B = N G B
                const double sc = (d == 1 ? 1.0 : 2.0) / (e * (double)n), sb = -(d == 1 ? 1.0 : 2.0) * cc / e;
                if (R > 0) {
                    cheb_combine_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(R * l, 256), 148 * 32), 256, 0, s>>>(
                        Cp, Bp, d == 1 ? nullptr : Ap, R, ldl, l, (T)sc, (T)sb, (T)-1.0);
                    CK_LAUNCH();
                }
                // rotate (A, B, C) <- (B, C, A or the third buffer)
                T* nextC = d == 1 ? Dp : Ap;
                Ap = Bp;
                Bp = Cp;
                Cp = nextC;
            }
            pf.end();
            T* scratch = Ap;  // free after the last step
            X = ew.orth(Bp, scratch, R, l, ldl, 2);  // 2 passes: the filtered columns differ in scale
            have_ritz = false;
        }
    }
    if (!have_ritz) ritz(X);
    std::vector<int64_t> ord(l);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return theta[a] > theta[b]; });
    lam_host.resize(k);
    std::vector<int32_t> sel(k);
    for (int64_t j = 0; j < k; ++j) {
        lam_host[j] = theta[ord[j]];
        sel[j] = (int32_t)ord[j];
    }
    // eigenvectors Q = X V[:, sel] (rows of this rank), on the tensor cores with
    // fp32-grade 3xTF32 products where the shape allows
    ProfScope pr("eig_ritz_vectors", s, 2.0 * (double)R * l * k, 0.0);
    DevMem Vk((size_t)l * k * sizeof(T), s), dsel((size_t)k * sizeof(int32_t), s);
    CK_CUDA(cudaMemcpyAsync(dsel.p, sel.data(), k * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    select_columns_kernel<T><<<blocks_for(l * k), 256, 0, s>>>(dptr<double>(V), l, dptr<int32_t>(dsel), k, dptr<T>(Vk));
    CK_LAUNCH();
    EpiStore<T> e{q_dev, k, 0, T(1), T(0)};
    bool done = false;
    if constexpr (std::is_same_v<T, float>) {
        if ((tf32_class(prec) || prec == k3xTF32) && R >= 512 && k % 4 == 0) {
            gemm_tf32(k3xTF32, s, R, k, l, kmaj(X, ldl), mnmaj(dptr<T>(Vk), k), e);
            done = true;
        }
    }
    if (!done && R > 0) gemm_simt<T>(s, R, k, l, 1, kmaj(X, ldl), mnmaj(dptr<T>(Vk), k), e);
    CK_CUDA(cudaStreamSynchronize(s));
}

template <class T>
void host_topk(const ModelDesc& md, const Cache<T>& c, int64_t k, int64_t oversample, int64_t power_iters,
               uint64_t seed, int prec, double* q_out, double* lambda_out, cudaStream_t s, int64_t cheb_steps = 0,
               int64_t cheb_degree = 0, double cheb_tol = 0.0) {
    DevMem q((size_t)md.P * k * sizeof(T), s);
    std::vector<double> lam;
    topk_core<T>(md, c, k, oversample, power_iters, seed, prec, dptr<T>(q), lam, s, nullptr, nullptr, 0, cheb_steps,
                 cheb_degree, cheb_tol);
    std::vector<T> hq((size_t)md.P * k);
    CK_CUDA(cudaMemcpyAsync(hq.data(), q.p, hq.size() * sizeof(T), cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 0; i < hq.size(); ++i) q_out[i] = (double)hq[i];
    for (int64_t j = 0; j < k; ++j) lambda_out[j] = lam[j];
}

template <class T>
void dev_topk(const ModelDesc& md, const Cache<T>& c, int64_t k, int64_t oversample, int64_t power_iters,
              uint64_t seed, int prec, T* q_dev, T* lam_dev, cudaStream_t s, const Comm* comm = nullptr,
              int64_t cheb_steps = 0, int64_t cheb_degree = 0, double cheb_tol = 0.0) {
    std::vector<double> lam;
    topk_core<T>(md, c, k, oversample, power_iters, seed, prec, q_dev, lam, s, comm, nullptr, 0, cheb_steps,
                 cheb_degree, cheb_tol);
    std::vector<T> hl(lam.begin(), lam.end());
    CK_CUDA(cudaMemcpyAsync(lam_dev, hl.data(), k * sizeof(T), cudaMemcpyHostToDevice, s));
    CK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace ck
