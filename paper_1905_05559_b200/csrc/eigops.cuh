// eigops.cuh -- what the reference does with eigenpairs (Q, lambda) once it
// has them (eigensolve.cpp:11-30 validate_eigen_pairs, :278-358 the low-rank
// operator Q diag(lambda) Q^T and its full-rank extension
// Q diag(lambda) Q^T + lambda_tilde (I - Q Q^T): materialize / apply /
// quadform), on the device.
//
//   materialize   one symmetric GEMM (Q diag(lambda - shift)) Q^T, K = k, on the
//                 engine of the curvature products (tcgen05 in the TF32 class,
//                 DMMA in fp64): lower tiles computed, mirrored in the epilogue,
//                 then shift added on the diagonal (shift = lambda_tilde or 0).
//                 Output bound: P^2 stored once.
//   apply         two HBM passes over Q (P x k): t = Q^T x (project_kernel,
//                 fixed-order two-stage reduction in fp64), then
//                 y = Q ((lambda - shift) t) + shift x (expand_kernel).  Several
//                 vectors share each pass.
//   quadform      sum_c lambda_c t_c^2 + lambda_tilde (x.x - t.t), from the
//                 projection pass alone (the reference's expression, fp64).
#pragma once

#include "common.cuh"
#include "curvature.cuh"
#include "eigen.cuh"
#include "gemm_tc.cuh"

namespace ck {
namespace eigops {

constexpr int kVecTile = 4;   // vectors sharing one pass over Q
constexpr int kColTile = 4;   // 32-column groups held in registers per pass (k <= 128 in one pass)

// qs[i][c] = q[i][c] (lambda[c] - shift), qp[i][c] = q[i][c]; columns [k, ldk) zero
template <class T>
__global__ void scale_cols_kernel(const T* __restrict__ q, int64_t ldq, const T* __restrict__ lam, T shift, int64_t p,
                                  int64_t k, T* __restrict__ qs, T* __restrict__ qp, int64_t ldk) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p * ldk) return;
    const int64_t r = i / ldk, c = i % ldk;
    const T v = c < k ? q[r * ldq + c] : T(0);
    qp[i] = v;
    qs[i] = c < k ? v * (lam[c] - shift) : T(0);
}

template <class T>
__global__ void add_diag_kernel(T* __restrict__ h, int64_t ldh, int64_t p, T v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < p) h[i * ldh + i] += v;
}

// H (p x p, ldh) = Q diag(lambda) Q^T [+ lambda_tilde (I - Q Q^T)]
template <class T>
void materialize(int prec, cudaStream_t s, int64_t p, int64_t k, const T* q, int64_t ldq, const T* lam, bool full,
                 double lambda_tilde, T* h, int64_t ldh) {
    if (k == 0) {  // no retained pairs: the zero matrix (the caller cleared h) plus lambda_tilde I
        if (full) {
            add_diag_kernel<T><<<(unsigned)ceil_div(p, 256), 256, 0, s>>>(h, ldh, p, (T)lambda_tilde);
            CK_LAUNCH();
        }
        return;
    }
    const int64_t ldk = round_up(k, 32);
    DevMem qs((size_t)p * ldk * sizeof(T), s), qp((size_t)p * ldk * sizeof(T), s);
    const T shift = full ? (T)lambda_tilde : T(0);
    ProfScope ps("eig_materialize", s, 2.0 * (double)p * (p + 1) / 2 * k, (double)sizeof(T) * p * p);
    scale_cols_kernel<T><<<(unsigned)ceil_div(p * ldk, 256), 256, 0, s>>>(q, ldq, lam, shift, p, k, dptr<T>(qs),
                                                                         dptr<T>(qp), ldk);
    CK_LAUNCH();
    EpiSymLower<T> e{h, ldh, T(1)};
    CurvGemm<T, EpiSymLower<T>>::run(prec, s, p, p, k, kmaj(dptr<T>(qs), ldk), kmaj(dptr<T>(qp), ldk), e);
    if (full) {
        add_diag_kernel<T><<<(unsigned)ceil_div(p, 256), 256, 0, s>>>(h, ldh, p, shift);
        CK_LAUNCH();
    }
}

// Partial projections of one row chunk: part[v][c][b] = sum_{i in chunk b} x[v][i] q[i][c]
// and part[v][k][b] = sum x[v][i]^2.  A warp takes rows i (four per iteration: 16
// loads in flight per lane), its lanes the columns c = lane + 32 j (coalesced rows
// of Q); the block's warps are summed through shared memory in warp order.
template <class T>
__global__ void __launch_bounds__(256) project_kernel(const T* __restrict__ q, int64_t ldq, int64_t p, int64_t k,
                                                      int64_t c0, const T* __restrict__ x, int64_t ldx, int nv,
                                                      int64_t chunk, double* __restrict__ part) {
    __shared__ double red[8][kVecTile][32 * kColTile + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = blockIdx.x * chunk, r1 = min(p, r0 + chunk);
    constexpr int RU = 4;  // rows per iteration
    T acc[kVecTile][kColTile] = {};
    T xx[kVecTile] = {};
    bool col[kColTile];
#pragma unroll
    for (int j = 0; j < kColTile; ++j) col[j] = c0 + lane + 32 * j < k;
    for (int64_t i = r0 + warp; i < r1; i += 8 * RU) {
        T qv[RU][kColTile], xv[RU][kVecTile];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int64_t r = i + 8 * u;
#pragma unroll
            for (int j = 0; j < kColTile; ++j) qv[u][j] = (r < r1 && col[j]) ? q[r * ldq + c0 + lane + 32 * j] : T(0);
#pragma unroll
            for (int v = 0; v < kVecTile; ++v) xv[u][v] = (r < r1 && v < nv) ? x[v * ldx + r] : T(0);
        }
#pragma unroll
        for (int u = 0; u < RU; ++u)
#pragma unroll
            for (int v = 0; v < kVecTile; ++v) {
#pragma unroll
                for (int j = 0; j < kColTile; ++j) acc[v][j] += xv[u][v] * qv[u][j];
                xx[v] += xv[u][v] * xv[u][v];
            }
    }
#pragma unroll
    for (int v = 0; v < kVecTile; ++v) {
#pragma unroll
        for (int j = 0; j < kColTile; ++j) red[warp][v][lane + 32 * j] = (double)acc[v][j];
        if (lane == 0) red[warp][v][32 * kColTile] = (double)xx[v];
    }
    __syncthreads();
    const int64_t nb = gridDim.x;
    for (int e = threadIdx.x; e < nv * (32 * kColTile + 1); e += 256) {
        const int v = e / (32 * kColTile + 1), cc = e % (32 * kColTile + 1);
        double sum = 0.0;
        for (int w = 0; w < 8; ++w) sum += red[w][v][cc];
        if (cc == 32 * kColTile) {
            if (c0 == 0) part[(v * (k + 1) + k) * nb + blockIdx.x] = sum;
        } else if (c0 + cc < k) {
            part[(v * (k + 1) + c0 + cc) * nb + blockIdx.x] = sum;
        }
    }
}

// sum of part[..][b] over the chunks b: lane l adds b = l, l + 32, ... in order,
// then a fixed shuffle tree (deterministic)
__device__ __forceinline__ double chunk_sum(const double* __restrict__ row, int64_t nb, int lane) {
    double s = 0.0;
    for (int64_t b = lane; b < nb; b += 32) s += row[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// t[v][c] = the chunk partials summed in fixed order (fp64); ts = (lambda - shift) t
// in T for the expansion; quad[v] = sum_c lambda_c t_c^2 + lambda_tilde (x.x - t.t)
// (eigensolve.cpp:294-299, :329-339).  One block per vector, one warp per column.
template <class T>
__global__ void __launch_bounds__(256) project_finish_kernel(const double* __restrict__ part, int64_t nblocks, int nv,
                                                             int64_t k, const T* __restrict__ lam, int full,
                                                             double lambda_tilde, T* __restrict__ ts, int64_t kt,
                                                             double* __restrict__ quad) {
    __shared__ double s_lt[8], s_tt[8];
    const int v = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* pv = part + (int64_t)v * (k + 1) * nblocks;
    double lt = 0.0, tt = 0.0;
    for (int64_t c = warp; c < k; c += 8) {
        const double t = chunk_sum(pv + c * nblocks, nblocks, lane);
        const double l = (double)lam[c];
        if (ts && lane == 0) ts[v * kt + c] = (T)((l - (full ? lambda_tilde : 0.0)) * t);
        lt += l * t * t;
        tt += t * t;
    }
    if (ts)  // the pad columns of the expansion's 16-byte groups
        for (int64_t c = k + threadIdx.x; c < kt; c += 256) ts[v * kt + c] = T(0);
    if (lane == 0) {
        s_lt[warp] = lt;
        s_tt[warp] = tt;
    }
    __syncthreads();
    if (warp == 0 && quad) {
        const double xx = chunk_sum(pv + k * nblocks, nblocks, lane);
        if (lane == 0) {
            double a = 0.0, b = 0.0;
            for (int i = 0; i < 8; ++i) {
                a += s_lt[i];
                b += s_tt[i];
            }
            quad[v] = full ? a + lambda_tilde * xx - lambda_tilde * b : a;
        }
    }
}

// y[v][i] = sum_c ts[v][c] q[i][c] + shift x[v][i].  A block stages kExpRows rows of
// Q (column chunks of ExpCols) in shared memory with coalesced loads; thread (row r,
// class g) then sums its row over the 16-byte column groups g, g + 4, ... (one
// LDS.128 of Q and one 16-byte load of ts per vector for W columns; the row pitch
// puts a quarter-warp's 16-byte reads on distinct banks), the four classes are
// added in fixed order, and y is stored coalesced along i.
constexpr int kExpRows = 64;
template <class T>
struct ExpTile {
    static constexpr int W = 16 / sizeof(T);           // elements per 16-byte group
    static constexpr int Cols = 1024 / sizeof(T);      // 256 (float) / 128 (double) columns per chunk
    static constexpr int Pitch = Cols + W;             // 260 / 130: 16-byte groups of 8 rows on distinct banks
    static constexpr size_t bytes = (size_t)(kExpRows * Pitch + 4 * kVecTile * kExpRows) * sizeof(T);
};

template <class T>
__global__ void __launch_bounds__(256) expand_kernel(const T* __restrict__ q, int64_t ldq, int64_t p, int64_t k,
                                                     const T* __restrict__ ts, int64_t kt, int nv, T shift,
                                                     const T* __restrict__ x, int64_t ldx, T* __restrict__ y,
                                                     int64_t ldy) {
    using E = ExpTile<T>;
    constexpr int W = E::W;
    struct alignas(16) Vec {
        T v[W];
    };
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* tile = reinterpret_cast<T*>(smem_raw);      // [kExpRows][Pitch]
    T* red = tile + kExpRows * E::Pitch;           // [4][kVecTile][kExpRows]
    const int t = threadIdx.x, r = t % kExpRows, g = t / kExpRows;
    const int64_t ntiles = ceil_div(p, kExpRows);
    for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        const int64_t i0 = tl * kExpRows;
        const int rows = (int)min((int64_t)kExpRows, p - i0);
        T acc[kVecTile] = {};
        for (int64_t c0 = 0; c0 < k; c0 += E::Cols) {
            const int cols = (int)min((int64_t)E::Cols, k - c0);
            const int colsw = (cols + W - 1) / W * W;
            __syncthreads();  // the previous chunk's readers are done
            if (ldq == k && cols == k) {  // the tile is one contiguous run of rows * k elements
                const T* src = q + i0 * k;
                const int total = rows * cols, dr = 256 / cols, dc = 256 % cols;
                int rr = t / cols, c = t % cols;
#pragma unroll 8
                for (int e = t; e < total; e += 256) {
                    tile[rr * E::Pitch + c] = src[e];
                    rr += dr;
                    c += dc;
                    if (c >= cols) {
                        c -= cols;
                        ++rr;
                    }
                }
            } else {
                for (int rr = t / 32; rr < rows; rr += 8) {
                    const T* src = q + (i0 + rr) * ldq + c0;
#pragma unroll 4
                    for (int c = t % 32; c < cols; c += 32) tile[rr * E::Pitch + c] = src[c];
                }
            }
            if (colsw != cols)  // zero the ragged end of the last 16-byte group
                for (int e = t; e < rows * (colsw - cols); e += 256)
                    tile[(e / (colsw - cols)) * E::Pitch + cols + e % (colsw - cols)] = T(0);
            __syncthreads();
            if (r < rows) {
                const T* row = tile + r * E::Pitch;
#pragma unroll 2
                for (int c = g * W; c < colsw; c += 4 * W) {
                    const Vec qv = *reinterpret_cast<const Vec*>(row + c);
#pragma unroll
                    for (int v = 0; v < kVecTile; ++v) {
                        if (v >= nv) break;
                        const Vec tv = *reinterpret_cast<const Vec*>(ts + v * kt + c0 + c);
#pragma unroll
                        for (int u = 0; u < W; ++u) acc[v] += qv.v[u] * tv.v[u];
                    }
                }
            }
        }
        __syncthreads();  // (k = 0: no chunk loop ran) red's previous readers are done
#pragma unroll
        for (int v = 0; v < kVecTile; ++v) red[(g * kVecTile + v) * kExpRows + r] = acc[v];
        __syncthreads();
        for (int e = t; e < nv * kExpRows; e += 256) {
            const int v = e / kExpRows, rr = e % kExpRows;
            if (rr >= rows) continue;
            T sum = red[(0 * kVecTile + v) * kExpRows + rr];
#pragma unroll
            for (int gg = 1; gg < 4; ++gg) sum += red[(gg * kVecTile + v) * kExpRows + rr];
            const int64_t i = i0 + rr;
            y[v * ldy + i] = sum + (shift != T(0) ? shift * x[v * ldx + i] : T(0));
        }
    }
}

// y (nvec x p, ldy) and/or quad (nvec, fp64) for x (nvec x p, ldx); y or quad may be null
template <class T>
void apply(cudaStream_t s, int64_t p, int64_t k, const T* q, int64_t ldq, const T* lam, bool full, double lambda_tilde,
           int64_t nvec, const T* x, int64_t ldx, T* y, int64_t ldy, double* quad) {
    if (nvec < 1) return;
    const int64_t nblocks = std::max<int64_t>(1, std::min<int64_t>(4 * 148, ceil_div(p, 256)));
    const int64_t chunk = ceil_div(p, nblocks);
    DevMem part((size_t)(nblocks * kVecTile * (k + 1)) * sizeof(double), s);
    const int64_t kt = round_up(std::max<int64_t>(k, 1), 4);
    DevMem ts((size_t)(kVecTile * kt) * sizeof(T), s);
    const T shift = full ? (T)lambda_tilde : T(0);
    const size_t smem = ExpTile<T>::bytes;
    func_attr_once((const void*)expand_kernel<T>, [smem] {
        CK_CUDA(cudaFuncSetAttribute(expand_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    ProfScope ps("eig_apply", s, 4.0 * (double)p * k * nvec, 2.0 * ceil_div(nvec, kVecTile) * sizeof(T) * p * k);
    for (int64_t v0 = 0; v0 < nvec; v0 += kVecTile) {
        const int nv = (int)std::min<int64_t>(kVecTile, nvec - v0);
        // (k = 0: one pass still sums x.x for the full-rank quadform)
        for (int64_t c0 = 0; c0 < std::max<int64_t>(k, 1); c0 += 32 * kColTile) {
            project_kernel<T><<<(unsigned)nblocks, 256, 0, s>>>(q, ldq, p, k, c0, x + v0 * ldx, ldx, nv, chunk,
                                                               dptr<double>(part));
            CK_LAUNCH();
        }
        project_finish_kernel<T><<<nv, 256, 0, s>>>(dptr<double>(part), nblocks, nv, k, lam, full ? 1 : 0, lambda_tilde,
                                                   y ? dptr<T>(ts) : nullptr, kt, quad ? quad + v0 : nullptr);
        CK_LAUNCH();
        if (!y) continue;
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(3 * 148, ceil_div(p, kExpRows)));
        expand_kernel<T><<<(unsigned)grid, 256, smem, s>>>(q, ldq, p, k, dptr<T>(ts), kt, nv, shift, x + v0 * ldx, ldx,
                                                          y + v0 * ldy, ldy);
        CK_LAUNCH();
    }
}

// max over i <= j of |(Q^T Q)[i][j] - delta_ij| from the fp64 Gram W (k x k)
__global__ void ortho_error_kernel(const double* __restrict__ W, int64_t k, double* __restrict__ out) {
    __shared__ double red[256];
    double m = 0.0;
    for (int64_t e = threadIdx.x; e < k * k; e += 256) {
        const int64_t i = e / k, j = e % k;
        if (j > i) continue;  // gram_dmma_kernel fills the lower tiles
        m = fmax(m, fabs(W[e] - (i == j ? 1.0 : 0.0)));
    }
    red[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < 256; ++i) m = fmax(m, red[i]);
        *out = m;
    }
}

// max |Q^T Q - I| (fp64 Gram on the FP64 tensor cores), for validate_eigen_pairs
template <class T>
double ortho_error(cudaStream_t s, int64_t p, int64_t k, const T* q, int64_t ldq) {
    DevMem W((size_t)(k * k + 1) * sizeof(double), s);
    CK_CUDA(cudaMemsetAsync(W.p, 0, (size_t)(k * k + 1) * sizeof(double), s));
    const int64_t lt = ceil_div(k, 64), tiles = lt * (lt + 1) / 2;
    const int64_t ksplit = std::min<int64_t>(ceil_div(4 * 148, tiles), std::max<int64_t>(1, p / 2048));
    gram_dmma_kernel<T><<<dim3((unsigned)tiles, (unsigned)ksplit), 128, 0, s>>>(q, ldq, p, k, ceil_div(p, ksplit),
                                                                            dptr<double>(W));
    CK_LAUNCH();
    ortho_error_kernel<<<1, 256, 0, s>>>(dptr<double>(W), k, dptr<double>(W) + k * k);
    CK_LAUNCH();
    double err = 0.0;
    CK_CUDA(cudaMemcpyAsync(&err, dptr<double>(W) + k * k, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaStreamSynchronize(s));
    return err;
}

}  // namespace eigops
}  // namespace ck
