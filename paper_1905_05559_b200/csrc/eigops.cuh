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

#include "comm.cuh"
#include "common.cuh"
#include "curvature.cuh"
#include "eigen.cuh"
#include "gemm_tc.cuh"

namespace ck {
namespace eigops {

constexpr int kVecTile = 4;   // vectors sharing one pass over Q

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
    static const bool lsu = getenv("CURVKIT_EIG_MAT_LSU") != nullptr;  // dev: blocks stored by the LSU instead of TMA boxes
    if (lsu) e.tma = 0;
    CurvGemm<T, EpiSymLower<T>>::run(prec, s, p, p, k, kmaj(dptr<T>(qs), ldk), kmaj(dptr<T>(qp), ldk), e);
    if (full) {
        add_diag_kernel<T><<<(unsigned)ceil_div(p, 256), 256, 0, s>>>(h, ldh, p, shift);
        CK_LAUNCH();
    }
}

template <class T>
struct alignas(16) Vec16 {
    static constexpr int W = 16 / sizeof(T);  // elements per 16-byte group
    T v[W];
};

// 16-byte read-once load (ld.global.cs: evict-first in L1/L2)
template <class T>
__device__ __forceinline__ Vec16<T> ld16_stream(const T* p) {
    uint4 u;
    asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p));
    Vec16<T> out;
    memcpy(&out, &u, 16);
    return out;
}

// Partial projections of one row chunk: part[v][c][b] = sum_{i in chunk b} x[v][i] q[i][c]
// and part[v][k][b] = sum x[v][i]^2.  A warp takes rows i, RU per iteration; lane l
// holds the 16-byte column group l of the pass (columns c0 + W l ..), so a row of
// the pass is one 16-byte load per lane (VEC: rows 16-byte aligned) and RU of them
// are in flight.  The block's warps are summed through shared memory in warp order.
template <class T, int NV, bool VEC>
__global__ void __launch_bounds__(256) project_kernel(const T* __restrict__ q, int64_t ldq, int64_t p, int64_t k,
                                                      int64_t c0, const T* __restrict__ x, int64_t ldx, int nv,
                                                      int64_t chunk, double* __restrict__ part) {
    using V = Vec16<T>;
    constexpr int W = V::W, PC = 32 * W, RU = 8;  // PC: columns per pass
    __shared__ double red[8][NV][PC + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = blockIdx.x * chunk, r1 = min(p, r0 + chunk);
    const int64_t cl = c0 + (int64_t)W * lane;  // this lane's first column
    // lanes past the last column group read group 0 instead (their sums are dropped below)
    const int64_t cld = cl < k ? cl : c0;
    T acc[NV][W] = {};
    T xx[NV] = {};
    auto rows_step = [&](int64_t i, auto full) {
        constexpr bool kFull = decltype(full)::value;  // all RU rows inside the chunk: loads without predicates
        V qv[RU];
        T xv[RU][NV];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int64_t r = i + 8 * u;
            const bool ok = kFull || r < r1;
            if constexpr (VEC) {
                if (ok) {
                    qv[u] = ld16_stream<T>(q + r * ldq + cld);
                } else {
#pragma unroll
                    for (int w = 0; w < W; ++w) qv[u].v[w] = T(0);
                }
            } else {
#pragma unroll
                for (int w = 0; w < W; ++w) qv[u].v[w] = (ok && cl + w < k) ? q[r * ldq + cl + w] : T(0);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) xv[u][v] = (ok && v < nv) ? x[v * ldx + r] : T(0);
        }
#pragma unroll
        for (int u = 0; u < RU; ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
#pragma unroll
                for (int w = 0; w < W; ++w) acc[v][w] += xv[u][v] * qv[u].v[w];
                xx[v] += xv[u][v] * xv[u][v];
            }
    };
    int64_t i = r0 + warp;
    for (; i + 8 * (RU - 1) < r1; i += 8 * RU) rows_step(i, std::true_type{});
    if (i < r1) rows_step(i, std::false_type{});
#pragma unroll
    for (int v = 0; v < NV; ++v) {
#pragma unroll
        for (int w = 0; w < W; ++w) red[warp][v][W * lane + w] = (double)acc[v][w];
        if (lane == 0) red[warp][v][PC] = (double)xx[v];
    }
    __syncthreads();
    const int64_t nb = gridDim.x;
    for (int e = threadIdx.x; e < nv * (PC + 1); e += 256) {
        const int v = e / (PC + 1), cc = e % (PC + 1);
        double sum = 0.0;
        for (int w = 0; w < 8; ++w) sum += red[w][v][cc];
        if (cc == PC) {
            if (c0 == 0) part[(v * (k + 1) + k) * nb + blockIdx.x] = sum;
        } else if (c0 + cc < k) {  // (a VEC group's columns past k were read from the row's pitch: dropped here)
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

// tsum[v][c] = the chunk partials of column c (c = k: x.x) summed in fixed order
// (fp64); one warp per column
__global__ void __launch_bounds__(256) project_sum_kernel(const double* __restrict__ part, int64_t nblocks, int64_t k,
                                                          double* __restrict__ tsum) {
    const int v = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c = (int64_t)blockIdx.x * 8 + warp;
    if (c > k) return;
    const double t = chunk_sum(part + ((int64_t)v * (k + 1) + c) * nblocks, nblocks, lane);
    if (lane == 0) tsum[(int64_t)v * (k + 1) + c] = t;
}

// ts = (lambda - shift) t in T for the expansion (pitch kt, pad zeroed);
// quad[v] = sum_c lambda_c t_c^2 + lambda_tilde (x.x - t.t) (eigensolve.cpp:294-299,
// :329-339).  One block per vector; fixed summation order.
template <class T>
__global__ void __launch_bounds__(256) project_finish_kernel(const double* __restrict__ tsum, int64_t k,
                                                             const T* __restrict__ lam, int full, double lambda_tilde,
                                                             T* __restrict__ ts, int64_t kt,
                                                             double* __restrict__ quad) {
    __shared__ double s_lt[256], s_tt[256];
    const int v = blockIdx.x;
    const double* tv = tsum + (int64_t)v * (k + 1);
    double lt = 0.0, tt = 0.0;
    for (int64_t c = threadIdx.x; c < kt; c += 256) {
        if (c >= k) {
            if (ts) ts[v * kt + c] = T(0);  // the pad columns of the expansion's 16-byte groups
            continue;
        }
        const double t = tv[c], l = (double)lam[c];
        if (ts) ts[v * kt + c] = (T)((l - (full ? lambda_tilde : 0.0)) * t);
        lt += l * t * t;
        tt += t * t;
    }
    s_lt[threadIdx.x] = lt;
    s_tt[threadIdx.x] = tt;
    __syncthreads();
    if (threadIdx.x == 0 && quad) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < 256; ++i) {
            a += s_lt[i];
            b += s_tt[i];
        }
        quad[v] = full ? a + lambda_tilde * tv[k] - lambda_tilde * b : a;
    }
}

// y[v][i] = sum_c ts[v][c] q[i][c] + shift x[v][i].  A block walks tiles of kExpRows
// rows of Q, in column chunks of at most ExpTile::Cols, through two shared-memory
// buffers: the 16-byte cp.async copies of the next (tile, chunk) are in flight while
// the current one is summed (VEC: rows 16-byte aligned; otherwise plain loads, one
// buffer).  The row pitch puts a quarter-warp's 16-byte reads on distinct banks.
// Thread (row r, class g) sums its row over the 16-byte column groups g, g + 4, ...
// (one LDS.128 of Q and one of the staged ts chunk per vector for W columns), the
// four classes are added in fixed order, and y is stored coalesced along i.
constexpr int kExpRows = 64;
template <class T>
struct ExpTile {
    static constexpr int W = 16 / sizeof(T);
    static constexpr int Cols = 1024 / sizeof(T);  // at most 256 (float) / 128 (double) columns per chunk
    // smallest pitch >= cols (a multiple of W) whose 4-byte word count is 4 mod 32
    static int pitch(int64_t k) {
        const int colsw = (int)round_up(std::min<int64_t>(k, Cols), W);
        const int mod = 32 / (int)(sizeof(T) / 4), want = W;  // elements: float 4 mod 32, double 2 mod 16
        int pt = colsw;
        while (pt % mod != want) pt += W;
        return pt;
    }
    // per buffer: the Q tile and the ts chunk [kVecTile][pitch]; then the class sums
    static size_t bytes(int64_t k, bool two) {
        return (size_t)((two ? 2 : 1) * (kExpRows + kVecTile) * pitch(k) + 4 * kVecTile * kExpRows) * sizeof(T);
    }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(gmem), "r"(src_bytes) : "memory");
}

template <class T, int NV, bool VEC>
__global__ void __launch_bounds__(256) expand_kernel(const T* __restrict__ q, int64_t ldq, int64_t p, int64_t k,
                                                     const T* __restrict__ ts, int64_t kt, int nv, int pitch, T shift,
                                                     const T* __restrict__ x, int64_t ldx, T* __restrict__ y,
                                                     int64_t ldy) {
    using E = ExpTile<T>;
    using V = Vec16<T>;
    constexpr int W = E::W, NB = VEC ? 2 : 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* tiles = reinterpret_cast<T*>(smem_raw);               // [NB][kExpRows + kVecTile][pitch]: Q rows, then ts rows
    const int bufsz = (kExpRows + kVecTile) * pitch;
    T* red = tiles + NB * bufsz;                             // [4][kVecTile][kExpRows]
    const int t = threadIdx.x, r = t % kExpRows, g = t / kExpRows;
    const int64_t ntiles = ceil_div(p, kExpRows);
    const int64_t nchunks = ceil_div(k, (int64_t)E::Cols);
    // this block's work items: (tile blockIdx.x + j gridDim.x, chunk ch), j-major, walked
    // by (j, ch) counters (no 64-bit divisions in the loop)
    const int nch = (int)nchunks;
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t nitems = my_tiles * nchunks;
    auto item_rows = [&](int64_t j, int ch, int64_t& i0, int64_t& c0, int& rows, int& cols) {
        i0 = (blockIdx.x + j * gridDim.x) * kExpRows;
        c0 = (int64_t)ch * E::Cols;
        rows = (int)min((int64_t)kExpRows, p - i0);
        cols = (int)min((int64_t)E::Cols, k - c0);
    };
    // stage item `it` into buffer `b`: cp.async (VEC; the ragged last group zero-filled
    // past k) or plain loads
    auto stage = [&](int64_t j, int ch, int b) {
        int64_t i0, c0;
        int rows, cols;
        item_rows(j, ch, i0, c0, rows, cols);
        T* tile = tiles + b * bufsz;
        const int nvr = (cols + W - 1) / W;
        // the chunk of ts (kt is a multiple of 4 and its pad is zero: whole 16-byte groups)
        for (int e = t; e < NV * nvr; e += 256) {
            const int v = e / nvr, cv = e % nvr;
            if constexpr (VEC) {
                cp_async16(tile + (kExpRows + v) * pitch + W * cv, ts + v * kt + c0 + W * cv, 16);
            } else {
#pragma unroll
                for (int w = 0; w < W; ++w) tile[(kExpRows + v) * pitch + W * cv + w] = ts[v * kt + c0 + W * cv + w];
            }
        }
        if constexpr (VEC) {
            const int total = rows * nvr, dr = 256 / nvr, dc = 256 % nvr;
            const int tail = (cols - W * (nvr - 1)) * (int)sizeof(T);  // valid bytes of a row's last group
            const T* gsrc = q + i0 * ldq + c0;
            const int ldqi = (int)ldq;  // (row offsets inside a tile fit 32 bits: 64 rows)
            int rr = t / nvr, cv = t % nvr;
            for (int e = t; e < total; e += 256) {
                cp_async16(tile + rr * pitch + W * cv, gsrc + rr * ldqi + W * cv, cv == nvr - 1 ? tail : 16);
                rr += dr;
                cv += dc;
                if (cv >= nvr) {
                    cv -= nvr;
                    ++rr;
                }
            }
        } else {
            for (int rr = t / 32; rr < rows; rr += 8) {
                const T* src = q + (i0 + rr) * ldq + c0;
#pragma unroll 4
                for (int c = t % 32; c < nvr * W; c += 32) tile[rr * pitch + c] = c < cols ? src[c] : T(0);
            }
        }
    };
    if constexpr (VEC) {
        if (nitems > 0) stage(0, 0, 0);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    T acc[NV] = {};
    int64_t j = 0;
    int ch = 0;
    for (int64_t it = 0; it < nitems; ++it) {
        int64_t i0, c0;
        int rows, cols;
        item_rows(j, ch, i0, c0, rows, cols);
        const int b = VEC ? (int)(it & 1) : 0;
        const int chn = ch + 1 < nch ? ch + 1 : 0;  // the next item
        const int64_t jn = chn ? j : j + 1;
        if constexpr (VEC) {
            if (it + 1 < nitems) stage(jn, chn, b ^ 1);  // (its last readers passed the barrier below)
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            stage(j, ch, 0);
        }
        __syncthreads();
        if (r < rows) {
            const T* row = tiles + b * bufsz + r * pitch;
            const T* st = tiles + b * bufsz + kExpRows * pitch;
            const int colsw = (cols + W - 1) / W * W;
#pragma unroll 4
            for (int c = g * W; c < colsw; c += 4 * W) {
                const V qv = *reinterpret_cast<const V*>(row + c);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const V tv = *reinterpret_cast<const V*>(st + v * pitch + c);
#pragma unroll
                    for (int u = 0; u < W; ++u) acc[v] += qv.v[u] * tv.v[u];
                }
            }
        }
        if (c0 + E::Cols >= k) {  // the tile's last chunk: add the four classes, store y
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                red[(g * kVecTile + v) * kExpRows + r] = acc[v];
                acc[v] = T(0);
            }
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
        __syncthreads();  // the buffer and red may be rewritten
        j = jn;
        ch = chn;
    }
    if constexpr (VEC) asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// k = 0: y = shift x
template <class T>
__global__ void scale_vec_kernel(const T* __restrict__ x, int64_t ldx, T* __restrict__ y, int64_t ldy, int64_t p,
                                 int nv, T shift) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p * nv) return;
    const int64_t v = i / p, j = i % p;
    y[v * ldy + j] = shift * x[v * ldx + j];
}

template <class T, int NV, bool VEC>
void launch_project(cudaStream_t s, int64_t nblocks, const T* q, int64_t ldq, int64_t p, int64_t k, int64_t c0,
                    const T* x, int64_t ldx, int nv, int64_t chunk, double* part) {
    project_kernel<T, NV, VEC><<<(unsigned)nblocks, 256, 0, s>>>(q, ldq, p, k, c0, x, ldx, nv, chunk, part);
    CK_LAUNCH();
}

template <class T, int NV, bool VEC>
void launch_expand(cudaStream_t s, const T* q, int64_t ldq, int64_t p, int64_t k, const T* ts, int64_t kt, int nv,
                   T shift, const T* x, int64_t ldx, T* y, int64_t ldy) {
    if (p == 0) return;  // a rank without rows (sharded apply)
    if (k == 0) {
        scale_vec_kernel<T><<<(unsigned)ceil_div(p * nv, 256), 256, 0, s>>>(x, ldx, y, ldy, p, nv, shift);
        CK_LAUNCH();
        return;
    }
    const size_t smem = ExpTile<T>::bytes(k, VEC), smem_max = ExpTile<T>::bytes(ExpTile<T>::Cols, VEC);
    func_attr_once((const void*)expand_kernel<T, NV, VEC>, [smem_max] {
        CK_CUDA(cudaFuncSetAttribute(expand_kernel<T, NV, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_max));
    });
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(6, (int64_t)(200 * 1024) / (int64_t)smem));
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(per_sm * 148, ceil_div(p, kExpRows)));
    expand_kernel<T, NV, VEC><<<(unsigned)grid, 256, smem, s>>>(q, ldq, p, k, ts, kt, nv, ExpTile<T>::pitch(k), shift,
                                                                x, ldx, y, ldy);
    CK_LAUNCH();
}

// y (nvec x p, ldy) and/or quad (nvec, fp64) for x (nvec x p, ldx); y or quad may be null.
// With a communicator, q, x and y hold this rank's parameter rows (the row shards of
// the sharded top-k solvers): the projections t = Q^T x and x.x are summed over the
// ranks -- one all-reduce of nvec (k + 1) doubles -- and every rank expands its own
// rows; quad is the whole vector's quadratic form, identical on every rank.
template <class T>
void apply(cudaStream_t s, int64_t p, int64_t k, const T* q, int64_t ldq, const T* lam, bool full, double lambda_tilde,
           int64_t nvec, const T* x, int64_t ldx, T* y, int64_t ldy, double* quad, const Comm* comm = nullptr) {
    if (nvec < 1) return;
    constexpr int W = Vec16<T>::W;
    const int64_t nblocks = std::max<int64_t>(1, std::min<int64_t>(4 * 148, ceil_div(p, 256)));
    const int64_t chunk = ceil_div(p, nblocks);
    DevMem part((size_t)(nblocks * kVecTile * (k + 1)) * sizeof(double), s);
    DevMem tsum((size_t)(kVecTile * (k + 1)) * sizeof(double), s);
    const int64_t kt = round_up(std::max<int64_t>(k, 1), 4);
    DevMem ts((size_t)(kVecTile * kt) * sizeof(T), s);
    const T shift = full ? (T)lambda_tilde : T(0);
    // 16-byte loads of Q when every row starts 16-byte aligned
    const bool vec = ldq % W == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0;
    ProfScope ps("eig_apply", s, 4.0 * (double)p * k * nvec, 2.0 * ceil_div(nvec, kVecTile) * sizeof(T) * p * k);
    for (int64_t v0 = 0; v0 < nvec; v0 += kVecTile) {
        const int nv = (int)std::min<int64_t>(kVecTile, nvec - v0);
        const T* xv = x + v0 * ldx;
        // (k = 0: one pass still sums x.x for the full-rank quadform)
        for (int64_t c0 = 0; c0 < std::max<int64_t>(k, 1); c0 += 32 * W) {
            double* pd = dptr<double>(part);
            if (nv == 1) {
                if (vec) launch_project<T, 1, true>(s, nblocks, q, ldq, p, k, c0, xv, ldx, nv, chunk, pd);
                else launch_project<T, 1, false>(s, nblocks, q, ldq, p, k, c0, xv, ldx, nv, chunk, pd);
            } else {
                if (vec) launch_project<T, kVecTile, true>(s, nblocks, q, ldq, p, k, c0, xv, ldx, nv, chunk, pd);
                else launch_project<T, kVecTile, false>(s, nblocks, q, ldq, p, k, c0, xv, ldx, nv, chunk, pd);
            }
        }
        project_sum_kernel<<<dim3((unsigned)ceil_div(k + 1, 8), (unsigned)nv), 256, 0, s>>>(dptr<double>(part), nblocks, k,
                                                                                          dptr<double>(tsum));
        CK_LAUNCH();
        if (comm) comm->sum(dptr<double>(tsum), (size_t)nv * (size_t)(k + 1), s);
        project_finish_kernel<T><<<nv, 256, 0, s>>>(dptr<double>(tsum), k, lam, full ? 1 : 0, lambda_tilde,
                                                   y ? dptr<T>(ts) : nullptr, kt, quad ? quad + v0 : nullptr);
        CK_LAUNCH();
        if (!y) continue;
        T* yv = y + v0 * ldy;
        auto ex = [&](auto nvc) {
            constexpr int NVC = decltype(nvc)::value;
            if (vec) launch_expand<T, NVC, true>(s, q, ldq, p, k, dptr<T>(ts), kt, nv, shift, xv, ldx, yv, ldy);
            else launch_expand<T, NVC, false>(s, q, ldq, p, k, dptr<T>(ts), kt, nv, shift, xv, ldx, yv, ldy);
        };
        switch (nv) {
            case 1: ex(std::integral_constant<int, 1>{}); break;
            case 2: ex(std::integral_constant<int, 2>{}); break;
            case 3: ex(std::integral_constant<int, 3>{}); break;
            default: ex(std::integral_constant<int, 4>{}); break;
        }
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
