// gemm_simt.cuh -- exact-FMA tiled GEMM for the f64 and f32 precision modes.
//
// C(b, m, n) = sum_k A(b, m, k) * B(b, n, k), with each operand either
// K-major (element (row, k) at p[row*ld + k]) or MN-major (p[k*ld + row]).
// The result is handed element by element to an epilogue functor, which
// owns the output layout (plain, symmetric mirror, Hessian block mapping,
// fused bias+activation, ...).  The tcgen05 kernel in gemm_tc.cuh shares the
// same operand/epilogue conventions for the TF32 modes.
#pragma once

#include "common.cuh"

namespace ck {

template <class T>
struct Opnd {
    const T* p = nullptr;
    int64_t ld = 0;
    int kmajor = 1;
    int64_t bstride = 0;  // batch stride in elements
    int rounded = 0;      // values already rounded to TF32 by their producer
    int once = 0;         // every element read by one tile only (L2 evict_first)
};

template <class T>
inline Opnd<T> pre_rounded(Opnd<T> o) {
    o.rounded = 1;
    return o;
}

template <class T>
inline Opnd<T> read_once(Opnd<T> o) {
    o.once = 1;
    return o;
}

template <class T>
__host__ __device__ inline Opnd<T> kmaj(const T* p, int64_t ld, int64_t bs = 0) {
    Opnd<T> o;
    o.p = p; o.ld = ld; o.kmajor = 1; o.bstride = bs;
    return o;
}
template <class T>
__host__ __device__ inline Opnd<T> mnmaj(const T* p, int64_t ld, int64_t bs = 0) {
    Opnd<T> o;
    o.p = p; o.ld = ld; o.kmajor = 0; o.bstride = bs;
    return o;
}

// Default: never skip a tile.
struct NoSkip {
    __device__ bool operator()(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
};

template <class T, int BM, int BN, int BK, int TM, int TN, class Epi>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_simt_kernel(int64_t M, int64_t N, int64_t K, Opnd<T> A, Opnd<T> B, Epi epi, int64_t kchunk) {
    constexpr int NTX = BN / TN, NTY = BM / TM, NT = NTX * NTY;
    __shared__ T As[BK][BM + 1];
    __shared__ T Bs[BK][BN + 1];
    const int bz = blockIdx.z;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    if (epi.skip(bz, m0, n0, BM, BN)) return;
    const T* Ap = A.p + bz * A.bstride;
    const T* Bp = B.p + bz * B.bstride;
    int64_t kbeg = 0;
    if (kchunk > 0) {  // split-K: grid.z indexes K ranges, operands are not batched
        kbeg = bz * kchunk;
        K = ::min(K, kbeg + kchunk);
        Ap = A.p;
        Bp = B.p;
    }
    const int tid = threadIdx.x, tx = tid % NTX, ty = tid / NTX;
    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

    for (int64_t k0 = kbeg; k0 < K; k0 += BK) {
        // A tile: BM x BK
        for (int e = tid; e < BM * BK; e += NT) {
            int r, kk;
            if (A.kmajor) { kk = e % BK; r = e / BK; } else { r = e % BM; kk = e / BM; }
            const int64_t gm = m0 + r, gk = k0 + kk;
            T v = T(0);
            if (gm < M && gk < K) v = A.kmajor ? Ap[gm * A.ld + gk] : Ap[gk * A.ld + gm];
            As[kk][r] = v;
        }
        for (int e = tid; e < BN * BK; e += NT) {
            int r, kk;
            if (B.kmajor) { kk = e % BK; r = e / BK; } else { r = e % BN; kk = e / BN; }
            const int64_t gn = n0 + r, gk = k0 + kk;
            T v = T(0);
            if (gn < N && gk < K) v = B.kmajor ? Bp[gn * B.ld + gk] : Bp[gk * B.ld + gn];
            Bs[kk][r] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            T a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + NTY * i];
#pragma unroll
            for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + NTX * j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int64_t gm = m0 + ty + NTY * i, gn = n0 + tx + NTX * j;
            if (gm < M && gn < N) epi(bz, gm, gn, acc[i][j]);
        }
}

// batch > 0: batched GEMM over grid.z.  kchunk > 0: split-K instead, grid.z =
// ceil(K / kchunk) ranges, the epilogue sees the range index as its batch.
template <class T, class Epi>
void gemm_simt(cudaStream_t s, int64_t M, int64_t N, int64_t K, int64_t batch, Opnd<T> A, Opnd<T> B,
               const Epi& epi, int64_t kchunk = 0) {
    if (M <= 0 || N <= 0 || batch <= 0) return;
    constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
    const int64_t gz = kchunk > 0 ? ceil_div(K, kchunk) : batch;
    dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(N, BN), (unsigned)gz);
    gemm_simt_kernel<T, BM, BN, BK, TM, TN, Epi><<<grid, (BM / TM) * (BN / TN), 0, s>>>(M, N, K, A, B, epi, kchunk);
    CK_LAUNCH();
}

// ---- common epilogues --------------------------------------------------------

// C[b][m*ldc + n] = alpha * acc (+ beta * C)
template <class T>
struct EpiStore {
    T* c;
    int64_t ldc, bstride;
    T alpha, beta;
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int b, int64_t m, int64_t n, T acc) const {
        T* p = c + b * bstride + m * ldc + n;
        *p = beta == T(0) ? alpha * acc : alpha * acc + beta * *p;
    }
    // tensor-core epilogue (see EpiBlock contract below)
    __device__ void block(int64_t row0, int64_t col0, int64_t M, int64_t N, const float (*buf)[36], const float*,
                          int lane) const {
        const int q = lane & 7, rsub = lane >> 3;
        const int64_t col = col0 + 4 * q;
        const bool vec = sizeof(T) == 4 && beta == T(0) && (ldc & 3) == 0;
        for (int it = 0; it < 8; ++it) {
            const int r = it * 4 + rsub;
            const int64_t row = row0 + r;
            if (row >= M) break;
            T* p = c + row * ldc + col;
            const float4 x = *reinterpret_cast<const float4*>(&buf[r][4 * q]);
            if constexpr (sizeof(T) == 4) {
                if (vec && col + 3 < N) {
                    __stcs(reinterpret_cast<float4*>(p), make_float4(alpha * x.x, alpha * x.y, alpha * x.z, alpha * x.w));
                    continue;
                }
            }
            const float xs[4] = {x.x, x.y, x.z, x.w};
            for (int u = 0; u < 4 && col + u < N; ++u)
                p[u] = beta == T(0) ? alpha * (T)xs[u] : alpha * (T)xs[u] + beta * p[u];
        }
    }
};

// Symmetric product (SYRK-style): only tiles touching the lower triangle run;
// each lower entry is written at (m, n) and mirrored to (n, m), so the result
// is exactly symmetric.
template <class T>
struct EpiSymLower {
    T* c;
    int64_t ldc;
    T alpha;
    // row shard: the GEMM's A operand starts at matrix row roff, so GEMM row m
    // is matrix row m + roff (columns are always absolute)
    int64_t roff = 0;
    // tensor-core epilogue: 32 x 32 blocks strictly below the diagonal go out
    // as two TMA boxes (entry block at (row, col), mirror at (col, row))
    static constexpr bool kTmaStore = true;
    int tma = 1;  // cleared by the launcher when C's pitch cannot be a TMA tensor (ldc % 4 != 0)
    __device__ bool tma_block(int64_t row0, int64_t col0, int64_t M, int64_t N, int64_t& gr0, int64_t& gc0) const {
        if (!tma || row0 + 32 > M || col0 + 32 > N) return false;
        gr0 = row0 + roff;
        gc0 = col0;
        return gc0 + 31 < gr0;
    }
    __device__ bool skip(int, int64_t m0, int64_t n0, int64_t bm, int64_t) const {
        return n0 > m0 + roff + bm - 1;
    }
    __device__ void operator()(int, int64_t m, int64_t n, T acc) const {
        m += roff;
        if (n > m) return;
        const T v = alpha * acc;
        c[m * ldc + n] = v;
        c[n * ldc + m] = v;
    }
    // the two stores of operator() separately (staged fp64 epilogue)
    __device__ void store_direct(int, int64_t m, int64_t n, T acc) const {
        m += roff;
        if (n <= m) c[m * ldc + n] = alpha * acc;
    }
    __device__ void store_mirror(int, int64_t m, int64_t n, T acc) const {
        m += roff;
        if (n <= m) c[n * ldc + m] = alpha * acc;
    }
    __device__ void block(int64_t row0, int64_t col0, int64_t M, int64_t N, const float (*buf)[36], const float* v,
                          int lane) const {
        {  // lower entries (col <= row): 16-byte vectors along rows
            const int q = lane & 7, rsub = lane >> 3;
            const int64_t col = col0 + 4 * q;
            for (int it = 0; it < 8; ++it) {
                const int r = it * 4 + rsub;
                if (row0 + r >= M) break;
                const int64_t row = row0 + r + roff;
                const float4 x = *reinterpret_cast<const float4*>(&buf[r][4 * q]);
                T* p = c + row * ldc + col;
                if constexpr (sizeof(T) == 4) {
                    if ((ldc & 3) == 0 && col + 3 <= row && col + 3 < N) {
                        __stcs(reinterpret_cast<float4*>(p),
                               make_float4(alpha * x.x, alpha * x.y, alpha * x.z, alpha * x.w));
                        continue;
                    }
                }
                const float xs[4] = {x.x, x.y, x.z, x.w};
                for (int u = 0; u < 4; ++u)
                    if (col + u < N && col + u <= row) __stcs(&p[u], alpha * (T)xs[u]);
            }
        }
        {  // mirrored strictly-lower entries: this lane's row, straight from registers
            if (row0 + lane < M) {
                const int64_t row = row0 + lane + roff;
#pragma unroll
                for (int cc = 0; cc < 32; ++cc)  // constant trip count keeps v[] in registers
                    if (col0 + cc < N && col0 + cc < row) __stcs(&c[(col0 + cc) * ldc + row], alpha * (T)v[cc]);
            }
        }
    }
};

}  // namespace ck
