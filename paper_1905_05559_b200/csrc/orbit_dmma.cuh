// orbit_dmma.cuh -- f64 symmetric-orbit diagonal blocks on the FP64 tensor
// cores (mma.sync m8n8k4 f64), used by Engine::orbit_block (curvature.cuh).
#pragma once

#include "common.cuh"

namespace ck {

__device__ __forceinline__ void dmma8x8x4(double* c, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// ---- f64 symmetric orbits (Engine::orbit_block): Z rows are pairs in 8 x 8
// blocks (block b = (ib, cb), row il * 8 + cl = (i = 8 ib + il, c = 8 cb + cl)),
// so one 64-row tile is one (i, c) block.  The tile is staged in shared memory
// and each of the four orbit images is written as 64-byte runs (8 consecutive
// c, or 8 consecutive i), four runs per warp store instead of scattered
// 8-byte stores.
template <class T>
struct OrbitArgs {
    const T* z;           // [rows][ldz] (K-major), rows = 64 x blocks of this chunk
    const T* pi;          // [np][ldz]
    int64_t ldz, np, K;
    const int2* blocks;   // (ib, cb) of the chunk's blocks
    const int2* oo;       // packed (o, o'')
    T* H;
    int64_t ldh, woff, boff, tk;
    T alpha;
};

template <class T>
__device__ __forceinline__ int64_t orbit_hidx(const OrbitArgs<T>& a, int64_t o, int64_t x) {
    return x < a.tk ? a.woff + o * a.tk + x : a.boff + o;
}

// The staged 64 x 64 tile S[row][col] (row = il * 8 + cl of block (ib, cb),
// col = packed (o, o'') n0 + col) to its four orbit images: 64-byte (f64) or
// 32-byte (f32) runs of 8 consecutive c (types 1, 4) or i (types 2, 3), four
// runs per warp store
template <class T, int SP>
__device__ __forceinline__ void orbit_store_tile(const OrbitArgs<T>& a, const T* S, int64_t n0, int2 blk, int warp,
                                                 int lane) {
    const int64_t i0 = 8 * (int64_t)blk.x, c0 = 8 * (int64_t)blk.y;
    const int e8 = lane & 7;
    for (int run = warp * 4 + (lane >> 3); run < 64 * 8; run += 16) {
        const int jl = run >> 3, w = run & 7;
        const int64_t j = n0 + jl;
        if (j >= a.np) continue;
        const int2 u = a.oo[j];
        {  // types 1 and 4: i = i0 + w fixed, c = c0 + e8 consecutive
            const int64_t i = i0 + w, c = c0 + e8;
            if (i <= a.tk && c <= a.tk) {
                const T v = S[(w * 8 + e8) * SP + jl];
                a.H[orbit_hidx(a, u.x, i) * a.ldh + orbit_hidx(a, u.y, c)] = v;   // (o, i; o'', c)
                a.H[orbit_hidx(a, u.y, i) * a.ldh + orbit_hidx(a, u.x, c)] = v;   // (o'', i; o, c)
            }
        }
        {  // types 2 and 3: c = c0 + w fixed, i = i0 + e8 consecutive
            const int64_t c = c0 + w, i = i0 + e8;
            if (i <= a.tk && c <= a.tk) {
                const T v = S[(e8 * 8 + w) * SP + jl];
                a.H[orbit_hidx(a, u.y, c) * a.ldh + orbit_hidx(a, u.x, i)] = v;   // (o'', c; o, i)
                a.H[orbit_hidx(a, u.x, c) * a.ldh + orbit_hidx(a, u.y, i)] = v;   // (o, c; o'', i)
            }
        }
    }
}

template <int BYTES>
__device__ __forceinline__ void cp_async_n(void* dst, const void* src, bool pred) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    const int n = pred ? BYTES : 0;  // zero-fill when out of range
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src), "n"(BYTES), "r"(n) : "memory");
}

__global__ void __launch_bounds__(128, 4) orbit_dmma_kernel(OrbitArgs<double> a) {
    constexpr int BM = 64, BN = 64, BK = 16, LD = BK + 4, SP = BN + 1;
    constexpr int TILE = 2 * BM * LD;  // As + Bs of one K-panel
    __shared__ double smem[BM * SP > 2 * TILE ? BM * SP : 2 * TILE];
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][4][2] = {};
    // K-panels double-buffered in shared memory by cp.async (no register prefetch)
    auto fetch = [&](int64_t k0, int buf) {
        double* As = smem + buf * TILE;
        double* Bs = As + BM * LD;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = t + 128 * j, r = e / BK, kk = e % BK;
            const int64_t gk = k0 + kk, gn = n0 + r;
            const bool ka = gk < a.K, kb = gn < a.np && gk < a.K;
            cp_async_n<8>(As + r * LD + kk, a.z + (m0 + r) * a.ldz + (ka ? gk : 0), ka);
            cp_async_n<8>(Bs + r * LD + kk, a.pi + (kb ? gn : 0) * a.ldz + (kb ? gk : 0), kb);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (a.K > 0) fetch(0, 0);
    int buf = 0;
    for (int64_t k0 = 0; k0 < a.K; k0 += BK, buf ^= 1) {
        if (k0 + BK < a.K) {
            fetch(k0 + BK, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double* As = smem + buf * TILE;
        const double* Bs = As + BM * LD;
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            double x[4], y[4];
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                x[f] = As[(wm + 8 * f + fr) * LD + k4 + fk];
                y[f] = Bs[(wn + 8 * f + fr) * LD + k4 + fk];
            }
#pragma unroll
            for (int fa = 0; fa < 4; ++fa)
#pragma unroll
                for (int fb = 0; fb < 4; ++fb) dmma8x8x4(acc[fa][fb], x[fa], y[fb]);
        }
        __syncthreads();
    }
    // stage the tile: S[row][col], row = il * 8 + cl
    double* S = smem;
#pragma unroll
    for (int fa = 0; fa < 4; ++fa)
#pragma unroll
        for (int fb = 0; fb < 4; ++fb)
#pragma unroll
            for (int h = 0; h < 2; ++h) S[(wm + 8 * fa + fr) * SP + wn + 8 * fb + 2 * fk + h] = a.alpha * acc[fa][fb][h];
    __syncthreads();
    orbit_store_tile<double, SP>(a, S, n0, a.blocks[blockIdx.x], warp, lane);
}


// f32: the same tiles and epilogue on FFMA (each thread an 8 x 4 micro-tile)
__global__ void __launch_bounds__(128, 4) orbit_simt_kernel(OrbitArgs<float> a) {
    constexpr int BM = 64, BN = 64, BK = 16, LD = BK + 1, SP = BN + 1;
    constexpr int TILE = 2 * BM * LD;
    __shared__ float smem[BM * SP > 2 * TILE ? BM * SP : 2 * TILE];
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const int tx = t % 16, ty = t / 16;  // columns tx + 16 c (c < 4), rows 8 ty + r (r < 8)
    float acc[8][4] = {};
    auto fetch = [&](int64_t k0, int buf) {
        float* As = smem + buf * TILE;
        float* Bs = As + BM * LD;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = t + 128 * j, r = e / BK, kk = e % BK;
            const int64_t gk = k0 + kk, gn = n0 + r;
            const bool ka = gk < a.K, kb = gn < a.np && gk < a.K;
            cp_async_n<4>(As + r * LD + kk, a.z + (m0 + r) * a.ldz + (ka ? gk : 0), ka);
            cp_async_n<4>(Bs + r * LD + kk, a.pi + (kb ? gn : 0) * a.ldz + (kb ? gk : 0), kb);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (a.K > 0) fetch(0, 0);
    int buf = 0;
    for (int64_t k0 = 0; k0 < a.K; k0 += BK, buf ^= 1) {
        if (k0 + BK < a.K) {
            fetch(k0 + BK, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const float* As = smem + buf * TILE;
        const float* Bs = As + BM * LD;
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float x[8], y[4];
#pragma unroll
            for (int r = 0; r < 8; ++r) x[r] = As[(8 * ty + r) * LD + kk];
#pragma unroll
            for (int c = 0; c < 4; ++c) y[c] = Bs[(tx + 16 * c) * LD + kk];
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(x[r], y[c], acc[r][c]);
        }
        __syncthreads();
    }
    float* S = smem;
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) S[(8 * ty + r) * SP + tx + 16 * c] = a.alpha * acc[r][c];
    __syncthreads();
    orbit_store_tile<float, SP>(a, S, n0, a.blocks[blockIdx.x], warp, lane);
}

}  // namespace ck
