// gemm_dmma.cuh -- fp64 GEMM on the FP64 tensor cores (mma.sync m8n8k4 f64)
// with the SIMT engine's contract: Opnd operands (K- or MN-major), batches
// over grid.z, Epi::skip per tile and an element-wise Epi epilogue.  The f64
// precision mode routes its large products here (CurvGemm<double>).
//
// A 128-thread block owns a 64 x 64 tile; each warp a 32 x 32 quarter as
// 4 x 4 fragments of 8 x 8.  Per K-panel of 16 the operand tiles are staged
// in shared memory as [row][k] (pitch 20 doubles: the 8 rows x 4 k of a
// fragment load hit distinct banks but for a 2-way overlap), double-buffered
// by cp.async so the next panel lands while this one is multiplied (the
// register-prefetch form reached 15.5 TF/s = 0.42 of the measured 37.2 TF/s
// DMMA peak at config 1).
#pragma once

#include "common.cuh"
#include "gemm_simt.cuh"
#include "orbit_dmma.cuh"

namespace ck {

// Epilogues that split each entry into a direct and a mirrored store
// (Epi::store_direct / Epi::store_mirror; together they equal Epi::operator())
template <class E, class = void>
struct EpiSplit : std::false_type {};
template <class E>
struct EpiSplit<E, std::void_t<decltype(&E::store_direct)>> : std::true_type {};


template <class Epi>
__global__ void __launch_bounds__(128, 4) gemm_dmma_kernel(int64_t M, int64_t N, int64_t K, Opnd<double> A,
                                                           Opnd<double> B, Epi epi) {
    constexpr int BM = 64, BN = 64, BK = 16, LD = BK + 4;
    constexpr int TILE = (BM + BN) * LD;  // As + Bs of one K-panel
    __shared__ double smem[2 * TILE];
    const int bz = blockIdx.z;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    if (epi.skip(bz, m0, n0, BM, BN)) return;
    const double* Ap = A.p + bz * A.bstride;
    const double* Bp = B.p + bz * B.bstride;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][4][2] = {};
    // K-panels double-buffered in shared memory by cp.async (zero-filled out of
    // range).  Element e of a 64 x 16 operand tile: K-major -> row e / 16, k
    // e % 16 (16 consecutive k of a row are contiguous); MN-major -> k e / 64,
    // row e % 64.
    auto fetch = [&](int64_t k0, int buf) {
        double* As = smem + buf * TILE;
        double* Bs = As + BM * LD;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = t + 128 * j;
            int r, kk;
            if (A.kmajor) { r = e / BK; kk = e % BK; } else { kk = e / BM; r = e % BM; }
            int64_t gm = m0 + r, gk = k0 + kk;
            bool ok = gm < M && gk < K;
            cp_async_n<8>(As + r * LD + kk, ok ? (A.kmajor ? Ap + gm * A.ld + gk : Ap + gk * A.ld + gm) : Ap, ok);
            if (B.kmajor) { r = e / BK; kk = e % BK; } else { kk = e / BN; r = e % BN; }
            gm = n0 + r;
            gk = k0 + kk;
            ok = gm < N && gk < K;
            cp_async_n<8>(Bs + r * LD + kk, ok ? (B.kmajor ? Bp + gm * B.ld + gk : Bp + gk * B.ld + gm) : Bp, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (K > 0) fetch(0, 0);
    int buf = 0;
    for (int64_t k0 = 0; k0 < K; k0 += BK, buf ^= 1) {
        if (k0 + BK < K) {
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
            double a[4], b[4];
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                a[f] = As[(wm + 8 * f + fr) * LD + k4 + fk];  // A(row, k)
                b[f] = Bs[(wn + 8 * f + fr) * LD + k4 + fk];  // B(k, col) = B(col, k) stored [col][k]
            }
#pragma unroll
            for (int fa = 0; fa < 4; ++fa)
#pragma unroll
                for (int fb = 0; fb < 4; ++fb) dmma8x8x4(acc[fa][fb], a[fa], b[fb]);
        }
        __syncthreads();
    }
    // D fragment: row fr, columns 2 fk + {0, 1}
    if constexpr (EpiSplit<Epi>::value) {
        // staged: the tile in shared memory, then the direct entries row by row
        // and the mirrored entries column by column, so both store streams are
        // 512-byte runs (per-element mirror stores walk down a column of H)
        constexpr int SP = BN + 1;
        double* S = smem;  // 64 x 65 <= the two K-panel buffers (after the last barrier)
#pragma unroll
        for (int fa = 0; fa < 4; ++fa)
#pragma unroll
            for (int fb = 0; fb < 4; ++fb)
#pragma unroll
                for (int h = 0; h < 2; ++h) S[(wm + 8 * fa + fr) * SP + wn + 8 * fb + 2 * fk + h] = acc[fa][fb][h];
        __syncthreads();
        for (int idx = t; idx < BM * BN; idx += 128) {
            const int r = idx / BN, c = idx % BN;
            if (m0 + r < M && n0 + c < N) epi.store_direct(bz, m0 + r, n0 + c, S[r * SP + c]);
        }
        for (int idx = t; idx < BM * BN; idx += 128) {
            const int c = idx / BM, r = idx % BM;
            if (m0 + r < M && n0 + c < N) epi.store_mirror(bz, m0 + r, n0 + c, S[r * SP + c]);
        }
    } else {
#pragma unroll
        for (int fa = 0; fa < 4; ++fa)
#pragma unroll
            for (int fb = 0; fb < 4; ++fb)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t gm = m0 + wm + 8 * fa + fr, gn = n0 + wn + 8 * fb + 2 * fk + h;
                    if (gm < M && gn < N) epi(bz, gm, gn, acc[fa][fb][h]);
                }
    }
}

template <class Epi>
void gemm_dmma(cudaStream_t s, int64_t M, int64_t N, int64_t K, int64_t batch, Opnd<double> A, Opnd<double> B,
               const Epi& epi) {
    if (M <= 0 || N <= 0 || batch <= 0) return;
    dim3 grid((unsigned)ceil_div(M, 64), (unsigned)ceil_div(N, 64), (unsigned)batch);
    gemm_dmma_kernel<Epi><<<grid, 128, 0, s>>>(M, N, K, A, B, epi);
    CK_LAUNCH();
}

// f64 curvature products on the FP64 tensor cores
template <class Epi>
struct CurvGemm<double, Epi> {
    static void run(int, cudaStream_t s, int64_t M, int64_t N, int64_t K, Opnd<double> A, Opnd<double> B,
                    const Epi& e) {
        gemm_dmma<Epi>(s, M, N, K, 1, A, B, e);
    }
};

}  // namespace ck
