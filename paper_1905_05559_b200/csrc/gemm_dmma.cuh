// gemm_dmma.cuh -- fp64 GEMM on the FP64 tensor cores (mma.sync m8n8k4 f64)
// with the SIMT engine's contract: Opnd operands (K- or MN-major), batches
// over grid.z, Epi::skip per tile and an element-wise Epi epilogue.  The f64
// precision mode routes its large products here (CurvGemm<double>).
//
// A 128-thread block owns a 64 x 64 tile; each warp a 32 x 32 quarter as
// 4 x 4 fragments of 8 x 8.  Per K-panel of 16 the operand tiles are staged
// in shared memory as [row][k] (pitch 20 doubles: the 8 rows x 4 k of a
// fragment load hit distinct banks but for a 2-way overlap) and the next
// panel is fetched into registers while this one is multiplied.
#pragma once

#include "common.cuh"
#include "gemm_simt.cuh"
#include "orbit_dmma.cuh"

namespace ck {


template <class Epi>
__global__ void __launch_bounds__(128) gemm_dmma_kernel(int64_t M, int64_t N, int64_t K, Opnd<double> A,
                                                        Opnd<double> B, Epi epi) {
    constexpr int BM = 64, BN = 64, BK = 16, LD = BK + 4;
    __shared__ double As[BM * LD], Bs[BN * LD];
    const int bz = blockIdx.z;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    if (epi.skip(bz, m0, n0, BM, BN)) return;
    const double* Ap = A.p + bz * A.bstride;
    const double* Bp = B.p + bz * B.bstride;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][4][2] = {};
    // 64 x 16 = 1024 elements per operand tile: 8 per thread.  Element e of
    // the tile: K-major operand -> row e / 16, k e % 16 (16 consecutive k of
    // a row are contiguous in memory); MN-major -> k e / 64, row e % 64.
    double ra[8], rb[8];
    auto fetch = [&](int64_t k0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = t + 128 * j;
            int r, kk;
            if (A.kmajor) { r = e / BK; kk = e % BK; } else { kk = e / BM; r = e % BM; }
            const int64_t gm = m0 + r, gk = k0 + kk;
            ra[j] = (gm < M && gk < K) ? (A.kmajor ? Ap[gm * A.ld + gk] : Ap[gk * A.ld + gm]) : 0.0;
            if (B.kmajor) { r = e / BK; kk = e % BK; } else { kk = e / BN; r = e % BN; }
            const int64_t gn = n0 + r, gk2 = k0 + kk;
            rb[j] = (gn < N && gk2 < K) ? (B.kmajor ? Bp[gn * B.ld + gk2] : Bp[gk2 * B.ld + gn]) : 0.0;
        }
    };
    if (K > 0) fetch(0);
    for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = t + 128 * j;
            int r, kk;
            if (A.kmajor) { r = e / BK; kk = e % BK; } else { kk = e / BM; r = e % BM; }
            As[r * LD + kk] = ra[j];
            if (B.kmajor) { r = e / BK; kk = e % BK; } else { kk = e / BN; r = e % BN; }
            Bs[r * LD + kk] = rb[j];
        }
        __syncthreads();
        if (k0 + BK < K) fetch(k0 + BK);
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
