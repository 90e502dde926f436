// symkr.cuh -- diagonal curvature blocks by the symmetric Khatri-Rao product.
//
// A diagonal layer block (tangent step k = m) of H, and of G = (1/N) J^T J, is
//
//   B[(o, i), (o'', c)] = alpha * sum_n abar[n, i] abar[n, c] Pi[o][o''][n]
//
// with abar = a_k plus its ones column (index T_k stands for the bias of unit
// o, row boff_k + o of H), Pi[o][o''] = the R-op profile G_k[o][o''] for H
// (curvature.cpp:43-72 restated per DESIGN.md section 2) and delta_k[., o] *
// delta_k[., o''] for G (the per-example gradient rows of
// autodiff.cpp:127-143 are delta (x) abar).  Pi is symmetric in (o, o''), and
// abar_i abar_c is symmetric in (i, c), so every value sits on an orbit of
// four entries:
//
//   (o, i; o'', c)   (o'', c; o, i)   (o, c; o'', i)   (o'', i; o, c)
//
// The kernel computes one representative per orbit (i <= c in 16 x 16 blocks,
// o <= o'' as packed columns) as a tensor-core GEMM
//
//   V[(i, c), j] = sum_n Z[(i, c), n] Pi_packed[j][n],   Z = abar_i * abar_c,
//
// i.e. half the multiply-adds of the lower-triangle GEMM, and writes each
// value to its four places.  Z is formed in shared memory by four transform
// warps from TMA-staged activation rows (8 + 16 rows per K-block instead of a
// 128-row tile); Pi_packed is the TMA-loaded B operand.  CTA pair (cta_group::2,
// M = 256 = 16 i x 16 c), N = up to 256 packed columns, TMEM double buffer.
// The epilogue stages each 8-column chunk in two layouts and stores 4-D TMA
// boxes (16 c x 8 i x E o'' or 8 i x 16 c x E o'') into H; the TMA clips
// everything at index T_k, and the bias entries (index T_k) are written by
// the lanes that hold them.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include "gemm_tc.cuh"

namespace ck {
namespace tc {
namespace sym {
using namespace ::ck::tc::pair;

constexpr int EPI_W = 8, TW_W = 4, TW_SETS = 2;  // TW_SETS sets of 4 transform warps take alternate K-blocks
constexpr int kThreads = 128 + 32 * EPI_W + 32 * TW_W * TW_SETS;
constexpr int TW0 = 4 + EPI_W;
constexpr int Z_BYTES = 128 * BK * 4;   // A operand (Z), 128 rows x 32 examples (shared-memory form)
#ifndef CURVKIT_SYMKR_BROWS
#define CURVKIT_SYMKR_BROWS 128
#endif
constexpr int B_ROWS = CURVKIT_SYMKR_BROWS;  // packed profile rows per CTA and stage (MMA N <= 2 B_ROWS)
constexpr int B_BYTES = B_ROWS * BK * 4;
constexpr int CH = 8;                   // epilogue chunk (packed columns)
constexpr int SLOT = CH * 128 * 4;      // one staging layout of one chunk
constexpr int EPI_BYTES = 2 * 2 * 2 * SLOT;  // group x double buffer x layout
constexpr int EPI_PAD = 4 * 1024;       // boxes of extent 8 may read past a slot
constexpr int MAX_SMEM = 227 * 1024;
// ZT (Z in TMEM): the transform writes Z with tcgen05.st into NZ slots of 32
// columns and the MMA reads A from TMEM (tcgen05.mma [d], [a], b), so Z never
// passes through shared memory; slot reuse is gated by an MMA commit (zfree).
constexpr int NZ = 4;
constexpr int ZSLOT0 = 512 - 32 * NZ;   // first Z column; accumulators at 0 and bn
// F16 (precision kF16S): Z and the packed profile are fp16, so one 128-byte
// operand row holds KB = 64 examples (4 kind::f16 MMAs of K = 16); the fp32
// abar^T rows of a K-block arrive as two 128-byte TMA boxes (examples
// [k0, k0 + 32) and [k0 + 32, k0 + 64)), each in its own 1 KB swizzle atom.
template <bool ZT, bool F16 = false>
struct Cfg {
    static constexpr int KB = F16 ? 64 : 32;           // examples per K-block
    static constexpr int HALVES = F16 ? 2 : 1;         // 32-example abar boxes per K-block
    static constexpr int I_HALF = 8 * BK * 4, C_HALF = 16 * BK * 4;
    static constexpr int I_BYTES = HALVES * I_HALF;    // abar^T rows of the CTA's 8 i
    static constexpr int C_BYTES = HALVES * C_HALF;    // abar^T rows of the 16 c
    static constexpr int STAGE = (ZT ? 0 : Z_BYTES) + B_BYTES + I_BYTES + C_BYTES;
    static constexpr int NST = std::min(8, (MAX_SMEM - 1024 - EPI_BYTES - EPI_PAD - 1024) / STAGE);
    static constexpr int SMEM_BYTES = 1024 + NST * STAGE + EPI_BYTES + EPI_PAD + 1024;
    static constexpr int MAX_BN = ZT ? std::min(ZSLOT0 / 2 / 16 * 16, 2 * B_ROWS) : 2 * B_ROWS;
    static constexpr int ACC_STRIDE = ZT ? 0 : 256;  // 0: accumulator acc at acc * bn
};

struct Params {
    const int4* tiles;   // (ib, cb, nt, -): 16-blocks ib <= cb of abar indices, packed column tile nt
    int64_t ntiles;
    const int4* pairs;   // (o, o'', box kind, -) of packed column j
    int64_t npairs, bn;  // packed columns, MMA N (multiple of 16, <= 256)
    int64_t tk, nk;      // T_k (abar has T_k + 1 rows), K-blocks of 32 examples
    int64_t U;           // T_{k+1}
    float* H;
    int64_t ldh, woff, boff;
    float alpha;
    int tma;             // H boxes by TMA (else every entry by the scalar path)
    int dev;             // dev experiments (CURVKIT_DEV_SYMKR): 1 no transform, 2 no epilogue stores, 32 MMA loop alone (+64 no per-K-block commits)
    // output rows: units [u0, u1) of the block; row (o, x) of the block is stored
    // at H row bwoff + (o - u0) T_k + x (weights) / bboff + (o - u0) (bias).  The
    // whole block is u0 = 0, u1 = U, bwoff = woff, bboff = boff (unit bands:
    // DESIGN.md section 7).  Columns are always the global ones.
    int64_t u0, u1, bwoff, bboff;
    // F16: power-of-two scales, Z row (i, c) = abar_i abar_c zscale[i] zscale[c]
    // (abar indices, padded to whole 16-blocks) and packed column j = Pi_j / pscale[j]
    const float* zscale;
    const float* pscale;
};

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

// the output streams through L2 with evict_first: the packed profile (the B
// operand, re-read by every tile square) keeps its lines
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1, int32_t c2,
                                             int32_t c3, uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;"
                 ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// Tile row rho (TMEM lane, Z row) -> (i, c) within the CTA's 8 x 16 block.  A warp
// covers 4 i x 8 c and each half-warp 2 i x 8 c, so the transform's abar loads touch
// 8 distinct c rows per half-warp (one shared-memory wavefront per LDS.128).
__device__ __forceinline__ void row_ic(int rho, int& il, int& cl) {
    const int w = rho >> 5;
    il = 4 * (w >> 1) + ((rho >> 3) & 3);
    cl = (rho & 7) + 8 * (w & 1);
}

// Split TMEM load: issue now, wait later (the wait passes the registers through,
// so the compiler cannot read them before the data has landed)
__device__ __forceinline__ void tmem_ld8_issue(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait8(uint32_t (&r)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
                 :
                 : "memory");
}

// inverse of row_ic: the tile row (TMEM lane, Z row) of (il, cl)
__device__ __forceinline__ int ic_row(int il, int cl) { return 32 * (2 * (il >> 2) + (cl >> 3)) + 8 * (il & 3) + (cl & 7); }

__device__ __forceinline__ float4 scale4(float4 v, float s) { return make_float4(v.x * s, v.y * s, v.z * s, v.w * s); }

// two fp32 -> packed fp16x2 (round to nearest even), the first in the low half
__device__ __forceinline__ uint32_t h2_bits(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// H column of (unit o, abar index x): weight (o, x) or the bias of o
__device__ __forceinline__ int64_t hidx(const Params& p, int64_t o, int64_t x) {
    return x < p.tk ? p.woff + o * p.tk + x : p.boff + o;
}
// storage row of (unit o, abar index x), -1 outside the output units
__device__ __forceinline__ int64_t srow(const Params& p, int64_t o, int64_t x) {
    if (o < p.u0 || o >= p.u1) return -1;
    return x < p.tk ? p.bwoff + (o - p.u0) * p.tk + x : p.bboff + (o - p.u0);
}

// H maps: [0..3] = orbit types 1..4 with o''-extent 8, [4..7] with extent 1
struct HMaps {
    CUtensorMap m[8];
};

template <bool ZT, bool BAND, bool F16 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
symkr_kernel(const __grid_constant__ CUtensorMap mapAbar8, const __grid_constant__ CUtensorMap mapAbar16,
             const __grid_constant__ CUtensorMap mapPi, const __grid_constant__ HMaps hm, Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    using K = Cfg<ZT, F16>;
    static_assert(!(ZT && F16), "Z in TMEM is a TF32-only variant");
    constexpr int STAGE = K::STAGE, NST = K::NST;
    constexpr int Z_OFF = 0, B_OFF = ZT ? 0 : Z_BYTES, I_OFF = B_OFF + B_BYTES, C_OFF = I_OFF + K::I_BYTES;
    uint8_t* epi_base = smem + NST * STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(epi_base + EPI_BYTES + EPI_PAD);
    uint64_t* full = bars;         // [8] leader: producer + 2 x 4 transform warps, B tx
    uint64_t* empty = bars + 8;    // [8] both CTAs (multicast commit)
    uint64_t* afull = bars + 16;   // [8] local: abar rows landed
    uint64_t* tfull = bars + 24;   // [2]
    uint64_t* tempty = bars + 26;  // [2] leader
    uint64_t* zfree = bars + 28;   // [NZ] both CTAs (ZT): the MMA of the slot's K-block is done
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 28 + NZ);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cta_rank();
    const int64_t pair_id = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int bn = (int)p.bn;

    if (warp == 0 && lane == 0) {
        prefetch_map(&mapAbar8);
        prefetch_map(&mapAbar16);
        prefetch_map(&mapPi);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1 + 2 * TW_W);
            mbar_init(&empty[s], 1);
            mbar_init(&afull[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * EPI_W);
        }
        for (int z = 0; z < NZ; ++z) mbar_init(&zfree[z], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0 && !(p.dev & 32)) {  // ---------------- producer
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol = evict_last_policy();
            for (int64_t t = pair_id; t < p.ntiles; t += npairs) {
                const int4 tl = __ldg(&p.tiles[t]);
                const int32_t i0 = tl.x * 16 + 8 * (int)rank, c0 = tl.y * 16;
                const int32_t b0 = (int32_t)(tl.z * p.bn + (p.bn / 2) * rank);
                for (int64_t kb = 0; kb < p.nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* st = smem + stage * STAGE;
                    const int32_t k0 = (int32_t)(kb * K::KB);
                    mbar_expect_tx(&afull[stage], (uint32_t)(K::I_BYTES + K::C_BYTES));
#pragma unroll
                    for (int h = 0; h < K::HALVES; ++h) {
                        tma_load_2d(st + I_OFF + h * K::I_HALF, &mapAbar8, &afull[stage], k0 + 32 * h, i0);
                        tma_load_2d(st + C_OFF + h * K::C_HALF, &mapAbar16, &afull[stage], k0 + 32 * h, c0);
                    }
                    const uint32_t fb = map_to_leader(smem_u32(&full[stage]));
                    if (rank == 0) mbar_expect_tx(&full[stage], (uint32_t)(2 * (p.bn / 2) * BK * 4));
                    tma2_2d(st + B_OFF, &mapPi, fb, k0, b0, pol);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ---------------- MMA issuer (leader CTA, whole warp, elected lane issues)
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            const uint32_t idesc = F16 ? idesc2_f16(bn, false, false) : idesc2_tf32(bn, false, false);
            const uint64_t zdesc0 = smem_desc(smem_u32(smem) + Z_OFF, 16, 1024, 2);
            const uint64_t bdesc0 = smem_desc(smem_u32(smem) + B_OFF, 16, 1024, 2);
            int zs = 0;
            for (int64_t t = pair_id; t < p.ntiles; t += npairs) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(acc * (K::ACC_STRIDE ? K::ACC_STRIDE : bn));
                for (int64_t kb = 0; kb < p.nk; ++kb) {
                    if (!(p.dev & 32)) mbar_wait(&full[stage], phase);  // dev 32: the MMA loop alone (no data)
                    tc_fence_after();
                    const uint64_t off = (uint64_t)((stage * STAGE) >> 4);  // descriptor address field: 16-byte units
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        if (elect_one()) {
                            if constexpr (ZT)
                                mma2_tf32_ts(d, tmem_base + (uint32_t)(ZSLOT0 + zs * 32 + ks * 8), bdesc0 + off + 2 * ks,
                                             idesc, (kb > 0 || ks > 0) ? 1u : 0u);
                            else if constexpr (F16)
                                mma2_f16(d, zdesc0 + off + 2 * ks, bdesc0 + off + 2 * ks, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
                            else
                                mma2_tf32(d, zdesc0 + off + 2 * ks, bdesc0 + off + 2 * ks, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
                        }
                        __syncwarp();
                    }
                    if (!(p.dev & 64)) {  // dev 64: no per-K-block commit
                        if (elect_one()) commit2(&empty[stage]);
                        __syncwarp();
                    }
                    if constexpr (ZT) {
                        if (elect_one()) commit2(&zfree[zs]);
                        __syncwarp();
                        if (++zs == NZ) zs = 0;
                    }
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
                if (elect_one()) commit2(&tfull[acc]);
                __syncwarp();
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp >= TW0) {  // ---------------- Z transform (both CTAs)
        if (p.dev & 32) goto done;
        const int set = (warp - TW0) / TW_W;
        const int rho = ((warp - TW0) % TW_W) * 32 + lane;  // tile row (row_ic)
        int il, cl;
        row_ic(rho, il, cl);
        const uint32_t fb0 = map_to_leader(smem_u32(&full[0]));
        int stage = 0, sidx = 0;
        uint32_t phase = 0;
        int64_t g = 0;  // K-block counter (ZT: Z slot g mod NZ)
        // blocked (shared-memory Z) form: thread = (chunk tq, 2 i of pair tip, 4 c of quad tcq)
        const int tid = ((warp - TW0) % TW_W) * 32 + lane;
        const int tq = tid & 7, tip = (tid >> 3) & 3, tcq = tid >> 5;
        for (int64_t t = pair_id; t < p.ntiles; t += npairs) {
            float zsx[2] = {1.f, 1.f}, zsy[4] = {1.f, 1.f, 1.f, 1.f};  // F16: the exact power-of-two zscale
            if constexpr (F16) {
                const int4 tl = __ldg(&p.tiles[t]);
#pragma unroll
                for (int a = 0; a < 2; ++a) zsx[a] = __ldg(&p.zscale[tl.x * 16 + 8 * (int)rank + 2 * tip + a]);
#pragma unroll
                for (int b = 0; b < 4; ++b) zsy[b] = __ldg(&p.zscale[tl.y * 16 + 4 * tcq + b]);
            }
            for (int64_t kb = 0; kb < p.nk; ++kb, ++g) {
                const int st_ = stage;
                const uint32_t ph_ = phase;
                if (++stage == NST) { stage = 0; phase ^= 1; }
                const bool mine = sidx == set;
                if (++sidx == TW_SETS) sidx = 0;
                // every set waits on every stage in order: a set that skipped stages
                // could otherwise see a completed phase of the same parity one lap early
                mbar_wait(&afull[st_], ph_);
                if (!mine) continue;
                uint8_t* st = smem + st_ * STAGE;
                const uint8_t* ri = st + I_OFF + il * 128;
                const uint8_t* rc = st + C_OFF + cl * 128;
                if constexpr (ZT) {
                    const int zs = (int)(g % NZ);
                    // slot reuse: the MMA of K-block g - NZ is done (phase g / NZ - 1 of zfree[zs];
                    // exact: that barrier cannot run ahead of this set's own K-block g)
                    if (g >= NZ) mbar_wait(&zfree[zs], (uint32_t)(((g / NZ) - 1) & 1));
                    if (!(p.dev & 1)) {
                        float z[32];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 x = *reinterpret_cast<const float4*>(ri + ((q ^ (il & 7)) << 4));
                            const float4 y = *reinterpret_cast<const float4*>(rc + ((q ^ (cl & 7)) << 4));
                            z[4 * q] = round_tf32(x.x * y.x);
                            z[4 * q + 1] = round_tf32(x.y * y.y);
                            z[4 * q + 2] = round_tf32(x.z * y.z);
                            z[4 * q + 3] = round_tf32(x.w * y.w);
                        }
                        // row rho of this CTA's Z = TMEM lane rho, K = the slot's 32 columns
                        tmem_st32(tmem_base + ((uint32_t)(rho & ~31) << 16) + (uint32_t)(ZSLOT0 + zs * 32), z);
                    }
                    tc_fence_before();
                } else if (!(p.dev & 1)) {
                    // Blocked: thread (group gq, chunk q) forms Z chunk q of the 2 i x 4 c
                    // rows of its group from 2 + 4 abar chunks, so every activation
                    // chunk it loads serves 4 (x) or 2 (y) Z rows -- the loads were two
                    // per Z chunk, and the shared-memory load wavefronts bounded the
                    // K-block period.  A quarter-warp is one group's 8 chunks: its loads
                    // and stores hit 8 distinct 16-byte bank slots.
                    uint8_t* zb = st + Z_OFF;
                    if constexpr (F16) {
                        // Z chunk q (8 fp16) = examples 8q .. 8q + 7 = fp32 chunks 2(q % 4)
                        // and 2(q % 4) + 1 of abar box h = q / 4; box h = 1 reads its chunks
                        // in the other order, so a quarter-warp's first load covers slots
                        // {0,2,4,6} (box 0) and {1,3,5,7} (box 1) without conflicts
                        const int h = tq >> 2, ca = 2 * (tq & 3) + h, cb = 2 * (tq & 3) + 1 - h;
                        float4 x0[2], x1[2], y0[4], y1[4];
#pragma unroll
                        for (int a = 0; a < 2; ++a) {
                            const int il = 2 * tip + a;
                            const uint8_t* r = st + I_OFF + h * K::I_HALF + il * 128;
                            const float4 u = *reinterpret_cast<const float4*>(r + ((ca ^ (il & 7)) << 4));
                            const float4 v = *reinterpret_cast<const float4*>(r + ((cb ^ (il & 7)) << 4));
                            x0[a] = scale4(h ? v : u, zsx[a]);
                            x1[a] = scale4(h ? u : v, zsx[a]);
                        }
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int cl = 4 * tcq + b;
                            const uint8_t* r = st + C_OFF + h * K::C_HALF + cl * 128;
                            const float4 u = *reinterpret_cast<const float4*>(r + ((ca ^ (cl & 7)) << 4));
                            const float4 v = *reinterpret_cast<const float4*>(r + ((cb ^ (cl & 7)) << 4));
                            y0[b] = scale4(h ? v : u, zsy[b]);
                            y1[b] = scale4(h ? u : v, zsy[b]);
                        }
#pragma unroll
                        for (int a = 0; a < 2; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                const int rho = ic_row(2 * tip + a, 4 * tcq + b);
                                uint4 w;
                                w.x = h2_bits(x0[a].x * y0[b].x, x0[a].y * y0[b].y);
                                w.y = h2_bits(x0[a].z * y0[b].z, x0[a].w * y0[b].w);
                                w.z = h2_bits(x1[a].x * y1[b].x, x1[a].y * y1[b].y);
                                w.w = h2_bits(x1[a].z * y1[b].z, x1[a].w * y1[b].w);
                                *reinterpret_cast<uint4*>(zb + rho * 128 + ((tq ^ (rho & 7)) << 4)) = w;
                            }
                    } else {
                        float4 x[2], y[4];
#pragma unroll
                        for (int a = 0; a < 2; ++a) {
                            const int il = 2 * tip + a;
                            x[a] = *reinterpret_cast<const float4*>(st + I_OFF + il * 128 + ((tq ^ (il & 7)) << 4));
                        }
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int cl = 4 * tcq + b;
                            y[b] = *reinterpret_cast<const float4*>(st + C_OFF + cl * 128 + ((tq ^ (cl & 7)) << 4));
                        }
#pragma unroll
                        for (int a = 0; a < 2; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                const int rho = ic_row(2 * tip + a, 4 * tcq + b);
                                *reinterpret_cast<float4*>(zb + rho * 128 + ((tq ^ (rho & 7)) << 4)) =
                                    make_float4(round_tf32(x[a].x * y[b].x), round_tf32(x[a].y * y[b].y),
                                                round_tf32(x[a].z * y[b].z), round_tf32(x[a].w * y[b].w));
                            }
                    }
                    fence_proxy_async();
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(fb0 + st_ * 8);
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue (both CTAs, 2 groups of 4 warps)
        const int ew = warp - 4;
        const int quad = warp % 4;   // TMEM lanes 32 quad .. + 31
        const int grp = ew / 4;      // column half of the tile
        const int rho = quad * 32 + lane;
        int il, cl;
        row_ic(rho, il, cl);
        uint8_t* gbase = epi_base + grp * 4 * SLOT;  // [buf][layout][CH][128] floats
        // (dev 1024 / 2048: evict_normal / evict_last instead)
        const uint64_t spol = (p.dev & 1024) ? evict_normal_policy() : (p.dev & 2048) ? evict_last_policy() : evict_first_policy();
        const uint32_t te_leader = map_to_leader(smem_u32(&tempty[0]));
        const int half = bn / 2;
        int acc = 0;
        uint32_t acc_phase = 0;
        int chunk = 0;
        for (int64_t t = pair_id; t < p.ntiles; t += npairs) {
            const int4 tl = __ldg(&p.tiles[t]);
            const int64_t i0 = tl.x * 16 + 8 * (int)rank, c0 = tl.y * 16;
            const int64_t ii = i0 + il, cc = c0 + cl;  // this lane's abar indices
            const bool box_ok = p.tma && i0 < p.tk && c0 < p.tk && !(p.dev & 2);
            // lanes holding a bias entry (index T_k) or, without TMA, any valid entry
            const bool scalar = (ii <= p.tk && cc <= p.tk) && (ii == p.tk || cc == p.tk || !p.tma) && !(p.dev & 2);
            const int64_t jt0 = (int64_t)tl.z * p.bn;
            // F16: undo the power-of-two scales (exact): alpha / (zscale[i] zscale[c]) per
            // lane, / pscale... per column (pscale holds the inverse column scale)
            float rsc = p.alpha;
            if constexpr (F16)
                rsc = p.alpha / (__ldg(&p.zscale[i0 + il]) * __ldg(&p.zscale[c0 + cl]));
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            // chunk n + 1's TMEM load is in flight while chunk n is staged and stored
            const uint32_t tacc = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * (K::ACC_STRIDE ? K::ACC_STRIDE : bn));
            const int jend = (grp + 1) * half;
            uint32_t r[CH];
            if (jt0 + grp * half < p.npairs) tmem_ld8_issue(tacc + (uint32_t)(grp * half), r);
            for (int jj0 = grp * half; jj0 < jend; jj0 += CH) {
                const int64_t J0 = jt0 + jj0;
                if (J0 >= p.npairs) break;  // uniform across the group
                float v[CH];
                tmem_ld_wait8(r);
                if constexpr (F16) {
#pragma unroll
                    for (int e = 0; e < CH; ++e)
                        v[e] = __uint_as_float(r[e]) * rsc * (J0 + e < p.npairs ? __ldg(&p.pscale[J0 + e]) : 0.f);
                } else {
#pragma unroll
                    for (int e = 0; e < CH; ++e) v[e] = __uint_as_float(r[e]) * rsc;
                }
                if (jj0 + CH < jend && J0 + CH < p.npairs) tmem_ld8_issue(tacc + (uint32_t)(jj0 + CH), r);
                const int ncol = (int)(p.npairs - J0 < CH ? p.npairs - J0 : CH);
                if (box_ok) {
                    float* sA = reinterpret_cast<float*>(gbase + (chunk & 1) * 2 * SLOT);
                    float* sB = sA + SLOT / 4;
                    // lanes 0..7 of every warp issue boxes (warp quad = orbit type); each
                    // waits for its own stores of two chunks ago before the buffer is reused
                    if (lane < CH) bulk_wait_read1();
                    named_sync(1 + grp, 128);
#pragma unroll
                    for (int e = 0; e < CH; ++e) {
                        sA[e * 128 + il * 16 + cl] = v[e];  // [o''][i][c]
                        sB[e * 128 + cl * 8 + il] = v[e];    // [o''][c][i]
                    }
                    fence_proxy_async();
                    named_sync(1 + grp, 128);
                    if (lane < ncol) {
                        // kind 1: extent-8 box from this column (the run fills the chunk or
                        // ends at U, where the TMA clips), 2: extent-1 box, 0: inside a box
                        const int4 bx = __ldg(&p.pairs[J0 + lane]);
                        // dev 256: skip types 2, 3 (32-byte rows); dev 512: skip types 1, 4 (64-byte rows)
                        const bool skip_t = ((p.dev & 256) && (quad == 1 || quad == 2)) ||
                                            ((p.dev & 512) && (quad == 0 || quad == 3));
                        if (bx.z && !skip_t) {
                            const CUtensorMap* mp = &hm.m[(bx.z == 1 ? 0 : 4) + quad];
                            const bool ic = quad == 0 || quad == 3;  // types 1, 4: [o''][i][c]
                            const float* src = (ic ? sA : sB) + lane * 128;
                            // the row unit is o (types 1, 3: dim 3) or o'' (types 2, 4: dim 2),
                            // counted from u0; rows outside the output units are clipped by TMA
                            // (a negative coordinate is an illegal TMA store on sm_100: images
                            // of types 1, 3 with o < u0 lie wholly outside and are skipped; o''
                            // >= u0 for every packed column)
                            const bool row_o = quad == 0 || quad == 2;
                            const int32_t d2 = bx.y - (row_o ? 0 : (int32_t)p.u0);
                            const int32_t d3 = bx.x - (row_o ? (int32_t)p.u0 : 0);
                            if (d3 >= 0 && !(p.dev & 4096)) {  // dev 4096: staging and barriers, no boxes
                                if (ic) tma_store_4d(mp, src, (int32_t)c0, (int32_t)i0, d2, d3, spol);
                                else tma_store_4d(mp, src, (int32_t)i0, (int32_t)c0, d2, d3, spol);
                            }
                        }
                    }
                    if (lane < CH) bulk_commit();  // one group per chunk and lane (wait_group.read 1 above)
                    ++chunk;
                }
                if (scalar) {
#pragma unroll
                    for (int e = 0; e < CH; ++e) {
                        if (e >= ncol) break;
                        const int4 pr = __ldg(&p.pairs[J0 + e]);
                        // the four orbit entries (row unit, col unit): (o,i;o'',c) (o'',c;o,i)
                        // (o,c;o'',i) (o'',i;o,c); rows outside the output units are skipped
                        if constexpr (!BAND) {  // the whole block: all four images
                            // (a separate instantiation: the band's row mapping in this
                            // loop measured 15% slower on the whole-block kernel)
                            const int64_t r1 = hidx(p, pr.x, ii), c1 = hidx(p, pr.y, cc);
                            const int64_t r3 = hidx(p, pr.x, cc), c3 = hidx(p, pr.y, ii);
                            p.H[r1 * p.ldh + c1] = v[e];
                            p.H[c1 * p.ldh + r1] = v[e];
                            p.H[r3 * p.ldh + c3] = v[e];
                            p.H[c3 * p.ldh + r3] = v[e];
                            continue;
                        }
                        const int64_t s1 = srow(p, pr.x, ii), s2 = srow(p, pr.y, cc);
                        const int64_t s3 = srow(p, pr.x, cc), s4 = srow(p, pr.y, ii);
                        if (s1 >= 0) p.H[s1 * p.ldh + hidx(p, pr.y, cc)] = v[e];
                        if (s2 >= 0) p.H[s2 * p.ldh + hidx(p, pr.x, ii)] = v[e];
                        if (s3 >= 0) p.H[s3 * p.ldh + hidx(p, pr.y, ii)] = v[e];
                        if (s4 >= 0) p.H[s4 * p.ldh + hidx(p, pr.x, cc)] = v[e];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(te_leader + acc * 8);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (lane < CH) bulk_wait_all();
    }
done:
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

}  // namespace sym

// 4-D map of one orbit type over the diagonal block's output rows at `base`
// (the entry of row (u0, 0), column (0, 0)): dims (d0, d1, d2, d3) with element
// strides (1, s1, s2, s3), box (b0, b1, E, 1)
inline CUtensorMap make_map_orbit(float* base, int64_t d0, int64_t d1, int64_t d2, int64_t d3, int64_t s1,
                                  int64_t s2, int64_t s3, int b0, int b1, int E) {
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2, (cuuint64_t)d3};
    cuuint64_t str[3] = {(cuuint64_t)s1 * 4, (cuuint64_t)s2 * 4, (cuuint64_t)s3 * 4};
    cuuint32_t box[4] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)E, 1}, es[4] = {1, 1, 1, 1};
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (str[0] & 15) || (str[1] & 15) || (str[2] & 15))
        throw CurvError(kCudaError, "orbit map: 16-byte alignment");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CurvError(kCudaError, "cuTensorMapEncodeTiled (orbit) failed: " + std::to_string((int)r));
    return m;
}

// out[j][.] = tf32(src[(o_j * U + o''_j)][.])  -- packed profile rows; t0 >= 0: src
// holds the tangents of units t0, t0 + 1, ... only and the symmetric entry
// src[((o''_j - t0) * U + o_j)] is read instead (unit bands)
__global__ void pack_profile_kernel(const float* __restrict__ src, const int4* __restrict__ pairs, int64_t U,
                                    int64_t ldn, float* __restrict__ out, int64_t npairs, int64_t t0) {
    for (int64_t j = blockIdx.y; j < npairs; j += gridDim.y) {  // grid.y <= 65535
        const int4 pr = pairs[j];
        const int64_t row = t0 < 0 ? pr.x * U + pr.y : (pr.y - t0) * U + pr.x;
        const float4* s = reinterpret_cast<const float4*>(src + row * ldn);
        float4* d = reinterpret_cast<float4*>(out + j * ldn);
        for (int64_t q = blockIdx.x * blockDim.x + threadIdx.x; q < ldn / 4; q += gridDim.x * blockDim.x) {
            float4 v = s[q];
            v.x = round_tf32(v.x); v.y = round_tf32(v.y); v.z = round_tf32(v.z); v.w = round_tf32(v.w);
            d[q] = v;
        }
    }
}

// out[j][n] = tf32(dT[o_j][n] * dT[o''_j][n])  -- OPG profiles delta_o delta_o''
__global__ void pack_delta_products_kernel(const float* __restrict__ dT, const int4* __restrict__ pairs, int64_t ldn,
                                           float* __restrict__ out, int64_t npairs) {
    for (int64_t j = blockIdx.y; j < npairs; j += gridDim.y) {  // grid.y <= 65535
        const int4 pr = pairs[j];
        const float4* a = reinterpret_cast<const float4*>(dT + pr.x * ldn);
        const float4* b = reinterpret_cast<const float4*>(dT + pr.y * ldn);
        float4* d = reinterpret_cast<float4*>(out + j * ldn);
        for (int64_t q = blockIdx.x * blockDim.x + threadIdx.x; q < ldn / 4; q += gridDim.x * blockDim.x) {
            const float4 x = a[q], y = b[q];
            d[q] = make_float4(round_tf32(x.x * y.x), round_tf32(x.y * y.y), round_tf32(x.z * y.z), round_tf32(x.w * y.w));
        }
    }
}

// ---- F16 operands (precision kF16S) ----------------------------------------
// Exact power-of-two scales put every operand into fp16's normal range with
// headroom: |abar_i zscale[i]| < 2^7 (so |Z| < 2^14) and |Pi_j| / pscale[j]
// < 2^14, products < 2^28 in the fp32 accumulator.  Values below 2^-14 of
// the scaled range (2^-28 of a row's largest) lose significand bits to fp16
// subnormals -- ~1e-9 relative contributions, far below the 2^-12 rounding
// of the 11-bit significand every operand shares with TF32.

__device__ __forceinline__ float block_absmax(float m, float* red) {
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) red[0] = m;
    }
    __syncthreads();
    m = red[0];
    __syncthreads();
    return m;
}

// 2^(cap - e) with max|x| < 2^e: |x| * scale < 2^cap (1 for an all-zero row)
__device__ __forceinline__ float pow2_scale(float m, int cap) {
    if (!(m > 0.f) || isinf(m)) return 1.f;
    int e;
    frexpf(m, &e);
    return ldexpf(1.f, max(-126, min(127, cap - e)));
}

// zscale[i] for the abar^T rows (rows >= `rows`: 1); one CTA per row
__global__ void zscale_kernel(const float* __restrict__ akT, int64_t rows, int64_t n, int64_t ldn,
                              float* __restrict__ zscale, int64_t padded) {
    __shared__ float red[32];
    for (int64_t r = blockIdx.x; r < padded; r += gridDim.x) {
        float m = 0.f;
        if (r < rows)
            for (int64_t q = threadIdx.x; q < n; q += blockDim.x) m = fmaxf(m, fabsf(akT[r * ldn + q]));
        m = block_absmax(m, red);
        if (threadIdx.x == 0) zscale[r] = r < rows ? pow2_scale(m, 7) : 1.f;
    }
}

// out[j][.] = fp16(Pi_j[.] * w_j), pscale[j] = 1 / w_j; Pi_j = the profile row
// (o_j U + o''_j) or delta_o delta_o''; one CTA per packed column, two passes
template <bool DELTA>
__global__ void pack_h_kernel(const float* __restrict__ src, const int4* __restrict__ pairs, int64_t U, int64_t n,
                              int64_t ldn, __half* __restrict__ out, float* __restrict__ pscale, int64_t npairs,
                              int64_t t0) {
    __shared__ float red[32];
    for (int64_t j = blockIdx.x; j < npairs; j += gridDim.x) {
        const int4 pr = pairs[j];
        const float* a = DELTA ? src + pr.x * ldn
                               : src + (t0 < 0 ? pr.x * U + pr.y : (pr.y - t0) * U + pr.x) * ldn;
        const float* b = src + pr.y * ldn;
        auto val = [&](int64_t q) { return q < n ? (DELTA ? a[q] * b[q] : a[q]) : 0.f; };
        float m = 0.f;
        for (int64_t q = threadIdx.x; q < n; q += blockDim.x) m = fmaxf(m, fabsf(val(q)));
        m = block_absmax(m, red);
        const float w = pow2_scale(m, 14);
        if (threadIdx.x == 0) pscale[j] = 1.f / w;
        __half2* d = reinterpret_cast<__half2*>(out + j * ldn);
        for (int64_t q = threadIdx.x; q < ldn / 2; q += blockDim.x)
            d[q] = __floats2half2_rn(val(2 * q) * w, val(2 * q + 1) * w);
    }
}

// jt[p][n] = fp16(delta_k[n][o] abar_k[n][x] * t_{k,o} u_{k,x}), inv[p] = 1 / (t u)
// for parameter row p = weight (k, o, x < T_k) or bias (k, o; x = T_k, the ones
// row); t and u are the per-row power-of-two scales of delta_k^T and abar_k^T
// (zscale_kernel), so |jt| < 2^14.  8 examples (one 16-byte store) per thread.
__global__ void jt_f16_kernel(JtF16Args a, const float* __restrict__ us, const float* __restrict__ ts,
                              int64_t us_ld, int64_t ts_ld, __half* __restrict__ jt, float* __restrict__ inv) {
    const int64_t q8 = a.ldn / 8;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t p = blockIdx.y; p < a.P; p += gridDim.y) {
        int k = 0;
        while (k + 1 < a.S && p >= a.woff[k + 1]) ++k;
        const int64_t tk = a.w[k], nwk = a.w[k + 1] * tk;
        const int64_t rel = p - a.woff[k];
        const int64_t o = rel < nwk ? rel / tk : rel - nwk, x = rel < nwk ? rel - o * tk : tk;
        const float sc = ts[k * ts_ld + o] * us[k * us_ld + x];
        if (e == 0) inv[p] = 1.f / sc;
        if (e >= q8) continue;
        const float4* d = reinterpret_cast<const float4*>(a.dT[k] + o * a.ldn) + 2 * e;
        const float4* b = reinterpret_cast<const float4*>(a.akT[k] + x * a.ldn) + 2 * e;
        const float4 d0 = d[0], d1 = d[1], b0 = b[0], b1 = b[1];
        uint4 wv;
        wv.x = sym::h2_bits((d0.x * b0.x) * sc, (d0.y * b0.y) * sc);
        wv.y = sym::h2_bits((d0.z * b0.z) * sc, (d0.w * b0.w) * sc);
        wv.z = sym::h2_bits((d1.x * b1.x) * sc, (d1.y * b1.y) * sc);
        wv.w = sym::h2_bits((d1.z * b1.z) * sc, (d1.w * b1.w) * sc);
        reinterpret_cast<uint4*>(jt + p * a.ldn)[e] = wv;
    }
}

// out[r] = max |src[r][0 .. n)|, one CTA per row
__global__ void row_absmax_kernel(const float* __restrict__ src, int64_t rows, int64_t n, int64_t ld,
                                  float* __restrict__ out) {
    __shared__ float red[32];
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        float m = 0.f;
        for (int64_t q = threadIdx.x; q < n; q += blockDim.x) m = fmaxf(m, fabsf(src[r * ld + q]));
        m = block_absmax(m, red);
        if (threadIdx.x == 0) out[r] = m;
    }
}

// a_m^T in fp16: out[c][e] = fp16(a[e][c] u_c), u_c = the power-of-two scale of
// column c (|a u| < 2^7), inv[c] = 1 / u_c; one CTA per column (c < cols)
__global__ void am_f16_kernel(const float* __restrict__ a, int64_t lda, int64_t cols, int64_t n, int64_t ldn,
                              __half* __restrict__ out, float* __restrict__ inv) {
    __shared__ float red[32];
    for (int64_t c = blockIdx.x; c < cols; c += gridDim.x) {
        float m = 0.f;
        for (int64_t e = threadIdx.x; e < n; e += blockDim.x) m = fmaxf(m, fabsf(a[e * lda + c]));
        m = block_absmax(m, red);
        const float u = pow2_scale(m, 7);
        if (threadIdx.x == 0) inv[c] = 1.f / u;
        for (int64_t e = threadIdx.x; e < ldn; e += blockDim.x)
            out[c * ldn + e] = __float2half_rn(e < n ? a[e * lda + c] * u : 0.f);
    }
}

// R rows of one chunk in fp16 (see rgen_kernel for the row layout and the
// register reuse): row r = (o'', tangent j) scaled by s_r = 2^(14 - e) with
// |R| <= max|a_i| max|P[o][o'']| + max|delta_o| max|Q[i][o'']| < 2^e (bias rows:
// max|P|); rinv[r] = 1 / s_r.  8 examples (one 16-byte store) per thread.
__global__ void rgen_f16_kernel(HessF16Args g, const float* __restrict__ amax, const float* __restrict__ dmax,
                                const float* __restrict__ pmax, const float* __restrict__ qmax, int64_t j0, int64_t J,
                                int64_t nopp, __half* __restrict__ R, float* __restrict__ rinv) {
    constexpr int SEG = 32;
    const int64_t q8 = g.ldn / 8;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nw = g.np * g.tk;
    const int64_t segs = ceil_div(J, SEG);
    for (int64_t sg = blockIdx.y; sg < nopp * segs; sg += gridDim.y) {
        const int64_t opp = sg / segs, jj0 = (sg - opp * segs) * SEG;
        const int64_t jj1 = jj0 + SEG < J ? jj0 + SEG : J;
        int64_t last_o = -1;
        float4 p0{}, p1{}, d0{}, d1{};  // the profile and delta vectors of the current unit o
        for (int64_t jj = jj0; jj < jj1; ++jj) {
            const int64_t j = j0 + jj;
            const bool wt = j < nw;
            const int64_t o = wt ? j / g.tk : j - nw;
            const int64_t i = wt ? j - o * g.tk : 0;
            const float bound = wt ? amax[i] * pmax[o * g.tm1 + opp] + dmax[o] * qmax[i * g.tm1 + opp]
                                   : pmax[o * g.tm1 + opp];
            const float sc = pow2_scale(bound, 14);
            const int64_t r = opp * J + jj;
            if (e == 0) rinv[r] = 1.f / sc;
            if (e >= q8) continue;
            if (o != last_o || !wt) {
                const float4* pp = reinterpret_cast<const float4*>(g.prof + (o * g.tm1 + opp) * g.ldn) + 2 * e;
                p0 = pp[0];
                p1 = pp[1];
                if (wt) {
                    const float4* dp = reinterpret_cast<const float4*>(g.dkT + o * g.ldn) + 2 * e;
                    d0 = dp[0];
                    d1 = dp[1];
                }
                last_o = wt ? o : -1;
            }
            float4 v0 = p0, v1 = p1;
            if (wt) {
                const float4* ap = reinterpret_cast<const float4*>(g.akT + i * g.ldn) + 2 * e;
                const float4* qp = reinterpret_cast<const float4*>(g.q + (i * g.tm1 + opp) * g.ldn) + 2 * e;
                const float4 a0 = ap[0], a1 = ap[1], q0 = qp[0], q1 = qp[1];
                v0.x *= a0.x; v0.y *= a0.y; v0.z *= a0.z; v0.w *= a0.w;
                v1.x *= a1.x; v1.y *= a1.y; v1.z *= a1.z; v1.w *= a1.w;
                v0.x += d0.x * q0.x; v0.y += d0.y * q0.y; v0.z += d0.z * q0.z; v0.w += d0.w * q0.w;
                v1.x += d1.x * q1.x; v1.y += d1.y * q1.y; v1.z += d1.z * q1.z; v1.w += d1.w * q1.w;
            }
            uint4 w;
            w.x = sym::h2_bits(v0.x * sc, v0.y * sc);
            w.y = sym::h2_bits(v0.z * sc, v0.w * sc);
            w.z = sym::h2_bits(v1.x * sc, v1.y * sc);
            w.w = sym::h2_bits(v1.z * sc, v1.w * sc);
            reinterpret_cast<uint4*>(R + r * g.ldn)[e] = w;
        }
    }
}

}  // namespace tc

template <>
struct HessF16<float> {
    struct Prep {
        DevMem amax, dmax, pmax, qmax, am16, aminv;
    };
    static bool prepare(cudaStream_t s, const HessF16Args& a, Prep& p) {
        if (a.ldn % 8 != 0 || !a.q) return false;
        p.amax = DevMem((size_t)(a.tk + 1) * 4, s);
        p.dmax = DevMem((size_t)a.np * 4, s);
        p.pmax = DevMem((size_t)a.np * a.tm1 * 4, s);
        p.qmax = DevMem((size_t)a.tk * a.tm1 * 4, s);
        auto rmax = [&](const float* src, int64_t rows, DevMem& out) {
            tc::row_absmax_kernel<<<(unsigned)std::min<int64_t>(rows, 8192), 256, 0, s>>>(src, rows, a.n, a.ldn,
                                                                                        dptr<float>(out));
            CK_LAUNCH();
        };
        rmax(a.akT, a.tk + 1, p.amax);
        rmax(a.dkT, a.np, p.dmax);
        rmax(a.prof, a.np * a.tm1, p.pmax);
        rmax(a.q, a.tk * a.tm1, p.qmax);
        p.am16 = DevMem((size_t)(a.tm + 1) * a.ldn * 2, s);
        p.aminv = DevMem((size_t)(a.tm + 1) * 4, s);
        tc::am_f16_kernel<<<(unsigned)std::min<int64_t>(a.tm + 1, 8192), 256, 0, s>>>(
            a.am, a.lda_m, a.tm + 1, a.n, a.ldn, dptr<__half>(p.am16), dptr<float>(p.aminv));
        CK_LAUNCH();
        return true;
    }
    static void chunk(cudaStream_t s, const HessF16Args& a, const Prep& p, int64_t j0, int64_t Jc, int64_t nopp,
                      DevMem& r16, DevMem& rinv, const EpiHess<float>& e, double req) {
        const int64_t rows = nopp * Jc;
        r16 = DevMem((size_t)rows * a.ldn * 2, s);
        rinv = DevMem((size_t)rows * 4, s);
        {
            ProfScope pr("hess_rgen", s, 0.0, 2.0 * (double)rows * a.ldn);
            const dim3 g((unsigned)ceil_div(a.ldn / 8, 128), (unsigned)std::min<int64_t>(nopp * ceil_div(Jc, 32), 65535));
            tc::rgen_f16_kernel<<<g, 128, 0, s>>>(a, dptr<float>(p.amax), dptr<float>(p.dmax), dptr<float>(p.pmax),
                                                  dptr<float>(p.qmax), j0, Jc, nopp, dptr<__half>(r16),
                                                  dptr<float>(rinv));
            CK_LAUNCH();
        }
        ProfScope pg("hess_gemm", s, 2.0 * (double)a.n * req, 4.0 * req);
        gemm_f16(s, rows, a.tm + 1, a.n, dptr<__half>(r16), a.ldn, dptr<__half>(p.am16), a.ldn, dptr<float>(rinv),
                 dptr<float>(p.aminv), e);
    }
};

template <>
struct OpgF16<float> {
    static bool build(cudaStream_t s, const JtF16Args& a, DevMem& jt, DevMem& inv) {
        if (a.ldn % 8 != 0) return false;
        int64_t ul = 0, tl = 0;
        for (int k = 0; k < a.S; ++k) {
            ul = std::max(ul, a.w[k] + 1);
            tl = std::max(tl, a.w[k + 1]);
        }
        DevMem us((size_t)a.S * ul * 4, s), ts((size_t)a.S * tl * 4, s);
        for (int k = 0; k < a.S; ++k) {
            tc::zscale_kernel<<<(unsigned)std::min<int64_t>(a.w[k] + 1, 4096), 256, 0, s>>>(
                a.akT[k], a.w[k] + 1, a.n, a.ldn, dptr<float>(us) + k * ul, a.w[k] + 1);
            CK_LAUNCH();
            tc::zscale_kernel<<<(unsigned)std::min<int64_t>(a.w[k + 1], 4096), 256, 0, s>>>(
                a.dT[k], a.w[k + 1], a.n, a.ldn, dptr<float>(ts) + k * tl, a.w[k + 1]);
            CK_LAUNCH();
        }
        jt = DevMem((size_t)a.P * a.ldn * 2, s);
        inv = DevMem((size_t)a.P * 4, s);
        dim3 g((unsigned)ceil_div(a.ldn / 8, 128), (unsigned)std::min<int64_t>(a.P, 65535));
        tc::jt_f16_kernel<<<g, 128, 0, s>>>(a, dptr<float>(us), dptr<float>(ts), ul, tl, dptr<__half>(jt),
                                           dptr<float>(inv));
        CK_LAUNCH();
        return true;
    }
    static void rect(cudaStream_t s, int64_t r0, int64_t r1, int64_t cols, int64_t n, const DevMem& jt, int64_t ldn,
                     const DevMem& inv, float* G, int64_t ldg, float alpha) {
        EpiSymLower<float> e{G, ldg, alpha, r0};
        gemm_f16(s, r1 - r0, cols, n, dptr<__half>(jt) + r0 * ldn, ldn, dptr<__half>(jt), ldn,
                 dptr<float>(inv) + r0, dptr<float>(inv), e);
    }
};

template <>
struct SymKr<float> {
    // Applicability of the TMA orbit epilogue (else the caller keeps the other kernels)
    static bool tma_ok(const float* H, int64_t ldh, int64_t woff, int64_t tk) {
        return ldh % 4 == 0 && woff % 4 == 0 && tk % 4 == 0 && (reinterpret_cast<uintptr_t>(H) & 15) == 0;
    }

    static bool run(int prec, cudaStream_t s, const SymKrArgs<float>& a) {
        if (!tf32_class(prec)) return false;
        const bool f16 = prec == kF16S;
        // without TMA-addressable H (pitch or offset not 16-byte aligned) every
        // entry takes the scalar path: slower, same values
        const int tma = tma_ok(a.H, a.ldh, a.woff, a.tk) ? 1 : 0;
        namespace sym = tc::sym;
        const int64_t U = a.U, tk = a.tk;
        // output units [u0, u1): the packed columns (o <= o'') with o'' in [u0, u1)
        // carry every entry of those units' rows whose column unit is <= the row's
        // (the entries of the other orbit images fall outside and are not stored)
        const int64_t u0 = a.u0, u1 = a.u1 < 0 ? U : a.u1;
        if (u0 < 0 || u1 > U || u0 >= u1) return true;
        const int64_t bwoff = a.bwoff < 0 ? a.woff : a.bwoff, bboff = a.bboff < 0 ? a.boff : a.bboff;
        // packed columns, o-major
        // (pair_q0 / pair_q1: a sub-range of o'' with the rows left unrestricted)
        const int64_t q0 = std::max(u0, a.pair_q0), q1 = a.pair_q1 < 0 ? u1 : std::min(u1, a.pair_q1);
        if (q0 >= q1) return true;
        std::vector<int4> pairs;
        for (int64_t o = 0; o < q1; ++o)
            for (int64_t q = std::max(o, q0); q < q1; ++q) pairs.push_back(make_int4((int)o, (int)q, 0, 0));
        const int64_t np = (int64_t)pairs.size();
        // TMA box decomposition per 8-column chunk (chunks start at multiples of 8:
        // tile widths are multiples of 16): runs of one o with consecutive o''; a
        // run ending at u1 may take the extent-8 box (the maps clip at u1)
        for (int64_t j0 = 0; j0 < np; j0 += sym::CH) {
            const int64_t j1 = std::min<int64_t>(np, j0 + sym::CH);
            for (int64_t e = j0; e < j1;) {
                int64_t L = 1;
                while (e + L < j1 && pairs[e + L].x == pairs[e].x) ++L;
                const bool wide = L == sym::CH || pairs[e].y + L == u1;
                if (wide) pairs[e].z = 1;
                else
                    for (int64_t u = 0; u < L; ++u) pairs[e + u].z = 2;
                e += L;
            }
        }
        // Z in shared memory (default) or in TMEM (CURVKIT_SYMKR_TS=1: correct, but measured
        // slower on B200 -- c1 1.08 vs 0.92 ms, c2 9.2 vs 8.6 ms, c3 97.7 vs 85.7 ms)
        static const bool zt_env = getenv("CURVKIT_SYMKR_TS") != nullptr;
        const bool zt = zt_env && !f16;
        const int64_t max_bn = zt ? sym::Cfg<true>::MAX_BN : sym::Cfg<false>::MAX_BN;
        const int64_t ntn = ceil_div(np, max_bn);
        const int64_t bn = round_up(ceil_div(np, ntn), 16);  // <= max_bn
        const int64_t nb = ceil_div(tk + 1, 16);  // 16-blocks of abar indices
        // Tile order = write locality: the ~74 tiles in flight walk an SB x SB square
        // of (ib, cb) blocks, so both the c-contiguous (types 1, 4) and the
        // i-contiguous (types 2, 3) row segments of concurrent tiles are adjacent in H.
        // measured: 5 best on c1 (0.92 vs 1.00 ms row-major); a packed profile larger than
        // ~1/4 of L2 is re-read from HBM once per square (c3: 330 MB, 55 squares, 33 GB of
        // reads), so larger squares there (c3 symkr 81.5 -> 79.5 ms at 10-25)
        static const int64_t SB_env = getenv("CURVKIT_SYMKR_SB") ? atoi(getenv("CURVKIT_SYMKR_SB")) : -1;
        const int64_t SB = SB_env >= 0 ? SB_env : ((double)np * a.ldn * (f16 ? 2 : 4) > 32e6 ? 12 : 5);
        std::vector<int4> tiles;
        if (SB <= 0) {
            for (int64_t ib = 0; ib < nb; ++ib)
                for (int64_t cb = ib; cb < nb; ++cb)
                    for (int64_t nt = 0; nt < ntn; ++nt) tiles.push_back(make_int4((int)ib, (int)cb, (int)nt, 0));
        } else {
            for (int64_t IB = 0; IB < nb; IB += SB)
                for (int64_t CB = IB; CB < nb; CB += SB)
                    for (int64_t nt = 0; nt < ntn; ++nt)
                        for (int64_t ib = IB; ib < std::min(nb, IB + SB); ++ib)
                            for (int64_t cb = std::max(ib, CB); cb < std::min(nb, CB + SB); ++cb)
                                tiles.push_back(make_int4((int)ib, (int)cb, (int)nt, 0));
        }
        const int4* dpairs = static_cast<const int4*>(cached_upload(pairs.data(), pairs.size() * sizeof(int4)));
        const int4* dtiles = static_cast<const int4*>(cached_upload(tiles.data(), tiles.size() * sizeof(int4)));
        // packed profiles (B operand, K-major rows of ldn examples), rounded to nearest TF32
        // (F16: scaled and rounded to nearest fp16, with the column scales)
        DevMem pi((size_t)np * a.ldn * (f16 ? 2 : 4), s);
        DevMem psc(f16 ? (size_t)np * 4 : 0, s), zsc(f16 ? (size_t)nb * 16 * 4 : 0, s);
        if (f16) {
            const unsigned g = (unsigned)std::min<int64_t>(np, 8 * tc::num_sms());
            if (a.delta_products)
                tc::pack_h_kernel<true><<<g, 256, 0, s>>>(a.prof, dpairs, U, a.n, a.ldn, dptr<__half>(pi), dptr<float>(psc), np, -1);
            else
                tc::pack_h_kernel<false><<<g, 256, 0, s>>>(a.prof, dpairs, U, a.n, a.ldn, dptr<__half>(pi), dptr<float>(psc), np,
                                                           a.prof_t0);
            CK_LAUNCH();
            tc::zscale_kernel<<<(unsigned)std::min<int64_t>(nb * 16, 4096), 256, 0, s>>>(a.akT, tk + 1, a.n, a.ldn,
                                                                                         dptr<float>(zsc), nb * 16);
        } else if (a.delta_products)
            tc::pack_delta_products_kernel<<<dim3((unsigned)ceil_div(a.ldn / 4, 256), (unsigned)std::min<int64_t>(np, 65535)), 256, 0, s>>>(
                a.prof, dpairs, a.ldn, dptr<float>(pi), np);
        else
            tc::pack_profile_kernel<<<dim3((unsigned)ceil_div(a.ldn / 4, 256), (unsigned)std::min<int64_t>(np, 65535)), 256, 0, s>>>(
                a.prof, dpairs, U, a.ldn, dptr<float>(pi), np, a.prof_t0);
        CK_LAUNCH();
        CUtensorMap m8 = tc::make_map(a.akT, tk + 1, a.n, a.ldn, 0, 8);
        CUtensorMap m16 = tc::make_map(a.akT, tk + 1, a.n, a.ldn, 0, 16);
        CUtensorMap mpi = f16 ? tc::make_map_f16(dptr<__half>(pi), np, a.n, a.ldn, (int)(bn / 2))
                              : tc::make_map(dptr<float>(pi), np, a.n, a.ldn, 0, (int)(bn / 2));
        tc::sym::HMaps hm;
        std::memset(&hm, 0, sizeof hm);
        const int64_t L = a.ldh, nu = u1 - u0;
        // row unit dims count from u0 (nu units), column unit dims end at u1: the
        // TMA clips every image whose row lies outside the output units
        float* base = a.H + bwoff * L + a.woff;
        for (int x = 0; tma && x < 2; ++x) {
            const int E = x == 0 ? 8 : 1;
            // type 1: H[(o,i),(o'',c)]  d = (c, i, o'' col, o row), strides (1, L, tk, tk L)
            hm.m[4 * x + 0] = tc::make_map_orbit(base, tk, tk, u1, nu, L, tk, tk * L, 16, 8, E);
            // type 2: H[(o'',c),(o,i)]  d = (i, c, o'' row, o col), strides (1, L, tk L, tk)
            hm.m[4 * x + 1] = tc::make_map_orbit(base, tk, tk, nu, u1, L, tk * L, tk, 8, 16, E);
            // type 3: H[(o,c),(o'',i)]  d = (i, c, o'' col, o row), strides (1, L, tk, tk L)
            hm.m[4 * x + 2] = tc::make_map_orbit(base, tk, tk, u1, nu, L, tk, tk * L, 8, 16, E);
            // type 4: H[(o'',i),(o,c)]  d = (c, i, o'' row, o col), strides (1, L, tk L, tk)
            hm.m[4 * x + 3] = tc::make_map_orbit(base, tk, tk, nu, u1, L, tk * L, tk, 16, 8, E);
        }
        sym::Params prm{dtiles, (int64_t)tiles.size(), dpairs, np, bn, tk,
                        ceil_div(a.n, f16 ? (int64_t)sym::Cfg<false, true>::KB : (int64_t)tc::BK), U, a.H, a.ldh,
                        a.woff, a.boff, a.alpha, tma, 0, u0, u1, bwoff, bboff,
                        f16 ? dptr<float>(zsc) : nullptr, f16 ? dptr<float>(psc) : nullptr};
        static const int dev = getenv("CURVKIT_DEV_SYMKR") ? atoi(getenv("CURVKIT_DEV_SYMKR")) : 0;
        prm.dev = dev;
        func_attr_once((const void*)sym::symkr_kernel<true, false>, [] {
            CK_CUDA(cudaFuncSetAttribute(sym::symkr_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         sym::Cfg<true>::SMEM_BYTES));
            CK_CUDA(cudaFuncSetAttribute(sym::symkr_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         sym::Cfg<false>::SMEM_BYTES));
            CK_CUDA(cudaFuncSetAttribute(sym::symkr_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         sym::Cfg<false>::SMEM_BYTES));
            CK_CUDA(cudaFuncSetAttribute(sym::symkr_kernel<false, false, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, sym::Cfg<false, true>::SMEM_BYTES));
            CK_CUDA(cudaFuncSetAttribute(sym::symkr_kernel<false, true, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, sym::Cfg<false, true>::SMEM_BYTES));
        });
        const int grid = 2 * (int)std::min<int64_t>((int64_t)tiles.size(), tc::num_sms() / 2);
        const bool band = u0 != 0 || u1 != U || bwoff != a.woff || bboff != a.boff;
        if (f16 && band)
            sym::symkr_kernel<false, true, true><<<grid, sym::kThreads, sym::Cfg<false, true>::SMEM_BYTES, s>>>(m8, m16, mpi, hm, prm);
        else if (f16)
            sym::symkr_kernel<false, false, true><<<grid, sym::kThreads, sym::Cfg<false, true>::SMEM_BYTES, s>>>(m8, m16, mpi, hm, prm);
        else if (band)
            sym::symkr_kernel<false, true><<<grid, sym::kThreads, sym::Cfg<false>::SMEM_BYTES, s>>>(m8, m16, mpi, hm, prm);
        else if (zt)
            sym::symkr_kernel<true, false><<<grid, sym::kThreads, sym::Cfg<true>::SMEM_BYTES, s>>>(m8, m16, mpi, hm, prm);
        else
            sym::symkr_kernel<false, false><<<grid, sym::kThreads, sym::Cfg<false>::SMEM_BYTES, s>>>(m8, m16, mpi, hm, prm);
        CK_LAUNCH();
        return true;
    }
};

}  // namespace ck
