// kr.cuh -- J X and J^T T for the randomized top-k OPG eigensolver without
// ever forming J (the N x P matrix of per-example gradients).
//
// Row n of J restricted to layer k's weights is the Khatri-Rao (row-wise
// Kronecker) product delta_k[n, :] (x) a_k[n, :] -- reference autodiff.cpp
// accumulates exactly these outer products per example -- and its bias part
// is delta_k[n, :].  Hence, with X_{k,o} = rows woff_k + o*T_k .. + T_k - 1
// of X (the tangents of output unit o's incoming weights):
//
//   (J X)[n, c]           = sum_k sum_o delta_k[n, o] (A_k X_{k,o})[n, c]
//                           + sum_k (delta_k Xb_k)[n, c]
//   (J^T T)[(k,o,i), c]   = sum_n a_k[n, i] delta_k[n, o] T[n, c]
//   (J^T T)[(k,o), c]     = (delta_k^T T)[o, c]                    (biases)
//
// The same flops as the dense products (2 N P l each) but the operands are
// the activations (N x T_k) and the l-column blocks, all L2-resident, instead
// of an N x P matrix streamed from HBM (84 GB for config 4): the products are
// tensor-core bound instead of HBM bound, and J's allocation and generation
// disappear.
//
// Both kernels are CTA-pair (cta_group::2) tcgen05 kind::tf32 GEMMs with
// 256 x 256 tiles whose N = 256 columns are two output units o (128 columns
// of c each, one per CTA of the pair):
//   kr_kernel<false>  (J X): D = A_k[n-tile, :] [X_{k,o} | X_{k,o+1}]; the
//       epilogue scales each TMEM row by delta_k[n, o] and accumulates over a
//       chunk of o in registers, then stores one K-slab of partial sums
//       (summed in fixed order afterwards: deterministic).
//   kr_kernel<true>   (J^T T): D = A_k^T[i-tile, :] [delta_o . T | delta_o+1 . T];
//       transform warps scale the TMA-loaded T tile's k-rows (examples) by
//       delta_k[n, o] in shared memory (a 128-byte swizzle row is one k, so
//       the scaling is swizzle-agnostic), round to nearest TF32, and hand the
//       stage to the MMA.
#pragma once

#include "gemm_tc.cuh"
#include "model.cuh"

namespace ck {
namespace tc {
namespace pair {

struct KrArgs {
    int64_t mt;           // row tiles (JX: n-tiles of 256 examples; JT: i-tiles of 256 inputs)
    int64_t nop;          // o pairs: ceil((oend - o0) / 2) (JT F16: o quads, ceil((oend - o0) / 4))
    int64_t chunk;        // JX: o pairs per work unit
    int64_t nk;           // k-blocks per o pair (JX: ceil(T_k / 32); JT: ceil(n / 32))
    int64_t tk, to, woff;  // T_k, T_{k+1}, first weight row of layer k in X / Y
    const float* delta;    // JX: delta_k (n x ldd); JT: delta_k^T (T_{k+1} x ldd, ldd >= 32 nk)
    int64_t ldd;
    int64_t n;             // examples
    float* out;            // JX: slab workspace (+ slab0 * slab); JT: Y (+ c0)
    int64_t ldo, slab;     // JX: floats per slab
    int64_t rows;          // JX: n ; JT: T_k
    int64_t l;             // live columns of this 128-wide column tile
    int64_t ksplit;        // JT: example slabs (partial Y in slab ks of out)
    int64_t o0, oend;      // output units o0 .. oend - 1 of the layer (a shard's range)
    int64_t prow0;         // parameter row held at row 0 of X (JX) / Y (JT)
    // F16 (precision kF16S, J X): inverse power-of-two scales of the fp16
    // operands -- per example row of a_k and per column c of X^T
    const float* rinv = nullptr;
    const float* cinv = nullptr;
    // F16 J^T T: max |delta_k[:, o]| per unit and max |T[:, c]| per column of this
    // tile: the operand scale of unit o, column c is pow2_scale(dmax tmax, 14)
    const float* dmax = nullptr;
    const float* tmax = nullptr;
};

constexpr int KR_BN = 256;

// JT F16 ("quad" units: each CTA of the pair computes TWO output units
// o, o + 2 against the same A and T tiles, i.e. four units per pair and two
// N = 256 MMAs per k-step into the whole TMEM): the B stage holds the raw fp32
// T^T tile (128 columns c x 64 examples, two 128-byte boxes), the second
// unit's fp16 operand (16 KB) and the two delta_o rows (256 bytes each); the
// transform writes the first unit's operand over box 0, row by row (each
// thread one row c, read before written)
template <bool JT, bool F16 = false>
struct KrCfg {
    static constexpr int THREADS = 128 + 32 * EPI_WARPS + (JT ? 128 : 0);
    static constexpr int A_BYTES = 128 * BK * 4;
    static constexpr int B_BYTES = (JT && F16) ? 3 * (KR_BN / 2) * BK * 4 + 1024 : (KR_BN / 2) * BK * 4;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_BYTES = 0;  // epilogues store from registers
    static constexpr int STAGES_ = (227 * 1024 - 1024 - EPI_BYTES - 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_ > 8 ? 8 : STAGES_;
    static constexpr int BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + 1024;
};

// F16 (J X only): A = a_k in fp16 (K-major over the inputs i, rows scaled by
// 1 / rinv), B = X^T in fp16 (K-major over the parameter rows, columns scaled
// by 1 / cinv); 64 inputs per 128-byte operand row, kind::f16 MMAs; the
// epilogue undoes both scales on the summed row (exact).
template <bool JT, bool F16 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(KrCfg<JT, F16>::THREADS, 1)
kr_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
          const __grid_constant__ CUtensorMap mapDelta, KrArgs ka,
          uint32_t mn_lbo, uint32_t mn_sbo, uint32_t mn_kstep, int a3d, int b3d) {
    using C = KrCfg<JT, F16>;
    constexpr int KBE = F16 ? 2 * BK : BK;  // K elements per 128-byte operand row
    constexpr bool QUAD = JT && F16;        // two units per CTA, no accumulator double buffer
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int NST = C::STAGES;
    uint8_t* stage_base = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * C::STAGE_BYTES + C::EPI_BYTES);
    uint64_t* full = bars;         // [8] leader: operand bytes (+ transform arrivals)
    uint64_t* empty = bars + 8;    // [8] both CTAs (multicast commit)
    uint64_t* bfull = bars + 16;   // [8] local: raw T tile landed (JT)
    uint64_t* tfull = bars + 24;   // [2]
    uint64_t* tempty = bars + 26;  // [2] leader
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 28);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cta_rank();
    const int64_t pair_id = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int64_t nchunk = JT ? ka.nop * ka.ksplit : ceil_div(ka.nop, ka.chunk);
    const int64_t nunits = ka.mt * nchunk;
    const int64_t kcb = JT ? ceil_div(ka.nk, ka.ksplit) : ka.nk;
    constexpr int TW0 = 4 + EPI_WARPS;
    // unit u -> (row tile, o-pair range, k-block range, slab); units sharing
    // an o range run side by side, so the B operand they stream stays in L2
    auto unit_of = [&](int64_t u, int64_t& mi, int64_t& op0, int64_t& op1, int64_t& kb0, int64_t& kb1,
                       int64_t& slab) {
        mi = u % ka.mt;
        const int64_t ch = u / ka.mt;
        if (JT) {
            op0 = ch % ka.nop;
            op1 = op0 + 1;
            slab = ch / ka.nop;
            kb0 = slab * kcb;
            kb1 = ::min(ka.nk, kb0 + kcb);
        } else {
            op0 = ch * ka.chunk;
            op1 = ::min(ka.nop, op0 + ka.chunk);
            slab = ch;
            kb0 = 0;
            kb1 = ka.nk;
        }
    };

    if (warp == 0 && lane == 0) {
        prefetch_map(&mapA);
        prefetch_map(&mapB);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], JT ? 1 + 2 * 4 : 2);
            mbar_init(&empty[s], 1);
            mbar_init(&bfull[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                     "n"(2 * KR_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol = evict_last_policy();
            for (int64_t u = pair_id; u < nunits; u += npairs) {
                int64_t mi, op0, op1, kb0, kb1, sl;
                unit_of(u, mi, op0, op1, kb0, kb1, sl);
                const int64_t r0 = mi * 256 + 128 * rank;  // this CTA's A rows
                for (int64_t op = op0; op < op1; ++op) {
                    const int64_t o = ka.o0 + (QUAD ? 4 : 2) * op + rank;  // this CTA's (first) output unit
                    for (int64_t kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = stage_base + stage * C::STAGE_BYTES;
                        uint8_t* sb = sa + C::A_BYTES;
                        const uint32_t fb = map_to_leader(smem_u32(&full[stage]));
                        const int64_t k0 = kb * KBE;
                        if constexpr (JT && F16) {
                            // A = a_k^T in fp16 (K-major over examples); raw T^T boxes + delta_o
                            if (rank == 0) mbar_expect_tx(&full[stage], (uint32_t)(2 * C::A_BYTES));
                            load_tile2<128>(sa, &mapA, fb, 0, 0, r0, k0, pol);
                            // both CTAs scale the same T^T tile: each loads one of its two
                            // boxes into both (the peer's stage is free: the pair MMA that
                            // last read it has committed to both CTAs' empty barriers)
                            mbar_expect_tx(&bfull[stage], (uint32_t)(2 * 16384 + 512));
                            tma_load_2d_mc(sb + rank * 16384, &mapB, &bfull[stage], (int32_t)(k0 + 32 * rank), 0,
                                           (uint16_t)3);
                            tma_load_2d(sb + 49152, &mapDelta, &bfull[stage], (int32_t)k0,
                                        (int32_t)(o < ka.oend ? o : ka.o0));
                            tma_load_2d(sb + 49152 + 256, &mapDelta, &bfull[stage], (int32_t)k0,
                                        (int32_t)(o + 2 < ka.oend ? o + 2 : ka.o0));
                        } else if constexpr (JT) {
                            if (rank == 0) mbar_expect_tx(&full[stage], (uint32_t)(2 * C::A_BYTES));
                            load_tile2<128>(sa, &mapA, fb, 1, a3d, r0, k0, pol);
                            mbar_expect_tx(&bfull[stage], (uint32_t)C::B_BYTES);
                            load_tile<128>(sb, &mapB, &bfull[stage], 1, b3d, 0, k0, 4);
                        } else {
                            if (rank == 0) mbar_expect_tx_cluster(&full[stage], (uint32_t)(2 * C::STAGE_BYTES));
                            else mbar_arrive_cluster(fb);
                            load_tile2<128>(sa, &mapA, fb, 0, 0, r0, k0, pol);
                            // rows of X past this unit's T_k meet zero-filled A columns
                            if constexpr (F16)  // X^T: K-major, rows = columns c of X
                                load_tile2<128>(sb, &mapB, fb, 0, 0, 0, ka.woff + o * ka.tk + k0 - ka.prow0, pol);
                            else
                                load_tile2<128>(sb, &mapB, fb, 1, b3d, 0, ka.woff + o * ka.tk + k0 - ka.prow0, pol);
                        }
                        if (++stage == NST) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ---------------- MMA issuer (leader CTA, whole warp; elected lane issues)
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            const uint32_t idesc = F16 ? idesc2_f16(KR_BN, false, false) : idesc2_tf32(KR_BN, JT, true);
            for (int64_t u = pair_id; u < nunits; u += npairs) {
                int64_t mi, op0, op1, kb0, kb1, sl;
                unit_of(u, mi, op0, op1, kb0, kb1, sl);
                for (int64_t op = op0; op < op1; ++op) {
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem_base + (uint32_t)(acc * KR_BN);  // QUAD: acc = 0, columns 0 .. 511
                    for (int64_t kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t sa = smem_u32(stage_base + stage * C::STAGE_BYTES);
                        const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
                        for (int ks = 0; ks < BK / 8; ++ks) {
                            const uint64_t ad = (JT && !F16) ? smem_desc(sa + ks * mn_kstep, mn_lbo, mn_sbo, 1)
                                                             : smem_desc(sa + ks * 32, 16, 1024, 2);
                            if constexpr (F16) {  // both K-major: K = 16 per MMA in the same 32 bytes
                                const uint64_t bd = smem_desc(sb + ks * 32, 16, 1024, 2);
                                if (elect_one()) {
                                    mma2_f16(d, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
                                    if constexpr (QUAD)  // the second unit pair: B at +32 KB, columns 256 ..
                                        mma2_f16(d + KR_BN, ad, smem_desc(sb + 32768 + ks * 32, 16, 1024, 2), idesc,
                                                 (kb > kb0 || ks > 0) ? 1u : 0u);
                                }
                                __syncwarp();
                            } else {
                                const uint64_t bd = smem_desc(sb + ks * mn_kstep, mn_lbo, mn_sbo, 1);
                                mma2_tf32_e(d, ad, bd, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
                            }
                        }
                        commit2_e(&empty[stage]);
                        if (++stage == NST) { stage = 0; phase ^= 1; }
                    }
                    commit2_e(&tfull[acc]);
                    if (QUAD || ++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
            }
        }
    } else if (JT && F16 && warp >= TW0) {  // ---------------- fp16 B rows (both CTAs)
        // thread t = column c of this CTA's unit o: row c of the raw T^T tile
        // (examples k0 .. k0 + 63 in two 128-byte boxes) times delta_o (staged
        // 256 bytes), scaled by the power of two of (o, c), rounded to fp16 and
        // written back as row c of box 0 (each thread reads its row first)
        const int c = threadIdx.x - TW0 * 32;
        const uint32_t fb0 = map_to_leader(smem_u32(&full[0]));
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t u = pair_id; u < nunits; u += npairs) {
            int64_t mi, op0, op1, kb0, kb1, sl;
            unit_of(u, mi, op0, op1, kb0, kb1, sl);
            const int64_t o = ka.o0 + 4 * op0 + rank;  // units o (box 0) and o + 2 (+32 KB)
            const float tm = c < ka.l ? __ldg(ka.tmax + c) : 0.f;
            const float sc0 = o < ka.oend ? pow2_scale(__ldg(ka.dmax + o) * tm, 14) : 0.f;
            const float sc1 = o + 2 < ka.oend ? pow2_scale(__ldg(ka.dmax + o + 2) * tm, 14) : 0.f;
            for (int64_t kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&bfull[stage], phase);
                uint8_t* sb = stage_base + stage * C::STAGE_BYTES + C::A_BYTES;
                const float4* dl = reinterpret_cast<const float4*>(sb + 49152);
                float4 x[16];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        x[8 * h + q] = *reinterpret_cast<const float4*>(sb + h * 16384 + c * 128 + ((q ^ (c & 7)) << 4));
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float sc = u ? sc1 : sc0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {  // output chunk q = examples 8q .. 8q + 7 = raw chunks 2q, 2q + 1
                        const float4 a0 = x[2 * q], a1 = x[2 * q + 1], d0 = dl[16 * u + 2 * q], d1 = dl[16 * u + 2 * q + 1];
                        uint4 w;
                        w.x = sym::h2_bits(a0.x * d0.x * sc, a0.y * d0.y * sc);
                        w.y = sym::h2_bits(a0.z * d0.z * sc, a0.w * d0.w * sc);
                        w.z = sym::h2_bits(a1.x * d1.x * sc, a1.y * d1.y * sc);
                        w.w = sym::h2_bits(a1.z * d1.z * sc, a1.w * d1.w * sc);
                        *reinterpret_cast<uint4*>(sb + u * 32768 + c * 128 + ((q ^ (c & 7)) << 4)) = w;
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(fb0 + stage * 8);
                if (++stage == NST) { stage = 0; phase ^= 1; }
            }
        }
    } else if (JT && warp >= TW0) {  // ---------------- T-tile scaling (both CTAs)
        // thread t scales the 16-byte chunks t + 128 r (r < 8) of this CTA's
        // 16 KB T tile, so one warp instruction covers 512 contiguous bytes
        // (no bank conflicts).  Chunk g sits in 128-byte row g / 8 = one k
        // (example) of a 32-column atom: k = t / 8 for even r, t / 8 + 16 for odd.
        const int t = threadIdx.x - TW0 * 32;
        const int klo = t / 8;
        const uint32_t fb0 = map_to_leader(smem_u32(&full[0]));
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t u = pair_id; u < nunits; u += npairs) {
            int64_t mi, op0, op1, kb0, kb1, sl;
            unit_of(u, mi, op0, op1, kb0, kb1, sl);
            const int64_t o = ka.o0 + 2 * op0 + rank;
            // delta_k^T row o, eight k-blocks ahead of the stages that need them
            const float* drow = ka.delta + (o < ka.oend ? o : ka.o0) * ka.ldd + klo;
            const float live = o < ka.oend ? 1.f : 0.f;
            for (int64_t kbg = kb0; kbg < kb1; kbg += 8) {
                float d0[8], d1[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const bool in = kbg + j < kb1;
                    d0[j] = in ? live * __ldg(drow + (kbg + j) * BK) : 0.f;
                    d1[j] = in ? live * __ldg(drow + (kbg + j) * BK + 16) : 0.f;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (kbg + j >= kb1) break;
                    mbar_wait(&bfull[stage], phase);
                    float4* p = reinterpret_cast<float4*>(stage_base + stage * C::STAGE_BYTES + C::A_BYTES) + t;
                    float4 x[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) x[r] = p[128 * r];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const float dv = (r & 1) ? d1[j] : d0[j];
                        x[r].x = round_tf32(x[r].x * dv); x[r].y = round_tf32(x[r].y * dv);
                        x[r].z = round_tf32(x[r].z * dv); x[r].w = round_tf32(x[r].w * dv);
                        p[128 * r] = x[r];
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(fb0 + stage * 8);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp >= 4 && warp < TW0) {  // ---------------- epilogue (both CTAs)
        const int ew = warp - 4;
        const int quad = warp % 4;   // TMEM lanes 32*quad .. +31
        const int chalf = ew / 4;
        const uint32_t te_leader = map_to_leader(smem_u32(&tempty[0]));
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t u = pair_id; u < nunits; u += npairs) {
            int64_t mi, op0, op1, kb0, kb1, sl;
            unit_of(u, mi, op0, op1, kb0, kb1, sl);
            const int64_t row0 = mi * 256 + 128 * rank + quad * 32;
            if constexpr (!JT) {
                // row n = row0 + lane; columns 64*chalf .. +63 of both o of each pair
                const int64_t nrow = row0 + lane;
                const bool live = nrow < ka.rows;
                float sum[64];
#pragma unroll
                for (int j = 0; j < 64; ++j) sum[j] = 0.f;
                for (int64_t op = op0; op < op1; ++op) {
                    mbar_wait(&tfull[acc], acc_phase);
                    tc_fence_after();
#pragma unroll
                    for (int x = 0; x < 2; ++x) {
                        const int64_t o = ka.o0 + 2 * op + x;
                        const float dv = (live && o < ka.oend) ? __ldg(ka.delta + nrow * ka.ldd + o) : 0.f;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            float v[32];
                            tmem_ld32(lane_base + (uint32_t)(acc * KR_BN + x * 128 + chalf * 64 + h * 32), v);
#pragma unroll
                            for (int j = 0; j < 32; ++j) sum[h * 32 + j] = fmaf(dv, v[j], sum[h * 32 + j]);
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(te_leader + acc * 8);
                    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
                if (live) {
                    if constexpr (F16) {  // undo the operand scales: row n, columns c
                        const float rs = __ldg(ka.rinv + nrow);
#pragma unroll
                        for (int j = 0; j < 64; ++j) sum[j] *= rs * __ldg(ka.cinv + chalf * 64 + j);
                    }
                    float4* dst = reinterpret_cast<float4*>(ka.out + sl * ka.slab + nrow * ka.ldo + chalf * 64);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        __stcs(dst + j, make_float4(sum[4 * j], sum[4 * j + 1], sum[4 * j + 2], sum[4 * j + 3]));
                }
            } else {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                // TMEM columns 128*chalf.. hold output unit o (QUAD: columns
                // 256 u + 128 chalf.. unit o0 + 4 op + 2 u + chalf); lane = input
                // i, whose 32-column run of Y row (woff + o T_k + i) is contiguous
                const int64_t i = row0 + lane;
                const bool vec = (ka.ldo & 3) == 0;
                const float ri = (F16 && i < ka.rows) ? __ldg(ka.rinv + i) : 1.f;
#pragma unroll 1
                for (int u = 0; u < (QUAD ? 2 : 1); ++u)
#pragma unroll 1
                for (int cb = 0; cb < 4; ++cb) {
                    const int64_t o = ka.o0 + (QUAD ? 4 : 2) * op0 + 2 * u + chalf;
                    float* yrow = ka.out + sl * ka.slab + (ka.woff + o * ka.tk + i - ka.prow0) * ka.ldo;
                    const float dm = (F16 && o < ka.oend) ? __ldg(ka.dmax + o) : 0.f;
                    const int64_t c0 = cb * 32;
                    if (c0 >= ka.l || o >= ka.oend) break;
                    float v[32];
                    tmem_ld32(lane_base + (uint32_t)(acc * KR_BN + u * KR_BN + chalf * 128 + cb * 32), v);
                    if constexpr (F16) {  // undo the operand scales (exact): row i, (unit o, column c)
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            v[j] *= c0 + j < ka.l ? ri / pow2_scale(dm * __ldg(ka.tmax + c0 + j), 14) : 0.f;
                    }
                    if (i < ka.rows) {
                        if (vec && c0 + 32 <= ka.l) {
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                __stcs(reinterpret_cast<float4*>(yrow + c0) + q,
                                       make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (c0 + j < ka.l) yrow[c0 + j] = v[j];
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(te_leader + acc * 8);
                if (QUAD || ++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(2 * KR_BN));
    }
}

}  // namespace pair

// out[r, c] = tf32(in[r, c]) for c < cols, 0 in the padding columns
__global__ void round_pad_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t rows, int64_t cols,
                                 int64_t ld) {
    const int64_t nq = ld / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * nq;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / nq, c = (i % nq) * 4;
        const float4 v = *reinterpret_cast<const float4*>(in + r * ld + c);
        float4 w;
        w.x = c + 0 < cols ? round_tf32(v.x) : 0.f;
        w.y = c + 1 < cols ? round_tf32(v.y) : 0.f;
        w.z = c + 2 < cols ? round_tf32(v.z) : 0.f;
        w.w = c + 3 < cols ? round_tf32(v.w) : 0.f;
        *reinterpret_cast<float4*>(out + r * ld + c) = w;
    }
}

// ---- F16 operands of J X (precision kF16S) ----------------------------------
// out[n][i] = fp16(a[n][i] w_n) for i < tk (0 up to ld16), w_n = 2^(7 - e) with
// max_i |a[n][i]| < 2^e, winv[n] = 1 / w_n; one CTA per example row
__global__ void a16_kernel(const float* __restrict__ a, int64_t lda, int64_t n, int64_t tk, int64_t ld16,
                           __half* __restrict__ out, float* __restrict__ winv) {
    __shared__ float red[32];
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        float m = 0.f;
        for (int64_t i = threadIdx.x; i < tk; i += blockDim.x) m = fmaxf(m, fabsf(a[r * lda + i]));
        m = block_absmax(m, red);
        const float w = pow2_scale(m, 7);
        if (threadIdx.x == 0) winv[r] = 1.f / w;
        for (int64_t i = threadIdx.x; i < ld16; i += blockDim.x)
            out[r * ld16 + i] = __float2half_rn(i < tk ? a[r * lda + i] * w : 0.f);
    }
}

// bits[c] = max over rows of |X[p][c]| (float bits; non-negative floats order as
// unsigned ints), c < l; thread c of a block walks a chunk of rows
__global__ void colmax_kernel(const float* __restrict__ X, int64_t ldx, int64_t R, int64_t l, int64_t rows_per_block,
                              unsigned* __restrict__ bits) {
    const int64_t c = blockIdx.y * (int64_t)blockDim.x + threadIdx.x;
    if (c >= l) return;
    const int64_t p0 = blockIdx.x * rows_per_block, p1 = min(R, p0 + rows_per_block);
    float m = 0.f;
    for (int64_t p = p0; p < p1; ++p) m = fmaxf(m, fabsf(X[p * ldx + c]));
    atomicMax(bits + c, __float_as_uint(m));
}

inline void colmax(cudaStream_t s, const float* X, int64_t ldx, int64_t R, int64_t l, unsigned* bits) {
    const int64_t rpb = 512, bx = std::min<int64_t>(round_up(l, 32), 256);
    colmax_kernel<<<dim3((unsigned)ceil_div(R, rpb), (unsigned)ceil_div(l, bx)), (unsigned)bx, 0, s>>>(X, ldx, R, l,
                                                                                                   rpb, bits);
    CK_LAUNCH();
}

// 2-D fp32 map without swizzle over rows x K (pitch ld), box (box_k, 1): one
// row segment (delta_k^T row o of the F16 J^T T stages)
inline CUtensorMap make_map_rowseg(const float* p, int64_t rows, int64_t K, int64_t ld, int box_k) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_k, 1}, es[2] = {1, 1};
    if ((reinterpret_cast<uintptr_t>(p) & 15) || (strides[0] & 15))
        throw CurvError(kCudaError, "TMA operand must be 16-byte aligned with a 16-byte row pitch");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CurvError(kCudaError, "cuTensorMapEncodeTiled (row) failed: " + std::to_string((int)r));
    return m;
}

// XT[c][p] = fp16(X[p][c0 + c] z_c) for c < lc, p < R (0 up to ld16), z_c =
// 2^(14 - e) with max_p |X[p][c]| < 2^e; zinv[c] = 1 / z_c.  32 x 32 tiles.
__global__ void xt16_kernel(const float* __restrict__ X, int64_t ldx, int64_t R, int64_t lc, int64_t c0,
                            const unsigned* __restrict__ bits, __half* __restrict__ XT, int64_t ld16,
                            float* __restrict__ zinv) {
    __shared__ float t[32][33];
    const int64_t p0 = (int64_t)blockIdx.x * 32, cb = (int64_t)blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t p = p0 + y, c = cb + threadIdx.x;
        t[y][threadIdx.x] = (p < R && c < lc) ? X[p * ldx + c0 + c] : 0.f;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t c = cb + y, p = p0 + threadIdx.x;
        if (c >= lc || p >= ld16) continue;
        const float z = pow2_scale(__uint_as_float(bits[c0 + c]), 14);
        if (blockIdx.x == 0 && threadIdx.x == 0) zinv[c] = 1.f / z;
        XT[c * ld16 + p] = __float2half_rn(t[threadIdx.x][y] * z);
    }
}

}  // namespace tc

// Rounded (to nearest TF32) copies of the activations and deltas of every
// layer, shared by all J X / J^T T products of one eigensolve.
struct KrOperands {
    DevMem mem;
    const float* a[kMaxLayers] = {};
    const float* d[kMaxLayers] = {};
    const float* dT[kMaxLayers] = {};  // delta_k^T (T_{k+1} x ldn, not rounded), zero padded
    int64_t ldn = 0;
    // F16 (kF16S): a_k in fp16 with per-example scales, for the J X products
    bool f16 = false;
    DevMem mem16;
    const __half* a16[kMaxLayers] = {};
    const float* winv[kMaxLayers] = {};
    int64_t lda16[kMaxLayers] = {};
    // ... and for J^T T: a_k^T in fp16 (T_k x ldn16) with per-input scales,
    // and max |delta_k[:, o]| per output unit
    const __half* aT16[kMaxLayers] = {};
    const float* uinv[kMaxLayers] = {};
    const float* dmax[kMaxLayers] = {};
    int64_t ldn16 = 0;

    KrOperands(const ModelDesc& md, const Cache<float>& c, cudaStream_t s, bool with_f16 = false) {
        ldn = round_up(c.n, 32);
        size_t total = 0;
        for (int k = 0; k < md.S; ++k) total += (size_t)c.n * (c.lda[k] + c.ldt[k]) + (size_t)md.w[k + 1] * ldn;
        mem = DevMem(total * sizeof(float), s);
        float* p = dptr<float>(mem);
        auto round = [&](const float* src, int64_t count) -> const float* {
            tc::round_tf32_kernel<<<(unsigned)std::min<int64_t>(ceil_div(count, 1024), 148 * 32), 256, 0, s>>>(src, p,
                                                                                                            count);
            CK_LAUNCH();
            const float* out = p;
            p += count;
            return out;
        };
        for (int k = 0; k < md.S; ++k) {
            a[k] = round(c.a[k], c.n * c.lda[k]);
            d[k] = round(c.delta[k], c.n * c.ldt[k]);
        }
        for (int k = 0; k < md.S; ++k) {
            transpose<float>(s, c.delta[k], c.ldt[k], 0, p, ldn, 0, c.n, md.w[k + 1], 1);
            dT[k] = p;
            p += (size_t)md.w[k + 1] * ldn;
        }
        if (!with_f16) return;
        f16 = true;
        size_t bytes = 0;
        ldn16 = round_up(c.n, 64);
        for (int k = 0; k < md.S; ++k) {
            lda16[k] = round_up(md.w[k], 64);
            bytes += (size_t)c.n * lda16[k] * 2 + (size_t)round_up(c.n, 4) * 4;
            bytes += (size_t)md.w[k] * ldn16 * 2 + (size_t)round_up(md.w[k], 4) * 4 + (size_t)round_up(md.w[k + 1], 4) * 4;
        }
        mem16 = DevMem(bytes, s);
        uint8_t* q = static_cast<uint8_t*>(mem16.p);
        for (int k = 0; k < md.S; ++k) {
            __half* h = reinterpret_cast<__half*>(q);
            q += (size_t)c.n * lda16[k] * 2;
            float* w = reinterpret_cast<float*>(q);
            q += (size_t)round_up(c.n, 4) * 4;
            tc::a16_kernel<<<(unsigned)std::min<int64_t>(c.n, 65535), 128, 0, s>>>(c.a[k], c.lda[k], c.n, md.w[k],
                                                                                 lda16[k], h, w);
            CK_LAUNCH();
            a16[k] = h;
            winv[k] = w;
        }
        for (int k = 0; k < md.S; ++k) {
            __half* h = reinterpret_cast<__half*>(q);
            q += (size_t)md.w[k] * ldn16 * 2;
            float* u = reinterpret_cast<float*>(q);
            q += (size_t)round_up(md.w[k], 4) * 4;
            float* dm = reinterpret_cast<float*>(q);
            q += (size_t)round_up(md.w[k + 1], 4) * 4;
            tc::am_f16_kernel<<<(unsigned)std::min<int64_t>(md.w[k], 8192), 256, 0, s>>>(c.a[k], c.lda[k], md.w[k], c.n,
                                                                                       ldn16, h, u);
            CK_LAUNCH();
            tc::row_absmax_kernel<<<(unsigned)std::min<int64_t>(md.w[k + 1], 8192), 256, 0, s>>>(dT[k], md.w[k + 1], c.n,
                                                                                               ldn, dm);
            CK_LAUNCH();
            aT16[k] = h;
            uinv[k] = u;
            dmax[k] = dm;
        }
    }
};

// Khatri-Rao products need 16-byte aligned pitches for TMA
inline bool kr_supported(const ModelDesc& md, const Cache<float>& c) {
    for (int k = 0; k < md.S; ++k)
        if (c.lda[k] % 4 || c.ldt[k] % 4) return false;
    return true;
}

template <bool JT, bool F16 = false>
void kr_launch(cudaStream_t s, const CUtensorMap& ma, const CUtensorMap& mb, const tc::pair::KrArgs& ka, int a3d,
               int b3d, const CUtensorMap* mdl = nullptr) {
    using C = tc::pair::KrCfg<JT, F16>;
    func_attr_once((const void*)tc::pair::kr_kernel<JT, F16>, [] {
        CK_CUDA(cudaFuncSetAttribute(tc::pair::kr_kernel<JT, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     C::BYTES));
    });
    const int64_t units = ka.mt * (JT ? ka.nop * ka.ksplit : ceil_div(ka.nop, ka.chunk));
    const int grid = 2 * (int)std::min<int64_t>(units, tc::num_sms() / 2);
    tc::pair::kr_kernel<JT, F16><<<grid, C::THREADS, C::BYTES, s>>>(ma, mb, mdl ? *mdl : mb, ka,
                                                                    (uint32_t)tc::BK * 128u, 512u, 1024u, a3d, b3d);
    CK_LAUNCH();
}

// Contiguous parameter rows [p0, p1) of one rank of the sharded top-k
// solver, cut at output-unit weight blocks (T_k rows each) and at 4-aligned
// bias blocks, balanced by parameter count (the J X and J^T T work of a row is
// proportional to it).  Per layer: the output units [oa, ob) whose weight
// rows the rank owns and its biases [ba, bb).
struct TopkShard {
    int64_t p0 = 0, p1 = 0;
    int64_t oa[kMaxLayers] = {}, ob[kMaxLayers] = {}, ba[kMaxLayers] = {}, bb[kMaxLayers] = {};
    int64_t rows() const { return p1 - p0; }

    // rows [p0, p1), which must start and end on unit boundaries
    static TopkShard range(const ModelDesc& md, int64_t p0, int64_t p1) {
        auto on_cut = [&](int64_t p) {
            if (p == 0 || p == md.P) return true;
            for (int k = 0; k < md.S; ++k) {
                if (p >= md.woff[k] && p < md.boff[k]) return (p - md.woff[k]) % md.w[k] == 0;
                if (p >= md.boff[k] && p <= md.boff[k] + md.w[k + 1]) return (p - md.boff[k]) % 4 == 0 || p == md.boff[k] + md.w[k + 1];
            }
            return false;
        };
        if (p0 < 0 || p1 > md.P || p0 > p1 || !on_cut(p0) || !on_cut(p1))
            throw CurvError(kContractError, "parameter range must start and end on an output-unit weight block or a "
                                            "4-aligned bias block");
        TopkShard t;
        t.p0 = p0;
        t.p1 = p1;
        for (int k = 0; k < md.S; ++k) {
            const int64_t tk = md.w[k], to = md.w[k + 1];
            auto units = [&](int64_t p) { return std::min(to, ceil_div(std::max<int64_t>(p - md.woff[k], 0), tk)); };
            auto biases = [&](int64_t p) { return std::min(to, std::max<int64_t>(p - md.boff[k], 0)); };
            t.oa[k] = units(p0);
            t.ob[k] = units(p1);
            t.ba[k] = biases(p0);
            t.bb[k] = biases(p1);
        }
        return t;
    }

    static TopkShard make(const ModelDesc& md, int64_t nshards, int64_t shard) {
        // unit boundaries in parameter order
        std::vector<int64_t> cut;
        for (int k = 0; k < md.S; ++k) {
            for (int64_t o = 0; o < md.w[k + 1]; ++o) cut.push_back(md.woff[k] + o * md.w[k]);
            for (int64_t b = 0; b < md.w[k + 1]; b += 4) cut.push_back(md.boff[k] + b);
        }
        cut.push_back(md.P);
        auto bound = [&](int64_t s) -> int64_t {
            if (s <= 0) return 0;
            if (s >= nshards) return md.P;
            const double target = (double)md.P * (double)s / (double)nshards;
            return *std::lower_bound(cut.begin(), cut.end(), (int64_t)std::ceil(target));
        };
        return range(md, bound(shard), bound(shard + 1));
    }
};

// T (n x l, ldt) = J[:, shard rows] X for X = the shard's rows (sh.rows() x l,
// ldx a multiple of 32).  Unsharded: TopkShard::make(md, 1, 0).
inline void kr_apply_j(const ModelDesc& md, const Cache<float>& c, const KrOperands& op, const TopkShard& sh,
                       const float* X, int64_t ldx, int64_t l, float* T, int64_t ldt, cudaStream_t s) {
    const int64_t n = c.n, R = sh.rows();
    const int64_t pairs = tc::num_sms() / 2;
    const int64_t mt = ceil_div(n, 256);
    // X rounded to nearest TF32 with zero padding columns
    DevMem xr((size_t)R * ldx * sizeof(float), s);
    tc::round_pad_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(R * ldx / 4, 256), 148 * 16)),
                           256, 0, s>>>(X, dptr<float>(xr), R, l, ldx);
    CK_LAUNCH();
    // work split: each layer's o pairs cut into chunks so ~8 units per SM pair
    int64_t chunk[kMaxLayers] = {}, nslab = 0, base[kMaxLayers] = {}, bslab[kMaxLayers] = {};
    for (int k = 0; k < md.S; ++k) {
        const int64_t nop = ceil_div(sh.ob[k] - sh.oa[k], 2);
        base[k] = nslab;
        if (nop > 0) {
            const int64_t want = std::max<int64_t>(1, ceil_div(8 * pairs, mt));
            chunk[k] = ceil_div(nop, std::min(nop, want));
            nslab += ceil_div(nop, chunk[k]);
        }
    }
    for (int k = 0; k < md.S; ++k) bslab[k] = sh.bb[k] > sh.ba[k] ? nslab++ : -1;
    const int64_t ldw = 128, slab = n * ldw;
    if (nslab == 0) {  // a shard without rows contributes zeros
        CK_CUDA(cudaMemset2DAsync(T, ldt * sizeof(float), 0, l * sizeof(float), n, s));
        return;
    }
    DevMem ws((size_t)(nslab * slab) * sizeof(float), s);
    // F16: X^T in fp16 with power-of-two column scales, per 128-column tile
    DevMem cbits, xt16, zinv;
    const int64_t ldR = round_up(R, 64);
    if (op.f16) {
        cbits = DevMem((size_t)l * 4, s);
        CK_CUDA(cudaMemsetAsync(cbits.p, 0, (size_t)l * 4, s));
        const int64_t rpb = 512;
        tc::colmax(s, X, ldx, R, l, dptr<unsigned>(cbits));
        xt16 = DevMem((size_t)128 * ldR * 2, s);
        zinv = DevMem((size_t)128 * 4, s);
    }
    for (int64_t c0 = 0; c0 < l; c0 += 128) {
        const int64_t lc = std::min<int64_t>(128, l - c0);
        const float* xc = dptr<float>(xr) + c0;
        const int b3 = ldx >= round_up(lc, 32) ? 1 : 0;
        if (op.f16) {
            CK_CUDA(cudaMemsetAsync(zinv.p, 0, (size_t)128 * 4, s));  // columns >= lc: scale 0
            tc::xt16_kernel<<<dim3((unsigned)ceil_div(ldR, 32), (unsigned)ceil_div(lc, 32)), dim3(32, 8), 0, s>>>(
                X, ldx, R, lc, c0, dptr<unsigned>(cbits), dptr<__half>(xt16), ldR, dptr<float>(zinv));
            CK_LAUNCH();
        }
        for (int k = 0; k < md.S; ++k) {
            const int64_t tk = md.w[k];
            if (sh.ob[k] > sh.oa[k]) {
                tc::pair::KrArgs ka{mt, ceil_div(sh.ob[k] - sh.oa[k], 2), chunk[k], ceil_div(tk, tc::BK), tk,
                                    md.w[k + 1], md.woff[k],
                                    c.delta[k], c.ldt[k], n, dptr<float>(ws) + base[k] * slab, ldw, slab, n, lc, 1,
                                    sh.oa[k], sh.ob[k], sh.p0};
                // the fp16 form reads X^T from parameter row woff + o T_k: TMA needs that
                // start 16-byte (8-half) aligned, else the TF32 form (a 4-input layer)
                const bool f16k = op.f16 && tk % 8 == 0 && (md.woff[k] - sh.p0) % 8 == 0;
                if (f16k) {
                    ka.nk = ceil_div(tk, 2 * tc::BK);
                    ka.rinv = op.winv[k];
                    ka.cinv = dptr<float>(zinv);
                    // K extent = the zero-padded row (a 4-input layer's 8-byte rows are below
                    // TMA's 16-byte minimum: the load faulted as an illegal instruction)
                    CUtensorMap ma = tc::make_map_f16(op.a16[k], n, op.lda16[k], op.lda16[k], 128);
                    CUtensorMap mb = tc::make_map_f16(dptr<__half>(xt16), lc, R, ldR, 128);
                    kr_launch<false, true>(s, ma, mb, ka, 0, 0);
                } else {
                    CUtensorMap ma = tc::make_map(op.a[k], n, tk, c.lda[k], 0, 128);
                    CUtensorMap mb = tc::make_map(xc, lc, R, ldx, 1, 128, b3);
                    kr_launch<false>(s, ma, mb, ka, 0, b3);
                }
            }
            if (bslab[k] >= 0)  // bias tangents: delta_k[:, ba..bb) Xb
                gemm_tf32(kTF32, s, n, lc, sh.bb[k] - sh.ba[k], pre_rounded(kmaj(op.d[k] + sh.ba[k], c.ldt[k])),
                          pre_rounded(mnmaj(xc + (md.boff[k] + sh.ba[k] - sh.p0) * ldx, ldx)),
                          EpiStore<float>{dptr<float>(ws) + bslab[k] * slab, ldw, 0, 1.f, 0.f});
        }
        tc::slab_sum_kernel<<<(unsigned)ceil_div(n * (ldw / 4), 256), 256, 0, s>>>(dptr<float>(ws), ldw, slab,
                                                                                  (int)nslab, n, lc, 1.f, T + c0, ldt);
        CK_LAUNCH();
    }
}

// Y (shard rows x l, ldy) = J[:, shard rows]^T T for T (n x l, ldtn; ldtn a
// multiple of 32)
inline void kr_apply_jt(const ModelDesc& md, const Cache<float>& c, const KrOperands& op, const TopkShard& sh,
                        const float* Tn, int64_t ldtn, int64_t l, float* Y, int64_t ldy, cudaStream_t s) {
    const int64_t n = c.n;
    const int64_t pairs = tc::num_sms() / 2;
    // F16: T^T per 128-column tile in fp32 (the kernel scales it by delta_o and
    // rounds to fp16 in shared memory) and max |T[:, c]| per column
    DevMem tbits, tt;
    if (op.f16) {
        tbits = DevMem((size_t)l * 4, s);
        CK_CUDA(cudaMemsetAsync(tbits.p, 0, (size_t)l * 4, s));
        tc::colmax(s, Tn, ldtn, n, l, dptr<unsigned>(tbits));
        tt = DevMem((size_t)128 * op.ldn * 4, s);
    }
    for (int64_t c0 = 0; c0 < l; c0 += 128) {
        const int64_t lc = std::min<int64_t>(128, l - c0);
        const float* tc0 = Tn + c0;
        const int b3 = ldtn >= round_up(lc, 32) ? 1 : 0;
        CUtensorMap mb = tc::make_map(tc0, lc, n, ldtn, 1, 128, b3);
        CUtensorMap mb16;
        if (op.f16) {
            transpose<float>(s, tc0, ldtn, 0, dptr<float>(tt), op.ldn, 0, n, lc, 1);
            mb16 = tc::make_map(dptr<float>(tt), lc, n, op.ldn, 0, 128);
        }
        for (int k = 0; k < md.S; ++k) {
            const int64_t tk = md.w[k], oa = sh.oa[k], ob = sh.ob[k];
            if (ob > oa) {
                const int a3 = c.lda[k] >= round_up(tk, 32) ? 1 : 0;
                const bool f16 = op.f16;
                CUtensorMap ma = f16 ? tc::make_map_f16(op.aT16[k], tk, n, op.ldn16, 128)
                                     : tc::make_map(op.a[k], tk, n, c.lda[k], 1, 128, a3);
                CUtensorMap mdl;
                if (f16) mdl = tc::make_map_rowseg(op.dT[k], md.w[k + 1], n, op.ldn, 64);
                auto launch = [&](tc::pair::KrArgs& ka) {
                    if (f16) {
                        ka.rinv = op.uinv[k];
                        ka.dmax = op.dmax[k];
                        ka.tmax = reinterpret_cast<const float*>(dptr<unsigned>(tbits)) + c0;
                        kr_launch<true, true>(s, ma, mb16, ka, 0, 0, &mdl);
                    } else {
                        kr_launch<true>(s, ma, mb, ka, a3, b3);
                    }
                };
                // (F16: units of four output units, two per CTA)
                const int64_t mt = ceil_div(tk, 256), nop = ceil_div(ob - oa, f16 ? 4 : 2),
                              nk = ceil_div(n, f16 ? 2 * tc::BK : tc::BK);
                // few (i-tile, o-pair) units (a narrow layer): split the examples
                // into slabs of partial products, summed in fixed order after
                int64_t ks = 1;
                if (mt * nop < 2 * pairs) ks = std::max<int64_t>(1, std::min(ceil_div(4 * pairs, mt * nop), nk / 8));
                if (ks > 1) ks = ceil_div(nk, ceil_div(nk, ks));  // every slab non-empty
                if (ks == 1) {
                    tc::pair::KrArgs ka{mt, nop, 1, nk, tk, md.w[k + 1], md.woff[k], op.dT[k], op.ldn, n, Y + c0, ldy,
                                        0, tk, lc, 1, oa, ob, sh.p0};
                    launch(ka);
                } else {
                    // slab rows (o - oa) T_k + i: woff 0 and prow0 = oa T_k
                    const int64_t rows = (ob - oa) * tk, slab = rows * 128;
                    DevMem ws((size_t)(ks * slab) * sizeof(float), s);
                    tc::pair::KrArgs ka{mt, nop, 1, nk, tk, md.w[k + 1], 0, op.dT[k], op.ldn, n, dptr<float>(ws),
                                        128, slab, tk, lc, ks, oa, ob, oa * tk};
                    launch(ka);
                    tc::slab_sum_kernel<<<(unsigned)ceil_div(rows * 32, 256), 256, 0, s>>>(
                        dptr<float>(ws), 128, slab, (int)ks, rows, lc, 1.f,
                        Y + (md.woff[k] + oa * tk - sh.p0) * ldy + c0, ldy);
                    CK_LAUNCH();
                }
            }
            if (sh.bb[k] > sh.ba[k])  // bias rows: delta_k[:, ba..bb)^T T (short M, long K: split over K)
                gemm_tf32_store(kTF32, s, sh.bb[k] - sh.ba[k], lc, n, pre_rounded(mnmaj(op.d[k] + sh.ba[k], c.ldt[k])),
                                mnmaj(tc0, ldtn), Y + (md.boff[k] + sh.ba[k] - sh.p0) * ldy + c0, ldy);
        }
    }
}

}  // namespace ck
