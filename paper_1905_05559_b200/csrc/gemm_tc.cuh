// gemm_tc.cuh -- tcgen05 TF32 GEMM for the curvature products (sm_100a).
//
// C(m, n) = sum_k A(m, k) B(n, k), A/B fp32 in HBM (K-major or MN-major),
// multiplied by kind::tf32 tensor-core MMAs with fp32 accumulation in TMEM.
//
//   warp 0      TMA producer: cp.async.bulk.tensor 2D tiles, SWIZZLE_128B,
//               4-stage smem ring (full/empty mbarriers)
//   warp 1      MMA issuer: one lane issues tcgen05.mma (M=128, N=BN, K=8)
//               and commits completion to the empty / tmem_full barriers
//   warp 2      TMEM allocator (2 x BN accumulator columns, double buffer)
//   warps 4-7   epilogue: tcgen05.ld 32x32 blocks -> smem transpose ->
//               coalesced stores through the epilogue functor (plain store,
//               symmetric mirror, Hessian block mapping)
// Persistent: one CTA per SM walks the tile list; tiles the functor marks
// as skippable (upper triangle of a symmetric product) cost nothing.
//
// k3xTF32 runs three MMAs per k-step on hi/lo TF32 splits of both operands
// (hi*hi + hi*lo + lo*hi); the lo parts are separate operands prepared by
// split_tf32_kernel.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "curvature.cuh"
#include "gemm_dmma.cuh"

namespace ck {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int STAGES = 4;
constexpr int kThreads = 256;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SWIZZLE_128B shared-memory matrix descriptor (sm_100 layout: version 1).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;       // version
    d |= (uint64_t)layout << 61;  // 2: SWIZZLE_128B, 1: SWIZZLE_128B_BASE32B
    return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, M=128, N=n.
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool a_mn, bool b_mn) {
    return (1u << 4)                       // D format f32
           | (2u << 7)                     // A tf32
           | (2u << 10)                    // B tf32
           | ((a_mn ? 1u : 0u) << 15)      // A major (0 K, 1 MN)
           | ((b_mn ? 1u : 0u) << 16)      // B major
           | ((uint32_t)(n >> 3) << 17)    // N / 8
           | ((uint32_t)(BM >> 4) << 24);  // M / 16
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// One lane of a converged warp.  The MMA issuers run as whole warps with
// warp-uniform descriptors and issue from the elected lane: a single-lane
// issuer makes ptxas wrap every tcgen05.mma in a uniform-register waterfall
// (ELECT / R2UR.BROADCAST / BRA.U.ANY), which measured ~200 clocks per MMA,
// well below the tensor pipe's rate (tools/mma_loop.cu).
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void mma_tf32_e(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (elect_one()) mma_tf32(d, a, b, idesc, acc);
    __syncwarp();
}
__device__ __forceinline__ void mma_commit_e(uint64_t* bar) {
    if (elect_one()) mma_commit(bar);
    __syncwarp();
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Epilogue block contract: after stage_block, buf[r][c] (16-byte aligned rows
// of 36 floats) holds acc(row0 + r, col0 + c) for the warp's 32 x 32 block and
// v[] still holds this lane's own row (row0 + lane) -- so stores along rows
// use buf (lanes across columns, 16-byte vectors) and transposed stores use v
// (lanes across rows, one register per column).
__device__ __forceinline__ void stage_block(float (*buf)[36], const float* v, int lane) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(&buf[lane][4 * q]) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    __syncwarp();
}

// ---------------------------------------------------------------- kernel
struct TcShape {
    int64_t M, N, K;
    int a_mn, b_mn;  // operand is MN-major
    int nsplit;      // 1: tf32, 3: 3xTF32 (hi*hi + hi*lo + lo*hi)
    uint32_t mn_lbo, mn_sbo, mn_kstep;  // MN-major descriptor strides (bytes)
    uint32_t mn_layout;                 // MN-major descriptor layout type
    int a_3d, b_3d;                     // MN-major operand loaded by one 3D TMA box
    int ksplit = 1;                     // pair kernel: K slabs per tile (Epi::block_split)
    int a_once = 0, b_once = 0;         // streamed operand: L2 evict_first
    int group_m = 16;                   // rasterisation group (m-tiles per column sweep)
    // pair kernel, precision kF16S: K-major fp16 operands (64 per 128-byte row,
    // kind::f16), scaled by exact powers of two; the epilogue multiplies entry
    // (r, c) by rsc[r] * csc[c] (the inverse scales) before storing
    int f16 = 0;
    const float* rsc = nullptr;
    const float* csc = nullptr;
    int dev = 0;  // dev (CURVKIT_DEV_PAIR): 1 no direct TMA boxes, 2 no mirror TMA boxes, 4 mirror blocks by the LSU
};

// Epilogues whose interior blocks are stored by TMA boxes (Epi::tma_block)
template <class E, class = void>
struct EpiTma : std::false_type {};
template <class E>
struct EpiTma<E, std::void_t<decltype(E::kTmaStore)>> : std::true_type {};

// Epilogues that take a K-slab index (split-K partial products)
template <class E, class = void>
struct EpiSplitK : std::false_type {};
template <class E>
struct EpiSplitK<E, std::void_t<decltype(E::kSplitK)>> : std::true_type {};

template <int BN>
struct TcSmem {
    static constexpr int A_BYTES = BM * BK * 4;  // 16 KB
    static constexpr int B_BYTES = BN * BK * 4;
    static constexpr int EPI_BYTES = 4 * 32 * 36 * 4;
    static constexpr int MAX_SMEM = 227 * 1024;
    __host__ __device__ static constexpr int stage_bytes(int nsplit) { return (A_BYTES + B_BYTES) * (nsplit == 1 ? 1 : 2); }
    __host__ __device__ static constexpr int stages(int nsplit) {
        const int st = (MAX_SMEM - 1024 - EPI_BYTES - 256) / stage_bytes(nsplit);
        return st > STAGES ? STAGES : st;
    }
    __host__ __device__ static constexpr int bytes(int nsplit) {
        return 1024 + stages(nsplit) * stage_bytes(nsplit) + EPI_BYTES + 256;
    }
};

// Load one operand tile (rows x BK) of a K-major or MN-major operand.
// MN-major tiles are [32-row atom][BK k-rows][32 elements]; a 3D map
// (elem-in-atom, k, atom) fetches all atoms of the tile in one box.
template <int ROWS>
__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int mn, int mn3d,
                                          int64_t r0, int64_t k0, int atoms) {
    if (!mn) {
        tma_load_2d(dst, map, bar, (int32_t)k0, (int32_t)r0);
    } else if (mn3d) {
        tma_load_3d(dst, map, bar, 0, (int32_t)k0, (int32_t)(r0 / 32));
    } else {
        for (int i = 0; i < atoms; ++i) tma_load_2d(dst + i * 4096, map, bar, (int32_t)(r0 + 32 * i), (int32_t)k0);
    }
}

template <int BN, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
               const __grid_constant__ CUtensorMap mapAlo, const __grid_constant__ CUtensorMap mapBlo, TcShape sh,
               Epi epi) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by offset from the __shared__ array, so the compiler
    // keeps the shared state space (LDS/STS, not generic LD/ST) for derived pointers
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int A_BYTES = TcSmem<BN>::A_BYTES, B_BYTES = TcSmem<BN>::B_BYTES;
    const int split = sh.nsplit == 1 ? 1 : 2;  // operand copies per stage (hi[, lo])
    const int STAGE_BYTES = (A_BYTES + B_BYTES) * split;
    const int NST = TcSmem<BN>::stages(sh.nsplit);
    uint8_t* stage_base = smem;
    float* epi_buf = reinterpret_cast<float*>(smem + NST * STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE_BYTES + TcSmem<BN>::EPI_BYTES);
    uint64_t* full = bars;                // [STAGES]
    uint64_t* empty = bars + STAGES;      // [STAGES]
    uint64_t* tfull = bars + 2 * STAGES;  // [2]
    uint64_t* tempty = tfull + 2;         // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t mt = ceil_div(sh.M, BM), nt = ceil_div(sh.N, BN);
    const int64_t ntiles = mt * nt;
    const int64_t nk = ceil_div(sh.K, BK);

    if (warp == 0 && lane == 0) {
        prefetch_map(&mapA);
        prefetch_map(&mapB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                     "n"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t m0 = (t / nt) * BM, n0 = (t % nt) * BN;
                if (epi.skip(0, m0, n0, BM, BN)) continue;
                // MN-major B of a ragged last tile: only the atoms that hold columns
                const int batoms = (sh.b_mn && !sh.b_3d) ? (int)::min((int64_t)(BN / 32), ceil_div(sh.N - n0, 32))
                                                         : BN / 32;
                const uint32_t bytes = (uint32_t)((A_BYTES + batoms * 4096 * (sh.b_mn && !sh.b_3d ? 1 : 0) +
                                                   (sh.b_mn && !sh.b_3d ? 0 : B_BYTES)) * split);
                for (int64_t kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], bytes);
                    uint8_t* sa = stage_base + stage * STAGE_BYTES;
                    uint8_t* sb = sa + A_BYTES * split;
                    const int64_t k0 = kb * BK;
                    load_tile<BM>(sa, &mapA, &full[stage], sh.a_mn, sh.a_3d, m0, k0, BM / 32);
                    load_tile<BN>(sb, &mapB, &full[stage], sh.b_mn, sh.b_3d, n0, k0, batoms);
                    if (split == 2) {
                        load_tile<BM>(sa + A_BYTES, &mapAlo, &full[stage], sh.a_mn, sh.a_3d, m0, k0, BM / 32);
                        load_tile<BN>(sb + B_BYTES, &mapBlo, &full[stage], sh.b_mn, sh.b_3d, n0, k0, batoms);
                    }
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        {  // ---------------- MMA issuer (whole warp; elected lane issues)
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t m0 = (t / nt) * BM, n0 = (t % nt) * BN;
                if (epi.skip(0, m0, n0, BM, BN)) continue;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                // ragged last N tile: the MMA only spans the live columns
                const int ntile = (int)::min((int64_t)BN, (sh.N - n0 + 15) / 16 * 16);
                const uint32_t idesc = idesc_tf32(ntile, sh.a_mn, sh.b_mn);
                const uint32_t d = tmem_base + (uint32_t)(acc * BN);
                for (int64_t kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(stage_base + stage * STAGE_BYTES);
                    const uint32_t sb = sa + A_BYTES * split;
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        // K-major: +32 B inside the 128 B swizzle row; MN-major: next 8-row group
                        const uint32_t aoff = sh.a_mn ? ks * sh.mn_kstep : ks * 32;
                        const uint32_t boff = sh.b_mn ? ks * sh.mn_kstep : ks * 32;
                        const uint32_t albo = sh.a_mn ? sh.mn_lbo : 16, blbo = sh.b_mn ? sh.mn_lbo : 16;
                        const uint32_t asbo = sh.a_mn ? sh.mn_sbo : 1024, bsbo = sh.b_mn ? sh.mn_sbo : 1024;
                        const uint32_t alay = sh.a_mn ? sh.mn_layout : 2, blay = sh.b_mn ? sh.mn_layout : 2;
                        const uint64_t ahi = smem_desc(sa + aoff, albo, asbo, alay);
                        const uint64_t bhi = smem_desc(sb + boff, blbo, bsbo, blay);
                        const uint32_t accf = (kb > 0 || ks > 0) ? 1u : 0u;
                        mma_tf32_e(d, ahi, bhi, idesc, accf);
                        if (split == 2) {
                            const uint64_t alo = smem_desc(sa + A_BYTES + aoff, albo, asbo, alay);
                            const uint64_t blo = smem_desc(sb + B_BYTES + boff, blbo, bsbo, blay);
                            mma_tf32_e(d, ahi, blo, idesc, 1u);
                            mma_tf32_e(d, alo, bhi, idesc, 1u);
                        }
                    }
                    mma_commit_e(&empty[stage]);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
                mma_commit_e(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue
        const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31
        float(*buf)[36] = reinterpret_cast<float(*)[36]>(epi_buf + ew * 32 * 36);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t m0 = (t / nt) * BM, n0 = (t % nt) * BN;
            if (epi.skip(0, m0, n0, BM, BN)) continue;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t row0 = m0 + ew * 32;
            for (int cb = 0; cb < BN / 32; ++cb) {
                const int64_t col0 = n0 + cb * 32;
                if (col0 >= sh.N) break;
                float v[32];
                tmem_ld32(tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * BN + cb * 32), v);
                if (row0 < sh.M) {
                    stage_block(buf, v, lane);
                    epi.block(row0, col0, sh.M, sh.N, buf, v, lane);
                    __syncwarp();
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(2 * BN));
    }
}

// ---------------------------------------------------------------- CTA pair
// cta_group::2: a cluster of two CTAs on one TPC computes a 256 x BN tile.
// Each CTA stages its own 128 rows of A and BN/2 rows of B; the leader
// (rank 0) issues M=256 MMAs that read both CTAs' shared memory, so every
// SM moves 2/3 of the operand bytes of the single-CTA 128 x BN tile for the
// same MMA work.  Completion is multicast to both CTAs' barriers.
namespace pair {

constexpr int EPI_WARPS = 8;
constexpr int kThreads2 = 128 + 32 * EPI_WARPS;  // warps 0-3 control, 4-11 epilogue

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t map_to_leader(uint32_t local_smem) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local_smem));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Remote arrive on a barrier in the pair (default .release.cta semantics, as
// CUTLASS's ClusterBarrier).  Waits stay CTA-scoped: a cluster-scope acquire
// in a polling loop makes ptxas emit an L1 invalidate (CCTL.IVALL) per poll.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_cluster(uint64_t* bar, uint32_t bytes) { mbar_expect_tx(bar, bytes); }

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }

// TMA into this CTA's smem, completion counted on the leader's barrier
// Operand tiles are re-read by neighbouring tiles: keep them in L2 against the
// P x P output stream (evict_last policy on every TMA load).
__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t evict_normal_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void tma2_2d(void* dst, const CUtensorMap* map, uint32_t bar_leader, int32_t c0,
                                        int32_t c1, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_leader), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
}
// one box written to the same offset in every CTA of `mask`, completing bytes
// on each destination CTA's barrier at the offset of `bar`
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                               int32_t c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tma2_3d(void* dst, const CUtensorMap* map, uint32_t bar_leader, int32_t c0,
                                        int32_t c1, int32_t c2, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_leader), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}

// Grouped rasterisation: consecutive tile indices walk GROUP_M m-tiles down a
// column before moving right, so the ~74 tiles in flight share a few A and B
// panels in L2.
constexpr int64_t GROUP_M = 16;
__device__ __forceinline__ void tile_coords(int64_t t, int64_t mt, int64_t nt, int64_t& mi, int64_t& ni,
                                            int64_t group = GROUP_M) {
    const int64_t per = group * nt;
    const int64_t g = t / per, local = t - g * per;
    const int64_t gm = ::min(group, mt - g * group);
    mi = g * group + local % gm;
    ni = local / gm;
}

template <int ROWS>
__device__ __forceinline__ void load_tile2(uint8_t* dst, const CUtensorMap* map, uint32_t bar, int mn, int mn3d,
                                           int64_t r0, int64_t k0, uint64_t pol) {
    if (!mn) {
        tma2_2d(dst, map, bar, (int32_t)k0, (int32_t)r0, pol);
    } else if (mn3d) {
        tma2_3d(dst, map, bar, 0, (int32_t)k0, (int32_t)(r0 / 32), pol);
    } else {
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i)
            tma2_2d(dst + i * 4096, map, bar, (int32_t)(r0 + 32 * i), (int32_t)k0, pol);
    }
}

__device__ __forceinline__ void mma2_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    const uint32_t z = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(z)
        : "memory");
}

// kind::f16: fp16 A and B (K = 16 per instruction, the same 32 bytes of a
// 128-byte swizzle row as one K = 8 tf32 step), fp32 accumulate
__device__ __forceinline__ void mma2_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    const uint32_t z = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(z)
        : "memory");
}

// A from TMEM (the "TS" form): a_tmem is this CTA's A tile column in TMEM
__device__ __forceinline__ void mma2_tf32_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
    const uint32_t z = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(tmem_d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc), "r"(z)
        : "memory");
}

// 32 lanes x 32 columns of 32-bit values from registers into TMEM
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]),
        "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]),
        "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void commit2(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}

// issue from the elected lane of a converged warp (see elect_one)
__device__ __forceinline__ void mma2_tf32_e(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (elect_one()) mma2_tf32(d, a, b, idesc, acc);
    __syncwarp();
}
__device__ __forceinline__ void mma2_tf32_ts_e(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (elect_one()) mma2_tf32_ts(d, a, b, idesc, acc);
    __syncwarp();
}
__device__ __forceinline__ void commit2_e(uint64_t* bar) {
    if (elect_one()) commit2(bar);
    __syncwarp();
}

// kind::f16 instruction descriptor, M = 256 (pair): D f32, A/B f16 (format 0)
__host__ __device__ constexpr uint32_t idesc2_f16(int n, bool a_mn, bool b_mn) {
    return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(256 >> 4) << 24);
}

__host__ __device__ constexpr uint32_t idesc2_tf32(int n, bool a_mn, bool b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
           ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA store of one smem box; bulk-group bookkeeping
// output boxes stream through L2 with evict_first (the operands keep their lines:
// config 3's symmetric kernel re-read half as much of its B operand from HBM)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(evict_first_policy())
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// all but the newest store group have read their shared-memory source
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int BN>
struct PairSmem {
    static constexpr int A_BYTES = 128 * BK * 4;       // own 128 rows
    static constexpr int B_BYTES = (BN / 2) * BK * 4;  // own half of B
    // per epilogue warp a 1024-aligned 8 KB slot: the 32 x 36 staging block, or two
    // swizzled 32 x 32 TMA store boxes (a block and its mirror: one store is in
    // flight while the other box is filled)
    static constexpr int EPI_SLOT = 8 * 1024;
    static constexpr int EPI_BYTES = EPI_WARPS * EPI_SLOT;
    static constexpr int MAX_SMEM = 227 * 1024;
    __host__ __device__ static constexpr int stage_bytes(int nsplit) { return (A_BYTES + B_BYTES) * (nsplit == 1 ? 1 : 2); }
    __host__ __device__ static constexpr int stages(int nsplit) {
        const int st = (MAX_SMEM - 1024 - EPI_BYTES - 512) / stage_bytes(nsplit);
        return st > 8 ? 8 : st;
    }
    __host__ __device__ static constexpr int bytes(int nsplit) {
        return 1024 + stages(nsplit) * stage_bytes(nsplit) + EPI_BYTES + 512;
    }
};

template <int BN, class Epi, bool F16 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
tc_gemm_pair_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ CUtensorMap mapAlo, const __grid_constant__ CUtensorMap mapBlo,
                    const __grid_constant__ CUtensorMap mapC, TcShape sh, Epi epi) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by offset from the __shared__ array, so the compiler
    // keeps the shared state space (LDS/STS, not generic LD/ST) for derived pointers
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    using S = PairSmem<BN>;
    const int split = sh.nsplit == 1 ? 1 : 2;
    const int STAGE_BYTES = S::stage_bytes(sh.nsplit);
    const int NST = S::stages(sh.nsplit);
    uint8_t* stage_base = smem;
    float* epi_buf = reinterpret_cast<float*>(smem + NST * STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE_BYTES + S::EPI_BYTES);
    uint64_t* full = bars;            // [8]  (leader's copy is the live one)
    uint64_t* empty = bars + 8;       // [8]  (both CTAs, multicast commit)
    uint64_t* tfull = bars + 16;      // [2]  (both CTAs, multicast commit)
    uint64_t* tempty = bars + 18;     // [2]  (leader's copy; remote arrivals)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 20);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cta_rank();
    const int64_t pair_id = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int64_t mt = ceil_div(sh.M, 256), nt = ceil_div(sh.N, BN);
    const int64_t ntiles = mt * nt;
    const int KBE = F16 ? 2 * BK : BK;  // K elements per 128-byte operand row
    const int64_t nk = ceil_div(sh.K, KBE);
    // work unit t = (K slab t / ntiles, tile t % ntiles): concurrent units
    // share a K slab, so the B rows they stream stay in L2
    const int64_t ksl = sh.ksplit > 1 ? sh.ksplit : 1;
    const int64_t nunits = ntiles * ksl;
    const int64_t kcb = ceil_div(nk, ksl);
    auto unit_of = [&](int64_t t, int64_t& mi, int64_t& ni, int64_t& kb0, int64_t& kb1) {
        tile_coords(t % ntiles, mt, nt, mi, ni, sh.group_m);
        kb0 = (t / ntiles) * kcb;
        kb1 = ::min(nk, kb0 + kcb);
    };

    if (warp == 0 && lane == 0) {
        prefetch_map(&mapA);
        prefetch_map(&mapB);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 2);  // leader arrive.expect_tx + peer arrive
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                     "n"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    auto tile_ntile = [&](int64_t n0) -> int {
        // live columns of this tile, in steps of 64 so each CTA's half is a
        // whole number of 32-row MN atoms
        return (int)::min((int64_t)BN, (sh.N - n0 + 63) / 64 * 64);
    };

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t bytes_leader = (uint32_t)(2 * STAGE_BYTES);
            const uint64_t keep = evict_last_policy(), stream = evict_first_policy();
            const uint64_t pa = sh.a_once ? stream : keep, pb = sh.b_once ? stream : keep;
            for (int64_t t = pair_id; t < nunits; t += npairs) {
                int64_t mi, ni, kb0, kb1;
                unit_of(t, mi, ni, kb0, kb1);
                const int64_t m0 = mi * 256, n0 = ni * BN;
                if (epi.skip(0, m0, n0, 256, BN)) continue;
                const int64_t half = tile_ntile(n0) / 2;
                const int64_t am0 = m0 + 128 * rank, bn0 = n0 + half * rank;
                for (int64_t kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t fb = map_to_leader(smem_u32(&full[stage]));
                    if (rank == 0) mbar_expect_tx_cluster(&full[stage], bytes_leader);
                    else mbar_arrive_cluster(fb);
                    uint8_t* sa = stage_base + stage * STAGE_BYTES;
                    uint8_t* sb = sa + S::A_BYTES * split;
                    const int64_t k0 = kb * KBE;
                    load_tile2<128>(sa, &mapA, fb, sh.a_mn, sh.a_3d, am0, k0, pa);
                    load_tile2<BN / 2>(sb, &mapB, fb, sh.b_mn, sh.b_3d, bn0, k0, pb);
                    if (split == 2) {
                        load_tile2<128>(sa + S::A_BYTES, &mapAlo, fb, sh.a_mn, sh.a_3d, am0, k0, pa);
                        load_tile2<BN / 2>(sb + S::B_BYTES, &mapBlo, fb, sh.b_mn, sh.b_3d, bn0, k0, pb);
                    }
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ---------------- MMA issuer (leader CTA, whole warp; elected lane issues)
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = pair_id; t < nunits; t += npairs) {
                int64_t mi, ni, kb0, kb1;
                unit_of(t, mi, ni, kb0, kb1);
                const int64_t m0 = mi * 256, n0 = ni * BN;
                if (epi.skip(0, m0, n0, 256, BN)) continue;
                mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t idesc = F16 ? idesc2_f16(tile_ntile(n0), false, false)
                                           : idesc2_tf32(tile_ntile(n0), sh.a_mn, sh.b_mn);
                const uint32_t d = tmem_base + (uint32_t)(acc * BN);
                for (int64_t kb = kb0; kb < kb1; ++kb) {
                    mbar_wait_cluster(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(stage_base + stage * STAGE_BYTES);
                    const uint32_t sb = sa + S::A_BYTES * split;
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        const uint32_t aoff = sh.a_mn ? ks * sh.mn_kstep : ks * 32;
                        const uint32_t boff = sh.b_mn ? ks * sh.mn_kstep : ks * 32;
                        const uint32_t albo = sh.a_mn ? sh.mn_lbo : 16, blbo = sh.b_mn ? sh.mn_lbo : 16;
                        const uint32_t asbo = sh.a_mn ? sh.mn_sbo : 1024, bsbo = sh.b_mn ? sh.mn_sbo : 1024;
                        const uint32_t alay = sh.a_mn ? sh.mn_layout : 2, blay = sh.b_mn ? sh.mn_layout : 2;
                        const uint64_t ahi = smem_desc(sa + aoff, albo, asbo, alay);
                        const uint64_t bhi = smem_desc(sb + boff, blbo, bsbo, blay);
                        if constexpr (F16) {  // K-major fp16: K = 16 per MMA, the same 32 bytes per step
                            if (elect_one()) mma2_f16(d, ahi, bhi, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
                            __syncwarp();
                            continue;
                        }
                        mma2_tf32_e(d, ahi, bhi, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
                        if (split == 2) {
                            mma2_tf32_e(d, ahi, smem_desc(sb + S::B_BYTES + boff, blbo, bsbo, blay), idesc, 1u);
                            mma2_tf32_e(d, smem_desc(sa + S::A_BYTES + aoff, albo, asbo, alay), bhi, idesc, 1u);
                        }
                    }
                    commit2_e(&empty[stage]);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
                commit2_e(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue (both CTAs, 8 warps)
        const int ew = warp - 4;
        const int quad = warp % 4;   // TMEM lanes 32*quad .. +31
        const int chalf = ew / 4;    // column half of the tile
        uint8_t* slot = reinterpret_cast<uint8_t*>(epi_buf) + ew * S::EPI_SLOT;
        float(*buf)[36] = reinterpret_cast<float(*)[36]>(slot);
        float* box = reinterpret_cast<float*>(slot);          // 32 rows x 128 B, 128-byte swizzle
        float* box2 = reinterpret_cast<float*>(slot + 4096);  // the mirrored block's box
        const uint32_t te_leader = map_to_leader(smem_u32(&tempty[0]));
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = pair_id; t < nunits; t += npairs) {
            int64_t mi, ni, kb0, kb1;
            unit_of(t, mi, ni, kb0, kb1);
            const int64_t m0 = mi * 256, n0 = ni * BN;
            if (epi.skip(0, m0, n0, 256, BN)) continue;
            mbar_wait_cluster(&tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t row0 = m0 + 128 * rank + quad * 32;
            for (int cb = chalf * (BN / 64); cb < (chalf + 1) * (BN / 64); ++cb) {
                const int64_t col0 = n0 + cb * 32;
                if (col0 >= sh.N) break;
                float v[32];
                tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN + cb * 32), v);
                if constexpr (F16) {  // undo the operands' power-of-two scales (exact)
                    const float rs = row0 + lane < sh.M ? sh.rsc[row0 + lane] : 0.f;
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] *= rs * (col0 + c < sh.N ? __ldg(&sh.csc[col0 + c]) : 0.f);
                }
                if (row0 < sh.M) {
                    if constexpr (EpiTma<Epi>::value) {
                        int64_t gr0, gc0;
                        if (epi.tma_block(row0, col0, sh.M, sh.N, gr0, gc0)) {
                            // store groups complete in order: with at most one pending, the
                            // store before the last one -- this box's previous use -- has read it
                            if (lane == 0) bulk_wait_read1();
                            __syncwarp();
#pragma unroll
                            for (int c = 0; c < 32; ++c) v[c] *= epi.alpha;
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                *reinterpret_cast<float4*>(box + lane * 32 + ((q ^ (lane & 7)) << 2)) =
                                    make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                            fence_proxy_async();
                            __syncwarp();
                            if (lane == 0) {
                                if (!(sh.dev & 1)) tma_store_2d(&mapC, box, (int32_t)gc0, (int32_t)gr0);
                                bulk_commit();
                                bulk_wait_read1();  // the previous mirror box has been read
                            }
                            __syncwarp();
                            if (sh.dev & 4) {
                                // mirrored block from registers: row gc0 + c of C gets this block's
                                // column c, the 32 lanes writing 128 contiguous bytes (LSU, no box)
                                float* mcol = epi.c + gc0 * epi.ldc + gr0 + lane;
#pragma unroll
                                for (int c = 0; c < 32; ++c) __stcs(mcol + c * epi.ldc, v[c]);
                                continue;
                            }
#pragma unroll
                            for (int c = 0; c < 32; ++c)
                                box2[c * 32 + ((((lane >> 2) ^ (c & 7)) << 2) | (lane & 3))] = v[c];
                            fence_proxy_async();
                            __syncwarp();
                            if (lane == 0) {
                                if (!(sh.dev & 2)) tma_store_2d(&mapC, box2, (int32_t)gr0, (int32_t)gc0);
                                bulk_commit();
                            }
                            continue;
                        }
                        // the staging block below overlaps both boxes: every store has read them
                        if (lane == 0) bulk_wait_read();
                        __syncwarp();
                    }
                    stage_block(buf, v, lane);
                    if constexpr (EpiSplitK<Epi>::value)
                        epi.block_split((int)(t / ntiles), row0, col0, sh.M, sh.N, buf, v, lane);
                    else
                        epi.block(row0, col0, sh.M, sh.N, buf, v, lane);
                    __syncwarp();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(te_leader + acc * 8);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if constexpr (EpiTma<Epi>::value)
            if (lane == 0) bulk_wait_all();  // epilogue stores complete before exit
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(2 * BN));
    }
}

// ---------------------------------------------------------------- fused Hessian block
// Weight-tangent rows of one Hessian block (k, m) without materialising R:
//   A[(o'', j), n] = a_k[n, i] * PV[o][o''][n]  (+ delta_k[n, o] * Q[o''][i][n]   if m < k)
// with j = o * T_k + i.  Per K-block the producer TMA-loads the activation
// tile a_k^T[i0 .. i0+127][n0 .. n0+31] (and the Q tile), four transform
// warps scale it in place (one thread per row, swizzle-aware 16-byte smem
// accesses), fence it into the async proxy and arrive on the leader's full
// barrier; the MMA then runs exactly as in tc_gemm_pair_kernel.  Rows are
// enumerated per o'' band (j >= jstart(o'')), so only tiles holding lower-
// triangle entries are visited.
struct FusedHess {
    const float* pv;   // [T_{k+1}][T_{m+1}][ldn]  (G or P_m, n-contiguous)
    const float* dT;   // delta_k^T [T_{k+1}][ldn]   (m < k only)
    int64_t ldn, tk, tm, tm1, nw;  // T_k, T_m, T_{m+1}, weight tangents T_{k+1} T_k
    int64_t qrows;     // rows per o'' slab of the extended Q^T (m < k)
    int diag, hasq;
    const int4* tiles;  // (o'', j0, n0, -) of every pair tile holding required entries
    int64_t ntiles;
    int64_t rows;       // tangent rows of the block: nw weights, then T_{k+1} biases (s = 1)
    int pv_tma;         // profile / delta rows of a CTA's weight rows staged by TMA (else __ldg)
    long long* trace = nullptr;  // dev: pipeline event stamps (8 x 1024) of CTA 0
    int tma_h = 0;               // interior 32 x 32 blocks stored by TMA (mapH)
    int dev = 0;                 // dev experiments (CURVKIT_DEV_FUSED): 1 no transform math, 2 no epilogue stores,
                                 // 4 mirror boxes by TMA (else coalesced register stores)
    // first output unit o whose profile row the producer stages for a CTA
    // whose first tangent row is jr (rows jr .. jr + 127 use units o_first ..)
    __host__ __device__ int64_t o_first(int64_t jr) const {
        const int64_t to = rows - nw;
        const int64_t o = jr < nw ? jr / tk : 0;
        return o < to ? o : to - 1;
    }
    // first tangent row of band o'' (aligned to the 256-row pair tile)
    __host__ __device__ int64_t jstart(int64_t opp) const {
        if (!diag) return 0;
        const int64_t s = (opp * tm) / 256 * 256;
        return s < rows ? s : rows;
    }
};

// control (4 warps), epilogue (8: two per TMEM lane quadrant, each half the
// tile width), transform (FUSED_TW: TW_SETS sets of 4 warps, one tile row per
// thread; set s transforms the k-blocks with global index = s mod TW_SETS,
// so a stage has TW_SETS MMA periods for its transform)
constexpr int FUSED_EPI = 8, FUSED_TW = 4;
constexpr int TW_SETS = FUSED_TW / 4;
constexpr int TW_CH = 8 / TW_SETS;  // 16-byte chunks per pass (TW_SETS passes bound the registers)
constexpr int PV_ROWS = 8;  // profile rows (output units o) staged per CTA and stage
constexpr bool STAGE_PV = true;  // profile rows ride the stage (TMA), no L2 round trip in the transform
constexpr int kFusedThreads = 128 + 32 * FUSED_EPI + 32 * FUSED_TW;

template <int BN>
struct FusedSmem {
    static constexpr int A_BYTES = 128 * BK * 4;
    static constexpr int B_BYTES = (BN / 2) * BK * 4;
    // per epilogue warp: a 1024-aligned 4 KB slot holding one swizzled 32 x 32
    // block (the TMA store box, or the staging block of the scalar path)
    static constexpr int EPI_SLOT = 4 * 1024;
    static constexpr int EPI_BYTES = FUSED_EPI * EPI_SLOT;
    static constexpr int MAX_SMEM = 227 * 1024;
    static constexpr int PV_BYTES = STAGE_PV ? PV_ROWS * BK * 4 : 0;  // one 128-byte row of examples per unit
    // stage: A | Q (m < k) | B | PV rows | delta^T rows (m < k)
    __host__ __device__ static constexpr int stage_bytes(int hasq) {
        return (A_BYTES + PV_BYTES) * (hasq ? 2 : 1) + B_BYTES;
    }
    __host__ __device__ static constexpr int stages(int hasq) {
        const int st = (MAX_SMEM - 1024 - EPI_BYTES - 1024) / stage_bytes(hasq);
        return st > 8 ? 8 : st;
    }
    __host__ __device__ static constexpr int bytes(int hasq) {
        return 1024 + stages(hasq) * stage_bytes(hasq) + EPI_BYTES + 1024;
    }
};

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}


// TS = true: the transform writes R into TMEM A slots (tcgen05.st) and the MMA
// reads A from TMEM, so R never passes through shared memory; 512 TMEM
// columns = 2 accumulators of BN (192) + TS_SLOTS A slots of one K-block.
constexpr int TS_SLOTS = 4;

template <int BN, class Epi, bool TS = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFusedThreads, 1)
tc_hess_fused_kernel(const __grid_constant__ CUtensorMap mapAk, const __grid_constant__ CUtensorMap mapQ,
                     const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapPV,
                     const __grid_constant__ CUtensorMap mapDT, const __grid_constant__ CUtensorMap mapH, FusedHess fh,
                     TcShape sh, Epi epi) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by offset from the __shared__ array, so the compiler
    // keeps the shared state space (LDS/STS, not generic LD/ST) for derived pointers
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    using S = FusedSmem<BN>;
    const int STAGE_BYTES = S::stage_bytes(fh.hasq);
    const int NST = S::stages(fh.hasq);
    const int A_OFF_Q = S::A_BYTES, B_OFF = S::A_BYTES * (fh.hasq ? 2 : 1);
    const int PV_OFF = B_OFF + S::B_BYTES, DT_OFF = PV_OFF + S::PV_BYTES;
    uint8_t* stage_base = smem;
    float* epi_buf = reinterpret_cast<float*>(smem + NST * STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE_BYTES + S::EPI_BYTES);
    uint64_t* full = bars;         // [8] leader: 1 producer + transform-warp arrivals, B tx
    uint64_t* empty = bars + 8;    // [8] both CTAs (multicast commit)
    uint64_t* afull = bars + 16;   // [8] local: A (Q, profile rows) landed
    uint64_t* tfull = bars + 24;   // [2]
    uint64_t* tempty = bars + 26;  // [2] leader
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 28);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cta_rank();
    // dev trace (fh.trace set): clock64 stamps of pipeline events in CTA 0
    constexpr int64_t TRN = 1024;
    long long* trace = (fh.trace && blockIdx.x == 0) ? fh.trace : nullptr;
    const int64_t pair_id = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int64_t ntiles = fh.ntiles;
    const int64_t nk = ceil_div(sh.K, BK);
    constexpr int TW0 = 4 + FUSED_EPI;  // first transform warp

    // tile t -> (o'', first tangent row j0, n0) from the host-built list of
    // tiles that hold required entries; rows of the pair tile are j0 .. j0+255
    // and the virtual GEMM row is o'' * nw + j
    auto tile_of = [&](int64_t t, int64_t& opp, int64_t& j0, int64_t& n0) {
        const int4 tl = __ldg(&fh.tiles[t]);
        opp = tl.x;
        j0 = tl.y;
        n0 = tl.z;
    };

    if (warp == 0 && lane == 0) {
        prefetch_map(&mapAk);
        prefetch_map(&mapB);
        if (fh.hasq) prefetch_map(&mapQ);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1 + 2 * 4);  // producer + one transform set (4 warps) of each CTA
            mbar_init(&empty[s], 1);
            mbar_init(&afull[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * FUSED_EPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    constexpr int TMEM_COLS = (TS || 2 * BN > 256) ? 512 : 256;
    static_assert(!TS || 2 * BN + 32 * TS_SLOTS <= 512, "TMEM budget");
    constexpr uint32_t A_COL0 = 2 * BN;  // first TMEM A slot (TS)
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    auto tile_ntile = [&](int64_t n0) -> int { return (int)::min((int64_t)BN, (sh.N - n0 + 63) / 64 * 64); };

    if (warp == 0) {
        if (lane == 0) {  // ---------------- producer
            int stage = 0;
            uint32_t phase = 0;
            int64_t tg = 0;
            const uint64_t pol = evict_last_policy();
            for (int64_t t = pair_id; t < ntiles; t += npairs) {
                int64_t opp, j0, n0;
                tile_of(t, opp, j0, n0);
                const int64_t jr = j0 + 128 * rank;           // this CTA's first tangent row
                const int64_t i0 = jr % fh.tk;                // row in the extended a_k^T
                const int64_t half = tile_ntile(n0) / 2;
                const int64_t bn0 = n0 + half * rank;
                for (int64_t kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (trace) { if (tg < TRN) trace[0 * TRN + tg] = clock64(); ++tg; }
                    uint8_t* sa = stage_base + stage * STAGE_BYTES;
                    const int64_t k0 = kb * BK;
                    mbar_expect_tx(&afull[stage], (uint32_t)((S::A_BYTES + (fh.pv_tma ? S::PV_BYTES : 0)) *
                                                             (fh.hasq ? 2 : 1)));
                    tma_load_2d(sa, &mapAk, &afull[stage], (int32_t)k0, (int32_t)i0);
                    if (fh.hasq) tma_load_2d(sa + A_OFF_Q, &mapQ, &afull[stage], (int32_t)k0, (int32_t)(opp * fh.qrows + i0));
                    if (fh.pv_tma) {  // profile rows (o_first .. + 7, o''), examples k0 .. k0 + 31
                        const int32_t of = (int32_t)fh.o_first(jr);
                        tma_load_3d(sa + PV_OFF, &mapPV, &afull[stage], (int32_t)k0, (int32_t)opp, of);
                        if (fh.hasq) tma_load_3d(sa + DT_OFF, &mapDT, &afull[stage], (int32_t)k0, 0, of);
                    }
                    const uint32_t fb = map_to_leader(smem_u32(&full[stage]));
                    if (rank == 0) mbar_expect_tx(&full[stage], (uint32_t)(2 * S::B_BYTES));
                    load_tile2<BN / 2>(sa + B_OFF, &mapB, fb, sh.b_mn, sh.b_3d, bn0, k0, pol);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ---------------- MMA issuer (leader CTA, whole warp; elected lane issues)
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int64_t tg = 0, tt = 0;
            for (int64_t t = pair_id; t < ntiles; t += npairs) {
                int64_t opp, j0, n0;
                tile_of(t, opp, j0, n0);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                ++tt;
                tc_fence_after();
                const uint32_t idesc = idesc2_tf32(tile_ntile(n0), false, sh.b_mn);
                const uint32_t d = tmem_base + (uint32_t)(acc * BN);
                for (int64_t kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    if (trace) { if (tg < TRN) trace[3 * TRN + tg] = clock64(); }
                    tc_fence_after();
                    const uint32_t sa = smem_u32(stage_base + stage * STAGE_BYTES);
                    const uint32_t sb = sa + B_OFF;
                    const uint32_t aslot = tmem_base + A_COL0 + (uint32_t)(tg % TS_SLOTS) * 32;
                    ++tg;
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ++ks) {
                        const uint32_t boff = sh.b_mn ? ks * sh.mn_kstep : ks * 32;
                        const uint32_t blbo = sh.b_mn ? sh.mn_lbo : 16, bsbo = sh.b_mn ? sh.mn_sbo : 1024;
                        const uint32_t blay = sh.b_mn ? sh.mn_layout : 2;
                        const uint64_t bd = smem_desc(sb + boff, blbo, bsbo, blay);
                        if constexpr (TS)
                            mma2_tf32_ts_e(d, aslot + ks * 8, bd, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
                        else
                            mma2_tf32_e(d, smem_desc(sa + ks * 32, 16, 1024, 2), bd, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
                    }
                    commit2_e(&empty[stage]);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
                commit2_e(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp >= TW0) {  // ---------------- A transform (both CTAs)
        const int set = (warp - TW0) >> 2;
        const int row = ((warp - TW0) & 3) * 32 + lane;  // tile row of this thread
        const uint32_t fb0 = map_to_leader(smem_u32(&full[0]));
        // running stage / phase of the k-block stream (all tiles), and its
        // position mod TW_SETS: no divisions in the loop
        int stage = 0, sidx = 0;
        uint32_t phase = 0;
        int g = 0;  // k-block index (trace; TS: A slot g % TS_SLOTS)
        // TS: the MMA of k-block g - TS_SLOTS (stage rs, phase rph) must be done
        // with A slot g % TS_SLOTS before it is overwritten
        int rs = 0;
        uint32_t rph = 0;
        const uint32_t tq = (uint32_t)(((warp - TW0) & 3) * 32) << 16;  // TMEM lane quadrant of this warp
        for (int64_t t = pair_id; t < ntiles; t += npairs) {
            int64_t opp, j0, n0;
            tile_of(t, opp, j0, n0);
            const int64_t j = ::min(j0 + 128 * rank + row, fh.rows - 1);  // rows past the band are masked later
            const bool bias = j >= fh.nw;  // bias tangent: s_n = 1, no delta*Q term
            const int64_t o = bias ? j - fh.nw : j / fh.tk;
            const float* pvrow = fh.pv + (o * fh.tm1 + opp) * fh.ldn;
            const float* drow = fh.hasq ? fh.dT + o * fh.ldn : nullptr;
            const int sw = row & 7;
            const bool trw = trace && threadIdx.x == TW0 * 32;
            // weight rows read their profile (and delta) row from the stage
            const int64_t slot = o - fh.o_first(j0 + 128 * rank);
            const bool staged = fh.pv_tma && !bias && slot >= 0 && slot < PV_ROWS;
            for (int64_t kb = 0; kb < nk; ++kb, ++g) {
                const bool mine = TW_SETS == 1 || sidx == set;
                const int st_ = stage;
                const uint32_t ph_ = phase;
                if (++stage == NST) { stage = 0; phase ^= 1; }
                if (TW_SETS > 1 && ++sidx == TW_SETS) sidx = 0;
                // every set waits on every stage in order: a set that skipped stages
                // could see a completed phase of the same parity one lap early
                mbar_wait(&afull[st_], ph_);
                if (!mine) continue;
                if constexpr (TS) {
                    if (g >= TS_SLOTS) {
                        mbar_wait(&empty[rs], rph);
                        if (++rs == NST) { rs = 0; rph ^= 1; }
                    }
                }
                if (trw && g < TRN) trace[1 * TRN + g] = clock64();
                if (fh.dev & 1) {  // dev: pipeline without the transform's shared-memory work
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(fb0 + st_ * 8);
                    continue;
                }
                uint8_t* st = stage_base + st_ * STAGE_BYTES;
                uint8_t* sa = st + row * 128;
                const int64_t n0k = kb * BK;
                const float4* pst = reinterpret_cast<const float4*>(st + PV_OFF + slot * 128);
                const float4* dst_ = reinterpret_cast<const float4*>(st + DT_OFF + slot * 128);
                // per pass: loads first, then the products, then the stores;
                // logical 16-byte chunk L holds examples n0k + 4L .. +3 and sits
                // at physical chunk L ^ (row & 7)
#pragma unroll
                for (int pass = 0; pass < TW_SETS; ++pass) {
                    const int L0 = pass * TW_CH;
                    float4 x[TW_CH], p[TW_CH];
#pragma unroll
                    for (int u = 0; u < TW_CH; ++u)
                        x[u] = *reinterpret_cast<const float4*>(sa + (((L0 + u) ^ sw) << 4));
                    if (staged) {
#pragma unroll
                        for (int u = 0; u < TW_CH; ++u) p[u] = pst[L0 + u];
                    } else {
#pragma unroll
                        for (int u = 0; u < TW_CH; ++u)
                            p[u] = __ldg(reinterpret_cast<const float4*>(pvrow + n0k + 4 * (L0 + u)));
                    }
#pragma unroll
                    for (int u = 0; u < TW_CH; ++u) {
                        if (bias) {
                            x[u] = p[u];
                        } else {
                            x[u].x *= p[u].x; x[u].y *= p[u].y; x[u].z *= p[u].z; x[u].w *= p[u].w;
                        }
                    }
                    if (fh.hasq && !bias) {
#pragma unroll
                        for (int u = 0; u < TW_CH; ++u) {
                            const float4 q = *reinterpret_cast<const float4*>(sa + A_OFF_Q + (((L0 + u) ^ sw) << 4));
                            const float4 dd = staged ? dst_[L0 + u]
                                                     : __ldg(reinterpret_cast<const float4*>(drow + n0k + 4 * (L0 + u)));
                            x[u].x += dd.x * q.x; x[u].y += dd.y * q.y; x[u].z += dd.z * q.z; x[u].w += dd.w * q.w;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < TW_CH; ++u) {  // round to nearest TF32 (the MMA would truncate)
                        x[u].x = round_tf32(x[u].x); x[u].y = round_tf32(x[u].y);
                        x[u].z = round_tf32(x[u].z); x[u].w = round_tf32(x[u].w);
                        if constexpr (!TS) *reinterpret_cast<float4*>(sa + (((L0 + u) ^ sw) << 4)) = x[u];
                    }
                    if constexpr (TS) {  // row = TMEM lane, k = column of A slot g % TS_SLOTS
                        static_assert(!TS || TW_SETS == 1, "TS transform writes whole rows");
                        tmem_st32(tmem_base + tq + A_COL0 + (uint32_t)(g % TS_SLOTS) * 32,
                                  reinterpret_cast<const float*>(x));
                    }
                }
                if (trw && g < TRN) trace[4 * TRN + g] = clock64();
                if constexpr (TS) tc_fence_before();
                else fence_proxy_async();
                if (trw && g < TRN) trace[5 * TRN + g] = clock64();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(fb0 + st_ * 8);
                if (trw && g < TRN) trace[2 * TRN + g] = clock64();
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue (both CTAs)
        const int ew = warp - 4;
        const int quad = warp % 4;
        const int chalf = ew / 4;
        uint8_t* slot = reinterpret_cast<uint8_t*>(epi_buf) + ew * S::EPI_SLOT;
        float* box = reinterpret_cast<float*>(slot);  // 32 rows x 128 B, 128-byte swizzle
        const uint32_t te_leader = map_to_leader(smem_u32(&tempty[0]));
        int acc = 0;
        uint32_t acc_phase = 0;
        const bool tre = trace && threadIdx.x == 4 * 32;
        int64_t tt = 0;
        for (int64_t t = pair_id; t < ntiles; t += npairs, ++tt) {
            int64_t opp, j0, n0;
            tile_of(t, opp, j0, n0);
            const int64_t m0 = opp * fh.rows + j0;
            mbar_wait(&tfull[acc], acc_phase);
            if (tre && tt < TRN) trace[6 * TRN + tt] = clock64();
            tc_fence_after();
            const int64_t row0 = m0 + 128 * rank + quad * 32;
            const int64_t band_end = (opp + 1) * fh.rows;  // rows beyond the band are not stored
            for (int cb = chalf * (BN / 64); cb < (chalf + 1) * (BN / 64); ++cb) {
                const int64_t col0 = n0 + cb * 32;
                if (col0 >= sh.N) break;
                float v[32];
                tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN + cb * 32), v);
                if (row0 < band_end && !(fh.dev & 2)) {
                    int64_t gr0, gc0;
                    // the slot is free once the previous box's TMA store has read it
                    if (lane == 0) bulk_wait_read();
                    __syncwarp();
                    const bool via_tma = fh.tma_h && epi.tma_block(row0, col0, band_end, sh.N, gr0, gc0);
                    const float sc = via_tma ? epi.alpha : 1.f;  // the scalar path applies alpha itself
                    // direct block: row = lane, 16-byte chunk q at q ^ (lane & 7)
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<float4*>(box + lane * 32 + ((q ^ (lane & 7)) << 2)) =
                            make_float4(sc * v[4 * q], sc * v[4 * q + 1], sc * v[4 * q + 2], sc * v[4 * q + 3]);
                    if (via_tma) {
                        fence_proxy_async();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&mapH, box, (int32_t)gc0, (int32_t)gr0);
                            bulk_commit();
                        }
                        if (epi.mirror) {
                            if (fh.dev & 4) {
                                if (lane == 0) bulk_wait_read();
                                __syncwarp();
                                // transposed box: row c holds this block's column c, element lane
#pragma unroll
                                for (int c = 0; c < 32; ++c)
                                    box[c * 32 + ((((lane >> 2) ^ (c & 7)) << 2) | (lane & 3))] = sc * v[c];
                                fence_proxy_async();
                                __syncwarp();
                                if (lane == 0) {
                                    tma_store_2d(&mapH, box, (int32_t)gr0, (int32_t)gc0);
                                    bulk_commit();
                                }
                            } else {
                                // mirrored block: H row gc0 + c gets this block's column c; the
                                // 32 lanes write 128 contiguous bytes per row (no shared memory)
                                float* mcol = epi.H + gc0 * epi.ldh + gr0 + lane;
#pragma unroll
                                for (int c = 0; c < 32; ++c) __stcs(mcol + c * epi.ldh, sc * v[c]);
                            }
                        }
                    } else {
                        __syncwarp();
                        epi.block_any(row0, col0, band_end, sh.N,
                                      [&](int r, int q) {
                                          return *reinterpret_cast<const float4*>(box + r * 32 + ((q ^ (r & 7)) << 2));
                                      },
                                      v, lane);
                        __syncwarp();
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(te_leader + acc * 8);
            if (tre && tt < TRN) trace[7 * TRN + tt] = clock64();
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (lane == 0) bulk_wait_all();  // epilogue stores complete before exit
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
    }
}

}  // namespace pair

// ---------------------------------------------------------------- host side
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw CurvError(kCudaError, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2D fp32 tensor map over an operand of `rows` x K (K-major: p[r*ld + k];
// MN-major: p[k*ld + r]), box = one BK x box_rows tile (or 32 x 32 pieces).
inline CUtensorMap make_map(const float* p, int64_t rows, int64_t K, int64_t ld, int mn, int box_rows,
                           bool mn3d = false) {
    CUtensorMap m;
    if (mn && mn3d) {
        // (element in 32-wide atom, k, atom): atom stride 128 B
        cuuint64_t dims3[3] = {32, (cuuint64_t)K, (cuuint64_t)ceil_div(rows, 32)};
        cuuint64_t str3[2] = {(cuuint64_t)ld * 4, 128};
        cuuint32_t box3[3] = {32, BK, (cuuint32_t)(box_rows / 32)}, es3[3] = {1, 1, 1};
        if ((reinterpret_cast<uintptr_t>(p) & 15) || (str3[0] & 15))
            throw CurvError(kCudaError, "TMA operand must be 16-byte aligned with a 16-byte row pitch");
        CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p), dims3, str3, box3, es3,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw CurvError(kCudaError, "cuTensorMapEncodeTiled (3D) failed: " + std::to_string((int)r));
        return m;
    }
    cuuint64_t dims[2], strides[1];
    cuuint32_t box[2], es[2] = {1, 1};
    if (!mn) {
        dims[0] = (cuuint64_t)K; dims[1] = (cuuint64_t)rows;
        box[0] = BK; box[1] = (cuuint32_t)box_rows;
    } else {
        dims[0] = (cuuint64_t)rows; dims[1] = (cuuint64_t)K;
        box[0] = 32; box[1] = BK;
    }
    strides[0] = (cuuint64_t)ld * 4;
    if ((reinterpret_cast<uintptr_t>(p) & 15) || (strides[0] & 15))
        throw CurvError(kCudaError, "TMA operand must be 16-byte aligned with a 16-byte row pitch");
    const CUtensorMapSwizzle swz = mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CurvError(kCudaError, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

// 2-D fp16 K-major map (rows x K, pitch ld halves), box (64, box_rows), 128-byte swizzle
inline CUtensorMap make_map_f16(const __half* p, int64_t rows, int64_t K, int64_t ld, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
    if ((reinterpret_cast<uintptr_t>(p) & 15) || (strides[0] & 15))
        throw CurvError(kCudaError, "TMA operand must be 16-byte aligned with a 16-byte row pitch");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(p), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CurvError(kCudaError, "cuTensorMapEncodeTiled (f16) failed: " + std::to_string((int)r));
    return m;
}

// 3D fp32 map without swizzle over p[(c * d1 + b) * ld0 + a] -- dims
// (d0, d1, d2), dim-2 stride s2 elements -- box (b0, b1, b2)
inline CUtensorMap make_map_plain3(const float* p, int64_t d0, int64_t d1, int64_t d2, int64_t s2, int b0, int b1,
                                   int b2) {
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
    cuuint64_t str[2] = {(cuuint64_t)d0 * 4, (cuuint64_t)s2 * 4};
    cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2}, es[3] = {1, 1, 1};
    if ((reinterpret_cast<uintptr_t>(p) & 15) || (str[0] & 15) || (str[1] & 15))
        throw CurvError(kCudaError, "TMA operand must be 16-byte aligned with 16-byte pitches");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p), dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CurvError(kCudaError, "cuTensorMapEncodeTiled (plain 3D) failed: " + std::to_string((int)r));
    return m;
}

// H (rows x ldh fp32, rows <= ldh) as 32 x 32 boxes with the 128-byte swizzle
inline CUtensorMap make_map_h(float* H, int64_t ldh) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)ldh, (cuuint64_t)ldh};
    cuuint64_t str[1] = {(cuuint64_t)ldh * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    if ((reinterpret_cast<uintptr_t>(H) & 15) || (str[0] & 15))
        throw CurvError(kCudaError, "TMA store target must be 16-byte aligned with a 16-byte row pitch");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, H, dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CurvError(kCudaError, "cuTensorMapEncodeTiled (H) failed: " + std::to_string((int)r));
    return m;
}

inline int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
}

// out = nearest TF32 of in, over a flat range (whole pitched buffers)
__global__ void round_tf32_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t count) {
    const int64_t n4 = count / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 v = reinterpret_cast<const float4*>(in)[i];
        v.x = round_tf32(v.x); v.y = round_tf32(v.y); v.z = round_tf32(v.z); v.w = round_tf32(v.w);
        reinterpret_cast<float4*>(out)[i] = v;
    }
    for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = round_tf32(in[i]);
}

// hi = tf32(x) (round to nearest), lo = tf32(x - hi); padding columns copied as 0
__global__ void split_tf32_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                  float* __restrict__ hi, float* __restrict__ lo) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows * cols) return;
    const int64_t off = (i / cols) * ld + i % cols;
    const float v = x[off];
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    const float hf = __uint_as_float(h);
    uint32_t l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(v - hf));
    hi[off] = hf;
    lo[off] = __uint_as_float(l);
}

template <int BN, class Epi>
void launch(cudaStream_t s, const TcShape& sh, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& alo,
            const CUtensorMap& blo, const Epi& e) {
    const int smem = TcSmem<BN>::bytes(sh.nsplit);
    func_attr_once((const void*)tc_gemm_kernel<BN, Epi>, [] {
        CK_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<BN, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     std::max(TcSmem<BN>::bytes(1), TcSmem<BN>::bytes(3))));
    });
    const int64_t tiles = ceil_div(sh.M, BM) * ceil_div(sh.N, BN);
    const int grid = (int)std::min<int64_t>(tiles, num_sms());
    tc_gemm_kernel<BN, Epi><<<grid, kThreads, smem, s>>>(a, b, alo, blo, sh, e);
    CK_LAUNCH();
}

template <int BN, class Epi, bool F16 = false>
void launch_pair(cudaStream_t s, const TcShape& sh, const CUtensorMap& a, const CUtensorMap& b,
                 const CUtensorMap& alo, const CUtensorMap& blo, const Epi& e) {
    using S = pair::PairSmem<BN>;
    const int smem = S::bytes(sh.nsplit);
    func_attr_once((const void*)pair::tc_gemm_pair_kernel<BN, Epi, F16>, [] {
        CK_CUDA(cudaFuncSetAttribute(pair::tc_gemm_pair_kernel<BN, Epi, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     std::max(S::bytes(1), S::bytes(3))));
    });
    const int64_t tiles = ceil_div(sh.M, 256) * ceil_div(sh.N, BN) * std::max(1, sh.ksplit);
    const int grid = 2 * (int)std::min<int64_t>(tiles, num_sms() / 2);
    CUtensorMap mc = a;  // unused unless the epilogue stores by TMA
    Epi ee = e;
    if constexpr (EpiTma<Epi>::value) {
        if (e.ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(e.c) & 15) == 0) mc = make_map_h(e.c, e.ldc);
        else ee.tma = 0;  // pitch not TMA-addressable: scalar epilogue for every block
    }
    pair::tc_gemm_pair_kernel<BN, Epi, F16><<<grid, pair::kThreads2, smem, s>>>(a, b, alo, blo, mc, sh, ee);
    CK_LAUNCH();
}

}  // namespace tc

// TF32 tensor-core GEMM with the generic epilogue contract (Epi::block).
template <class Epi>
void gemm_tf32(int prec, cudaStream_t s, int64_t M, int64_t N, int64_t K, Opnd<float> A, Opnd<float> B,
               const Epi& e, int ksplit = 1) {
    if (M <= 0 || N <= 0) return;
    // MN-major 32-bit operands use the 128B swizzle with 32B atoms
    // (SWIZZLE_128B_BASE32B, TMA SWIZZLE_128B_ATOM_32B): LBO = stride between
    // 32-element MN slices (BK rows x 128 B), SBO = stride between 4-row K
    // groups, one K=8 MMA step = 8 rows.  Plain SWIZZLE_128B reads zeros here.
    // a 3D box may read up to the next multiple of 32 rows: only when the
    // pitch covers it (reads past `rows` land in masked output rows/columns)
    const int a3 = (!A.kmajor && A.ld >= round_up(M, 32)) ? 1 : 0;
    const int b3 = (!B.kmajor && B.ld >= round_up(N, 32)) ? 1 : 0;
    tc::TcShape sh{M, N, K, A.kmajor ? 0 : 1, B.kmajor ? 0 : 1, prec == k3xTF32 ? 3 : 1,
                   (uint32_t)tc::BK * 128u, 512u, 1024u, 1u, a3, b3, ksplit, A.once, B.once};
    static const int group_env = getenv("CURVKIT_GROUP_M") ? atoi(getenv("CURVKIT_GROUP_M")) : 0;  // dev knob
    if (group_env > 0) sh.group_m = group_env;
    static const int dev_env = getenv("CURVKIT_DEV_PAIR") ? atoi(getenv("CURVKIT_DEV_PAIR")) : 0;  // dev ablations
    sh.dev = dev_env;
    const int bn = N >= 192 ? 256 : (N > 64 ? 128 : 64);
    DevMem alo, blo, ahi, bhi;
    const float* pa = A.p;
    const float* pb = B.p;
    const float* pal = A.p;
    const float* pbl = B.p;
    if (sh.nsplit == 1) {
        // the MMA truncates fp32 to TF32 (a bias towards zero in every
        // product): operands not pre-rounded by their producer get a
        // round-to-nearest copy (same layout and pitch, padding included)
        auto round_copy = [&](const Opnd<float>& o, int64_t rows, DevMem& out) -> const float* {
            const int64_t r = o.kmajor ? rows : K, c = o.kmajor ? K : rows;
            // last row only up to what a TMA box can touch (never past the source)
            const int64_t count = (r - 1) * o.ld + std::min(o.ld, round_up(c, 32)) / 4 * 4;
            out = DevMem((size_t)count * 4, s);
            tc::round_tf32_kernel<<<(unsigned)std::min<int64_t>(ceil_div(count, 1024), 148 * 32), 256, 0, s>>>(
                o.p, dptr<float>(out), count);
            CK_LAUNCH();
            return dptr<float>(out);
        };
        if (!A.rounded) pa = round_copy(A, M, ahi);
        if (!B.rounded) {
            if (B.p == A.p && B.ld == A.ld && B.kmajor == A.kmajor) pb = pa;
            else pb = round_copy(B, N, bhi);
        }
        pal = pa;
        pbl = pb;
    }
    if (sh.nsplit == 3) {
        // split both operands into hi/lo TF32 parts (same layout and pitch)
        auto split = [&](const Opnd<float>& o, int64_t rows, DevMem& hi, DevMem& lo) {
            const int64_t r = o.kmajor ? rows : K, c = o.kmajor ? K : rows;
            hi = DevMem((size_t)r * o.ld * 4, s);
            lo = DevMem((size_t)r * o.ld * 4, s);
            tc::split_tf32_kernel<<<(unsigned)ceil_div(r * c, 256), 256, 0, s>>>(o.p, r, c, o.ld, dptr<float>(hi),
                                                                                 dptr<float>(lo));
            CK_LAUNCH();
        };
        split(A, M, ahi, alo);
        pa = dptr<float>(ahi);
        pal = dptr<float>(alo);
        if (B.p == A.p && B.ld == A.ld && B.kmajor == A.kmajor) {
            pb = pa;
            pbl = pal;
        } else {
            split(B, N, bhi, blo);
            pb = dptr<float>(bhi);
            pbl = dptr<float>(blo);
        }
    }
    // CTA-pair (cta_group::2) tiles of 256 x bn when M gives every pair work;
    // each CTA then stages only bn/2 rows of B.
    static const bool no_pair = getenv("CURVKIT_NO_PAIR") != nullptr;
    // (M = 256 exactly fills one pair tile: a 4-unit band of a 64-input layer, config 3 W = 8)
    const bool use_pair = (!no_pair && bn >= 128 && (M >= 512 || M == 256)) || ksplit > 1;
    if (ksplit > 1 && (bn < 128 || M < 512)) throw CurvError(kRuntimeError, "split-K needs the CTA-pair kernel");
    const int box_b = use_pair ? bn / 2 : bn;
    CUtensorMap ma = tc::make_map(pa, M, K, A.ld, sh.a_mn, tc::BM, a3);
    CUtensorMap mb = tc::make_map(pb, N, K, B.ld, sh.b_mn, box_b, b3);
    CUtensorMap mal = tc::make_map(pal, M, K, A.ld, sh.a_mn, tc::BM, a3);
    CUtensorMap mbl = tc::make_map(pbl, N, K, B.ld, sh.b_mn, box_b, b3);
    if (use_pair) {
        if (bn == 256) tc::launch_pair<256>(s, sh, ma, mb, mal, mbl, e);
        else tc::launch_pair<128>(s, sh, ma, mb, mal, mbl, e);
        return;
    }
    if (bn == 256) tc::launch<256>(s, sh, ma, mb, mal, mbl, e);
    else if (bn == 128) tc::launch<128>(s, sh, ma, mb, mal, mbl, e);
    else tc::launch<64>(s, sh, ma, mb, mal, mbl, e);
}

// kF16S GEMM on the CTA-pair kernel: K-major fp16 operands A (M x K, lda) and
// B (N x K, ldb) pre-scaled by exact powers of two, entry (r, c) multiplied by
// rsc[r] * csc[c] before the epilogue.  M >= 512 and N > 64 (pair tiles).
template <class Epi>
void gemm_f16(cudaStream_t s, int64_t M, int64_t N, int64_t K, const __half* A, int64_t lda, const __half* B,
              int64_t ldb, const float* rsc, const float* csc, const Epi& e) {
    if (M <= 0 || N <= 0) return;
    if (M < 512 || N <= 64) throw CurvError(kRuntimeError, "gemm_f16: needs M >= 512 and N > 64");
    tc::TcShape sh{M, N, K, 0, 0, 1, (uint32_t)tc::BK * 128u, 512u, 1024u, 1u, 0, 0};
    sh.f16 = 1;
    sh.rsc = rsc;
    sh.csc = csc;
    const int bn = N >= 192 ? 256 : 128;
    CUtensorMap ma = tc::make_map_f16(A, M, K, lda, tc::BM);
    CUtensorMap mb = tc::make_map_f16(B, N, K, ldb, bn / 2);
    if (bn == 256) tc::launch_pair<256, Epi, true>(s, sh, ma, mb, ma, mb, e);
    else tc::launch_pair<128, Epi, true>(s, sh, ma, mb, ma, mb, e);
}

namespace tc {
// K-slab partial products: slab k of the workspace holds the tile products
// over its K range (plain stores, no atomics)
struct EpiSlab {
    static constexpr bool kSplitK = true;
    float* ws;
    int64_t ldw, slab;
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int, int64_t, int64_t, float) const {}
    __device__ void block_split(int k, int64_t row0, int64_t col0, int64_t M, int64_t N, const float (*buf)[36],
                                const float* v, int lane) const {
        EpiStore<float>{ws + k * slab, ldw, 0, 1.f, 0.f}.block(row0, col0, M, N, buf, v, lane);
    }
    __device__ void block(int64_t row0, int64_t col0, int64_t M, int64_t N, const float (*buf)[36], const float* v,
                          int lane) const {
        block_split(0, row0, col0, M, N, buf, v, lane);
    }
};

// C = sum over slabs in fixed order (deterministic), 4 columns per thread
__global__ void slab_sum_kernel(const float* __restrict__ ws, int64_t ldw, int64_t slab, int nslab, int64_t M,
                                int64_t N, float alpha, float* __restrict__ C, int64_t ldc) {
    const int64_t nq = ldw / 4;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M * nq) return;
    const int64_t r = i / nq, c = (i % nq) * 4;
    if (c >= N) return;
    float4 acc = __ldcs(reinterpret_cast<const float4*>(ws + r * ldw + c));
    for (int k = 1; k < nslab; ++k) {
        const float4 x = __ldcs(reinterpret_cast<const float4*>(ws + k * slab + r * ldw + c));
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    const float a[4] = {acc.x, acc.y, acc.z, acc.w};
    for (int u = 0; u < 4 && c + u < N; ++u) C[r * ldc + c + u] = alpha * a[u];
}
}  // namespace tc

// C (M x N, ldc) = A B on the tensor cores.  When the tile grid alone leaves
// most SM pairs idle (short M, long K: J X with M = N examples) K is cut into
// slabs whose partial tiles are summed afterwards in fixed order.
inline void gemm_tf32_store(int prec, cudaStream_t s, int64_t M, int64_t N, int64_t K, Opnd<float> A,
                            Opnd<float> B, float* C, int64_t ldc, float alpha = 1.f) {
    const int bn = N >= 192 ? 256 : (N > 64 ? 128 : 64);
    const int64_t pairs = tc::num_sms() / 2;
    const int64_t tiles = ceil_div(M, 256) * ceil_div(N, bn);
    const int64_t nk = ceil_div(K, tc::BK);
    int64_t ks = 1;
    if (bn >= 128 && M >= 512 && tiles < pairs && nk >= 64) {
        const int64_t target = std::min<int64_t>(ceil_div(8 * pairs, tiles), nk / 16);
        const int64_t kcb = ceil_div(nk, target);
        ks = ceil_div(nk, kcb);  // every slab non-empty
    }
    if (ks <= 1) {
        gemm_tf32(prec, s, M, N, K, A, B, EpiStore<float>{C, ldc, 0, alpha, 0.f});
        return;
    }
    const int64_t ldw = round_up(N, 4), slab = M * ldw;
    DevMem ws((size_t)(ks * slab) * sizeof(float), s);
    gemm_tf32(prec, s, M, N, K, A, B, tc::EpiSlab{dptr<float>(ws), ldw, slab}, (int)ks);
    tc::slab_sum_kernel<<<(unsigned)ceil_div(M * (ldw / 4), 256), 256, 0, s>>>(dptr<float>(ws), ldw, slab, (int)ks,
                                                                              M, N, alpha, C, ldc);
    CK_LAUNCH();
}

// Fused Hessian block (TF32 only): weight-tangent rows of block (k, m) with
// the A operand generated in shared memory (see tc_hess_fused_kernel).
template <>
struct HessFused<float> {
    static bool run(int prec, cudaStream_t s, const HessFusedArgs<float>& a, const EpiHess<float>& e) {
        if (!tf32_class(prec)) return false;
        namespace pair = tc::pair;
        // A from TMEM (R never in shared memory) is correct but measured slower
        // on B200 (5.3 vs 4.2 clocks per N column per k-block): opt-in only
        static const bool ts = getenv("CURVKIT_HESS_TS") != nullptr;
        static const bool ss192 = getenv("CURVKIT_HESS_SS192") != nullptr;  // dev: control for the TS variant
        if (ss192) return launch<192, false>(s, a, e);
        if constexpr (pair::TW_SETS == 1)
            if (ts) return launch<192, true>(s, a, e);
        return launch<256, false>(s, a, e);
    }

    template <int BN, bool TS>
    static bool launch(cudaStream_t s, const HessFusedArgs<float>& a, const EpiHess<float>& e) {
        namespace pair = tc::pair;
        pair::FusedHess fh{a.pv, a.dT, a.ldn, a.tk, a.tm, a.tm1, a.nw, a.qrows, a.diag, a.qT ? 1 : 0, nullptr, 0,
                           a.rows, 0};
        // a CTA's 128 weight rows span at most 127 / T_k + 2 output units
        const int64_t to = a.rows - a.nw;
        fh.pv_tma = (pair::STAGE_PV && 127 / a.tk + 2 <= pair::PV_ROWS) ? 1 : 0;
        CUtensorMap mpv = tc::make_map_plain3(a.pv, a.ldn, a.tm1, to, a.tm1 * a.ldn, 32, 1, pair::PV_ROWS);
        CUtensorMap mdt = a.qT ? tc::make_map_plain3(a.dT, a.ldn, 1, to, a.ldn, 32, 1, pair::PV_ROWS) : mpv;
        const int64_t N = a.tm + 1;  // weight columns + bias column of block m
        // tile list: every (o'' band, 256-row j tile, n tile) holding a required entry
        std::vector<int4> list;
        for (int64_t o = 0; o < a.tm1; ++o)
            for (int64_t j0 = fh.jstart(o); j0 < a.rows; j0 += 256) {
                // tangent rows of this pair tile must intersect the owned shard
                if (e.woffk + j0 + 256 <= e.rlo || e.woffk + j0 >= e.rhi) continue;
                for (int64_t n0 = 0; n0 < N; n0 += BN)
                    if (!e.skip(0, o * a.rows + j0, n0, 256, BN))
                        list.push_back(make_int4((int)o, (int)j0, (int)n0, 0));
            }
        if (list.empty()) return true;
        // partial-width column tiles (the bias column's tail, N = T_m + 1) last: the
        // persistent pairs' final round then gets the short tiles (the transform
        // cost of a tile does not shrink with its width)
        std::stable_partition(list.begin(), list.end(), [&](const int4& t) { return t.z + BN <= N; });
        fh.tiles = static_cast<const int4*>(cached_upload(list.data(), list.size() * sizeof(int4)));
        fh.ntiles = (int64_t)list.size();
        const int b3 = a.lda_m >= round_up(N, 32) ? 1 : 0;
        tc::TcShape sh{0, N, a.n, 0, 1, 1, (uint32_t)tc::BK * 128u, 512u, 1024u, 1u, 0, b3};
        CUtensorMap mak = tc::make_map(a.akT, a.ak_rows, a.n, a.ldn, 0, 128);
        CUtensorMap mq = a.qT ? tc::make_map(a.qT, a.q_rows_total, a.n, a.ldn, 0, 128) : mak;
        // B = a_m, rounded to nearest TF32 (n rows x lda_m, padding included)
        DevMem amr((size_t)a.n * a.lda_m * 4, s);
        tc::round_tf32_kernel<<<(unsigned)std::min<int64_t>(ceil_div(a.n * a.lda_m, 1024), 148 * 32), 256, 0, s>>>(
            a.am, dptr<float>(amr), a.n * a.lda_m);
        CK_LAUNCH();
        CUtensorMap mb = tc::make_map(dptr<float>(amr), N, a.n, a.lda_m, 1, BN / 2, b3);
        using S = pair::FusedSmem<BN>;
        func_attr_once((const void*)pair::tc_hess_fused_kernel<BN, EpiHess<float>, TS>, [] {
            CK_CUDA(cudaFuncSetAttribute(pair::tc_hess_fused_kernel<BN, EpiHess<float>, TS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, std::max(S::bytes(0), S::bytes(1))));
        });
        int grid = 2 * (int)std::min<int64_t>(fh.ntiles, tc::num_sms() / 2);
        if (const char* g = getenv("CURVKIT_DEV_GRID")) grid = std::min(grid, 2 * (atoi(g) / 2));  // dev: fewer SMs
        static const bool tracing = getenv("CURVKIT_TRACE") != nullptr;
        DevMem trbuf;
        if (tracing) {
            trbuf = DevMem(8 * 1024 * sizeof(long long), s);
            CK_CUDA(cudaMemsetAsync(trbuf.p, 0, 8 * 1024 * sizeof(long long), s));
            fh.trace = dptr<long long>(trbuf);
        }
        // H as a 2D map of 32 x 32 boxes (128-byte swizzle) for the epilogue
        fh.tma_h = (e.ldh % 4 == 0 && (reinterpret_cast<uintptr_t>(e.H) & 15) == 0) ? 1 : 0;
        static const int dev = getenv("CURVKIT_DEV_FUSED") ? atoi(getenv("CURVKIT_DEV_FUSED")) : 0;
        fh.dev = dev;
        CUtensorMap mh = fh.tma_h ? tc::make_map_h(e.H, e.ldh) : mb;
        pair::tc_hess_fused_kernel<BN, EpiHess<float>, TS><<<grid, pair::kFusedThreads, S::bytes(fh.hasq), s>>>(
            mak, mq, mb, mpv, mdt, mh, fh, sh, e);
        CK_LAUNCH();
        if (tracing) {
            std::vector<long long> h(8 * 1024);
            CK_CUDA(cudaMemcpyAsync(h.data(), trbuf.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s));
            CK_CUDA(cudaStreamSynchronize(s));
            static int call = 0;
            char fn[64];
            snprintf(fn, sizeof fn, "gpurun_out/trace_%d.bin", call++);
            if (FILE* f = fopen(fn, "wb")) {
                fwrite(h.data(), sizeof(long long), h.size(), f);
                fclose(f);
            }
        }
        return true;
    }
};

// Route TF32 precisions of the large curvature GEMMs to the tensor cores.
template <class Epi>
struct CurvGemm<float, Epi> {
    static void run(int prec, cudaStream_t s, int64_t M, int64_t N, int64_t K, Opnd<float> A, Opnd<float> B,
                    const Epi& e) {
        if (tf32_class(prec) || prec == k3xTF32) gemm_tf32(tc_form(prec), s, M, N, K, A, B, e);
        else gemm_simt<float>(s, M, N, K, 1, A, B, e);
    }
};

}  // namespace ck

#include "symkr.cuh"
