// Dev microbenchmark: the symkr MMA issue loop in isolation (cta_group::2,
// kind::tf32, M = 256, N = bn, 4 MMAs per 32-example K-block advancing inside
// the 128-byte swizzle atom, NST rotating smem stages, optional commit per
// K-block).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dev/mma_loop tools/dev/mma_loop.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int n, int mn = 0) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)mn << 15) | ((uint32_t)mn << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

// whole-warp issue: every lane computes the (uniform) descriptors, one elected lane issues
__global__ void __cluster_dims__(2, 1, 1) warp_kernel(int kblocks, int n, int nst, int stage_bytes, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, cbar;
    __shared__ uint32_t tmem_holder;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < nst * stage_bytes / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.25f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&cbar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x / 32 == 0)
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_holder)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_holder;
    if (threadIdx.x / 32 == 0 && rank == 0) {
        const uint32_t id = idesc(n), z = 0;
        const uint64_t a0 = sdesc(su32(sm), 16, 1024, 2), b0 = sdesc(su32(sm) + 16384, 16, 1024, 2);
        long long t0 = clock64();
        int st = 0;
        for (int kb = 0; kb < kblocks; ++kb) {
            const uint64_t off = (uint64_t)((st * stage_bytes) >> 4);
            const uint32_t d = tmem + (uint32_t)(((kb >> 5) & 1) * 256);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t ad = a0 + off + (uint64_t)(ks * 2), bd = b0 + off + (uint64_t)(ks * 2);
                const uint32_t acc = ((kb & 31) > 0 || ks > 0) ? 1u : 0u;
                if (elect_one())
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(d),
                                 "l"(ad), "l"(bd), "r"(id), "r"(acc), "r"(z) : "memory");
                __syncwarp();
            }
            if (elect_one())
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&cbar)), "h"((uint16_t)3) : "memory");
            __syncwarp();
            if (++st == nst) st = 0;
        }
        if (elect_one()) {
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar)), "h"((uint16_t)1) : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(done) : "r"(su32(&bar)) : "memory");
            out[blockIdx.x] = clock64() - t0;
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x / 32 == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__global__ void __cluster_dims__(2, 1, 1) loop_kernel(int kblocks, int n, int nst, int stage_bytes, int kadv, int commit,
                                                       int vary_stage, long long* out, int ts, int mn) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, cbar;
    __shared__ uint32_t tmem_holder;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < nst * stage_bytes / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.25f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&cbar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x / 32 == 0)
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_holder)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_holder;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t id = idesc(n, mn), z = 0;
        long long t0 = clock64();
        for (int kb = 0; kb < kblocks; ++kb) {
            const int st = vary_stage ? kb % nst : 0;
            const uint32_t sa = su32(sm + st * stage_bytes), sb = sa + 16384;
            const uint32_t d = tmem + (uint32_t)(((kb / 32) & 1) * 256);
            for (int ks = 0; ks < 4; ++ks) {
                // K-major: 32-byte K step inside the 128-byte atom; MN-major (SWIZZLE_128B_BASE32B):
                // LBO = 32 x 128 B, SBO 512 B, K step of 8 rows = 1024 B
                const uint64_t ad = mn ? sdesc(sa + (kadv ? ks * 1024 : 0), 4096, 512, 1) : sdesc(sa + (kadv ? ks * 32 : 0), 16, 1024, 2);
                const uint64_t bd = mn ? sdesc(sb + (kadv ? ks * 1024 : 0), 4096, 512, 1) : sdesc(sb + (kadv ? ks * 32 : 0), 16, 1024, 2);
                const uint32_t acc = (kb % 32 > 0 || ks > 0) ? 1u : 0u;
                if (ts) {
                    const uint32_t d2 = tmem + (uint32_t)(((kb / 32) & 1) * 176);
                    const uint32_t at = tmem + 352u + (uint32_t)((kb % 5) * 32 + ks * 8);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(d2),
                                 "r"(at), "l"(bd), "r"(id), "r"(acc), "r"(z) : "memory");
                } else {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(d),
                                 "l"(ad), "l"(bd), "r"(id), "r"(acc), "r"(z) : "memory");
                }
            }
            if (commit)
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&cbar)), "h"((uint16_t)3) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar)), "h"((uint16_t)1) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(su32(&bar)) : "memory");
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x / 32 == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    const int smem = 5 * 35840;
    cudaFuncSetAttribute(loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    struct V { const char* name; int n, kadv, commit, vary, ts, mn; } vs[] = {
        {"SS N176 K-adv + stages         ", 176, 1, 1, 1, 0, 0}, {"SS N256 K-adv + stages         ", 256, 1, 1, 1, 0, 0},
        {"SS N128 K-adv + stages         ", 128, 1, 1, 1, 0, 0}, {"TS N176 K-adv + stages         ", 176, 1, 1, 1, 1, 0},
        {"TS N128 K-adv + stages         ", 128, 1, 1, 1, 1, 0}, {"SS N256 MN-major + stages      ", 256, 1, 1, 1, 0, 1},
        {"SS N256 stages, no K-adv       ", 256, 0, 1, 1, 0, 0}};
    for (auto& v : vs) {
        const int kb = 2048;
        for (int rep = 0; rep < 2; ++rep)
            loop_kernel<<<148, 128, smem>>>(kb, v.n, 5, 35840, v.kadv, v.commit, v.vary, d, v.ts, v.mn);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; i += 2) mx = h[i] > mx ? h[i] : mx;
        printf("%s: %7.1f clk per K-block (ideal %d)  %s\n", v.name, (double)mx / kb, 4 * v.n / 2, cudaGetErrorString(e));
    }
    cudaFuncSetAttribute(warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int nn : {128, 176, 256}) {
        const int kb = 2048;
        for (int rep = 0; rep < 2; ++rep) warp_kernel<<<148, 128, smem>>>(kb, nn, 5, 35840, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; i += 2) mx = h[i] > mx ? h[i] : mx;
        printf("warp-uniform issue N%d + stages + commit: %7.1f clk per K-block (ideal %d)  %s\n", nn, (double)mx / kb, 2 * nn, cudaGetErrorString(e));
    }
    return 0;
}
