// Dev microbenchmark: issue rate of back-to-back tcgen05.mma (no data
// dependencies, operands = whatever is in shared memory) for the shapes and
// operand layouts the curvature kernels use.  Prints clocks per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
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
// kind: 0 tf32, 1 bf16
__host__ __device__ constexpr uint32_t idesc(int kind, int m, int n, bool a_mn, bool b_mn) {
    return (1u << 4) | ((kind == 0 ? 2u : 1u) << 7) | ((kind == 0 ? 2u : 1u) << 10) | ((a_mn ? 1u : 0u) << 15) |
           ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// TS = 1: A operand from TMEM (columns 384.., cta_group::2 tf32 only)
template <int CG, int KIND, int TS = 0>
__global__ void __cluster_dims__(2, 1, 1) mma_rate(int reps, int n, int a_mn, int b_mn, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_holder;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        if (CG == 2)
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_holder)));
        else
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_holder)));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_holder;
    const int m = CG == 2 ? 256 : 128;
    const uint32_t id = idesc(KIND, m, n, a_mn, b_mn);
    if (threadIdx.x == 0 && (CG == 1 || rank == 0)) {
        const uint32_t a = su32(sm), b = su32(sm + 32 * 1024);
        const uint64_t ad = a_mn ? sdesc(a, 4096, 512, 1) : sdesc(a, 16, 1024, 2);
        const uint64_t bd = b_mn ? sdesc(b, 4096, 512, 1) : sdesc(b, 16, 1024, 2);
        const uint32_t z = 0;
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            const uint32_t d = tmem + (uint32_t)((r & 1) * 256);
            if (TS) {
                const uint32_t d2 = tmem + (uint32_t)((r & 1) * 192);
                asm volatile("tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, {%4, %4, %4, %4, %4, %4, %4, %4}, 1;" ::"r"(d2),
                             "r"(tmem + 384u + (uint32_t)((r & 3) * 32)), "l"(bd), "r"(id), "r"(z) : "memory");
            } else if (CG == 2) {
                if (KIND == 0)
                    asm volatile("tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%4, %4, %4, %4, %4, %4, %4, %4}, 1;" ::"r"(d),
                                 "l"(ad), "l"(bd), "r"(id), "r"(z) : "memory");
                else
                    asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%4, %4, %4, %4, %4, %4, %4, %4}, 1;" ::"r"(d),
                                 "l"(ad), "l"(bd), "r"(id), "r"(z) : "memory");
            } else {
                if (KIND == 0)
                    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(ad), "l"(bd), "r"(id) : "memory");
                else
                    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(ad), "l"(bd), "r"(id) : "memory");
            }
        }
        if (CG == 2)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar)), "h"((uint16_t)1) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(su32(&bar)) : "memory");
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) {
        if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int CG, int KIND, int TS = 0>
void run(const char* name, int n, int a_mn, int b_mn, int grid) {
    long long* d;
    cudaMalloc(&d, grid * sizeof(long long));
    cudaMemset(d, 0, grid * sizeof(long long));
    cudaFuncSetAttribute(mma_rate<CG, KIND, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int reps = 4096;
    mma_rate<CG, KIND, TS><<<grid, 128, 64 * 1024>>>(reps, n, a_mn, b_mn, d);
    mma_rate<CG, KIND, TS><<<grid, 128, 64 * 1024>>>(reps, n, a_mn, b_mn, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[296] = {0};
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    const int m = CG == 2 ? 256 : 128;
    const int k = KIND == 0 ? 8 : 16;
    const double clk = (double)mx / reps;
    // flops per SM per clock: M x N x K x 2 / CG per MMA
    printf("%-28s grid %3d  M %d N %3d K %2d a_mn %d b_mn %d : %7.1f clk/MMA  %6.0f flop/clk/SM  (%s)\n", name, grid, m, n, k,
           a_mn, b_mn, clk, 2.0 * m * n * k / CG / clk, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    for (int grid : {2, 148}) {
        run<2, 0, 1>("tf32 TS cta_group::2 N192", 192, 0, 0, grid);
        run<2, 0, 1>("tf32 TS cta_group::2 N176", 176, 0, 0, grid);
        run<2, 0, 0>("tf32 SS cta_group::2 N176", 176, 0, 0, grid);
        run<2, 0>("tf32 cta_group::2 KK", 256, 0, 0, grid);
        run<2, 0>("tf32 cta_group::2 K,MN", 256, 0, 1, grid);
        run<2, 0>("tf32 cta_group::2 MN,MN", 256, 1, 1, grid);
        run<2, 0>("tf32 cta_group::2 KK N128", 128, 0, 0, grid);
        run<2, 0>("tf32 cta_group::2 KK N64", 64, 0, 0, grid);
        run<1, 0>("tf32 cta_group::1 KK", 256, 0, 0, grid);
        run<2, 1>("bf16 cta_group::2 KK", 256, 0, 0, grid);
        run<1, 1>("bf16 cta_group::1 KK", 256, 0, 0, grid);
    }
    return 0;
}
