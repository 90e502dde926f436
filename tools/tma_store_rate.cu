// Dev microbenchmark: TMA store (cp.async.bulk.tensor ... global.shared::cta)
// throughput for the box shapes of the curvature epilogues, every SM storing
// into its own region of a P x P fp32 matrix (ld = 25472, as config 1).
//   shape 0: 2-D 32 x 32 box (128-byte rows; SYRK / fused Hessian epilogue)
//   shape 1: 4-D 16 c x 8 i x 8 o'' box (64-byte rows; orbit types 1, 4)
//   shape 2: 4-D 8 i x 16 c x 8 o'' box (32-byte rows; orbit types 2, 3)
//   shapes 3, 4: shapes 1, 2 with 16 o'' (twice the rows per box)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_store_rate tools/tma_store_rate.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void store_kernel(const __grid_constant__ CUtensorMap map, int shape, int boxes_per_warp, int warps,
                             long long* out) {
    extern __shared__ __align__(1024) float sm[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 16 * 1024; i += blockDim.x) sm[i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    long long t0 = clock64();
    if (warp < warps && lane == 0) {
        const float* src = sm + warp * (shape >= 3 ? 2048 : 1024);  // 4 / 8 KB per warp
        for (int b = 0; b < boxes_per_warp; ++b) {
            // each CTA walks its own band of rows; boxes spread like the kernels' tiles
            const int blk = blockIdx.x * warps * boxes_per_warp + warp * boxes_per_warp + b;
            if (shape == 0) {
                const int r = (blk % 790) * 32, c = (blk / 790 % 790) * 32;
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&map),
                             "r"(su32(src)), "r"(c), "r"(r) : "memory");
            } else {
                // (d0, d1, o'', o) for 784-wide units: d0 block, d1 block, o'' run start, o
                const int o = blk % 32, ob = (blk / 32) % 4, d1b = (blk / 128) % 49, d0b = (blk / 6272) % 49;
                const int sh = shape >= 3 ? shape - 2 : shape;
                const int c0 = sh == 1 ? d0b * 16 : d1b * 8, c1 = sh == 1 ? d1b * 8 : d0b * 16;
                asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(&map),
                             "r"(su32(src)), "r"(c0), "r"(c1), "r"(shape >= 3 ? (ob & 1) * 16 : ob * 8), "r"(o) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const int64_t P = 25450, ld = 25472, T = 784, U = 32;
    float* H;
    cudaMalloc(&H, (size_t)P * ld * 4);
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int shape = 0; shape < 5; ++shape) {
        const int sh = shape >= 3 ? shape - 2 : shape, E = shape >= 3 ? 16 : 8;
        CUtensorMap m;
        CUresult r;
        if (shape == 0) {
            cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)P}, str[1] = {(cuuint64_t)ld * 4};
            cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, H, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            // type 1: (c, i, o'', o) strides (1, ld, T, T ld); type 2: (i, c, o'', o) strides (1, ld, T ld, T)
            cuuint64_t dims[4] = {(cuuint64_t)T, (cuuint64_t)T, (cuuint64_t)U, (cuuint64_t)U};
            cuuint64_t str[3] = {(cuuint64_t)ld * 4, (cuuint64_t)(sh == 1 ? T : T * ld) * 4,
                                 (cuuint64_t)(sh == 1 ? T * ld : T) * 4};
            cuuint32_t box[4] = {(cuuint32_t)(sh == 1 ? 16 : 8), (cuuint32_t)(sh == 1 ? 8 : 16), (cuuint32_t)E, 1},
                       es[4] = {1, 1, 1, 1};
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, H, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
        for (int warps : {1, 2, 4, 8}) {
            const int bpw = (shape >= 3 ? 2048 : 4096) / warps;
            for (int rep = 0; rep < 2; ++rep) store_kernel<<<148, 256, 64 * 1024>>>(m, shape, bpw, warps, d);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            store_kernel<<<148, 256, 64 * 1024>>>(m, shape, bpw, warps, d);
            cudaEventRecord(e1);
            cudaError_t err = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = 148.0 * warps * bpw * (shape >= 3 ? 8192 : 4096);
            printf("shape %d (%s) warps %d: %.3f ms, %.2f TB/s  %s\n", shape,
                   shape == 0 ? "32x32, 128 B rows" : shape == 1 ? "16x8x8, 64 B rows" : shape == 2 ? "8x16x8, 32 B rows" : shape == 3 ? "16x8x16, 64 B rows" : "8x16x16, 32 B rows", warps, ms,
                   bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
        }
    }
    return 0;
}
