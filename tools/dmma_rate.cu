// FP64 tensor-core peak on this GPU: back-to-back mma.sync.m8n8k4.f64 (DMMA)
// from every warp of every SM, operands in registers, 8 independent
// accumulator chains per warp.  Prints TFLOP/s per warps-per-SM setting; the
// best figure is the fp64 roofline denominator bench.py uses
// (profiles/fp64_peak.json).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_rate tools/dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__global__ void dmma_loop(int reps, double seed, double* out) {
    double acc[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
    const double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int c = 0; c < 8; ++c) dmma(acc[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
    if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains live
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 1024 * sizeof(double));
    const int reps = 1 << 14;
    double best = 0.0;
    for (int warps : {4, 8, 16, 32}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        dmma_loop<<<sms * 4, warps * 32 / 4>>>(reps / 8, 1.0, d);  // warm-up (clocks up)
        dmma_loop<<<sms * 4, warps * 32 / 4>>>(reps, 1.0, d);
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) dmma_loop<<<sms * 4, warps * 32 / 4>>>(reps, 1.0, d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 5.0 * sms * 4 * (warps / 4) * (double)reps * 8 * 512;  // 8x8x4 x 2 per DMMA
        const double tf = flops / (ms * 1e-3) / 1e12;
        best = tf > best ? tf : best;
        printf("warps/SM %2d: %8.3f ms  %6.2f TFLOP/s fp64 (%s)\n", warps, ms, tf, cudaGetErrorString(cudaGetLastError()));
    }
    printf("{\"fp64_tflops\": %.2f}\n", best);
    return 0;
}
