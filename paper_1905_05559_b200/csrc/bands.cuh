// bands.cuh -- unit bands: the multi-GPU layout of H and G.
//
// The rows of layer k's parameter block belong to its output units: unit o
// owns the weight rows (o, i), i < T_k, and the bias row o (model.hpp:44-46
// flatten order).  Shard r of W owns the units [u0[k], u1[k]) of every layer
// and stores the rows of those units, compact: per layer the weight rows of
// its units, then their bias rows.  In the unit-major order (layers, then
// units) the matrix is the symmetric completion of its block-lower triangle,
// whose row blocks are exactly these bands: a shard computes only entries
// whose column unit is <= the row's unit (the unit-diagonal squares whole), so
// the shards together compute each symmetric pair once, with no exchange.
// The final gather puts the bands' rows into place and mirrors the upper
// unit-major triangle (symmetrize_units_kernel).
//
// The reference shards Hessian columns over threads (curvature.cpp:39-71);
// this is the same "independent slices of the output" idea, cut so that each
// slice is balanced and symmetric work is not repeated.
#pragma once

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "model.cuh"

namespace ck {

struct UnitBand {
    int S = 0;
    int64_t u0[kMaxLayers] = {}, u1[kMaxLayers] = {};  // output units of layer k
    int64_t bw[kMaxLayers] = {}, bb[kMaxLayers] = {};  // band row of weight row (u0, 0) / of bias u0
    int64_t rows = 0;

    // Unit cuts.  A unit's cost in layer k: the diagonal block grows with the
    // packed unit pairs below it, u (u + 1) / 2 orbit columns of
    // (T_k + 1)(T_k + 2) / 2 values, the blocks left of it linearly, u (T_k + 1)
    // rows of woff_k columns -- 2 N flops per value or entry either way.  Every
    // layer but the most expensive one is cut so each shard gets ~1/W of it; the
    // most expensive layer (config 3: layer 0, 92% of the work) is then cut so
    // each shard's TOTAL is ~1/W, absorbing the lumps of the small layers (10
    // units over 8 shards).  Cuts fall on multiples of 4 units: every band row
    // range then starts 16-byte aligned, so the bias rows take the J GEMM too
    // (an unaligned start sent them to the fused block kernel: 1.5-1.8 ms of a
    // 15 ms band at c3, W = 8) -- except in the first layer, which has no
    // rectangle rows and keeps unit granularity (a 4-unit step of its largest
    // units is ~3% of the whole job).
    static double layer_cost(const ModelDesc& md, int k, int64_t u) {
        const int64_t tk = md.w[k];
        const double orb = (double)(tk + 1) * (double)(tk + 2) / 2.0, rect = (double)(tk + 1) * (double)md.woff[k];
        return (double)u * (u + 1) / 2.0 * orb + (double)u * rect;
    }
    // smallest u on a multiple of 4 nearest to cost_k(u) = target, in [0, U]
    static int64_t cut_for(const ModelDesc& md, int k, double target) {
        const int64_t U = md.w[k + 1];
        int64_t lo = 0, hi = U;  // smallest u with cost(u) >= target
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (layer_cost(md, k, mid) >= target) hi = mid;
            else lo = mid + 1;
        }
        if (lo > 0 && target - layer_cost(md, k, lo - 1) < layer_cost(md, k, lo) - target) --lo;  // nearer
        if (md.woff[k] == 0) return lo;  // no rectangle rows in the first layer: any unit aligns
        const int64_t q = (lo + 2) / 4 * 4;
        return q < U ? q : U;
    }
    static UnitBand make(const ModelDesc& md, int64_t W, int64_t r) {
        if (W < 1 || r < 0 || r >= W) throw CurvError(kContractError, "shard_units: need 0 <= shard < nshards");
        UnitBand b;
        b.S = md.S;
        // cut[k][s]: first unit of shard s in layer k (s = 0 .. W)
        std::vector<std::vector<int64_t>> cut(md.S, std::vector<int64_t>(W + 1));
        int a = 0;
        double total = 0.0;
        for (int k = 0; k < md.S; ++k) {
            const int64_t U = md.w[k + 1];
            const double ck = layer_cost(md, k, U);
            total += ck;
            if (ck > layer_cost(md, a, md.w[a + 1])) a = k;
            for (int64_t s = 0; s <= W; ++s)
                cut[k][s] = s == 0 ? 0 : s == W ? U : cut_for(md, k, ck * (double)s / (double)W);
        }
        for (int64_t s = 1; s < W; ++s) {  // the absorbing layer
            double other = 0.0;
            for (int k = 0; k < md.S; ++k)
                if (k != a) other += layer_cost(md, k, cut[k][s]);
            const double t = std::max(0.0, total * (double)s / (double)W - other);
            cut[a][s] = std::max(cut[a][s - 1], cut_for(md, a, t));
        }
        for (int k = 0; k < md.S; ++k) {
            b.u0[k] = cut[k][r];
            b.u1[k] = std::max(b.u0[k], cut[k][r + 1]);
        }
        for (int k = 0; k < md.S; ++k) {
            const int64_t nu = b.u1[k] - b.u0[k];
            b.bw[k] = b.rows;
            b.bb[k] = b.rows + nu * md.w[k];
            b.rows += nu * (md.w[k] + 1);
        }
        return b;
    }

    // contiguous global row ranges of the band: (global row, band row, count)
    struct Range {
        int64_t g, b, n;
    };
    std::vector<Range> ranges(const ModelDesc& md) const {
        std::vector<Range> out;
        for (int k = 0; k < md.S; ++k) {
            const int64_t nu = u1[k] - u0[k];
            if (nu <= 0) continue;
            out.push_back({md.woff[k] + u0[k] * md.w[k], bw[k], nu * md.w[k]});
            out.push_back({md.boff[k] + u0[k], bb[k], nu});
        }
        return out;
    }
};

// unit id of every row in the unit-major order (layers, then units)
__global__ void unit_ids_kernel(ModelDesc md, int32_t* __restrict__ g) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < md.P; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t base = 0;
        int k = 0;
        while (k + 1 < md.S && r >= md.woff[k + 1]) {
            base += md.w[k + 1];
            ++k;
        }
        const int64_t o = r < md.boff[k] ? (r - md.woff[k]) / md.w[k] : r - md.boff[k];
        g[r] = (int32_t)(base + o);
    }
}

// F[r][c] <- F[c][r] for every entry whose column unit follows the row's
// (the upper unit-major triangle), 32 x 32 tiles through shared memory
template <class T>
__global__ void symmetrize_units_kernel(T* __restrict__ F, int64_t ld, int64_t P, const int32_t* __restrict__ g) {
    __shared__ T t[32][33];
    __shared__ int32_t gr[32], gc[32];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    if (ty == 0) {
        gr[tx] = r0 + tx < P ? g[r0 + tx] : INT32_MAX;
        gc[tx] = c0 + tx < P ? g[c0 + tx] : -1;
    }
    __syncthreads();
    // any entry of the tile with g(col) > g(row)?
    int lo = gr[tx], hi = gc[tx];
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (hi <= lo) return;  // uniform over the block (every warp reduces the same arrays)
    for (int y = ty; y < 32; y += 8) {  // t[x][y] = F[c0 + y][r0 + x]: coalesced along the source row
        const int64_t sr = c0 + y, sc = r0 + tx;
        if (sr < P && sc < P) t[tx][y] = F[sr * ld + sc];
    }
    __syncthreads();
    for (int y = ty; y < 32; y += 8) {
        const int64_t r = r0 + y, c = c0 + tx;
        if (r < P && c < P && gc[tx] > gr[y]) F[r * ld + c] = t[y][tx];
    }
}

template <class T>
void symmetrize_units(const ModelDesc& md, T* F, int64_t ld, cudaStream_t s) {
    DevMem g((size_t)md.P * sizeof(int32_t), s);
    unit_ids_kernel<<<(unsigned)std::min<int64_t>(ceil_div(md.P, 256), 1024), 256, 0, s>>>(md, dptr<int32_t>(g));
    CK_LAUNCH();
    dim3 grid((unsigned)ceil_div(md.P, 32), (unsigned)ceil_div(md.P, 32));
    symmetrize_units_kernel<T><<<grid, dim3(32, 8), 0, s>>>(F, ld, md.P, dptr<int32_t>(g));
    CK_LAUNCH();
}

// full rows <- band rows (a copy per contiguous range)
template <class T>
void band_scatter(const ModelDesc& md, const UnitBand& b, const T* band, int64_t ld, T* full, int64_t ldf, cudaStream_t s) {
    for (const auto& r : b.ranges(md))
        CK_CUDA(cudaMemcpy2DAsync(full + r.g * ldf, ldf * sizeof(T), band + r.b * ld, ld * sizeof(T), md.P * sizeof(T),
                                  r.n, cudaMemcpyDeviceToDevice, s));
}

}  // namespace ck
