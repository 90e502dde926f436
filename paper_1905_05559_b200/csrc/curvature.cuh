// curvature.cuh -- orchestration of the curvature products on one GPU.
//
//   hvp      batched Pearlmutter R-op (autodiff.cpp:158-244): every layer of
//            the R-forward / R-backward pass and the final accumulation is
//            a GEMM over (direction x example) rows.
//   hessian  exact H (curvature.cpp:33-92).  Column p of H is the HVP on the
//            basis vector e_p.  For e_p a weight (o, i) of step k the R-state
//            factorises as s_n * f(n, o) with s_n = a_k[n][i], so the R-op
//            only runs for the T_{k+1} "profiles" o (plus T_k profiles i for
//            the explicit delta*RW term below the tangent layer), and every
//            block of H is one GEMM  R (rows (o'', p), K = n) x a_m (n x T_m+1)
//            whose A operand R is an elementwise product of profiles and
//            activations.  The lower block triangle is computed and mirrored.
//   opg      G = (1/N) J^T J as a symmetric (lower-triangle) GEMM over J.
#pragma once

#include <algorithm>
#include <vector>

#include "bands.cuh"
#include "common.cuh"
#include "gemm_simt.cuh"
#include "model.cuh"
#include "orbit_dmma.cuh"
#include "prof.cuh"

namespace ck {

// Large curvature GEMMs.  TF32 modes are routed to the tcgen05 kernel by
// the specialisations in gemm_tc.cuh; everything else runs SIMT FMAs.
template <class T, class Epi>
struct CurvGemm {
    static void run(int prec, cudaStream_t s, int64_t M, int64_t N, int64_t K, Opnd<T> A, Opnd<T> B,
                    const Epi& e) {
        (void)prec;
        gemm_simt<T>(s, M, N, K, 1, A, B, e);
    }
};

// Fused weight-tangent Hessian block: the R operand is formed on chip from
// the extended activation tile and the profiles.  Specialised for TF32 in
// gemm_tc.cuh; returns false where no fused kernel exists (then the R
// operand is materialised by rgen_kernel).
template <class T>
struct HessFusedArgs {
    const T* akT;       // a_k^T extended: row r holds a_k[., r mod T_k]
    int64_t ak_rows;
    const T* qT;        // Q_m^T extended [T_{m+1}][qrows][ldn] or null (m == k)
    int64_t qrows, q_rows_total;
    const T* pv;        // G or P_m transposed [T_{k+1}][T_{m+1}][ldn]
    const T* dT;        // delta_k^T [T_{k+1}][ldn]
    const T* am;        // a_m [n][lda_m] (B operand, MN-major)
    int64_t lda_m, ldn, n, tk, tm, tm1, nw;
    int diag;
    int64_t rows;  // all tangent rows of step k (weights then biases)
};

template <class T>
struct HessFused {
    static bool run(int, cudaStream_t, const HessFusedArgs<T>&, const EpiHess<T>&) { return false; }
};

// Diagonal layer block (k = m) by the symmetric Khatri-Rao product (symkr.cuh):
// B[(o,i),(o'',c)] = alpha sum_n abar_i abar_c Pi[o][o''] written with its
// four symmetric images.  TF32 only; returns false where it does not apply.
template <class T>
struct SymKrArgs {
    const T* akT;        // abar_k^T [T_k + 1][ldn] (row T_k = ones)
    const T* prof;       // H: profiles [U][U][ldn]; G: delta_k^T [U][ldn]
    int delta_products;  // 1: Pi[o][o''] = delta_o * delta_o'' (OPG)
    int64_t ldn, n, tk, U;
    T* H;
    int64_t ldh, woff, boff;
    T alpha;
    // output units [u0, u1) (u1 < 0: all) stored at band rows bwoff / bboff (< 0:
    // the block's own rows woff / boff): see symkr.cuh Params and bands.cuh
    int64_t u0 = 0, u1 = -1, bwoff = -1, bboff = -1;
    // >= 0: prof holds only the tangents of units prof_t0, prof_t0 + 1, ... and
    // Pi[o][o''] is read as prof[(o'' - prof_t0) U + o] (the profile is symmetric)
    int64_t prof_t0 = -1;
    // whole-block assembly in pieces: only the packed columns (o, o'') with o'' in
    // [pair_q0, pair_q1) (pair_q1 < 0: all), all four images of each stored.  Run
    // over descending o'' ranges, the rows of a range's units are complete when its
    // launch ends (the host-buffer OPG downloads them while the next range runs).
    int64_t pair_q0 = 0, pair_q1 = -1;
};

// kF16S OPG rectangles (blocks m < k): J^T in fp16 with an exact power-of-two
// scale per parameter row (symkr.cuh), multiplied on the fp16 datapath
struct JtF16Args {
    int S;
    const float* akT[kMaxLayers];  // abar_k^T [T_k + 1][ldn] (row T_k = ones)
    const float* dT[kMaxLayers];   // delta_k^T [T_{k+1}][ldn]
    int64_t w[kMaxLayers + 1], woff[kMaxLayers], boff[kMaxLayers];
    int64_t P, n, ldn;
};
template <class T>
struct OpgF16 {
    // J^T (P x ldn fp16) and the inverse row scales (P floats); false: no fp16 form
    static bool build(cudaStream_t, const JtF16Args&, DevMem&, DevMem&) { return false; }
    // G rows [r0, r1) x columns [0, cols) = alpha J^T[r0:r1] J^T[0:cols]^T, mirrored
    static void rect(cudaStream_t, int64_t, int64_t, int64_t, int64_t, const DevMem&, int64_t, const DevMem&, T*,
                     int64_t, T) {}
};

// kF16S Hessian blocks m < k through R in HBM (symkr.cuh): R rows in fp16 with
// an exact power-of-two scale from a per-row bound, a_m^T in fp16 with per-index
// scales, the fp16 pair GEMM
struct HessF16Args {
    const float* prof;  // P_m transposed [T_{k+1}][T_{m+1}][ldn]
    const float* q;     // Q_m transposed [T_k][T_{m+1}][ldn]
    const float* akT;   // a_k^T [T_k + 1][ldn]
    const float* dkT;   // delta_k^T [T_{k+1}][ldn]
    const float* am;    // a_m [n][lda_m] (column T_m = ones)
    int64_t lda_m, ldn, n, tk, np, tm, tm1;
};
template <class T>
struct HessF16 {
    struct Prep {
        DevMem amax, dmax, pmax, qmax, am16, aminv;
    };
    static bool prepare(cudaStream_t, const HessF16Args&, Prep&) { return false; }
    static void chunk(cudaStream_t, const HessF16Args&, const Prep&, int64_t, int64_t, int64_t, DevMem&, DevMem&,
                      const EpiHess<T>&, double) {}
};

template <class T>
struct SymKr {
    static bool tma_ok(const T*, int64_t, int64_t, int64_t) { return false; }
    static bool run(int, cudaStream_t, const SymKrArgs<T>&) { return false; }
};

// ---- symmetric orbits in the f32 / f64 modes (Engine::orbit_block) ----
// The same one-value-per-orbit scheme as symkr.cuh: Z[(i,c)][n] = abar_i abar_c
// is materialised for a chunk of pair blocks, V = Z Pi_packed^T runs on the
// FP64 tensor cores / FFMA (orbit_dmma.cuh), each value goes to its four places.

// Z[q][n] = akT[i_q][n] * akT[c_q][n]
template <class T>
__global__ void orbit_z_kernel(const T* __restrict__ akT, int64_t ldn, const int2* __restrict__ ic, int64_t q0,
                               int64_t nq, int64_t n, T* __restrict__ z) {
    const int64_t q = q0 + blockIdx.y;
    if (blockIdx.y >= nq) return;
    const int2 p = ic[q];
    const T* a = akT + p.x * ldn;
    const T* b = akT + p.y * ldn;
    T* out = z + (int64_t)blockIdx.y * ldn;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[i] * b[i];
}

// packed profiles: out[j][n] = src[(o_j U + o''_j)][n] (H) or dk[o_j][n] dk[o''_j][n] (OPG)
template <class T>
__global__ void orbit_pack_kernel(const T* __restrict__ src, const int2* __restrict__ oo, int64_t U, int64_t ldn,
                                  int64_t n, int delta_products, T* __restrict__ out, int64_t np) {
    for (int64_t j = blockIdx.y; j < np; j += gridDim.y) {  // grid.y <= 65535
        const int2 p = oo[j];
        T* d = out + j * ldn;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
            d[i] = delta_products ? src[p.x * ldn + i] * src[p.y * ldn + i] : src[(p.x * U + p.y) * ldn + i];
    }
}

// PV[o][o''][n] = dk[o][n] * dm[o''][n]  (OPG profile of block (k, m))
template <class T>
__global__ void outer_delta_kernel(const T* __restrict__ dk, const T* __restrict__ dm, int64_t um, int64_t ldn,
                                   T* __restrict__ pv) {
    const int64_t o = blockIdx.z, oo = blockIdx.y;
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < ldn; n += (int64_t)gridDim.x * blockDim.x)
        pv[(o * um + oo) * ldn + n] = dk[o * ldn + n] * dm[oo * ldn + n];
}

// out[r][.] = in[r mod period][.]  (row replication for the extended tiles)
template <class T>
__global__ void replicate_rows_kernel(const T* __restrict__ in, int64_t period, int64_t ld, T* __restrict__ out,
                                      int64_t rows, int64_t in_bstride, int64_t out_bstride) {
    const int64_t b = blockIdx.y;
    if constexpr (sizeof(T) == 4) {
        if (ld % 4 == 0 && in_bstride % 4 == 0 && out_bstride % 4 == 0 && rows * ld / 4 < (int64_t(1) << 31)) {
            const uint32_t q = (uint32_t)(ld / 4), total = (uint32_t)(rows * q);
            const float4* src = reinterpret_cast<const float4*>(in + b * in_bstride);
            float4* dst = reinterpret_cast<float4*>(out + b * out_bstride);
            for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
                const uint32_t r = i / q;
                __stcs(dst + i, __ldg(src + (size_t)(r % (uint32_t)period) * q + (i - r * q)));
            }
            return;
        }
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * ld; i += (int64_t)gridDim.x * blockDim.x)
        out[b * out_bstride + i] = in[b * in_bstride + ((i / ld) % period) * ld + i % ld];
}

// QX[o''][r][n] = QT[(r mod T_k)][o''][n]
template <class T>
__global__ void qext_kernel(const T* __restrict__ qt, int64_t tk, int64_t tm1, int64_t ldn, T* __restrict__ qx,
                            int64_t rows) {
    const int64_t opp = blockIdx.y;
    if constexpr (sizeof(T) == 4) {
        // 16-byte vectors along n (ldn is a multiple of 32); row index math in 32 bits
        const uint32_t q = (uint32_t)(ldn / 4), total = (uint32_t)(rows * q);
        const float4* src = reinterpret_cast<const float4*>(qt);
        float4* dst = reinterpret_cast<float4*>(qx) + (size_t)opp * rows * q;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
            const uint32_t r = i / q, e = i - r * q;
            __stcs(dst + i, __ldg(src + ((size_t)(r % (uint32_t)tk) * tm1 + opp) * q + e));
        }
    } else {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * ldn;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t r = i / ldn, e = i - r * ldn;
            qx[(opp * rows + r) * ldn + e] = qt[((r % tk) * tm1 + opp) * ldn + e];
        }
    }
}

// rz_k[b] = a_k RW_k[b]^T + Rb_k[b]
template <class T>
struct EpiRzBias {
    T* out; int64_t ld, bs; const T* rb; int64_t rbs;
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int b, int64_t m, int64_t o, T acc) const {
        out[b * bs + m * ld + o] = acc + rb[b * rbs + o];
    }
};

// batched view of EpiRback: direction b, example m -> stacked row b*n + m
template <class T>
struct EpiRb2 {
    EpiRback<T> inner; int64_t bs;
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int b, int64_t m, int64_t cc, T acc) const {
        inner(0, b * inner.n + m, cc, acc);
    }
};

inline unsigned blocks_for(int64_t n, int t = 256) { return (unsigned)ceil_div(n, t); }

template <class T>
struct Engine {
    const ModelDesc& md;
    cudaStream_t s;
    int prec;
    // opg_kr: restrict the diagonal blocks' packed columns (SymKrArgs::pair_q0 / pair_q1)
    int64_t pair_q0 = 0, pair_q1 = -1;

    // ---------------------------------------------------------------- grad
    void grad(const Cache<T>& c, T* g) {
        for (int k = 0; k < md.S; ++k) {
            EpiHv<T> e{g, 0, md.woff[k], md.boff[k], md.w[k], T(1), 0};
            gemm_simt<T>(s, md.w[k + 1], md.w[k] + 1, c.n, 1, mnmaj(c.delta[k], c.ldt[k]),
                         mnmaj(c.a[k], c.lda[k]), e);
        }
    }

    // ---------------------------------------------------------------- hvp
    // V: nv directions, row b at V + b*ldv (canonical flat order).
    void hvp(const T* params, const Cache<T>& c, const T* V, int64_t nv, int64_t ldv, T* HV, int64_t ldhv,
             T alpha) {
        const int S = md.S;
        const int64_t n = c.n;
        std::vector<DevMem> keep;
        T* rz[kMaxLayers] = {};
        T* ra[kMaxLayers] = {};
        T* rd[kMaxLayers] = {};
        for (int k = 0; k < S; ++k) {
            keep.emplace_back((size_t)nv * n * c.ldt[k] * sizeof(T), s);
            rz[k] = dptr<T>(keep.back());
            keep.emplace_back((size_t)nv * n * c.ldt[k] * sizeof(T), s);
            rd[k] = dptr<T>(keep.back());
            if (k > 0) {
                keep.emplace_back((size_t)nv * n * c.lda[k] * sizeof(T), s);
                ra[k] = dptr<T>(keep.back());
                CK_CUDA(cudaMemsetAsync(ra[k], 0, (size_t)nv * n * c.lda[k] * sizeof(T), s));
            }
        }
        // R-forward
        for (int k = 0; k < S; ++k) {
            const int64_t tin = md.w[k], tout = md.w[k + 1];
            const int64_t bsz = n * c.ldt[k];
            EpiRzBias<T> e1{rz[k], c.ldt[k], bsz, V + md.boff[k], ldv};
            gemm_simt<T>(s, n, tout, tin, nv, kmaj(c.a[k], c.lda[k], 0), kmaj(V + md.woff[k], tin, ldv), e1);
            if (k > 0) {
                EpiStore<T> e2{rz[k], c.ldt[k], bsz, T(1), T(1)};
                gemm_simt<T>(s, n, tout, tin, nv, kmaj(ra[k], c.lda[k], n * c.lda[k]),
                             kmaj(params + md.woff[k], tin, 0), e2);
            }
            if (k + 1 < S) {
                // ra_{k+1} = act'(z_k) * rz_k  (rows = nv * n)
                rop_act_kernel<T><<<blocks_for(nv * n * tout), 256, 0, s>>>(
                    rz[k], c.ldt[k], c.z[k], c.ldt[k], n, nv * n, tout, md.act, ra[k + 1], c.lda[k + 1]);
                CK_LAUNCH();
            }
        }
        // R-backward
        rop_softmax_kernel<T><<<blocks_for(nv * n, 128), 128, 0, s>>>(
            rz[S - 1], c.ldt[S - 1], c.a[S], c.lda[S], n, nv * n, md.w[S], md.mode, rd[S - 1], c.ldt[S - 1]);
        CK_LAUNCH();
        for (int k = S - 2; k >= 0; --k) {
            const int64_t t1 = md.w[k + 1], t2 = md.w[k + 2];
            // treat (direction, example) rows as one stacked operand
            EpiRback<T> e1{rd[k], c.ldt[k], c.z[k], c.up[k], c.ldt[k], rz[k], c.ldt[k], n, md.act, 0, 0, 0};
            gemm_simt<T>(s, nv * n, t1, t2, 1, kmaj(rd[k + 1], c.ldt[k + 1]), mnmaj(params + md.woff[k + 1], t1), e1);
            // + delta_{k+1} RW_{k+1}[b]  (batched over directions), then apply
            EpiRb2<T> e2{EpiRback<T>{rd[k], c.ldt[k], c.z[k], c.up[k], c.ldt[k], rz[k], c.ldt[k], n, md.act, 0, 1, 1}, 0};
            gemm_simt<T>(s, n, t1, t2, nv, kmaj(c.delta[k + 1], c.ldt[k + 1], 0),
                         mnmaj(V + md.woff[k + 1], t1, ldv), e2);
        }
        // accumulate: hv_k = sum_n rd_k (x) a_k + delta_k (x) ra_k, bias = sum_n rd_k
        for (int k = 0; k < S; ++k) {
            const int64_t tin = md.w[k], tout = md.w[k + 1];
            EpiHv<T> e1{HV, ldhv, md.woff[k], md.boff[k], tin, alpha, 0};
            gemm_simt<T>(s, tout, tin + 1, n, nv, mnmaj(rd[k], c.ldt[k], n * c.ldt[k]), mnmaj(c.a[k], c.lda[k], 0), e1);
            if (k > 0) {
                EpiHv<T> e2{HV, ldhv, md.woff[k], md.boff[k], tin, alpha, 1};
                gemm_simt<T>(s, tout, tin + 1, n, nv, mnmaj(c.delta[k], c.ldt[k], 0),
                             mnmaj(ra[k], c.lda[k], n * c.lda[k]), e2);
            }
        }
    }

    // ---------------------------------------------------------------- opg
    // Rows [rb, re) of the lower triangle and their mirrors (a row shard; the
    // full product is rb = 0, re = P).  rb must be a multiple of 4 (TMA base).
    // In TF32 mode J must have been stored rounded (jacobian(..., rn = true)).
    void opg(const T* J, int64_t ldj, int64_t n, T* G, int64_t ldg, int64_t rb = 0, int64_t re = -1) {
        if (re < 0 || re > md.P) re = md.P;
        if (rb >= re) return;
        EpiSymLower<T> e{G, ldg, T(1) / T(n), rb};
        const double entries = (double)re * (re + 1) / 2.0 - (double)rb * (rb + 1) / 2.0;
        ProfScope ps("opg_gemm", s, 2.0 * entries * (double)n,
                     (double)sizeof(T) * ((double)n * re + 2.0 * entries));
        CurvGemm<T, EpiSymLower<T>>::run(prec, s, re - rb, re, n, pre_rounded(mnmaj(J + rb, ldj)), pre_rounded(mnmaj(J, ldj)), e);
    }

    // Diagonal block of layer k by symmetric orbits in the f32 / f64 modes (the
    // TF32 modes take symkr.cuh).  prof = profiles [U][U][ldn] (H) or delta_k^T
    // [U][ldn] (OPG, delta_products).  Z = abar_i abar_c is materialised for
    // pairs in 8 x 8 (i, c) blocks, one 64-row tile per block (orbit_dmma_kernel
    // f64 / orbit_simt_kernel f32, orbit_dmma.cuh), the tile staged in shared
    // memory and written as runs of 8 for all four orbit images.  A row shard
    // takes the block range matching its share of the block's lower triangle.
    void orbit_block(int k, const T* akT, const T* prof, int delta_products, int64_t ldn, int64_t n, T* H,
                         int64_t ldh, int64_t rlo, int64_t rhi) {
        const int64_t tk = md.w[k], U = md.w[k + 1], Pk = md.block_size(k);
        const int64_t nb = ceil_div(tk + 1, 8);
        std::vector<int2> blocks, ic, oo;
        for (int64_t ib = 0; ib < nb; ++ib)
            for (int64_t cb = ib; cb < nb; ++cb) blocks.push_back(make_int2((int)ib, (int)cb));
        for (const int2& b : blocks)
            for (int il = 0; il < 8; ++il)
                for (int cl = 0; cl < 8; ++cl)  // padding rows read row T_k (masked at the store)
                    ic.push_back(make_int2((int)std::min<int64_t>(8 * b.x + il, tk), (int)std::min<int64_t>(8 * b.y + cl, tk)));
        for (int64_t o = 0; o < U; ++o)
            for (int64_t q = o; q < U; ++q) oo.push_back(make_int2((int)o, (int)q));
        const int64_t nbk = (int64_t)blocks.size(), np = (int64_t)oo.size();
        auto tri = [&](int64_t r) {
            const double j = (double)std::clamp<int64_t>(r - md.woff[k], 0, Pk);
            return j * (j + 1.0) / ((double)Pk * (Pk + 1.0));
        };
        const int64_t ba = rlo <= md.woff[k] ? 0 : std::min<int64_t>(nbk, (int64_t)(tri(rlo) * (double)nbk));
        const int64_t bb = rhi >= md.woff[k] + Pk ? nbk : std::min<int64_t>(nbk, (int64_t)(tri(rhi) * (double)nbk));
        if (ba >= bb) return;
        const int2* dblocks = static_cast<const int2*>(cached_upload(blocks.data(), blocks.size() * sizeof(int2)));
        const int2* dic = static_cast<const int2*>(cached_upload(ic.data(), ic.size() * sizeof(int2)));
        const int2* doo = static_cast<const int2*>(cached_upload(oo.data(), oo.size() * sizeof(int2)));
        DevMem pi((size_t)np * ldn * sizeof(T), s);
        orbit_pack_kernel<T><<<dim3((unsigned)ceil_div(n, 256), (unsigned)std::min<int64_t>(np, 65535)), 256, 0, s>>>(
            prof, doo, U, ldn, n, delta_products, dptr<T>(pi), np);
        CK_LAUNCH();
        // Z chunks of whole blocks (<= ~512 MB, <= 32768 rows: grid.y of orbit_z_kernel)
        const int64_t cblk = std::clamp<int64_t>((int64_t(512) << 20) / (64 * ldn * (int64_t)sizeof(T)), 1, 512);
        DevMem z((size_t)std::min(cblk, bb - ba) * 64 * ldn * sizeof(T), s);
        for (int64_t b0 = ba; b0 < bb; b0 += cblk) {
            const int64_t nbc = std::min(cblk, bb - b0);
            orbit_z_kernel<T><<<dim3((unsigned)ceil_div(n, 256), (unsigned)(64 * nbc)), 256, 0, s>>>(
                akT, ldn, dic, 64 * b0, 64 * nbc, n, dptr<T>(z));
            CK_LAUNCH();
            OrbitArgs<T> oa{dptr<T>(z), dptr<T>(pi), ldn, np, n, dblocks + b0, doo, H, ldh, md.woff[k],
                            md.boff[k], tk, T(1) / T(n)};
            if constexpr (sizeof(T) == 8)
                orbit_dmma_kernel<<<dim3((unsigned)nbc, (unsigned)ceil_div(np, 64)), 128, 0, s>>>(oa);
            else
                orbit_simt_kernel<<<dim3((unsigned)nbc, (unsigned)ceil_div(np, 64)), 128, 0, s>>>(oa);
            CK_LAUNCH();
        }
    }

    // OPG without J (TF32): G[(k,o,i),(m,o'',c)] = (1/N) sum_n abar_k,i abar_m,c
    // delta_k,o delta_m,o'' -- the per-example gradient rows are delta (x) abar
    // (autodiff.cpp:127-143).  Diagonal blocks by the symmetric Khatri-Rao
    // kernel (one value per orbit); the blocks m < k of a layer k form one
    // rectangular tensor-core GEMM over J (or, where its rows are not
    // 16-byte addressable, the fused block kernel with the profile
    // delta_k,o delta_m,o'' and no Q term).  Same row-shard contract as opg();
    // returns false where the route does not apply (then J + SYRK).
    //
    // band != null: G holds the unit band's rows (bands.cuh), TF32 only.
    bool opg_kr(const Cache<T>& c, T* G, int64_t ldg, int64_t rlo = 0, int64_t rhi = INT64_MAX,
                const UnitBand* band = nullptr) {
        const bool tc = tf32_class(prec) && sizeof(T) == 4;
        if (band && !tc) throw CurvError(kContractError, "unit-band assembly needs TF32 precision");
        if (!(tc || prec == kF32 || prec == kF64) || sym_off()) {
            if (band) throw CurvError(kContractError, "unit-band assembly needs the symmetric-orbit kernels");
            return false;
        }
        const int S = md.S;
        const int64_t n = c.n, ldn = round_up(n, 32);
        std::vector<DevMem> keep;
        // every buffer here is written in full, padding included (transposes pad
        // with zeros; replicate_rows and outer_delta copy or multiply whole rows)
        auto buf = [&](int64_t rows, int64_t ld) {
            keep.emplace_back((size_t)rows * ld * sizeof(T), s);
            return dptr<T>(keep.back());
        };
        T* akT[kMaxLayers] = {};
        T* dT[kMaxLayers] = {};
        DevMem J;  // per-example gradients (rounded to TF32), only for the blocks m < k
        int64_t ldj = 0;
        DevMem jt16, jt16inv;  // F16S: J^T in fp16 and its inverse row scales
        {
            ProfScope prep("opg_prep", s, 0.0, 0.0);
            TransposeBatch<T> tb(s);  // all layers' copies in one launch
            for (int k = 0; k < S; ++k) {
                akT[k] = buf(md.w[k] + 1, ldn);
                tb.add(c.a[k], c.lda[k], 0, akT[k], ldn, 0, n, md.w[k] + 1, 1);
                dT[k] = buf(md.w[k + 1], ldn);
                tb.add(c.delta[k], c.ldt[k], 0, dT[k], ldn, 0, n, md.w[k + 1], 1);
            }
            tb.flush();
        }
        for (int k = 0; k < S; ++k) {
            const int64_t Pk = md.block_size(k), tk = md.w[k], uk = md.w[k + 1];
            if (band ? band->u0[k] >= band->u1[k] : (md.woff[k] + Pk <= rlo || md.woff[k] >= rhi)) continue;
            {
                // packed unit pairs (o <= o'') computed: all, or o'' in the band
                const int64_t v0 = band ? band->u0[k] : 0, v1 = band ? band->u1[k] : uk;
                const double pairs = ((double)v1 * (v1 + 1) - (double)v0 * (v0 + 1)) / 2.0;
                const double orbits = pairs * (double)(tk + 1) * (tk + 2) / 2.0;
                const double stored = band ? (double)(v1 - v0) * (tk + 1) * (double)(md.woff[k] + (v1) * (tk + 1))
                                           : (double)Pk * Pk;
                ProfScope ps("opg_symkr", s, 2.0 * (double)n * orbits, (double)sizeof(T) * stored);
                if (tc) {
                    SymKrArgs<T> sa{akT[k], dT[k], 1, ldn, n, tk, uk, G, ldg, md.woff[k], md.boff[k], T(1) / T(n)};
                    if (band) {
                        sa.u0 = band->u0[k];
                        sa.u1 = band->u1[k];
                        sa.bwoff = band->bw[k];
                        sa.bboff = band->bb[k];
                    } else {
                        sa.pair_q0 = pair_q0;
                        sa.pair_q1 = pair_q1;
                    }
                    if (!SymKr<T>::run(prec, s, sa)) throw CurvError(kCudaError, "opg_kr: diagonal block kernel unavailable");
                } else {
                    orbit_block(k, akT[k], dT[k], 1, ldn, n, G, ldg, rlo, rhi);
                }
            }
            if (k == 0) continue;
            // blocks m < k: rectangular GEMMs G[rows of k, columns of layers < k] =
            // (1/N) J_k^T J_<k on the tensor cores (the SYRK engine), mirrored; a band
            // stores its weight rows and its bias rows (two ranges), unmirrored
            struct Rows {
                int64_t r0, r1, b;  // global rows [r0, r1) stored from band row b (-1: in place)
            };
            std::vector<Rows> rows;
            if (band) {
                rows.push_back({md.woff[k] + band->u0[k] * tk, md.woff[k] + band->u1[k] * tk, band->bw[k]});
                rows.push_back({md.boff[k] + band->u0[k], md.boff[k] + band->u1[k], band->bb[k]});
            } else {
                rows.push_back({std::max(rlo, md.woff[k]), std::min(rhi, md.woff[k] + Pk), -1});
            }
            T* akX = nullptr;
            for (const Rows& rr : rows) {
                const int64_t r0 = rr.r0, r1 = rr.r1;
                if (r0 >= r1) continue;
                // F16S: the whole-block rectangle on the fp16 datapath (J^T in fp16, built once)
                if (prec == kF16S && !band && r1 - r0 >= 512 && md.woff[k] > 64) {
                    if (!jt16.p) {
                        JtF16Args ja{};
                        ja.S = md.S;
                        for (int q = 0; q < md.S; ++q) {
                            ja.akT[q] = reinterpret_cast<const float*>(akT[q]);
                            ja.dT[q] = reinterpret_cast<const float*>(dT[q]);
                            ja.woff[q] = md.woff[q];
                            ja.boff[q] = md.boff[q];
                        }
                        for (int q = 0; q <= md.S; ++q) ja.w[q] = md.w[q];
                        ja.P = md.P;
                        ja.n = n;
                        ja.ldn = ldn;
                        ProfScope pj("opg_jt16", s, 0.0, 2.0 * (double)md.P * ldn);
                        if (!OpgF16<T>::build(s, ja, jt16, jt16inv)) jt16 = DevMem();
                    }
                    if (jt16.p) {
                        ProfScope ps("opg_gemm", s, 2.0 * (double)(r1 - r0) * md.woff[k] * n,
                                     (double)sizeof(T) * 2.0 * (double)(r1 - r0) * md.woff[k]);
                        OpgF16<T>::rect(s, r0, r1, md.woff[k], n, jt16, ldn, jt16inv, G, ldg, T(1) / T(n));
                        continue;
                    }
                }
                if (r0 % 4 == 0 || !tc) {
                    if (!J.p) {  // (jacobian() times itself as "jacobian")
                        ldj = round_up(md.P, 32);
                        J = DevMem((size_t)n * ldj * sizeof(T), s);
                        jacobian<T>(md, c, 0, n, dptr<T>(J), ldj, s, tc);
                    }
                    ProfScope ps("opg_gemm", s, 2.0 * (double)(r1 - r0) * md.woff[k] * n,
                                 (double)sizeof(T) * (band ? 1.0 : 2.0) * (double)(r1 - r0) * md.woff[k]);
                    auto opj = [&](const T* p) { return tc ? pre_rounded(mnmaj(p, ldj)) : mnmaj(p, ldj); };
                    if constexpr (sizeof(T) == 4) {
                        if (band) {
                            gemm_tf32_store(prec, s, r1 - r0, md.woff[k], n, opj(dptr<T>(J) + r0), opj(dptr<T>(J)),
                                            G + rr.b * ldg, ldg, T(1) / T(n));
                            continue;
                        }
                    }
                    EpiSymLower<T> e{G, ldg, T(1) / T(n), r0};
                    CurvGemm<T, EpiSymLower<T>>::run(prec, s, r1 - r0, md.woff[k], n, opj(dptr<T>(J) + r0), opj(dptr<T>(J)), e);
                    continue;
                }
                const int64_t ak_rows = tk + 256;
                if (!akX) {
                    akX = buf(ak_rows, ldn);
                    replicate_rows_kernel<T><<<dim3(blocks_for(ak_rows * ldn), 1), 256, 0, s>>>(akT[k], tk, ldn, akX,
                                                                                                ak_rows, 0, 0);
                    CK_LAUNCH();
                }
                for (int m = k - 1; m >= 0; --m) {
                    const int64_t tm = md.w[m], um = md.w[m + 1];
                    T* pv = buf(uk * um, ldn);
                    outer_delta_kernel<T><<<dim3((unsigned)ceil_div(ldn, 256), (unsigned)um, (unsigned)uk), 256, 0, s>>>(
                        dT[k], dT[m], um, ldn, pv);
                    CK_LAUNCH();
                    HessFusedArgs<T> fa{akX, ak_rows, nullptr, ak_rows, um * ak_rows, pv, dT[k], c.a[m], c.lda[m], ldn,
                                        n, tk, tm, um, uk * tk, 0, Pk};
                    EpiHess<T> e{G, ldg, Pk, 0, md.woff[k], md.woff[m], md.boff[m], tm, T(1) / T(n), 0, band ? 0 : 1,
                                 band ? r0 : rlo, band ? r1 : rhi, band ? r0 - rr.b : 0};
                    const double req = (double)(r1 - r0) * um * (tm + 1);
                    ProfScope ps("opg_fused", s, 2.0 * (double)n * req, (double)sizeof(T) * (band ? 1.0 : 2.0) * req);
                    if (!HessFused<T>::run(prec, s, fa, e)) throw CurvError(kCudaError, "opg_kr: block kernel unavailable");
                }
            }
        }
        return true;
    }

    // ---------------------------------------------------------------- hessian
    // Profiles for tangent step k (see file comment):
    //   G  [T_{k+1}][n][ldt_k]       rdelta_k for rz_k = e_o
    //   Pm [T_{k+1}][n][ldt_m]       rdelta_m, m < k, same tangents
    //   Qm [T_k][n][ldt_m]           rdelta_m from the explicit delta*RW term
    size_t chunk_bytes = size_t(256) << 20;  // R operand chunk (streamed once from HBM)
    // dev control: CURVKIT_NO_SYMKR=1 keeps diagonal blocks on the lower-triangle kernels
    static bool sym_off() {
        static const bool off = getenv("CURVKIT_NO_SYMKR") != nullptr;
        return off;
    }

    // Output entries of one (k, m, chunk) block that the assembly needs: all
    // of an off-diagonal block, the lower triangle (gc <= gr) of a diagonal one.
    double hess_required_entries(int k, int m, int64_t j0, int64_t Jc) const {
        const int64_t tm = md.w[m], tm1 = md.w[m + 1];
        if (m != k) return (double)Jc * tm1 * (tm + 1);
        // row j of the block needs clamp(j - o*tm + 1, 0, tm) weight columns of
        // band o and the bias column when j >= tm*tm1 + o: closed-form sums
        auto S = [tm](int64_t x, int64_t a) -> double {  // sum_{j<x} clamp(j - a + 1, 0, tm)
            if (x <= a) return 0.0;
            const double r = (double)std::min(x - a, tm);
            return r * (r + 1.0) / 2.0 + (double)std::max<int64_t>(0, x - a - tm) * (double)tm;
        };
        const int64_t j1 = j0 + Jc, bias0 = md.boff[m] - md.woff[m];
        double cnt = 0.0;
        for (int64_t o = 0; o < tm1; ++o) {
            cnt += S(j1, o * tm) - S(j0, o * tm);
            cnt += (double)std::max<int64_t>(0, j1 - std::max(j0, bias0 + o));
        }
        return cnt;
    }

    // Tangent rows [rlo, rhi) of H (their lower entries and mirrors); the full
    // assembly is rlo = 0, rhi = P.  Layers with no owned row are skipped.
    // band != null: H holds the unit band's rows (bands.cuh), TF32 only.
    void hessian(const T* params, const Cache<T>& c, T* H, int64_t ldh, bool verify, int64_t rlo = 0,
                 int64_t rhi = INT64_MAX, const UnitBand* band = nullptr) {
        const int S = md.S;
        const int64_t n = c.n;
        if (band && (!tf32_class(prec) || sizeof(T) != 4 || verify || sym_off()))
            throw CurvError(kContractError, "unit-band assembly needs TF32 precision");
        for (int k = 0; k < S; ++k) {
            const int64_t np = md.w[k + 1];
            if (band ? band->u0[k] >= band->u1[k] : (md.woff[k] + md.block_size(k) <= rlo || md.woff[k] >= rhi))
                continue;
            std::vector<DevMem> keep;
            // R-op profile buffers: every kernel below writes its output's logical
            // extent and reads only logical extents (checked with CURVKIT_POISON)
            auto buf = [&](int64_t rows, int64_t ld) {
                keep.emplace_back((size_t)rows * ld * sizeof(T), s);
                return dptr<T>(keep.back());
            };
            // for the n-contiguous copies below: transpose, replicate_rows and qext
            // write every element of their rows, the padding included (zeros)
            auto buf_full = [&](int64_t rows, int64_t ld) {
                keep.emplace_back((size_t)rows * ld * sizeof(T), s);
                return dptr<T>(keep.back());
            };
            // Unit bands run the R-op only for the tangents of their own units
            // [t0, t1): P[o][.] and PV[o][.] are needed for the rows of unit o alone
            // (the symmetric kernel reads PV[o''][o] for its packed columns o <= o'',
            // o'' in the band); Q_m does not depend on the row's unit.
            static const bool fused_env = getenv("CURVKIT_HESS_FUSED") != nullptr;
            const bool band_rgen = band && !fused_env;
            const int64_t t0 = band_rgen ? band->u0[k] : 0, nt = band_rgen ? band->u1[k] - band->u0[k] : np;
            ProfScope prof_stage("hess_profiles", s, 0.0, 0.0);
            T* G = buf(nt * n, c.ldt[k]);
            T* rzp[kMaxLayers] = {};
            if (k == S - 1) {
                profile_output_kernel<T><<<blocks_for(nt * n * np), 256, 0, s>>>(c.a[S], c.lda[S], np, n, md.mode, G,
                                                                                  c.ldt[k], t0, nt);
                CK_LAUNCH();
            } else {
                // R-forward above the tangent layer
                rzp[k + 1] = buf(nt * n, c.ldt[k + 1]);
                profile_first_rz_kernel<T><<<blocks_for(nt * n * md.w[k + 2]), 256, 0, s>>>(
                    c.z[k], c.ldt[k], params + md.woff[k + 1], md.w[k + 1], md.w[k + 2], n, md.act, rzp[k + 1],
                    c.ldt[k + 1], t0, nt);
                CK_LAUNCH();
                for (int kp = k + 1; kp + 1 < S; ++kp) {
                    T* ra = buf(nt * n, c.lda[kp + 1]);
                    rop_act_kernel<T><<<blocks_for(nt * n * md.w[kp + 1]), 256, 0, s>>>(
                        rzp[kp], c.ldt[kp], c.z[kp], c.ldt[kp], n, nt * n, md.w[kp + 1], md.act, ra, c.lda[kp + 1]);
                    CK_LAUNCH();
                    rzp[kp + 1] = buf(nt * n, c.ldt[kp + 1]);
                    EpiStore<T> e{rzp[kp + 1], c.ldt[kp + 1], 0, T(1), T(0)};
                    gemm_simt<T>(s, nt * n, md.w[kp + 2], md.w[kp + 1], 1, kmaj(ra, c.lda[kp + 1]),
                                 kmaj(params + md.woff[kp + 1], md.w[kp + 1]), e);
                }
                // R-backward down to the tangent layer
                T* rdn = buf(nt * n, c.ldt[S - 1]);
                rop_softmax_kernel<T><<<blocks_for(nt * n, 128), 128, 0, s>>>(
                    rzp[S - 1], c.ldt[S - 1], c.a[S], c.lda[S], n, nt * n, md.w[S], md.mode, rdn, c.ldt[S - 1]);
                CK_LAUNCH();
                for (int kp = S - 2; kp >= k; --kp) {
                    T* out = kp == k ? G : buf(nt * n, c.ldt[kp]);
                    EpiRback<T> e{out, c.ldt[kp], c.z[kp], c.up[kp], c.ldt[kp], rzp[kp], c.ldt[kp], n, md.act,
                                  kp == k ? 1 : 0, 1, 0, t0};
                    gemm_simt<T>(s, nt * n, md.w[kp + 1], md.w[kp + 2], 1, kmaj(rdn, c.ldt[kp + 1]),
                                 mnmaj(params + md.woff[kp + 1], md.w[kp + 1]), e);
                    rdn = out;
                }
            }
            // P and Q profiles below the tangent layer
            T* Pm[kMaxLayers] = {};
            T* Qm[kMaxLayers] = {};
            if (k > 0) {
                const int64_t nq = md.w[k];
                T* prevP = G;
                for (int m = k - 1; m >= 0; --m) {
                    Pm[m] = buf(nt * n, c.ldt[m]);
                    EpiRback<T> e{Pm[m], c.ldt[m], c.z[m], nullptr, c.ldt[m], nullptr, 0, n, md.act, 0, 1, 0};
                    gemm_simt<T>(s, nt * n, md.w[m + 1], md.w[m + 2], 1, kmaj(prevP, c.ldt[m + 1]),
                                 mnmaj(params + md.woff[m + 1], md.w[m + 1]), e);
                    prevP = Pm[m];
                }
                Qm[k - 1] = buf(nq * n, c.ldt[k - 1]);
                profile_q_kernel<T><<<blocks_for(nq * n * nq), 256, 0, s>>>(c.z[k - 1], c.ldt[k - 1], nq, n, md.act,
                                                                             Qm[k - 1], c.ldt[k - 1]);
                CK_LAUNCH();
                for (int m = k - 2; m >= 0; --m) {
                    Qm[m] = buf(nq * n, c.ldt[m]);
                    EpiRback<T> e{Qm[m], c.ldt[m], c.z[m], nullptr, c.ldt[m], nullptr, 0, n, md.act, 0, 1, 0};
                    gemm_simt<T>(s, nq * n, md.w[m + 1], md.w[m + 2], 1, kmaj(Qm[m + 1], c.ldt[m + 1]),
                                 mnmaj(params + md.woff[m + 1], md.w[m + 1]), e);
                }
            }
            prof_stage.end();
            ProfScope prep_stage("hess_prep", s, 0.0, 0.0);
            TransposeBatch<T> tb(s);  // the copies below in one launch
            // n-contiguous copies for the R generator (all reads 16-byte vectors);
            // a 32-multiple pitch keeps every K-block of 32 examples inside a row
            const int64_t ldn = round_up(n, 32);
            const int64_t tk = md.w[k];
            T* akT = buf_full(tk + 1, ldn);
            tb.add(c.a[k], c.lda[k], 0, akT, ldn, 0, n, tk + 1, 1);
            T* dkT = buf_full(np, ldn);
            tb.add(c.delta[k], c.ldt[k], 0, dkT, ldn, 0, n, np, 1);
            T* GT = buf_full(nt * np, ldn);
            tb.add(G, c.ldt[k], n * c.ldt[k], GT, ldn, np * ldn, n, np, nt);
            T* PT[kMaxLayers] = {};
            T* QT[kMaxLayers] = {};
            for (int m = k - 1; m >= 0; --m) {
                const int64_t tm1 = md.w[m + 1];
                PT[m] = buf_full(nt * tm1, ldn);
                tb.add(Pm[m], c.ldt[m], n * c.ldt[m], PT[m], ldn, tm1 * ldn, n, tm1, nt);
                QT[m] = buf_full(tk * tm1, ldn);
                tb.add(Qm[m], c.ldt[m], n * c.ldt[m], QT[m], ldn, tm1 * ldn, n, tm1, tk);
            }
            tb.flush();
            // Extended copies for the fused TF32 kernel: a 128-row activation
            // tile starting anywhere in [0, T_k) reads rows r -> r mod T_k.
            const bool fused = tf32_class(prec) && sizeof(T) == 4;
            const int64_t ak_rows = tk + 256;
            T* akX = nullptr;
            T* QX[kMaxLayers] = {};
            // built before the block loop when a fused block is certain (m < k, or a
            // diagonal block without the symmetric kernel), else on first use
            auto build_ext = [&]() {
                akX = buf_full(ak_rows, ldn);
                replicate_rows_kernel<T><<<dim3(blocks_for(ak_rows * ldn), 1), 256, 0, s>>>(akT, tk, ldn, akX, ak_rows, 0, 0);
                CK_LAUNCH();
                for (int m = k - 1; m >= 0; --m) {
                    const int64_t tm1 = md.w[m + 1];
                    QX[m] = buf_full(tm1 * ak_rows, ldn);
                    // QT[m] is [i][o''][n]; QX[m] is [o''][r][n] with r -> i = r mod T_k
                    qext_kernel<T><<<dim3(blocks_for(ak_rows * ldn / 4), (unsigned)tm1), 256, 0, s>>>(
                        QT[m], tk, tm1, ldn, QX[m], ak_rows);
                    CK_LAUNCH();
                }
            };
            // (blocks m < k take R in HBM unless CURVKIT_HESS_FUSED, below)
            if (fused && ((k > 0 && fused_env) || verify || sym_off())) build_ext();
            prep_stage.end();
            // blocks (k, m), m <= k
            const int64_t Pk = md.block_size(k);
            const int64_t nw = md.w[k + 1] * tk;
            const int64_t ldr = ldn;
            for (int m = k; m >= 0; --m) {
                // weight tangents through the fused kernel where it exists; the
                // chunked R path below then only covers the bias tangents
                int64_t jbeg = 0;
                if (fused && m == k && !verify && !sym_off()) {
                    // diagonal block: one value per symmetric orbit (a row shard takes
                    // its share of the block's lower triangle as a range of orbit tiles)
                    const int64_t v0 = band ? band->u0[k] : 0, v1 = band ? band->u1[k] : np;
                    const double f = ((double)v1 * (v1 + 1) - (double)v0 * (v0 + 1)) / ((double)np * (np + 1));
                    const double orbits = (double)np * (np + 1) / 2.0 * (double)(tk + 1) * (tk + 2) / 2.0;
                    ProfScope ps("hess_symkr", s, 2.0 * (double)n * orbits * f, (double)sizeof(T) * (double)Pk * Pk * f);
                    SymKrArgs<T> sa{akT, GT, 0, ldn, n, tk, np, H, ldh, md.woff[k], md.boff[k], T(1) / T(n)};
                    if (band) {
                        sa.u0 = v0;
                        sa.u1 = v1;
                        sa.bwoff = band->bw[k];
                        sa.bboff = band->bb[k];
                        if (band_rgen) sa.prof_t0 = t0;
                    }
                    if (SymKr<T>::run(prec, s, sa)) jbeg = Pk;
                    else if (band) throw CurvError(kCudaError, "hessian: diagonal block kernel unavailable");
                }
                if (!fused && (prec == kF32 || prec == kF64) && m == k && !verify && !sym_off()) {
                    const double orbits = (double)np * (np + 1) / 2.0 * (double)(tk + 1) * (tk + 2) / 2.0;
                    ProfScope ps("hess_orbit", s, 2.0 * (double)n * orbits, (double)sizeof(T) * (double)Pk * Pk);
                    orbit_block(k, akT, GT, 0, ldn, n, H, ldh, rlo, rhi);
                    jbeg = Pk;
                }
                // Blocks m < k (TF32 class, whole blocks): R generated into HBM in 2 GB
                // chunks (rounded to TF32, write-bound) and the pair GEMM (~570 TF/s)
                // instead of the fused kernel, whose k-block pipeline runs at ~0.34 of
                // the TF32 peak for reasons DESIGN.md section 4 did not isolate (c2:
                // 7.2 -> 5.2 ms), unit bands included (the chunks then cover the band's
                // weight and bias tangent rows).  CURVKIT_HESS_FUSED=1 selects the
                // fused kernel everywhere.
                const bool rgen_tc = fused && !fused_env && m < k;
                if (band && m == k) continue;  // the symmetric kernel wrote the band's diagonal block
                if (fused && jbeg < Pk && !rgen_tc) {
                    if (!akX) build_ext();
                    const int64_t tm = md.w[m], tm1 = md.w[m + 1];
                    HessFusedArgs<T> fa{akX, ak_rows, m == k ? nullptr : QX[m], ak_rows, tm1 * ak_rows,
                                        m == k ? GT : PT[m], dkT, c.a[m], c.lda[m], ldn, n, tk, tm, tm1, nw,
                                        (m == k && !verify) ? 1 : 0, Pk};
                    if (band) {  // m < k: the band's weight rows, then its bias rows, unmirrored
                        const int64_t u0 = band->u0[k], u1 = band->u1[k];
                        const int64_t rg[2][3] = {{md.woff[k] + u0 * tk, md.woff[k] + u1 * tk, band->bw[k]},
                                                  {md.boff[k] + u0, md.boff[k] + u1, band->bb[k]}};
                        for (const auto& g : rg) {
                            EpiHess<T> e{H, ldh, Pk, 0, md.woff[k], md.woff[m], md.boff[m], tm, T(1) / T(n), 0, 0,
                                         g[0], g[1], g[0] - g[2]};
                            const double req = (double)(g[1] - g[0]) * tm1 * (tm + 1);
                            ProfScope ps("hess_fused", s, 2.0 * (double)n * req, (double)sizeof(T) * req);
                            if (!HessFused<T>::run(prec, s, fa, e)) throw CurvError(kCudaError, "hessian: block kernel unavailable");
                        }
                        continue;
                    }
                    EpiHess<T> e{H, ldh, Pk, 0, md.woff[k], md.woff[m], md.boff[m], tm, T(1) / T(n),
                                 m == k ? 1 : 0, (m == k && verify) ? 0 : 1, rlo, rhi};
                    const int64_t js = std::clamp<int64_t>(rlo - md.woff[k], 0, Pk);
                    const int64_t je = std::clamp<int64_t>(rhi - md.woff[k], 0, Pk);
                    const double req = Profiler::get().on ? hess_required_entries(k, m, js, je - js) : 0.0;
                    ProfScope ps("hess_fused", s, 2.0 * (double)n * req, (double)sizeof(T) * req);
                    if (HessFused<T>::run(prec, s, fa, e)) jbeg = Pk;
                }
                const int64_t tm = md.w[m], tm1 = md.w[m + 1];
                // F16S: the same chunks with R in fp16 and the fp16 GEMM
                typename HessF16<T>::Prep hp;
                HessF16Args ha{};
                bool f16r = false;
                if (rgen_tc && !band && prec == kF16S && tm + 1 > 64 && jbeg < Pk) {
                    ha = HessF16Args{reinterpret_cast<const float*>(PT[m]), reinterpret_cast<const float*>(QT[m]),
                                     reinterpret_cast<const float*>(akT), reinterpret_cast<const float*>(dkT),
                                     reinterpret_cast<const float*>(c.a[m]), c.lda[m], ldn, n, tk, np, tm, tm1};
                    ProfScope pp("hess_prep16", s, 0.0, 0.0);
                    f16r = HessF16<T>::prepare(s, ha, hp);
                }
                // tangent-row ranges of block k to generate: everything left (whole
                // assembly), or the band's weight rows and bias rows, stored at the
                // band's row offsets without mirrors
                struct JRange { int64_t lo, hi, rlo, rhi, rsh; };
                std::vector<JRange> ranges;
                if (band) {
                    const int64_t u0 = band->u0[k], u1 = band->u1[k];
                    ranges.push_back({u0 * tk, u1 * tk, md.woff[k] + u0 * tk, md.woff[k] + u1 * tk,
                                      md.woff[k] + u0 * tk - band->bw[k]});
                    ranges.push_back({nw + u0, nw + u1, md.boff[k] + u0, md.boff[k] + u1, md.boff[k] + u0 - band->bb[k]});
                } else {
                    ranges.push_back({jbeg, Pk, rlo, rhi, 0});
                }
                int64_t span = 0;
                for (const JRange& r : ranges) span = std::max(span, r.hi - r.lo);
                int64_t J = (int64_t)((rgen_tc ? size_t(2) << 30 : chunk_bytes) / ((size_t)tm1 * ldr * sizeof(T)));
                J = std::max<int64_t>(128, J / 128 * 128);
                J = std::min<int64_t>(J, round_up(span, 128));
                DevMem rbuf(span > 0 ? (size_t)tm1 * J * ldr * sizeof(T) : 0, s);
                for (const JRange& jr : ranges)
                for (int64_t j0 = jr.lo; j0 < jr.hi; j0 += J) {
                    const int64_t Jc = std::min<int64_t>(J, jr.hi - j0);
                    const int64_t rlo = jr.rlo, rhi = jr.rhi;
                    const int mirror = band ? 0 : ((m == k && verify) ? 0 : 1);
                    if (md.woff[k] + j0 + Jc <= rlo || md.woff[k] + j0 >= rhi) continue;  // no owned row
                    // R rows (o'', jj) whose block entries are all above the
                    // diagonal are neither generated nor multiplied
                    int64_t opp_hi = tm1;
                    if (m == k && !verify && j0 + Jc - 1 < tm * tm1) opp_hi = std::min(tm1, (j0 + Jc - 1) / tm + 1);
                    const int64_t rows = opp_hi * Jc;
                    if (f16r && rows >= 512) {
                        EpiHess<T> e{H, ldh, Jc, j0, md.woff[k], md.woff[m], md.boff[m], tm, T(1) / T(n),
                                     m == k ? 1 : 0, mirror, rlo, rhi, jr.rsh};
                        const double req = Profiler::get().on ? hess_required_entries(k, m, j0, Jc) : 0.0;
                        DevMem r16, rinv;
                        HessF16<T>::chunk(s, ha, hp, j0, Jc, opp_hi, r16, rinv, e, req);
                        continue;
                    }
                    RGenArgs<T> g{m == k ? GT : PT[m], m == k ? nullptr : QT[m], akT, dkT, ldn, n, tk, np, tm1,
                                  j0, Jc, rows, dptr<T>(rbuf), ldr, rgen_tc ? 1 : 0, t0};
                    {
                        ProfScope ps("hess_rgen", s, 0.0, (double)sizeof(T) * rows * ldr);
                        const dim3 grid((unsigned)ceil_div(ldr / 4, 256),
                                        (unsigned)std::min<int64_t>(opp_hi * ceil_div(Jc, RGEN_SEG), 65535));
                        rgen_kernel<T><<<grid, 256, 0, s>>>(g);
                        CK_LAUNCH();
                    }
                    EpiHess<T> e{H, ldh, Jc, j0, md.woff[k], md.woff[m], md.boff[m], tm, T(1) / T(n),
                                 m == k ? 1 : 0, mirror, rlo, rhi, jr.rsh};
                    // algorithmic work is counted only while profiling (host loop)
                    const double req = Profiler::get().on ? hess_required_entries(k, m, j0, Jc) : 0.0;
                    ProfScope ps("hess_gemm", s, 2.0 * (double)n * req, (double)sizeof(T) * ((double)rows * ldr + req));
                    Opnd<T> ra = kmaj(dptr<T>(rbuf), ldr);
                    if (rgen_tc) ra = pre_rounded(ra);
                    CurvGemm<T, EpiHess<T>>::run(prec, s, rows, tm + 1, n, ra, mnmaj(c.a[m], c.lda[m]), e);
                }
            }
        }
    }
};

// ---- verify mode: asymmetry of the diagonal layer blocks, then symmetrize --
template <class T>
__global__ void symmetrize_block_kernel(T* H, int64_t ldh, int64_t off, int64_t size, unsigned long long* asym_bits) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= size * size) return;
    const int64_t i = idx / size, j = idx % size;
    if (j <= i) return;
    T* a = H + (off + i) * ldh + off + j;
    T* b = H + (off + j) * ldh + off + i;
    const double d = fabs((double)*a - (double)*b);
    atomicMax(asym_bits, (unsigned long long)__double_as_longlong(d));
    const T avg = T(0.5) * (*a + *b);
    *a = avg;
    *b = avg;
}

template <class T>
__global__ void absmax_kernel(const T* H, int64_t ldh, int64_t rows, int64_t cols, unsigned long long* bits) {
    double m = 0.0;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < rows * cols;
         idx += (int64_t)gridDim.x * blockDim.x) {
        m = fmax(m, fabs((double)H[(idx / cols) * ldh + idx % cols]));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(bits, (unsigned long long)__double_as_longlong(m));
}

}  // namespace ck
