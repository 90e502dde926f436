// model.cuh -- device-side forward/backward cache, per-example Jacobian,
// Pearlmutter R-op (HVP) and the basis-tangent Hessian factorization.
//
// Reference behaviour followed:
//   forward_backward      autodiff.cpp:53-103
//   per_example_grad_rows autodiff.cpp:127-143
//   hvp_from_cache        autodiff.cpp:158-244
//   assemble_hessian      curvature.cpp:33-92 (columns = HVPs on e_p)
//
// Layout in HBM (row-major everywhere, n = example index):
//   a[k]     n x lda[k]  activations entering step k; column T_k holds 1.0
//            so a GEMM against a[k] yields weight and bias sums together
//   z/delta/up[k]  n x ldt[k]  (ldt = round_up(T_{k+1}, 4))
//   profiles [p][n][t]  one n x ldt slab per tangent profile p, contiguous,
//            so a stack of profiles is a plain (p*n) x ldt GEMM operand.
#pragma once

#include "common.cuh"
#include "gemm_simt.cuh"
#include "prof.cuh"

namespace ck {

// ---------------------------------------------------------------------------
// device buffers (stream-ordered pool allocations)
// ---------------------------------------------------------------------------
struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    DevMem() = default;
    DevMem(size_t b, cudaStream_t st) : bytes(b), s(st) {
        if (b) CK_CUDA(cudaMallocAsync(&p, b, st));
        // dev check (CURVKIT_POISON=1): new buffers start as NaN bytes, so a read of
        // anything no kernel or memset wrote shows up in the parity tests
        static const bool poison = getenv("CURVKIT_POISON") != nullptr;
        if (b && poison) CK_CUDA(cudaMemsetAsync(p, 0xFF, b, st));
    }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    DevMem(DevMem&& o) noexcept { *this = std::move(o); }
    DevMem& operator=(DevMem&& o) noexcept {
        release();
        p = o.p; bytes = o.bytes; s = o.s;
        o.p = nullptr; o.bytes = 0;
        return *this;
    }
    ~DevMem() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
    }
};

template <class T>
inline T* dptr(const DevMem& m) { return static_cast<T*>(m.p); }

template <class T>
struct Cache {
    int64_t n = 0;
    T* a[kMaxLayers] = {};
    int64_t lda[kMaxLayers] = {};
    T* z[kMaxLayers] = {};
    T* delta[kMaxLayers] = {};
    T* up[kMaxLayers] = {};
    int64_t ldt[kMaxLayers] = {};
    DevMem mem;
};

// ---------------------------------------------------------------------------
// forward / backward
// ---------------------------------------------------------------------------
template <class Tin, class T>
__global__ void pack_input_kernel(const Tin* __restrict__ x, int64_t n, int64_t t0, T* __restrict__ a,
                                  int64_t lda) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * lda) return;
    const int64_t r = idx / lda, c = idx % lda;
    a[idx] = c < t0 ? (T)x[r * t0 + c] : (c == t0 ? T(1) : T(0));
}

// z = a W^T + b ; hidden: a_next = act(z) (+ ones column)
template <class T>
struct EpiForward {
    const T* bias;
    T* z;
    int64_t ldz;
    T* anext;  // nullptr for the output step
    int64_t ldan, tout;
    int act;
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int, int64_t m, int64_t c, T acc) const {
        const T v = acc + bias[c];
        z[m * ldz + c] = v;
        if (anext) {
            anext[m * ldan + c] = act_value<T>(act, v);
            if (c == 0) anext[m * ldan + tout] = T(1);
        }
    }
};

// softmax output + delta = p - y (autodiff.cpp:34-49, 85-90)
template <class T>
__global__ void output_layer_kernel(const T* __restrict__ z, int64_t ldz, const int32_t* __restrict__ labels,
                                    int64_t n, int64_t tl, int mode, T* __restrict__ prob, int64_t ldp,
                                    T* __restrict__ delta) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    const T* zr = z + r * ldz;
    T* pr = prob + r * ldp;
    T* dr = delta + r * ldz;
    if (mode == kRawMean) {
        for (int64_t m = 0; m < tl; ++m) { pr[m] = zr[m]; dr[m] = T(1); }
        return;
    }
    T zmax = zr[0];
    for (int64_t m = 1; m < tl; ++m) zmax = zr[m] > zmax ? zr[m] : zmax;
    T sum = T(0);
    for (int64_t m = 0; m < tl; ++m) { const T e = d_exp(zr[m] - zmax); pr[m] = e; sum += e; }
    const int32_t y = labels[r];
    for (int64_t m = 0; m < tl; ++m) {
        const T p = pr[m] / sum;
        pr[m] = p;
        dr[m] = p - (m == y ? T(1) : T(0));
    }
}

// up = delta_{k+1} W_{k+1};  delta_k = up * act'(z_k)
template <class T>
struct EpiBackward {
    const T* z;
    T* up;
    T* delta;
    int64_t ld;
    int act;
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int, int64_t m, int64_t c, T acc) const {
        up[m * ld + c] = acc;
        delta[m * ld + c] = acc * act_deriv<T>(act, z[m * ld + c]);
    }
};

template <class T>
void alloc_cache(const ModelDesc& md, int64_t n, Cache<T>& c, cudaStream_t s) {
    c.n = n;
    size_t total = 0;
    for (int k = 0; k <= md.S; ++k) {
        c.lda[k] = round_up(md.w[k] + 1, 32);
        total += (size_t)n * c.lda[k];
    }
    for (int k = 0; k < md.S; ++k) {
        c.ldt[k] = round_up(md.w[k + 1], 4);
        total += 3 * (size_t)n * c.ldt[k];
    }
    c.mem = DevMem(total * sizeof(T), s);
    T* p = dptr<T>(c.mem);
    for (int k = 0; k <= md.S; ++k) { c.a[k] = p; p += n * c.lda[k]; }
    for (int k = 0; k < md.S; ++k) {
        c.z[k] = p; p += n * c.ldt[k];
        c.delta[k] = p; p += n * c.ldt[k];
        c.up[k] = p; p += n * c.ldt[k];
    }
    CK_CUDA(cudaMemsetAsync(c.mem.p, 0, total * sizeof(T), s));
}

// Dense GEMM dispatcher used by the small model GEMMs: SIMT in every mode
// (their cost is O(N * P) against the O(N * P^2) curvature products).
// Split-K partial sums: split z writes its own M x N slab (deterministic;
// the slabs are summed in a fixed order by finalize_kernel).
template <class T>
struct EpiPartial {
    T* ws;
    int64_t ld, slab;
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int z, int64_t m, int64_t n, T acc) const { ws[z * slab + m * ld + n] = acc; }
};

template <class T, class Epi>
__global__ void finalize_kernel(const T* __restrict__ ws, int64_t splits, int64_t M, int64_t N, Epi epi) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M * N) return;
    T acc = T(0);
    for (int64_t z = 0; z < splits; ++z) acc += ws[z * M * N + i];
    epi(0, i / N, i % N, acc);
}

// Tall-K, narrow-output layer GEMMs (e.g. 1000 x 32 x 784) give the 64 x 64
// tile grid only a few CTAs: split K across grid.z so all SMs stream the
// operands, then apply the layer epilogue in one elementwise pass.
template <class T, class Epi>
void model_gemm(cudaStream_t s, int64_t M, int64_t N, int64_t K, Opnd<T> A, Opnd<T> B, const Epi& e) {
    const int64_t tiles = ceil_div(M, 64) * ceil_div(N, 64);
    int64_t splits = std::min<int64_t>(ceil_div(2 * 148, tiles), K / 32);
    if (splits < 2) {
        gemm_simt<T>(s, M, N, K, 1, A, B, e);
        return;
    }
    const int64_t kc = round_up(ceil_div(K, splits), 16);
    splits = ceil_div(K, kc);
    DevMem ws((size_t)splits * M * N * sizeof(T), s);
    EpiPartial<T> ep{dptr<T>(ws), N, M * N};
    gemm_simt<T>(s, M, N, K, 1, A, B, ep, kc);
    finalize_kernel<T, Epi><<<(unsigned)ceil_div(M * N, 256), 256, 0, s>>>(dptr<T>(ws), splits, M, N, e);
    CK_LAUNCH();
}

template <class T>
void forward_backward(const ModelDesc& md, const T* params, const int32_t* labels, Cache<T>& c,
                      cudaStream_t s) {
    const int S = md.S;
    const int64_t n = c.n;
    double fl = 0.0;
    for (int k = 0; k < S; ++k) fl += 4.0 * n * md.w[k] * md.w[k + 1];
    ProfScope ps("fwd_bwd", s, fl, 0.0);
    for (int k = 0; k < S; ++k) {
        const T* W = params + md.woff[k];
        const T* b = params + md.boff[k];
        EpiForward<T> e{b, c.z[k], c.ldt[k], k + 1 < S ? c.a[k + 1] : nullptr, c.lda[k + 1], md.w[k + 1], md.act};
        model_gemm<T>(s, n, md.w[k + 1], md.w[k], kmaj(c.a[k], c.lda[k]), kmaj(W, md.w[k]), e);
    }
    output_layer_kernel<T><<<(unsigned)ceil_div(n, 128), 128, 0, s>>>(
        c.z[S - 1], c.ldt[S - 1], labels, n, md.w[S], md.mode, c.a[S], c.lda[S], c.delta[S - 1]);
    CK_LAUNCH();
    for (int k = S - 2; k >= 0; --k) {
        const T* W1 = params + md.woff[k + 1];  // T_{k+2} x T_{k+1}
        EpiBackward<T> e{c.z[k], c.up[k], c.delta[k], c.ldt[k], md.act};
        model_gemm<T>(s, n, md.w[k + 1], md.w[k + 2], kmaj(c.delta[k + 1], c.ldt[k + 1]), mnmaj(W1, md.w[k + 1]), e);
    }
}

// ---------------------------------------------------------------------------
// per-example gradients: J[n][p] (autodiff.cpp:127-143).  Pure HBM write
// stream: every CTA owns one example row and walks it with 16-byte stores.
// ---------------------------------------------------------------------------
struct LayerTable {
    int S;
    int64_t tin[kMaxLayers], tout[kMaxLayers], woff[kMaxLayers], boff[kMaxLayers];
    int64_t lda[kMaxLayers], ldt[kMaxLayers];
};

inline LayerTable make_table(const ModelDesc& md, const int64_t* lda, const int64_t* ldt) {
    LayerTable t{};
    t.S = md.S;
    for (int k = 0; k < md.S; ++k) {
        t.tin[k] = md.w[k]; t.tout[k] = md.w[k + 1];
        t.woff[k] = md.woff[k]; t.boff[k] = md.boff[k];
        t.lda[k] = lda[k]; t.ldt[k] = ldt[k];
    }
    return t;
}

template <class T>
struct CachePtrs {
    const T* a[kMaxLayers];
    const T* delta[kMaxLayers];
};

template <class T>
__device__ __forceinline__ T jac_entry(const LayerTable& t, const CachePtrs<T>& cp, int64_t row, int64_t col) {
    int k = 0;
    while (k + 1 < t.S && col >= t.woff[k + 1]) ++k;
    const int64_t e = col - t.woff[k];
    const int64_t nw = t.tin[k] * t.tout[k];
    const T* d = cp.delta[k] + row * t.ldt[k];
    if (e < nw) {
        const int64_t o = e / t.tin[k], i = e - o * t.tin[k];
        return d[o] * cp.a[k][row * t.lda[k] + i];
    }
    return d[e - nw];
}

template <class T>
__global__ void __launch_bounds__(256) jacobian_kernel(LayerTable t, CachePtrs<T> cp, int64_t P, T* __restrict__ J,
                                                       int64_t ldj, int64_t row0, int rn_tf32, int vec) {
    const int64_t row = row0 + blockIdx.y;
    T* out = J + (int64_t)blockIdx.y * ldj;
    constexpr int V = 16 / sizeof(T);
    for (int64_t c0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * V; c0 < P;
         c0 += (int64_t)gridDim.x * blockDim.x * V) {
        T v[V];
#pragma unroll
        for (int u = 0; u < V; ++u) v[u] = c0 + u < P ? jac_entry(t, cp, row, c0 + u) : T(0);
        if constexpr (sizeof(T) == 4) {
            if (rn_tf32) {
#pragma unroll
                for (int u = 0; u < V; ++u) v[u] = round_tf32(v[u]);
            }
        }
        if (vec && c0 + V <= P) {  // 16-byte aligned rows: vector stores (the pitch padding untouched)
            if constexpr (sizeof(T) == 4) {
                *reinterpret_cast<float4*>(out + c0) = make_float4(v[0], v[1], v[2], v[3]);
            } else {
                *reinterpret_cast<double2*>(out + c0) = make_double2(v[0], v[1]);
            }
        } else {
            for (int u = 0; u < V && c0 + u < P; ++u) out[c0 + u] = v[u];
        }
    }
}

// Structured writer: one CTA per (example row, layer k) keeps its activation
// chunk a_k[n, 4t .. 4t+3] in registers and streams the T_{k+1} rows
// delta_k[n, o] * a_k[n, :] of the weight block, then the bias entries.
// Needs T_k % 4 == 0 and 16-byte aligned block starts (checked by the host).
template <class T>
__global__ void __launch_bounds__(256) jacobian_rows_kernel(LayerTable t, CachePtrs<T> cp, T* __restrict__ J,
                                                            int64_t ldj, int64_t row0, int rn_tf32) {
    const int k = blockIdx.y;
    const int64_t row = row0 + blockIdx.x;
    const int64_t tin = t.tin[k], tout = t.tout[k];
    T* out = J + (int64_t)blockIdx.x * ldj;
    const T* a = cp.a[k] + row * t.lda[k];
    const T* d = cp.delta[k] + row * t.ldt[k];
    auto rnd = [&](T v) -> T {
        if constexpr (sizeof(T) == 4) return rn_tf32 ? round_tf32(v) : v;
        return v;
    };
    for (int64_t i4 = threadIdx.x; i4 * 4 < tin; i4 += blockDim.x) {
        const T a0 = a[4 * i4], a1 = a[4 * i4 + 1], a2 = a[4 * i4 + 2], a3 = a[4 * i4 + 3];
        T* dst = out + t.woff[k] + 4 * i4;
        for (int64_t o = 0; o < tout; ++o) {
            const T dv = __ldg(&d[o]);
            if constexpr (sizeof(T) == 4) {
                __stcs(reinterpret_cast<float4*>(dst + o * tin),
                       make_float4(rnd(dv * a0), rnd(dv * a1), rnd(dv * a2), rnd(dv * a3)));
            } else {
                dst[o * tin] = dv * a0; dst[o * tin + 1] = dv * a1;
                dst[o * tin + 2] = dv * a2; dst[o * tin + 3] = dv * a3;
            }
        }
    }
    for (int64_t o = threadIdx.x; o < tout; o += blockDim.x) out[t.boff[k] + o] = rnd(d[o]);
}

// rn_tf32: store J pre-rounded to TF32 (round to nearest) when it only feeds
// TF32 tensor-core products; the MMA itself truncates the low mantissa bits,
// which biases every product towards zero.
template <class T>
void jacobian(const ModelDesc& md, const Cache<T>& c, int64_t row0, int64_t rows, T* J, int64_t ldj,
              cudaStream_t s, bool rn_tf32 = false) {
    ProfScope ps("jacobian", s, 0.0, (double)sizeof(T) * rows * md.P);
    LayerTable t = make_table(md, c.lda, c.ldt);
    CachePtrs<T> cp;
    for (int k = 0; k < md.S; ++k) { cp.a[k] = c.a[k]; cp.delta[k] = c.delta[k]; }
    bool structured = (ldj % 4 == 0) && (reinterpret_cast<uintptr_t>(J) & 15) == 0;
    for (int k = 0; k < md.S; ++k) structured = structured && md.w[k] % 4 == 0 && md.woff[k] % 4 == 0;
    if (structured) {
        for (int64_t r = 0; r < rows; r += (int64_t)1 << 30) {
            const int64_t rr = std::min<int64_t>((int64_t)1 << 30, rows - r);
            jacobian_rows_kernel<T><<<dim3((unsigned)rr, (unsigned)md.S), 256, 0, s>>>(t, cp, J + r * ldj, ldj,
                                                                                      row0 + r, rn_tf32 ? 1 : 0);
            CK_LAUNCH();
        }
        return;
    }
    const int64_t per_block = 256 * (16 / sizeof(T));
    // any pitch: vector stores only where every row start is 16-byte aligned
    const int vec = (ldj * (int64_t)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(J) & 15) == 0;
    const unsigned gx = (unsigned)std::min<int64_t>(ceil_div(md.P, per_block), 64);
    for (int64_t r = 0; r < rows; r += 65535) {
        const int64_t rr = std::min<int64_t>(65535, rows - r);
        jacobian_kernel<T><<<dim3(gx, (unsigned)rr), 256, 0, s>>>(t, cp, md.P, J + r * ldj, ldj, row0 + r,
                                                                   rn_tf32 ? 1 : 0, vec);
        CK_LAUNCH();
    }
}

// ---------------------------------------------------------------------------
// elementwise helpers for the R-op
// ---------------------------------------------------------------------------

// out[r][c] = f(row-wise cache values) over `rows` = nprof * n rows
template <class T>
__global__ void rop_act_kernel(const T* __restrict__ in, int64_t ldi, const T* __restrict__ z, int64_t ldz,
                               int64_t n, int64_t rows, int64_t cols, int act, T* __restrict__ out, int64_t ldo) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= rows * cols) return;
    const int64_t r = idx / cols, c = idx % cols, e = r % n;
    out[r * ldo + c] = act_deriv<T>(act, z[e * ldz + c]) * in[r * ldi + c];
}

// rdelta_out = p * (rz - p . rz) for each (profile, example) row; zero in
// raw_mean_output mode (autodiff.cpp:190-205).
template <class T>
__global__ void rop_softmax_kernel(const T* __restrict__ rz, int64_t ldr, const T* __restrict__ prob, int64_t ldp,
                                   int64_t n, int64_t rows, int64_t tl, int mode, T* __restrict__ out, int64_t ldo) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int64_t e = r % n;
    const T* pr = prob + e * ldp;
    const T* x = rz + r * ldr;
    T* o = out + r * ldo;
    if (mode == kRawMean) {
        for (int64_t m = 0; m < tl; ++m) o[m] = T(0);
        return;
    }
    T pd = T(0);
    for (int64_t m = 0; m < tl; ++m) pd += pr[m] * x[m];
    for (int64_t m = 0; m < tl; ++m) o[m] = pr[m] * (x[m] - pd);
}

// R-backward epilogue: rd = acc (+ existing) ;  final = rd*act'(z) + up*act''(z)*rz
// `accum` adds into out first (second GEMM of the pair).  unit_prof >= 0
// marks the tangent layer itself, where rz = e_o (o = row / n).
template <class T>
struct EpiRback {
    T* out;
    int64_t ldo;
    const T* z;
    const T* up;
    int64_t ldz;
    const T* rz;  // may be null
    int64_t ldr;
    int64_t n;
    int act;
    int unit_prof;  // 1: rz is e_{row/n} (profile tangent layer)
    int finalize;   // 0: store raw acc (first of two GEMMs); 1: acc(+out) then apply
    int accum;
    int64_t o0 = 0;  // unit_prof: row block b holds the tangent of unit o0 + b (unit bands)
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int, int64_t r, int64_t c, T acc) const {
        T v = acc;
        if (accum) v += out[r * ldo + c];
        if (finalize) {
            const int64_t e = r % n;
            const T zz = z[e * ldz + c];
            T rzv = T(0);
            if (unit_prof) rzv = (c == o0 + r / n) ? T(1) : T(0);
            else if (rz) rzv = rz[r * ldr + c];
            v = v * act_deriv<T>(act, zz) + (up ? up[e * ldz + c] * act_second<T>(act, zz) * rzv : T(0));
        }
        out[r * ldo + c] = v;
    }
};

// prof[o - o0][n][t] = act'(z_k[n][o]) * W_{k+1}[t][o]   (R-forward one step above
// the tangent layer for rz_k = e_o), tangents o in [o0, o0 + no)
template <class T>
__global__ void profile_first_rz_kernel(const T* __restrict__ zk, int64_t ldz, const T* __restrict__ W1,
                                        int64_t t1, int64_t t2, int64_t n, int act, T* __restrict__ out,
                                        int64_t ldo, int64_t o0, int64_t no) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= no * n * t2) return;
    const int64_t t = idx % t2, r = idx / t2, o = o0 + r / n, e = r % n;
    out[r * ldo + t] = act_deriv<T>(act, zk[e * ldz + o]) * W1[t * t1 + o];
}

// G_{S-1}[o - o0][n][t] = p_t (delta_{to} - p_o): output-layer Hessian columns,
// tangents o in [o0, o0 + no)
template <class T>
__global__ void profile_output_kernel(const T* __restrict__ prob, int64_t ldp, int64_t tl, int64_t n, int mode,
                                      T* __restrict__ out, int64_t ldo, int64_t o0, int64_t no) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= no * n * tl) return;
    const int64_t t = idx % tl, r = idx / tl, o = o0 + r / n, e = r % n;
    T v = T(0);
    if (mode == kSoftmaxCE) {
        const T pt = prob[e * ldp + t], po = prob[e * ldp + o];
        v = pt * ((t == o ? T(1) : T(0)) - po);
    }
    out[r * ldo + t] = v;
}

// Q_{k-1}[i][n][t] = act'(z_{k-1}[n][i]) * [t == i]
template <class T>
__global__ void profile_q_kernel(const T* __restrict__ z, int64_t ldz, int64_t tk, int64_t n, int act,
                                 T* __restrict__ out, int64_t ldo) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= tk * n * tk) return;
    const int64_t t = idx % tk, r = idx / tk, i = r / n, e = r % n;
    out[r * ldo + t] = t == i ? act_deriv<T>(act, z[e * ldz + i]) : T(0);
}

// ---------------------------------------------------------------------------
// R operand for one Hessian block: rows (o'', jj) of the tangent chunk
//   m == k: R = s_n * G[o][n][o'']
//   m <  k: R = s_n * Pm[o][n][o''] + [weight tangent] delta_k[n][o] * Qm[i][n][o'']
// with s_n = a_k[n][i] for weight tangents (o, i) and 1 for bias tangents.
// ---------------------------------------------------------------------------
template <class T>
struct RGenArgs {
    const T* prof;  // G (m == k) or Pm, transposed: [T_{k+1} - o0][T_{m+1}][ldn]
    const T* q;     // Qm transposed [T_k][T_{m+1}][ldn], or null
    const T* akT;   // a_k transposed [T_k + 1][ldn]
    const T* dkT;   // delta_k transposed [T_{k+1}][ldn]
    int64_t ldn;
    int64_t n, tink, toutk, tm1;  // T_k, T_{k+1}, T_{m+1}
    int64_t j0, J, rows;          // rows = (o'' rows generated) * J
    T* R;
    int64_t ldr;
    int round = 0;                // store R rounded to nearest TF32 (the tensor-core GEMM's A operand)
    int64_t o0 = 0;               // prof holds the tangents of units o0, o0 + 1, ... (unit bands)
};

// CTA (x: a 256-wide slice of the 4-example groups along n, y: a segment of
// RGEN_SEG consecutive rows of one o'' band).  Consecutive rows share their
// unit o (the tangent order is (o, i)), so a thread keeps the profile and
// delta vectors of the current o in registers and loads only a_k[i] and
// Q[i][o''] per row: two 16-byte loads per 16-byte R store instead of four
// (c2: 3.2 -> 1.7 ms for 4.4 GB of R).  Keeping a segment of i in registers
// and walking o instead (~0.3 loads per store) ran slower (3.3 ms: 121
// registers, too few warps for the store stream).
constexpr int RGEN_SEG = 32;
template <class T>
__global__ void __launch_bounds__(256) rgen_kernel(RGenArgs<T> g) {
    const int64_t n4 = g.ldr / 4;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n4) return;
    const int64_t nw = g.toutk * g.tink;
    const int64_t segs = ceil_div(g.J, RGEN_SEG);
    using V = typename std::conditional<sizeof(T) == 4, float4, double4>::type;
    for (int64_t sg = blockIdx.y; sg < (g.rows / g.J) * segs; sg += gridDim.y) {
        const int64_t opp = sg / segs, jj0 = (sg - opp * segs) * RGEN_SEG;
        const int64_t jj1 = jj0 + RGEN_SEG < g.J ? jj0 + RGEN_SEG : g.J;
        int64_t last_o = -1;
        V p{}, d{};
        for (int64_t jj = jj0; jj < jj1; ++jj) {
            const int64_t j = g.j0 + jj;
            const bool wt = j < nw;
            const int64_t o = wt ? j / g.tink : j - nw;
            const int64_t i = wt ? j - o * g.tink : 0;
            if (o != last_o || !wt) {
                p = reinterpret_cast<const V*>(g.prof + ((o - g.o0) * g.tm1 + opp) * g.ldn)[e];
                if (g.q) d = reinterpret_cast<const V*>(g.dkT + o * g.ldn)[e];
                last_o = wt ? o : -1;
            }
            // four consecutive weight tangents of one unit: their eight loads are issued
            // before the first store (the compiler will not move loads across the stores
            // to R on its own)
            if (wt && g.q && jj + 4 <= jj1 && i + 4 <= g.tink) {
                V sv[4], qv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    sv[u] = reinterpret_cast<const V*>(g.akT + (i + u) * g.ldn)[e];
                    qv[u] = reinterpret_cast<const V*>(g.q + ((i + u) * g.tm1 + opp) * g.ldn)[e];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    V r = p;  // (the same operation order as the single-row form below)
                    r.x *= sv[u].x; r.y *= sv[u].y; r.z *= sv[u].z; r.w *= sv[u].w;
                    r.x += d.x * qv[u].x; r.y += d.y * qv[u].y; r.z += d.z * qv[u].z; r.w += d.w * qv[u].w;
                    if constexpr (sizeof(T) == 4) {
                        if (g.round) {
                            r.x = round_tf32(r.x); r.y = round_tf32(r.y); r.z = round_tf32(r.z); r.w = round_tf32(r.w);
                        }
                        __stcs(reinterpret_cast<V*>(g.R + (opp * g.J + jj + u) * g.ldr) + e, r);
                    } else {
                        reinterpret_cast<V*>(g.R + (opp * g.J + jj + u) * g.ldr)[e] = r;
                    }
                }
                jj += 3;  // (the loop adds the fourth)
                continue;
            }
            V r = p;
            if (wt) {
                const V s = reinterpret_cast<const V*>(g.akT + i * g.ldn)[e];
                r.x *= s.x; r.y *= s.y; r.z *= s.z; r.w *= s.w;
                if (g.q) {
                    const V qv = reinterpret_cast<const V*>(g.q + (i * g.tm1 + opp) * g.ldn)[e];
                    r.x += d.x * qv.x; r.y += d.y * qv.y; r.z += d.z * qv.z; r.w += d.w * qv.w;
                }
            }
            if constexpr (sizeof(T) == 4) {
                if (g.round) {
                    r.x = round_tf32(r.x); r.y = round_tf32(r.y); r.z = round_tf32(r.z); r.w = round_tf32(r.w);
                }
                __stcs(reinterpret_cast<V*>(g.R + (opp * g.J + jj) * g.ldr) + e, r);
            } else {
                reinterpret_cast<V*>(g.R + (opp * g.J + jj) * g.ldr)[e] = r;
            }
        }
    }
}

// out[b][c][r] = in[b][r][c]  (rows x cols per batch; 32x32 smem tiles)
template <class T>
__device__ __forceinline__ void transpose_tile(const T* __restrict__ in, int64_t ldi, int64_t bsi, T* __restrict__ out,
                                               int64_t ldo, int64_t bso, int64_t rows, int64_t cols, int64_t bx,
                                               int64_t by, int64_t bz) {
    __shared__ T tile[32][33];
    const int64_t r0 = bx * 32, c0 = by * 32;
    const T* ip = in + bz * bsi;
    T* op = out + bz * bso;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t r = r0 + y, c = c0 + threadIdx.x;
        tile[y][threadIdx.x] = (r < rows && c < cols) ? ip[r * ldi + c] : T(0);
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t c = c0 + y, r = r0 + threadIdx.x;
        if (c < cols && r < ldo) op[c * ldo + r] = r < rows ? tile[threadIdx.x][y] : T(0);
    }
}

template <class T>
__global__ void transpose_kernel(const T* __restrict__ in, int64_t ldi, int64_t bsi, T* __restrict__ out,
                                 int64_t ldo, int64_t bso, int64_t rows, int64_t cols) {
    transpose_tile<T>(in, ldi, bsi, out, ldo, bso, rows, cols, blockIdx.x, blockIdx.y, blockIdx.z);
}

// Several independent transposes in one launch (the per-layer n-contiguous
// copies of the curvature prep): block b belongs to the last job whose
// first block is <= b.
template <class T>
struct TransposeJobs {
    static constexpr int kMax = 8;
    struct Job {
        const T* in;
        T* out;
        int64_t ldi, bsi, ldo, bso, rows, cols, bx, by, block0;
    } j[kMax];
    int n = 0;
    int64_t blocks = 0;
};

template <class T>
__global__ void transpose_jobs_kernel(const __grid_constant__ TransposeJobs<T> J) {
    const int64_t b = blockIdx.x;
    int q = 0;
    while (q + 1 < J.n && b >= J.j[q + 1].block0) ++q;
    const auto& t = J.j[q];
    const int64_t lb = b - t.block0;
    transpose_tile<T>(t.in, t.ldi, t.bsi, t.out, t.ldo, t.bso, t.rows, t.cols, lb % t.bx, (lb / t.bx) % t.by,
                      lb / (t.bx * t.by));
}

// same arguments as transpose(); jobs are launched together by flush()
template <class T>
struct TransposeBatch {
    cudaStream_t s;
    TransposeJobs<T> J{};
    explicit TransposeBatch(cudaStream_t st) : s(st) {}
    void add(const T* in, int64_t ldi, int64_t bsi, T* out, int64_t ldo, int64_t bso, int64_t rows, int64_t cols,
             int64_t batch) {
        if (J.n == TransposeJobs<T>::kMax) flush();
        auto& t = J.j[J.n++];
        t = {in, out, ldi, bsi, ldo, bso, rows, cols, ceil_div(ldo, 32), ceil_div(cols, 32), J.blocks};
        J.blocks += t.bx * t.by * batch;
    }
    void flush() {
        if (J.n == 0) return;
        transpose_jobs_kernel<T><<<(unsigned)J.blocks, dim3(32, 8), 0, s>>>(J);
        CK_LAUNCH();
        J.n = 0;
        J.blocks = 0;
    }
    // never launches (a destructor must not throw): callers flush() explicitly;
    // jobs still pending here belong to a call that is unwinding on an error
    ~TransposeBatch() { J.n = 0; }
};

template <class T>
void transpose(cudaStream_t s, const T* in, int64_t ldi, int64_t bsi, T* out, int64_t ldo, int64_t bso, int64_t rows,
               int64_t cols, int64_t batch) {
    // covers padding columns r in [rows, ldo) with zeros
    dim3 grid((unsigned)ceil_div(ldo, 32), (unsigned)ceil_div(cols, 32), (unsigned)batch);
    transpose_kernel<T><<<grid, dim3(32, 8), 0, s>>>(in, ldi, bsi, out, ldo, bso, rows, cols);
    CK_LAUNCH();
}

// Hessian block epilogue: GEMM row r = (o'', jj), column c = input unit of
// layer m (c == T_m is the bias column, fed by the ones column of a_m).
template <class T>
struct EpiHess {
    T* H;
    int64_t ldh;
    int64_t J, j0, woffk, woffm, boffm, tm;
    T alpha;
    int diag;    // m == k
    int mirror;  // write the transposed entry too
    // shard of tangent rows owned by this call (global H row of the lower
    // entry); entries of other rows and their mirrors are left untouched
    int64_t rlo = 0, rhi = INT64_MAX;
    // band output (unit bands): H holds row gr at H + (gr - rsh) * ldh; no mirrors
    int64_t rsh = 0;
    __host__ __device__ __forceinline__ bool owns(int64_t gr) const { return gr >= rlo && gr < rhi; }
    __host__ __device__ __forceinline__ int64_t gcol(int64_t opp, int64_t c) const {
        return c < tm ? woffm + opp * tm + c : boffm + opp;
    }
    __host__ __device__ bool skip(int, int64_t r0, int64_t c0, int64_t bm, int64_t) const {
        if (!diag || !mirror) return false;
        const int64_t opp_min = r0 / J;
        const int64_t jj_max = (r0 + bm - 1) / J > opp_min ? J - 1 : (r0 + bm - 1) % J;
        const int64_t gr_max = woffk + j0 + jj_max;
        return gcol(opp_min, c0) > gr_max;
    }
    __device__ void operator()(int, int64_t r, int64_t c, T acc) const {
        const int64_t opp = r / J, jj = r - opp * J;
        const int64_t gr = woffk + j0 + jj, gc = gcol(opp, c);
        const T v = alpha * acc;
        if (!owns(gr)) return;
        if (diag && mirror) {
            if (gc > gr) return;
            H[(gr - rsh) * ldh + gc] = v;
            H[gc * ldh + gr] = v;
        } else {
            H[(gr - rsh) * ldh + gc] = v;
            if (mirror) H[gc * ldh + gr] = v;
        }
    }
    // the two stores of operator() separately (staged fp64 epilogue)
    __device__ void store_direct(int, int64_t r, int64_t c, T acc) const {
        const int64_t opp = r / J, jj = r - opp * J;
        const int64_t gr = woffk + j0 + jj, gc = gcol(opp, c);
        if (!owns(gr) || (diag && mirror && gc > gr)) return;
        H[(gr - rsh) * ldh + gc] = alpha * acc;
    }
    __device__ void store_mirror(int, int64_t r, int64_t c, T acc) const {
        if (!mirror) return;
        const int64_t opp = r / J, jj = r - opp * J;
        const int64_t gr = woffk + j0 + jj, gc = gcol(opp, c);
        if (!owns(gr) || (diag && gc > gr)) return;
        H[gc * ldh + gr] = alpha * acc;
    }
    // 32 x 32 block stored by two TMA boxes (direct at (gr0, gc0), mirror at
    // (gc0, gr0); gr0 returned as the storage row): rows in one band and owned, columns inside the weight
    // columns, and on diagonal blocks strictly below the diagonal
    __device__ bool tma_block(int64_t row0, int64_t col0, int64_t M, int64_t N, int64_t& gr0, int64_t& gc0) const {
        if (row0 + 32 > M || col0 + 32 > N || col0 + 32 > tm) return false;
        const int64_t opp = row0 / J, jj = row0 - opp * J;
        if (jj + 32 > J) return false;
        gr0 = woffk + j0 + jj;
        if (gr0 < rlo || gr0 + 32 > rhi) return false;
        gc0 = woffm + opp * tm + col0;
        const bool ok = !(diag && mirror && gc0 + 31 >= gr0);
        gr0 -= rsh;  // storage row (band output); mirrors are off there
        return ok;
    }
    // register-only epilogue (fused kernel): lane = row row0 + lane holds the
    // 32 accumulators of columns col0 .. col0 + 31 in v[]; the row's entries
    // are 128 contiguous bytes of H (16-byte stores), the mirrored column
    // entries are one coalesced 128-byte store per column
    __device__ void block_regs(int64_t row0, int64_t col0, int64_t M, int64_t N, const float* v, int lane) const {
        const bool tri = diag && mirror;
        const int64_t r = row0 + lane;
        if (r >= M) return;
        const int64_t opp = r / J, jj = r - opp * J;
        const int64_t gr = woffk + j0 + jj;
        if (!owns(gr)) return;
        const int ncols = (int)::min((int64_t)32, N - col0);
        const int64_t wbase = woffm + opp * tm;
        T* row = H + (gr - rsh) * ldh;
        if constexpr (sizeof(T) == 4) {
            // whole 32-column run inside the weight columns and the triangle
            const int64_t gc0 = wbase + col0;
            if (ncols == 32 && col0 + 32 <= tm && ((gc0 | ldh) & 3) == 0 && (!tri || gc0 + 31 <= gr)) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    __stcs(reinterpret_cast<float4*>(row + gc0) + q,
                           make_float4(alpha * v[4 * q], alpha * v[4 * q + 1], alpha * v[4 * q + 2], alpha * v[4 * q + 3]));
                if (mirror) {
#pragma unroll
                    for (int cc = 0; cc < 32; ++cc)
                        if (!tri || gc0 + cc < gr) __stcs(&H[(gc0 + cc) * ldh + gr], alpha * (T)v[cc]);
                }
                return;
            }
        }
#pragma unroll
        for (int cc = 0; cc < 32; ++cc) {  // constant trip count keeps v[] in registers
            const int64_t c = col0 + cc;
            const int64_t gc = c < tm ? wbase + c : boffm + opp;
            if (cc < ncols && (!tri || gc <= gr)) {
                __stcs(&row[gc], alpha * (T)v[cc]);
                if (mirror && (!tri || gc < gr)) __stcs(&H[gc * ldh + gr], alpha * (T)v[cc]);
            }
        }
    }
    // tensor-core epilogue (32 x 32 block, coalesced in both store directions)
    __device__ void block(int64_t row0, int64_t col0, int64_t M, int64_t N, const float (*buf)[36], const float* v,
                          int lane) const {
        block_any(row0, col0, M, N, [&](int r, int q) { return *reinterpret_cast<const float4*>(&buf[r][4 * q]); },
                  v, lane);
    }
    // same, the staged block read through get(r, q) = columns 4q .. 4q+3 of row r
    template <class Get>
    __device__ void block_any(int64_t row0, int64_t col0, int64_t M, int64_t N, Get get, const float* v,
                              int lane) const {
        const bool tri = diag && mirror;
        // one division per block; each row's (o'', jj) follows by carrying
        const int64_t opp0 = row0 / J, jj0 = row0 - opp0 * J;
        const int nrows = (int)::min((int64_t)32, M - row0);
        {  // direct: H[gr][gc], 16-byte vectors along gc
            const int q = lane & 7, rsub = lane >> 3;
            const int64_t c = col0 + 4 * q;
            for (int it = 0; it < 8; ++it) {
                const int r = it * 4 + rsub;
                if (r >= nrows) break;
                int64_t opp = opp0, jj = jj0 + r;
                while (jj >= J) { jj -= J; ++opp; }
                const int64_t gr = woffk + j0 + jj, wb = woffm + opp * tm;
                if (!owns(gr)) continue;
                const float4 x = get(r, q);
                T* row = H + (gr - rsh) * ldh;
                if constexpr (sizeof(T) == 4) {
                    const int64_t gc = wb + c;
                    if (c + 3 < tm && c + 3 < N && ((gc | ldh) & 3) == 0 && (!tri || gc + 3 <= gr)) {
                        __stcs(reinterpret_cast<float4*>(row + gc),
                               make_float4(alpha * x.x, alpha * x.y, alpha * x.z, alpha * x.w));
                        continue;
                    }
                }
                const float xs[4] = {x.x, x.y, x.z, x.w};
                for (int u = 0; u < 4; ++u) {
                    const int64_t cc = c + u;
                    if (cc >= N) break;
                    const int64_t gc = cc < tm ? wb + cc : boffm + opp;
                    if (!tri || gc <= gr) __stcs(&row[gc], alpha * (T)xs[u]);
                }
            }
        }
        if (mirror && lane < nrows) {  // transposed: H[gc][gr], this lane's row from registers
            int64_t opp = opp0, jj = jj0 + lane;
            while (jj >= J) { jj -= J; ++opp; }
            const int64_t gr = woffk + j0 + jj;
            const int ncols = owns(gr) ? (int)::min((int64_t)32, N - col0) : 0;
            const int64_t wbase = woffm + opp * tm;
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {  // constant trip count keeps v[] in registers
                const int64_t c = col0 + cc;
                const int64_t gc = c < tm ? wbase + c : boffm + opp;
                if (cc < ncols && (!tri || gc < gr)) __stcs(&H[gc * ldh + gr], alpha * (T)v[cc]);
            }
        }
    }
};

// HVP accumulation epilogue: rows o of step k, column c (c == T_k: bias)
template <class T>
struct EpiHv {
    T* hv;
    int64_t ldhv;  // stride between directions
    int64_t woff, boff, tin;
    T alpha;
    int accum;
    __device__ bool skip(int, int64_t, int64_t, int64_t, int64_t) const { return false; }
    __device__ void operator()(int b, int64_t o, int64_t c, T acc) const {
        T* p = hv + b * ldhv + (c < tin ? woff + o * tin + c : boff + o);
        *p = accum ? *p + alpha * acc : alpha * acc;
    }
};

}  // namespace ck
