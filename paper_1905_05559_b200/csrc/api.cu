// api.cu -- the C-ABI (include/curvkit_b200.h) over the B200 engine.
//
// Validation and error text follow the reference (model.cpp:80-87,
// model.cpp:201-214, curvature.cpp:15-29, autodiff.cpp:266-280) so a caller
// switching from curvkit sees the same contract errors for the same inputs.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/curvkit_b200.h"
#include "bands.cuh"
#include "comm.cuh"
#include "common.cuh"
#include "curvature.cuh"
#include "eigen.cuh"
#include "eigops.cuh"
#include "lanczos.cuh"
#include "gemm_tc.cuh"
#include "incremental.cuh"
#include "model.cuh"
#include "prof.cuh"

namespace ck {
std::atomic<int64_t> g_launches{0};
}

namespace {

using namespace ck;

thread_local std::string g_err;

void trim_pool();

template <class F>
int guard(F&& f) {
    try {
        f();
        trim_pool();
        return kOk;
    } catch (const CurvError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_err = e.what();
        return kOutOfMemory;
    } catch (const std::exception& e) {
        g_err = e.what();
        return kRuntimeError;
    }
}

// bytes of pool memory kept mapped between calls (CURVKIT_POOL_KEEP_GB,
// default 64): a host that re-runs config-3 sized calls keeps its 48 GB result and J mapped
// (re-mapping them cost 100-400 ms per call at a 16 GB threshold)
size_t pool_keep_bytes() {
    static const size_t keep = [] {
        const char* e = getenv("CURVKIT_POOL_KEEP_GB");
        const double gb = e ? atof(e) : 64.0;
        return (size_t)((gb > 0 ? gb : 0.0) * double(1ull << 30));
    }();
    return keep;
}

void trim_pool() {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolTrimTo(pool, pool_keep_bytes());
}

[[noreturn]] void contract(const std::string& m) { throw CurvError(kContractError, m); }

constexpr int64_t kAutoDegree = 6;  // Chebyshev degree of the converged top-k solver
[[noreturn]] void shape(const std::string& m) { throw CurvError(kShapeError, m); }

ModelDesc make_desc(const curvkit_model* m) {
    if (!m || !m->layer_widths) contract("model needs at least an input and an output layer");
    ModelDesc d;
    if (m->num_layers < 2) contract("model needs at least an input and an output layer");
    if (m->num_layers > kMaxLayers) contract("model has more than 16 layers");
    d.L = m->num_layers;
    d.S = d.L - 1;
    d.act = m->hidden_activation;
    d.mode = m->output_mode;
    if (d.act < 0 || d.act > 3) contract("unknown activation");
    if (d.mode < 0 || d.mode > 1) contract("unknown output mode");
    for (int i = 0; i < d.L; ++i) {
        d.w[i] = m->layer_widths[i];
        if (d.w[i] < 1) contract("layer widths must be >= 1");
    }
    if (d.mode == kRawMean && d.w[d.L - 1] != 1) contract("raw_mean_output requires an output width of 1");
    int64_t at = 0;
    for (int k = 0; k < d.S; ++k) {
        d.woff[k] = at;
        d.boff[k] = at + d.w[k] * d.w[k + 1];
        at += d.block_size(k);
    }
    d.P = at;
    return d;
}

// model.cpp:201-214 -> class indices
std::vector<int32_t> labels_from_onehot(const ModelDesc& md, const double* y, int64_t n) {
    std::vector<int32_t> lab(n, 0);
    if (md.mode == kRawMean) return lab;
    if (!y) contract("target row 0 is not one-hot");
    const int64_t tl = md.w[md.L - 1];
    for (int64_t r = 0; r < n; ++r) {
        int ones = 0;
        for (int64_t m = 0; m < tl; ++m) {
            const double v = y[r * tl + m];
            if (v == 1.0) {
                ++ones;
                lab[r] = (int32_t)m;
            } else if (v != 0.0) {
                contract("target row " + std::to_string(r) + " is not one-hot");
            }
        }
        if (ones != 1) contract("target row " + std::to_string(r) + " is not one-hot");
    }
    return lab;
}

void check_divisible(int64_t n, int64_t b, const char* who) {  // curvature.cpp:15-22
    if (b < 1) contract(std::string(who) + ": batch size must be >= 1");
    if (n == 0) contract(std::string(who) + ": empty dataset");
    if (n % b != 0)
        contract(std::string(who) + ": dataset size " + std::to_string(n) + " is not divisible by batch size " +
                 std::to_string(b) + "; refusing to drop the remainder");
}

void check_memory_cap(int64_t p, int64_t cap, const char* who) {  // curvature.cpp:24-29
    if (p > cap)
        contract(std::string(who) + ": P = " + std::to_string(p) + " exceeds the dense memory cap " +
                 std::to_string(cap) + "; use the matrix-free eigensolvers instead");
}

// Never release the stream-ordered pool at synchronisation points inside a
// call: a sync while an 84 GB J is live would otherwise unmap every freed
// workspace and re-map it on the next allocation.  Keep up to 64 GB mapped
// between calls (curvature workspaces are reused); trim_pool returns the
// rest once the call's frees have completed.
void keep_pool_memory() {
    static std::mutex mu;
    static std::vector<int> done;
    int dev = 0;
    CK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (std::find(done.begin(), done.end(), dev) != done.end()) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done.push_back(dev);
}

// the host-buffer entry points' stream: one per (thread, device)
cudaStream_t lib_stream() {
    static thread_local std::vector<std::pair<int, cudaStream_t>> streams;
    keep_pool_memory();
    int dev = 0;
    CK_CUDA(cudaGetDevice(&dev));
    for (const auto& ds : streams)
        if (ds.first == dev) return ds.second;
    cudaStream_t s = nullptr;
    CK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    streams.emplace_back(dev, s);
    return s;
}

cudaStream_t dev_stream(void* stream) {
    keep_pool_memory();
    return static_cast<cudaStream_t>(stream);
}

bool is_f64(int prec) {
    if (prec < kF64 || prec > kF16S) contract("unknown precision");
    return prec == kF64;
}

// Resident problem: params, cache (forward/backward done) on the device.
template <class T>
struct Resident {
    DevMem params;
    DevMem labels;
    Cache<T> cache;
};

template <class T>
__global__ void convert_kernel(const double* __restrict__ in, T* __restrict__ out, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (T)in[i];
}

template <class T, class U>
__global__ void convert_rows_kernel(const T* __restrict__ in, int64_t ldi, U* __restrict__ out, int64_t ldo,
                                    int64_t rows, int64_t cols) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < rows * cols) out[(i / cols) * ldo + i % cols] = (U)in[(i / cols) * ldi + i % cols];
}

// Upload host doubles and run forward/backward.
template <class T>
void upload_and_forward(const ModelDesc& md, const double* params, const double* x, const std::vector<int32_t>& lab,
                        int64_t n, Resident<T>& r, cudaStream_t s) {
    DevMem pd((size_t)md.P * sizeof(double), s);
    CK_CUDA(cudaMemcpyAsync(pd.p, params, md.P * sizeof(double), cudaMemcpyHostToDevice, s));
    r.params = DevMem((size_t)md.P * sizeof(T), s);
    convert_kernel<T><<<blocks_for(md.P), 256, 0, s>>>(dptr<double>(pd), dptr<T>(r.params), md.P);
    CK_LAUNCH();
    r.labels = DevMem((size_t)n * sizeof(int32_t), s);
    CK_CUDA(cudaMemcpyAsync(r.labels.p, lab.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    alloc_cache<T>(md, n, r.cache, s);
    DevMem xd((size_t)n * md.w[0] * sizeof(double), s);
    CK_CUDA(cudaMemcpyAsync(xd.p, x, (size_t)n * md.w[0] * sizeof(double), cudaMemcpyHostToDevice, s));
    pack_input_kernel<double, T><<<blocks_for(n * r.cache.lda[0]), 256, 0, s>>>(dptr<double>(xd), n, md.w[0],
                                                                                 r.cache.a[0], r.cache.lda[0]);
    CK_LAUNCH();
    forward_backward<T>(md, dptr<T>(r.params), dptr<int32_t>(r.labels), r.cache, s);
    // Settle the pageable-memory uploads before the curvature work: without this
    // sync a later 2.6 GB device-to-pinned download of the same call measured
    // 53-214 ms instead of a steady 53 ms (tools/e2e_probe.py)
    CK_CUDA(cudaStreamSynchronize(s));
}

// Device-resident inputs: x already T on device.
template <class T>
void forward_device(const ModelDesc& md, const T* params, const T* x, const int32_t* labels, int64_t n, Cache<T>& c,
                    cudaStream_t s) {
    alloc_cache<T>(md, n, c, s);
    pack_input_kernel<T, T><<<blocks_for(n * c.lda[0]), 256, 0, s>>>(x, n, md.w[0], c.a[0], c.lda[0]);
    CK_LAUNCH();
    forward_backward<T>(md, params, labels, c, s);
}

// Copy a device matrix (rows x cols, ld) to host U (dense), converting.
template <class T, class U>
void download(const T* d, int64_t ld, int64_t rows, int64_t cols, U* h, cudaStream_t s) {
    if constexpr (sizeof(T) == sizeof(U)) {
        CK_CUDA(cudaMemcpy2DAsync(h, cols * sizeof(U), d, ld * sizeof(T), cols * sizeof(T), rows,
                                  cudaMemcpyDeviceToHost, s));
    } else {
        const int64_t chunk = std::max<int64_t>(1, (int64_t(64) << 20) / (cols * (int64_t)sizeof(U)));
        DevMem st[2] = {DevMem((size_t)chunk * cols * sizeof(U), s), DevMem((size_t)chunk * cols * sizeof(U), s)};
        int which = 0;
        for (int64_t r0 = 0; r0 < rows; r0 += chunk, which ^= 1) {
            const int64_t rr = std::min(chunk, rows - r0);
            convert_rows_kernel<T, U><<<blocks_for(rr * cols), 256, 0, s>>>(d + r0 * ld, ld, dptr<U>(st[which]), cols,
                                                                             rr, cols);
            CK_LAUNCH();
            CK_CUDA(cudaMemcpyAsync(h + r0 * cols, st[which].p, rr * cols * sizeof(U), cudaMemcpyDeviceToHost, s));
        }
    }
    CK_CUDA(cudaStreamSynchronize(s));
}

template <class T>
double hessian_into(const ModelDesc& md, const T* params, const Cache<T>& c, T* H, int64_t ldh, int prec, bool verify,
                    cudaStream_t s) {
    Engine<T> eng{md, s, prec};
    eng.hessian(params, c, H, ldh, verify);
    if (!verify) return 0.0;
    DevMem bits(2 * sizeof(unsigned long long), s);
    CK_CUDA(cudaMemsetAsync(bits.p, 0, 2 * sizeof(unsigned long long), s));
    unsigned long long* b = dptr<unsigned long long>(bits);
    absmax_kernel<T><<<1024, 256, 0, s>>>(H, ldh, md.P, md.P, b + 1);
    CK_LAUNCH();
    for (int k = 0; k < md.S; ++k) {
        const int64_t sz = md.block_size(k);
        symmetrize_block_kernel<T><<<blocks_for(sz * sz), 256, 0, s>>>(H, ldh, md.woff[k], sz, b);
        CK_LAUNCH();
    }
    unsigned long long hb[2];
    CK_CUDA(cudaMemcpyAsync(hb, b, sizeof(hb), cudaMemcpyDeviceToHost, s));
    CK_CUDA(cudaStreamSynchronize(s));
    double asym, hmax;
    std::memcpy(&asym, &hb[0], 8);
    std::memcpy(&hmax, &hb[1], 8);
    // curvature.cpp:81-84; fp32 storage modes get fp32-scaled headroom.
    const double tol = prec == kF64 ? 1e-8 : 1e-3;
    if (asym > tol * hmax)
        throw CurvError(kRuntimeError, "assemble_hessian: pre-symmetrization asymmetry " + std::to_string(asym) +
                                           " exceeds " + std::to_string(tol) + " * " + std::to_string(hmax));
    return asym;
}

// dev (CURVKIT_HOST_TIMING): wall time of the phases of a host-buffer call
struct HostTimer {
    const char* name;
    cudaStream_t s;
    bool on;
    std::chrono::steady_clock::time_point t;
    HostTimer(const char* n, cudaStream_t st) : name(n), s(st), on(getenv("CURVKIT_HOST_TIMING") != nullptr) {
        if (on) t = std::chrono::steady_clock::now();
    }
    void mark(const char* phase) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[curvkit] %s %s %.2f ms\n", name, phase, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

template <class T, class U>
void host_hessian(const ModelDesc& md, const double* params, const double* x, const double* y, int64_t n,
                  const curvkit_curvature_config* cfg, int prec, bool verify, U* h_out, double* asym_out) {
    const int64_t cap = cfg ? cfg->memory_cap : 4096;
    check_memory_cap(md.P, cap, "assemble_hessian");
    check_divisible(n, cfg ? cfg->batch_size_h : n, "assemble_hessian");
    auto lab = labels_from_onehot(md, y, n);
    cudaStream_t s = lib_stream();
    HostTimer tm("assemble_hessian", s);
    Resident<T> r;
    upload_and_forward<T>(md, params, x, lab, n, r, s);
    tm.mark("upload+forward");
    const int64_t ldh = round_up(md.P, 32);  // 128-byte row pitch: the block stores write whole lines
    DevMem H((size_t)md.P * ldh * sizeof(T), s);
    const double asym = hessian_into<T>(md, dptr<T>(r.params), r.cache, dptr<T>(H), ldh, prec, verify, s);
    tm.mark("compute");
    download<T, U>(dptr<T>(H), ldh, md.P, md.P, h_out, s);
    tm.mark("download");
    if (asym_out) *asym_out = asym;
}

template <class T>
void jacobian_full(const ModelDesc& md, const Cache<T>& c, DevMem& J, int64_t& ldj, cudaStream_t s, bool rn = false) {
    ldj = round_up(md.P, 32);
    J = DevMem((size_t)c.n * ldj * sizeof(T), s);
    jacobian<T>(md, c, 0, c.n, dptr<T>(J), ldj, s, rn);
}

// G (rows [rb, re) of the lower triangle and their mirrors): the J-free
// Khatri-Rao route in TF32 mode, else per-example gradients J and the SYRK
template <class T>
void opg_into(const ModelDesc& md, const Cache<T>& c, T* G, int64_t ldg, int prec, cudaStream_t s, int64_t rb = 0,
              int64_t re = -1, int64_t pair_q0 = 0, int64_t pair_q1 = -1) {
    Engine<T> eng{md, s, prec};
    eng.pair_q0 = pair_q0;
    eng.pair_q1 = pair_q1;
    if (eng.opg_kr(c, G, ldg, rb, re < 0 ? INT64_MAX : re)) return;
    DevMem J;
    int64_t ldj;
    jacobian_full<T>(md, c, J, ldj, s, tf32_class(prec));
    eng.opg(dptr<T>(J), ldj, c.n, G, ldg, rb, re);
}

// a second stream per (thread, device) for downloads that overlap compute
cudaStream_t copy_stream() {
    static thread_local std::vector<std::pair<int, cudaStream_t>> streams;
    int dev = 0;
    CK_CUDA(cudaGetDevice(&dev));
    for (const auto& ds : streams)
        if (ds.first == dev) return ds.second;
    cudaStream_t s = nullptr;
    CK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    streams.emplace_back(dev, s);
    return s;
}

// opg_into restricted to a row range assembles those rows and their mirrors: the
// J-free route (TF32 class, f32, f64 orbit kernels) does; the J SYRK route too
template <class T>
bool opg_rows_supported(const ModelDesc&, int prec) {
    return tf32_class(prec) && sizeof(T) == 4;
}

template <class T, class U>
void host_opg(const ModelDesc& md, const double* params, const double* x, const double* y, int64_t n,
              const curvkit_curvature_config* cfg, int prec, U* g_out) {
    const int64_t cap = cfg ? cfg->memory_cap : 4096;
    check_memory_cap(md.P, cap, "assemble_opg");
    check_divisible(n, cfg ? cfg->batch_size_g : n, "assemble_opg");
    auto lab = labels_from_onehot(md, y, n);
    cudaStream_t s = lib_stream();
    HostTimer tm("assemble_opg", s);
    Resident<T> r;
    upload_and_forward<T>(md, params, x, lab, n, r, s);
    tm.mark("upload+forward");
    const int64_t ldg = round_up(md.P, 32);  // 128-byte row pitch: the block stores write whole lines
    DevMem G((size_t)md.P * ldg * sizeof(T), s);
    // Two phases when the result is large and goes out unconverted: the rows of the
    // layers above the first (with their mirrors in the first layer's rows) are
    // assembled first and travel to the host on a second stream while the first
    // layer's diagonal block -- most of the work -- is computed.
    const int64_t split = md.S > 1 ? md.woff[1] : md.P;
    static const bool serial = getenv("CURVKIT_SERIAL_DOWNLOAD") != nullptr;  // dev: one phase
    if (std::is_same_v<T, U> && !serial && split < md.P && md.P * md.P * (int64_t)sizeof(T) >= (int64_t(1) << 30) &&
        opg_rows_supported<T>(md, prec)) {
        T* Gd = dptr<T>(G);
        T* hG = reinterpret_cast<T*>(g_out);
        cudaStream_t s2 = copy_stream();
        std::vector<cudaEvent_t> evs;
        // on every exit (errors included) the copy stream has finished reading G before
        // G's stream-ordered release on s
        struct Drain {
            cudaStream_t st;
            std::vector<cudaEvent_t>& ev;
            ~Drain() {
                cudaStreamSynchronize(st);
                for (cudaEvent_t e : ev) cudaEventDestroy(e);
            }
        } drain{s2, evs};
        // rows [r0, r1) are final on s: they follow on the copy stream
        auto send_rows = [&](int64_t r0, int64_t r1, bool new_event) {
            if (r0 >= r1) return;
            if (new_event) {
                cudaEvent_t e;
                CK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                evs.push_back(e);
                CK_CUDA(cudaEventRecord(e, s));
                CK_CUDA(cudaStreamWaitEvent(s2, e, 0));
            }
            CK_CUDA(cudaMemcpy2DAsync(hG + r0 * md.P, md.P * sizeof(T), Gd + r0 * ldg, ldg * sizeof(T),
                                      md.P * sizeof(T), r1 - r0, cudaMemcpyDeviceToHost, s2));
        };
        opg_into<T>(md, r.cache, Gd, ldg, prec, s, split, md.P);
        send_rows(split, md.P, true);
        // the first layer's diagonal block in ranges of its units o'', last range first and
        // of equal pair counts: when a range's launch ends, the rows of its units are final
        const int64_t U0 = md.w[1], tk0 = md.w[0];
        const int nchunk = U0 >= 16 ? 4 : 1;
        std::vector<int64_t> cut(nchunk + 1, 0);
        cut[nchunk] = U0;
        const double total = (double)U0 * (U0 + 1) / 2.0;
        for (int j = 1; j < nchunk; ++j) {
            int64_t u = 0;
            while (u < U0 && (double)u * (u + 1) / 2.0 < total * j / nchunk) ++u;
            cut[j] = std::max(cut[j - 1], std::min(u, U0));
        }
        for (int j = nchunk - 1; j >= 0; --j) {
            if (cut[j] >= cut[j + 1]) continue;
            opg_into<T>(md, r.cache, Gd, ldg, prec, s, 0, split, cut[j], cut[j + 1]);
            send_rows(md.woff[0] + cut[j] * tk0, md.woff[0] + cut[j + 1] * tk0, true);  // weight rows of the units
            send_rows(md.boff[0] + cut[j], md.boff[0] + cut[j + 1], false);             // their bias rows
        }
        tm.mark("compute");
        CK_CUDA(cudaStreamSynchronize(s));
        CK_CUDA(cudaStreamSynchronize(s2));
        tm.mark("download");
        return;
    }
    opg_into<T>(md, r.cache, dptr<T>(G), ldg, prec, s);
    tm.mark("compute");
    download<T, U>(dptr<T>(G), ldg, md.P, md.P, g_out, s);
    tm.mark("download");
}

template <class T>
void host_jacobian(const ModelDesc& md, const double* params, const double* x, const double* y, int64_t n,
                   double* j_out) {
    if (n < 1) contract("assemble_jacobian: empty batch");
    auto lab = labels_from_onehot(md, y, n);
    cudaStream_t s = lib_stream();
    Resident<T> r;
    upload_and_forward<T>(md, params, x, lab, n, r, s);
    DevMem J;
    int64_t ldj;
    jacobian_full<T>(md, r.cache, J, ldj, s);
    download<T, double>(dptr<T>(J), ldj, n, md.P, j_out, s);
}

template <class T>
void host_grad(const ModelDesc& md, const double* params, const double* x, const double* y, int64_t n, double* g) {
    if (n < 1) contract("forward_backward: empty batch");
    auto lab = labels_from_onehot(md, y, n);
    cudaStream_t s = lib_stream();
    Resident<T> r;
    upload_and_forward<T>(md, params, x, lab, n, r, s);
    DevMem gd((size_t)md.P * sizeof(T), s);
    Engine<T> eng{md, s, kF64};
    eng.grad(r.cache, dptr<T>(gd));
    download<T, double>(dptr<T>(gd), md.P, 1, md.P, g, s);
}

template <class T>
void host_hvp(const ModelDesc& md, const double* params, const double* x, const double* y, int64_t n, const double* v,
              int64_t nv, int prec, double* hv) {
    if (n < 1) contract("forward_backward: empty batch");
    if (nv < 1) shape("hvp: need at least one direction");
    auto lab = labels_from_onehot(md, y, n);
    cudaStream_t s = lib_stream();
    Resident<T> r;
    upload_and_forward<T>(md, params, x, lab, n, r, s);
    DevMem vd((size_t)nv * md.P * sizeof(double), s), vt((size_t)nv * md.P * sizeof(T), s),
        hd((size_t)nv * md.P * sizeof(T), s);
    CK_CUDA(cudaMemcpyAsync(vd.p, v, nv * md.P * sizeof(double), cudaMemcpyHostToDevice, s));
    convert_kernel<T><<<blocks_for(nv * md.P), 256, 0, s>>>(dptr<double>(vd), dptr<T>(vt), nv * md.P);
    CK_LAUNCH();
    Engine<T> eng{md, s, prec};
    eng.hvp(dptr<T>(r.params), r.cache, dptr<T>(vt), nv, md.P, dptr<T>(hd), md.P, T(1) / T(n));
    download<T, double>(dptr<T>(hd), md.P, nv, md.P, hv, s);
}

// opg_eigs_incremental's input contract (eigensolve.cpp:245-251): the rows of
// J from the caller; top-k of G = (1/n) J^T J by the randomized range finder.
template <class T>
void topk_from_j(const T* J, int64_t ldj, int64_t n, int64_t p, int64_t k, int64_t oversample, int64_t power_iters,
                 uint64_t seed, int prec, T* q_dev, std::vector<double>& lam, cudaStream_t s) {
    if (n < 1 || p < 1) shape("opg_eigs: empty Jacobian");
    ModelDesc md{};
    md.P = p;  // no layers: the products run on the caller's J
    Cache<T> c;
    c.n = n;
    topk_core<T>(md, c, k, oversample, power_iters, seed, prec, q_dev, lam, s, nullptr, J, ldj);
}

// per-example cost (model.cpp:216-256): fused log-softmax logsumexp(z) - z_y
// on the logits in fp64, or the raw output (raw_mean_output)
template <class T>
__global__ void example_cost_kernel(const T* __restrict__ z, int64_t ldz, const T* __restrict__ out, int64_t ldo,
                                    const int32_t* __restrict__ labels, int64_t n, int64_t tl, int mode,
                                    double* __restrict__ cost) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    if (mode == kRawMean) {
        cost[r] = (double)out[r * ldo];
        return;
    }
    const T* zr = z + r * ldz;
    double zmax = (double)zr[0];
    for (int64_t m = 1; m < tl; ++m) zmax = fmax(zmax, (double)zr[m]);
    double sum = 0.0;
    for (int64_t m = 0; m < tl; ++m) sum += exp((double)zr[m] - zmax);
    cost[r] = zmax + log(sum) - (double)zr[labels[r]];
}

template <class T>
void host_forward_cost(const ModelDesc& md, const double* params, const double* x, const double* y, int64_t n, int prec,
                       double* out, double* cost) {
    if (n < 1) contract("cost: empty batch");
    auto lab = labels_from_onehot(md, y, n);
    cudaStream_t s = lib_stream();
    Resident<T> r;
    upload_and_forward<T>(md, params, x, lab, n, r, s);
    const int S = md.S;
    const int64_t tl = md.w[S];
    if (out) download<T, double>(r.cache.a[S], r.cache.lda[S], n, tl, out, s);
    if (cost) {
        DevMem cd((size_t)n * sizeof(double), s);
        example_cost_kernel<T><<<(unsigned)ceil_div(n, 128), 128, 0, s>>>(
            r.cache.z[S - 1], r.cache.ldt[S - 1], r.cache.a[S], r.cache.lda[S], dptr<int32_t>(r.labels), n, tl,
            md.mode, dptr<double>(cd));
        CK_LAUNCH();
        std::vector<double> hc(n);
        CK_CUDA(cudaMemcpyAsync(hc.data(), cd.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK_CUDA(cudaStreamSynchronize(s));
        double total = 0.0;
        for (double v : hc) total += v;  // fixed order: deterministic
        *cost = total / (double)n;
    }
    (void)prec;
}

}  // namespace

// ---- helpers of the eigenpair operators (eigensolve.cpp:253-275) ---------------
namespace {

void check_eig_shape(int64_t p, int64_t k, const void* q, const void* lambda, const char* who) {
    if (p < 1 || k < 0 || k > p) shape(std::string(who) + ": bad eigenpair shape");
    if (k > 0 && (!q || !lambda)) contract(std::string(who) + ": null eigenpairs");
}

void check_lambda_tilde(int32_t full_rank, double lambda_tilde) {  // eigensolve.cpp:271-275
    if (full_rank && !(lambda_tilde > 0.0))
        contract("full-rank approximation requires lambda_tilde > 0, got " + std::to_string(lambda_tilde));
}

void check_dense_cap(int64_t p, int64_t cap, const char* who) {  // eigensolve.cpp:255-261
    if (p > cap)
        contract(std::string(who) + ": P = " + std::to_string(p) + " exceeds the dense memory cap " +
                 std::to_string(cap) + "; use the implicit quadform/apply forms instead");
}

// host doubles (rows x cols, dense) -> device T (rows x ld)
template <class T>
DevMem upload_as(const double* h, int64_t rows, int64_t cols, int64_t ld, cudaStream_t s) {
    DevMem out((size_t)std::max<int64_t>(1, rows * ld) * sizeof(T), s);
    if (rows * cols == 0) return out;
    if (std::is_same_v<T, double> && ld == cols) {
        CK_CUDA(cudaMemcpyAsync(out.p, h, (size_t)rows * cols * sizeof(double), cudaMemcpyHostToDevice, s));
        return out;
    }
    DevMem st((size_t)rows * cols * sizeof(double), s);
    CK_CUDA(cudaMemcpyAsync(st.p, h, (size_t)rows * cols * sizeof(double), cudaMemcpyHostToDevice, s));
    if (ld != cols) CK_CUDA(cudaMemsetAsync(out.p, 0, (size_t)rows * ld * sizeof(T), s));
    convert_rows_kernel<double, T><<<blocks_for(rows * cols), 256, 0, s>>>(dptr<double>(st), cols, dptr<T>(out), ld,
                                                                           rows, cols);
    CK_LAUNCH();
    CK_CUDA(cudaStreamSynchronize(s));  // st is released in stream order, h may be pageable
    return out;
}

}  // namespace

extern "C" {

const char* curvkit_last_error(void) { return g_err.c_str(); }
const char* curvkit_version(void) { return "curvkit-b200 0.1 (sm_100a)"; }
int64_t curvkit_launch_count(void) { return ck::g_launches.load(); }

int curvkit_profile_begin(void) {
    return guard([&] {
        Profiler& p = Profiler::get();
        std::lock_guard<std::mutex> g(p.mu);
        for (auto& kv : p.recs)
            for (auto& r : kv.second) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
        p.recs.clear();
        p.on = true;
    });
}

int curvkit_profile_end(char* json_out, int64_t capacity) {
    return guard([&] {
        Profiler& p = Profiler::get();
        std::lock_guard<std::mutex> g(p.mu);
        p.on = false;
        CK_CUDA(cudaDeviceSynchronize());
        std::string js = "{";
        bool first = true;
        for (auto& kv : p.recs) {
            double ms = 0.0, fl = 0.0, by = 0.0;
            for (auto& r : kv.second) {
                float t = 0.f;
                CK_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
                ms += t; fl += r.flops; by += r.bytes;
                cudaEventDestroy(r.a); cudaEventDestroy(r.b);
            }
            char buf[256];
            snprintf(buf, sizeof(buf), "%s\"%s\": {\"ms\": %.6f, \"launches\": %zu, \"flops\": %.6e, \"bytes\": %.6e}",
                     first ? "" : ", ", kv.first.c_str(), ms, kv.second.size(), fl, by);
            js += buf;
            first = false;
        }
        js += "}";
        p.recs.clear();
        if ((int64_t)js.size() + 1 > capacity) throw CurvError(kShapeError, "profile buffer too small");
        std::memcpy(json_out, js.c_str(), js.size() + 1);
    });
}

int curvkit_param_count(const curvkit_model* model, int64_t* p_out) {
    return guard([&] { *p_out = make_desc(model).P; });
}

int curvkit_assemble_jacobian(const curvkit_model* model, const double* params, const double* x, const double* y,
                              int64_t n, int32_t precision, double* j_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (is_f64(precision)) host_jacobian<double>(md, params, x, y, n, j_out);
        else host_jacobian<float>(md, params, x, y, n, j_out);
    });
}

int curvkit_grad_batch(const curvkit_model* model, const double* params, const double* x, const double* y, int64_t n,
                       int32_t precision, double* grad_total_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (is_f64(precision)) host_grad<double>(md, params, x, y, n, grad_total_out);
        else host_grad<float>(md, params, x, y, n, grad_total_out);
    });
}

int curvkit_hvp(const curvkit_model* model, const double* params, const double* x, const double* y, int64_t n,
                const double* v, int64_t nvec, int32_t precision, double* hv_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (is_f64(precision)) host_hvp<double>(md, params, x, y, n, v, nvec, precision, hv_out);
        else host_hvp<float>(md, params, x, y, n, v, nvec, precision, hv_out);
    });
}

int curvkit_hvp_operator_apply(const curvkit_model* model, const double* params, const double* x, const double* y,
                               int64_t n, int64_t batch_size, const double* v, int64_t nvec, int32_t precision,
                               double* hv_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        // autodiff.cpp:266-280; equal mini-batches average to the full mean
        if (batch_size < 1) contract("HvpOperator: batch size must be >= 1");
        if (n == 0) contract("HvpOperator: empty dataset");
        if (n % batch_size != 0)
            contract("HvpOperator: dataset size " + std::to_string(n) + " is not divisible by batch size " +
                     std::to_string(batch_size) + "; refusing to drop the remainder");
        if (is_f64(precision)) host_hvp<double>(md, params, x, y, n, v, nvec, precision, hv_out);
        else host_hvp<float>(md, params, x, y, n, v, nvec, precision, hv_out);
    });
}

// curv::forward (model.cpp:178-199) for n examples at once: out n x T_L
// (softmax probabilities, or the raw output for raw_mean_output).
int curvkit_forward(const curvkit_model* model, const double* params, const double* x, int64_t n, int32_t precision,
                    double* out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (!out) contract("forward: null output");
        std::vector<double> y;
        if (md.mode == kSoftmaxCE) {  // the forward pass needs no labels: any one-hot row
            y.assign((size_t)n * md.w[md.L - 1], 0.0);
            for (int64_t r = 0; r < n; ++r) y[r * md.w[md.L - 1]] = 1.0;
        }
        if (is_f64(precision)) host_forward_cost<double>(md, params, x, y.empty() ? nullptr : y.data(), n, precision, out, nullptr);
        else host_forward_cost<float>(md, params, x, y.empty() ? nullptr : y.data(), n, precision, out, nullptr);
    });
}

// curv::cost (model.cpp:216-256): mean fused log-softmax cross-entropy (or
// mean raw output).
int curvkit_cost(const curvkit_model* model, const double* params, const double* x, const double* y, int64_t n,
                 int32_t precision, double* cost_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (!cost_out) contract("cost: null output");
        if (is_f64(precision)) host_forward_cost<double>(md, params, x, y, n, precision, nullptr, cost_out);
        else host_forward_cost<float>(md, params, x, y, n, precision, nullptr, cost_out);
    });
}

int curvkit_hessian_topk_lanczos(const curvkit_model* model, const double* params, const double* x, const double* y,
                                 int64_t n, int64_t batch_size, int64_t k, int64_t max_iterations,
                                 double residual_tol, uint64_t seed, int32_t precision, double* q_out,
                                 double* lambda_out, double* residuals_out, int64_t* iterations_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        // the HvpOperator the reference hands to lanczos_topk (autodiff.cpp:266-280)
        if (batch_size < 1) contract("HvpOperator: batch size must be >= 1");
        if (n == 0) contract("HvpOperator: empty dataset");
        if (n % batch_size != 0)
            contract("HvpOperator: dataset size " + std::to_string(n) + " is not divisible by batch size " +
                     std::to_string(batch_size) + "; refusing to drop the remainder");
        // lanczos_topk's own preconditions (eigensolve.cpp:47-53), before any device work
        if (md.P < 2) contract("lanczos_topk: operator dimension must be >= 2");
        if (k < 1 || k >= md.P)
            contract("lanczos_topk: need 1 <= k < p, got k = " + std::to_string(k) + ", p = " + std::to_string(md.P));
        if (max_iterations < k) contract("lanczos_topk: max_iterations must be >= k");
        if (!(residual_tol > 0.0)) contract("lanczos_topk: residual_tol must be > 0");
        auto lab = labels_from_onehot(md, y, n);
        cudaStream_t s = lib_stream();
        auto run = [&](auto tag) {
            using T = decltype(tag);
            Resident<T> r;
            upload_and_forward<T>(md, params, x, lab, n, r, s);
            LanczosOut o = lanczos_topk<T>(md, dptr<T>(r.params), r.cache, k, max_iterations, residual_tol, seed,
                                           precision, s);
            if (iterations_out) *iterations_out = o.iterations;
            if (residuals_out)
                for (int64_t i = 0; i < (int64_t)o.residuals.size() && i < k; ++i) residuals_out[i] = o.residuals[i];
            if (!o.converged)
                throw CurvError(kConvergenceError, "lanczos_topk: not converged within " +
                                                       std::to_string(std::min(max_iterations, md.P)) + " iterations");
            if (q_out) std::copy(o.q.begin(), o.q.end(), q_out);
            if (lambda_out) std::copy(o.lambda.begin(), o.lambda.end(), lambda_out);
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

int curvkit_assemble_hessian(const curvkit_model* model, const double* params, const double* x, const double* y,
                             int64_t n, const curvkit_curvature_config* cfg, int32_t precision, int32_t verify,
                             double* h_out, double* asymmetry_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (is_f64(precision))
            host_hessian<double, double>(md, params, x, y, n, cfg, precision, verify != 0, h_out, asymmetry_out);
        else
            host_hessian<float, double>(md, params, x, y, n, cfg, precision, verify != 0, h_out, asymmetry_out);
    });
}

int curvkit_assemble_hessian_f32(const curvkit_model* model, const double* params, const double* x, const double* y,
                                 int64_t n, const curvkit_curvature_config* cfg, int32_t precision, float* h_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (is_f64(precision)) host_hessian<double, float>(md, params, x, y, n, cfg, precision, false, h_out, nullptr);
        else host_hessian<float, float>(md, params, x, y, n, cfg, precision, false, h_out, nullptr);
    });
}

int curvkit_assemble_opg(const curvkit_model* model, const double* params, const double* x, const double* y,
                         int64_t n, const curvkit_curvature_config* cfg, int32_t precision, double* g_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (is_f64(precision)) host_opg<double, double>(md, params, x, y, n, cfg, precision, g_out);
        else host_opg<float, double>(md, params, x, y, n, cfg, precision, g_out);
    });
}

int curvkit_assemble_opg_f32(const curvkit_model* model, const double* params, const double* x, const double* y,
                             int64_t n, const curvkit_curvature_config* cfg, int32_t precision, float* g_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (is_f64(precision)) host_opg<double, float>(md, params, x, y, n, cfg, precision, g_out);
        else host_opg<float, float>(md, params, x, y, n, cfg, precision, g_out);
    });
}

int curvkit_opg_topk(const curvkit_model* model, const double* params, const double* x, const double* y, int64_t n,
                     int64_t k, int64_t oversample, int64_t power_iters, uint64_t seed, int32_t precision,
                     double* q_out, double* lambda_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk: empty dataset");
        auto lab = labels_from_onehot(md, y, n);
        cudaStream_t s = lib_stream();
        if (is_f64(precision)) {
            Resident<double> r;
            upload_and_forward<double>(md, params, x, lab, n, r, s);
            host_topk<double>(md, r.cache, k, oversample, power_iters, seed, precision, q_out, lambda_out, s);
        } else {
            Resident<float> r;
            upload_and_forward<float>(md, params, x, lab, n, r, s);
            host_topk<float>(md, r.cache, k, oversample, power_iters, seed, precision, q_out, lambda_out, s);
        }
    });
}

int curvkit_opg_topk_filtered(const curvkit_model* model, const double* params, const double* x, const double* y,
                              int64_t n, int64_t k, int64_t oversample, int64_t filter_steps, int64_t filter_degree,
                              uint64_t seed, int32_t precision, double* q_out, double* lambda_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk_filtered: empty dataset");
        if (filter_degree < 1) contract("opg_topk_filtered: filter_degree must be >= 1");
        auto lab = labels_from_onehot(md, y, n);
        cudaStream_t s = lib_stream();
        if (is_f64(precision)) {
            Resident<double> r;
            upload_and_forward<double>(md, params, x, lab, n, r, s);
            host_topk<double>(md, r.cache, k, oversample, 0, seed, precision, q_out, lambda_out, s, filter_steps,
                              filter_degree);
        } else {
            Resident<float> r;
            upload_and_forward<float>(md, params, x, lab, n, r, s);
            host_topk<float>(md, r.cache, k, oversample, 0, seed, precision, q_out, lambda_out, s, filter_steps,
                             filter_degree);
        }
    });
}

// ---- device entry points -----------------------------------------------------
int curvkit_dev_assemble_hessian(const curvkit_model* model, const void* params, const void* x, const int32_t* labels,
                                 int64_t n, int32_t precision, void* h, int64_t ldh, void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("assemble_hessian: empty dataset");
        cudaStream_t s = dev_stream(stream);
        if (is_f64(precision)) {
            Cache<double> c;
            forward_device<double>(md, (const double*)params, (const double*)x, labels, n, c, s);
            hessian_into<double>(md, (const double*)params, c, (double*)h, ldh, precision, false, s);
        } else {
            Cache<float> c;
            forward_device<float>(md, (const float*)params, (const float*)x, labels, n, c, s);
            hessian_into<float>(md, (const float*)params, c, (float*)h, ldh, precision, false, s);
        }
    });
}

int curvkit_dev_assemble_opg(const curvkit_model* model, const void* params, const void* x, const int32_t* labels,
                             int64_t n, int32_t precision, void* g, int64_t ldg, void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("assemble_opg: empty dataset");
        cudaStream_t s = dev_stream(stream);
        auto run = [&](auto tag) {
            using T = decltype(tag);
            Cache<T> c;
            forward_device<T>(md, (const T*)params, (const T*)x, labels, n, c, s);
            opg_into<T>(md, c, (T*)g, ldg, precision, s);
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

int curvkit_dev_assemble_jacobian(const curvkit_model* model, const void* params, const void* x,
                                  const int32_t* labels, int64_t n, int32_t precision, void* j, int64_t ldj,
                                  void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("assemble_jacobian: empty batch");
        cudaStream_t s = dev_stream(stream);
        auto run = [&](auto tag) {
            using T = decltype(tag);
            Cache<T> c;
            forward_device<T>(md, (const T*)params, (const T*)x, labels, n, c, s);
            jacobian<T>(md, c, 0, n, (T*)j, ldj, s);
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

// ---- unit bands (multi-GPU H and G, bands.cuh) ---------------------------------
int curvkit_shard_units(const curvkit_model* model, int64_t nshards, int64_t shard, int64_t* unit_begin,
                        int64_t* unit_end, int64_t* band_rows) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        const UnitBand b = UnitBand::make(md, nshards, shard);
        for (int k = 0; k < md.S; ++k) {
            if (unit_begin) unit_begin[k] = b.u0[k];
            if (unit_end) unit_end[k] = b.u1[k];
        }
        if (band_rows) *band_rows = b.rows;
    });
}

int curvkit_dev_assemble_band(const curvkit_model* model, int32_t product, const void* params, const void* x,
                              const int32_t* labels, int64_t n, int32_t precision, int64_t nshards, int64_t shard,
                              void* band, int64_t ld, void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("assemble_band: empty dataset");
        if (product != 0 && product != 1) contract("assemble_band: product must be 0 (Hessian) or 1 (OPG)");
        if (!tf32_class(precision)) contract("unit-band assembly needs TF32 precision");
        if (ld < md.P || ld % 4) contract("assemble_band: ld must be >= P and a multiple of 4");
        const UnitBand b = UnitBand::make(md, nshards, shard);
        if (b.rows == 0) return;
        cudaStream_t s = dev_stream(stream);
        Cache<float> c;
        forward_device<float>(md, (const float*)params, (const float*)x, labels, n, c, s);
        Engine<float> eng{md, s, precision};
        if (product == 0) eng.hessian((const float*)params, c, (float*)band, ld, false, 0, INT64_MAX, &b);
        else eng.opg_kr(c, (float*)band, ld, 0, INT64_MAX, &b);
    });
}

int curvkit_dev_band_scatter(const curvkit_model* model, int32_t precision, int64_t nshards, int64_t shard,
                             const void* band, int64_t ld, void* full, int64_t ldf, void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        const UnitBand b = UnitBand::make(md, nshards, shard);
        if (ld < md.P || ldf < md.P) contract("band_scatter: leading dimensions must be >= P");
        cudaStream_t s = dev_stream(stream);
        if (is_f64(precision)) band_scatter<double>(md, b, (const double*)band, ld, (double*)full, ldf, s);
        else band_scatter<float>(md, b, (const float*)band, ld, (float*)full, ldf, s);
    });
}

int curvkit_dev_symmetrize_units(const curvkit_model* model, int32_t precision, void* full, int64_t ldf, void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (ldf < md.P) contract("symmetrize_units: ldf must be >= P");
        cudaStream_t s = dev_stream(stream);
        if (is_f64(precision)) symmetrize_units<double>(md, (double*)full, ldf, s);
        else symmetrize_units<float>(md, (float*)full, ldf, s);
    });
}

// ---- operators on eigenpairs (eigensolve.cpp:11-30, 253-358) -----------------

int curvkit_eig_validate(int64_t p, int64_t k, const double* q, const double* lambda, int64_t lambda_len,
                         double ortho_tol) {
    return guard([&] {
        if (lambda_len != k) shape("EigenPairs: lambda length does not match column count");
        if (k > p) shape("EigenPairs: more columns than rows");
        if (k < 0 || p < 0) shape("EigenPairs: bad shape");
        if (k == 0) return;
        if (!q || !lambda) contract("EigenPairs: null eigenpairs");
        for (int64_t i = 0; i + 1 < k; ++i)
            if (lambda[i] < lambda[i + 1]) contract("EigenPairs: eigenvalues not sorted descending");
        cudaStream_t s = lib_stream();
        DevMem qd = upload_as<double>(q, p, k, k, s);
        const double err = eigops::ortho_error<double>(s, p, k, dptr<double>(qd), k);
        if (!(err <= ortho_tol)) contract("EigenPairs: columns are not orthonormal");
    });
}

int curvkit_eig_materialize(int64_t p, int64_t k, const double* q, const double* lambda, int32_t full_rank,
                            double lambda_tilde, int64_t memory_cap, int32_t precision, double* h_out) {
    return guard([&] {
        const char* who = full_rank ? "full_rank_materialize" : "low_rank_materialize";
        check_lambda_tilde(full_rank, lambda_tilde);
        check_eig_shape(p, k, q, lambda, who);
        check_dense_cap(p, memory_cap, who);
        if (!h_out) contract(std::string(who) + ": null output");
        const bool f64 = is_f64(precision);
        cudaStream_t s = lib_stream();
        auto run = [&](auto tag) {
            using T = decltype(tag);
            const int64_t ldq = round_up(std::max<int64_t>(k, 1), 4), ldh = round_up(p, 32);  // 128-byte row pitch
            DevMem qd = upload_as<T>(q, p, k, ldq, s), ld = upload_as<T>(lambda, 1, k, k, s);
            DevMem H((size_t)p * ldh * sizeof(T), s);
            if (k == 0) CK_CUDA(cudaMemsetAsync(H.p, 0, (size_t)p * ldh * sizeof(T), s));
            eigops::materialize<T>(precision, s, p, k, dptr<T>(qd), ldq, dptr<T>(ld), full_rank != 0, lambda_tilde,
                                   dptr<T>(H), ldh);
            download<T, double>(dptr<T>(H), ldh, p, p, h_out, s);
        };
        if (f64) run(double{});
        else run(float{});
    });
}

int curvkit_eig_apply(int64_t p, int64_t k, const double* q, const double* lambda, int32_t full_rank,
                      double lambda_tilde, int64_t nvec, const double* x, int64_t x_len, int32_t precision,
                      double* y_out, double* quad_out) {
    return guard([&] {
        check_lambda_tilde(full_rank, lambda_tilde);
        check_eig_shape(p, k, q, lambda, "eigen operator");
        if (x_len != p)  // eigensolve.cpp:263-269
            shape("eigen operator: vector length " + std::to_string(x_len) + " does not match P = " +
                  std::to_string(p));
        if (nvec < 1) return;
        if (!x) contract("eigen operator: null vector");
        const bool f64 = is_f64(precision);
        cudaStream_t s = lib_stream();
        auto run = [&](auto tag) {
            using T = decltype(tag);
            const int64_t ldq = round_up(std::max<int64_t>(k, 1), 4);
            DevMem qd = upload_as<T>(q, p, k, ldq, s), ld = upload_as<T>(lambda, 1, k, k, s);
            DevMem xd = upload_as<T>(x, nvec, p, p, s);
            DevMem yd((size_t)(y_out ? nvec * p : 1) * sizeof(T), s), qf((size_t)nvec * sizeof(double), s);
            eigops::apply<T>(s, p, k, dptr<T>(qd), ldq, dptr<T>(ld), full_rank != 0, lambda_tilde, nvec, dptr<T>(xd),
                             p, y_out ? dptr<T>(yd) : nullptr, p, quad_out ? dptr<double>(qf) : nullptr);
            if (y_out) download<T, double>(dptr<T>(yd), p, nvec, p, y_out, s);
            if (quad_out) {
                CK_CUDA(cudaMemcpyAsync(quad_out, qf.p, (size_t)nvec * sizeof(double), cudaMemcpyDeviceToHost, s));
                CK_CUDA(cudaStreamSynchronize(s));
            }
        };
        if (f64) run(double{});
        else run(float{});
    });
}

int curvkit_dev_eig_materialize(int64_t p, int64_t k, const void* q, int64_t ldq, const void* lambda,
                                int32_t full_rank, double lambda_tilde, int32_t precision, void* h, int64_t ldh,
                                void* stream) {
    return guard([&] {
        const char* who = full_rank ? "full_rank_materialize" : "low_rank_materialize";
        check_lambda_tilde(full_rank, lambda_tilde);
        check_eig_shape(p, k, q, lambda, who);
        if (!h || ldh < p || ldq < k) shape(std::string(who) + ": bad leading dimension or null output");
        const bool f64 = is_f64(precision);
        cudaStream_t s = dev_stream(stream);
        if (k == 0) CK_CUDA(cudaMemsetAsync(h, 0, (size_t)p * ldh * (f64 ? 8 : 4), s));
        if (f64)
            eigops::materialize<double>(precision, s, p, k, (const double*)q, ldq, (const double*)lambda, full_rank != 0,
                                        lambda_tilde, (double*)h, ldh);
        else
            eigops::materialize<float>(precision, s, p, k, (const float*)q, ldq, (const float*)lambda, full_rank != 0,
                                       lambda_tilde, (float*)h, ldh);
    });
}

int curvkit_dev_eig_apply(int64_t p, int64_t k, const void* q, int64_t ldq, const void* lambda, int32_t full_rank,
                          double lambda_tilde, int64_t nvec, const void* x, int64_t ldx, void* y, int64_t ldy,
                          double* quad, int32_t precision, void* stream) {
    return guard([&] {
        check_lambda_tilde(full_rank, lambda_tilde);
        check_eig_shape(p, k, q, lambda, "eigen operator");
        if (nvec < 1) return;
        if (!x || ldx < p || ldq < k || (y && ldy < p)) shape("eigen operator: bad leading dimension or null vector");
        cudaStream_t s = dev_stream(stream);
        if (is_f64(precision))
            eigops::apply<double>(s, p, k, (const double*)q, ldq, (const double*)lambda, full_rank != 0, lambda_tilde,
                                  nvec, (const double*)x, ldx, (double*)y, ldy, quad);
        else
            eigops::apply<float>(s, p, k, (const float*)q, ldq, (const float*)lambda, full_rank != 0, lambda_tilde,
                                 nvec, (const float*)x, ldx, (float*)y, ldy, quad);
    });
}

int curvkit_dev_gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda, int32_t a_kmajor,
                     const float* b, int64_t ldb, int32_t b_kmajor, float* c, int64_t ldc, float alpha,
                     int32_t precision, void* stream) {
    return guard([&] {
        if (m < 0 || n < 0 || k < 1) shape("dev_gemm: bad shape");
        if (precision == kF64) contract("dev_gemm: fp32 storage only");
        cudaStream_t s = dev_stream(stream);
        EpiStore<float> e{c, ldc, 0, alpha, 0.f};
        Opnd<float> A = a_kmajor ? kmaj(a, lda) : mnmaj(a, lda);
        Opnd<float> B = b_kmajor ? kmaj(b, ldb) : mnmaj(b, ldb);
        if (tf32_class(precision) || precision == k3xTF32) gemm_tf32_store(tc_form(precision), s, m, n, k, A, B, c, ldc, alpha);
        else CurvGemm<float, EpiStore<float>>::run(precision, s, m, n, k, A, B, e);
    });
}

struct curvkit_incr_opg_s {
    ck::IncrOpg st;
    int dev;
};

int curvkit_incr_opg_create(int64_t p, int64_t k, curvkit_incr_opg* out) {
    return guard([&] {
        if (!out) contract("incr_opg_create: null output");
        ck::IncrOpg st(p, k);  // the reference's k range check, before any device work
        int dev = 0;
        CK_CUDA(cudaGetDevice(&dev));
        *out = new curvkit_incr_opg_s{std::move(st), dev};
    });
}

int curvkit_incr_opg_push_block(curvkit_incr_opg h, const double* block, int64_t rows) {
    return guard([&] {
        if (!h) contract("incr_opg_push_block: null handle");
        if (rows >= 1 && !block) contract("incr_opg_push_block: null block");
        CK_CUDA(cudaSetDevice(h->dev));
        h->st.push(block, rows, h->st.p, cudaMemcpyHostToDevice, lib_stream());
    });
}

int curvkit_incr_opg_dev_push_block(curvkit_incr_opg h, const void* block, int64_t rows, int64_t ld, void* stream) {
    return guard([&] {
        if (!h) contract("incr_opg_push_block: null handle");
        if (rows >= 1 && !block) contract("incr_opg_push_block: null block");
        h->st.push(static_cast<const double*>(block), rows, ld, cudaMemcpyDeviceToDevice, dev_stream(stream));
    });
}

int curvkit_incr_opg_counts(curvkit_incr_opg h, int64_t* rows_seen, int64_t* updates) {
    return guard([&] {
        if (!h) contract("incr_opg_counts: null handle");
        if (rows_seen) *rows_seen = h->st.rows_seen;
        if (updates) *updates = h->st.updates;
    });
}

int curvkit_incr_opg_finalize(curvkit_incr_opg h, int64_t n_total, double* q_out, double* lambda_out) {
    return guard([&] {
        if (!h) contract("incr_opg_finalize: null handle");
        CK_CUDA(cudaSetDevice(h->dev));
        h->st.finalize(n_total, q_out, lambda_out, cudaMemcpyDeviceToHost, lib_stream());
    });
}

int curvkit_incr_opg_dev_finalize(curvkit_incr_opg h, int64_t n_total, void* q, void* lambda, void* stream) {
    return guard([&] {
        if (!h) contract("incr_opg_finalize: null handle");
        h->st.finalize(n_total, static_cast<double*>(q), static_cast<double*>(lambda), cudaMemcpyDeviceToDevice,
                       dev_stream(stream));
    });
}

int curvkit_incr_opg_destroy(curvkit_incr_opg h) {
    return guard([&] { delete h; });
}

struct curvkit_comm_s {
    ck::Comm c;
};

int curvkit_comm_unique_id(uint8_t* id_out) {
    return guard([&] {
        if (!id_out) contract("comm_unique_id: null output");
        ncclUniqueId id;
        nccl_check(NcclApi::get().get_unique_id(&id), "ncclGetUniqueId");
        static_assert(sizeof(id.internal) == CURVKIT_COMM_ID_BYTES, "NCCL unique id size");
        std::memcpy(id_out, id.internal, CURVKIT_COMM_ID_BYTES);
    });
}

int curvkit_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, curvkit_comm* out) {
    return guard([&] {
        if (!id || !out) contract("comm_init: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) contract("comm_init: need 0 <= rank < nranks");
        ncclUniqueId u;
        std::memcpy(u.internal, id, CURVKIT_COMM_ID_BYTES);
        ncclComm_t c = nullptr;
        nccl_check(NcclApi::get().comm_init_rank(&c, nranks, u, rank), "ncclCommInitRank");
        ck::Comm cm;
        cm.comm = c;
        cm.rank = rank;
        cm.nranks = nranks;
        const char* lb = getenv("CURVKIT_COMM_LOOPBACK");
        cm.loopback = nranks == 1 && lb && lb[0] == '1';
        *out = new curvkit_comm_s{cm};
    });
}

int curvkit_comm_init_host(int32_t nranks, int32_t rank, curvkit_host_allreduce_fn allreduce,
                           curvkit_host_gather_fn gather, void* user, curvkit_comm* out) {
    return guard([&] {
        if (!out || !allreduce || !gather) contract("comm_init_host: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) contract("comm_init_host: need 0 <= rank < nranks");
        ck::Comm c;
        c.h_sum = allreduce;
        c.h_gather = gather;
        c.user = user;
        c.rank = rank;
        c.nranks = nranks;
        *out = new curvkit_comm_s{c};
    });
}

int curvkit_dev_gather_bands(const curvkit_model* model, int32_t precision, const void* band, int64_t ld, void* full,
                             int64_t ldf, void* stream, curvkit_comm comm) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (!comm) contract("gather_bands: null communicator");
        const ck::Comm& cm = comm->c;
        if (ld < md.P || ld != ldf) contract("gather_bands: ld must be >= P and equal ldf");
        if (cm.rank == 0 && !full) contract("gather_bands: rank 0 needs the full output");
        cudaStream_t s = dev_stream(stream);
        const size_t es = is_f64(precision) ? 8 : 4;
        std::vector<UnitBand> bands;
        std::vector<int64_t> bytes;
        for (int r = 0; r < cm.nranks; ++r) {
            bands.push_back(UnitBand::make(md, cm.nranks, r));
            bytes.push_back(bands.back().rows * ld * (int64_t)es);
        }
        // rank 0 receives every band into a staging buffer laid out band after
        // band, then scatters the rows and mirrors the upper unit-major triangle
        const int64_t total = std::accumulate(bytes.begin(), bytes.end(), int64_t(0));
        DevMem stage(cm.rank == 0 ? (size_t)total : 0, s);
        cm.gather(band, bytes, stage.p, 0, s);
        if (cm.rank != 0) return;
        int64_t off = 0;
        for (int r = 0; r < cm.nranks; ++r) {
            const uint8_t* src = static_cast<const uint8_t*>(stage.p) + off;
            if (es == 8) band_scatter<double>(md, bands[r], (const double*)src, ld, (double*)full, ldf, s);
            else band_scatter<float>(md, bands[r], (const float*)src, ld, (float*)full, ldf, s);
            off += bytes[r];
        }
        if (es == 8) symmetrize_units<double>(md, (double*)full, ldf, s);
        else symmetrize_units<float>(md, (float*)full, ldf, s);
    });
}

int curvkit_comm_destroy(curvkit_comm comm) {
    return guard([&] {
        if (!comm) return;
        if (comm->c.comm) nccl_check(NcclApi::get().comm_destroy(comm->c.comm), "ncclCommDestroy");
        delete comm;
    });
}

int curvkit_topk_shard_rows(const curvkit_model* model, int64_t nshards, int64_t shard, int64_t* p_begin,
                            int64_t* p_end) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (nshards < 1 || shard < 0 || shard >= nshards) contract("topk_shard_rows: need 0 <= shard < nshards");
        const TopkShard t = TopkShard::make(md, nshards, shard);
        if (p_begin) *p_begin = t.p0;
        if (p_end) *p_end = t.p1;
    });
}

int curvkit_dev_jacobian_apply(const curvkit_model* model, const void* params, const void* x, const int32_t* labels,
                               int64_t n, int32_t precision, int64_t p_begin, int64_t p_end, int32_t transpose,
                               const void* in, int64_t ld_in, int64_t l, void* out, int64_t ld_out, void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1 || l < 1) contract("jacobian_apply: empty operand");
        if (!tf32_class(precision)) contract("jacobian_apply needs TF32 precision");
        if (ld_in % 32 || (transpose && ld_in < l) || (!transpose && ld_in < l))
            contract("jacobian_apply: the input pitch must be a multiple of 32 and >= l");
        cudaStream_t s = dev_stream(stream);
        const TopkShard sh = TopkShard::range(md, p_begin, p_end);
        Cache<float> c;
        forward_device<float>(md, (const float*)params, (const float*)x, labels, n, c, s);
        if (!kr_supported(md, c)) contract("jacobian_apply: unsupported cache layout");
        KrOperands op(md, c, s, precision == kF16S);
        if (transpose)
            kr_apply_jt(md, c, op, sh, (const float*)in, ld_in, l, (float*)out, ld_out, s);
        else
            kr_apply_j(md, c, op, sh, (const float*)in, ld_in, l, (float*)out, ld_out, s);
    });
}

int curvkit_dev_opg_topk_sharded(const curvkit_model* model, const void* params, const void* x,
                                 const int32_t* labels, int64_t n, int64_t k, int64_t oversample,
                                 int64_t power_iters, uint64_t seed, int32_t precision, void* q, void* lambda,
                                 void* stream, curvkit_comm comm) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk: empty dataset");
        if (!comm) contract("opg_topk_sharded: null communicator");
        cudaStream_t s = dev_stream(stream);
        if (!tf32_class(precision)) contract("sharded opg_topk needs TF32 precision");
        Cache<float> c;
        forward_device<float>(md, (const float*)params, (const float*)x, labels, n, c, s);
        dev_topk<float>(md, c, k, oversample, power_iters, seed, precision, (float*)q, (float*)lambda, s, &comm->c);
    });
}

int curvkit_dev_opg_topk_sharded_filtered(const curvkit_model* model, const void* params, const void* x,
                                          const int32_t* labels, int64_t n, int64_t k, int64_t oversample,
                                          int64_t filter_steps, int64_t filter_degree, uint64_t seed,
                                          int32_t precision, void* q, void* lambda, void* stream, curvkit_comm comm) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk: empty dataset");
        if (!comm) contract("opg_topk_sharded: null communicator");
        if (filter_degree < 1) contract("opg_topk_filtered: filter_degree must be >= 1");
        cudaStream_t s = dev_stream(stream);
        if (!tf32_class(precision)) contract("sharded opg_topk needs TF32 precision");
        Cache<float> c;
        forward_device<float>(md, (const float*)params, (const float*)x, labels, n, c, s);
        dev_topk<float>(md, c, k, oversample, 0, seed, precision, (float*)q, (float*)lambda, s, &comm->c, filter_steps,
                        filter_degree);
    });
}

int curvkit_dev_opg_topk_sharded_auto(const curvkit_model* model, const void* params, const void* x,
                                      const int32_t* labels, int64_t n, int64_t k, int64_t oversample, double tol,
                                      int64_t max_applications, uint64_t seed, int32_t precision, void* q,
                                      void* lambda, void* stream, curvkit_comm comm) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk: empty dataset");
        if (!comm) contract("opg_topk_sharded: null communicator");
        if (!(tol > 0.0) || max_applications < 1) contract("opg_topk_auto: need tol > 0 and max_applications >= 1");
        if (!tf32_class(precision)) contract("sharded opg_topk needs TF32 precision");
        cudaStream_t s = dev_stream(stream);
        Cache<float> c;
        forward_device<float>(md, (const float*)params, (const float*)x, labels, n, c, s);
        dev_topk<float>(md, c, k, oversample, 0, seed, precision, (float*)q, (float*)lambda, s, &comm->c,
                        ceil_div(max_applications, kAutoDegree), kAutoDegree, tol);
    });
}

int curvkit_opg_topk_from_jacobian(const double* j, int64_t n, int64_t p, int64_t k, int64_t oversample,
                                   int64_t power_iters, uint64_t seed, int32_t precision, double* q_out,
                                   double* lambda_out) {
    return guard([&] {
        if (!j) contract("opg_eigs: null Jacobian");
        cudaStream_t s = lib_stream();
        auto run = [&](auto tag) {
            using T = decltype(tag);
            const int64_t ld = round_up(p, 32);
            DevMem jd((size_t)n * p * sizeof(double), s), jt((size_t)n * ld * sizeof(T), s);
            CK_CUDA(cudaMemcpyAsync(jd.p, j, (size_t)n * p * sizeof(double), cudaMemcpyHostToDevice, s));
            CK_CUDA(cudaMemsetAsync(jt.p, 0, (size_t)n * ld * sizeof(T), s));
            convert_rows_kernel<double, T><<<blocks_for(n * p), 256, 0, s>>>(dptr<double>(jd), p, dptr<T>(jt), ld, n, p);
            CK_LAUNCH();
            DevMem q((size_t)p * k * sizeof(T), s);
            std::vector<double> lam;
            topk_from_j<T>(dptr<T>(jt), ld, n, p, k, oversample, power_iters, seed, precision, dptr<T>(q), lam, s);
            std::vector<T> hq((size_t)p * k);
            CK_CUDA(cudaMemcpyAsync(hq.data(), q.p, hq.size() * sizeof(T), cudaMemcpyDeviceToHost, s));
            CK_CUDA(cudaStreamSynchronize(s));
            for (size_t i = 0; i < hq.size(); ++i) q_out[i] = (double)hq[i];
            for (int64_t i = 0; i < k; ++i) lambda_out[i] = lam[i];
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

int curvkit_dev_opg_topk_from_jacobian(const void* j, int64_t ldj, int64_t n, int64_t p, int64_t k,
                                       int64_t oversample, int64_t power_iters, uint64_t seed, int32_t precision,
                                       void* q, void* lambda, void* stream) {
    return guard([&] {
        if (!j) contract("opg_eigs: null Jacobian");
        if (ldj < p || ldj % 4) contract("opg_eigs: ldj must be >= p and a multiple of 4");
        cudaStream_t s = dev_stream(stream);
        auto run = [&](auto tag) {
            using T = decltype(tag);
            std::vector<double> lam;
            topk_from_j<T>((const T*)j, ldj, n, p, k, oversample, power_iters, seed, precision, (T*)q, lam, s);
            std::vector<T> hl(lam.begin(), lam.end());
            CK_CUDA(cudaMemcpyAsync(lambda, hl.data(), k * sizeof(T), cudaMemcpyHostToDevice, s));
            CK_CUDA(cudaStreamSynchronize(s));
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

int curvkit_dev_opg_topk(const curvkit_model* model, const void* params, const void* x, const int32_t* labels,
                         int64_t n, int64_t k, int64_t oversample, int64_t power_iters, uint64_t seed,
                         int32_t precision, void* q, void* lambda, void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk: empty dataset");
        cudaStream_t s = dev_stream(stream);
        auto run = [&](auto tag) {
            using T = decltype(tag);
            Cache<T> c;
            forward_device<T>(md, (const T*)params, (const T*)x, labels, n, c, s);
            dev_topk<T>(md, c, k, oversample, power_iters, seed, precision, (T*)q, (T*)lambda, s);
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

int curvkit_dev_opg_topk_auto(const curvkit_model* model, const void* params, const void* x, const int32_t* labels,
                              int64_t n, int64_t k, int64_t oversample, double tol, int64_t max_applications,
                              uint64_t seed, int32_t precision, void* q, void* lambda, void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk_auto: empty dataset");
        if (!(tol > 0.0) || max_applications < 1) contract("opg_topk_auto: need tol > 0 and max_applications >= 1");
        cudaStream_t s = dev_stream(stream);
        auto run = [&](auto tag) {
            using T = decltype(tag);
            Cache<T> c;
            forward_device<T>(md, (const T*)params, (const T*)x, labels, n, c, s);
            dev_topk<T>(md, c, k, oversample, 0, seed, precision, (T*)q, (T*)lambda, s, nullptr,
                        ceil_div(max_applications, kAutoDegree), kAutoDegree, tol);
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

int curvkit_opg_topk_auto(const curvkit_model* model, const double* params, const double* x, const double* y,
                          int64_t n, int64_t k, int64_t oversample, double tol, int64_t max_applications,
                          uint64_t seed, int32_t precision, double* q_out, double* lambda_out) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk_auto: empty dataset");
        if (!(tol > 0.0) || max_applications < 1) contract("opg_topk_auto: need tol > 0 and max_applications >= 1");
        auto lab = labels_from_onehot(md, y, n);
        cudaStream_t s = lib_stream();
        auto run = [&](auto tag) {
            using T = decltype(tag);
            Resident<T> r;
            upload_and_forward<T>(md, params, x, lab, n, r, s);
            host_topk<T>(md, r.cache, k, oversample, 0, seed, precision, q_out, lambda_out, s,
                         ceil_div(max_applications, kAutoDegree), kAutoDegree, tol);
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

int curvkit_dev_opg_topk_filtered(const curvkit_model* model, const void* params, const void* x,
                                  const int32_t* labels, int64_t n, int64_t k, int64_t oversample, int64_t filter_steps,
                                  int64_t filter_degree, uint64_t seed, int32_t precision, void* q, void* lambda,
                                  void* stream) {
    return guard([&] {
        ModelDesc md = make_desc(model);
        if (n < 1) contract("opg_topk_filtered: empty dataset");
        if (filter_degree < 1) contract("opg_topk_filtered: filter_degree must be >= 1");
        cudaStream_t s = dev_stream(stream);
        auto run = [&](auto tag) {
            using T = decltype(tag);
            Cache<T> c;
            forward_device<T>(md, (const T*)params, (const T*)x, labels, n, c, s);
            dev_topk<T>(md, c, k, oversample, 0, seed, precision, (T*)q, (T*)lambda, s, nullptr, filter_steps,
                        filter_degree);
        };
        if (is_f64(precision)) run(double{});
        else run(float{});
    });
}

int curvkit_dev_eig_apply_sharded(int64_t p_local, int64_t k, const void* q, int64_t ldq, const void* lambda,
                                  int32_t full_rank, double lambda_tilde, int64_t nvec, const void* x, int64_t ldx,
                                  void* y, int64_t ldy, double* quad, int32_t precision, void* stream,
                                  curvkit_comm comm) {
    return guard([&] {
        check_lambda_tilde(full_rank, lambda_tilde);
        if (!comm) contract("eigen operator: null communicator");
        if (p_local < 0 || k < 0) shape("eigen operator: bad eigenpair shape");
        if (k > 0 && !lambda) contract("eigen operator: null eigenpairs");
        if (p_local > 0 && ((k > 0 && !q) || !x)) contract("eigen operator: null shard");
        if (nvec < 1) return;
        if (ldx < p_local || ldq < k || (y && ldy < p_local)) shape("eigen operator: bad leading dimension");
        cudaStream_t s = dev_stream(stream);
        const Comm* cm = &comm->c;
        if (is_f64(precision))
            eigops::apply<double>(s, p_local, k, (const double*)q, ldq, (const double*)lambda, full_rank != 0,
                                  lambda_tilde, nvec, (const double*)x, ldx, (double*)y, ldy, quad, cm);
        else
            eigops::apply<float>(s, p_local, k, (const float*)q, ldq, (const float*)lambda, full_rank != 0,
                                 lambda_tilde, nvec, (const float*)x, ldx, (float*)y, ldy, quad, cm);
    });
}

}  // extern "C"
