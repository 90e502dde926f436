// common.cuh -- shared definitions for the curvkit B200 library.
//
// Model description, canonical flat-parameter offsets (reference
// model.cpp:142-151), activation functions and their first/second
// derivatives (model.cpp:9-50), error plumbing for the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <cstring>
#include <vector>

namespace ck {

constexpr int kMaxLayers = 16;

enum Status : int {
    kOk = 0,
    kShapeError = 1,     // curv::ShapeError
    kContractError = 2,  // curv::ContractError
    kRuntimeError = 3,   // std::runtime_error in the reference
    kConvergenceError = 4,
    kCudaError = 5,
    kOutOfMemory = 6,
};

enum Act : int { kIdentity = 0, kSigmoid = 1, kTanh = 2, kRelu = 3 };
enum OutMode : int { kSoftmaxCE = 0, kRawMean = 1 };

// Arithmetic the path computes in.  kF64/kF32 run exact-FMA SIMT tiles;
// kTF32 runs tcgen05 kind::tf32 MMAs with fp32 accumulation in TMEM;
// k3xTF32 splits each fp32 operand into a TF32 hi part and a TF32 lo part
// and accumulates hi*hi + hi*lo + lo*hi (fp32-grade products).
// kF16S is the TF32 precision class on the fp16 datapath: operands are
// scaled by exact powers of two into fp16 range and rounded to nearest fp16
// -- the same 11-bit significand as TF32 -- and the tcgen05 kind::f16 MMA
// accumulates their exact products in fp32; the scales are undone in the
// epilogue (exact).  Twice the TF32 tensor rate at half the operand bytes.
// Kernels without an fp16 variant run their TF32 form in this mode.
enum Precision : int { kF64 = 0, kF32 = 1, kTF32 = 2, k3xTF32 = 3, kF16S = 4 };
// the tensor-core (TF32-precision) class: TF32 or F16S
__host__ __device__ inline bool tf32_class(int p) { return p == kTF32 || p == kF16S; }
// what a kernel without an fp16 form runs
__host__ __device__ inline int tc_form(int p) { return p == kF16S ? (int)kTF32 : p; }

struct CurvError : std::runtime_error {
    int code;
    CurvError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK_CUDA(expr)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            throw ::ck::CurvError(e_ == cudaErrorMemoryAllocation ? ::ck::kOutOfMemory      \
                                                                  : ::ck::kCudaError,       \
                                  std::string(#expr) + ": " + cudaGetErrorString(e_));     \
    } while (0)

extern std::atomic<int64_t> g_launches;  // kernels launched by this library

#define CK_LAUNCH()                                                   \
    do {                                                              \
        ::ck::g_launches.fetch_add(1, std::memory_order_relaxed);     \
        CK_CUDA(cudaGetLastError());                                  \
    } while (0)

struct ModelDesc {
    int L = 0;  // number of layers (widths)
    int S = 0;  // number of affine steps, L - 1
    int act = kTanh;
    int mode = kSoftmaxCE;
    int64_t w[kMaxLayers] = {};
    int64_t woff[kMaxLayers] = {};  // start of W_k in the flat vector
    int64_t boff[kMaxLayers] = {};  // start of b_k
    int64_t P = 0;

    int64_t tin(int k) const { return w[k]; }
    int64_t tout(int k) const { return w[k + 1]; }
    int64_t block_size(int k) const { return w[k] * w[k + 1] + w[k + 1]; }
};

__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
__host__ __device__ inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// fp32 -> nearest TF32 (10-bit mantissa), kept in fp32 storage
// Round-half-away on the magnitude bits: the result of cvt.rna.tf32.f32 for
// every finite value, +-Inf and quiet NaNs, in two integer ops (ptxas expands
// cvt.rna.tf32 into an Inf test plus predicated adds and moves).
__device__ __forceinline__ float round_tf32(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// ---- activations (model.cpp:9-50) -------------------------------------------

template <class T>
__device__ __forceinline__ T d_exp(T x);
template <>
__device__ __forceinline__ float d_exp<float>(float x) { return expf(x); }
template <>
__device__ __forceinline__ double d_exp<double>(double x) { return exp(x); }

template <class T>
__device__ __forceinline__ T d_tanh(T x);
template <>
__device__ __forceinline__ float d_tanh<float>(float x) { return tanhf(x); }
template <>
__device__ __forceinline__ double d_tanh<double>(double x) { return tanh(x); }

template <class T>
__device__ __forceinline__ T act_value(int a, T z) {
    switch (a) {
        case kSigmoid:
            return z >= T(0) ? T(1) / (T(1) + d_exp(-z)) : d_exp(z) / (T(1) + d_exp(z));
        case kTanh: return d_tanh(z);
        case kRelu: return z > T(0) ? z : T(0);
        default: return z;
    }
}

template <class T>
__device__ __forceinline__ T act_deriv(int a, T z) {
    switch (a) {
        case kSigmoid: {
            const T s = act_value(kSigmoid, z);
            return s * (T(1) - s);
        }
        case kTanh: {
            const T t = d_tanh(z);
            return T(1) - t * t;
        }
        case kRelu: return z > T(0) ? T(1) : T(0);
        default: return T(1);
    }
}

template <class T>
__device__ __forceinline__ T act_second(int a, T z) {
    switch (a) {
        case kSigmoid: {
            const T s = act_value(kSigmoid, z);
            return s * (T(1) - s) * (T(1) - T(2) * s);
        }
        case kTanh: {
            const T t = d_tanh(z);
            return T(-2) * t * (T(1) - t * t);
        }
        default: return T(0);
    }
}

// Read-only launch tables (tile lists, packed index pairs) keyed by content:
// uploaded once per device and reused, so repeated calls of the same shape
// launch without a pageable host-to-device copy.  Bounded: at most 64 tables
// and 256 MB per device, least recently used evicted first (after a device
// synchronisation, since a queued kernel may still read it).
inline uint64_t content_hash(const void* p, size_t bytes) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    uint64_t h = 0x9E3779B97F4A7C15ull ^ bytes;
    size_t i = 0;
    for (; i + 8 <= bytes; i += 8) {
        uint64_t w;
        std::memcpy(&w, b + i, 8);
        h = (h ^ w) * 0xBF58476D1CE4E5B9ull;
        h ^= h >> 31;
    }
    for (; i < bytes; ++i) h = (h ^ b[i]) * 0x94D049BB133111EBull;
    return h;
}

inline const void* cached_upload(const void* host, size_t bytes) {
    struct Entry {
        int dev;
        uint64_t hash;
        std::vector<uint8_t> content;
        void* d;
        uint64_t used;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    static uint64_t tick = 0;
    constexpr size_t kMaxEntries = 64, kMaxBytes = size_t(256) << 20;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t h = content_hash(host, bytes);
    std::lock_guard<std::mutex> g(mu);
    for (Entry& e : cache)
        if (e.dev == dev && e.hash == h && e.content.size() == bytes && std::memcmp(e.content.data(), host, bytes) == 0) {
            e.used = ++tick;
            return e.d;
        }
    auto held = [&] {
        size_t n = 0, b = 0;
        for (const Entry& e : cache)
            if (e.dev == dev) { ++n; b += e.content.size(); }
        return std::make_pair(n, b);
    };
    for (auto hb = held(); hb.first > 0 && (hb.first >= kMaxEntries || hb.second + bytes > kMaxBytes); hb = held()) {
        size_t lru = cache.size();
        for (size_t i = 0; i < cache.size(); ++i)
            if (cache[i].dev == dev && (lru == cache.size() || cache[i].used < cache[lru].used)) lru = i;
        cudaDeviceSynchronize();  // a queued launch may still read the table
        cudaFree(cache[lru].d);
        cache.erase(cache.begin() + (ptrdiff_t)lru);
    }
    void* d = nullptr;
    if (cudaMalloc(&d, bytes ? bytes : 1) != cudaSuccess) throw std::runtime_error("cached_upload: cudaMalloc failed");
    if (bytes && cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cached_upload: cudaMemcpy failed");
    const uint8_t* hb = static_cast<const uint8_t*>(host);
    cache.push_back(Entry{dev, h, std::vector<uint8_t>(hb, hb + bytes), d, ++tick});
    return d;
}

// cudaFuncSetAttribute acts per device: run `set` once per (device, kernel key)
template <class F>
inline void func_attr_once(const void* key, F&& set) {
    static std::mutex mu;
    static std::vector<std::pair<int, const void*>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    for (const auto& d : done)
        if (d.first == dev && d.second == key) return;
    set();
    done.emplace_back(dev, key);
}

}  // namespace ck
