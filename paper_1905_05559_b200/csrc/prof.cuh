// prof.cuh -- optional CUDA-event timing of the library's hot kernels.
//
// When enabled (curvkit_profile_begin), every instrumented region records a
// start/stop event pair on the stream it launches on, together with its
// algorithmic FLOPs and bytes.  curvkit_profile_end() synchronises, sums the
// per-region durations and returns them as JSON, which bench.py turns into
// the roofline numbers.  Disabled, a region costs one branch.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace ck {

struct ProfRec {
    cudaEvent_t a, b;
    double flops, bytes;
};

struct Profiler {
    bool on = false;
    std::mutex mu;
    std::map<std::string, std::vector<ProfRec>> recs;

    static Profiler& get() {
        static Profiler p;
        return p;
    }
};

struct ProfScope {
    const char* name;
    cudaStream_t s;
    double flops, bytes;
    cudaEvent_t a = nullptr;
    ProfScope(const char* n, cudaStream_t st, double f, double by) : name(n), s(st), flops(f), bytes(by) {
        if (!Profiler::get().on) return;
        cudaEventCreate(&a);
        cudaEventRecord(a, s);
    }
    ~ProfScope() { end(); }
    void end() {
        if (!a) return;
        cudaEvent_t b;
        cudaEventCreate(&b);
        cudaEventRecord(b, s);
        Profiler& p = Profiler::get();
        std::lock_guard<std::mutex> g(p.mu);
        p.recs[name].push_back({a, b, flops, bytes});
        a = nullptr;
    }
};

}  // namespace ck
