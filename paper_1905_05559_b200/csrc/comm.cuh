// comm.cuh -- NCCL communicator for the parameter-row-sharded top-k solver.
//
// NCCL is opened at run time (dlopen), not linked: a process that already
// loaded one (torch bundles its own libnccl.so.2) keeps using that copy, so
// the library never brings a second NCCL with the same soname into it.
// Collectives run on the caller's stream over NVLink / NVSwitch.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "common.cuh"

namespace ck {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;

    static NcclApi& get() {
        static NcclApi api;
        static std::once_flag once;
        static std::string err;
        std::call_once(once, [] {
            void* h = nullptr;
            if (const char* path = getenv("CURVKIT_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)
            if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) {
                const char* e = dlerror();
                err = e ? e : "libnccl.so.2 not found";
                return;
            }
            api.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
            api.comm_init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
            api.comm_destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
            api.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
            api.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
        });
        if (!api.all_reduce) throw CurvError(kRuntimeError, "NCCL unavailable: " + err);
        return api;
    }
};

inline void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* s = NcclApi::get().error_string ? NcclApi::get().error_string(r) : "?";
        throw CurvError(kRuntimeError, std::string(what) + ": " + s);
    }
}

// One rank of a communicator; nranks == 1 makes every collective a no-op.
struct Comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;

    template <class T>
    void sum(T* buf, size_t count, cudaStream_t s) const {
        if (nranks == 1 || count == 0) return;
        const ncclDataType_t t = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
        nccl_check(NcclApi::get().all_reduce(buf, buf, count, t, ncclSum, comm, s), "ncclAllReduce");
    }
};

}  // namespace ck
