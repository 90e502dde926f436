// comm.cuh -- the communicator of the multi-GPU entry points.
//
// Two transports behind one interface:
//   NCCL  (curvkit_comm_init): collectives on the caller's stream over NVLink /
//         NVSwitch.  NCCL is opened at run time (dlopen), not linked: a process
//         that already loaded one (torch bundles libnccl.so.2) keeps using it.
//   host  (curvkit_comm_init_host): the caller's own collectives on host
//         memory (an MPI / gloo / torch.distributed binding passed as C
//         callbacks); the library stages each exchange through host memory.
//         Used where NCCL cannot run (ranks sharing one GPU in tests).
// The multi-GPU algorithms issue the same exchanges on either transport:
// sum (all-reduce) and gather (variable-size blocks to one root).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/curvkit_b200.h"
#include "common.cuh"

namespace ck {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
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
            api.send = reinterpret_cast<decltype(&ncclSend)>(dlsym(h, "ncclSend"));
            api.recv = reinterpret_cast<decltype(&ncclRecv)>(dlsym(h, "ncclRecv"));
            api.group_start = reinterpret_cast<decltype(&ncclGroupStart)>(dlsym(h, "ncclGroupStart"));
            api.group_end = reinterpret_cast<decltype(&ncclGroupEnd)>(dlsym(h, "ncclGroupEnd"));
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

// One rank of a communicator; nranks == 1 makes every collective a local copy.
struct Comm {
    ncclComm_t comm = nullptr;  // NCCL transport, or
    curvkit_host_allreduce_fn h_sum = nullptr;  // the host transport
    curvkit_host_gather_fn h_gather = nullptr;
    void* user = nullptr;
    int rank = 0, nranks = 1;
    // One-rank NCCL communicators opened under CURVKIT_COMM_LOOPBACK=1 still issue
    // their collectives (an in-place all-reduce over one rank, a send/recv pair
    // to itself): the NCCL calls of the multi-GPU paths run on a one-GPU box.
    bool loopback = false;

    bool host() const { return comm == nullptr && h_sum != nullptr; }

    // buf <- sum over ranks (identical bytes on every rank afterwards)
    template <class T>
    void sum(T* buf, size_t count, cudaStream_t s) const {
        if ((nranks == 1 && !loopback) || count == 0) return;
        if (host()) {
            std::vector<T> h(count);
            CK_CUDA(cudaMemcpyAsync(h.data(), buf, count * sizeof(T), cudaMemcpyDeviceToHost, s));
            CK_CUDA(cudaStreamSynchronize(s));
            if (h_sum(h.data(), (int64_t)count, sizeof(T) == 8 ? 1 : 0, user) != 0)
                throw CurvError(kRuntimeError, "host all-reduce callback failed");
            CK_CUDA(cudaMemcpyAsync(buf, h.data(), count * sizeof(T), cudaMemcpyHostToDevice, s));
            CK_CUDA(cudaStreamSynchronize(s));
            return;
        }
        const ncclDataType_t t = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
        nccl_check(NcclApi::get().all_reduce(buf, buf, count, t, ncclSum, comm, s), "ncclAllReduce");
    }

    // Rank r's `bytes[r]` device bytes at `send` land at recv + sum_{q<r} bytes[q]
    // on `root` (recv is only used there).
    void gather(const void* send, const std::vector<int64_t>& bytes, void* recv, int root, cudaStream_t s) const {
        std::vector<int64_t> off(nranks + 1, 0);
        for (int r = 0; r < nranks; ++r) off[r + 1] = off[r] + bytes[r];
        if (nranks == 1 && loopback && !host()) {
            NcclApi& api = NcclApi::get();
            if (!api.send || !api.recv || !api.group_start) throw CurvError(kRuntimeError, "NCCL send/recv unavailable");
            if (bytes[0] <= 0) return;
            nccl_check(api.group_start(), "ncclGroupStart");
            nccl_check(api.recv(recv, (size_t)bytes[0], ncclInt8, 0, comm, s), "ncclRecv");
            nccl_check(api.send(send, (size_t)bytes[0], ncclInt8, 0, comm, s), "ncclSend");
            nccl_check(api.group_end(), "ncclGroupEnd");
            return;
        }
        if (nranks == 1 || (!host() && rank == root)) {
            if (rank == root && bytes[rank] > 0)
                CK_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + off[rank], send, (size_t)bytes[rank],
                                        cudaMemcpyDeviceToDevice, s));
            if (nranks == 1) return;
        }
        if (host()) {
            // in pieces of at most 256 MB per rank (bands of config 3 are tens of GB):
            // every rank makes the same number of callback calls, piece c of rank r
            // being bytes [c * PIECE, min(bytes[r], (c + 1) * PIECE)) of its block
            constexpr int64_t PIECE = int64_t(256) << 20;
            int64_t mx = 0;
            for (int r = 0; r < nranks; ++r) mx = std::max(mx, bytes[r]);
            const int64_t npieces = std::max<int64_t>(1, ceil_div(mx, PIECE));
            std::vector<uint8_t> hs((size_t)std::min(bytes[rank], PIECE));
            std::vector<uint8_t> hr;
            std::vector<int64_t> sz(nranks), po(nranks + 1);
            for (int64_t c = 0; c < npieces; ++c) {
                po[0] = 0;
                for (int r = 0; r < nranks; ++r) {
                    sz[r] = std::clamp<int64_t>(bytes[r] - c * PIECE, 0, PIECE);
                    po[r + 1] = po[r] + sz[r];
                }
                if (sz[rank] > 0)
                    CK_CUDA(cudaMemcpyAsync(hs.data(), static_cast<const uint8_t*>(send) + c * PIECE, (size_t)sz[rank],
                                            cudaMemcpyDeviceToHost, s));
                CK_CUDA(cudaStreamSynchronize(s));
                if (rank == root) hr.resize((size_t)po[nranks]);
                if (h_gather(hs.data(), sz[rank], rank == root ? hr.data() : nullptr, sz.data(), root, user) != 0)
                    throw CurvError(kRuntimeError, "host gather callback failed");
                if (rank == root)
                    for (int r = 0; r < nranks; ++r)
                        if (sz[r] > 0)
                            CK_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + off[r] + c * PIECE, hr.data() + po[r],
                                                    (size_t)sz[r], cudaMemcpyHostToDevice, s));
                CK_CUDA(cudaStreamSynchronize(s));
            }
            return;
        }
        NcclApi& api = NcclApi::get();
        if (!api.send || !api.recv || !api.group_start) throw CurvError(kRuntimeError, "NCCL send/recv unavailable");
        nccl_check(api.group_start(), "ncclGroupStart");
        if (rank == root) {
            for (int r = 0; r < nranks; ++r)
                if (r != root && bytes[r] > 0)
                    nccl_check(api.recv(static_cast<uint8_t*>(recv) + off[r], (size_t)bytes[r], ncclInt8, r, comm, s),
                               "ncclRecv");
        } else if (bytes[rank] > 0) {
            nccl_check(api.send(send, (size_t)bytes[rank], ncclInt8, root, comm, s), "ncclSend");
        }
        nccl_check(api.group_end(), "ncclGroupEnd");
    }
};

}  // namespace ck
