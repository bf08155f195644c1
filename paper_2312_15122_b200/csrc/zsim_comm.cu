// Episode-statistics exchange across GPUs over NCCL.
//
// The batch is scenario-sharded: rank r simulates its own slice and nothing
// crosses GPUs per step.  Once per rollout the int64 stats vector
// (zsim_episode_stats) is summed over all GPUs with one ncclAllReduce -- an
// integer sum, exact and independent of the reduction order, which honours the
// fixed-order contract of the reference's AllReducer
// (core/train/transport.hpp:59-61) -- and the fp64 Aggregate partial sums
// (zsim_episode_metrics, metrics.hpp:56-69) are all-gathered so every rank
// adds them in rank order (zsim_aggregate_finalize), reproducible for a given
// sharding.
//
// NCCL is resolved at first use with dlopen("libnccl.so.2"): a process that
// already loaded NCCL (torch) shares that copy, and the library itself loads
// on hosts without NCCL.  Two ways to build a communicator:
//  * one process per GPU (torchrun): rank 0 calls zsim_comm_unique_id, the
//    128-byte id is broadcast by the caller's plumbing, every rank calls
//    zsim_comm_init_rank;
//  * one process driving every GPU (SURVEY §8e's ncclCommInitAll layout):
//    zsim_comm_init_all, then one host thread and stream per GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/zsim_gpu.h"

extern "C" void zsim_internal_set_last_error(const char* m);  // zsim_capi.cu

struct zsim_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0;
    int rank = 0;
    int device = 0;
};

namespace {

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            n.error = std::string("NCCL unavailable: ") + (e ? e : "dlopen(libnccl.so.2) failed");
            return;
        }
        auto sym = [&](const char* s) {
            void* p = dlsym(h, s);
            if (!p && n.error.empty()) n.error = std::string("NCCL symbol missing: ") + s;
            return p;
        };
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.CommGetAsyncError = reinterpret_cast<decltype(n.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!n.error.empty()) throw Fail(ZSIM_RUNTIME, n.error);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Fail(ZSIM_RUNTIME, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Fail(ZSIM_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return ZSIM_OK;
    } catch (const Fail& e) {
        zsim_internal_set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        zsim_internal_set_last_error(e.what());
        return ZSIM_RUNTIME;
    }
}

void need(const zsim_comm* c) {
    if (!c || !c->comm) throw Fail(ZSIM_INVALID_ARGUMENT, "null communicator");
}

}  // namespace

extern "C" {

ZSIM_API int zsim_comm_available(void) {
    return guarded([] { (void)nccl(); }) == ZSIM_OK ? 1 : 0;
}

ZSIM_API int zsim_comm_unique_id(uint8_t id[ZSIM_COMM_ID_BYTES]) {
    return guarded([&] {
        if (!id) throw Fail(ZSIM_INVALID_ARGUMENT, "null id buffer");
        static_assert(sizeof(ncclUniqueId) == ZSIM_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

ZSIM_API int zsim_comm_init_rank(const uint8_t id[ZSIM_COMM_ID_BYTES], int32_t nranks, int32_t rank, int32_t device,
                                 zsim_comm** out) {
    return guarded([&] {
        if (!id || !out) throw Fail(ZSIM_INVALID_ARGUMENT, "null argument");
        *out = nullptr;
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Fail(ZSIM_INVALID_ARGUMENT, "bad rank / nranks");
        cuda_ok(cudaSetDevice(device), "cudaSetDevice");
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        auto* c = new zsim_comm();
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, u, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

ZSIM_API int zsim_comm_init_all(int32_t ndev, const int32_t* devices, zsim_comm** out) {
    return guarded([&] {
        if (!out || ndev < 1) throw Fail(ZSIM_INVALID_ARGUMENT, "bad arguments");
        std::vector<int> devs(static_cast<size_t>(ndev));
        for (int i = 0; i < ndev; ++i) devs[size_t(i)] = devices ? devices[i] : i;
        std::vector<ncclComm_t> comms(static_cast<size_t>(ndev));
        nccl_check(nccl().CommInitAll(comms.data(), ndev, devs.data()), "ncclCommInitAll");
        for (int i = 0; i < ndev; ++i) {
            auto* c = new zsim_comm();
            c->comm = comms[size_t(i)];
            c->nranks = ndev;
            c->rank = i;
            c->device = devs[size_t(i)];
            out[i] = c;
        }
    });
}

ZSIM_API int zsim_comm_destroy(zsim_comm* c) {
    return guarded([&] {
        if (!c) return;
        if (c->comm) nccl_check(nccl().CommDestroy(c->comm), "ncclCommDestroy");
        delete c;
    });
}

ZSIM_API int zsim_comm_check(zsim_comm* c) {
    return guarded([&] {
        need(c);
        ncclResult_t a = ncclSuccess;
        nccl_check(nccl().CommGetAsyncError(c->comm, &a), "ncclCommGetAsyncError");
        nccl_check(a, "NCCL asynchronous error");
    });
}

ZSIM_API int zsim_stats_allreduce(zsim_comm* c, int64_t* stats_dev, int32_t n, void* stream) {
    return guarded([&] {
        need(c);
        if (!stats_dev || n <= 0) throw Fail(ZSIM_INVALID_ARGUMENT, "bad stats buffer");
        nccl_check(nccl().AllReduce(stats_dev, stats_dev, size_t(n), ncclInt64, ncclSum, c->comm,
                                    static_cast<cudaStream_t>(stream)),
                   "ncclAllReduce(stats)");
    });
}

ZSIM_API int zsim_metric_sums_allgather(zsim_comm* c, const double* sums_dev, int32_t n, double* gathered_dev,
                                        void* stream) {
    return guarded([&] {
        need(c);
        if (!sums_dev || !gathered_dev || n <= 0) throw Fail(ZSIM_INVALID_ARGUMENT, "bad metric buffers");
        nccl_check(nccl().AllGather(sums_dev, gathered_dev, size_t(n), ncclFloat64, c->comm,
                                    static_cast<cudaStream_t>(stream)),
                   "ncclAllGather(metric sums)");
    });
}

ZSIM_API int zsim_comm_group(int32_t begin) {
    return guarded([&] {
        nccl_check(begin ? nccl().GroupStart() : nccl().GroupEnd(), begin ? "ncclGroupStart" : "ncclGroupEnd");
    });
}

}  // extern "C"
