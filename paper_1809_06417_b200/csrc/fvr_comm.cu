// fvr_comm.cu -- the loop's one collective per iteration:
// an owned NCCL communicator and the all-reduce(sum) of the i64 exchange
// buffer [packed correction | squared-residual partials | volume partials].
//
// The reference has no distribution; what this replaces is the
// per-view loop and the fixed-order merge of adjust_pass (reconstruct.py:
// 181-226): each rank back-projects its own views and the integer sum over
// ranks is exact and order-independent, so every GPU count gives the same
// bits.
//
// NCCL is resolved at run time from the libnccl.so.2 already mapped into the
// process (torch's copy) -- or loaded by soname / FVR_NCCL_LIB -- so the
// library never pins a second NCCL build and the build needs no NCCL link.
// The unique id crosses ranks through the caller's rendezvous (the torch
// store), as plain bytes.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "fvr_internal.cuh"

namespace fvr {
namespace {

// nccl.h (2.x) ABI pieces used here
typedef int nccl_result_t;
typedef void* nccl_comm_t;
struct nccl_unique_id {
    char internal[FVR_COMM_ID_BYTES];
};
constexpr int kNcclSum = 0;
constexpr int kNcclInt64 = 4;
constexpr int kNcclFloat32 = 7;
constexpr int kNcclFloat64 = 8;

struct NcclApi {
    nccl_result_t (*get_version)(int*) = nullptr;
    nccl_result_t (*get_unique_id)(nccl_unique_id*) = nullptr;
    nccl_result_t (*comm_init_rank)(nccl_comm_t*, int, nccl_unique_id, int) = nullptr;
    nccl_result_t (*comm_destroy)(nccl_comm_t) = nullptr;
    nccl_result_t (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(nccl_result_t) = nullptr;
    bool ok = false;
    std::string why;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        if (const char* p = std::getenv("FVR_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already mapped (torch)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = "libnccl.so.2 not found (import torch first, or set FVR_NCCL_LIB)";
            return;
        }
        a.get_version = reinterpret_cast<decltype(a.get_version)>(dlsym(h, "ncclGetVersion"));
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_version && a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce &&
               a.error_string;
        if (!a.ok) a.why = "libnccl.so.2 lacks an expected symbol";
    });
    return a;
}

int nccl_error(const char* what, nccl_result_t r) {
    return set_error(FVR_ERR_CUDA, std::string(what) + ": " + api().error_string(r));
}

}  // namespace
}  // namespace fvr

using namespace fvr;

extern "C" int fvr_comm_available(void) { return api().ok ? 1 : 0; }

extern "C" int fvr_comm_nccl_version(int32_t* version) {
    if (!api().ok) return set_error(FVR_ERR_CUDA, api().why);
    int v = 0;
    const nccl_result_t r = api().get_version(&v);
    if (r != 0) return nccl_error("ncclGetVersion", r);
    *version = v;
    return FVR_OK;
}

extern "C" int fvr_comm_unique_id(uint8_t* id_out) {
    if (!id_out) return set_error(FVR_ERR_INVALID, "fvr_comm_unique_id: null output");
    if (!api().ok) return set_error(FVR_ERR_CUDA, api().why);
    nccl_unique_id id;
    const nccl_result_t r = api().get_unique_id(&id);
    if (r != 0) return nccl_error("ncclGetUniqueId", r);
    std::memcpy(id_out, id.internal, FVR_COMM_ID_BYTES);
    return FVR_OK;
}

extern "C" int fvr_comm_init(int32_t rank, int32_t world, const uint8_t* unique_id, int32_t device,
                             fvr_comm_t* comm_out) {
    if (!comm_out || !unique_id) return set_error(FVR_ERR_INVALID, "fvr_comm_init: null argument");
    if (world < 1 || rank < 0 || rank >= world) return set_error(FVR_ERR_INVALID, "fvr_comm_init: bad rank/world");
    if (!api().ok) return set_error(FVR_ERR_CUDA, api().why);
    if (cudaSetDevice(device) != cudaSuccess) return set_error(FVR_ERR_CUDA, "fvr_comm_init: cudaSetDevice failed");
    nccl_unique_id id;
    std::memcpy(id.internal, unique_id, FVR_COMM_ID_BYTES);
    nccl_comm_t c = nullptr;
    const nccl_result_t r = api().comm_init_rank(&c, world, id, rank);
    if (r != 0) return nccl_error("ncclCommInitRank", r);
    *comm_out = c;
    return FVR_OK;
}

extern "C" int fvr_allreduce_sum(fvr_comm_t comm, void* buf, int64_t count, int32_t dtype, void* stream) {
    if (!comm) return set_error(FVR_ERR_INVALID, "fvr_allreduce_sum: no communicator");
    if (count < 0) return set_error(FVR_ERR_INVALID, "fvr_allreduce_sum: negative count");
    if (count == 0) return FVR_OK;
    int nt;
    switch (dtype) {
        case FVR_DT_INT64: nt = kNcclInt64; break;
        case FVR_DT_FLOAT32: nt = kNcclFloat32; break;
        case FVR_DT_FLOAT64: nt = kNcclFloat64; break;
        default: return set_error(FVR_ERR_INVALID, "fvr_allreduce_sum: dtype must be FVR_DT_INT64/FLOAT32/FLOAT64");
    }
    const nccl_result_t r = api().all_reduce(buf, buf, (size_t)count, nt, kNcclSum, comm, (cudaStream_t)stream);
    if (r != 0) return nccl_error("ncclAllReduce", r);
    return FVR_OK;
}

extern "C" int fvr_comm_destroy(fvr_comm_t comm) {
    if (!comm) return FVR_OK;
    if (!api().ok) return set_error(FVR_ERR_CUDA, api().why);
    const nccl_result_t r = api().comm_destroy(comm);
    if (r != 0) return nccl_error("ncclCommDestroy", r);
    return FVR_OK;
}
