// Minimal NCCL binding, resolved at run time (dlopen "libnccl.so.2") so the
// single-GPU library has no hard NCCL dependency and shares whichever libnccl
// the process (e.g. torch) already mapped.  Used only when world > 1.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

namespace tsd {

struct NcclApi {
    ncclResult_t (*get_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    bool ok = false;
};

inline NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_id = (decltype(a.get_id))dlsym(h, "ncclGetUniqueId");
        a.init_rank = (decltype(a.init_rank))dlsym(h, "ncclCommInitRank");
        a.destroy = (decltype(a.destroy))dlsym(h, "ncclCommDestroy");
        a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
        a.ok = a.get_id && a.init_rank && a.destroy && a.all_reduce;
        return a;
    }();
    return api;
}

inline bool nccl_get_unique_id(uint8_t out[128]) {
    NcclApi& a = nccl_api();
    if (!a.ok) return false;
    ncclUniqueId id;
    if (a.get_id(&id) != ncclSuccess) return false;
    memcpy(out, &id, sizeof(id) < 128 ? sizeof(id) : 128);
    return true;
}

inline void* nccl_init(const uint8_t id_bytes[128], int rank, int world) {
    NcclApi& a = nccl_api();
    if (!a.ok) return nullptr;
    ncclUniqueId id;
    memcpy(&id, id_bytes, sizeof(id) < 128 ? sizeof(id) : 128);
    ncclComm_t comm = nullptr;
    if (a.init_rank(&comm, world, id, rank) != ncclSuccess) return nullptr;
    return comm;
}

inline void nccl_destroy(void* comm) {
    NcclApi& a = nccl_api();
    if (a.ok && comm) a.destroy((ncclComm_t)comm);
}

// kind: 0 u8 min (== AND on {0,1} flags), 1 u32 max, 2 u64 min, 3 i32 sum
inline bool nccl_allreduce(void* comm, void* buf, size_t cnt, int kind, cudaStream_t st) {
    NcclApi& a = nccl_api();
    if (!a.ok || !comm) return false;
    ncclDataType_t dt = ncclUint8;
    ncclRedOp_t op = ncclMin;
    switch (kind) {
        case 0: dt = ncclUint8; op = ncclMin; break;
        case 1: dt = ncclUint32; op = ncclMax; break;
        case 2: dt = ncclUint64; op = ncclMin; break;
        default: dt = ncclInt32; op = ncclSum; break;
    }
    return a.all_reduce(buf, buf, cnt, dt, op, (ncclComm_t)comm, st) == ncclSuccess;
}

}  // namespace tsd
