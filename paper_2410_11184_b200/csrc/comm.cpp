// comm.cpp -- the library-owned NCCL communicator of the sharded
// many-ciphertext Softmax (SURVEY 8(b) hs_comm_init).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- the copy torch
// already loaded when there is one), so the library itself has no link-time
// NCCL dependency and loads on machines without it; only hs_comm_* need it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "hs_internal.h"

namespace {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl()
{
    static NcclApi api;
    static std::once_flag once;
    static std::string why;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char *e = dlerror();  // one call: dlerror() clears the message
            why = e ? e : "dlopen failed";
            return;
        }
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
        api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
        api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
        api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
        api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
    });
    if (!api.getUniqueId || !api.commInitRank || !api.commDestroy || !api.allGather)
        throw HsError(HS_ENCCL, "libnccl.so.2 not available: " + why);
    return api;
}

void check(ncclResult_t r, const char *what)
{
    if (r != ncclSuccess) {
        const NcclApi &a = nccl();
        throw HsError(HS_ENCCL, std::string(what) + ": " + (a.errorString ? a.errorString(r) : "nccl error"));
    }
}

}  // namespace

struct hs_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
};

int comm_world(const hs_comm *c) { return c->world; }

void comm_all_gather(const hs_comm *c, const u64 *partial, u64 *gathered, size_t words, cudaStream_t st)
{
    check(nccl().allGather(partial, gathered, words, ncclUint64, c->comm, st), "ncclAllGather");
}

// in-place uint64 sum over the ranks (the caller reduces mod q afterwards:
// exact while world * max prime < 2^64)
void comm_all_reduce_u64(const hs_comm *c, u64 *buf, size_t words, cudaStream_t st)
{
    if (!nccl().allReduce) throw HsError(HS_ENCCL, "ncclAllReduce not available");
    check(nccl().allReduce(buf, buf, words, ncclUint64, ncclSum, c->comm, st), "ncclAllReduce");
}

void comm_unique_id(uint8_t uid[128])
{
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    check(nccl().getUniqueId(&id), "ncclGetUniqueId");
    memcpy(uid, &id, 128);
}

hs_comm *comm_create(int rank, int world, const uint8_t uid[128])
{
    ncclUniqueId id;
    memcpy(&id, uid, 128);
    std::unique_ptr<hs_comm> h(new hs_comm);
    h->rank = rank;
    h->world = world;
    check(nccl().commInitRank(&h->comm, world, id, rank), "ncclCommInitRank");
    return h.release();
}

void comm_destroy(hs_comm *comm)
{
    if (!comm) return;
    try {
        if (comm->comm) nccl().commDestroy(comm->comm);
    } catch (...) {
    }
    delete comm;
}
