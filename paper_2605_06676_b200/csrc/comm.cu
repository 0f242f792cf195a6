// comm.cu -- multi-GPU plumbing of the head-sharded path: one process per GPU,
// NCCL over NVLink 5 / NVSwitch.  The data path itself has no collective: every (seq, layer,
// head) is scored, selected, compacted and decoded on the rank that owns it.  The only
// exchanges are
//   * the LKV-H logits: each rank holds its own heads' logits (head_scores of its heads,
//     policy.cpp:106-108); one allgatherv gives every rank all n logits, and every rank then
//     solves the global lambda redundantly and bit-identically (K2), so the budgets and the
//     per-rank ragged offsets agree everywhere without a second exchange;
//   * the decode outputs: each rank's [n_seq][its layers][Hq][d] block goes to the root
//     (gatherv) or to everyone (allgatherv), batched over layers and steps by the caller.
// Messages are a few KB, so these are latency-bound: a grouped broadcast / send-recv per rank.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch process that is the
// NCCL torch already loaded; in a plain C++ process it is the system library.  No link-time
// dependency, and a box without NCCL only loses these entry points (LKV_ERR_NCCL).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "../../include/lkv_b200.h"

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
    bool ok = false;
    std::string why;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
        bool all = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) all = false;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.Broadcast, "ncclBroadcast");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GetErrorString, "ncclGetErrorString");
        api.ok = all;
        if (!all) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

}  // namespace

struct lkv_comm_s {
    ncclComm_t comm;
    int n_ranks, rank;
};

// error reporting lives in c_api.cu
lkv_status lkv_internal_fail(lkv_status code, const std::string& msg);

#define LKV_NCCL(call, where)                                                                              \
    do {                                                                                                   \
        const ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess)                                                                             \
            return lkv_internal_fail(LKV_ERR_NCCL, std::string(where) + ": " + nccl().GetErrorString(r_)); \
    } while (0)

extern "C" {

lkv_status lkv_comm_get_unique_id(void* id) {
    if (!id) return lkv_internal_fail(LKV_ERR_CONTRACT, "comm_get_unique_id: id is null");
    if (!nccl().ok) return lkv_internal_fail(LKV_ERR_NCCL, nccl().why);
    static_assert(sizeof(ncclUniqueId) == LKV_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId u;
    LKV_NCCL(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    memcpy(id, &u, sizeof u);
    return LKV_OK;
}

lkv_status lkv_comm_init(lkv_comm_t* out, const void* id, int32_t n_ranks, int32_t rank) {
    if (!out || !id) return lkv_internal_fail(LKV_ERR_CONTRACT, "comm_init: null argument");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return lkv_internal_fail(LKV_ERR_CONTRACT, "comm_init: bad rank");
    if (!nccl().ok) return lkv_internal_fail(LKV_ERR_NCCL, nccl().why);
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    ncclComm_t c = nullptr;
    LKV_NCCL(nccl().CommInitRank(&c, n_ranks, u, rank), "ncclCommInitRank");
    *out = new lkv_comm_s{c, n_ranks, rank};
    return LKV_OK;
}

lkv_status lkv_comm_destroy(lkv_comm_t c) {
    if (!c) return LKV_OK;
    const ncclResult_t r = nccl().CommDestroy(c->comm);
    delete c;
    if (r != ncclSuccess) return lkv_internal_fail(LKV_ERR_NCCL, std::string("ncclCommDestroy: ") + nccl().GetErrorString(r));
    return LKV_OK;
}

int32_t lkv_comm_size(lkv_comm_t c) { return c ? c->n_ranks : 0; }
int32_t lkv_comm_rank(lkv_comm_t c) { return c ? c->rank : -1; }

static lkv_status check_v(lkv_comm_t c, const int64_t* bytes, const int64_t* displs) {
    if (!c || !bytes || !displs) return lkv_internal_fail(LKV_ERR_CONTRACT, "comm: null communicator or size table");
    for (int r = 0; r < c->n_ranks; ++r)
        if (bytes[r] < 0 || displs[r] < 0) return lkv_internal_fail(LKV_ERR_CONTRACT, "comm: negative size/displacement");
    return LKV_OK;
}

// recv[displs[r] .. + bytes[r]) <- rank r's send, on every rank (ncclBroadcast per rank, grouped).
lkv_status lkv_comm_allgatherv(lkv_comm_t c, const void* send, void* recv, const int64_t* bytes, const int64_t* displs,
                               lkv_stream_t stream) {
    lkv_status st = check_v(c, bytes, displs);
    if (st) return st;
    if (!recv || (bytes[c->rank] > 0 && !send)) return lkv_internal_fail(LKV_ERR_CONTRACT, "allgatherv: null buffer");
    LKV_NCCL(nccl().GroupStart(), "ncclGroupStart");
    for (int r = 0; r < c->n_ranks; ++r) {
        if (bytes[r] == 0) continue;
        const ncclResult_t e = nccl().Broadcast(r == c->rank ? send : nullptr, static_cast<char*>(recv) + displs[r],
                                                (size_t)bytes[r], ncclUint8, r, c->comm, (cudaStream_t)stream);
        if (e != ncclSuccess) {
            nccl().GroupEnd();
            return lkv_internal_fail(LKV_ERR_NCCL, std::string("ncclBroadcast: ") + nccl().GetErrorString(e));
        }
    }
    LKV_NCCL(nccl().GroupEnd(), "ncclGroupEnd");
    return LKV_OK;
}

// On `root`: recv[displs[r] .. + bytes[r]) <- rank r's send (grouped send/recv; recv may be
// NULL elsewhere).
lkv_status lkv_comm_gatherv(lkv_comm_t c, const void* send, void* recv, const int64_t* bytes, const int64_t* displs,
                            int32_t root, lkv_stream_t stream) {
    lkv_status st = check_v(c, bytes, displs);
    if (st) return st;
    if (root < 0 || root >= c->n_ranks) return lkv_internal_fail(LKV_ERR_CONTRACT, "gatherv: bad root");
    if (c->rank == root && !recv) return lkv_internal_fail(LKV_ERR_CONTRACT, "gatherv: root needs recv");
    if (bytes[c->rank] > 0 && !send) return lkv_internal_fail(LKV_ERR_CONTRACT, "gatherv: null send");
    const cudaStream_t s = (cudaStream_t)stream;
    if (c->rank == root && bytes[root] > 0) {  // own block: a device copy, not a self send
        if (cudaMemcpyAsync(static_cast<char*>(recv) + displs[root], send, (size_t)bytes[root],
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return lkv_internal_fail(LKV_ERR_CUDA, "gatherv: own block copy failed");
    }
    LKV_NCCL(nccl().GroupStart(), "ncclGroupStart");
    ncclResult_t e = ncclSuccess;
    if (c->rank == root) {
        for (int r = 0; r < c->n_ranks && e == ncclSuccess; ++r)
            if (r != root && bytes[r] > 0)
                e = nccl().Recv(static_cast<char*>(recv) + displs[r], (size_t)bytes[r], ncclUint8, r, c->comm, s);
    } else if (bytes[c->rank] > 0) {
        e = nccl().Send(send, (size_t)bytes[c->rank], ncclUint8, root, c->comm, s);
    }
    const ncclResult_t g = nccl().GroupEnd();
    if (e != ncclSuccess) return lkv_internal_fail(LKV_ERR_NCCL, std::string("ncclSend/Recv: ") + nccl().GetErrorString(e));
    if (g != ncclSuccess) return lkv_internal_fail(LKV_ERR_NCCL, std::string("ncclGroupEnd: ") + nccl().GetErrorString(g));
    return LKV_OK;
}

}  // extern "C"
