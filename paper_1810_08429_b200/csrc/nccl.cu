// NCCL for the sharded matvec (block-row partition, all-gather
// of x and of the forward coefficients x-hat over NVLink / NVSwitch).  NCCL
// is resolved at run time (dlopen of libnccl.so.2: inside a torch process
// this is torch's already-loaded NCCL, elsewhere the system one), so the
// library has no link-time NCCL dependency and C hosts without NCCL still
// load it.  The all-gather is also a node kind of the native product
// executor (csrc/plan.cu), captured into the product's CUDA graph.
#include <dlfcn.h>
#include <mutex>

#include "common.cuh"

namespace {

typedef struct { char internal[128]; } NcclUniqueId;   // ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128)
typedef void* NcclComm;
constexpr int NCCL_FLOAT64 = 8;                        // ncclFloat64 / ncclDouble

struct NcclApi {
    int (*get_unique_id)(NcclUniqueId*) = nullptr;
    int (*comm_init_rank)(NcclComm*, int, NcclUniqueId, int) = nullptr;
    int (*comm_destroy)(NcclComm) = nullptr;
    int (*all_gather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
    const char* (*error_string)(int) = nullptr;
    bool ok = false;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

void load_nccl() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);      // the copy torch loaded, if any
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_nccl.get_unique_id = (int (*)(NcclUniqueId*))dlsym(h, "ncclGetUniqueId");
    g_nccl.comm_init_rank = (int (*)(NcclComm*, int, NcclUniqueId, int))dlsym(h, "ncclCommInitRank");
    g_nccl.comm_destroy = (int (*)(NcclComm))dlsym(h, "ncclCommDestroy");
    g_nccl.all_gather = (int (*)(const void*, void*, size_t, int, NcclComm, cudaStream_t))dlsym(h, "ncclAllGather");
    g_nccl.error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.comm_destroy && g_nccl.all_gather &&
                g_nccl.error_string;
}

int need_nccl() {
    std::call_once(g_nccl_once, load_nccl);
    if (!g_nccl.ok) {
        gcb::set_error(GC_ERR_CUDA, "NCCL (libnccl.so.2) not available");
        return GC_ERR_CUDA;
    }
    return GC_OK;
}

int nccl_status(int r, const char* what) {
    if (r == 0) return GC_OK;
    gcb::set_error(GC_ERR_CUDA, "%s: %s", what, g_nccl.error_string ? g_nccl.error_string(r) : "NCCL error");
    return GC_ERR_CUDA;
}

}  // namespace

extern "C" int gc_nccl_unique_id(void* id) {
    if (!id) { gcb::set_error(GC_ERR_CONFIG, "gc_nccl_unique_id: null output"); return GC_ERR_CONFIG; }
    if (int rc = need_nccl()) return rc;
    return nccl_status(g_nccl.get_unique_id((NcclUniqueId*)id), "ncclGetUniqueId");
}

extern "C" int gc_nccl_comm_init(const void* id, int32_t nranks, int32_t rank, void** comm) {
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) {
        gcb::set_error(GC_ERR_CONFIG, "gc_nccl_comm_init: bad arguments");
        return GC_ERR_CONFIG;
    }
    if (int rc = need_nccl()) return rc;
    NcclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    NcclComm c = nullptr;
    if (int rc = nccl_status(g_nccl.comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank")) return rc;
    *comm = c;
    return GC_OK;
}

extern "C" int gc_nccl_comm_destroy(void* comm) {
    if (!comm) return GC_OK;
    if (int rc = need_nccl()) return rc;
    return nccl_status(g_nccl.comm_destroy((NcclComm)comm), "ncclCommDestroy");
}

// recv (nranks * count doubles) = concatenation over ranks of send (count
// doubles); in place when send is recv's own slot (recv + rank * count).
extern "C" int gc_nccl_all_gather(const double* send, double* recv, int64_t count, void* comm, void* stream) {
    if (!send || !recv || !comm || count < 0) {
        gcb::set_error(GC_ERR_CONFIG, "gc_nccl_all_gather: bad arguments");
        return GC_ERR_CONFIG;
    }
    if (int rc = need_nccl()) return rc;
    return nccl_status(g_nccl.all_gather(send, recv, (size_t)count, NCCL_FLOAT64, (NcclComm)comm,
                                         (cudaStream_t)stream), "ncclAllGather");
}
