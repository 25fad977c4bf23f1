// Native product executor: the matvec DAG of h2.PanelPlan (panel phases,
// memsets, the external-order gather / scatter) captured into one CUDA
// graph by C++ on its own streams and events, then launched with one call
// per product (h2.py:63-80 as a single C entry point).  The Python plan
// builds the phase descriptors; gc_plan_run re-points the graph's gather /
// scatter nodes at the caller's x / y when they change
// (cudaGraphExecKernelNodeSetParams) and launches the executable graph.
#include <cstring>
#include <vector>

#include "common.cuh"

extern "C" int gc_panelmv(int64_t nitems, const int64_t* items, const int32_t* xidx, const double* A0,
                          const double* A1, const double* in0, const double* in1, double* out, double* scratch,
                          int64_t nred, const int64_t* red, int32_t* arrivals, int32_t chain, int32_t priority,
                          uint64_t* trace, void* stream);
extern "C" int gc_gather_inv(const double* x, const int64_t* iperm, int64_t n, double* xt, void* stream);
extern "C" int gc_scatter2_inv(const double* yt, const double* yt2, const int64_t* iperm, int64_t n, double* y,
                               void* stream);
extern "C" int gc_nccl_all_gather(const double* send, double* recv, int64_t count, void* comm, void* stream);
extern "C" int gc_graph_retarget(void* graph, void* exec, int32_t kernel, int32_t arg, const void* old_ptr,
                                 const void* new_ptr, int32_t* count);

namespace {

// node kinds
enum { NODE_PANEL = 0, NODE_MEMSET = 1, NODE_GATHER = 2, NODE_SCATTER = 3, NODE_ALLGATHER = 4 };

struct Node {
    int64_t kind, stream, priority, chain, ndeps, dep_off;
    // panel: items, nitems, xidx, A0, A1, in0, in1, out, scratch, nred, red, arrivals
    // memset: ptr, bytes; gather: x, iperm, n, xt; scatter: yt, yt2, iperm, n, y;
    // all-gather: send, recv, count (doubles per rank), NCCL communicator
    int64_t a[12];
};

struct Plan {
    std::vector<Node> nodes;
    std::vector<int64_t> deps;
    int nstreams = 0;
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    const void* cap_x = nullptr;      // captured gather input / scatter output
    const void* cap_y = nullptr;
    const void* bound_x = nullptr;    // currently bound in the executable graph
    const void* bound_y = nullptr;
};

int launch_node(const Node& nd, cudaStream_t st) {
    const int64_t* a = nd.a;
    switch (nd.kind) {
        case NODE_PANEL:
            return gc_panelmv(a[1], (const int64_t*)a[0], (const int32_t*)a[2], (const double*)a[3],
                              (const double*)a[4], (const double*)a[5], (const double*)a[6], (double*)a[7],
                              (double*)a[8], a[9], (const int64_t*)a[10], (int32_t*)a[11], (int32_t)nd.chain,
                              (int32_t)nd.priority, nullptr, st);
        case NODE_MEMSET: {
            cudaError_t e = cudaMemsetAsync((void*)a[0], 0, (size_t)a[1], st);
            return e == cudaSuccess ? GC_OK : gcb::cuda_status(e, "gc_plan memset");
        }
        case NODE_GATHER:
            return gc_gather_inv((const double*)a[0], (const int64_t*)a[1], a[2], (double*)a[3], st);
        case NODE_SCATTER:
            return gc_scatter2_inv((const double*)a[0], (const double*)a[1], (const int64_t*)a[2], a[3],
                                   (double*)a[4], st);
        case NODE_ALLGATHER:
            return gc_nccl_all_gather((const double*)a[0], (double*)a[1], a[2], (void*)a[3], st);
        default:
            gcb::set_error(GC_ERR_CONFIG, "gc_plan: unknown node kind %lld", (long long)nd.kind);
            return GC_ERR_CONFIG;
    }
}

void destroy(Plan* p) {
    if (!p) return;
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    for (auto e : p->events) cudaEventDestroy(e);
    for (auto s : p->streams) cudaStreamDestroy(s);
    delete p;
}

}  // namespace

using namespace gcb;

// nodes [host] (n, 18) int64 rows: kind, stream, priority, chain, ndeps,
// dep_off, then 12 arguments (see Node); deps [host] = concatenated
// dependency node indices (each < its node's index); stream_prio [host]
// (nstreams) = creation priority of each stream (stream 0 carries the
// first node and the final join).  Captures the DAG in node order on the
// plan's streams into one graph and instantiates it.  *out = the plan.
extern "C" int gc_plan_create(int64_t n, const int64_t* nodes, int64_t ndeps, const int64_t* deps,
                              int64_t nstreams, const int32_t* stream_prio, void** out) {
    if (!out || n <= 0 || !nodes || nstreams <= 0 || !stream_prio) {
        set_error(GC_ERR_CONFIG, "gc_plan_create: bad arguments");
        return GC_ERR_CONFIG;
    }
    *out = nullptr;
    Plan* p = new Plan();
    p->nodes.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t* r = nodes + 18 * i;
        Node& nd = p->nodes[(size_t)i];
        nd.kind = r[0], nd.stream = r[1], nd.priority = r[2], nd.chain = r[3], nd.ndeps = r[4], nd.dep_off = r[5];
        for (int k = 0; k < 12; ++k) nd.a[k] = r[6 + k];
        if (nd.stream < 0 || nd.stream >= nstreams || nd.dep_off < 0 || nd.dep_off + nd.ndeps > ndeps) {
            destroy(p);
            set_error(GC_ERR_CONFIG, "gc_plan_create: node %lld has a bad stream or dependency range", (long long)i);
            return GC_ERR_CONFIG;
        }
        for (int64_t k = 0; k < nd.ndeps; ++k)
            if (deps[nd.dep_off + k] < 0 || deps[nd.dep_off + k] >= i) {
                destroy(p);
                set_error(GC_ERR_CONFIG, "gc_plan_create: node %lld depends on a later node", (long long)i);
                return GC_ERR_CONFIG;
            }
        if (nd.kind == NODE_GATHER) p->cap_x = (const void*)nd.a[0];
        if (nd.kind == NODE_SCATTER) p->cap_y = (const void*)nd.a[4];
    }
    p->deps.assign(deps, deps + ndeps);
    p->nstreams = (int)nstreams;
    cudaError_t e = cudaSuccess;
    for (int s = 0; s < nstreams && e == cudaSuccess; ++s) {
        cudaStream_t st;
        e = cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, stream_prio[s]);
        if (e == cudaSuccess) p->streams.push_back(st);
    }
    for (int64_t i = 0; i < n && e == cudaSuccess; ++i) {
        cudaEvent_t ev;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) p->events.push_back(ev);
    }
    if (e != cudaSuccess) {
        destroy(p);
        return cuda_status(e, "gc_plan_create streams");
    }
    // capture: fork every side stream from stream 0, nodes in order, join
    cudaStream_t origin = p->streams[0];
    int rc = GC_OK;
    cudaEvent_t fork;
    e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(origin, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        destroy(p);
        return cuda_status(e, "gc_plan_create begin capture");
    }
    cudaEventRecord(fork, origin);
    std::vector<int64_t> last(nstreams, -1);
    std::vector<char> used(nstreams, 0);
    used[0] = 1;
    for (int64_t i = 0; i < n && rc == GC_OK; ++i) {
        const Node& nd = p->nodes[(size_t)i];
        cudaStream_t st = p->streams[(size_t)nd.stream];
        if (!used[nd.stream]) {
            cudaStreamWaitEvent(st, fork, 0);
            used[nd.stream] = 1;
        }
        for (int64_t k = 0; k < nd.ndeps; ++k) {
            const int64_t d = p->deps[nd.dep_off + k];
            if (p->nodes[(size_t)d].stream != nd.stream) cudaStreamWaitEvent(st, p->events[(size_t)d], 0);
        }
        rc = launch_node(nd, st);
        if (rc == GC_OK) cudaEventRecord(p->events[(size_t)i], st);
        last[nd.stream] = i;
    }
    for (int s = 1; s < nstreams && rc == GC_OK; ++s)
        if (last[s] >= 0) cudaStreamWaitEvent(origin, p->events[(size_t)last[s]], 0);
    cudaGraph_t g = nullptr;
    cudaError_t ee = cudaStreamEndCapture(origin, &g);
    cudaEventDestroy(fork);
    if (rc != GC_OK || ee != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        destroy(p);
        return rc != GC_OK ? rc : cuda_status(ee, "gc_plan_create end capture");
    }
    p->graph = g;
    // per-node launch priorities (the schedule's bucket / chain ordering)
    // apply inside a graph only with this flag
    e = cudaGraphInstantiateWithFlags(&p->exec, g, cudaGraphInstantiateFlagUseNodePriority);
    if (e != cudaSuccess) {
        destroy(p);
        return cuda_status(e, "gc_plan_create instantiate");
    }
    p->bound_x = p->cap_x;
    p->bound_y = p->cap_y;
    *out = p;
    return GC_OK;
}

// One product: re-point the gather input at x and the scatter output at y
// (device or mapped pinned host memory, external order) when they changed,
// then launch the graph on `stream`.  x / y may be NULL: keep the binding.
extern "C" int gc_plan_run(void* plan, const double* x, double* y, void* stream) {
    Plan* p = (Plan*)plan;
    if (!p || !p->exec) { set_error(GC_ERR_STATE, "gc_plan_run: no plan"); return GC_ERR_STATE; }
    int32_t cnt = 0;
    if (x && (const void*)x != p->bound_x) {
        if (!p->cap_x) { set_error(GC_ERR_CONFIG, "gc_plan_run: plan has no gather node"); return GC_ERR_CONFIG; }
        if (int rc = gc_graph_retarget(p->graph, p->exec, 2, 0, p->cap_x, x, &cnt)) return rc;
        if (cnt != 1) { set_error(GC_ERR_STATE, "gc_plan_run: %d gather nodes re-pointed", cnt); return GC_ERR_STATE; }
        p->bound_x = x;
    }
    if (y && (const void*)y != p->bound_y) {
        if (!p->cap_y) { set_error(GC_ERR_CONFIG, "gc_plan_run: plan has no scatter node"); return GC_ERR_CONFIG; }
        if (int rc = gc_graph_retarget(p->graph, p->exec, 3, 4, p->cap_y, y, &cnt)) return rc;
        if (cnt != 1) { set_error(GC_ERR_STATE, "gc_plan_run: %d scatter nodes re-pointed", cnt); return GC_ERR_STATE; }
        p->bound_y = y;
    }
    cudaError_t e = cudaGraphLaunch(p->exec, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "gc_plan_run");
    return GC_OK;
}

// The synchronous host-vector product (h2.mvm) as one call: copy the
// caller's host x (any host memory, n_in doubles) into the pinned staging
// buffer x_pinned, run the graph reading x_pinned and writing the pinned y
// directly (over the host link), and wait for it on `stream`.
extern "C" int gc_plan_run_host(void* plan, const double* x_host, double* x_pinned, int64_t n_in, double* y_pinned,
                                void* stream) {
    if (!x_host || !x_pinned || !y_pinned || n_in < 0) {
        set_error(GC_ERR_CONFIG, "gc_plan_run_host: bad arguments");
        return GC_ERR_CONFIG;
    }
    std::memcpy(x_pinned, x_host, (size_t)n_in * sizeof(double));
    if (int rc = gc_plan_run(plan, x_pinned, y_pinned, stream)) return rc;
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "gc_plan_run_host");
    return GC_OK;
}

extern "C" int gc_plan_destroy(void* plan) {
    destroy((Plan*)plan);
    return GC_OK;
}
