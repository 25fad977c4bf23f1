// Error plumbing, launch accounting, permutation gather/scatter, chart
// quadrature points and the FP64 throughput probe.
#include <atomic>
#include <cmath>
#include <stdarg.h>
#include <string.h>

#include "common.cuh"

namespace gcb {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

void set_error(int code, const char* fmt, ...) {
    (void)code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t err, const char* what) {
    set_error(GC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(err));
    return GC_ERR_CUDA;
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

// xt[i] = x[perm[i]]
__global__ void k_gather(const double* __restrict__ x, const int64_t* __restrict__ perm,
                         int64_t n, double* __restrict__ xt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        xt[i] = __ldg(x + __ldg(perm + i));
}

// y[perm[i]] = yt[i]
__global__ void k_scatter(const double* __restrict__ yt, const int64_t* __restrict__ perm,
                          int64_t n, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[__ldg(perm + i)] = yt[i];
}

// y[perm[i]] = yt[i] + yt2[i]
__global__ void k_scatter2(const double* __restrict__ yt, const double* __restrict__ yt2,
                           const int64_t* __restrict__ perm, int64_t n, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[__ldg(perm + i)] = yt[i] + yt2[i];
}

// The same two steps indexed from the external side (iperm = inverse of
// perm): reads of x / writes of y are contiguous, so x and y may live in
// mapped pinned host memory (the product graph reads and writes the
// caller's host buffers directly, h2.mvm).
// xt[iperm[j]] = x[j].  The product's first forward tier is its programmatic
// dependent (PDL): released at once, it stages its matrix while this runs.
__global__ void k_gather_inv(const double* __restrict__ x, const int64_t* __restrict__ iperm,
                             int64_t n, double* __restrict__ xt) {
    asm volatile("griddepcontrol.launch_dependents;");
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        xt[__ldg(iperm + j)] = x[j];
}

// y[j] = yt[iperm[j]] + yt2[iperm[j]].  Launched as the programmatic
// dependent of the leaf-row tier (PDL): it loads its indices, then waits
// for the tier's results.
__global__ void k_scatter2_inv(const double* __restrict__ yt, const double* __restrict__ yt2,
                               const int64_t* __restrict__ iperm, int64_t n, double* __restrict__ y) {
    const int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t i0 = j0 < n ? __ldg(iperm + j0) : 0;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (j0 < n) y[j0] = yt[i0] + yt2[i0];
    for (int64_t j = j0 + (int64_t)gridDim.x * blockDim.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = __ldg(iperm + j);
        y[j] = yt[i] + yt2[i];
    }
}

// Plane chart data and cluster support of every triangle (geometry.py:266-293
// chart_pack, :324-338 control_points, clustering.py:107-128 support boxes,
// TriangleMesh.centroids) in numpy's operation order, without contraction,
// so the results are bit-identical to the host arrays:
//   nodes 3..5 = 0.5 * (p_i + p_j); du, dv = sum_a g[a] * node[a] in node
//   order; n = cross(du, dv) (a1*b2 - a2*b1, ...); gram = sqrt((n0^2 +
//   n1^2) + n2^2); control points 3..5 = 0.5 * ((4 m - p_i) - p_j); lo / hi
//   = min / max over the 6 control points; centroid = ((a + b) + c) / 3.
// Outputs: corners (nt,3,3), gram (nt), normal (nt,3), support (nt,9) =
// [lo | hi | centroid] (the cluster tree's per-dof pack).
struct ChartGrads { double gu[6], gv[6]; };

__global__ void k_chart_pack(const double* __restrict__ verts, const int64_t* __restrict__ tris, int64_t nt,
                             ChartGrads g, double* __restrict__ corners, double* __restrict__ gram,
                             double* __restrict__ normal, double* __restrict__ support) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt;
         t += (int64_t)gridDim.x * blockDim.x) {
        double node[6][3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int64_t v = tris[3 * t + k];
#pragma unroll
            for (int c = 0; c < 3; ++c) node[k][c] = verts[3 * v + c];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            node[3][c] = __dmul_rn(0.5, __dadd_rn(node[0][c], node[1][c]));
            node[4][c] = __dmul_rn(0.5, __dadd_rn(node[1][c], node[2][c]));
            node[5][c] = __dmul_rn(0.5, __dadd_rn(node[2][c], node[0][c]));
        }
        double du[3], dv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double a = 0.0, b = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                a = __dadd_rn(a, __dmul_rn(g.gu[k], node[k][c]));
                b = __dadd_rn(b, __dmul_rn(g.gv[k], node[k][c]));
            }
            du[c] = a;
            dv[c] = b;
        }
        const double n0 = __dsub_rn(__dmul_rn(du[1], dv[2]), __dmul_rn(du[2], dv[1]));
        const double n1 = __dsub_rn(__dmul_rn(du[2], dv[0]), __dmul_rn(du[0], dv[2]));
        const double n2 = __dsub_rn(__dmul_rn(du[0], dv[1]), __dmul_rn(du[1], dv[0]));
        gram[t] = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(n0, n0), __dmul_rn(n1, n1)), __dmul_rn(n2, n2)));
        normal[3 * t] = n0;
        normal[3 * t + 1] = n1;
        normal[3 * t + 2] = n2;
        double* sp = support + 9 * t;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            corners[9 * t + c] = node[0][c];
            corners[9 * t + 3 + c] = node[1][c];
            corners[9 * t + 6 + c] = node[2][c];
            // np.minimum(lo, q) = lo < q ? lo : q (x86 MINPD: the second
            // operand on ties, so signed zeros land as numpy's do)
            double lo = node[0][c], hi = node[0][c];
            lo = lo < node[1][c] ? lo : node[1][c];
            hi = hi > node[1][c] ? hi : node[1][c];
            lo = lo < node[2][c] ? lo : node[2][c];
            hi = hi > node[2][c] ? hi : node[2][c];
            const int ij[3][2] = {{0, 1}, {1, 2}, {2, 0}};
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                const double q = __dmul_rn(
                    0.5, __dsub_rn(__dsub_rn(__dmul_rn(4.0, node[3 + e][c]), node[ij[e][0]][c]), node[ij[e][1]][c]));
                lo = lo < q ? lo : q;
                hi = hi > q ? hi : q;
            }
            sp[c] = lo;
            sp[3 + c] = hi;
            sp[6 + c] = __ddiv_rn(__dadd_rn(__dadd_rn(node[0][c], node[1][c]), node[2][c]), 3.0);
        }
    }
}

// xq[t,m,c] = sum_a n6[m,a] * node[t,a,c], sequential, no contraction; nodes
// 3..5 are the straight midpoints 0.5*(p_i + p_j) (geometry.py:278-280).
__global__ void k_surface_points(const double* __restrict__ corners, int64_t nt,
                                 const double* __restrict__ n6, int64_t mq,
                                 double* __restrict__ xq) {
    int64_t total = nt * mq;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t t = i / mq;
        int m = (int)(i % mq);
        const double* p = corners + 9 * t;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double node[6];
            node[0] = p[c];
            node[1] = p[3 + c];
            node[2] = p[6 + c];
            node[3] = __dmul_rn(0.5, __dadd_rn(node[0], node[1]));
            node[4] = __dmul_rn(0.5, __dadd_rn(node[1], node[2]));
            node[5] = __dmul_rn(0.5, __dadd_rn(node[2], node[0]));
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < 6; ++a) acc = __dadd_rn(acc, __dmul_rn(n6[m * 6 + a], node[a]));
            xq[i * 3 + c] = acc;
        }
    }
}

// one CTA per matrix: out[off + c*rows + r] = in[off + r*cols + c]
__global__ void k_batched_transpose(const int64_t* __restrict__ desc, const double* __restrict__ in,
                                    double* __restrict__ out) {
    const int64_t off = desc[3 * blockIdx.x], rows = desc[3 * blockIdx.x + 1],
                  cols = desc[3 * blockIdx.x + 2];
    for (int64_t e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int64_t c = e / rows, r = e - c * rows;
        out[off + e] = in[off + r * cols + c];
    }
}

// 8 independent DFMA chains per thread
__global__ void k_dfma_probe(int64_t iters, double* out) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double m = 0.999999, c = 1e-7;
    for (int64_t i = 0; i < iters; ++i) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
    double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

static inline int grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 148 * 64) b = 148 * 64;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gc_abi_version(void) { return GC_ABI_VERSION; }
const char* gc_last_error(void) { return g_err; }
uint64_t gc_launch_count(void) { return g_launches.load(); }
void gc_reset_launch_count(void) { g_launches.store(0); }

int gc_gather(const double* x, const int64_t* perm, int64_t n, double* xt, void* stream) {
    if (n <= 0) return GC_OK;
    k_gather<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, perm, n, xt);
    GC_CHECK_LAUNCH("gc_gather");
    return GC_OK;
}

int gc_scatter(const double* yt, const int64_t* perm, int64_t n, double* y, void* stream) {
    if (n <= 0) return GC_OK;
    k_scatter<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(yt, perm, n, y);
    GC_CHECK_LAUNCH("gc_scatter");
    return GC_OK;
}

int gc_scatter2(const double* yt, const double* yt2, const int64_t* perm, int64_t n, double* y,
                void* stream) {
    if (n <= 0) return GC_OK;
    k_scatter2<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(yt, yt2, perm, n, y);
    GC_CHECK_LAUNCH("gc_scatter2");
    return GC_OK;
}

// Re-point a pointer argument of the gather / scatter kernel nodes of an
// instantiated CUDA graph (cudaGraphExecKernelNodeSetParams): the product
// graph then reads the caller's x and writes the caller's y directly, with
// no device copies around the replay.  kernel 0 = k_gather (4 arguments),
// 1 = k_scatter2 (5), 2 = k_gather_inv (4), 3 = k_scatter2_inv (5); only nodes whose captured argument `arg` (the value
// in the graph, which exec updates do not change) equals old_ptr change.
// *count = nodes updated.
int gc_graph_retarget(void* graph, void* exec, int32_t kernel, int32_t arg, const void* old_ptr,
                      const void* new_ptr, int32_t* count) {
    const void* fns[4] = {(const void*)k_gather, (const void*)k_scatter2, (const void*)k_gather_inv,
                          (const void*)k_scatter2_inv};
    const void* fn = kernel >= 0 && kernel < 4 ? fns[kernel] : nullptr;
    const int nargs = (kernel & 1) ? 5 : 4;
    if (!fn || arg < 0 || arg >= nargs || !graph || !exec) {
        set_error(GC_ERR_CONFIG, "gc_graph_retarget: bad kernel/arg/graph");
        return GC_ERR_CONFIG;
    }
    // captured nodes may carry the host stub or the driver function handle
    cudaFunction_t drv = nullptr;
    if (cudaGetFuncBySymbol(&drv, fn) != cudaSuccess) drv = nullptr;
    size_t n = 0;
    cudaError_t e = cudaGraphGetNodes((cudaGraph_t)graph, nullptr, &n);
    if (e != cudaSuccess) return cuda_status(e, "gc_graph_retarget nodes");
    cudaGraphNode_t stack_nodes[256];
    cudaGraphNode_t* nodes = n <= 256 ? stack_nodes : (cudaGraphNode_t*)malloc(n * sizeof(cudaGraphNode_t));
    e = cudaGraphGetNodes((cudaGraph_t)graph, nodes, &n);
    int32_t cnt = 0;
    for (size_t i = 0; e == cudaSuccess && i < n; ++i) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nodes[i], &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams p;
        if (cudaGraphKernelNodeGetParams(nodes[i], &p) != cudaSuccess) continue;
        if (p.func != fn && (drv == nullptr || p.func != (void*)drv)) continue;
        if (*(void* const*)p.kernelParams[arg] != old_ptr) continue;
        void* args[5];
        for (int a = 0; a < nargs; ++a) args[a] = p.kernelParams[a];
        void* nv = const_cast<void*>(new_ptr);
        args[arg] = &nv;
        p.kernelParams = args;
        p.extra = nullptr;
        e = cudaGraphExecKernelNodeSetParams((cudaGraphExec_t)exec, nodes[i], &p);
        ++cnt;
    }
    if (nodes != stack_nodes) free(nodes);
    (void)cudaGetLastError();
    if (e != cudaSuccess) return cuda_status(e, "gc_graph_retarget");
    if (count) *count = cnt;
    return GC_OK;
}

int gc_gather_inv(const double* x, const int64_t* iperm, int64_t n, double* xt, void* stream) {
    if (n <= 0) return GC_OK;
    k_gather_inv<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, iperm, n, xt);
    GC_CHECK_LAUNCH("gc_gather_inv");
    return GC_OK;
}

int gc_scatter2_inv(const double* yt, const double* yt2, const int64_t* iperm, int64_t n, double* y,
                    void* stream) {
    if (n <= 0) return GC_OK;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(n, 256));
    cfg.blockDim = dim3(256);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_scatter2_inv, yt, yt2, iperm, n, y);
    if (e != cudaSuccess) return cuda_status(e, "gc_scatter2_inv");
    count_launch();
    return GC_OK;
}

int gc_surface_points(const double* corners, int64_t nt, const double* n6, int64_t mq,
                      double* xq, void* stream) {
    if (nt <= 0) return GC_OK;
    if (mq <= 0) {
        set_error(GC_ERR_CONFIG, "gc_surface_points: mq must be positive");
        return GC_ERR_CONFIG;
    }
    k_surface_points<<<grid_for(nt * mq, 256), 256, 0, (cudaStream_t)stream>>>(
        corners, nt, n6, mq, xq);
    GC_CHECK_LAUNCH("gc_surface_points");
    return GC_OK;
}

int gc_chart_pack(const double* verts, const int64_t* tris, int64_t nt, const double* gu, const double* gv,
                  double* corners, double* gram, double* normal, double* support, void* stream) {
    if (nt <= 0) return GC_OK;
    if (!verts || !tris || !gu || !gv || !corners || !gram || !normal || !support) {
        set_error(GC_ERR_CONFIG, "gc_chart_pack: null argument");
        return GC_ERR_CONFIG;
    }
    ChartGrads g;
    for (int k = 0; k < 6; ++k) g.gu[k] = gu[k], g.gv[k] = gv[k];
    k_chart_pack<<<grid_for(nt, 256), 256, 0, (cudaStream_t)stream>>>(verts, tris, nt, g, corners, gram, normal,
                                                                      support);
    GC_CHECK_LAUNCH("gc_chart_pack");
    return GC_OK;
}

int gc_batched_transpose(int64_t nn, const int64_t* desc, const double* in, double* out,
                         void* stream) {
    if (nn <= 0) return GC_OK;
    k_batched_transpose<<<(unsigned)nn, 256, 0, (cudaStream_t)stream>>>(desc, in, out);
    GC_CHECK_LAUNCH("gc_batched_transpose");
    return GC_OK;
}

int gc_host_norm3(const double* v, int64_t n, double* out, int mode) {
    // host helper: Euclidean norms of n 3-vectors with a chosen rounding
    // sequence (mode 0: sqrt(fma(z,z,fma(y,y,x*x))), the OpenBLAS ddot tail;
    // mode 1: sqrt((x*x + y*y) + z*z) without contraction)
    if (n < 0 || (mode != 0 && mode != 1)) {
        set_error(GC_ERR_CONFIG, "gc_host_norm3: bad arguments");
        return GC_ERR_CONFIG;
    }
    for (int64_t i = 0; i < n; ++i) {
        const double x = v[3 * i], y = v[3 * i + 1], z = v[3 * i + 2];
        volatile double xx = x * x;
        double s;
        if (mode == 0) {
            s = std::fma(z, z, std::fma(y, y, (double)xx));
        } else {
            volatile double yy = y * y, zz = z * z;
            volatile double t = (double)xx + (double)yy;
            s = (double)t + (double)zz;
        }
        out[i] = std::sqrt(s);
    }
    return GC_OK;
}

int gc_dfma_probe(int64_t blocks, int64_t threads, int64_t iters, double* out, void* stream) {
    k_dfma_probe<<<(int)blocks, (int)threads, 0, (cudaStream_t)stream>>>(iters, out);
    GC_CHECK_LAUNCH("gc_dfma_probe");
    return GC_OK;
}

}  // extern "C"

// out[off[i] + j] = start[i] + j for j < len[i] (int32): the input-index
// lists of the matvec panels, expanded on the device from per-block ranges
__global__ void k_expand_ranges_impl(int64_t n, const int64_t* __restrict__ start, const int64_t* __restrict__ len,
                                const int64_t* __restrict__ off, int32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const int64_t s = start[i], L = len[i], o = off[i];
        for (int64_t j = threadIdx.x; j < L; j += blockDim.x) out[o + j] = (int32_t)(s + j);
    }
}

extern "C" int gc_expand_ranges(int64_t n, const int64_t* start, const int64_t* len, const int64_t* off,
                                int32_t* out, void* stream) {
    if (n <= 0) return GC_OK;
    const int64_t grid = n < 148 * 64 ? n : 148 * 64;
    k_expand_ranges_impl<<<(unsigned)grid, 64, 0, (cudaStream_t)stream>>>(n, start, len, off, out);
    GC_CHECK_LAUNCH("k_expand_ranges");
    return GC_OK;
}
