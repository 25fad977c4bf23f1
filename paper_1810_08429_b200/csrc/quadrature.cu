// Batched Galerkin pair quadrature for the single-layer kernel 1/(4 pi r),
// piecewise-constant basis, plane charts (assembly.py:159-216).
//
// Disjoint pairs (the regular q_reg^2 x q_reg^2 tensor rule) are one thread
// per matrix entry: the q^2 row points stay in registers, the column points
// are broadcast across the warp, and 1/r comes from a MUFU seed plus one
// cubic-corrected Newton step (common.cuh rsqrt_fast).  Singular pairs
// (Sauter-Schwab vertex / edge / identical rules) are queued by the block
// kernel and integrated by a CTA-per-4-tasks kernel: 256 threads split the
// rule points, every rule point loaded once serves 4 tasks, and a fixed
// reduction tree makes each value independent of how tasks were grouped.
#include "common.cuh"

namespace gcb {

// sum_i sum_j w_i w_j / |X_i - Y_j| with X in registers (M compile-time)
template <int M>
__device__ __forceinline__ double disjoint_sum(const double* __restrict__ xq_t,
                                               const double* __restrict__ xq_s,
                                               const double* __restrict__ wq) {
    double X[M][3];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        X[i][0] = __ldg(xq_t + 3 * i);
        X[i][1] = __ldg(xq_t + 3 * i + 1);
        X[i][2] = __ldg(xq_t + 3 * i + 2);
    }
    double wi[M];
#pragma unroll
    for (int i = 0; i < M; ++i) wi[i] = __ldg(wq + i);
    double total = 0.0;
#pragma unroll 1
    for (int j = 0; j < M; ++j) {
        const double y0 = __ldg(xq_s + 3 * j), y1 = __ldg(xq_s + 3 * j + 1),
                     y2 = __ldg(xq_s + 3 * j + 2);
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double d0 = X[i][0] - y0, d1 = X[i][1] - y1, d2 = X[i][2] - y2;
            double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
            acc = fma(wi[i], rsqrt_fast(r2), acc);
        }
        total = fma(wi[j], acc, total);
    }
    return total;
}

// generic (any mq) variant reading both point sets from L1
__device__ double disjoint_sum_any(const double* __restrict__ xq_t,
                                   const double* __restrict__ xq_s,
                                   const double* __restrict__ wq, int mq) {
    double total = 0.0;
    for (int j = 0; j < mq; ++j) {
        const double y0 = __ldg(xq_s + 3 * j), y1 = __ldg(xq_s + 3 * j + 1),
                     y2 = __ldg(xq_s + 3 * j + 2);
        double acc = 0.0;
        for (int i = 0; i < mq; ++i) {
            double d0 = __ldg(xq_t + 3 * i) - y0, d1 = __ldg(xq_t + 3 * i + 1) - y1,
                   d2 = __ldg(xq_t + 3 * i + 2) - y2;
            double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
            acc = fma(__ldg(wq + i), rsqrt_fast(r2), acc);
        }
        total = fma(__ldg(wq + j), acc, total);
    }
    return total;
}

template <int M>
__device__ __forceinline__ double disjoint_entry(const gc_geom& g, int64_t t, int64_t s) {
    double sum;
    if (M > 0)
        sum = disjoint_sum<(M > 0 ? M : 1)>(g.xq + t * 3 * M, g.xq + s * 3 * M, g.wq);
    else
        sum = disjoint_sum_any(g.xq + t * 3 * g.mq, g.xq + s * 3 * g.mq, g.wq, (int)g.mq);
    return (__ldg(g.gram + t) * __ldg(g.gram + s) * INV_FOUR_PI) * sum;
}

__device__ __forceinline__ void push_task(gc_queue q, int kase, int64_t t, int64_t s, int px,
                                          int py, int64_t out_idx, int32_t* flags) {
    int slot = atomicAdd(q.count + kase, 1);
    if (slot >= q.cap[kase]) {
        atomicOr(flags, FLAG_OVERFLOW);
        return;
    }
    int64_t* dst = q.tasks[kase] + 4 * (int64_t)slot;
    dst[0] = t;
    dst[1] = s;
    dst[2] = (int64_t)px | ((int64_t)py << 8);
    dst[3] = out_idx;
}

// one CTA per block, one thread per entry, column-major output
template <int M>
__global__ void __launch_bounds__(256) k_assemble_blocks(gc_geom g, const int64_t* __restrict__ desc,
                                                         const int64_t* __restrict__ row_idx,
                                                         const int64_t* __restrict__ col_idx,
                                                         double* __restrict__ out, gc_queue q,
                                                         int32_t* flags) {
    const int64_t* d = desc + 5 * (int64_t)blockIdx.x;
    const int64_t row_off = d[0], col_off = d[2], out_off = d[4];
    const int nr = (int)d[1], nc = (int)d[3];
    const int total = nr * nc;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        int a = e % nr, b = e / nr;
        int64_t t = __ldg(row_idx + row_off + a);
        int64_t s = __ldg(col_idx + col_off + b);
        int64_t tv[3], sv[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            tv[k] = __ldg(g.tri_vid + 3 * t + k);
            sv[k] = __ldg(g.tri_vid + 3 * s + k);
        }
        int px, py;
        int kase = classify_pair(tv, sv, &px, &py);
        if (kase == 0)
            out[out_off + e] = disjoint_entry<M>(g, t, s);
        else
            push_task(q, kase, t, s, px, py, out_off + e, flags);
    }
}

// evaluator seam, disjoint case: one thread per task
template <int M>
__global__ void k_pair_disjoint(gc_geom g, int64_t B, const int64_t* __restrict__ rows,
                                const int64_t* __restrict__ cols, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = disjoint_entry<M>(g, __ldg(rows + i), __ldg(cols + i));
}

// pack seam arrays into queue-format tasks
__global__ void k_pack_tasks(int64_t B, const int64_t* rows, const int64_t* cols,
                             const int64_t* px, const int64_t* py, int64_t* tasks) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B;
         i += (int64_t)gridDim.x * blockDim.x) {
        tasks[4 * i] = rows[i];
        tasks[4 * i + 1] = cols[i];
        tasks[4 * i + 2] = px[i] | (py[i] << 8);
        tasks[4 * i + 3] = i;
    }
}

constexpr int SING_THREADS = 256;
constexpr int SING_G = 4;  // tasks per CTA

// Singular pairs.  Vertex/edge: D = x1 E1 + x2 E2 - y1 F1 - y2 F2 with
// E_k = P_k - P_0 (row chart after its alignment permutation), F likewise
// for the column chart; P_0 == Q_0 is the shared vertex, so the difference
// is formed without cancellation.  Identical: D = dx E1 + dy E2.
template <int KASE>
__global__ void __launch_bounds__(SING_THREADS) k_singular(gc_geom g, const double* __restrict__ rule,
                                                           int64_t P, const int64_t* __restrict__ tasks,
                                                           int64_t ntasks, double* __restrict__ out) {
    const int64_t first = (int64_t)blockIdx.x * SING_G;
    double E1[SING_G][3], E2[SING_G][3], F1[SING_G][3], F2[SING_G][3];
    double scale[SING_G];
    int64_t oidx[SING_G];
#pragma unroll
    for (int k = 0; k < SING_G; ++k) {
        int64_t id = first + k;
        bool live = id < ntasks;
        const int64_t* tk = tasks + 4 * (live ? id : first);
        int64_t t = tk[0], s = tk[1], pp = tk[2];
        oidx[k] = live ? tk[3] : -1;
        int px = (int)(pp & 0xff), py = (int)((pp >> 8) & 0xff);
        const double* ct = g.corners + 9 * t;
        const double* cs = g.corners + 9 * s;
        int p0 = kPerms3[px][0], p1 = kPerms3[px][1], p2 = kPerms3[px][2];
        int q0 = kPerms3[py][0], q1 = kPerms3[py][1], q2 = kPerms3[py][2];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            E1[k][c] = ct[3 * p1 + c] - ct[3 * p0 + c];
            E2[k][c] = ct[3 * p2 + c] - ct[3 * p0 + c];
            F1[k][c] = cs[3 * q1 + c] - cs[3 * q0 + c];
            F2[k][c] = cs[3 * q2 + c] - cs[3 * q0 + c];
        }
        scale[k] = g.gram[t] * g.gram[s] * INV_FOUR_PI;
    }
    double acc[SING_G];
#pragma unroll
    for (int k = 0; k < SING_G; ++k) acc[k] = 0.0;
    const double* rx1 = rule;
    const double* rx2 = rule + P;
    const double* ry1 = rule + 2 * P;
    const double* ry2 = rule + 3 * P;
    const double* rw = rule + 4 * P;
    for (int64_t p = threadIdx.x; p < P; p += SING_THREADS) {
        const double x1 = __ldg(rx1 + p), x2 = __ldg(rx2 + p), w = __ldg(rw + p);
        if (KASE == 3) {
#pragma unroll
            for (int k = 0; k < SING_G; ++k) {
                double d0 = fma(x1, E1[k][0], x2 * E2[k][0]);
                double d1 = fma(x1, E1[k][1], x2 * E2[k][1]);
                double d2 = fma(x1, E1[k][2], x2 * E2[k][2]);
                double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
                acc[k] = fma(w, rsqrt_fast(r2), acc[k]);
            }
        } else {
            const double y1 = __ldg(ry1 + p), y2 = __ldg(ry2 + p);
#pragma unroll
            for (int k = 0; k < SING_G; ++k) {
                double d[3];
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    d[c] = fma(x1, E1[k][c], fma(x2, E2[k][c], -fma(y1, F1[k][c], y2 * F2[k][c])));
                double r2 = fma(d[2], d[2], fma(d[1], d[1], d[0] * d[0]));
                acc[k] = fma(w, rsqrt_fast(r2), acc[k]);
            }
        }
    }
    // fixed-order reduction: warp butterfly, then warp partials in order
    __shared__ double part[SING_THREADS / 32][SING_G];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < SING_G; ++k) {
        double v = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) part[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < SING_G) {
        const int k = threadIdx.x;
        double v = 0.0;
        for (int w = 0; w < SING_THREADS / 32; ++w) v += part[w][k];
        if (oidx[k] >= 0) out[oidx[k]] = scale[k] * v;
    }
}

static int launch_singular(const gc_geom& g, const gc_rules& r, int kase, const int64_t* tasks,
                           int64_t n, double* out, cudaStream_t st) {
    if (n <= 0) return GC_OK;
    if (!r.table[kase] || r.npts[kase] <= 0) {
        set_error(GC_ERR_CONFIG, "singular rule for case %d not uploaded", kase);
        return GC_ERR_CONFIG;
    }
    int64_t grid = (n + SING_G - 1) / SING_G;
    if (grid > 0x7fffffffLL) {
        set_error(GC_ERR_CONFIG, "too many singular tasks");
        return GC_ERR_CONFIG;
    }
    switch (kase) {
        case 1: k_singular<1><<<(unsigned)grid, SING_THREADS, 0, st>>>(g, r.table[1], r.npts[1], tasks, n, out); break;
        case 2: k_singular<2><<<(unsigned)grid, SING_THREADS, 0, st>>>(g, r.table[2], r.npts[2], tasks, n, out); break;
        case 3: k_singular<3><<<(unsigned)grid, SING_THREADS, 0, st>>>(g, r.table[3], r.npts[3], tasks, n, out); break;
        default: set_error(GC_ERR_CONFIG, "bad singular case %d", kase); return GC_ERR_CONFIG;
    }
    GC_CHECK_LAUNCH("k_singular");
    return GC_OK;
}

template <int M>
static void launch_blocks(const gc_geom& g, int64_t nb, const int64_t* desc, int threads,
                          const int64_t* ri, const int64_t* ci, double* out, gc_queue q,
                          int32_t* flags, cudaStream_t st) {
    k_assemble_blocks<M><<<(unsigned)nb, threads, 0, st>>>(g, desc, ri, ci, out, q, flags);
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gc_pair_eval(const gc_geom* gp, const gc_rules* rp, int kase, int64_t B, const int64_t* rows,
                 const int64_t* cols, const int64_t* px, const int64_t* py, double* out,
                 void* stream) {
    if (!gp || !rp) { set_error(GC_ERR_CONFIG, "null geometry/rules"); return GC_ERR_CONFIG; }
    if (B <= 0) return GC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const gc_geom g = *gp;
    if (kase == 0) {
        int64_t grid = (B + 127) / 128;
        if (grid > 148 * 64) grid = 148 * 64;
        if (g.mq == 9)
            k_pair_disjoint<9><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        else if (g.mq == 4)
            k_pair_disjoint<4><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        else if (g.mq == 16)
            k_pair_disjoint<16><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        else
            k_pair_disjoint<0><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        GC_CHECK_LAUNCH("k_pair_disjoint");
        return GC_OK;
    }
    if (kase < 1 || kase > 3) { set_error(GC_ERR_CONFIG, "bad case %d", kase); return GC_ERR_CONFIG; }
    int64_t* tasks = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&tasks, (size_t)B * 4 * sizeof(int64_t), st);
    if (e != cudaSuccess) return cuda_status(e, "gc_pair_eval alloc");
    int64_t grid = (B + 255) / 256;
    if (grid > 148 * 64) grid = 148 * 64;
    k_pack_tasks<<<(unsigned)grid, 256, 0, st>>>(B, rows, cols, px, py, tasks);
    GC_CHECK_LAUNCH("k_pack_tasks");
    int rc = launch_singular(g, *rp, kase, tasks, B, out, st);
    cudaFreeAsync(tasks, st);
    return rc;
}

int gc_assemble_blocks(const gc_geom* gp, int64_t nb, const int64_t* desc,
                       int64_t max_block_entries, const int64_t* row_idx, const int64_t* col_idx,
                       double* out, gc_queue* qp, int32_t* flags, void* stream) {
    if (!gp || !qp) { set_error(GC_ERR_CONFIG, "null geometry/queue"); return GC_ERR_CONFIG; }
    if (nb <= 0) return GC_OK;
    if (nb > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "too many blocks"); return GC_ERR_CONFIG; }
    int threads = max_block_entries >= 256 ? 256 : (max_block_entries > 32 ? (int)((max_block_entries + 31) / 32 * 32) : 32);
    cudaStream_t st = (cudaStream_t)stream;
    const gc_geom g = *gp;
    switch (g.mq) {
        case 9: launch_blocks<9>(g, nb, desc, threads, row_idx, col_idx, out, *qp, flags, st); break;
        case 4: launch_blocks<4>(g, nb, desc, threads, row_idx, col_idx, out, *qp, flags, st); break;
        case 16: launch_blocks<16>(g, nb, desc, threads, row_idx, col_idx, out, *qp, flags, st); break;
        default: launch_blocks<0>(g, nb, desc, threads, row_idx, col_idx, out, *qp, flags, st); break;
    }
    GC_CHECK_LAUNCH("k_assemble_blocks");
    return GC_OK;
}

int gc_singular_flush(const gc_geom* gp, const gc_rules* rp, gc_queue* qp, double* out,
                      int64_t* counts_out, void* stream) {
    if (!gp || !rp || !qp) { set_error(GC_ERR_CONFIG, "null argument"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    int32_t counts[4] = {0, 0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(counts, qp->count, sizeof(counts), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_singular_flush counts");
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_status(e, "gc_singular_flush sync");
    for (int k = 1; k <= 3; ++k) {
        if (counts[k] > qp->cap[k]) {
            set_error(GC_ERR_STATE, "singular queue %d overflow (%d > %lld)", k, counts[k],
                      (long long)qp->cap[k]);
            return GC_ERR_STATE;
        }
        if (counts_out) counts_out[k] = counts[k];
        int rc = launch_singular(*gp, *rp, k, qp->tasks[k], counts[k], out, st);
        if (rc) return rc;
    }
    e = cudaMemsetAsync(qp->count, 0, 4 * sizeof(int32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "gc_singular_flush reset");
    return GC_OK;
}

}  // extern "C"
