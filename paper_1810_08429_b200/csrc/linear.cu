// Piecewise-linear Galerkin basis (assembly.py:54-135,
// 175-214, 279-304): every triangle pair contributes a 3x3 matrix of
// integrals k(x, y) phi_a(x) phi_c(y) (phi the barycentric hat functions of
// the two triangles), which is scattered onto the vertex DOFs.
//
// Three kernels:
//  * k_lin_pairs: one thread per triangle pair.  Classifies the pair;
//    disjoint pairs integrate the q^2 x q^2 tensor rule into 9 accumulators
//    (per column point: 3 row-weighted partial sums, then 9 FMAs); singular
//    pairs are pushed to the per-case queues.
//  * k_lin_singular: the reference's full Sauter-Schwab rules (the xi
//    factorisation of the constant basis does not apply: the hat functions
//    are affine in xi), one warp per pair, lanes over the rule points, a
//    fixed butterfly for the 9 sums.  Pair values are kept in the canonical
//    permuted local order of batchexec.py:70-76.
//  * k_lin_gather: one thread per block entry sums, in a fixed order, the
//    contributions of every (row triangle, column triangle) pair touching
//    the two vertices - the deterministic replacement of the executor's
//    np.add.at scatter (batchexec.py:200-209).
#include "common.cuh"

namespace gcb {

template <bool DLP>
__device__ __forceinline__ double lin_kern(double d0, double d1, double d2, double n0, double n1, double n2) {
    const double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
    const double ri = rsqrt_fast(r2);
    if (!DLP) return ri;
    const double dot = fma(d2, n2, fma(d1, n1, d0 * n0));
    return dot * (ri * ri * ri);
}

// regular rule: weights and the barycentric values of its points
struct LinRule {
    double w[64];
    double b[64][3];
};

__device__ __forceinline__ void lin_push(const gc_queue& q, int kase, int64_t t, int64_t s, int px, int py,
                                         int64_t idx, int32_t* flags) {
    const int slot = atomicAdd(q.count + kase, 1);
    if (slot >= q.cap[kase]) {
        atomicOr(flags, FLAG_OVERFLOW);
        return;
    }
    int64_t* dst = q.tasks[kase] + 4 * (int64_t)slot;
    dst[0] = t;
    dst[1] = s;
    dst[2] = (int64_t)px | ((int64_t)py << 8);
    dst[3] = idx;
}

// tasks: (t, s) per pair; U: 9 values per pair (canonical permuted order);
// pp: px | py << 8 per pair
// Pair i of a batch: explicit (t, s) from `tasks`, or - `blk` given - the
// pair (tri_r[tr_off + p], tri_c[tc_off + q]) of the block whose task range
// holds i (blk rows: task_base, n_col_tris, tr_off, tc_off; ascending
// task_base), p = local / n_col_tris, q = local % n_col_tris.  The product
// of the row and column triangle tables never exists in memory.
struct PairSource {
    const int64_t* tasks;
    const int64_t* blk;
    int64_t nblk;
    const int64_t* tri_r;
    const int64_t* tri_c;
};

__device__ __forceinline__ void pair_of(const PairSource& ps, int64_t i, int64_t& t, int64_t& s) {
    if (ps.blk == nullptr) {
        t = __ldg(ps.tasks + 2 * i);
        s = __ldg(ps.tasks + 2 * i + 1);
        return;
    }
    int64_t lo = 0, hi = ps.nblk - 1;
    while (lo < hi) {                                   // last block with task_base <= i
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(ps.blk + 4 * mid) <= i) lo = mid; else hi = mid - 1;
    }
    const int64_t* b = ps.blk + 4 * lo;
    const int64_t local = i - __ldg(b), tc = __ldg(b + 1);
    const int64_t pr = local / tc, qc = local - pr * tc;
    t = __ldg(ps.tri_r + __ldg(b + 2) + pr);
    s = __ldg(ps.tri_c + __ldg(b + 3) + qc);
}

template <int M, bool DLP>
__global__ void __launch_bounds__(128) k_lin_pairs(gc_geom g, LinRule lr, PairSource ps,
                                                   int64_t n, double* __restrict__ U, int32_t* __restrict__ pp,
                                                   gc_queue q, int32_t* flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t t, s;
        pair_of(ps, i, t, s);
        int64_t tv[3], sv[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            tv[k] = __ldg(g.tri_vid + 3 * t + k);
            sv[k] = __ldg(g.tri_vid + 3 * s + k);
        }
        int px, py;
        const int kase = classify_pair(tv, sv, &px, &py);
        pp[i] = px | (py << 8);
        if (kase != 0) {
            lin_push(q, kase, t, s, px, py, i, flags);
            continue;
        }
        const double* xt = g.xq + t * 3 * M;
        const double* xs = g.xq + s * 3 * M;
        double X[M][3];
#pragma unroll
        for (int k = 0; k < M; ++k) {
            X[k][0] = __ldg(xt + 3 * k);
            X[k][1] = __ldg(xt + 3 * k + 1);
            X[k][2] = __ldg(xt + 3 * k + 2);
        }
        double n0 = 0.0, n1 = 0.0, n2 = 0.0;
        if (DLP) {
            n0 = __ldg(g.normals + 3 * s);
            n1 = __ldg(g.normals + 3 * s + 1);
            n2 = __ldg(g.normals + 3 * s + 2);
        }
        // curved charts: per-point Gramians (row always, column for the
        // single layer) and per-point normals (double layer)
        const bool curv = g.gq != nullptr;
        double acc[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
#pragma unroll 1
        for (int j = 0; j < M; ++j) {
            const double y0 = __ldg(xs + 3 * j), y1 = __ldg(xs + 3 * j + 1), y2 = __ldg(xs + 3 * j + 2);
            if (DLP && curv) {
                n0 = __ldg(g.nq + (s * M + j) * 3);
                n1 = __ldg(g.nq + (s * M + j) * 3 + 1);
                n2 = __ldg(g.nq + (s * M + j) * 3 + 2);
            }
            double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
            for (int k = 0; k < M; ++k) {
                const double wxk = curv ? lr.w[k] * __ldg(g.gq + t * M + k) : lr.w[k];
                const double wk = wxk * lin_kern<DLP>(X[k][0] - y0, X[k][1] - y1, X[k][2] - y2, n0, n1, n2);
                p0 = fma(wk, lr.b[k][0], p0);
                p1 = fma(wk, lr.b[k][1], p1);
                p2 = fma(wk, lr.b[k][2], p2);
            }
            const double wj = (curv && !DLP) ? lr.w[j] * __ldg(g.gq + s * M + j) : lr.w[j];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double f = wj * lr.b[j][c];
                acc[0][c] = fma(p0, f, acc[0][c]);
                acc[1][c] = fma(p1, f, acc[1][c]);
                acc[2][c] = fma(p2, f, acc[2][c]);
            }
        }
        double sc = INV_FOUR_PI;
        if (!curv) {
            const double gt = __ldg(g.gram + t) * INV_FOUR_PI;
            sc = DLP ? gt : gt * __ldg(g.gram + s);
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int c = 0; c < 3; ++c) U[9 * i + 3 * a + c] = sc * acc[a][c];
    }
}

// singular pairs, the full rule: table SoA (x1, x2, y1, y2, w) x P
template <bool DLP>
__global__ void __launch_bounds__(128) k_lin_singular(gc_geom g, const double* __restrict__ rule, int P,
                                                      const int64_t* __restrict__ tasks, int64_t n,
                                                      double* __restrict__ U) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t task = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); task < n; task += nw) {
        const int64_t* tk = tasks + 4 * task;
        const int64_t t = tk[0], s = tk[1], pk = tk[2], idx = tk[3];
        const int px = (int)(pk & 0xff), py = (int)((pk >> 8) & 0xff);
        const double* ct = g.corners + 9 * t;
        const double* cs = g.corners + 9 * s;
        const int p0 = kPerms3[px][0], p1 = kPerms3[px][1], p2 = kPerms3[px][2];
        const int q0 = kPerms3[py][0], q1 = kPerms3[py][1], q2 = kPerms3[py][2];
        double E1[3], E2[3], F1[3], F2[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            E1[c] = ct[3 * p1 + c] - ct[3 * p0 + c];
            E2[c] = ct[3 * p2 + c] - ct[3 * p0 + c];
            F1[c] = cs[3 * q1 + c] - cs[3 * q0 + c];
            F2[c] = cs[3 * q2 + c] - cs[3 * q0 + c];
        }
        double n0 = 0.0, n1 = 0.0, n2 = 0.0;
        if (DLP) {
            n0 = g.normals[3 * s];
            n1 = g.normals[3 * s + 1];
            n2 = g.normals[3 * s + 2];
        }
        double acc[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] = 0.0;
        for (int p = lane; p < P; p += 32) {
            const double x1 = __ldg(rule + p), x2 = __ldg(rule + P + p);
            const double y1 = __ldg(rule + 2 * P + p), y2 = __ldg(rule + 3 * P + p);
            const double w = __ldg(rule + 4 * P + p);
            double d[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) d[c] = fma(x1, E1[c], fma(x2, E2[c], -fma(y1, F1[c], y2 * F2[c])));
            const double wk = w * lin_kern<DLP>(d[0], d[1], d[2], n0, n1, n2);
            const double bx[3] = {1.0 - x1 - x2, x1, x2};
            const double by[3] = {1.0 - y1 - y2, y1, y2};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double f = wk * bx[a];
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[3 * a + c] = fma(f, by[c], acc[3 * a + c]);
            }
        }
#pragma unroll
        for (int k = 0; k < 9; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
        if (lane == 0) {
            const double gt = g.gram[t] * INV_FOUR_PI;
            const double sc = DLP ? gt : gt * g.gram[s];
#pragma unroll
            for (int k = 0; k < 9; ++k) U[9 * idx + k] = sc * acc[k];
        }
    }
}

__device__ __constant__ static const int8_t kInvPerms3[6][3] = {
    {0, 1, 2}, {2, 0, 1}, {1, 2, 0}, {0, 2, 1}, {2, 1, 0}, {1, 0, 2}};

// desc (nb, 7): row_ptr_off, nr, col_ptr_off, nc, out_off, task_base, ncol_tris
// rptr/cptr: CSR offsets per DOF into rlist/clist (packed (table_row << 2) | slot)
__global__ void k_lin_gather(int64_t nb, const int64_t* __restrict__ desc, const int64_t* __restrict__ rptr,
                             const int64_t* __restrict__ rlist, const int64_t* __restrict__ cptr,
                             const int64_t* __restrict__ clist, const double* __restrict__ U,
                             const int32_t* __restrict__ pp, double* __restrict__ out) {
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int64_t* d = desc + 7 * b;
        const int64_t ro = d[0], co = d[2], out_off = d[4], base = d[5], tc = d[6];
        const int nr = (int)d[1], nc = (int)d[3];
        for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) {
            const int i = e % nr, j = e / nr;
            double sum = 0.0;
            for (int64_t u = rptr[ro + i]; u < rptr[ro + i + 1]; ++u) {
                const int64_t rp = rlist[u] >> 2;
                const int k = (int)(rlist[u] & 3);
                for (int64_t v = cptr[co + j]; v < cptr[co + j + 1]; ++v) {
                    const int64_t cq = clist[v] >> 2;
                    const int l = (int)(clist[v] & 3);
                    const int64_t task = base + rp * tc + cq;
                    const int32_t w = pp[task];
                    const int a = kInvPerms3[w & 0xff][k], c = kInvPerms3[(w >> 8) & 0xff][l];
                    sum += U[9 * task + 3 * a + c];
                }
            }
            out[out_off + (int64_t)j * nr + i] = sum;
        }
    }
}

}  // namespace gcb

using namespace gcb;

static int lin_pairs(const gc_geom* gp, const double* rule_w, const double* rule_b, int64_t n,
                     const PairSource& ps, double* U, int32_t* pp, gc_queue* qp, int32_t* flags,
                     void* stream);

extern "C" int gc_lin_pairs(const gc_geom* gp, const double* rule_w, const double* rule_b, int64_t n,
                            const int64_t* tasks, double* U, int32_t* pp, gc_queue* qp, int32_t* flags,
                            void* stream) {
    const PairSource ps{tasks, nullptr, 0, nullptr, nullptr};
    return lin_pairs(gp, rule_w, rule_b, n, ps, U, pp, qp, flags, stream);
}

extern "C" int gc_lin_pairs_blocks(const gc_geom* gp, const double* rule_w, const double* rule_b, int64_t n,
                                   int64_t nblk, const int64_t* blk, const int64_t* tri_r, const int64_t* tri_c,
                                   double* U, int32_t* pp, gc_queue* qp, int32_t* flags, void* stream) {
    if (nblk <= 0 || !blk || !tri_r || !tri_c) { set_error(GC_ERR_CONFIG, "gc_lin_pairs_blocks: no blocks"); return GC_ERR_CONFIG; }
    const PairSource ps{nullptr, blk, nblk, tri_r, tri_c};
    return lin_pairs(gp, rule_w, rule_b, n, ps, U, pp, qp, flags, stream);
}

static int lin_pairs(const gc_geom* gp, const double* rule_w, const double* rule_b, int64_t n,
                     const PairSource& ps, double* U, int32_t* pp, gc_queue* qp, int32_t* flags,
                     void* stream) {
    if (!gp || !qp || !rule_w || !rule_b) { set_error(GC_ERR_CONFIG, "gc_lin_pairs: null argument"); return GC_ERR_CONFIG; }
    if (n <= 0) return GC_OK;
    const gc_geom g = *gp;
    if (g.kernel && !g.normals) { set_error(GC_ERR_CONFIG, "double layer needs gc_geom.normals"); return GC_ERR_CONFIG; }
    if (g.mq != 9 && g.mq != 4 && g.mq != 16) {
        set_error(GC_ERR_CONFIG, "gc_lin_pairs: regular order q_reg in {2, 3, 4} (got %lld points)", (long long)g.mq);
        return GC_ERR_CONFIG;
    }
    LinRule lr;
    for (int k = 0; k < 64; ++k) {
        lr.w[k] = k < g.mq ? rule_w[k] : 0.0;
        for (int c = 0; c < 3; ++c) lr.b[k][c] = k < g.mq ? rule_b[3 * k + c] : 0.0;
    }
    cudaStream_t st = (cudaStream_t)stream;
    int64_t grid = (n + 127) / 128;
    if (grid > 148 * 32) grid = 148 * 32;
    const gc_queue q = *qp;
#define LIN_LAUNCH(M)                                                                                   \
    do {                                                                                                \
        if (g.kernel)                                                                                   \
            k_lin_pairs<M, true><<<(unsigned)grid, 128, 0, st>>>(g, lr, ps, n, U, pp, q, flags);        \
        else                                                                                            \
            k_lin_pairs<M, false><<<(unsigned)grid, 128, 0, st>>>(g, lr, ps, n, U, pp, q, flags);       \
    } while (0)
    if (g.mq == 9) LIN_LAUNCH(9);
    else if (g.mq == 4) LIN_LAUNCH(4);
    else LIN_LAUNCH(16);
#undef LIN_LAUNCH
    GC_CHECK_LAUNCH("k_lin_pairs");
    return GC_OK;
}

extern "C" int gc_lin_singular(const gc_geom* gp, const gc_rules* rp, gc_queue* qp, double* U,
                               int64_t* counts_out, void* stream) {
    if (!gp || !rp || !qp) { set_error(GC_ERR_CONFIG, "gc_lin_singular: null argument"); return GC_ERR_CONFIG; }
    if (gp->gq) { set_error(GC_ERR_CONFIG, "curved charts: flush with gc_curved_singular"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    int32_t counts[4] = {0, 0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(counts, qp->count, sizeof(counts), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_status(e, "gc_lin_singular counts");
    const gc_geom g = *gp;
    for (int k = 1; k <= 3; ++k) {
        if (counts[k] > qp->cap[k]) {
            set_error(GC_ERR_STATE, "singular queue %d overflow (%d > %lld)", k, counts[k], (long long)qp->cap[k]);
            return GC_ERR_STATE;
        }
        if (counts_out) counts_out[k] = counts[k];
        if (counts[k] == 0) continue;
        if (!rp->table[k] || rp->npts[k] <= 0) { set_error(GC_ERR_CONFIG, "full rule %d not uploaded", k); return GC_ERR_CONFIG; }
        int64_t grid = (counts[k] + 3) / 4;
        if (grid > 148 * 16) grid = 148 * 16;
        if (g.kernel)
            k_lin_singular<true><<<(unsigned)grid, 128, 0, st>>>(g, rp->table[k], (int)rp->npts[k], qp->tasks[k], counts[k], U);
        else
            k_lin_singular<false><<<(unsigned)grid, 128, 0, st>>>(g, rp->table[k], (int)rp->npts[k], qp->tasks[k], counts[k], U);
        GC_CHECK_LAUNCH("k_lin_singular");
    }
    e = cudaMemsetAsync(qp->count, 0, 4 * sizeof(int32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "gc_lin_singular reset");
    return GC_OK;
}

extern "C" int gc_lin_gather(int64_t nb, const int64_t* desc, const int64_t* rptr, const int64_t* rlist,
                             const int64_t* cptr, const int64_t* clist, const double* U, const int32_t* pp,
                             double* out, void* stream) {
    if (nb <= 0) return GC_OK;
    int64_t grid = nb < 148 * 32 ? nb : 148 * 32;
    k_lin_gather<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(nb, desc, rptr, rlist, cptr, clist, U, pp, out);
    GC_CHECK_LAUNCH("k_lin_gather");
    return GC_OK;
}

// ---------------------------------------------------------------------------
// Collocation (assembly.py:219-276, 340-362): rows are surface points (mesh
// vertices), columns the linear basis.  A task (v, s) is the single
// integral of k(x_v, y) phi_c(y) over triangle s: the regular rule (the
// q_reg chart points of s) when v is not a corner of s, else the collapsed
// Gauss rule with v rotated to corner 0 (duffy_rule(0, q_sing)), where
// y - x_v = y1 E1 + y2 E2 carries no cancellation.  Values in the rotated
// (canonical) column order: U[9 i + c], pp[i] = rotation << 8.
__device__ __constant__ static const int8_t kOrder6c[3][6] = {
    {0, 1, 2, 3, 4, 5}, {1, 2, 0, 4, 5, 3}, {2, 0, 1, 5, 3, 4}};

struct ColRule {
    double w[64];        // regular rule weights
    double b[64][3];     // regular rule barycentrics
    double sw[64];       // singular (collapsed) rule weights
    double sp[64][2];    // singular rule points
    int ms;              // singular rule size
};

template <bool DLP>
__global__ void __launch_bounds__(128) k_col_pairs(gc_geom g, ColRule cr, const double* __restrict__ verts,
                                                   PairSource ps, int64_t n, double* __restrict__ U,
                                                   int32_t* __restrict__ pp, int32_t* nsing) {
    const int M = (int)g.mq;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v, s;
        pair_of(ps, i, v, s);
        int rot = -1;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (rot < 0 && __ldg(g.tri_vid + 3 * s + k) == v) rot = k;
        const double x0 = verts[3 * v], x1 = verts[3 * v + 1], x2 = verts[3 * v + 2];
        double n0 = 0.0, n1 = 0.0, n2 = 0.0;
        if (DLP) {
            n0 = __ldg(g.normals + 3 * s);
            n1 = __ldg(g.normals + 3 * s + 1);
            n2 = __ldg(g.normals + 3 * s + 2);
        }
        double acc[3] = {0.0, 0.0, 0.0};
        const bool curv = g.gq != nullptr;
        if (rot >= 0 && nsing != nullptr) atomicAdd(nsing, 1);
        if (curv && rot >= 0) {
            // curved chart, point at a corner: the rotated quadratic chart at
            // the collapsed rule's points (assembly.py:254-265)
            const double* P6 = g.nodes6 + 18 * s;
            const double* N6 = g.nrm6 + 18 * s;
            for (int m = 0; m < cr.ms; ++m) {
                const double y1 = cr.sp[m][0], y2 = cr.sp[m][1];
                const double l0 = 1.0 - y1 - y2;
                const double sh[6] = {l0 * (2.0 * l0 - 1.0), y1 * (2.0 * y1 - 1.0), y2 * (2.0 * y2 - 1.0),
                                      4.0 * l0 * y1, 4.0 * y1 * y2, 4.0 * y2 * l0};
                double Y[3], Nn[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double ay = 0.0, an = 0.0;
#pragma unroll
                    for (int a = 0; a < 6; ++a) {
                        ay = fma(sh[a], P6[3 * kOrder6c[rot][a] + c], ay);
                        an = fma(sh[a], N6[3 * kOrder6c[rot][a] + c], an);
                    }
                    Y[c] = ay;
                    Nn[c] = an;
                }
                const double gy = sqrt(fma(Nn[2], Nn[2], fma(Nn[1], Nn[1], Nn[0] * Nn[0])));
                const double k = lin_kern<DLP>(x0 - Y[0], x1 - Y[1], x2 - Y[2], Nn[0], Nn[1], Nn[2]);
                const double wk = cr.sw[m] * (DLP ? k : gy * k);
                const double b[3] = {l0, y1, y2};
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[c] = fma(wk, b[c], acc[c]);
            }
        } else if (rot < 0) {
            const double* yq = g.xq + s * 3 * M;
            for (int m = 0; m < M; ++m) {
                if (DLP && curv) {
                    n0 = __ldg(g.nq + (s * M + m) * 3);
                    n1 = __ldg(g.nq + (s * M + m) * 3 + 1);
                    n2 = __ldg(g.nq + (s * M + m) * 3 + 2);
                }
                const double k = lin_kern<DLP>(x0 - __ldg(yq + 3 * m), x1 - __ldg(yq + 3 * m + 1),
                                               x2 - __ldg(yq + 3 * m + 2), n0, n1, n2);
                const double wk = (curv && !DLP ? cr.w[m] * __ldg(g.gq + s * M + m) : cr.w[m]) * k;
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[c] = fma(wk, cr.b[m][c], acc[c]);
            }
        } else {
            // rotation rot puts corner rot first: PERMS3[rot] = (rot, rot+1, rot+2)
            const double* cs = g.corners + 9 * s;
            const int q0 = kPerms3[rot][0], q1 = kPerms3[rot][1], q2 = kPerms3[rot][2];
            double E1[3], E2[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                E1[c] = cs[3 * q1 + c] - cs[3 * q0 + c];
                E2[c] = cs[3 * q2 + c] - cs[3 * q0 + c];
            }
            for (int m = 0; m < cr.ms; ++m) {
                const double y1 = cr.sp[m][0], y2 = cr.sp[m][1];
                // x_v - y = -(y1 E1 + y2 E2)
                const double d0 = -fma(y1, E1[0], y2 * E2[0]);
                const double d1 = -fma(y1, E1[1], y2 * E2[1]);
                const double d2 = -fma(y1, E1[2], y2 * E2[2]);
                const double wk = cr.sw[m] * lin_kern<DLP>(d0, d1, d2, n0, n1, n2);
                const double b[3] = {1.0 - y1 - y2, y1, y2};
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[c] = fma(wk, b[c], acc[c]);
            }
        }
        const double sc = (DLP || curv) ? INV_FOUR_PI : __ldg(g.gram + s) * INV_FOUR_PI;
        if (rot < 0) rot = 0;
        pp[i] = rot << 8;
#pragma unroll
        for (int c = 0; c < 3; ++c) U[9 * i + c] = sc * acc[c];
    }
}

static int col_pairs(const gc_geom* gp, const double* verts, const double* reg_w, const double* reg_b,
                     int64_t ms, const double* sing_w, const double* sing_p, int64_t n, const PairSource& ps,
                     double* U, int32_t* pp, int32_t* nsing, void* stream);

extern "C" int gc_col_pairs(const gc_geom* gp, const double* verts, const double* reg_w, const double* reg_b,
                            int64_t ms, const double* sing_w, const double* sing_p, int64_t n,
                            const int64_t* tasks, double* U, int32_t* pp, void* stream) {
    const PairSource ps{tasks, nullptr, 0, nullptr, nullptr};
    return col_pairs(gp, verts, reg_w, reg_b, ms, sing_w, sing_p, n, ps, U, pp, nullptr, stream);
}

extern "C" int gc_col_pairs_blocks(const gc_geom* gp, const double* verts, const double* reg_w,
                                   const double* reg_b, int64_t ms, const double* sing_w, const double* sing_p,
                                   int64_t n, int64_t nblk, const int64_t* blk, const int64_t* pts_r,
                                   const int64_t* tri_c, double* U, int32_t* pp, int32_t* nsing, void* stream) {
    if (nblk <= 0 || !blk || !pts_r || !tri_c) { set_error(GC_ERR_CONFIG, "gc_col_pairs_blocks: no blocks"); return GC_ERR_CONFIG; }
    const PairSource ps{nullptr, blk, nblk, pts_r, tri_c};
    return col_pairs(gp, verts, reg_w, reg_b, ms, sing_w, sing_p, n, ps, U, pp, nsing, stream);
}

static int col_pairs(const gc_geom* gp, const double* verts, const double* reg_w, const double* reg_b,
                     int64_t ms, const double* sing_w, const double* sing_p, int64_t n, const PairSource& ps,
                     double* U, int32_t* pp, int32_t* nsing, void* stream) {
    if (!gp || !verts || !reg_w || !reg_b || !sing_w || !sing_p) {
        set_error(GC_ERR_CONFIG, "gc_col_pairs: null argument");
        return GC_ERR_CONFIG;
    }
    if (n <= 0) return GC_OK;
    const gc_geom g = *gp;
    if (g.kernel && !g.normals) { set_error(GC_ERR_CONFIG, "double layer needs gc_geom.normals"); return GC_ERR_CONFIG; }
    if (g.mq < 1 || g.mq > 64 || ms < 1 || ms > 64) {
        set_error(GC_ERR_CONFIG, "gc_col_pairs: rules of 1..64 points (q <= 8)");
        return GC_ERR_CONFIG;
    }
    ColRule cr;
    for (int k = 0; k < 64; ++k) {
        cr.w[k] = k < g.mq ? reg_w[k] : 0.0;
        for (int c = 0; c < 3; ++c) cr.b[k][c] = k < g.mq ? reg_b[3 * k + c] : 0.0;
        cr.sw[k] = k < ms ? sing_w[k] : 0.0;
        cr.sp[k][0] = k < ms ? sing_p[2 * k] : 0.0;
        cr.sp[k][1] = k < ms ? sing_p[2 * k + 1] : 0.0;
    }
    cr.ms = (int)ms;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t grid = (n + 127) / 128;
    if (grid > 148 * 32) grid = 148 * 32;
    if (g.kernel)
        k_col_pairs<true><<<(unsigned)grid, 128, 0, st>>>(g, cr, verts, ps, n, U, pp, nsing);
    else
        k_col_pairs<false><<<(unsigned)grid, 128, 0, st>>>(g, cr, verts, ps, n, U, pp, nsing);
    GC_CHECK_LAUNCH("k_col_pairs");
    return GC_OK;
}
