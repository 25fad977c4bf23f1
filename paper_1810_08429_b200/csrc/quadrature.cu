// Batched Galerkin pair quadrature, piecewise-constant basis, plane charts
// (assembly.py:159-216): the single-layer kernel 1/(4 pi r) and (DLP) the
// double-layer kernel <x - y, n_y>/(4 pi r^3), n_y the column triangle's
// chart normal (|n_y| carries the column Gramian, assembly.py:196-201).
//
// Disjoint pairs (the regular q_reg^2 x q_reg^2 tensor rule): one CTA per
// block.  The block's row and column quadrature points are staged in shared
// memory; each thread owns one row (its q^2 points in registers) and two
// adjacent columns, so every shared-memory read of a column point feeds
// q^2 independent distance evaluations.  1/r is a MUFU seed plus one
// cubic-corrected Newton step (common.cuh rsqrt_fast).
//
// Singular pairs (Sauter-Schwab vertex / edge / identical) are queued by the
// block kernel and integrated by persistent warps: the rule (xi-reduced, see
// quadrature.reduced_sauter_rule) sits in shared memory, each warp takes 2
// tasks at a time, lane l evaluates rule points l, l+32, ... and a fixed
// butterfly sums the lanes - every value is independent of how tasks were
// grouped or scheduled, so assembly is bitwise reproducible.
#include "common.cuh"

namespace gcb {

// integrand without 1/(4 pi): 1/r (single layer) or <d, n>/r^3 (double layer)
template <bool DLP>
__device__ __forceinline__ double kern(double d0, double d1, double d2, double n0, double n1, double n2) {
    const double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
    const double ri = rsqrt_fast(r2);
    if (!DLP) return ri;
    const double dot = fma(d2, n2, fma(d1, n1, d0 * n0));
    return dot * (ri * ri * ri);
}

// sum_i sum_j w_i w_j / |X_i - Y_j| reading both point sets from global
// (evaluator seam, one thread per task)
template <int M, bool DLP>
__device__ __forceinline__ double disjoint_sum(const double* __restrict__ xq_t,
                                               const double* __restrict__ xq_s,
                                               const double* __restrict__ wq, const double* ns) {
    double X[M][3];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        X[i][0] = __ldg(xq_t + 3 * i);
        X[i][1] = __ldg(xq_t + 3 * i + 1);
        X[i][2] = __ldg(xq_t + 3 * i + 2);
    }
    const double n0 = DLP ? ns[0] : 0.0, n1 = DLP ? ns[1] : 0.0, n2 = DLP ? ns[2] : 0.0;
    double total = 0.0;
#pragma unroll 1
    for (int j = 0; j < M; ++j) {
        const double y0 = __ldg(xq_s + 3 * j), y1 = __ldg(xq_s + 3 * j + 1),
                     y2 = __ldg(xq_s + 3 * j + 2);
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < M; ++i)
            acc = fma(__ldg(wq + i), kern<DLP>(X[i][0] - y0, X[i][1] - y1, X[i][2] - y2, n0, n1, n2), acc);
        total = fma(__ldg(wq + j), acc, total);
    }
    return total;
}

template <bool DLP>
__device__ double disjoint_sum_any(const double* __restrict__ xq_t,
                                   const double* __restrict__ xq_s,
                                   const double* __restrict__ wq, int mq, const double* ns) {
    const double n0 = DLP ? ns[0] : 0.0, n1 = DLP ? ns[1] : 0.0, n2 = DLP ? ns[2] : 0.0;
    double total = 0.0;
    for (int j = 0; j < mq; ++j) {
        const double y0 = __ldg(xq_s + 3 * j), y1 = __ldg(xq_s + 3 * j + 1),
                     y2 = __ldg(xq_s + 3 * j + 2);
        double acc = 0.0;
        for (int i = 0; i < mq; ++i)
            acc = fma(__ldg(wq + i), kern<DLP>(__ldg(xq_t + 3 * i) - y0, __ldg(xq_t + 3 * i + 1) - y1,
                                               __ldg(xq_t + 3 * i + 2) - y2, n0, n1, n2), acc);
        total = fma(__ldg(wq + j), acc, total);
    }
    return total;
}

// entry scale: (gram_t / 4 pi) * gram_s (single layer) or gram_t / 4 pi
// (double layer: the column Gramian is |n_y|)
template <bool DLP>
__device__ __forceinline__ double entry_scale(const gc_geom& g, int64_t t, int64_t s) {
    const double gt = __ldg(g.gram + t) * INV_FOUR_PI;
    return DLP ? gt : gt * __ldg(g.gram + s);
}

template <int M, bool DLP>
__device__ __forceinline__ double disjoint_entry(const gc_geom& g, int64_t t, int64_t s) {
    double sum;
    const double* ns = DLP ? g.normals + 3 * s : nullptr;
    if (M > 0)
        sum = disjoint_sum<(M > 0 ? M : 1), DLP>(g.xq + t * 3 * M, g.xq + s * 3 * M, g.wq, ns);
    else
        sum = disjoint_sum_any<DLP>(g.xq + t * 3 * g.mq, g.xq + s * 3 * g.mq, g.wq, (int)g.mq, ns);
    return entry_scale<DLP>(g, t, s) * sum;  // same association as k_assemble_blocks
}

__device__ __forceinline__ void push_task(const gc_queue& q, int kase, int64_t t, int64_t s, int px,
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

constexpr int BLK_THREADS = 256;

struct RuleW;
static void e_copy_weights(const gc_geom& g, RuleW& rw, int M);

// quadrature weights as a kernel parameter: they live in the constant bank
// and feed the DFMAs directly instead of occupying 2*M registers
struct RuleW {
    double w[64];
};

// One CTA per block; column-major output.  Shared memory: row points
// (nr*M*3), column points (nc*M*3) and both vertex-id lists; the caller
// sizes the dynamic allocation for the largest block.  NT = 128 for the
// 16x16 near-field blocks (one thread per column pair), 256 otherwise.
template <int M, int NT, bool DLP, bool CURV>
__global__ void __launch_bounds__(NT) k_assemble_blocks(
    gc_geom g, RuleW rw, const int64_t* __restrict__ desc, const int64_t* __restrict__ row_idx,
    const int64_t* __restrict__ col_idx, double* __restrict__ out, gc_queue q, int32_t* flags) {
    extern __shared__ double sm[];
    const int64_t* d = desc + 5 * (int64_t)blockIdx.x;
    const int64_t row_off = d[0], col_off = d[2], out_off = d[4];
    const int nr = (int)d[1], nc = (int)d[3];
    double* Xs = sm;                                   // nr * M * 3
    double* Ys = Xs + nr * M * 3;                      // nc * M * 3
    int64_t* tvs = (int64_t*)(Ys + nc * M * 3);        // nr * 4: id, v0, v1, v2
    int64_t* svs = tvs + 4 * nr;                       // nc * 4
    for (int e = threadIdx.x; e < nr; e += NT) {
        const int64_t t = __ldg(row_idx + row_off + e);
        tvs[4 * e] = t;
#pragma unroll
        for (int k = 0; k < 3; ++k) tvs[4 * e + 1 + k] = __ldg(g.tri_vid + 3 * t + k);
    }
    for (int e = threadIdx.x; e < nc; e += NT) {
        const int64_t s = __ldg(col_idx + col_off + e);
        svs[4 * e] = s;
#pragma unroll
        for (int k = 0; k < 3; ++k) svs[4 * e + 1 + k] = __ldg(g.tri_vid + 3 * s + k);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nr * M * 3; e += NT) {
        const int a = e / (M * 3);
        Xs[e] = __ldg(g.xq + tvs[4 * a] * (M * 3) + (e - a * M * 3));
    }
    for (int e = threadIdx.x; e < nc * M * 3; e += NT) {
        const int b = e / (M * 3);
        Ys[e] = __ldg(g.xq + svs[4 * b] * (M * 3) + (e - b * M * 3));
    }
    __syncthreads();
    const int npairs = (nc + 1) / 2;
    for (int e = threadIdx.x; e < nr * npairs; e += NT) {
        const int a = e % nr, b0 = 2 * (e / nr);
        const bool two = b0 + 1 < nc;
        const int64_t t = tvs[4 * a];
        const int64_t tv[3] = {tvs[4 * a + 1], tvs[4 * a + 2], tvs[4 * a + 3]};
        bool live[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            live[c] = false;
            if (c == 1 && !two) continue;
            const int b = b0 + c;
            const int64_t sv[3] = {svs[4 * b + 1], svs[4 * b + 2], svs[4 * b + 3]};
            int px, py;
            const int kase = classify_pair(tv, sv, &px, &py);
            if (kase == 0)
                live[c] = true;
            else
                push_task(q, kase, t, svs[4 * b], px, py, out_off + (int64_t)b * nr + a, flags);
        }
        if (!live[0] && !live[1]) continue;
        double X[M][3];
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) X[i][k] = Xs[(a * M + i) * 3 + k];
        const int b1 = two ? b0 + 1 : b0;
        const double* Y0 = Ys + b0 * M * 3;
        const double* Y1 = Ys + b1 * M * 3;
        const int64_t s0 = svs[4 * b0], s1 = svs[4 * b1];
        double na[3] = {0.0, 0.0, 0.0}, nb[3] = {0.0, 0.0, 0.0};
        if (DLP && !CURV) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                na[k] = __ldg(g.normals + 3 * s0 + k);
                nb[k] = __ldg(g.normals + 3 * s1 + k);
            }
        }
        // curved charts: the point Gramians fold into the weights (row
        // always; column for the single layer - the double layer's |n_y| is
        // the interpolated normal)
        double wx[CURV ? M : 1];
        if (CURV) {
#pragma unroll
            for (int i = 0; i < M; ++i) wx[i] = rw.w[i] * __ldg(g.gq + t * M + i);
        }
        double tot0 = 0.0, tot1 = 0.0;
#pragma unroll 1
        for (int j = 0; j < M; ++j) {
            const double u0 = Y0[3 * j], u1 = Y0[3 * j + 1], u2 = Y0[3 * j + 2];
            const double v0 = Y1[3 * j], v1 = Y1[3 * j + 1], v2 = Y1[3 * j + 2];
            if (DLP && CURV) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    na[k] = __ldg(g.nq + (s0 * M + j) * 3 + k);
                    nb[k] = __ldg(g.nq + (s1 * M + j) * 3 + k);
                }
            }
            double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const double wi = CURV ? wx[CURV ? i : 0] : rw.w[i];
                acc0 = fma(wi, kern<DLP>(X[i][0] - u0, X[i][1] - u1, X[i][2] - u2, na[0], na[1], na[2]), acc0);
                acc1 = fma(wi, kern<DLP>(X[i][0] - v0, X[i][1] - v1, X[i][2] - v2, nb[0], nb[1], nb[2]), acc1);
            }
            double wy0 = rw.w[j], wy1 = rw.w[j];
            if (CURV && !DLP) {
                wy0 *= __ldg(g.gq + s0 * M + j);
                wy1 *= __ldg(g.gq + s1 * M + j);
            }
            tot0 = fma(wy0, acc0, tot0);
            tot1 = fma(wy1, acc1, tot1);
        }
        const double sc0 = CURV ? INV_FOUR_PI : entry_scale<DLP>(g, t, s0);
        const double sc1 = CURV ? INV_FOUR_PI : entry_scale<DLP>(g, t, s1);
        if (live[0]) out[out_off + (int64_t)b0 * nr + a] = sc0 * tot0;
        if (live[1]) out[out_off + (int64_t)(b0 + 1) * nr + a] = sc1 * tot1;
    }
}

static void e_copy_weights(const gc_geom& g, RuleW& rw, int M) {
    for (int i = 0; i < 64; ++i) rw.w[i] = (i < M && g.wq_host) ? g.wq_host[i] : 0.0;
}

// Higher regular orders (q_reg^2 = M > 16, M <= 64): same structure as
// k_assemble_blocks, the row's points held in registers MC at a time.
template <int MC, int NT, bool DLP>
__global__ void __launch_bounds__(NT) k_assemble_blocks_big(
    gc_geom g, RuleW rw, int M, const int64_t* __restrict__ desc, const int64_t* __restrict__ row_idx,
    const int64_t* __restrict__ col_idx, double* __restrict__ out, gc_queue q, int32_t* flags) {
    extern __shared__ double sm[];
    const int64_t* d = desc + 5 * (int64_t)blockIdx.x;
    const int64_t row_off = d[0], col_off = d[2], out_off = d[4];
    const int nr = (int)d[1], nc = (int)d[3];
    double* Xs = sm;
    double* Ys = Xs + nr * M * 3;
    int64_t* tvs = (int64_t*)(Ys + nc * M * 3);
    int64_t* svs = tvs + 4 * nr;
    for (int e = threadIdx.x; e < nr; e += NT) {
        const int64_t t = __ldg(row_idx + row_off + e);
        tvs[4 * e] = t;
        for (int k = 0; k < 3; ++k) tvs[4 * e + 1 + k] = __ldg(g.tri_vid + 3 * t + k);
    }
    for (int e = threadIdx.x; e < nc; e += NT) {
        const int64_t s = __ldg(col_idx + col_off + e);
        svs[4 * e] = s;
        for (int k = 0; k < 3; ++k) svs[4 * e + 1 + k] = __ldg(g.tri_vid + 3 * s + k);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nr * M * 3; e += NT) {
        const int a = e / (M * 3);
        Xs[e] = __ldg(g.xq + tvs[4 * a] * (M * 3) + (e - a * M * 3));
    }
    for (int e = threadIdx.x; e < nc * M * 3; e += NT) {
        const int b = e / (M * 3);
        Ys[e] = __ldg(g.xq + svs[4 * b] * (M * 3) + (e - b * M * 3));
    }
    __syncthreads();
    const int npairs = (nc + 1) / 2;
    for (int e = threadIdx.x; e < nr * npairs; e += NT) {
        const int a = e % nr, b0 = 2 * (e / nr);
        const bool two = b0 + 1 < nc;
        const int64_t t = tvs[4 * a];
        const int64_t tv[3] = {tvs[4 * a + 1], tvs[4 * a + 2], tvs[4 * a + 3]};
        bool live[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            live[c] = false;
            if (c == 1 && !two) continue;
            const int b = b0 + c;
            const int64_t sv[3] = {svs[4 * b + 1], svs[4 * b + 2], svs[4 * b + 3]};
            int px, py;
            const int kase = classify_pair(tv, sv, &px, &py);
            if (kase == 0)
                live[c] = true;
            else
                push_task(q, kase, t, svs[4 * b], px, py, out_off + (int64_t)b * nr + a, flags);
        }
        if (!live[0] && !live[1]) continue;
        const int b1 = two ? b0 + 1 : b0;
        const double* Y0 = Ys + b0 * M * 3;
        const double* Y1 = Ys + b1 * M * 3;
        double na[3] = {0.0, 0.0, 0.0}, nb[3] = {0.0, 0.0, 0.0};
        if (DLP) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                na[k] = __ldg(g.normals + 3 * svs[4 * b0] + k);
                nb[k] = __ldg(g.normals + 3 * svs[4 * b1] + k);
            }
        }
        double tot0 = 0.0, tot1 = 0.0;
        for (int i0 = 0; i0 < M; i0 += MC) {
            double X[MC][3], wi[MC];
#pragma unroll
            for (int i = 0; i < MC; ++i) {
                const bool in = i0 + i < M;
#pragma unroll
                for (int k = 0; k < 3; ++k) X[i][k] = in ? Xs[(a * M + i0 + i) * 3 + k] : 1e30;
                wi[i] = in ? rw.w[i0 + i] : 0.0;
            }
#pragma unroll 1
            for (int j = 0; j < M; ++j) {
                const double u0 = Y0[3 * j], u1 = Y0[3 * j + 1], u2 = Y0[3 * j + 2];
                const double v0 = Y1[3 * j], v1 = Y1[3 * j + 1], v2 = Y1[3 * j + 2];
                double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                for (int i = 0; i < MC; ++i) {
                    // padded points (weight 0) sit far away: finite, nonzero r2
                    acc0 = fma(wi[i], kern<DLP>(X[i][0] - u0, X[i][1] - u1, X[i][2] - u2, na[0], na[1], na[2]), acc0);
                    acc1 = fma(wi[i], kern<DLP>(X[i][0] - v0, X[i][1] - v1, X[i][2] - v2, nb[0], nb[1], nb[2]), acc1);
                }
                tot0 = fma(rw.w[j], acc0, tot0);
                tot1 = fma(rw.w[j], acc1, tot1);
            }
        }
        if (live[0]) out[out_off + (int64_t)b0 * nr + a] = entry_scale<DLP>(g, t, svs[4 * b0]) * tot0;
        if (live[1]) out[out_off + (int64_t)(b0 + 1) * nr + a] = entry_scale<DLP>(g, t, svs[4 * b1]) * tot1;
    }
}

// generic-order fallback (any q_reg): one thread per entry, points from L1
__global__ void __launch_bounds__(BLK_THREADS) k_assemble_blocks_any(
    gc_geom g, const int64_t* __restrict__ desc, const int64_t* __restrict__ row_idx,
    const int64_t* __restrict__ col_idx, double* __restrict__ out, gc_queue q, int32_t* flags) {
    const int64_t* d = desc + 5 * (int64_t)blockIdx.x;
    const int64_t row_off = d[0], col_off = d[2], out_off = d[4];
    const int nr = (int)d[1], nc = (int)d[3];
    for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) {
        const int a = e % nr, b = e / nr;
        const int64_t t = __ldg(row_idx + row_off + a), s = __ldg(col_idx + col_off + b);
        int64_t tv[3], sv[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            tv[k] = __ldg(g.tri_vid + 3 * t + k);
            sv[k] = __ldg(g.tri_vid + 3 * s + k);
        }
        int px, py;
        const int kase = classify_pair(tv, sv, &px, &py);
        if (kase == 0)
            out[out_off + e] = g.kernel ? disjoint_entry<0, true>(g, t, s) : disjoint_entry<0, false>(g, t, s);
        else
            push_task(q, kase, t, s, px, py, out_off + e, flags);
    }
}

// evaluator seam, disjoint case: one thread per task
template <int M, bool DLP>
__global__ void k_pair_disjoint(gc_geom g, int64_t B, const int64_t* __restrict__ rows,
                                const int64_t* __restrict__ cols, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = disjoint_entry<M, DLP>(g, __ldg(rows + i), __ldg(cols + i));
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

#ifndef GC_SING_THREADS
#define GC_SING_THREADS 128
#endif
constexpr int SING_THREADS = GC_SING_THREADS;
constexpr int SING_WARPS = SING_THREADS / 32;
#ifndef GC_SING_G
#define GC_SING_G 4
#endif
constexpr int SING_G = GC_SING_G;   // tasks per warp
// per case (vertex NC=4, edge NC=3, identical NC=2); a task's value does not
// depend on it (lane-strided points, then the same shuffle tree)
#ifndef GC_SING_G4
#define GC_SING_G4 SING_G
#endif
#ifndef GC_SING_G3
#define GC_SING_G3 SING_G
#endif
#ifndef GC_SING_G2
#define GC_SING_G2 SING_G
#endif
template <int NC>
constexpr int sing_group() { return NC == 4 ? GC_SING_G4 : NC == 3 ? GC_SING_G3 : GC_SING_G2; }

// Singular pairs with the xi-reduced rule: D = sum_k coef[k] G_k,
//   NC = 4 (vertex):    G = (E1, E2, -F1, -F2)
//   NC = 3 (edge):      G = (E1, E2, -F2)          (E1 == F1)
//   NC = 2 (identical): G = (E1, E2)               (E == F)
// with E_k = P_k - P_0, F_k = Q_k - Q_0 after the alignment permutations;
// P_0 == Q_0 is the shared vertex, so D carries no cancellation.  The rule
// table (NC coefficient columns + weight, SoA, P points) is staged in
// shared memory when it fits, else read through L1.
template <int NC, bool SMEM, bool DLP, int SG = sing_group<NC>()>
__global__ void __launch_bounds__(SING_THREADS) k_singular(gc_geom g, const double* __restrict__ rule,
                                                           int P, const int64_t* __restrict__ tasks,
                                                           int64_t ntasks, double* __restrict__ out,
                                                           const int32_t* __restrict__ count) {
    extern __shared__ double sr[];
    // count: the queue's device counter (the asynchronous flush); ntasks is
    // then the capacity (overflow was flagged by the producer)
    if (count) ntasks = min((int64_t)*count, ntasks);
    const double* R = rule;
    if (SMEM) {
        for (int i = threadIdx.x; i < (NC + 1) * P; i += SING_THREADS) sr[i] = rule[i];
        __syncthreads();
        R = sr;
    }
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * SING_WARPS;
    const int64_t ngroups = (ntasks + SG - 1) / SG;
    for (int64_t grp = (int64_t)blockIdx.x * SING_WARPS + (threadIdx.x >> 5); grp < ngroups;
         grp += nwarps) {
        double G[SG][NC][3];
        double scale[SG];
        double nrm[SG][3];
        int64_t oidx[SG];
#pragma unroll
        for (int k = 0; k < SG; ++k) {
            const int64_t id = grp * SG + k;
            const bool live = id < ntasks;
            const int64_t* tk = tasks + 4 * (live ? id : grp * SG);
            const int64_t t = tk[0], s = tk[1], pp = tk[2];
            oidx[k] = live ? tk[3] : -1;
            const int px = (int)(pp & 0xff), py = (int)((pp >> 8) & 0xff);
            const double* ct = g.corners + 9 * t;
            const double* cs = g.corners + 9 * s;
            const int p0 = kPerms3[px][0], p1 = kPerms3[px][1], p2 = kPerms3[px][2];
            const int q0 = kPerms3[py][0], q1 = kPerms3[py][1], q2 = kPerms3[py][2];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                G[k][0][c] = ct[3 * p1 + c] - ct[3 * p0 + c];
                G[k][1][c] = ct[3 * p2 + c] - ct[3 * p0 + c];
                if (NC == 4) {
                    G[k][2 % NC][c] = -(cs[3 * q1 + c] - cs[3 * q0 + c]);
                    G[k][3 % NC][c] = -(cs[3 * q2 + c] - cs[3 * q0 + c]);
                } else if (NC == 3) {
                    G[k][2 % NC][c] = -(cs[3 * q2 + c] - cs[3 * q0 + c]);
                }
            }
            scale[k] = DLP ? g.gram[t] * INV_FOUR_PI : g.gram[t] * g.gram[s] * INV_FOUR_PI;
#pragma unroll
            for (int c = 0; c < 3; ++c) nrm[k][c] = DLP ? g.normals[3 * s + c] : 0.0;
        }
        double acc[SG];
#pragma unroll
        for (int k = 0; k < SG; ++k) acc[k] = 0.0;
        for (int p = lane; p < P; p += 32) {
            double cf[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) cf[j] = R[j * P + p];
            const double w = R[NC * P + p];
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                double dd[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double v = cf[0] * G[k][0][c];
#pragma unroll
                    for (int j = 1; j < NC; ++j) v = fma(cf[j], G[k][j][c], v);
                    dd[c] = v;
                }
                acc[k] = fma(w, kern<DLP>(dd[0], dd[1], dd[2], nrm[k][0], nrm[k][1], nrm[k][2]), acc[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < SG; ++k) {
            double v = acc[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && oidx[k] >= 0) out[oidx[k]] = scale[k] * v;
        }
    }
}

template <int NC, bool DLP>
static int launch_singular_nc(const gc_geom& g, const double* table, int64_t P, const int64_t* tasks,
                              int64_t n, double* out, cudaStream_t st, const int32_t* count) {
    const size_t bytes = (size_t)(NC + 1) * P * sizeof(double);
    const int64_t groups = (n + sing_group<NC>() - 1) / sing_group<NC>();
    int64_t grid = (groups + SING_WARPS - 1) / SING_WARPS;     // capped below: persistent warps
    if (bytes <= 200 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_singular<NC, true, DLP>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return cuda_status(e, "k_singular smem attribute");
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_singular<NC, true, DLP>, SING_THREADS, bytes);
        if (per_sm < 1) per_sm = 1;
        if (grid > 148LL * per_sm) grid = 148LL * per_sm;
        k_singular<NC, true, DLP><<<(unsigned)grid, SING_THREADS, bytes, st>>>(g, table, (int)P, tasks, n, out,
                                                                                 count);
    } else {
        if (grid > 148LL * 8) grid = 148LL * 8;
        k_singular<NC, false, DLP><<<(unsigned)grid, SING_THREADS, 0, st>>>(g, table, (int)P, tasks, n, out,
                                                                              count);
    }
    GC_CHECK_LAUNCH("k_singular");
    return GC_OK;
}

static int launch_singular(const gc_geom& g, const gc_rules& r, int kase, const int64_t* tasks,
                           int64_t n, double* out, cudaStream_t st, const int32_t* count = nullptr) {
    if (n <= 0) return GC_OK;
    if (!r.table[kase] || r.npts[kase] <= 0) {
        set_error(GC_ERR_CONFIG, "singular rule for case %d not uploaded", kase);
        return GC_ERR_CONFIG;
    }
    if (g.kernel && !g.normals) { set_error(GC_ERR_CONFIG, "double layer needs gc_geom.normals"); return GC_ERR_CONFIG; }
    switch (kase * 2 + (g.kernel ? 1 : 0)) {
        case 2: return launch_singular_nc<4, false>(g, r.table[1], r.npts[1], tasks, n, out, st, count);
        case 3: return launch_singular_nc<4, true>(g, r.table[1], r.npts[1], tasks, n, out, st, count);
        case 4: return launch_singular_nc<3, false>(g, r.table[2], r.npts[2], tasks, n, out, st, count);
        case 5: return launch_singular_nc<3, true>(g, r.table[2], r.npts[2], tasks, n, out, st, count);
        case 6: return launch_singular_nc<2, false>(g, r.table[3], r.npts[3], tasks, n, out, st, count);
        case 7: return launch_singular_nc<2, true>(g, r.table[3], r.npts[3], tasks, n, out, st, count);
        default: set_error(GC_ERR_CONFIG, "bad singular case %d", kase); return GC_ERR_CONFIG;
    }
}

template <int M, int NT, bool DLP, bool CURV = false>
static int launch_blocks_nt(const gc_geom& g, const RuleW& rw, int64_t nb, const int64_t* desc,
                            size_t bytes, const int64_t* ri, const int64_t* ci, double* out,
                            const gc_queue& q, int32_t* flags, cudaStream_t st) {
    if (g.gq && !CURV)
        return launch_blocks_nt<M, NT, DLP, true>(g, rw, nb, desc, bytes, ri, ci, out, q, flags, st);
    cudaError_t e = cudaFuncSetAttribute(k_assemble_blocks<M, NT, DLP, CURV>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return cuda_status(e, "k_assemble_blocks smem attribute");
    k_assemble_blocks<M, NT, DLP, CURV><<<(unsigned)nb, NT, bytes, st>>>(g, rw, desc, ri, ci, out, q, flags);
    GC_CHECK_LAUNCH("k_assemble_blocks");
    return GC_OK;
}

template <int M>
static int launch_blocks(const gc_geom& g, int64_t nb, const int64_t* desc, int64_t max_rows,
                         int64_t max_cols, const int64_t* ri, const int64_t* ci, double* out,
                         gc_queue q, int32_t* flags, cudaStream_t st) {
    const size_t bytes = (size_t)(max_rows + max_cols) * (M * 3 * sizeof(double) + 4 * sizeof(int64_t));
    if (bytes > 200 * 1024) {
        k_assemble_blocks_any<<<(unsigned)nb, BLK_THREADS, 0, st>>>(g, desc, ri, ci, out, q, flags);
        GC_CHECK_LAUNCH("k_assemble_blocks_any");
        return GC_OK;
    }
    if (!g.wq_host) { set_error(GC_ERR_CONFIG, "gc_geom.wq_host is required"); return GC_ERR_CONFIG; }
    RuleW rw;
    e_copy_weights(g, rw, M);
    const bool small = max_rows * ((max_cols + 1) / 2) <= 128;
    if (g.kernel)
        return small ? launch_blocks_nt<M, 128, true>(g, rw, nb, desc, bytes, ri, ci, out, q, flags, st)
                     : launch_blocks_nt<M, 256, true>(g, rw, nb, desc, bytes, ri, ci, out, q, flags, st);
    return small ? launch_blocks_nt<M, 128, false>(g, rw, nb, desc, bytes, ri, ci, out, q, flags, st)
                 : launch_blocks_nt<M, 256, false>(g, rw, nb, desc, bytes, ri, ci, out, q, flags, st);
}

template <int MC, int NT, bool DLP>
static int launch_big(const gc_geom& g, const RuleW& rw, int M, int64_t nb, const int64_t* desc,
                      size_t bytes, const int64_t* ri, const int64_t* ci, double* out, const gc_queue& q,
                      int32_t* flags, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(k_assemble_blocks_big<MC, NT, DLP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return cuda_status(e, "k_assemble_blocks_big smem");
    k_assemble_blocks_big<MC, NT, DLP><<<(unsigned)nb, NT, bytes, st>>>(g, rw, M, desc, ri, ci, out, q, flags);
    GC_CHECK_LAUNCH("k_assemble_blocks_big");
    return GC_OK;
}

}  // namespace gcb

using namespace gcb;

extern "C" {

int gc_pair_eval(const gc_geom* gp, const gc_rules* rp, int kase, int64_t B, const int64_t* rows,
                 const int64_t* cols, const int64_t* px, const int64_t* py, double* out,
                 void* stream) {
    if (!gp || !rp) { set_error(GC_ERR_CONFIG, "null geometry/rules"); return GC_ERR_CONFIG; }
    if (B <= 0) return GC_OK;
    if (gp->gq) { set_error(GC_ERR_CONFIG, "curved charts: evaluate with gc_curved_pairs"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    const gc_geom g = *gp;
    if (kase == 0) {
        int64_t grid = (B + 127) / 128;
        if (grid > 148 * 64) grid = 148 * 64;
        if (g.kernel && !g.normals) { set_error(GC_ERR_CONFIG, "double layer needs gc_geom.normals"); return GC_ERR_CONFIG; }
        if (g.mq == 9 && g.kernel)
            k_pair_disjoint<9, true><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        else if (g.mq == 9)
            k_pair_disjoint<9, false><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        else if (g.mq == 4 && g.kernel)
            k_pair_disjoint<4, true><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        else if (g.mq == 4)
            k_pair_disjoint<4, false><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        else if (g.kernel)
            k_pair_disjoint<0, true><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
        else
            k_pair_disjoint<0, false><<<(unsigned)grid, 128, 0, st>>>(g, B, rows, cols, out);
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

int gc_assemble_blocks(const gc_geom* gp, int64_t nb, const int64_t* desc, int64_t max_rows,
                       int64_t max_cols, const int64_t* row_idx, const int64_t* col_idx,
                       double* out, gc_queue* qp, int32_t* flags, void* stream) {
    if (!gp || !qp) { set_error(GC_ERR_CONFIG, "null geometry/queue"); return GC_ERR_CONFIG; }
    if (nb <= 0) return GC_OK;
    if (nb > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "too many blocks"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    const gc_geom g = *gp;
    if (g.kernel && !g.normals) { set_error(GC_ERR_CONFIG, "double layer needs gc_geom.normals"); return GC_ERR_CONFIG; }
    if (g.gq) {
        // curved charts: the shared-memory block kernel with per-point Gramians
        const size_t bytes = (size_t)(max_rows + max_cols) * (g.mq * 3 * sizeof(double) + 4 * sizeof(int64_t));
        if ((g.mq != 4 && g.mq != 9 && g.mq != 16) || bytes > 200 * 1024) {
            set_error(GC_ERR_CONFIG, "curved charts: q_reg in {2, 3, 4} and blocks of <= %lld entries per side",
                      (long long)(200 * 1024 / (g.mq * 24 + 32)));
            return GC_ERR_CONFIG;
        }
    }
    switch (g.mq) {
        case 9: return launch_blocks<9>(g, nb, desc, max_rows, max_cols, row_idx, col_idx, out, *qp, flags, st);
        case 4: return launch_blocks<4>(g, nb, desc, max_rows, max_cols, row_idx, col_idx, out, *qp, flags, st);
        case 16: return launch_blocks<16>(g, nb, desc, max_rows, max_cols, row_idx, col_idx, out, *qp, flags, st);
        default:
            if (g.mq > 16 && g.mq <= 64) {
                if (!g.wq_host) { set_error(GC_ERR_CONFIG, "gc_geom.wq_host is required"); return GC_ERR_CONFIG; }
                const int M = (int)g.mq;
                const size_t bytes = (size_t)(max_rows + max_cols) * (M * 3 * sizeof(double) + 4 * sizeof(int64_t));
                if (bytes <= 200 * 1024) {
                    RuleW rw;
                    e_copy_weights(g, rw, M);
                    const bool small = max_rows * ((max_cols + 1) / 2) <= 128;
                    if (g.kernel)
                        return small ? launch_big<8, 128, true>(g, rw, M, nb, desc, bytes, row_idx, col_idx, out, *qp, flags, st)
                                     : launch_big<8, 256, true>(g, rw, M, nb, desc, bytes, row_idx, col_idx, out, *qp, flags, st);
                    return small ? launch_big<8, 128, false>(g, rw, M, nb, desc, bytes, row_idx, col_idx, out, *qp, flags, st)
                                 : launch_big<8, 256, false>(g, rw, M, nb, desc, bytes, row_idx, col_idx, out, *qp, flags, st);
                }
            }
            k_assemble_blocks_any<<<(unsigned)nb, BLK_THREADS, 0, st>>>(g, desc, row_idx, col_idx, out, *qp, flags);
            GC_CHECK_LAUNCH("k_assemble_blocks_any");
            return GC_OK;
    }
}

int gc_singular_flush(const gc_geom* gp, const gc_rules* rp, gc_queue* qp, double* out,
                      int64_t* counts_out, void* stream) {
    if (!gp || !rp || !qp) { set_error(GC_ERR_CONFIG, "null argument"); return GC_ERR_CONFIG; }
    if (gp->gq) { set_error(GC_ERR_CONFIG, "curved charts: flush with gc_curved_singular"); return GC_ERR_CONFIG; }
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

// The same flush without a host synchronisation: the singular kernels run
// persistent warps that read their task counts from the queue's device
// counters (clamped to the capacity; an overflow was flagged on the device
// by the producer), the counters are copied to counts_dev (int32 x 4,
// device memory, may be NULL) and reset - all stream-ordered, so assembly
// returns while the quadrature runs.
int gc_singular_flush_async(const gc_geom* gp, const gc_rules* rp, gc_queue* qp, double* out,
                            int32_t* counts_dev, void* stream) {
    if (!gp || !rp || !qp) { set_error(GC_ERR_CONFIG, "null argument"); return GC_ERR_CONFIG; }
    if (gp->gq) { set_error(GC_ERR_CONFIG, "curved charts: flush with gc_curved_singular"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    for (int k = 1; k <= 3; ++k) {
        if (qp->cap[k] <= 0) continue;
        int rc = launch_singular(*gp, *rp, k, qp->tasks[k], qp->cap[k], out, st, qp->count + k);
        if (rc) return rc;
    }
    cudaError_t e = cudaSuccess;
    if (counts_dev) e = cudaMemcpyAsync(counts_dev, qp->count, 4 * sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(qp->count, 0, 4 * sizeof(int32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "gc_singular_flush_async");
    return GC_OK;
}

}  // extern "C"
