// Quadratic (curved) charts (geometry.py:69-114,
// 266-293; assembly.py:175-214): the chart of a triangle interpolates its 6
// nodes (vertices + curved edge midpoints) with the quadratic Lagrange
// basis, and the Gramian at a point is the norm of the interpolated node
// normals.  Distances are no longer affine in the Sauter-Schwab radial
// coordinate, so singular pairs use the reference's full rules with the
// charts evaluated point by point.
//
// k_curved_singular: one warp per queued singular pair, lanes over the rule
// points (SoA x1, x2, y1, y2, w), fixed butterfly sums.  W = 1 (constant
// basis: out[idx]) or 9 (linear basis: U[9 idx + 3a + c], canonical
// permuted order).
#include "common.cuh"

namespace gcb {

__device__ __constant__ static const int8_t kOrder6[6][6] = {
    {0, 1, 2, 3, 4, 5}, {1, 2, 0, 4, 5, 3}, {2, 0, 1, 5, 3, 4},
    {0, 2, 1, 5, 4, 3}, {2, 1, 0, 4, 3, 5}, {1, 0, 2, 3, 5, 4}};

__device__ __forceinline__ void shape6(double x, double y, double* n) {
    const double l0 = 1.0 - x - y;
    n[0] = l0 * (2.0 * l0 - 1.0);
    n[1] = x * (2.0 * x - 1.0);
    n[2] = y * (2.0 * y - 1.0);
    n[3] = 4.0 * l0 * x;
    n[4] = 4.0 * x * y;
    n[5] = 4.0 * y * l0;
}

// v = sum_a n[a] * P[perm[a]] (sequential, as assembly._interp6)
__device__ __forceinline__ void interp6(const double* n, const double* P, const int8_t* perm, double* v) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < 6; ++a) acc = fma(n[a], P[3 * perm[a] + c], acc);
        v[c] = acc;
    }
}

template <bool DLP, int W>
__global__ void __launch_bounds__(128) k_curved_singular(gc_geom g, const double* __restrict__ rule, int P,
                                                         const int64_t* __restrict__ tasks, int64_t n,
                                                         double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t task = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); task < n; task += nw) {
        const int64_t* tk = tasks + 4 * task;
        const int64_t t = tk[0], s = tk[1], pk = tk[2], idx = tk[3];
        const int8_t* ox = kOrder6[pk & 0xff];
        const int8_t* oy = kOrder6[(pk >> 8) & 0xff];
        const double* Pt = g.nodes6 + 18 * t;
        const double* Ps = g.nodes6 + 18 * s;
        const double* Nt = g.nrm6 + 18 * t;
        const double* Ns = g.nrm6 + 18 * s;
        double acc[W];
#pragma unroll
        for (int k = 0; k < W; ++k) acc[k] = 0.0;
        for (int p = lane; p < P; p += 32) {
            const double x1 = __ldg(rule + p), x2 = __ldg(rule + P + p);
            const double y1 = __ldg(rule + 2 * P + p), y2 = __ldg(rule + 3 * P + p);
            const double w = __ldg(rule + 4 * P + p);
            double nx[6], ny[6], X[3], Y[3], GX[3], GY[3];
            shape6(x1, x2, nx);
            shape6(y1, y2, ny);
            interp6(nx, Pt, ox, X);
            interp6(ny, Ps, oy, Y);
            interp6(nx, Nt, ox, GX);
            interp6(ny, Ns, oy, GY);
            const double d0 = X[0] - Y[0], d1 = X[1] - Y[1], d2 = X[2] - Y[2];
            const double r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
            const double ri = rsqrt_fast(r2);
            const double gx = sqrt(fma(GX[2], GX[2], fma(GX[1], GX[1], GX[0] * GX[0])));
            double kg;
            if (DLP) {
                const double dot = fma(d2, GY[2], fma(d1, GY[1], d0 * GY[0]));
                kg = dot * (ri * ri * ri) * gx;
            } else {
                const double gy = sqrt(fma(GY[2], GY[2], fma(GY[1], GY[1], GY[0] * GY[0])));
                kg = gx * gy * ri;
            }
            const double wk = w * kg;
            if (W == 1) {
                acc[0] += wk;
            } else {
                const double bx[3] = {1.0 - x1 - x2, x1, x2};
                const double by[3] = {1.0 - y1 - y2, y1, y2};
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[(3 * a + c) % W] = fma(wk * bx[a], by[c], acc[(3 * a + c) % W]);
            }
        }
#pragma unroll
        for (int k = 0; k < W; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < W; ++k) out[(int64_t)W * idx + k] = INV_FOUR_PI * acc[k];
        }
    }
}

}  // namespace gcb

using namespace gcb;

// singular pairs of curved charts; rules r->table[c] = full Sauter-Schwab
// SoA (x1, x2, y1, y2, w); width 1 (constant basis, out indexed by the
// task's output index) or 9 (linear basis).  Reads the queue counters
// (one stream synchronisation), launches, re-arms the queue.
extern "C" int gc_curved_singular(const gc_geom* gp, const gc_rules* rp, gc_queue* qp, int64_t width,
                                  double* out, int64_t* counts_out, void* stream) {
    if (!gp || !rp || !qp) { set_error(GC_ERR_CONFIG, "gc_curved_singular: null argument"); return GC_ERR_CONFIG; }
    if (!gp->nodes6 || !gp->nrm6) { set_error(GC_ERR_CONFIG, "curved charts need gc_geom.nodes6/nrm6"); return GC_ERR_CONFIG; }
    if (width != 1 && width != 9) { set_error(GC_ERR_CONFIG, "gc_curved_singular: width 1 or 9"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    int32_t counts[4] = {0, 0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(counts, qp->count, sizeof(counts), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_status(e, "gc_curved_singular counts");
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
        const int P = (int)rp->npts[k];
        if (width == 1) {
            if (g.kernel) k_curved_singular<true, 1><<<(unsigned)grid, 128, 0, st>>>(g, rp->table[k], P, qp->tasks[k], counts[k], out);
            else k_curved_singular<false, 1><<<(unsigned)grid, 128, 0, st>>>(g, rp->table[k], P, qp->tasks[k], counts[k], out);
        } else {
            if (g.kernel) k_curved_singular<true, 9><<<(unsigned)grid, 128, 0, st>>>(g, rp->table[k], P, qp->tasks[k], counts[k], out);
            else k_curved_singular<false, 9><<<(unsigned)grid, 128, 0, st>>>(g, rp->table[k], P, qp->tasks[k], counts[k], out);
        }
        GC_CHECK_LAUNCH("k_curved_singular");
    }
    e = cudaMemsetAsync(qp->count, 0, 4 * sizeof(int32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "gc_curved_singular reset");
    return GC_OK;
}

// The same integration for an explicit task list (t, s, px | py << 8, idx)
// and rule (SoA x1, x2, y1, y2, w of P points): the evaluator seam on
// curved charts, where the disjoint case runs the regular q^2 x q^2 tensor
// rule through this kernel too.
extern "C" int gc_curved_pairs(const gc_geom* gp, const double* rule, int64_t P, const int64_t* tasks,
                               int64_t n, int64_t width, double* out, void* stream) {
    if (!gp || !rule || !tasks) { set_error(GC_ERR_CONFIG, "gc_curved_pairs: null argument"); return GC_ERR_CONFIG; }
    if (!gp->nodes6 || !gp->nrm6) { set_error(GC_ERR_CONFIG, "curved charts need gc_geom.nodes6/nrm6"); return GC_ERR_CONFIG; }
    if (width != 1 && width != 9) { set_error(GC_ERR_CONFIG, "gc_curved_pairs: width 1 or 9"); return GC_ERR_CONFIG; }
    if (n <= 0) return GC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t grid = (n + 3) / 4;
    if (grid > 148 * 16) grid = 148 * 16;
    const gc_geom g = *gp;
    if (width == 1) {
        if (g.kernel) k_curved_singular<true, 1><<<(unsigned)grid, 128, 0, st>>>(g, rule, (int)P, tasks, n, out);
        else k_curved_singular<false, 1><<<(unsigned)grid, 128, 0, st>>>(g, rule, (int)P, tasks, n, out);
    } else {
        if (g.kernel) k_curved_singular<true, 9><<<(unsigned)grid, 128, 0, st>>>(g, rule, (int)P, tasks, n, out);
        else k_curved_singular<false, 9><<<(unsigned)grid, 128, 0, st>>>(g, rule, (int)P, tasks, n, out);
    }
    GC_CHECK_LAUNCH("k_curved_singular");
    return GC_OK;
}
