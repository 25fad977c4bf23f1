// Green quadrature factors of cluster-basis nodes (assembly.py:371-455,
// quadrature.py:95-126), one CTA per node, one thread per (row, box point).
//
// Pivot sets are chosen by argmax over these entries, so every operation
// follows the reference's rounding: no FMA contraction (__d*_rn
// intrinsics), sequential point sums starting from 0, 1/(4 pi r) formed as
// 1/(FOUR_PI*r), and r^3 rounded once (cube_rn).  The only known difference
// is numpy's SIMD r**3, which is within 1 ulp of cube_rn.
#include "common.cuh"

namespace gcb {

constexpr int GREEN_THREADS = 256;
constexpr int GREEN_MAX_K = 6 * 8 * 8;  // m <= 8

// Box-boundary rules of a batch of nodes (quadrature.green_box_rule):
// face (axis, low/high side) -> m x m tensor Gauss points, with the
// reference's operation order for points and weights.
__global__ void k_green_box_rules(int m, const double* __restrict__ g01,
                                  const double* __restrict__ w01, int64_t nn,
                                  const double* __restrict__ boxes, double* __restrict__ z,
                                  double* __restrict__ sq, double* __restrict__ nz) {
    const int K = 6 * m * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn * K;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t node = e / K;
        const int k = (int)(e % K);
        const double* bx = boxes + 8 * node;
        const int face = k / (m * m), ij = k % (m * m), i = ij / m, j = ij % m;
        const int axis = face >> 1, hi_side = face & 1;
        const int b = axis == 0 ? 1 : 0, c = axis == 2 ? 1 : 2;
        double lo[3], hi[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = __dsub_rn(bx[a], bx[6]);
            hi[a] = __dadd_rn(bx[3 + a], bx[6]);
        }
        const double span_b = __dsub_rn(hi[b], lo[b]), span_c = __dsub_rn(hi[c], lo[c]);
        double p[3], n[3] = {0.0, 0.0, 0.0};
        p[axis] = hi_side ? hi[axis] : lo[axis];
        p[b] = __dadd_rn(lo[b], __dmul_rn(span_b, g01[i]));
        p[c] = __dadd_rn(lo[c], __dmul_rn(span_c, g01[j]));
        n[axis] = hi_side ? 1.0 : -1.0;
        const double wz = __dmul_rn(__dmul_rn(__dmul_rn(w01[i], w01[j]), span_b), span_c);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            z[3 * e + a] = p[a];
            nz[3 * e + a] = n[a];
        }
        sq[e] = __dsqrt_rn(wz);
    }
}

// moments of one triangle at box point (z, n): sum_p wgt_p g / h, with
// wgt_p = gram * w_p (constant basis) or (b_p[a] * (gram * w_p)) (linear
// basis, the hat function of corner a), in the reference's order
template <bool LIN>
__device__ __forceinline__ void tri_moments(const gc_geom& g, int64_t t, int a, double z0, double z1, double z2,
                                            double n0, double n1, double n2, double& ig, double& ih, bool& touch) {
    const int mq = (int)g.mq;
    const double gram = g.gq ? 0.0 : g.gram[t];
    const double* xq = g.xq + t * 3 * mq;
    for (int p = 0; p < mq; ++p) {
        const double d0 = __dsub_rn(xq[3 * p], z0);
        const double d1 = __dsub_rn(xq[3 * p + 1], z1);
        const double d2 = __dsub_rn(xq[3 * p + 2], z2);
        const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
        const double rr = __dsqrt_rn(r2);
        touch |= (rr <= 1e-12);
        const double gk = __ddiv_rn(1.0, __dmul_rn(FOUR_PI, rr));
        const double dot = __dadd_rn(__dadd_rn(__dmul_rn(d0, n0), __dmul_rn(d1, n1)), __dmul_rn(d2, n2));
        const double hk = __ddiv_rn(dot, __dmul_rn(FOUR_PI, cube_rn(rr)));
        double gw = __dmul_rn(g.gq ? g.gq[t * mq + p] : gram, g.wq[p]);   // curved: |n| per point
        if (LIN) gw = __dmul_rn(g.bq[3 * p + a], gw);
        ig = __dadd_rn(ig, __dmul_rn(gw, gk));
        ih = __dadd_rn(ih, __dmul_rn(gw, hk));
    }
}

// One CTA per node; rule (K points) staged in shared memory; one thread per
// (row, box point) entry of the R x 2K factor.  LIN: rows are vertices and
// each row sums its star triangles' hat-weighted moments (assembly.py:406-
// 415: per corner a, then triangle order, each a full point sum added to
// the running total).
template <bool LIN, bool POINT>
__global__ void __launch_bounds__(GREEN_THREADS) k_green_factor(
    gc_geom g, int side, int K, const int64_t* __restrict__ desc,
    const double* __restrict__ dtau, const double* __restrict__ zr, const double* __restrict__ sqr,
    const double* __restrict__ nzr, const int64_t* __restrict__ rows, double* __restrict__ out,
    int32_t* flags) {
    __shared__ double z[GREEN_MAX_K][3];
    __shared__ double nn3[GREEN_MAX_K][3];
    __shared__ double sq[GREEN_MAX_K];
    const int node = blockIdx.x;
    const int64_t rows_off = desc[5 * node], R = desc[5 * node + 1];
    const int64_t out_off = desc[5 * node + 2], rule = desc[5 * node + 3];
    if (side < 0) side = (int)desc[5 * node + 4];      // per-node side
    const double d_tau = dtau[node];
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            z[k][a] = zr[(rule * K + k) * 3 + a];
            nn3[k][a] = nzr[(rule * K + k) * 3 + a];
        }
        sq[k] = sqr[rule * K + k];
    }
    __syncthreads();

    const int64_t W = 2 * (int64_t)K;
    bool touch = false;
    for (int64_t e = threadIdx.x; e < R * K; e += blockDim.x) {
        const int64_t r = e / K;
        const int k = (int)(e % K);
        const int64_t dof = rows[rows_off + r];
        const double z0 = z[k][0], z1 = z[k][1], z2 = z[k][2];
        const double n0 = nn3[k][0], n1 = nn3[k][1], n2 = nn3[k][2];
        double ig = 0.0, ih = 0.0;
        if (POINT) {
            // collocation rows: point evaluations at the vertex (assembly.py:427-433)
            const double d0 = __dsub_rn(g.verts[3 * dof], z0);
            const double d1 = __dsub_rn(g.verts[3 * dof + 1], z1);
            const double d2 = __dsub_rn(g.verts[3 * dof + 2], z2);
            const double rr = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
            touch |= (rr <= 1e-12);
            ig = __ddiv_rn(1.0, __dmul_rn(FOUR_PI, rr));
            const double dot = __dadd_rn(__dadd_rn(__dmul_rn(d0, n0), __dmul_rn(d1, n1)), __dmul_rn(d2, n2));
            ih = __ddiv_rn(dot, __dmul_rn(FOUR_PI, cube_rn(rr)));
        } else if (LIN) {
            for (int64_t u = g.vstar_ptr[dof]; u < g.vstar_ptr[dof + 1]; ++u) {
                double vg = 0.0, vh = 0.0;
                const int64_t ent = g.vstar_ent[u];
                tri_moments<true>(g, ent >> 2, (int)(ent & 3), z0, z1, z2, n0, n1, n2, vg, vh, touch);
                ig = __dadd_rn(ig, vg);
                ih = __dadd_rn(ih, vh);
            }
        } else {
            tri_moments<false>(g, dof, 0, z0, z1, z2, n0, n1, n2, ig, ih, touch);
        }
        double* row = out + out_off + r * W;
        if (side == 0) {
            row[k] = __dmul_rn(sq[k], ig);
            row[K + k] = __dmul_rn(__dmul_rn(-d_tau, sq[k]), ih);
        } else {
            row[k] = __dmul_rn(sq[k], ih);
            row[K + k] = __dmul_rn(__ddiv_rn(sq[k], d_tau), ig);
        }
    }
    if (touch) atomicOr(flags, FLAG_TOUCH);
}

}  // namespace gcb

using namespace gcb;

extern "C" int gc_green_box_rules(int m, const double* g01, const double* w01, int64_t nn,
                                  const double* box, double* z, double* sq, double* nz,
                                  void* stream) {
    if (m < 1 || m > 8) { set_error(GC_ERR_CONFIG, "green order m=%d outside [1, 8]", m); return GC_ERR_CONFIG; }
    if (nn <= 0) return GC_OK;
    int64_t total = nn * 6 * m * m;
    int64_t grid = (total + 255) / 256;
    if (grid > 148 * 32) grid = 148 * 32;
    k_green_box_rules<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(m, g01, w01, nn, box, z, sq, nz);
    GC_CHECK_LAUNCH("k_green_box_rules");
    return GC_OK;
}

extern "C" int gc_green_factor(const gc_geom* gp, int side, int64_t K, int64_t nn,
                               const int64_t* desc, const double* dtau, const double* z,
                               const double* sq, const double* nz, const int64_t* rows,
                               double* out, int32_t* flags, void* stream) {
    if (!gp) { set_error(GC_ERR_CONFIG, "null geometry"); return GC_ERR_CONFIG; }
    if (side < -1 || side > 1) { set_error(GC_ERR_CONFIG, "side must be 0 (row), 1 (col) or -1 (per node)"); return GC_ERR_CONFIG; }
    if (K < 1 || K > GREEN_MAX_K) { set_error(GC_ERR_CONFIG, "rule size K=%lld outside [1, %d]", (long long)K, GREEN_MAX_K); return GC_ERR_CONFIG; }
    if (nn <= 0) return GC_OK;
    if (gp->basis == 1) {
        if (!gp->vstar_ptr || !gp->vstar_ent || !gp->bq) {
            set_error(GC_ERR_CONFIG, "linear basis needs gc_geom.vstar_ptr/vstar_ent/bq");
            return GC_ERR_CONFIG;
        }
        k_green_factor<true, false><<<(unsigned)nn, GREEN_THREADS, 0, (cudaStream_t)stream>>>(
            *gp, side, (int)K, desc, dtau, z, sq, nz, rows, out, flags);
    } else if (gp->basis == 2) {
        if (!gp->verts) { set_error(GC_ERR_CONFIG, "collocation rows need gc_geom.verts"); return GC_ERR_CONFIG; }
        k_green_factor<false, true><<<(unsigned)nn, GREEN_THREADS, 0, (cudaStream_t)stream>>>(
            *gp, side, (int)K, desc, dtau, z, sq, nz, rows, out, flags);
    } else {
        k_green_factor<false, false><<<(unsigned)nn, GREEN_THREADS, 0, (cudaStream_t)stream>>>(
            *gp, side, (int)K, desc, dtau, z, sq, nz, rows, out, flags);
    }
    GC_CHECK_LAUNCH("k_green_factor");
    return GC_OK;
}
