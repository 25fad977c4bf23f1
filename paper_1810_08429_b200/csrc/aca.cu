// Batched full-pivot cross approximation (gca.aca_interpolation,
// gca.py:41-79): one CTA per cluster-basis node.
//
// The residual lives in shared memory when it fits (R x W <= ~200 KB, i.e.
// every node at m = 3) and in place in the factor buffer otherwise.  Each
// step is one pass over the residual that applies the rank-one update
// R -= u (x) R[i,:] with the reference's rounding (product, then
// difference; no FMA) and, in the same pass, tracks the next pivot (largest
// |R|, first in row-major order) and the squared Frobenius norm; one fixed-
// order block reduction per step.  Pivots follow from argmax and exact
// elementwise updates, so they match the reference bit for bit unless the
// stopping test sits within rounding of eps*||A|| (the reference's norm is
// a BLAS dot; ours is a fixed tree).
//
// V = U (U|piv)^-1: U|piv is unit lower triangular in pivot order, so each
// row of V is one back substitution against the r x r pivot block (read
// from the cached U scratch), then V[piv] = I exactly.
#include "common.cuh"

namespace gcb {

struct MaxLoc {
    double v;
    int i;
    double ss;
};

__device__ __forceinline__ void merge(MaxLoc& a, double v, int i, double ss) {
    if (v > a.v || (v == a.v && i < a.i)) { a.v = v; a.i = i; }
    a.ss += ss;
}

// merge for a thread's own elements, visited in increasing flat index:
// the first maximum stays without an index comparison
__device__ __forceinline__ void merge_next(MaxLoc& a, double v, int i, double ss) {
    if (v > a.v) { a.v = v; a.i = i; }
    a.ss += ss;
}

// block-wide (max |.|, first flat index, sum of squares) with a fixed tree
template <int NT>
__device__ MaxLoc block_reduce(MaxLoc x, double* sv, int* si, double* ss) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, x.v, o);
        const int i = __shfl_xor_sync(0xffffffffu, x.i, o);
        const double s = __shfl_xor_sync(0xffffffffu, x.ss, o);
        if (v > x.v || (v == x.v && i < x.i)) { x.v = v; x.i = i; }
        x.ss = x.ss + s;  // commutative: both partners hold the same sum
    }
    if (lane == 0) { sv[warp] = x.v; si[warp] = x.i; ss[warp] = x.ss; }
    __syncthreads();
    MaxLoc r{-1.0, INT_MAX, 0.0};
    for (int w = 0; w < NT / 32; ++w) merge(r, sv[w], si[w], ss[w]);
    __syncthreads();
    return r;
}

// One CTA per node.  Flat residual index e = a*W + b is walked with int32
// increments (no per-element division); NT = 1024 for batches of few large
// nodes (the top tree levels), 256 otherwise.
template <int NT>
__global__ void __launch_bounds__(NT) k_aca(const int64_t* __restrict__ desc, int W, double eps,
                                            int max_rank, double* fac, int64_t* __restrict__ piv_out,
                                            int64_t* __restrict__ rank_out, double* __restrict__ v_out,
                                            double* __restrict__ u, int max_rows, int resid_in_smem) {
    extern __shared__ double smem[];
    const int node = blockIdx.x;
    const int64_t fac_off = desc[4 * node], piv_off = desc[4 * node + 2], v_off = desc[4 * node + 3];
    const int R = (int)desc[4 * node + 1];
    int limit = max_rank > 0 ? max_rank : W;
    if (R < limit) limit = R;

    double* res = resid_in_smem ? smem : fac + fac_off;
    double* tail = resid_in_smem ? smem + (size_t)max_rows * W : smem;
    double* prow = tail;                        // W
    double* ucol = prow + W;                    // max_rows
    int* pivs = (int*)(ucol + max_rows);        // max_rows
    int* pivpos = pivs + max_rows;              // max_rows: row -> k or -1
    double* sv = (double*)(pivpos + max_rows);  // 2*max_rows ints: 8-byte aligned
    int* si = (int*)(sv + NT / 32);
    double* ss = (double*)(si + NT / 32 + ((NT / 32) & 1));
    __shared__ int s_rank;

    const int N = R * W;
    const int da = NT / W, db = NT % W;
    const int a0 = threadIdx.x / W, b0 = threadIdx.x % W;
    MaxLoc loc{-1.0, INT_MAX, 0.0};
    for (int e = threadIdx.x; e < N; e += NT) {
        const double x = fac[fac_off + e];
        if (resid_in_smem) res[e] = x;
        merge_next(loc, fabs(x), e, x * x);
    }
    for (int a = threadIdx.x; a < R; a += NT) pivpos[a] = -1;
    MaxLoc st = block_reduce<NT>(loc, sv, si, ss);
    const double thr = eps * sqrt(st.ss);
    int rank = 0;
    double* U = u + v_off;
    while (rank < limit && sqrt(st.ss) > thr) {
        const int i = st.i / W, j = st.i - (st.i / W) * W;
        const double pv = res[st.i];
        if (pv == 0.0) break;
        for (int b = threadIdx.x; b < W; b += NT) prow[b] = res[i * W + b];
        for (int a = threadIdx.x; a < R; a += NT) {
            const double ua = __ddiv_rn(res[a * W + j], pv);
            ucol[a] = ua;
            U[(int64_t)a * limit + rank] = ua;
        }
        if (threadIdx.x == 0) { pivs[rank] = i; pivpos[i] = rank; }
        __syncthreads();
        loc = MaxLoc{-1.0, INT_MAX, 0.0};
        int a = a0, b = b0;
        for (int e = threadIdx.x; e < N; e += NT) {
            const double x = __dsub_rn(res[e], __dmul_rn(ucol[a], prow[b]));
            res[e] = x;
            merge_next(loc, fabs(x), e, x * x);
            a += da;
            b += db;
            if (b >= W) { b -= W; ++a; }
        }
        st = block_reduce<NT>(loc, sv, si, ss);
        ++rank;
    }
    if (threadIdx.x == 0) {
        rank_out[node] = rank;
        s_rank = rank;
    }
    for (int k = threadIdx.x; k < rank; k += NT) piv_out[piv_off + k] = pivs[k];
    __syncthreads();
    const int r = s_rank;
    if (r == 0) return;
    // V = U (U|piv)^-1: stage the r x r pivot block M[k][l] = U[piv_k, l] in
    // shared memory (the residual is dead now), then one back substitution
    // per row: v[l] = U[a,l] - sum_{k>l} v[k] M[k][l]; V[piv] = I exactly
    double* M = smem;
    const bool m_in_smem = resid_in_smem && (int64_t)r * r <= (int64_t)max_rows * W;
    if (m_in_smem) {
        for (int e = threadIdx.x; e < r * r; e += NT) {
            const int k = e / r, l = e - (e / r) * r;
            M[e] = U[(int64_t)pivs[k] * limit + l];
        }
        __syncthreads();
    }
    double* V = v_out + v_off;
    for (int a = threadIdx.x; a < R; a += NT) {
        const int pk = pivpos[a];
        if (pk >= 0) {
            for (int l = 0; l < r; ++l) V[(int64_t)a * r + l] = (l == pk) ? 1.0 : 0.0;
            continue;
        }
        for (int l = r - 1; l >= 0; --l) {
            double sacc = U[(int64_t)a * limit + l];
            for (int k = l + 1; k < r; ++k) {
                const double mk = m_in_smem ? M[k * r + l] : U[(int64_t)pivs[k] * limit + l];
                sacc = fma(-V[(int64_t)a * r + k], mk, sacc);
            }
            V[(int64_t)a * r + l] = sacc;
        }
    }
}

}  // namespace gcb

using namespace gcb;

template <int NT>
static int launch_aca(int64_t nn, const int64_t* desc, int64_t W, double eps, int64_t max_rank,
                      double* fac, int64_t* piv, int64_t* rank, double* v, double* u,
                      int64_t max_rows, cudaStream_t st) {
    const size_t tail = (size_t)W * 8 + (size_t)(max_rows + 1) * 8 * 2 + (NT / 32) * 24 + 16;
    const size_t resid = (size_t)max_rows * W * 8;
    const int in_smem = (resid + tail) <= 200 * 1024;
    const size_t bytes = (in_smem ? resid : 0) + tail;
    if (bytes > 227 * 1024) { set_error(GC_ERR_CONFIG, "gc_aca: %lld rows too many", (long long)max_rows); return GC_ERR_CONFIG; }
    cudaError_t e = cudaFuncSetAttribute(k_aca<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return cuda_status(e, "gc_aca smem attribute");
    k_aca<NT><<<(unsigned)nn, NT, bytes, st>>>(desc, (int)W, eps, (int)max_rank, fac, piv, rank, v, u,
                                               (int)max_rows, in_smem);
    GC_CHECK_LAUNCH("k_aca");
    return GC_OK;
}

extern "C" int gc_aca(int64_t nn, const int64_t* desc, int64_t W, double eps, int64_t max_rank,
                      double* fac, int64_t* piv, int64_t* rank, double* v, double* u,
                      int64_t max_rows, void* stream) {
    if (nn <= 0) return GC_OK;
    if (W <= 0 || max_rows < 0) { set_error(GC_ERR_CONFIG, "gc_aca: bad shape"); return GC_ERR_CONFIG; }
    if (!(eps >= 0.0)) { set_error(GC_ERR_CONFIG, "gc_aca: eps must be >= 0"); return GC_ERR_CONFIG; }
    if (max_rows * W >= (1LL << 31)) { set_error(GC_ERR_CONFIG, "gc_aca: factor too large"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    // few large nodes (top tree levels): 1024 threads per node
    if (nn < 148 && max_rows * W >= 4096)
        return launch_aca<1024>(nn, desc, W, eps, max_rank, fac, piv, rank, v, u, max_rows, st);
    return launch_aca<256>(nn, desc, W, eps, max_rank, fac, piv, rank, v, u, max_rows, st);
}
