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

constexpr int ACA_THREADS = 256;
constexpr int ACA_WARPS = ACA_THREADS / 32;

struct MaxLoc {
    double v;
    int64_t i;
    double ss;
};

__device__ __forceinline__ void merge(MaxLoc& a, double v, int64_t i, double ss) {
    if (v > a.v || (v == a.v && i < a.i)) { a.v = v; a.i = i; }
    a.ss += ss;
}

// block-wide (max |.|, first index, sum of squares) with a fixed tree
__device__ MaxLoc block_reduce(MaxLoc x, double* sv, int64_t* si, double* ss) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, x.v, o);
        const long long i = __shfl_xor_sync(0xffffffffu, (long long)x.i, o);
        const double s = __shfl_xor_sync(0xffffffffu, x.ss, o);
        if (v > x.v || (v == x.v && i < x.i)) { x.v = v; x.i = i; }
        x.ss = x.ss + s;  // commutative: both partners hold the same sum
    }
    if (lane == 0) { sv[warp] = x.v; si[warp] = x.i; ss[warp] = x.ss; }
    __syncthreads();
    MaxLoc r{-1.0, INT64_MAX, 0.0};
    for (int w = 0; w < ACA_WARPS; ++w) merge(r, sv[w], si[w], ss[w]);
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(ACA_THREADS) k_aca(const int64_t* __restrict__ desc, int64_t W,
                                                     double eps, int64_t max_rank, double* fac,
                                                     int64_t* __restrict__ piv_out,
                                                     int64_t* __restrict__ rank_out,
                                                     double* __restrict__ v_out,
                                                     double* __restrict__ u, int64_t max_rows,
                                                     int resid_in_smem) {
    extern __shared__ double smem[];
    const int node = blockIdx.x;
    const int64_t fac_off = desc[4 * node], R = desc[4 * node + 1];
    const int64_t piv_off = desc[4 * node + 2], v_off = desc[4 * node + 3];
    int64_t limit = max_rank > 0 ? max_rank : W;
    if (R < limit) limit = R;

    double* res = resid_in_smem ? smem : fac + fac_off;
    double* tail = resid_in_smem ? smem + max_rows * W : smem;
    double* prow = tail;                         // W
    double* ucol = prow + W;                     // max_rows
    int64_t* pivs = (int64_t*)(ucol + max_rows); // max_rows
    int64_t* pivpos = pivs + max_rows;           // max_rows: row -> k or -1
    double* sv = (double*)(pivpos + max_rows);
    int64_t* si = (int64_t*)(sv + ACA_WARPS);
    double* ss = (double*)(si + ACA_WARPS);
    __shared__ int64_t s_state[2];

    const int64_t N = R * W;
    MaxLoc loc{-1.0, INT64_MAX, 0.0};
    for (int64_t e = threadIdx.x; e < N; e += ACA_THREADS) {
        double x = fac[fac_off + e];
        if (resid_in_smem) res[e] = x;
        merge(loc, fabs(x), e, x * x);
    }
    for (int64_t a = threadIdx.x; a < R; a += ACA_THREADS) pivpos[a] = -1;
    MaxLoc st = block_reduce(loc, sv, si, ss);
    const double thr = eps * sqrt(st.ss);
    int64_t rank = 0;
    double* U = u + v_off;
    while (rank < limit && sqrt(st.ss) > thr) {
        const int64_t i = st.i / W, j = st.i % W;
        const double pv = res[st.i];
        if (pv == 0.0) break;
        for (int64_t b = threadIdx.x; b < W; b += ACA_THREADS) prow[b] = res[i * W + b];
        for (int64_t a = threadIdx.x; a < R; a += ACA_THREADS) {
            const double ua = __ddiv_rn(res[a * W + j], pv);
            ucol[a] = ua;
            U[a * limit + rank] = ua;
        }
        if (threadIdx.x == 0) { pivs[rank] = i; pivpos[i] = rank; }
        __syncthreads();
        loc = MaxLoc{-1.0, INT64_MAX, 0.0};
        for (int64_t e = threadIdx.x; e < N; e += ACA_THREADS) {
            const int64_t a = e / W, b = e - a * W;
            const double x = __dsub_rn(res[e], __dmul_rn(ucol[a], prow[b]));
            res[e] = x;
            merge(loc, fabs(x), e, x * x);
        }
        st = block_reduce(loc, sv, si, ss);
        ++rank;
    }
    if (threadIdx.x == 0) {
        rank_out[node] = rank;
        s_state[0] = rank;
    }
    for (int64_t k = threadIdx.x; k < rank; k += ACA_THREADS) piv_out[piv_off + k] = pivs[k];
    __syncthreads();
    const int64_t r = s_state[0];
    if (r == 0) return;
    // V row a: solve v M = U[a,:], M[k][l] = U[piv_k, l] unit lower triangular
    double* V = v_out + v_off;
    for (int64_t a = threadIdx.x; a < R; a += ACA_THREADS) {
        const int64_t pk = pivpos[a];
        if (pk >= 0) {
            for (int64_t l = 0; l < r; ++l) V[a * r + l] = (l == pk) ? 1.0 : 0.0;
            continue;
        }
        for (int64_t l = r - 1; l >= 0; --l) {
            double s = U[a * limit + l];
            for (int64_t k = l + 1; k < r; ++k) s = fma(-V[a * r + k], U[pivs[k] * limit + l], s);
            V[a * r + l] = s;
        }
    }
}

}  // namespace gcb

using namespace gcb;

extern "C" int gc_aca(int64_t nn, const int64_t* desc, int64_t W, double eps, int64_t max_rank,
                      double* fac, int64_t* piv, int64_t* rank, double* v, double* u,
                      int64_t max_rows, void* stream) {
    if (nn <= 0) return GC_OK;
    if (W <= 0 || max_rows < 0) { set_error(GC_ERR_CONFIG, "gc_aca: bad shape"); return GC_ERR_CONFIG; }
    if (!(eps >= 0.0)) { set_error(GC_ERR_CONFIG, "gc_aca: eps must be >= 0"); return GC_ERR_CONFIG; }
    const size_t tail = (size_t)W * 8 + (size_t)max_rows * 8 * 3 + ACA_WARPS * 24;
    const size_t resid = (size_t)max_rows * W * 8;
    int in_smem = (resid + tail) <= 200 * 1024;
    size_t bytes = (in_smem ? resid : 0) + tail;
    if (bytes > 227 * 1024) { set_error(GC_ERR_CONFIG, "gc_aca: %lld rows too many", (long long)max_rows); return GC_ERR_CONFIG; }
    cudaError_t e = cudaFuncSetAttribute(k_aca, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return cuda_status(e, "gc_aca smem attribute");
    k_aca<<<(unsigned)nn, ACA_THREADS, bytes, (cudaStream_t)stream>>>(desc, W, eps, max_rank, fac, piv,
                                                                      rank, v, u, max_rows, in_smem);
    GC_CHECK_LAUNCH("k_aca");
    return GC_OK;
}
