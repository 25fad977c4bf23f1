// Tiered transforms of the matvec (plan time).  The forward transform of a
// nested basis is a chain of one dependent launch per tree height; under the
// bandwidth-bound coupling phase each of those levels costs a loaded memory
// round trip and a wait for SM slots.  A tier of consecutive heights
// (b_prev, b] is instead applied in ONE launch from the x-hat of its
// frontier (the live nodes at heights <= b_prev whose parent lies in the
// tier; the degrees of freedom themselves for the lowest tier), with the
// explicit composed transfers
//     M_u = stack over live children c of (M_c E_c | E_c if c is frontier),
//     M_leaf = V_leaf,
// where E_c = rows [child_row(c), +rank(c)) of the parent's V-hat
// (gca.py:162-220 nested-basis recursion, multiplied out).  The backward
// transform reads the same numbers transposed and regrouped per frontier
// node.  Both kernels run once per plan; the product kernels are the panel
// kernels of h2mv.cu.
#include "common.cuh"

namespace gcb {

constexpr int TIER_THREADS = 256;

// desc (6 x int64): s_off (-1: identity), m, kc, e_off, ku, out_off
//   out[m x ku] = S[m x kc] @ E[kc x ku]   (S = M + s_off, E = V + e_off)
//   or, s_off < 0, out = E[m x ku] (copy)
// all row-major; each output entry sums over kc in order (deterministic).
// Work is cut into tiles of TIER_TILE outputs: tile (2 x int64) = desc
// index, first output; one CTA per tile (the top nodes' blocks are large).
constexpr int TIER_TILE = 1024;

__global__ void __launch_bounds__(TIER_THREADS) k_tier_compose(int64_t ntiles, const int64_t* __restrict__ tiles,
                                                               const int64_t* __restrict__ desc,
                                                               const double* __restrict__ V, double* M) {
    for (int64_t b = blockIdx.x; b < ntiles; b += gridDim.x) {
        const int64_t* d = desc + 6 * tiles[2 * b];
        const int64_t e0 = tiles[2 * b + 1];
        const int64_t s_off = d[0], m = d[1], kc = d[2], e_off = d[3], ku = d[4], o_off = d[5];
        const double* __restrict__ E = V + e_off;
        double* out = M + o_off;
        const int64_t total = m * ku;
        const int64_t e1 = e0 + TIER_TILE < total ? e0 + TIER_TILE : total;
        if (s_off < 0) {
            for (int64_t e = e0 + threadIdx.x; e < e1; e += TIER_THREADS) out[e] = E[e];
            continue;
        }
        const double* S = M + s_off;
        for (int64_t e = e0 + threadIdx.x; e < e1; e += TIER_THREADS) {
            const int64_t i = e / ku, j = e - i * ku;
            const double* Si = S + i * kc;
            double acc = 0.0;
            for (int64_t t = 0; t < kc; ++t) acc = fma(Si[t], __ldg(E + t * ku + j), acc);
            out[e] = acc;
        }
    }
}

// desc (5 x int64): src_off, ld, rows, cols, dst_off
//   dst[dst_off + c * rows + r] = src[src_off + r * ld + c]
__global__ void __launch_bounds__(TIER_THREADS) k_block_transpose(int64_t n, const int64_t* __restrict__ desc,
                                                                  const double* __restrict__ src,
                                                                  double* __restrict__ dst) {
    for (int64_t b = blockIdx.x; b < n; b += gridDim.x) {
        const int64_t* d = desc + 5 * b;
        const int64_t s_off = d[0], ld = d[1], rows = d[2], cols = d[3], o_off = d[4];
        for (int64_t e = threadIdx.x; e < rows * cols; e += TIER_THREADS) {
            const int64_t c = e / rows, r = e - c * rows;
            dst[o_off + e] = __ldg(src + s_off + r * ld + c);
        }
    }
}

}  // namespace gcb

using namespace gcb;

// One height of a tier's composition: n descriptors (6 x int64, [dev]) cut
// into ntiles tiles (2 x int64, [dev]: descriptor, first output; see
// gc_tier_tile); M may be read (children's blocks, written by an earlier
// call) and written (this height's blocks) - the regions are disjoint.
extern "C" int gc_tier_compose(int64_t ntiles, const int64_t* tiles, const int64_t* desc, const double* V,
                               double* M, void* stream) {
    if (ntiles <= 0) return GC_OK;
    if (!tiles || !desc || !V || !M) { set_error(GC_ERR_CONFIG, "gc_tier_compose: null argument"); return GC_ERR_CONFIG; }
    const int64_t grid = ntiles < 148 * 16 ? ntiles : 148 * 16;
    k_tier_compose<<<(unsigned)grid, TIER_THREADS, 0, (cudaStream_t)stream>>>(ntiles, tiles, desc, V, M);
    GC_CHECK_LAUNCH("k_tier_compose");
    return GC_OK;
}

extern "C" int64_t gc_tier_tile(void) { return TIER_TILE; }

extern "C" int gc_block_transpose(int64_t n, const int64_t* desc, const double* src, double* dst, void* stream) {
    if (n <= 0) return GC_OK;
    if (!desc || !src || !dst) { set_error(GC_ERR_CONFIG, "gc_block_transpose: null argument"); return GC_ERR_CONFIG; }
    const int64_t grid = n < 148 * 8 ? n : 148 * 8;
    k_block_transpose<<<(unsigned)grid, TIER_THREADS, 0, (cudaStream_t)stream>>>(n, desc, src, dst);
    GC_CHECK_LAUNCH("k_block_transpose");
    return GC_OK;
}
