// Cluster-tree construction on the device (clustering.py:131-162, the
// level-wise form of clustering.build_cluster_tree): per tree depth,
//   * k_seg_box   - segmented min/max of the support boxes (exact, so the
//                   reduction order is free);
//   * k_seg_keys  - the split coordinate of every dof of every splitting
//                   node (-0.0 canonicalised to +0.0: numpy's comparison
//                   sort treats them as equal, a radix sort would not);
//   * two stable CUB radix sorts - by the key, then by the segment (LSD
//                   order: segments in place, keys ascending inside, ties in
//                   row order) - the reference's per-node argsort(kind=
//                   "stable"); one launch pair over all nodes of the depth
//                   (CUB's segmented sort falls back to one-block sorts for
//                   the large top-level segments); once every segment is
//                   short, one stable segmented sort (gc_tree_split_small);
//   * k_seg_permute - applies the order to the permutation and to the
//                   packed (lo | hi | point) rows.
//   * k_seg_axis  - the longest box axis of every splitting node.
// The tree's shape depends only on the dof count and the leaf size, so the
// host lays out every depth's frontier up front and the depths run back to
// back on the stream; boxes and the permutation come back once.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "common.cuh"

namespace gcb {

constexpr int TREE_THREADS = 256;

// box[6 s ..] = (min lo, max hi) over pack rows [start[s], stop[s])
__global__ void __launch_bounds__(TREE_THREADS) k_seg_box(int64_t nseg, const int64_t* __restrict__ start,
                                                          const int64_t* __restrict__ stop,
                                                          const double* __restrict__ pack, double* __restrict__ box) {
    __shared__ double red[6][TREE_THREADS];
    for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (int64_t r = start[sg] + threadIdx.x; r < stop[sg]; r += TREE_THREADS) {
            const double* p = pack + 9 * r;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                v[k] = fmin(v[k], p[k]);
                v[3 + k] = fmax(v[3 + k], p[3 + k]);
            }
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) red[k][threadIdx.x] = v[k];
        __syncthreads();
        for (int o = TREE_THREADS / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    red[k][threadIdx.x] = fmin(red[k][threadIdx.x], red[k][threadIdx.x + o]);
                    red[3 + k][threadIdx.x] = fmax(red[3 + k][threadIdx.x], red[3 + k][threadIdx.x + o]);
                }
            }
            __syncthreads();
        }
        if (threadIdx.x < 6) box[6 * sg + threadIdx.x] = red[threadIdx.x][0];
        __syncthreads();
    }
}

// segment s: rows [start, start + len) -> items [head, head + len)
__global__ void __launch_bounds__(TREE_THREADS) k_seg_keys(int64_t nseg, const int64_t* __restrict__ start,
                                                           const int64_t* __restrict__ len,
                                                           const int64_t* __restrict__ head,
                                                           const int64_t* __restrict__ axis,
                                                           const double* __restrict__ pack,
                                                           double* __restrict__ keys, int32_t* __restrict__ vals) {
    for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        const int64_t s = start[sg], h = head[sg], L = len[sg];
        const int ax = (int)axis[sg];
        for (int64_t i = threadIdx.x; i < L; i += TREE_THREADS) {
            keys[h + i] = pack[9 * (s + i) + 6 + ax] + 0.0;     // -0.0 -> +0.0
            vals[h + i] = (int32_t)(s + i);
        }
    }
}

// seg[j] = the segment whose rows [start[s], start[s] + len[s]) hold row[j]
// (segment starts ascending)
__global__ void k_seg_of(int64_t n, int64_t nseg, const int64_t* __restrict__ start, const int32_t* __restrict__ row,
                         int32_t* __restrict__ seg) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = row[j];
        int64_t lo = 0, hi = nseg;                  // first start > r
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (start[mid] <= r) lo = mid + 1; else hi = mid;
        }
        seg[j] = (int32_t)(lo - 1);
    }
}

// new[dst[i]] = old[src[i]] for the permutation and the packed rows
__global__ void k_seg_permute(int64_t n, const int32_t* __restrict__ dst, const int32_t* __restrict__ src,
                              const int64_t* __restrict__ perm_old, int64_t* __restrict__ perm_new,
                              const double* __restrict__ pack_old, double* __restrict__ pack_new) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = dst[i], s = src[i];
        perm_new[d] = perm_old[s];
#pragma unroll
        for (int k = 0; k < 9; ++k) pack_new[9 * d + k] = pack_old[9 * s + k];
    }
}

// longest box axis of the splitting nodes (np.argmax: first maximum wins)
__global__ void k_seg_axis(int64_t k, const int64_t* __restrict__ rows, const double* __restrict__ box,
                           int64_t* __restrict__ axis) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const double* b = box + 6 * rows[i];
        const double e0 = __dsub_rn(b[3], b[0]), e1 = __dsub_rn(b[4], b[1]), e2 = __dsub_rn(b[5], b[2]);
        int64_t ax = 0;
        double m = e0;
        if (e1 > m) { ax = 1; m = e1; }
        if (e2 > m) ax = 2;
        axis[i] = ax;
    }
}

}  // namespace gcb

using namespace gcb;

// split axes of k nodes whose boxes are the rows [dev] of box (6 per row)
extern "C" int gc_tree_axis(int64_t k, const int64_t* rows, const double* box, int64_t* axis, void* stream) {
    if (k <= 0) return GC_OK;
    const int64_t grid = (k + 255) / 256 < 148 * 8 ? (k + 255) / 256 : 148 * 8;
    k_seg_axis<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(k, rows, box, axis);
    GC_CHECK_LAUNCH("k_seg_axis");
    return GC_OK;
}

extern "C" int gc_tree_boxes(int64_t nseg, const int64_t* start, const int64_t* stop, const double* pack,
                             double* box, void* stream) {
    if (nseg <= 0) return GC_OK;
    const int64_t grid = nseg < 148 * 16 ? nseg : 148 * 16;
    k_seg_box<<<(unsigned)grid, TREE_THREADS, 0, (cudaStream_t)stream>>>(nseg, start, stop, pack, box);
    GC_CHECK_LAUNCH("k_seg_box");
    return GC_OK;
}

// CUB temp-storage bytes of a split step with nitems dofs in nseg segments
extern "C" int gc_tree_sort_bytes(int64_t nitems, int64_t nseg, int64_t* bytes) {
    size_t t1 = 0, t2 = 0, t3 = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, t1, (const double*)nullptr, (double*)nullptr,
                                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)nitems);
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(nullptr, t2, (const int32_t*)nullptr, (int32_t*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, (int)nitems);
    if (e == cudaSuccess)
        e = cub::DeviceSegmentedSort::StableSortPairs(nullptr, t3, (const double*)nullptr, (double*)nullptr,
                                                      (const int32_t*)nullptr, (int32_t*)nullptr, (int)nitems,
                                                      (int)(nseg > 0 ? nseg : 1), (const int32_t*)nullptr,
                                                      (const int32_t*)nullptr);
    if (e != cudaSuccess) return cuda_status(e, "gc_tree_sort_bytes");
    size_t t = t1 > t2 ? t1 : t2;
    *bytes = (int64_t)(t > t3 ? t : t3);
    return GC_OK;
}

// One split step: keys of the splitting segments, stable segmented sort,
// permutation of perm / pack from the *_old to the *_new buffers (which the
// caller initialised as copies of the old ones).  seg arrays [dev] per
// segment: start, len, head, axis; offsets [dev] (nseg+1) int32 item
// offsets.  Scratch (caller-owned, [dev]): keys 2*nitems doubles, vals
// 2*nitems int32, temp of gc_tree_sort_bytes bytes.
extern "C" int gc_tree_split(int64_t nseg, const int64_t* seg_start, const int64_t* seg_len,
                             const int64_t* seg_head, const int64_t* seg_axis, const int32_t* offsets,
                             int64_t nitems, const double* pack_old, double* pack_new,
                             const int64_t* perm_old, int64_t* perm_new, double* keys, int32_t* vals,
                             void* temp, int64_t temp_bytes, void* stream) {
    if (nseg <= 0 || nitems <= 0) return GC_OK;
    if (nitems > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "gc_tree_split: too many dofs"); return GC_ERR_CONFIG; }
    if (!keys || !vals || !temp) { set_error(GC_ERR_CONFIG, "gc_tree_split: scratch missing"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    double* keys_out = keys + nitems;
    int32_t* vals_out = vals + nitems;
    const int64_t grid = nseg < 148 * 16 ? nseg : 148 * 16;
    k_seg_keys<<<(unsigned)grid, TREE_THREADS, 0, st>>>(nseg, seg_start, seg_len, seg_head, seg_axis, pack_old,
                                                        keys, vals);
    GC_CHECK_LAUNCH("k_seg_keys");
    (void)offsets;
    // pass 1: all items by key (stable); pass 2: by segment (stable).  The
    // key buffers are dead after pass 1: they hold the segment ids
    // (keys[0..n)) and the final source rows (keys_out[0..n)).
    size_t tb = (size_t)temp_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys_out, vals, vals_out, (int)nitems, 0, 64, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_tree_split sort (key)");
    int32_t* segk = reinterpret_cast<int32_t*>(keys);
    int32_t* segk_out = segk + nitems;
    int32_t* src_final = reinterpret_cast<int32_t*>(keys_out);
    int64_t pgrid = (nitems + 255) / 256;
    if (pgrid > 148 * 32) pgrid = 148 * 32;
    k_seg_of<<<(unsigned)pgrid, 256, 0, st>>>(nitems, nseg, seg_start, vals_out, segk);
    GC_CHECK_LAUNCH("k_seg_of");
    int end_bit = 1;
    while (end_bit < 31 && (1LL << end_bit) < nseg) ++end_bit;
    tb = (size_t)temp_bytes;
    e = cub::DeviceRadixSort::SortPairs(temp, tb, segk, segk_out, vals_out, src_final, (int)nitems, 0, end_bit, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_tree_split sort (segment)");
    count_launch(2);
    k_seg_permute<<<(unsigned)pgrid, 256, 0, st>>>(nitems, vals, src_final, perm_old, perm_new, pack_old, pack_new);
    GC_CHECK_LAUNCH("k_seg_permute");
    return GC_OK;
}

// gc_tree_split for depths whose segments are all short: one stable
// segmented sort (CUB picks warp / block sorts per segment size) instead of
// the two full-width radix sorts; the same order (key ascending, ties in
// row order) and the same permutation.
extern "C" int gc_tree_split_small(int64_t nseg, const int64_t* seg_start, const int64_t* seg_len,
                                   const int64_t* seg_head, const int64_t* seg_axis, const int32_t* offsets,
                                   int64_t nitems, const double* pack_old, double* pack_new,
                                   const int64_t* perm_old, int64_t* perm_new, double* keys, int32_t* vals,
                                   void* temp, int64_t temp_bytes, void* stream) {
    if (nseg <= 0 || nitems <= 0) return GC_OK;
    if (nitems > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "gc_tree_split_small: too many dofs"); return GC_ERR_CONFIG; }
    if (!keys || !vals || !temp || !offsets) {
        set_error(GC_ERR_CONFIG, "gc_tree_split_small: scratch missing");
        return GC_ERR_CONFIG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t grid = nseg < 148 * 16 ? nseg : 148 * 16;
    k_seg_keys<<<(unsigned)grid, TREE_THREADS, 0, st>>>(nseg, seg_start, seg_len, seg_head, seg_axis, pack_old,
                                                        keys, vals);
    GC_CHECK_LAUNCH("k_seg_keys");
    size_t tb = (size_t)temp_bytes;
    cudaError_t e = cub::DeviceSegmentedSort::StableSortPairs(temp, tb, keys, keys + nitems, vals, vals + nitems,
                                                              (int)nitems, (int)nseg, offsets, offsets + 1, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_tree_split_small sort");
    count_launch(1);
    int64_t pgrid = (nitems + 255) / 256;
    if (pgrid > 148 * 32) pgrid = 148 * 32;
    k_seg_permute<<<(unsigned)pgrid, 256, 0, st>>>(nitems, vals, vals + nitems, perm_old, perm_new, pack_old,
                                                  pack_new);
    GC_CHECK_LAUNCH("k_seg_permute");
    return GC_OK;
}
