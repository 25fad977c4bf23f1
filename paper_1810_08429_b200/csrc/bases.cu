// Per-level bookkeeping of the nested cluster bases (gca.py:162-220, the
// level-synchronous form of gca.build_cluster_bases) on the device: the
// factor row lists of the nodes of one tree height (leaf dofs, or the
// children's pivots left then right), the factor / ACA descriptors, and
// after the ACA the local -> global pivot map, ranks and V offsets.  The
// host keeps only the launches and one small read per level (the level's
// row totals, which size the factor, ACA and V buffers).
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace gcb {

// R[pos0 + i] of node nodes[i] of one basis side: its leaf size, or the sum
// of its children's ranks; rows_node[node] = R (the store's per-node rows)
__global__ void k_bases_R(int64_t n, const int64_t* __restrict__ nodes, const int64_t* __restrict__ left,
                          const int64_t* __restrict__ right, const int64_t* __restrict__ start,
                          const int64_t* __restrict__ stop, const int64_t* __restrict__ rank, int64_t pos0,
                          int64_t W, int64_t* __restrict__ R, int64_t* __restrict__ lim, int64_t* __restrict__ vcap,
                          int64_t* __restrict__ rows_node) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = nodes[i];
        const int64_t l = left[u];
        const int64_t r = l < 0 ? stop[u] - start[u] : rank[l] + rank[right[u]];
        const int64_t lm = r < W ? r : W;
        R[pos0 + i] = r;
        lim[pos0 + i] = lm;
        vcap[pos0 + i] = r * lm;
        rows_node[u] = r;
    }
}

// rows of node i: leaf -> perm[start ..], else gpiv[piv_off[left] ..] then
// gpiv[piv_off[right] ..]; descriptors of gc_green_factor (rows_off, R,
// fac_off, box index, side) and gc_aca (fac_off, R, piv_off_l, v_off)
__global__ void k_bases_rows(int64_t n, const int64_t* __restrict__ nodes, const int64_t* __restrict__ left,
                             const int64_t* __restrict__ right, const int64_t* __restrict__ start,
                             const int64_t* __restrict__ rank, const int64_t* __restrict__ piv_off,
                             const int64_t* __restrict__ gpiv, const int64_t* __restrict__ perm, int64_t pos0,
                             int64_t box0, int64_t side, int64_t W, const int64_t* __restrict__ R,
                             const int64_t* __restrict__ rows_off, const int64_t* __restrict__ piv_off_l,
                             const int64_t* __restrict__ v_off, int64_t* __restrict__ rows,
                             int64_t* __restrict__ fdesc, int64_t* __restrict__ adesc) {
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const int64_t u = nodes[i], p = pos0 + i;
        const int64_t l = left[u], ro = rows_off[p], r = R[p];
        if (l < 0) {
            for (int64_t j = threadIdx.x; j < r; j += blockDim.x) rows[ro + j] = perm[start[u] + j];
        } else {
            const int64_t rl = rank[l], pl = piv_off[l], pr = piv_off[right[u]];
            for (int64_t j = threadIdx.x; j < r; j += blockDim.x)
                rows[ro + j] = j < rl ? gpiv[pl + j] : gpiv[pr + j - rl];
        }
        if (threadIdx.x == 0) {
            int64_t* f = fdesc + 5 * p;
            f[0] = ro; f[1] = r; f[2] = ro * W; f[3] = box0 + p; f[4] = side;
            int64_t* a = adesc + 4 * p;
            a[0] = ro * W; a[1] = r; a[2] = piv_off_l[p]; a[3] = v_off[p];
        }
    }
}

// out: R_max, rows total, limit total, vcap total, then v_off at every side
// boundary (n_bound positions)
__global__ void k_bases_totals(int64_t nn, const int64_t* __restrict__ R, const int64_t* __restrict__ lim,
                               const int64_t* __restrict__ vcap, const int64_t* __restrict__ rows_off,
                               const int64_t* __restrict__ piv_off_l, const int64_t* __restrict__ v_off,
                               const int64_t* __restrict__ bounds, int64_t n_bound, int64_t* __restrict__ out) {
    __shared__ int64_t red[256];
    int64_t m = 0;
    for (int64_t i = threadIdx.x; i < nn; i += blockDim.x) m = R[i] > m ? R[i] : m;
    red[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o && red[threadIdx.x + o] > red[threadIdx.x]) red[threadIdx.x] = red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = red[0];
        out[1] = rows_off[nn - 1] + R[nn - 1];
        out[2] = piv_off_l[nn - 1] + lim[nn - 1];
        out[3] = v_off[nn - 1] + vcap[nn - 1];
    }
    for (int64_t b = threadIdx.x; b < n_bound; b += blockDim.x) {
        const int64_t q = bounds[b];
        out[4 + b] = q < nn ? v_off[q] : v_off[nn - 1] + vcap[nn - 1];
    }
}

// after the ACA: rank[node], piv_off[node] = cursor + exclusive sum of the
// side's ranks, the global pivots gpiv[...] = rows[rows_off + local pivot],
// v_off_node[node] = v_base + v_off[p] - v_off[pos0]; the cursor advances
__global__ void k_bases_post(int64_t n, const int64_t* __restrict__ nodes, int64_t pos0,
                             const int64_t* __restrict__ rank_l, const int64_t* __restrict__ rk_off,
                             const int64_t* __restrict__ piv_l, const int64_t* __restrict__ piv_off_l,
                             const int64_t* __restrict__ rows, const int64_t* __restrict__ rows_off,
                             const int64_t* __restrict__ v_off, int64_t v_base, int64_t* __restrict__ cursor,
                             int64_t* __restrict__ rank, int64_t* __restrict__ piv_off, int64_t* __restrict__ gpiv,
                             int64_t* __restrict__ v_off_node) {
    const int64_t c0 = *cursor;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const int64_t u = nodes[i], p = pos0 + i;
        const int64_t rk = rank_l[p], base = c0 + rk_off[i];
        for (int64_t k = threadIdx.x; k < rk; k += blockDim.x)
            gpiv[base + k] = rows[rows_off[p] + piv_l[piv_off_l[p] + k]];
        if (threadIdx.x == 0) {
            rank[u] = rk;
            piv_off[u] = base;
            v_off_node[u] = v_base + v_off[p] - v_off[pos0];
        }
    }
}

__global__ void k_bases_cursor(int64_t n, const int64_t* __restrict__ rank_l, int64_t pos0,
                               const int64_t* __restrict__ rk_off, int64_t* __restrict__ cursor) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && n > 0) *cursor += rk_off[n - 1] + rank_l[pos0 + n - 1];
}

}  // namespace gcb

using namespace gcb;

extern "C" {

// scratch bytes of the scans of a level of nn nodes
int gc_bases_scan_bytes(int64_t nn, int64_t* bytes) {
    size_t tb = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int64_t*)nullptr, (int64_t*)nullptr, (int)nn);
    if (e != cudaSuccess) return cuda_status(e, "gc_bases_scan_bytes");
    *bytes = (int64_t)tb;
    return GC_OK;
}

// R / limit / vcap of the nodes of one side (positions pos0 .. pos0 + n of
// the level); tree arrays [dev] per tree node, rank [dev] per tree node.
int gc_bases_R(int64_t n, const int64_t* nodes, const int64_t* left, const int64_t* right, const int64_t* start,
               const int64_t* stop, const int64_t* rank, int64_t pos0, int64_t W, int64_t* R, int64_t* lim,
               int64_t* vcap, int64_t* rows_node, void* stream) {
    if (n <= 0) return GC_OK;
    const int64_t grid = (n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8;
    k_bases_R<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(n, nodes, left, right, start, stop, rank, pos0, W, R,
                                                               lim, vcap, rows_node);
    GC_CHECK_LAUNCH("k_bases_R");
    return GC_OK;
}

// the level's offsets (exclusive scans of R, limit, vcap) and totals
// (out: R_max, rows, limits, vcap, then v_off at the n_bound side bounds)
int gc_bases_scan(int64_t nn, const int64_t* R, const int64_t* lim, const int64_t* vcap, int64_t* rows_off,
                  int64_t* piv_off_l, int64_t* v_off, const int64_t* bounds, int64_t n_bound, int64_t* out,
                  void* temp, int64_t temp_bytes, void* stream) {
    if (nn <= 0) return GC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    size_t tb = (size_t)temp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb, R, rows_off, (int)nn, st);
    if (e == cudaSuccess) { tb = (size_t)temp_bytes; e = cub::DeviceScan::ExclusiveSum(temp, tb, lim, piv_off_l, (int)nn, st); }
    if (e == cudaSuccess) { tb = (size_t)temp_bytes; e = cub::DeviceScan::ExclusiveSum(temp, tb, vcap, v_off, (int)nn, st); }
    if (e != cudaSuccess) return cuda_status(e, "gc_bases_scan");
    k_bases_totals<<<1, 256, 0, st>>>(nn, R, lim, vcap, rows_off, piv_off_l, v_off, bounds, n_bound, out);
    GC_CHECK_LAUNCH("k_bases_totals");
    count_launch(3);
    return GC_OK;
}

// row lists and descriptors of one side's nodes
int gc_bases_rows(int64_t n, const int64_t* nodes, const int64_t* left, const int64_t* right, const int64_t* start,
                  const int64_t* rank, const int64_t* piv_off, const int64_t* gpiv, const int64_t* perm, int64_t pos0,
                  int64_t box0, int64_t side, int64_t W, const int64_t* R, const int64_t* rows_off,
                  const int64_t* piv_off_l, const int64_t* v_off, int64_t* rows, int64_t* fdesc, int64_t* adesc,
                  void* stream) {
    if (n <= 0) return GC_OK;
    const int64_t grid = n < 148 * 16 ? n : 148 * 16;
    k_bases_rows<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(n, nodes, left, right, start, rank, piv_off, gpiv,
                                                                  perm, pos0, box0, side, W, R, rows_off, piv_off_l,
                                                                  v_off, rows, fdesc, adesc);
    GC_CHECK_LAUNCH("k_bases_rows");
    return GC_OK;
}

// after the ACA of the level: global pivots / ranks / offsets of one side
int gc_bases_post(int64_t n, const int64_t* nodes, int64_t pos0, const int64_t* rank_l, const int64_t* piv_l,
                  const int64_t* piv_off_l, const int64_t* rows, const int64_t* rows_off, const int64_t* v_off,
                  int64_t v_base, int64_t* cursor, int64_t* rank, int64_t* piv_off, int64_t* gpiv,
                  int64_t* v_off_node, int64_t* rk_off, void* temp, int64_t temp_bytes, void* stream) {
    if (n <= 0) return GC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    size_t tb = (size_t)temp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb, rank_l + pos0, rk_off, (int)n, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_bases_post scan");
    const int64_t grid = n < 148 * 16 ? n : 148 * 16;
    k_bases_post<<<(unsigned)grid, 64, 0, st>>>(n, nodes, pos0, rank_l, rk_off, piv_l, piv_off_l, rows, rows_off,
                                               v_off, v_base, cursor, rank, piv_off, gpiv, v_off_node);
    GC_CHECK_LAUNCH("k_bases_post");
    k_bases_cursor<<<1, 32, 0, st>>>(n, rank_l, pos0, rk_off, cursor);
    GC_CHECK_LAUNCH("k_bases_cursor");
    count_launch(1);
    return GC_OK;
}

}  // extern "C"
