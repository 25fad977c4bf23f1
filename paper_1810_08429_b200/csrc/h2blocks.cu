// Block tables of build_h2 (gca.py:282-312) on the device: from the block
// tree's leaves in depth-first order, the coupling (admissible) or
// near-field (inadmissible) blocks of one kind, their sizes (pivot counts or
// cluster sizes), storage offsets grouped by block row (stable in DFS order:
// the blocks of one block row form one contiguous panel of the matvec), and
// the assembly descriptors of the non-empty blocks.  Replaces the host
// numpy pass over every leaf (gathers, a stable argsort per kind, stacks
// and the descriptor uploads).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"

namespace gcb {

struct BlkIn {
    const int64_t* leaf_ids;   // nl leaves (DFS order)
    const int64_t* node_row;   // block-tree node -> row / col cluster
    const int64_t* node_col;
    const int8_t* node_state;  // 0 admissible, 1 inadmissible
    const int64_t* r_start;    // cluster trees
    const int64_t* r_stop;
    const int64_t* c_start;
    const int64_t* c_stop;
    const int64_t* r_rank;     // bases (coupling blocks)
    const int64_t* r_poff;
    const int64_t* c_rank;
    const int64_t* c_poff;
    const int8_t* r_ok;        // coupling: row cluster has basis content / column pivots available
    const int8_t* c_ok;
    int64_t lo, hi;            // block-row shard [lo, hi) of tree positions, lo < 0: none
    int32_t near;              // 0 coupling, 1 near field
};

__global__ void k_blk_flag(int64_t nl, BlkIn in, char* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = in.leaf_ids[i];
        const int64_t r = in.node_row[b];
        bool f = in.node_state[b] == (in.near ? 1 : 0);
        if (in.lo >= 0) f = f && in.r_start[r] >= in.lo && in.r_stop[r] <= in.hi;
        flag[i] = f;
    }
}

// block j < count: row / col cluster, sizes, storage key; padding entries
// sort last with size 0
__global__ void k_blk_fill(int64_t nl, BlkIn in, const int64_t* __restrict__ count, const int64_t* __restrict__ sel,
                           int64_t sentinel, int64_t* __restrict__ row, int64_t* __restrict__ col,
                           int64_t* __restrict__ nr, int64_t* __restrict__ nc, int64_t* __restrict__ key,
                           int64_t* __restrict__ size, int64_t* __restrict__ idx,
                           unsigned long long* __restrict__ bad) {
    const int64_t n = *count;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nl; j += (int64_t)gridDim.x * blockDim.x) {
        idx[j] = j;
        if (j >= n) {
            key[j] = sentinel;
            size[j] = 0;
            continue;
        }
        const int64_t b = in.leaf_ids[sel[j]];
        const int64_t r = in.node_row[b], c = in.node_col[b];
        if (!in.near && (!in.r_ok[r] || !in.c_ok[c])) atomicAdd(bad, 1ULL);
        const int64_t a = in.near ? in.r_stop[r] - in.r_start[r] : in.r_rank[r];
        const int64_t d = in.near ? in.c_stop[c] - in.c_start[c] : in.c_rank[c];
        row[j] = r;
        col[j] = c;
        nr[j] = a;
        nc[j] = d;
        size[j] = a * d;
        key[j] = in.lo >= 0 ? 2 * r + !(in.c_start[c] >= in.lo && in.c_stop[c] <= in.hi) : r;
    }
}

__global__ void k_blk_gather(int64_t nl, const int64_t* __restrict__ order, const int64_t* __restrict__ size,
                             int64_t* __restrict__ ss) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nl; j += (int64_t)gridDim.x * blockDim.x)
        ss[j] = size[order[j]];
}

// host table (6 columns of stride count): row, col, nr, nc, off, order; the
// keep flags (non-empty blocks)
__global__ void k_blk_scatter(int64_t nl, const int64_t* __restrict__ count, const int64_t* __restrict__ order,
                              const int64_t* __restrict__ soff, const int64_t* __restrict__ row,
                              const int64_t* __restrict__ col, const int64_t* __restrict__ nr,
                              const int64_t* __restrict__ nc, int64_t* __restrict__ off, int64_t* __restrict__ table,
                              char* __restrict__ keep) {
    const int64_t n = *count;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nl; j += (int64_t)gridDim.x * blockDim.x) {
        if (j >= n) {
            keep[j] = 0;
            continue;
        }
        off[order[j]] = soff[j];
        table[j] = row[j];
        table[n + j] = col[j];
        table[2 * n + j] = nr[j];
        table[3 * n + j] = nc[j];
        table[5 * n + j] = order[j];
        keep[j] = nr[j] > 0 && nc[j] > 0;
    }
}

__global__ void k_blk_desc(int64_t nl, BlkIn in, const int64_t* __restrict__ count, const int64_t* __restrict__ nkeep,
                           const int64_t* __restrict__ kept, const int64_t* __restrict__ off,
                           int64_t* __restrict__ table, int64_t* __restrict__ desc) {
    const int64_t n = *count, m = *nkeep;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nl; j += (int64_t)gridDim.x * blockDim.x) {
        if (j < n) table[4 * n + j] = off[j];
        if (j >= m) continue;
        const int64_t q = kept[j];
        const int64_t r = table[q], c = table[n + q];
        int64_t* d = desc + 5 * j;
        d[0] = in.near ? in.r_start[r] : in.r_poff[r];
        d[1] = table[2 * n + q];
        d[2] = in.near ? in.c_start[c] : in.c_poff[c];
        d[3] = table[3 * n + q];
        d[4] = off[q];
    }
}

// totals: count, kept, max nr, max nc (kept blocks), entries
__global__ void k_blk_totals(const int64_t* __restrict__ count, const int64_t* __restrict__ nkeep,
                             const int64_t* __restrict__ desc, const int64_t* __restrict__ soff,
                             const int64_t* __restrict__ ss, int64_t* __restrict__ tot) {
    __shared__ int64_t red[2][256];
    const int64_t n = *count, m = *nkeep;
    int64_t a = 0, b = 0;
    for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
        a = desc[5 * j + 1] > a ? desc[5 * j + 1] : a;
        b = desc[5 * j + 3] > b ? desc[5 * j + 3] : b;
    }
    red[0][threadIdx.x] = a;
    red[1][threadIdx.x] = b;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            if (red[0][threadIdx.x + o] > red[0][threadIdx.x]) red[0][threadIdx.x] = red[0][threadIdx.x + o];
            if (red[1][threadIdx.x + o] > red[1][threadIdx.x]) red[1][threadIdx.x] = red[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        tot[0] = n;
        tot[1] = m;
        tot[2] = red[0][0];
        tot[3] = red[1][0];
        tot[4] = n ? soff[n - 1] + ss[n - 1] : 0;
    }
}

}  // namespace gcb

using namespace gcb;

namespace {

size_t blk_temp(int64_t nl) {
    size_t t1 = 0, t2 = 0, t3 = 0;
    thrust::counting_iterator<int64_t> it(0);
    cub::DeviceSelect::Flagged(nullptr, t1, it, (const char*)nullptr, (int64_t*)nullptr, (int64_t*)nullptr, (int)nl);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (const int64_t*)nullptr, (int64_t*)nullptr, (const int64_t*)nullptr,
                                    (int64_t*)nullptr, (int)nl);
    cub::DeviceScan::ExclusiveSum(nullptr, t3, (const int64_t*)nullptr, (int64_t*)nullptr, (int)nl);
    size_t t = t1 > t2 ? t1 : t2;
    return t > t3 ? t : t3;
}

}  // namespace

extern "C" {

int gc_h2_blocks_bytes(int64_t nl, int64_t* bytes) {
    *bytes = (int64_t)blk_temp(nl > 0 ? nl : 1);
    return GC_OK;
}

// One kind of blocks (near = 0 coupling, 1 near field) of nl leaves; see
// include/gcb200.h.
int gc_h2_blocks(int64_t nl, const int64_t* leaf_ids, const int64_t* node_row, const int64_t* node_col,
                 const int8_t* node_state, const int64_t* r_start, const int64_t* r_stop, const int64_t* c_start,
                 const int64_t* c_stop, const int64_t* r_rank, const int64_t* r_poff, const int64_t* c_rank,
                 const int64_t* c_poff, const int8_t* r_ok, const int8_t* c_ok, int64_t lo, int64_t hi,
                 int32_t near, int32_t key_bits, int64_t* table,
                 int64_t* desc, int64_t* totals, int64_t* scratch, char* flags, void* temp, int64_t temp_bytes,
                 void* stream) {
    if (nl <= 0) return GC_OK;
    if (nl > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "gc_h2_blocks: too many leaves"); return GC_ERR_CONFIG; }
    if (key_bits < 1 || key_bits > 63) { set_error(GC_ERR_CONFIG, "gc_h2_blocks: key bits"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    BlkIn in{leaf_ids, node_row, node_col, node_state, r_start, r_stop, c_start, c_stop, r_rank, r_poff, c_rank,
             c_poff, r_ok, c_ok, lo, hi, near};
    int64_t* sel = scratch;
    int64_t* row = scratch + nl;
    int64_t* col = scratch + 2 * nl;
    int64_t* nr = scratch + 3 * nl;
    int64_t* nc = scratch + 4 * nl;
    int64_t* key = scratch + 5 * nl;
    int64_t* size = scratch + 6 * nl;
    int64_t* idx = scratch + 7 * nl;
    int64_t* key_out = scratch + 8 * nl;
    int64_t* order = scratch + 9 * nl;
    int64_t* ss = scratch + 10 * nl;
    int64_t* soff = scratch + 11 * nl;
    int64_t* off = key;                 // dead after the sort
    int64_t* kept = idx;                // dead after the sort
    int64_t* count = totals + 5;
    int64_t* nkeep = totals + 6;
    char* flag = flags;
    char* keep = flags + nl;
    const int64_t grid = (nl + 255) / 256 < 148 * 16 ? (nl + 255) / 256 : 148 * 16;
    const int64_t sentinel = (1LL << (key_bits - 1)) - 1 + (1LL << (key_bits - 1));
    k_blk_flag<<<(unsigned)grid, 256, 0, st>>>(nl, in, flag);
    GC_CHECK_LAUNCH("k_blk_flag");
    size_t tb = (size_t)temp_bytes;
    thrust::counting_iterator<int64_t> it(0);
    cudaError_t e = cub::DeviceSelect::Flagged(temp, tb, it, flag, sel, count, (int)nl, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2_blocks select");
    k_blk_fill<<<(unsigned)grid, 256, 0, st>>>(nl, in, count, sel, sentinel, row, col, nr, nc, key, size, idx,
                                                reinterpret_cast<unsigned long long*>(totals + 7));
    GC_CHECK_LAUNCH("k_blk_fill");
    tb = (size_t)temp_bytes;
    e = cub::DeviceRadixSort::SortPairs(temp, tb, key, key_out, idx, order, (int)nl, 0, key_bits, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2_blocks sort");
    k_blk_gather<<<(unsigned)grid, 256, 0, st>>>(nl, order, size, ss);
    GC_CHECK_LAUNCH("k_blk_gather");
    tb = (size_t)temp_bytes;
    e = cub::DeviceScan::ExclusiveSum(temp, tb, ss, soff, (int)nl, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2_blocks scan");
    k_blk_scatter<<<(unsigned)grid, 256, 0, st>>>(nl, count, order, soff, row, col, nr, nc, off, table, keep);
    GC_CHECK_LAUNCH("k_blk_scatter");
    tb = (size_t)temp_bytes;
    e = cub::DeviceSelect::Flagged(temp, tb, it, keep, kept, nkeep, (int)nl, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2_blocks keep");
    k_blk_desc<<<(unsigned)grid, 256, 0, st>>>(nl, in, count, nkeep, kept, off, table, desc);
    GC_CHECK_LAUNCH("k_blk_desc");
    k_blk_totals<<<1, 256, 0, st>>>(count, nkeep, desc, soff, ss, totals);
    GC_CHECK_LAUNCH("k_blk_totals");
    count_launch(4);
    return GC_OK;
}

}  // extern "C"
