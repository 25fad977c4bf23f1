// The whole H2 matvec (h2.mvm, h2.py:63-80) as ONE persistent cooperative
// kernel: every tree level of the forward transform, the coupling phase,
// the coupling reduction, every level of the backward transform and the
// final leaf-basis + near-field + permutation stage run as stages of a
// single launch separated by grid barriers.  The ~20 launches (and their
// drain/launch gaps) of the level-by-level formulation collapse to one;
// the near-field panels run in the same stage as the coupling panels.
//
// Work items (8 x int64):
//   [0] type | a_sel << 4 | in_sel << 8 | out_sel << 12 | acc << 16
//       type 0: panel product -> out[out_off + t]  (acc: += instead of =)
//       type 1: panel product -> scratch[out_off + t]
//       type 2: reduce: out[out_off + t] (+)= sum_{i<aux2} scratch[aux + i*T + t]
//       type 3: leaf final: y[perm_out[out_off + t]] = yt[out_off + t] + panel(t)
//   [1] a_off  [2] xi_off  [3] out_off  [4] T  [5] nrows  [6] c0 / aux  [7] tw / aux2
// Panel product over the column slice t in [c0, c0+tw) (tw = 0: all T):
//   s[t] = sum_{r < nrows} A[a_off + r*T + t] * in[xidx[xi_off + r]].
// Panels are split by columns, never by rows, so no partial sums exist.
// Every output element has one writer and a fixed summation order, so the
// result is bitwise identical to the multi-launch formulation's order
// within each item and deterministic run to run.
#include <cuda/atomic>

#include "common.cuh"

namespace gcb {

constexpr int PM_THREADS = 256;
constexpr int PM_UNROLL = 16;

struct MvProgram {
    const int64_t* items;
    const int32_t* xidx;
    const int32_t* stage_off;   // nstages + 1
    int32_t nstages;
    int32_t pad;
    const int64_t* perm_in;     // xt[i] = x[perm_in[i]]
    const int64_t* perm_out;    // y[perm_out[i]] = yt[i] + ...
    int64_t n_in;
    int64_t zero_len;           // yhat entries zeroed in stage 0
    const double* mat[4];       // panel matrices
    double* buf[8];             // 0 x, 1 xt, 2 xhat, 3 yhat, 4 yt, 5 y, 6 scratch
    unsigned int* barrier;      // zeroed before launch
    long long* timing;          // optional: globaltimer after each stage (block 0)
};

__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned int, cuda::thread_scope_device> a(*bar);
        __threadfence();
        a.fetch_add(1u, cuda::memory_order_release);
        while (a.load(cuda::memory_order_acquire) < target) __nanosleep(32);
        __threadfence();
    }
    __syncthreads();
}

__device__ void panel_item(const MvProgram& P, const int64_t* it, double* xs, double* red) {
    const int64_t head = it[0];
    const int type = (int)(head & 15), a_sel = (int)((head >> 4) & 15);
    const int in_sel = (int)((head >> 8) & 15), out_sel = (int)((head >> 12) & 15);
    const bool acc_out = ((head >> 16) & 1) != 0;
    const int64_t a_off = it[1], xi_off = it[2], out_off = it[3];
    const int T = (int)it[4], nrows = (int)it[5], c0 = (int)it[6];
    const int tw = it[7] > 0 ? (int)it[7] : T;          // column slice [c0, c0 + tw)
    const double* __restrict__ A = P.mat[a_sel] + a_off;
    const double* __restrict__ x = P.buf[in_sel];
    const int32_t* __restrict__ xi = P.xidx + xi_off;
    const int tt = tw < PM_THREADS ? (tw > 0 ? tw : 1) : PM_THREADS;
    const int ng = PM_THREADS / tt;
    const int g = threadIdx.x / tt;
    // first batch of matrix loads is issued before the (dependent) input
    // gather so the two memory round trips overlap
    double a0[PM_UNROLL];
    {
        const int t = c0 + (int)(threadIdx.x % tt);
        const bool live = g < ng && t < c0 + tw;
#pragma unroll
        for (int j = 0; j < PM_UNROLL; ++j) {
            const int r = g + j * ng;
            a0[j] = (live && r < nrows) ? __ldcs(A + (int64_t)r * T + t) : 0.0;
        }
    }
    // inputs may have been written by other CTAs in an earlier stage of this
    // launch: read them through L2 (ld.global.cg), never from a stale L1 line
    for (int r = threadIdx.x; r < nrows; r += PM_THREADS) xs[r] = __ldcg(x + __ldg(xi + r));
    __syncthreads();
    for (int t0 = c0; t0 < c0 + tw; t0 += tt) {
        const int t = t0 + (int)(threadIdx.x % tt);
        const bool live = g < ng && t < c0 + tw;
        double acc = 0.0;
        if (live) {
            const double* __restrict__ At = A + t;
            int r = g;
            if (t0 == c0) {
#pragma unroll
                for (int j = 0; j < PM_UNROLL; ++j)
                    if (r + j * ng < nrows) acc = fma(a0[j], xs[r + j * ng], acc);
                r += PM_UNROLL * ng;
            }
            for (; r + (PM_UNROLL - 1) * ng < nrows; r += PM_UNROLL * ng) {
                double a[PM_UNROLL];
#pragma unroll
                for (int j = 0; j < PM_UNROLL; ++j) a[j] = __ldcs(At + (int64_t)(r + j * ng) * T);
#pragma unroll
                for (int j = 0; j < PM_UNROLL; ++j) acc = fma(a[j], xs[r + j * ng], acc);
            }
            for (; r < nrows; r += ng) acc = fma(__ldcs(At + (int64_t)r * T), xs[r], acc);
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < tt && t < c0 + tw) {
            double s = red[threadIdx.x];
            for (int q = 1; q < ng; ++q) s += red[q * tt + threadIdx.x];
            if (type == 0) {
                double* o = P.buf[out_sel] + out_off + t;
                *o = acc_out ? __ldcg(o) + s : s;
            } else if (type == 1) {
                P.buf[6][out_off + t] = s;
            } else {  // type 3: leaf final
                const int64_t i = out_off + t;
                P.buf[5][__ldg(P.perm_out + i)] = __ldcg(P.buf[4] + i) + s;
            }
        }
        __syncthreads();
    }
}

__device__ void reduce_item(const MvProgram& P, const int64_t* it) {
    const int64_t head = it[0];
    const int out_sel = (int)((head >> 12) & 15);
    const bool acc_out = ((head >> 16) & 1) != 0;
    const int64_t out_off = it[3], T = it[4], so = it[6], ni = it[7];
    const double* sc = P.buf[6];
    for (int64_t t = threadIdx.x; t < T; t += PM_THREADS) {
        double v = __ldcg(sc + so + t);
        for (int64_t i = 1; i < ni; ++i) v += __ldcg(sc + so + i * T + t);
        double* o = P.buf[out_sel] + out_off + t;
        *o = acc_out ? __ldcg(o) + v : v;
    }
}

__global__ void __launch_bounds__(PM_THREADS, 4) k_h2mv_persistent(MvProgram P) {
    extern __shared__ double xs[];      // max rows over all items
    __shared__ double red[PM_THREADS];
    const unsigned int G = gridDim.x;
    // stage 0: permuted input and zeroed coupling accumulators
    {
        const int64_t stride = (int64_t)G * PM_THREADS;
        for (int64_t i = blockIdx.x * (int64_t)PM_THREADS + threadIdx.x; i < P.n_in; i += stride)
            P.buf[1][i] = __ldcg(P.buf[0] + __ldg(P.perm_in + i));
        for (int64_t i = blockIdx.x * (int64_t)PM_THREADS + threadIdx.x; i < P.zero_len; i += stride)
            P.buf[3][i] = 0.0;
    }
    if (P.timing && blockIdx.x == 0 && threadIdx.x == 0) P.timing[0] = global_ns();
    unsigned int target = G;
    grid_barrier(P.barrier, target);
    if (P.timing && blockIdx.x == 0 && threadIdx.x == 0) P.timing[1] = global_ns();
    for (int s = 0; s < P.nstages; ++s) {
        const int b = P.stage_off[s], e = P.stage_off[s + 1];
        for (int i = b + (int)blockIdx.x; i < e; i += (int)G) {
            const int64_t* it = P.items + 8 * (int64_t)i;
            if ((it[0] & 15) == 2)
                reduce_item(P, it);
            else
                panel_item(P, it, xs, red);
        }
        if (P.timing && blockIdx.x == 0 && threadIdx.x == 0) P.timing[2 + 2 * s] = global_ns();
        if (s + 1 < P.nstages) {
            target += G;
            grid_barrier(P.barrier, target);
        }
        if (P.timing && blockIdx.x == 0 && threadIdx.x == 0) P.timing[3 + 2 * s] = global_ns();
    }
}

}  // namespace gcb

using namespace gcb;

extern "C" int gc_h2mv_persistent(const int64_t* items, const int32_t* xidx,
                                  const int32_t* stage_off, int32_t nstages,
                                  const int64_t* perm_in, const int64_t* perm_out, int64_t n_in,
                                  int64_t zero_len, const double* const* mats, double* const* bufs,
                                  unsigned int* barrier, int32_t grid, long long* timing,
                                  int32_t max_rows, void* stream) {
    MvProgram P;
    P.items = items;
    P.xidx = xidx;
    P.stage_off = stage_off;
    P.nstages = nstages;
    P.pad = 0;
    P.perm_in = perm_in;
    P.perm_out = perm_out;
    P.n_in = n_in;
    P.zero_len = zero_len;
    for (int i = 0; i < 4; ++i) P.mat[i] = mats[i];
    for (int i = 0; i < 8; ++i) P.buf[i] = bufs[i];
    P.barrier = barrier;
    P.timing = timing;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t smem = (size_t)(max_rows > 0 ? max_rows : 1) * sizeof(double);
    if (smem > 160 * 1024) { set_error(GC_ERR_CONFIG, "panel with %d rows is too long", max_rows); return GC_ERR_CONFIG; }
    cudaError_t e = cudaFuncSetAttribute(k_h2mv_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2mv_persistent smem attribute");
    int max_blocks = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks, k_h2mv_persistent, PM_THREADS, smem);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2mv_persistent occupancy");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int cap = max_blocks * sms;
    if (grid <= 0 || grid > cap) grid = cap;
    e = cudaMemsetAsync(barrier, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2mv_persistent barrier reset");
    void* args[] = {&P};
    e = cudaLaunchCooperativeKernel((const void*)k_h2mv_persistent, dim3(grid), dim3(PM_THREADS),
                                    args, smem, st);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2mv_persistent launch");
    count_launch();
    return GC_OK;
}

extern "C" int gc_h2mv_grid(int32_t max_rows, int32_t* grid_out) {
    int max_blocks = 0, dev = 0, sms = 0;
    const size_t smem = (size_t)(max_rows > 0 ? max_rows : 1) * sizeof(double);
    cudaFuncSetAttribute(k_h2mv_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks, k_h2mv_persistent,
                                                                  PM_THREADS, smem);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2mv_grid");
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    *grid_out = max_blocks * sms;
    return GC_OK;
}
