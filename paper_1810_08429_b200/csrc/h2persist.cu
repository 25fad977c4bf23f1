// The whole H2 matvec (h2.mvm, h2.py:63-80) as ONE persistent cooperative
// kernel driven by dataflow counters instead of level barriers.
//
// Every product phase is a list of work items over contiguous panels
// (forward transform per tree height, coupling per row cluster, near field
// per row leaf, backward transform per height, final leaf basis + near sum
// + output permutation).  Panels are split by output COLUMNS only, so every
// output element is written by exactly one item with a fixed summation
// order: the result is bitwise deterministic and there are no partial sums.
//
// CTAs walk the global item list round-robin (item i -> CTA i mod G).  An
// item names up to two (counter, target) conditions it waits for and up to
// two counters it bumps when done; dependencies always point to earlier
// items, so with all CTAs co-resident (cooperative launch) the walk cannot
// deadlock.  Static operands (descriptor, input indices, the first batch of
// matrix rows) are loaded BEFORE waiting, so after a dependency resolves an
// item costs one L2 round trip for its inputs plus the stream of the rest of
// its panel.  The latency-bound transform levels no longer pay a launch or
// a grid barrier each.
//
// Work item (8 x int64):
//   [0] type | a_sel<<4 | in_sel<<8 | out_sel<<12 | add_sel<<20
//       type 0: out[out_off + t] = (add ? add[out_off + t] : 0) + s[t]
//       type 2: out[out_off + t] = sum_{i < nrows} scratch[a_off + i*T + t]
//       type 3: y[perm_out[out_off + t]] = add[out_off + t] + s[t]
//   [1] a_off  [2] xi_off  [3] out_off  [4] T (row stride)  [5] nrows
//   [6] c0 | tw << 16 | sig1 << 32 | sig2 << 40     (column slice, signals)
//   [7] wait1 | wait2 << 32, wait = counter << 24 | target   (counter 127: none)
//   s[t] = sum_{r < nrows} A[a_off + r*T + t] * in[xidx[xi_off + r]],  t in [c0, c0+tw)
#include <cuda/atomic>
#include <string.h>

#include "common.cuh"

namespace gcb {

constexpr int PM_THREADS = 256;
constexpr int PM_UNROLL = 16;
constexpr int PM_NONE = 127;
constexpr int PM_SEG0 = 128;     // sync slots 128..: per-segment take counters
constexpr int PM_MAXSEG = 120;

struct MvProgram {
    const int64_t* items;
    const int32_t* xidx;
    int64_t nitems;
    const int64_t* perm_in;     // xt[i] = x[perm_in[i]]
    const int64_t* perm_out;    // y[perm_out[i]] = ...
    int64_t n_in;
    int64_t zero_len;           // buf[3] entries zeroed before the walk
    const double* mat[4];       // panel matrices
    double* buf[8];             // 0 x, 1 xt, 2 x-hat, 3 y-hat (coupling), 4 y-hat, 5 yt (near), 6 y, 7 scratch
    unsigned int* sync;         // [0] start barrier, [1..] dataflow counters; zeroed before launch
    int32_t nseg;               // item segments:
    const int32_t* seg;         // [dev] (nseg, 3): begin, end, unused
    int32_t nlists;             // segment lists in priority order (readiness
    int32_t list_end[8];        // monotone along each list): [end[l-1], end[l])
    long long* timing;          // optional: per item (wait start, wait end, done)
};

__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ bool counter_reached(const unsigned int* ctr, unsigned int target) {
    cuda::atomic_ref<unsigned int, cuda::thread_scope_device> a(*const_cast<unsigned int*>(ctr));
    return a.load(cuda::memory_order_acquire) >= target;
}

template <typename Prog>
__device__ __forceinline__ bool deps_ready(const Prog& P, int64_t w7) {
    const unsigned int w1 = (unsigned int)(w7 & 0xffffffff), w2 = (unsigned int)(w7 >> 32);
    if ((w1 >> 24) != PM_NONE && !counter_reached(P.sync + 1 + (w1 >> 24), w1 & 0xffffff)) return false;
    if ((w2 >> 24) != PM_NONE && !counter_reached(P.sync + 1 + (w2 >> 24), w2 & 0xffffff)) return false;
    return true;
}

__device__ __forceinline__ void wait_counter(unsigned int* ctr, unsigned int target) {
    cuda::atomic_ref<unsigned int, cuda::thread_scope_device> a(*ctr);
    while (a.load(cuda::memory_order_acquire) < target) __nanosleep(20);
}

__device__ void run_item(const MvProgram& P, const int64_t* it, double* xs, double* red,
                         long long* tm) {
    const int64_t head = it[0];
    const int type = (int)(head & 15), a_sel = (int)((head >> 4) & 15);
    const int in_sel = (int)((head >> 8) & 15), out_sel = (int)((head >> 12) & 15);
    const int add_sel = (int)((head >> 20) & 15);
    const int64_t a_off = it[1], xi_off = it[2], out_off = it[3];
    const int T = (int)it[4], nrows = (int)it[5];
    const int64_t w6 = it[6], w7 = it[7];
    const int c0 = (int)(w6 & 0xffff);
    const int tw = ((w6 >> 16) & 0xffff) ? (int)((w6 >> 16) & 0xffff) : T;
    const double* __restrict__ A = P.mat[a_sel] + a_off;
    const int32_t* __restrict__ xi = P.xidx + xi_off;
    const int tt = tw < PM_THREADS ? (tw > 0 ? tw : 1) : PM_THREADS;
    const int ng = PM_THREADS / tt;
    const int g = threadIdx.x / tt;
    // static operands first: the first batch of matrix rows and the input
    // indices do not depend on other items
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
    int32_t myidx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int r = threadIdx.x + j * PM_THREADS;
        myidx[j] = r < nrows ? __ldg(xi + r) : 0;
    }
    // dependencies (none when launched phase by phase: P.sync == nullptr)
    if (tm && threadIdx.x == 0) tm[0] = global_ns();
    if (threadIdx.x == 0 && P.sync) {
        const unsigned int w1 = (unsigned int)(w7 & 0xffffffff), w2 = (unsigned int)(w7 >> 32);
        if ((w1 >> 24) != PM_NONE) wait_counter(P.sync + 1 + (w1 >> 24), w1 & 0xffffff);
        if ((w2 >> 24) != PM_NONE) wait_counter(P.sync + 1 + (w2 >> 24), w2 & 0xffffff);
        __threadfence();
    }
    __syncthreads();
    if (tm && threadIdx.x == 0) tm[1] = global_ns();
    // inputs were written by other CTAs: read through L2 (ld.global.cg)
    const double* __restrict__ x = P.buf[in_sel];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int r = threadIdx.x + j * PM_THREADS;
        if (r < nrows) xs[r] = __ldcg(x + myidx[j]);
    }
    for (int r = threadIdx.x + 4 * PM_THREADS; r < nrows; r += PM_THREADS)
        xs[r] = __ldcg(x + __ldg(xi + r));
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
            const int64_t i = out_off + t;
            if (add_sel) s = __ldcg(P.buf[add_sel] + i) + s;
            if (type == 3)
                P.buf[6][__ldg(P.perm_out + i)] = s;
            else
                P.buf[out_sel][i] = s;
        }
        __syncthreads();
    }
    // signals (after every thread's stores: barrier above, then a fence)
    if (threadIdx.x == 0 && P.sync) {
        const int s1 = (int)((w6 >> 32) & 0xff), s2 = (int)((w6 >> 40) & 0xff);
        __threadfence();
        if (s1 != PM_NONE) atomicAdd(P.sync + 1 + s1, 1u);
        if (s2 != PM_NONE) atomicAdd(P.sync + 1 + s2, 1u);
        if (tm) tm[2] = global_ns();
    }
}

// type 2: out[out_off + t] = sum_{i < nrows} scratch[a_off + i*T + t] (partials of a
// row-split panel, summed in chunk order)
__device__ void reduce_item(const MvProgram& P, const int64_t* it, long long* tm) {
    const int64_t head = it[0];
    const int out_sel = (int)((head >> 12) & 15);
    const int64_t so = it[1], out_off = it[3], T = it[4], nch = it[5];
    const int64_t w6 = it[6], w7 = it[7];
    if (threadIdx.x == 0 && P.sync) {
        if (tm) tm[0] = global_ns();
        const unsigned int w1 = (unsigned int)(w7 & 0xffffffff), w2 = (unsigned int)(w7 >> 32);
        if ((w1 >> 24) != PM_NONE) wait_counter(P.sync + 1 + (w1 >> 24), w1 & 0xffffff);
        if ((w2 >> 24) != PM_NONE) wait_counter(P.sync + 1 + (w2 >> 24), w2 & 0xffffff);
        __threadfence();
        if (tm) tm[1] = global_ns();
    }
    __syncthreads();
    const double* sc = P.buf[7];
    for (int64_t t = threadIdx.x; t < T; t += PM_THREADS) {
        double v = __ldcg(sc + so + t);
        for (int64_t i = 1; i < nch; ++i) v += __ldcg(sc + so + i * T + t);
        P.buf[out_sel][out_off + t] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0 && P.sync) {
        const int s1 = (int)((w6 >> 32) & 0xff), s2 = (int)((w6 >> 40) & 0xff);
        __threadfence();
        if (s1 != PM_NONE) atomicAdd(P.sync + 1 + s1, 1u);
        if (s2 != PM_NONE) atomicAdd(P.sync + 1 + s2, 1u);
        if (tm) tm[2] = global_ns();
    }
}

__global__ void __launch_bounds__(PM_THREADS, 4) k_h2mv_persistent(MvProgram P) {
    extern __shared__ double xs[];      // longest panel's inputs
    __shared__ double red[PM_THREADS];
    const unsigned int G = gridDim.x;
    {   // permuted input and zeroed coupling accumulators, one grid barrier
        const int64_t stride = (int64_t)G * PM_THREADS;
        for (int64_t i = blockIdx.x * (int64_t)PM_THREADS + threadIdx.x; i < P.n_in; i += stride)
            P.buf[1][i] = __ldcg(P.buf[0] + __ldg(P.perm_in + i));
        for (int64_t i = blockIdx.x * (int64_t)PM_THREADS + threadIdx.x; i < P.zero_len; i += stride)
            P.buf[3][i] = 0.0;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(P.sync, 1u);
            wait_counter(P.sync, G);
            __threadfence();
        }
        __syncthreads();
    }
    if (P.timing && blockIdx.x == 0 && threadIdx.x == 0) P.timing[3 * P.nitems] = global_ns();
    // Scheduler.  Items form segments (runs with one shared dependency) in
    // priority order: transform chains, coupling by deadline, filler.
    // Thread 0 takes from the first segment that is both non-exhausted and
    // ready, with one atomicAdd on that segment's counter (an overshoot just
    // means exhausted), so a taken item never waits, CTAs never block one
    // another and the walk is deadlock-free for any dependency DAG.
    __shared__ long long s_taken;
    __shared__ int s_cur[8];                 // per list: first non-exhausted segment
    __shared__ unsigned char s_ready[PM_MAXSEG];
    if (threadIdx.x < 8) s_cur[threadIdx.x] = threadIdx.x ? P.list_end[threadIdx.x - 1] : 0;
    for (int q = threadIdx.x; q < PM_MAXSEG; q += PM_THREADS) s_ready[q] = 0;
    __syncthreads();
    for (;;) {
        if (threadIdx.x == 0) {
            long long taken = -1;
            unsigned int spins = 0;
            for (;;) {
                bool left = false;
                for (int l = 0; l < P.nlists && taken < 0; ++l) {
                    int q = s_cur[l];
                    while (q < P.list_end[l]) {
                        const int b = P.seg[3 * q], e = P.seg[3 * q + 1];
                        unsigned int* ctr = P.sync + 1 + PM_SEG0 + q;
                        cuda::atomic_ref<unsigned int, cuda::thread_scope_device> a(*ctr);
                        if (b + (int)a.load(cuda::memory_order_relaxed) >= e) { s_cur[l] = ++q; continue; }
                        left = true;
                        if (!s_ready[q]) {
                            // readiness is monotone along a list: stop at the
                            // first segment that is not ready yet
                            if (!deps_ready(P, P.items[8 * (int64_t)b + 7])) break;
                            s_ready[q] = 1;
                        }
                        const unsigned int k = a.fetch_add(1u, cuda::memory_order_relaxed);
                        if (b + (int)k < e) { taken = b + k; break; }
                        s_cur[l] = ++q;
                    }
                }
                if (taken >= 0 || !left) break;
                __nanosleep(spins < 16 ? 32 : 128);
                ++spins;
            }
            __threadfence();
            s_taken = taken;
        }
        __syncthreads();
        const long long i = s_taken;
        __syncthreads();
        if (i < 0) break;
        const int64_t* it = P.items + 8 * i;
        long long* tm = P.timing ? P.timing + 3 * i : nullptr;
        if ((it[0] & 15) == 2)
            reduce_item(P, it, tm);
        else
            run_item(P, it, xs, red, tm);
    }
}

}  // namespace gcb

using namespace gcb;

extern "C" int gc_h2mv_persistent(const int64_t* items, const int32_t* xidx, int64_t nitems,
                                  int32_t nseg, const int32_t* seg, int32_t nlists,
                                  const int32_t* list_end,
                                  const int64_t* perm_in, const int64_t* perm_out, int64_t n_in,
                                  int64_t zero_len, const double* const* mats, double* const* bufs,
                                  unsigned int* sync, int32_t nsync, int32_t grid,
                                  long long* timing, int32_t max_rows, void* stream) {
    MvProgram P;
    P.items = items;
    P.xidx = xidx;
    P.nitems = nitems;
    if (nseg < 1 || nseg > PM_MAXSEG) { set_error(GC_ERR_CONFIG, "1..%d item segments", PM_MAXSEG); return GC_ERR_CONFIG; }
    if (nsync < 1 + PM_SEG0 + nseg) { set_error(GC_ERR_CONFIG, "sync array too small"); return GC_ERR_CONFIG; }
    P.nseg = nseg;
    P.seg = seg;
    if (nlists < 1 || nlists > 8) { set_error(GC_ERR_CONFIG, "1..8 segment lists"); return GC_ERR_CONFIG; }
    P.nlists = nlists;
    for (int l = 0; l < 8; ++l) P.list_end[l] = l < nlists ? list_end[l] : nseg;
    P.perm_in = perm_in;
    P.perm_out = perm_out;
    P.n_in = n_in;
    P.zero_len = zero_len;
    for (int i = 0; i < 4; ++i) P.mat[i] = mats[i];
    for (int i = 0; i < 8; ++i) P.buf[i] = bufs[i];
    P.sync = sync;
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
    e = cudaMemsetAsync(sync, 0, (size_t)nsync * sizeof(unsigned int), st);
    if (e != cudaSuccess) return cuda_status(e, "gc_h2mv_persistent counter reset");
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

// ---------------------------------------------------------------------------
// The same work items launched phase by phase (one CTA per item, no
// scheduling): the multi-launch formulation used inside a CUDA graph.
namespace gcb {

__global__ void __launch_bounds__(PM_THREADS) k_run_items(MvProgram P, int64_t first) {
    extern __shared__ double xs[];
    __shared__ double red[PM_THREADS];
    const int64_t* it = P.items + 8 * (first + blockIdx.x);
    if ((it[0] & 15) == 2)
        reduce_item(P, it, nullptr);
    else
        run_item(P, it, xs, red, nullptr);
}

}  // namespace gcb

extern "C" int gc_run_items(const int64_t* items, int64_t first, int64_t count, const int32_t* xidx,
                            const double* const* mats, double* const* bufs, unsigned int* sync,
                            int32_t max_rows, const int64_t* perm_out, void* stream) {
    using namespace gcb;
    if (count <= 0) return GC_OK;
    if (count > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "too many items"); return GC_ERR_CONFIG; }
    MvProgram P;
    memset(&P, 0, sizeof(P));
    P.items = items;
    P.xidx = xidx;
    P.nitems = first + count;
    P.perm_out = perm_out;
    for (int i = 0; i < 4; ++i) P.mat[i] = mats[i];
    for (int i = 0; i < 8; ++i) P.buf[i] = bufs[i];
    P.sync = nullptr;   // stream order replaces the dataflow counters
    (void)sync;
    const size_t smem = (size_t)(max_rows > 0 ? max_rows : 1) * sizeof(double);
    if (smem > 160 * 1024) { set_error(GC_ERR_CONFIG, "panel with %d rows is too long", max_rows); return GC_ERR_CONFIG; }
    cudaError_t e = cudaFuncSetAttribute(k_run_items, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "gc_run_items smem attribute");
    k_run_items<<<(unsigned)count, PM_THREADS, smem, (cudaStream_t)stream>>>(P, first);
    GC_CHECK_LAUNCH("k_run_items");
    return GC_OK;
}
