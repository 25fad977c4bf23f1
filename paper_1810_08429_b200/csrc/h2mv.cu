// The H2 matvec (h2.py:19-80) as panel products: every phase - forward
// transform (V^T x, composed transfers), coupling (S x-hat), backward
// transform, near-field SpMV, leaf rows - is out[t] (+)= sum_k A[k*T + t]
// in[idx[k]] over contiguous row-major panels, cut into work items.
#include "common.cuh"

// ---------------------------------------------------------------------------
// Panel products (the mvm hot path).  A "panel" is one contiguous row-major
// K x T matrix (all coupling blocks of one row cluster stored back to back,
// all near-field blocks of one row leaf, one V-hat, ...).  The panels of a
// phase are cut into work items of ~32 KB so every CTA streams the same
// amount of HBM; items of a multi-item panel write partial sums to scratch
// and the last CTA of the panel adds them in item order (bitwise deterministic).
namespace gcb {

constexpr int PAN_THREADS = 256;
#ifndef GC_PAN_UNROLL
#define GC_PAN_UNROLL 8
#endif
constexpr int PAN_UNROLL = GC_PAN_UNROLL;
#ifndef GC_PAN_MINB
#define GC_PAN_MINB 6
#endif
constexpr int PAN_MAX_ROWS = 1024;   // rows per work item (x gathered to smem)

// item (8 x int64): a_off, xi_off, out_off, T, nrows, mode, red, 0
//   mode bit0 A1, bit1 in1, bit2 direct to out, bit3 accumulate into out,
//   bit4 prefetch the item's matrix chunk into L2 before the input gather,
//   bit5 the input is in0 + in1 (both at the gathered indices);
//   red = reduction slot of a split panel (items without bit2 write partial
//   sums to scratch[out_off..]).
// red slot (5 x int64): out_off, T, scratch_off, nitems, accumulate.
// The item's input entries are gathered into shared memory first, so the
// streaming loop over A has no dependent loads: PAN_UNROLL independent 8-byte loads
// per thread are in flight before the first FMA.  The last CTA to finish a
// split panel (arrival counter) adds its partial sums in item order, so the
// result is bitwise deterministic without a second launch; it re-arms the
// counter for the next product.
struct PanelSmem {
    double red[PAN_THREADS];
    double xs[PAN_MAX_ROWS];
    int last;
};

struct PanelPhase {           // one phase (forward level, bucket, ...) of the product
    const int64_t* items;
    int64_t nitems;
    const int32_t* xidx;
    const double* A0;
    const double* A1;
    const double* in0;
    const double* in1;
    double* out;
    double* scratch;
    const int64_t* red;
    int* arrivals;
    unsigned long long* trace;   // optional: min start / max end %globaltimer (ns)
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Diagnostics (PanelPhase.trace, scripts/timeline.py): trace[0] / [1] =
// min CTA start / max CTA end (%globaltimer, ns); when trace[2] = n > 0,
// CTA b < n also records its own [start, end] at trace[4 + 2b].
__device__ __forceinline__ void trace_begin(const PanelPhase& P) {
    if (P.trace == nullptr || threadIdx.x != 0) return;
    const unsigned long long t = globaltimer();
    atomicMin(P.trace, t);
    if (P.trace[2] > blockIdx.x) P.trace[4 + 2 * (int64_t)blockIdx.x] = t;
}

__device__ __forceinline__ void trace_end(const PanelPhase& P) {
    if (P.trace == nullptr) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long t = globaltimer();
        atomicMax(P.trace + 1, t);
        if (P.trace[2] > blockIdx.x) P.trace[5 + 2 * (int64_t)blockIdx.x] = t;
    }
}

__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(127);
    const uintptr_t hi = reinterpret_cast<uintptr_t>(p) + bytes;
    for (uintptr_t l = lo + 128 * threadIdx.x; l < hi; l += 128 * PAN_THREADS)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
}


// load the item's inputs into smem (WAIT: griddepcontrol.wait between the
// input-independent prologue and the first read of the input vector)
template <bool WAIT>
__device__ __forceinline__ void panel_item(const PanelPhase& P, int64_t item, PanelSmem& sm) {
    const int64_t* it = P.items + 8 * item;
    const int64_t a_off = it[0], xi_off = it[1], out_off = it[2];
    const int T = (int)it[3], nrows = (int)it[4], mode = (int)it[5];
    const double* __restrict__ A = ((mode & 1) ? P.A1 : P.A0) + a_off;
    const double* x = (mode & 2) ? P.in1 : P.in0;
    const int32_t* __restrict__ xi = P.xidx + xi_off;
    if (WAIT) {
        int* xsi = reinterpret_cast<int*>(sm.red);
        prefetch_l2(A, 8 * (int64_t)nrows * T);
        const bool staged = nrows <= 2 * PAN_THREADS;
        if (staged)
            for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) xsi[r] = __ldg(xi + r);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (mode & 32) {
            for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) {
                const int i = staged ? xsi[r] : __ldg(xi + r);
                sm.xs[r] = __ldcg(P.in0 + i) + __ldcg(P.in1 + i);
            }
        } else if (staged) {
            for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) sm.xs[r] = __ldcg(x + xsi[r]);
        } else {
            for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) sm.xs[r] = __ldcg(x + __ldg(xi + r));
        }
    } else {
        if (mode & 32) {
            for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) {
                const int i = __ldg(xi + r);
                sm.xs[r] = __ldcg(P.in0 + i) + __ldcg(P.in1 + i);
            }
        } else {
            for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) sm.xs[r] = __ldcg(x + __ldg(xi + r));
        }
    }
    __syncthreads();
    const int tt = T < PAN_THREADS ? T : PAN_THREADS;
    const int ng = PAN_THREADS / tt;
    const int g = threadIdx.x / tt;
    for (int t0 = 0; t0 < T; t0 += tt) {
        const int t = t0 + (int)(threadIdx.x % tt);
        const bool live = g < ng && t < T;
        double acc = 0.0;
        if (live) {
            const double* __restrict__ At = A + t;
            int r = g;
            for (; r + (PAN_UNROLL - 1) * ng < nrows; r += PAN_UNROLL * ng) {
                double a[PAN_UNROLL];
#pragma unroll
                for (int j = 0; j < PAN_UNROLL; ++j) a[j] = __ldcs(At + (int64_t)(r + j * ng) * T);
                // pins the batch: ptxas otherwise may sink loads between the
                // FMAs under the 40-register cap (WARPSYNC.ALL, no wait)
                __syncwarp(__activemask());
#pragma unroll
                for (int j = 0; j < PAN_UNROLL; ++j) acc = fma(a[j], sm.xs[r + j * ng], acc);
            }
            for (; r < nrows; r += ng) acc = fma(__ldcs(At + (int64_t)r * T), sm.xs[r], acc);
        }
        sm.red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < tt && t < T) {
            double s = sm.red[threadIdx.x];
            for (int q = 1; q < ng; ++q) s += sm.red[q * tt + threadIdx.x];
            if (mode & 4) {
                double* o = P.out + out_off + t;
                *o = (mode & 8) ? __ldcg(o) + s : s;
            } else {
                P.scratch[out_off + t] = s;
            }
        }
        __syncthreads();
    }
    if (mode & 4) return;
    const int slot = (int)it[6];
    const int64_t* rd = P.red + 5 * (int64_t)slot;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) sm.last = atomicAdd(P.arrivals + slot, 1) == (int)rd[3] - 1;
    __syncthreads();
    if (!sm.last) return;
    __threadfence();
    const int64_t o_off = rd[0], so = rd[2];
    const int RT = (int)rd[1], ni = (int)rd[3];
    const bool accum = rd[4] != 0;
    for (int t = threadIdx.x; t < RT; t += PAN_THREADS) {
        double v = __ldcg(P.scratch + so + t);
#pragma unroll 8
        for (int i = 1; i < ni; ++i) v += __ldcg(P.scratch + so + (int64_t)i * RT + t);
        P.out[o_off + t] = accum ? __ldcg(P.out + o_off + t) + v : v;
    }
    __syncthreads();
    if (threadIdx.x == 0) P.arrivals[slot] = 0;
}

// One phase, one CTA per item.  CHAIN: launched with programmatic stream
// serialization - the kernel starts while its predecessor drains, reads its
// descriptor and indices and prefetches its matrix chunk into L2, then
// waits (griddepcontrol.wait) before it touches the input vector; the
// dependent launch is released at the CTA's start.
template <bool CHAIN>
__global__ void __launch_bounds__(PAN_THREADS, GC_PAN_MINB) k_panelmv(PanelPhase P) {
    __shared__ PanelSmem sm;
    if (CHAIN) asm volatile("griddepcontrol.launch_dependents;");
    trace_begin(P);
    panel_item<CHAIN>(P, blockIdx.x, sm);
    trace_end(P);
}

// Two small whole panels per CTA: threads [0,128) run item 2b, [128,256)
// item 2b+1, each half with the k_panelmv mapping over 128 threads (same
// per-output summation order as k_panelmv at 128 threads).  For the latency-
// bound tier phases whose panels are small (the lowest forward tier, the
// leaf rows): half as many CTAs, so about half the waves of per-CTA round
// trips.  Items must be direct (no split), T <= 128, nrows <= PAIR_MAX_ROWS.
constexpr int PAIR_THREADS = PAN_THREADS / 2;
constexpr int PAIR_MAX_ROWS = PAN_MAX_ROWS / 2;
#ifndef GC_PAIR_UNROLL
#define GC_PAIR_UNROLL 8
#endif
#ifndef GC_PAIR_MINB
#define GC_PAIR_MINB 6
#endif
constexpr int PAIR_UNROLL = GC_PAIR_UNROLL;

template <bool CHAIN>
__global__ void __launch_bounds__(PAN_THREADS, GC_PAIR_MINB) k_panel_pair(PanelPhase P) {
    __shared__ PanelSmem sm;                       // xs / red split in halves
    if (CHAIN) asm volatile("griddepcontrol.launch_dependents;");
    trace_begin(P);
    const int half = threadIdx.x / PAIR_THREADS, ltid = threadIdx.x % PAIR_THREADS;
    const int64_t item = 2 * (int64_t)blockIdx.x + half;
    const bool has = item < P.nitems;
    double* xs = sm.xs + half * PAIR_MAX_ROWS;
    double* red = sm.red + half * PAIR_THREADS;
    const int64_t* it = P.items + 8 * (has ? item : 0);
    const int64_t a_off = it[0], xi_off = it[1], out_off = it[2];
    const int T = has ? (int)it[3] : 1, nrows = has ? (int)it[4] : 0, mode = (int)it[5];
    const double* __restrict__ A = ((mode & 1) ? P.A1 : P.A0) + a_off;
    const int32_t* __restrict__ xi = P.xidx + xi_off;
    if (CHAIN) {
        if (has) prefetch_l2(A, 8 * (int64_t)nrows * T);
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (mode & 32) {
        for (int r = ltid; r < nrows; r += PAIR_THREADS) {
            const int i = __ldg(xi + r);
            xs[r] = __ldcg(P.in0 + i) + __ldcg(P.in1 + i);
        }
    } else {
        const double* x = (mode & 2) ? P.in1 : P.in0;
        for (int r = ltid; r < nrows; r += PAIR_THREADS) xs[r] = __ldcg(x + __ldg(xi + r));
    }
    __syncthreads();
    const int tt = T < PAIR_THREADS ? T : PAIR_THREADS;
    const int ng = PAIR_THREADS / tt;
    const int g = ltid / tt;
    const int t = ltid % tt;
    double acc = 0.0;
    if (has && g < ng) {
        const double* __restrict__ At = A + t;
        int r = g;
        for (; r + (PAIR_UNROLL - 1) * ng < nrows; r += PAIR_UNROLL * ng) {
            double a[PAIR_UNROLL];
#pragma unroll
            for (int j = 0; j < PAIR_UNROLL; ++j) a[j] = __ldcs(At + (int64_t)(r + j * ng) * T);
            __syncwarp(__activemask());                                  // pins the batch (see panel_item)
#pragma unroll
            for (int j = 0; j < PAIR_UNROLL; ++j) acc = fma(a[j], xs[r + j * ng], acc);
        }
        for (; r < nrows; r += ng) acc = fma(__ldcs(At + (int64_t)r * T), xs[r], acc);
    }
    red[ltid] = acc;
    __syncthreads();
    if (has && ltid < tt) {
        double v = red[ltid];
        for (int q = 1; q < ng; ++q) v += red[q * tt + ltid];
        double* o = P.out + out_off + t;
        *o = (mode & 8) ? __ldcg(o) + v : v;
    }
    trace_end(P);
}

// ---------------------------------------------------------------------------
// Bulk phases (coupling buckets, near field): one CTA per item as in
// k_panelmv, but the item's matrix streams through a 2-stage shared-memory
// ring filled by 1-D TMA bulk copies (cp.async.bulk, completion on one
// mbarrier per stage).  Thread 0 issues the first two 16 KB chunks before
// the index -> input gather, so the matrix stream overlaps the item's
// prologue, and the bytes in flight (32 KB per CTA) do not cost registers.
// Thread (g, t) sums the same rows in the same order as k_panelmv: the
// results are bitwise identical.  Requires T <= PAN_THREADS; every matrix
// buffer must be readable 16 bytes past its end (device.padded_empty).
constexpr int RING_STAGES = 2;
constexpr int RING_ELEMS = 2048;                  // 16 KB per stage

struct RingSmem {
    double stage[RING_STAGES][RING_ELEMS + 2];    // + 16-byte alignment slack
    double red[PAN_THREADS];
    double xs[PAN_MAX_ROWS];
    unsigned long long full[RING_STAGES];
    int last;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void ring_issue(RingSmem& sm, int st, const double* A, int c, int rps, int nrows,
                                           int T) {
    const int r0 = c * rps;
    const int nr = min(rps, nrows - r0);
    const uintptr_t sa = reinterpret_cast<uintptr_t>(A + (int64_t)r0 * T);
    const unsigned lead = (unsigned)((sa & 15) >> 3);
    const unsigned bytes = ((unsigned)(nr * T + (int)lead) * 8u + 15u) & ~15u;
    const uint32_t bar = smem_u32(&sm.full[st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(sm.stage[st])), "l"(sa & ~uintptr_t(15)), "r"(bytes), "r"(bar) : "memory");
}

__device__ __forceinline__ void ring_wait(RingSmem& sm, int st, unsigned parity) {
    const uint32_t bar = smem_u32(&sm.full[st]);
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    }
}

__global__ void __launch_bounds__(PAN_THREADS, 4) k_panel_ring(PanelPhase P) {
    extern __shared__ __align__(128) unsigned char ring_raw[];
    RingSmem& sm = *reinterpret_cast<RingSmem*>(ring_raw);
    trace_begin(P);
    const int64_t* it = P.items + 8 * (int64_t)blockIdx.x;
    const int64_t a_off = it[0], xi_off = it[1], out_off = it[2];
    const int T = (int)it[3], nrows = (int)it[4], mode = (int)it[5];
    const double* __restrict__ A = ((mode & 1) ? P.A1 : P.A0) + a_off;
    const int rps = RING_ELEMS / T;
    const int nch = (nrows + rps - 1) / rps;
    if (threadIdx.x == 0) {
        for (int st = 0; st < RING_STAGES; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.full[st])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int c = 0; c < RING_STAGES && c < nch; ++c) ring_issue(sm, c, A, c, rps, nrows, T);
    }
    const int32_t* __restrict__ xi = P.xidx + xi_off;
    if (mode & 32) {
        for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) {
            const int i = __ldg(xi + r);
            sm.xs[r] = __ldcg(P.in0 + i) + __ldcg(P.in1 + i);
        }
    } else {
        const double* x = (mode & 2) ? P.in1 : P.in0;
        for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) sm.xs[r] = __ldcg(x + __ldg(xi + r));
    }
    __syncthreads();
    const int tt = T;                                      // T <= PAN_THREADS
    const int ng = PAN_THREADS / tt;
    const int g = threadIdx.x / tt, t = threadIdx.x % tt;
    const bool live = g < ng;
    double acc = 0.0;
    for (int c = 0; c < nch; ++c) {
        const int st = c % RING_STAGES;
        ring_wait(sm, st, (unsigned)(c / RING_STAGES) & 1u);
        const int r0 = c * rps;
        const int nr = min(rps, nrows - r0);
        const double* sa = sm.stage[st] + ((reinterpret_cast<uintptr_t>(A + (int64_t)r0 * T) & 15) >> 3);
        if (live) {
            int r = ((g - r0 % ng) % ng + ng) % ng;
            const double* pa = sa + r * T + t;
            const double* px = sm.xs + r0 + r;
            const int sa_step = ng * T;
            for (; r + 3 * ng < nr; r += 4 * ng) {
                acc = fma(pa[0], px[0], acc);
                acc = fma(pa[sa_step], px[ng], acc);
                acc = fma(pa[2 * sa_step], px[2 * ng], acc);
                acc = fma(pa[3 * sa_step], px[3 * ng], acc);
                pa += 4 * sa_step;
                px += 4 * ng;
            }
            for (; r < nr; r += ng) {
                acc = fma(pa[0], px[0], acc);
                pa += sa_step;
                px += ng;
            }
        }
        __syncthreads();                                   // stage st consumed
        if (threadIdx.x == 0 && c + RING_STAGES < nch) ring_issue(sm, st, A, c + RING_STAGES, rps, nrows, T);
    }
    sm.red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < tt) {
        double s = sm.red[threadIdx.x];
        for (int q = 1; q < ng; ++q) s += sm.red[q * tt + threadIdx.x];
        if (mode & 4) {
            double* o = P.out + out_off + t;
            *o = (mode & 8) ? __ldcg(o) + s : s;
        } else {
            P.scratch[out_off + t] = s;
        }
    }
    if (!(mode & 4)) {
        // split panel: the last arriving item adds the partial sums in item order
        const int slot = (int)it[6];
        const int64_t* rd = P.red + 5 * (int64_t)slot;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) sm.last = atomicAdd(P.arrivals + slot, 1) == (int)rd[3] - 1;
        __syncthreads();
        if (sm.last) {
            __threadfence();
            const int64_t o_off = rd[0], so = rd[2];
            const int RT = (int)rd[1], ni = (int)rd[3];
            const bool accum = rd[4] != 0;
            for (int tq = threadIdx.x; tq < RT; tq += PAN_THREADS) {
                double v = __ldcg(P.scratch + so + tq);
#pragma unroll 8
                for (int i = 1; i < ni; ++i) v += __ldcg(P.scratch + so + (int64_t)i * RT + tq);
                P.out[o_off + tq] = accum ? __ldcg(P.out + o_off + tq) + v : v;
            }
            __syncthreads();
            if (threadIdx.x == 0) P.arrivals[slot] = 0;
        }
    }
    trace_end(P);
}

}  // namespace gcb

using namespace gcb;

static int check_phase(int64_t nitems, int64_t nred, const int64_t* red, const int32_t* arrivals) {
    if (nitems > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "too many work items"); return GC_ERR_CONFIG; }
    if (nred > 0 && (red == nullptr || arrivals == nullptr)) {
        set_error(GC_ERR_CONFIG, "gc_panelmv: split panels need red and arrivals");
        return GC_ERR_CONFIG;
    }
    return GC_OK;
}

extern "C" int gc_panelmv(int64_t nitems, const int64_t* items, const int32_t* xidx,
                          const double* A0, const double* A1, const double* in0,
                          const double* in1, double* out, double* scratch, int64_t nred,
                          const int64_t* red, int32_t* arrivals, int32_t chain, int32_t priority,
                          uint64_t* trace, void* stream) {
    using namespace gcb;
    if (nitems <= 0) return GC_OK;
    if (int rc = check_phase(nitems, nred, red, arrivals)) return rc;
    const PanelPhase P{items, nitems, xidx, A0, A1, in0, in1, out, scratch, red, arrivals,
                       (unsigned long long*)trace};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nitems);
    cfg.blockDim = dim3(PAN_THREADS);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (chain & 3) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (priority != 0) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na].val.priority = priority;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e;
    if (chain & 32) {
        // bulk phase on the TMA ring kernel (items with T <= 256)
        int dev = 0;
        e = cudaGetDevice(&dev);
        if (e == cudaSuccess)     // function attributes are per device context: set on every launch
            e = cudaFuncSetAttribute(k_panel_ring, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(RingSmem));
        if (e != cudaSuccess) return cuda_status(e, "k_panel_ring smem attribute");
        cfg.dynamicSmemBytes = sizeof(RingSmem);
        e = cudaLaunchKernelEx(&cfg, k_panel_ring, P);
    } else if (chain & 16) {
        // two whole small panels per CTA (direct items, T <= 128, <= 512 rows)
        cfg.gridDim = dim3((unsigned)((nitems + 1) / 2));
        e = (chain & 3) ? cudaLaunchKernelEx(&cfg, k_panel_pair<true>, P)
                        : cudaLaunchKernelEx(&cfg, k_panel_pair<false>, P);
    } else {
        e = (chain & 1) ? cudaLaunchKernelEx(&cfg, k_panelmv<true>, P)
                        : cudaLaunchKernelEx(&cfg, k_panelmv<false>, P);
    }
    if (e != cudaSuccess) return cuda_status(e, "k_panelmv");
    count_launch();
    return GC_OK;
}

extern "C" int gc_priority_range(int32_t* least, int32_t* greatest) {
    using namespace gcb;
    int l = 0, g = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&l, &g);
    if (e != cudaSuccess) return cuda_status(e, "gc_priority_range");
    *least = l;
    *greatest = g;
    return GC_OK;
}
