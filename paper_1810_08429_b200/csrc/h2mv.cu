// Segmented block-row products: the one kernel form behind every H2 matvec
// phase (h2.py:19-80) - forward transform (V^T x, V-hat^T x-hat), coupling
// (S x-hat), backward transform (E y-hat) and the near-field SpMV (N x).
//
// Matrices are stored so that the product reads contiguous rows of A
// (out[t] += sum_k A[k*lda + t] in[k]): a group of T threads covers the T
// outputs of a segment and streams one row of A per step with coalesced
// loads; ng = 256/T groups split the k range round-robin and are summed in
// group order at the end, so every output has exactly one writer and a
// fixed summation order (bitwise deterministic, no atomics).
#include "common.cuh"

namespace gcb {

constexpr int SEG_THREADS = 256;

__global__ void __launch_bounds__(SEG_THREADS) k_segmv(const int64_t* __restrict__ seg,
                                                       const int64_t* __restrict__ blk,
                                                       const double* __restrict__ A0,
                                                       const double* __restrict__ A1,
                                                       const double* __restrict__ in0,
                                                       const double* __restrict__ in1,
                                                       double* __restrict__ out, int accumulate) {
    __shared__ double red[SEG_THREADS];
    const int64_t* sd = seg + 4 * (int64_t)blockIdx.x;
    const int64_t out_off = sd[0];
    const int T = (int)sd[1];
    const int64_t b0 = sd[2], b1 = sd[3];
    const int tt = T < SEG_THREADS ? T : SEG_THREADS;   // threads per group
    const int ng = SEG_THREADS / tt;                     // groups
    const int g = threadIdx.x / tt;
    for (int t0 = 0; t0 < T; t0 += tt) {
        const int t = t0 + (int)(threadIdx.x % tt);
        const bool live = g < ng && t < T;
        double acc = 0.0;
        if (live) {
            for (int64_t b = b0; b < b1; ++b) {
                const int64_t* bd = blk + 6 * b;
                const int64_t a_off = bd[0], K = bd[1], lda = bd[2], in_off = bd[3];
                const int sel = (int)bd[4];
                const double* A = ((sel & 1) ? A1 : A0) + a_off + t * bd[5];
                const double* x = ((sel & 2) ? in1 : in0) + in_off;
                int64_t k = g;
                for (; k + 3 * ng < K; k += 4 * ng) {
                    const double a0 = __ldg(A + k * lda), a1 = __ldg(A + (k + ng) * lda);
                    const double a2 = __ldg(A + (k + 2 * ng) * lda), a3 = __ldg(A + (k + 3 * ng) * lda);
                    const double x0 = __ldg(x + k), x1 = __ldg(x + k + ng);
                    const double x2 = __ldg(x + k + 2 * ng), x3 = __ldg(x + k + 3 * ng);
                    acc = fma(a0, x0, acc);
                    acc = fma(a1, x1, acc);
                    acc = fma(a2, x2, acc);
                    acc = fma(a3, x3, acc);
                }
                for (; k < K; k += ng) acc = fma(__ldg(A + k * lda), __ldg(x + k), acc);
            }
        }
        if (ng == 1) {
            if (live) {
                double* o = out + out_off + t;
                *o = accumulate ? *o + acc : acc;
            }
            continue;
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < tt && t < T) {
            double s = red[threadIdx.x];
            for (int q = 1; q < ng; ++q) s += red[q * tt + threadIdx.x];
            double* o = out + out_off + t;
            *o = accumulate ? *o + s : s;
        }
        __syncthreads();
    }
}

}  // namespace gcb

using namespace gcb;

extern "C" int gc_segmv(int64_t nseg, const int64_t* seg, const int64_t* blk, const double* A0,
                        const double* A1, const double* in0, const double* in1, double* out,
                        int accumulate, int64_t max_T, void* stream) {
    (void)max_T;
    if (nseg <= 0) return GC_OK;
    if (nseg > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "too many segments"); return GC_ERR_CONFIG; }
    k_segmv<<<(unsigned)nseg, SEG_THREADS, 0, (cudaStream_t)stream>>>(seg, blk, A0, A1, in0, in1,
                                                                      out, accumulate);
    GC_CHECK_LAUNCH("k_segmv");
    return GC_OK;
}

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
// streaming loop over A has no dependent loads: 16 independent 8-byte loads
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

__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(127);
    const uintptr_t hi = reinterpret_cast<uintptr_t>(p) + bytes;
    for (uintptr_t l = lo + 128 * threadIdx.x; l < hi; l += 128 * PAN_THREADS)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
}

__device__ __forceinline__ void prefetch_item(const PanelPhase& P, int64_t i) {
    const int64_t* it = P.items + 8 * i;
    const double* A = ((it[5] & 1) ? P.A1 : P.A0) + it[0];
    prefetch_l2(A, 8 * it[3] * it[4]);
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
        // bulk: start the item's matrix stream (L2 prefetch of the whole
        // chunk) before the dependent index -> input gather
        if (mode & 16) prefetch_l2(A, 8 * (int64_t)nrows * T);
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
// waits (griddepcontrol.wait) before it touches the input vector.
// TRIGGER 1: the dependent launch is released at the CTA's start (its CTAs
// then wait on SM slots); 2: after the CTA's item is done (the dependent
// only overlaps this kernel's drain and keeps its slots free for the bulk).
template <bool CHAIN, int TRIGGER>
__global__ void __launch_bounds__(PAN_THREADS, GC_PAN_MINB) k_panelmv(PanelPhase P) {
    __shared__ PanelSmem sm;
    if (CHAIN && TRIGGER == 1) asm volatile("griddepcontrol.launch_dependents;");
    if (P.trace != nullptr && threadIdx.x == 0) atomicMin(P.trace, globaltimer());
    panel_item<CHAIN>(P, blockIdx.x, sm);
    if (CHAIN && TRIGGER == 2) asm volatile("griddepcontrol.launch_dependents;");
    if (P.trace != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(P.trace + 1, globaltimer());
    }
}

// Two small whole panels per CTA: threads [0,128) run item 2b, [128,256)
// item 2b+1, each half with the k_panelmv mapping over 128 threads (same
// per-output summation order as k_panelmv at 128 threads).  For the latency-
// bound tier phases whose panels are small (the lowest forward tier, the
// leaf rows): half as many CTAs, so about half the waves of per-CTA round
// trips.  Items must be direct (no split), T <= 128, nrows <= PAIR_MAX_ROWS.
constexpr int PAIR_THREADS = PAN_THREADS / 2;
constexpr int PAIR_MAX_ROWS = PAN_MAX_ROWS / 2;

template <bool CHAIN>
__global__ void __launch_bounds__(PAN_THREADS, 6) k_panel_pair(PanelPhase P) {
    __shared__ PanelSmem sm;                       // xs / red split in halves
    if (CHAIN) asm volatile("griddepcontrol.launch_dependents;");
    if (P.trace != nullptr && threadIdx.x == 0) atomicMin(P.trace, globaltimer());
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
        for (; r + (PAN_UNROLL - 1) * ng < nrows; r += PAN_UNROLL * ng) {
            double a[PAN_UNROLL];
#pragma unroll
            for (int j = 0; j < PAN_UNROLL; ++j) a[j] = __ldcs(At + (int64_t)(r + j * ng) * T);
#pragma unroll
            for (int j = 0; j < PAN_UNROLL; ++j) acc = fma(a[j], xs[r + j * ng], acc);
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
    if (P.trace != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(P.trace + 1, globaltimer());
    }
}

// ---------------------------------------------------------------------------
// Bulk phases (coupling buckets, near field): a TMA-fed streaming kernel.
// A co-resident grid (2 CTAs per SM); CTA b owns the items
// [cta_begin[b], cta_begin[b+1]) (equal bytes per CTA, set on the host).
// One producer thread streams each item's matrix rows into a 4-stage
// shared-memory ring with cp.async.bulk (row-aligned chunks of <= 16 KB,
// completion counted on an mbarrier); 8 consumer warps gather the item's
// input entries, wait for a stage, FMA it against them and release the
// stage.  DRAM sees one long stream of 16 KB bulk reads per CTA with up to
// 64 KB in flight, independent of the consumers' gather/reduce latency.
// Summation order is fixed by (item, chunk, row group): deterministic.
// Every matrix buffer must be readable 16 bytes past its last element (the
// bulk copies are widened to 16-byte boundaries).
constexpr int ST_STAGES = 4;
constexpr int ST_ELEMS = 2048;                 // 16 KB of matrix per stage
constexpr int ST_PAD = 4;                      // 16-byte widening slack (doubles)
constexpr int ST_CONSUMERS = 256;
constexpr int ST_THREADS = ST_CONSUMERS + 32;  // + 1 producer warp
constexpr int ST_MAX_T = 1024;                 // 4 outputs per consumer thread

struct StreamSmem {
    double stage[ST_STAGES][ST_ELEMS + ST_PAD];
    double xs[PAN_MAX_ROWS];
    double red[ST_CONSUMERS];
    unsigned long long full[ST_STAGES];
    unsigned long long empty[ST_STAGES];
    int last;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    const uint32_t a = smem_u32(b);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done) : "r"(a), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(ST_CONSUMERS) : "memory");
}

__global__ void __launch_bounds__(ST_THREADS) k_panel_stream(PanelPhase P, const int64_t* __restrict__ cta_begin) {
    extern __shared__ __align__(128) unsigned char st_raw[];
    StreamSmem& sm = *reinterpret_cast<StreamSmem*>(st_raw);
    const int tid = threadIdx.x;
    const int64_t beg = cta_begin[blockIdx.x], end = cta_begin[blockIdx.x + 1];
    if (tid == 0) {
        for (int s = 0; s < ST_STAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], ST_CONSUMERS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (P.trace != nullptr && tid == 0) atomicMin(P.trace, globaltimer());
    if (tid >= ST_CONSUMERS) {
        // producer: one lane streams every chunk of every owned item
        if (tid == ST_CONSUMERS) {
            int stage = 0;
            unsigned phase = 0;
            for (int64_t i = beg; i < end; ++i) {
                const int64_t* it = P.items + 8 * i;
                const int T = (int)it[3], nrows = (int)it[4], mode = (int)it[5];
                const double* A = ((mode & 1) ? P.A1 : P.A0) + it[0];
                const int rc = ST_ELEMS / T;
                for (int r0 = 0; r0 < nrows; r0 += rc) {
                    const int rows = min(rc, nrows - r0);
                    const uintptr_t src = reinterpret_cast<uintptr_t>(A + (int64_t)r0 * T);
                    const uintptr_t al = src & ~uintptr_t(15);
                    const unsigned bytes = (unsigned)(((src - al) + (uintptr_t)rows * T * 8 + 15) & ~uintptr_t(15));
                    mbar_wait(&sm.empty[stage], phase ^ 1);
                    mbar_expect_tx(&sm.full[stage], bytes);
                    bulk_g2s(sm.stage[stage], reinterpret_cast<const void*>(al), bytes, &sm.full[stage]);
                    if (++stage == ST_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
        return;
    }
    // consumers
    const int lane = tid & 31;
    int stage = 0;
    unsigned phase = 0;
    for (int64_t i = beg; i < end; ++i) {
        const int64_t* it = P.items + 8 * i;
        const int64_t out_off = it[2];
        const int T = (int)it[3], nrows = (int)it[4], mode = (int)it[5];
        const double* A = ((mode & 1) ? P.A1 : P.A0) + it[0];
        const double* x = (mode & 2) ? P.in1 : P.in0;
        const int32_t* __restrict__ xi = P.xidx + it[1];
        consumers_sync();                                     // xs / red free
        for (int r = tid; r < nrows; r += ST_CONSUMERS) sm.xs[r] = __ldcg(x + __ldg(xi + r));
        consumers_sync();
        const int tt = T < ST_CONSUMERS ? T : ST_CONSUMERS;
        const int ng = ST_CONSUMERS / tt;
        const int g = tid / tt, tl = tid - g * tt;
        const int J = (T + ST_CONSUMERS - 1) / ST_CONSUMERS;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const int rc = ST_ELEMS / T;
        for (int r0 = 0; r0 < nrows; r0 += rc) {
            const int rows = min(rc, nrows - r0);
            const uintptr_t src = reinterpret_cast<uintptr_t>(A + (int64_t)r0 * T);
            const int lead = (int)((src & 15) >> 3);
            mbar_wait(&sm.full[stage], phase);
            const double* C = sm.stage[stage] + lead;
            const double* xr = sm.xs + r0;
            if (g < ng) {
                if (J == 1) {
                    double a0 = 0.0, a1 = 0.0;
                    int lr = g;
                    for (; lr + ng < rows; lr += 2 * ng) {
                        a0 = fma(C[lr * T + tl], xr[lr], a0);
                        a1 = fma(C[(lr + ng) * T + tl], xr[lr + ng], a1);
                    }
                    if (lr < rows) a0 = fma(C[lr * T + tl], xr[lr], a0);
                    acc[0] += a0 + a1;
                } else {
                    for (int lr = 0; lr < rows; ++lr) {
                        const double xv = xr[lr];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int t = tl + ST_CONSUMERS * j;
                            if (j < J && t < T) acc[j] = fma(C[lr * T + t], xv, acc[j]);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[stage]);
            if (++stage == ST_STAGES) { stage = 0; phase ^= 1; }
        }
        double* dst = (mode & 4) ? P.out + out_off : P.scratch + out_off;
        const bool add = (mode & 12) == 12;
        if (J == 1) {
            sm.red[tid] = acc[0];
            consumers_sync();
            if (tid < T) {
                double s = sm.red[tid];
                for (int q = 1; q < ng; ++q) s += sm.red[q * T + tid];
                dst[tid] = add ? __ldcg(dst + tid) + s : s;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int t = tl + ST_CONSUMERS * j;
                if (j < J && t < T) dst[t] = add ? __ldcg(dst + t) + acc[j] : acc[j];
            }
        }
        if (mode & 4) continue;
        // split panel: the last CTA to finish adds the partial sums in item order
        const int slot = (int)it[6];
        const int64_t* rd = P.red + 5 * (int64_t)slot;
        __threadfence();
        consumers_sync();
        if (tid == 0) sm.last = atomicAdd(P.arrivals + slot, 1) == (int)rd[3] - 1;
        consumers_sync();
        if (!sm.last) continue;
        __threadfence();
        const int64_t o_off = rd[0], so = rd[2];
        const int RT = (int)rd[1], ni = (int)rd[3];
        const bool accum = rd[4] != 0;
        for (int t = tid; t < RT; t += ST_CONSUMERS) {
            double v = __ldcg(P.scratch + so + t);
            for (int k = 1; k < ni; ++k) v += __ldcg(P.scratch + so + (int64_t)k * RT + t);
            P.out[o_off + t] = accum ? __ldcg(P.out + o_off + t) + v : v;
        }
        consumers_sync();
        if (tid == 0) P.arrivals[slot] = 0;
    }
    if (P.trace != nullptr) {
        consumers_sync();
        if (tid == 0) atomicMax(P.trace + 1, globaltimer());
    }
}

// ---------------------------------------------------------------------------
// Bulk phases, one CTA per item, TMA-fed: thread 0 launches ONE cp.async.bulk
// of the item's whole contiguous matrix chunk (<= TMA_ITEM_ELEMS doubles)
// into shared memory, tracked by an mbarrier, and the CTA gathers the
// item's input entries while the bytes are in flight; then it computes
// from shared memory.  Every CTA puts its whole item in flight at once and
// the hardware scheduler keeps 3 CTAs per SM streaming (the index -> input
// gather no longer serialises with the matrix stream).
constexpr int TMA_ITEM_ELEMS = 7168;            // 56 KB per item: 3 CTAs per SM

struct TmaSmem {
    double a[TMA_ITEM_ELEMS + ST_PAD];
    double xs[PAN_MAX_ROWS];
    double red[PAN_THREADS];
    unsigned long long full;
    int last;
};

__global__ void __launch_bounds__(PAN_THREADS) k_panel_tma(PanelPhase P) {
    extern __shared__ __align__(128) unsigned char tma_raw[];
    TmaSmem& sm = *reinterpret_cast<TmaSmem*>(tma_raw);
    const int tid = threadIdx.x;
    const int64_t* it = P.items + 8 * (int64_t)blockIdx.x;
    const int64_t a_off = it[0], xi_off = it[1], out_off = it[2];
    const int T = (int)it[3], nrows = (int)it[4], mode = (int)it[5];
    const double* A = ((mode & 1) ? P.A1 : P.A0) + a_off;
    const uintptr_t src = reinterpret_cast<uintptr_t>(A);
    const uintptr_t al = src & ~uintptr_t(15);
    const int lead = (int)((src - al) >> 3);
    if (tid == 0) {
        if (P.trace != nullptr) atomicMin(P.trace, globaltimer());
        mbar_init(&sm.full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const unsigned bytes = (unsigned)(((src - al) + (uintptr_t)nrows * T * 8 + 15) & ~uintptr_t(15));
        mbar_expect_tx(&sm.full, bytes);
        bulk_g2s(sm.a, reinterpret_cast<const void*>(al), bytes, &sm.full);
    }
    const double* x = (mode & 2) ? P.in1 : P.in0;
    const int32_t* __restrict__ xi = P.xidx + xi_off;
    for (int r = tid; r < nrows; r += PAN_THREADS) sm.xs[r] = __ldcg(x + __ldg(xi + r));
    __syncthreads();                                  // xs ready, barrier initialised
    mbar_wait(&sm.full, 0);
    const double* C = sm.a + lead;
    const int tt = T < PAN_THREADS ? T : PAN_THREADS;
    const int ng = PAN_THREADS / tt;
    const int g = tid / tt;
    for (int t0 = 0; t0 < T; t0 += tt) {
        const int t = t0 + (tid % tt);
        double acc = 0.0;
        if (g < ng && t < T) {
            double a1 = 0.0;
            int r = g;
            for (; r + ng < nrows; r += 2 * ng) {
                acc = fma(C[r * T + t], sm.xs[r], acc);
                a1 = fma(C[(r + ng) * T + t], sm.xs[r + ng], a1);
            }
            if (r < nrows) acc = fma(C[r * T + t], sm.xs[r], acc);
            acc += a1;
        }
        sm.red[tid] = acc;
        __syncthreads();
        if (tid < tt && t < T) {
            double s = sm.red[tid];
            for (int q = 1; q < ng; ++q) s += sm.red[q * tt + tid];
            if (mode & 4) {
                double* o = P.out + out_off + t;
                *o = (mode & 8) ? __ldcg(o) + s : s;
            } else {
                P.scratch[out_off + t] = s;
            }
        }
        __syncthreads();
    }
    if (!(mode & 4)) {
        const int slot = (int)it[6];
        const int64_t* rd = P.red + 5 * (int64_t)slot;
        __threadfence();
        __syncthreads();
        if (tid == 0) sm.last = atomicAdd(P.arrivals + slot, 1) == (int)rd[3] - 1;
        __syncthreads();
        if (sm.last) {
            __threadfence();
            const int64_t o_off = rd[0], so = rd[2];
            const int RT = (int)rd[1], ni = (int)rd[3];
            const bool accum = rd[4] != 0;
            for (int t = tid; t < RT; t += PAN_THREADS) {
                double v = __ldcg(P.scratch + so + t);
                for (int k = 1; k < ni; ++k) v += __ldcg(P.scratch + so + (int64_t)k * RT + t);
                P.out[o_off + t] = accum ? __ldcg(P.out + o_off + t) + v : v;
            }
            __syncthreads();
            if (tid == 0) P.arrivals[slot] = 0;
        }
    }
    if (P.trace != nullptr) {
        __syncthreads();
        if (tid == 0) atomicMax(P.trace + 1, globaltimer());
    }
}

// Grid-wide barrier (co-resident grid): every CTA adds 1 except CTA 0,
// which adds 2^31 - (nb - 1), so each barrier flips bit 31 of the counter
// and the counter never needs re-arming between launches.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nb = gridDim.x;
        const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (nb - 1) : 1u;
        __threadfence();
        const unsigned old = atomicAdd(bar, inc);
        unsigned cur;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
    }
    __syncthreads();
}

// Warp-granular item (the chain's levels are too small to give every CTA
// an item: a level has ~10^3 items of a few KB, so one warp owns one item
// and a CTA works 8 items at once).  Lane l owns outputs t = t0 + l + 32 j,
// j < J, and runs the rows of the item in order (fixed summation order).
constexpr int WARP_MAX_ROWS = 256;

template <int J>
__device__ __forceinline__ void warp_rows(const double* __restrict__ A, int T, int t0, int nrows,
                                          const double* xs, int lane, double* acc) {
    constexpr int U = 16 / J;                     // rows in flight
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] = 0.0;
    const int tl = t0 + lane;
    int r = 0;
    for (; r + U <= nrows; r += U) {
        double a[U][J];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int t = tl + 32 * j;
                a[u][j] = t < T ? __ldcs(A + (int64_t)(r + u) * T + t) : 0.0;
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < J; ++j) acc[j] = fma(a[u][j], xs[r + u], acc[j]);
    }
    for (; r < nrows; ++r)
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int t = tl + 32 * j;
            if (t < T) acc[j] = fma(__ldcs(A + (int64_t)r * T + t), xs[r], acc[j]);
        }
}

__device__ void warp_item(const PanelPhase& P, int64_t item, double* xs, int lane) {
    const int64_t* it = P.items + 8 * item;
    const int64_t a_off = it[0], xi_off = it[1], out_off = it[2];
    const int T = (int)it[3], nrows = (int)it[4], mode = (int)it[5];
    const double* __restrict__ A = ((mode & 1) ? P.A1 : P.A0) + a_off;
    const double* x = (mode & 2) ? P.in1 : P.in0;
    const int32_t* __restrict__ xi = P.xidx + xi_off;
    if (mode & 32) {
        for (int r = lane; r < nrows; r += 32) {
            const int i = __ldg(xi + r);
            xs[r] = __ldcg(P.in0 + i) + __ldcg(P.in1 + i);
        }
    } else {
        for (int r = lane; r < nrows; r += 32) xs[r] = __ldcg(x + __ldg(xi + r));
    }
    __syncwarp();
    double* dst = (mode & 4) ? P.out + out_off : P.scratch + out_off;
    for (int t0 = 0; t0 < T; t0 += 256) {
        const int span = T - t0;
        double acc[8];
        if (span > 128) warp_rows<8>(A, T, t0, nrows, xs, lane, acc);
        else if (span > 64) warp_rows<4>(A, T, t0, nrows, xs, lane, acc);
        else if (span > 32) warp_rows<2>(A, T, t0, nrows, xs, lane, acc);
        else warp_rows<1>(A, T, t0, nrows, xs, lane, acc);
        const int J = span > 128 ? 8 : span > 64 ? 4 : span > 32 ? 2 : 1;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int t = t0 + lane + 32 * j;
            if (j < J && t < T) dst[t] = (mode & 12) == 12 ? __ldcg(dst + t) + acc[j] : acc[j];
        }
    }
    __syncwarp();
    if (mode & 4) return;
    const int slot = (int)it[6];
    const int64_t* rd = P.red + 5 * (int64_t)slot;
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicAdd(P.arrivals + slot, 1) == (int)rd[3] - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
    const int64_t o_off = rd[0], so = rd[2];
    const int RT = (int)rd[1], ni = (int)rd[3];
    const bool accum = rd[4] != 0;
    for (int t = lane; t < RT; t += 32) {
        double v = __ldcg(P.scratch + so + t);
        for (int i = 1; i < ni; ++i) v += __ldcg(P.scratch + so + (int64_t)i * RT + t);
        P.out[o_off + t] = accum ? __ldcg(P.out + o_off + t) + v : v;
    }
    __syncwarp();
    if (lane == 0) P.arrivals[slot] = 0;
}

// One warp per item (a whole small panel: the many tiny panels of the
// lower transform levels - leaf bases of 16 rows, sibling transfers): 8
// items per CTA instead of one, so a level of 2048 panels is 256 CTAs.
// CHAIN: programmatic dependent launch as in k_panelmv.
template <bool CHAIN>
__global__ void __launch_bounds__(PAN_THREADS) k_panel_warp(PanelPhase P) {
    __shared__ double xs[PAN_THREADS / 32][WARP_MAX_ROWS];
    if (CHAIN) asm volatile("griddepcontrol.launch_dependents;");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t item = (int64_t)blockIdx.x * (PAN_THREADS / 32) + warp;
    if (P.trace != nullptr && threadIdx.x == 0) atomicMin(P.trace, globaltimer());
    if (CHAIN) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (item < P.nitems) warp_item(P, item, xs[warp], lane);
    if (P.trace != nullptr) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(P.trace + 1, globaltimer());
    }
}

// A run of consecutive chain phases (transform levels) in ONE co-resident
// launch: warps stride over each phase's items, prefetch their items of
// the next phase into L2, and the grid meets at a barrier between phases.
__global__ void __launch_bounds__(PAN_THREADS) k_panel_chain(const PanelPhase* __restrict__ phases,
                                                             int nphase, unsigned* bar) {
    __shared__ double xs[PAN_THREADS / 32][WARP_MAX_ROWS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (PAN_THREADS / 32) + warp;
    const int64_t nw = (int64_t)gridDim.x * (PAN_THREADS / 32);
    for (int ph = 0; ph < nphase; ++ph) {
        const PanelPhase P = phases[ph];
        for (int64_t i = gw; i < P.nitems; i += nw) warp_item(P, i, xs[warp], lane);
        if (ph + 1 < nphase) {
            const PanelPhase& Q = phases[ph + 1];
            for (int64_t i = gw; i < Q.nitems; i += nw) {
                const int64_t* it = Q.items + 8 * i;
                const double* A = ((it[5] & 1) ? Q.A1 : Q.A0) + it[0];
                const uintptr_t lo = reinterpret_cast<uintptr_t>(A) & ~uintptr_t(127);
                const uintptr_t hi = reinterpret_cast<uintptr_t>(A + it[3] * it[4]);
                for (uintptr_t l = lo + 128 * lane; l < hi; l += 128 * 32)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
            }
            grid_barrier(bar);
        }
    }
}

}  // namespace gcb

// the persistent chain kernel carries the device's highest scheduling
// priority, so its CTAs are dispatched ahead of the queued bulk phases
static int top_priority() {
    int least = 0, greatest = 0;
    if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return 0;
    return greatest;
}

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
    if (chain & 16) {
        // two whole small panels per CTA (direct items, T <= 128, <= 512 rows)
        cfg.gridDim = dim3((unsigned)((nitems + 1) / 2));
        e = (chain & 3) ? cudaLaunchKernelEx(&cfg, k_panel_pair<true>, P)
                        : cudaLaunchKernelEx(&cfg, k_panel_pair<false>, P);
    } else if (chain & 4) {
        // warp-granular items (whole panels of <= WARP_MAX_ROWS rows)
        cfg.gridDim = dim3((unsigned)((nitems + PAN_THREADS / 32 - 1) / (PAN_THREADS / 32)));
        e = (chain & 3) ? cudaLaunchKernelEx(&cfg, k_panel_warp<true>, P)
                        : cudaLaunchKernelEx(&cfg, k_panel_warp<false>, P);
    } else {
        e = chain == 1   ? cudaLaunchKernelEx(&cfg, k_panelmv<true, 1>, P)
          : chain == 2 ? cudaLaunchKernelEx(&cfg, k_panelmv<true, 2>, P)
                       : cudaLaunchKernelEx(&cfg, k_panelmv<false, 0>, P);
    }
    if (e != cudaSuccess) return cuda_status(e, "k_panelmv");
    count_launch();
    return GC_OK;
}

extern "C" int gc_panel_chain_grid(int64_t* grid) {
    using namespace gcb;
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_panel_chain, PAN_THREADS, 0);
    if (e != cudaSuccess) return cuda_status(e, "gc_panel_chain_grid");
    // two CTAs per SM: enough memory parallelism for the small transform
    // levels, and room left on every SM for the concurrent bulk phases
    *grid = (int64_t)sms * (per_sm < 2 ? per_sm : 2);
    return GC_OK;
}

extern "C" int gc_panel_chain(int64_t nphase, const void* phases, int64_t grid, uint32_t* barrier,
                              void* stream) {
    using namespace gcb;
    if (nphase <= 0) return GC_OK;
    if (grid <= 0 || barrier == nullptr) { set_error(GC_ERR_CONFIG, "gc_panel_chain: bad grid"); return GC_ERR_CONFIG; }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(PAN_THREADS);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributePriority;
    attr[1].val.priority = top_priority();
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_panel_chain, (const PanelPhase*)phases, (int)nphase,
                                       (unsigned*)barrier);
    if (e != cudaSuccess) return cuda_status(e, "k_panel_chain");
    count_launch();
    return GC_OK;
}

extern "C" int64_t gc_panel_phase_bytes(void) { return (int64_t)sizeof(gcb::PanelPhase); }

extern "C" int gc_priority_range(int32_t* least, int32_t* greatest) {
    using namespace gcb;
    int l = 0, g = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&l, &g);
    if (e != cudaSuccess) return cuda_status(e, "gc_priority_range");
    *least = l;
    *greatest = g;
    return GC_OK;
}

extern "C" int gc_panel_stream_grid(int64_t* grid) {
    using namespace gcb;
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_panel_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(StreamSmem));
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_panel_stream, ST_THREADS, sizeof(StreamSmem));
    if (e != cudaSuccess) return cuda_status(e, "gc_panel_stream_grid");
    *grid = (int64_t)sms * (per_sm < 2 ? per_sm : 2);
    return GC_OK;
}

extern "C" int gc_panel_stream(int64_t nitems, const int64_t* items, const int32_t* xidx,
                               const double* A0, const double* A1, const double* in0,
                               const double* in1, double* out, double* scratch, int64_t nred,
                               const int64_t* red, int32_t* arrivals, const int64_t* cta_begin,
                               int64_t grid, int32_t priority, uint64_t* trace, void* stream) {
    using namespace gcb;
    if (nitems <= 0) return GC_OK;
    if (int rc = check_phase(nitems, nred, red, arrivals)) return rc;
    if (grid <= 0 || cta_begin == nullptr) { set_error(GC_ERR_CONFIG, "gc_panel_stream: bad grid"); return GC_ERR_CONFIG; }
    const PanelPhase P{items, nitems, xidx, A0, A1, in0, in1, out, scratch, red, arrivals,
                       (unsigned long long*)trace};
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_panel_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(StreamSmem));
        if (e != cudaSuccess) return cuda_status(e, "k_panel_stream smem attribute");
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(ST_THREADS);
    cfg.dynamicSmemBytes = sizeof(StreamSmem);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (priority != 0) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na].val.priority = priority;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_panel_stream, P, cta_begin);
    if (e != cudaSuccess) return cuda_status(e, "k_panel_stream");
    count_launch();
    return GC_OK;
}

extern "C" int gc_panel_tma(int64_t nitems, const int64_t* items, const int32_t* xidx,
                            const double* A0, const double* A1, const double* in0,
                            const double* in1, double* out, double* scratch, int64_t nred,
                            const int64_t* red, int32_t* arrivals, int32_t priority, uint64_t* trace,
                            void* stream) {
    using namespace gcb;
    if (nitems <= 0) return GC_OK;
    if (int rc = check_phase(nitems, nred, red, arrivals)) return rc;
    const PanelPhase P{items, nitems, xidx, A0, A1, in0, in1, out, scratch, red, arrivals,
                       (unsigned long long*)trace};
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_panel_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(TmaSmem));
        if (e != cudaSuccess) return cuda_status(e, "k_panel_tma smem attribute");
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nitems);
    cfg.blockDim = dim3(PAN_THREADS);
    cfg.dynamicSmemBytes = sizeof(TmaSmem);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (priority != 0) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na].val.priority = priority;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_panel_tma, P);
    if (e != cudaSuccess) return cuda_status(e, "k_panel_tma");
    count_launch();
    return GC_OK;
}

extern "C" int64_t gc_panel_tma_item_elems(void) { return gcb::TMA_ITEM_ELEMS; }
