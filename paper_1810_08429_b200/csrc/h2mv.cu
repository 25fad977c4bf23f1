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
// and k_panel_reduce adds them in item order (bitwise deterministic).
namespace gcb {

constexpr int PAN_THREADS = 256;
constexpr int PAN_UNROLL = 16;
constexpr int PAN_MAX_ROWS = 1024;   // rows per work item (x gathered to smem)

// item: a_off, xi_off, out_off, T, nrows, mode (bit0 A1, bit1 in1,
//       bit2 direct to out, bit3 accumulate into out)
// The item's input entries are gathered into shared memory first, so the
// streaming loop over A has no dependent loads: 16 independent 8-byte loads
// per thread are in flight before the first FMA.
__global__ void __launch_bounds__(PAN_THREADS) k_panelmv(
    const int64_t* __restrict__ items, const int32_t* __restrict__ xidx,
    const double* __restrict__ A0, const double* __restrict__ A1,
    const double* __restrict__ in0, const double* __restrict__ in1,
    double* __restrict__ out, double* __restrict__ scratch) {
    __shared__ double red[PAN_THREADS];
    __shared__ double xs[PAN_MAX_ROWS];
    const int64_t* it = items + 6 * (int64_t)blockIdx.x;
    const int64_t a_off = it[0], xi_off = it[1], out_off = it[2];
    const int T = (int)it[3], nrows = (int)it[4], mode = (int)it[5];
    const double* __restrict__ A = ((mode & 1) ? A1 : A0) + a_off;
    const double* __restrict__ x = (mode & 2) ? in1 : in0;
    const int32_t* __restrict__ xi = xidx + xi_off;
    for (int r = threadIdx.x; r < nrows; r += PAN_THREADS) xs[r] = __ldg(x + __ldg(xi + r));
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
                for (int j = 0; j < PAN_UNROLL; ++j) acc = fma(a[j], xs[r + j * ng], acc);
            }
            for (; r < nrows; r += ng) acc = fma(__ldcs(At + (int64_t)r * T), xs[r], acc);
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < tt && t < T) {
            double s = red[threadIdx.x];
            for (int q = 1; q < ng; ++q) s += red[q * tt + threadIdx.x];
            if (mode & 4) {
                double* o = out + out_off + t;
                *o = (mode & 8) ? *o + s : s;
            } else {
                scratch[out_off + t] = s;
            }
        }
        __syncthreads();
    }
}

// red: out_off, T, scratch_off, nitems, accumulate
__global__ void k_panel_reduce(int64_t nred, const int64_t* __restrict__ red,
                               const double* __restrict__ scratch, double* __restrict__ out) {
    for (int64_t s = blockIdx.x; s < nred; s += gridDim.x) {
        const int64_t* r = red + 5 * s;
        const int64_t out_off = r[0], T = r[1], so = r[2], ni = r[3];
        const bool accum = r[4] != 0;
        for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
            double v = scratch[so + t];
            for (int64_t i = 1; i < ni; ++i) v += scratch[so + i * T + t];
            out[out_off + t] = accum ? out[out_off + t] + v : v;
        }
    }
}

}  // namespace gcb

extern "C" int gc_panelmv(int64_t nitems, const int64_t* items, const int32_t* xidx,
                          const double* A0, const double* A1, const double* in0,
                          const double* in1, double* out, double* scratch, int64_t nred,
                          const int64_t* red, void* stream) {
    using namespace gcb;
    if (nitems <= 0) return GC_OK;
    if (nitems > 0x7fffffffLL) { set_error(GC_ERR_CONFIG, "too many work items"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    k_panelmv<<<(unsigned)nitems, PAN_THREADS, 0, st>>>(items, xidx, A0, A1, in0, in1, out, scratch);
    GC_CHECK_LAUNCH("k_panelmv");
    if (nred > 0) {
        int64_t grid = nred < 148 * 16 ? nred : 148 * 16;
        k_panel_reduce<<<(unsigned)grid, 128, 0, st>>>(nred, red, scratch, out);
        GC_CHECK_LAUNCH("k_panel_reduce");
    }
    return GC_OK;
}
