// Device-side Krylov iteration around the H2 matvec (SURVEY §8f rank 3,
// the consumers of h2.py:190-253): conjugate-gradient vector updates with
// the scalars kept in device memory, and a deterministic dot product
// (fixed grid, fixed per-thread order, fixed reduction tree), so a solve
// is bitwise reproducible and the only host traffic per iteration is the
// residual norm read for the stopping test.
#include "common.cuh"

namespace gcb {

constexpr int KR_THREADS = 256;
constexpr int KR_BLOCKS = 148 * 4;

// scalar slots of the CG state vector s[]
enum { S_RR = 0, S_PQ = 1, S_RRNEW = 2, S_BETA = 3, S_ALPHA = 4, S_STOP = 5, S_N = 8 };

__device__ __forceinline__ double block_sum(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
#pragma unroll
    for (int o = KR_THREADS / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// partial[b] = sum over this block's grid-stride elements of a*b
__global__ void __launch_bounds__(KR_THREADS) k_dot_partial(int64_t n, const double* __restrict__ a,
                                                            const double* __restrict__ b,
                                                            double* __restrict__ partial) {
    __shared__ double sh[KR_THREADS];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)KR_THREADS + threadIdx.x; i < n; i += (int64_t)KR_BLOCKS * KR_THREADS)
        acc = fma(a[i], b[i], acc);
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// out = sum of the KR_BLOCKS partials (fixed tree); mode 1 also forms the
// CG scalars beta = out / s[RR], s[RR] = out (after a step)
__global__ void __launch_bounds__(KR_THREADS) k_dot_final(const double* __restrict__ partial, double* s,
                                                          int slot, int mode) {
    __shared__ double sh[KR_THREADS];
    double acc = 0.0;
    for (int i = threadIdx.x; i < KR_BLOCKS; i += KR_THREADS) acc += partial[i];
    const double v = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        s[slot] = v;
        if (mode == 1) {
            const double rr = s[S_RR];
            s[S_BETA] = rr != 0.0 ? v / rr : 0.0;
            s[S_RR] = v;
        }
    }
}

// alpha = s[RR] / s[PQ]; x += alpha p; r -= alpha q; partial sums of r.r.
// pq <= 0 (not SPD along p) sets s[STOP] and leaves x, r unchanged.
__global__ void __launch_bounds__(KR_THREADS) k_cg_step(int64_t n, const double* s_in, double* __restrict__ x,
                                                        double* __restrict__ r, const double* __restrict__ p,
                                                        const double* __restrict__ q, double* __restrict__ partial,
                                                        double* s_out) {
    __shared__ double sh[KR_THREADS];
    const double pq = s_in[S_PQ];
    const bool stop = !(pq > 0.0);
    const double alpha = stop ? 0.0 : s_in[S_RR] / pq;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)KR_THREADS + threadIdx.x; i < n; i += (int64_t)KR_BLOCKS * KR_THREADS) {
        double ri = r[i];
        if (!stop) {
            x[i] = fma(alpha, p[i], x[i]);
            ri = fma(-alpha, q[i], ri);
            r[i] = ri;
        }
        acc = fma(ri, ri, acc);
    }
    const double v = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s_out[S_ALPHA] = alpha;
        s_out[S_STOP] = stop ? 1.0 : 0.0;
    }
}

// p = r + beta p
__global__ void __launch_bounds__(KR_THREADS) k_cg_dir(int64_t n, const double* __restrict__ s,
                                                       const double* __restrict__ r, double* __restrict__ p) {
    const double beta = s[S_BETA];
    for (int64_t i = blockIdx.x * (int64_t)KR_THREADS + threadIdx.x; i < n; i += (int64_t)KR_BLOCKS * KR_THREADS)
        p[i] = fma(beta, p[i], r[i]);
}

// CGNR step (h2.py:236-245): stop if q.q == 0, else alpha = s[0] / q.q,
// x += alpha p, r -= alpha q; partial sums of r.r
__global__ void __launch_bounds__(KR_THREADS) k_cgnr_step(int64_t n, double* s, double* __restrict__ x,
                                                          double* __restrict__ r, const double* __restrict__ p,
                                                          const double* __restrict__ q,
                                                          double* __restrict__ partial) {
    __shared__ double sh[KR_THREADS];
    const double qq = s[S_PQ];
    const bool stop = qq == 0.0;
    const double alpha = stop ? 0.0 : s[S_RR] / qq;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)KR_THREADS + threadIdx.x; i < n; i += (int64_t)KR_BLOCKS * KR_THREADS) {
        double ri = r[i];
        if (!stop) {
            x[i] = fma(alpha, p[i], x[i]);
            ri = fma(-alpha, q[i], ri);
            r[i] = ri;
        }
        acc = fma(ri, ri, acc);
    }
    const double v = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s[S_ALPHA] = alpha;
        s[S_STOP] = stop ? 1.0 : 0.0;
    }
}

// z /= sqrt(s[0])  (the power iteration's normalisation, h2.py:170-171)
__global__ void __launch_bounds__(KR_THREADS) k_scale_inv_norm(int64_t n, double* __restrict__ z,
                                                               const double* __restrict__ s) {
    const double nz = sqrt(s[0]);
    for (int64_t i = blockIdx.x * (int64_t)KR_THREADS + threadIdx.x; i < n; i += (int64_t)KR_BLOCKS * KR_THREADS)
        z[i] = z[i] / nz;
}

// b -= a
__global__ void __launch_bounds__(KR_THREADS) k_sub(int64_t n, const double* __restrict__ a,
                                                    double* __restrict__ b) {
    for (int64_t i = blockIdx.x * (int64_t)KR_THREADS + threadIdx.x; i < n; i += (int64_t)KR_BLOCKS * KR_THREADS)
        b[i] = b[i] - a[i];
}

}  // namespace gcb

using namespace gcb;

extern "C" int gc_dot(int64_t n, const double* a, const double* b, double* partial, double* out,
                      void* stream) {
    if (n < 0) { set_error(GC_ERR_CONFIG, "gc_dot: negative length"); return GC_ERR_CONFIG; }
    cudaStream_t st = (cudaStream_t)stream;
    k_dot_partial<<<KR_BLOCKS, KR_THREADS, 0, st>>>(n, a, b, partial);
    GC_CHECK_LAUNCH("k_dot_partial");
    k_dot_final<<<1, KR_THREADS, 0, st>>>(partial, out, 0, 0);
    GC_CHECK_LAUNCH("k_dot_final");
    return GC_OK;
}

extern "C" int gc_cg_pq(int64_t n, const double* p, const double* q, double* partial, double* s,
                        void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    k_dot_partial<<<KR_BLOCKS, KR_THREADS, 0, st>>>(n, p, q, partial);
    GC_CHECK_LAUNCH("k_dot_partial");
    k_dot_final<<<1, KR_THREADS, 0, st>>>(partial, s, S_PQ, 0);
    GC_CHECK_LAUNCH("k_dot_final");
    return GC_OK;
}

extern "C" int gc_cg_update(int64_t n, double* x, double* r, double* p, const double* q,
                            double* partial, double* s, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    k_cg_step<<<KR_BLOCKS, KR_THREADS, 0, st>>>(n, s, x, r, p, q, partial, s);
    GC_CHECK_LAUNCH("k_cg_step");
    k_dot_final<<<1, KR_THREADS, 0, st>>>(partial, s, S_RRNEW, 1);
    GC_CHECK_LAUNCH("k_dot_final");
    k_cg_dir<<<KR_BLOCKS, KR_THREADS, 0, st>>>(n, s, r, p);
    GC_CHECK_LAUNCH("k_cg_dir");
    return GC_OK;
}

extern "C" int64_t gc_krylov_partials(void) { return KR_BLOCKS; }

// CGNR (h2.py:222-253).  State s[]: [0] s.s, [1] q.q, [2] r.r, [3] beta,
// [4] new s.s, [5] stop flag.  gc_cgnr_step: q.q, then the x / r update and
// r.r; gc_cgnr_dir: new s.s, beta = new / s[0], p = s + beta p, s[0] = new.
extern "C" int gc_cgnr_step(int64_t n, double* x, double* r, const double* p, const double* q,
                            double* partial, double* s, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    k_dot_partial<<<KR_BLOCKS, KR_THREADS, 0, st>>>(n, q, q, partial);
    GC_CHECK_LAUNCH("k_dot_partial");
    k_dot_final<<<1, KR_THREADS, 0, st>>>(partial, s, S_PQ, 0);
    GC_CHECK_LAUNCH("k_dot_final");
    k_cgnr_step<<<KR_BLOCKS, KR_THREADS, 0, st>>>(n, s, x, r, p, q, partial);
    GC_CHECK_LAUNCH("k_cgnr_step");
    k_dot_final<<<1, KR_THREADS, 0, st>>>(partial, s, S_RRNEW, 0);
    GC_CHECK_LAUNCH("k_dot_final");
    return GC_OK;
}

extern "C" int gc_cgnr_dir(int64_t n, const double* sv, double* p, double* partial, double* s, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    k_dot_partial<<<KR_BLOCKS, KR_THREADS, 0, st>>>(n, sv, sv, partial);
    GC_CHECK_LAUNCH("k_dot_partial");
    k_dot_final<<<1, KR_THREADS, 0, st>>>(partial, s, 4, 1);
    GC_CHECK_LAUNCH("k_dot_final");
    k_cg_dir<<<KR_BLOCKS, KR_THREADS, 0, st>>>(n, s, sv, p);
    GC_CHECK_LAUNCH("k_cg_dir");
    return GC_OK;
}

extern "C" int gc_scale_inv_norm(int64_t n, double* z, const double* s, void* stream) {
    k_scale_inv_norm<<<KR_BLOCKS, KR_THREADS, 0, (cudaStream_t)stream>>>(n, z, s);
    GC_CHECK_LAUNCH("k_scale_inv_norm");
    return GC_OK;
}

extern "C" int gc_axpy_neg(int64_t n, const double* a, double* b, void* stream) {
    k_sub<<<KR_BLOCKS, KR_THREADS, 0, (cudaStream_t)stream>>>(n, a, b);
    GC_CHECK_LAUNCH("k_sub");
    return GC_OK;
}
