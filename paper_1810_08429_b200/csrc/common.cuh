// Shared device helpers and the error / launch-accounting plumbing of the
// C-ABI library (include/gcb200.h).  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/gcb200.h"

namespace gcb {

// 1/(4 pi) and 4 pi exactly as numpy forms them (4.0 * np.pi)
constexpr double FOUR_PI = 12.566370614359172;
constexpr double INV_FOUR_PI = 0.07957747154594767;

// ---- status plumbing -------------------------------------------------------
void set_error(int code, const char* fmt, ...);
int cuda_status(cudaError_t err, const char* what);
void count_launch(int n = 1);

#define GC_CHECK_LAUNCH(what)                                              \
    do {                                                                   \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return ::gcb::cuda_status(_e, what);        \
        ::gcb::count_launch();                                             \
    } while (0)

// device-side error flags (bit 0: geometry touch guard, bit 1: queue overflow)
constexpr int FLAG_TOUCH = 1;
constexpr int FLAG_OVERFLOW = 2;

// ---- fast FP64 reciprocal square root -------------------------------------
// MUFU-based approximation refined by one Newton step with the cubic term:
// y1 = y0 (1 + e/2 + 3e^2/8), e = 1 - x y0^2.  With |e| ~ 2^-21 the
// truncation error is ~e^3 < 2^-62: full double accuracy (<= 1-2 ulp) for
// 5 FP64 instructions plus one MUFU.
__device__ __forceinline__ double rsqrt_fast(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double t = x * y;
    double e = fma(-t, y, 1.0);
    double p = fma(e, 0.375, 0.5);
    return fma(y * e, p, y);
}

// r^3 rounded once (double-double product then one rounding): matches the
// correctly rounded cube, which agrees with numpy's SIMD r**3 in ~95% of
// cases and is never more than 1 ulp away from it.
__device__ __forceinline__ double cube_rn(double r) {
    double p = __dmul_rn(r, r);
    double pe = fma(r, r, -p);
    double hi = __dmul_rn(p, r);
    double lo = fma(p, r, -hi);
    lo = fma(pe, r, lo);
    return __dadd_rn(hi, lo);
}

// permutation table PERMS3 (quadrature.py:26-31 / quadrature.PERMS3)
__device__ __constant__ static const int8_t kPerms3[6][3] = {
    {0, 1, 2}, {1, 2, 0}, {2, 0, 1}, {0, 2, 1}, {2, 1, 0}, {1, 0, 2}};
__device__ __constant__ static const int8_t kPermId[3][3] = {
    // kPermId[a][b]: id of the permutation starting (a, b, 3-a-b)
    {-1, 0, 3}, {5, -1, 1}, {2, 4, -1}};

// Classification of one triangle pair by shared vertex ids: case code
// 0 disjoint / 1 vertex / 2 edge / 3 identical and the alignment
// permutation ids (same rules as quadrature.classify_pairs).
__device__ __forceinline__ int classify_pair(const int64_t* tv, const int64_t* sv,
                                             int* px, int* py) {
    int rhit = 0, chit = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            if (tv[a] == sv[b]) { rhit |= 1 << a; chit |= 1 << b; }
    int shared = __popc(rhit);
    *px = 0; *py = 0;
    if (shared == 1) {
        *px = __ffs(rhit) - 1;
        *py = __ffs(chit) - 1;
    } else if (shared == 2) {
        // rotation putting the shared edge in slots 0, 1 (register selects:
        // no dynamically indexed local arrays)
        const int missing = __ffs(~rhit & 7) - 1;
        const int rot = (missing + 1) % 3;
        *px = rot;
        const int64_t g0 = rot == 0 ? tv[0] : (rot == 1 ? tv[1] : tv[2]);
        const int64_t g1 = rot == 0 ? tv[1] : (rot == 1 ? tv[2] : tv[0]);
        const int c0 = (sv[0] == g0) ? 0 : (sv[1] == g0 ? 1 : 2);
        const int c1 = (sv[0] == g1) ? 0 : (sv[1] == g1 ? 1 : 2);
        // id of the permutation (c0, c1, 3-c0-c1): see kPermId
        *py = c0 == 0 ? (c1 == 1 ? 0 : 3) : (c0 == 1 ? (c1 == 2 ? 1 : 5) : (c1 == 0 ? 2 : 4));
    }
    return shared;
}

}  // namespace gcb
