// Read bandwidth of 1-D TMA bulk copies (cp.async.bulk global -> shared,
// mbarrier completion) against plain 8-byte streaming loads, on random
// (incompressible) data: each CTA streams its contiguous chunk through a
// ring of S stages of B bytes, consumer threads sum every element.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe scripts/tma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_fill(double* a, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t h = i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 32;
        a[i] = (double)(h >> 11) * 0x1.0p-53 - 0.5;
    }
}

template <int U>
__global__ void k_chunk(const double* __restrict__ a, size_t chunk, double* out) {
    const double* p = a + blockIdx.x * chunk;
    double acc = 0;
    size_t i = threadIdx.x;
    for (; i + (U - 1) * blockDim.x < chunk; i += U * blockDim.x) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    for (; i < chunk; i += blockDim.x) acc += __ldcs(p + i);
    if (acc == 1.2345) out[0] = acc;
}

// S stages of B bytes; thread 0 produces, all threads consume
__global__ void k_tma(const double* __restrict__ a, size_t chunk, int S, int B, double* out, int skew) {
    extern __shared__ __align__(128) unsigned char raw[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(raw);
    double* ring = reinterpret_cast<double*>(raw + 128);
    const int E = B / 8;
    // skew: chunks start 16 bytes past an 8 KB-aligned address and are 16
    // bytes shorter than the stage (the layout of the matvec's work items)
    const double* p = a + blockIdx.x * chunk + 2 * skew;
    const int nch = (int)(chunk / E) - 1;
    const unsigned Bc = B - 16 * skew;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + s)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int c) {
        const int s = c % S;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(Bc) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(ring + (size_t)s * E)), "l"(p + (size_t)c * E), "r"(Bc), "r"(su32(full + s)) : "memory");
    };
    if (threadIdx.x == 0)
        for (int c = 0; c < S && c < nch; ++c) issue(c);
    double acc = 0;
    for (int c = 0; c < nch; ++c) {
        const int s = c % S;
        const unsigned par = (c / S) & 1;
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0,1,0,q;\n}\n"
                         : "=r"(done) : "r"(su32(full + s)), "r"(par) : "memory");
        for (int i = threadIdx.x; i < E; i += blockDim.x) acc += ring[(size_t)s * E + i];
        __syncthreads();
        if (threadIdx.x == 0 && c + S < nch) issue(c + S);
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    const size_t bytes = 1ull << 30, n = bytes / 8;
    double *a, *out;
    cudaMalloc(&a, bytes + 4096);
    cudaMalloc(&out, 8);
    k_fill<<<4096, 256>>>(a, n);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(e0);
        const int R = 10;
        for (int r = 0; r < R; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t e = cudaGetLastError();
        printf("%-40s %7.0f GB/s %s\n", name, bytes * (double)R / (ms * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
    };
    for (int ctas : {148 * 4, 148 * 64}) {
        size_t chunk = n / ctas;
        char nm[64];
        snprintf(nm, 64, "ldcs U8 256thr ctas %d", ctas);
        run(nm, [&] { k_chunk<8><<<ctas, 256>>>(a, chunk, out); });
    }
    for (int skew : {0, 1, 3})
    for (int S : {2, 4, 6}) {
        for (int B : {8192, 16384}) {
            const int smem = 128 + S * B;
            if (smem > 220 * 1024) continue;
            cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            int per = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tma, 128, smem);
            for (int mult : {1}) {
                int ctas = 148 * per * mult;
                size_t chunk = n / ctas;
                chunk -= chunk % (B / 8);
                char nm[64];
                snprintf(nm, 64, "tma skew %d S%d B%d per_sm %d ctas %d", skew, S, B, per, ctas);
                run(nm, [&] { k_tma<<<ctas, 128, smem>>>(a, chunk, S, B, out, skew); });
            }
        }
    }
    return 0;
}
