// Read-bandwidth ceiling on this GPU for the access shapes of the matvec:
// grid-stride streaming vs one contiguous chunk per CTA (the panel kernel's
// shape), plain 8-byte loads vs 16-byte vector loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe scripts/bw_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_stride(const double* __restrict__ a, size_t n, double* out) {
    double acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc += __ldcs(a + i);
    if (acc == 1.2345) out[0] = acc;
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

template <int U>
__global__ void k_chunk2(const double2* __restrict__ a, size_t chunk2, double* out) {
    const double2* p = a + blockIdx.x * chunk2;
    double acc = 0;
    size_t i = threadIdx.x;
    for (; i + (U - 1) * blockDim.x < chunk2; i += U * blockDim.x) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    const size_t bytes = 1ull << 30, n = bytes / 8;
    double *a, *out;
    cudaMalloc(&a, bytes);
    cudaMalloc(&out, 8);
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(e0);
        const int R = 20;
        for (int r = 0; r < R; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %8.1f GB/s\n", name, bytes * (double)R / (ms * 1e-3) / 1e9);
    };
    run("grid-stride 148x8x256", [&] { k_stride<<<148 * 8, 256>>>(a, n, out); });
    run("grid-stride 148x16x128", [&] { k_stride<<<148 * 16, 128>>>(a, n, out); });
    for (size_t kb : {16, 32, 64, 128, 256}) {
        const size_t chunk = kb * 1024 / 8;
        char name[64];
        snprintf(name, 64, "chunk %zu KB / CTA, U8", kb);
        run(name, [&] { k_chunk<8><<<(unsigned)(n / chunk), 256>>>(a, chunk, out); });
        snprintf(name, 64, "chunk %zu KB / CTA, U16", kb);
        run(name, [&] { k_chunk<16><<<(unsigned)(n / chunk), 256>>>(a, chunk, out); });
        snprintf(name, 64, "chunk %zu KB / CTA, double2 U8", kb);
        run(name, [&] { k_chunk2<8><<<(unsigned)(n / chunk), 256>>>((const double2*)a, chunk / 2, out); });
    }
    cudaError_t err = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
