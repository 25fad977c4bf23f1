/* The matvec hot kernel driven from C through the C-ABI only (no Python):
 * one panel product with gc_panelmv, then the same product captured and
 * replayed by the native executor (gc_plan_create / gc_plan_run), checked
 * against a plain C loop; then an NCCL communicator and all-gather through
 * gc_nccl_*.  Needs a GPU (tests/test_abi.py, -m gpu). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "gcb200.h"

#define K 300
#define T 48

int main(void) {
    double *hA = malloc(sizeof(double) * K * T), hx[K], ref[T], got[T];
    int32_t hidx[K];
    for (int i = 0; i < K * T; ++i) hA[i] = sin(0.37 * i);
    for (int k = 0; k < K; ++k) { hx[k] = cos(0.11 * k); hidx[k] = k; }
    for (int t = 0; t < T; ++t) {
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += hA[k * T + t] * hx[k];
        ref[t] = s;
    }
    /* one whole-panel item: a_off, xi_off, out_off, T, nrows, mode (4 = direct), red, 0 */
    int64_t item[8] = {0, 0, 0, T, K, 4, -1, 0};
    double *A, *x, *out, *scratch;
    int64_t *items;
    int32_t *xidx, *arrivals;
    cudaMalloc((void**)&A, sizeof(double) * K * T + 64);
    cudaMalloc((void**)&x, sizeof(double) * K);
    cudaMalloc((void**)&out, sizeof(double) * T);
    cudaMalloc((void**)&scratch, sizeof(double));
    cudaMalloc((void**)&items, sizeof(item));
    cudaMalloc((void**)&xidx, sizeof(hidx));
    cudaMalloc((void**)&arrivals, sizeof(int32_t));
    cudaMemcpy(A, hA, sizeof(double) * K * T, cudaMemcpyHostToDevice);
    cudaMemcpy(x, hx, sizeof(hx), cudaMemcpyHostToDevice);
    cudaMemcpy(items, item, sizeof(item), cudaMemcpyHostToDevice);
    cudaMemcpy(xidx, hidx, sizeof(hidx), cudaMemcpyHostToDevice);
    cudaMemset(arrivals, 0, sizeof(int32_t));
    if (gc_panelmv(1, items, xidx, A, NULL, x, NULL, out, scratch, 0, NULL, arrivals, 0, 0, NULL, NULL)) {
        printf("gc_panelmv: %s\n", gc_last_error());
        return 1;
    }
    cudaMemcpy(got, out, sizeof(got), cudaMemcpyDeviceToHost);
    double err = 0.0, nrm = 0.0;
    for (int t = 0; t < T; ++t) { err += (got[t] - ref[t]) * (got[t] - ref[t]); nrm += ref[t] * ref[t]; }
    if (!(sqrt(err) <= 1e-13 * sqrt(nrm))) { printf("panel mismatch %g\n", sqrt(err / nrm)); return 2; }
    /* the same product as a one-node plan on the native executor */
    cudaMemset(out, 0, sizeof(double) * T);
    int64_t node[18] = {0, 0, 0, 0, 0, 0,
                        (int64_t)(intptr_t)items, 1, (int64_t)(intptr_t)xidx, (int64_t)(intptr_t)A, 0,
                        (int64_t)(intptr_t)x, 0, (int64_t)(intptr_t)out, (int64_t)(intptr_t)scratch, 0, 0,
                        (int64_t)(intptr_t)arrivals};
    int64_t deps[1] = {0};
    int32_t prio[1] = {0};
    void* plan = NULL;
    if (gc_plan_create(1, node, 0, deps, 1, prio, &plan)) { printf("gc_plan_create: %s\n", gc_last_error()); return 3; }
    for (int rep = 0; rep < 3; ++rep)
        if (gc_plan_run(plan, NULL, NULL, NULL)) { printf("gc_plan_run: %s\n", gc_last_error()); return 4; }
    cudaDeviceSynchronize();
    double got2[T];
    cudaMemcpy(got2, out, sizeof(got2), cudaMemcpyDeviceToHost);
    for (int t = 0; t < T; ++t)
        if (got2[t] != got[t]) { printf("plan result differs at %d\n", t); return 5; }
    /* the synchronous host-vector call: a plan without gather / scatter
     * nodes must refuse host pointers */
    double* pin = NULL;
    cudaMallocHost((void**)&pin, sizeof(double) * (K + T));
    if (gc_plan_run_host(plan, hx, pin, K, pin + K, NULL) != GC_ERR_CONFIG) {
        printf("gc_plan_run_host accepted a plan without gather / scatter nodes\n");
        return 11;
    }
    cudaFreeHost(pin);
    gc_plan_destroy(plan);
    /* NCCL through the C-ABI (world of one): communicator from a unique id,
     * an in-place all-gather (send = the rank's own slot of recv) */
    char uid[128];
    void* comm = NULL;
    if (gc_nccl_unique_id(uid) || gc_nccl_comm_init(uid, 1, 0, &comm)) {
        printf("nccl init: %s\n", gc_last_error());
        return 8;
    }
    if (gc_nccl_all_gather(out, out, T, comm, NULL) || cudaDeviceSynchronize() != cudaSuccess) {
        printf("nccl all-gather: %s\n", gc_last_error());
        return 9;
    }
    double back[T];
    cudaMemcpy(back, out, sizeof(back), cudaMemcpyDeviceToHost);
    for (int t = 0; t < T; ++t)
        if (back[t] != got[t]) { printf("all-gather changed the data\n"); return 10; }
    gc_nccl_comm_destroy(comm);
    printf("C-ABI panel product ok (rel err %.1e)\n", sqrt(err / nrm));
    free(hA);
    return 0;
}
