// Micro-benchmark (debug aid): latency of one chol_diag_warp call (32 x 32 diagonal block factor +
// inverse) on one warp, in SM cycles (clock64) and ns (globaltimer).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o diag_bench diag_bench.cu
#include <cstdio>
#include "../../paper_2003_02978_b200/csrc/kernels.cuh"
#include "../../paper_2003_02978_b200/csrc/wide_chol.cuh"
using namespace smf;
__global__ void bench(double* A, int B, long long* out) {
    __shared__ double D[kChB * kChD], Dinv[kChB * kChD];
    int ok = 1;
    long long t0 = clock64(), g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const int reps = 50;
    for (int r = 0; r < reps; ++r) ok &= chol_diag_warp(A, B, 0, 32, 1e-30, D, Dinv);
    long long t1 = clock64(), g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / reps; out[1] = (g1 - g0) / reps; out[2] = ok; }
}
int main() {
    const int B = 32;
    double h[B * B];
    for (int i = 0; i < B; ++i)
        for (int j = 0; j < B; ++j) h[i * B + j] = (i == j ? B + 1.0 : 1.0 / (1 + i + j));
    double* A; long long* o;
    cudaMalloc(&A, sizeof(h)); cudaMalloc(&o, 24);
    cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int it = 0; it < 3; ++it) bench<<<1, 32>>>(A, B, o);
    long long r[3];
    cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost);
    printf("chol_diag_warp 32x32: %lld clock64 ticks, %lld ns per call (ok=%lld)\n", r[0], r[1], r[2]);
    return 0;
}
