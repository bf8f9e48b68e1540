// Microbenchmark: sustained read bandwidth from L2 (working set < 126 MB) vs HBM on B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) rd(const float4* __restrict__ p, size_t n, int reps, float* out) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            float4 v = __ldcg(p + i);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t maxb = (size_t)4 << 30;
    float4* buf;
    cudaMalloc(&buf, maxb);
    cudaMemset(buf, 0, maxb);
    float* out;
    cudaMalloc(&out, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    size_t sizes[] = {(size_t)16 << 20, (size_t)32 << 20, (size_t)48 << 20, (size_t)64 << 20, (size_t)96 << 20,
                      (size_t)128 << 20, (size_t)256 << 20, (size_t)4 << 30};
    for (size_t bytes : sizes) {
        size_t n = bytes / 16;
        int reps = (int)(((size_t)16 << 30) / bytes);
        if (reps < 2) reps = 2;
        rd<<<sms * 4, 512>>>(buf, n, 1, out);
        cudaEventRecord(a);
        rd<<<sms * 4, 512>>>(buf, n, reps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("working set %8.1f MB: %.2f TB/s\n", bytes / 1048576.0, (double)bytes * reps / (ms * 1e-3) / 1e12);
    }
    return 0;
}
