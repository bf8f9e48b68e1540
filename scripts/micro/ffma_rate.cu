// Microbenchmark: sustained FFMA issue rate of an 8x8 register outer product on sm_100a.
// Variant A: operands in registers only (no smem). Variant B: with 4 LDS.128 per 64 FFMA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) outer_regs(float* out, int iters, float s) {
    float acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = 0.f;
    float xa[8], xb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { xa[i] = threadIdx.x * 0.001f + i; xb[i] = s * i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[i * 8 + k] = fmaf(xa[i], xb[k], acc[i * 8 + k]);
#pragma unroll
        for (int i = 0; i < 8; ++i) { xa[i] += 1e-7f; xb[i] -= 1e-7f; }
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 64; ++i) t += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void __launch_bounds__(256, 1) outer_smem(float* out, int iters, int stride) {
    __shared__ __align__(16) float buf[128 * 84];
    for (int i = threadIdx.x; i < 128 * 84; i += blockDim.x) buf[i] = i * 1e-4f;
    __syncthreads();
    float acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = 0.f;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int R = lane % 10, C = lane / 10;   // 4 x 10 pattern in a warp
    for (int it = 0; it < iters; ++it) {
        const int r = (it * 8 + w) & 127;
        const float4* row = reinterpret_cast<const float4*>(buf + r * 84);
        const float4 a0 = row[2 * R], a1 = row[2 * R + 1], b0 = row[2 * C], b1 = row[2 * C + 1];
        const float xa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float xb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[i * 8 + k] = fmaf(xa[i], xb[k], acc[i * 8 + k]);
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 64; ++i) t += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 4 * 256 * sizeof(float));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps = 4; warps <= 16; warps *= 2) {
        int threads = warps * 32, iters = 20000;
        outer_regs<<<sms, threads>>>(out, 10, 1.f);
        cudaEventRecord(a);
        outer_regs<<<sms, threads>>>(out, iters, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double fma = (double)sms * threads * iters * 64;
        printf("regs  warps/SM=%2d: %.2f TFMA/s = %.1f FMA/clk/SM at 1.965 GHz\n", warps, fma / ms / 1e9,
               fma / (ms * 1e-3) / sms / 1.965e9);
        outer_smem<<<sms, threads>>>(out, 10, 84);
        cudaEventRecord(a);
        outer_smem<<<sms, threads>>>(out, iters, 84);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("smem  warps/SM=%2d: %.2f TFMA/s = %.1f FMA/clk/SM\n", warps, fma / ms / 1e9,
               fma / (ms * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
