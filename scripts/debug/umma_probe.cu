// Minimal tcgen05 kind::tf32 probe: D[128 x 16] = A[128 x 8] . B[16 x 8]^T with
// operands written by threads in one of several smem layouts; checks the
// result against the CPU. variant: 0 = TMEM st/ld roundtrip, 1 = MN-major SW64,
// 2 = K-major no swizzle, 3 = MN-major SW128, 4 = K-major SW32.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_2003_02978_b200/csrc/ptx.cuh"
using namespace smf;

__device__ float Aval(int m, int k) { return (float)((m * 3 + k * 7) % 11) - 5.f; }
__device__ float Bval(int n, int k) { return (float)((n * 5 + k * 3) % 7) - 3.f; }

__global__ void probe(int variant, float* out, uint32_t* info) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    unsigned char* A = base;             // 32 KB region
    unsigned char* Bm = base + 32768;    // 32 KB region
    __shared__ uint64_t bar;
    __shared__ uint32_t tsh;
    int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 65536 / 4; i += blockDim.x) ((float*)base)[i] = 0.f;
    __syncthreads();
    // write operands: element (mn, k)
    auto put = [&](unsigned char* R, int mn, int k, float v) {
        uint32_t off;
        if (variant == 1) {          // MN-major SW64: chunk = mn/16 (stride 4096), row k at 64 B, swizzle
            uint32_t slot = ((mn % 16) / 4) ^ ((k >> 1) & 3);
            off = (mn / 16) * 4096 + k * 64 + slot * 16 + (mn % 4) * 4;
        } else if (variant == 3) {   // MN-major SW128: chunk = mn/32 (stride 8192), row k at 128 B
            uint32_t slot = ((mn % 32) / 4) ^ (k & 7);
            off = (mn / 32) * 8192 + k * 128 + slot * 16 + (mn % 4) * 4;
        } else if (variant == 2) {   // K-major interleave: core matrix (8 mn rows x 16 B) = 128 B;
            // K chunk (4 elts) stride LBO = 128 B, mn group of 8 stride SBO = 256 B
            off = (mn / 8) * 256 + (k / 4) * 128 + (mn % 8) * 16 + (k % 4) * 4;
        } else if (variant == 5) {   // K-major SW128: rows of 128 B (32 tf32 along K), 8-row atoms 1024 B
            uint32_t o = mn * 128 + (k / 4) * 16;
            o ^= ((o >> 7) & 7) << 4;
            off = o + (k % 4) * 4;
        } else {                     // K-major SW32: rows of 32 B (8 tf32 along K), mn rows stride 32 B,
            // 8-row atoms of 256 B, SBO = 256
            uint32_t o = mn * 32 + (k / 4) * 16;
            o ^= ((o >> 7) & 1) << 4;
            off = o + (k % 4) * 4;
        }
        *(float*)(R + off) = v;
    };
    if (variant > 0) {
        const int KK = variant == 5 ? 32 : 8;
        for (int i = tid; i < 128 * KK; i += blockDim.x) put(A, i / KK, i % KK, Aval(i / KK, i % KK));
        for (int i = tid; i < 16 * KK; i += blockDim.x) put(Bm, i / KK, i % KK, Bval(i / KK, i % KK));
    }
    fence_proxy_async();
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (wid == 0) tmem_alloc(&tsh, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tm = tsh;
    if (tid == 0) info[0] = tm;
    if (variant == 0) {
        // each warp stores 16 columns of its lane quarter then loads them back
        uint32_t r[16];
        for (int j = 0; j < 16; ++j) r[j] = __float_as_uint((float)(tid * 100 + j));
        uint32_t a = tm + ((uint32_t)(32 * wid) << 16);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                     "tcgen05.wait::st.sync.aligned;\n" :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                     "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
    } else if (tid == 0) {
        uint32_t sa = smem_u32(A), sb = smem_u32(Bm);
        uint64_t da, db;
        if (variant == 1) { da = umma_desc(sa, 4096, 512, 4); db = umma_desc(sb, 4096, 512, 4); }
        else if (variant == 3) { da = umma_desc(sa, 8192, 1024, 2); db = umma_desc(sb, 8192, 1024, 2); }
        else if (variant == 2) { da = umma_desc(sa, 128, 256, 0); db = umma_desc(sb, 128, 256, 0); }
        else if (variant == 5) { da = umma_desc(sa, 16, 1024, 2); db = umma_desc(sb, 16, 1024, 2); }
        else { da = umma_desc(sa, 0, 256, 6); db = umma_desc(sb, 0, 256, 6); }
        uint32_t amaj = (variant == 1 || variant == 3) ? 1u : 0u;
        uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (amaj << 15) | (amaj << 16) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
        info[1] = idesc; info[2] = (uint32_t)da; info[3] = (uint32_t)(da >> 32);
        if (variant == 5) {
            for (int ks = 0; ks < 4; ++ks)
                mma_tf32(tm, umma_desc(sa + ks * 32, 16, 1024, 2), umma_desc(sb + ks * 32, 16, 1024, 2), idesc, ks > 0);
        } else
            mma_tf32(tm, da, db, idesc, 0u);
        mma_commit(&bar);
    }
    if (variant > 0) mbar_wait(&bar, 0);
    tc_fence_after();
    {
        float v[16], u[16];
        tmem_ld16x2(tm + ((uint32_t)(32 * wid) << 16), tm + ((uint32_t)(32 * wid) << 16) + 16, v, u);
        for (int j = 0; j < 16; ++j) out[tid * 16 + j] = v[j];
    }
    tc_fence_before();
    __syncthreads();
    if (wid == 0) { tc_fence_after(); tmem_dealloc(tm, 32); }
}

int main() {
    float* d; uint32_t* inf;
    cudaMalloc(&d, 128 * 16 * 4); cudaMalloc(&inf, 64);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    for (int variant = 0; variant <= 5; ++variant) {
        cudaMemset(d, 0, 128 * 16 * 4);
        probe<<<1, 128, 70000>>>(variant, d, inf);
        cudaError_t e = cudaDeviceSynchronize();
        float h[128 * 16]; uint32_t hi[4];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        cudaMemcpy(hi, inf, 16, cudaMemcpyDeviceToHost);
        double err = 0; int nz = 0;
        for (int m = 0; m < 128; ++m) for (int n = 0; n < 16; ++n) {
            double ref = 0;
            if (variant == 0) ref = m * 100 + n;
            else for (int k = 0; k < (variant == 5 ? 32 : 8); ++k) ref += (double)(((m * 3 + k * 7) % 11) - 5) * (double)(((n * 5 + k * 3) % 7) - 3);
            err = fmax(err, fabs(h[m * 16 + n] - ref)); nz += h[m * 16 + n] != 0.f;
        }
        printf("variant %d: %s tmem=%u idesc=%08x desc=%08x%08x max err %g nonzero %d | D[0][0..3] %g %g %g %g\n", variant,
               cudaGetErrorString(e), hi[0], hi[1], hi[3], hi[2], err, nz, h[0], h[1], h[2], h[3]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
