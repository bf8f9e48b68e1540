// Probe of k1_stats_tc on several long columns (pilot c = 0, ghat = 0, so x = L and
// rho = -1): per column, sym(P) summed over the CTA slots vs the fp64 sum of e e^T,
// e = [L, -1, 1, 0...]. Reports the worst rows. Built with -D knobs to bisect.
#define SMF_DEBUG_K1TC 1
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include <cstring>
#include <cudaTypedefs.h>
#include "../../paper_2003_02978_b200/csrc/kernels.cuh"
using namespace smf;

int main(int argc, char** argv) {
    constexpr int NQ = 18, B = 72;
    using K = K1TC<NQ>;
    const int N = argc > 1 ? atoi(argv[1]) : 20000, cols = argc > 2 ? atoi(argv[2]) : 4;
    const int G = argc > 3 ? atoi(argv[3]) : 148;
    std::vector<float> L((size_t)cols * N * B);
    std::mt19937 rng(7);
    std::uniform_real_distribution<float> U(0.5f, 1.5f);
    for (auto& x : L) x = U(rng);
    float *dL, *dpil, *dgh;
    double* dpart;
    cudaMalloc(&dL, L.size() * 4);
    cudaMemcpy(dL, L.data(), L.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&dpil, cols * B * 4); cudaMemset(dpil, 0, cols * B * 4);
    cudaMalloc(&dgh, cols * B * 4); cudaMemset(dgh, 0, cols * B * 4);
    const int BE = K::BE, tpc = (N + 63) / 64;
    const long long ttot = (long long)cols * tpc;
    int S = 1;
    for (int b = 0; b < G; ++b) { long long t0 = b * ttot / G, t1 = (b + 1) * ttot / G; if (t1 > t0) S = std::max(S, (int)((t1 - 1) / tpc - t0 / tpc + 1)); }
    size_t pb = (size_t)G * S * BE * BE * 8;
    cudaMalloc(&dpart, pb); cudaMemset(dpart, 0, pb);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap mm, tm; memset(&mm, 0, sizeof(mm)); memset(&tm, 0, sizeof(tm));
    cuuint64_t dims[3] = {(cuuint64_t)B, (cuuint64_t)N, (cuuint64_t)cols};
    cuuint64_t strides[2] = {(cuuint64_t)B * 4, (cuuint64_t)N * B * 4};
    cuuint32_t box[3] = {32, 64, 1}, box2[3] = {8, 64, 1}, es[3] = {1, 1, 1};
    enc(&mm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dL, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dL, dims, strides, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    double* ddbg; cudaMalloc(&ddbg, (size_t)G * 64 * 80 * 8); cudaMemset(ddbg, 0, (size_t)G * 64 * 80 * 8);
    StatsArgs a; a.dbg = ddbg;
    a.pil32 = dpil; a.ghat32 = dgh; a.part1 = dpart; a.cols = cols; a.N = N; a.B = B;
    a.tpc = tpc; a.G = G; a.S = S; a.ttot = ttot;
    cudaFuncSetAttribute(k1_stats_tc<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
    k1_stats_tc<NQ><<<G, K::NT, K::SMEM>>>(mm, tm, a);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s  (N %d cols %d G %d S %d RS %d flush %d)\n", cudaGetErrorString(e), N, cols, G, S, K::RS, kFlushTC);
    std::vector<double> P(pb / 8);
    cudaMemcpy(P.data(), dpart, pb, cudaMemcpyDeviceToHost);
    for (int c = 0; c < cols; ++c) {
        std::vector<double> Pc((size_t)BE * BE, 0.0), ref((size_t)BE * BE, 0.0);
        for (int b = 0; b < G; ++b) {
            long long t0 = b * ttot / G, t1 = (b + 1) * ttot / G;
            if (t1 <= t0) continue;
            int c0 = (int)(t0 / tpc), c1 = (int)((t1 - 1) / tpc);
            if (c < c0 || c > c1) continue;
            for (size_t k = 0; k < Pc.size(); ++k) Pc[k] += P[((size_t)b * S + (c - c0)) * BE * BE + k];
        }
        for (int p = 0; p < N; ++p) {
            double ev[96] = {0};
            for (int bb = 0; bb < B; ++bb) ev[bb] = L[((size_t)c * N + p) * B + bb];
            ev[B] = -1.0; ev[B + 1] = 1.0;
            for (int i = 0; i < B + 2; ++i) for (int k = 0; k < B + 2; ++k) ref[i * BE + k] += ev[i] * ev[k];
        }
        std::vector<double> rowerr(BE, 0.0);
        for (int i = 0; i < BE; ++i) for (int k = 0; k < BE; ++k) {
            double sy = 0.5 * (Pc[i * BE + k] + Pc[k * BE + i]);
            double d = fabs(sy - ref[i * BE + k]) / (fabs(ref[i * BE + k]) + 1e-30);
            if (ref[i * BE + k] != 0) rowerr[i] = fmax(rowerr[i], d);
        }
        printf("col %d rows with rel err > 1e-5:", c);
        double mx = 0;
        for (int i = 0; i < B + 2; ++i) { mx = fmax(mx, rowerr[i]); if (rowerr[i] > 1e-5) printf(" %d(%.1e)", i, rowerr[i]); }
        printf("   max %.2e\n", mx);
    }
    // per-CTA check of the emitted sym(P) against the host sum over the CTA's pixels
    int nbad = 0; double worst = 0;
    for (int b = 0; b < G; ++b) {
        long long t0 = b * ttot / G, t1 = (b + 1) * ttot / G;
        if (t1 <= t0) continue;
        int c0 = (int)(t0 / tpc);
        std::vector<double> ref2((size_t)BE * BE, 0.0);
        for (int sl = 0; sl < S; ++sl) {
            std::fill(ref2.begin(), ref2.end(), 0.0);
            bool any = false;
            for (long long t = t0; t < t1; ++t) {
                int c = (int)(t / tpc), tt = (int)(t % tpc);
                if (c - c0 != sl) continue;
                any = true;
                for (int r = 0; r < 64; ++r) { int p = tt * 64 + r; if (p >= N) continue;
                    double e[80] = {0}; for (int k = 0; k < B; ++k) e[k] = L[((size_t)c * N + p) * B + k]; e[B] = -1; e[B + 1] = 1;
                    for (int ii = 0; ii < B + 2; ++ii) for (int k = 0; k <= ii; ++k) ref2[ii * BE + k] += e[ii] * e[k]; }
            }
            if (!any) continue;
            const double* Pb = &P[((size_t)b * S + sl) * BE * BE];
            double w = 0; int wi = 0, wk = 0;
            for (int ii = 0; ii < B + 2; ++ii) for (int k = 0; k <= ii; ++k) {
                double sy = 0.5 * (Pb[ii * BE + k] + Pb[k * BE + ii]);
                double d = fabs(sy - ref2[ii * BE + k]) / fabs(ref2[ii * BE + k]);
                if (d > w) { w = d; wi = ii; wk = k; }
            }
            worst = fmax(worst, w);
            if (w > 1e-5 && nbad < 20) { printf("CTA %d slot %d (tiles %lld..%lld): worst rel %.2e at (%d,%d) got %.5f exp %.5f\n", b, sl, t0, t1 - 1, w, wi, wk,
                0.5 * (Pb[wi * BE + wk] + Pb[wk * BE + wi]), ref2[wi * BE + wk]); ++nbad; }
        }
    }
    printf("per-CTA worst rel %.2e, bad CTAs %d\n", worst, nbad);
    return 0;
}
