// wide.cuh -- the hot path for any band count B (the narrow kernels in kernels.cuh
// need B % 4 == 0 and B <= 96: a pixel row in registers, TMA tiles with 16-byte
// rows). Used for the full-spectrum stress configuration (B = 425, 380-2510 nm,
// BASELINE.json configs[3]). Same method, same readings, same column state as the
// narrow path (ColState, K3 partial layout [G][S][B+3]); only the data movement
// differs:
//  K1w k1w_stats   Fig. alg lines 2-3: extended-row SYRK (x = L - sigma c, rho, 1;
//                  DESIGN.md 6.1) on FFMA 8x8 register blocks; CTA (g, c) owns 128
//                  lower-triangle blocks of column c and streams all its pixels
//                  through a shared-memory tile (the NG CTAs of a column are launch-
//                  adjacent, so the column is read from HBM once and from L2 NG times).
//  K2w k2w_init    lines 2-3, 5-6: C0 from the blocks (fp64), ridge, blocked in-place
//                  Gauss-Jordan inverse A^-1 = (C0 + rho I)^-1 in global memory (the
//                  B x B fp64 matrix, 1.44 MB at B = 425, exceeds shared memory),
//                  z0 = A^-1 t0, q0, mhat.
//      k2w_update  lines 9-16: the narrow Woodbury update with A^-1 streamed from
//                  global memory.
//  K3w k3w_sweep   per pixel (albedo, projection, thresholded update, beta) with a
//                  warp per pixel over a shared-memory tile of contiguous pixel rows,
//                  then the sufficient statistics sum beta L' with a thread per band.
#pragma once
#include "kernels.cuh"

namespace smf {

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Copy n contiguous floats global -> shared with cp.async: 16-byte pieces where
// source and destination share the same alignment phase, 4-byte pieces otherwise.
// dst must have the same (address mod 16) as src for the 16-byte path; callers pass
// a destination offset chosen that way (see wide_tile_shift).
__device__ __forceinline__ void cp_async_floats(float* dst, const float* src, int n, int tid, int nt) {
    const uint32_t d0 = smem_u32(dst);
    const int head = (int)((16 - ((uintptr_t)src & 15)) & 15) / 4;   // floats before a 16-B boundary
    if (((d0 ^ (uint32_t)(uintptr_t)src) & 15) == 0 && n > head) {
        const int h = head < n ? head : n;
        for (int i = tid; i < h; i += nt) cp_async4(d0 + 4 * i, src + i);
        const int nv = (n - h) / 4;
        for (int i = tid; i < nv; i += nt) cp_async16(d0 + 4 * (h + 4 * i), src + h + 4 * i);
        for (int i = h + 4 * nv + tid; i < n; i += nt) cp_async4(d0 + 4 * i, src + i);
    } else {
        for (int i = tid; i < n; i += nt) cp_async4(d0 + 4 * i, src + i);
    }
}

// shift (in floats, 0..3) that gives a shared tile the alignment phase of its source
__device__ __forceinline__ int wide_tile_shift(const float* src) { return (int)(((uintptr_t)src & 15) >> 2); }

// ---------------------------------------------------------------- K1w
constexpr int kWideT1 = 32;      // pixels per K1w shared tile
constexpr int kWideNT1 = 128;    // threads (= 8x8 blocks) per K1w CTA
constexpr int kWideRun1 = 16;    // K1w tiles per fp32 run before the fp64 fold

struct WideStatsArgs {
    const float* L;
    const float* pil32;
    const float* ghat32;
    double* part;     // [cols][NG * 128][64] blocks of the extended-row second moments
    int cols, N, B, BE, NB, NG;
};

__host__ inline size_t k1w_smem(int B, int BE) { return ((size_t)kWideT1 * BE + 2 * (size_t)B) * 4 + 16; }

__global__ void __launch_bounds__(kWideNT1, 2) k1w_stats(WideStatsArgs a) {
    extern __shared__ __align__(16) float w1_smem[];
    float* ext = w1_smem;                       // [kWideT1][BE]
    float* pil = ext + kWideT1 * a.BE;          // [B]
    float* gh = pil + a.B;                      // [B]
    const int g = blockIdx.x, c = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int blk = g * kWideNT1 + tid;
    const bool active = blk < a.NB;
    int R = 0, C = 0;
    if (active) blk_rc(blk, R, C);
    for (int b = tid; b < a.B; b += kWideNT1) {
        pil[b] = a.pil32[(size_t)c * a.B + b];
        gh[b] = a.ghat32[(size_t)c * a.B + b];
    }
    const float* Lc = a.L + (size_t)c * a.N * a.B;
    float acc[64];
    double acc64[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        acc[i] = 0.f;
        acc64[i] = 0.0;
    }
    int run = 0;
    for (int p0 = 0; p0 < a.N; p0 += kWideT1) {
        __syncthreads();   // previous tile consumed (and pil/gh loaded)
        // extended rows: warp w takes pixels w, w + 4, ...; sigma = L . ghat (fixed order)
        for (int pp = wid; pp < kWideT1; pp += kWideNT1 / 32) {
            const int p = p0 + pp;
            float* row = ext + pp * a.BE;
            if (p < a.N) {
                const float* Lp = Lc + (size_t)p * a.B;
                float sg = 0.f;
                for (int b = lane; b < a.B; b += 32) sg = fmaf(__ldg(Lp + b), gh[b], sg);
                sg = warp_sum_f(sg);
                for (int b = lane; b < a.B; b += 32) row[b] = fmaf(-sg, pil[b], __ldg(Lp + b));
                for (int b = a.B + lane; b < a.BE; b += 32) row[b] = b == a.B ? sg - 1.f : (b == a.B + 1 ? 1.f : 0.f);
            } else {
                for (int b = lane; b < a.BE; b += 32) row[b] = 0.f;
            }
        }
        __syncthreads();
        if (active) {
            const float* ra = ext + R * 8;
            const float* rb = ext + C * 8;
#pragma unroll 2
            for (int pp = 0; pp < kWideT1; ++pp) {
                const float4 a0 = *reinterpret_cast<const float4*>(ra + pp * a.BE);
                const float4 a1 = *reinterpret_cast<const float4*>(ra + pp * a.BE + 4);
                const float4 b0 = *reinterpret_cast<const float4*>(rb + pp * a.BE);
                const float4 b1 = *reinterpret_cast<const float4*>(rb + pp * a.BE + 4);
                const float xa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float xb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[i * 8 + k] = fmaf(xa[i], xb[k], acc[i * 8 + k]);
            }
        }
        if (++run == kWideRun1) {
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                acc64[i] += (double)acc[i];
                acc[i] = 0.f;
            }
            run = 0;
        }
    }
    if (active) {
        double* out = a.part + ((size_t)c * a.NG * kWideNT1 + blk) * 64;
#pragma unroll
        for (int i = 0; i < 64; ++i) out[i] = acc64[i] + (double)acc[i];
    }
}

// ---------------------------------------------------------------- K2w init
constexpr int kWideNT2 = 256;
constexpr int kWideMaxBPT2 = 8;   // bands per thread in k2w_update (B <= 2048)
constexpr int kGJ = 32;          // Gauss-Jordan block size

struct WideInitArgs {
    ColState cs;
    const float* pil32;
    const double* part;    // K1w blocks [cols][NG*128][64]
    double* mean_out;      // optional [cols][B]
    double* cov_out;       // optional [cols][B][B]
    int cols, N, B, BE, NG, use_albedo, stats_only;
    double ridge_rel;
};

__host__ inline size_t k2w_init_smem(int B) { return (size_t)(5 * B + kGJ * kGJ + 32 * 4) * 8; }

// In-place blocked Gauss-Jordan inverse of the SPD matrix A (B x B, row-major, global)
// by one CTA: for every diagonal block K, D = A_KK^-1 (shared memory, unblocked GJ),
// R = D A_K* (row panel), A_ij -= A_iK R_Kj, A_iK = -A_iK D, A_KK = D. No pivoting: for
// an SPD matrix the pivots are the Cholesky pivots squared; a pivot <= tol flags NOT_SPD.
__device__ bool wide_gj_inverse(double* A, int B, double tol, double* D /* [kGJ][kGJ] smem */) {
    const int tid = threadIdx.x, nt = blockDim.x;
    __shared__ int sh_bad;
    if (tid == 0) sh_bad = 0;
    __syncthreads();
    for (int k0 = 0; k0 < B; k0 += kGJ) {
        const int nb = min(kGJ, B - k0);
        // (a) D = inverse of the diagonal block (unblocked GJ in shared memory, zero-padded)
        for (int e = tid; e < kGJ * kGJ; e += nt) D[e] = 0.0;
        __syncthreads();
        for (int e = tid; e < nb * nb; e += nt) D[(e / nb) * kGJ + e % nb] = A[(size_t)(k0 + e / nb) * B + k0 + e % nb];
        __syncthreads();
        for (int j = 0; j < nb; ++j) {
            const double piv = D[j * kGJ + j];
            if (!(piv > tol) || !isfinite(piv)) {
                if (tid == 0) sh_bad = 1;
                __syncthreads();
                return false;
            }
            const double p = 1.0 / piv;
            // rank-1 update of the other entries, then row / column j
            for (int e = tid; e < nb * nb; e += nt) {
                const int r = e / nb, cc = e % nb;
                if (r != j && cc != j) D[r * kGJ + cc] -= D[r * kGJ + j] * p * D[j * kGJ + cc];
            }
            __syncthreads();
            for (int e = tid; e < nb; e += nt) {
                if (e != j) {
                    D[j * kGJ + e] *= p;
                    D[e * kGJ + j] *= -p;
                }
            }
            __syncthreads();
            if (tid == 0) D[j * kGJ + j] = p;
            __syncthreads();
        }
        // (b) row panel R_Kj = D A_Kj and (c) trailing update A_ij -= A_iK R_Kj for
        // i, j outside the block: thread per column j, R_.j kept in registers; the old
        // column panel A_iK (same for every thread) is read through L1 as broadcasts
        for (int j = tid; j < B; j += nt) {
            if (j >= k0 && j < k0 + nb) continue;
            double rp[kGJ];
#pragma unroll
            for (int s2 = 0; s2 < kGJ; ++s2) rp[s2] = s2 < nb ? A[(size_t)(k0 + s2) * B + j] : 0.0;
            double rn[kGJ];
#pragma unroll
            for (int r = 0; r < kGJ; ++r) {
                double v = 0.0;
#pragma unroll
                for (int s2 = 0; s2 < kGJ; ++s2) v = fma(D[r * kGJ + s2], rp[s2], v);   // D is zero-padded
                rn[r] = v;
            }
#pragma unroll
            for (int r = 0; r < kGJ; ++r)
                if (r < nb) A[(size_t)(k0 + r) * B + j] = rn[r];
            for (int i = 0; i < B; ++i) {
                if (i >= k0 && i < k0 + nb) continue;
                const double* Ai = A + (size_t)i * B + k0;
                double v = A[(size_t)i * B + j];
#pragma unroll
                for (int s2 = 0; s2 < kGJ; ++s2) v = fma(-(s2 < nb ? Ai[s2] : 0.0), rn[s2], v);
                A[(size_t)i * B + j] = v;
            }
        }
        __syncthreads();
        // (d) column panel A_iK = -A_iK D, (e) A_KK = D
        for (int i = tid; i < B; i += nt) {
            if (i >= k0 && i < k0 + nb) continue;
            double row[kGJ];
#pragma unroll
            for (int s2 = 0; s2 < kGJ; ++s2) row[s2] = s2 < nb ? A[(size_t)i * B + k0 + s2] : 0.0;
#pragma unroll
            for (int r = 0; r < kGJ; ++r) {
                double v = 0.0;
#pragma unroll
                for (int s2 = 0; s2 < kGJ; ++s2) v = fma(row[s2], D[s2 * kGJ + r], v);
                if (r < nb) A[(size_t)i * B + k0 + r] = -v;
            }
        }
        for (int e = tid; e < nb * nb; e += nt) A[(size_t)(k0 + e / nb) * B + k0 + e % nb] = D[(e / nb) * kGJ + e % nb];
        __syncthreads();
    }
    return sh_bad == 0;
}

__global__ void __launch_bounds__(kWideNT2) k2w_init(WideInitArgs a) {
    extern __shared__ double w2_smem[];
    const int B = a.B, tid = threadIdx.x, c = blockIdx.x, nt = blockDim.x;
    double* dm = w2_smem;        // [B] mean(L) - c, later mu0
    double* srx = dm + B;        // [B]
    double* cv = srx + B;        // [B] pilot c
    double* vt = cv + B;         // [B] t0
    double* mh = vt + B;         // [B] fp32 mhat (as double)
    double* D = mh + B;          // [kGJ][kGJ]
    double* scratch = D + kGJ * kGJ;   // [32][4]
    __shared__ int bad;
    __shared__ double sh_tol, sh_mm;
    const double invN = 1.0 / (double)a.N;
    const double* S = a.part + (size_t)c * a.NG * kWideNT1 * 64;
    double* A = a.cs.ainv + (size_t)c * B * B;
    if (tid == 0) bad = COL_OK;
    __syncthreads();
    const double Sr = ext_entry(S, B + 1, B, 0), Srr = ext_entry(S, B, B, 0);
    int nonfinite = 0;
    for (int b = tid; b < B; b += nt) {
        cv[b] = (double)a.pil32[(size_t)c * B + b];
        srx[b] = ext_entry(S, B, b, 0);
        dm[b] = (ext_entry(S, B + 1, b, 0) + Sr * cv[b]) * invN;
        if (!isfinite(dm[b])) nonfinite = 1;
    }
    __syncthreads();
    // C0 = (Sxx + Srx c^T + c Srx^T + Srr c c^T)/N - dm dm^T  (fp64, lower + mirror)
    for (size_t e = tid; e < (size_t)B * B; e += nt) {
        const int i = (int)(e / B), k = (int)(e % B);
        if (i < k) continue;
        const double s2 = ext_entry(S, i, k, 0) + srx[i] * cv[k] + cv[i] * srx[k] + Srr * cv[i] * cv[k];
        const double v = s2 * invN - dm[i] * dm[k];
        if (!isfinite(v)) nonfinite = 1;
        A[(size_t)i * B + k] = v;
        A[(size_t)k * B + i] = v;
    }
    if (nonfinite) atomicExch(&bad, COL_NONFINITE);
    __syncthreads();
    for (int b = tid; b < B; b += nt) {
        const double m = cv[b] + dm[b];
        a.cs.mbar[(size_t)c * B + b] = m;
        a.cs.mu[(size_t)c * B + b] = m;
        if (a.mean_out) a.mean_out[(size_t)c * B + b] = m;
        dm[b] = m;
    }
    if (a.cov_out)
        for (size_t e = tid; e < (size_t)B * B; e += nt) a.cov_out[(size_t)c * B * B + e] = A[e];
    if (a.stats_only) return;
    __syncthreads();
    {
        double loc[1] = {0.0};   // trace
        for (int b = tid; b < B; b += nt) loc[0] += A[(size_t)b * B + b];
        block_sum<1>(loc, scratch);
        if (tid == 0) {
            const double rho = a.ridge_rel * loc[0] / (double)B;
            double amax = 0.0;
            for (int b = 0; b < B; ++b) {
                A[(size_t)b * B + b] += rho;
                amax = fmax(amax, A[(size_t)b * B + b]);
            }
            sh_tol = (double)B * 2.220446049250313e-16 * amax;
        }
        double mm_loc[1] = {0.0};
        for (int b = tid; b < B; b += nt) mm_loc[0] += dm[b] * dm[b];
        block_sum<1>(mm_loc, scratch);
        if (tid == 0) {
            if (bad == COL_OK && a.use_albedo && !(mm_loc[0] > 0.0)) bad = COL_DEGENERATE_MEAN;
            sh_mm = mm_loc[0];
        }
        __syncthreads();
    }
    int st = bad;
    if (st == COL_OK && !wide_gj_inverse(A, B, sh_tol, D)) st = COL_NOT_SPD;
    __syncthreads();
    const double mm = sh_mm;
    for (int b = tid; b < B; b += nt) {
        vt[b] = dm[b] * (double)a.cs.s[b];
        const float m32 = (float)(dm[b] / mm);
        a.cs.mhat32[(size_t)c * B + b] = m32;
        mh[b] = (double)m32;
    }
    __syncthreads();
    double qc[3] = {0.0, 0.0, 0.0};
    for (int b = tid; b < B; b += nt) {
        double y = 0.0;
        for (int i = 0; i < B; ++i) y = fma(A[(size_t)i * B + b], vt[i], y);
        const float z32 = (float)y;
        a.cs.z32[(size_t)c * B + b] = z32;
        a.cs.tprev[(size_t)c * B + b] = vt[b];
        a.cs.yprev[(size_t)c * B + b] = y;
        qc[0] += vt[b] * y;
        qc[1] += mh[b] * (double)z32;
        qc[2] += dm[b] * (double)z32;
    }
    block_sum<3>(qc, scratch);
    if (tid == 0) {
        if (st == COL_OK && (!(qc[0] > 0.0) || !isfinite(qc[0]) || !isfinite(qc[1]) || !isfinite(qc[2])))
            st = COL_DEGENERATE_TARGET;
        a.cs.q64[c] = qc[0];
        a.cs.q32[c] = (float)qc[0];
        a.cs.kc32[2 * c] = (float)qc[1];
        a.cs.kc32[2 * c + 1] = (float)qc[2];
        a.cs.status[c] = st;
    }
}

// ---------------------------------------------------------------- K2w update
__host__ inline size_t k2w_update_smem(int B) { return (size_t)(2 * B + 32 * 9) * 8; }

__global__ void __launch_bounds__(kWideNT2) k2w_update(UpdateArgs a) {
    extern __shared__ double w3_smem[];
    const int B = a.B, tid = threadIdx.x, c = blockIdx.x, nt = blockDim.x;
    double* sh_t = w3_smem;        // [B]
    double* sh_h = sh_t + B;       // [B]
    double* scratch = sh_h + B;    // [32][9]
    __shared__ double sh_coef[3], sh_s[3];
    __shared__ int sh_st;
    ColState& cs = a.cs;
    if (cs.status[c] != COL_OK) return;   // uniform per block
    const double* Ainv = cs.ainv + (size_t)c * B * B;
    // 1. sufficient statistics of the previous sweep (fixed CTA order)
    const long long c0 = (long long)c * a.tpc, c1 = c0 + a.tpc;
    int b0 = (int)((c0 * a.G) / a.ttot);
    while (b0 > 0 && tile_begin(b0, a.ttot, a.G) > c0) --b0;
    while (tile_begin(b0 + 1, a.ttot, a.G) <= c0) ++b0;
    const int W = B + 3;
    const double invN = 1.0 / (double)a.N;
    if (tid == 0) {
        double s0 = 0.0, s2 = 0.0, ss = 0.0;
        for (int b = b0; b < a.G && tile_begin(b, a.ttot, a.G) < c1; ++b) {
            const int slot = c - (int)(tile_begin(b, a.ttot, a.G) / a.tpc);
            const double* P = a.part3 + ((size_t)b * a.S + slot) * W;
            s0 += P[0];
            s2 += P[1];
            ss += P[2];
        }
        sh_s[0] = s0;
        sh_s[1] = s2;
        sh_s[2] = ss;
    }
    __syncthreads();
    const double bbar = sh_s[0] * invN, b2 = sh_s[1] * invN, bs = sh_s[2] * invN;
    double yt_r[kWideMaxBPT2], yh_r[kWideMaxBPT2];
#pragma unroll
    for (int jj = 0; jj < kWideMaxBPT2; ++jj) {
        const int j = tid + jj * nt;
        if (j >= B) break;
        double sv = 0.0;
        for (int b = b0; b < a.G && tile_begin(b, a.ttot, a.G) < c1; ++b) {
            const int slot = c - (int)(tile_begin(b, a.ttot, a.G) / a.tpc);
            sv += a.part3[((size_t)b * a.S + slot) * W + 3 + j];
        }
        const size_t o = (size_t)c * B + j;
        const double mb = cs.mbar[o], tp = cs.tprev[o], mhj = (double)cs.mhat32[o];
        const double h = sv * invN + (bs * mhj - bbar * mb);   // (1/N) sum beta (L - mu0)
        const double mu = mb - bbar * tp;                       // Eq. 10 / line 10
        sh_t[j] = mu * (double)cs.s[j];                         // Eq. 9
        sh_h[j] = h;
        cs.mu[o] = mu;
    }
    __syncthreads();
    // 2. y_t = A^-1 t, y_h = A^-1 h (A^-1 symmetric: column access, coalesced); 3. G
    double gv[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) gv[i] = 0.0;
#pragma unroll
    for (int jj = 0; jj < kWideMaxBPT2; ++jj) {
        const int j = tid + jj * nt;
        if (j >= B) break;
        double yt = 0.0, yh = 0.0;
#pragma unroll 4
        for (int i = 0; i < B; ++i) {
            const double v = __ldg(Ainv + (size_t)i * B + j);
            yt = fma(v, sh_t[i], yt);
            yh = fma(v, sh_h[i], yh);
        }
        yt_r[jj] = yt;
        yh_r[jj] = yh;
        const size_t o = (size_t)c * B + j;
        const double u[3] = {cs.tprev[o], sh_t[j], sh_h[j]}, y[3] = {cs.yprev[o], yt, yh};
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int q2 = 0; q2 < 3; ++q2) gv[r * 3 + q2] += u[r] * y[q2];
    }
    block_sum<9>(gv, scratch);
    if (tid == 0) {
        // C^k = C0 + U M U^T, M in the basis (t', t, h)
        const double M[3][3] = {{bbar * bbar, -bbar * bbar, 0.0}, {-bbar * bbar, b2, -1.0}, {0.0, -1.0, 0.0}};
        double K[3][3], v[3], x[3];
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j) {
                double s2 = (i == j) ? 1.0 : 0.0;
                for (int l = 0; l < 3; ++l) s2 += gv[i * 3 + l] * M[l][j];
                K[i][j] = s2;
            }
            v[i] = gv[i * 3 + 1];
        }
        int st = COL_OK;
        if (!solve3(K, v, x)) st = COL_NOT_SPD;
        for (int i = 0; i < 3; ++i) {
            double s2 = 0.0;
            for (int l = 0; l < 3; ++l) s2 += M[i][l] * x[l];
            sh_coef[i] = s2;
        }
        sh_st = st;
    }
    __syncthreads();
    // 4. z = y_t - Y M (I + G M)^-1 U^T A^-1 t (Woodbury), q, mhat.z, mu.z
    double qc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int jj = 0; jj < kWideMaxBPT2; ++jj) {
        const int j = tid + jj * nt;
        if (j >= B) break;
        const size_t o = (size_t)c * B + j;
        const double yt = yt_r[jj], yh = yh_r[jj], yp = cs.yprev[o];
        const double z = yt - (yp * sh_coef[0] + yt * sh_coef[1] + yh * sh_coef[2]);
        const float z32 = (float)z;
        const double t = sh_t[j];
        qc[0] += t * z;
        qc[1] += (double)cs.mhat32[o] * (double)z32;
        qc[2] += cs.mu[o] * (double)z32;
        cs.z32[o] = z32;
        cs.tprev[o] = t;
        cs.yprev[o] = yt;
    }
    block_sum<3>(qc, scratch);
    if (tid == 0) {
        int st = sh_st;
        if (st == COL_OK && (!(qc[0] > 0.0) || !isfinite(qc[0]) || !isfinite(qc[1]) || !isfinite(qc[2])))
            st = COL_DEGENERATE_TARGET;
        cs.q64[c] = qc[0];
        cs.q32[c] = (float)qc[0];
        cs.kc32[2 * c] = (float)qc[1];
        cs.kc32[2 * c + 1] = (float)qc[2];
        cs.status[c] = st;
    }
}

// ---------------------------------------------------------------- K3w sweep
constexpr int kWideT3 = 32;       // pixels per K3w tile
constexpr int kWideNT3 = 256;     // threads per K3w CTA (8 warps, 4 pixels each)
constexpr int kWideMaxBPT = 8;    // bands per thread in the beta L' accumulation (B <= 2048)

__host__ inline size_t k3w_tile_floats(int B) { return ((size_t)kWideT3 * B + 4 + 3) / 4 * 4; }
__host__ inline size_t k3w_smem(int B) { return (2 * k3w_tile_floats(B) + 2 * (size_t)B) * 4 + 16; }

__global__ void __launch_bounds__(kWideNT3, 1) k3w_sweep(SweepArgs a, const float* L) {
    extern __shared__ __align__(16) float w4_smem[];
    const int B = a.B, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const size_t TF = ((size_t)kWideT3 * B + 4 + 3) / 4 * 4;   // floats per tile buffer (+ shift room)
    float* buf0 = w4_smem;
    float* zs = w4_smem + 2 * TF;      // [B]
    float* ms = zs + B;                // [B]
    __shared__ float sh_beta[kWideT3], sh_sc[kWideT3];
    __shared__ float sh_par[4];
    __shared__ int sh_st;
    __shared__ double red[kWideNT3 / 32][3];
    const long long tb = tile_begin(blockIdx.x, a.ttot, a.G), te = tile_begin(blockIdx.x + 1, a.ttot, a.G);
    const int ntl = (int)(te - tb);
    const int cfirst = (int)(tb / a.tpc);
    const bool accum = a.k < a.n_iter;
    const int nbt = (B + kWideNT3 - 1) / kWideNT3;   // bands per thread (<= kWideMaxBPT)

    // tile i -> shared buffer i % 2, shifted to the source's 16-byte phase
    auto tile_src = [&](long long gt, int& rows) -> const float* {
        const int c = (int)(gt / a.tpc), tt = (int)(gt - (long long)c * a.tpc);
        const int p0 = tt * kWideT3;
        rows = min(kWideT3, a.N - p0);
        return L + ((size_t)c * a.N + p0) * B;
    };
    auto load_tile = [&](int i) {
        int rows;
        const float* src = tile_src(tb + i, rows);
        float* dst = buf0 + (i & 1) * TF + wide_tile_shift(src);
        cp_async_floats(dst, src, rows * B, tid, kWideNT3);
        cp_async_commit();
    };
    if (ntl > 0) load_tile(0);

    float acc[kWideMaxBPT];
#pragma unroll
    for (int j = 0; j < kWideMaxBPT; ++j) acc[j] = 0.f;
    float sb = 0.f, sb2 = 0.f, sbs = 0.f;   // per-thread partials (thread 0.. of the beta loop)

    auto flush = [&](int slot) {
        // band sums: thread j owns bands j, j + NT, ...; scalar sums reduced over the CTA
        double* P = a.part3 + ((size_t)blockIdx.x * a.S + slot) * (B + 3);
#pragma unroll
        for (int j = 0; j < kWideMaxBPT; ++j) {
            const int b = tid + j * kWideNT3;
            if (j < nbt && b < B) P[3 + b] = (double)acc[j];
            acc[j] = 0.f;
        }
        float v3[3] = {sb, sb2, sbs};
#pragma unroll
        for (int q = 0; q < 3; ++q) v3[q] = warp_sum_f(v3[q]);
        if (lane == 0)
            for (int q = 0; q < 3; ++q) red[wid][q] = (double)v3[q];
        __syncthreads();
        if (tid < 3) {
            double s = 0.0;
            for (int w = 0; w < kWideNT3 / 32; ++w) s += red[w][tid];
            P[tid] = s;
        }
        __syncthreads();
        sb = sb2 = sbs = 0.f;
    };

    int cur = -1;
    float mz = 0.f, cz = 0.f, q = 1.f, mmf = 1.f;
    int cst = 0;
    TileCursor ccur(tb, a.tpc);
    for (int i = 0; i < ntl; ++i, ccur.next()) {
        const int c = ccur.c;
        const int p0 = ccur.tt * kWideT3;
        const int rows = min(kWideT3, a.N - p0);
        if (i + 1 < ntl) load_tile(i + 1);
        if (c != cur) {
            if (cur >= 0 && accum) flush(cur - cfirst);
            for (int b = tid; b < B; b += kWideNT3) {
                zs[b] = a.z32[(size_t)c * B + b];
                ms[b] = a.mhat32[(size_t)c * B + b];
            }
            if (tid == 0) {
                sh_par[0] = a.kc32[2 * c];
                sh_par[1] = a.kc32[2 * c + 1];
                sh_par[2] = a.q32[c];
                sh_st = a.status[c];
            }
            __syncthreads();
            // |mu0|^2 in fp32 from mhat, fixed order (warp 0), identical for all threads
            if (wid == 0) {
                float s2 = 0.f;
                for (int b = lane; b < B; b += 32) s2 = fmaf(ms[b], ms[b], s2);
                s2 = warp_sum_f(s2);
                if (lane == 0) sh_par[3] = s2 > 0.f ? 1.f / s2 : 0.f;
            }
            __syncthreads();
            mz = sh_par[0];
            cz = sh_par[1];
            q = sh_par[2];
            mmf = sh_par[3];
            cst = sh_st;
            cur = c;
        }
        if (i + 1 < ntl) cp_async_wait_1(); else cp_async_wait_all();
        __syncthreads();   // tile i landed for every thread
        int rr;
        const float* T = buf0 + (i & 1) * TF + wide_tile_shift(tile_src(tb + i, rr));
        // ---- phase A: warp per pixel (albedo, projection, update)
        for (int pp = wid; pp < kWideT3; pp += kWideNT3 / 32) {
            float beta = 0.f, sc = 0.f;
            if (pp < rows) {
                const size_t pix = (size_t)c * a.N + p0 + pp;
                if (cst != COL_OK) {
                    if (lane == 0) {
                        a.enh[pix] = __int_as_float(0x7fc00000);
                        a.alb[pix] = __int_as_float(0x7fc00000);
                    }
                } else {
                    const float* row = T + (size_t)pp * B;
                    float r = 0.f;
                    for (int b = lane; b < B; b += 32) r = fmaf(row[b], ms[b], r);
                    r = warp_sum_f(r);                       // albedo factor (Eq. 7)
                    sc = r * mmf;
                    float dz = 0.f;
                    for (int b = lane; b < B; b += 32) dz = fmaf(fmaf(-sc, ms[b], row[b]), zs[b], dz);
                    dz = warp_sum_f(dz);
                    const float pz = dz + fmaf(sc, mz, -cz);  // (L - mu^k).z
                    const float rr2 = a.use_albedo ? r : 1.f;
                    const float rt = a.use_albedo ? fmaxf(r, a.r_floor) : 1.f;
                    float out;
                    if (a.k == 0) {
                        const float a0 = pz / (rt * q);
                        out = a.n_iter == 0 ? a0 : (a0 > 0.f ? a0 : 0.f);
                    } else {
                        const float aprev = a.use_sparsity ? a.enh[pix] : 0.f;
                        const float w = a.use_sparsity ? 1.f / (aprev + a.eps) : 0.f;
                        const float x = (pz - w) / (rt * q);
                        out = x > 0.f ? x : 0.f;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        a.enh[pix] = out;
                        if (a.k == 0) a.alb[pix] = rr2;
                    }
                    beta = rt * out;
                }
            }
            if (lane == 0) {
                sh_beta[pp] = beta;
                sh_sc[pp] = sc;
                sb += beta;
                sb2 = fmaf(beta, beta, sb2);
                sbs = fmaf(beta, sc, sbs);
            }
        }
        __syncthreads();
        // ---- phase B: sum beta L' with a thread per band
        if (accum && cst == COL_OK) {
#pragma unroll
            for (int j = 0; j < kWideMaxBPT; ++j) {
                const int b = tid + j * kWideNT3;
                if (j < nbt && b < B) {
                    const float mb = ms[b];
                    float s = acc[j];
                    for (int pp = 0; pp < rows; ++pp) s = fmaf(sh_beta[pp], fmaf(-sh_sc[pp], mb, T[(size_t)pp * B + b]), s);
                    acc[j] = s;
                }
            }
        }
        __syncthreads();   // buffer i & 1 free for tile i + 2
    }
    if (cur >= 0 && accum) flush(cur - cfirst);
}

}  // namespace smf
