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
//                  Cholesky A0 = C0 + rho I = L L^T in global memory (wide_chol.cuh; the
//                  B x B fp64 matrix, 1.44 MB at B = 425, exceeds shared memory),
//                  z0 = L^-T L^-1 t0, q0, mhat.
//      k2w_update  lines 9-16: the Woodbury update of the narrow path on the Cholesky
//                  factor (forward solves for W = L^-1 U, one backward solve for z).
//  The statistics themselves default to the exact-integer tensor-core kernels of
//  widei8.cuh (k1w_stats / k1w_stats_tc remain selectable).
//  K3w k3w_sweep   per pixel (albedo, projection, thresholded update, beta) with a
//                  warp per pixel over a shared-memory tile of contiguous pixel rows,
//                  then the sufficient statistics sum beta L' with a thread per band.
#pragma once
#include "kernels.cuh"
#include "wide_chol.cuh"

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
// K3w ring: at most S - 1 newer groups may stay pending
__device__ __forceinline__ void cp_async_wait_ring() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

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
constexpr int kWideT1 = 30;      // pixels per K1w shared tile (two tiles + pilot fit 2 CTAs/SM)
constexpr int kWideNT1 = 256;    // threads (= 8x8 blocks) per K1w CTA
constexpr int kWideRun1 = 16;    // K1w tiles per fp32 run before the fp64 fold

struct WideStatsArgs {
    const float* L;
    const float* pil32;
    const float* ghat32;
    double* part;     // [cols][NG * 128][64] blocks of the extended-row second moments
    int cols, N, B, BE, NB, NG;
    int mask;         // nodata masking: such rows contribute nothing
    float nodata;
};

__host__ inline size_t k1w_smem(int B, int BE) { return (2 * (size_t)kWideT1 * BE + 2 * (size_t)B) * 4 + 16; }

// One CTA per (block group g, column c): the column's pixel rows arrive by cp.async
// straight into the extended-row layout of a double-buffered tile (row stride BE),
// are turned into extended rows in place (warp per 4 pixels, interleaved), and feed
// 128 8x8 FFMA register blocks.
__global__ void __launch_bounds__(kWideNT1, 2) k1w_stats(WideStatsArgs a) {
    extern __shared__ __align__(16) float w1_smem[];
    float* ext = w1_smem;                          // [2][kWideT1][BE]
    float* pil = ext + 2 * kWideT1 * a.BE;         // [B]
    float* gh = pil + a.B;                         // [B]
    const int g = blockIdx.x, c = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int B = a.B, BE = a.BE;
    const int blk = g * kWideNT1 + tid;
    const bool active = blk < a.NB;
    int R = 0, C = 0;
    if (active) blk_rc(blk, R, C);
    for (int b = tid; b < B; b += kWideNT1) {
        pil[b] = a.pil32[(size_t)c * B + b];
        gh[b] = a.ghat32[(size_t)c * B + b];
    }
    const float* Lc = a.L + (size_t)c * a.N * B;
    const int ntile = (a.N + kWideT1 - 1) / kWideT1;
    auto load_tile = [&](int t) {
        const int p0 = t * kWideT1, rows = min(kWideT1, a.N - p0);
        float* buf = ext + (t & 1) * kWideT1 * BE;
        const uint32_t d0 = smem_u32(buf);
        const float* src = Lc + (size_t)p0 * B;
        for (int r = 0; r < rows; ++r)
            for (int b = tid; b < B; b += kWideNT1) cp_async4(d0 + 4 * (r * BE + b), src + (size_t)r * B + b);
        cp_async_commit();
    };
    load_tile(0);
    // fp32 register runs are folded into this thread's fp64 partial block in global
    // memory (L2-resident, 512 B per thread), keeping registers for the FFMA tile
    double* out = a.part + ((size_t)c * a.NG * kWideNT1 + blk) * 64;
    float acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = 0.f;
    int run = 0;
    bool first_fold = true;
    auto fold = [&]() {
        if (active) {
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                out[i] = (first_fold ? 0.0 : out[i]) + (double)acc[i];
                acc[i] = 0.f;
            }
        }
        first_fold = false;
    };
    for (int t = 0; t < ntile; ++t) {
        const int p0 = t * kWideT1, rows = min(kWideT1, a.N - p0);
        float* buf = ext + (t & 1) * kWideT1 * BE;
        __syncthreads();                       // buffer (t+1)&1 no longer read by anyone
        if (t + 1 < ntile) {
            load_tile(t + 1);
            cp_async_wait_1();
        } else {
            cp_async_wait_all();
        }
        __syncthreads();                       // tile t landed
        // extended rows in place: x = L - sigma c, rho = sigma - 1, 1, zero pad; a warp
        // per 8 pixels, their sigma dot products interleaved
        {
            constexpr int PW = (kWideT1 + kWideNT1 / 32 - 1) / (kWideNT1 / 32);   // pixels per warp
            const int pp0 = wid * PW;
            float sg[PW];
            unsigned bad = 0u;   // bit u: pixel pp0 + u is nodata (masking)
#pragma unroll
            for (int u = 0; u < PW; ++u) sg[u] = 0.f;
            for (int b = lane; b < B; b += 32) {
                const float gb = gh[b];
#pragma unroll
                for (int u = 0; u < PW; ++u)
                    if (pp0 + u < rows) {
                        const float lv = buf[(pp0 + u) * BE + b];
                        sg[u] = fmaf(lv, gb, sg[u]);
                        if (a.mask && is_nodata(lv, a.nodata)) bad |= 1u << u;
                    }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                bad |= __shfl_xor_sync(0xffffffffu, bad, off);
#pragma unroll
                for (int u = 0; u < PW; ++u) sg[u] += __shfl_xor_sync(0xffffffffu, sg[u], off);
            }
            for (int b = lane; b < BE; b += 32) {
                const float pb = b < B ? pil[b] : 0.f;
#pragma unroll
                for (int u = 0; u < PW; ++u) {
                    const int pp = pp0 + u;
                    if (pp >= kWideT1) break;
                    float* row = buf + pp * BE;
                    float v;
                    if (pp >= rows || (bad >> u & 1u)) v = 0.f;
                    else if (b < B) v = fmaf(-sg[u], pb, row[b]);
                    else v = b == B ? sg[u] - 1.f : (b == B + 1 ? 1.f : 0.f);
                    row[b] = v;
                }
            }
        }
        __syncthreads();
        if (active) {
            const float* ra = buf + R * 8;
            const float* rb = buf + C * 8;
#pragma unroll 3
            for (int pp = 0; pp < kWideT1; ++pp) {
                const float4 a0 = *reinterpret_cast<const float4*>(ra + pp * BE);
                const float4 a1 = *reinterpret_cast<const float4*>(ra + pp * BE + 4);
                const float4 b0 = *reinterpret_cast<const float4*>(rb + pp * BE);
                const float4 b1 = *reinterpret_cast<const float4*>(rb + pp * BE + 4);
                const float xa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float xb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[i * 8 + k] = fmaf(xa[i], xb[k], acc[i * 8 + k]);
            }
        }
        if (++run == kWideRun1) {
            fold();
            run = 0;
        }
    }
    if (run > 0 || first_fold) fold();
}

// ---------------------------------------------------------------- K2w init
constexpr int kWideNT2 = 128;    // k2w_update threads (5 CTAs per SM: one wave of 598 columns)
constexpr int kWideNTI = 512;     // k2w_init threads (1 CTA per SM)

struct WideInitArgs {
    ColState cs;
    const float* pil32;
    const double* part;    // K1w blocks [cols][NG*128][64], or (BEp > 0) k1w_stats_tc [cols][BEp][BEp]
    int BEp;
    double* mean_out;      // optional [cols][B]
    double* cov_out;       // optional [cols][B][B]
    int cols, N, B, BE, NG, use_albedo, stats_only;
    int energy;            // the energy trace needs tr(A0^-1)
    int sym;               // the block-pair partials are exactly symmetric (int8 SYRK): no (P + P^T)/2
    double ridge_rel;
    int c0 = 0;            // first column of this launch (grid.x columns from c0)
};

// shared: dm, srx, cv, vt, mh [B]; D, Dinv [32][33]; the panel Cp [B][32] (after the
// factorisation reused for the solves: x [2][B], red [16][2][32], yv [2][32]); scratch [32][4]
__host__ __device__ inline size_t k2w_init_panel(int B) {
    const size_t p = (size_t)B * kChB, q = (size_t)2 * B + 16 * 2 * 32 + 2 * 32;
    return p > q ? p : q;
}
__host__ inline size_t k2w_init_smem(int B) { return (size_t)(5 * B + 2 * kChB * kChD + k2w_init_panel(B) + 32 * 4) * 8 + 32; }

__global__ void __launch_bounds__(kWideNTI, 1) k2w_init(WideInitArgs a) {
    extern __shared__ double w2_smem[];
    const int B = a.B, tid = threadIdx.x, c = a.c0 + blockIdx.x, nt = blockDim.x;
    double* dm = w2_smem;        // [B] mean(L) - c, later mu0
    double* srx = dm + B;        // [B]
    double* cv = srx + B;        // [B] pilot c
    double* vt = cv + B;         // [B] t0
    double* mh = vt + B;         // [B] fp32 mhat (as double)
    double* D = mh + B;          // [kChB][kChD] diagonal block
    double* Dinv = D + kChB * kChD;                  // [kChB][kChD] its inverse
    double* Cp = Dinv + kChB * kChD + ((5 * B) & 1);   // [B][kChB] panel (16-byte aligned)
    double* scratch = Cp + k2w_init_panel(B);   // [32][4]
    __shared__ int bad, chol_flag;
    __shared__ double sh_tol, sh_mm;
    const int BEp = a.BEp;
    const double* S = BEp > 0 ? a.part + (size_t)c * BEp * BEp : a.part + (size_t)c * a.NG * kWideNT1 * 64;
    // entry (i, k) of the extended-row second moments: FFMA 8x8 blocks, or the tensor-core
    // block-pair matrix (diagonal 128-blocks symmetrised, (P + P^T)/2; lower blocks as is)
    auto ext = [&](int i, int k) -> double {
        if (BEp == 0) return ext_entry(S, i, k, 0);
        if (i < k) {
            const int t = i;
            i = k;
            k = t;
        }
        if (!a.sym && (i >> 7) == (k >> 7)) return 0.5 * (S[(size_t)i * BEp + k] + S[(size_t)k * BEp + i]);
        return S[(size_t)i * BEp + k];
    };
    double* A = a.cs.ainv + (size_t)c * B * wide_ld(B);   // row stride wide_ld(B)
    if (tid == 0) bad = COL_OK;
    __syncthreads();
    const double Nv = a.cs.mask ? ext(B + 1, B + 1) : (double)a.N;   // valid rows when masking
    const double invN = 1.0 / Nv;
    if (tid == 0) {
        a.cs.nvalid[c] = Nv;
        if (!(Nv >= 2.0)) bad = COL_INSUFFICIENT;
    }
    __syncthreads();
    const double Sr = ext(B + 1, B), Srr = ext(B, B);
    int nonfinite = 0;
    for (int b = tid; b < B; b += nt) {
        cv[b] = (double)a.pil32[(size_t)c * B + b];
        srx[b] = ext(B, b);
        dm[b] = (ext(B + 1, b) + Sr * cv[b]) * invN;
        if (!isfinite(dm[b])) nonfinite = 1;
    }
    __syncthreads();
    // C0 = (Sxx + Srx c^T + c Srx^T + Srr c c^T)/N - dm dm^T  (fp64, lower + mirror)
    // a warp per row, lanes over the columns k <= i (coalesced partial reads, no divisions);
    // the partial reads of kAsm column strides are issued before any store (the stores to A
    // could alias them as far as the compiler knows)
    constexpr int kAsm = 8;
    for (int i = tid >> 5; i < B; i += nt >> 5)
        for (int k0 = tid & 31; k0 <= i; k0 += 32 * kAsm) {
            double e[kAsm];
#pragma unroll
            for (int u = 0; u < kAsm; ++u) {
                const int k = k0 + 32 * u;
                e[u] = k <= i ? ext(i, k) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kAsm; ++u) {
                const int k = k0 + 32 * u;
                if (k > i) break;
                const double s2 = e[u] + srx[i] * cv[k] + cv[i] * srx[k] + Srr * cv[i] * cv[k];
                const double v = s2 * invN - dm[i] * dm[k];
                if (!isfinite(v)) nonfinite = 1;
                A[(size_t)i * wide_ld(B) + k] = v;   // lower triangle only (the Cholesky reads nothing else)
                if (a.cov_out) {
                    a.cov_out[(size_t)c * B * B + (size_t)i * B + k] = v;
                    a.cov_out[(size_t)c * B * B + (size_t)k * B + i] = v;
                }
            }
        }
    if (nonfinite && bad == COL_OK) atomicCAS(&bad, COL_OK, COL_NONFINITE);
    __syncthreads();
    for (int b = tid; b < B; b += nt) {
        const double m = cv[b] + dm[b];
        a.cs.mbar[(size_t)c * B + b] = m;
        a.cs.mu[(size_t)c * B + b] = m;
        if (a.mean_out) a.mean_out[(size_t)c * B + b] = m;
        dm[b] = m;
    }
    if (a.stats_only) return;
    __syncthreads();
    {
        double loc[1] = {0.0};   // trace
        for (int b = tid; b < B; b += nt) loc[0] += A[(size_t)b * wide_ld(B) + b];
        block_sum<1>(loc, scratch);
        // ridge and the pivot tolerance's max diagonal, one diagonal entry per thread (with the
        // two changes here: 0.917 -> 0.895 ms per wave of 148 stress columns)
        const double rho = a.ridge_rel * loc[0] / (double)B;
        if (tid == 0) a.cs.rho64[c] = rho;
        double amax = 0.0;
        for (int b = tid; b < B; b += nt) {
            double* d = A + (size_t)b * wide_ld(B) + b;
            const double v = *d + rho;
            *d = v;
            amax = fmax(amax, v);
        }
        for (int off = 16; off > 0; off >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
        __syncthreads();   // scratch reuse (block_sum above)
        if ((tid & 31) == 0) scratch[tid >> 5] = amax;
        __syncthreads();
        if (tid == 0) {
            for (int w = 0; w < (nt + 31) / 32; ++w) amax = fmax(amax, scratch[w]);
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
    if (st == COL_OK && !wide_cholesky(A, B, sh_tol, D, Dinv, Cp, &chol_flag)) st = COL_NOT_SPD;
    __syncthreads();
    const double mm = sh_mm;
    for (int b = tid; b < B; b += nt) {
        vt[b] = dm[b] * (double)a.cs.s[b];
        const float m32 = (float)(dm[b] / mm);
        a.cs.mhat32[(size_t)c * B + b] = m32;
        mh[b] = (double)m32;
    }
    // z0 = A0^-1 t0 = L^-T (L^-1 t0); L^-1 t0 is kept (yprev) for the first Woodbury update
    double* xw = Cp;                    // [B]
    double* xz = Cp + B;                // [B]
    double* red = Cp + 2 * (size_t)B;   // [nwarps][2][32]
    double* yv = red + 16 * 2 * 32;     // [2][32]
    for (int b = tid; b < B; b += nt) xw[b] = st == COL_OK ? vt[b] : 0.0;
    __syncthreads();
    if (st == COL_OK) {   // uniform
        tri_fwd<1>(A, B, xw, D, red, yv);
        for (int b = tid; b < B; b += nt) xz[b] = xw[b];
        __syncthreads();
        tri_bwd<1>(A, B, xz, D, red, yv);
    }
    double qc[3] = {0.0, 0.0, 0.0};
    for (int b = tid; b < B; b += nt) {
        const double y = st == COL_OK ? xz[b] : 0.0;
        const float z32 = (float)y;
        a.cs.z32[(size_t)c * B + b] = z32;
        a.cs.tprev[(size_t)c * B + b] = vt[b];
        a.cs.yprev[(size_t)c * B + b] = st == COL_OK ? xw[b] : 0.0;
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
        a.cs.nlit[c] = 0;
    }
    // tr((C0 + rho I)^-1) = ||L^-1||_F^2 for the energy trace: forward solves of the unit
    // vectors, four at a time (only when the trace is on)
    double tl[1] = {0.0};
    if (a.energy && st == COL_OK) {
        double* xu = Cp;   // [2][B]
        for (int i0 = 0; i0 < B; i0 += 2) {
            __syncthreads();
            for (int e = tid; e < 2 * B; e += nt) xu[e] = (e % B == i0 + e / B) ? 1.0 : 0.0;
            __syncthreads();
            tri_fwd<2>(A, B, xu, D, red, yv);
            for (int e = tid; e < 2 * B; e += nt)
                if (i0 + e / B < B) tl[0] += xu[e] * xu[e];
        }
    }
    block_sum<1>(tl, scratch);
    if (tid == 0) {
        a.cs.tra[c] = tl[0];
        a.cs.tq[c] = (double)B - a.cs.rho64[c] * tl[0];
    }
}

// ---------------------------------------------------------------- K2w update
// shared: t [B], x_f [2][B] (forward: t, h -> L^-1 t, L^-1 h), with the energy trace x_b [4][B]
// (backward right-hand sides; otherwise the one backward right-hand side replaces w_t in x_f),
// yv [4][32], scratch [96], then (128-byte aligned) the factor ring [kTsS][kTsT][32][32] of the
// streamed solves (wide_chol.cuh; 2 stages of 2 tiles: 44.9 KB in all at B = 425, five CTAs per
// SM), which the
// literal path reuses as the diagonal block [32][33] and reduction [4][2][32] of tri_fwd
__host__ inline size_t k2w_update_smem(int B, int energy) {
    return (size_t)((energy ? 7 : 3) * B + 4 * 32 + 96 + 16 + kTsS * kStageD) * 8;
}
constexpr int kLitRows = 32;   // residual rows per chunk of the wide literal check
// doubles of global scratch per column for the wide literal check (packed C^k + residual rows)
__host__ inline long long lit_doubles(int B) { return (long long)B * (B + 1) / 2 + (long long)kLitRows * B; }

// Woodbury update on the Cholesky factor A0 = L L^T (wide_chol.cuh):
// W = L^-1 U with U = [t', t, h] (w' = L^-1 t' kept from the previous update in yprev), G =
// U^T A0^-1 U = W^T W, coef = M (I + G M)^-1 W^T w_t, z = L^-T (w_t - W coef). The energy trace
// also needs Y = A0^-1 U = L^-T W (three more backward right-hand sides, same pass over L).
__global__ void __launch_bounds__(kWideNT2, 5) k2w_update(UpdateArgs a, const __grid_constant__ CUtensorMap fmap) {
    extern __shared__ double w3_smem[];
    const int B = a.B, tid = threadIdx.x, c = blockIdx.x, nt = blockDim.x;
    double* sh_t = w3_smem;          // [B] t^k
    double* xf = sh_t + B;           // [2][B]
    // backward right-hand sides: [4][B] with the energy trace, else in place of w_t (xf[0..B))
    double* xb = a.energy_on ? xf + 2 * B : xf;
    double* yv = xf + (a.energy_on ? 6 : 2) * B;   // [4][32]
    double* scratch = yv + 4 * 32;   // [96]: block_sum [4 warps][<= 18], literal check [32][3]
    double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(scratch + 96) + 127) & ~(uintptr_t)127);
    __shared__ double sh_coef[3], sh_s[3], sh_g[9];
    __shared__ int sh_st, sh_lit;
    __shared__ __align__(8) uint64_t ts_full[kTsS], ts_empty[kTsS];
    ColState& cs = a.cs;
    if (cs.status[c] != COL_OK) return;   // uniform per block
    const double* Lf = cs.ainv + (size_t)c * B * wide_ld(B);   // the solve-ready factor (row stride wide_ld(B))
    // the factor stream (forward then backward pass) starts before the statistics gather
    TileStream ts;
    ts_init(ts, ring, ts_full, ts_empty, &fmap, B, c, 2);
    if (tid == 0) {
        prefetch_tmap(&fmap);
        ts_issue(ts, kTsS);
    }
    // 1. sufficient statistics of the previous sweep (fixed CTA order)
    const long long c0 = (long long)c * a.tpc, c1 = c0 + a.tpc;
    int b0 = (int)((c0 * a.G) / a.ttot);
    while (b0 > 0 && tile_begin(b0, a.ttot, a.G) > c0) --b0;
    while (tile_begin(b0 + 1, a.ttot, a.G) <= c0) ++b0;
    const int W = B + kPartExtra;
    const double invN = 1.0 / cs.nvalid[c];
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
    for (int j = tid; j < B; j += nt) {
        double sv = 0.0;
        for (int b = b0; b < a.G && tile_begin(b, a.ttot, a.G) < c1; ++b) {
            const int slot = c - (int)(tile_begin(b, a.ttot, a.G) / a.tpc);
            sv += a.part3[((size_t)b * a.S + slot) * W + 3 + j];
        }
        const size_t o = (size_t)c * B + j;
        const double mb = cs.mbar[o], tp = cs.tprev[o], mhj = (double)cs.mhat32[o];
        const double h = sv * invN + (bs * mhj - bbar * mb);   // (1/N) sum beta (L - mu0)
        const double mu = mb - bbar * tp;                       // Eq. 10 / line 10
        const double t = mu * (double)cs.s[j];                  // Eq. 9
        sh_t[j] = t;
        xf[j] = t;
        xf[B + j] = h;
        cs.mu[o] = mu;
    }
    __syncthreads();
    // 2. W = L^-1 [t, h]; 3. G = W^T W with W = [w', w_t, w_h] (U^T A0^-1 U)
    tri_stream<2, true>(ts, B, xf, yv);
    double gv[9];   // G = W^T W (kept in shared memory for the energy trace's YY step)
#pragma unroll
    for (int i = 0; i < 9; ++i) gv[i] = 0.0;
    for (int j = tid; j < B; j += nt) {
        const size_t o = (size_t)c * B + j;
        const double w[3] = {cs.yprev[o], xf[j], xf[B + j]};
        const double u[3] = {cs.tprev[o], sh_t[j], 0.0};
        (void)u;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int q2 = 0; q2 < 3; ++q2) gv[r * 3 + q2] += w[r] * w[q2];
    }
    block_sum<9>(gv, scratch);
    if (tid == 0) {
        for (int i = 0; i < 9; ++i) sh_g[i] = gv[i];
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
        const bool solved = solve3(K, v, x);
        if (!solved) st = COL_NOT_SPD;
        for (int i = 0; i < 3; ++i) {
            double s2 = 0.0;
            for (int l = 0; l < 3; ++l) s2 += M[i][l] * x[l];
            sh_coef[i] = s2;
        }
        sh_st = st;
        sh_lit = a.lit_mode == 2 || (a.lit_mode == 1 && (!solved || !(min_eig3(K) > kLitTau)));
    }
    __syncthreads();
    if (sh_lit) {
        // lines 10-16 literally (reading C16''), C^k and the residual rows in global scratch;
        // then w' = L^-1 t^k for the next Woodbury update (the prefetched backward tiles are
        // drained first: the ring becomes tri_fwd's diagonal block and reduction buffer)
        ts_drain(ts);
        __syncthreads();
        double* Dsm = ring;                 // [32][33]
        double* red = ring + kChB * kChD;   // [4][2][32]
        double* Cp = a.lit + (size_t)c * a.lit_stride;
        const int stl = literal_iteration(a, c, nullptr, Cp, Cp + (size_t)B * (B + 1) / 2, kLitRows, xf, scratch);
        if (stl != COL_NOT_SPD) {
            for (int j = tid; j < B; j += nt) xf[j] = cs.tprev[(size_t)c * B + j];
            __syncthreads();
            tri_fwd<1>(Lf, B, xf, Dsm, red, yv);
            for (int j = tid; j < B; j += nt) cs.yprev[(size_t)c * B + j] = xf[j];
        }
        if (tid == 0) {
            cs.status[c] = stl;
            cs.nlit[c] += 1;
        }
        return;
    }
    // 4. z = L^-T (w_t - W coef) (Woodbury); with the energy trace also Y = L^-T W
    const int nr = a.energy_on ? 4 : 1;
    for (int j = tid; j < B; j += nt) {
        const double wp = cs.yprev[(size_t)c * B + j], wt = xf[j], wh = xf[B + j];
        cs.yprev[(size_t)c * B + j] = wt;   // w' = L^-1 t for the next update
        xb[j] = wt - (wp * sh_coef[0] + wt * sh_coef[1] + wh * sh_coef[2]);
        if (nr == 4) {
            xb[B + j] = wp;
            xb[2 * B + j] = wt;
            xb[3 * B + j] = wh;
        }
    }
    __syncthreads();
    if (nr == 4)
        tri_stream<4, false>(ts, B, xb, yv);
    else
        tri_stream<1, false>(ts, B, xb, yv);
    if (a.energy_on) {
        double yy[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) yy[i] = 0.0;
        for (int j = tid; j < B; j += nt) {
            const double y[3] = {xb[B + j], xb[2 * B + j], xb[3 * B + j]};
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int q2 = 0; q2 < 3; ++q2) yy[r * 3 + q2] += y[r] * y[q2];
        }
        block_sum<9>(yy, scratch);
        if (tid == 0) {
            const double M[3][3] = {{bbar * bbar, -bbar * bbar, 0.0}, {-bbar * bbar, b2, -1.0}, {0.0, -1.0, 0.0}};
            cs.tq[c] = woodbury_trace(M, sh_g, yy, B, cs.rho64[c], cs.tra[c], bbar);
        }
    }
    // 5. q, mhat.z, mu.z; state for the next iteration (w' = L^-1 t)
    double qc[3] = {0.0, 0.0, 0.0};
    for (int j = tid; j < B; j += nt) {
        const size_t o = (size_t)c * B + j;
        const double z = xb[j];
        const float z32 = (float)z;
        const double t = sh_t[j];
        qc[0] += t * z;
        qc[1] += (double)cs.mhat32[o] * (double)z32;
        qc[2] += cs.mu[o] * (double)z32;
        cs.z32[o] = z32;
        cs.tprev[o] = t;
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
#ifndef SMF_WT3
#define SMF_WT3 16
#endif
#ifndef SMF_WS3
#define SMF_WS3 2
#endif
constexpr int kWideT3 = SMF_WT3;  // pixels per K3w tile
constexpr int kWideS3 = SMF_WS3;  // K3w ring depth (tiles in flight)
constexpr int kWideNT3 = 128;     // threads per K3w CTA (4 warps; 4 CTAs per SM)

// floats per tile buffer: 32 rows + 4 floats of alignment shift + 32 floats of zero pad
// (the register pass reads up to 32 J - B floats past a row; the pad keeps that finite)
__host__ __device__ inline size_t k3w_tile_floats(int B) { return ((size_t)kWideT3 * B + 4 + 32 + 3) / 4 * 4; }
__host__ inline int k3w_j(int B) {
    const int j = (B + 31) / 32;
    return j <= 2 ? 2 : j <= 4 ? 4 : j <= 8 ? 8 : j <= 14 ? 14 : j <= 20 ? 20 : j <= 28 ? 28 : 0;
}
__host__ inline size_t k3w_smem(int B) {
    const int J = k3w_j(B);
    return (kWideS3 * k3w_tile_floats(B) + 2 * (size_t)(J > 0 ? 32 * J : B)) * 4 + 16;
}

// Warp reduce-scatter of P (1, 2 or 4) fp32 sums: lane l returns the full sum of value
// l / (32 / P). P - 1 + 5 - log2(P) shuffles instead of 5 P.
template <int P>
__device__ __forceinline__ float warp_rs_f(const float (&v)[P]) {
    const int lane = threadIdx.x & 31;
    float x0 = v[0], x1 = P > 1 ? v[P > 1 ? 1 : 0] : 0.f;
    int o = 16;
    if constexpr (P == 4) {   // 4 -> 2 values (lanes with bit 4 keep values 2, 3)
        const bool up = lane & 16;
        const float s0 = up ? v[0] : v[2], s1 = up ? v[1] : v[3];
        x0 = (up ? v[2] : v[0]) + __shfl_xor_sync(0xffffffffu, s0, 16);
        x1 = (up ? v[3] : v[1]) + __shfl_xor_sync(0xffffffffu, s1, 16);
        o = 8;
    }
    if constexpr (P >= 2) {   // 2 -> 1 value
        const bool up = lane & o;
        x0 = (up ? x1 : x0) + __shfl_xor_sync(0xffffffffu, up ? x0 : x1, o);
        o >>= 1;
    }
    for (; o >= 1; o >>= 1) x0 += __shfl_xor_sync(0xffffffffu, x0, o);
    return x0;
}

// J = elements per lane of a pixel row (B <= 32 J). A warp processes PB pixels at once
// (their dot products interleaved for ILP): lane l holds bands l + 32 j of each row in
// registers from the albedo dot through the projection to the sum of beta L' (the
// statistics for k + 1), so the tile is read from shared memory once; the xor
// butterflies leave every lane with the full dots, so all lanes evaluate the pixel update
// identically and lane 0 stores it. Per-lane sums are combined across the warps in a
// fixed order (fp64) at each column-slot flush.
// MASK: nodata masking compiled in (the checks cost ~45 % of the sweep's time when
// present, so the common no-masking launch uses the MASK = false instance)
template <int J, bool MASK>
__global__ void __launch_bounds__(kWideNT3, 4) k3w_sweep(SweepArgs a, const float* L) {
    constexpr int NW = kWideNT3 / 32;
#ifndef SMF_K3W_PB
#define SMF_K3W_PB 4
#endif
    constexpr int PB = J >= 20 ? 1 : (J <= 14 ? SMF_K3W_PB : 2);   // pixels per warp pass (registers: PB x J row elements)
    extern __shared__ __align__(16) float w4_smem[];
    const int B = a.B, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const size_t TF = k3w_tile_floats(B);
    float* buf0 = w4_smem;
    float* zs = w4_smem + kWideS3 * TF;   // [32 J], zero beyond B
    float* ms = zs + 32 * J;           // [32 J], zero beyond B
    __shared__ float sh_aprev[kWideT3];
    __shared__ uint64_t full[kWideS3];  // bulk path: one TMA bulk copy per tile
    __shared__ float sh_par[4];
    __shared__ int sh_st;
    __shared__ double red[NW][5];
    __shared__ float reda[NW][32 * J];  // per-warp sum beta L' at a flush
    const long long tb = tile_begin(blockIdx.x, a.ttot, a.G), te = tile_begin(blockIdx.x + 1, a.ttot, a.G);
    const int ntl = (int)(te - tb);
    const int cfirst = (int)(tb / a.tpc);
    const bool accum = a.k < a.n_iter;    // statistics for iteration k + 1
    const bool acce = accum || a.energy;   // partials written (energy: every sweep)
    // zero the ring once: the pads past the tile data stay zero
    for (size_t e = tid; e < kWideS3 * TF; e += kWideNT3) buf0[e] = 0.f;
    if (tid == 0) {
        for (int q2 = 0; q2 < kWideS3; ++q2) mbar_init(&full[q2], 1);
        fence_mbar_init();
    }
    fence_proxy_async();
    __syncthreads();

    // tile addresses from cursors (column, tile-in-column): no 64-bit divisions per tile
    auto tile_src = [&](const TileCursor& tc, int& rows) -> const float* {
        const int p0 = tc.tt * kWideT3;
        rows = min(kWideT3, a.N - p0);
        return L + ((size_t)tc.c * a.N + p0) * B;
    };
    TileCursor lcur(tb, a.tpc);   // next tile to load
    auto load_tile = [&](int i) {
        int rows;
        const float* src = tile_src(lcur, rows);
        lcur.next();
        float* dst = buf0 + (i % kWideS3) * TF + wide_tile_shift(src);
        if (a.bulk) {   // one TMA bulk copy (source 16-byte aligned, 16-byte multiple)
            if (tid == 0) {
                const uint32_t bytes = (uint32_t)rows * B * 4;
                mbar_arrive_expect_tx(&full[i % kWideS3], bytes);
                bulk_load(dst, src, bytes, &full[i % kWideS3]);
            }
        } else {
            cp_async_floats(dst, src, rows * B, tid, kWideNT3);
        }
    };
    // prologue: tiles 0 .. S-2 in flight (one commit group per tile, empty groups past the end)
    for (int i = 0; i < kWideS3 - 1; ++i) {
        if (i < ntl) load_tile(i);
        cp_async_commit();
    }

    float acc[J];
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] = 0.f;
    float sb = 0.f, sb2 = 0.f, sbs = 0.f, sbp = 0.f, swa = 0.f;   // lanes < PB: their pixels' sums

    auto flush = [&](int slot) {
        double* P = a.part3 + ((size_t)blockIdx.x * a.S + slot) * (B + kPartExtra);
#pragma unroll
        for (int j = 0; j < J; ++j) {
            reda[wid][lane + 32 * j] = acc[j];
            acc[j] = 0.f;
        }
        float v5[5] = {sb, sb2, sbs, sbp, swa};   // nonzero in lanes < PB only
#pragma unroll
        for (int q5 = 0; q5 < 5; ++q5) v5[q5] = warp_sum_f(v5[q5]);
        if (lane == 0)
            for (int q5 = 0; q5 < 5; ++q5) red[wid][q5] = (double)v5[q5];
        __syncthreads();
        for (int b = tid; b < B; b += kWideNT3) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += (double)reda[w][b];
            P[3 + b] = s;
        }
        if (tid < 5) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += red[w][tid];
            P[tid < 3 ? tid : B + tid] = s;   // [0..2] and [B+3], [B+4]
        }
        __syncthreads();
        sb = sb2 = sbs = sbp = swa = 0.f;
    };

    int cur = -1;
    float mz = 0.f, cz = 0.f, q = 1.f, mmf = 1.f;
    int cst = 0;
    float msr[J], zsr[J];   // this lane's m-hat and z entries (zero beyond B)
    // alpha^{k-1} of the next tile's pixels, loaded one tile ahead (threads < kWideT3) so its
    // global-memory latency is off the per-tile critical path (Eq. 5 reweighting term)
    const bool need_prev = a.k > 0 && a.use_sparsity;
    TileCursor pcur(tb, a.tpc);
    auto aprev_load = [&]() -> float {
        const int pp = pcur.tt * kWideT3 + tid;
        const float v = (need_prev && tid < kWideT3 && pp < a.N) ? a.enh[(size_t)pcur.c * a.N + pp] : 0.f;
        pcur.next();
        return v;
    };
    float apf = ntl > 0 ? aprev_load() : 0.f;
    TileCursor ccur(tb, a.tpc);
    for (int i = 0; i < ntl; ++i, ccur.next()) {
        const float ap_cur = apf;
        if (i + 1 < ntl) apf = aprev_load();
        const int c = ccur.c;
        const int p0 = ccur.tt * kWideT3;
        const int rows = min(kWideT3, a.N - p0);
        // refill: tile i + S - 1 into the slot freed by tile i - 1 (end-of-tile barrier)
        if (i + kWideS3 - 1 < ntl) load_tile(i + kWideS3 - 1);
        cp_async_commit();
        if (c != cur) {
            if (cur >= 0 && acce) flush(cur - cfirst);
            for (int b = tid; b < 32 * J; b += kWideNT3) {
                zs[b] = b < B ? a.z32[(size_t)c * B + b] : 0.f;
                ms[b] = b < B ? a.mhat32[(size_t)c * B + b] : 0.f;
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
#pragma unroll
            for (int j = 0; j < J; ++j) {
                msr[j] = ms[lane + 32 * j];
                zsr[j] = zs[lane + 32 * j];
            }
            mz = sh_par[0];
            cz = sh_par[1];
            q = sh_par[2];
            mmf = sh_par[3];
            cst = sh_st;
            cur = c;
        }
        if (tid < kWideT3) sh_aprev[tid] = ap_cur;   // (unused for failed columns / past N)
        if (a.bulk)
            mbar_wait(&full[i % kWideS3], (i / kWideS3) & 1);
        else
            cp_async_wait_ring();   // this thread's copies of tile i have landed
        __syncthreads();        // ... and everyone's; sh_aprev visible
        int rr_;
        const float* T = buf0 + (i % kWideS3) * TF + wide_tile_shift(tile_src(ccur, rr_));
        for (int base = wid * PB; base < rows; base += NW * PB) {
            float v[PB][J], r[PB], dz[PB], r2[PB], dz2[PB];   // two partial sums per dot (ILP)
            int bad[PB];
#pragma unroll
            for (int pb = 0; pb < PB; ++pb) {
                r[pb] = 0.f;
                r2[pb] = 0.f;
                bad[pb] = 0;
                const float* row = T + (size_t)(base + pb) * B;
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    // with masking, elements past the row belong to the next pixel: zero them
                    // (0 * NaN of a neighbouring nodata pixel must not reach this one);
                    // without it a non-finite neighbour makes the column NONFINITE anyway
                    const bool inrow = !MASK || lane + 32 * j < B;
                    v[pb][j] = inrow ? row[lane + 32 * j] : 0.f;
                    if (j & 1) r2[pb] = fmaf(v[pb][j], msr[j], r2[pb]);
                    else r[pb] = fmaf(v[pb][j], msr[j], r[pb]);
                    if (MASK && inrow && is_nodata(v[pb][j], a.nodata)) bad[pb] = 1;
                }
                r[pb] += r2[pb];
            }
            if (MASK) {
#pragma unroll
                for (int pb = 0; pb < PB; ++pb) bad[pb] = __any_sync(0xffffffffu, bad[pb]);
            }
            // the PB dots reduced together (reduce-scatter: lane l ends with the dot of pixel
            // l / (32 / PB)), then gathered back to every lane for the centring
            const float rmine = warp_rs_f<PB>(r);
#pragma unroll
            for (int pb = 0; pb < PB; ++pb) r[pb] = __shfl_sync(0xffffffffu, rmine, pb * (32 / PB));
            float scv[PB];
#pragma unroll
            for (int pb = 0; pb < PB; ++pb) {
                scv[pb] = r[pb] * mmf;   // albedo-centred radiance L' = L - sc mhat
                dz[pb] = 0.f;
                dz2[pb] = 0.f;
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    v[pb][j] = fmaf(-scv[pb], msr[j], v[pb][j]);
                    if (j & 1) dz2[pb] = fmaf(v[pb][j], zsr[j], dz2[pb]);
                    else dz[pb] = fmaf(v[pb][j], zsr[j], dz[pb]);
                }
                dz[pb] += dz2[pb];
            }
            // pixel tails in parallel: lane l evaluates pixel l / (32 / PB) (the PB tails share
            // one instruction stream; lanes 0, 32 / PB, ... store), then beta is broadcast
            const float dzm = warp_rs_f<PB>(dz);
            const int myp = lane / (32 / PB);
            const float r0 = rmine, sc = rmine * mmf;
            int badm = bad[0];
#pragma unroll
            for (int pb = 1; pb < PB; ++pb)
                if (myp == pb) badm = bad[pb];
            const int ppm = base + myp;
            float beta = 0.f;
            const bool mine = (lane & (32 / PB - 1)) == 0 && ppm < rows;
            if (ppm < rows) {
                const size_t pix = (size_t)c * a.N + p0 + ppm;
                if (cst != COL_OK || badm) {   // failed column or nodata pixel
                    if (mine) {
                        a.enh[pix] = __int_as_float(0x7fc00000);
                        a.alb[pix] = __int_as_float(0x7fc00000);
                    }
                } else {
                    const float pz = dzm + fmaf(sc, mz, -cz);   // (L - mu^k).z
                    const float rt = a.use_albedo ? fmaxf(r0, a.r_floor) : 1.f;
                    float out;
                    float w = 0.f;
                    if (a.k == 0) {
                        const float a0 = pz / (rt * q);                       // line 6
                        out = a.n_iter == 0 ? a0 : (a0 > 0.f ? a0 : 0.f);     // reading C3
                        if (mine) a.alb[pix] = a.use_albedo ? r0 : 1.f;      // Eq. 7
                    } else {
                        w = a.use_sparsity ? 1.f / (sh_aprev[ppm] + a.eps) : 0.f;   // Eq. 5
                        const float x = (pz - w) / (rt * q);                       // line 16
                        out = x > 0.f ? x : 0.f;                                   // C14
                    }
                    beta = rt * out;
                    if (mine) {
                        a.enh[pix] = out;
                        if (a.energy) {
                            sbp = fmaf(beta, pz, sbp);
                            swa = fmaf(rt * w, fabsf(out), swa);
                        }
                        sb += beta;
                        sb2 = fmaf(beta, beta, sb2);
                        sbs = fmaf(beta, sc, sbs);
                    }
                }
            }
            if (accum) {
#pragma unroll
                for (int pb = 0; pb < PB; ++pb) {
                    const float bp = __shfl_sync(0xffffffffu, beta, pb * (32 / PB));   // 0 for skipped pixels
                    if (base + pb < rows && bp != 0.f) {   // warp-uniform
#pragma unroll
                        for (int j = 0; j < J; ++j) acc[j] = fmaf(bp, v[pb][j], acc[j]);
                    }
                }
            }
        }
        fence_proxy_async();   // generic reads of slot i % S before its async-proxy refill
        __syncthreads();       // slot i % S free for tile i + S
    }
    if (cur >= 0 && acce) flush(cur - cfirst);
}

}  // namespace smf

namespace smf {
// ---------------------------------------------------------------- K1w on tensor cores
// The wide extended-row SYRK as tcgen05 kind::tf32 MMAs over 128 x 128 band blocks of
// the extended row (BE padded to NBLK * 128). CTA (pair, column) owns one lower block
// pair (m >= n) of one column and streams the column's pixels in 32-pixel K-blocks:
// 8 transform warps, one per band row of the pair's two blocks (thread b loads L[p][b]
// for the K-block's 32 pixels -- coalesced across the warp -- forms x = L - sigma_p c,
// rho = sigma - 1, 1, splits h = RN-tf32(x), l = x - h and writes both K-major
// SWIZZLE_128B rows with STS.128); one MMA thread; 4 epilogue warps (TMEM lanes).
// Off-diagonal pairs accumulate S_mn = h_m h_n^T + h_m l_n^T + l_m h_n^T (two MMAs per
// K-step), diagonal pairs P = h_m h_m^T + 2 h_m l_m^T (one MMA, symmetrised by k2w_init),
// i.e. the split of reading C21. fp32 TMEM runs of kRunW K-blocks are folded by the
// epilogue into the column's fp64 partial matrix [BEp][BEp] in global memory (L2).
// sigma_p = L_p . ghat comes from k1w_sigma (one pass, fp32, the same product order as
// the FFMA kernels use for their own transform).
#ifndef SMF_KRUNW
#define SMF_KRUNW 16
#endif
constexpr int kRunW = SMF_KRUNW;  // K-blocks (32 px each) per fp32 TMEM run
constexpr int kTW = 13 * 32;      // threads: 8 transform + 4 epilogue + 1 MMA warps

struct WideTCArgs {
    const float* L;
    const float* pil32;
    const float* ghat32;
    const float* sigma;   // [cols][N] (NaN = nodata row when masking)
    double* part;         // [cols][BEp][BEp]
    int cols, N, B, NBLK;
    int mask;
};

__global__ void k1w_sigma(const float* __restrict__ L, const float* __restrict__ ghat32, float* __restrict__ sigma,
                          int cols, int N, int B, int mask, float nodata) {
    // a warp per pixel: lanes stride the bands, fixed-order butterfly; with masking a
    // nodata pixel gets sigma = NaN, which the SYRK treats as "no row"
    const int lane = threadIdx.x & 31;
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= (long long)cols * N) return;
    const int c = (int)(gw / N);
    const float* Lp = L + (size_t)gw * B;
    const float* g = ghat32 + (size_t)c * B;
    float s = 0.f;
    int bad = 0;
    for (int b = lane; b < B; b += 32) {
        const float lv = __ldg(Lp + b);
        s = fmaf(lv, __ldg(g + b), s);
        if (mask) bad |= is_nodata(lv, nodata);
    }
    s = warp_sum_f(s);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) sigma[gw] = bad ? __int_as_float(0x7fc00000) : s;
}

__host__ inline size_t k1w_tc_smem() { return 2 * (size_t)512 * 128 + 1024; }   // 2 stages x 512 rows x 128 B

__global__ void __launch_bounds__(kTW, 1) k1w_stats_tc(WideTCArgs a) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* ops = align1024(smem_raw);   // [2][512 rows][128 B]
    constexpr int STAGE = 512 * 128;
    __shared__ uint64_t op_full[2], op_empty[2], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_sh;
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    // pair index -> (m, n), m >= n (row-major lower triangle of the block grid)
    int m = 0, n = blockIdx.x;
    while (n > m) {
        n -= m + 1;
        ++m;
    }
    const bool diag = m == n;
    const int c = blockIdx.y, B = a.B, N = a.N;
    const int BEp = a.NBLK * 128;
    const int nkb = (N + 31) / 32;
    const uint32_t idesc256 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc128 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

    for (int i = tid; i < 2 * STAGE / 16; i += kTW) reinterpret_cast<float4*>(ops)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid == 0) {
        for (int s2 = 0; s2 < 2; ++s2) {
            mbar_init(&op_full[s2], 8);
            mbar_init(&op_empty[s2], 1);
            mbar_init(&acc_full[s2], 1);
            mbar_init(&acc_empty[s2], 4);
        }
        fence_mbar_init();
    }
    if (wid == 12) tmem_alloc(&tmem_sh, 512);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_sh;

    if (wid < 8) {
        // ===================== transform: thread = one band row of the pair =====================
        // threads 0..127: block m (H_m rows 0..127, L_m rows 128..255);
        // threads 128..255: block n (H_n rows 256..383, L_n rows 384..511), idle on the diagonal
        const int half = tid >> 7, r = tid & 127;
        const int blk = half ? n : m;
        const int b = blk * 128 + r;                 // extended-row index
        const bool work = !(diag && half);
        const float cb = b < B ? a.pil32[(size_t)c * B + b] : 0.f;
        const float* Lc = a.L + (size_t)c * N * B;
        const float* sg = a.sigma + (size_t)c * N;
        const uint32_t ops0 = smem_u32(ops);
        const uint32_t rowH = (uint32_t)(half ? 256 + r : r) * 128, rowL = rowH + 128 * 128;
        const uint32_t sw = (uint32_t)(r & 7);
        // Register double buffer (measured: one K-block's loads took ~2000 of its ~3000
        // cycles when issued after the previous K-block was published): the 32 radiance
        // values of K-block kb + 1 and lane j's sigma of pixel p0 + j are in flight while
        // K-block kb is transformed; sigma is broadcast with shuffles.
        const int bl = b < B ? b : B - 1;
        const bool all_bands = __all_sync(0xffffffffu, b < B);   // no extended-row entry in this warp
        auto load = [&](int kb, float (&lv)[32], float& sl) {
            const int p0 = kb * 32;
#pragma unroll
            for (int j = 0; j < 32; ++j) lv[j] = __ldg(Lc + (size_t)min(p0 + j, N - 1) * B + bl);
            sl = __ldg(sg + min(p0 + lane, N - 1));
        };
        auto process = [&](int kb, float (&lv)[32], const float sl) {
            const int s2 = kb & 1;
            if (kb >= 2) mbar_wait(&op_empty[s2], ((kb >> 1) - 1) & 1);
            if (work) {
                const int p0 = kb * 32;
                // the extended-row entry selected per band kind (in place); the common case
                // (a band row, a full K-block, no masking) is one shuffle and one FFMA
                if (all_bands && p0 + 32 <= N && !a.mask) {   // warp-uniform (shuffles below)
#pragma unroll
                    for (int j = 0; j < 32; ++j) lv[j] = fmaf(-__shfl_sync(0xffffffffu, sl, j), cb, lv[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float sv = __shfl_sync(0xffffffffu, sl, j);
                        const float xb = fmaf(-sv, cb, lv[j]);
                        const float v = b < B ? xb : (b == B ? sv - 1.f : (b == B + 1 ? 1.f : 0.f));
                        lv[j] = (p0 + j < N && !(a.mask && isnan(sv))) ? v : 0.f;
                    }
                }
                const uint32_t base = ops0 + s2 * STAGE;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float4 h, l;
                    h.x = tf32_rna(lv[4 * q + 0]);
                    h.y = tf32_rna(lv[4 * q + 1]);
                    h.z = tf32_rna(lv[4 * q + 2]);
                    h.w = tf32_rna(lv[4 * q + 3]);
                    l.x = lv[4 * q + 0] - h.x;
                    l.y = lv[4 * q + 1] - h.y;
                    l.z = lv[4 * q + 2] - h.z;
                    l.w = lv[4 * q + 3] - h.w;
                    const uint32_t off = (((uint32_t)q ^ sw) << 4);
                    sts4(base + rowH + off, h);
                    sts4(base + rowL + off, l);
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&op_full[s2]);
        };
        float la[32], lb[32], sa = 0.f, sb = 0.f;
        if (work) load(0, la, sa);
        for (int kb = 0; kb < nkb; kb += 2) {
            if (work && kb + 1 < nkb) load(kb + 1, lb, sb);
            process(kb, la, sa);
            if (kb + 1 < nkb) {
                if (work && kb + 2 < nkb) load(kb + 2, la, sa);
                process(kb + 1, lb, sb);
            }
        }
    } else if (wid < 12) {
        // ===================== epilogue: TMEM -> fp64 partial (global) =====================
        const int e = wid - 8, row = 32 * e + lane;      // D row = band of block m
        double* prow = a.part + ((size_t)c * BEp + m * 128 + row) * BEp + n * 128;
        int g = 0, run = 0;
        bool first = true;
        for (int kb = 0; kb < nkb; ++kb) {
            ++run;
            if (kb != nkb - 1 && run < kRunW) continue;
            run = 0;
            const int ab = g & 1;
            mbar_wait(&acc_full[ab], (g >> 1) & 1);
            tc_fence_after();
            const uint32_t t0 = tmem + ((uint32_t)(32 * e) << 16) + (uint32_t)(ab * 256);
            // this thread's row: 16-column chunks, 16-byte accesses, the next chunk's old
            // values in flight while the current one is added (latency of the L2 round trip
            // paid about once per flush instead of once per chunk)
            double2* prow2 = reinterpret_cast<double2*>(prow);
            double2 cur[8], nxt[8];
            if (!first) {
#pragma unroll
                for (int k = 0; k < 8; ++k) cur[k] = prow2[k];
            }
#pragma unroll 1
            for (int n0 = 0; n0 < 128; n0 += 16) {
                if (!first && n0 + 16 < 128) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) nxt[k] = prow2[(n0 + 16) / 2 + k];
                }
                float v[16], u[16];
                tmem_ld16x2(t0 + n0, t0 + 128 + n0, v, u);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    double2 s;
                    s.x = (double)v[2 * k] + (diag ? 2.0 : 1.0) * (double)u[2 * k];
                    s.y = (double)v[2 * k + 1] + (diag ? 2.0 : 1.0) * (double)u[2 * k + 1];
                    if (!first) {
                        s.x += cur[k].x;
                        s.y += cur[k].y;
                    }
                    prow2[n0 / 2 + k] = s;
                    cur[k] = nxt[k];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            ++g;
            first = false;
        }
    } else {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            const uint32_t ops0 = smem_u32(ops);
            int g = 0, run = 0;
            bool fresh = true;
            for (int kb = 0; kb < nkb; ++kb) {
                const int s2 = kb & 1, ab = g & 1;
                if (fresh && g >= 2) mbar_wait(&acc_empty[ab], ((g >> 1) - 1) & 1);
                mbar_wait(&op_full[s2], (kb >> 1) & 1);
                tc_fence_after();
                const uint32_t sb = ops0 + s2 * STAGE;
                const uint32_t d = tmem + (uint32_t)(ab * 256);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t ko = ks * 32;
                    const uint64_t dHm = umma_desc(sb + ko, 16, 1024, 2);                   // rows 0..127
                    const uint64_t dLm = umma_desc(sb + 128 * 128 + ko, 16, 1024, 2);       // rows 128..255
                    const uint64_t dHn = umma_desc(sb + 256 * 128 + ko, 16, 1024, 2);       // rows 256..511
                    const uint32_t acc0 = (fresh && ks == 0) ? 0u : 1u;
                    if (diag) {
                        mma_tf32(d, dHm, dHm, idesc256, acc0);                 // [h h^T | h l^T]
                    } else {
                        mma_tf32(d, dHm, dHn, idesc256, acc0);                 // [h_m h_n^T | h_m l_n^T]
                        mma_tf32(d, dLm, dHn, idesc128, 1u);                   // += l_m h_n^T
                    }
                }
                fresh = false;
                mma_commit(&op_empty[s2]);
                if (kb == nkb - 1 || ++run == kRunW) {
                    mma_commit(&acc_full[ab]);
                    ++g;
                    run = 0;
                    fresh = true;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (wid == 12) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}
}  // namespace smf
