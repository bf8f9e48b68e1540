// kernels.cuh -- the hot-path kernels of the B200 sparse albedo-corrected matched
// filter (Foote et al., arXiv 2003.02978; PAPER.md Fig. alg).
//
//  K1 k1_stats      Fig. alg lines 2-3: per-column first and second moments of the
//                   radiances (batched SYRK on FFMA 8x8 register tiles over
//                   TMA-staged, SWIZZLE_128B pixel tiles). Accuracy: each pixel is
//                   shifted by a pilot mean c and its component along c removed,
//                   L - c = x + rho c, so the fp32 products x x^T are ~20x smaller
//                   than (L-c)(L-c)^T; fp32 runs are flushed to fp64 once per tile
//                   and the exact identity is re-assembled in fp64 by K2.
//  K2 k2_init       lines 2-3, 5-6: reduce K1 partials -> mu0, C0; ridge; in-place
//                   Gauss-Jordan inverse A^-1 = (C0 + rho I)^-1 (fp64, smem);
//                   z0 = A^-1 t0, q0, c0 = mu0.z0, mhat = mu0/|mu0|^2.
//     k2_update     lines 9-16 per iteration: reduce the sweep's sufficient
//                   statistics -> mu^k (Eq. 10), C^k = C0 + rank-3 update (exact
//                   form of Eq. 11); Woodbury on A^-1:
//                   z^k = (C^k + rho I)^-1 t^k, q^k, c^k.
//  K3 k3_sweep      per pixel, one pass over the cube per iteration: albedo r_i
//                   (Eq. 7), whitened projection p_i = (L_i - mu^k).z^k (line 16),
//                   reweight w = 1/(alpha^{k-1} + eps) (Eq. 5), thresholded update
//                   (Eq. 6/8, line 16) and beta_i = r~_i alpha_i^k with the
//                   sufficient statistics of iteration k+1 (sum beta, beta^2,
//                   beta s, beta L'). Persistent CTAs over a balanced static
//                   partition of the tile stream; 3-stage TMA ring; the pixel row
//                   and the 72 band sums live in registers.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace smf {

constexpr int kTileRows = 128;    // pixels per TMA tile
constexpr int kStages = 3;        // K3 TMA ring depth
constexpr int kStages1 = 2;       // K1 TMA ring depth (K1 is FFMA-bound)
constexpr int kPilotRows = 32;    // pixels averaged for the K1 pilot shift

enum { COL_OK = 0, COL_NONFINITE = 1, COL_DEGENERATE_MEAN = 2, COL_NOT_SPD = 3, COL_DEGENERATE_TARGET = 4 };

// Shared-memory tile geometry: bands split into `nfull` 32-band regions
// (SWIZZLE_128B rows of 128 B) plus one tail region of `tailw` floats
// (8/16/32 -> SWIZZLE_32B/64B/128B). Each region holds kTileRows rows.
struct TileGeom {
    int B, nfull, tailw, stage_bytes;
    __host__ __device__ static TileGeom make(int B) {
        TileGeom g;
        g.B = B;
        g.nfull = B / 32;
        int rem = B % 32;
        g.tailw = rem == 0 ? 0 : (rem <= 8 ? 8 : (rem <= 16 ? 16 : 32));
        int bytes = kTileRows * (g.nfull * 128 + g.tailw * 4);
        g.stage_bytes = (bytes + 1023) / 1024 * 1024;
        return g;
    }
    __host__ __device__ uint32_t tx_bytes() const { return kTileRows * (nfull * 128 + tailw * 4); }
    // byte offset of quad q (bands 4q..4q+3) of row r within a stage
    __device__ __forceinline__ uint32_t quad_off(int r, int q) const {
        if (q < nfull * 8) return (q >> 3) * (kTileRows * 128) + swz_off(r, q & 7, 128);
        return nfull * (kTileRows * 128) + swz_off(r, q - nfull * 8, tailw * 4);
    }
};

// Issue the TMA loads of one tile (rows row0.., column c) into `stage`.
__device__ __forceinline__ void issue_tile(const TileGeom& g, unsigned char* stage, uint64_t* bar,
                                           const CUtensorMap* tm_main, const CUtensorMap* tm_tail, int row0,
                                           int c) {
    mbar_arrive_expect_tx(bar, g.tx_bytes());
    for (int f = 0; f < g.nfull; ++f)
        tma_load_3d(stage + f * (kTileRows * 128), tm_main, bar, f * 32, row0, c);
    if (g.tailw) tma_load_3d(stage + g.nfull * (kTileRows * 128), tm_tail, bar, g.nfull * 32, row0, c);
}

__device__ __forceinline__ unsigned char* align1024(unsigned char* p) {
    return reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ---------------------------------------------------------------- K1
// Partial layout per (column, chunk), fp64, width k1_width(B):
//   [nb][64]  sum x x^T per 8x8 block (lower triangle of blocks, row-major in block)
//   [Bp]      sum x          (Bp = nblk*8)
//   [Bp]      sum rho x
//   [2]       sum rho, sum rho^2
// with L - c = x + rho c (c = pilot mean of the first kPilotRows pixels).
struct StatsArgs {
    const float* L;      // radiance [cols][N][B]
    float* pilot;        // [cols][B] pilot shift (written by chunk 0)
    double* part1;       // [cols][nch1][k1_width]
    int cols, N, B, tpc, nch1, tiles_per_cta, nblk, nb, G1;
};

__host__ __device__ inline int k1_width(int nblk) { return nblk * (nblk + 1) / 2 * 64 + 2 * nblk * 8 + 2; }

constexpr int kFlushTiles1 = 2;    // K1 fp32 run length: tiles between fp64 flushes

// K1 dynamic smem: [kStages1 stages][64][NA] fp64 block accumulators
// [G1*nblk][16] fp64 diagonal-thread band sums, NA = G1*nb active threads.
__host__ __device__ inline size_t k1_smem_bytes(int B) {
    const int nblk = (B + 7) / 8, nb = nblk * (nblk + 1) / 2, G1 = 256 / nb;
    return (size_t)kStages1 * TileGeom::make(B).stage_bytes + (size_t)64 * G1 * nb * 8 +
           (size_t)G1 * nblk * 16 * 8 + 1024;
}

// Block (R, C) of the 8x8-blocked lower triangle, blk = R(R+1)/2 + C.
__device__ __forceinline__ void blk_rc(int blk, int& R, int& C) {
    int r = 0;
    while ((r + 1) * (r + 2) / 2 <= blk) ++r;
    R = r;
    C = blk - r * (r + 1) / 2;
}

__global__ void __launch_bounds__(256, 1)
    k1_stats(const __grid_constant__ CUtensorMap tm_main, const __grid_constant__ CUtensorMap tm_tail,
             StatsArgs a) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* stages = align1024(smem_raw);
    __shared__ uint64_t full[kStages1];
    __shared__ __align__(16) float pil[256];    // pilot c (zero-padded to nblk*8)
    __shared__ __align__(16) float ghat[256];   // c / |c|^2
    __shared__ float rho_s[kTileRows];
    __shared__ double red_r[kTileRows * 2];
    const TileGeom g = TileGeom::make(a.B);
    const int NA = a.G1 * a.nb;                 // active threads
    double* acc64 = reinterpret_cast<double*>(stages + kStages1 * g.stage_bytes);   // [64][NA]
    double* dsum = acc64 + (size_t)64 * NA;    // [G1*nblk][16]: sum x (8), sum rho x (8)
    const int tid = threadIdx.x;
    const int c = blockIdx.y, j = blockIdx.x;
    const int t0 = j * a.tiles_per_cta;
    const int t1 = min(t0 + a.tiles_per_cta, a.tpc);
    const int ntl = t1 - t0;
    const int Bq = a.nblk * 2;   // quads covered by the blocks

    if (tid == 0) {
        for (int s = 0; s < kStages1; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        for (int i = 0; i < kStages1 && i < ntl; ++i)
            issue_tile(g, stages + i * g.stage_bytes, &full[i], &tm_main, &tm_tail, (t0 + i) * kTileRows, c);
    }
    // pilot shift: fp32 mean of the first kPilotRows pixels, identical in every CTA
    const int np = min(kPilotRows, a.N);
    const size_t cbase = (size_t)c * a.N * a.B;
    if (tid < a.nblk * 8) {
        float sum = 0.f;
        if (tid < a.B)
            for (int p = 0; p < np; ++p) sum += a.L[cbase + (size_t)p * a.B + tid];
        pil[tid] = tid < a.B ? sum / (float)np : 0.f;
        if (j == 0 && tid < a.B) a.pilot[(size_t)c * a.B + tid] = pil[tid];
    }
    for (int i = tid; i < 64 * NA + a.G1 * a.nblk * 16; i += blockDim.x) acc64[i] = 0.0;
    __syncthreads();
    if (tid == 0) {
        double cc = 0.0;
        for (int b = 0; b < a.B; ++b) cc += (double)pil[b] * (double)pil[b];
        red_r[0] = cc;
    }
    __syncthreads();
    if (tid < a.nblk * 8) ghat[tid] = red_r[0] > 0.0 ? (float)((double)pil[tid] / red_r[0]) : 0.f;
    __syncthreads();

    const int blk = tid % a.nb, grp = tid / a.nb;
    const bool active = grp < a.G1;
    int R = 0, C = 0;
    blk_rc(blk, R, C);
    const bool diag = R == C;
    float acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = 0.f;
    double* dmine = dsum + (size_t)(grp * a.nblk + R) * 16;
    float ms[8], mr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ms[i] = mr[i] = 0.f;
    double r1 = 0.0, r2 = 0.0;   // row owners: sum rho, sum rho^2

    for (int it = 0; it < ntl; ++it) {
        const int s = it % kStages1;
        mbar_wait(&full[s], (it / kStages1) & 1);
        unsigned char* st = stages + s * g.stage_bytes;
        const int rowbase = (t0 + it) * kTileRows;
        // (1) rewrite the tile in place: x = (L - c) - rho c, rho = (L - c).ghat; rows >= N -> 0
        if (tid < kTileRows) {
            const bool valid = rowbase + tid < a.N;
            float rho = 0.f;
            for (int q = 0; q < Bq; ++q) {
                float4 v = *reinterpret_cast<const float4*>(st + g.quad_off(tid, q));
                const float4 cq = *reinterpret_cast<const float4*>(&pil[4 * q]);
                const float4 gq = *reinterpret_cast<const float4*>(&ghat[4 * q]);
                rho = fmaf(v.x - cq.x, gq.x, rho);
                rho = fmaf(v.y - cq.y, gq.y, rho);
                rho = fmaf(v.z - cq.z, gq.z, rho);
                rho = fmaf(v.w - cq.w, gq.w, rho);
            }
            if (!valid) rho = 0.f;
            for (int q = 0; q < Bq; ++q) {
                float4* pv = reinterpret_cast<float4*>(st + g.quad_off(tid, q));
                float4 v = *pv;
                const float4 cq = *reinterpret_cast<const float4*>(&pil[4 * q]);
                float4 x;
                x.x = fmaf(-rho, cq.x, v.x - cq.x);
                x.y = fmaf(-rho, cq.y, v.y - cq.y);
                x.z = fmaf(-rho, cq.z, v.z - cq.z);
                x.w = fmaf(-rho, cq.w, v.w - cq.w);
                if (!valid) x = make_float4(0.f, 0.f, 0.f, 0.f);
                *pv = x;
            }
            rho_s[tid] = rho;
            r1 += (double)rho;
            r2 += (double)rho * (double)rho;
        }
        __syncthreads();
        // (2) 8x8 block outer products (fp32 run over this tile's rows)
        if (active) {
#pragma unroll 1
            for (int r = grp; r < kTileRows; r += a.G1) {
                const float4 a0 = *reinterpret_cast<const float4*>(st + g.quad_off(r, 2 * R));
                const float4 a1 = *reinterpret_cast<const float4*>(st + g.quad_off(r, 2 * R + 1));
                const float4 b0 = *reinterpret_cast<const float4*>(st + g.quad_off(r, 2 * C));
                const float4 b1 = *reinterpret_cast<const float4*>(st + g.quad_off(r, 2 * C + 1));
                const float xa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float xb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[i * 8 + k] = fmaf(xa[i], xb[k], acc[i * 8 + k]);
                if (diag) {
                    const float rho = rho_s[r];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        ms[i] += xa[i];
                        mr[i] = fmaf(rho, xa[i], mr[i]);
                    }
                }
            }
            // (3) flush the fp32 run to fp64 every kFlushTiles1 tiles
            if ((it + 1) % kFlushTiles1 == 0 || it + 1 == ntl) {
#pragma unroll
                for (int i = 0; i < 64; ++i) {
                    acc64[(size_t)i * NA + tid] += (double)acc[i];
                    acc[i] = 0.f;
                }
                if (diag) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        dmine[i] += (double)ms[i];
                        dmine[8 + i] += (double)mr[i];
                        ms[i] = mr[i] = 0.f;
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0 && it + kStages1 < ntl)
            issue_tile(g, stages + s * g.stage_bytes, &full[s], &tm_main, &tm_tail,
                       (t0 + it + kStages1) * kTileRows, c);
    }
    __syncthreads();
    // cross-group reduction in fixed group order
    const int W1 = k1_width(a.nblk);
    double* out = a.part1 + ((size_t)c * a.nch1 + j) * W1;
    for (int e = tid; e < a.nb * 64; e += blockDim.x) {
        const int b = e >> 6, i = e & 63;
        double v = 0.0;
        for (int q = 0; q < a.G1; ++q) v += acc64[(size_t)i * NA + q * a.nb + b];
        out[e] = v;
    }
    // band sums from the diagonal-block threads, fixed group order
    const int Bp = a.nblk * 8;
    for (int b = tid; b < Bp; b += blockDim.x) {
        double sx = 0.0, srx = 0.0;
        for (int q = 0; q < a.G1; ++q) {
            const double* d = dsum + (size_t)(q * a.nblk + (b >> 3)) * 16;
            sx += d[b & 7];
            srx += d[8 + (b & 7)];
        }
        out[a.nb * 64 + b] = sx;
        out[a.nb * 64 + Bp + b] = srx;
    }
    // rho sums from the row owners, fixed order
    if (tid < kTileRows) {
        red_r[tid * 2] = r1;
        red_r[tid * 2 + 1] = r2;
    }
    __syncthreads();
    if (tid == 0) {
        double s1 = 0.0, s2 = 0.0;
        for (int t = 0; t < kTileRows; ++t) {
            s1 += red_r[t * 2];
            s2 += red_r[t * 2 + 1];
        }
        out[a.nb * 64 + 2 * Bp] = s1;
        out[a.nb * 64 + 2 * Bp + 1] = s2;
    }
}

// ---------------------------------------------------------------- shared column state
struct ColState {
    double* mbar;     // [cols][B] mu0
    double* mu;       // [cols][B] mu^k
    double* tprev;    // [cols][B] t^{k-1}
    double* yprev;    // [cols][B] A^-1 t^{k-1}
    double* ainv;     // [cols][B][B] (C0 + rho I)^-1
    double* q64;      // [cols]
    float* z32;       // [cols][B]   z^k
    float* mhat32;    // [cols][B]   mu0 / |mu0|^2
    float* kc32;      // [cols][2]   (mhat.z^k, mu^k.z^k)
    float* q32;       // [cols]
    int* status;      // [cols]
    const float* s;   // [B] unit absorption spectrum
};

// Deterministic block reduction of NV values per thread (fixed order).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch /* [32][NV] */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) scratch[w * NV + i] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double t = 0.0;
        for (int q = 0; q < nw; ++q) t += scratch[q * NV + i];
        v[i] = t;
    }
}

// ---------------------------------------------------------------- K2 init
struct InitArgs {
    ColState cs;
    const float* pilot;
    const double* part1;
    double* mean_out;   // optional [cols][B] (smf_initial_statistics)
    double* cov_out;    // optional [cols][B][B]
    int cols, N, B, nch1, nblk, use_albedo, stats_only;
    double ridge_rel;
};

__host__ inline size_t k2_init_smem(int B) { return (size_t)B * B * 8 + 6 * (size_t)B * 8 + 32 * 4 * 8; }

__global__ void __launch_bounds__(256) k2_init(InitArgs a) {
    extern __shared__ double sm2[];
    const int B = a.B, tid = threadIdx.x, c = blockIdx.x;
    double* A = sm2;               // [B][B]
    double* dm = A + B * B;        // [B] mean of L - c, later mu0
    double* srx = dm + B;          // [B] sum rho x
    double* cv = srx + B;          // [B] pilot c
    double* rowj = cv + B;         // [B]
    double* colj = rowj + B;       // [B]
    double* vt = colj + B;         // [B] t0
    double* scratch = vt + B;      // [32][4]
    __shared__ int bad;
    __shared__ double sh_tol, sh_mm, sh_r1, sh_r2;
    const int nb = a.nblk * (a.nblk + 1) / 2, Bp = a.nblk * 8;
    const int W1 = k1_width(a.nblk);
    const double* P = a.part1 + (size_t)c * a.nch1 * W1;
    const double invN = 1.0 / (double)a.N;
    if (tid == 0) {
        bad = COL_OK;
        double s1 = 0.0, s2 = 0.0;
        for (int j = 0; j < a.nch1; ++j) {
            s1 += P[(size_t)j * W1 + nb * 64 + 2 * Bp];
            s2 += P[(size_t)j * W1 + nb * 64 + 2 * Bp + 1];
        }
        sh_r1 = s1;
        sh_r2 = s2;
    }
    __syncthreads();
    // sum (L - c) = sum x + (sum rho) c ;  dm = mean(L) - c
    for (int b = tid; b < B; b += blockDim.x) {
        double sx = 0.0, sr = 0.0;
        for (int j = 0; j < a.nch1; ++j) {
            sx += P[(size_t)j * W1 + nb * 64 + b];
            sr += P[(size_t)j * W1 + nb * 64 + Bp + b];
        }
        cv[b] = (double)a.pilot[(size_t)c * B + b];
        srx[b] = sr;
        dm[b] = (sx + sh_r1 * cv[b]) * invN;
    }
    __syncthreads();
    // sum (L-c)(L-c)^T = Sxx + Srx c^T + c Srx^T + Srr c c^T ;  C0 = that/N - dm dm^T
    int nonfinite = 0;
    for (int e = tid; e < B * B; e += blockDim.x) {
        int i = e / B, k = e % B;
        if (i < k) continue;
        int R = i >> 3, C = k >> 3;
        int off = (R * (R + 1) / 2 + C) * 64 + (i & 7) * 8 + (k & 7);
        double sxx = 0.0;
        for (int j = 0; j < a.nch1; ++j) sxx += P[(size_t)j * W1 + off];
        double s2 = sxx + srx[i] * cv[k] + cv[i] * srx[k] + sh_r2 * cv[i] * cv[k];
        double v = s2 * invN - dm[i] * dm[k];
        if (!isfinite(v)) nonfinite = 1;
        A[i * B + k] = v;
        A[k * B + i] = v;
    }
    for (int b = tid; b < B; b += blockDim.x)
        if (!isfinite(dm[b])) nonfinite = 1;
    if (nonfinite) atomicExch(&bad, COL_NONFINITE);
    __syncthreads();
    for (int b = tid; b < B; b += blockDim.x) {
        double m = cv[b] + dm[b];
        a.cs.mbar[(size_t)c * B + b] = m;
        a.cs.mu[(size_t)c * B + b] = m;
        if (a.mean_out) a.mean_out[(size_t)c * B + b] = m;
        dm[b] = m;   // dm now holds mu0
    }
    if (a.cov_out)
        for (int e = tid; e < B * B; e += blockDim.x) a.cov_out[(size_t)c * B * B + e] = A[e];
    if (a.stats_only) return;
    __syncthreads();
    // ridge (reading C9): rho = ridge_rel * tr(C0)/B; singularity tolerance as the oracle's Cholesky
    if (tid == 0) {
        double tr = 0.0, amax = 0.0;
        for (int b = 0; b < B; ++b) tr += A[b * B + b];
        double rho = a.ridge_rel * tr / (double)B;
        for (int b = 0; b < B; ++b) {
            A[b * B + b] += rho;
            amax = fmax(amax, A[b * B + b]);
        }
        sh_tol = (double)B * 2.220446049250313e-16 * amax;
    }
    {
        double mm_loc[1] = {0.0};
        for (int b = tid; b < B; b += blockDim.x) mm_loc[0] += dm[b] * dm[b];
        block_sum<1>(mm_loc, scratch);
        if (tid == 0) {
            if (bad == COL_OK && a.use_albedo && !(mm_loc[0] > 0.0)) bad = COL_DEGENERATE_MEAN;
            sh_mm = mm_loc[0];
        }
    }
    __syncthreads();
    // in-place Gauss-Jordan inverse of the SPD matrix A = C0 + rho I (no pivoting;
    // pivot j equals the j-th Cholesky pivot squared, checked like the oracle's)
    for (int j = 0; j < B && bad == COL_OK; ++j) {
        for (int k = tid; k < B; k += blockDim.x) {
            rowj[k] = A[j * B + k];
            colj[k] = A[k * B + j];
        }
        __syncthreads();
        const double piv = rowj[j];
        if (!(piv > sh_tol) || !isfinite(piv)) {
            if (tid == 0) bad = COL_NOT_SPD;
            __syncthreads();
            break;
        }
        const double p = 1.0 / piv;
        for (int e = tid; e < B * B; e += blockDim.x) {
            int i = e / B, k = e % B;
            double v;
            if (i == j && k == j) v = p;
            else if (i == j) v = rowj[k] * p;
            else if (k == j) v = -colj[i] * p;
            else v = A[e] - colj[i] * rowj[k] * p;
            A[e] = v;
        }
        __syncthreads();
    }
    int st = bad;
    const double mm = sh_mm;
    // A^-1 to global; t0 = mu0 (.) s; y = A^-1 t0
    for (int e = tid; e < B * B; e += blockDim.x) a.cs.ainv[(size_t)c * B * B + e] = A[e];
    for (int b = tid; b < B; b += blockDim.x) {
        vt[b] = dm[b] * (double)a.cs.s[b];
        const float mh = (float)(dm[b] / mm);
        a.cs.mhat32[(size_t)c * B + b] = mh;
        rowj[b] = (double)mh;   // the fp32 mhat the sweep uses
    }
    __syncthreads();
    double qc[3] = {0.0, 0.0, 0.0};
    for (int b = tid; b < B; b += blockDim.x) {
        double y = 0.0;
        for (int i = 0; i < B; ++i) y += A[i * B + b] * vt[i];
        const float z32 = (float)y;
        a.cs.z32[(size_t)c * B + b] = z32;
        a.cs.tprev[(size_t)c * B + b] = vt[b];
        a.cs.yprev[(size_t)c * B + b] = y;
        qc[0] += vt[b] * y;
        qc[1] += rowj[b] * (double)z32;   // mhat . z (as the sweep sees them)
        qc[2] += dm[b] * (double)z32;     // mu0 . z
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

// ---------------------------------------------------------------- K2 update
// K3 partial layout per (CTA, column slot), fp64, width B + 3:
//   [0] sum beta, [1] sum beta^2, [2] sum beta s, [3 + b] sum beta L'_b
// with s_i = r_i |mu0|^2 (as fp32) and L'_i = L_i - s_i mhat (albedo-centred radiance).
struct UpdateArgs {
    ColState cs;
    const double* part3;   // [G][S][B+3]
    int cols, N, B, tpc, G, S;
    long long ttot;
};

__host__ __device__ __forceinline__ long long tile_begin(long long b, long long ttot, int G) {
    return b * ttot / G;
}

// Solve the 3x3 system K x = v by Gaussian elimination with partial pivoting.
__device__ __forceinline__ bool solve3(double K[3][3], double v[3], double x[3]) {
    for (int col = 0; col < 3; ++col) {
        int piv = col;
        for (int r = col + 1; r < 3; ++r)
            if (fabs(K[r][col]) > fabs(K[piv][col])) piv = r;
        if (!(fabs(K[piv][col]) > 0.0)) return false;
        if (piv != col) {
            for (int k = 0; k < 3; ++k) {
                double t = K[col][k];
                K[col][k] = K[piv][k];
                K[piv][k] = t;
            }
            double t = v[col];
            v[col] = v[piv];
            v[piv] = t;
        }
        for (int r = col + 1; r < 3; ++r) {
            double f = K[r][col] / K[col][col];
            for (int k = col; k < 3; ++k) K[r][k] -= f * K[col][k];
            v[r] -= f * v[col];
        }
    }
    for (int r = 2; r >= 0; --r) {
        double s = v[r];
        for (int k = r + 1; k < 3; ++k) s -= K[r][k] * x[k];
        x[r] = s / K[r][r];
    }
    return isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]);
}

__global__ void __launch_bounds__(128) k2_update(UpdateArgs a) {
    const int B = a.B, tid = threadIdx.x, c = blockIdx.x;
    __shared__ double sh_t[128], sh_h[128];
    __shared__ double scratch[32 * 9];
    __shared__ double sh_coef[3];
    __shared__ double sh_s[3];
    __shared__ int sh_st;
    ColState& cs = a.cs;
    const int st0 = cs.status[c];
    if (st0 != COL_OK) return;   // uniform per block
    // 1. sufficient statistics of sweep k-1 (fixed CTA order)
    const long long c0 = (long long)c * a.tpc, c1 = c0 + a.tpc;
    int b0 = (int)((c0 * a.G) / a.ttot);
    while (b0 > 0 && tile_begin(b0, a.ttot, a.G) > c0) --b0;
    while (tile_begin(b0 + 1, a.ttot, a.G) <= c0) ++b0;
    const int W = B + 3;
    double sv = 0.0, s0 = 0.0, s2 = 0.0, ss = 0.0;
    for (int b = b0; b < a.G && tile_begin(b, a.ttot, a.G) < c1; ++b) {
        const int slot = c - (int)(tile_begin(b, a.ttot, a.G) / a.tpc);
        const double* P = a.part3 + ((size_t)b * a.S + slot) * W;
        if (tid < B) sv += P[3 + tid];
        if (tid == 0) {
            s0 += P[0];
            s2 += P[1];
            ss += P[2];
        }
    }
    if (tid == 0) {
        sh_s[0] = s0;
        sh_s[1] = s2;
        sh_s[2] = ss;
    }
    __syncthreads();
    const double invN = 1.0 / (double)a.N;
    const double bbar = sh_s[0] * invN, b2 = sh_s[1] * invN, bs = sh_s[2] * invN;
    double mb = 0.0, tp = 0.0, t = 0.0, h = 0.0, mu = 0.0, yp = 0.0, mh = 0.0;
    if (tid < B) {
        const size_t o = (size_t)c * B + tid;
        mb = cs.mbar[o];
        tp = cs.tprev[o];
        yp = cs.yprev[o];
        mh = (double)cs.mhat32[o];
        // h = (1/N) sum beta (L - mu0) = (1/N)[sum beta L' + (sum beta s) mhat] - bbar mu0
        h = sv * invN + (bs * mh - bbar * mb);
        mu = mb - bbar * tp;                 // Eq. 10 / line 10
        t = mu * (double)cs.s[tid];          // Eq. 9
        sh_t[tid] = t;
        sh_h[tid] = h;
    }
    __syncthreads();
    // 2. y_t = A^-1 t, y_h = A^-1 h  (A^-1 symmetric: row i, column = tid -> coalesced)
    double yt = 0.0, yh = 0.0;
    if (tid < B) {
        const double* Ai = cs.ainv + (size_t)c * B * B + tid;
#pragma unroll 8
        for (int i = 0; i < B; ++i) {
            const double v = Ai[(size_t)i * B];
            yt = fma(v, sh_t[i], yt);
            yh = fma(v, sh_h[i], yh);
        }
    }
    // 3. G_ij = u_i . y_j, u = (t', t, h), y = (A^-1 t', A^-1 t, A^-1 h)
    double gv[9];
    {
        const double u[3] = {tp, t, h}, y[3] = {yp, yt, yh};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) gv[i * 3 + j] = tid < B ? u[i] * y[j] : 0.0;
    }
    block_sum<9>(gv, scratch);
    if (tid == 0) {
        // C^k = C0 + U M U^T, M in the basis (t', t, h)
        const double M[3][3] = {{bbar * bbar, -bbar * bbar, 0.0}, {-bbar * bbar, b2, -1.0}, {0.0, -1.0, 0.0}};
        double K[3][3], v[3], x[3];
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j) {
                double s = (i == j) ? 1.0 : 0.0;
                for (int l = 0; l < 3; ++l) s += gv[i * 3 + l] * M[l][j];
                K[i][j] = s;
            }
            v[i] = gv[i * 3 + 1];   // u_i^T A^-1 t
        }
        int st = COL_OK;
        if (!solve3(K, v, x)) st = COL_NOT_SPD;
        for (int i = 0; i < 3; ++i) {
            double s = 0.0;
            for (int l = 0; l < 3; ++l) s += M[i][l] * x[l];
            sh_coef[i] = s;
        }
        sh_st = st;
    }
    __syncthreads();
    // 4. z = y_t - Y M (I + G M)^-1 U^T A^-1 t   (Woodbury)
    double z = 0.0;
    float z32 = 0.f;
    if (tid < B) {
        z = yt - (yp * sh_coef[0] + yt * sh_coef[1] + yh * sh_coef[2]);
        z32 = (float)z;
    }
    double qc[3] = {tid < B ? t * z : 0.0, tid < B ? mh * (double)z32 : 0.0, tid < B ? mu * (double)z32 : 0.0};
    block_sum<3>(qc, scratch);
    int st = sh_st;
    if (st == COL_OK && (!(qc[0] > 0.0) || !isfinite(qc[0]) || !isfinite(qc[1]) || !isfinite(qc[2])))
        st = COL_DEGENERATE_TARGET;
    if (tid < B) {
        const size_t o = (size_t)c * B + tid;
        cs.z32[o] = z32;
        cs.tprev[o] = t;
        cs.yprev[o] = yt;
        cs.mu[o] = mu;
    }
    if (tid == 0) {
        cs.q64[c] = qc[0];
        cs.q32[c] = (float)qc[0];
        cs.kc32[2 * c] = (float)qc[1];
        cs.kc32[2 * c + 1] = (float)qc[2];
        cs.status[c] = st;
    }
}

// ---------------------------------------------------------------- K3 sweep
struct SweepArgs {
    float* enh;            // [cols][N] alpha (read alpha^{k-1}, write alpha^k)
    float* alb;            // [cols][N] albedo r (written at k = 0)
    const float* z32;
    const float* mhat32;
    const float* kc32;
    const float* q32;
    const double* mm64;    // unused placeholder (|mu0|^2 derived from mhat)
    const int* status;
    double* part3;         // [G][S][B+3]
    int cols, N, B, tpc, G, S;
    long long ttot;
    int k, n_iter, use_sparsity, use_albedo;
    float eps, r_floor;
};

template <int NQ>
struct SweepGeom {
    static constexpr int NFULL = NQ / 8;
    static constexpr int TQ = NQ % 8;
    static constexpr int TAILW = TQ == 0 ? 0 : (TQ <= 2 ? 8 : (TQ <= 4 ? 16 : 32));
    static constexpr int STAGE = ((kTileRows * (NFULL * 128 + TAILW * 4)) + 1023) / 1024 * 1024;
    static constexpr uint32_t TX = kTileRows * (NFULL * 128 + TAILW * 4);
    static __device__ __forceinline__ uint32_t quad_off(int r, int q) {
        if (q < NFULL * 8) return (q >> 3) * (kTileRows * 128) + swz_off(r, q & 7, 128);
        return NFULL * (kTileRows * 128) + swz_off(r, q - NFULL * 8, TAILW * 4);
    }
};

template <int NQ>
__global__ void __launch_bounds__(kTileRows, 2)
    k3_sweep(const __grid_constant__ CUtensorMap tm_main, const __grid_constant__ CUtensorMap tm_tail,
             SweepArgs a) {
    using Gm = SweepGeom<NQ>;
    constexpr int B4 = NQ * 4;
    constexpr int W = B4 + 3;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* stages = align1024(smem_raw);
    __shared__ uint64_t full[kStages];
    __shared__ __align__(16) float zs[B4];
    __shared__ __align__(16) float ms[B4];
    __shared__ double red[kTileRows / 32][W];
    __shared__ float sh_par[4];
    __shared__ int sh_st;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long tb = tile_begin(blockIdx.x, a.ttot, a.G), te = tile_begin(blockIdx.x + 1, a.ttot, a.G);
    const int ntl = (int)(te - tb);
    const int cfirst = (int)(tb / a.tpc);
    const bool accum = a.k < a.n_iter;

    if (tid == 0) {
        prefetch_tmap(&tm_main);
        if (Gm::TAILW) prefetch_tmap(&tm_tail);
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int i) {
        const long long g = tb + i;
        const int c = (int)(g / a.tpc), row0 = (int)(g % a.tpc) * kTileRows;
        unsigned char* st = stages + (i % kStages) * Gm::STAGE;
        uint64_t* bar = &full[i % kStages];
        mbar_arrive_expect_tx(bar, Gm::TX);
#pragma unroll
        for (int f = 0; f < Gm::NFULL; ++f) tma_load_3d(st + f * (kTileRows * 128), &tm_main, bar, f * 32, row0, c);
        if (Gm::TAILW) tma_load_3d(st + Gm::NFULL * (kTileRows * 128), &tm_tail, bar, Gm::NFULL * 32, row0, c);
    };
    if (tid == 0)
        for (int i = 0; i < kStages && i < ntl; ++i) issue(i);

    float acc[B4];
#pragma unroll
    for (int i = 0; i < B4; ++i) acc[i] = 0.f;
    float sb = 0.f, sb2 = 0.f, sbs = 0.f;

    auto flush = [&](int slot) {
        // fixed-order warp butterfly, then fp64 across warps -> part3[blockIdx][slot]
#pragma unroll
        for (int i = 0; i < B4; ++i) {
            float v = acc[i];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            acc[i] = v;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            sb += __shfl_xor_sync(0xffffffffu, sb, off);
            sb2 += __shfl_xor_sync(0xffffffffu, sb2, off);
            sbs += __shfl_xor_sync(0xffffffffu, sbs, off);
        }
        if (lane == 0) {
            red[wid][0] = sb;
            red[wid][1] = sb2;
            red[wid][2] = sbs;
#pragma unroll
            for (int i = 0; i < B4; ++i) red[wid][3 + i] = acc[i];
        }
        __syncthreads();
        if (tid < W) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < kTileRows / 32; ++q) s += red[q][tid];
            a.part3[((size_t)blockIdx.x * a.S + slot) * W + tid] = s;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < B4; ++i) acc[i] = 0.f;
        sb = sb2 = sbs = 0.f;
    };

    int cur = -1;
    float mz = 0.f, cz = 0.f, q = 1.f, mmf = 1.f;
    int cst = 0;
    for (int i = 0; i < ntl; ++i) {
        const long long g = tb + i;
        const int c = (int)(g / a.tpc);
        const int row0 = (int)(g % a.tpc) * kTileRows;
        if (c != cur) {
            if (cur >= 0 && accum) flush(cur - cfirst);
            if (tid < B4) {
                zs[tid] = a.z32[(size_t)c * a.B + tid];
                ms[tid] = a.mhat32[(size_t)c * a.B + tid];
            }
            if (tid == 0) {
                sh_par[0] = a.kc32[2 * c];       // mhat . z
                sh_par[1] = a.kc32[2 * c + 1];   // mu^k . z
                sh_par[2] = a.q32[c];
                sh_st = a.status[c];
            }
            __syncthreads();
            if (tid == 0) {
                // |mu0|^2 in fp32 from mhat (1/|mhat|^2), identical for every thread
                float s2 = 0.f;
                for (int b = 0; b < B4; ++b) s2 = fmaf(ms[b], ms[b], s2);
                sh_par[3] = s2 > 0.f ? 1.f / s2 : 0.f;
            }
            __syncthreads();
            mz = sh_par[0];
            cz = sh_par[1];
            q = sh_par[2];
            mmf = sh_par[3];
            cst = sh_st;
            cur = c;
        }
        const int p = row0 + tid;
        const bool valid = p < a.N;
        const size_t pix = (size_t)c * a.N + p;
        float aprev = 0.f;
        if (valid && a.k > 0 && a.use_sparsity && cst == COL_OK) aprev = a.enh[pix];
        const int s = i % kStages;
        mbar_wait(&full[s], (i / kStages) & 1);
        if (valid) {
            if (cst != COL_OK) {
                a.enh[pix] = __int_as_float(0x7fc00000);
                a.alb[pix] = __int_as_float(0x7fc00000);
            } else {
                const unsigned char* st = stages + s * Gm::STAGE;
                float4 Lq[NQ];
#pragma unroll
                for (int m = 0; m < NQ; ++m) Lq[m] = *reinterpret_cast<const float4*>(st + Gm::quad_off(tid, m));
                // albedo factor r = L.mhat (Eq. 7, mhat = mu0/|mu0|^2)
                float dm[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int m = 0; m < NQ; ++m) {
                    const float4 mq = *reinterpret_cast<const float4*>(&ms[4 * m]);
                    dm[m & 3] = dot4(Lq[m], mq, dm[m & 3]);
                }
                const float r = (dm[0] + dm[1]) + (dm[2] + dm[3]);
                // albedo-centred radiance L' = L - s mhat, s = r |mu0|^2 (removes the
                // component along mu0; the projection and the sums use L')
                const float sc = r * mmf;
                float dz[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int m = 0; m < NQ; ++m) {
                    const float4 mq = *reinterpret_cast<const float4*>(&ms[4 * m]);
                    const float4 zq = *reinterpret_cast<const float4*>(&zs[4 * m]);
                    Lq[m].x = fmaf(-sc, mq.x, Lq[m].x);
                    Lq[m].y = fmaf(-sc, mq.y, Lq[m].y);
                    Lq[m].z = fmaf(-sc, mq.z, Lq[m].z);
                    Lq[m].w = fmaf(-sc, mq.w, Lq[m].w);
                    dz[m & 3] = dot4(Lq[m], zq, dz[m & 3]);
                }
                // (L - mu^k).z = L'.z + s (mhat.z) - mu^k.z
                const float pz = ((dz[0] + dz[1]) + (dz[2] + dz[3])) + fmaf(sc, mz, -cz);
                const float rr = a.use_albedo ? r : 1.f;
                const float rt = a.use_albedo ? fmaxf(r, a.r_floor) : 1.f;
                float out;
                if (a.k == 0) {
                    const float a0 = pz / (rt * q);                        // line 6
                    out = a.n_iter == 0 ? a0 : (a0 > 0.f ? a0 : 0.f);      // reading C3
                    a.alb[pix] = rr;
                } else {
                    const float w = a.use_sparsity ? 1.f / (aprev + a.eps) : 0.f;   // Eq. 5
                    const float x = (pz - w) / (rt * q);                             // line 16
                    out = x > 0.f ? x : 0.f;                                         // reading C14
                }
                a.enh[pix] = out;
                if (accum) {
                    const float beta = rt * out;
                    sb += beta;
                    sb2 = fmaf(beta, beta, sb2);
                    sbs = fmaf(beta, sc, sbs);
#pragma unroll
                    for (int m = 0; m < NQ; ++m) {
                        acc[4 * m + 0] = fmaf(beta, Lq[m].x, acc[4 * m + 0]);
                        acc[4 * m + 1] = fmaf(beta, Lq[m].y, acc[4 * m + 1]);
                        acc[4 * m + 2] = fmaf(beta, Lq[m].z, acc[4 * m + 2]);
                        acc[4 * m + 3] = fmaf(beta, Lq[m].w, acc[4 * m + 3]);
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0 && i + kStages < ntl) issue(i + kStages);
    }
    if (cur >= 0 && accum) flush(cur - cfirst);
}

// ---------------------------------------------------------------- misc
__global__ void k_copy_status(const int* src, int32_t* dst, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i];
}

struct ModelArgs {
    const double* mu;
    const double* q64;
    double* mu_out;
    double* q_out;
    int cols, B;
};

__global__ void k_column_model(ModelArgs a) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (a.mu_out && i < a.cols * a.B) a.mu_out[i] = a.mu[i];
    if (a.q_out && i < a.cols) a.q_out[i] = a.q64[i];
}

}  // namespace smf
