// wide_chol.cuh -- the wide path's factorisation (Fig. alg line 16's (C + rho I)^-1 products,
// P:358-381) as a Cholesky factor A0 = C0 + rho I = L L^T instead of an explicit inverse:
//
//  wide_cholesky   in-place right-looking blocked Cholesky of one column's A0 (row-major B x B
//                  in global memory, lower triangle) by one CTA: a warp factors each 32 x 32
//                  diagonal block in shared memory (pivot test of reading C16': a pivot <= tol
//                  is NOT_SPD, as the oracle's Cholesky), a thread per row solves the panel
//                  L_iK = A_iK L_KK^-T with the inverted diagonal block, and 4 x 4 register
//                  tiles of the lower trailing triangle take A_ij -= L_iK . L_jK (j <= i)
//                  with the panel staged in shared memory.
//                  B^3/6 FMA -- a sixth of the Gauss-Jordan inverse it replaces -- and the
//                  shrinking trailing triangle is the only global traffic.
//  tri_fwd<NR>     L x = b for NR right-hand sides: per 32-row block an off-diagonal GEMV
//                  with every load of the block in flight at once (threads stride columns,
//                  a transpose-reduction per 16 rows), then x_J = L_JJ^-1 y_J with the
//                  inverted diagonal block stored in the factor (no sequential chain).
//  tri_bwd<NR>     L^T x = b, the same on the mirrored upper triangle (L^T stored there, so
//                  the backward GEMV also reads rows).
// The Woodbury update needs A0^-1 only through G = U^T A0^-1 U = W^T W with
// W = L^-1 U (forward solves) and z = L^-T (L^-1 t - W coef) (one backward solve), so the
// per-iteration reads of L are the same bytes the explicit inverse cost.
#pragma once
#include <cstdint>

namespace smf {

constexpr int kChB = 32;         // block width of the factorisation and the solves
// row stride of the stored factor: even, so every row is 16-byte aligned (the solves read
// row segments as double2)
__host__ __device__ inline int wide_ld(int B) { return (B + 1) & ~1; }
constexpr int kChD = kChB + 1;   // padded row stride of the shared diagonal block

// Factor and invert the diagonal block at k0 (nb <= 32 rows) by the calling warp. Lane l holds
// row l in registers; the column loop is rolled and the row registers rotate one place per
// step, so the current column is always r[0] and every register index is a compile-time
// constant (the inner 31-wide updates are unrolled: independent FMAs fed by shuffles). The
// fully unrolled 32 x 32 version (~20 K straight-line instructions per call, on the
// look-ahead's critical path once per panel step) was instruction-fetch bound inside the
// kernel (`scripts/micro/diag_bench.cu` times one call in isolation: 13.7 us now). The pivot
// uses the hardware reciprocal square root with Newton steps (the IEEE sqrt and division are
// long software sequences on this serial chain). The inverse (lane c computes column c of
// L_KK^-1, right-looking with the reciprocal pivots) rotates the same way. Writes L to D and
// L^-1 to Dinv (lower triangles, zeros elsewhere). Returns false (warp-uniformly) on a pivot
// <= tol or non-finite.
__device__ __forceinline__ bool chol_diag_warp(const double* A, int B, int k0, int nb, double tol, double* D,
                                            double* Dinv) {
    const int lane = threadIdx.x & 31;
    const double* Ar = A + (size_t)(k0 + (lane < nb ? lane : 0)) * wide_ld(B) + k0;
    double r[kChB];
#pragma unroll
    for (int m = 0; m < kChB; ++m) r[m] = (lane < nb && m <= lane) ? Ar[m] : 0.0;
    bool ok = true;
    double rdl = 0.0;   // lane j: 1 / L_jj
#pragma unroll 1
    for (int j = 0; j < nb; ++j) {
        const double d = __shfl_sync(0xffffffffu, r[0], j);
        if (!(d > tol) || !isfinite(d)) ok = false;   // warp-uniform (the factor is then discarded)
        // 1/sqrt(d) by the hardware reciprocal-square-root seed and Newton steps, g = d / sqrt(d):
        // the IEEE sqrt and division are software sequences of ~1000 cycles each on this
        // critical path (one pivot after another); ~1 ulp apart from them
        const double ginv = rsqrt(d);
        const double g = d * ginv;
        if (lane == j) {
            r[0] = g;
            rdl = ginv;   // reciprocal pivot for the inverse below
        }
        else if (lane > j) r[0] *= ginv;   // L_lj
        const double lj = r[0];
#pragma unroll
        for (int m = 1; m < kChB; ++m) {   // original column j + m
            const double lmj = __shfl_sync(0xffffffffu, r[0], (j + m) & 31);
            if (lane >= j + m) r[m] = fma(-lj, lmj, r[m]);
        }
        D[lane * kChD + j] = r[0];   // column j of row `lane` is final
#pragma unroll
        for (int m = 0; m < kChB - 1; ++m) r[m] = r[m + 1];
        r[kChB - 1] = 0.0;
    }
    for (int j = nb; j < kChB; ++j) D[lane * kChD + j] = 0.0;
    __syncwarp();
    if (ok) {
        double x[kChB];   // x[i] = row k + i of column `lane` at step k
#pragma unroll
        for (int i = 0; i < kChB; ++i) x[i] = (i == lane && i < nb) ? 1.0 : 0.0;
#pragma unroll 1
        for (int k = 0; k < nb; ++k) {
            const double xk = x[0] * __shfl_sync(0xffffffffu, rdl, k);
            Dinv[k * kChD + lane] = xk;
            const double* Dk = D + k;   // column k of L, rows k + i
#pragma unroll
            for (int i = 1; i < kChB; ++i) {
                const double l = k + i < nb ? Dk[(k + i) * kChD] : 0.0;
                x[i] = fma(-l, xk, x[i]);
            }
#pragma unroll
            for (int i = 0; i < kChB - 1; ++i) x[i] = x[i + 1];
            x[kChB - 1] = 0.0;
        }
        for (int i = nb; i < kChB; ++i) Dinv[i * kChD + lane] = 0.0;
    }
    __syncwarp();
    return ok;
}

// The panel Cp holds row r's 32 values as 16 double2 pairs, pair s2 at slot s2 ^ cp_swz(r): the
// trailing tiles of a warp read rows 4 apart (tile columns J, J + 1, ...), which an unswizzled
// stride maps onto the same banks.
__device__ __forceinline__ int cp_swz(int r) { return (r >> 2) & 7; }

// 4 x 4 register tile (I, J) of the trailing update A_ij -= Cp_i . Cp_j (j <= i) below row
// and right of column t0 (tile rows t0 + 4I.., columns t0 + 4J..; t0 is a multiple of 4, so
// a tile's four rows share one swizzle).
__device__ __forceinline__ void chol_tile(double* A, int B, int t0, int I, int J, const double* Cp) {
    const int i0 = t0 + 4 * I, j0 = t0 + 4 * J;
    double acc[4][4];
#pragma unroll
    for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) acc[a2][b2] = 0.0;
    const double2* ri[4];
    const double2* rj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        ri[q] = reinterpret_cast<const double2*>(Cp + min(i0 + q, B - 1) * kChB);
        rj[q] = reinterpret_cast<const double2*>(Cp + min(j0 + q, B - 1) * kChB);
    }
    const int dg = cp_swz(i0) ^ cp_swz(j0);   // slot p of row i pairs with slot p ^ dg of row j
    double old[4][4];   // the 16 old values in flight while the products accumulate
#pragma unroll
    for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) {
            const int i = i0 + a2, j = j0 + b2;
            old[a2][b2] = (i < B && j <= i) ? A[(size_t)i * wide_ld(B) + j] : 0.0;
        }
#pragma unroll 4
    for (int p = 0; p < kChB / 2; ++p) {
        double2 va[4], vb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            va[q] = ri[q][p];
            vb[q] = rj[q][p ^ dg];
        }
#pragma unroll
        for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2)
                acc[a2][b2] = fma(va[a2].y, vb[b2].y, fma(va[a2].x, vb[b2].x, acc[a2][b2]));
    }
#pragma unroll
    for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) {
            const int i = i0 + a2, j = j0 + b2;
            if (i < B && j <= i) A[(size_t)i * wide_ld(B) + j] = old[a2][b2] - acc[a2][b2];
        }
}

__device__ __forceinline__ void tri_decode(int e, int& I, int& J) {
    I = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
    while ((I + 1) * (I + 2) / 2 <= e) ++I;
    while (I * (I + 1) / 2 > e) --I;
    J = e - I * (I + 1) / 2;
}

// In-place Cholesky of A (row-major B x B, global; the lower triangle holds A on entry).
// On exit the matrix holds the solve-ready factor M:
//   off-diagonal blocks, lower: L;  upper: L^T (mirrored, so both solves read rows);
//   diagonal blocks: lower (incl. diagonal) L_KK^-1, strictly upper (L_KK^-1)^T.
// Look-ahead: once the trailing update has finished the next block column, warp 0 factors
// the next diagonal block while the other warps apply the rest of the trailing update.
// D, Dinv: shared [kChB][kChD]; Cp: shared [B][kChB] (16-byte aligned, swizzled pairs); flag:
// shared int. Returns false (uniformly) on a non-positive or non-finite pivot (<= tol).

__device__ bool wide_cholesky(double* A, int B, double tol, double* D, double* Dinv, double* Cp, int* flag) {
    const int tid = threadIdx.x, nt = blockDim.x, wid = tid >> 5;
    if (tid == 0) *flag = 0;
    __syncthreads();
    if (wid == 0 && !chol_diag_warp(A, B, 0, min(kChB, B), tol, D, Dinv) && (tid & 31) == 0) *flag = 1;
    __syncthreads();
    if (*flag) return false;
    for (int k0 = 0; k0 < B; k0 += kChB) {
        const int nb = min(kChB, B - k0);
        // (a) the factored block (D, Dinv) is final: write L_KK^-1 and its transpose
        for (int e = tid; e < nb * nb; e += nt) {
            const int r = e / nb, cc = e - r * nb;
            A[(size_t)(k0 + r) * wide_ld(B) + k0 + cc] = cc <= r ? Dinv[r * kChD + cc] : Dinv[cc * kChD + r];
        }
        // (b) panel: x = a L_KK^-T for every row below the block (thread per row), staged in
        // Cp, written to the lower part and mirrored (L^T) into the upper part
        for (int i = k0 + nb + tid; i < B; i += nt) {
            double a_[kChB];
            double* Ai = A + (size_t)i * wide_ld(B) + k0;
#pragma unroll
            for (int s = 0; s < kChB; ++s) a_[s] = s < nb ? Ai[s] : 0.0;
#pragma unroll
            for (int s = 0; s < kChB; ++s) {
                double v = 0.0;
                if (s < nb) {
#pragma unroll
                    for (int t = 0; t <= s; ++t) v = fma(a_[t], Dinv[s * kChD + t], v);
                    Ai[s] = v;
                    A[(size_t)(k0 + s) * wide_ld(B) + i] = v;
                }
                Cp[i * kChB + (((s >> 1) ^ cp_swz(i)) << 1) + (s & 1)] = v;   // zero past nb
            }
        }
        __syncthreads();
        const int t0 = k0 + nb;
        if (t0 >= B) break;
        const int T = B - t0, n4 = (T + 3) >> 2, nb2 = min(kChB, T), c4 = (nb2 + 3) >> 2;
        // (c1) the trailing tiles of the next block column (tile columns J < c4, rows I >= J)
        {
            const int tri = c4 * (c4 + 1) / 2, n1 = tri + (n4 - c4) * c4;
            for (int e = tid; e < n1; e += nt) {
                int I, J;
                if (e < tri) {
                    tri_decode(e, I, J);
                } else {
                    I = c4 + (e - tri) / c4;
                    J = (e - tri) % c4;
                }
                chol_tile(A, B, t0, I, J, Cp);
            }
        }
        __syncthreads();
        // (a') warp 0 factors the next diagonal block while (c2) the other warps update the
        // rest of the trailing triangle (tile columns J >= c4)
        if (wid == 0) {
            if (!chol_diag_warp(A, B, t0, nb2, tol, D, Dinv) && (tid & 31) == 0) *flag = 1;
        } else {
            const int m = n4 - c4, n2 = m * (m + 1) / 2;
            for (int e = tid - 32; e < n2; e += nt - 32) {
                int I, J;
                tri_decode(e, I, J);
                chol_tile(A, B, t0, I + c4, J + c4, Cp);
            }
        }
        __syncthreads();
        if (*flag) return false;
    }
    return true;
}

// y_r = x_r - sum_{cc in [cs, ce)} M[J0 + r][cc] x[cc] for the nb <= 32 rows of block J0 and NR
// right-hand sides (x: shared [NR][B]); result in yv (shared [NR][32]). blockDim.x / 32 threads
// share a row (a warp covers 32 / tpr rows, the row segments it reads are 8 * tpr bytes wide);
// each thread issues up to 32 of its row's loads at once, so a block step costs one or two
// global round trips; the row's threads reduce with shuffles.
#ifndef SMF_GEMV_BATCH
#define SMF_GEMV_BATCH 16
#endif
constexpr int kGemvBatch = SMF_GEMV_BATCH;   // doubles in flight per thread in the solves' GEMVs
constexpr int kGemvPairs = kGemvBatch / 2;   // ... loaded as double2 pairs

template <int NR>
__device__ __forceinline__ void row_gemv(const double* __restrict__ M, int B, int J0, int nb, int cs, int ce,
                                         const double* x, double* /*red*/, double* yv) {
    const int tid = threadIdx.x, tpr = blockDim.x >> 5;   // threads per row (4 or 8)
    const int r = tid / tpr, cq = tid - r * tpr;
    double acc[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[q] = 0.0;
    // rows are 16-byte aligned (wide_ld): each load fetches a column pair (cc, cc + 1), cc even
    const double* Mr = M + (size_t)(J0 + (r < nb ? r : 0)) * wide_ld(B);
    const int cs2 = cs & ~1;
    for (int base = cs2 + 2 * cq; base < ce; base += 2 * kGemvPairs * tpr) {
        double2 lv[kGemvPairs];
#pragma unroll
        for (int u = 0; u < kGemvPairs; ++u) {
            const int cc = base + 2 * u * tpr;
            lv[u] = (r < nb && cc < ce) ? *reinterpret_cast<const double2*>(Mr + cc) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kGemvPairs; ++u) {
            const int cc = base + 2 * u * tpr;
            const bool ok0 = cc >= cs && cc < ce, ok1 = cc + 1 >= cs && cc + 1 < ce;
            const double l0 = ok0 ? lv[u].x : 0.0, l1 = ok1 ? lv[u].y : 0.0;
            const int c0 = ok0 ? cc : 0, c1 = ok1 ? cc + 1 : 0;
#pragma unroll
            for (int q = 0; q < NR; ++q) acc[q] = fma(l1, x[q * B + c1], fma(l0, x[q * B + c0], acc[q]));
        }
    }
#pragma unroll
    for (int q = 0; q < NR; ++q)
        for (int off = 1; off < tpr; off <<= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
    if (cq == 0 && r < nb)
#pragma unroll
        for (int q = 0; q < NR; ++q) yv[q * 32 + r] = x[q * B + J0 + r] - acc[q];
    __syncthreads();
}

// Stage diagonal block [J0, J0 + nb) of M (lower: L_JJ^-1, upper: its transpose) into Dsm.
__device__ __forceinline__ void stage_diag(const double* __restrict__ M, int B, int J0, int nb, double* Dsm) {
    for (int e = threadIdx.x; e < kChB * kChB; e += blockDim.x) {
        const int i = e >> 5, l = e & 31;
        Dsm[i * kChD + l] = (i < nb && l < nb) ? M[(size_t)(J0 + i) * wide_ld(B) + J0 + l] : 0.0;
    }
}

// L x = b in place for NR (1 or 2) right-hand sides x[nr * B + i] (shared). Whole block;
// Dsm [kChB][kChD], red [nwarps][NR][32], yv [NR][32] shared.
template <int NR>
__device__ void tri_fwd(const double* __restrict__ M, int B, double* x, double* Dsm, double* red, double* yv) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int J0 = 0; J0 < B; J0 += kChB) {
        const int nb = min(kChB, B - J0);
        stage_diag(M, B, J0, nb, Dsm);
        row_gemv<NR>(M, B, J0, nb, 0, J0, x, red, yv);
        __syncwarp();
        if (wid == 0 && lane < nb) {   // x_J = L_JJ^-1 y_J (lower part of the staged block)
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                double v = 0.0;
                for (int r = 0; r <= lane; ++r) v = fma(Dsm[lane * kChD + r], yv[q * 32 + r], v);
                x[q * B + J0 + lane] = v;
            }
        }
        __syncthreads();
    }
}

// L^T x = b in place (the mirrored upper part holds L^T). Same shared buffers as tri_fwd.
template <int NR>
__device__ void tri_bwd(const double* __restrict__ M, int B, double* x, double* Dsm, double* red, double* yv) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nblk = (B + kChB - 1) / kChB;
    for (int jb = nblk - 1; jb >= 0; --jb) {
        const int J0 = jb * kChB, nb = min(kChB, B - J0);
        stage_diag(M, B, J0, nb, Dsm);
        row_gemv<NR>(M, B, J0, nb, J0 + nb, B, x, red, yv);
        __syncwarp();
        if (wid == 0 && lane < nb) {   // x_J = L_JJ^-T y_J (upper part incl. the diagonal)
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                double v = 0.0;
                for (int r = lane; r < nb; ++r) v = fma(Dsm[lane * kChD + r], yv[q * 32 + r], v);
                x[q * B + J0 + lane] = v;
            }
        }
        __syncthreads();
    }
}


// ---------------------------------------------------------------- streamed solves (k2w_update)
// The per-iteration solves read the whole solve-ready factor once forward (lower part, row
// blocks top-down) and once backward (mirrored upper part, bottom-up): 2 x 105 tiles of 32 x 32
// fp64 at B = 425. The tile loads do not depend on the solution, only the FMAs do, so the
// factor is streamed through a ring of S shared-memory stages by TMA (3-D map {B, B, cols} over
// the [cols][B][wide_ld(B)] factor; rows and columns past B are zero-filled) in the exact order
// the solves consume it, and the HBM stream runs ahead of the dependent chain by S tiles --
// across the forward/backward boundary and the 3 x 3 algebra between them too. Thread 0
// issues the loads (it waits on a stage's `empty` barrier, which the four warps arrive on
// after reading the tile); no producer warp, so the 128-thread generic loops are unchanged.
// Consumption: warp w owns tile rows 8w..8w+7, lane = tile column (conflict-free 256-byte
// row reads); per-lane partial sums of the row block are reduced once per row block by a
// butterfly reduce-scatter.
constexpr int kTileD = kChB * kChB;   // doubles per factor tile
#ifndef SMF_K2W_STAGES
#define SMF_K2W_STAGES 2
#endif
constexpr int kTsS = SMF_K2W_STAGES;  // ring depth (k2w_update: five CTAs per SM at B = 425)
// Tiles per stage: the kernel is bound by each warp's instruction latency chain (an mbarrier
// wait, a release and the ring bookkeeping per stage), not by bytes in flight, so a stage holds
// two adjacent off-diagonal tiles of a row block (the last one of an odd count and the
// diagonal tile travel alone): 63 instead of 105 stages per pass at B = 425 for the same
// 32 KB ring as four one-tile stages.
#ifndef SMF_K2W_PAIR
#define SMF_K2W_PAIR 1
#endif
constexpr int kTsT = SMF_K2W_PAIR ? 2 : 1;
constexpr int kStageD = kTsT * kTileD;   // doubles per stage

// Stage index / phase bookkeeping is incremental (no divisions) and the issuing thread walks
// the tile order with a cursor (no triangular decode): thread 0 is also a consumer, so every
// cycle it spends issuing is on warp 0's path.
struct TileStream {
    double* ring;          // [kTsS][kTsT][32][32] shared, 128-byte aligned
    uint64_t* full;        // [kTsS] TMA completion
    uint64_t* empty;       // [kTsS] one arrival per warp
    const CUtensorMap* map;
    int nblk, col;
    int total;             // stages in the whole sequence (forward + backward)
    int consumed;          // every thread: stages consumed (program order)
    int cs, cph;           // every thread: stage and full-barrier phase of the next tile to consume
    // thread 0 (issuer): tiles issued, stage / empty phase of the next issue, tile cursor
    int issued, ps, pph, pI, pJ, pfwd;
};

__device__ __forceinline__ void ts_init(TileStream& ts, double* ring, uint64_t* full, uint64_t* empty,
                                        const CUtensorMap* map, int B, int col, int npass) {
    ts.ring = ring;
    ts.full = full;
    ts.empty = empty;
    ts.map = map;
    ts.nblk = (B + kChB - 1) / kChB;
    ts.col = col;
    int per_pass = 0;   // a row block with n off-diagonal tiles: ceil(n / kTsT) stages + the diagonal's
    for (int n = 0; n < ts.nblk; ++n) per_pass += (n + kTsT - 1) / kTsT + 1;
    ts.total = npass * per_pass;
    ts.consumed = 0;
    ts.cs = 0;
    ts.cph = 0;
    ts.issued = 0;
    ts.ps = 0;
    ts.pph = 0;
    ts.pI = 0;
    ts.pJ = 0;
    ts.pfwd = 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTsS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], blockDim.x >> 5);
        }
        fence_mbar_init();
    }
}

// Thread 0: issue tiles up to (not including) `upto`. Order: forward row blocks I = 0.. with
// J = 0..I (diagonal last), then backward row blocks I = nblk-1..0 with J = nblk-1..I.
__device__ __forceinline__ void ts_issue(TileStream& ts, int upto) {
    while (ts.issued < ts.total && ts.issued < upto) {
        if (ts.issued >= kTsS) {
            mbar_wait(&ts.empty[ts.ps], (uint32_t)ts.pph);   // the stage's previous tile released
            fence_proxy_async();   // the warps' generic reads of the stage before the async refill
        }
        // an off-diagonal tile takes the row block's next off-diagonal tile along
        const int Jn = ts.pfwd ? ts.pJ + 1 : ts.pJ - 1;
        const bool two = kTsT == 2 && ts.pJ != ts.pI && Jn != ts.pI;
        double* dst = ts.ring + (size_t)ts.ps * kStageD;
        mbar_arrive_expect_tx(&ts.full[ts.ps], (two ? 2 : 1) * kTileD * 8);
        tma_load_3d(dst, ts.map, &ts.full[ts.ps], ts.pJ * kChB, ts.pI * kChB, ts.col);
        if (two) {
            tma_load_3d(dst + kTileD, ts.map, &ts.full[ts.ps], Jn * kChB, ts.pI * kChB, ts.col);
            ts.pJ = Jn;   // the cursor step below then leaves the pair
        }
        ++ts.issued;
        if (++ts.ps == kTsS) {
            ts.ps = 0;
            if (ts.issued > kTsS) ts.pph ^= 1;   // the first round of issues waits on no release
        }
        if (ts.pfwd) {
            if (++ts.pJ > ts.pI) {
                ts.pJ = 0;
                if (++ts.pI == ts.nblk) {
                    ts.pfwd = 0;
                    ts.pI = ts.pJ = ts.nblk - 1;
                }
            }
        } else if (--ts.pJ < ts.pI) {
            --ts.pI;
            ts.pJ = ts.nblk - 1;
        }
    }
}

__device__ __forceinline__ const double* ts_acquire(TileStream& ts) {
    if (threadIdx.x == 0) ts_issue(ts, ts.consumed + kTsS);
    mbar_wait(&ts.full[ts.cs], (uint32_t)ts.cph);
    return ts.ring + (size_t)ts.cs * kStageD;
}

__device__ __forceinline__ void ts_release(TileStream& ts) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&ts.empty[ts.cs]);
    ++ts.consumed;
    if (++ts.cs == kTsS) {
        ts.cs = 0;
        ts.cph ^= 1;
    }
}

// Thread 0 waits for every issued tile still in flight (before the ring's memory is reused or
// the CTA exits off the streamed sequence); the caller synchronises the block afterwards.
__device__ __forceinline__ void ts_drain(TileStream& ts) {
    if (threadIdx.x == 0) {
        int s = ts.cs, ph = ts.cph;
        for (int i = ts.consumed; i < ts.issued; ++i) {
            mbar_wait(&ts.full[s], (uint32_t)ph);
            if (++s == kTsS) {
                s = 0;
                ph ^= 1;
            }
        }
    }
}

// One butterfly step of the reduce-scatter: N values -> N/2, keeping the upper half if `up`.
template <int N>
__device__ __forceinline__ void rs_step(double* v, int o, bool up) {
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
        const double send = up ? v[k] : v[k + N / 2];
        const double keep = up ? v[k + N / 2] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
}

// Sum each of V (8, 16 or 32) per-lane values over the warp; lane l ends with the total of value
// l / (32 / V) (every lane of its group of 32 / V lanes holds it).
template <int V>
__device__ __forceinline__ double reduce_scatter(double (&v)[V]) {
    static_assert(V == 8 || V == 16 || V == 32, "reduce_scatter: V in {8, 16, 32}");
    const int lane = threadIdx.x & 31;
    int o = 16;
    if constexpr (V >= 32) { rs_step<32>(v, o, lane & o); o >>= 1; }
    if constexpr (V >= 16) { rs_step<16>(v, o, lane & o); o >>= 1; }
    rs_step<8>(v, o, lane & o); o >>= 1;
    rs_step<4>(v, o, lane & o); o >>= 1;
    rs_step<2>(v, o, lane & o); o >>= 1;
    for (; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    return v[0];
}

// Streamed L x = b (FWD) or L^T x = b (!FWD) in place for NR right-hand sides x [NR][B]
// (shared); yv [NR][32] shared. 128 threads. Consumes the next nblk (nblk + 1) / 2 tiles.
template <int NR, bool FWD>
__device__ __forceinline__ void tri_stream(TileStream& ts, int B, double* x, double* yv) {
    constexpr int V = 8 * NR;
    const int tid = threadIdx.x, lane = tid & 31, r0 = (tid >> 5) * 8;
    const int nblk = ts.nblk;
    const int idx = lane / (32 / V), ri = r0 + idx / NR, qi = idx % NR;
    const bool writer = (lane & (32 / V - 1)) == 0;
    for (int step = 0; step < nblk; ++step) {
        const int I = FWD ? step : nblk - 1 - step;
        const int nb = min(kChB, B - I * kChB);
        double acc[V];
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = 0.0;
        const int nJ = FWD ? I : nblk - 1 - I;   // off-diagonal tiles of the row block
        for (int jj = 0; jj < nJ; jj += kTsT) {
            const int J = FWD ? jj : nblk - 1 - jj;
            const int cJ = J * kChB + lane;
            const bool two = kTsT == 2 && jj + 1 < nJ;   // the stage holds tile J and the next one (block-uniform)
            const int cJ2 = cJ + (FWD ? kChB : -kChB);
            double xv[NR], xv2[NR];
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                xv[q] = cJ < B ? x[q * B + cJ] : 0.0;
                xv2[q] = (two && cJ2 < B) ? x[q * B + cJ2] : 0.0;
            }
            const double* T = ts_acquire(ts);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double l = T[(r0 + i) * kChB + lane];
#pragma unroll
                for (int q = 0; q < NR; ++q) acc[i * NR + q] = fma(l, xv[q], acc[i * NR + q]);
            }
            if (two) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const double l = T[kTileD + (r0 + i) * kChB + lane];
#pragma unroll
                    for (int q = 0; q < NR; ++q) acc[i * NR + q] = fma(l, xv2[q], acc[i * NR + q]);
                }
            }
            ts_release(ts);
        }
        double red = reduce_scatter<V>(acc);
        if (writer && ri < nb) yv[qi * 32 + ri] = x[qi * B + I * kChB + ri] - red;
        __syncthreads();
        // x_I = L_II^-1 y (lower part incl. the diagonal) or L_II^-T y (upper part)
        double yl[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) yl[q] = lane < nb ? yv[q * 32 + lane] : 0.0;
        const double* T = ts_acquire(ts);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = r0 + i;
            const double l = (FWD ? lane <= r : lane >= r) ? T[r * kChB + lane] : 0.0;
#pragma unroll
            for (int q = 0; q < NR; ++q) acc[i * NR + q] = l * yl[q];
        }
        ts_release(ts);
        red = reduce_scatter<V>(acc);
        if (writer && ri < nb) x[qi * B + I * kChB + ri] = red;
        __syncthreads();
    }
}

}  // namespace smf
