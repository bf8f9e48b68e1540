// widei8.cuh -- the wide path's initial statistics (Fig. alg lines 2-3) as an
// exact-integer tensor-core SYRK (tcgen05 kind::i8, int32 accumulation in TMEM).
//
// Why integers (reading C21'): the tf32 two-term split (k1w_stats_tc) is exact
// per product, but its fp32 TMEM accumulation over runs of hundreds of pixels left C0 with a
// ~3e-6 relative error at B = 425 -- 40x a one-ulp input perturbation, enough to move
// well-conditioned pixels of the 598 x 4000 x 425 stress cube past the C18 bar. Here every
// extended-row entry v (x = L - sigma c, rho = sigma - 1, 1) is fixed-point
// quantised per (column, row) against its column maximum, q = rint(v 2^(27-e)) with
// |v| < 2^e (an int32, |q| < 2^27), and split into four balanced signed base-128 digits
// q = 2^21 s1 + 2^14 s2 + 2^7 s3 + s4, |s| <= 64. The SYRK sum_i q_a q_b is then
//   2^42 S11 + 2^35 (S12+S21) + 2^28 (S13+S22+S31) + 2^21 (S14+S23+S32+S41) + dropped,
// each S an exact int32 sum accumulated by the tensor cores (no accumulation error at all);
// the dropped digit products (k + l >= 6) are below 2^-26 of a product and zero-mean, and
// the rounding of q is 2^-28 of the row maximum -- C0 to ~1e-9 relative, better than the
// fp32 FFMA kernel.
//
//  k1w_scan   one cube read: sigma_p = L_p . ghat (the pilot projection, as k1w_sigma) and
//             the per-(column, row) maximum |v| (atomicMax on the float bits)
//  k1w_quant  one cube read: digits of every v, written K-major (pixels contiguous) as the
//             int8 slice cube [cols][4][R = B + 2][Np] (transposed through shared memory)
//  k1w_syrk_i8  persistent; a work item = (column, 128 x 128 row-block pair m >= n); TMA
//             loads the 4 (diagonal) or 8 slice tiles of 128 rows x 64 pixels per K tile
//             (SWIZZLE_64B); one thread issues the 10 (diagonal pairs: 7) digit products per
//             32-pixel K step as 6 (4) kind::i8 MMAs -- two products per N = 256 instruction
//             where they fill adjacent accumulators -- into four int32 TMEM accumulators (all
//             512 columns); 4 epilogue warps combine them in fp64
//             (exact power-of-two scales)
//             into the column's [BEp][BEp] partial that k2w_init consumes.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace smf {

constexpr int kI8Blk = 128;        // rows per block (TMEM lanes / MMA M and N)
constexpr int kI8S = 4;            // digits (slices) per value
constexpr int kI8Tile = 64;        // pixels per K tile (one 64-byte swizzle row per band row)
constexpr int kI8QTile = 128;      // pixels per k1w_quant block
constexpr int kI8Stages = 3;       // TMA ring depth of the SYRK
#ifndef SMF_I8_EPIW
#define SMF_I8_EPIW 4              // epilogue warps: 4, or 8 (two per TMEM lane quadrant, 64 columns each; measured equal)
#endif
constexpr int kI8EpiW = SMF_I8_EPIW;
constexpr int kI8NT = 64 + 32 * kI8EpiW;   // SYRK threads: TMA warp, MMA warp, the epilogue warps
constexpr int kI8MaxRun = 2048;    // K tiles per int32 run (131072 pixels: 4 digit products <= 4 * 64^2 per pixel)
constexpr uint32_t kI8TileBytes = kI8Blk * kI8Tile;   // one slice of one block: 8 KB
constexpr int kI8ScanPix = 128;    // pixels per k1w_scan block
#ifndef SMF_I8_PAIRN
#define SMF_I8_PAIRN 1             // A/B switch: 0 = one 128 x 128 digit product per MMA
#endif

__host__ __device__ inline size_t k1w_i8_smem() { return (size_t)kI8Stages * 2 * kI8S * kI8TileBytes + 1024; }
__host__ __device__ inline size_t k1w_quant_smem() { return (size_t)kI8S * 64 * 33 * 4; }

// exponent e of a row maximum: vmax 2^-e in [0.5, 1) (0 for an all-zero row; clamped so that
// 2^(27-e) stays a normal float)
__device__ __forceinline__ int i8_exponent(unsigned vbits) {
    const float v = __uint_as_float(vbits);
    if (!(v > 0.f)) return 0;
    int e;
    frexpf(v, &e);
    return max(e, -100);
}

struct I8ScanArgs {
    const float* L;
    const float* pil32;    // pilot mean c [cols][B]
    const float* ghat32;   // c / |c|^2 [cols][B]
    float* sigma;          // out [cols][N] (NaN = nodata row when masking)
    unsigned* vmax;        // out [cols][BEq] float bits, zeroed by k0_pilot; +inf = non-finite data
    int cols, N, B, BEq, mask;
    float nodata;
    int c0 = 0;            // first column of this launch (grid.y columns from c0)
};

constexpr int kI8ScanJ = 20;   // bands per lane held in registers (B <= 640)
__host__ inline int k1w_scan_j(int B) { return B <= 64 ? 2 : B <= 128 ? 4 : B <= 256 ? 8 : B <= 448 ? 14 : 20; }

// grid (ceil(N / kI8ScanPix), cols), 256 threads: a warp per pixel (lane l holds bands
// l + 32 j in registers), sigma by a fixed-order butterfly (as k1w_sigma), then the row
// maxima of v = L - sigma c kept per lane across the warp's pixels, combined across warps in
// shared memory and merged into vmax with one atomicMax per (block, row)
template <int J>
__global__ void __launch_bounds__(256, 4) k1w_scan(I8ScanArgs a) {
    const int c = a.c0 + blockIdx.y, p0 = blockIdx.x * kI8ScanPix, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int np = min(kI8ScanPix, a.N - p0), B = a.B;
    __shared__ float red[8][kI8ScanJ * 32 + 2];
    __shared__ float gs[kI8ScanJ * 32], cs_[kI8ScanJ * 32];
    const float* Lc = a.L + ((size_t)c * a.N + p0) * B;
    for (int b = tid; b < 32 * J; b += blockDim.x) {
        gs[b] = b < B ? a.ghat32[(size_t)c * B + b] : 0.f;
        cs_[b] = b < B ? a.pil32[(size_t)c * B + b] : 0.f;
    }
    float mx[J];
#pragma unroll
    for (int j = 0; j < J; ++j) mx[j] = 0.f;
    __syncthreads();
    float mrho = 0.f, mone = 0.f;
    const float kInf = __int_as_float(0x7f800000);
    for (int pp = wid; pp < np; pp += 8) {
        const float* Lp = Lc + (size_t)pp * B;
        float v[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int b = lane + 32 * j;
            v[j] = b < B ? __ldg(Lp + b) : 0.f;
        }
        float sum = 0.f;
        int bad = 0;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            if (lane + 32 * j < B) {
                sum = fmaf(v[j], gs[lane + 32 * j], sum);
                if (a.mask) bad |= is_nodata(v[j], a.nodata);
            }
        }
        const float sg0 = warp_sum_f(sum);
        bad = __any_sync(0xffffffffu, bad);
        const float sg = bad ? __int_as_float(0x7fc00000) : sg0;
        if (lane == 0) a.sigma[(size_t)c * a.N + p0 + pp] = sg;
        if (a.mask && bad) continue;   // nodata pixel: no row (warp-uniform)
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const float x = fabsf(fmaf(-sg, cs_[lane + 32 * j], v[j]));   // zero past B (v = c = 0)
            mx[j] = x <= 3.402823466e38f ? fmaxf(mx[j], x) : kInf;
        }
        const float rho = fabsf(sg - 1.f);
        mrho = rho <= 3.402823466e38f ? fmaxf(mrho, rho) : kInf;
        mone = 1.f;
    }
#pragma unroll
    for (int j = 0; j < J; ++j) red[wid][lane + 32 * j] = mx[j];
    if (lane == 0) {
        red[wid][kI8ScanJ * 32] = mrho;
        red[wid][kI8ScanJ * 32 + 1] = mone;
    }
    __syncthreads();
    for (int b = tid; b < B + 2; b += blockDim.x) {
        const int col = b < B ? b : kI8ScanJ * 32 + (b - B);
        float m = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) m = fmaxf(m, red[w][col]);   // +inf survives fmaxf
        if (m > 0.f) atomicMax(a.vmax + (size_t)c * a.BEq + b, __float_as_uint(m));
    }
}

struct I8QuantArgs {
    const float* L;
    const float* pil32;
    const float* sigma;
    const unsigned* vmax;
    int8_t* slices;        // out [cols][4][R][Np]
    int cols, N, B, R, Np, BEq, mask;
    int c0 = 0;            // first column of this launch
};

constexpr int kI8QRows = 64;   // extended rows per k1w_quant block
constexpr int kI8QTiles = 4;   // 128-pixel tiles per k1w_quant block (amortises the per-row setup)

// grid (ceil(Np / 512), ceil(R / 64), cols), 256 threads, k1w_quant_smem() dynamic smem.
// Every extended row is v = fma(-sigma, beta_r, L_r) + gamma_r (band rows: beta = c_r, gamma =
// 0, bit-identical to k1w_scan's v; rho row: beta = -1, gamma = -1; the 1 row: beta = 0,
// gamma = 1; rows >= R: 0). A non-finite v becomes 0 -- which also zeroes nodata pixels
// (sigma = NaN) and the pixels past N (sigma set to NaN here); non-finite data was flagged by
// k1w_scan (+inf row maximum) and turns the partial into NaN in the SYRK epilogue.
__global__ void __launch_bounds__(256, 4) k1w_quant(I8QuantArgs a) {
    extern __shared__ uint32_t qsm[];   // [4][64 rows][33 words]: 4 pixels per word, padded
    const int rb = blockIdx.y, c = a.c0 + blockIdx.z, tid = threadIdx.x;
    const int B = a.B, R = a.R;
    __shared__ float sh_sig[kI8QTile];
    const int rbase = rb * kI8QRows;
    // per-thread row constants, once per block (the block walks kI8QTiles pixel tiles)
    const int r = tid & (kI8QRows - 1), q = tid >> 6, gr = rbase + r;
    const unsigned vb = gr < R ? a.vmax[(size_t)c * a.BEq + gr] : 0u;
    const float sc = ldexpf(1.f, 27 - i8_exponent(vb));
    const float beta = gr < B ? a.pil32[(size_t)c * B + gr] : (gr == B ? -1.f : 0.f);
    const float gamma = gr == B ? -1.f : (gr == B + 1 ? 1.f : 0.f);
    const bool band = gr < B;
    const int nrows = min(kI8QRows, R - rbase);
    for (int pt = blockIdx.x * kI8QTiles; pt < min((int)(blockIdx.x + 1) * kI8QTiles, (a.Np + kI8QTile - 1) / kI8QTile);
         ++pt) {
        const int pbase = pt * kI8QTile;
        __syncthreads();   // the previous tile's sigma / words are consumed
        for (int p = tid; p < kI8QTile; p += blockDim.x) {
            const int gp = pbase + p;
            sh_sig[p] = gp < a.N ? a.sigma[(size_t)c * a.N + gp] : __int_as_float(0x7fc00000);
        }
        const int nvalid = a.N - pbase;   // pixels of this tile that exist (may exceed 128)
        // block-uniform 64-bit base + 32-bit per-thread offsets (p B + gr < 2^31): one integer
        // add per load instead of a 64-bit multiply-add chain
        const float* Lt = a.L + ((size_t)c * a.N + pbase) * B;
        const uint32_t o0 = (uint32_t)(4 * q * B + gr), o16 = (uint32_t)(16 * B), oB = (uint32_t)B;
        float lv[2][4][4];   // all 32 of this thread's radiances in flight at once
        if (band && nvalid >= kI8QTile) {   // full tile: no per-load bounds
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int k = 0; k < 4; ++k) lv[h][u][k] = __ldg(Lt + (o0 + (uint32_t)(4 * h + u) * o16 + k * oB));
        } else {
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int p = 4 * (q + 4 * (4 * h + u)) + k;
                        lv[h][u][k] =
                            (band && p < nvalid) ? __ldg(Lt + (o0 + (uint32_t)(4 * h + u) * o16 + k * oB)) : 0.f;
                    }
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int w = q + 4 * (4 * h + u);
                unsigned dgk[4][kI8S];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float v = fmaf(-sh_sig[4 * w + k], beta, lv[h][u][k]) + gamma;
                    v = fabsf(v) <= 3.402823466e38f ? v : 0.f;
                    // q = rint(v 2^(27-e)), |q| < 2^27 (v 2^(27-e) is exact: a power-of-two
                    // scaling). Its signed base-128 digits d_k in [-64, 63] (top digit [-64, 64])
                    // are the plain base-128 digits of q + 64 (1 + 2^7 + 2^14 + 2^21) minus 64 --
                    // no carries -- so a digit is a shift and a mask, and the -64 is one
                    // per-byte subtraction per word
                    const unsigned qb = (unsigned)(__float2int_rn(v * sc) + 0x8102040);
                    dgk[k][3] = qb & 127u;
                    dgk[k][2] = (qb >> 7) & 127u;
                    dgk[k][1] = (qb >> 14) & 127u;
                    dgk[k][0] = qb >> 21;
                }
#pragma unroll
                for (int d = 0; d < kI8S; ++d) {
                    const uint32_t lo = __byte_perm(dgk[0][d], dgk[1][d], 0x0040);
                    const uint32_t hi = __byte_perm(dgk[2][d], dgk[3][d], 0x0040);
                    // per byte b in [0, 127]: b - 64 as int8 = b ^ 0x40 ^ ((~b & 0x40) << 1) (no
                    // borrows between bytes; __vsub4 is a multi-instruction sequence)
                    const uint32_t wb = __byte_perm(lo, hi, 0x5410);
                    qsm[(d * kI8QRows + r) * 33 + w] = wb ^ 0x40404040u ^ ((~wb & 0x40404040u) << 1);
                }
            }
        __syncthreads();
        // write out: warp = 8 rows per pass, lane = word (128 B per row segment); 32-bit word
        // offsets from a per-slice base (a column's slices are 4 R Np bytes), no per-store
        // 64-bit address arithmetic
        const int w = tid & 31, pw_lim = min(kI8QTile, a.Np - pbase) / 4;   // Np is a multiple of 16
        if (w < pw_lim) {
            const uint32_t wpr = (uint32_t)a.Np >> 2;   // words per slice row
            const uint32_t* qs = qsm + w;
            const int r0 = tid >> 5;
#pragma unroll
            for (int sl = 0; sl < kI8S; ++sl) {
                // block-uniform base, 32-bit word offsets (a column's slices are 4 R Np bytes)
                uint32_t* dst = reinterpret_cast<uint32_t*>(a.slices + (((size_t)c * kI8S + sl) * R + rbase) * a.Np +
                                                            pbase);
                if (nrows == kI8QRows) {
#pragma unroll
                    for (int i = 0; i < kI8QRows / 8; ++i) {
                        const int rr = r0 + 8 * i;
                        dst[(uint32_t)rr * wpr + w] = qs[(sl * kI8QRows + rr) * 33];
                    }
                } else {
                    for (int rr = r0; rr < nrows; rr += 8) dst[(uint32_t)rr * wpr + w] = qs[(sl * kI8QRows + rr) * 33];
                }
            }
        }
    }
}

// D[tmem] (+)= A[smem] . B[smem]^T, kind::i8 (signed int8 operands, int32 accumulate).
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 32-lane x 16-column int32 TMEM load of this thread's lane (no wait)
__device__ __forceinline__ void tmem_ld16_s32(uint32_t addr, int (&x)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = (int)r[i];
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

struct I8SyrkArgs {
    const unsigned* vmax;   // [cols][BEq]
    double* part;           // out [cols][BEp][BEp] (lower blocks m >= n; diagonal blocks full)
    int cols, N, R, BEq, BEp, NBLK, npairs, nitems;
    int c0 = 0;             // first column of this launch (items cover columns c0 .. c0 + nitems / npairs - 1)
};

__global__ void __launch_bounds__(kI8NT, 1)
    k1w_syrk_i8(const __grid_constant__ CUtensorMap tm, I8SyrkArgs a) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* ring = align1024(smem_raw);   // [kI8Stages][2 blocks x 4 slices][128 rows][64 B]
    constexpr uint32_t STAGE = 2 * kI8S * kI8TileBytes;
    __shared__ uint64_t full[kI8Stages], empty[kI8Stages], acc_full, acc_empty;
    __shared__ uint32_t tmem_sh;
    __shared__ double colsc[2][kI8Blk];   // epilogue: 2^e_j of the item's columns (by item parity)
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    const int ntile = (a.N + kI8Tile - 1) / kI8Tile;
    // M = N = 128, int8 x int8 -> s32, both K-major
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kI8Blk >> 3) << 17) |
                           ((uint32_t)(kI8Blk >> 4) << 24);
    // the same with N = 256: two adjacent digit slices of the B block per instruction
    const uint32_t idesc2 = (idesc & ~(0x3fu << 17)) | ((uint32_t)(2 * kI8Blk >> 3) << 17);
    if (tid == 0) {
        prefetch_tmap(&tm);
        for (int s = 0; s < kI8Stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&acc_full, 1);
        mbar_init(&acc_empty, kI8EpiW);
        fence_mbar_init();
    }
    if (wid == 1) tmem_alloc(&tmem_sh, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_sh;
    auto item_mn = [&](int it, int& c, int& m, int& n) {
        const int cl = it / a.npairs;
        c = a.c0 + cl;
        n = it - cl * a.npairs;
        m = 0;
        while (n > m) {
            n -= m + 1;
            ++m;
        }
    };

    if (wid == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            uint32_t g = 0;
            for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
                int c, m, n;
                item_mn(it, c, m, n);
                const bool diag = m == n;
                for (int kt = 0; kt < ntile; ++kt, ++g) {
                    const int s = g % kI8Stages;
                    if (g >= kI8Stages) mbar_wait(&empty[s], ((g / kI8Stages) - 1) & 1);
                    unsigned char* st = ring + s * STAGE;
                    mbar_arrive_expect_tx(&full[s], (diag ? kI8S : 2 * kI8S) * kI8TileBytes);
                    for (int sl = 0; sl < kI8S; ++sl)
                        tma_load_3d(st + sl * kI8TileBytes, &tm, &full[s], kt * kI8Tile, m * kI8Blk, c * kI8S + sl);
                    if (!diag)
                        for (int sl = 0; sl < kI8S; ++sl)
                            tma_load_3d(st + (kI8S + sl) * kI8TileBytes, &tm, &full[s], kt * kI8Tile, n * kI8Blk,
                                        c * kI8S + sl);
                }
            }
        }
    } else if (wid == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            const uint32_t ring0 = smem_u32(ring);
            uint32_t g = 0, runs = 0;
            for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
                int c, m, n;
                item_mn(it, c, m, n);
                const bool diag = m == n;
                for (int kt0 = 0; kt0 < ntile; kt0 += kI8MaxRun) {
                    const int kt1 = min(ntile, kt0 + kI8MaxRun);
                    if (runs >= 1) mbar_wait(&acc_empty, (runs - 1) & 1);   // epilogue drained TMEM
                    tc_fence_after();
                    for (int kt = kt0; kt < kt1; ++kt, ++g) {
                        const int s = g % kI8Stages;
                        mbar_wait(&full[s], (g / kI8Stages) & 1);
                        tc_fence_after();
                        const uint32_t sa = ring0 + s * STAGE, sb = diag ? sa : sa + kI8S * kI8TileBytes;
#pragma unroll
                        for (int ks = 0; ks < kI8Tile / 32; ++ks) {
                            uint64_t ad[kI8S], bd[kI8S];
#pragma unroll
                            for (int d = 0; d < kI8S; ++d) {   // SWIZZLE_64B K-major: 8-row groups 512 B apart
                                ad[d] = umma_desc(sa + d * kI8TileBytes + ks * 32, 16, 512, 4);
                                bd[d] = umma_desc(sb + d * kI8TileBytes + ks * 32, 16, 512, 4);
                            }
                            const uint32_t acc = (kt == kt0 && ks == 0) ? 0u : 1u;
                            // accumulator j (TMEM columns 128 j) collects the digit products of
                            // weight 2^(42 - 7 j): k + l = j (0-based digit indices). A diagonal
                            // block pair (m = n) needs only k <= l for j = 1, 3 (the k > l products
                            // are transposes; the epilogue doubles those accumulators and k2w_init
                            // symmetrises the block): 7 products instead of 10. j = 2 mixes the
                            // cross product with the square D1 D1^T, so it keeps all three.
#if SMF_I8_PAIRN
                            // Two products per instruction where they land in adjacent
                            // accumulators: the digit slices of a block are adjacent 8 KB tiles of
                            // the stage, so B = [D_l ; D_l+1] is one 256-row operand and
                            // D_k [D_l ; D_l+1]^T fills accumulators k + l and k + l + 1 (N = 256)
                            // with one read of A: 6 (diagonal pairs: 4) MMAs instead of 10 (7).
                            mma_i8(tmem, ad[0], bd[0], idesc2, acc);             // (0,0) (0,1)
                            mma_i8(tmem + 256, ad[0], bd[2], idesc2, acc);       // (0,2) (0,3)
                            if (!diag) {
                                mma_i8(tmem + 128, ad[1], bd[0], idesc2, 1u);    // (1,0) (1,1)
                                mma_i8(tmem + 384, ad[1], bd[2], idesc, 1u);     // (1,2)
                                mma_i8(tmem + 256, ad[2], bd[0], idesc2, 1u);    // (2,0) (2,1)
                                mma_i8(tmem + 384, ad[3], bd[0], idesc, 1u);     // (3,0)
                            } else {
                                mma_i8(tmem + 256, ad[1], bd[1], idesc2, 1u);    // (1,1) (1,2)
                                mma_i8(tmem + 256, ad[2], bd[0], idesc, 1u);     // (2,0)
                            }
#else
#pragma unroll
                            for (int j = 0; j < kI8S; ++j)
#pragma unroll
                                for (int k = 0; k <= j; ++k)
                                    if (!(diag && (j & 1) && k > j - k))
                                        mma_i8(tmem + 128 * j, ad[k], bd[j - k], idesc, k == 0 ? acc : 1u);
#endif
                        }
                        mma_commit(&empty[s]);
                    }
                    mma_commit(&acc_full);
                    ++runs;
                }
            }
        }
    } else {
        // ===================== epilogue: TMEM int32 -> fp64 partial =====================
        // v = sumq 2^(e_i + e_j - 33) as two exact power-of-two multiplications: the row's factor
        // in a register, the 128 column factors of the item in shared memory (one per epilogue
        // thread, double-buffered by item parity: one named barrier per item). A non-finite row
        // maximum (flagged by k1w_scan) makes its factor NaN, which the products propagate. The
        // per-element __ldg + frexpf + ldexp of the first version was ~110 instructions per
        // element: ~a fifth of the kernel, with the tensor pipe idle (the accumulators are
        // single-buffered: all 512 TMEM columns hold one item).
        const int q = wid & 3;                 // TMEM lane quadrant this warp may access
        const int rl = 32 * q + lane;          // row within the block
        const int half = (wid - 2) >> 2;       // column half of this warp (8 epilogue warps)
        constexpr int kColsW = kI8Blk * 4 / kI8EpiW;   // columns per warp: 128 or 64
        const double kNaN = __longlong_as_double(0x7ff8000000000000ULL);
        auto pow2 = [](int e) { return __longlong_as_double((long long)(e + 1023) << 52); };   // -1022 <= e <= 1023
        uint32_t runs = 0;
        int par = 0;
        for (int it = blockIdx.x; it < a.nitems; it += gridDim.x, par ^= 1) {
            int c, m, n;
            item_mn(it, c, m, n);
            const unsigned* vm = a.vmax + (size_t)c * a.BEq;
            const int gi = m * kI8Blk + rl, gjt = n * kI8Blk + rl;
            const unsigned vbi = gi < a.R ? vm[gi] : 0u;
            const unsigned vbj = gjt < a.R ? vm[gjt] : 0u;
            const bool badi = !(__uint_as_float(vbi) <= 3.402823466e38f);
            const bool badj = !(__uint_as_float(vbj) <= 3.402823466e38f);
            const double si = badi ? kNaN : pow2(i8_exponent(vbi) - 33);
            if (half == 0) colsc[par][rl] = badj ? kNaN : pow2(i8_exponent(vbj));
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kI8EpiW) : "memory");   // the epilogue warps
            const double* sj = colsc[par];
            double* prow = a.part + ((size_t)c * a.BEp + gi) * a.BEp + (size_t)n * kI8Blk;
            // diagonal pairs carry the odd-j cross products once (see the MMA issuer): doubled here
            const double w1 = m == n ? 32768.0 : 16384.0, w3 = m == n ? 2.0 : 1.0;
            for (int kt0 = 0; kt0 < ntile; kt0 += kI8MaxRun) {
                mbar_wait(&acc_full, runs & 1);
                tc_fence_after();
                const uint32_t t0 = tmem + ((uint32_t)(32 * q) << 16);
#pragma unroll 1
                for (int j0 = half * kColsW; j0 < (half + 1) * kColsW; j0 += 16) {
                    int x[kI8S][16];
#pragma unroll
                    for (int d = 0; d < kI8S; ++d) tmem_ld16_s32(t0 + 128 * d + j0, x[d]);
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 16; k += 2) {
                        double2 v;
                        // sum_i q_a q_b = 2^42 x0 + 2^35 x1 + 2^28 x2 + 2^21 x3 (each term exact in
                        // fp64; the sum rounds once per term at 2^-53), in units of 2^21
                        v.x = ((((double)x[0][k] * 2097152.0 + (double)x[1][k] * w1) + (double)x[2][k] * 128.0) +
                               (double)x[3][k] * w3) * si * sj[j0 + k];
                        v.y = ((((double)x[0][k + 1] * 2097152.0 + (double)x[1][k + 1] * w1) +
                                (double)x[2][k + 1] * 128.0) + (double)x[3][k + 1] * w3) * si * sj[j0 + k + 1];
                        double2* dst = reinterpret_cast<double2*>(prow + j0 + k);   // 16-byte aligned (BEp % 128 == 0)
                        if (kt0 > 0) {
                            const double2 o = *dst;
                            v.x += o.x;
                            v.y += o.y;
                        }
                        *dst = v;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty);
                ++runs;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (wid == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace smf
