// smf.cu -- C ABI of libsmf.so (include/smf.h): context, validation, workspace
// layout, TMA descriptors and the launch sequence of the B200 hot path.
//
// Launch sequence of smf_retrieve (all on the caller's stream):
//   K1 k1_stats (once)  -> K2 k2_init (once)  -> K3 k3_sweep(k=0)
//   -> for k = 1..N_iter: K2 k2_update(k) -> K3 k3_sweep(k)
// i.e. (N_iter + 2) passes over the radiance cube.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3 (no-op unless a tool is attached)

#include "../../include/smf.h"
#include "kernels.cuh"
#include "wide.cuh"
#include "widei8.cuh"

using namespace smf;

struct smf_ctx {
    int device = 0;
    int bands = 0;
    int sm_count = 0;
    float* s_dev = nullptr;
    bool s_set = false;
    double eps = 1e-2, ridge = 0.0, r_floor = 0.05;
    int n_iter = 30, use_sparsity = 1, use_albedo = 1;
    int stats_kernel = SMF_STATS_AUTO;
    int energy = 0;   // energy trace (smf_set_energy_trace)
    int group = 1;    // detector columns per partition (smf_set_grouping)
    int mask = 0;     // nodata masking (smf_set_nodata)
    float nodata = -9999.f;
    int lit_mode = SMF_COVCHECK_AUTO;   // literal covariance check (smf_set_covariance_check)
    int diag = 0;                       // per-iteration diagnostics (smf_set_diagnostics)
    int nvtx = -1;                      // NVTX range per launch (smf_set_nvtx; -1: SMF_NVTX env)
    int last_launches = 0;
    char err[512] = {0};
    // profiling (smf_profile_*): events bracketing each launch
    bool prof = false;
    struct Rec { int kind; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    // smf_retrieve_host state
    cudaStream_t h_stream = nullptr;   // compute
    cudaStream_t h_up = nullptr;       // host -> device copies
    cudaStream_t h_down = nullptr;     // device -> host copies
    cudaEvent_t h_ev[8] = {};          // [0,2) uploaded, [2,4) computed, [4,6) downloaded
    void* h_buf = nullptr;
    size_t h_buf_bytes = 0;
    // CUDA-graph mode (smf_set_graph): the launch sequence of the last smf_retrieve,
    // captured once and replayed while the call's arguments and settings are unchanged
    int graph = 0;
    unsigned gen = 0;                  // bumped by every setter: invalidates the graph
    cudaGraphExec_t gexec = nullptr;
    struct GKey {
        const void* rad; int cols, pixels; const void* enh; const void* alb; const void* ws;
        const void* status; const void* stream; unsigned gen;
        bool operator==(const GKey& o) const {
            return rad == o.rad && cols == o.cols && pixels == o.pixels && enh == o.enh && alb == o.alb &&
                   ws == o.ws && status == o.status && stream == o.stream && gen == o.gen;
        }
    } gkey = {};
    int glaunches = 0;
    // wide path: the last partial wave of k2w_init runs on this stream beside the other
    // columns' statistics (retrieve_eager); created on first use
    cudaStream_t aux = nullptr;
    cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
};

namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

void load_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

void set_err(smf_ctx* ctx, const char* fmt, ...) {
    if (!ctx) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
    va_end(ap);
}

smf_status cuda_fail(smf_ctx* ctx, cudaError_t e, const char* where) {
    set_err(ctx, "%s: %s", where, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SMF_ERR_OUT_OF_MEMORY : SMF_ERR_CUDA;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

cudaEvent_t get_event(smf_ctx* ctx) {
    if (!ctx->pool.empty()) {
        cudaEvent_t e = ctx->pool.back();
        ctx->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

bool nvtx_on(const smf_ctx* ctx) {
    static const int env = [] {
        const char* e = std::getenv("SMF_NVTX");
        return (e && e[0] == '1') ? 1 : 0;
    }();
    return ctx->nvtx < 0 ? env != 0 : ctx->nvtx != 0;
}

const char* kernel_kind_name(int kind) {
    switch (kind) {
        case SMF_KERNEL_STATS: return "smf:stats (K0/K1, Fig. alg lines 2-3)";
        case SMF_KERNEL_INIT: return "smf:init (K2, lines 2-6)";
        case SMF_KERNEL_UPDATE: return "smf:update (K2, lines 9-16)";
        case SMF_KERNEL_SWEEP: return "smf:sweep (K3, lines 5, 9, 16)";
    }
    return "smf:other";
}

// Bracket one launch with events when profiling is on, and with an NVTX range when
// NVTX is on (host-side range around the enqueue; tools map it to the launch).
struct ProfScope {
    smf_ctx* ctx;
    cudaStream_t st;
    int kind;
    cudaEvent_t a = nullptr;
    bool nv = false;
    ProfScope(smf_ctx* c, cudaStream_t s, int k) : ctx(c), st(s), kind(k) {
        nv = nvtx_on(ctx);
        if (nv) nvtxRangePushA(kernel_kind_name(kind));
        if (ctx->prof) {
            a = get_event(ctx);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (ctx->prof && a) {
            cudaEvent_t b = get_event(ctx);
            cudaEventRecord(b, st);
            ctx->recs.push_back({kind, a, b});
        }
        if (nv) nvtxRangePop();
    }
};

// Static, balanced partition of the global tile stream (column-major tiles) over
// the persistent sweep CTAs; S = max columns touched by one CTA.
struct Plan {
    int cols, N, B, tpc, G, S;
    long long ttot;
    // K1 (persistent, one CTA per SM, own tile height T1 and partition)
    int G1, S1, W1, T1, tpc1, NT1, be_full;
    bool k1tc;
    // wide path (any B): K1w block grid, K3w tiles of kWideT3 pixels
    bool wide, widetc, widei8;
    int R8, Np8, BEq8;          // int8 statistics: extended rows B + 2, padded pixels, vmax stride
    size_t o_vmax, o_slices;
    int BEw, NBw, NGw, NBLKw;
    size_t o_sigma;
    long long ttot1;
    size_t smem1, smem2, smem3;
    // workspace offsets
    size_t o_mbar, o_mu, o_tprev, o_yprev, o_ainv, o_q64, o_z32, o_mhat, o_kc, o_q32, o_status, o_pilot, o_ghat, o_part1,
        o_part3, o_tra, o_rho, o_tq, o_energy, o_nvalid, o_nlit, o_lit, o_dnnz, o_dq, o_dst, o_dlit, total;
    long long lit_stride;   // doubles per column of the wide literal-check scratch
    int n_energy;   // energy rows (n_iter + 1) or 0
    int n_diag;     // diagnostics rows (n_iter + 1) or 0
};

int sweep_blocks_per_sm(int B);
size_t k1_smem(int B);
int k1_rows(int B);
int stats_threads(int B);
bool k1tc_fits(int B);
int k1tc_be(int B);
size_t k1tc_smem(int B);
bool narrow(int B) { return B >= 4 && B <= 96 && B % 4 == 0; }
int wide_blocks_per_sm(int B);
void* k2_init_kernel(int B) {
    switch ((B + 7) / 8) {
#define SMF_K2I(n) \
    case n: return reinterpret_cast<void*>(&k2_init<n>);
        SMF_K2I(1) SMF_K2I(2) SMF_K2I(3) SMF_K2I(4) SMF_K2I(5) SMF_K2I(6) SMF_K2I(7) SMF_K2I(8) SMF_K2I(9)
        SMF_K2I(10) SMF_K2I(11) SMF_K2I(12)
#undef SMF_K2I
        default: return nullptr;
    }
}

bool make_plan(const smf_ctx* ctx, int cols, int N, Plan& p) {
    const int B = ctx->bands;
    p.cols = cols;
    p.N = N;
    p.B = B;
    p.wide = !narrow(B);
    p.tpc = (N + (p.wide ? kWideT3 : kTileRows) - 1) / (p.wide ? kWideT3 : kTileRows);
    p.ttot = (long long)cols * p.tpc;
    int per_sm = std::max(1, p.wide ? wide_blocks_per_sm(B) : sweep_blocks_per_sm(B));
    static const int per_sm_env = [] {   // SMF_SWEEP_CTAS_PER_SM: sweep occupancy override (A/B)
        const char* e = std::getenv("SMF_SWEEP_CTAS_PER_SM");
        return e ? std::atoi(e) : 0;
    }();
    if (per_sm_env > 0) per_sm = std::min(per_sm, per_sm_env);
    long long G = (long long)ctx->sm_count * per_sm;
    if (G > p.ttot) G = p.ttot;
    p.G = (int)G;
    int S = 1;
    for (int b = 0; b < p.G; ++b) {
        long long t0 = tile_begin(b, p.ttot, p.G), t1 = tile_begin(b + 1, p.ttot, p.G);
        if (t1 > t0) S = std::max(S, (int)((t1 - 1) / p.tpc - t0 / p.tpc + 1));
    }
    p.S = S;
    p.BEw = (B + 2 + 7) / 8 * 8;
    p.NBw = (p.BEw / 8) * (p.BEw / 8 + 1) / 2;
    p.NGw = (p.NBw + kWideNT1 - 1) / kWideNT1;
    p.NBLKw = (B + 2 + 127) / 128;
    p.widetc = p.wide && ctx->stats_kernel == SMF_STATS_TENSOR;
    p.widei8 = p.wide && (ctx->stats_kernel == SMF_STATS_AUTO || ctx->stats_kernel == SMF_STATS_INT8);
    p.R8 = B + 2;
    p.Np8 = (N + 15) / 16 * 16;
    p.k1tc = !p.wide && ctx->stats_kernel != SMF_STATS_FFMA && k1tc_fits(B);
    p.T1 = p.k1tc ? kTileTC : k1_rows(B);
    p.NT1 = p.k1tc ? K1TC<1>::NT : stats_threads(B);
    p.be_full = p.k1tc ? k1tc_be(B) : 0;
    p.tpc1 = (N + p.T1 - 1) / p.T1;
    p.ttot1 = (long long)cols * p.tpc1;
    p.G1 = (int)std::min<long long>(std::min(ctx->sm_count, kMaxSlots1), p.ttot1);
    p.S1 = 1;
    for (int b = 0; b < p.G1; ++b) {
        long long t0 = tile_begin(b, p.ttot1, p.G1), t1 = tile_begin(b + 1, p.ttot1, p.G1);
        if (t1 > t0) p.S1 = std::max(p.S1, (int)((t1 - 1) / p.tpc1 - t0 / p.tpc1 + 1));
    }
    p.W1 = p.k1tc ? p.be_full * p.be_full : k1_width_host(B);
    if (p.wide) {
        p.smem1 = p.widetc ? k1w_tc_smem() : (p.widei8 ? k1w_i8_smem() : k1w_smem(B, p.BEw));
        p.smem2 = k2w_init_smem(B);
        p.smem3 = k3w_smem(B);
    } else {
        TileGeom g = TileGeom::make(B);
        p.smem1 = p.k1tc ? k1tc_smem(B) : k1_smem(B);
        p.smem2 = k2_init_smem(B, p.W1);
        p.smem3 = (size_t)kStages * g.stage_bytes + 1024;
    }
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = align_up(o + bytes, 256);
        return r;
    };
    const size_t cb = (size_t)cols * B;
    p.o_mbar = take(cb * 8);
    p.o_mu = take(cb * 8);
    p.o_tprev = take(cb * 8);
    p.o_yprev = take(cb * 8);
    p.o_ainv = take(cb * (p.wide ? wide_ld(B) : B) * 8);   // wide: the factor's rows padded to an even stride
    p.o_q64 = take((size_t)cols * 8);
    p.o_z32 = take(cb * 4);
    p.o_mhat = take(cb * 4);
    p.o_kc = take((size_t)cols * 8);
    p.o_q32 = take((size_t)cols * 4);
    p.o_status = take((size_t)cols * 4);
    p.o_pilot = take(cb * 4);
    p.o_ghat = take(cb * 4);
    const size_t bep = (size_t)p.NBLKw * 128;
    p.BEq8 = (int)bep;
    p.o_part1 = p.wide ? take((p.widetc || p.widei8) ? (size_t)cols * bep * bep * 8
                                                     : (size_t)cols * p.NGw * kWideNT1 * 64 * 8)
                       : take((size_t)p.G1 * p.S1 * p.W1 * 8);
    p.o_sigma = take((p.widetc || p.widei8) ? (size_t)cols * N * 4 : 0);
    p.o_vmax = take(p.widei8 ? (size_t)cols * p.BEq8 * 4 : 0);
    p.o_slices = take(p.widei8 ? (size_t)cols * kI8S * p.R8 * p.Np8 : 0);
    p.o_part3 = take((size_t)p.G * p.S * (B + kPartExtra) * 8);
    p.o_tra = take((size_t)cols * 8);
    p.o_rho = take((size_t)cols * 8);
    p.o_tq = take((size_t)cols * 8);
    p.o_nvalid = take((size_t)cols * 8);
    p.n_energy = ctx->energy ? ctx->n_iter + 1 : 0;
    p.o_energy = take((size_t)std::max(p.n_energy, 1) * cols * 8);
    p.o_nlit = take((size_t)cols * 4);
    // wide literal covariance check (reading C16''): per-column fp64 scratch, aliased onto the
    // K1w partials (dead once k2w_init has consumed them) when they are large enough
    p.lit_stride = p.wide ? lit_doubles(B) : 0;
    const size_t part1_bytes = p.wide ? ((p.widetc || p.widei8) ? (size_t)cols * bep * bep * 8
                                                                : (size_t)cols * p.NGw * kWideNT1 * 64 * 8)
                                      : 0;
    const size_t lit_bytes = (size_t)cols * p.lit_stride * 8;
    p.o_lit = !p.wide ? 0 : (lit_bytes <= part1_bytes ? p.o_part1 : take(lit_bytes));
    p.n_diag = ctx->diag ? ctx->n_iter + 1 : 0;
    const size_t nd = (size_t)std::max(p.n_diag, 1) * cols;
    p.o_dnnz = take(nd * 8);
    p.o_dq = take(nd * 8);
    p.o_dst = take(nd * 4);
    p.o_dlit = take(nd * 4);
    p.total = o;
    return true;
}

template <int NQ>
void* sweep_fn() {
    return reinterpret_cast<void*>(&k3_sweep<NQ>);
}

void* sweep_kernel(int B) {
    switch (B / 4) {
        case 1: return sweep_fn<1>();
        case 2: return sweep_fn<2>();
        case 3: return sweep_fn<3>();
        case 4: return sweep_fn<4>();
        case 5: return sweep_fn<5>();
        case 6: return sweep_fn<6>();
        case 7: return sweep_fn<7>();
        case 8: return sweep_fn<8>();
        case 9: return sweep_fn<9>();
        case 10: return sweep_fn<10>();
        case 11: return sweep_fn<11>();
        case 12: return sweep_fn<12>();
        case 13: return sweep_fn<13>();
        case 14: return sweep_fn<14>();
        case 15: return sweep_fn<15>();
        case 16: return sweep_fn<16>();
        case 17: return sweep_fn<17>();
        case 18: return sweep_fn<18>();
        case 19: return sweep_fn<19>();
        case 20: return sweep_fn<20>();
        case 21: return sweep_fn<21>();
        case 22: return sweep_fn<22>();
        case 23: return sweep_fn<23>();
        case 24: return sweep_fn<24>();
        default: return nullptr;
    }
}

template <int NQ>
void* stats_fn() {
    return reinterpret_cast<void*>(&k1_stats<NQ>);
}

template <int NQ>
size_t stats_smem() {
    return k1_smem_bytes<NQ>();
}

#define SMF_NQ_CASES(M) \
    M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16) M(17) M(18) M(19) \
        M(20) M(21) M(22) M(23) M(24)

void* stats_kernel(int B) {
    switch (B / 4) {
#define SMF_CASE(n) \
    case n: return stats_fn<n>();
        SMF_NQ_CASES(SMF_CASE)
#undef SMF_CASE
        default: return nullptr;
    }
}

template <int NQ>
void* stats_tc_fn() {
    return reinterpret_cast<void*>(&k1_stats_tc<NQ>);
}

void* stats_tc_kernel(int B) {
    switch (B / 4) {
#define SMF_CASE(n) \
    case n: return K1TC<n>::FITS ? stats_tc_fn<n>() : nullptr;
        SMF_NQ_CASES(SMF_CASE)
#undef SMF_CASE
        default: return nullptr;
    }
}

bool k1tc_fits(int B) { return stats_tc_kernel(B) != nullptr; }

int k1tc_be(int B) {
    switch (B / 4) {
#define SMF_CASE(n) \
    case n: return K1TC<n>::BE;
        SMF_NQ_CASES(SMF_CASE)
#undef SMF_CASE
        default: return 0;
    }
}

size_t k1tc_smem(int B) {
    switch (B / 4) {
#define SMF_CASE(n) \
    case n: return K1TC<n>::SMEM;
        SMF_NQ_CASES(SMF_CASE)
#undef SMF_CASE
        default: return 0;
    }
}

int k1_rows(int B) {
    switch (B / 4) {
#define SMF_CASE(n) \
    case n: return K1Geom<n>::T;
        SMF_NQ_CASES(SMF_CASE)
#undef SMF_CASE
        default: return kTileRows;
    }
}

int stats_threads(int B) {
    switch (B / 4) {
#define SMF_CASE(n) \
    case n: return K1Geom<n>::NT;
        SMF_NQ_CASES(SMF_CASE)
#undef SMF_CASE
        default: return 0;
    }
}

size_t k1_smem(int B) {
    switch (B / 4) {
#define SMF_CASE(n) \
    case n: return stats_smem<n>();
        SMF_NQ_CASES(SMF_CASE)
#undef SMF_CASE
        default: return 0;
    }
}

int sweep_blocks_per_sm(int B) {
    void* fn = sweep_kernel(B);
    if (!fn) return 0;
    TileGeom g = TileGeom::make(B);
    size_t smem = (size_t)kStages * g.stage_bytes + 1024;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kTileRows, smem) != cudaSuccess) return 1;
    return std::max(n, 1);
}

// Programmatic dependent launch (SMF_PDL=0 turns it off): the kernel may be scheduled
// while its predecessor in the stream drains; it runs its prologue (barrier init, TMEM
// allocation, the first TMA loads of the read-only cube) and then blocks in griddep_wait()
// until the predecessor has completed. Only kernels that call griddep_wait() use it.
bool pdl_on() {
    static const bool on = [] {
        const char* e = std::getenv("SMF_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st) {
    if (!pdl_on()) return cudaLaunchKernel(fn, grid, block, args, smem, st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

// smf_retrieve_host chunking: ~24 chunks of whole detector groups -- the exposed tail
// (the last chunk's retrieval and download) shrinks with the chunk while every chunk's
// retrieval still hides under the next upload (SMF_HOST_CHUNKS overrides the target).
int host_chunk_cols(int group, int cols) {
    static const int target = [] {
        const char* e = std::getenv("SMF_HOST_CHUNKS");
        const int v = e ? std::atoi(e) : 24;
        return v > 0 ? v : 24;
    }();
    const int G = std::max(1, std::min(group, cols));
    const int ngroups = (cols + G - 1) / G;
    const int want = std::max(1, std::min(target, cols / 16));
    return (ngroups + want - 1) / want * G;
}

// Serpentine sweep order (narrow path): alternate sweeps walk each CTA's tile range
// backwards so the start of a pass hits the L2-resident tail of the previous one.
// SMF_SERPENTINE=0 turns it off (A/B measurement).
bool serpentine() {
    static const bool on = [] {
        const char* e = std::getenv("SMF_SERPENTINE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Tiles per sweep CTA whose L2 lines are kept (evict_last) for the next, reversed pass:
// SMF_L2KEEP_MB (default 48) of the 126 MB L2 spread over the sweep grid; 0 = no hints.
int l2_keep_tiles(const Plan& p) {
    static const long mb = [] {
        const char* e = std::getenv("SMF_L2KEEP_MB");
        return e ? std::atol(e) : 48L;
    }();
    if (p.wide || mb <= 0 || p.G <= 0) return 0;
    const double tile = (double)kTileRows * p.B * 4.0;
    return (int)std::max(1.0, (double)mb * 1048576.0 / ((double)p.G * tile));
}

template <bool MASK>
void* wide_sweep_kernel_t(int B) {
    switch (k3w_j(B)) {
        case 2: return reinterpret_cast<void*>(&k3w_sweep<2, MASK>);
        case 4: return reinterpret_cast<void*>(&k3w_sweep<4, MASK>);
        case 8: return reinterpret_cast<void*>(&k3w_sweep<8, MASK>);
        case 14: return reinterpret_cast<void*>(&k3w_sweep<14, MASK>);
        case 20: return reinterpret_cast<void*>(&k3w_sweep<20, MASK>);
        case 28: return reinterpret_cast<void*>(&k3w_sweep<28, MASK>);
        default: return nullptr;
    }
}

void* wide_sweep_kernel(int B, bool mask = false) {
    return mask ? wide_sweep_kernel_t<true>(B) : wide_sweep_kernel_t<false>(B);
}

int wide_blocks_per_sm(int B) {
    void* fn = wide_sweep_kernel(B);
    if (!fn) return 0;
    const size_t smem = k3w_smem(B);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kWideNT3, smem) != cudaSuccess) return 0;
    return n;
}

// narrow kernels for B % 4 == 0, B <= 96; the wide path for any other B whose K3w
// tile (two buffers of kWideT3 rows) fits in shared memory
bool supported(int B) {
    if (narrow(B)) return true;
    // 626: the largest band count the parity suite exercises (the shared-memory budgets of
    // the wide kernels would allow up to ~660 since the Cholesky replaced the Gauss-Jordan)
    return B >= 1 && B <= 626 && k3w_j(B) > 0 && k3w_smem(B) <= 220 * 1024 &&
           k2w_init_smem(B) <= 220 * 1024 && k1w_smem(B, (B + 2 + 7) / 8 * 8) <= 220 * 1024;
}

CUresult make_maps(const float* rad, int cols, int N, int B, CUtensorMap* main_map, CUtensorMap* tail_map,
                   int rows = kTileRows) {
    TileGeom g = TileGeom::make(B);
    cuuint64_t dims[3] = {(cuuint64_t)B, (cuuint64_t)N, (cuuint64_t)cols};
    cuuint64_t strides[2] = {(cuuint64_t)B * 4, (cuuint64_t)N * B * 4};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = CUDA_SUCCESS;
    memset(main_map, 0, sizeof(CUtensorMap));
    memset(tail_map, 0, sizeof(CUtensorMap));
    if (g.nfull > 0) {
        cuuint32_t box[3] = {32, (cuuint32_t)rows, 1};
        r = g_encode(main_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)rad, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return r;
    }
    if (g.tailw > 0) {
        cuuint32_t box[3] = {(cuuint32_t)g.tailw, (cuuint32_t)rows, 1};
        CUtensorMapSwizzle sw = g.tailw == 8 ? CU_TENSOR_MAP_SWIZZLE_32B
                                : g.tailw == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_128B;
        r = g_encode(tail_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)rad, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return r;
}

// The wide path's solve-ready factor [cols][B][wide_ld(B)] fp64 as a 3-D map {B, B, cols} with
// 32 x 32 boxes (rows/columns past B zero-filled) for k2w_update's streamed solves.
CUresult make_factor_map(const double* f, int cols, int B, CUtensorMap* map) {
    cuuint64_t dims[3] = {(cuuint64_t)B, (cuuint64_t)B, (cuuint64_t)cols};
    cuuint64_t strides[2] = {(cuuint64_t)wide_ld(B) * 8, (cuuint64_t)B * wide_ld(B) * 8};
    cuuint32_t box[3] = {(cuuint32_t)kChB, (cuuint32_t)kChB, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    memset(map, 0, sizeof(CUtensorMap));
    return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)f, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

ColState col_state(const Plan& p, unsigned char* ws, const float* s, const smf_ctx* ctx) {
    ColState cs;
    cs.mbar = (double*)(ws + p.o_mbar);
    cs.mu = (double*)(ws + p.o_mu);
    cs.tprev = (double*)(ws + p.o_tprev);
    cs.yprev = (double*)(ws + p.o_yprev);
    cs.ainv = (double*)(ws + p.o_ainv);
    cs.q64 = (double*)(ws + p.o_q64);
    cs.z32 = (float*)(ws + p.o_z32);
    cs.mhat32 = (float*)(ws + p.o_mhat);
    cs.kc32 = (float*)(ws + p.o_kc);
    cs.q32 = (float*)(ws + p.o_q32);
    cs.status = (int*)(ws + p.o_status);
    cs.s = s;
    cs.tra = (double*)(ws + p.o_tra);
    cs.rho64 = (double*)(ws + p.o_rho);
    cs.tq = (double*)(ws + p.o_tq);
    cs.nvalid = (double*)(ws + p.o_nvalid);
    cs.nlit = (int*)(ws + p.o_nlit);
    cs.mask = ctx->mask;
    cs.nodata = ctx->nodata;
    return cs;
}

smf_status validate(smf_ctx* ctx, const void* rad, int cols, int pixels, const void* ws) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    if (!rad || !ws || cols < 1 || pixels < 2) {
        set_err(ctx, "invalid argument (radiance/workspace NULL, cols < 1 or pixels < 2)");
        return SMF_ERR_INVALID_ARGUMENT;
    }
    if (!ctx->s_set) {
        set_err(ctx, "absorption spectrum not set (smf_set_absorption)");
        return SMF_ERR_NOT_CONFIGURED;
    }
    // the narrow path reads the cube through TMA tensor maps (16-byte aligned base); the wide
    // path handles any float-aligned cube (per-row cp.async when the rows are not 16-byte runs)
    if ((((uintptr_t)rad & 15) && narrow(ctx->bands)) || ((uintptr_t)rad & 3) || ((uintptr_t)ws & 255)) {
        set_err(ctx, "radiance must be 16-byte (narrow path) / 4-byte (wide path) and workspace 256-byte aligned");
        return SMF_ERR_INVALID_ARGUMENT;
    }
    if (!g_encode) {
        set_err(ctx, "cuTensorMapEncodeTiled unavailable (driver too old?)");
        return SMF_ERR_CUDA;
    }
    return SMF_OK;
}

// Detector grouping: partitions of G adjacent columns plus a
// ragged remainder; G >= cols is the all-detectors mode.
struct GroupLayout {
    int G, nfull, rem, parts;
    size_t o_full, o_rem, o_status, total;
    static GroupLayout make(int cols, int group) {
        GroupLayout g;
        g.G = group >= cols ? cols : group;
        g.nfull = cols / g.G;
        g.rem = cols - g.nfull * g.G;
        g.parts = g.nfull + (g.rem > 0 ? 1 : 0);
        g.o_full = g.o_rem = g.o_status = g.total = 0;
        return g;
    }
    size_t bytes(const smf_ctx* ctx, int pixels) {
        smf_ctx tmp = *ctx;   // plan without grouping
        tmp.group = 1;
        Plan pf, pr;
        make_plan(&tmp, nfull, G * pixels, pf);
        size_t o = 0;
        o_full = o;
        o = align_up(o + pf.total, 256);
        if (rem > 0) {
            make_plan(&tmp, 1, rem * pixels, pr);
            o_rem = o;
            o = align_up(o + pr.total, 256);
        }
        o_status = o;
        o = align_up(o + (size_t)parts * 4, 256);
        total = o;
        return total;
    }
};

// Columns of the wide int8 path whose k2w_init is split off the main launch (0: no split): the
// partial last wave, when it is at most half a wave. SMF_TAIL_SPLIT=0 disables it (A/B).
int wide_tail_mode() {
    static const int mode = [] {
        const char* e = std::getenv("SMF_TAIL_SPLIT");
        return e ? std::atoi(e) : 1;
    }();
    return mode;
}

int wide_tail_cols(const smf_ctx* ctx, const Plan& p) {
    const int on = wide_tail_mode();
    if (!on || !p.wide || !p.widei8 || ctx->prof || p.cols <= ctx->sm_count) return 0;
    const int tail = p.cols % ctx->sm_count;
    return tail <= ctx->sm_count / 2 ? tail : 0;
}

// K0 pilot + K1 stats + K2 init (shared by retrieve and initial_statistics)
// Wide int8 path only: columns [c0, c0 + nc) of the plan (nc < 0: all), and k2w_init on st_init
// (ordered behind this range's statistics by ctx->aux_fork) instead of st.
smf_status launch_stats(smf_ctx* ctx, const Plan& p, const float* rad, unsigned char* ws, cudaStream_t st,
                        double* mean_out, double* cov_out, int stats_only, int& launches, int c0 = 0, int nc = -1,
                        cudaStream_t st_init = nullptr) {
    if (nc < 0) nc = p.cols;
    const bool fork = st_init != nullptr && st_init != st;
    CUtensorMap mm, tm;
    if (!p.wide) {
        CUresult cr = make_maps(rad, p.cols, p.N, p.B, &mm, &tm, p.T1);
        if (cr != CUDA_SUCCESS) {
            set_err(ctx, "cuTensorMapEncodeTiled (K1) failed (%d)", (int)cr);
            return SMF_ERR_CUDA;
        }
    }
    PilotArgs pa;
    pa.L = rad;
    pa.pil32 = (float*)(ws + p.o_pilot);
    pa.ghat32 = (float*)(ws + p.o_ghat);
    pa.cols = p.cols;
    pa.N = p.N;
    pa.B = p.B;
    pa.mask = ctx->mask;
    pa.nodata = ctx->nodata;
    pa.vmax = p.widei8 ? (unsigned*)(ws + p.o_vmax) : nullptr;
    pa.BEq = p.BEq8;
    pa.c0 = c0;
    {
        ProfScope ps(ctx, st, SMF_KERNEL_STATS);
        k0_pilot<<<nc, 128, 0, st>>>(pa);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "k0_pilot launch");
    ++launches;
    if (p.wide && p.widei8) {
        // exact-integer tensor-core statistics (widei8.cuh): scan (sigma, row maxima) ->
        // quantise to the int8 slice cube -> kind::i8 SYRK into the [BEp][BEp] partials
        I8ScanArgs sc;
        sc.L = rad;
        sc.pil32 = pa.pil32;
        sc.ghat32 = pa.ghat32;
        sc.sigma = (float*)(ws + p.o_sigma);
        sc.vmax = (unsigned*)(ws + p.o_vmax);
        sc.cols = p.cols;
        sc.N = p.N;
        sc.B = p.B;
        sc.BEq = p.BEq8;
        sc.mask = ctx->mask;
        sc.nodata = ctx->nodata;
        sc.c0 = c0;
        {
            ProfScope ps(ctx, st, SMF_KERNEL_STATS);
            const dim3 grid((p.N + kI8ScanPix - 1) / kI8ScanPix, nc);
            switch (k1w_scan_j(p.B)) {
                case 2: k1w_scan<2><<<grid, 256, 0, st>>>(sc); break;
                case 4: k1w_scan<4><<<grid, 256, 0, st>>>(sc); break;
                case 8: k1w_scan<8><<<grid, 256, 0, st>>>(sc); break;
                case 14: k1w_scan<14><<<grid, 256, 0, st>>>(sc); break;
                default: k1w_scan<20><<<grid, 256, 0, st>>>(sc); break;
            }
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_scan launch");
        ++launches;
        I8QuantArgs qa;
        qa.L = rad;
        qa.pil32 = pa.pil32;
        qa.sigma = sc.sigma;
        qa.vmax = sc.vmax;
        qa.slices = (int8_t*)(ws + p.o_slices);
        qa.cols = p.cols;
        qa.N = p.N;
        qa.B = p.B;
        qa.R = p.R8;
        qa.Np = p.Np8;
        qa.BEq = p.BEq8;
        qa.mask = ctx->mask;
        qa.c0 = c0;
        e = cudaFuncSetAttribute(k1w_quant, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k1w_quant_smem());
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_quant smem attribute");
        {
            ProfScope ps(ctx, st, SMF_KERNEL_STATS);
            k1w_quant<<<dim3((p.Np8 + kI8QTile * kI8QTiles - 1) / (kI8QTile * kI8QTiles), (p.R8 + kI8QRows - 1) / kI8QRows, nc), 256,
                        k1w_quant_smem(), st>>>(qa);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_quant launch");
        ++launches;
        CUtensorMap tq;
        {
            cuuint64_t dims[3] = {(cuuint64_t)p.Np8, (cuuint64_t)p.R8, (cuuint64_t)p.cols * kI8S};
            cuuint64_t strides[2] = {(cuuint64_t)p.Np8, (cuuint64_t)p.R8 * p.Np8};
            cuuint32_t box[3] = {(cuuint32_t)kI8Tile, (cuuint32_t)kI8Blk, 1};
            cuuint32_t estr[3] = {1, 1, 1};
            memset(&tq, 0, sizeof(tq));
            CUresult cr = g_encode(&tq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)qa.slices, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) {
                set_err(ctx, "cuTensorMapEncodeTiled (int8 slices) failed (%d)", (int)cr);
                return SMF_ERR_CUDA;
            }
        }
        I8SyrkArgs ya;
        ya.vmax = sc.vmax;
        ya.part = (double*)(ws + p.o_part1);
        ya.cols = p.cols;
        ya.N = p.N;
        ya.R = p.R8;
        ya.BEq = p.BEq8;
        ya.BEp = p.NBLKw * 128;
        ya.NBLK = p.NBLKw;
        ya.npairs = p.NBLKw * (p.NBLKw + 1) / 2;
        ya.nitems = nc * ya.npairs;
        ya.c0 = c0;
        e = cudaFuncSetAttribute(k1w_syrk_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k1w_i8_smem());
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_syrk_i8 smem attribute");
        {
            ProfScope ps(ctx, st, SMF_KERNEL_STATS);
            k1w_syrk_i8<<<std::min(ya.nitems, ctx->sm_count), kI8NT, k1w_i8_smem(), st>>>(tq, ya);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_syrk_i8 launch");
        ++launches;
    }
    if (p.wide && p.widetc) {
        float* sigma = (float*)(ws + p.o_sigma);
        {
            ProfScope ps(ctx, st, SMF_KERNEL_STATS);
            const long long warps = (long long)p.cols * p.N;
            k1w_sigma<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(rad, pa.ghat32, sigma, p.cols, p.N, p.B,
                                                                            ctx->mask, ctx->nodata);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_sigma launch");
        ++launches;
        WideTCArgs ta;
        ta.L = rad;
        ta.pil32 = pa.pil32;
        ta.ghat32 = pa.ghat32;
        ta.sigma = sigma;
        ta.part = (double*)(ws + p.o_part1);
        ta.cols = p.cols;
        ta.N = p.N;
        ta.B = p.B;
        ta.NBLK = p.NBLKw;
        ta.mask = ctx->mask;
        e = cudaFuncSetAttribute(k1w_stats_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem1);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_stats_tc smem attribute");
        {
            ProfScope ps(ctx, st, SMF_KERNEL_STATS);
            k1w_stats_tc<<<dim3(p.NBLKw * (p.NBLKw + 1) / 2, p.cols), kTW, p.smem1, st>>>(ta);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_stats_tc launch");
        ++launches;
    }
    if (p.wide) {
        WideStatsArgs wa;
        wa.L = rad;
        wa.pil32 = pa.pil32;
        wa.ghat32 = pa.ghat32;
        wa.part = (double*)(ws + p.o_part1);
        wa.cols = p.cols;
        wa.N = p.N;
        wa.B = p.B;
        wa.BE = p.BEw;
        wa.NB = p.NBw;
        wa.NG = p.NGw;
        wa.mask = ctx->mask;
        wa.nodata = ctx->nodata;
        if (!p.widetc && !p.widei8) {
            e = cudaFuncSetAttribute(k1w_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem1);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_stats smem attribute");
            {
                ProfScope ps(ctx, st, SMF_KERNEL_STATS);
                k1w_stats<<<dim3(p.NGw, p.cols), kWideNT1, p.smem1, st>>>(wa);
            }
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(ctx, e, "k1w_stats launch");
            ++launches;
        }
        WideInitArgs ia;
        ia.cs = col_state(p, ws, ctx->s_dev, ctx);
        ia.pil32 = pa.pil32;
        ia.part = wa.part;
        ia.BEp = (p.widetc || p.widei8) ? p.NBLKw * 128 : 0;
        ia.mean_out = mean_out;
        ia.cov_out = cov_out;
        ia.cols = p.cols;
        ia.N = p.N;
        ia.B = p.B;
        ia.BE = p.BEw;
        ia.NG = p.NGw;
        ia.use_albedo = ctx->use_albedo;
        ia.stats_only = stats_only;
        ia.energy = ctx->energy;
        ia.sym = 0;   // diagonal 128-blocks are (P + P^T)/2 for every statistics kernel (int8: 7-MMA diagonal pairs)
        ia.ridge_rel = ctx->ridge;
        ia.c0 = c0;
        cudaStream_t si = st;
        if (fork) {   // this range's k2w_init on st_init, behind its statistics
            e = cudaEventRecord(ctx->aux_fork, st);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(st_init, ctx->aux_fork, 0);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "k2w_init fork");
            si = st_init;
        }
        e = cudaFuncSetAttribute(k2w_init, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem2);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k2w_init smem attribute");
        {
            ProfScope ps(ctx, si, SMF_KERNEL_INIT);
            // a power of two of warps (the solves share each row among blockDim / 32 threads)
            int nti = 32;
            while (nti < kWideNTI && nti < p.B) nti *= 2;
            k2w_init<<<nc, nti, p.smem2, si>>>(ia);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k2w_init launch");
        ++launches;
        return SMF_OK;
    }
    StatsArgs sa;
    sa.pil32 = pa.pil32;
    sa.ghat32 = pa.ghat32;
    sa.part1 = (double*)(ws + p.o_part1);
    sa.cols = p.cols;
    sa.N = p.N;
    sa.B = p.B;
    sa.tpc = p.tpc1;
    sa.G = p.G1;
    sa.S = p.S1;
    sa.ttot = p.ttot1;
    sa.mask = ctx->mask;
    sa.nodata = ctx->nodata;
    void* k1 = p.k1tc ? stats_tc_kernel(p.B) : stats_kernel(p.B);
    e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem1);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "k1_stats smem attribute");
    {
        ProfScope ps(ctx, st, SMF_KERNEL_STATS);
        void* args[] = {(void*)&mm, (void*)&tm, (void*)&sa};
        e = launch_pdl(k1, dim3(p.G1), dim3(p.NT1), args, p.smem1, st);
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "k1_stats launch");
    ++launches;
    InitArgs ia;
    ia.cs = col_state(p, ws, ctx->s_dev, ctx);
    ia.pil32 = pa.pil32;
    ia.part1 = sa.part1;
    ia.mean_out = mean_out;
    ia.cov_out = cov_out;
    ia.cols = p.cols;
    ia.N = p.N;
    ia.B = p.B;
    ia.W1 = p.W1;
    ia.tpc = p.tpc1;
    ia.G1 = p.G1;
    ia.S1 = p.S1;
    ia.ttot = p.ttot1;
    ia.be_full = p.be_full;
    ia.use_albedo = ctx->use_albedo;
    ia.stats_only = stats_only;
    ia.ridge_rel = ctx->ridge;
    void* k2fn = k2_init_kernel(p.B);
    e = cudaFuncSetAttribute(k2fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem2);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "k2_init smem attribute");
    {
        ProfScope ps(ctx, st, SMF_KERNEL_INIT);
        void* args[] = {(void*)&ia};
        e = launch_pdl(k2fn, dim3(p.cols), dim3(256), args, p.smem2, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k2_init launch");
    }
    ++launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "k2_init launch");
    return SMF_OK;
}

}  // namespace

extern "C" {

int smf_abi_version(void) { return SMF_ABI_VERSION; }

int smf_supported_bands(int bands) { return supported(bands) ? 1 : 0; }

const char* smf_status_string(smf_status s) {
    switch (s) {
        case SMF_OK: return "SMF_OK";
        case SMF_ERR_INVALID_ARGUMENT: return "SMF_ERR_INVALID_ARGUMENT";
        case SMF_ERR_NOT_CONFIGURED: return "SMF_ERR_NOT_CONFIGURED";
        case SMF_ERR_SHAPE: return "SMF_ERR_SHAPE";
        case SMF_ERR_NUMERICAL: return "SMF_ERR_NUMERICAL";
        case SMF_ERR_CUDA: return "SMF_ERR_CUDA";
        case SMF_ERR_OUT_OF_MEMORY: return "SMF_ERR_OUT_OF_MEMORY";
    }
    return "SMF_UNKNOWN";
}

const char* smf_last_error(const smf_ctx* ctx) { return ctx ? ctx->err : "NULL context"; }

int smf_last_launch_count(const smf_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

smf_status smf_create(smf_ctx** out, int bands) {
    if (!out) return SMF_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (bands < 1) return SMF_ERR_INVALID_ARGUMENT;
    if (!supported(bands)) return SMF_ERR_SHAPE;
    smf_ctx* ctx = new (std::nothrow) smf_ctx();
    if (!ctx) return SMF_ERR_OUT_OF_MEMORY;
    ctx->bands = bands;
    cudaError_t e = cudaGetDevice(&ctx->device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, ctx->device);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->s_dev, sizeof(float) * bands);
    if (e != cudaSuccess) {
        delete ctx;
        return e == cudaErrorMemoryAllocation ? SMF_ERR_OUT_OF_MEMORY : SMF_ERR_CUDA;
    }
    std::call_once(g_encode_once, load_encode);
    *out = ctx;
    return SMF_OK;
}

smf_status smf_profile_enable(smf_ctx* ctx, int enable) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    for (auto& r : ctx->recs) {
        ctx->pool.push_back(r.a);
        ctx->pool.push_back(r.b);
    }
    ctx->recs.clear();
    ctx->prof = enable != 0;
    return SMF_OK;
}

smf_status smf_profile_read(smf_ctx* ctx, int kind, double* total_ms, int* launches) {
    if (!ctx || !total_ms || !launches) return SMF_ERR_INVALID_ARGUMENT;
    double tot = 0.0;
    int n = 0;
    for (auto& r : ctx->recs) {
        if (r.kind != kind) continue;
        cudaError_t e = cudaEventSynchronize(r.b);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "profile_read");
        tot += ms;
        ++n;
    }
    *total_ms = tot;
    *launches = n;
    return SMF_OK;
}

void smf_destroy(smf_ctx* ctx) {
    if (!ctx) return;
    smf_profile_enable(ctx, 0);
    for (auto e : ctx->pool) cudaEventDestroy(e);
    cudaFree(ctx->s_dev);
    if (ctx->h_buf) cudaFree(ctx->h_buf);
    if (ctx->h_stream) cudaStreamDestroy(ctx->h_stream);
    if (ctx->h_up) cudaStreamDestroy(ctx->h_up);
    if (ctx->h_down) cudaStreamDestroy(ctx->h_down);
    for (auto ev : ctx->h_ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    if (ctx->aux_fork) cudaEventDestroy(ctx->aux_fork);
    if (ctx->aux_join) cudaEventDestroy(ctx->aux_join);
    delete ctx;
}

smf_status smf_set_absorption(smf_ctx* ctx, const float* s_host, int bands) {
    if (!ctx || !s_host) return SMF_ERR_INVALID_ARGUMENT;
    ++ctx->gen;
    if (bands != ctx->bands) {
        set_err(ctx, "bands %d != context bands %d", bands, ctx->bands);
        return SMF_ERR_SHAPE;
    }
    cudaError_t e = cudaMemcpy(ctx->s_dev, s_host, sizeof(float) * bands, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "set_absorption");
    ctx->s_set = true;
    return SMF_OK;
}

smf_status smf_set_regularisation(smf_ctx* ctx, double epsilon, double ridge_rel, double r_floor) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    ++ctx->gen;
    if (!(epsilon > 0.0) || !(ridge_rel >= 0.0) || !(r_floor > 0.0)) {
        set_err(ctx, "need epsilon > 0, ridge_rel >= 0, r_floor > 0");
        return SMF_ERR_INVALID_ARGUMENT;
    }
    ctx->eps = epsilon;
    ctx->ridge = ridge_rel;
    ctx->r_floor = r_floor;
    return SMF_OK;
}

smf_status smf_set_iterations(smf_ctx* ctx, int n_iter, int use_sparsity, int use_albedo) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    ++ctx->gen;
    if (n_iter < 0) {
        set_err(ctx, "n_iter < 0");
        return SMF_ERR_INVALID_ARGUMENT;
    }
    ctx->n_iter = n_iter;
    ctx->use_sparsity = use_sparsity ? 1 : 0;
    ctx->use_albedo = use_albedo ? 1 : 0;
    return SMF_OK;
}

smf_status smf_set_nodata(smf_ctx* ctx, int enable, float value) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    ++ctx->gen;
    ctx->mask = enable ? 1 : 0;
    ctx->nodata = value;
    return SMF_OK;
}

smf_status smf_set_energy_trace(smf_ctx* ctx, int enable) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    ++ctx->gen;
    ctx->energy = enable ? 1 : 0;
    return SMF_OK;
}

smf_status smf_energy_trace(smf_ctx* ctx, const void* workspace, int cols, int pixels, double* energy_out,
                            void* stream) {
    if (!ctx || !workspace || !energy_out || cols < 1 || pixels < 2) return SMF_ERR_INVALID_ARGUMENT;
    if (!ctx->energy) {
        set_err(ctx, "energy trace not enabled (smf_set_energy_trace)");
        return SMF_ERR_NOT_CONFIGURED;
    }
    GroupLayout g = GroupLayout::make(cols, ctx->group);
    cudaError_t e = cudaSuccess;
    if (g.G == 1) {
        Plan p;
        make_plan(ctx, cols, pixels, p);
        e = cudaMemcpyAsync(energy_out, (const unsigned char*)workspace + p.o_energy, (size_t)p.n_energy * cols * 8,
                            cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
    } else {
        // [n_iter+1][partitions]: the full groups, then the remainder partition
        g.bytes(ctx, pixels);
        smf_ctx tmp = *ctx;
        tmp.group = 1;
        Plan pf;
        make_plan(&tmp, g.nfull, g.G * pixels, pf);
        const unsigned char* ws = (const unsigned char*)workspace;
        e = cudaMemcpy2DAsync(energy_out, (size_t)g.parts * 8, ws + g.o_full + pf.o_energy, (size_t)g.nfull * 8,
                              (size_t)g.nfull * 8, pf.n_energy, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
        if (e == cudaSuccess && g.rem > 0) {
            Plan pr;
            make_plan(&tmp, 1, g.rem * pixels, pr);
            e = cudaMemcpy2DAsync(energy_out + g.nfull, (size_t)g.parts * 8, ws + g.o_rem + pr.o_energy, 8, 8,
                                  pr.n_energy, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
        }
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "energy_trace copy");
    return SMF_OK;
}

smf_status smf_set_covariance_check(smf_ctx* ctx, int mode) {
    if (!ctx || mode < SMF_COVCHECK_OFF || mode > SMF_COVCHECK_ALWAYS) return SMF_ERR_INVALID_ARGUMENT;
    ++ctx->gen;
    ctx->lit_mode = mode;
    return SMF_OK;
}

smf_status smf_set_nvtx(smf_ctx* ctx, int enable) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    ctx->nvtx = enable ? 1 : 0;
    return SMF_OK;
}

smf_status smf_set_diagnostics(smf_ctx* ctx, int enable) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    ++ctx->gen;
    ctx->diag = enable ? 1 : 0;
    return SMF_OK;
}

// Copy a per-partition record array [rows][plan cols] (offset `which` of each plan) of the last
// retrieve into dst [rows][partitions], following the grouping layout (full groups, remainder).
static cudaError_t copy_records(smf_ctx* ctx, const unsigned char* ws, int cols, int pixels, size_t Plan::*which,
                                int rows, size_t elem, void* dst, cudaStream_t st) {
    if (!dst) return cudaSuccess;
    GroupLayout g = GroupLayout::make(cols, ctx->group);
    if (g.G == 1) {
        Plan p;
        make_plan(ctx, cols, pixels, p);
        return cudaMemcpyAsync(dst, ws + p.*which, (size_t)rows * cols * elem, cudaMemcpyDeviceToDevice, st);
    }
    g.bytes(ctx, pixels);
    smf_ctx tmp = *ctx;
    tmp.group = 1;
    Plan pf;
    make_plan(&tmp, g.nfull, g.G * pixels, pf);
    cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)g.parts * elem, ws + g.o_full + pf.*which, (size_t)g.nfull * elem,
                                      (size_t)g.nfull * elem, rows, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && g.rem > 0) {
        Plan pr;
        make_plan(&tmp, 1, g.rem * pixels, pr);
        e = cudaMemcpy2DAsync((unsigned char*)dst + (size_t)g.nfull * elem, (size_t)g.parts * elem,
                              ws + g.o_rem + pr.*which, elem, elem, rows, cudaMemcpyDeviceToDevice, st);
    }
    return e;
}

smf_status smf_iteration_diagnostics(smf_ctx* ctx, const void* workspace, int cols, int pixels, int64_t* nnz_out,
                                     double* q_out, int32_t* status_out, int32_t* literal_out, void* stream) {
    if (!ctx || !workspace || cols < 1 || pixels < 2) return SMF_ERR_INVALID_ARGUMENT;
    if (!ctx->diag) {
        set_err(ctx, "diagnostics not enabled (smf_set_diagnostics)");
        return SMF_ERR_NOT_CONFIGURED;
    }
    const unsigned char* ws = (const unsigned char*)workspace;
    const int rows = ctx->n_iter + 1;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = copy_records(ctx, ws, cols, pixels, &Plan::o_dnnz, rows, 8, nnz_out, st);
    if (e == cudaSuccess) e = copy_records(ctx, ws, cols, pixels, &Plan::o_dq, rows, 8, q_out, st);
    if (e == cudaSuccess) e = copy_records(ctx, ws, cols, pixels, &Plan::o_dst, rows, 4, status_out, st);
    if (e == cudaSuccess) e = copy_records(ctx, ws, cols, pixels, &Plan::o_dlit, rows, 4, literal_out, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "iteration_diagnostics copy");
    return SMF_OK;
}

smf_status smf_set_stats_kernel(smf_ctx* ctx, int kind) {
    if (!ctx || kind < SMF_STATS_AUTO || kind > SMF_STATS_INT8) return SMF_ERR_INVALID_ARGUMENT;
    if (kind == SMF_STATS_INT8 && narrow(ctx->bands)) {
        set_err(ctx, "int8 statistics kernel is the wide path's (bands %d use the narrow kernels)", ctx->bands);
        return SMF_ERR_SHAPE;
    }
    ++ctx->gen;
    if (kind == SMF_STATS_TENSOR && narrow(ctx->bands) && !k1tc_fits(ctx->bands)) {
        set_err(ctx, "tensor-core statistics kernel unavailable for %d bands", ctx->bands);
        return SMF_ERR_SHAPE;
    }
    ctx->stats_kernel = kind;
    return SMF_OK;
}

int smf_stats_kernel_used(const smf_ctx* ctx) {
    if (!ctx) return -1;
    const bool tc = narrow(ctx->bands) ? k1tc_fits(ctx->bands) : true;
    if (!narrow(ctx->bands) && (ctx->stats_kernel == SMF_STATS_AUTO || ctx->stats_kernel == SMF_STATS_INT8))
        return SMF_STATS_INT8;
    return (ctx->stats_kernel != SMF_STATS_FFMA && tc) ? SMF_STATS_TENSOR : SMF_STATS_FFMA;
}

smf_status smf_convert_layout(const float* in, int lines, int samples, int bands, int layout, float* out,
                              void* stream) {
    if (!in || !out || (const void*)in == (const void*)out || lines < 1 || samples < 1 || bands < 1 ||
        (layout != SMF_LAYOUT_BIL && layout != SMF_LAYOUT_BIP))
        return SMF_ERR_INVALID_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    if (layout == SMF_LAYOUT_BIP) {
        const int warps = 8, gx = std::min((samples + warps - 1) / warps, 64);
        k_bip_to_cpb<<<dim3(gx, std::min(lines, 65535)), warps * 32, 0, st>>>(in, out, lines, samples, bands);
    } else {
        k_bil_to_cpb<<<dim3((samples + 31) / 32, (bands + 31) / 32, std::min(lines, 65535)), dim3(32, 8), 0, st>>>(
            in, out, lines, samples, bands);
    }
    return cudaGetLastError() == cudaSuccess ? SMF_OK : SMF_ERR_CUDA;
}

smf_status smf_group_partitions(int cols, int group, int* n_partitions, int* first_cols) {
    if (cols < 1 || group < 1 || !n_partitions) return SMF_ERR_INVALID_ARGUMENT;
    const GroupLayout g = GroupLayout::make(cols, group);
    *n_partitions = g.parts;
    if (first_cols)
        for (int k = 0; k < g.parts; ++k) first_cols[k] = k * g.G;
    return SMF_OK;
}

smf_status smf_set_grouping(smf_ctx* ctx, int group) {
    if (!ctx || group < 1) return SMF_ERR_INVALID_ARGUMENT;
    ++ctx->gen;
    ctx->group = group;
    return SMF_OK;
}

smf_status smf_workspace_bytes(const smf_ctx* ctx, int cols, int pixels, size_t* bytes) {
    if (!ctx || !bytes || cols < 1 || pixels < 2) return SMF_ERR_INVALID_ARGUMENT;
    GroupLayout g = GroupLayout::make(cols, ctx->group);
    if (g.G == 1) {
        Plan p;
        make_plan(ctx, cols, pixels, p);
        *bytes = p.total;
        return SMF_OK;
    }
    *bytes = g.bytes(ctx, pixels);
    return SMF_OK;
}

static smf_status retrieve_eager(smf_ctx* ctx, const float* radiance, int cols, int pixels, float* enhancement,
                                 float* albedo, void* workspace, int32_t* column_status, void* stream) {
    if (ctx && ctx->group > 1 && cols >= 1) {
        // detector grouping: the full groups are one retrieval over nfull partitions of
        // G * pixels rows (the G columns of a group are contiguous in [cols][pixels][bands]),
        // the ragged remainder a second one; partition status expanded to columns
        GroupLayout g = GroupLayout::make(cols, ctx->group);
        if (g.G > 1) {
            if (!radiance || !workspace || !enhancement || !albedo || pixels < 2) return SMF_ERR_INVALID_ARGUMENT;
            g.bytes(ctx, pixels);   // region offsets
            unsigned char* ws = (unsigned char*)workspace;
            int32_t* pst = (int32_t*)(ws + g.o_status);
            const int saved = ctx->group;
            ctx->group = 1;
            smf_status rc = retrieve_eager(ctx, radiance, g.nfull, g.G * pixels, enhancement, albedo,
                                         ws + g.o_full, pst, stream);
            int launches = ctx->last_launches;
            if (rc == SMF_OK && g.rem > 0) {
                const size_t off = (size_t)g.nfull * g.G * pixels;
                rc = retrieve_eager(ctx, radiance + off * ctx->bands, 1, g.rem * pixels, enhancement + off,
                                  albedo + off, ws + g.o_rem, pst + g.nfull, stream);
                launches += ctx->last_launches;
            }
            ctx->group = saved;
            if (rc != SMF_OK) return rc;
            if (column_status) {
                k_expand_status<<<(cols + 255) / 256, 256, 0, (cudaStream_t)stream>>>(pst, column_status, cols, g.G);
                ++launches;
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) return cuda_fail(ctx, e, "expand status");
            }
            ctx->last_launches = launches;
            return SMF_OK;
        }
    }
    smf_status v = validate(ctx, radiance, cols, pixels, workspace);
    if (v != SMF_OK) return v;
    if (!enhancement || !albedo || (void*)enhancement == (void*)albedo ||
        (void*)enhancement == (void*)radiance || (void*)albedo == (void*)radiance) {
        set_err(ctx, "enhancement/albedo NULL or aliased");
        return SMF_ERR_INVALID_ARGUMENT;
    }
    ctx->last_launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    Plan p;
    make_plan(ctx, cols, pixels, p);
    CUtensorMap mm, tm;
    if (!p.wide) {
        CUresult cr = make_maps(radiance, cols, pixels, ctx->bands, &mm, &tm);
        if (cr != CUDA_SUCCESS) {
            set_err(ctx, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
            return SMF_ERR_CUDA;
        }
    }
    unsigned char* ws = (unsigned char*)workspace;
    int launches = 0;
    smf_status rc = SMF_OK;
    const int tail = wide_tail_cols(ctx, p);
    if (tail > 0) {
        // k2w_init runs one CTA per SM and every column costs the same, so the last
        // cols % SMs columns would hold a few SMs for a whole extra wave (598 columns on 148
        // SMs: 6 columns, ~0.9 ms). Their statistics go first and their k2w_init runs on a
        // second (high-priority) stream beside the other columns' statistics kernels; the
        // partitions are independent and every kernel is per-column deterministic,
        // so the results are bit-identical to the single-range launch order.
        if (!ctx->aux) {
            int lo = 0, hi = 0;
            cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
            if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, hi);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->aux_fork, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->aux_join, cudaEventDisableTiming);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "auxiliary stream");
        }
        cudaError_t e = cudaSuccess;
        if (wide_tail_mode() == 2) {   // the tail's statistics on the second stream too
            e = cudaEventRecord(ctx->aux_fork, st);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->aux, ctx->aux_fork, 0);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "tail fork");
            rc = launch_stats(ctx, p, radiance, ws, ctx->aux, nullptr, nullptr, 0, launches, cols - tail, tail);
        } else {
            rc = launch_stats(ctx, p, radiance, ws, st, nullptr, nullptr, 0, launches, cols - tail, tail, ctx->aux);
        }
        if (rc != SMF_OK) return rc;
        e = cudaEventRecord(ctx->aux_join, ctx->aux);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k2w_init join record");
        rc = launch_stats(ctx, p, radiance, ws, st, nullptr, nullptr, 0, launches, 0, cols - tail);
        if (rc != SMF_OK) return rc;
        e = cudaStreamWaitEvent(st, ctx->aux_join, 0);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k2w_init join");
    } else {
        rc = launch_stats(ctx, p, radiance, ws, st, nullptr, nullptr, 0, launches);
        if (rc != SMF_OK) return rc;
    }
    ColState cs = col_state(p, ws, ctx->s_dev, ctx);
    SweepArgs sa;
    sa.enh = enhancement;
    sa.alb = albedo;
    sa.z32 = cs.z32;
    sa.mhat32 = cs.mhat32;
    sa.kc32 = cs.kc32;
    sa.q32 = cs.q32;
    sa.status = cs.status;
    sa.part3 = (double*)(ws + p.o_part3);
    sa.cols = cols;
    sa.N = pixels;
    sa.B = p.B;
    sa.tpc = p.tpc;
    sa.G = p.G;
    sa.S = p.S;
    sa.ttot = p.ttot;
    sa.n_iter = ctx->n_iter;
    sa.use_sparsity = ctx->use_sparsity;
    sa.use_albedo = ctx->use_albedo;
    sa.eps = (float)ctx->eps;
    sa.r_floor = (float)ctx->r_floor;
    sa.energy = ctx->energy;
    sa.mask = ctx->mask;
    sa.nodata = ctx->nodata;
    sa.bulk = p.wide && ((uintptr_t)radiance % 16 == 0) && ((size_t)pixels * p.B % 4 == 0) &&
              ((size_t)(pixels % kWideT3) * p.B % 4 == 0);
    UpdateArgs ua;
    ua.cs = cs;
    ua.part3 = sa.part3;
    ua.energy = (double*)(ws + p.o_energy);
    ua.k = 0;
    ua.energy_on = ctx->energy;
    ua.cols = cols;
    ua.N = pixels;
    ua.B = p.B;
    ua.tpc = p.tpc;
    ua.G = p.G;
    ua.S = p.S;
    ua.ttot = p.ttot;
    ua.L = radiance;
    ua.enh = enhancement;
    ua.alb = albedo;
    ua.lit = (double*)(ws + p.o_lit);
    ua.lit_stride = p.lit_stride;
    ua.r_floor = (float)ctx->r_floor;
    ua.use_albedo = ctx->use_albedo;
    ua.lit_mode = ctx->lit_mode;
    CUtensorMap fmap;   // wide: the solve-ready factor, streamed by k2w_update's solves
    if (p.wide) {
        CUresult cr = make_factor_map(cs.ainv, cols, p.B, &fmap);
        if (cr != CUDA_SUCCESS) {
            set_err(ctx, "cuTensorMapEncodeTiled (factor) failed (%d)", (int)cr);
            return SMF_ERR_CUDA;
        }
    }
    DiagArgs da;
    da.enh = enhancement;
    da.cs = cs;
    da.nnz = (long long*)(ws + p.o_dnnz);
    da.q = (double*)(ws + p.o_dq);
    da.st = (int*)(ws + p.o_dst);
    da.lit = (int*)(ws + p.o_dlit);
    da.cols = cols;
    da.N = pixels;
    const size_t smem_up = p.wide ? k2w_update_smem(p.B, ctx->energy) : (size_t)p.B * p.B * 8;
    void* ufn = p.wide ? reinterpret_cast<void*>(&k2w_update) : reinterpret_cast<void*>(&k2_update);
    cudaError_t e0 = cudaFuncSetAttribute(ufn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_up);
    if (e0 != cudaSuccess) return cuda_fail(ctx, e0, "k2_update smem attribute");
    void* kfn = p.wide ? wide_sweep_kernel(p.B, ctx->mask != 0) : sweep_kernel(p.B);
    e0 = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem3);
    if (e0 != cudaSuccess) return cuda_fail(ctx, e0, "k3_sweep smem attribute");
    for (int k = 0; k <= ctx->n_iter; ++k) {
        if (k > 0) {
            {
                ProfScope ps(ctx, st, SMF_KERNEL_UPDATE);
                if (p.wide)
                    k2w_update<<<cols, kWideNT2, smem_up, st>>>(ua, fmap);
                else {
                    void* args[] = {(void*)&ua};
                    e0 = launch_pdl(reinterpret_cast<const void*>(&k2_update), dim3(cols), dim3(128), args, smem_up,
                                    st);
                    if (e0 != cudaSuccess) return cuda_fail(ctx, e0, "k2_update launch");
                }
            }
            e0 = cudaGetLastError();
            if (e0 != cudaSuccess) return cuda_fail(ctx, e0, "k2_update launch");
            ++launches;
        }
        sa.k = k;
        sa.rev = serpentine() && p.wide == 0 ? (k & 1) == 0 : 0;   // K1 walks forward
        sa.keep = serpentine() ? l2_keep_tiles(p) : 0;
        cudaError_t e;
        {
            ProfScope ps(ctx, st, SMF_KERNEL_SWEEP);
            if (p.wide) {
                const float* rad = radiance;
                void* args[] = {(void*)&sa, (void*)&rad};
                e = cudaLaunchKernel(kfn, dim3(p.G), dim3(kWideNT3), args, p.smem3, st);
            } else {
                void* args[] = {(void*)&mm, (void*)&tm, (void*)&sa};
                e = launch_pdl(kfn, dim3(p.G), dim3(kTileRows), args, p.smem3, st);
            }
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "sweep launch");
        ++launches;
        if (ctx->energy) {   // Eq. 8 energy of iteration k from the sweep's partials
            ua.k = k;
            k_energy<<<(cols + 127) / 128, 128, 0, st>>>(ua);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(ctx, e, "k_energy launch");
            ++launches;
        }
        if (ctx->diag) {   // per-iteration nonzero count, q^k, status, literal checks
            da.k = k;
            k_diag<<<cols, 256, 0, st>>>(da);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(ctx, e, "k_diag launch");
            ++launches;
        }
    }
    if (column_status) {
        k_copy_status<<<(cols + 255) / 256, 256, 0, st>>>(cs.status, column_status, cols);
        ++launches;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "retrieve launch");
    ctx->last_launches = launches;
    return SMF_OK;
}

smf_status smf_retrieve(smf_ctx* ctx, const float* radiance, int cols, int pixels, float* enhancement,
                        float* albedo, void* workspace, int32_t* column_status, void* stream) {
    if (!ctx || !ctx->graph || ctx->prof || !stream)   // (the legacy stream cannot be captured)
        return retrieve_eager(ctx, radiance, cols, pixels, enhancement, albedo, workspace, column_status, stream);
    cudaStream_t st = (cudaStream_t)stream;
    const smf_ctx::GKey key = {radiance, cols, pixels, enhancement, albedo, workspace, column_status, stream,
                               ctx->gen};
    if (!(ctx->gexec && key == ctx->gkey)) {
        if (ctx->gexec) {
            cudaGraphExecDestroy(ctx->gexec);
            ctx->gexec = nullptr;
        }
        cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "graph capture begin");
        smf_status rc = retrieve_eager(ctx, radiance, cols, pixels, enhancement, albedo, workspace, column_status,
                                       stream);
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(st, &graph);
        if (rc != SMF_OK) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "graph capture end");
        e = cudaGraphInstantiate(&ctx->gexec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            ctx->gexec = nullptr;
            return cuda_fail(ctx, e, "graph instantiate");
        }
        ctx->gkey = key;
        ctx->glaunches = ctx->last_launches;
    }
    cudaError_t e = cudaGraphLaunch(ctx->gexec, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "graph launch");
    ctx->last_launches = ctx->glaunches;
    return SMF_OK;
}

smf_status smf_set_graph(smf_ctx* ctx, int enable) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    ctx->graph = enable ? 1 : 0;
    if (!ctx->graph && ctx->gexec) {
        cudaGraphExecDestroy(ctx->gexec);
        ctx->gexec = nullptr;
    }
    return SMF_OK;
}

smf_status smf_synchronize(smf_ctx* ctx, void* stream, const int32_t* column_status, int cols,
                           int* first_failed_column) {
    if (!ctx) return SMF_ERR_INVALID_ARGUMENT;
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "synchronize");
    if (first_failed_column) *first_failed_column = -1;
    if (!column_status || cols < 1) return SMF_OK;
    int32_t* h = new (std::nothrow) int32_t[cols];
    if (!h) return SMF_ERR_OUT_OF_MEMORY;
    e = cudaMemcpy(h, column_status, sizeof(int32_t) * cols, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        delete[] h;
        return cuda_fail(ctx, e, "synchronize status");
    }
    int first = -1;
    for (int c = 0; c < cols && first < 0; ++c)
        if (h[c] != SMF_COL_OK) first = c;
    delete[] h;
    if (first_failed_column) *first_failed_column = first;
    if (first >= 0) {
        set_err(ctx, "column %d failed", first);
        return SMF_ERR_NUMERICAL;
    }
    return SMF_OK;
}

smf_status smf_host_chunk_cols(const smf_ctx* ctx, int cols, int* chunk_cols) {
    if (!ctx || !chunk_cols || cols < 1) return SMF_ERR_INVALID_ARGUMENT;
    *chunk_cols = host_chunk_cols(ctx->group, cols);
    return SMF_OK;
}

smf_status smf_retrieve_host(smf_ctx* ctx, const float* radiance_host, int cols, int pixels,
                             float* enhancement_host, float* albedo_host, int32_t* column_status_host) {
    // Columns are independent partitions, so the cube is streamed in column
    // chunks through two device buffers: the upload of chunk i+1 (copy engine, h_up)
    // overlaps the retrieval of chunk i (h_stream) and the download of chunk i-1 (h_down).
    if (!ctx || !radiance_host || !enhancement_host || !albedo_host || cols < 1 || pixels < 2)
        return SMF_ERR_INVALID_ARGUMENT;
    cudaError_t e = cudaSuccess;
    if (!ctx->h_stream) {
        e = cudaStreamCreateWithFlags(&ctx->h_stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->h_up, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->h_down, cudaStreamNonBlocking);
        for (int k = 0; k < 6 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&ctx->h_ev[k], cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "stream create");
    }
    const int ccols = host_chunk_cols(ctx->group, cols);   // whole detector groups (last may be short)
    const int nchunks = (cols + ccols - 1) / ccols;           // every chunk non-empty
    size_t ws_bytes = 0, ws_last = 0;
    smf_workspace_bytes(ctx, ccols, pixels, &ws_bytes);
    smf_workspace_bytes(ctx, cols - (nchunks - 1) * ccols > 0 ? cols - (nchunks - 1) * ccols : ccols, pixels,
                        &ws_last);
    ws_bytes = std::max(ws_bytes, ws_last);
    const size_t col_rad = (size_t)pixels * ctx->bands * 4, col_map = (size_t)pixels * 4;
    const size_t rad_bytes = align_up((size_t)ccols * col_rad, 256);
    const size_t map_bytes = align_up((size_t)ccols * col_map, 256);
    const size_t st_bytes = align_up((size_t)cols * 4, 256);
    const size_t need = 2 * (rad_bytes + 2 * map_bytes) + st_bytes + ws_bytes;
    if (need > ctx->h_buf_bytes) {
        if (ctx->h_buf) cudaFree(ctx->h_buf);
        ctx->h_buf = nullptr;
        ctx->h_buf_bytes = 0;
        e = cudaMalloc(&ctx->h_buf, need);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "retrieve_host alloc");
        ctx->h_buf_bytes = need;
    }
    unsigned char* b = (unsigned char*)ctx->h_buf;
    float *d_rad[2], *d_enh[2], *d_alb[2];
    for (int k = 0; k < 2; ++k) {
        unsigned char* base = b + k * (rad_bytes + 2 * map_bytes);
        d_rad[k] = (float*)base;
        d_enh[k] = (float*)(base + rad_bytes);
        d_alb[k] = (float*)(base + rad_bytes + map_bytes);
    }
    int32_t* d_st = (int32_t*)(b + 2 * (rad_bytes + 2 * map_bytes));
    void* d_ws = b + 2 * (rad_bytes + 2 * map_bytes) + st_bytes;
    cudaEvent_t* up = ctx->h_ev;          // chunk i uploaded into slot i % 2
    cudaEvent_t* done = ctx->h_ev + 2;    // chunk i computed
    cudaEvent_t* down = ctx->h_ev + 4;    // chunk i downloaded (slot free)
    int launches = 0;
    for (int i = 0; i < nchunks; ++i) {
        const int c0 = i * ccols, nc = std::min(ccols, cols - c0), k = i & 1;
        if (nc <= 0) break;
        // upload: slot k is free once chunk i-2 has been computed
        if (i >= 2) e = cudaStreamWaitEvent(ctx->h_up, done[k], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_rad[k], radiance_host + (size_t)c0 * pixels * ctx->bands, (size_t)nc * col_rad,
                                cudaMemcpyHostToDevice, ctx->h_up);
        if (e == cudaSuccess) e = cudaEventRecord(up[k], ctx->h_up);
        // compute: after the upload, and after chunk i-2's outputs have left slot k
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->h_stream, up[k], 0);
        if (e == cudaSuccess && i >= 2) e = cudaStreamWaitEvent(ctx->h_stream, down[k], 0);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "retrieve_host upload");
        smf_status rc = retrieve_eager(ctx, d_rad[k], nc, pixels, d_enh[k], d_alb[k], d_ws, d_st + c0, ctx->h_stream);
        if (rc != SMF_OK) return rc;
        launches += ctx->last_launches;
        e = cudaEventRecord(done[k], ctx->h_stream);
        // download
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->h_down, done[k], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(enhancement_host + (size_t)c0 * pixels, d_enh[k], (size_t)nc * col_map,
                                cudaMemcpyDeviceToHost, ctx->h_down);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(albedo_host + (size_t)c0 * pixels, d_alb[k], (size_t)nc * col_map,
                                cudaMemcpyDeviceToHost, ctx->h_down);
        if (e == cudaSuccess) e = cudaEventRecord(down[k], ctx->h_down);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "retrieve_host download");
    }
    ctx->last_launches = launches;
    if (column_status_host) {
        e = cudaStreamWaitEvent(ctx->h_down, done[(nchunks - 1) & 1], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(column_status_host, d_st, (size_t)cols * 4, cudaMemcpyDeviceToHost, ctx->h_down);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->h_down);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->h_stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "retrieve_host sync");
    if (column_status_host)
        for (int c = 0; c < cols; ++c)
            if (column_status_host[c] != SMF_COL_OK) return SMF_ERR_NUMERICAL;
    return SMF_OK;
}

smf_status smf_column_model(smf_ctx* ctx, const void* workspace, int cols, int pixels, double* mu_out,
                            double* q_out, void* stream) {
    if (!ctx || !workspace || cols < 1 || pixels < 2) return SMF_ERR_INVALID_ARGUMENT;
    // per partition (the grouping layout resolved as for the energy trace): mu [parts][B], q [parts]
    const unsigned char* ws = (const unsigned char*)workspace;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = copy_records(ctx, ws, cols, pixels, &Plan::o_mu, 1, (size_t)ctx->bands * 8, mu_out, st);
    if (e == cudaSuccess) e = copy_records(ctx, ws, cols, pixels, &Plan::o_q64, 1, 8, q_out, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "column_model");
    return SMF_OK;
}

smf_status smf_initial_statistics(smf_ctx* ctx, const float* radiance, int cols, int pixels, double* mean_out,
                                  double* cov_out, void* workspace, void* stream) {
    smf_status v = validate(ctx, radiance, cols, pixels, workspace);
    if (v != SMF_OK) return v;
    Plan p;
    make_plan(ctx, cols, pixels, p);
    int launches = 0;
    return launch_stats(ctx, p, radiance, (unsigned char*)workspace, (cudaStream_t)stream, mean_out, cov_out, 1,
                        launches);
}

}  // extern "C"
