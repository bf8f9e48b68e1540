/*
 * smf.h -- C ABI of libsmf.so: the B200 (sm_100a) hot path of the sparse,
 * albedo-corrected matched filter of Foote et al., "Fast and Accurate
 * Retrieval of Methane Concentration from Imaging Spectrometer Data Using
 * Sparsity Prior" (IEEE TGRS 2020, arXiv 2003.02978).
 *
 * Citations: P:n = line n of the paper text; "Fig. alg line k" =
 * line k of its algorithm figure "AlbedoReWeightL1Filter".
 *
 * The operation (smf_retrieve) is the procedure AlbedoReWeightL1Filter(D, s,
 * N_iter) run independently on every detector column of a radiance
 * cube (one partition = one column):
 *   mu0, C0 (lines 2-3) -> albedo r_i (line 5, Eq. 7) -> alpha0 (line 6, Eq. 3)
 *   -> N_iter x { w (line 9, Eq. 5), mu^k, C^k (lines 10-14, Eq. 10-11),
 *                 alpha^k = max((.)-w)/(r q), 0) (line 16, Eq. 6/8) }.
 * The variant switches follow the figure's caption: sparsity off
 * => w = 0; albedo off => r = 1. Readings of points the paper leaves open
 * (clamping alpha0 before it feeds w^1/mu^1/C^1, the ridge, r floor, signed
 * zero, 1/N) are listed in DESIGN.md section 2 and are the oracle's too.
 *
 * Conventions for every call:
 *  - Every call returns smf_status; nothing throws or aborts across the ABI.
 *  - Device pointers are CUDA device (or managed) memory owned by the CALLER;
 *    the library never frees them. Host pointers are read during the call only.
 *  - Layouts are C-contiguous: radiance [cols][pixels][bands] fp32 (column
 *    major over detectors, pixels = along-track lines, bands contiguous);
 *    enhancement / albedo [cols][pixels] fp32; column_status [cols] int32.
 *  - Units: radiance arbitrary (the method is invariant to L -> cL);
 *    s in (ppm m)^-1 (d ln L / d(ppm m), negative in absorption bands, P:119,
 *    P:410); enhancement alpha in ppm m.
 *  - stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Context threading: one retrieve in flight per (context, workspace) pair;
 *    separate contexts are independent. A context binds to the CUDA device
 *    current at smf_create.
 */
#ifndef SMF_H
#define SMF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMF_ABI_VERSION 1

typedef struct smf_ctx smf_ctx; /* opaque, library-owned (create/destroy) */

typedef enum {
    SMF_OK = 0,
    SMF_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, bands < 1, cols < 1, pixels < 2,
                                     n_iter < 0, eps <= 0, ridge < 0, r_floor <= 0,
                                     aliasing outputs */
    SMF_ERR_NOT_CONFIGURED = 2,   /* retrieve before smf_set_absorption */
    SMF_ERR_SHAPE = 3,            /* bands != context bands, workspace too small,
                                     or a shape this build does not support
                                     (see smf_supported_bands) */
    SMF_ERR_NUMERICAL = 4,        /* >= 1 column failed; per-column codes in column_status */
    SMF_ERR_CUDA = 5,             /* CUDA runtime error; text via smf_last_error() */
    SMF_ERR_OUT_OF_MEMORY = 6
} smf_status;

/* Per-column status codes written to column_status (device int32 [cols]). A
 * failed column's enhancement and albedo are NaN; other columns are unaffected
 * (cf. the paper skipping censored regions). */
enum {
    SMF_COL_OK = 0,
    SMF_COL_NONFINITE = 1,         /* a non-finite radiance value in the column */
    SMF_COL_DEGENERATE_MEAN = 2,   /* mu0 . mu0 = 0 with albedo correction (Eq. 7 undefined) */
    SMF_COL_NOT_SPD = 3,           /* C^k + rho I not numerically positive definite */
    SMF_COL_DEGENERATE_TARGET = 4, /* t^T (C^k+rho I)^-1 t <= 0 or non-finite (Eq. 3/6 undefined) */
    SMF_COL_INSUFFICIENT = 5       /* nodata masking left fewer than 2 valid pixels in the partition */
};

/* Create a context for `bands` spectral bands on the current CUDA device.
 * Defaults: eps = 1e-2 ppm m, ridge_rel = 0, r_floor = 0.05, n_iter = 30,
 * sparsity and albedo correction on. *out = NULL on failure. */
smf_status smf_create(smf_ctx** out, int bands);

/* Destroy a context (NULL-safe). Does not touch caller-owned buffers. */
void smf_destroy(smf_ctx* ctx);

/* Set the unit absorption spectrum s (host fp32 [bands], copied). s is the
 * per-band slope d ln L / d(ppm m); the target spectrum is
 * t = mu (.) s (Eq. 9), recomputed from mu^k every iteration. */
smf_status smf_set_absorption(smf_ctx* ctx, const float* s_host, int bands);

/* Regularisation constants:
 *  epsilon   > 0: the reweighting stabiliser of Eq. 5, w = 1/(alpha + eps);
 *  ridge_rel >= 0: rho = ridge_rel * tr(C0)/bands, computed once per column from
 *              C0 and added to every factored covariance (C0 and all C^k);
 *              0 reproduces the paper's unregularised covariance;
 *  r_floor   > 0: r~ = max(r, r_floor) wherever r enters the iteration
 *              (denominator and signal removal); the raw r is reported. */
smf_status smf_set_regularisation(smf_ctx* ctx, double epsilon, double ridge_rel, double r_floor);

/* N_iter >= 0 (30 in the paper) and the Table I switches
 * (P:389-391): use_sparsity = 0 enforces w = 0; use_albedo = 0
 * sets r = 1. N_iter = 0 returns the unclamped closed form alpha0 (Eq. 3,
 * divided by r~ when albedo correction is on). */
smf_status smf_set_iterations(smf_ctx* ctx, int n_iter, int use_sparsity, int use_albedo);

/* Device workspace bytes needed by smf_retrieve for this shape (host call). */
smf_status smf_workspace_bytes(const smf_ctx* ctx, int cols, int pixels, size_t* bytes);

/* Bands supported by this build: returns 1 if `bands` is supported, else 0.
 * This build supports every band count 1 <= bands <= 626 (narrow kernels for
 * bands % 4 == 0 up to 96, the wide path otherwise; 626 is the largest band count the
 * parity suite exercises). */
int smf_supported_bands(int bands);

/* The retrieval. Validates host-side arguments synchronously, enqueues every
 * step on `stream` (all arithmetic in this library's CUDA kernels) and
 * returns without synchronising.
 *   radiance      device fp32 [cols][pixels][bands], read-only, 16-byte aligned when
 *                 bands % 4 == 0 and bands <= 96 (TMA path), else 4-byte aligned
 *   enhancement   device fp32 [cols][pixels] out: alpha^{N_iter} in ppm m
 *   albedo        device fp32 [cols][pixels] out: raw r_i (Eq. 7), 1 if albedo off
 *   workspace     device, >= smf_workspace_bytes(cols, pixels), 256-byte aligned
 *   column_status device int32 [cols] out, or NULL
 * enhancement and albedo must not alias each other or the radiance.
 * Ordering: everything is ordered after the work already in `stream` and complete when
 * `stream` reaches the point after this call. On the wide path with more columns than SMs the
 * initial factorisation of the last cols mod SMs columns (independent partitions)
 * runs on a second stream the context owns, forked from and joined back into `stream` by
 * events inside this call -- a caller only ever synchronises with `stream`. */
smf_status smf_retrieve(smf_ctx* ctx, const float* radiance, int cols, int pixels,
                        float* enhancement, float* albedo, void* workspace,
                        int32_t* column_status, void* stream);

/* CUDA-graph mode (enable != 0; default off): smf_retrieve captures its launch
 * sequence (statistics, factorisation, N_iter + 1 sweeps and updates) into a CUDA
 * graph on the first call and replays it with one cudaGraphLaunch while the call's
 * pointers, shape and stream and the context's settings (every smf_set_* call
 * invalidates it) are unchanged; results are bitwise those of the eager launches.
 * Calls on the legacy default stream (stream == NULL) and calls with profiling on
 * run eagerly. smf_retrieve_host always runs eagerly. */
smf_status smf_set_graph(smf_ctx* ctx, int enable);

/* Wait for `stream`, then read `column_status` (device int32 [cols], as passed
 * to smf_retrieve) and report the first failed column (-1 if none).
 * Returns SMF_ERR_NUMERICAL if any column failed, SMF_ERR_CUDA on a CUDA error. */
smf_status smf_synchronize(smf_ctx* ctx, void* stream, const int32_t* column_status, int cols,
                           int* first_failed_column);

/* End-to-end convenience call with HOST buffers (pinned for full overlap;
 * pageable works): streams the cube through the device in column chunks (columns
 * are independent partitions) -- the host->device copy of chunk i+1
 * overlaps smf_retrieve of chunk i and the device->host copy of chunk i-1 on three
 * internal streams, with context-owned device buffers (two chunk slots + one
 * workspace, grown on demand and reused across calls) -- then synchronises.
 * Each chunk's results are bitwise those of smf_retrieve on the same columns (the
 * whole-cube launch differs only in the per-column fp reduction order).
 * Returns SMF_ERR_NUMERICAL if any column failed. */
smf_status smf_retrieve_host(smf_ctx* ctx, const float* radiance_host, int cols, int pixels,
                             float* enhancement_host, float* albedo_host,
                             int32_t* column_status_host);

/* Columns per chunk that smf_retrieve_host uses for a cube of `cols` columns with
 * this context's grouping (whole detector groups per chunk; ~24 chunks, at most
 * cols/16; the last chunk may be shorter). Writes *chunk_cols; SMF_ERR_INVALID_ARGUMENT for a
 * NULL pointer or cols < 1. */
smf_status smf_host_chunk_cols(const smf_ctx* ctx, int cols, int* chunk_cols);

/* Per-partition background model after the last smf_retrieve (N_iter >= 1) that used
 * `workspace`: mu^{N_iter} (device fp64 [partitions][bands], or NULL) and
 * q^{N_iter} = t^T (C+rho I)^-1 t (device fp64 [partitions], or NULL); partitions =
 * cols without grouping, else the full groups then the remainder (smf_group_partitions).
 * Enqueued on `stream`. */
smf_status smf_column_model(smf_ctx* ctx, const void* workspace, int cols, int pixels,
                            double* mu_out, double* q_out, void* stream);

/* Initial statistics only (Fig. alg lines 2-3): mu0 (device fp64 [cols][bands])
 * and C0 (device fp64 [cols][bands][bands], population 1/N covariance, no
 * ridge), using the same statistics kernel as smf_retrieve. */
smf_status smf_initial_statistics(smf_ctx* ctx, const float* radiance, int cols, int pixels,
                                  double* mean_out, double* cov_out, void* workspace,
                                  void* stream);

/* Which kernel computes the initial statistics (Fig. alg lines 2-3, the
 * batched bands x bands SYRK): SMF_STATS_AUTO (default: the narrow path's tf32
 * tensor-core kernel where the shape fits, the wide path's int8 kernel), SMF_STATS_FFMA
 * (fp32 FFMA 8x8 register tiles), SMF_STATS_TENSOR (tcgen05 kind::tf32 with the
 * two-term accuracy-preserving split of DESIGN.md 5.5; SMF_ERR_SHAPE if this band
 * count has no tensor-core variant), SMF_STATS_INT8 (wide path only, DESIGN.md 5.6:
 * tcgen05 kind::i8 on a three-digit fixed-point split with exact int32 accumulation;
 * SMF_ERR_SHAPE for narrow band counts). smf_stats_kernel_used returns the kernel AUTO
 * resolves to, -1 for a NULL context. */
enum { SMF_STATS_AUTO = 0, SMF_STATS_FFMA = 1, SMF_STATS_TENSOR = 2, SMF_STATS_INT8 = 3 };
smf_status smf_set_stats_kernel(smf_ctx* ctx, int kind);
int smf_stats_kernel_used(const smf_ctx* ctx);

/* Nodata masking (the paper skips censored regions). With
 * enable != 0 a pixel is nodata when any of its bands is non-finite or equals `value`
 * (AVIRIS-NG files use -9999): it is left out of every statistic of its partition
 * (mean, covariance, the iteration's sufficient statistics; N counts valid pixels only)
 * and its enhancement and albedo are NaN; a partition with fewer than 2 valid pixels
 * gets SMF_COL_INSUFFICIENT. Disabled (default), any non-finite value fails its column
 * with SMF_COL_NONFINITE. */
smf_status smf_set_nodata(smf_ctx* ctx, int enable, float value);

/* On-device layout conversion of a radiance cube as stored on disk (AVIRIS-NG style,
 * SPEC S:23) into the retrieval layout [samples][lines][bands] (samples =
 * detector columns = cols, lines = along-track pixels):
 *   SMF_LAYOUT_BIL: in [lines][bands][samples] (band interleaved by line);
 *   SMF_LAYOUT_BIP: in [lines][samples][bands] (band interleaved by pixel).
 * in, out: device fp32, caller-owned, must not overlap; enqueued on `stream`. Any
 * number of lines (the kernels grid-stride over lines). */
enum { SMF_LAYOUT_BIL = 0, SMF_LAYOUT_BIP = 1 };
smf_status smf_convert_layout(const float* in, int lines, int samples, int bands, int layout, float* out,
                              void* stream);

/* Detector grouping (the paper processes 5 adjacent detectors per
 * partition, and all 598 together for the convergence study):
 * with group = G > 1, smf_retrieve pools G adjacent columns into one partition
 * (one mean, covariance, target and albedo reference per partition, Fig. alg applied
 * to the partition's G * pixels rows); the cols % G columns left over form a ragged
 * remainder partition (598 = 119 x 5 + 3), and G >= cols is the all-columns mode.
 * Layouts are unchanged ([cols][pixels][bands] in, [cols][pixels] out, column_status
 * per column = the status of its partition); smf_workspace_bytes accounts for the
 * grouping; smf_energy_trace then returns [N_iter + 1][partitions]. G = 1 (default)
 * is one partition per column. smf_column_model reports per partition;
 * smf_initial_statistics always treats each column as a partition.
 * smf_group_partitions: number of partitions and (optional, host int[n]) the first
 * column of each. */
smf_status smf_set_grouping(smf_ctx* ctx, int group);
smf_status smf_group_partitions(int cols, int group, int* n_partitions, int* first_cols);

/* Energy trace (the objective of Eq. 8, tracked over the iterations in
 * Fig. 4). When enabled, smf_retrieve also records per column and per
 * iteration k = 0..N_iter
 *   E_k = sum_i d_i^T (C^k + rho I)^-1 d_i + sum_i r~_i w_i^k |alpha_i^k|,
 *   d_i = L_i - r~_i alpha_i^k t^k - mu^k
 * with the statistics mu^k, C^k, t^k and the weights w^k of iteration k at the updated
 * alpha^k (alpha0 as stored, w^0 = 0; reading C19). It is assembled exactly
 * from per-column sufficient statistics (no per-pixel whitening): two more sums in the
 * sweep and a rank-3 Woodbury trace, plus one small kernel launch per sweep.
 * smf_energy_trace copies the trace of the last smf_retrieve that used `workspace`
 * (device fp64 [N_iter + 1][cols], NaN for failed columns) to energy_out, enqueued on
 * `stream`; SMF_ERR_NOT_CONFIGURED if the trace was not enabled. The workspace size
 * depends on this switch and N_iter (query smf_workspace_bytes after setting them). */
smf_status smf_set_energy_trace(smf_ctx* ctx, int enable);
smf_status smf_energy_trace(smf_ctx* ctx, const void* workspace, int cols, int pixels, double* energy_out,
                            void* stream);

/* Per-iteration positive-definiteness of C^k + rho I (Fig. alg lines 14-16; the
 * oracle factors every C^k and reports a Cholesky pivot <= bands * 2^-52 * max diag as
 * SMF_COL_NOT_SPD, reading C16'). The hot path never forms C^k: it applies the
 * exact rank-3 identity C^k = C0 + U M U^T through a Woodbury solve on (C0 + rho I)^-1, whose
 * fp32-statistics precision cannot resolve a collapse of C^k below ~1e-6 of C0. So each
 * iteration also computes the smallest eigenvalue of (C0+rho I)^-1 (C^k+rho I) from the 3 x 3
 * Woodbury capacitance, and when it is <= 1e-3 (mode SMF_COVCHECK_AUTO, default) or always
 * (SMF_COVCHECK_ALWAYS) the column's iteration is done literally in fp64, as the oracle does
 * it (reading C16''): mu^k from line 10, C^k = (1/N) sum d_i d_i^T from the residuals (lines
 * 12-14), a Cholesky with the oracle's pivot criterion (NOT_SPD on failure), and z^k, q^k from
 * its triangular solves. SMF_COVCHECK_OFF keeps only the Woodbury path (NOT_SPD when its 3 x 3
 * capacitance is exactly singular) -- for measurement. Realistic columns never trigger the
 * literal path (smallest eigenvalue >= 0.03 on every config measured), so it costs nothing
 * there; a triggered column costs O(N bands^2) fp64 work in its update kernel. */
enum { SMF_COVCHECK_OFF = 0, SMF_COVCHECK_AUTO = 1, SMF_COVCHECK_ALWAYS = 2 };
smf_status smf_set_covariance_check(smf_ctx* ctx, int mode);

/* Per-iteration diagnostics (the exact-zero fraction of P:733-736).
 * When enabled (enable != 0; default off), smf_retrieve records after every sweep
 * k = 0..N_iter, per partition: the number of pixels with alpha_i^k > 0, q^k = t^T (C^k+rho
 * I)^-1 t, the partition status, and the cumulative number of iterations whose C^k was
 * recomputed literally (smf_set_covariance_check). One extra small kernel per sweep (it reads
 * the [cols][pixels] enhancement map once). smf_iteration_diagnostics copies the records of
 * the last smf_retrieve that used `workspace` to caller device buffers laid out
 * [N_iter + 1][partitions] (any pointer may be NULL), enqueued on `stream`;
 * SMF_ERR_NOT_CONFIGURED if diagnostics were not enabled. The workspace size depends on this
 * switch and N_iter (query smf_workspace_bytes after setting them). */
smf_status smf_set_diagnostics(smf_ctx* ctx, int enable);
smf_status smf_iteration_diagnostics(smf_ctx* ctx, const void* workspace, int cols, int pixels, int64_t* nnz_out,
                                     double* q_out, int32_t* status_out, int32_t* literal_out, void* stream);

/* NVTX ranges (enable != 0): every kernel enqueue of smf_retrieve is wrapped in an NVTX
 * range named after its step (smf:stats / smf:init / smf:update / smf:sweep, with the
 * algorithm lines it implements), for timeline tools. Default: off unless the environment
 * variable SMF_NVTX=1 is set when the first range would be pushed. No effect on results. */
smf_status smf_set_nvtx(smf_ctx* ctx, int enable);

/* Kernel launches enqueued by the last smf_retrieve call on this context. */
int smf_last_launch_count(const smf_ctx* ctx);

/* Per-kernel timing (measurement aid for bench.py): while enabled, every
 * kernel launch of smf_retrieve is bracketed by two CUDA events recorded on
 * the launching stream. smf_profile_enable(ctx, 1) also clears previous
 * records. smf_profile_read synchronises on the recorded events and returns,
 * for one kernel kind (SMF_KERNEL_*), the summed device duration in ms and
 * the number of launches recorded since the last enable. */
enum { SMF_KERNEL_STATS = 0, SMF_KERNEL_INIT = 1, SMF_KERNEL_UPDATE = 2, SMF_KERNEL_SWEEP = 3 };
smf_status smf_profile_enable(smf_ctx* ctx, int enable);
smf_status smf_profile_read(smf_ctx* ctx, int kernel_kind, double* total_ms, int* launches);

const char* smf_status_string(smf_status status);
const char* smf_last_error(const smf_ctx* ctx);
int smf_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SMF_H */
