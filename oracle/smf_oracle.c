/*
 * smf_oracle.c -- fp64 CPU ORACLE for the albedo-corrected reweighted-l1
 * matched filter (Foote et al., arXiv 2003.02978, "AlbedoReWeightL1Filter",
 * PAPER.md Fig. alg).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2003_02978_b200/csrc); the product path never calls it.
 *
 * It is a literal, step-by-step transcription of the algorithm figure in
 * fp64, one partition = one detector column:
 *   line 2   mu0 = (1/N) sum L_i
 *   line 3   C0  = (1/N) sum (L_i - mu0)(L_i - mu0)^T      (outer product, reading C1)
 *   line 5   r_i = L_i.mu0 / mu0.mu0                         (frozen, reading C2)
 *   line 6   alpha0_i = (L_i-mu0)^T C0^-1 t0 / (r_i t0^T C0^-1 t0),  t0 = mu0 (.) s
 *   line 9   w_i = 1/(alpha_i^{k-1} + eps)                   (0 if sparsity off)
 *   line 10  mu^k = (1/N) sum (L_i - r_i alpha_i^{k-1} mu^{k-1} (.) s)
 *   line 12  d_i = L_i - r_i alpha_i^{k-1} mu^k (.) s - mu^k
 *   line 14  C^k = (1/N) sum d_i d_i^T                        (recomputed from residuals)
 *   line 16  alpha_i^k = max(((L_i-mu^k)^T C^k^-1 t^k - w_i) / (r_i t^k^T C^k^-1 t^k), 0)
 * Readings of silent / ambiguous points:
 *   C3  alpha0 is clamped at 0 before it feeds w^1, mu^1, C^1;
 *       the unclamped alpha0 is returned only when n_iter == 0.
 *   C7  eps is a parameter (default 1e-2 ppm m).
 *   C8  1/N normalisation.
 *   C9  a ridge rho = lambda_rel * tr(C0)/B, computed ONCE from C0, is added
 *       to every factored covariance (C0 and every C^k); lambda_rel = 0 is
 *       the paper-faithful default.
 *   C10 r~ = max(r, r_floor) wherever r enters the iteration; raw r reported.
 *   C14 max(x, 0) is (x > 0 ? x : +0.0).
 *   C15/C16 per-column status; a failed column is NaN-filled.
 * C^{-1} products use this file's own Cholesky (plain loops, no BLAS).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_OK = 0, OR_NONFINITE = 1, OR_DEGENERATE_MEAN = 2, OR_NOT_SPD = 3,
       OR_DEGENERATE_TARGET = 4, OR_BAD_ARG = 5, OR_NOMEM = 6 };

/* ---- step functions (each exported so tests can pin it alone) ---------- */

/* Fig. alg line 2 / Eq. 10 with alpha = 0: arithmetic mean of N rows. */
void oracle_mean(int N, int B, const double* L, double* mu) {
    for (int b = 0; b < B; ++b) mu[b] = 0.0;
    for (int i = 0; i < N; ++i)
        for (int b = 0; b < B; ++b) mu[b] += L[(size_t)i * B + b];
    for (int b = 0; b < B; ++b) mu[b] /= (double)N;
}

/* Fig. alg line 3 / line 14 / Eq. 11: (1/N) sum d_i d_i^T of the given rows
 * (rows are already the deviations d_i). Full symmetric output. */
void oracle_second_moment(int N, int B, const double* D, double* C) {
    for (int a = 0; a < B * B; ++a) C[a] = 0.0;
    for (int i = 0; i < N; ++i) {
        const double* d = D + (size_t)i * B;
        for (int a = 0; a < B; ++a) {
            double da = d[a];
            double* Ca = C + (size_t)a * B;
            for (int b = 0; b <= a; ++b) Ca[b] += da * d[b];
        }
    }
    for (int a = 0; a < B; ++a)
        for (int b = 0; b <= a; ++b) {
            C[(size_t)a * B + b] /= (double)N;
            C[(size_t)b * B + a] = C[(size_t)a * B + b];
        }
}

/* Lower Cholesky factor A = G G^T in place (lower triangle of A used).
 * Returns 0, or k+1 when pivot k is not numerically positive: not finite or
 * <= n * 2^-52 * max_i A_ii (reading C16: a numerically singular covariance
 * is reported as NOT_SPD instead of factored through a rounding-level pivot). */
int oracle_cholesky(int n, double* A) {
    double amax = 0.0;
    for (int j = 0; j < n; ++j) amax = fmax(amax, A[(size_t)j * n + j]);
    const double tol = (double)n * 2.220446049250313e-16 * amax;
    for (int j = 0; j < n; ++j) {
        double d = A[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
        if (!(d > tol) || !isfinite(d)) return j + 1;
        double g = sqrt(d);
        A[(size_t)j * n + j] = g;
        for (int i = j + 1; i < n; ++i) {
            double v = A[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) v -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
            A[(size_t)i * n + j] = v / g;
        }
        for (int i = 0; i < j; ++i) A[(size_t)i * n + j] = 0.0;
    }
    return 0;
}

/* Solve G G^T x = b with the lower factor G (forward then back substitution). */
void oracle_chol_solve(int n, const double* G, const double* b, double* x) {
    for (int i = 0; i < n; ++i) {
        double v = b[i];
        for (int k = 0; k < i; ++k) v -= G[(size_t)i * n + k] * x[k];
        x[i] = v / G[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double v = x[i];
        for (int k = i + 1; k < n; ++k) v -= G[(size_t)k * n + i] * x[k];
        x[i] = v / G[(size_t)i * n + i];
    }
}

/* x = (A + rho I)^-1 b for symmetric A; returns 0 or OR_NOT_SPD. */
int oracle_spd_solve(int n, const double* A, double rho, const double* b, double* x) {
    double* G = (double*)malloc(sizeof(double) * (size_t)n * n);
    if (!G) return OR_NOMEM;
    memcpy(G, A, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) G[(size_t)i * n + i] += rho;
    int rc = oracle_cholesky(n, G) ? OR_NOT_SPD : OR_OK;
    if (rc == OR_OK) oracle_chol_solve(n, G, b, x);
    free(G);
    return rc;
}

/* Eq. 7 / Fig. alg line 5: r = L.mu / mu.mu */
double oracle_albedo(int B, const double* L, const double* mu) {
    double num = 0.0, den = 0.0;
    for (int b = 0; b < B; ++b) { num += L[b] * mu[b]; den += mu[b] * mu[b]; }
    return num / den;
}

/* Eq. 5: w = 1/(alpha + eps) */
double oracle_reweight(double alpha_prev, double eps) { return 1.0 / (alpha_prev + eps); }

/* Eq. 6 / Fig. alg line 16 for one pixel given its numerator
 * num = (L-mu)^T C^-1 t and the denominator factor q = t^T C^-1 t. */
double oracle_ista_update(double num, double w, double r, double q) {
    double x = (num - w) / (r * q);
    return x > 0.0 ? x : 0.0;   /* reading C14: canonical +0 */
}

/* Eq. 3 for every row: alpha_i = (L_i-mu)^T C^-1 t / t^T C^-1 t; status. */
int oracle_mf_closed_form(int N, int B, const double* L, const double* mu, const double* C,
                          const double* t, double* alpha) {
    double* z = (double*)malloc(sizeof(double) * B);
    if (!z) return OR_NOMEM;
    int rc = oracle_spd_solve(B, C, 0.0, t, z);
    if (rc == OR_OK) {
        double q = 0.0;
        for (int b = 0; b < B; ++b) q += t[b] * z[b];
        if (!(q > 0.0) || !isfinite(q)) rc = OR_DEGENERATE_TARGET;
        for (int i = 0; i < N && rc == OR_OK; ++i) {
            double p = 0.0;
            for (int b = 0; b < B; ++b) p += (L[(size_t)i * B + b] - mu[b]) * z[b];
            alpha[i] = p / q;
        }
    }
    free(z);
    return rc;
}

/* ---- the procedure ------------------------------------------------------ */

typedef struct {
    /* every pointer optional (NULL = not recorded); k = 0..n_iter */
    double* mu;          /* [n_iter+1][B]  mu^k                                 */
    double* cov;         /* [n_iter+1][B][B] C^k (without ridge)                */
    double* q;           /* [n_iter+1]     t^k^T (C^k+rho I)^-1 t^k             */
    double* alpha_hist;  /* [n_iter+1][N]  alpha^k (k=0: unclamped alpha0)      */
    int64_t* nnz;        /* [n_iter+1]     # alpha^k > 0                        */
    double* rho;         /* [1]                                                  */
    double* energy;      /* [n_iter+1]     Eq. 8 at iteration k (see below)      */
} oracle_diag;

static void nan_fill(int N, double* alpha, double* r) {
    for (int i = 0; i < N; ++i) { alpha[i] = NAN; r[i] = NAN; }
}

/* Eq. 8, the objective tracked in Fig. 4, as printed (no 1/2,
 * cf. reading C4): E = sum_i d_i^T (C + rho I)^-1 d_i + sum_i r~_i w_i alpha_i with
 * d_i = L_i - r~_i alpha_i t - mu. Per pixel: forward substitution with this file's
 * Cholesky factor G of C + rho I, so d^T (C+rho I)^-1 d = |G^-1 d|^2. w may be NULL
 * (w = 0). Returns NaN if C + rho I is not SPD. */
double oracle_energy(int N, int B, const double* L, const double* mu, const double* C, double rho,
                     const double* t, const double* alpha, const double* rt, const double* w) {
    double* G = (double*)malloc(sizeof(double) * (size_t)B * B);
    double* d = (double*)malloc(sizeof(double) * B);
    double* y = (double*)malloc(sizeof(double) * B);
    double E = NAN;
    if (!G || !d || !y) goto out;
    for (int a = 0; a < B * B; ++a) G[a] = C[a];
    for (int b = 0; b < B; ++b) G[(size_t)b * B + b] += rho;
    if (oracle_cholesky(B, G) != OR_OK) goto out;
    E = 0.0;
    for (int i = 0; i < N; ++i) {
        for (int b = 0; b < B; ++b) d[b] = L[(size_t)i * B + b] - rt[i] * alpha[i] * t[b] - mu[b];
        double q = 0.0;
        for (int r = 0; r < B; ++r) {           /* y = G^-1 d (lower triangular) */
            double v = d[r];
            for (int c = 0; c < r; ++c) v -= G[(size_t)r * B + c] * y[c];
            y[r] = v / G[(size_t)r * B + r];
            q += y[r] * y[r];
        }
        E += q + (w ? rt[i] * w[i] * fabs(alpha[i]) : 0.0);
    }
out:
    free(G); free(d); free(y);
    return E;
}

/* One partition (column). L: fp32 [N][B] row-major (promoted to fp64).
 * Returns an OR_* status; on failure alpha and r are NaN. */
int oracle_retrieve_column(const float* Lf, int N, int B, const float* sf, int n_iter,
                           int use_sparsity, int use_albedo, double eps, double lambda_rel,
                           double r_floor, double* alpha, double* r, const oracle_diag* dg) {
    if (N < 2 || B < 1 || n_iter < 0 || !(eps > 0.0) || lambda_rel < 0.0 || !(r_floor > 0.0))
        return OR_BAD_ARG;
    size_t NB = (size_t)N * B;
    double* L = (double*)malloc(sizeof(double) * NB);
    double* D = (double*)malloc(sizeof(double) * NB);
    double* C = (double*)malloc(sizeof(double) * (size_t)B * B);
    double* mu = (double*)malloc(sizeof(double) * B);
    double* mu_prev = (double*)malloc(sizeof(double) * B);
    double* t = (double*)malloc(sizeof(double) * B);
    double* ts = (double*)malloc(sizeof(double) * B);
    double* z = (double*)malloc(sizeof(double) * B);
    double* s = (double*)malloc(sizeof(double) * B);
    double* rt = (double*)malloc(sizeof(double) * N);   /* r~ */
    double* w = (double*)malloc(sizeof(double) * N);
    int rc = OR_OK;
    if (!L || !D || !C || !mu || !mu_prev || !t || !ts || !z || !s || !rt || !w) { rc = OR_NOMEM; goto done; }

    for (size_t e = 0; e < NB; ++e) {
        L[e] = (double)Lf[e];
        if (!isfinite(L[e])) { rc = OR_NONFINITE; goto done; }   /* reading C15 */
    }
    for (int b = 0; b < B; ++b) s[b] = (double)sf[b];

    /* line 2 */
    oracle_mean(N, B, L, mu);
    /* line 3 (reading C1: outer product) */
    for (int i = 0; i < N; ++i)
        for (int b = 0; b < B; ++b) D[(size_t)i * B + b] = L[(size_t)i * B + b] - mu[b];
    oracle_second_moment(N, B, D, C);
    double tr = 0.0;
    for (int b = 0; b < B; ++b) tr += C[(size_t)b * B + b];
    double rho = lambda_rel * tr / (double)B;               /* reading C9 */
    if (dg && dg->rho) dg->rho[0] = rho;

    /* lines 4-5 */
    double mm = 0.0;
    for (int b = 0; b < B; ++b) mm += mu[b] * mu[b];
    if (use_albedo && !(mm > 0.0)) { rc = OR_DEGENERATE_MEAN; goto done; }
    for (int i = 0; i < N; ++i) {
        r[i] = use_albedo ? oracle_albedo(B, L + (size_t)i * B, mu) : 1.0;
        rt[i] = use_albedo ? (r[i] > r_floor ? r[i] : r_floor) : 1.0;   /* reading C10 */
    }

    /* line 6 */
    for (int b = 0; b < B; ++b) t[b] = mu[b] * s[b];
    if (oracle_spd_solve(B, C, rho, t, z) != OR_OK) { rc = OR_NOT_SPD; goto done; }
    double q = 0.0;
    for (int b = 0; b < B; ++b) q += t[b] * z[b];
    if (!(q > 0.0) || !isfinite(q)) { rc = OR_DEGENERATE_TARGET; goto done; }
    int64_t nz = 0;
    for (int i = 0; i < N; ++i) {
        double p = 0.0;
        for (int b = 0; b < B; ++b) p += (L[(size_t)i * B + b] - mu[b]) * z[b];
        alpha[i] = p / (rt[i] * q);
        nz += alpha[i] > 0.0;
    }
    if (dg) {
        if (dg->mu) memcpy(dg->mu, mu, sizeof(double) * B);
        if (dg->cov) memcpy(dg->cov, C, sizeof(double) * (size_t)B * B);
        if (dg->q) dg->q[0] = q;
        if (dg->alpha_hist) memcpy(dg->alpha_hist, alpha, sizeof(double) * N);
        if (dg->nnz) dg->nnz[0] = nz;
    }
    if (n_iter > 0)
        for (int i = 0; i < N; ++i) alpha[i] = alpha[i] > 0.0 ? alpha[i] : 0.0;   /* reading C3 */
    /* energy trace (reading C19): E_k = Eq. 8 with the statistics mu^k, C^k, t^k and the
     * weights w^k of iteration k, at the updated alpha^k (alpha0 as stored; w^0 = 0) */
    if (dg && dg->energy) dg->energy[0] = oracle_energy(N, B, L, mu, C, rho, t, alpha, rt, NULL);
    if (n_iter == 0) goto done;                               /* unclamped alpha0 */

    memcpy(mu_prev, mu, sizeof(double) * B);

    for (int k = 1; k <= n_iter; ++k) {
        /* line 9 */
        for (int i = 0; i < N; ++i) w[i] = use_sparsity ? oracle_reweight(alpha[i], eps) : 0.0;
        /* line 10: mu^k = (1/N) sum (L_i - r_i alpha_i mu^{k-1} (.) s) */
        for (int b = 0; b < B; ++b) ts[b] = mu_prev[b] * s[b];
        for (int i = 0; i < N; ++i)
            for (int b = 0; b < B; ++b)
                D[(size_t)i * B + b] = L[(size_t)i * B + b] - rt[i] * alpha[i] * ts[b];
        oracle_mean(N, B, D, mu);
        /* lines 11-13: d_i = L_i - r_i alpha_i mu^k (.) s - mu^k */
        for (int b = 0; b < B; ++b) t[b] = mu[b] * s[b];
        for (int i = 0; i < N; ++i)
            for (int b = 0; b < B; ++b)
                D[(size_t)i * B + b] = L[(size_t)i * B + b] - rt[i] * alpha[i] * t[b] - mu[b];
        /* line 14 */
        oracle_second_moment(N, B, D, C);
        /* line 16 */
        if (oracle_spd_solve(B, C, rho, t, z) != OR_OK) { rc = OR_NOT_SPD; goto done; }
        q = 0.0;
        for (int b = 0; b < B; ++b) q += t[b] * z[b];
        if (!(q > 0.0) || !isfinite(q)) { rc = OR_DEGENERATE_TARGET; goto done; }
        nz = 0;
        for (int i = 0; i < N; ++i) {
            double p = 0.0;
            for (int b = 0; b < B; ++b) p += (L[(size_t)i * B + b] - mu[b]) * z[b];
            alpha[i] = oracle_ista_update(p, w[i], rt[i], q);
            nz += alpha[i] > 0.0;
        }
        if (dg) {
            if (dg->mu) memcpy(dg->mu + (size_t)k * B, mu, sizeof(double) * B);
            if (dg->cov) memcpy(dg->cov + (size_t)k * B * B, C, sizeof(double) * (size_t)B * B);
            if (dg->q) dg->q[k] = q;
            if (dg->alpha_hist) memcpy(dg->alpha_hist + (size_t)k * N, alpha, sizeof(double) * N);
            if (dg->nnz) dg->nnz[k] = nz;
            if (dg->energy) dg->energy[k] = oracle_energy(N, B, L, mu, C, rho, t, alpha, rt, w);
        }
        memcpy(mu_prev, mu, sizeof(double) * B);
    }

done:
    if (rc != OR_OK && rc != OR_BAD_ARG && rc != OR_NOMEM) nan_fill(N, alpha, r);
    free(L); free(D); free(C); free(mu); free(mu_prev); free(t); free(ts); free(z); free(s);
    free(rt); free(w);
    return rc;
}

/* Whole cube [cols][N][B]: columns are independent partitions,
 * run in parallel over `threads` OpenMP threads (0 = library default).
 * alpha, r: fp64 [cols][N]; status: int32 [cols]. Returns # failed columns. */
int oracle_retrieve(const float* cube, int cols, int N, int B, const float* s, int n_iter,
                    int use_sparsity, int use_albedo, double eps, double lambda_rel,
                    double r_floor, double* alpha, double* r, int32_t* status, int threads) {
    int failed = 0;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : failed)
#endif
    for (int c = 0; c < cols; ++c) {
        int rc = oracle_retrieve_column(cube + (size_t)c * N * B, N, B, s, n_iter, use_sparsity,
                                        use_albedo, eps, lambda_rel, r_floor,
                                        alpha + (size_t)c * N, r + (size_t)c * N, NULL);
        status[c] = rc;
        failed += rc != OR_OK;
    }
    return failed;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
