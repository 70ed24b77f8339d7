/*
 * ssa.h -- C-ABI of libssa.so, the B200 (sm_100a) hot path of fast Basic SSA
 * (Korobeynikov, "Computation- and Space-Efficient Implementation of SSA",
 * arXiv:0911.4498).  Citations are PAPER.md line ranges with section / algorithm.
 *
 * Problem statement (sec 2): a real series F = (f_1..f_N), N > 2, window
 * 1 < L < N, K = N - L + 1, trajectory matrix X (L x K, x_ij = f_{i+j-1},
 * PAPER.md:84-94 sec 2.1).  The library computes the k leading singular triples
 * (sigma_i, u_i, v_i) of X (sec 2.2, X = U Sigma V^T -- see DESIGN.md
 * reading R3) without ever forming X, and the elementary reconstructed series
 * g_i = diagonal averaging of sigma_i u_i v_i^T (sec 2.4, 747-828 sec 5).
 *
 * Conventions shared by every entry point:
 *  - All numbers are IEEE binary64 (double).  Arrays are dense, C row-major, with
 *    the shapes written next to each argument; no padding in caller buffers.
 *  - Pointers named d_* are DEVICE pointers on the plan's device (e.g. torch CUDA
 *    tensors' data_ptr()), h_* are HOST pointers (pageable or pinned).  The caller
 *    owns every buffer passed in; inputs are read-only.  Device buffers must be
 *    8-byte aligned (16-byte for d_spec).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every
 *    device-pointer call is asynchronous with respect to the host: it only enqueues
 *    kernels on `stream` -- except ssa_run_host and the H-matrix calls, which
 *    synchronize `stream` (documented there).  Argument validation happens synchronously
 *    before anything is enqueued.
 *  - Errors are status codes; no exception crosses the ABI.  ssa_last_error() returns
 *    a thread-local human-readable detail for the last non-OK status.
 *  - A plan owns all its device workspace (spectra, Krylov bases, bidiagonal factors,
 *    scratch), allocated once in ssa_plan_create, so out-of-memory is reported there;
 *    the only exceptions are scratch buffers grown on first use by ssa_run_host,
 *    ssa_reconstruct_grouped (long path) and ssa_bootstrap, which then report
 *    OUT_OF_MEMORY themselves.  Plans are not thread-safe; use one plan per concurrent
 *    stream.
 */
#ifndef SSA_H_
#define SSA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ssa_plan_s* ssa_plan_t;

typedef enum {
  SSA_OK = 0,
  SSA_ERR_INVALID_ARGUMENT = 1, /* bad sizes / null pointers; non-finite series (d_info) */
  SSA_ERR_NOT_CONVERGED = 2,    /* some series did not meet tol within max_steps       */
  SSA_ERR_OUT_OF_MEMORY = 3,    /* workspace allocation failed in ssa_plan_create       */
  SSA_ERR_CUDA = 4,             /* a CUDA runtime call failed (detail in ssa_last_error)*/
  SSA_ERR_INTERNAL = 5,
  SSA_ERR_UNSUPPORTED = 6       /* valid request this build cannot run (e.g. FFT size) */
} ssa_status;

/* Options of the truncated SVD (sec 3.1-3.2).  Fill with ssa_options_default first. */
typedef struct {
  double tol;            /* stop when every one of the k leading Ritz triples has residual
                            alpha_{m+1} |P_{m+1,i}| <= tol * omega_1 (R7; the paper
                            gives no criterion).  Default 1e-12.        */
  int32_t max_steps;     /* m_max, Lanczos steps cap; default max(256, 8k) clipped to
                            min(L, K).  Fixes the Krylov basis workspace size.             */
  int32_t check_every;   /* run the convergence test every c steps once m >= k; default 4 */
  uint64_t seed;         /* start vector p_0 (Alg. 1 line 1): uniform(-1,1)
                            entries from a counter-based hash of (seed, series, i); dflt 42 */
  int32_t reorth;        /* 3 = partial reorthogonalization (PRO: Simon /
                            Larsen omega recurrences estimate the orthogonality level of
                            each new Lanczos vector; when it exceeds reorth_eta the vector,
                            and the next one of the same side, are orthogonalized against
                            the whole basis) -- the default, R22;
                            1 = full reorthogonalization (FRO, sec 3.2.2)
                            by classical Gram-Schmidt with a DGKS second pass when the norm
                            drops below 1/sqrt(2); 2 = FRO, always two passes.  The long-
                            series path (M > 16384) runs 3 as 1.                          */
  int32_t reserved;      /* flags: 1 = per-phase cycle counters (ssa_plan_profile); 2 = bidiagonal
                            SVD by implicit-shift QR instead of TGK inverse iteration; 4 = use
                            the long-series (multi-CTA FFT) path even when M <= 16384 (tests) */
  double reorth_eta;     /* PRO threshold on the estimated orthogonality level; default
                            eps^(3/4) = 1.82e-12 (tighter than Larsen's sqrt(eps) so the Ritz
                            vectors stay orthogonal to ~1e-12, R22); must lie in
                            (0, 1e-6] when reorth = 3, ignored otherwise.                 */
  int64_t series_base;   /* global index of the plan's series 0 in the start-vector hash
                            (seed, series, i): a shard [b0, b1) of a larger batch set to b0
                            gets bit-identical results to the unsharded run (SURVEY.md
                            8(e)).  Default 0.                                             */
  int32_t restart_dim;   /* thick-restarted Lanczos bidiagonalization (sec 3.3,
                            "restarting schemes"): the Krylov dimension d, i.e. at most d+1
                            basis vectors per side are stored (O(d(L+K)) memory); when the
                            basis is full the restart keeps restart_keep Ritz triples and the
                            residual direction (R23).  0 (default) = no restart.
                            Requires k + 2 <= d <= min(L, K) - 1 and the batched path
                            (M <= 16384); reorthogonalization inside a cycle is FRO (reorth
                            3 runs as 1).  max_steps then caps the TOTAL steps (default
                            max(512, 16 k)) and no longer sizes the bases.                  */
  int32_t restart_keep;  /* Ritz triples kept at a thick restart, k <= p <= min(d - 2, 64); 0 = d / 2
                            (at least k).                                                  */
} ssa_options;

/* Per-series outcome of ssa_decompose (device array, one entry per series). */
typedef struct {
  int32_t steps;          /* m: Lanczos steps in B_m                                       */
  int32_t converged;      /* 1 if all k residuals met tol                                  */
  int32_t breakdown_step; /* first step with alpha or beta < 1e-12 * running max, else 0   */
  int32_t reorth_extra;   /* number of DGKS second passes taken                            */
  int32_t status;         /* ssa_status for this series (INVALID_ARGUMENT if non-finite)   */
  int32_t restarts;       /* breakdown restarts (fresh seeded vectors, R11)      */
  double max_residual;    /* max_i alpha_{m+1}|P_{m+1,i}| / omega_1 over the k triples     */
  double sigma1;          /* omega_1                                                       */
  int32_t rows_u;         /* Krylov basis rows of U read by reorthogonalization (all passes) */
  int32_t rows_v;         /* the same for V  (bytes read = 8 (rows_u L + rows_v K))          */
  int32_t reorth_steps;   /* half-steps that reorthogonalized (all of them under FRO)      */
  int32_t reserved;       /* thick restarts taken (restart_dim > 0), else 0                  */
} ssa_series_info;

/* Fill *opt with the defaults above (max_steps = 0 means "derive from k, L, K"). */
ssa_status ssa_options_default(ssa_options* opt);

/* Create a plan for `batch` independent series of length N with window L and k triples.
 * Validation: N >= 3; 2 <= L <= N-1; 1 <= k <= min(L, K);
 * batch >= 1.  k = 0 is accepted for plans used only for ssa_spectrum / ssa_matvec /
 * ssa_hankelize.  The FFT size M is the smallest power of two >= N (R5).
 * `device` is the CUDA ordinal.  opt may be NULL (defaults).  On success *out owns
 * device workspace sized for ssa_decompose (about 8 B * batch_in_flight * (m_max+1) *
 * (L+K) for the Krylov bases plus spectra). */
ssa_status ssa_plan_create(int64_t N, int64_t L, int32_t k, int64_t batch,
                           const ssa_options* opt, int device, ssa_plan_t* out);
void ssa_plan_destroy(ssa_plan_t plan);

int64_t ssa_plan_fft_size(ssa_plan_t plan);     /* M, or -1 for a NULL plan */
int32_t ssa_plan_max_steps(ssa_plan_t plan);    /* resolved m_max            */

/* Spectrum of each series (Alg. 2 lines 1-2, computed once and reused,
 * PAPER.md:699-702): d_spec[b][q] = sum_{n<N} f_{n+1} exp(-2 pi i q n / M), q = 0..M/2,
 * stored as interleaved (re, im) pairs.  This is the paper's c-hat up to the phase
 * exp(-2 pi i q L / M) (R1/R5; the correlation form needs no rotation).
 *   d_series: [batch][N]     d_spec: [batch][M/2+1][2] */
ssa_status ssa_spectrum(ssa_plan_t plan, const double* d_series, double* d_spec, void* stream);

/* Hankel matrix-vector products through the stored spectra (Alg. 2 / Alg. 3,
 * PAPER.md:680-729 sec 4.3; Alg. 3 output slice read as p'_L..p'_N, R1):
 *   transpose = 0 : d_y[b] = X_b d_x[b]     d_x: [batch][K]   d_y: [batch][L]
 *   transpose = 1 : d_y[b] = X_b^T d_x[b]   d_x: [batch][L]   d_y: [batch][K]
 * computed as y = irfft(spec * conj(rfft(x, M)))[0 : len(y)]; X is never formed. */
ssa_status ssa_matvec(ssa_plan_t plan, const double* d_spec, const double* d_x, double* d_y,
                      int transpose, void* stream);

/* The same products for nvec vectors per series in one call, every vector of series b
 * against the one stored spectrum of b (the products of a series share its spectrum, read
 * from HBM once per call instead of once per product):
 *   transpose = 0 : d_y[b][i] = X_b d_x[b][i]    d_x: [batch][nvec][K]  d_y: [batch][nvec][L]
 *   transpose = 1 : d_y[b][i] = X_b^T d_x[b][i]  d_x: [batch][nvec][L]  d_y: [batch][nvec][K]
 * nvec >= 1 and batch * nvec < 2^31, else SSA_ERR_INVALID_ARGUMENT.  Enqueue only. */
ssa_status ssa_matvec_multi(ssa_plan_t plan, const double* d_spec, const double* d_x, double* d_y,
                            int32_t nvec, int transpose, void* stream);

/* Rank-1 Hankelization (diagonal averaging of sigma u v^T) of nterms terms per series via
 * linear convolution (sec 5, Eqs. hankelization1/conv, Alg. 4 with the
 * weights read as division by the antidiagonal counts c_t = min(t, L, K, N-t+1),
 * DESIGN.md R2):
 *   d_out[b][i][t-1] = sigma[b][i] * (u' * v')_t / c_t,  t = 1..N
 *   d_sigma: [batch][nterms]  d_U: [batch][nterms][L]  d_V: [batch][nterms][K]
 *   d_out: [batch][nterms][N] */
ssa_status ssa_hankelize(ssa_plan_t plan, const double* d_sigma, const double* d_U, const double* d_V,
                         int32_t nterms, double* d_out, void* stream);

/* Truncated SVD of each trajectory matrix by Golub-Kahan-Lanczos bidiagonalization
 * (Alg. 1, sec 3.1) with full reorthogonalization,
 * every product by the FFT correlation above, then the SVD of the (m+1) x m lower
 * bidiagonal B_m on device and Ritz assembly U_k = U_{m+1} P_k,
 * V_k = V_m Q_k (Eq. 1):
 *   d_series: [batch][N]   d_sigma: [batch][k] (descending)   d_U: [batch][k][L]
 *   d_V: [batch][k][K]     d_info: [batch] or NULL
 * Each u_i is sign-canonicalized (largest-|.| entry positive, lowest index on ties; v_i
 * flipped with it).  Per-series failures (non-finite input -> INVALID_ARGUMENT, not
 * converged -> NOT_CONVERGED with the best triples written) are reported in d_info after
 * the stream synchronizes; the return value covers validation and launch only.
 * Two execution paths, both enqueue-only: the batched path (one CTA per series, every
 * series of the batch in flight) when the series' kernel fits one CTA's shared memory
 * (M <= 16384, and for M = 16384 only while the per-series basis fits), otherwise the
 * long-series path, which decomposes the series of the batch ONE AFTER ANOTHER, each with
 * the whole GPU (four-step FFT products, grid-wide reorthogonalization; the Lanczos loop of
 * each series is one CUDA graph launch with device-side decisions). */
ssa_status ssa_decompose(ssa_plan_t plan, const double* d_series, double* d_sigma, double* d_U,
                         double* d_V, ssa_series_info* d_info, void* stream);

/* Elementary reconstructed series of the k triples (grouping with
 * I_j = {j} combined with averaging; equals ssa_hankelize with nterms = k).
 *   d_out: [batch][k][N] */
ssa_status ssa_reconstruct(ssa_plan_t plan, const double* d_sigma, const double* d_U, const double* d_V,
                           double* d_out, void* stream);

/* Grouped reconstruction (Basic SSA steps 3-4, PAPER.md:131-146 grouping and 148-167
 * diagonal averaging): for each group I_g = { i : groups[i] == g } the series
 *   g~_g = hankelization( sum_{i in I_g} sigma_i u_i v_i^T ) = sum_{i in I_g} g~_i
 * (averaging is linear), computed as one inverse FFT of the summed
 * product spectra per group (M <= 8192 and not the long path), else as elementary series
 * in plan scratch summed per group.
 *   groups: HOST [k], groups[i] in [0, ngroups) or -1 (triple left out); read during the
 *           call only.  ngroups in [1, k].  An empty group yields a zero series.
 *   d_sigma, d_U, d_V: as ssa_reconstruct.   d_out: [batch][ngroups][N]
 * Errors: INVALID_ARGUMENT for NULL pointers, k = 0 plans, ngroups or a group id out of
 * range; OUT_OF_MEMORY if the scratch of the long path cannot be allocated. */
ssa_status ssa_reconstruct_grouped(ssa_plan_t plan, const double* d_sigma, const double* d_U, const double* d_V,
                                   const int32_t* groups, int32_t ngroups, double* d_out, void* stream);

/* Heterogeneity matrix for structural-change detection (sec 6.2):
 *   G[i][j] = 1 - sum_{m=1}^{K2} sum_{r in I} (U_r^(i)T X_m^(j))^2 / sum_{m=1}^{K2} |X_m^(j)|^2
 * where U_r^(i) (r in I) are left singular vectors of the base window
 * (f_i .. f_{i+B-1}), i = 1..N-B+1, and X_m^(j), m = 1..K2 = T-L+1, the L-lagged vectors of
 * the test window (f_j .. f_{j+T-1}), j = 1..N-T+1 (R21: windows of length B
 * and T).  The base windows are decomposed by the batched ssa_decompose (its options and
 * tolerances), the projections of every test window come from one FFT Hankel product
 * X_F^T U_r^(i) of the whole series per (i, r).
 *   d_series: [N] device;  I: HOST [nI] distinct 1-based triple indices, each <= min(L, B-L+1)
 *   d_G: [N-B+1][N-T+1] device;  d_info: [N-B+1] per-window decompose info, or NULL
 * Needs N >= 3, 2 <= L < B <= N, L <= T <= N.  The one-shot call creates the plan below,
 * executes it and destroys it.  Returns NOT_CONVERGED (G still written) if a base window
 * did not converge. */
ssa_status ssa_hmatrix(const double* d_series, int64_t N, int64_t B, int64_t T, int64_t L, const int32_t* I,
                       int32_t nI, const ssa_options* opt, int device, double* d_G, ssa_series_info* d_info,
                       void* stream);

/* The same as a plan (sub-plans and workspace allocated once, OUT_OF_MEMORY reported at
 * creation) and an execution that can be repeated on new series of length N; exec
 * synchronizes `stream` to read the per-window info.  Not thread-safe per plan. */
typedef struct ssa_hplan_s* ssa_hplan_t;
ssa_status ssa_hmatrix_plan_create(int64_t N, int64_t B, int64_t T, int64_t L, const int32_t* I, int32_t nI,
                                   const ssa_options* opt, int device, ssa_hplan_t* out);
ssa_status ssa_hmatrix_exec(ssa_hplan_t hplan, const double* d_series, double* d_G, ssa_series_info* d_info,
                            void* stream);
void ssa_hmatrix_plan_destroy(ssa_hplan_t hplan);

/* Bootstrap study of the rank-d reconstruction (sec 6.3): for the plan's
 * batch = R replicates F'_r = F + noise_sigma * eps_r of the clean series F, the k = d
 * leading triples of each (ssa_decompose) are grouped into one component and averaged
 * (ssa_reconstruct_grouped) into G_r, then per point t:
 *   mean[t] = (1/R) sum_r G_r[t],  var[t] = 1/(R-1) sum_r (G_r[t] - mean[t])^2,
 *   mse[t]  = (1/R) sum_r (G_r[t] - F[t])^2      (bias = mean - F;  mse = bias^2 + (R-1)/R var)
 *   d_series: [N] the clean F;  d_eps: [R][N] the noise (caller-drawn, seeded: the library
 *   draws no random numbers for this);  d_mean, d_var, d_mse: [N] (var, mse nullable);
 *   d_G: [R][N] reconstructions or NULL (plan scratch);  d_info: [R] or NULL.
 * The plan's workspace grows by 2 R N doubles on first use. */
ssa_status ssa_bootstrap(ssa_plan_t plan, const double* d_series, const double* d_eps, double noise_sigma,
                         double* d_mean, double* d_var, double* d_mse, double* d_G, ssa_series_info* d_info,
                         void* stream);

/* End-to-end call on HOST buffers: copies h_series to the device, runs ssa_decompose and
 * ssa_reconstruct on plan-owned device buffers, copies sigma, U, V, the reconstructions
 * and info back, and synchronizes `stream`.  Any output pointer may be NULL to skip its
 * copy.  Returns NOT_CONVERGED / INVALID_ARGUMENT if any series reported it.
 *   h_series: [batch][N]  h_sigma: [batch][k]  h_U: [batch][k][L]  h_V: [batch][k][K]
 *   h_recon: [batch][k][N]  h_info: [batch] */
ssa_status ssa_run_host(ssa_plan_t plan, const double* h_series, double* h_sigma, double* h_U,
                        double* h_V, double* h_recon, ssa_series_info* h_info, void* stream);

const char* ssa_status_string(ssa_status s);
const char* ssa_last_error(void);

/* Number of kernels the library enqueued since the plan was created (for bench.py's
 * gpu_launches claim). */
int64_t ssa_plan_launch_count(ssa_plan_t plan);

/* Device time (ms, CUDA events recorded on the launching stream around each kernel) of
 * the most recent launch of each phase of this plan: out_ms[0] spectrum, [1] Lanczos
 * bidiagonalization, [2] bidiagonal SVD, [3] Ritz assembly, [4] hankelization.  Blocks
 * until those events completed; phases never launched are reported as -1.  (When a
 * decompose call is split into several chunks, the times are those of the last chunk.) */
ssa_status ssa_plan_phase_ms(ssa_plan_t plan, double out_ms[5]);

/* Diagnostic: if the plan was created with (options.reserved & 1), the decompose kernel
 * accumulates SM clock cycles per phase summed over all CTAs and launches:
 * out[0] FFT products, [1] reorthogonalization, [2] convergence tests, [3] final
 * bidiagonal QR, [4] forming P_k / Q_k, [5] Ritz assembly + signs, [6] number of
 * convergence tests, [7] other.  INVALID_ARGUMENT if profiling is off. */
ssa_status ssa_plan_profile(ssa_plan_t plan, int64_t out[8]);

/* Diagnostic / test hook: after ssa_decompose (synchronizes the device), copy the
 * Lanczos bidiagonal factors of the series of the LAST decompose chunk (all series when
 * the batch fits one chunk): h_alpha[b][j] = alpha_j, h_beta[b][j] = beta_j for
 * j = 0..m_max+2 (1-based as in Alg. 1; unused entries undefined) and
 * h_steps[b] = m.  Shapes: [nb][m_max+3], [nb][m_max+3], [nb]. */
ssa_status ssa_plan_bidiagonals(ssa_plan_t plan, double* h_alpha, double* h_beta, int32_t* h_steps);

#ifdef __cplusplus
}
#endif
#endif /* SSA_H_ */
