/*
 * sl7.h -- C ABI of the B200-native Seven-League (7L) online path generator.
 *
 * The method (arXiv 2302.05170, "GPU acceleration of the Seven-League scheme", PAPER.md):
 * for each of N_P Monte Carlo paths and each large step t_i -> t_{i+1} = t_i + dt
 * (Algorithm I):
 *   step 3 (Eq. 6.4): predict the m conditional collocation points
 *           y_j = H_hat_j(Y_i, dt, theta) with a trained MLP (or, in the "exact-collocation"
 *           modes, with the closed form H_j of Eq. 6.3 for GBM / OU (Eq. 6.6));
 *   step 6: draw X_hat ~ N(0,1)  (Philox4x32-10 + Box-Muller keyed by
 *           (seed, path, step), see sl7_philox_u32 below);
 *   steps 5-6: Y_{i+1} = g_m(X_hat), g_m the (barycentric)
 *           Lagrange interpolant through (x_j, y_j) on the m Gauss-Hermite nodes x_j;
 *   steps 7-8: collect all paths at t_{i+1}, loop until T.
 *
 * Everything between sl7_simulate's entry and its return runs in the library's own CUDA
 * kernels for sm_100a.  There is no CPU fallback: on a machine without a usable device every
 * compute entry point returns SL7_ECUDA.
 *
 * Conventions
 *   - "d_" pointers are DEVICE pointers on the context's device, "h_" pointers are HOST
 *     pointers.  The caller owns every buffer it passes; the library never frees them.
 *   - All compute calls are asynchronous on the caller's CUDA stream (opts->stream, a
 *     cudaStream_t; NULL = legacy default stream) unless stated otherwise.  Argument errors are
 *     detected synchronously, before any launch, and leave the outputs untouched.
 *   - Every call returns an sl7_status; sl7_last_error(ctx) gives a one-line message naming the
 *     offending field (e.g. "layer_dims", "version").
 *   - A context is bound to one device and is NOT thread-safe; use one context per thread.
 */
#ifndef SL7_H
#define SL7_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SL7_ABI_VERSION 2
#define SL7_MAX_M 16          /* nodes per collocation grid */
#define SL7_MAX_WIDTH 64      /* hidden width of the MLP */
#define SL7_MAX_HIDDEN 6      /* hidden layers of the MLP */
#define SL7_MAX_THETA 8       /* model parameters appended to the network input */
#define SL7_STATS_HEAD 8      /* doubles before the histogram in the stats vector */

typedef struct sl7_ctx_s* sl7_ctx;

typedef enum {
  SL7_OK = 0,
  SL7_EINVAL = 1,        /* an argument is out of range (message names it) */
  SL7_ESTATE = 2,        /* call out of order, e.g. ANN mode before sl7_load_weights */
  SL7_EFORMAT = 3,       /* malformed weights blob (message names the field) */
  SL7_ENOMEM = 4,        /* host or device allocation failed */
  SL7_ECUDA = 5,         /* no device / launch or copy failure (message holds cudaGetErrorString) */
  SL7_ENONFINITE = 6,    /* sl7_stats: at least one non-finite terminal value was counted */
  SL7_EUNSUPPORTED = 7   /* valid request this build does not implement (e.g. a precision mode) */
} sl7_status;

/* Hidden-layer activation (PAPER.md:85 uses Softplus; BASELINE configs 0,1,3 use tanh). */
typedef enum { SL7_ACT_TANH = 0, SL7_ACT_SOFTPLUS = 1 } sl7_act;

/* What sl7_simulate writes.
 *  FULL:     d_out[i * n_paths + p] = Y_hat_i of path p, i = 0..n_steps (row 0 = Y0), fp32,
 *            step-major (SPEC's N_P x (N+1) PathSet, transposed for coalescing).
 *  TERMINAL: d_out[p] = Y_hat_{n_steps} of path p.
 *  STATS:    no path output; only the fused statistics (d_stats required).
 * In FULL and TERMINAL modes statistics are also accumulated when d_stats != NULL. */
typedef enum { SL7_OUT_FULL = 0, SL7_OUT_TERMINAL = 1, SL7_OUT_STATS = 2 } sl7_out;

/* Arithmetic of the ANN contractions (hidden layers 2..L and the output layer).
 *  FP32:  CUDA-core fp32 FFMA, accurate activations ("exact mode").
 *  BF16:  tcgen05 tensor cores, operands rounded to bf16 (RNE), fp32 accumulate, fp32 bias and
 *         activations (tanh on MUFU.TANH, <= 1e-5 relative); reproduces the quantisation-aware oracle O6
 *         (DESIGN.md).  BF16 and TF32 draw X_hat with the fast Box-Muller of SL7_FLAG_FAST_NORMALS.
 *  TF32:  tcgen05 kind::tf32 (K = 8 per instruction), operands rounded with cvt.rna (ties away, 11
 *         significant bits), fp32 accumulate; reproduces O6 with TF32 rounding.
 *  SPLIT: tcgen05 with every operand split into three bf16 parts (a = a0 + a1 + a2, same for W) and
 *         the six partial products of size >= 2^-16 accumulated in fp32: fp32-class results (checked
 *         against the plain float64 oracle at the fp32 tolerance) at tensor-core speed.
 * Layer 1 (rank-1 in Y once dt and theta are folded into its bias) is always fp32. */
typedef enum { SL7_PREC_FP32 = 0, SL7_PREC_TF32 = 1, SL7_PREC_BF16 = 2, SL7_PREC_SPLIT = 3 } sl7_prec;

/* Source of the collocation points y_j (step 3 of Algorithm I).
 *  ANN:        the loaded MLP, input (Y, dt, theta...) (Eq. 6.4).
 *  EXACT_GBM:  y_j = Y exp((mu - sigma^2/2) dt + sigma sqrt(dt) x_j), theta = (mu, sigma).
 *  EXACT_OU:   y_j = Y e^{-lam dt} + Ybar (1 - e^{-lam dt}) + sigma sqrt((1-e^{-2 lam dt})/(2 lam)) x_j
 *              (Eq. 6.6), theta = (Ybar, lam, sigma); series form when lam*dt < 1e-6.
 *  EXACT_CIR:  y_j = c F^{-1}(Phi(x_j)), F the noncentral chi-square CDF with d = 4 kappa Ybar / sigma^2
 *              degrees of freedom and noncentrality Y+ e^{-kappa dt} / c, c = sigma^2 (1 - e^{-kappa dt})
 *              / (4 kappa), Y+ = max(Y, 0) (the CIR transition law, Eq. 6.3); theta = (kappa, Ybar,
 *              sigma), all > 0.  Evaluated per path and step in float64 (Poisson mixture of incomplete
 *              gammas, bracketed Newton): a reference generator, ~100x slower than the other modes.
 *              Scheme 7L only; SL7_FLAG_SPECIALIZED is not available. */
typedef enum { SL7_COLLOC_ANN = 0, SL7_COLLOC_EXACT_GBM = 1, SL7_COLLOC_EXACT_OU = 2,
               SL7_COLLOC_EXACT_CIR = 3 } sl7_colloc;

/* Path-wise reference evaluated on the SAME normals, for the strong error E|Y_T - Y(T)|
 * (PAPER.md:81, :16, :110).  GBM: Y(T) = Y0 exp((mu - s^2/2) T + s sqrt(dt) sum_i X_i),
 * ref_theta = (mu, s).  OU: the exact Eq. 6.6 transition per step, ref_theta = (Ybar, lam, s). */
typedef enum { SL7_REF_NONE = 0, SL7_REF_GBM = 1, SL7_REF_OU = 2 } sl7_ref;

/* Scheme.  7L: Algorithm I, the predictor runs for every path.
 * CDC: the 7L-CDC variant: per step the predictor runs only at the m marginal
 * collocation points z_k = empirical quantiles of the current states of ALL paths of the call at the
 * levels Phi(x_k) (plotting position (k - 0.5)/M, linear interpolation; exact order statistics by radix
 * select on the device), and each path's conditional points are the Lagrange interpolant of the table
 * rows on the z_k at its own state; repeated z_k (step 0) use the nearest row.  The marginal points
 * couple the paths, so one sl7_simulate CDC call holds the whole path set (opts->ref must be NONE); runs
 * sharded over ranks use the sl7_cdc_* calls below.
 * CDC_PRED: the 7L-CDC variant with the marginal collocation points taken from the predictor itself,
 * z_k(t_i) = H(Y0, t_i = i dt, theta)_k ("only requires the ANNs to compute a small number of marginal
 * collocation points"; reading R-26 of DESIGN.md); t_0 has every path at Y0 (nearest row).
 * The table is then the same for every path set, so there are no selection passes and no exchange:
 * shard it like SL7_SCHEME_7L with path_offset.  The network must be fitted for horizons up to T: with a
 * blob that carries its fitted domain (flags bit 2), a call whose horizons dt..(n_steps-1) dt or whose Y0
 * leave that box fails with SL7_EINVAL instead of extrapolating.  The hull clamp truncates the tails; a
 * CDC_PRED run with a stats vector reports how often it acted: E1 (slot 6, unused otherwise since the CDC
 * schemes take no strong-error reference) = the number of path-steps whose state was outside
 * [z_0, z_{m-1}] and clamped, E2 = 0 (sl7_stats then reports E1 / n as strong_err: clamped steps per path). */
typedef enum { SL7_SCHEME_7L = 0, SL7_SCHEME_CDC = 1, SL7_SCHEME_CDC_PRED = 2 } sl7_scheme;

typedef struct {
  sl7_prec prec;            /* ANN arithmetic (ignored by the exact modes) */
  sl7_colloc colloc;        /* source of y_j */
  uint64_t path_offset;     /* global index of this call's first path (Philox counter, sharding) */
  void* stream;             /* cudaStream_t of the caller (e.g. torch.cuda.current_stream()) */
  double hist_lo, hist_hi;  /* histogram range; n_bins equal bins [lo + k w, lo + (k+1) w) */
  double shift;             /* shift for the power sums S_k = sum (Y_T - shift)^k */
  int32_t n_bins;           /* 0 = no histogram; else 1..16384 (shared-memory histogram) */
  int32_t accumulate;       /* 0: zero d_stats first; 1: add into it (chunked / resumed runs) */
  sl7_ref ref;              /* strong-error reference (SL7_REF_NONE: E1 = E2 = 0) */
  double ref_theta[3];
  uint32_t flags;           /* SL7_FLAG_* below; 0 = defaults */
  sl7_scheme scheme;        /* SL7_SCHEME_7L (Algorithm I), SL7_SCHEME_CDC or SL7_SCHEME_CDC_PRED */
} sl7_run_opts;

/* opts->flags (exact-collocation modes and 7L-CDC (FAST_NORMALS only); ignored by the 7L ANN kernels):
 *  SL7_FLAG_FAST_NORMALS : Box-Muller with MUFU lg2 (exact series for u -> 1) and MUFU sin/cos on the
 *                          angle reduced exactly to (-pi, pi): ~4x fewer instructions,
 *                          |X_hat - X| <= 2e-6 (1 + |X|) (measured 1.1e-6).
 *  SL7_FLAG_SPECIALIZED  : evaluate g_m in closed form for the linear structure of the exact points:
 *                          GBM y_j = Y c_j  =>  g_m(Z) = Y Q(Z), Q the degree-(m-1) interpolant of c_j
 *                          in monomial form (Horner; m <= 8); OU y_j = mean + std x_j  =>  g_m(Z) =
 *                          mean + std Z (linear reproduction).  Same interpolant, fewer operations. */
#define SL7_FLAG_FAST_NORMALS 1u
#define SL7_FLAG_SPECIALIZED 2u

/* Summary computed on the host from a (possibly all-reduced) stats vector. */
typedef struct {
  uint64_t n, n_nonfinite;
  double mean, var;         /* population variance (divisor n) */
  double skew, exkurt;
  double strong_err;        /* E1 / n = mean |Y_T - Y(T)| (0 without a reference) */
  double rms_err;           /* sqrt(E2 / n) */
  const double* q_levels;   /* in: n_q probability levels in (0,1) */
  double* q_values;         /* out: n_q quantiles from the histogram CDF; NaN if the level falls
                               in the under/overflow bin or no histogram was kept */
  int32_t n_q;
} sl7_summary;

/* Create a context on `device`.
 * m           : collocation nodes, 1..SL7_MAX_M (m=5 in PAPER.md:83).
 * layer_dims  : [d_in, h_1..h_L, m] of the MLP (4 hidden x 50), or NULL with
 *               n_dims = 0 for a context that only runs the exact-collocation modes.
 *               d_in = 2 + n_theta (input order (Y, dt, theta...)), 1 <= L <= SL7_MAX_HIDDEN,
 *               h_l <= SL7_MAX_WIDTH, last entry == m.
 * act         : hidden activation.
 * Host setup done here (once): Gauss-Hermite nodes (Sturm-sequence bisection on the He_k recurrence +
 * Newton, in double), barycentric
 * weights, fp32 hi/lo node split.  Errors: SL7_EINVAL (m, layer_dims), SL7_ECUDA (device). */
sl7_status sl7_create(int32_t m, const int32_t* layer_dims, int32_t n_dims, sl7_act act,
                      int32_t device, sl7_ctx* out);

/* Load the trained network (Algorithm I step 1 output) from a blob; copied, so the
 * caller may free it on return.  Little-endian "SL7W" container:
 *   char magic[4] = "SL7W"; u32 version = 1; u32 n_dims; u32 dims[n_dims]; u32 act; u32 flags
 *   (bit0 has_norm, bit1 residual, bit2 has_domain; other bits rejected); then per layer l:
 *   f32 W[out][in] (row-major), f32 b[out]; if has_norm: f32 in_shift[d_in], in_scale[d_in],
 *   out_shift[m], out_scale[m]; if has_domain: f32 dom_lo[d_in], dom_hi[d_in], the box of raw features
 *   (Y, dt, theta...) the network was fitted on
 *   (network sees (f - in_shift)/in_scale; prediction is out * out_scale + out_shift, or out without
 *   has_norm).  residual (reading R-11 in DESIGN.md): y_j = Y + sqrt(dt) * prediction_j, so the
 *   network carries only the step's spread and bf16 / tf32 rounding no longer scales with |Y|.
 * The size must match exactly.  dims/act must equal the context's.  Errors: SL7_EFORMAT. */
sl7_status sl7_load_weights(sl7_ctx ctx, const void* blob, size_t nbytes);

/* Run Algorithm I steps 2-8 for paths [opts->path_offset, opts->path_offset + n_paths).
 * Y0        : initial value (rounded to fp32; FULL row 0).
 * dt        : large step, > 0; t_i = i dt, T = n_steps dt.
 * n_steps   : >= 1.   theta/n_theta : model parameters (see sl7_colloc; ANN: n_theta = d_in-2).
 * n_paths   : >= 1; path_offset + n_paths must not overflow 2^64.
 * seed      : Philox key.  Step i of path p uses normal Z_{4b + (i & 3)}, b = i >> 2, of
 *             Philox4x32-10(key = (seed_lo, seed_hi), counter = (b, 0, p_lo, p_hi)).
 * d_out     : device fp32 buffer of sl7_out_elems(n_steps, n_paths, out_mode) elements, or NULL
 *             in STATS mode.
 * d_stats   : device fp64 buffer of sl7_stats_elems(opts->n_bins) elements, or NULL (FULL /
 *             TERMINAL without statistics).  Layout: [n, n_nonfinite, S1, S2, S3, S4, E1, E2,
 *             hist_under, hist[0..n_bins-1], hist_over]; sums over finite Y_T only.
 * Asynchronous on opts->stream.  Errors: SL7_EINVAL, SL7_ESTATE, SL7_EUNSUPPORTED, SL7_ECUDA. */
sl7_status sl7_simulate(sl7_ctx ctx, double Y0, double dt, int32_t n_steps, const double* theta,
                        int32_t n_theta, uint64_t n_paths, uint64_t seed, sl7_out out_mode,
                        const sl7_run_opts* opts, float* d_out, double* d_stats);

/* Same as sl7_simulate but with HOST buffers (end-to-end use): the library stages through
 * context-owned device scratch, copies results back on opts->stream and synchronises it before
 * returning.  h_out/h_stats as d_out/d_stats (h_stats is always overwritten unless
 * opts->accumulate, in which case it is added into).  *h2d_bytes / *d2h_bytes (may be NULL)
 * receive the bytes moved across PCIe by this call. */
sl7_status sl7_simulate_host(sl7_ctx ctx, double Y0, double dt, int32_t n_steps, const double* theta,
                             int32_t n_theta, uint64_t n_paths, uint64_t seed, sl7_out out_mode,
                             const sl7_run_opts* opts, float* h_out, double* h_stats,
                             uint64_t* h2d_bytes, uint64_t* d2h_bytes);

/* Pipelined form of sl7_simulate_host: enqueues the kernels on opts->stream and the result copies into
 * h_out / h_stats on a context-owned copy stream, and returns without waiting, so the next call's kernels
 * overlap this call's device->host copies.  The host buffers should be page-locked (cudaHostAlloc /
 * torch pin_memory) -- pageable buffers work but serialise -- and must not be read (or, with
 * opts->accumulate, h_stats modified) before sl7_sync(ctx) returns.  The context alternates between two
 * device staging slots; a call waits on the device for the copies of the call two before it.  Byte
 * counts as sl7_simulate_host.  Errors: as sl7_simulate_host (launch errors surface at the latest in
 * sl7_sync). */
sl7_status sl7_simulate_host_async(sl7_ctx ctx, double Y0, double dt, int32_t n_steps, const double* theta,
                                   int32_t n_theta, uint64_t n_paths, uint64_t seed, sl7_out out_mode,
                                   const sl7_run_opts* opts, float* h_out, double* h_stats,
                                   uint64_t* h2d_bytes, uint64_t* d2h_bytes);
/* Wait until every sl7_simulate_host_async result of this context is in host memory. */
sl7_status sl7_sync(sl7_ctx ctx);

/* Moments, strong error and quantiles from a HOST copy of a stats vector (which the caller may
 * have all-reduced across ranks first).  Algorithm I step 7 collects the paths at each t_i into "a complete
 * set"; the distribution of that set at T and its path-wise error against the exact solution
 * on the same normals (Eq. 6.6, "used to compute the reference value to the path-wise error and the strong
 * convergence") are what this summarises: population mean / variance / skew / excess
 * kurtosis from the shifted power sums, strong error E1 / n and RMS sqrt(E2 / n), and quantiles by linear
 * interpolation of the histogram CDF.  opts supplies shift, hist_lo, hist_hi, n_bins (and scheme: see
 * SL7_SCHEME_CDC_PRED for the E1 slot of that scheme).
 * Returns SL7_ENONFINITE (after filling *out) if n_nonfinite > 0; SL7_EINVAL if n == 0. */
sl7_status sl7_stats(const double* h_stats, const sl7_run_opts* opts, sl7_summary* out);

/* Raw Philox4x32-10 outputs of the path generator's RNG (step a1), for verification:
 * d_out[k * n_paths + q] = r_k of path (path_offset + q) at block `block`, k = 0..3. */
sl7_status sl7_philox_u32(uint64_t seed, uint64_t path_offset, uint64_t n_paths, uint32_t block,
                          uint32_t* d_out, void* stream);

/* The normals the path generator consumes: d_out[i * n_paths + q] = X_hat of path
 * (path_offset + q) at step i, i = 0..n_steps-1, computed by the same device code as the step
 * kernels.  flags: 0 = libm Box-Muller (ANN kernels and default exact kernels), SL7_FLAG_FAST_NORMALS
 * = the fast variant the exact kernels use under that flag. */
sl7_status sl7_normals(uint64_t seed, uint64_t path_offset, uint64_t n_paths, int32_t n_steps,
                       uint32_t flags, float* d_out, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Sharded 7L-CDC (PAPER.md:48, :106-108 on several GPUs).  The marginal collocation points z_k are
 * quantiles of ALL paths, so a run whose paths are split over ranks exchanges, per large step, the four
 * radix-select digit histograms.  The caller drives the step loop and owns the reduction:
 *
 *   sl7_cdc_init(ctx, ..., n_local, ..., opts{path_offset = first global path of this rank}, d_state)
 *   for step i in 0..n_steps-1:
 *     for pass in 0..3:
 *       sl7_cdc_hist(ctx, d_state, pass, d_hist)      local digit counts of this pass
 *       all-reduce(SUM) d_hist over the ranks           (e.g. torch.distributed / NCCL, same stream)
 *       sl7_cdc_select(ctx, pass, d_hist)               every rank fixes the same digits
 *     sl7_cdc_step(ctx, i, d_state, d_state, last ? d_stats : NULL)
 *   all-reduce(SUM) d_stats
 *
 * With one rank this is exactly sl7_simulate(scheme = CDC) (bit for bit); with several, every path's
 * states equal those of the single-rank run over the union of the paths.
 * d_hist: device u64[sl7_cdc_hist_elems()] ([2 SL7_MAX_M slots][256 digits]); d_state: device fp32
 * [n_local], updated in place (d_in == d_out allowed).  opts as for sl7_simulate with scheme CDC (the
 * histogram/shift fields describe the statistics sl7_cdc_step adds into d_stats; d_stats is NOT zeroed).
 * All calls are asynchronous on opts->stream of sl7_cdc_init.  Errors: as sl7_simulate; SL7_ESTATE if
 * sl7_cdc_init has not succeeded; SL7_EINVAL for pass outside 0..3 or step outside 0..n_steps-1. */
size_t sl7_cdc_hist_elems(void);
sl7_status sl7_cdc_init(sl7_ctx ctx, double Y0, double dt, int32_t n_steps, const double* theta,
                        int32_t n_theta, uint64_t n_paths, uint64_t seed, const sl7_run_opts* opts,
                        float* d_state);
sl7_status sl7_cdc_hist(sl7_ctx ctx, const float* d_state, int32_t pass, uint64_t* d_hist);
sl7_status sl7_cdc_select(sl7_ctx ctx, int32_t pass, const uint64_t* d_hist);
sl7_status sl7_cdc_step(sl7_ctx ctx, int32_t step, const float* d_in, float* d_out, double* d_stats);

/* ---------------------------------------------------------------------------------------------
 * Euler-Maruyama comparator and offline training-set generation.
 * --------------------------------------------------------------------------------------------- */

/* SDE models of Eq. 6.1 with their Euler-Maruyama coefficients (Eq. 6.2):
 *  GBM: a = mu Y,              b = sigma Y;            theta = (mu, sigma), sigma >= 0
 *  OU:  a = lam (Ybar - Y),    b = sigma;              theta = (Ybar, lam, sigma), lam, sigma >= 0
 *  CIR: a = kappa (Ybar - Y+), b = sigma sqrt(Y+);     theta = (kappa, Ybar, sigma), kappa, sigma >= 0,
 *       Y+ = max(Y, 0) ("full truncation"; the plain scheme is undefined for Y < 0, R-22). */
typedef enum { SL7_MODEL_GBM = 1, SL7_MODEL_OU = 2, SL7_MODEL_CIR = 3 } sl7_model;

/* Euler-Maruyama paths on the path generator's RNG, the classical comparator of the 7L scheme
 * (PAPER.md:32 Eq. 6.2; strong convergence contrast PAPER.md:16, :110).  Each large step dt is taken
 * as `substeps` (K >= 1) equal sub-steps dtau = dt / K:
 *     Y <- Y + a(Y) dtau + b(Y) sqrt(dtau) X,
 * fine step k = i K + s of path p consuming normal Z_{4b + (k & 3)}, b = k >> 2, of the same Philox
 * stream as sl7_simulate (so K = 1 shares the 7L scheme's normals step for step).  Outputs, d_out /
 * d_stats layouts, path_offset sharding and asynchrony are those of sl7_simulate (FULL records the
 * large steps).  opts: path_offset, stream, hist_lo/hi, shift, n_bins, accumulate, ref/ref_theta
 * (the reference runs on the FINE normals: GBM exact, OU exact Eq. 6.6 transition per sub-step) and
 * flags (SL7_FLAG_FAST_NORMALS only); prec, colloc and scheme are ignored.
 * Errors: SL7_EINVAL (model, theta, substeps, n_steps * substeps > 2^31, as sl7_simulate), SL7_ECUDA. */
sl7_status sl7_simulate_em(sl7_ctx ctx, sl7_model model, double Y0, double dt, int32_t n_steps,
                           int32_t substeps, const double* theta, int32_t n_theta, uint64_t n_paths,
                           uint64_t seed, sl7_out out_mode, const sl7_run_opts* opts, float* d_out,
                           double* d_stats);

/* Offline training-set generation (Algorithm I step 1; "the Euler-Maruyama scheme will
 * be used to generate the training data set ... tiny time steps").
 * h_features : HOST float64 rows [n_rows][2 + n_theta] = (y_start, dt, theta...) (theta order of
 *              sl7_model; dt > 0).
 * n_inner    : M >= m inner Monte Carlo paths per row.   dtau : target fine step, > 0.
 * Row r runs K_r = ceil(dt_r / dtau) Euler sub-steps of dt_r / K_r on M paths with
 * global ids path_offset + r M + q (q < M), each fine step k on Z_{p,k} as in sl7_simulate_em; its
 * labels are the empirical quantiles of the M terminal values at the levels Phi(x_j) of the context's
 * m Gauss-Hermite nodes (plotting position (k - 0.5)/M, linear interpolation between order statistics;
 * non-finite values excluded; NaN labels if none is finite).
 * d_terminal : device fp32 [n_rows][M] terminal values, or NULL (context scratch, processed in chunks).
 * d_labels   : device fp64 [n_rows][m], ascending per row.
 * opts: path_offset, stream, flags (SL7_FLAG_FAST_NORMALS only); the rest is ignored.
 * Asynchronous on opts->stream (the feature rows are copied before return).  Errors: SL7_EINVAL
 * (model, features, M, dtau, K_r > 2^31, path-id overflow), SL7_ENOMEM, SL7_ECUDA. */
sl7_status sl7_training_set(sl7_ctx ctx, sl7_model model, const double* h_features, uint64_t n_rows,
                            uint32_t n_inner, double dtau, uint64_t seed, const sl7_run_opts* opts,
                            float* d_terminal, double* d_labels);

/* Host setup introspection (no device needed): the context-independent grid of m nodes in
 * double (x[m], ascending) and barycentric weights w[m] = 1 / prod_{k != j}(x_j - x_k). */
sl7_status sl7_gh_grid(int32_t m, double* x, double* w);

size_t sl7_out_elems(int32_t n_steps, uint64_t n_paths, sl7_out mode); /* (n+1)N_P | N_P | 0 */
size_t sl7_stats_elems(int32_t n_bins);                                /* 8 + n_bins + 2 */
const char* sl7_last_error(sl7_ctx ctx);   /* never NULL; ctx may be NULL (thread-global msg) */
const char* sl7_status_str(sl7_status s);
int32_t sl7_abi_version(void);
void sl7_destroy(sl7_ctx ctx);              /* NULL is a no-op */

#ifdef __cplusplus
}
#endif
#endif /* SL7_H */
