/*
 * mdhp.h — C ABI of libmdhp.so, the B200 (sm_100a) MDHP-GDS hot path.
 *
 * MDHP-GDS (arxiv 2411.10258, "MDHP-Net") fits the parameters (theta, alpha, beta) of a
 * multi-dimensional Hawkes process with exponential kernels,
 *     lambda^i(t) = theta_i + sum_j sum_{k: T_j^k < t} alpha_ij exp(-beta_ij (t - T_j^k))   Eq.(2)
 * by gradient ascent on the closed-form log-likelihood
 *     lnL = Part1 + Part2 + Part3                                                      Eq.(5)
 *     Part1 = sum_i sum_{t in dim i} ln lambda^i(t)
 *     Part2 = -T_span sum_i theta_i
 *     Part3 = sum_i sum_j (alpha_ij / beta_ij) sum_k ( exp(-beta_ij (T_span - T_j^k)) - 1 )
 * with loss -lnL and "a PyTorch optimizer", independently per observation
 * window.  ("P:n" = line n of the paper text; "S:n" = line n of SPEC.md.)
 *
 * The three calls follow the paper's statement of the problem (north_star):
 *   mdhp_pack_windows  input = per-window marked event streams + horizon T;
 *                      the parameter-independent precompute ("decoupling"),
 *                      without the O(N^2) tMpT tensor.
 *   mdhp_loglik_grad   lnL of Eq.(5) and its gradient for a batch of windows.
 *   mdhp_fit           projected gradient descent / Adam on -lnL with the positivity
 *                      projection, stopping and rollback rules of DESIGN.md "Fit"
 *                      (SPEC S:159-160).
 *
 * CONVENTIONS (all calls)
 *   - D (number of marks / ECUs / message IDs) is 1..32.  Marks are 0..D-1.
 *   - alpha, beta are row-major D x D per window: element [i*D + j] is the excitation of
 *     TARGET i by SOURCE j, as in Eq.(2) P:107 (reading R1).
 *   - Parameter and result arrays are indexed by the ORIGINAL window index w (CSR order):
 *     theta [W][D], alpha [W][D][D], beta [W][D][D], loglik [W], win_status [W].
 *   - Every pointer argument named in a call is a CUDA DEVICE pointer on the current device,
 *     except the descriptor/config structs (host) and the *_host buffers of mdhp_fit_host.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls
 *     enqueue work on `stream` and return without synchronising, except where noted.
 *   - OWNERSHIP: the caller owns every buffer.  The library keeps no device memory between
 *     calls; temporary workspaces are stream-ordered (cudaMallocAsync/cudaFreeAsync) and
 *     freed before the call returns control of the stream.  The library is reentrant.
 *   - ERRORS: every int-returning call returns MDHP_OK (0) or a negative MDHP_E* code and
 *     sets a thread-local message readable with mdhp_last_error().  Data problems of a
 *     single window never fail a call: they are reported in that window's status word and
 *     the window is skipped (its outputs are set to NaN); other windows proceed.
 */
#ifndef MDHP_H_
#define MDHP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- return codes */
#define MDHP_OK       0
#define MDHP_EINVAL  -1   /* NULL pointer, bad config value                              */
#define MDHP_EDIM    -2   /* D outside 1..32, negative sizes                              */
#define MDHP_ESIZE   -3   /* packed buffer smaller than mdhp_packed_bytes()               */
#define MDHP_ECUDA   -5   /* a CUDA runtime call or kernel launch failed                  */

/* ---------------------------------------------------------------- per-window status bits */
#define MDHP_ST_OK            0
#define MDHP_ST_EMPTY         (1 << 0)  /* no events: allowed; lnL = -T sum theta */
#define MDHP_ST_UNSORTED      (1 << 1)  /* t decreases inside the window           */
#define MDHP_ST_OUT_OF_RANGE  (1 << 2)  /* t < 0, t > T or t not finite            */
#define MDHP_ST_BAD_MARK      (1 << 3)  /* mark outside 0..D-1                            */
#define MDHP_ST_SAME_DIM_TIE  (1 << 4)  /* two events of one mark share a time after      */
                                        /* conversion to fp32 (R10)      */
#define MDHP_ST_DEGENERATE    (1 << 5)  /* EQ6 with max(t) == min(t)              */
#define MDHP_ST_NONFINITE     (1 << 6)  /* fit: a non-finite lnL/gradient was met         */
#define MDHP_ST_DIVERGED      (1 << 7)  /* fit: halving budget exhausted          */
#define MDHP_ST_CONVERGED     (1 << 8)  /* fit: stopped by tol_rel / patience     */
#define MDHP_ST_BAD_T         (1 << 9)  /* T not finite or <= 0                           */
#define MDHP_ST_INVALID       (MDHP_ST_UNSORTED | MDHP_ST_OUT_OF_RANGE | MDHP_ST_BAD_MARK | \
                               MDHP_ST_SAME_DIM_TIE | MDHP_ST_DEGENERATE | MDHP_ST_BAD_T)

/* ---------------------------------------------------------------- packing */
#define MDHP_TIME_RAW   0   /* analysis time = t, horizon T                                  */
#define MDHP_TIME_UNIT  1   /* analysis time = t / T, horizon 1 (exact time rescaling: lnL   */
                            /* shifts by -N ln T, rates scale by T; R8)             */
#define MDHP_TIME_EQ6   2   /* Eq.(6) P:372-374 with the window's joint min/max over all     */
                            /* dims mapped to [eq6_lo, eq6_hi]; horizon eq6_hi */

#define MDHP_TIE_ERROR  0   /* a same-mark tie after fp32 conversion flags SAME_DIM_TIE        */
#define MDHP_TIE_NUDGE  1   /* in stream order y_k = max(fl32(x_k), y_{k-1}); if the */
                            /* previous event of the same mark has time y_k, y_k = next float up  */

typedef struct {
    int32_t D;            /* number of marks, 1..32                                         */
    int32_t time_mode;    /* MDHP_TIME_*                                                    */
    int64_t n_windows;    /* W >= 0                                                         */
    int64_t n_events;     /* E >= 0 (total over all windows, = win_off[W])                  */
    double  eq6_lo;       /* EQ6 target range (ignored otherwise)                           */
    double  eq6_hi;
    int32_t tie_policy;   /* MDHP_TIE_ERROR | MDHP_TIE_NUDGE                                */
    int32_t reserved;     /* 0                                                              */
} mdhp_pack_desc;

/* Bytes the packed buffer needs for this descriptor (a pure function of D, W, E).          */
size_t mdhp_packed_bytes(const mdhp_pack_desc* desc);

/*
 * mdhp_pack_windows — validate and convert a CSR batch of windows into the packed,
 * self-contained device layout that mdhp_loglik_grad / mdhp_fit consume.
 *
 *   t        [E] fp64   event times; window w owns t[win_off[w] .. win_off[w+1]), which
 *                       must be non-decreasing with 0 <= t <= T[w] (each window starts with
 *                       empty history at 0, R9).  Cross-mark ties are allowed and
 *                       resolved by the strict inequality of Eq.(2) (R2).
 *   mark     [E] int32  0..D-1
 *   win_off  [W+1] int64, win_off[0] = 0, non-decreasing, win_off[W] = E
 *   T        [W] fp64   window horizons T_span
 *   packed   device buffer of packed_bytes >= mdhp_packed_bytes(desc); fully (re)written
 *   win_status [W] int32 out: MDHP_ST_* validation bits (0 or EMPTY when usable)
 *
 * Per event the packer stores the fp32 analysis time (round-to-nearest of the mode's
 * conversion, see MDHP_TIME_*), the mark, and the fp32 gap to the previous event of the
 * same mark.  Per window and mark it stores the event count, and the power moments
 * m_p = sum_k (u_k / u_max)^p, p = 1..17, of u_k = T - t_k, which the Part3 epilogue uses
 * when beta * u_max <= 2 (no cancellation at small beta, R20).  Windows are
 * ordered longest first for scheduling (results do not depend on that order).
 * Asynchronous.  Returns MDHP_EINVAL / MDHP_EDIM / MDHP_ESIZE / MDHP_ECUDA on misuse only.
 */
int mdhp_pack_windows(const mdhp_pack_desc* desc, const double* t, const int32_t* mark,
                      const int64_t* win_off, const double* T, void* packed,
                      size_t packed_bytes, int32_t* win_status, void* stream);

/*
 * mdhp_loglik_grad — Eq.(5) and its analytic gradient for every window of a packed batch.
 *
 *   theta [W][D], alpha [W][D][D], beta [W][D][D]  fp32, in the packed time units; invariants
 *                 theta > 0, alpha >= 0, beta > 0 are the caller's responsibility
 *   loglik [W]    fp64 out: lnL (NaN for invalid windows)
 *   g_theta [W][D], g_alpha [W][D][D], g_beta [W][D][D]  fp32 out: d lnL / d(.)
 *                 (all three NULL -> lnL only; otherwise all three must be non-NULL)
 * Gradient formulas: d theta_i = sum_{n in i} 1/lambda_n - T;
 *   d alpha_ij = sum_{n in i} R_ij(t_n)/lambda_n + E_ij/beta_ij;
 *   d beta_ij  = -alpha_ij sum_{n in i} Q_ij(t_n)/lambda_n + alpha_ij H_ij / beta_ij^2, with
 *   R, Q the decayed sums of Eq.(2) and of (t - t_k) times its terms, E_ij = sum_k (e^{-b u_k} - 1),
 *   H_ij = sum_k (1 - e^{-b u_k}(1 + b u_k)).
 * Precision: fp32 evaluation; windows whose fp32 lnL could miss 1e-4 relative (R24)
 * are re-evaluated in fp64 on the GPU (lnL and gradients; see mdhp_loglik_exact).
 * Asynchronous (one stream-ordered workspace of 256 + 4 W bytes).
 */
int mdhp_loglik_grad(const mdhp_pack_desc* desc, const void* packed,
                     const float* theta, const float* alpha, const float* beta,
                     double* loglik, float* g_theta, float* g_alpha, float* g_beta,
                     const int32_t* win_status, void* stream);

/*
 * mdhp_loglik_exact — the same outputs as mdhp_loglik_grad, every window evaluated in fp64 on
 * the GPU (state, exponentials, logarithms and sums in double, from the packed fp32 analysis
 * times; Part3 terms summed directly as sum_k expm1(-beta u_k)).  mdhp_loglik_grad and
 * mdhp_fit run this evaluation automatically on the windows whose fp32 lnL could miss 1e-4
 * relative (R24: lnL a cancellation of much larger terms); this entry point applies
 * it to the whole batch (reference-quality GPU evaluation, ~100x the fp32 cost).
 * Same arguments and layout as mdhp_loglik_grad.  Asynchronous.
 */
int mdhp_loglik_exact(const mdhp_pack_desc* desc, const void* packed,
                      const float* theta, const float* alpha, const float* beta,
                      double* loglik, float* g_theta, float* g_alpha, float* g_beta,
                      const int32_t* win_status, void* stream);

/*
 * mdhp_loglik_dense — ABLATION: lnL of Eq.(5) evaluated the way the
 * paper's Algorithms 1-3 do, i.e. by summing over ALL causal pairs (O(N^2)
 * exponentials per window instead of the recurrence's 2 D N), in the Eq.(5)-correct form
 * (causal mask, Part3 with "-1"; R4/R5).  Same arguments and layout as
 * mdhp_loglik_grad without gradients.  Not used by mdhp_fit; it exists to measure the paper's
 * method on the same GPU and as an independent GPU cross-check.  Asynchronous.
 */
int mdhp_loglik_dense(const mdhp_pack_desc* desc, const void* packed, const float* theta,
                      const float* alpha, const float* beta, double* loglik,
                      const int32_t* win_status, void* stream);

/* ---------------------------------------------------------------- fit */
#define MDHP_OPT_GD    0
#define MDHP_OPT_ADAM  1       /* torch.optim.Adam semantics (amsgrad off, no weight decay) */
#define MDHP_FIT_THETA 1u
#define MDHP_FIT_ALPHA 2u
#define MDHP_FIT_BETA  4u

typedef struct {
    int32_t  max_iters;     /* >= 0 iterations (evaluations followed by a step)            */
    int32_t  optimizer;     /* MDHP_OPT_GD | MDHP_OPT_ADAM                                 */
    float    lr;            /* > 0                                                          */
    float    adam_b1, adam_b2, adam_eps;
    int32_t  loss_mean;     /* 0: loss = -lnL;  1: loss = -lnL / N_w               */
    float    tol_rel;       /* <= 0: fixed-iteration mode; else stop after `patience`       */
    int32_t  patience;      /*   consecutive |dlnL| <= tol_rel*max(|lnL_prev|,1)    */
    float    min_param;     /* projection floor for theta and beta; alpha floor is 0 */
    uint32_t fit_mask;      /* MDHP_FIT_* groups that are updated; others keep their init   */
    int32_t  max_halvings;  /* non-finite evaluation: roll back, halve lr           */
    int32_t  adam_step0;    /* Adam steps already taken (bias-correction offset) when resuming
                               from a returned opt_state; 0 for a fresh fit.  fit(k) then
                               fit(m, opt_state, adam_step0 = k) == fit(k + m) in fixed-
                               iteration mode (checkpoint / resume)        */
    int32_t  time_chunks;   /* 0 or 1: throughput layout (32/Dp windows per warp).  C >= 2, for
                               D <= 8: each window's events are cut into C' = min(pow2 <= C,
                               32/Dp) time chunks run in parallel by C' lane groups (chunked
                               scan inside the warp, DESIGN.md a6), 32/(Dp C') windows per warp:
                               shorter per-window chains for single windows (latency mode,
                               C' = 32/Dp: one window per warp) and small batches.  Results
                               agree with C = 0 within fp32 rounding (another fixed summation
                               order), deterministically.  Ignored for D > 8.                */
} mdhp_fit_config;

/*
 * mdhp_fit — the whole MDHP-GDS iteration loop on the device, every window independently:
 *   repeat: evaluate (lnL, grad) -> non-finite? roll back + halve lr -> stopping test ->
 *           GD / Adam step on -lnL -> projection   (DESIGN.md "Fit" gives the exact loop).
 *
 *   theta, alpha, beta  in: initial parameters; out: fitted (projected) parameters
 *   opt_state [W][2][D + 2 D^2] fp32 Adam moments (m then v, each in theta|alpha|beta order),
 *             in/out; NULL -> zero-initialised internal workspace (resume = pass it back
 *             with cfg->adam_step0 = the iterations already run)
 *   loglik [W]   fp64 out: lnL at the returned parameters (fp32 evaluation, fp64 on the GPU for
 *                the windows of DESIGN.md R24)
 *   iters  [W]   int32 out: iterations run
 *   win_status [W] in: from mdhp_pack_windows; out: its validation bits (MDHP_ST_INVALID | EMPTY)
 *                OR-ed with this call's NONFINITE / DIVERGED / CONVERGED (outcome bits of an
 *                earlier call on the same batch are not carried over)
 *   lnl_trace [W][max_iters] fp32 out or NULL: lnL of every evaluation (NaN after the stop)
 * One persistent kernel launch for the iteration loop (+1 for the fp64 re-evaluation of
 * cancellation windows).  Each CTA allocates tensor memory (TMEM) for the windows' optimizer
 * state (pow2(7 Dp + 3) columns; 128 at D = 16) and frees it before it exits; kernels of other
 * streams that hold TMEM on the same SMs can delay it.  Asynchronous.
 */
int mdhp_fit(const mdhp_pack_desc* desc, const void* packed, const mdhp_fit_config* cfg,
             float* theta, float* alpha, float* beta, float* opt_state,
             double* loglik, int32_t* iters, int32_t* win_status, float* lnl_trace,
             void* stream);

/*
 * mdhp_fit_host — end-to-end convenience call on HOST buffers (pinned memory recommended):
 * copies the CSR batch and initial parameters to the device, packs, fits, and copies the
 * fitted parameters, loglik, iters and status back.  Same arguments as pack + fit with host
 * pointers (win_off_host[0] must be 0 and win_off_host[W] = n_events, else MDHP_EINVAL).
 * Synchronous (returns after the device->host copies completed).  From 4,096 windows on, the
 * batch is processed as 4 window ranges: the uploads run on a private copy stream and overlap
 * the fits on `stream`, each range's results go back while the next range fits (windows are
 * independent: the outputs equal those of pack + fit on the whole batch).
 * Workspace comes from the device's default stream-ordered memory pool; mdhp_fit and
 * mdhp_fit_host raise that pool's release threshold (once per device) so repeated calls reuse
 * the memory instead of re-mapping it (cudaMemPoolTrimTo releases it).
 */
int mdhp_fit_host(const mdhp_pack_desc* desc, const double* t_host, const int32_t* mark_host,
                  const int64_t* win_off_host, const double* T_host,
                  const mdhp_fit_config* cfg, float* theta_host, float* alpha_host,
                  float* beta_host, double* loglik_host, int32_t* iters_host,
                  int32_t* win_status_host, void* stream);

/* ---------------------------------------------------------------- long single sequences (a7)
 * One long marked sequence on [0, T] (e.g. BASELINE config 4: D = 16, 1e6 events over 1000 s),
 * evaluated and fitted by a chunked parallel scan: the sequence is cut into chunks of about
 * chunk_events events (never inside a group of equal times), each chunk's times are stored
 * relative to its base (the previous chunk's last event; fp64 difference rounded to fp32, so
 * resolution stays ~1e-7 s), chunk-local decayed states are combined by an exclusive scan of
 * their affine maps (S <- e^{-beta L} S + S_loc, Q <- e^{-beta L}(Q + L S) + Q_loc), and every
 * chunk then re-runs the event loop from its carried-in state.  Same Eq.(5) lnL and gradients
 * as mdhp_loglik_grad (row a7).  Times are RAW (seconds).             */
typedef struct {
    int32_t D;             /* 1..32                                                         */
    int32_t chunk_events;  /* >= 8; 256 is a good default                                   */
    int64_t n_events;      /* N >= 0 (of this slice, see f1 below)                          */
    double  T;             /* horizon T_span > 0                                             */
    double  t0;            /* slice base: 0 for a whole sequence; for rank r > 0 of a sliced */
                           /* sequence, the time of the previous slice's last event          */
    int32_t has_history;   /* 0: empty history at t0 (whole sequence / rank 0); 1: the state */
                           /* carried in from earlier slices applies (rank > 0)              */
    int32_t reserved;      /* 0                                                              */
} mdhp_seq_desc;

size_t mdhp_seq_packed_bytes(const mdhp_seq_desc* desc);

/* A chunk_events value for an N-event sequence of D marks on the CURRENT device: the smallest
 * size (>= 8) whose chunks fill whole waves of the phase-3 kernel (SM count x its occupancy x
 * chunks per warp), so no SM runs one more block than the others in a partial last wave
 * (a chunk never exceeds chunk_events events, tie groups aside, so ceil(N / size) bounds the
 * chunk count).  At least 256 events per chunk once a wave is full.  Returns the size, or a
 * negative MDHP_E* code (EDIM: D outside 1..32 or N < 0; ECUDA).  Host-only, synchronous.
 * Not in the paper: a launch-shape helper for the chunked scan of row a7.                    */
int32_t mdhp_seq_chunk_hint(int32_t D, int64_t n_events);

/* t [N] fp64 non-decreasing in [0, T], mark [N] int32 in 0..D-1 (device).  status [1] int32
 * (device) receives the MDHP_ST_* validation bits.  Asynchronous.                          */
int mdhp_seq_pack(const mdhp_seq_desc* desc, const double* t, const int32_t* mark,
                  void* packed, size_t packed_bytes, int32_t* status, void* stream);

/* theta [D], alpha [D][D], beta [D][D] fp32; loglik [1] fp64; g_* as in mdhp_loglik_grad
 * (all NULL -> lnL only).  NaN outputs for an invalid sequence.  Asynchronous.              */
int mdhp_seq_loglik_grad(const mdhp_seq_desc* desc, const void* packed, const float* theta,
                         const float* alpha, const float* beta, double* loglik, float* g_theta,
                         float* g_alpha, float* g_beta, void* stream);

/* The loop of mdhp_fit for one sequence: per iteration 3 scan phases + reduce + one fused
 * epilogue/step kernel; the stop/rollback state lives on the device (no host sync).
 * opt_state [2][D + 2 D^2] or NULL; loglik [1]; iters [1]; status [1] out; lnl_trace
 * [max_iters] or NULL.  Asynchronous.                                                      */
int mdhp_seq_fit(const mdhp_seq_desc* desc, const void* packed, const mdhp_fit_config* cfg,
                 float* theta, float* alpha, float* beta, float* opt_state, double* loglik,
                 int32_t* iters, int32_t* status, float* lnl_trace, void* stream);

/* ---------------------------------------------------------------- f1: one sequence over GPUs
 * SURVEY 8(f) f1.  Rank r holds a contiguous slice of the sequence (packed with t0 = previous
 * slice's last event and has_history = r > 0).  Per evaluation:
 *   1. mdhp_seq_maps   local chunk states + the slice's composite affine map from a zero state
 *                      (rankmap = {S, Q'} per pair at the slice's last event, rankspan = its span)
 *   2. all_gather of (rankmap, rankspan) over ranks          [the exchange: 2 D^2 + 1 floats/rank]
 *   3. mdhp_seq_parts  carried-in state = earlier slices' maps composed in order, then the chunk
 *                      scan, the event loop and fixed-order sums -> parts (2 D^2 + D + 1 fp64:
 *                      gR, gQ interleaved, g_theta, sum lg2 lambda) and fin (end state)
 *   4. all_reduce(sum) of parts; fin of the last rank is the global final state
 *   5. mdhp_seq_finish epilogue (and with cfg, one step of the DESIGN.md "Fit" loop), identical
 *                      on every rank.  Stats (counts, u_max, moments, tail) are combined once per
 *                      fit: mdhp_seq_stats per rank -> all_gather -> mdhp_seq_stats_combine.
 * Exact decomposition: the same lnL and gradients as the single-GPU path up to fp32 rounding.
 * `work` is a caller-owned device buffer of mdhp_seq_work_bytes() bytes, initialised with
 * mdhp_seq_work_init (cfg NULL for evaluation only).  All calls are asynchronous.            */
size_t mdhp_seq_work_bytes(const mdhp_seq_desc* desc);
int mdhp_seq_work_init(const mdhp_seq_desc* desc, void* work, const mdhp_fit_config* cfg,
                       void* stream);
int mdhp_seq_maps(const mdhp_seq_desc* desc, const void* packed, const float* beta, void* work,
                  float* rankmap, float* rankspan, int32_t fit, void* stream);
int mdhp_seq_parts(const mdhp_seq_desc* desc, const void* packed, const float* theta,
                   const float* alpha, const float* beta, const float* maps, const float* spans,
                   int32_t rank, void* work, double* parts, float* fin, int32_t grad, int32_t fit,
                   void* stream);
int mdhp_seq_stats(const mdhp_seq_desc* desc, const void* packed, double* stats, void* stream);
int mdhp_seq_stats_combine(int32_t D, int32_t R, const double* gathered, double* combined,
                           void* stream);
int mdhp_seq_finish(const mdhp_seq_desc* desc, int64_t n_events_total, const double* stats,
                    const double* parts, const float* fin, float* theta, float* alpha, float* beta,
                    double* loglik, float* g_theta, float* g_alpha, float* g_beta,
                    const mdhp_fit_config* cfg, void* work, float* opt_state, float* lnl_trace,
                    int32_t* status, int32_t* iters, int32_t final_eval, const void* packed,
                    void* stream);

/* Byte offsets of the packed sections (introspection for tests/tools), in this order:
 * [0] begin i64[W]  [1] n i32[W]  [2] T32 f32[W]  [3] perm i32[W]  [4] t32 f32[Epad]
 * [5] dtp f32[Epad] [6] mark u8[Epad]  [7] cnt i32[W][Dp]  [8] umax f32[W][Dp]
 * [9] mom f32[W][Dp][17]  [10] sort scratch  [11] total bytes  [12] Epad  [13] Dp.
 * Dp = D rounded up to a power of two.  Returns MDHP_OK or MDHP_EINVAL / MDHP_EDIM.        */
int mdhp_packed_layout(const mdhp_pack_desc* desc, size_t offsets[14]);

/* ---------------------------------------------------------------- f4: MDHP-LSTM Hawkes gate */
/*
 * mdhp_hawkes_features — SURVEY 8(f) row f4: the Hawkes gate of the MDHP-LSTM cell, Eq.(7)
 * third line, for every window of a batch of fitted parameters:
 *
 *     hks[w][h] = tanh( sum_ij A[h][i*D+j] alpha[w][i][j]
 *                       - sum_ij B[h][i*D+j] beta[w][i][j] * T_span[w]
 *                       + sum_j  C[h][j] theta[w][j] )
 *
 * (SPEC S:366-381 reading: alpha^x, beta^x flattened row-major, the product beta^x T_span^x
 * entrywise; computed once per window.)  One tensor-core GEMM (tcgen05 kind::tf32, TMEM
 * accumulator) with a fused tanh epilogue.  Inputs are rounded to TF32 (round-to-nearest)
 * before the products, so the pre-activation carries an error <= ~2^-10 * sum_k |W_hk X_wk|
 * (R22); accumulation is fp32.
 *
 *   D                 1..32
 *   n_windows         W >= 0
 *   H                 hidden size: a multiple of 16, <= 256, or a multiple of 256
 *   theta [W][D], alpha [W][D][D], beta [W][D][D]   fp32 device (e.g. mdhp_fit output)
 *   T_span [W]        fp32 device: window horizon in the parameters' time units
 *   A [H][D*D], B [H][D*D], C [H][D]                fp32 device, row-major
 *   hks [W][H]        fp32 device out (16-byte aligned)
 * Returns MDHP_OK, MDHP_EINVAL (NULL pointer), MDHP_EDIM (D or H out of range), MDHP_ECUDA.
 * Asynchronous on `stream`; no workspace.
 */
int mdhp_hawkes_features(int32_t D, int64_t n_windows, int32_t H, const float* theta,
                         const float* alpha, const float* beta, const float* T_span,
                         const float* A, const float* B, const float* C, float* hks,
                         void* stream);

/* ---------------------------------------------------------------- misc */
const char* mdhp_last_error(void);   /* thread-local message of the last failing call     */
uint64_t    mdhp_launch_count(void); /* kernels this library has launched (process-wide)   */
int32_t     mdhp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MDHP_H_ */
