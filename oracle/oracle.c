/*
 * oracle.c — plain, slow, fp64 CPU oracle for MDHP-GDS (arxiv 2411.10258).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2411_10258_b200/csrc), and it
 * includes nothing from there.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n.
 *
 * Contents
 *   oracle_convert_window  the packing definition: fp64 event times -> fp32 analysis
 *                          times (RAW / UNIT / EQ6 standardisation, Eq.(6)),
 *                          validation, per-window status.
 *   oracle_loglik_def      Eq.(5) written out literally: O(N^2) pairwise
 *                          sums for Part1, Part2 = -T*sum(theta), Part3 with its "-1",
 *                          and the analytic partial derivatives of each term.
 *   oracle_loglik_rec      the same quantity by the eager exponential recursion
 *                          (the multi-dimensional form of Ozaki's recursion cited at
 *                          P:270): all D*D pair states decayed at every tie group.
 *                          O(N*D^2); used where O(N^2) is too slow (long windows, fits).
 *   oracle_fit             projected gradient ascent on lnL with the
 *                          optimizer/stopping definition of DESIGN.md section "Fit".
 *   *_batch                the same over many windows, on a pthread pool.
 *   oracle_hawkes_features the MDHP-LSTM Hawkes gate, Eq.(7) third line:
 *                          hks = tanh(A alpha - B (beta T_span) + C theta) per window
 *                          (SURVEY 8(f) row f4), plain loops in fp64.
 *
 * Conventions: alpha, beta are D*D row-major [i][j] = target i, source j (Eq.(2) P:107:
 * lambda^i sums over sources j).  theta is length D.  Times are fp64: the fp32 analysis times
 * produced by oracle_convert_window promoted exactly, or raw fp64 times (long sequences).
 */
#include <math.h>
#include <float.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ---- per-window status bits; values chosen here, independently
 *      matched by the CUDA path's own definition in include/mdhp.h. ---- */
#define OR_OK             0
#define OR_EMPTY          (1 << 0)
#define OR_UNSORTED       (1 << 1)
#define OR_OUT_OF_RANGE   (1 << 2)
#define OR_BAD_MARK       (1 << 3)
#define OR_SAME_DIM_TIE   (1 << 4)
#define OR_DEGENERATE     (1 << 5)
#define OR_NONFINITE      (1 << 6)
#define OR_DIVERGED       (1 << 7)
#define OR_CONVERGED      (1 << 8)
#define OR_BAD_T          (1 << 9)
#define OR_INVALID_MASK   (OR_UNSORTED | OR_OUT_OF_RANGE | OR_BAD_MARK | OR_SAME_DIM_TIE | OR_DEGENERATE | OR_BAD_T)

#define OR_TIME_RAW  0
#define OR_TIME_UNIT 1
#define OR_TIME_EQ6  2

/* -------------------------------------------------------------------------------------
 * Packing definition.
 *   RAW : x = t,                         T' = T
 *   UNIT: x = t / T,                     T' = 1       (time rescaling; R8)
 *   EQ6 : x = (t-mn)/(mx-mn)*(hi-lo)+lo, T' = hi      (Eq.(6), joint min/max over
 *                                                      all dims of the window)
 * then t32 = (float)x (round to nearest), T32 = (float)T'.
 * Validation, on the input order:  T finite and > 0 (else BAD_T); every t finite with
 * 0 <= t <= T (else OUT_OF_RANGE); 0 <= mark < D (else BAD_MARK); t non-decreasing
 * (else UNSORTED); after rounding, no two events of the same mark share a t32
 * (else SAME_DIM_TIE, S:106 / DESIGN.md R10; with tie_policy NUDGE such events are moved up
 * instead, see below); EQ6 with mx == mn -> DEGENERATE.
 * An empty window is valid (status EMPTY).  Returns the status word.
 * ------------------------------------------------------------------------------------- */
int oracle_convert_window(int D, int time_mode, double lo, double hi, int tie_policy, int64_t n,
                          const double* t, const int32_t* mark, double T,
                          float* t32_out, float* T32_out)
{
    int status = OR_OK;
    if (!(T > 0.0) || !isfinite(T)) status |= OR_BAD_T;
    if (n == 0) status |= OR_EMPTY;
    double mn = INFINITY, mx = -INFINITY;
    for (int64_t k = 0; k < n; k++) {
        if (!isfinite(t[k]) || t[k] < 0.0 || t[k] > T) status |= OR_OUT_OF_RANGE;
        if (mark[k] < 0 || mark[k] >= D) status |= OR_BAD_MARK;
        if (k > 0 && t[k] < t[k - 1]) status |= OR_UNSORTED;
        if (t[k] < mn) mn = t[k];
        if (t[k] > mx) mx = t[k];
    }
    double Tp = T;
    if (time_mode == OR_TIME_UNIT) Tp = 1.0;
    if (time_mode == OR_TIME_EQ6) {
        Tp = hi;
        if (n > 0 && !(mx > mn)) status |= OR_DEGENERATE;
    }
    for (int64_t k = 0; k < n; k++) {
        double x = t[k];
        if (time_mode == OR_TIME_UNIT) x = t[k] / T;
        else if (time_mode == OR_TIME_EQ6) x = (t[k] - mn) / (mx - mn) * (hi - lo) + lo;
        t32_out[k] = (float)x;
    }
    *T32_out = (float)Tp;
    /* tie_policy 1 = NUDGE, the rule of include/mdhp.h MDHP_TIE_NUDGE, applied
       literally in stream order: y_k = max(fl32(x_k), y_{k-1}); if the previous event of the same
       mark has time y_k, y_k = nextafterf(y_k, +inf). */
    if (tie_policy == 1 && !(status & (OR_BAD_MARK | OR_UNSORTED))) {
        float floor_ = -INFINITY;
        for (int64_t k = 0; k < n; k++) {
            float y = t32_out[k] > floor_ ? t32_out[k] : floor_;
            for (int64_t q = k - 1; q >= 0; q--) {        /* previous event of the same mark */
                if (mark[q] == mark[k]) {
                    if (t32_out[q] == y) y = nextafterf(y, INFINITY);
                    break;
                }
            }
            t32_out[k] = y;
            floor_ = y;
        }
    }
    /* same-dim ties after rounding: compare every pair of events with equal mark that
       are adjacent among that mark's events (plain O(N*D) scan, no cleverness). */
    if (!(status & (OR_BAD_MARK | OR_UNSORTED))) {
        for (int j = 0; j < D; j++) {
            int have = 0; float prev = 0.0f;
            for (int64_t k = 0; k < n; k++) {
                if (mark[k] != j) continue;
                if (have && t32_out[k] == prev) status |= OR_SAME_DIM_TIE;
                prev = t32_out[k]; have = 1;
            }
        }
    }
    return status;
}

/* -------------------------------------------------------------------------------------
 * Eq.(5), written out.
 *   Part1 = sum_i sum_{t in dim i} ln( theta_i + sum_j sum_{k: T_j^k < t} a_ij e^{-b_ij (t - T_j^k)} )
 *   Part2 = -T * sum_i theta_i
 *   Part3 = sum_i sum_j (a_ij / b_ij) sum_k ( e^{-b_ij (T - T_j^k)} - 1 )
 * The inner constraint "k ^ T_j^k < t" is read as all k with T_j^k < t, strictly (Eq.(4)
 * P:283 "k : T_j^k < t"; R2), so coincident cross-dim events do not excite each
 * other.  Part3 keeps the "-1" of Eq.(5)/App. B, not Algorithm 3's form
 * (R4).  (e - 1) is evaluated with expm1, which is that quantity, accurately.
 *
 * Gradients (analytic partial derivatives of the three parts; the paper uses autograd):
 *   d/d theta_i : sum_{n in i} 1/lambda_n                                 - T
 *   d/d a_ij    : sum_{n in i} sum_{k in j, t_k<t_n} e^{-b(t_n-t_k)}/lambda_n + (1/b) sum_k (e^{-b u_k}-1)
 *   d/d b_ij    : -a sum_{n in i} sum_{k in j,t_k<t_n} (t_n-t_k) e^{-b(t_n-t_k)}/lambda_n
 *                 - (a/b^2) sum_k (e^{-b u_k}-1) - (a/b) sum_k u_k e^{-b u_k},   u_k = T - t_k
 * gamma_out (optional) receives Gamma of App. B = T sum theta - Part3.
 * Any gradient pointer may be NULL.
 * ------------------------------------------------------------------------------------- */
double oracle_loglik_def(int D, int64_t n, const double* t, const int32_t* mark, double T,
                         const double* theta, const double* alpha, const double* beta,
                         double* g_theta, double* g_alpha, double* g_beta, double* gamma_out)
{
    if (g_theta) for (int i = 0; i < D; i++) g_theta[i] = 0.0;
    if (g_alpha) for (int i = 0; i < D * D; i++) g_alpha[i] = 0.0;
    if (g_beta)  for (int i = 0; i < D * D; i++) g_beta[i] = 0.0;
    double* ra = (double*)calloc((size_t)D, sizeof(double));   /* sum_k e^{..}      per source j */
    double* rq = (double*)calloc((size_t)D, sizeof(double));   /* sum_k dt e^{..}   per source j */

    /* Part1 */
    double part1 = 0.0;
    for (int64_t nn = 0; nn < n; nn++) {
        int i = mark[nn];
        double tn = (double)t[nn];
        for (int j = 0; j < D; j++) { ra[j] = 0.0; rq[j] = 0.0; }
        for (int64_t k = 0; k < n; k++) {
            double tk = (double)t[k];
            if (!(tk < tn)) continue;                 /* strict: T_j^k < t */
            int j = mark[k];
            double dt = tn - tk;
            double e = exp(-beta[i * D + j] * dt);
            ra[j] += e;
            rq[j] += dt * e;
        }
        double lam = theta[i];
        for (int j = 0; j < D; j++) lam += alpha[i * D + j] * ra[j];
        part1 += log(lam);
        double w = 1.0 / lam;
        if (g_theta) g_theta[i] += w;
        for (int j = 0; j < D; j++) {
            if (g_alpha) g_alpha[i * D + j] += ra[j] * w;
            if (g_beta)  g_beta[i * D + j]  += -alpha[i * D + j] * rq[j] * w;
        }
    }

    /* Part2 */
    double sum_theta = 0.0;
    for (int i = 0; i < D; i++) sum_theta += theta[i];
    double part2 = -T * sum_theta;
    if (g_theta) for (int i = 0; i < D; i++) g_theta[i] -= T;

    /* Part3 */
    double part3 = 0.0;
    for (int i = 0; i < D; i++) {
        for (int j = 0; j < D; j++) {
            double a = alpha[i * D + j], b = beta[i * D + j];
            double E = 0.0, F = 0.0;          /* E = sum_k (e^{-b u_k} - 1), F = sum_k u_k e^{-b u_k} */
            for (int64_t k = 0; k < n; k++) {
                if (mark[k] != j) continue;
                double u = T - (double)t[k];
                E += expm1(-b * u);
                F += u * exp(-b * u);
            }
            part3 += (a / b) * E;
            if (g_alpha) g_alpha[i * D + j] += E / b;
            if (g_beta)  g_beta[i * D + j]  += -(a / (b * b)) * E - (a / b) * F;
        }
    }
    free(ra); free(rq);
    if (gamma_out) *gamma_out = T * sum_theta - part3;
    return part1 + part2 + part3;
}

/* -------------------------------------------------------------------------------------
 * The eager recursion (Ozaki's univariate recursion, applied to every pair (i,j)):
 *   R_ij(t) = sum_{k in j, t_k < t} e^{-b_ij (t - t_k)},  Q_ij(t) = sum_k (t - t_k) e^{-b_ij (t-t_k)}
 * Between tie groups (maximal runs of equal t):  Q <- e^{-b D}(Q + D R),  R <- e^{-b D} R.
 * Inside a group every member reads (R, Q) before any member is added (strict inequality),
 * then every member of source j adds 1 to R_.j.  Part3 terms are computed directly per
 * event as in oracle_loglik_def (expm1), not as R(T) - N.
 * Same outputs as oracle_loglik_def.
 * ------------------------------------------------------------------------------------- */
double oracle_loglik_rec(int D, int64_t n, const double* t, const int32_t* mark, double T,
                         const double* theta, const double* alpha, const double* beta,
                         double* g_theta, double* g_alpha, double* g_beta, double* gamma_out)
{
    size_t DD = (size_t)D * D;
    double* R  = (double*)calloc(DD, sizeof(double));
    double* Q  = (double*)calloc(DD, sizeof(double));
    double* gR = (double*)calloc(DD, sizeof(double));
    double* gQ = (double*)calloc(DD, sizeof(double));
    double* gt = (double*)calloc((size_t)D, sizeof(double));
    double* E  = (double*)calloc(DD, sizeof(double));
    double* F  = (double*)calloc(DD, sizeof(double));
    double tau = 0.0, part1 = 0.0;

    int64_t g0 = 0;
    while (g0 < n) {
        double tg = (double)t[g0];
        int64_t g1 = g0;
        while (g1 < n && (double)t[g1] == tg) g1++;
        double dl = tg - tau;
        if (dl != 0.0) {
            for (size_t p = 0; p < DD; p++) {
                double e = exp(-beta[p] * dl);
                Q[p] = e * (Q[p] + dl * R[p]);
                R[p] = e * R[p];
            }
            tau = tg;
        }
        for (int64_t nn = g0; nn < g1; nn++) {         /* read: lambda at t, strict past */
            int i = mark[nn];
            double lam = theta[i];
            for (int j = 0; j < D; j++) lam += alpha[i * D + j] * R[i * D + j];
            part1 += log(lam);
            double w = 1.0 / lam;
            gt[i] += w;
            for (int j = 0; j < D; j++) {
                gR[i * D + j] += R[i * D + j] * w;
                gQ[i * D + j] += Q[i * D + j] * w;
            }
        }
        for (int64_t nn = g0; nn < g1; nn++) {         /* then add the group's events */
            int j = mark[nn];
            for (int i = 0; i < D; i++) R[i * D + j] += 1.0;
        }
        g0 = g1;
    }
    for (int64_t k = 0; k < n; k++) {                  /* compensator terms, directly */
        int j = mark[k];
        double u = T - (double)t[k];
        for (int i = 0; i < D; i++) {
            double b = beta[i * D + j];
            E[i * D + j] += expm1(-b * u);
            F[i * D + j] += u * exp(-b * u);
        }
    }
    double sum_theta = 0.0, part3 = 0.0;
    for (int i = 0; i < D; i++) sum_theta += theta[i];
    for (int i = 0; i < D; i++) {
        if (g_theta) g_theta[i] = gt[i] - T;
        for (int j = 0; j < D; j++) {
            size_t p = (size_t)i * D + j;
            double a = alpha[p], b = beta[p];
            part3 += (a / b) * E[p];
            if (g_alpha) g_alpha[p] = gR[p] + E[p] / b;
            if (g_beta)  g_beta[p]  = -a * gQ[p] - (a / (b * b)) * E[p] - (a / b) * F[p];
        }
    }
    if (gamma_out) *gamma_out = T * sum_theta - part3;
    free(R); free(Q); free(gR); free(gQ); free(gt); free(E); free(F);
    return part1 - T * sum_theta + part3;
}

/* -------------------------------------------------------------------------------------
 * Fit (P:322 loss = -lnL, "a PyTorch optimizer"; SPEC S:159-160,
 * S:182-185 for projection, stopping, rollback and defaults).  Loss L = -lnL (SUM) or
 * -lnL/N (MEAN).  g_L = -grad(lnL) * scale.
 *   GD  : p <- p - lr_w * g_L
 *   ADAM: PyTorch torch.optim.Adam, amsgrad=False, weight_decay=0:
 *         m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2;
 *         p <- p - (lr_w / (1 - b1^s)) * m / ( sqrt(v) / sqrt(1 - b2^s) + eps ),   s = step count
 *   project: alpha <- max(alpha, 0); beta <- max(beta, floor); theta <- max(theta, floor)
 * Loop (identical on the GPU):
 *   it = 0
 *   while it < max_iters:
 *     evaluate (lnL, grad) at p
 *     if non-finite: status |= NONFINITE; if no previous point or halvings == max_halvings -> DIVERGED (p <- previous
 *                    point if any), stop;  else p <- previous point, lr_w /= 2, halvings++,
 *                    it++, continue
 *     if tol_rel > 0 and it has a previous lnL: stall = (|lnL - prev| <= tol_rel*max(|prev|,1)) ? stall+1 : 0
 *                    if stall >= patience -> CONVERGED, stop
 *     prev = lnL; previous point <- p; s++; step; project; it++
 *   lnL_out = lnL(p) at the returned p;  iters_out = it
 * ------------------------------------------------------------------------------------- */
typedef struct {
    int32_t max_iters;
    int32_t optimizer;       /* 0 = GD, 1 = ADAM */
    double  lr, b1, b2, eps;
    int32_t loss_mean;       /* 0 = SUM (-lnL), 1 = MEAN (-lnL / N) */
    double  tol_rel;
    int32_t patience;
    double  min_param;
    uint32_t fit_mask;       /* 1 = theta, 2 = alpha, 4 = beta */
    int32_t max_halvings;
    int32_t use_def;         /* 1: evaluate with oracle_loglik_def, 0: oracle_loglik_rec */
} oracle_fit_cfg;

static int all_finite(const double* x, size_t n) {
    for (size_t k = 0; k < n; k++) if (!isfinite(x[k])) return 0;
    return 1;
}

int oracle_fit(int D, int64_t n, const double* t, const int32_t* mark, double T,
               const oracle_fit_cfg* cfg, double* theta, double* alpha, double* beta,
               double* lnl_out, int32_t* iters_out, double* trace)
{
    size_t DD = (size_t)D * D, P = 2 * DD + D;
    /* parameter vector layout: [theta (D) | alpha (D*D) | beta (D*D)] */
    double* p    = (double*)malloc(P * sizeof(double));
    double* prev = (double*)malloc(P * sizeof(double));
    double* g    = (double*)malloc(P * sizeof(double));
    double* m    = (double*)calloc(P, sizeof(double));
    double* v    = (double*)calloc(P, sizeof(double));
    memcpy(p, theta, D * sizeof(double));
    memcpy(p + D, alpha, DD * sizeof(double));
    memcpy(p + D + DD, beta, DD * sizeof(double));
    double (*ll)(int, int64_t, const double*, const int32_t*, double, const double*, const double*,
                 const double*, double*, double*, double*, double*) =
        cfg->use_def ? oracle_loglik_def : oracle_loglik_rec;

    int status = 0, have_prev = 0, have_lnl = 0, stall = 0, halv = 0;
    double lr_w = cfg->lr, lnl_prev = 0.0;
    double scale = (cfg->loss_mean && n > 0) ? 1.0 / (double)n : 1.0;
    int64_t s = 0;
    int32_t it = 0;
    while (it < cfg->max_iters) {
        double lnl = ll(D, n, t, mark, T, p, p + D, p + D + DD, g, g + D, g + D + DD, NULL);
        if (!isfinite(lnl) || !all_finite(g, P)) {
            status |= OR_NONFINITE;
            if (!have_prev || halv >= cfg->max_halvings) {
                if (have_prev) memcpy(p, prev, P * sizeof(double));
                status |= OR_DIVERGED;
                break;
            }
            memcpy(p, prev, P * sizeof(double));
            lr_w *= 0.5; halv++; it++;
            continue;
        }
        if (trace) trace[it] = lnl;
        if (cfg->tol_rel > 0.0 && have_lnl) {
            double thr = cfg->tol_rel * fmax(fabs(lnl_prev), 1.0);
            stall = (fabs(lnl - lnl_prev) <= thr) ? stall + 1 : 0;
            if (stall >= cfg->patience) { status |= OR_CONVERGED; break; }
        }
        lnl_prev = lnl; have_lnl = 1;
        memcpy(prev, p, P * sizeof(double)); have_prev = 1;
        s++;
        double bc1 = 1.0 - pow(cfg->b1, (double)s), bc2 = 1.0 - pow(cfg->b2, (double)s);
        for (size_t q = 0; q < P; q++) {
            uint32_t grp = q < (size_t)D ? 1u : (q < (size_t)D + DD ? 2u : 4u);
            if (!(cfg->fit_mask & grp)) continue;
            double gl = -g[q] * scale;                    /* gradient of the loss */
            if (cfg->optimizer == 0) {
                p[q] -= lr_w * gl;
            } else {
                m[q] = cfg->b1 * m[q] + (1.0 - cfg->b1) * gl;
                v[q] = cfg->b2 * v[q] + (1.0 - cfg->b2) * gl * gl;
                double denom = sqrt(v[q]) / sqrt(bc2) + cfg->eps;
                p[q] -= (lr_w / bc1) * m[q] / denom;
            }
            double lo = (grp == 2u) ? 0.0 : cfg->min_param;
            if (p[q] < lo) p[q] = lo;
        }
        it++;
    }
    double lnl_fin = ll(D, n, t, mark, T, p, p + D, p + D + DD, NULL, NULL, NULL, NULL);
    memcpy(theta, p, D * sizeof(double));
    memcpy(alpha, p + D, DD * sizeof(double));
    memcpy(beta, p + D + DD, DD * sizeof(double));
    *lnl_out = lnl_fin;
    *iters_out = it;
    free(p); free(prev); free(g); free(m); free(v);
    return status;
}

/* -------------------------------------------------------------------------------------
 * Batches over windows (CSR: events of window w are [win_off[w], win_off[w+1]) ), on a
 * pthread pool of `nthreads` threads with a shared atomic window counter.
 * Parameter arrays are [W][D], [W][D*D], [W][D*D].
 * ------------------------------------------------------------------------------------- */
typedef struct {
    int kind;            /* 0 = loglik (rec), 1 = loglik (def), 2 = fit */
    int D; int64_t W;
    const double* t; const int32_t* mark; const int64_t* off; const double* T;
    double *theta, *alpha, *beta;
    double *lnl, *g_theta, *g_alpha, *g_beta;
    const oracle_fit_cfg* cfg; int32_t* iters; int32_t* status;
    int64_t next;
    pthread_mutex_t mu;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* J = (batch_job*)arg;
    size_t D = (size_t)J->D, DD = D * D;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t w = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (w >= J->W) break;
        int64_t a = J->off[w], n = J->off[w + 1] - a;
        const double* tw = J->t + a; const int32_t* mw = J->mark + a;
        if (J->kind == 2) {
            J->status[w] = oracle_fit(J->D, n, tw, mw, J->T[w], J->cfg, J->theta + w * D,
                                      J->alpha + w * DD, J->beta + w * DD, J->lnl + w,
                                      J->iters + w, NULL);
        } else {
            double (*ll)(int, int64_t, const double*, const int32_t*, double, const double*,
                         const double*, const double*, double*, double*, double*, double*) =
                J->kind == 1 ? oracle_loglik_def : oracle_loglik_rec;
            J->lnl[w] = ll(J->D, n, tw, mw, J->T[w], J->theta + w * D, J->alpha + w * DD,
                           J->beta + w * DD, J->g_theta ? J->g_theta + w * D : NULL,
                           J->g_alpha ? J->g_alpha + w * DD : NULL,
                           J->g_beta ? J->g_beta + w * DD : NULL, NULL);
        }
    }
    return NULL;
}

static void run_batch(batch_job* J, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    pthread_mutex_init(&J->mu, NULL);
    J->next = 0;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int k = 0; k < nthreads; k++) pthread_create(&th[k], NULL, batch_worker, J);
    for (int k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    free(th);
    pthread_mutex_destroy(&J->mu);
}

void oracle_loglik_batch(int use_def, int D, int64_t W, const double* t, const int32_t* mark,
                         const int64_t* win_off, const double* T, const double* theta,
                         const double* alpha, const double* beta, double* lnl,
                         double* g_theta, double* g_alpha, double* g_beta, int nthreads)
{
    batch_job J;
    memset(&J, 0, sizeof(J));
    J.kind = use_def ? 1 : 0; J.D = D; J.W = W; J.t = t; J.mark = mark; J.off = win_off; J.T = T;
    J.theta = (double*)theta; J.alpha = (double*)alpha; J.beta = (double*)beta;
    J.lnl = lnl; J.g_theta = g_theta; J.g_alpha = g_alpha; J.g_beta = g_beta;
    run_batch(&J, nthreads);
}

void oracle_fit_batch(int D, int64_t W, const double* t, const int32_t* mark,
                      const int64_t* win_off, const double* T, const oracle_fit_cfg* cfg,
                      double* theta, double* alpha, double* beta, double* lnl,
                      int32_t* iters, int32_t* status, int nthreads)
{
    batch_job J;
    memset(&J, 0, sizeof(J));
    J.kind = 2; J.D = D; J.W = W; J.t = t; J.mark = mark; J.off = win_off; J.T = T;
    J.theta = theta; J.alpha = alpha; J.beta = beta; J.lnl = lnl;
    J.cfg = cfg; J.iters = iters; J.status = status;
    run_batch(&J, nthreads);
}

/* ---- Eq.(7) third line: hks^t = tanh(A alpha^x - B (beta^x T_span^x) + C theta^x).
 * alpha^x, beta^x are the window's D*D matrices flattened row-major (index i*D+j), the product
 * beta^x T_span^x entrywise (SPEC S:366-374 reading), theta^x the D baselines.  A, B are
 * H x D*D and C is H x D, row-major.  hks is W x H.  gross (optional, W x H) receives
 * sum_k |W_hk X_wk| of the pre-activation, the scale of its rounding error on other hardware. */
void oracle_hawkes_features(int D, int64_t W, int H, const double* theta, const double* alpha,
                            const double* beta, const double* T_span, const double* A,
                            const double* B, const double* C, double* hks, double* gross)
{
    const int DD = D * D;
    for (int64_t w = 0; w < W; w++) {
        const double* al = alpha + w * DD;
        const double* be = beta + w * DD;
        const double* th = theta + w * D;
        for (int h = 0; h < H; h++) {
            double z = 0.0, g = 0.0;
            for (int k = 0; k < DD; k++) {
                z += A[(int64_t)h * DD + k] * al[k];
                g += fabs(A[(int64_t)h * DD + k] * al[k]);
            }
            for (int k = 0; k < DD; k++) {
                z -= B[(int64_t)h * DD + k] * (be[k] * T_span[w]);
                g += fabs(B[(int64_t)h * DD + k] * (be[k] * T_span[w]));
            }
            for (int j = 0; j < D; j++) {
                z += C[(int64_t)h * D + j] * th[j];
                g += fabs(C[(int64_t)h * D + j] * th[j]);
            }
            hks[w * H + h] = tanh(z);
            if (gross) gross[w * H + h] = g;
        }
    }
}
