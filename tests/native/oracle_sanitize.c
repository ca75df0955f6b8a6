/* Host sanitizer driver for the oracle (ASan/UBSan on the host code).
 * Compiled together with oracle/oracle.c under -fsanitize=address,undefined by
 * tests/test_oracle_sanitizers.py; exercises every exported oracle function on small inputs,
 * including empty windows, ties, the EQ6 time mode, both optimizers, rollback and the pthread
 * batch paths.  Exit code 0 = no sanitizer report (the sanitizers abort on the first error). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t max_iters, optimizer;
    double lr, b1, b2, eps;
    int32_t loss_mean;
    double tol_rel;
    int32_t patience;
    double min_param;
    uint32_t fit_mask;
    int32_t max_halvings, use_def;
} cfg_t;

int oracle_convert_window(int D, int time_mode, double lo, double hi, int tie_policy, int64_t n,
                          const double* t, const int32_t* mark, double T, float* t32, float* T32);
double oracle_loglik_def(int D, int64_t n, const double* t, const int32_t* mark, double T,
                         const double* th, const double* al, const double* be, double* gt,
                         double* ga, double* gb, double* gamma);
double oracle_loglik_rec(int D, int64_t n, const double* t, const int32_t* mark, double T,
                         const double* th, const double* al, const double* be, double* gt,
                         double* ga, double* gb, double* gamma);
int oracle_fit(int D, int64_t n, const double* t, const int32_t* mark, double T, const cfg_t* cfg,
               double* th, double* al, double* be, double* lnl, int32_t* iters, double* trace);
void oracle_loglik_batch(int use_def, int D, int64_t W, const double* t, const int32_t* mark,
                         const int64_t* off, const double* T, const double* th, const double* al,
                         const double* be, double* lnl, double* gt, double* ga, double* gb, int nt);
void oracle_fit_batch(int D, int64_t W, const double* t, const int32_t* mark, const int64_t* off,
                      const double* T, const cfg_t* cfg, double* th, double* al, double* be,
                      double* lnl, int32_t* iters, int32_t* status, int nt);
void oracle_hawkes_features(int D, int64_t W, int H, const double* th, const double* al,
                            const double* be, const double* T, const double* A, const double* B,
                            const double* C, double* hks, double* gross);

static double urand(uint64_t* s) {
    *s = *s * 6364136223846793005ull + 1442695040888963407ull;
    return (double)(*s >> 11) / 9007199254740992.0;
}

int main(void) {
    const int D = 3, W = 4;
    uint64_t seed = 2024;
    /* four windows: 0 events, 1 event, ties (same time, different marks), 40 random events */
    int64_t off[5] = {0, 0, 1, 4, 44};
    double t[44];
    int32_t m[44];
    t[0] = 0.5; m[0] = 2;
    t[1] = 0.25; m[1] = 0; t[2] = 0.25; m[2] = 1; t[3] = 0.75; m[3] = 0;
    double acc = 0.0;
    for (int k = 4; k < 44; k++) {
        acc += 0.02 * urand(&seed);
        t[k] = acc;
        m[k] = (int32_t)(urand(&seed) * D) % D;
    }
    double T[4] = {1.0, 1.0, 1.0, 1.0};
    double th[4 * 3], al[4 * 9], be[4 * 9];
    for (int k = 0; k < 4 * 3; k++) th[k] = 0.5 + urand(&seed);
    for (int k = 0; k < 4 * 9; k++) { al[k] = 0.3 * urand(&seed); be[k] = 1.0 + 3.0 * urand(&seed); }

    /* conversion in every time mode and tie policy */
    float t32[44], T32;
    for (int mode = 0; mode < 3; mode++)
        for (int tie = 0; tie < 2; tie++)
            for (int w = 0; w < W; w++) {
                int64_t a = off[w], n = off[w + 1] - off[w];
                oracle_convert_window(D, mode, 0.0, 1.0, tie, n, t + a, m + a, T[w], t32, &T32);
            }
    /* likelihood + gradients, both routes, with and without gradient outputs */
    double gt[3], ga[9], gb[9], gamma;
    for (int w = 0; w < W; w++) {
        int64_t a = off[w], n = off[w + 1] - off[w];
        double l1 = oracle_loglik_def(D, n, t + a, m + a, T[w], th + 3 * w, al + 9 * w, be + 9 * w,
                                      gt, ga, gb, &gamma);
        double l2 = oracle_loglik_rec(D, n, t + a, m + a, T[w], th + 3 * w, al + 9 * w, be + 9 * w,
                                      gt, ga, gb, &gamma);
        double l3 = oracle_loglik_rec(D, n, t + a, m + a, T[w], th + 3 * w, al + 9 * w, be + 9 * w,
                                      NULL, NULL, NULL, NULL);
        if (!(fabs(l1 - l2) <= 1e-9 * fabs(l1) + 1e-12) || l2 != l3) {
            fprintf(stderr, "window %d: def %.17g rec %.17g\n", w, l1, l2);
            return 2;
        }
    }
    /* fits: GD (mean loss) and Adam with a trace; a huge lr to force rollback/halving */
    cfg_t c = {30, 0, 0.2, 0.9, 0.999, 1e-8, 1, 0.0, 10, 1e-4, 7u, 8, 0};
    double trace[64];
    for (int opt = 0; opt < 2; opt++)
        for (int w = 0; w < W; w++) {
            int64_t a = off[w], n = off[w + 1] - off[w];
            double pt[3], pa[9], pb[9], lnl;
            int32_t it;
            memcpy(pt, th + 3 * w, sizeof pt); memcpy(pa, al + 9 * w, sizeof pa);
            memcpy(pb, be + 9 * w, sizeof pb);
            c.optimizer = opt;
            c.lr = opt ? 0.05 : 0.2;
            oracle_fit(D, n, t + a, m + a, T[w], &c, pt, pa, pb, &lnl, &it, trace);
        }
    c.optimizer = 0; c.lr = 1e6; c.loss_mean = 0;
    {
        double pt[3], pa[9], pb[9], lnl;
        int32_t it;
        memcpy(pt, th + 9, sizeof pt); memcpy(pa, al + 27, sizeof pa); memcpy(pb, be + 27, sizeof pb);
        oracle_fit(D, 40, t + 4, m + 4, 1.0, &c, pt, pa, pb, &lnl, &it, NULL);
    }
    /* batch paths on a pthread pool */
    double lnl[4], bgt[12], bga[36], bgb[36];
    oracle_loglik_batch(0, D, W, t, m, off, T, th, al, be, lnl, bgt, bga, bgb, 3);
    oracle_loglik_batch(1, D, W, t, m, off, T, th, al, be, lnl, NULL, NULL, NULL, 2);
    int32_t iters[4], status[4];
    c.lr = 0.05; c.optimizer = 1; c.max_iters = 10;
    double bth[12], bal[36], bbe[36];
    memcpy(bth, th, sizeof bth); memcpy(bal, al, sizeof bal); memcpy(bbe, be, sizeof bbe);
    oracle_fit_batch(D, W, t, m, off, T, &c, bth, bal, bbe, lnl, iters, status, 4);
    /* Hawkes-gate features */
    const int H = 5;
    double A[5 * 9], B[5 * 9], C[5 * 3], hks[4 * 5], gross[4 * 5];
    for (int k = 0; k < 45; k++) { A[k] = urand(&seed) - 0.5; B[k] = urand(&seed) - 0.5; }
    for (int k = 0; k < 15; k++) C[k] = urand(&seed) - 0.5;
    oracle_hawkes_features(D, W, H, th, al, be, T, A, B, C, hks, gross);
    oracle_hawkes_features(D, W, H, th, al, be, T, A, B, C, hks, NULL);
    printf("oracle sanitizer run ok\n");
    return 0;
}
