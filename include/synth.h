/*
 * synth.h — C ABI of libmdhp_synth.so: seeded synthetic MDHP event streams on the GPU.
 *
 * INPUT SYNTHESIS ONLY.  Neither the oracle nor the hot path (libmdhp.so) uses this library;
 * tests and bench.py call it to make inputs of the shapes of BASELINE.json's configs.  It
 * simulates the Eq.(2) intensity by Ogata thinning: propose at the
 * total intensity just after the last event (non-increasing between events since alpha >= 0),
 * decay every pair state by the gap, accept dimension i with probability lambda_i / bound.
 * Randomness is Philox4x32-10 keyed by (seed, global window index), so a window's events do
 * not depend on how windows are batched or sharded.
 *
 * All pointers are device pointers; `stream` is a cudaStream_t passed as void*.  Returns 0 on
 * success, -1 on bad arguments, -5 on a CUDA error (message via synth_last_error()).
 */
#ifndef MDHP_SYNTH_H_
#define MDHP_SYNTH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Parameter recipe: per-ID stationary rates r_i log-uniform in
 * [rate_lo, rate_hi] scaled to total_rate; branching G = alpha/beta with G_ii ~ U(g_self) and
 * k_cross entries per row ~ U(g_cross); attack windows (probability attack_frac; STEIA9 keeps
 * normal/attack balanced) set G_aa = 0.7 and one G_ab = 0.2 on n_attack IDs; the max
 * row sum of G is rescaled to <= rho (rho_attack in attack windows), a bound on the spectral
 * radius; beta_ij log-uniform in [beta_lo, beta_hi]; alpha = G * beta; theta = max((I-G) r, 0.05 r). */
typedef struct {
    double total_rate, rate_lo, rate_hi, beta_lo, beta_hi;
    double g_self_lo, g_self_hi, g_cross_lo, g_cross_hi;
    double rho, attack_frac, rho_attack;
    int32_t k_cross, n_attack;
} synth_recipe;

/* theta [W][D], alpha [W][D][D], beta [W][D][D] fp32 out (row i = target, col j = source);
 * attack [W] uint8 out (may be NULL).  Windows are first_window .. first_window + W - 1.   */
int synth_params(int32_t D, int64_t W, int64_t first_window, uint64_t seed,
                 const synth_recipe* rc, float* theta, float* alpha, float* beta,
                 uint8_t* attack, void* stream);

/* Ogata thinning on [0, T] with empty history.  Two passes with identical random streams:
 *   count pass  (win_off == NULL): counts[w] = number of events of window w
 *   write pass  (win_off != NULL): events of window w written to t_out/mark_out starting at
 *               win_off[w] (must equal the exclusive prefix sum of the count pass)
 * max_events caps a window (status: counts[w] = -1 if exceeded).                           */
int synth_ogata(int32_t D, int64_t W, int64_t first_window, uint64_t seed, double T,
                const float* theta, const float* alpha, const float* beta, int64_t max_events,
                const int64_t* win_off, int64_t* counts, double* t_out, int32_t* mark_out,
                void* stream);

/* Time-exciting injection strategies (Table II): attack-rate shapes g(u) on the
 * normalised window u = t/T in [0,1]; constants in DESIGN.md R23.                   */
#define SYNTH_NONE 0
#define SYNTH_PLA  1   /* power-law acceleration   g = a u^b                                  */
#define SYNTH_DEA  2   /* delayed escalation       W1 a1 u^(a1-1) | W2 a2 e^{gamma (u - t1)}   */
#define SYNTH_ASA  3   /* adaptive stealth         C e^{gamma u} / (1 + e^{gamma (u - t0)})^2  */
#define SYNTH_DAM  4   /* multi-strategy           w a1 u^(a1-1) + (1 - w) a2 e^{a2 u}         */

/* synth_ogata plus injections: in every window with attack[w] != 0, an independent
 * Algorithm-4 (NPP) stream — candidate gaps Exponential(mean 1/inj_rate) in u,
 * accepted with probability g(u)/g_max — is superposed on the Hawkes events, all on one ID
 * drawn uniformly per window; the Hawkes part is the same stream synth_ogata produces.
 * strategy SYNTH_NONE ignores attack (then it equals synth_ogata).                          */
int synth_ogata_inject(int32_t D, int64_t W, int64_t first_window, uint64_t seed, double T,
                       const float* theta, const float* alpha, const float* beta,
                       int64_t max_events, const int64_t* win_off, int64_t* counts,
                       double* t_out, int32_t* mark_out, const uint8_t* attack,
                       int32_t strategy, double inj_rate, void* stream);

/* The injection sampler alone (Algorithm 4 on [0,1], same stream as synth_ogata_inject):
 * count pass (win_off == NULL) -> counts[w]; write pass -> normalised times u_out.        */
int synth_npp(int64_t W, int64_t first_window, uint64_t seed, int32_t strategy, double rate,
              const int64_t* win_off, int64_t* counts, double* u_out, void* stream);

const char* synth_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MDHP_SYNTH_H_ */
