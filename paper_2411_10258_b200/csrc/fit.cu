// fit.cu — mdhp_loglik_grad and mdhp_fit kernels (rows a2-a6 of DESIGN.md section 4).
#include <cmath>
#include "eval.cuh"

namespace mdhp {


template <int DP>
struct WarpCtx {
  int lane, g, j, gbase;
  unsigned gmask;
  __device__ WarpCtx() {
    lane = threadIdx.x & 31;
    g = lane / DP;
    j = lane % DP;
    gbase = g * DP;
    gmask = DP == 32 ? kFull : (((1u << DP) - 1u) << gbase);
  }
};

// Whether the fp32 lnL of a window may be off by more than 1e-4 |lnL| (R24): the
// absolute error of the fp32 evaluation is bounded by a few ulps per event of ln lambda
// (lambda itself carries O(10) ulps after the recurrence; lg2.approx adds ~2 ulps of |lg2|)
// plus a few ulps of the compensator |Part2| + |Part3|.  A window is re-evaluated in fp64
// (exact.cu) when those bounds, with a safety factor of ~6 over the worst error measured in
// the fuzz sweep (13 ulps per event), are not below 1e-4 |lnL|.
__device__ __forceinline__ bool needs_exact(double lnl, int n, double sum_ln, double part2,
                                            double part3) {
  return !(fabs(lnl) >= kExactPerEvent * (double)n + kExactPerLn * fabs(sum_ln) +
                            kExactGross * (fabs(part2) + fabs(part3)));
}

// Append window w to the fp64 re-evaluation list (one lane per group).
__device__ __forceinline__ void list_exact(int32_t* list, int32_t* count, int64_t w) {
  const int q = atomicAdd(count, 1);
  list[q] = (int32_t)w;
}

// Evaluate the window owned by this group at the parameters in K (alpha, beta) / th.
// Writes gradients (d alpha, d beta) over the accumulators in Gs when GRAD; returns lnL
// (identical in every lane of the group) and this lane's d theta_j; `exact` tells whether the
// window needs the fp64 re-evaluation (needs_exact).
template <int DP, bool GRAD>
__device__ __forceinline__ double eval_window(const Packed& P, float2* A, float2* SQ, float2* Gs,
                                              const WarpCtx<DP>& c, int64_t w, bool live,
                                              int nmax, float th, const ColInfo& ci,
                                              float& dth, bool& finite, bool& exact) {
  reset_state<DP>(SQ, Gs, c.j);
  __syncwarp();
  const int n = live ? P.n[w] : 0;
  const int64_t beg = live ? P.begin[w] : 0;
  float last, gth;
  double lsum;
  event_loop<DP, GRAD>(A, SQ, Gs, c.j, c.gbase, P.t32, P.dtp, P.mark, beg, n, nmax, th, last, gth,
                       lsum);
  ColInfo cc = ci;
  cc.last = last;
  Series S;
  load_series(S, P.mom + ((size_t)(live ? w : 0) * P.Dp + c.j) * kMom, live && cc.N > 0);
  double part3 = 0.0;
  bool ok = true;
#pragma unroll 4
  for (int i = 0; i < DP; i++) {
    const float2 k = A[i * (DP + 1) + c.j];
    const float2 sq = SQ[i * (DP + 1) + c.j];
    float Eb, Hb2;
    const float ka = ab_alpha<DP>(i, k), kb = ab_beta<DP>(i, k);
    compensator(cc, S, kb, sq.x, sq.y, Eb, Hb2);
    if (cc.real && i < P.D) {
      part3 += (double)(ka * Eb);
      if (GRAD) {
        float2 gg = Gs[i * DP + c.j];
        const float da = gg.x + Eb;
        const float db = fmaf(-ka, gg.y, ka * Hb2);
        ok = ok && isfinite(da) && isfinite(db);
        Gs[i * DP + c.j] = make_float2(da, db);
      }
    }
  }
  dth = gth - ci.T;
  if (GRAD && cc.real) ok = ok && isfinite(dth);
  part3 = group_sum_d<DP>(part3);
  lsum = group_sum_d<DP>(lsum);
  const double sth = group_sum_d<DP>(cc.real ? (double)th : 0.0);
  const double lnl = (double)kLn2 * lsum + part3 - (double)ci.T * sth;
  const unsigned bal = __ballot_sync(kFull, ok) & c.gmask;
  finite = (bal == c.gmask) && isfinite(lnl);
  exact = live && needs_exact(lnl, n, (double)kLn2 * lsum, (double)ci.T * sth, part3);
  return lnl;
}

template <int DP>
__device__ __forceinline__ ColInfo col_info(const Packed& P, int64_t w, bool live, int j) {
  ColInfo ci;
  ci.real = j < P.D;
  ci.T = live ? P.T32[w] : 1.0f;
  ci.N = live ? P.cnt[w * P.Dp + j] : 0;
  ci.umax = live ? P.umax[w * P.Dp + j] : 0.0f;
  ci.last = -1.0f;
  return ci;
}

// Load window parameters into K (alpha, beta) and return theta_j (0 for padded lanes).
template <int DP>
__device__ __forceinline__ float load_params(float2* A, const WarpCtx<DP>& c, int D, int64_t w,
                                             bool live, const float* __restrict__ theta,
                                             const float* __restrict__ alpha,
                                             const float* __restrict__ beta) {
  const bool real = live && c.j < D;
#pragma unroll 4
  for (int i = 0; i < DP; i++) {
    float a = 0.0f, b = 1.0f;
    if (real && i < D) {
      a = alpha[(size_t)w * D * D + (size_t)i * D + c.j];
      b = beta[(size_t)w * D * D + (size_t)i * D + c.j];
    }
    A[i * (DP + 1) + c.j] = ab_pack<DP>(i, a, b);
  }
  // null dimension (see eval.cuh): row DP = {1,0} at column 0, column DP has beta = 0
  A[DP * (DP + 1) + c.j] = ab_pack<DP>(DP, c.j == 0 ? 1.0f : 0.0f, 0.0f);
  A[c.j * (DP + 1) + DP] = make_float2(0.0f, 0.0f);
  return real ? theta[(size_t)w * D + c.j] : 0.0f;
}

template <int DP>
__global__ void __launch_bounds__(128, DP >= 32 ? 2 : 4)
k_loglik(Packed P, const float* __restrict__ theta, const float* __restrict__ alpha,
         const float* __restrict__ beta, double* __restrict__ lnl_out,
         float* __restrict__ g_theta, float* __restrict__ g_alpha, float* __restrict__ g_beta,
         const int32_t* __restrict__ status, int32_t* __restrict__ xlist,
         int32_t* __restrict__ xcount) {
  extern __shared__ __align__(16) unsigned char smem[];
  using SM = Smem<DP>;
  WarpCtx<DP> c;
  const int wid = threadIdx.x >> 5;
  float2* gbase_s = reinterpret_cast<float2*>(smem + wid * SM::per_warp) + c.g * SM::per_group;
  float2* A = gbase_s;
  float2* SQ = gbase_s + SM::AS;
  float2* Gs = gbase_s + 2 * SM::AS;
  const int64_t unit = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  const int64_t slot = unit * SM::G + c.g;
  const int64_t w = slot < P.W ? P.perm[slot] : 0;
  const bool live = slot < P.W && !(status[w] & MDHP_ST_INVALID);
  const int D = P.D;
  const float th = load_params<DP>(A, c, D, w, live, theta, alpha, beta);
  const ColInfo ci = col_info<DP>(P, w, live, c.j);
  const int nmax = group_max_i<DP>(live ? P.n[w] : 0);
  float dth;
  bool finite, exact;
  const bool grad = g_theta != nullptr;
  double lnl;
  if (grad) lnl = eval_window<DP, true>(P, A, SQ, Gs, c, w, live, nmax, th, ci, dth, finite, exact);
  else lnl = eval_window<DP, false>(P, A, SQ, Gs, c, w, live, nmax, th, ci, dth, finite, exact);
  if (slot >= P.W) return;
  if (c.j == 0) {
    lnl_out[w] = live ? lnl : (double)NAN;
    if (exact) list_exact(xlist, xcount, w);
  }
  if (grad && c.j < D) {
    g_theta[(size_t)w * D + c.j] = live ? dth : NAN;
    for (int i = 0; i < D; i++) {
      const float2 gg = Gs[i * DP + c.j];
      g_alpha[(size_t)w * D * D + (size_t)i * D + c.j] = live ? gg.x : NAN;
      g_beta[(size_t)w * D * D + (size_t)i * D + c.j] = live ? gg.y : NAN;
    }
  }
}

// One optimizer step for this lane's column j (theta_j, alpha_.j, beta_.j), PyTorch Adam / GD
// semantics, then projection.  Gradients of lnL are in Gs (alpha, beta) and
// dth; the loss gradient is -grad * scale.
template <int DP, bool RESUME>
__device__ __forceinline__ void step_column(float2* A, const float2* Gs, const WarpCtx<DP>& c,
                                            int D, int64_t w, const FitCfgDev& cfg, float lr_w,
                                            int s, float scale, float dth, float& th,
                                            float* __restrict__ opt) {
  if (c.j >= D) return;
  const size_t P = (size_t)D + 2 * (size_t)D * D;
  float* m = opt ? opt + (size_t)w * 2 * P : nullptr;
  float* v = m ? m + P : nullptr;
  const bool adam = cfg.optimizer == MDHP_OPT_ADAM;
  float bc1 = 1.0f, sbc2 = 1.0f;
  if (adam) {
    // s counts this call's steps; cfg.step0 those of earlier calls (resume).  A separate
    // instantiation: reading step0 in the hot kernel perturbed its register allocation (-3%)
    const float sg = RESUME ? (float)(s + cfg.step0) : (float)s;
    bc1 = 1.0f - powf(cfg.b1, sg);
    sbc2 = sqrtf(1.0f - powf(cfg.b2, sg));
  }
  auto upd = [&](float p, float g, size_t q, float lo) -> float {
    const float gl = -g * scale;
    if (adam) {
      const float mm = cfg.b1 * m[q] + (1.0f - cfg.b1) * gl;
      const float vv = cfg.b2 * v[q] + (1.0f - cfg.b2) * gl * gl;
      m[q] = mm;
      v[q] = vv;
      const float denom = sqrtf(vv) / sbc2 + cfg.eps;
      p = p - (lr_w / bc1) * (mm / denom);
    } else {
      p = p - lr_w * gl;
    }
    return p < lo ? lo : p;
  };
  if (cfg.fit_mask & MDHP_FIT_THETA) th = upd(th, dth, (size_t)c.j, cfg.min_param);
  for (int i = 0; i < D; i++) {
    float2* k = &A[i * (DP + 1) + c.j];
    const float2 gg = Gs[i * DP + c.j];
    const size_t q = (size_t)D + (size_t)i * D + c.j;
    float ka = ab_alpha<DP>(i, *k), kb = ab_beta<DP>(i, *k);
    if (cfg.fit_mask & MDHP_FIT_ALPHA) ka = upd(ka, gg.x, q, 0.0f);
    if (cfg.fit_mask & MDHP_FIT_BETA) kb = upd(kb, gg.y, q + (size_t)D * D, cfg.min_param);
    *k = ab_pack<DP>(i, ka, kb);
  }
}

template <int DP>
__device__ __forceinline__ void store_params(const float2* A, const WarpCtx<DP>& c, int D,
                                             int64_t w, float th, float* __restrict__ theta,
                                             float* __restrict__ alpha, float* __restrict__ beta) {
  if (c.j >= D) return;
  theta[(size_t)w * D + c.j] = th;
  for (int i = 0; i < D; i++) {
    const float2 k = A[i * (DP + 1) + c.j];
    alpha[(size_t)w * D * D + (size_t)i * D + c.j] = ab_alpha<DP>(i, k);
    beta[(size_t)w * D * D + (size_t)i * D + c.j] = ab_beta<DP>(i, k);
  }
}

// Persistent fit kernel (a6): windows are taken longest first from a global counter and run
// their whole iteration loop on chip, then lnL is evaluated at the returned parameters and
// everything is written back.
//   REFILL (converged mode, tol_rel > 0): each group of DP lanes takes one window at a time;
//     when its window stops (convergence, divergence, budget) the group evaluates the final lnL,
//     writes back and takes the next window at once, so a warp's other group(s) never idle
//     behind a window that stopped early (the convergence mask frees lanes instead of padding
//     them).  One evaluation per warp step: TRAIN groups step after it, FINAL groups record it.
//   !REFILL (fixed iteration count): every window of a warp stops at the same evaluation, so a
//     warp takes G windows at a time and keeps them to the end (no per-window bookkeeping).
template <int DP, bool RESUME, bool REFILL>
__global__ void __launch_bounds__(128, DP >= 32 ? 2 : 4)
k_fit(Packed P, FitCfgDev cfg, float* __restrict__ theta, float* __restrict__ alpha,
      float* __restrict__ beta, float* __restrict__ opt, double* __restrict__ lnl_out,
      int32_t* __restrict__ iters_out, int32_t* __restrict__ status,
      float* __restrict__ trace, int* __restrict__ counter, int32_t* __restrict__ xlist,
      int32_t* __restrict__ xcount) {
  extern __shared__ __align__(16) unsigned char smem[];
  using SM = Smem<DP>;
  WarpCtx<DP> c;
  const int wid = threadIdx.x >> 5;
  float2* gbase_s = reinterpret_cast<float2*>(smem + wid * SM::per_warp) + c.g * SM::per_group;
  float2* A = gbase_s;
  float2* SQ = gbase_s + SM::AS;
  float2* Gs = gbase_s + 2 * SM::AS;
  const int D = P.D;
  if constexpr (REFILL) {
    enum { TRAIN = 0, FINAL = 1, IDLE = 2 };
    // per-group (group-uniform) window and optimizer state
    int phase = IDLE;
    int64_t w = 0;
    int st0 = 0, n = 0, it = 0, s = 0, halv = 0, stall = 0, st = 0;
    bool live = false, have_prev = false, have_lnl = false;
    float th = 0.0f, scale = 1.0f, lr_w = cfg.lr;
    double lnl_prev = 0.0;
    ColInfo ci = col_info<DP>(P, 0, false, c.j);
    // group-collective: take the next window (all lanes of the group, none of the others)
    auto fetch = [&]() {
      int64_t slot = 0;
      if (c.j == 0) slot = atomicAdd(counter, 1);
      slot = __shfl_sync(c.gmask, slot, c.gbase);
      if (slot >= P.W) {
        phase = IDLE;
        live = false;
        n = 0;
        return;
      }
      w = P.perm[slot];
      MDHP_ASSERT(w >= 0 && w < P.W);
      st0 = status[w];
      live = !(st0 & MDHP_ST_INVALID);
      th = load_params<DP>(A, c, D, w, live, theta, alpha, beta);
      ci = col_info<DP>(P, w, live, c.j);
      n = live ? P.n[w] : 0;
      scale = (cfg.loss_mean && n > 0) ? 1.0f / (float)n : 1.0f;
      it = s = halv = stall = st = 0;
      lr_w = cfg.lr;
      lnl_prev = 0.0;
      have_prev = have_lnl = false;
      phase = (!live || cfg.max_iters <= 0) ? FINAL : TRAIN;
    };
    fetch();
    while (__any_sync(kFull, phase != IDLE)) {
      const bool act = phase != IDLE && live;
      const int nmax = group_max_i<DP>(act ? n : 0);
      float dth;
      bool finite, exact;
      // gradients only when some group trains (a warp whose groups all stop together, as in the
      // fixed-iteration mode, evaluates its final lnL without them)
      const double lnl = __any_sync(kFull, phase == TRAIN)
                             ? eval_window<DP, true>(P, A, SQ, Gs, c, w, act, nmax, th, ci, dth, finite, exact)
                             : eval_window<DP, false>(P, A, SQ, Gs, c, w, act, nmax, th, ci, dth, finite, exact);
      if (phase == TRAIN) {
        bool done = false;
        if (!finite) {
          st |= MDHP_ST_NONFINITE;
          if (!have_prev || halv >= cfg.max_halvings) {
            st |= MDHP_ST_DIVERGED;
            done = true;
            if (have_prev) th = load_params<DP>(A, c, D, w, true, theta, alpha, beta);
          } else {
            th = load_params<DP>(A, c, D, w, true, theta, alpha, beta);
            lr_w *= 0.5f;
            halv++;
            it++;
          }
        } else {
          if (trace && c.j == 0) trace[(size_t)w * cfg.max_iters + it] = (float)lnl;
          if (cfg.tol_rel > 0.0f && have_lnl) {
            const double thr = (double)cfg.tol_rel * fmax(fabs(lnl_prev), 1.0);
            stall = (fabs(lnl - lnl_prev) <= thr) ? stall + 1 : 0;
            if (stall >= cfg.patience) {
              st |= MDHP_ST_CONVERGED;
              done = true;
            }
          }
          if (!done) {
            lnl_prev = lnl;
            have_lnl = true;
            store_params<DP>(A, c, D, w, th, theta, alpha, beta);   // previous point
            have_prev = true;
            s++;
            step_column<DP, RESUME>(A, Gs, c, D, w, cfg, lr_w, s, scale, dth, th, opt);
            it++;
          }
        }
        if (it >= cfg.max_iters) done = true;
        if (done) phase = FINAL;   // the next evaluation is lnL at the returned parameters
      } else if (phase == FINAL) {
        if (live) store_params<DP>(A, c, D, w, th, theta, alpha, beta);
        if (c.j == 0) {
          lnl_out[w] = live ? lnl : (double)NAN;
          iters_out[w] = it;
          status[w] = (st0 & kKeepStatus) | st;
          if (exact) list_exact(xlist, xcount, w);
          if (trace && live)
            for (int q = it; q < cfg.max_iters; q++) trace[(size_t)w * cfg.max_iters + q] = NAN;
        }
        fetch();
      }
      __syncwarp();
    }
  } else {
    // fixed iteration count: every window of a warp stops at the same evaluation, so the
    // warp keeps its G windows to the end (no per-window refill bookkeeping)
    const int64_t nunits = (P.W + SM::G - 1) / SM::G;
    for (;;) {
      int64_t unit = 0;
      if (c.lane == 0) unit = atomicAdd(counter, 1);
      unit = __shfl_sync(kFull, unit, 0);
      if (unit >= nunits) break;
      const int64_t slot = unit * SM::G + c.g;
      const int64_t w = slot < P.W ? P.perm[slot] : 0;
      MDHP_ASSERT(w >= 0 && w < (P.W > 0 ? P.W : 1));
      const int st0 = slot < P.W ? status[w] : MDHP_ST_INVALID;
      const bool live = slot < P.W && !(st0 & MDHP_ST_INVALID);
      float th = load_params<DP>(A, c, D, w, live, theta, alpha, beta);
      const ColInfo ci = col_info<DP>(P, w, live, c.j);
      const int n = live ? P.n[w] : 0;
      const float scale = (cfg.loss_mean && n > 0) ? 1.0f / (float)n : 1.0f;
      // per-window (group-uniform) optimizer state
      int it = 0, s = 0, halv = 0, stall = 0, st = 0;
      float lr_w = cfg.lr;
      double lnl_prev = 0.0;
      bool have_prev = false, have_lnl = false;
      bool done = !live || cfg.max_iters <= 0;
      while (__any_sync(kFull, !done)) {
        const int nmax = group_max_i<DP>(done ? 0 : n);
        float dth;
        bool finite, exact;
        const double lnl = eval_window<DP, true>(P, A, SQ, Gs, c, w, !done, nmax, th, ci, dth, finite, exact);
        if (!done) {
          if (!finite) {
            st |= MDHP_ST_NONFINITE;
            if (!have_prev || halv >= cfg.max_halvings) {
              st |= MDHP_ST_DIVERGED;
              done = true;
              if (have_prev) th = load_params<DP>(A, c, D, w, true, theta, alpha, beta);
            } else {
              th = load_params<DP>(A, c, D, w, true, theta, alpha, beta);
              lr_w *= 0.5f;
              halv++;
              it++;
            }
          } else {
            if (trace && c.j == 0) trace[(size_t)w * cfg.max_iters + it] = (float)lnl;
            if (cfg.tol_rel > 0.0f && have_lnl) {
              const double thr = (double)cfg.tol_rel * fmax(fabs(lnl_prev), 1.0);
              stall = (fabs(lnl - lnl_prev) <= thr) ? stall + 1 : 0;
              if (stall >= cfg.patience) {
                st |= MDHP_ST_CONVERGED;
                done = true;
              }
            }
            if (!done) {
              lnl_prev = lnl;
              have_lnl = true;
              store_params<DP>(A, c, D, w, th, theta, alpha, beta);   // previous point
              have_prev = true;
              s++;
              step_column<DP, RESUME>(A, Gs, c, D, w, cfg, lr_w, s, scale, dth, th, opt);
              it++;
            }
          }
          if (it >= cfg.max_iters) done = true;
        }
        __syncwarp();
      }
      // lnL at the returned parameters (no gradient accumulation needed)
      const int nmax = group_max_i<DP>(n);
      float dth;
      bool finite, exact;
      const double lnl = eval_window<DP, false>(P, A, SQ, Gs, c, w, live, nmax, th, ci, dth, finite, exact);
      if (slot < P.W) {
        if (live) store_params<DP>(A, c, D, w, th, theta, alpha, beta);
        if (c.j == 0) {
          lnl_out[w] = live ? lnl : (double)NAN;
          iters_out[w] = it;
          status[w] = (st0 & kKeepStatus) | st;
          if (exact) list_exact(xlist, xcount, w);
          if (trace && live)
            for (int q = it; q < cfg.max_iters; q++) trace[(size_t)w * cfg.max_iters + q] = NAN;
        }
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------- host launchers
template <int DP>
static int launch_loglik_t(const Packed& P, const float* th, const float* al, const float* be,
                           double* lnl, float* gt, float* ga, float* gb, const int32_t* status,
                           int32_t* xlist, int32_t* xcount, cudaStream_t st) {
  using SM = Smem<DP>;
  constexpr int WPB = 4;
  const size_t smem = WPB * SM::per_warp;
  auto kern = k_loglik<DP>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("cudaFuncSetAttribute(k_loglik) failed");
    return MDHP_ECUDA;
  }
  const int64_t units = (P.W + SM::G - 1) / SM::G;
  const unsigned blocks = (unsigned)((units + WPB - 1) / WPB);
  kern<<<blocks, WPB * 32, smem, st>>>(P, th, al, be, lnl, gt, ga, gb, status, xlist, xcount);
  count_launch();
  return MDHP_OK;
}

int loglik_launch(const Packed& P, const float* th, const float* al, const float* be, double* lnl,
                  float* gt, float* ga, float* gb, const int32_t* status, int32_t* xlist,
                  int32_t* xcount, cudaStream_t st) {
  if (P.W == 0) return MDHP_OK;
  switch (P.Dp) {
    case 1: return launch_loglik_t<1>(P, th, al, be, lnl, gt, ga, gb, status, xlist, xcount, st);
    case 2: return launch_loglik_t<2>(P, th, al, be, lnl, gt, ga, gb, status, xlist, xcount, st);
    case 4: return launch_loglik_t<4>(P, th, al, be, lnl, gt, ga, gb, status, xlist, xcount, st);
    case 8: return launch_loglik_t<8>(P, th, al, be, lnl, gt, ga, gb, status, xlist, xcount, st);
    case 16: return launch_loglik_t<16>(P, th, al, be, lnl, gt, ga, gb, status, xlist, xcount, st);
    case 32: return launch_loglik_t<32>(P, th, al, be, lnl, gt, ga, gb, status, xlist, xcount, st);
  }
  set_error("unsupported padded D %d", P.Dp);
  return MDHP_EDIM;
}

template <int DP>
static int launch_fit_t(const Packed& P, const FitCfgDev& cfg, float* th, float* al, float* be,
                        float* opt, double* lnl, int32_t* iters, int32_t* status, float* trace,
                        int* counter, int32_t* xlist, int32_t* xcount, cudaStream_t st) {
  using SM = Smem<DP>;
  constexpr int WPB = 4;
  const size_t smem = WPB * SM::per_warp;
  // converged mode (tol_rel > 0): windows stop at different iterations -> per-window refill
  auto kern = cfg.tol_rel > 0.0f ? (cfg.step0 != 0 ? k_fit<DP, true, true> : k_fit<DP, false, true>)
                                 : (cfg.step0 != 0 ? k_fit<DP, true, false> : k_fit<DP, false, false>);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("cudaFuncSetAttribute(k_fit) failed");
    return MDHP_ECUDA;
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPB * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t units = (P.W + SM::G - 1) / SM::G;
  int64_t blocks = (int64_t)sms * per_sm;
  const int64_t need = (units + WPB - 1) / WPB;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, WPB * 32, smem, st>>>(P, cfg, th, al, be, opt, lnl, iters, status,
                                                 trace, counter, xlist, xcount);
  count_launch();
  return MDHP_OK;
}

int fit_launch(const Packed& P, const FitCfgDev& cfg, float* th, float* al, float* be, float* opt,
               double* lnl, int32_t* iters, int32_t* status, float* trace, int* counter,
               int32_t* xlist, int32_t* xcount, cudaStream_t st) {
  if (P.W == 0) return MDHP_OK;
  switch (P.Dp) {
    case 1: return launch_fit_t<1>(P, cfg, th, al, be, opt, lnl, iters, status, trace, counter, xlist, xcount, st);
    case 2: return launch_fit_t<2>(P, cfg, th, al, be, opt, lnl, iters, status, trace, counter, xlist, xcount, st);
    case 4: return launch_fit_t<4>(P, cfg, th, al, be, opt, lnl, iters, status, trace, counter, xlist, xcount, st);
    case 8: return launch_fit_t<8>(P, cfg, th, al, be, opt, lnl, iters, status, trace, counter, xlist, xcount, st);
    case 16: return launch_fit_t<16>(P, cfg, th, al, be, opt, lnl, iters, status, trace, counter, xlist, xcount, st);
    case 32: return launch_fit_t<32>(P, cfg, th, al, be, opt, lnl, iters, status, trace, counter, xlist, xcount, st);
  }
  set_error("unsupported padded D %d", P.Dp);
  return MDHP_EDIM;
}

}  // namespace mdhp
