// fit.cu — mdhp_loglik_grad and mdhp_fit kernels (rows a2-a6 of DESIGN.md section 4).
#include <cmath>
#include <cstdio>
#include <cstdlib>
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
  using SM = Smem<DP>;
  reset_state<DP>(SQ, Gs, c.j);
  __syncwarp();
  const int n = live ? P.n[w] : 0;
  const int64_t beg = live ? P.begin[w] : 0;
  float last, gth;
  double lsum;
  event_loop<DP, GRAD, true>(A, SQ, Gs, c.j, c.gbase, P.t32, P.dtp, P.mark, beg, n, nmax, th, last, gth,
                       lsum);
  ColInfo cc = ci;
  cc.last = last;
  Series S;
  load_series(S, P.mom + ((size_t)(live ? w : 0) * P.Dp + c.j) * kMom, live && cc.N > 0);
  double part3 = 0.0;
  bool ok = true;
#pragma unroll 4
  for (int i = 0; i < DP; i++) {
    const float2 k = A[SM::e(i, c.j)];
    const float2 sq = SQ[SM::e(i, c.j)];
    float Eb, Hb2;
    // A holds beta' = -beta log2 e; the compensator takes beta (one rounding of beta' * -ln 2)
    const float ka = ab_alpha<DP>(i, k), kb = ab_beta<DP>(i, k) * -kLn2;
    compensator(cc, S, kb, sq.x, sq.y, Eb, Hb2);
    if (cc.real && i < P.D) {
      part3 += (double)(ka * Eb);
      if (GRAD) {
        float2 gg = gsum<DP>(Gs, i, c.j);
        const float da = gg.x + Eb;
        const float db = fmaf(-ka, gg.y, ka * Hb2);
        ok = ok && isfinite(da) && isfinite(db);
        Gs[SM::ge(i, c.j)] = make_float2(da, db);
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

// Load window parameters into A = {alpha, beta' = -beta log2 e} and return theta_j (0 for
// padded lanes).
template <int DP>
__device__ __forceinline__ float load_params(float2* A, const WarpCtx<DP>& c, int D, int64_t w,
                                             bool live, const float* __restrict__ theta,
                                             const float* __restrict__ alpha,
                                             const float* __restrict__ beta) {
  using SM = Smem<DP>;
  const bool real = live && c.j < D;
#pragma unroll 4
  for (int i = 0; i < DP; i++) {
    float a = 0.0f, b = 1.0f;
    if (real && i < D) {
      a = alpha[(size_t)w * D * D + (size_t)i * D + c.j];
      b = beta[(size_t)w * D * D + (size_t)i * D + c.j];
    }
    A[SM::e(i, c.j)] = ab_pack<DP>(i, a, b * -kLog2e);
  }
  // null dimension (see eval.cuh): row DP = {1,0} at column 0, column DP has beta = 0
  A[SM::e(DP, c.j)] = ab_pack<DP>(DP, c.j == 0 ? 1.0f : 0.0f, 0.0f);
  if constexpr (!SM::SW) A[SM::e(c.j, DP)] = make_float2(0.0f, 0.0f);
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
  float2* gbase_s = reinterpret_cast<float2*>(smem + wid * SM::per_warp) + SM::group_off(c.g);
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
      const float2 gg = Gs[SM::ge(i, c.j)];
      g_alpha[(size_t)w * D * D + (size_t)i * D + c.j] = live ? gg.x : NAN;
      g_beta[(size_t)w * D * D + (size_t)i * D + c.j] = live ? gg.y : NAN;
    }
  }
}

// ---------------------------------------------------------------- optimizer state in TMEM
// Per window and lane j (source column j / target row j of the window's group), the state of
// the fit that is not needed by the event loop lives in tensor memory for the whole fit and
// touches global memory once at the start and once at the end (DESIGN.md a6): the exact beta
// of column j (shared memory holds beta' = -beta log2 e for the event loop), the previous point
// (rollback) and the Adam moments.  Columns (per lane, DP = padded D):
template <int DP>
struct TmCols {
  static constexpr uint32_t BETA = 0, PA = DP, PB = 2 * DP, MA = 3 * DP, MB = 4 * DP,
                            VA = 5 * DP, VB = 6 * DP, PT = 7 * DP, MT = 7 * DP + 1,
                            VT = 7 * DP + 2, N = 7 * DP + 3;
  static constexpr uint32_t ALLOC = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : N <= 256 ? 256 : 512;
  static constexpr int CH = DP < 8 ? DP : 8;   // columns per tcgen05.ld/st batch
};

enum { ACT_NONE = 0, ACT_STEP = 1, ACT_ROLLBACK = 2 };

// Load window w's parameters (init) into A = {alpha, beta'} (shared) and its exact beta and
// Adam moments (opt_state or zeros) into TMEM; returns theta_j.  Warp-collective: lanes with
// load == false keep their TMEM columns (read and written back) and their A rows.
template <int DP>
__device__ __forceinline__ float load_window(float2* A, const WarpCtx<DP>& c, int D, int64_t w,
                                             bool load, bool live, uint32_t tm, float th_keep,
                                             const float* __restrict__ theta,
                                             const float* __restrict__ alpha,
                                             const float* __restrict__ beta,
                                             const float* __restrict__ opt) {
  using SM = Smem<DP>;
  using L = TmCols<DP>;
  constexpr int CH = L::CH;
  const bool real = load && live && c.j < D;
  const size_t P = (size_t)D + 2 * (size_t)D * D;
  const float* m = (opt && real) ? opt + (size_t)w * 2 * P : nullptr;
  const float* v = m ? m + P : nullptr;
#pragma unroll
  for (int k = 0; k < DP; k += CH) {
    float bx[CH], ma[CH], mb[CH], va[CH], vb[CH];
    tm_ld<CH>(tm + L::BETA + k, bx);
    tm_ld<CH>(tm + L::MA + k, ma);
    tm_ld<CH>(tm + L::MB + k, mb);
    tm_ld<CH>(tm + L::VA + k, va);
    tm_ld<CH>(tm + L::VB + k, vb);
    tm_wait_ld();
    tm_fence_regs(bx); tm_fence_regs(ma); tm_fence_regs(mb); tm_fence_regs(va); tm_fence_regs(vb);
#pragma unroll
    for (int u = 0; u < CH; u++) {
      const int i = k + u;
      if (load) {
        float a = 0.0f, b = 1.0f;
        const bool r = real && i < D;
        if (r) {
          a = alpha[(size_t)w * D * D + (size_t)i * D + c.j];
          b = beta[(size_t)w * D * D + (size_t)i * D + c.j];
        }
        A[SM::e(i, c.j)] = ab_pack<DP>(i, a, b * -kLog2e);
        bx[u] = b;
        const size_t qa = (size_t)D + (size_t)i * D + c.j, qb = qa + (size_t)D * D;
        ma[u] = (m && r) ? m[qa] : 0.0f;
        mb[u] = (m && r) ? m[qb] : 0.0f;
        va[u] = (v && r) ? v[qa] : 0.0f;
        vb[u] = (v && r) ? v[qb] : 0.0f;
      }
    }
    tm_st<CH>(tm + L::BETA + k, bx);
    tm_st<CH>(tm + L::MA + k, ma);
    tm_st<CH>(tm + L::MB + k, mb);
    tm_st<CH>(tm + L::VA + k, va);
    tm_st<CH>(tm + L::VB + k, vb);
  }
  float mt[1], vt[1];
  tm_ld<1>(tm + L::MT, mt);
  tm_ld<1>(tm + L::VT, vt);
  tm_wait_ld();
  tm_fence_regs(mt); tm_fence_regs(vt);
  float th = th_keep;
  if (load) {
    mt[0] = m ? m[c.j] : 0.0f;
    vt[0] = v ? v[c.j] : 0.0f;
    th = real ? theta[(size_t)w * D + c.j] : 0.0f;
    // null dimension (see eval.cuh): row DP = {1,0} at column 0, column DP has beta = 0
    A[SM::e(DP, c.j)] = ab_pack<DP>(DP, c.j == 0 ? 1.0f : 0.0f, 0.0f);
    if constexpr (!SM::SW) A[SM::e(c.j, DP)] = make_float2(0.0f, 0.0f);
  }
  tm_st<1>(tm + L::MT, mt);
  tm_st<1>(tm + L::VT, vt);
  tm_wait_st();
  return th;
}

// Write window w's parameters (alpha from A, exact beta from TMEM, theta) and, when the caller
// passed opt_state, its Adam moments back to global memory.  Warp-collective (TMEM reads);
// only lanes with `store` write.
template <int DP>
__device__ __forceinline__ void store_window(const float2* A, const WarpCtx<DP>& c, int D,
                                             int64_t w, bool store, float th, uint32_t tm,
                                             float* __restrict__ theta, float* __restrict__ alpha,
                                             float* __restrict__ beta, float* __restrict__ opt) {
  using SM = Smem<DP>;
  using L = TmCols<DP>;
  constexpr int CH = L::CH;
  const bool real = store && c.j < D;
  const size_t P = (size_t)D + 2 * (size_t)D * D;
  float* m = (opt && real) ? opt + (size_t)w * 2 * P : nullptr;
  float* v = m ? m + P : nullptr;
#pragma unroll
  for (int k = 0; k < DP; k += CH) {
    float bx[CH], ma[CH], mb[CH], va[CH], vb[CH];
    tm_ld<CH>(tm + L::BETA + k, bx);
    tm_ld<CH>(tm + L::MA + k, ma);
    tm_ld<CH>(tm + L::MB + k, mb);
    tm_ld<CH>(tm + L::VA + k, va);
    tm_ld<CH>(tm + L::VB + k, vb);
    tm_wait_ld();
    tm_fence_regs(bx); tm_fence_regs(ma); tm_fence_regs(mb); tm_fence_regs(va); tm_fence_regs(vb);
#pragma unroll
    for (int u = 0; u < CH; u++) {
      const int i = k + u;
      if (real && i < D) {
        const size_t q = (size_t)w * D * D + (size_t)i * D + c.j;
        alpha[q] = ab_alpha<DP>(i, A[SM::e(i, c.j)]);
        beta[q] = bx[u];
        if (m) {
          const size_t qa = (size_t)D + (size_t)i * D + c.j, qb = qa + (size_t)D * D;
          m[qa] = ma[u]; m[qb] = mb[u]; v[qa] = va[u]; v[qb] = vb[u];
        }
      }
    }
  }
  float mt[1], vt[1];
  tm_ld<1>(tm + L::MT, mt);
  tm_ld<1>(tm + L::VT, vt);
  tm_wait_ld();
  tm_fence_regs(mt); tm_fence_regs(vt);
  if (real) {
    theta[(size_t)w * D + c.j] = th;
    if (m) {
      m[c.j] = mt[0];
      v[c.j] = vt[0];
    }
  }
}

// One optimizer action per group, warp-collective (oracle_fit):
//   ACT_STEP      previous point <- current; PyTorch Adam / GD step on the loss -lnL * scale
//                 for the groups in fit_mask; projection (alpha >= 0; beta, theta >= floor)
//   ACT_ROLLBACK  current <- previous point (non-finite evaluation)
//   ACT_NONE      nothing (the lane's TMEM columns are written back unchanged)
// Gradients of lnL are in Gs (d alpha, d beta) and dth.  A holds {alpha, beta'}.
template <int DP, bool RESUME>
__device__ __forceinline__ void opt_action(float2* A, const float2* Gs, const WarpCtx<DP>& c,
                                           int D, const FitCfgDev& cfg, int act, float lr_w,
                                           int s, float scale, float dth, float& th, uint32_t tm) {
  using SM = Smem<DP>;
  using L = TmCols<DP>;
  constexpr int CH = L::CH;
  const bool real = c.j < D;
  const bool step = act == ACT_STEP, rb = act == ACT_ROLLBACK;
  const bool adam = cfg.optimizer == MDHP_OPT_ADAM;
  float bc1 = 1.0f, sbc2 = 1.0f;
  if (adam && step) {
    // s counts this call's steps; cfg.step0 those of earlier calls (resume)
    const float sg = RESUME ? (float)(s + cfg.step0) : (float)s;
    bc1 = 1.0f - powf(cfg.b1, sg);
    sbc2 = sqrtf(1.0f - powf(cfg.b2, sg));
  }
  auto upd = [&](float p, float g, float& mm, float& vv, float lo) -> float {
    const float gl = -g * scale;
    if (adam) {
      mm = cfg.b1 * mm + (1.0f - cfg.b1) * gl;
      vv = cfg.b2 * vv + (1.0f - cfg.b2) * gl * gl;
      const float denom = sqrtf(vv) / sbc2 + cfg.eps;
      p = p - (lr_w / bc1) * (mm / denom);
    } else {
      p = p - lr_w * gl;
    }
    return p < lo ? lo : p;
  };
  const bool fa = cfg.fit_mask & MDHP_FIT_ALPHA, fb = cfg.fit_mask & MDHP_FIT_BETA,
             ft = cfg.fit_mask & MDHP_FIT_THETA;
  // alpha column (previous point, moments), then beta (exact value, previous point, moments):
  // two passes keep fewer registers live outside the event loop
#pragma unroll
  for (int k = 0; k < DP; k += CH) {
    float pa[CH], ma[CH], va[CH];
    tm_ld<CH>(tm + L::PA + k, pa);
    tm_ld<CH>(tm + L::MA + k, ma);
    tm_ld<CH>(tm + L::VA + k, va);
    tm_wait_ld();
    tm_fence_regs(pa); tm_fence_regs(ma); tm_fence_regs(va);
#pragma unroll
    for (int u = 0; u < CH; u++) {
      const int i = k + u;
      if (real && i < D && act != ACT_NONE) {
        float2* e = &A[SM::e(i, c.j)];
        float a = ab_alpha<DP>(i, *e);
        if (step) {
          pa[u] = a;
          if (fa) a = upd(a, Gs[SM::ge(i, c.j)].x, ma[u], va[u], 0.0f);
        } else {
          a = pa[u];
        }
        *e = ab_pack<DP>(i, a, ab_beta<DP>(i, *e));
      }
    }
    tm_st<CH>(tm + L::PA + k, pa);
    tm_st<CH>(tm + L::MA + k, ma);
    tm_st<CH>(tm + L::VA + k, va);
  }
#pragma unroll
  for (int k = 0; k < DP; k += CH) {
    float bx[CH], pb[CH], mb[CH], vb[CH];
    tm_ld<CH>(tm + L::BETA + k, bx);
    tm_ld<CH>(tm + L::PB + k, pb);
    tm_ld<CH>(tm + L::MB + k, mb);
    tm_ld<CH>(tm + L::VB + k, vb);
    tm_wait_ld();
    tm_fence_regs(bx); tm_fence_regs(pb); tm_fence_regs(mb); tm_fence_regs(vb);
#pragma unroll
    for (int u = 0; u < CH; u++) {
      const int i = k + u;
      if (real && i < D && act != ACT_NONE) {
        float b = bx[u];
        if (step) {
          pb[u] = b;
          if (fb) b = upd(b, Gs[SM::ge(i, c.j)].y, mb[u], vb[u], cfg.min_param);
        } else {
          b = pb[u];
        }
        bx[u] = b;
        float2* e = &A[SM::e(i, c.j)];
        *e = ab_pack<DP>(i, ab_alpha<DP>(i, *e), b * -kLog2e);
      }
    }
    tm_st<CH>(tm + L::BETA + k, bx);
    tm_st<CH>(tm + L::PB + k, pb);
    tm_st<CH>(tm + L::MB + k, mb);
    tm_st<CH>(tm + L::VB + k, vb);
  }
  float pt[1], mt[1], vt[1];
  tm_ld<1>(tm + L::PT, pt);
  tm_ld<1>(tm + L::MT, mt);
  tm_ld<1>(tm + L::VT, vt);
  tm_wait_ld();
  tm_fence_regs(pt); tm_fence_regs(mt); tm_fence_regs(vt);
  if (real && step) {
    pt[0] = th;
    if (ft) th = upd(th, dth, mt[0], vt[0], cfg.min_param);
  } else if (real && rb) {
    th = pt[0];
  }
  tm_st<1>(tm + L::PT, pt);
  tm_st<1>(tm + L::MT, mt);
  tm_st<1>(tm + L::VT, vt);
  tm_wait_st();
}

// Per-window (group-uniform) control of the fit loop (identical to
// oracle_fit): decides the optimizer action after an evaluation and advances the counters.
struct WinCtl {
  int it = 0, s = 0, halv = 0, stall = 0, st = 0;
  float lr_w = 0.0f;
  double lnl_prev = 0.0;
  bool have_prev = false, have_lnl = false;
  // returns the action; sets done when the window stops
  __device__ __forceinline__ int decide(const FitCfgDev& cfg, double lnl, bool finite, bool& done,
                                        float* trace, int64_t w, bool lane0) {
    int act = ACT_NONE;
    if (!finite) {
      st |= MDHP_ST_NONFINITE;
      if (!have_prev || halv >= cfg.max_halvings) {
        st |= MDHP_ST_DIVERGED;
        done = true;
        if (have_prev) act = ACT_ROLLBACK;
      } else {
        act = ACT_ROLLBACK;
        lr_w *= 0.5f;
        halv++;
        it++;
      }
    } else {
      if (trace && lane0) trace[(size_t)w * cfg.max_iters + it] = (float)lnl;
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
        have_prev = true;
        s++;
        act = ACT_STEP;
        it++;
      }
    }
    if (it >= cfg.max_iters) done = true;
    return act;
  }
};

// Persistent fit kernel (a6): windows are taken longest first from a global counter and run
// their whole iteration loop on chip (state in shared memory, optimizer state in TMEM), then
// lnL is evaluated at the returned parameters and everything is written back.
//   REFILL (converged mode, tol_rel > 0): each group of DP lanes takes one window at a time;
//     when its window stops (convergence, divergence, budget) the group evaluates the final lnL,
//     writes back and takes the next window at once, so a warp's other group(s) never idle
//     behind a window that stopped early (the convergence mask frees lanes instead of padding
//     them).  One evaluation per warp step: TRAIN groups step after it, FINAL groups record it.
//   !REFILL (fixed iteration count): every window of a warp stops at the same evaluation, so a
//     warp takes G windows at a time and keeps them to the end (no per-window bookkeeping).
//   LAT (Dp = 8, batches that fit one wave at 8 warps per SM, e.g. BASELINE cfg2): the same
//     kernel without the 128-register cap of 16 warps per SM, so ptxas keeps the chunk's
//     addresses and partial results in registers instead of re-deriving them (the kernel is
//     bound by each warp's dependent chain there, not by throughput; +6% on cfg2).  With fixed
//     iterations it runs one CTA of 8 warps per SM and cfg.slot_order = 1: warp slot (CTA b,
//     warp w) takes unit order(w) * gridDim + b, order = 0 for warp 0, 1-6 for warps 1-3 and
//     5-7, 7 for warp 4, so the gridDim longest units (perm is longest-first) run on warp 0 of
//     every SM with no other busy warp on its sub-partition (warps w and w+4 share one), and
//     the batch time -- set by the warps holding the longest windows -- approaches their
//     uncontended chain (profiles/r02_cfg2_latency_profiles.txt).
template <int DP, bool RESUME, bool REFILL, bool LAT = false>
__global__ void __launch_bounds__(LAT ? 256 : 128, DP >= 32 ? 2 : LAT ? 1 : 4)
k_fit(Packed P, FitCfgDev cfg, float* __restrict__ theta, float* __restrict__ alpha,
      float* __restrict__ beta, float* __restrict__ opt, double* __restrict__ lnl_out,
      int32_t* __restrict__ iters_out, int32_t* __restrict__ status,
      float* __restrict__ trace, int* __restrict__ counter, int32_t* __restrict__ xlist,
      int32_t* __restrict__ xcount) {
  extern __shared__ __align__(16) unsigned char smem[];
  using SM = Smem<DP>;
  using TL = TmCols<DP>;
  WarpCtx<DP> c;
  const int wid = threadIdx.x >> 5;
  float2* gbase_s = reinterpret_cast<float2*>(smem + wid * SM::per_warp) + SM::group_off(c.g);
  float2* A = gbase_s;
  float2* SQ = gbase_s + SM::AS;
  float2* Gs = gbase_s + 2 * SM::AS;
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + (blockDim.x >> 5) * SM::per_warp);
  // warps w and w + 4 of an 8-warp CTA share TMEM lanes 32 (w % 4) ..: separate column blocks
  const uint32_t tcols = TL::ALLOC * (blockDim.x > 128 ? 2u : 1u);
  const uint32_t tbase = tm_alloc(slot, tcols);
  const uint32_t tm = tbase + ((uint32_t)((wid & 3) * 32) << 16) + (uint32_t)(wid >> 2) * TL::ALLOC;
  const int D = P.D;
  if constexpr (REFILL) {
    enum { TRAIN = 0, FINAL = 1, IDLE = 2 };
    int phase = IDLE;
    int64_t w = 0;
    int st0 = 0, n = 0;
    bool live = false;
    float th = 0.0f, scale = 1.0f;
    WinCtl ctl;
    ColInfo ci = col_info<DP>(P, 0, false, c.j);
    // group-collective: the next window index (all lanes of the group)
    auto fetch = [&]() -> bool {
      int64_t sl = 0;
      if (c.j == 0) sl = atomicAdd(counter, 1);
      sl = __shfl_sync(c.gmask, sl, c.gbase);
      if (sl >= P.W) {
        phase = IDLE;
        live = false;
        n = 0;
        return false;
      }
      w = P.perm[sl];
      MDHP_ASSERT(w >= 0 && w < P.W);
      st0 = status[w];
      live = !(st0 & MDHP_ST_INVALID);
      ci = col_info<DP>(P, w, live, c.j);
      n = live ? P.n[w] : 0;
      scale = (cfg.loss_mean && n > 0) ? 1.0f / (float)n : 1.0f;
      ctl = WinCtl();
      ctl.lr_w = cfg.lr;
      phase = (!live || cfg.max_iters <= 0) ? FINAL : TRAIN;
      return true;
    };
    bool got = fetch();
    th = load_window<DP>(A, c, D, w, got, live, tm, th, theta, alpha, beta, opt);
    while (__any_sync(kFull, phase != IDLE)) {
      const bool act_eval = phase != IDLE && live;
      const int nmax = group_max_i<DP>(act_eval ? n : 0);
      float dth;
      bool finite, exact;
      // gradients only when some group trains (a warp whose groups all stop together, as in the
      // fixed-iteration mode, evaluates its final lnL without them)
      const double lnl = __any_sync(kFull, phase == TRAIN)
                             ? eval_window<DP, true>(P, A, SQ, Gs, c, w, act_eval, nmax, th, ci, dth, finite, exact)
                             : eval_window<DP, false>(P, A, SQ, Gs, c, w, act_eval, nmax, th, ci, dth, finite, exact);
      int act = ACT_NONE;
      bool fin = false;
      if (phase == TRAIN) {
        bool done = false;
        act = ctl.decide(cfg, lnl, finite, done, trace, w, c.j == 0);
        if (done) phase = FINAL;   // the next evaluation is lnL at the returned parameters
      } else if (phase == FINAL) {
        fin = true;
        if (c.j == 0) {
          lnl_out[w] = live ? lnl : (double)NAN;
          iters_out[w] = ctl.it;
          status[w] = (st0 & kKeepStatus) | ctl.st;
          if (exact) list_exact(xlist, xcount, w);
          if (trace && live)
            for (int q = ctl.it; q < cfg.max_iters; q++) trace[(size_t)w * cfg.max_iters + q] = NAN;
        }
      }
      if (__any_sync(kFull, act != ACT_NONE))
        opt_action<DP, RESUME>(A, Gs, c, D, cfg, act, ctl.lr_w, ctl.s, scale, dth, th, tm);
      if (__any_sync(kFull, fin)) {
        store_window<DP>(A, c, D, w, fin && live, th, tm, theta, alpha, beta, opt);
        bool nw = false;
        if (fin) nw = fetch();
        th = load_window<DP>(A, c, D, w, nw, live, tm, th, theta, alpha, beta, opt);
      }
      __syncwarp();
    }
  } else {
    const int64_t nunits = (P.W + SM::G - 1) / SM::G;
    bool taken = false;
    for (;;) {
      int64_t unit = 0;
      if (LAT && cfg.slot_order) {   // one static unit per warp slot (see above)
        if (taken) break;
        taken = true;
        const int order = wid == 0 ? 0 : wid < 4 ? wid : wid > 4 ? wid - 1 : 7;
        unit = (int64_t)order * gridDim.x + blockIdx.x;
      } else {
        if (c.lane == 0) unit = atomicAdd(counter, 1);
        unit = __shfl_sync(kFull, unit, 0);
      }
      if (unit >= nunits) break;
      const int64_t slot_w = unit * SM::G + c.g;
      const int64_t w = slot_w < P.W ? P.perm[slot_w] : 0;
      MDHP_ASSERT(w >= 0 && w < (P.W > 0 ? P.W : 1));
      const int st0 = slot_w < P.W ? status[w] : MDHP_ST_INVALID;
      const bool live = slot_w < P.W && !(st0 & MDHP_ST_INVALID);
      float th = load_window<DP>(A, c, D, w, true, live, tm, 0.0f, theta, alpha, beta, opt);
      const ColInfo ci = col_info<DP>(P, w, live, c.j);
      const int n = live ? P.n[w] : 0;
      const float scale = (cfg.loss_mean && n > 0) ? 1.0f / (float)n : 1.0f;
      WinCtl ctl;
      ctl.lr_w = cfg.lr;
      bool done = !live || cfg.max_iters <= 0;
      while (__any_sync(kFull, !done)) {
        const int nmax = group_max_i<DP>(done ? 0 : n);
        float dth;
        bool finite, exact;
        const double lnl = eval_window<DP, true>(P, A, SQ, Gs, c, w, !done, nmax, th, ci, dth, finite, exact);
        int act = ACT_NONE;
        if (!done) act = ctl.decide(cfg, lnl, finite, done, trace, w, c.j == 0);
        if (__any_sync(kFull, act != ACT_NONE))
          opt_action<DP, RESUME>(A, Gs, c, D, cfg, act, ctl.lr_w, ctl.s, scale, dth, th, tm);
        __syncwarp();
      }
      // lnL at the returned parameters (no gradient accumulation needed)
      const int nmax = group_max_i<DP>(n);
      float dth;
      bool finite, exact;
      const double lnl = eval_window<DP, false>(P, A, SQ, Gs, c, w, live, nmax, th, ci, dth, finite, exact);
      store_window<DP>(A, c, D, w, slot_w < P.W && live, th, tm, theta, alpha, beta, opt);
      if (slot_w < P.W && c.j == 0) {
        lnl_out[w] = live ? lnl : (double)NAN;
        iters_out[w] = ctl.it;
        status[w] = (st0 & kKeepStatus) | ctl.st;
        if (exact) list_exact(xlist, xcount, w);
        if (trace && live)
          for (int q = ctl.it; q < cfg.max_iters; q++) trace[(size_t)w * cfg.max_iters + q] = NAN;
      }
      __syncwarp();
    }
  }
  tm_free(tbase, tcols);
}

// ---------------------------------------------------------------- time chunks (latency mode)
// mdhp_fit_config.time_chunks = C >= 2, Dp <= 8: each window's events are cut into C
// consecutive time chunks (boundaries on 8-event blocks, never inside a tie group), one per
// group of Dp lanes, so a warp holds 32/(Dp C) windows and a window's sequential event chain
// is ~C times shorter.  C = 32/Dp (one window per warp) is the latency mode for single windows
// (BASELINE cfg1); smaller C trades chain length against windows per warp for small batches.
// Per evaluation (the a7 chunked scan inside a warp):
//   phase 1: every group sums its chunk's local state at the chunk's last event t_e from an
//            empty history (local_direct: direct sums, no recurrence chain);
//   scan:    the affine maps of a window's chunks (decay over the chunk span + local state,
//            seq.cu AffMap) are scanned across its groups with warp shuffles; the state carried
//            into chunk q is the composite of chunks 0..q-1, anchored at the chunk base t_b (the
//            previous chunk's last event);
//   phase 3: every group runs the full event loop of its chunk from the carried state;
//   then a window's gradient accumulators, sum ln lambda and sum 1/lambda are added over its
//   groups in a fixed order (identical in every group) and every group finishes the epilogue
//   from the window's last chunk's final state, so all groups of a window hold the same lnL,
//   gradients and (after opt_action) parameters.  Results equal the throughput layout's within
//   fp32 rounding (a different but fixed summation order), deterministic run to run.
struct TcChunk {
  int b, n;           // first event (relative to the window) and count of this group's chunk
  int clampo;         // offset of the window's null chunk, relative to b
  float tb, te;       // chunk base (last event before it, -1 if none) and last event time
};

template <int CPW>
__device__ __forceinline__ TcChunk tc_chunk(const Packed& P, int64_t beg, int n, int q) {
  // boundaries b_0 = 0 <= b_1 <= ... <= b_C = n: near k n / C, on 8-event blocks, moved past
  // cross-mark tie groups (a chunk must not start at a time equal to its base)
  int lo = 0, hi = n;
  int prev = 0;
  for (int k = 1; k <= q + 1 && k <= CPW; k++) {
    int b = k == CPW ? n : (int)(((int64_t)n * k / CPW) & ~(int64_t)7);
    if (b < prev) b = prev;
    while (b > 0 && b < n && P.t32[beg + b] == P.t32[beg + b - 1]) b = min(b + 8, n);
    if (k == q) lo = b;
    if (k == q + 1) hi = b;
    prev = b;
  }
  TcChunk ch;
  ch.b = lo;
  ch.n = hi - lo;
  ch.clampo = ((n + 7) & ~7) - lo;
  ch.tb = lo > 0 ? P.t32[beg + lo - 1] : -1.0f;
  ch.te = hi > 0 ? P.t32[beg + hi - 1] : -1.0f;
  return ch;
}

struct TcMap {
  float E, L, Sb, Qb;   // decay over the span, span, state added (S, Q') -- seq.cu AffMap
};
__device__ __forceinline__ TcMap tc_compose(const TcMap& m1, const TcMap& m2) {
  TcMap r;
  r.E = m2.E * m1.E;
  r.L = m1.L + m2.L;
  r.Sb = fmaf(m2.E, m1.Sb, m2.Sb);
  r.Qb = fmaf(m2.E, fmaf(m2.L, m1.Sb, m1.Qb), m2.Qb);
  return r;
}

// Evaluation of the window whose chunk q (= c.g % CPW) this group holds; see above.
template <int DP, int CPW, bool GRAD>
__device__ __forceinline__ double eval_window_tc(const Packed& P, float2* A, float2* SQ,
                                                 float2* Gs, float2* wbase, const WarpCtx<DP>& c,
                                                 int64_t w, bool live, const TcChunk& ch,
                                                 float th, const ColInfo& ci, float& dth,
                                                 bool& finite, bool& exact) {
  using SM = Smem<DP>;
  constexpr int WL = DP * CPW;                 // lanes of one window
  const int q = c.g % CPW;                     // this group's chunk of its window
  const int g0 = c.g - q;                      // the window's first group
  const unsigned wmask = WL == 32 ? kFull : (((1u << WL) - 1u) << (g0 * DP));
  const int64_t beg = live ? P.begin[w] : 0;
  const int n = live ? ch.n : 0;
  const int nmax = group_max_i<DP>(n);
  // ---- phase 1: the chunk's local state at its last event te (direct sums, local_direct)
  reset_state<DP>(SQ, Gs, c.j);
  __syncwarp();
  local_direct<DP>(A, SQ, Gs, c.j, P.t32, P.dtp, P.mark, beg + ch.b, n, nmax, ch.te, ch.clampo);
  // ---- this chunk's affine map per pair (r, j): decay over the span, local state at te
  TcMap m[DP];
  const float L = ch.te - ch.tb;
#pragma unroll
  for (int r = 0; r < DP; r++) {
    const float2 k = A[SM::e(r, c.j)];
    const float b = ab_beta<DP>(r, k);   // beta' (A holds -beta log2 e)
    const float2 sq = SQ[SM::e(r, c.j)];
    m[r].E = ex2f(b * L);
    m[r].L = L;
    m[r].Sb = sq.x;
    m[r].Qb = sq.y;
  }
  // ---- inclusive scan of the maps over the window's groups (lane j of chunk q <- q - k)
#pragma unroll
  for (int k = 1; k < CPW; k <<= 1) {
#pragma unroll
    for (int r = 0; r < DP; r++) {
      TcMap up;
      up.E = __shfl_up_sync(kFull, m[r].E, k * DP);
      up.L = __shfl_up_sync(kFull, m[r].L, k * DP);
      up.Sb = __shfl_up_sync(kFull, m[r].Sb, k * DP);
      up.Qb = __shfl_up_sync(kFull, m[r].Qb, k * DP);
      if (q >= k) m[r] = tc_compose(up, m[r]);
    }
  }
  // ---- phase 3: the full event loop of the chunk from the carried state (the composite of
  // the window's earlier chunks applied to the empty initial state), anchored at tb
  __syncwarp();
#pragma unroll
  for (int r = 0; r < DP; r++) {
    const float cs = __shfl_up_sync(kFull, m[r].Sb, DP);
    const float cq = __shfl_up_sync(kFull, m[r].Qb, DP);
    SQ[SM::e(r, c.j)] = q > 0 ? make_float2(cs, cq) : make_float2(0.0f, 0.0f);
    gzero<DP>(Gs, r, c.j);
  }
  __syncwarp();
  float last, gth;
  double lsum;
  event_loop<DP, GRAD, true, true>(A, SQ, Gs, c.j, c.gbase, P.t32, P.dtp, P.mark, beg + ch.b, n,
                                   nmax, th, last, gth, lsum, ch.b > 0 ? ch.tb : -1.0f,
                                   ch.clampo, ch.tb);
  // ---- sums over the window's chunks, in the same order in every group of the window
#pragma unroll
  for (int o = DP; o < WL; o <<= 1) gth += __shfl_xor_sync(kFull, gth, o);
#pragma unroll
  for (int o = WL / 2; o >= 1; o >>= 1) lsum += __shfl_xor_sync(kFull, lsum, o);
  __syncwarp();
  float2 gtot[DP];
  if (GRAD) {
#pragma unroll
    for (int r = 0; r < DP; r++) {
      float2 a = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int qq = 0; qq < CPW; qq++) {
        const float2 v = gsum<DP>(wbase + SM::group_off(g0 + qq) + 2 * SM::AS, r, c.j);
        a.x += v.x;
        a.y += v.y;
      }
      gtot[r] = a;
    }
  }
  // ---- epilogue from the window's last chunk's final state (its SQ, its lanes' last times)
  const int gl = g0 + CPW - 1;
  const float2* SQl = wbase + SM::group_off(gl) + SM::AS;
  ColInfo cc = ci;
  cc.last = __shfl_sync(kFull, last, gl * DP + c.j);
  Series S;
  load_series(S, P.mom + ((size_t)(live ? w : 0) * P.Dp + c.j) * kMom, live && cc.N > 0);
  double part3 = 0.0;
  bool ok = true;
  float2 gout[DP];
#pragma unroll 4
  for (int i = 0; i < DP; i++) {
    const float2 k = A[SM::e(i, c.j)];
    const float2 sq = SQl[SM::e(i, c.j)];
    float Eb, Hb2;
    const float ka = ab_alpha<DP>(i, k), kb = ab_beta<DP>(i, k) * -kLn2;
    compensator(cc, S, kb, sq.x, sq.y, Eb, Hb2);
    gout[i] = make_float2(0.0f, 0.0f);
    if (cc.real && i < P.D) {
      part3 += (double)(ka * Eb);
      if (GRAD) {
        const float da = gtot[i].x + Eb;
        const float db = fmaf(-ka, gtot[i].y, ka * Hb2);
        ok = ok && isfinite(da) && isfinite(db);
        gout[i] = make_float2(da, db);
      }
    }
  }
  __syncwarp();   // every group has read the others' accumulators
  if (GRAD) {
#pragma unroll
    for (int i = 0; i < DP; i++) Gs[SM::ge(i, c.j)] = gout[i];
  }
  dth = gth - ci.T;
  if (GRAD && cc.real) ok = ok && isfinite(dth);
  part3 = group_sum_d<DP>(part3);
  const double sth = group_sum_d<DP>(cc.real ? (double)th : 0.0);
  const double lnl = (double)kLn2 * lsum + part3 - (double)ci.T * sth;
  const unsigned bal = __ballot_sync(kFull, ok) & wmask;
  finite = (bal == wmask) && isfinite(lnl);
  const int ntot = live ? P.n[w] : 0;
  exact = live && needs_exact(lnl, ntot, (double)kLn2 * lsum, (double)ci.T * sth, part3);
  __syncwarp();
  return lnl;
}

template <int DP, int CPW, bool RESUME>
__global__ void __launch_bounds__(128, 4)
k_fit_tc(Packed P, FitCfgDev cfg, float* __restrict__ theta, float* __restrict__ alpha,
         float* __restrict__ beta, float* __restrict__ opt, double* __restrict__ lnl_out,
         int32_t* __restrict__ iters_out, int32_t* __restrict__ status,
         float* __restrict__ trace, int* __restrict__ counter, int32_t* __restrict__ xlist,
         int32_t* __restrict__ xcount) {
  extern __shared__ __align__(16) unsigned char smem[];
  using SM = Smem<DP>;
  using TL = TmCols<DP>;
  static_assert(DP <= 8 && CPW >= 2 && CPW * DP <= 32, "time chunks: Dp <= 8, 2 <= C <= 32/Dp");
  constexpr int WPW = 32 / (DP * CPW);   // windows per warp
  WarpCtx<DP> c;
  const int wid = threadIdx.x >> 5;
  float2* wbase = reinterpret_cast<float2*>(smem + wid * SM::per_warp);
  float2* A = wbase + SM::group_off(c.g);
  float2* SQ = A + SM::AS;
  float2* Gs = A + 2 * SM::AS;
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + (blockDim.x >> 5) * SM::per_warp);
  const uint32_t tbase = tm_alloc(slot, TL::ALLOC);
  const uint32_t tm = tbase + ((uint32_t)((wid & 3) * 32) << 16);
  const int D = P.D;
  const int q = c.g % CPW;
  const bool first_lane = (c.lane % (DP * CPW)) == 0;   // the window's lane 0
  const int64_t nunits = (P.W + WPW - 1) / WPW;
  for (;;) {
    int64_t unit = 0;
    if (c.lane == 0) unit = atomicAdd(counter, 1);
    unit = __shfl_sync(kFull, unit, 0);
    if (unit >= nunits) break;
    const int64_t slot_w = unit * WPW + c.g / CPW;
    const int64_t w = slot_w < P.W ? P.perm[slot_w] : 0;
    MDHP_ASSERT(w >= 0 && w < (P.W > 0 ? P.W : 1));
    const int st0 = slot_w < P.W ? status[w] : MDHP_ST_INVALID;
    const bool live = slot_w < P.W && !(st0 & MDHP_ST_INVALID);
    float th = load_window<DP>(A, c, D, w, true, live, tm, 0.0f, theta, alpha, beta, opt);
    const ColInfo ci = col_info<DP>(P, w, live, c.j);
    const int n = live ? P.n[w] : 0;
    const TcChunk ch = tc_chunk<CPW>(P, live ? P.begin[w] : 0, n, q);
    const float scale = (cfg.loss_mean && n > 0) ? 1.0f / (float)n : 1.0f;
    WinCtl ctl;
    ctl.lr_w = cfg.lr;
    bool done = !live || cfg.max_iters <= 0;
    while (__any_sync(kFull, !done)) {   // windows of a warp stop independently (mask)
      float dth;
      bool finite, exact;
      const double lnl = eval_window_tc<DP, CPW, true>(P, A, SQ, Gs, wbase, c, w, live && !done, ch,
                                                       th, ci, dth, finite, exact);
      int act = ACT_NONE;
      if (!done) act = ctl.decide(cfg, lnl, finite, done, trace, w, first_lane);
      if (__any_sync(kFull, act != ACT_NONE))
        opt_action<DP, RESUME>(A, Gs, c, D, cfg, act, ctl.lr_w, ctl.s, scale, dth, th, tm);
      __syncwarp();
    }
    float dth;
    bool finite, exact;
    const double lnl = eval_window_tc<DP, CPW, false>(P, A, SQ, Gs, wbase, c, w, live, ch, th, ci,
                                                      dth, finite, exact);
    store_window<DP>(A, c, D, w, slot_w < P.W && live && q == 0, th, tm, theta, alpha, beta, opt);
    if (slot_w < P.W && first_lane) {
      lnl_out[w] = live ? lnl : (double)NAN;
      iters_out[w] = ctl.it;
      status[w] = (st0 & kKeepStatus) | ctl.st;
      if (exact) list_exact(xlist, xcount, w);
      if (trace && live)
        for (int k = ctl.it; k < cfg.max_iters; k++) trace[(size_t)w * cfg.max_iters + k] = NAN;
    }
    __syncwarp();
  }
  tm_free(tbase, TL::ALLOC);
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
  const size_t smem = WPB * SM::per_warp + 16;   // + the TMEM base address slot
  // converged mode (tol_rel > 0): windows stop at different iterations -> per-window refill
  auto kern = cfg.tol_rel > 0.0f ? (cfg.step0 != 0 ? k_fit<DP, true, true> : k_fit<DP, false, true>)
                                 : (cfg.step0 != 0 ? k_fit<DP, true, false> : k_fit<DP, false, false>);
  // time chunks (Dp <= 8): C chunks per window, 32/(Dp C) windows per warp (k_fit_tc)
  int cpw = 1;
  if constexpr (DP <= 8) {
    if (cfg.time_chunks >= 2) {
      cpw = 2;
      while (cpw * 2 <= cfg.time_chunks && cpw * 2 * DP <= 32) cpw *= 2;
      const bool rs = cfg.step0 != 0;
      switch (cpw) {
        case 2: kern = rs ? k_fit_tc<DP, 2, true> : k_fit_tc<DP, 2, false>; break;
        case 4: kern = rs ? k_fit_tc<DP, (DP <= 8 ? 4 : 2), true> : k_fit_tc<DP, (DP <= 8 ? 4 : 2), false>; break;
        case 8: kern = rs ? k_fit_tc<DP, (DP <= 4 ? 8 : 2), true> : k_fit_tc<DP, (DP <= 4 ? 8 : 2), false>; break;
        case 16: kern = rs ? k_fit_tc<DP, (DP <= 2 ? 16 : 2), true> : k_fit_tc<DP, (DP <= 2 ? 16 : 2), false>; break;
        default: kern = rs ? k_fit_tc<DP, (DP <= 1 ? 32 : 2), true> : k_fit_tc<DP, (DP <= 1 ? 32 : 2), false>; break;
      }
    }
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  FitCfgDev kc = cfg;
  if constexpr (DP == 8) {
    const int64_t u8 = (P.W + SM::G - 1) / SM::G;
    if (cpw == 1 && u8 <= (int64_t)sms * 8) {   // one wave at 8 warps/SM
      const bool rs = cfg.step0 != 0;
      kern = cfg.tol_rel > 0.0f ? (rs ? k_fit<DP, true, true, true> : k_fit<DP, false, true, true>)
                                : (rs ? k_fit<DP, true, false, true> : k_fit<DP, false, false, true>);
      // fixed iterations, at most 7 units per SM: one 8-warp CTA per SM with the static
      // sub-partition-aware unit order (k_fit LAT)
      if (cfg.tol_rel <= 0.0f && u8 <= (int64_t)sms * 7 && !getenv("MDHP_NO_SLOT_ORDER")) {
        const size_t smem8 = 8 * SM::per_warp + 16;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8) != cudaSuccess) {
          set_error("cudaFuncSetAttribute(k_fit) failed");
          return MDHP_ECUDA;
        }
        kc.slot_order = 1;
        kern<<<(unsigned)sms, 256, smem8, st>>>(P, kc, th, al, be, opt, lnl, iters, status, trace, counter,
                                               xlist, xcount);
        count_launch();
        return MDHP_OK;
      }
    }
  }
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("cudaFuncSetAttribute(k_fit) failed");
    return MDHP_ECUDA;
  }
  // CTAs per SM from registers, shared memory and TMEM columns.  (The occupancy API reports 1
  // for kernels that allocate tensor memory; the hardware runs as many as the resources allow
  // and tcgen05.alloc would wait for columns, so the grid is sized from the resources here.)
  cudaFuncAttributes fa;
  int smem_sm = 0, smem_rsv = 0;
  if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess ||
      cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess) {
    set_error("k_fit: device attribute query failed");
    return MDHP_ECUDA;
  }
  const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
  const int by_regs = 65536 / (regs_warp * WPB);
  const int by_smem = smem_sm / (int)(smem + fa.sharedSizeBytes + smem_rsv);
  const int by_tmem = 512 / (int)TmCols<DP>::ALLOC;
  per_sm = by_regs < by_smem ? by_regs : by_smem;
  if (per_sm > by_tmem) per_sm = by_tmem;
  if (per_sm > 2048 / (WPB * 32)) per_sm = 2048 / (WPB * 32);
  if (getenv("MDHP_DEBUG_LAUNCH"))
    fprintf(stderr, "k_fit<%d>: per_sm=%d (regs %d smem %d tmem %d) smem=%zu regs=%d local=%zu\n", DP,
            per_sm, by_regs, by_smem, by_tmem, smem, fa.numRegs, fa.localSizeBytes);
  if (per_sm < 1) per_sm = 1;
  const int64_t wpu = cpw > 1 ? SM::G / cpw : SM::G;   // windows per warp unit
  const int64_t units = (P.W + wpu - 1) / wpu;
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
