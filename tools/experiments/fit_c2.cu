// fit_c2.cu — mdhp_loglik_grad / mdhp_fit kernels for Dp = 16 with the C2 mapping
// (eval_c2.cuh: 8 lanes per window, two columns per lane, 4 windows per warp).  The optimizer
// loop is the one of fit.cu: DESIGN.md "Fit".
#include <cmath>
#include "eval_c2.cuh"

namespace mdhp {

constexpr int kC2WPB = 4;   // warps per block; 26 KB of shared memory per warp

__global__ void __launch_bounds__(kC2WPB * 32, 2)
k_loglik_c2(Packed P, const float* __restrict__ theta, const float* __restrict__ alpha,
            const float* __restrict__ beta, double* __restrict__ lnl_out,
            float* __restrict__ g_theta, float* __restrict__ g_alpha, float* __restrict__ g_beta,
            const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wid = threadIdx.x >> 5;
  const C2Lane L(smem + wid * C2::per_warp);
  const int64_t slot = ((int64_t)blockIdx.x * kC2WPB + wid) * C2::GW + L.g;
  const int64_t w = slot < P.W ? P.perm[slot] : 0;
  const bool live = slot < P.W && !(status[w] & MDHP_ST_INVALID);
  const int D = P.D;
  const float2 th = c2_load_params(L, D, w, live, theta, alpha, beta);
  const int nmax = group_max_i<8>(live ? P.n[w] : 0);
  float2 dth;
  bool finite;
  const bool grad = g_theta != nullptr;
  double lnl;
  if (grad) lnl = c2_eval<true>(P, L, w, live, nmax, th, dth, finite);
  else lnl = c2_eval<false>(P, L, w, live, nmax, th, dth, finite);
  if (slot >= P.W) return;
  if (L.c == 0) lnl_out[w] = live ? lnl : (double)NAN;
  if (grad) {
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int j = L.c + 8 * q;
      if (j >= D) continue;
      g_theta[(size_t)w * D + j] = live ? (q ? dth.y : dth.x) : NAN;
      for (int r = 0; r < D; r++) {
        const float2 gg = at2<float2>(L.G, L.off(r, j));
        g_alpha[(size_t)w * D * D + (size_t)r * D + j] = live ? gg.x : NAN;
        g_beta[(size_t)w * D * D + (size_t)r * D + j] = live ? gg.y : NAN;
      }
    }
  }
}

// One optimizer step for this lane's columns c and c+8 (fit.cu step_column semantics).
__device__ __forceinline__ void c2_step(const C2Lane& L, int D, int64_t w, const FitCfgDev& cfg,
                                        float lr_w, int s, float scale, float2 dth, float2& th,
                                        float* __restrict__ opt) {
  const size_t P = (size_t)D + 2 * (size_t)D * D;
  float* m = opt ? opt + (size_t)w * 2 * P : nullptr;
  float* v = m ? m + P : nullptr;
  const bool adam = cfg.optimizer == MDHP_OPT_ADAM;
  float bc1 = 1.0f, sbc2 = 1.0f;
  if (adam) {
    bc1 = 1.0f - powf(cfg.b1, (float)s);
    sbc2 = sqrtf(1.0f - powf(cfg.b2, (float)s));
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
#pragma unroll
  for (int qq = 0; qq < 2; qq++) {
    const int j = L.c + 8 * qq;
    if (j >= D) continue;
    if (cfg.fit_mask & MDHP_FIT_THETA) {
      if (qq == 0) th.x = upd(th.x, dth.x, (size_t)j, cfg.min_param);
      else th.y = upd(th.y, dth.y, (size_t)j, cfg.min_param);
    }
    for (int r = 0; r < D; r++) {
      const int o = L.off(r, j);
      float2& k = at2<float2>(L.A, o);
      const float2 gg = at2<float2>(L.G, o);
      const size_t q = (size_t)D + (size_t)r * D + j;
      if (cfg.fit_mask & MDHP_FIT_ALPHA) k.x = upd(k.x, gg.x, q, 0.0f);
      if (cfg.fit_mask & MDHP_FIT_BETA) k.y = upd(k.y, gg.y, q + (size_t)D * D, cfg.min_param);
    }
  }
}

__device__ __forceinline__ void c2_store(const C2Lane& L, int D, int64_t w, float2 th,
                                         float* __restrict__ theta, float* __restrict__ alpha,
                                         float* __restrict__ beta) {
#pragma unroll
  for (int q = 0; q < 2; q++) {
    const int j = L.c + 8 * q;
    if (j >= D) continue;
    theta[(size_t)w * D + j] = q ? th.y : th.x;
    for (int r = 0; r < D; r++) {
      const float2 k = at2<float2>(L.A, L.off(r, j));
      alpha[(size_t)w * D * D + (size_t)r * D + j] = k.x;
      beta[(size_t)w * D * D + (size_t)r * D + j] = k.y;
    }
  }
}

__global__ void __launch_bounds__(kC2WPB * 32, 2)
k_fit_c2(Packed P, FitCfgDev cfg, float* __restrict__ theta, float* __restrict__ alpha,
         float* __restrict__ beta, float* __restrict__ opt, double* __restrict__ lnl_out,
         int32_t* __restrict__ iters_out, int32_t* __restrict__ status,
         float* __restrict__ trace, int* __restrict__ counter) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wid = threadIdx.x >> 5;
  const C2Lane L(smem + wid * C2::per_warp);
  const int D = P.D;
  const int64_t nunits = (P.W + C2::GW - 1) / C2::GW;
  for (;;) {
    int64_t unit = 0;
    if (L.lane == 0) unit = atomicAdd(counter, 1);
    unit = __shfl_sync(kFull, unit, 0);
    if (unit >= nunits) break;
    const int64_t slot = unit * C2::GW + L.g;
    const int64_t w = slot < P.W ? P.perm[slot] : 0;
    MDHP_ASSERT(w >= 0 && w < (P.W > 0 ? P.W : 1));
    const int st0 = slot < P.W ? status[w] : MDHP_ST_INVALID;
    const bool live = slot < P.W && !(st0 & MDHP_ST_INVALID);
    float2 th = c2_load_params(L, D, w, live, theta, alpha, beta);
    const int n = live ? P.n[w] : 0;
    const float scale = (cfg.loss_mean && n > 0) ? 1.0f / (float)n : 1.0f;
    int it = 0, s = 0, halv = 0, stall = 0, st = 0;
    float lr_w = cfg.lr;
    double lnl_prev = 0.0;
    bool have_prev = false, have_lnl = false;
    bool done = !live || cfg.max_iters <= 0;
    while (__any_sync(kFull, !done)) {
      const int nmax = group_max_i<8>(done ? 0 : n);
      float2 dth;
      bool finite;
      const double lnl = c2_eval<true>(P, L, w, !done, nmax, th, dth, finite);
      if (!done) {
        if (!finite) {
          st |= MDHP_ST_NONFINITE;
          if (!have_prev || halv >= cfg.max_halvings) {
            st |= MDHP_ST_DIVERGED;
            done = true;
            if (have_prev) th = c2_load_params(L, D, w, true, theta, alpha, beta);
          } else {
            th = c2_load_params(L, D, w, true, theta, alpha, beta);
            lr_w *= 0.5f;
            halv++;
            it++;
          }
        } else {
          if (trace && L.c == 0) trace[(size_t)w * cfg.max_iters + it] = (float)lnl;
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
            c2_store(L, D, w, th, theta, alpha, beta);   // previous point
            have_prev = true;
            s++;
            c2_step(L, D, w, cfg, lr_w, s, scale, dth, th, opt);
            it++;
          }
        }
        if (it >= cfg.max_iters) done = true;
      }
      __syncwarp();
    }
    const int nmax = group_max_i<8>(n);
    float2 dth;
    bool finite;
    const double lnl = c2_eval<false>(P, L, w, live, nmax, th, dth, finite);
    if (slot < P.W) {
      if (live) c2_store(L, D, w, th, theta, alpha, beta);
      if (L.c == 0) {
        lnl_out[w] = live ? lnl : (double)NAN;
        iters_out[w] = it;
        status[w] = st0 | st;
        if (trace && live)
          for (int q = it; q < cfg.max_iters; q++) trace[(size_t)w * cfg.max_iters + q] = NAN;
      }
    }
    __syncwarp();
  }
}

int loglik_launch_c2(const Packed& P, const float* th, const float* al, const float* be,
                     double* lnl, float* gt, float* ga, float* gb, const int32_t* status,
                     cudaStream_t st) {
  const size_t smem = kC2WPB * C2::per_warp;
  if (cudaFuncSetAttribute(k_loglik_c2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("cudaFuncSetAttribute(k_loglik_c2) failed");
    return MDHP_ECUDA;
  }
  const int64_t units = (P.W + C2::GW - 1) / C2::GW;
  const unsigned blocks = (unsigned)((units + kC2WPB - 1) / kC2WPB);
  k_loglik_c2<<<blocks, kC2WPB * 32, smem, st>>>(P, th, al, be, lnl, gt, ga, gb, status);
  count_launch();
  return MDHP_OK;
}

int fit_launch_c2(const Packed& P, const FitCfgDev& cfg, float* th, float* al, float* be,
                  float* opt, double* lnl, int32_t* iters, int32_t* status, float* trace,
                  int* counter, cudaStream_t st) {
  const size_t smem = kC2WPB * C2::per_warp;
  if (cudaFuncSetAttribute(k_fit_c2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("cudaFuncSetAttribute(k_fit_c2) failed");
    return MDHP_ECUDA;
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fit_c2, kC2WPB * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t units = (P.W + C2::GW - 1) / C2::GW;
  int64_t blocks = (int64_t)sms * per_sm;
  const int64_t need = (units + kC2WPB - 1) / kC2WPB;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  k_fit_c2<<<(unsigned)blocks, kC2WPB * 32, smem, st>>>(P, cfg, th, al, be, opt, lnl, iters, status,
                                                        trace, counter);
  count_launch();
  return MDHP_OK;
}

}  // namespace mdhp
