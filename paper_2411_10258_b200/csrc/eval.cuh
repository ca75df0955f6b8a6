// eval.cuh — per-window evaluation of Eq.(5) and its gradient on sm_100a (rows a2-a5 of
// DESIGN.md section 4).
//
// Mapping: a window is owned by a GROUP of DP lanes (DP = D padded to a power of two), so a
// warp holds G = 32/DP windows.  Lane j of a group owns source column j for the row read and
// target row j for the column update.  The per-window state lives in shared memory:
//   K[i][j] = {alpha_ij, beta_ij, S_ij, Q'_ij}  (row stride DP+1 float4: conflict-free rows
//                                                and columns)
//   G[i][j] = {gR_ij, gQ_ij}                    gradient accumulators
// where S_ij = sum_{k in j} e^{-beta_ij (last_j - t_k)} is anchored at last_j, the time of the
// latest event of source j, and Q'_ij = sum_{k in j} (last_j - t_k) e^{-beta_ij (last_j - t_k)}.
//
// Event n (time t, mark i), lazily (2 D exponentials per event instead of the D^2 of an eager
// update, and O(N D) work instead of the paper's O(N^2) tMpT broadcast):
//   row read  (lane j):  e = 2^{-beta_ij (t - last_j) log2 e};  R = e S_ij - [last_j == t]
//                        Q = e (Q'_ij + (t - last_j) S_ij);   lambda = theta_i + sum_j alpha_ij R
//                        (warp-shuffle reduction over the group);  w = 1/lambda;
//                        sum ln lambda += lg2(lambda) ln 2;  gR_ij += R w;  gQ_ij += Q w;
//                        g_theta_i += w   (Eq.(2) P:107 with the strict T_j^k < t, R2)
//   column update (lane j = target row, source i):  d = 2^{-beta_ji (t - last_i) log2 e};
//                        Q'_ji = d (Q'_ji + (t - last_i) S_ji);  S_ji = d S_ji + 1;  last_i = t
// The "[last_j == t]" term removes a cross-mark event at exactly t (tie groups, R2/R10).
//
// Epilogue (Part2, Part3 of Eq.(5) and the compensator gradients, App. B), per (i,j):
//   beta u_max > 2:  E_ij = e^{-beta (T-last_j)} S_ij - N_j,  F_ij = e^{..}(Q'_ij + (T-last_j) S_ij),
//                    E/beta,  H/beta^2 = (-E - beta F)/beta^2
//   beta u_max <= 2: power series in x = beta u_max with the packed moments m_p (exact to
//                    ~1e-10 relative, no cancellation as beta -> 0; R20)
//   lnL = ln2 sum lg2(lambda) - T sum theta + sum alpha E/beta
//   d alpha = gR + E/beta;   d beta = -alpha gQ + alpha H/beta^2;   d theta = g_theta - T
#pragma once
#include "common.cuh"

namespace mdhp {

__constant__ float c_inv_fact[kMom + 1] = {
    1.0f, 1.0f, 0.5f, 1.6666666666666666e-01f, 4.1666666666666664e-02f, 8.3333333333333332e-03f,
    1.3888888888888889e-03f, 1.9841269841269841e-04f, 2.4801587301587302e-05f,
    2.7557319223985893e-06f, 2.7557319223985888e-07f, 2.5052108385441720e-08f,
    2.0876756987868100e-09f, 1.6059043836821613e-10f, 1.1470745597729725e-11f,
    7.6471637318198164e-13f, 4.7794773323873853e-14f, 2.8114572543455206e-15f};

template <int DP>
struct Smem {
  static constexpr int G = 32 / DP;                 // windows (groups) per warp
  static constexpr int KS = DP * (DP + 1);          // float4 per group in K
  static constexpr int GS = DP * DP;                // float2 per group in G
  static constexpr size_t per_warp = (size_t)G * (KS * sizeof(float4) + GS * sizeof(float2));
};

// Zero the dynamic state (S, Q', gR, gQ) of this lane's column j.
template <int DP>
__device__ __forceinline__ void reset_state(float4* K, float2* Gs, int j) {
#pragma unroll
  for (int i = 0; i < DP; i++) {
    float4* p = &K[i * (DP + 1) + j];
    p->z = 0.0f;
    p->w = 0.0f;
    Gs[i * DP + j] = make_float2(0.0f, 0.0f);
  }
}

// The event loop of one window-evaluation.  All 32 lanes must call it (shuffles); groups whose
// window has fewer events than `nmax` (the max over the warp) idle through the tail.
// Returns via references: last (time of the latest event of source j), gth (sum 1/lambda over
// events of mark j) and lsum (sum over events of lg2 lambda; identical in all lanes of a group).
template <int DP, bool GRAD>
__device__ __forceinline__ void event_loop(float4* __restrict__ K, float2* __restrict__ Gs,
                                           const int j, const int gbase,
                                           const float* __restrict__ t32,
                                           const float* __restrict__ dtp,
                                           const uint8_t* __restrict__ mk, const int64_t beg,
                                           const int n, const int nmax, const float th,
                                           float& last, float& gth, double& lsum) {
  last = -1.0f;
  gth = 0.0f;
  lsum = 0.0;
  float4 ta = make_float4(0, 0, 0, 0), tb = ta, da = ta, db = ta;
  uint2 mm = make_uint2(0, 0);
  if (n > 0) {
    const float4* tp = reinterpret_cast<const float4*>(t32 + beg);
    const float4* dp = reinterpret_cast<const float4*>(dtp + beg);
    ta = __ldg(tp);
    tb = __ldg(tp + 1);
    da = __ldg(dp);
    db = __ldg(dp + 1);
    mm = __ldg(reinterpret_cast<const uint2*>(mk + beg));
  }
  for (int base = 0; base < nmax; base += 8) {
    // prefetch the next chunk of 8 events (broadcast loads: every lane of the group reads
    // the same 16-byte words; L1/L2 resident across fit iterations)
    float4 nta = ta, ntb = tb, nda = da, ndb = db;
    uint2 nmm = mm;
    if (base + 8 < n) {
      const float4* tp = reinterpret_cast<const float4*>(t32 + beg + base + 8);
      const float4* dp = reinterpret_cast<const float4*>(dtp + beg + base + 8);
      nta = __ldg(tp);
      ntb = __ldg(tp + 1);
      nda = __ldg(dp);
      ndb = __ldg(dp + 1);
      nmm = __ldg(reinterpret_cast<const uint2*>(mk + beg + base + 8));
    }
    float lacc = 0.0f;
#pragma unroll
    for (int s = 0; s < 8; s++) {
      const bool act = base + s < n;
      const float t = s == 0 ? ta.x : s == 1 ? ta.y : s == 2 ? ta.z : s == 3 ? ta.w
                    : s == 4 ? tb.x : s == 5 ? tb.y : s == 6 ? tb.z : tb.w;
      const float dc = s == 0 ? da.x : s == 1 ? da.y : s == 2 ? da.z : s == 3 ? da.w
                     : s == 4 ? db.x : s == 5 ? db.y : s == 6 ? db.z : db.w;
      const unsigned word = s < 4 ? mm.x : mm.y;
      int i = (int)((word >> (8 * (s & 3))) & 0xffu);
      i = act ? i : 0;
      const float4 kr = K[i * (DP + 1) + j];
      const float4 kc = K[j * (DP + 1) + i];
      const float dr = t - last;
      const float er = ex2f(kr.y * (dr * -kLog2e));
      const float ec = ex2f(kc.y * (dc * -kLog2e));
      const float tie = (dr == 0.0f) ? 1.0f : 0.0f;
      const float R = fmaf(er, kr.z, -tie);
      float p = kr.x * R;
      p = group_sum<DP>(p);
      const float lam = p + __shfl_sync(kFull, th, gbase + i);
      if (GRAD) {
        const float Q = er * fmaf(dr, kr.z, kr.w);
        const float w = rcpf(lam);
        float2 gg = Gs[i * DP + j];
        gg.x = fmaf(R, w, gg.x);
        gg.y = fmaf(Q, w, gg.y);
        if (act) Gs[i * DP + j] = gg;
        gth += (act && i == j) ? w : 0.0f;
      }
      lacc += act ? lg2f(lam) : 0.0f;
      const float Sn = fmaf(ec, kc.z, 1.0f);
      const float Qn = ec * fmaf(dc, kc.z, kc.w);
      if (act) {
        float2* pc = reinterpret_cast<float2*>(&K[j * (DP + 1) + i]) + 1;
        *pc = make_float2(Sn, Qn);
        if (i == j) last = t;
      }
      __syncwarp();
    }
    lsum += (double)lacc;
    ta = nta; tb = ntb; da = nda; db = ndb; mm = nmm;
  }
}

// Per-lane epilogue data of source column j.
struct ColInfo {
  float T, last, umax;
  int N;       // events of mark j
  bool real;   // j < D
};

// Series coefficients for the small-beta branch (column j): E/beta = umax * sum_p c_p x^(p-1),
// H/beta^2 = umax^2 * sum_{p>=2} h_p x^(p-2), with c_p = (-1)^p m_p / p!, h_p = (p-1) c_p.
struct Series {
  float c[kMom - 1];   // c_1..c_16
};

__device__ __forceinline__ void load_series(Series& S, const float* __restrict__ mom, bool have) {
#pragma unroll
  for (int p = 1; p < kMom; p++) {
    const float m = have ? __ldg(mom + (p - 1)) : 0.0f;
    const float c = m * c_inv_fact[p];
    S.c[p - 1] = (p & 1) ? -c : c;
  }
}

// E/beta and H/beta^2 of pair (i, j) given its state; see the header comment.
__device__ __forceinline__ void compensator(const ColInfo& ci, const Series& S, float b, float Sij,
                                            float Qij, float& Eb, float& Hb2) {
  if (ci.N == 0) {
    Eb = 0.0f;
    Hb2 = 0.0f;
    return;
  }
  const float x = b * ci.umax;
  if (x <= 2.0f) {
    float e = S.c[kMom - 2];
#pragma unroll
    for (int p = kMom - 3; p >= 0; p--) e = fmaf(e, x, S.c[p]);
    float h = 15.0f * S.c[kMom - 2];
#pragma unroll
    for (int p = kMom - 3; p >= 1; p--) h = fmaf(h, x, (float)p * S.c[p]);
    Eb = ci.umax * e;
    Hb2 = ci.umax * ci.umax * h;
  } else {
    const float dl = ci.T - ci.last;
    const float e = ex2f(b * (dl * -kLog2e));
    const float E = fmaf(e, Sij, -(float)ci.N);
    const float F = e * fmaf(dl, Sij, Qij);
    const float ib = 1.0f / b;
    Eb = E * ib;
    Hb2 = (-E - b * F) * ib * ib;
  }
}

}  // namespace mdhp
