// eval_c2.cuh — D = 16 (Dp = 16) evaluation with 8 lanes per window and two columns per lane,
// 4 windows per warp (the "C2" mapping; rows a2-a5).
//
// Same arithmetic as eval.cuh, different ownership: lane c of a group owns source columns c and
// c+8 (row reads, gradient accumulators) and target rows c and c+8 (column updates), so the
// per-event overhead (mark decode, addressing, reduction, selects, loop) is shared by 4 events
// per warp-step instead of 2.
//
// Shared-memory layout.  Two windows (h = 0, 1: groups 2p and 2p+1, the two halves of one
// half-warp) share a "pair arena".  Every 128-byte line holds 8 float2 of window 0 (units 0-7)
// and 8 of window 1 (units 8-15), so 64-bit accesses of the two windows never meet in a bank.
// Entry (r, col) of window h, r in 0..16 (16 = the null row), col in 0..15:
//     byte = (2 r + col / 8) * 128 + 64 h + 8 * ((col + r) mod 8)
// Row r, columns c and c+8 of lane c: 8 distinct slots, second column at +128 B.
// Column i, rows c and c+8 of lane c: 8 distinct slots (the skew), second row at +2048 B.
// Null events (mark 16) read the null row (lambda = 1) and rewrite the column-16 entries they
// read with an increment of 0 (an identity), so no storage beyond row 16 is needed.
#pragma once
#include "eval.cuh"

namespace mdhp {

struct C2 {
  static constexpr int DP = 16;
  static constexpr int LW = 8;                          // lanes per window
  static constexpr int GW = 4;                          // windows per warp
  static constexpr int ROWB = 256;                      // bytes per row (2 lines)
  static constexpr int ARR = (DP + 1) * ROWB;           // one array (rows 0..16) of a pair
  static constexpr int PAIR = 3 * ARR;                  // A, SQ, G
  static constexpr size_t per_warp = 2 * PAIR;          // 26112 B
};

struct C2Lane {
  int lane, g, c, h, pair;
  unsigned gmask;
  char* A;    // pair arena arrays
  char* SQ;
  char* G;
  int rowc;   // 64 h
  int colc;   // 256 c + 64 h
  __device__ C2Lane(unsigned char* warp_smem) {
    lane = threadIdx.x & 31;
    g = lane >> 3;
    c = lane & 7;
    h = g & 1;
    pair = g >> 1;
    gmask = 0xffu << (8 * g);
    char* base = reinterpret_cast<char*>(warp_smem) + pair * C2::PAIR;
    A = base;
    SQ = base + C2::ARR;
    G = base + 2 * C2::ARR;
    rowc = 64 * h;
    colc = 256 * c + 64 * h;
  }
  // byte offset of entry (r, col) of this lane's window
  __device__ __forceinline__ int off(int r, int col) const {
    return (2 * r + (col >> 3)) * 128 + 64 * h + 8 * ((col + r) & 7);
  }
};

template <typename T>
__device__ __forceinline__ T& at2(char* base, int off) {
  return *reinterpret_cast<T*>(base + off);
}

// Zero S, Q', gR, gQ of this lane's columns (all rows), set the null row (S = 1 at column 0).
__device__ __forceinline__ void c2_reset(const C2Lane& L) {
#pragma unroll
  for (int r = 0; r < C2::DP; r++) {
    const int o0 = L.off(r, L.c);
    at2<float2>(L.SQ, o0) = make_float2(0.0f, 0.0f);
    at2<float2>(L.SQ, o0 + 128) = make_float2(0.0f, 0.0f);
    at2<float2>(L.G, o0) = make_float2(0.0f, 0.0f);
    at2<float2>(L.G, o0 + 128) = make_float2(0.0f, 0.0f);
  }
  const int on = L.off(C2::DP, L.c);
  at2<float2>(L.SQ, on) = make_float2(L.c == 0 ? 1.0f : 0.0f, 0.0f);
  at2<float2>(L.SQ, on + 128) = make_float2(0.0f, 0.0f);
}

// Load alpha, beta of this lane's columns; null row {1, 0} at column 0, {0, 0} elsewhere.
// Returns theta of columns c and c+8 (0 for padded / dead).
__device__ __forceinline__ float2 c2_load_params(const C2Lane& L, int D, int64_t w, bool live,
                                                 const float* __restrict__ theta,
                                                 const float* __restrict__ alpha,
                                                 const float* __restrict__ beta) {
#pragma unroll
  for (int q = 0; q < 2; q++) {
    const int j = L.c + 8 * q;
    const bool real = live && j < D;
#pragma unroll 4
    for (int r = 0; r < C2::DP; r++) {
      float a = 0.0f, b = 1.0f;
      if (real && r < D) {
        a = alpha[(size_t)w * D * D + (size_t)r * D + j];
        b = beta[(size_t)w * D * D + (size_t)r * D + j];
      }
      at2<float2>(L.A, L.off(r, j)) = make_float2(a, b);
    }
    at2<float2>(L.A, L.off(C2::DP, j)) = make_float2(j == 0 ? 1.0f : 0.0f, 0.0f);
  }
  const float t0 = (live && L.c < D) ? theta[(size_t)w * D + L.c] : 0.0f;
  const float t1 = (live && L.c + 8 < D) ? theta[(size_t)w * D + L.c + 8] : 0.0f;
  return make_float2(t0, t1);
}

// One chunk of 8 events for the 4 windows of the warp.
template <bool GRAD>
__device__ __forceinline__ void c2_chunk(const Chunk& ck, const C2Lane& L, float2 th,
                                         float& lastA, float& lastB, float& gthA, float& gthB,
                                         double& lsum) {
  constexpr int DP = C2::DP;
  const int c = L.c;
  float pv[8], R0[8], R1[8], Q0[8], Q1[8];
  float lacc = 0.0f;
#pragma unroll
  for (int s = 0; s < 8; s++) {
    const float t = s == 0 ? ck.ta.x : s == 1 ? ck.ta.y : s == 2 ? ck.ta.z : s == 3 ? ck.ta.w
                  : s == 4 ? ck.tb.x : s == 5 ? ck.tb.y : s == 6 ? ck.tb.z : ck.tb.w;
    const float dc = s == 0 ? ck.da.x : s == 1 ? ck.da.y : s == 2 ? ck.da.z : s == 3 ? ck.da.w
                   : s == 4 ? ck.db.x : s == 5 ? ck.db.y : s == 6 ? ck.db.z : ck.db.w;
    const unsigned word = s < 4 ? ck.mm.x : ck.mm.y;
    const int i = (int)__byte_perm(word, 0u, 0x4440u | (unsigned)(s & 3));   // mark (null: 16)
    MDHP_ASSERT(i >= 0 && i <= DP);
    const int sk = ((c + i) & 7) * 8;
    const int ro = i * 256 + L.rowc + sk;                 // (i, c); (i, c+8) at +128
    const int co = (i >> 3) * 128 + L.colc + sk;          // (c, i); (c+8, i) at +2048
    const float2 a0 = at2<float2>(L.A, ro), a1 = at2<float2>(L.A, ro + 128);
    const float2 s0 = at2<float2>(L.SQ, ro), s1 = at2<float2>(L.SQ, ro + 128);
    const float b0 = at2<float2>(L.A, co).y, b1 = at2<float2>(L.A, co + 2048).y;
    const float2 q0 = at2<float2>(L.SQ, co), q1 = at2<float2>(L.SQ, co + 2048);
    const float d0 = t - lastA, d1 = t - lastB;
    const float e0 = ex2f(a0.y * (d0 * -kLog2e)), e1 = ex2f(a1.y * (d1 * -kLog2e));
    const float nd = dc * -kLog2e;
    const float f0 = ex2f(b0 * nd), f1 = ex2f(b1 * nd);
    const float r0 = fmaf(e0, s0.x, fsel_eqf(d0, 0.0f, -1.0f, 0.0f));   // strict T_j^k < t
    const float r1 = fmaf(e1, s1.x, fsel_eqf(d1, 0.0f, -1.0f, 0.0f));
    const float thi = fsel_eqi(i, c, th.x, fsel_eqi(i, c + 8, th.y, 0.0f));
    pv[s] = fmaf(a0.x, r0, fmaf(a1.x, r1, thi));
    const float add = fsel_eqi(i, DP, 0.0f, 1.0f);      // null event: identity rewrite
    at2<float2>(L.SQ, co) = make_float2(fmaf(f0, q0.x, add), f0 * fmaf(dc, q0.x, q0.y));
    at2<float2>(L.SQ, co + 2048) = make_float2(fmaf(f1, q1.x, add), f1 * fmaf(dc, q1.x, q1.y));
    lastA = fsel_eqi(i, c, t, lastA);
    lastB = fsel_eqi(i, c + 8, t, lastB);
    if (GRAD) {
      R0[s] = r0;
      R1[s] = r1;
      Q0[s] = e0 * fmaf(d0, s0.x, s0.y);
      Q1[s] = e1 * fmaf(d1, s1.x, s1.y);
    }
    __syncwarp();
  }
  const float lam = reduce_scatter8<8>(pv, c);   // lane c: intensity of event c of its window
  lacc += lg2f(lam);
  if (GRAD) {
    const float w = rcpf(lam);
#pragma unroll
    for (int s = 0; s < 8; s++) {
      const float ws = __shfl_sync(kFull, w, 8 * L.g + s);
      const unsigned word = s < 4 ? ck.mm.x : ck.mm.y;
      const int i = (int)__byte_perm(word, 0u, 0x4440u | (unsigned)(s & 3));
      const int ro = i * 256 + L.rowc + ((c + i) & 7) * 8;
      float2 g0 = at2<float2>(L.G, ro), g1 = at2<float2>(L.G, ro + 128);
      g0.x = fmaf(R0[s], ws, g0.x);
      g0.y = fmaf(Q0[s], ws, g0.y);
      g1.x = fmaf(R1[s], ws, g1.x);
      g1.y = fmaf(Q1[s], ws, g1.y);
      at2<float2>(L.G, ro) = g0;
      at2<float2>(L.G, ro + 128) = g1;
      gthA += fsel_eqi(i, c, ws, 0.0f);
      gthB += fsel_eqi(i, c + 8, ws, 0.0f);
    }
  }
  lsum += (double)lacc;
}

template <bool GRAD>
__device__ __forceinline__ void c2_event_loop(const C2Lane& L, const float* __restrict__ t32,
                                              const float* __restrict__ dtp,
                                              const uint8_t* __restrict__ mk, int64_t beg, int n,
                                              int nmax, float2 th, float& lastA, float& lastB,
                                              float& gthA, float& gthB, double& lsum) {
  lastA = -1.0f;
  lastB = -1.0f;
  gthA = 0.0f;
  gthB = 0.0f;
  lsum = 0.0;
  const float* tw = t32 + beg;
  const float* dw = dtp + beg;
  const uint8_t* mw = mk + beg;
  const int npad = (n + 7) & ~7;
  MDHP_ASSERT(n >= 0 && nmax >= n);
  Chunk c0, c1;
  load_chunk(c0, tw, dw, mw, 0 < n ? 0 : npad);
  for (int base = 0; base < nmax; base += 16) {
    load_chunk(c1, tw, dw, mw, min(base + 8, npad));
    c2_chunk<GRAD>(c0, L, th, lastA, lastB, gthA, gthB, lsum);
    load_chunk(c0, tw, dw, mw, min(base + 16, npad));
    c2_chunk<GRAD>(c1, L, th, lastA, lastB, gthA, gthB, lsum);
  }
}

// Per-window evaluation (event loop + epilogue).  On return (GRAD) the G arena holds
// (d alpha, d beta) for this lane's columns; dth = d theta for columns c, c+8.
template <bool GRAD>
__device__ __forceinline__ double c2_eval(const Packed& P, const C2Lane& L, int64_t w, bool live,
                                          int nmax, float2 th, float2& dth, bool& finite) {
  c2_reset(L);
  __syncwarp();
  const int n = live ? P.n[w] : 0;
  const int64_t beg = live ? P.begin[w] : 0;
  float lastA, lastB, gthA, gthB;
  double lsum;
  c2_event_loop<GRAD>(L, P.t32, P.dtp, P.mark, beg, n, nmax, th, lastA, lastB, gthA, gthB, lsum);
  const int D = P.D;
  const float T = live ? P.T32[w] : 1.0f;
  double part3 = 0.0;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 2; q++) {
    const int j = L.c + 8 * q;
    ColInfo ci;
    ci.real = j < D;
    ci.T = T;
    ci.N = live ? P.cnt[w * P.Dp + j] : 0;
    ci.umax = live ? P.umax[w * P.Dp + j] : 0.0f;
    ci.last = q == 0 ? lastA : lastB;
    Series S;
    load_series(S, P.mom + ((size_t)(live ? w : 0) * P.Dp + j) * kMom, live && ci.N > 0);
#pragma unroll 4
    for (int r = 0; r < C2::DP; r++) {
      const int o = L.off(r, j);
      const float2 k = at2<float2>(L.A, o);
      const float2 sq = at2<float2>(L.SQ, o);
      float Eb, Hb2;
      compensator(ci, S, k.y, sq.x, sq.y, Eb, Hb2);
      if (ci.real && r < D) {
        part3 += (double)(k.x * Eb);
        if (GRAD) {
          const float2 gg = at2<float2>(L.G, o);
          const float da = gg.x + Eb;
          const float db = fmaf(-k.x, gg.y, k.x * Hb2);
          ok = ok && isfinite(da) && isfinite(db);
          at2<float2>(L.G, o) = make_float2(da, db);
        }
      }
    }
  }
  dth = make_float2(gthA - T, gthB - T);
  if (GRAD) {
    if (L.c < D) ok = ok && isfinite(dth.x);
    if (L.c + 8 < D) ok = ok && isfinite(dth.y);
  }
  part3 = group_sum_d<8>(part3);
  lsum = group_sum_d<8>(lsum);
  double sthv = 0.0;
  if (L.c < D) sthv += (double)th.x;
  if (L.c + 8 < D) sthv += (double)th.y;
  const double sth = group_sum_d<8>(sthv);
  const double lnl = (double)kLn2 * lsum + part3 - (double)T * sth;
  const unsigned bal = __ballot_sync(kFull, ok) & L.gmask;
  finite = (bal == L.gmask) && isfinite(lnl);
  return lnl;
}

}  // namespace mdhp
