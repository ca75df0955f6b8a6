// eval.cuh — per-window evaluation of Eq.(5) and its gradient on sm_100a (rows a2-a5 of
// DESIGN.md section 4).
//
// Mapping: a window is owned by a GROUP of DP lanes (DP = D padded to a power of two), so a
// warp holds G = 32/DP windows.  Lane j of a group owns source column j for the row read and
// target row j for the column update.  The per-window state lives in shared memory as three
// float2 arrays (64-bit accesses are served per half-warp, so with an odd row stride DP+1 both
// row and column accesses of a group are bank-conflict free; measured in profiles/):
//   A[i][j]  = {alpha_ij, beta_ij}      parameters (row stride DP+1)
//   SQ[i][j] = {S_ij, Q'_ij}            recurrence state (row stride DP+1)
//   G[i][j]  = {gR_ij, gQ_ij}           gradient accumulators (row stride DP; rows only)
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
  // DP >= 16: each group owns (DP+1) x (DP+1) arrays with odd row stride DP+1 (row and column
  //   accesses of a group's 16 or 32 lanes are conflict-free).
  // DP <= 8 (SW, swizzled): the 16/DP groups of a half-warp share rows of 16 float2 (128 B):
  //   group h of the half-warp owns float2 DP*h .. DP*h+DP-1 of every row, and element (r, c)
  //   sits at 16 r + ((c ^ r) & (DP-1)) from the group's base, so a row read (lanes c) and a
  //   column access (lanes r) of each group hit DP distinct 8-byte bank pairs inside the
  //   group's own half of the 16 pairs: 64-bit accesses of a half-warp are conflict-free
  //   whatever the groups' marks (the odd-stride layout measured 46% excess wavefronts at
  //   DP = 8, profiles/r02_cfg2_*).  The null column (index DP) has no storage there: the
  //   event loop never stores to it and nothing reads it.
  static constexpr bool SW = DP <= 8;
  static constexpr int RS = SW ? 16 : DP + 1;       // row stride of A and SQ (float2 units)
  static constexpr int AS = (DP + 1) * RS;          // float2 from A to SQ (and SQ to G): DP
                                                    // real rows + the null row DP
  static constexpr int GS = SW ? AS : (DP + 1) * DP;   // float2 of G (+ null row)
  // DP = 8: NGC copies of G, event s of a chunk accumulating into copy s % NGC, so pass 2's
  // read-modify-writes of NGC consecutive events are independent and issue together (the
  // serial LDS -> FFMA -> STS chain of the 8 events was ~30% of the latency-bound cfg2 loop,
  // profiles/r02_cfg2_*); readers add the copies (gsum).  At DP = 16/32 the kernels are bound
  // by shared-memory throughput, not latency, and keep one copy.
  static constexpr int NGC = DP == 8 ? 4 : 1;
  static constexpr int P = SW ? 16 / DP : 1;        // groups sharing one row block
  static constexpr int per_group = 2 * AS + NGC * GS;   // float2 per group (SW: per block of P)
  static constexpr size_t per_warp = (size_t)(G / P) * per_group * sizeof(float2);
  // float2 offset of group g's A from the warp's base
  __host__ __device__ static constexpr int group_off(int g) {
    return SW ? (g / P) * per_group + (g % P) * DP : g * per_group;
  }
  // float2 offset of element (r, c) of A / SQ (e) and of G (ge) from the array base
  __host__ __device__ static constexpr int e(int r, int c) {
    return SW ? r * 16 + ((c ^ r) & (DP - 1)) : r * (DP + 1) + c;
  }
  __host__ __device__ static constexpr int ge(int r, int c) {
    return SW ? r * 16 + ((c ^ r) & (DP - 1)) : r * DP + c;
  }
};

// Gradient accumulator (r, c) summed over the NGC copies (fixed order), and zeroing of all
// copies.  Gs = the group's G base (A + 2 AS).
template <int DP>
__device__ __forceinline__ float2 gsum(const float2* Gs, int r, int c) {
  using SM = Smem<DP>;
  float2 a = Gs[SM::ge(r, c)];
#pragma unroll
  for (int k = 1; k < SM::NGC; k++) {
    const float2 v = Gs[k * SM::GS + SM::ge(r, c)];
    a.x += v.x;
    a.y += v.y;
  }
  return a;
}
template <int DP>
__device__ __forceinline__ void gzero(float2* Gs, int r, int c) {
  using SM = Smem<DP>;
#pragma unroll
  for (int k = 0; k < SM::NGC; k++) Gs[k * SM::GS + SM::ge(r, c)] = make_float2(0.0f, 0.0f);
}

// Parameter pair order in A.  Half of the pairs are stored {beta, alpha} instead of
// {alpha, beta}, chosen so that the 32-bit beta column read of the event loop hits even banks
// in one half-warp and odd banks in the other (one wavefront instead of two; 7% of all shared
// wavefronts at D = 16) for two selects per event in the row read:
//   DP <= 16: the upper half-warp (lanes 16-31; whole groups) stores its pairs swapped.
//   DP == 32 (one window per warp) would have to swap by row (r >= 16), which needs a per-event
//   predicate in the row read; measured 1% slower on cfg3, so DP = 32 keeps one order.
// Every access to A goes through these helpers (r = row index of the pair).
template <int DP>
__device__ __forceinline__ bool ab_swapped(int r) {
  (void)r;
  return DP <= 16 && (threadIdx.x & 16) != 0;
}
template <int DP>
__device__ __forceinline__ float2 ab_pack(int r, float a, float b) {
  return ab_swapped<DP>(r) ? make_float2(b, a) : make_float2(a, b);
}
template <int DP>
__device__ __forceinline__ float ab_alpha(int r, float2 k) {
  return ab_swapped<DP>(r) ? k.y : k.x;
}
template <int DP>
__device__ __forceinline__ float ab_beta(int r, float2 k) {
  return ab_swapped<DP>(r) ? k.x : k.y;
}

// The null dimension DP.  A padding slot or the tail of a shorter window in the warp is the
// event (t = -2, gap 0, mark DP).  With row DP = {alpha, beta} = {1, 0} at column 0 and {0, 0}
// elsewhere, S_DP,0 = 1 and column DP's beta = 0, such an event reads lambda = 1 exactly
// (lg2 = 0), never ties (t < every last >= -1), only touches column DP (never read by a real
// row) and accumulates its gradient terms into the never-read row DP of G.  So the event loop
// needs no per-event predicate.
constexpr float kNullT = -2.0f;

// Zero the dynamic state (S, Q', gR, gQ) of this lane's column j and its row-j entry of the
// null column; (re)set the null row.
template <int DP>
__device__ __forceinline__ void reset_state(float2* SQ, float2* Gs, int j) {
  using SM = Smem<DP>;
#pragma unroll
  for (int i = 0; i < DP; i++) {
    SQ[SM::e(i, j)] = make_float2(0.0f, 0.0f);
    gzero<DP>(Gs, i, j);
  }
  SQ[SM::e(DP, j)] = make_float2(j == 0 ? 1.0f : 0.0f, 0.0f);
  if constexpr (!SM::SW) SQ[SM::e(j, DP)] = make_float2(0.0f, 0.0f);
}

// Reduce-scatter of 8 per-lane values v[0..7] over the DP lanes of a group (DP >= 8): on
// return v[0] holds the group sum of value e = (j >> (log2 DP - 3)) & 7.  8 shuffles for 8 sums
// (DP = 16) instead of 8 x log2(DP) for 8 butterflies.
template <int DP>
__device__ __forceinline__ float reduce_scatter8(float (&v)[8], int j) {
  {
    const bool hi = (j & (DP / 2)) != 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const float mine = hi ? v[4 + k] : v[k];
      const float oth = hi ? v[k] : v[4 + k];
      v[k] = mine + __shfl_xor_sync(kFull, oth, DP / 2);
    }
  }
  {
    const bool hi = (j & (DP / 4)) != 0;
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const float mine = hi ? v[2 + k] : v[k];
      const float oth = hi ? v[k] : v[2 + k];
      v[k] = mine + __shfl_xor_sync(kFull, oth, DP / 4);
    }
  }
  {
    const bool hi = (j & (DP / 8)) != 0;
    const float mine = hi ? v[1] : v[0];
    const float oth = hi ? v[0] : v[1];
    v[0] = mine + __shfl_xor_sync(kFull, oth, DP / 8);
  }
#pragma unroll
  for (int o = DP / 16; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(kFull, v[0], o);
  return v[0];
}

template <int DP>
struct Log2 {
  static constexpr int v = DP <= 1 ? 0 : 1 + Log2<DP / 2>::v;
};
template <>
struct Log2<1> {
  static constexpr int v = 0;
};

// The event loop of one window-evaluation.  All 32 lanes must call it (shuffles); groups whose
// window has fewer events than `nmax` (the max over the warp) idle through the tail.
// Returns via references: last (time of the latest event of source j), gth (sum 1/lambda over
// events of mark j) and lsum (this lane's share of sum_n lg2 lambda_n; the group sum is the
// total).
//
// DP >= 8 processes events in chunks of 8: pass 1 does the row reads and column updates of the
// 8 events in order and keeps each event's partial sum alpha_ij R_ij (+ theta_i on lane i),
// R_ij and Q_ij in registers; one reduce-scatter gives every lane the intensity of one event
// (one rcp and one lg2 per lane per chunk instead of per event); pass 2 broadcasts w = 1/lambda
// per event (1 shuffle) and accumulates the gradients.  DP <= 4 reduces each event directly.
struct Chunk {
  float4 ta, tb, da, db;
  uint2 mm;
};

// Chunk loads use 32-bit event offsets from the window base.  Offsets past the window are
// clamped to its null chunk (the 8 null events the packer stores after every window), so
// every load is unconditional.
__device__ __forceinline__ void load_chunk(Chunk& c, const float* t32, const float* dtp,
                                           const uint8_t* mk, int off) {
  MDHP_ASSERT(off >= 0 && (off & 7) == 0);
  const float4* tp = reinterpret_cast<const float4*>(t32 + off);
  const float4* dp = reinterpret_cast<const float4*>(dtp + off);
  c.ta = __ldg(tp);
  c.tb = __ldg(tp + 1);
  c.da = __ldg(dp);
  c.db = __ldg(dp + 1);
  c.mm = __ldg(reinterpret_cast<const uint2*>(mk + off));
}

// (x == y) ? a : b as one compare + one FSEL (keeps the compiler from SEL + I2FP sequences)
__device__ __forceinline__ float fsel_eqf(float x, float y, float a, float b) {
  float r;
  asm("{\n\t.reg .pred p;\n\tsetp.eq.f32 p, %1, %2;\n\tselp.f32 %0, %3, %4, p;\n\t}"
      : "=f"(r) : "f"(x), "f"(y), "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fsel_eqi(int x, int y, float a, float b) {
  float r;
  asm("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, %2;\n\tselp.f32 %0, %3, %4, p;\n\t}"
      : "=f"(r) : "r"(x), "r"(y), "f"(a), "f"(b));
  return r;
}

// 1.0f if x == 0 else 0.0f, as one FSET (a select of -1/0 compiles to SEL + I2FP)
__device__ __forceinline__ float fset_eq0(float x) {
  float r;
  asm("set.eq.f32.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
  return r;
}

// Shared-memory accesses of the event loop through explicit 32-bit shared addresses: one
// IMAD/LEA per array per event (the compiler otherwise re-derives (j*RS + i)*8 + base with
// two or three integer ops).  The state (SQ, G) accesses are volatile with a memory clobber
// (their order carries the recurrence); the parameter loads (A, constant during an event
// loop) are plain asm so the compiler may hoist them across the state stores.
__device__ __forceinline__ float2 lda2(uint32_t a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
template <int OFF>
__device__ __forceinline__ float lda1o(uint32_t a) {
  float v;
  asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
  return v;
}
__device__ __forceinline__ float2 lds2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
template <int OFF>
__device__ __forceinline__ float2 lds2o(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2+%3];"
               : "=f"(v.x), "=f"(v.y) : "r"(a), "n"(OFF) : "memory");
  return v;
}
template <int OFF>
__device__ __forceinline__ float lds1o(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF) : "memory");
  return v;
}
__device__ __forceinline__ void sts1(uint32_t a, float x) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory");
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
template <int OFF>
__device__ __forceinline__ void sts2o(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0+%1], {%2, %3};" ::"r"(a), "n"(OFF), "f"(x), "f"(y)
               : "memory");
}

// One chunk of 8 events (see event_loop).  A, SQ, Gs are one group's arrays laid out
// contiguously (SQ = A + AS, Gs = A + 2 AS; Smem<DP>).  PRE: A holds beta' = -beta log2(e)
// (the fit and loglik kernels) instead of beta (the sequence path), so every exponential is
// ex2(beta' * dt) without the extra multiply.
template <int DP, bool GRAD, bool PRE, bool TC = false>
__device__ __forceinline__ void process_chunk(const Chunk& ck, const float2* __restrict__ A,
                                              float2* __restrict__ SQ, float2* __restrict__ Gs,
                                              const int j, const int gbase, const float th,
                                              float& last, float& gth, double& lsum,
                                              const float tb = 0.0f) {
  using SM = Smem<DP>;
  constexpr bool SW = SM::SW;
  constexpr int RS = SM::RS;
  constexpr int LG = Log2<DP>::v;
  constexpr int kSQ = SM::AS * 8, kG = 2 * SM::AS * 8;   // byte offsets from A
  MDHP_ASSERT(SQ == A + SM::AS && Gs == A + 2 * SM::AS);
  uint32_t sA = static_cast<uint32_t>(__cvta_generic_to_shared(A));
  // The parameter loads (lda*) are non-volatile asm so that ptxas may move them across the
  // state stores inside the chunk; every address derives from sA, which this empty volatile
  // asm (a compiler memory barrier) redefines here, so no parameter load is hoisted above the
  // start of the chunk -- i.e. above the parameter writes of the fit (opt_action,
  // load_window).  (Without it a loop-invariant address, e.g. Dp = 1, let the compiler hoist
  // the load out of the fit loop.)
  asm volatile("" : "+r"(sA) :: "memory");
  // per-lane bases.  Odd stride: row i of column j at rowb + i*RS*8, column i of row j at
  // colb + i*8, gradient row i of column j at rowb + kG + i*DP*8.  SW: element (r, c) at
  // sA + 128 r + 8 x with x = (c ^ r) & (DP-1); the row read (i, j) and the column access
  // (j, i) of an event share x = (i ^ j) & (DP-1); gradients at the row-read address + kG.
  const uint32_t rowb = SW ? sA : sA + 8u * j;
  const uint32_t colb = SW ? sA + 128u * j : sA + 8u * RS * j;
  // beta of a column pair: word 1, or word 0 where the pair is stored swapped
  const uint32_t colbb = colb + (ab_swapped<DP>(j) ? 0u : 4u);
  float pv[8], Rv[8], Qv[8];
  float lacc = 0.0f;
  // DP <= 8 and DP = 32 (latency-bound: few warps per SM): the column decay factors ec of the
  // chunk's 8 events depend only on parameters (beta'_ji) and gaps, so their loads and
  // exponentials are issued here, ahead of the chunk's state stores, which takes the beta load
  // and the MUFU off the event-to-event chain (state load -> FFMA -> state store).  (ptxas
  // cannot move the loads above the stores itself: it cannot prove the addresses disjoint.)
  // cfg3 (DP = 32) +4.6%; DP = 16 (bound by the shared-memory slot, not latency) unchanged.
  // SW: the addresses of the chunk's 8 events come from two byte-parallel words per 4 events:
  // y = 16 i + ((i ^ j) & (DP-1)) (the row element (i, j) in float2 units from the group base,
  // <= 135, one byte) and x = 8 ((i ^ j) & (DP-1)) (the column element's byte offset), so an
  // event needs one PRMT + one LEA/IADD per address instead of a PRMT-XOR-shift-mask-IMAD
  // chain; y == 16 j exactly when i == j.
  uint32_t yw[2] = {0u, 0u}, xw[2] = {0u, 0u};
  const int j16 = 16 * j;
  if constexpr (SW) {
    const uint32_t J4 = (uint32_t)j * 0x01010101u;
    constexpr uint32_t M4 = (uint32_t)(DP - 1) * 0x01010101u;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t m4 = h == 0 ? ck.mm.x : ck.mm.y;
      const uint32_t t4 = (m4 ^ J4) & M4;
      yw[h] = (m4 << 4) | t4;   // marks <= 8: no carry across bytes
      xw[h] = t4 << 3;
    }
  }
  auto byte_of = [](uint32_t w, int s) -> uint32_t { return __byte_perm(w, 0u, 0x4440u | (unsigned)(s & 3)); };
  constexpr bool HOIST = DP <= 8 || DP == 32;
  float ecs[8];
  if constexpr (HOIST) {
#pragma unroll
    for (int s = 0; s < 8; s++) {
      const float t = s == 0 ? ck.ta.x : s == 1 ? ck.ta.y : s == 2 ? ck.ta.z : s == 3 ? ck.ta.w
                    : s == 4 ? ck.tb.x : s == 5 ? ck.tb.y : s == 6 ? ck.tb.z : ck.tb.w;
      float dc = s == 0 ? ck.da.x : s == 1 ? ck.da.y : s == 2 ? ck.da.z : s == 3 ? ck.da.w
               : s == 4 ? ck.db.x : s == 5 ? ck.db.y : s == 6 ? ck.db.z : ck.db.w;
      if constexpr (TC) dc = fminf(dc, t - tb);
      (void)t;
      const int i = (int)__byte_perm(s < 4 ? ck.mm.x : ck.mm.y, 0u, 0x4440u | (unsigned)(s & 3));
      const uint32_t cab = SW ? colbb + byte_of(xw[s >> 2], s) : colbb + ((uint32_t)i << 3);
      const float bc = lda1o<0>(cab);
      ecs[s] = PRE ? ex2f(bc * dc) : ex2f(bc * (dc * -kLog2e));
    }
  }
#pragma unroll
  for (int s = 0; s < 8; s++) {
    const float t = s == 0 ? ck.ta.x : s == 1 ? ck.ta.y : s == 2 ? ck.ta.z : s == 3 ? ck.ta.w
                  : s == 4 ? ck.tb.x : s == 5 ? ck.tb.y : s == 6 ? ck.tb.z : ck.tb.w;
    float dc = s == 0 ? ck.da.x : s == 1 ? ck.da.y : s == 2 ? ck.da.z : s == 3 ? ck.da.w
             : s == 4 ? ck.db.x : s == 5 ? ck.db.y : s == 6 ? ck.db.z : ck.db.w;
    // TC (a time chunk of a window whose carried-in state is anchored at the chunk base tb):
    // the first event of a mark in the chunk re-anchors from tb, not from the mark's previous
    // event (gap = t - tb, the smaller of the two; fp32 subtraction is monotone)
    if constexpr (TC) dc = fminf(dc, t - tb);
    const unsigned word = s < 4 ? ck.mm.x : ck.mm.y;
    const int i = (int)__byte_perm(word, 0u, 0x4440u | (unsigned)(s & 3));   // mark (null: DP)
    MDHP_ASSERT(i >= 0 && i <= DP);
    uint32_t ra, ca, cab;
    // ii: the mark for the i == j / null tests (SW: y, compared with 16 j / 16 DP)
    int ii = i, jj = j, inull = DP;
    if constexpr (SW) {
      const uint32_t y = byte_of(yw[s >> 2], s), x = byte_of(xw[s >> 2], s);
      ra = sA + 8u * y;
      ca = colb + x;
      cab = colbb + x;
      ii = (int)y;
      jj = j16;
      inull = 16 * DP;
    } else {
      ra = rowb + (uint32_t)i * (8u * RS);
      ca = colb + ((uint32_t)i << 3);
      cab = colbb + ((uint32_t)i << 3);
    }
    MDHP_ASSERT(ra + 8 <= sA + 8u * (uint32_t)SM::AS && ca + kSQ + 8 <= sA + 8u * (uint32_t)(2 * SM::AS));
    const float2 ar = lda2(ra);
    const float2 sr = lds2o<kSQ>(ra);
    const float2 sc = lds2o<kSQ>(ca);
    const float dr = t - last;
    const float a_ij = ab_alpha<DP>(i, ar), b_ij = ab_beta<DP>(i, ar);
    const float er = PRE ? ex2f(b_ij * dr) : ex2f(b_ij * (dr * -kLog2e));
    float ec;
    if constexpr (HOIST) {
      ec = ecs[s];
      (void)cab;
    } else {
      const float bc = lda1o<0>(cab);
      ec = PRE ? ex2f(bc * dc) : ex2f(bc * (dc * -kLog2e));
    }
    const float R = fmaf(er, sr.x, -fset_eq0(dr));   // strict T_j^k < t
    // theta_i enters after the reduction for DP >= 8 (below), through lane i for DP <= 4
    const float p = DP >= 8 ? a_ij * R : fmaf(a_ij, R, fsel_eqi(ii, jj, th, 0.0f));
    // SW: the null column has no storage; a null event's column update is not stored
    if (!SW || ii < inull) sts2o<kSQ>(ca, fmaf(ec, sc.x, 1.0f), ec * fmaf(dc, sc.x, sc.y));
    last = fsel_eqi(ii, jj, t, last);
    if constexpr (DP >= 8) {
      pv[s] = p;
      if (GRAD) {
        Rv[s] = R;
        Qv[s] = er * fmaf(dr, sr.x, sr.y);
      }
    } else {
      const float lam = group_sum<DP>(p);
      if (GRAD) {
        const float w = rcpf(lam);
        const uint32_t ga = SW ? ra : rowb + ((uint32_t)i * (8u * DP));
        MDHP_ASSERT(ga + kG + 8 <= sA + 8u * (uint32_t)(2 * SM::AS + SM::GS));
        const float2 gg = lds2o<kG>(ga);
        sts2o<kG>(ga, fmaf(R, w, gg.x), fmaf(er * fmaf(dr, sr.x, sr.y), w, gg.y));
        gth += fsel_eqi(ii, jj, w, 0.0f);
      }
      lacc += (j == 0) ? lg2f(lam) : 0.0f;
    }
    // no __syncwarp per event (it cost an issue slot each): the state accesses are volatile asm
    // in program order and the warp is converged, so the shared-memory unit sees one event's
    // column stores before the next event's row loads
  }
  __syncwarp();
  if constexpr (DP >= 8) {
    // this lane now holds event e's sum over sources; add theta of its mark (0 for a null
    // event), which lane gbase + mark holds
    const int e = (j >> (LG - 3)) & 7;
    const int ie = (int)__byte_perm(e < 4 ? ck.mm.x : ck.mm.y, 0u, 0x4440u | (unsigned)(e & 3));
    const float the = __shfl_sync(kFull, th, gbase + (ie & (DP - 1)));
    const float lam = reduce_scatter8<DP>(pv, j) + (ie < DP ? the : 0.0f);
    if ((j & ((DP >> 3) - 1)) == 0) lacc += lg2f(lam);
    if (GRAD) {
      const float w = rcpf(lam);
      // broadcast the 8 weights through shared memory (one store + two broadcast loads = 3
      // slots) instead of 8 shuffles: shuffles and shared wavefronts share one slot per clock
      // (profiles/r01_ubench_b200.txt).  Scratch: the never-read null row of G (null events of
      // this chunk overwrite it in the pass below, after it has been read).
      // (DP <= 16; for DP = 32, one window per warp, the shuffles measured faster).
      float4 wa = make_float4(0.f, 0.f, 0.f, 0.f), wb = wa;
      if constexpr (DP <= 16) {
        const uint32_t scr = sA + kG + (SW ? 128u * DP : 8u * DP * DP);   // G's null row
        if ((j & ((DP >> 3) - 1)) == 0) sts1(scr + 4u * e, w);
        __syncwarp();
        wa = lds4(scr);
        wb = lds4(scr + 16u);
      }
      // NGC consecutive events at a time, event s into copy s % NGC: their loads issue
      // together, then their stores (the copies never alias)
      constexpr int NGC = SM::NGC;
#pragma unroll
      for (int s0 = 0; s0 < 8; s0 += NGC) {
        float2 gg[NGC];
        uint32_t ga[NGC];
        float wsv[NGC];
#pragma unroll
        for (int u = 0; u < NGC; u++) {
          const int s = s0 + u;
          wsv[u] = DP > 16 ? __shfl_sync(kFull, w, gbase + (s << (LG - 3)))
                 : s == 0 ? wa.x : s == 1 ? wa.y : s == 2 ? wa.z : s == 3 ? wa.w
                 : s == 4 ? wb.x : s == 5 ? wb.y : s == 6 ? wb.z : wb.w;
          const unsigned word = s < 4 ? ck.mm.x : ck.mm.y;
          // re-extract the mark (shift/mask, not pass 1's PRMT) so that pass 1's 8 "i == j"
          // predicates are not kept live across the reduction (ptxas would pack them into a
          // register with two LOP3 each)
          int i = (int)((word >> (8 * (s & 3))) & 0xffu), jj = j;
          MDHP_ASSERT(i >= 0 && i <= DP);
          if constexpr (SW) {   // y (see above): the row element (i, j) of G
            i = (int)byte_of(yw[s >> 2], s);
            jj = j16;
            ga[u] = (sA + kG + 8u * (uint32_t)(u * SM::GS)) + 8u * (uint32_t)i;
          } else {
            ga[u] = (rowb + kG) + ((uint32_t)i << (3 + LG)) + 8u * (uint32_t)(u * SM::GS);
          }
          MDHP_ASSERT(ga[u] >= sA + kG && ga[u] + 8 <= sA + 8u * (uint32_t)(2 * SM::AS + NGC * SM::GS));
          gg[u] = lds2(ga[u]);
          if constexpr (NGC > 1) gth += fsel_eqi(i, jj, wsv[u], 0.0f);
          else {
            sts2o<0>(ga[u], fmaf(Rv[s], wsv[u], gg[u].x), fmaf(Qv[s], wsv[u], gg[u].y));
            gth += fsel_eqi(i, jj, wsv[u], 0.0f);
          }
        }
        if constexpr (NGC > 1) {
#pragma unroll
          for (int u = 0; u < NGC; u++)
            sts2o<0>(ga[u], fmaf(Rv[s0 + u], wsv[u], gg[u].x), fmaf(Qv[s0 + u], wsv[u], gg[u].y));
        }
      }
    }
  }
  lsum += (double)lacc;
}

// The event loop of one window-evaluation, two chunks per iteration with explicit buffers so
// the prefetch of chunk c+1 overlaps chunk c without register rotation.
template <int DP, bool GRAD, bool PRE, bool TC = false>
__device__ __forceinline__ void event_loop(const float2* __restrict__ A, float2* __restrict__ SQ,
                                           float2* __restrict__ Gs,
                                           const int j, const int gbase,
                                           const float* __restrict__ t32,
                                           const float* __restrict__ dtp,
                                           const uint8_t* __restrict__ mk, const int64_t beg,
                                           const int n, const int nmax, const float th,
                                           float& last, float& gth, double& lsum,
                                           const float last0 = -1.0f, const int clampo = -1,
                                           const float tb = 0.0f) {
  // last0: anchor of the initial state (-1: empty history; 0: a carried-in state anchored at
  // the chunk base, seq.cu; tb: a time chunk of a window, TC)
  last = last0;
  gth = 0.0f;
  lsum = 0.0;
  // window base pointers; chunk offsets are clamped to the window's null chunk at npad (a time
  // chunk of a window passes the offset of its window's null chunk, clampo)
  const float* tw = t32 + beg;
  const float* dw = dtp + beg;
  const uint8_t* mw = mk + beg;
  const int npadn = (n + 7) & ~7;
  const int npad = clampo >= 0 ? clampo : npadn;
  MDHP_ASSERT(n >= 0 && nmax >= n);
  // offsets at or past this window's (chunk's) padded end go to the null chunk
  auto co = [&](int off) { return off < npadn ? off : npad; };
  Chunk c0, c1;
  load_chunk(c0, tw, dw, mw, co(0));
  if constexpr (TC) {
    // one chunk per iteration: the time-chunked kernel runs twice the warps over two hot loops
    // (phase 1 and this one), and a two-chunk body left a third of its issue slots waiting on
    // instruction fetch (ncu "no_instruction", profiles/r02_cfg2_tc*)
    for (int base = 0; base < nmax; base += 8) {
      load_chunk(c1, tw, dw, mw, co(base + 8));
      process_chunk<DP, GRAD, PRE, TC>(c0, A, SQ, Gs, j, gbase, th, last, gth, lsum, tb);
      c0 = c1;
    }
    return;
  }
  for (int base = 0; base < nmax; base += 16) {
    load_chunk(c1, tw, dw, mw, co(base + 8));
    process_chunk<DP, GRAD, PRE, TC>(c0, A, SQ, Gs, j, gbase, th, last, gth, lsum, tb);
    // no early exit: a second chunk past nmax is all null events (exact no-ops), and one basic
    // block per iteration lets ptxas overlap chunk c's reduction with chunk c+1's row reads
    load_chunk(c0, tw, dw, mw, co(base + 16));
    process_chunk<DP, GRAD, PRE, TC>(c1, A, SQ, Gs, j, gbase, th, last, gth, lsum, tb);
  }
}

// Phase 1 of a time-chunked window (k_fit_tc): the chunk's local state at its last event te,
// from an empty history, as direct sums instead of the column recurrence:
//   S_ji(te) = sum_{k in chunk, mark i} 2^{beta'_ji (te - t_k)},  Q'_ji(te) = sum (te - t_k) 2^{..}
// -- the lazy recurrence's state re-anchored at te, exact up to rounding, with the same one
// exponential per event and lane.  The terms are independent (no event-to-event chain: the
// recurrence made this phase as slow as the full evaluation), so lane j accumulates its row j
// through the NGC copies of G (scratch here; zeroed by reset_state, re-zeroed for phase 3),
// NGC events at a time, and finally writes the copies' sum into SQ.  Loads as event_loop.
template <int DP>
__device__ __forceinline__ void local_direct(const float2* __restrict__ A, float2* __restrict__ SQ,
                                             float2* __restrict__ Gs, const int j,
                                             const float* __restrict__ t32,
                                             const float* __restrict__ dtp,
                                             const uint8_t* __restrict__ mk, const int64_t beg,
                                             const int n, const int nmax, const float te,
                                             const int clampo) {
  using SM = Smem<DP>;
  static_assert(SM::SW, "time chunks: Dp <= 8");
  constexpr int NGC = SM::NGC;
  constexpr int kG = 2 * SM::AS * 8;
  uint32_t sA = static_cast<uint32_t>(__cvta_generic_to_shared(A));
  asm volatile("" : "+r"(sA) :: "memory");   // see process_chunk
  const uint32_t colb = sA + 128u * j;
  const uint32_t colbb = colb + (ab_swapped<DP>(j) ? 0u : 4u);
  const uint32_t J4 = (uint32_t)j * 0x01010101u;
  constexpr uint32_t M4 = (uint32_t)(DP - 1) * 0x01010101u;
  const float* tw = t32 + beg;
  const float* dw = dtp + beg;
  const uint8_t* mw = mk + beg;
  auto run8 = [&](const Chunk& ck) {
    const uint32_t xw[2] = {((ck.mm.x ^ J4) & M4) << 3, ((ck.mm.y ^ J4) & M4) << 3};
#pragma unroll
    for (int s0 = 0; s0 < 8; s0 += NGC) {
      uint32_t ga[NGC];
      float2 gg[NGC];
      float cv[NGC], dv[NGC];
      bool real[NGC];
#pragma unroll
      for (int u = 0; u < NGC; u++) {
        const int s = s0 + u;
        const float t = s == 0 ? ck.ta.x : s == 1 ? ck.ta.y : s == 2 ? ck.ta.z : s == 3 ? ck.ta.w
                      : s == 4 ? ck.tb.x : s == 5 ? ck.tb.y : s == 6 ? ck.tb.z : ck.tb.w;
        const int i = (int)__byte_perm(s < 4 ? ck.mm.x : ck.mm.y, 0u, 0x4440u | (unsigned)(s & 3));
        MDHP_ASSERT(i >= 0 && i <= DP);
        const uint32_t x = __byte_perm(xw[s >> 2], 0u, 0x4440u | (unsigned)(s & 3));
        real[u] = i < DP;   // the null column has no storage (SW)
        dv[u] = te - t;
        cv[u] = ex2f(lda1o<0>(colbb + x) * dv[u]);
        ga[u] = colb + x + kG + 8u * (uint32_t)(u * SM::GS);
        MDHP_ASSERT(ga[u] + 8 <= sA + 8u * (uint32_t)(2 * SM::AS + NGC * SM::GS));
        gg[u] = lds2(ga[u]);
      }
#pragma unroll
      for (int u = 0; u < NGC; u++)
        if (real[u]) sts2o<0>(ga[u], gg[u].x + cv[u], fmaf(dv[u], cv[u], gg[u].y));
    }
  };
  const int npadn = (n + 7) & ~7;
  auto co = [&](int off) { return off < npadn ? off : clampo; };
  Chunk c0, c1;
  load_chunk(c0, tw, dw, mw, co(0));
  for (int base = 0; base < nmax; base += 8) {
    load_chunk(c1, tw, dw, mw, co(base + 8));
    run8(c0);
    c0 = c1;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < DP; i++) SQ[SM::e(j, i)] = gsum<DP>(Gs, j, i);
  __syncwarp();
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
