// common.cuh — packed layout and device helpers shared by the libmdhp kernels (sm_100a).
// Nothing here is shared with oracle/ (DESIGN.md "Independence").
#pragma once
#include <cstdint>
#include <cstddef>
#include <cassert>
#include <cuda_runtime.h>
#include "../../include/mdhp.h"

// Device-side bounds checks, compiled in only for the debug library (build.py debug=True,
// -DMDHP_DEBUG); the tests run the GPU suites against it (compute-sanitizer is closed here).
#ifdef MDHP_DEBUG
#define MDHP_ASSERT(x) assert(x)
#else
#define MDHP_ASSERT(x) ((void)0)
#endif

namespace mdhp {

constexpr int kAlignEv = 8;     // window event ranges start on 8-event boundaries
constexpr int kWinStride = 16;  // begin(w) = roundup8(win_off[w]) + 16 w: every window is
                                // followed by its padding to 8 and 8 null events (eval.cuh)
constexpr int kMom = 17;        // power moments m_1..m_17 of u/u_max per (window, mark)
constexpr int kSortBuckets = 65536;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr unsigned kFull = 0xffffffffu;
// fp64 re-evaluation threshold (fit.cu needs_exact, R24): a window is re-evaluated in
// fp64 unless |lnL| >= kExactPerEvent N + kExactPerLn |sum ln lambda| + kExactGross (|Part2| +
// |Part3|)
constexpr double kExactPerEvent = 0.05;
constexpr double kExactPerLn = 0.01;
constexpr double kExactGross = 0.02;
// status bits a fit call keeps from its input (validation); the fit's own outcome bits
// (NONFINITE, DIVERGED, CONVERGED) are those of this call only
constexpr int kKeepStatus = MDHP_ST_INVALID | MDHP_ST_EMPTY;

inline int pad_dims(int D) {
  int p = 1;
  while (p < D) p <<= 1;
  return p;
}

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Byte layout of the packed buffer; a pure function of (D, W, E) so that every call can
// recompute it from the descriptor (no device->host read of a header is ever needed).
struct Layout {
  int D, Dp;
  int64_t W, E, Epad;
  size_t begin, n, T32, perm, t32, dtp, mark, cnt, umax, mom, sort_cnt, total;
};

__host__ __device__ inline Layout make_layout(int D, int64_t W, int64_t E) {
  Layout L;
  L.D = D;
  int p = 1;
  while (p < D) p <<= 1;
  L.Dp = p;
  L.W = W;
  L.E = E;
  L.Epad = ((E + kAlignEv - 1) / kAlignEv) * kAlignEv + (int64_t)kWinStride * W + kAlignEv;
  size_t o = 0;
  L.begin = o;    o = align256(o + sizeof(int64_t) * W);
  L.n = o;        o = align256(o + sizeof(int32_t) * W);
  L.T32 = o;      o = align256(o + sizeof(float) * W);
  L.perm = o;     o = align256(o + sizeof(int32_t) * W);
  L.t32 = o;      o = align256(o + sizeof(float) * L.Epad);
  L.dtp = o;      o = align256(o + sizeof(float) * L.Epad);
  L.mark = o;     o = align256(o + sizeof(uint8_t) * L.Epad);
  L.cnt = o;      o = align256(o + sizeof(int32_t) * W * L.Dp);
  L.umax = o;     o = align256(o + sizeof(float) * W * L.Dp);
  L.mom = o;      o = align256(o + sizeof(float) * W * L.Dp * kMom);
  L.sort_cnt = o; o = align256(o + sizeof(int32_t) * (kSortBuckets + 1));
  L.total = o;
  return L;
}

// Device view of a packed buffer.
struct Packed {
  const int64_t* begin;   // [W] first padded event slot of window w
  const int32_t* n;       // [W] events
  const float* T32;       // [W] horizon in analysis units
  const int32_t* perm;    // [W] windows, longest first
  const float* t32;       // [Epad]
  const float* dtp;       // [Epad] gap to the previous event of the same mark (t + 1 if none)
  const uint8_t* mark;    // [Epad]
  const int32_t* cnt;     // [W][Dp]
  const float* umax;      // [W][Dp] T - first event time of the mark (0 if none)
  const float* mom;       // [W][Dp][kMom]
  int64_t W;
  int D, Dp;
};

inline Packed view(const Layout& L, const void* base) {
  const char* b = static_cast<const char*>(base);
  Packed P;
  P.begin = reinterpret_cast<const int64_t*>(b + L.begin);
  P.n = reinterpret_cast<const int32_t*>(b + L.n);
  P.T32 = reinterpret_cast<const float*>(b + L.T32);
  P.perm = reinterpret_cast<const int32_t*>(b + L.perm);
  P.t32 = reinterpret_cast<const float*>(b + L.t32);
  P.dtp = reinterpret_cast<const float*>(b + L.dtp);
  P.mark = reinterpret_cast<const uint8_t*>(b + L.mark);
  P.cnt = reinterpret_cast<const int32_t*>(b + L.cnt);
  P.umax = reinterpret_cast<const float*>(b + L.umax);
  P.mom = reinterpret_cast<const float*>(b + L.mom);
  P.W = L.W;
  P.D = L.D;
  P.Dp = L.Dp;
  return P;
}

// ---------------------------------------------------------------- device math (MUFU)
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Asynchronous global -> shared copies (cp.async, L1-allocating): a prologue that stages many
// small loads pays one round trip at the final wait instead of one per dependent store.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gsrc) {
  static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "cp.async size");
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(gsrc), "n"(BYTES)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------- TMEM as per-lane storage
// tcgen05.ld/st with the 32x32b shape move 32-bit columns between thread l of a warp and TMEM
// lane 32*(warp%4)+l: a per-lane array indexed by a warp-uniform column.  The fit kernel keeps
// each window's optimizer state there (k_fit, DESIGN.md a6).  All lanes of a warp must execute
// these (.sync.aligned); values loaded by tm_ld are valid only after tm_wait_ld on them.
template <int N>
__device__ __forceinline__ void tm_ld(uint32_t a, float (&v)[N]) {
  static_assert(N == 1 || N == 2 || N == 4 || N % 8 == 0, "tm_ld width");
  if constexpr (N == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(v[0]) : "r"(a));
  } else if constexpr (N == 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                 : "=f"(v[0]), "=f"(v[1]) : "r"(a));
  } else if constexpr (N == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
  } else {
#pragma unroll
    for (int k = 0; k < N; k += 8)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=f"(v[k]), "=f"(v[k + 1]), "=f"(v[k + 2]), "=f"(v[k + 3]), "=f"(v[k + 4]),
                     "=f"(v[k + 5]), "=f"(v[k + 6]), "=f"(v[k + 7])
                   : "r"(a + (uint32_t)k));
  }
}
template <int N>
__device__ __forceinline__ void tm_st(uint32_t a, const float (&v)[N]) {
  static_assert(N == 1 || N == 2 || N == 4 || N % 8 == 0, "tm_st width");
  if constexpr (N == 1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a), "f"(v[0]) : "memory");
  } else if constexpr (N == 2) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "f"(v[0]),
                 "f"(v[1]) : "memory");
  } else if constexpr (N == 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]) : "memory");
  } else {
#pragma unroll
    for (int k = 0; k < N; k += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                   ::"r"(a + (uint32_t)k), "f"(v[k]), "f"(v[k + 1]), "f"(v[k + 2]), "f"(v[k + 3]),
                   "f"(v[k + 4]), "f"(v[k + 5]), "f"(v[k + 6]), "f"(v[k + 7]) : "memory");
  }
}
// Wait for the outstanding tcgen05.ld of this thread; the registers pass through the asm so no
// use of them can be scheduled before the wait.
__device__ __forceinline__ void tm_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tm_fence_regs(float (&v)[N]) {
#pragma unroll
  for (int k = 0; k < N; k++) asm volatile("" : "+f"(v[k]));
}
__device__ __forceinline__ void tm_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// Allocate `cols` (a power of two >= 32) TMEM columns for the CTA (warp 0), publish the base
// through shared memory and synchronise the CTA; returns the base address.
__device__ __forceinline__ uint32_t tm_alloc(uint32_t* slot, uint32_t cols) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(slot))),
                 "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  return *reinterpret_cast<volatile uint32_t*>(slot);
}
__device__ __forceinline__ void tm_free(uint32_t base, uint32_t cols) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols)
                 : "memory");
}

template <int DP>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = DP / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
template <int DP>
__device__ __forceinline__ double group_sum_d(double v) {
#pragma unroll
  for (int o = DP / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
template <int DP>
__device__ __forceinline__ int group_max_i(int v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

struct FitCfgDev {
  int max_iters, optimizer, loss_mean, patience, max_halvings;
  float lr, b1, b2, eps, tol_rel, min_param;
  unsigned fit_mask;
  int step0;   // Adam steps of earlier calls (resume)
  int time_chunks;   // time chunks per window (k_fit_tc), 0/1 = throughput layout
  int slot_order = 0;   // launcher-internal (k_fit LAT, fixed iterations): 1 = static unit per
                        // warp slot, longest units alone on their SM sub-partition
};

// launch counter (process-wide), incremented by every launch site
void count_launch(int k = 1);
uint64_t launches_so_far();
void set_error(const char* fmt, ...);

}  // namespace mdhp
