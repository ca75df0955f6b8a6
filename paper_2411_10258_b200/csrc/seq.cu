// seq.cu — long single sequences (row a7 of DESIGN.md section 4): chunked parallel scan of the
// exponential-decay recurrence.
//
// The recurrence state of Eq.(2) for every pair (i, j) evolves between events as a
// linear map: over a gap L, S <- e^{-beta L} S and Q <- e^{-beta L}(Q + L S), and an event of
// source j adds 1 to S_.j.  So a long sequence can be cut into chunks (never inside a tie group):
//   phase 1 (k_seq_local)  every chunk's local state at its last event from an empty
//                          history, as direct sums (2 D^2 floats);
//   phase 2 (k_seq_scan)   exclusive scan of the affine maps (decay over the chunk span + local
//                          state), segmented over chunks, per pair -> the state carried into each
//                          chunk, anchored at the chunk base (the previous chunk's last event);
//   phase 3 (k_seq_eval)   every chunk re-runs the full event loop (row reads, lambda, gradient
//                          accumulation) from its carried-in state;
//   phase 4 (k_seq_reduce, k_seq_finish)  fixed-order sums over chunks, the Part2/Part3
//                          epilogue from the global final state, and (fit) one optimizer step.
// Chunk-relative fp32 times (fp64 base per chunk) keep ~1e-7 s resolution over 1000 s.
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include "eval.cuh"

namespace mdhp {

constexpr int kSeqWPB = 4;

struct SeqLayout {
  int D, Dp;
  int64_t N, C, Epad;
  size_t cstart, cbeg, cspan, t32, dtp, mark, ccnt, cfirst, cmom, cnt, umax, mom, tail, status,
      total;
};

__host__ __device__ inline SeqLayout make_seq_layout(int D, int64_t N, int ce) {
  SeqLayout L;
  L.D = D;
  int p = 1;
  while (p < D) p <<= 1;
  L.Dp = p;
  L.N = N;
  L.C = N > 0 ? (N + ce - 1) / ce : 0;
  L.Epad = ((N + 7) / 8) * 8 + 16 * L.C + 8;
  size_t o = 0;
  L.cstart = o; o = align256(o + sizeof(int64_t) * (L.C + 1));
  L.cbeg = o;   o = align256(o + sizeof(int64_t) * L.C);
  L.cspan = o;  o = align256(o + sizeof(float) * L.C);
  L.t32 = o;    o = align256(o + sizeof(float) * L.Epad);
  L.dtp = o;    o = align256(o + sizeof(float) * L.Epad);
  L.mark = o;   o = align256(o + L.Epad);
  L.ccnt = o;   o = align256(o + sizeof(int32_t) * L.C * L.Dp);
  L.cfirst = o; o = align256(o + sizeof(double) * L.C * L.Dp);
  L.cmom = o;   o = align256(o + sizeof(float) * L.C * L.Dp * kMom);
  L.cnt = o;    o = align256(o + sizeof(int32_t) * L.Dp);
  L.umax = o;   o = align256(o + sizeof(float) * L.Dp);
  L.mom = o;    o = align256(o + sizeof(float) * L.Dp * kMom);
  L.tail = o;   o = align256(o + sizeof(float) * 2);
  L.status = o; o = align256(o + sizeof(int32_t));
  L.total = o;
  return L;
}

template <typename T>
__host__ __device__ inline T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}
template <typename T>
__host__ __device__ inline const T* at(const void* base, size_t off) {
  return reinterpret_cast<const T*>(static_cast<const char*>(base) + off);
}

// ---------------------------------------------------------------- packing
__global__ void k_seq_bounds(int64_t N, int64_t C, int ce, const double* __restrict__ t,
                             int64_t* __restrict__ cstart, int64_t* __restrict__ cbeg) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c > C) return;
  int64_t b = c * ce;
  if (b > N) b = N;
  while (b > 0 && b < N && t[b] == t[b - 1]) b++;   // never split a tie group
  cstart[c] = b;
  if (c < C) cbeg[c] = ((b + 7) & ~int64_t(7)) + 16 * c;
}

// One warp per chunk: relative times, same-mark gaps, validation, per-chunk counts/first times.
__global__ void __launch_bounds__(kSeqWPB * 32)
k_seq_events(int D, int Dp, int64_t N, int64_t C, double T, double t0, const double* __restrict__ t,
             const int32_t* __restrict__ mark, const int64_t* __restrict__ cstart,
             const int64_t* __restrict__ cbeg, float* __restrict__ cspan, float* __restrict__ o_t,
             float* __restrict__ o_d, uint8_t* __restrict__ o_m, int32_t* __restrict__ ccnt,
             double* __restrict__ cfirst, int32_t* __restrict__ status) {
  __shared__ double s_last[kSeqWPB][32];
  __shared__ double s_first[kSeqWPB][32];
  __shared__ int s_cnt[kSeqWPB][32];
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kSeqWPB + wp;
  if (c >= C) return;
  const int64_t a = cstart[c], z = cstart[c + 1], n = z - a, beg = cbeg[c];
  MDHP_ASSERT(a >= 0 && z <= N && n >= 0 && (beg & 7) == 0);
  const double tau = a > 0 ? t[a - 1] : t0;   // chunk base: previous event (or the slice base)
  s_last[wp][lane] = 0.0;
  s_first[wp][lane] = 0.0;
  s_cnt[wp][lane] = 0;
  __syncwarp();
  int st = 0;
  double carry = tau;
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t k = base + lane;
    const bool in = k < n;
    const double tk = in ? t[a + k] : 0.0;
    const int mk = in ? mark[a + k] : 0;
    const bool okmark = in && mk >= 0 && mk < D;
    if (in) {
      if (!isfinite(tk) || tk < 0.0 || tk > T) st |= MDHP_ST_OUT_OF_RANGE;
      if (!okmark) st |= MDHP_ST_BAD_MARK;
    }
    double tprev = __shfl_up_sync(kFull, tk, 1);
    if (lane == 0) tprev = carry;
    if (in && tk < tprev) st |= MDHP_ST_UNSORTED;
    carry = __shfl_sync(kFull, tk, 31);
    const unsigned key = okmark ? (unsigned)mk : (64u + lane);
    const unsigned grp = __match_any_sync(kFull, key);
    const unsigned lower = grp & ((1u << lane) - 1u);
    const int src = lower ? (31 - __clz(lower)) : lane;
    const double tin = __shfl_sync(kFull, tk, src);
    const int cnt_before = okmark ? s_cnt[wp][mk] : 0;
    const bool has_prev = lower != 0 || cnt_before > 0;
    const double tp = lower ? tin : (okmark && cnt_before > 0 ? s_last[wp][mk] : tau);
    if (okmark && has_prev && tk == tp) st |= MDHP_ST_SAME_DIM_TIE;
    if (in) {
      o_t[beg + k] = __double2float_rn(__dsub_rn(tk, tau));
      o_d[beg + k] = __double2float_rn(__dsub_rn(tk, tp));
      o_m[beg + k] = okmark ? (uint8_t)mk : (uint8_t)0xFF;
    }
    if (okmark && !lower && cnt_before == 0) s_first[wp][mk] = tk;
    __syncwarp();
    const bool is_last = okmark && (grp & ~((2u << lane) - 1u)) == 0u;
    if (is_last) {
      s_last[wp][mk] = tk;
      s_cnt[wp][mk] = cnt_before + __popc(grp);
    }
    __syncwarp();
  }
  const int64_t npad = ((n + 7) & ~int64_t(7)) + 8;   // padding + one null chunk
  for (int64_t k = n + lane; k < npad; k += 32) {
    o_t[beg + k] = kNullT;
    o_d[beg + k] = 0.0f;
    o_m[beg + k] = (uint8_t)Dp;
  }
  if (lane < Dp) {
    ccnt[c * Dp + lane] = lane < D ? s_cnt[wp][lane] : 0;
    cfirst[c * Dp + lane] = s_first[wp][lane];
  }
  st = __reduce_or_sync(kFull, st);
  if (lane == 0) {
    cspan[c] = n > 0 ? __double2float_rn(__dsub_rn(t[z - 1], tau)) : 0.0f;
    if (st) atomicOr(status, st);
  }
}

// Per-mark totals, first times -> u_max, and the tail T - (last event).  One block of 256
// threads over chunks; integer sums and a min over chunk indices are order-independent.
__global__ void __launch_bounds__(256)
k_seq_stats(int D, int Dp, int64_t N, int64_t C, double T, const double* __restrict__ t,
            const int32_t* __restrict__ ccnt, const double* __restrict__ cfirst,
            int32_t* __restrict__ cnt, float* __restrict__ umax, float* __restrict__ tail,
            int32_t* __restrict__ status) {
  __shared__ int s_cnt[32];
  __shared__ unsigned long long s_firstc[32];
  const int tid = threadIdx.x;
  if (tid < 32) {
    s_cnt[tid] = 0;
    s_firstc[tid] = ~0ull;
  }
  __syncthreads();
  for (int j = 0; j < Dp; j++) {
    int tot = 0;
    unsigned long long fc = ~0ull;
    for (int64_t c = tid; c < C; c += blockDim.x) {
      const int k = ccnt[c * Dp + j];
      tot += k;
      if (k > 0 && (unsigned long long)c < fc) fc = (unsigned long long)c;
    }
    if (tot) atomicAdd(&s_cnt[j], tot);
    if (fc != ~0ull) atomicMin(&s_firstc[j], fc);
  }
  __syncthreads();
  if (tid < Dp) {
    const int j = tid;
    const int tot = j < D ? s_cnt[j] : 0;
    cnt[j] = tot;
    umax[j] = (tot > 0) ? __double2float_rn(__dsub_rn(T, cfirst[(int64_t)s_firstc[j] * Dp + j])) : 0.0f;
  }
  if (tid == 0) {
    tail[0] = N > 0 ? __double2float_rn(__dsub_rn(T, t[N - 1])) : (float)T;
    tail[1] = (float)T;
    if (!(T > 0.0) || !isfinite(T)) atomicOr(status, MDHP_ST_BAD_T);
    if (N == 0) atomicOr(status, MDHP_ST_EMPTY);
  }
}

// Per-chunk power moments (lane = mark, fixed order), r = (T - t)/u_max in fp64.
__global__ void __launch_bounds__(kSeqWPB * 32)
k_seq_moments(int D, int Dp, int64_t C, double T, const double* __restrict__ t,
              const int32_t* __restrict__ mark, const int64_t* __restrict__ cstart,
              const float* __restrict__ umax, float* __restrict__ cmom) {
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kSeqWPB + wp;
  if (c >= C) return;
  const int64_t a = cstart[c], z = cstart[c + 1];
  const double um = lane < D ? (double)umax[lane] : 0.0;
  float acc[kMom];
#pragma unroll
  for (int p = 0; p < kMom; p++) acc[p] = 0.0f;
  for (int64_t base = a; base < z; base += 32) {
    const int64_t k = base + lane;
    const double tk = k < z ? t[k] : 0.0;
    const int mk = k < z ? mark[k] : -1;
    const int cntk = (int)min((int64_t)32, z - base);
    for (int s = 0; s < cntk; s++) {
      const double ts = __shfl_sync(kFull, tk, s);
      const int ms = __shfl_sync(kFull, mk, s);
      if (ms == lane) {
        const float r = um > 0.0 ? __double2float_rn((T - ts) / um) : 0.0f;
        float pw = r;
#pragma unroll
        for (int p = 0; p < kMom; p++) {
          acc[p] = __fadd_rn(acc[p], pw);
          pw = __fmul_rn(pw, r);
        }
      }
    }
  }
  if (lane < Dp) {
#pragma unroll
    for (int p = 0; p < kMom; p++) cmom[(c * Dp + lane) * kMom + p] = acc[p];
  }
}

__global__ void __launch_bounds__(256)
k_seq_momsum(int Dp, int64_t C, const float* __restrict__ cmom, float* __restrict__ mom) {
  __shared__ double red[256];
  const int q = blockIdx.x;   // (mark, p)
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < C; c += 256) s += (double)cmom[c * Dp * kMom + q];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o >= 1; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) mom[q] = (float)red[0];
}

// ---------------------------------------------------------------- evaluation workspace
#ifndef MDHP_SCAN_P
#define MDHP_SCAN_P 4
#endif
constexpr int kScanP = MDHP_SCAN_P, kScanS = 1024 / MDHP_SCAN_P;   // pairs x segments per scan
                                                                  // block (1024 threads)

// Phase-3 blocks: 4 warps x G chunks each; every block writes one record of partial sums.
inline int64_t seq_eval_blocks(int Dp, int64_t C) {
  const int64_t per = 4 * (32 / Dp);
  return (C + per - 1) / per;
}

struct SeqWork {
  float2* loc;     // [C][D*D]  local state at chunk end (target-major pairs)
  float2* carry;   // [C][D*D]  state carried into the chunk, anchored at its base
  float2* fin;     // [D*D]     state after the last event, anchored there
  float2* gsum;    // [D*D]
  float* gth;      // [Dp]
  double* ls;      // [1]
  int* ctl;        // optimizer control block (seq fit)
  float* prev;     // [D + 2 D^2] previous point (rollback)
  float* opt;      // [2 (D + 2 D^2)] Adam moments when the caller passes none
  double* rpart;   // [phase-3 blocks][2 D^2 + D + 1] per-block partial sums
  float4* segmap;  // [D*D][kScanS + 1] scan segment maps kept between mdhp_seq_maps and _parts (f1)
  size_t bytes;
};

inline SeqWork make_seq_work(void* base, int D, int Dp, int64_t C) {
  SeqWork w;
  const size_t DD = (size_t)D * D, P = (size_t)D + 2 * DD;
  size_t o = 0;
  auto take = [&](size_t nb) { size_t r = o; o = align256(o + nb); return r; };
  const size_t a = take(sizeof(float2) * C * DD), b = take(sizeof(float2) * C * DD),
               f = take(sizeof(float2) * DD), gs = take(sizeof(float2) * DD),
               gt = take(sizeof(float) * Dp), ls = take(sizeof(double)),
               ct = take(sizeof(int) * 64), pv = take(sizeof(float) * P), op = take(sizeof(float) * 2 * P),
               rp = take(sizeof(double) * (size_t)seq_eval_blocks(Dp, C) * (2 * DD + D + 1)),
               sg = take(sizeof(float4) * DD * (kScanS + 1));
  char* B = static_cast<char*>(base);
  w.loc = reinterpret_cast<float2*>(B + a);
  w.carry = reinterpret_cast<float2*>(B + b);
  w.fin = reinterpret_cast<float2*>(B + f);
  w.gsum = reinterpret_cast<float2*>(B + gs);
  w.gth = reinterpret_cast<float*>(B + gt);
  w.ls = reinterpret_cast<double*>(B + ls);
  w.ctl = reinterpret_cast<int*>(B + ct);
  w.prev = reinterpret_cast<float*>(B + pv);
  w.opt = reinterpret_cast<float*>(B + op);
  w.rpart = reinterpret_cast<double*>(B + rp);
  w.segmap = reinterpret_cast<float4*>(B + sg);
  w.bytes = o;
  return w;
}

// optimizer control block (device), one sequence
struct SeqCtl {
  int done, it, s, halv, stall, st, have_prev, have_lnl;
  float lr_w;
  int pad;
  double lnl_prev, lnl_last;
};

// Phase 1: every chunk's local state at its last event (chunk-relative time Lc), from an
// empty history, as direct sums instead of the column recurrence (as local_direct in eval.cuh):
//   S_ji(Lc) = sum_{k in chunk, mark i} e^{-beta_ji (Lc - t_k)},  Q_ji(Lc) = sum (Lc - t_k) e^{..}
// -- the recurrence's state re-anchored at Lc, exact up to rounding, one exponential per event
// and lane as before.  The terms are independent, so lane j accumulates its row j (private to
// the lane: no warp barrier per event) through kLocNC copies, kLocNC events at a time, instead
// of a load -> FMA -> store chain through every event.
constexpr int kLocNC = 2;
template <int DP>
__global__ void __launch_bounds__(128)
k_seq_local(int D, int64_t C, const int64_t* __restrict__ cstart, const int64_t* __restrict__ cbeg,
            const float* __restrict__ cspan, const float* __restrict__ t32,
            const float* __restrict__ dtp, const uint8_t* __restrict__ mk,
            const float* __restrict__ beta, float2* __restrict__ loc, const int* __restrict__ ctl) {
  if (ctl && ctl[0]) return;
  constexpr int G = 32 / DP, RS = DP + 1, CS = DP * RS;   // CS: float2 per copy
  extern __shared__ __align__(16) unsigned char smem_l[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane / DP, j = lane % DP;
  float2* SQ = reinterpret_cast<float2*>(smem_l) + (size_t)(wid * G + g) * kLocNC * CS;
  float* B = reinterpret_cast<float*>(reinterpret_cast<float2*>(smem_l) + (size_t)4 * G * kLocNC * CS) +
             (size_t)(wid * G + g) * CS;
  const int64_t c = ((int64_t)blockIdx.x * 4 + wid) * G + g;
  const bool live = c < C;
  const int n = live ? (int)(cstart[c + 1] - cstart[c]) : 0;
  // lane = column here (coalesced rows of beta): B[r][j] = beta_rj, SQ copies [r][j] = 0
  for (int r = 0; r < DP; r++) {
#pragma unroll
    for (int k = 0; k < kLocNC; k++) SQ[k * CS + r * RS + j] = make_float2(0.0f, 0.0f);
    if (r < D && j < D) cp_async<4>(&B[r * RS + j], beta + (size_t)r * D + j);
    else B[r * RS + j] = 0.0f;
  }
  cp_async_wait_all();
  // column DP: the null event's (never read) column
#pragma unroll
  for (int k = 0; k < kLocNC; k++) SQ[k * CS + j * RS + DP] = make_float2(0.0f, 0.0f);
  B[j * RS + DP] = 0.0f;
  __syncwarp();
  int nmax = n;
  for (int o = 16; o >= 1; o >>= 1) nmax = max(nmax, __shfl_xor_sync(kFull, nmax, o));
  const int64_t beg = live ? cbeg[c] : 0;
  const float Lc = live ? cspan[c] : 0.0f;
  // 8 events per vector load (the chunk layout is the window layout: 8-aligned, padded with
  // null events up to a multiple of 8 plus one null chunk), the next chunk prefetched
  const float* tw = t32 + beg;
  const float* dw = dtp + beg;
  const uint8_t* mw = mk + beg;
  const int npad = (n + 7) & ~7;
  auto local8 = [&](const Chunk& ck) {
#pragma unroll
    for (int s0 = 0; s0 < 8; s0 += kLocNC) {
      float2 v[kLocNC];
      float cv[kLocNC], dv[kLocNC];
      int ad[kLocNC];
#pragma unroll
      for (int u = 0; u < kLocNC; u++) {
        const int s = s0 + u;
        const float t = s == 0 ? ck.ta.x : s == 1 ? ck.ta.y : s == 2 ? ck.ta.z : s == 3 ? ck.ta.w
                      : s == 4 ? ck.tb.x : s == 5 ? ck.tb.y : s == 6 ? ck.tb.z : ck.tb.w;
        const int i = (int)__byte_perm(s < 4 ? ck.mm.x : ck.mm.y, 0u, 0x4440u | (unsigned)(s & 3));
        MDHP_ASSERT(i >= 0 && i <= DP);   // DP: null event (beta 0: adds to the unread column DP)
        dv[u] = Lc - t;
        cv[u] = ex2f(B[j * RS + i] * (dv[u] * -kLog2e));
        ad[u] = u * CS + j * RS + i;
        v[u] = SQ[ad[u]];
      }
#pragma unroll
      for (int u = 0; u < kLocNC; u++) SQ[ad[u]] = make_float2(v[u].x + cv[u], fmaf(dv[u], cv[u], v[u].y));
    }
  };
  Chunk c0, c1;
  load_chunk(c0, tw, dw, mw, 0 < n ? 0 : npad);
  for (int base = 0; base < nmax; base += 16) {
    load_chunk(c1, tw, dw, mw, min(base + 8, npad));
    local8(c0);
    load_chunk(c0, tw, dw, mw, min(base + 16, npad));
    local8(c1);
  }
  // local state at the chunk end, written row by row with lane = column (coalesced); element
  // (r, j) was accumulated by lane r
  __syncwarp();
  for (int r = 0; r < D; r++) {
    if (live && j < D) {
      float2 s = SQ[r * RS + j];
#pragma unroll
      for (int k = 1; k < kLocNC; k++) {
        const float2 x = SQ[k * CS + r * RS + j];
        s.x += x.x;
        s.y += x.y;
      }
      loc[(size_t)c * D * D + (size_t)r * D + j] = s;
    }
  }
}

// Phase 2: exclusive scan of the per-chunk affine maps.  Block = kScanP pairs x kScanS segments
// of chunks (thread = (segment, pair), pair fastest: a warp's loads of a chunk's pair row fill
// whole 32-byte sectors); each thread composes its segment in order, the segment maps are
// scanned across the block (warp shuffles, then a scan of the warp totals), then each thread
// re-walks its segment writing the carried states.  (kScanP = 32 with 32 segments was measured 2x slower: too few blocks.)
struct AffMap {
  float E, L, Sb, Qb;
};
__device__ __forceinline__ AffMap compose(const AffMap& m1, const AffMap& m2) {
  AffMap r;
  r.E = m2.E * m1.E;
  r.L = m1.L + m2.L;
  r.Sb = fmaf(m2.E, m1.Sb, m2.Sb);
  r.Qb = fmaf(m2.E, fmaf(m2.L, m1.Sb, m1.Qb), m2.Qb);
  return r;
}

constexpr int kScanB = 4;                  // chunks per load batch of a segment walk

__global__ void __launch_bounds__(kScanP * kScanS)
k_seq_scan(int D, int64_t C, const float* __restrict__ cspan, const float* __restrict__ beta,
           const float2* __restrict__ loc, float2* __restrict__ carry, float2* __restrict__ fin,
           const int* __restrict__ ctl, const float2* __restrict__ maps,
           const float* __restrict__ spans, int rank, float2* __restrict__ rankmap,
           float* __restrict__ rankspan, int mode, float4* __restrict__ segmap) {
  // mode 0: whole scan; 1 (f1 mdhp_seq_maps): slice map only, the segment maps kept in segmap;
  // 2 (f1 mdhp_seq_parts, same beta and local states): the kept segment maps replace the first
  // walk and the block scan, only the carried states are written
  if (ctl && ctl[0]) return;
  __shared__ AffMap sm[32][kScanP];   // per-warp totals (32 warps of 1024 threads)
  const int lane = threadIdx.x % kScanP, seg = threadIdx.x / kScanP;
  const int64_t DD = (int64_t)D * D;
  const int64_t p = (int64_t)blockIdx.x * kScanP + lane;
  const bool valid = p < DD;
  const float b = valid ? beta[p] : 0.0f;
  const int64_t per = (C + kScanS - 1) / kScanS;
  const int64_t c0 = min(C, (int64_t)seg * per), c1 = min(C, c0 + per);
  AffMap m{1.0f, 0.0f, 0.0f, 0.0f}, prevm{1.0f, 0.0f, 0.0f, 0.0f};
  const size_t sgb = (size_t)p * (kScanS + 1);
  if (mode == 2) {
    if (valid) {
      const float4 a = segmap[sgb + seg];
      prevm = AffMap{a.x, a.y, a.z, a.w};
      if (seg == kScanS - 1) {
        const float4 t = segmap[sgb + kScanS];
        m = AffMap{t.x, t.y, t.z, t.w};
      }
    }
  } else {
    // segment walks in batches of kScanB chunks: all loads of a batch are issued before the
    // (sequential) compose chain uses them, instead of one L2 round trip per chunk
    if (valid) {
      for (int64_t c = c0; c < c1; c += kScanB) {
        float Lb[kScanB];
        float2 lb[kScanB];
#pragma unroll
        for (int k = 0; k < kScanB; k++) {
          const bool in = c + k < c1;
          Lb[k] = in ? cspan[c + k] : 0.0f;
          lb[k] = in ? loc[(c + k) * DD + p] : make_float2(0.0f, 0.0f);
        }
#pragma unroll
        for (int k = 0; k < kScanB; k++) {
          if (c + k < c1) {
            const AffMap mc{ex2f(b * (Lb[k] * -kLog2e)), Lb[k], lb[k].x, lb[k].y};
            m = compose(m, mc);
          }
        }
      }
    }
    // inclusive scan of the segment maps (per pair, over segments) in two levels: shuffles
    // within each warp (32 / kScanP segments), then one warp per pair scans the 32 warp totals
    // (2 block barriers instead of the 2 log2(kScanS) of a Hillis-Steele scan over the block)
    static_assert(kScanP * kScanS == 1024 && 32 % kScanP == 0 && kScanP <= 32, "scan shape");
    const int wl = threadIdx.x & 31, wid = threadIdx.x >> 5;
    auto shfl_up_map = [](const AffMap& x, int o) {
      return AffMap{__shfl_up_sync(kFull, x.E, o), __shfl_up_sync(kFull, x.L, o),
                    __shfl_up_sync(kFull, x.Sb, o), __shfl_up_sync(kFull, x.Qb, o)};
    };
#pragma unroll
    for (int o = kScanP; o < 32; o <<= 1) {
      const AffMap up = shfl_up_map(m, o);
      if (wl >= o) m = compose(up, m);
    }
    if (wl >= 32 - kScanP) sm[wid][lane] = m;     // this warp's total (its last segment), per pair
    __syncthreads();
    if (wid < kScanP) {                           // warp q scans the 32 warp totals of pair q
      AffMap t = sm[wl][wid];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const AffMap up = shfl_up_map(t, o);
        if (wl >= o) t = compose(up, t);
      }
      sm[wl][wid] = t;
    }
    __syncthreads();
    if (wid > 0) m = compose(sm[wid - 1][lane], m);   // inclusive map through this segment
    // inclusive map through the previous segment (the second walk's starting point)
    const AffMap up1 = shfl_up_map(m, kScanP);
    prevm = wl >= kScanP ? up1 : (wid > 0 ? sm[wid - 1][lane] : AffMap{1.0f, 0.0f, 0.0f, 0.0f});
    if (mode == 1 && valid && segmap) {
      segmap[sgb + seg] = make_float4(prevm.E, prevm.L, prevm.Sb, prevm.Qb);
      if (seg == kScanS - 1) segmap[sgb + kScanS] = make_float4(m.E, m.L, m.Sb, m.Qb);
    }
  }
  if (!valid) return;
  // state carried into this slice (f1, multi-GPU): the earlier slices' maps composed in order
  float2 x0 = make_float2(0.0f, 0.0f);
  if (maps) {
    for (int r = 0; r < rank; r++) {
      const float L = spans[r];
      const float2 l = maps[(size_t)r * DD + p];
      const float e = ex2f(b * (L * -kLog2e));
      x0 = make_float2(fmaf(e, x0.x, l.x), fmaf(e, fmaf(L, x0.x, x0.y), l.y));
    }
  }
  auto apply = [&](const AffMap& M, float2 x) {
    return make_float2(fmaf(M.E, x.x, M.Sb), fmaf(M.E, fmaf(M.L, x.x, x.y), M.Qb));
  };
  if (seg == kScanS - 1) {
    fin[p] = apply(m, x0);
    if (rankmap) rankmap[p] = make_float2(m.Sb, m.Qb);
    if (rankspan && p == 0) rankspan[0] = m.L;
  }
  if (mode == 1) return;
  // state entering segment seg = (inclusive map of segment seg-1) applied to the carried state
  float2 x = seg > 0 ? apply(prevm, x0) : x0;
  for (int64_t c = c0; c < c1; c += kScanB) {
    float Lb[kScanB];
    float2 lb[kScanB];
#pragma unroll
    for (int k = 0; k < kScanB; k++) {
      const bool in = c + k < c1;
      Lb[k] = in ? cspan[c + k] : 0.0f;
      lb[k] = in ? loc[(c + k) * DD + p] : make_float2(0.0f, 0.0f);
    }
#pragma unroll
    for (int k = 0; k < kScanB; k++) {
      if (c + k < c1) {
        carry[(c + k) * DD + p] = x;
        const float e = ex2f(b * (Lb[k] * -kLog2e));
        x = make_float2(fmaf(e, x.x, lb[k].x), fmaf(e, fmaf(Lb[k], x.x, x.y), lb[k].y));
      }
    }
  }
}

// Phase 3: full event loop per chunk from its carried-in state; per-chunk partial sums.
template <int DP>
__global__ void __launch_bounds__(128, 4)
k_seq_eval(int D, int64_t C, const int64_t* __restrict__ cstart, const int64_t* __restrict__ cbeg,
           const float* __restrict__ t32, const float* __restrict__ dtp,
           const uint8_t* __restrict__ mk, const float* __restrict__ theta,
           const float* __restrict__ alpha, const float* __restrict__ beta,
           const float2* __restrict__ carry, double* __restrict__ rpart, int grad,
           const int* __restrict__ ctl, int has_history) {
  if (ctl && ctl[0] == 1 && grad) return;
  extern __shared__ __align__(16) unsigned char smem[];
  using SM = Smem<DP>;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane / DP, j = lane % DP;
  const int gbase = g * DP;
  float2* base = reinterpret_cast<float2*>(smem + wid * SM::per_warp) + SM::group_off(g);
  float2* A = base;
  float2* SQ = base + SM::AS;
  float2* Gs = base + 2 * SM::AS;
  const int64_t c = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wid) * SM::G + g;
  const bool live = c < C;
  const size_t DD = (size_t)D * D;
  // parameters and the carried-in state go straight to shared memory with cp.async (one round
  // trip at the wait below instead of one per row: this prologue was ~15% of the kernel)
  for (int i = 0; i < DP; i++) {
    const bool real = live && i < D && j < D;
    float2* a = &A[SM::e(i, j)];
    if (real) {
      float* af = reinterpret_cast<float*>(a);
      const bool sw = ab_swapped<DP>(i);
      cp_async<4>(af + (sw ? 1 : 0), alpha + (size_t)i * D + j);
      cp_async<4>(af + (sw ? 0 : 1), beta + (size_t)i * D + j);
      cp_async<8>(&SQ[SM::e(i, j)], carry + (size_t)c * DD + (size_t)i * D + j);
    } else {
      *a = ab_pack<DP>(i, 0.0f, 1.0f);
      SQ[SM::e(i, j)] = make_float2(0.0f, 0.0f);
    }
    gzero<DP>(Gs, i, j);
  }
  cp_async_wait_all();
  A[SM::e(DP, j)] = ab_pack<DP>(DP, j == 0 ? 1.0f : 0.0f, 0.0f);
  SQ[SM::e(DP, j)] = make_float2(j == 0 ? 1.0f : 0.0f, 0.0f);
  if constexpr (!SM::SW) {   // the swizzled layout has no null column (eval.cuh Smem)
    A[SM::e(j, DP)] = make_float2(0.0f, 0.0f);
    SQ[SM::e(j, DP)] = make_float2(0.0f, 0.0f);
  }
  const float th = (live && j < D) ? theta[j] : 0.0f;
  __syncwarp();
  const int n = live ? (int)(cstart[c + 1] - cstart[c]) : 0;
  int nmax = n;
  for (int o = 16; o >= 1; o >>= 1) nmax = max(nmax, __shfl_xor_sync(kFull, nmax, o));
  float last, gth;
  double lsum;
  // chunk 0 starts from an empty history (anchor -1, as a window); later chunks from a state
  // anchored at their base (relative time 0; their events are strictly later, R2/R10)
  const float last0 = (c == 0 && !has_history) ? -1.0f : 0.0f;
  if (grad)
    event_loop<DP, true, false>(A, SQ, Gs, j, gbase, t32, dtp, mk, live ? cbeg[c] : 0, n, nmax, th, last,
                         gth, lsum, last0);
  else
    event_loop<DP, false, false>(A, SQ, Gs, j, gbase, t32, dtp, mk, live ? cbeg[c] : 0, n, nmax, th,
                          last, gth, lsum, last0);
  lsum = group_sum_d<DP>(lsum);
  // Phase 4a, first stage, fused: the block's 4G chunks are summed in a fixed order (fp64) into
  // one record [2 D^2 gradient accumulators | D g_theta | sum lg2 lambda]; groups past the
  // last chunk (their loads were clamped to chunk 0's events) are skipped.  Scratch for g_theta
  // and the lsum: the group's parameter array A (no longer read).
  float* scf = reinterpret_cast<float*>(A);
  double* scd = reinterpret_cast<double*>(A + SM::e(1, 0));
  scf[j] = gth;
  if (j == 0) scd[0] = lsum;
  __syncthreads();
  constexpr int NG = 4 * SM::G;   // chunks (groups) per block
  const int NE = (int)(2 * DD) + D + 1;
  const int nq = (int)min((int64_t)NG, C - (int64_t)blockIdx.x * NG);
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    // the element's float offset from a group's base, computed once per element (not per chunk:
    // the runtime divisions by D were ~15% of this kernel); kind 0: a gradient accumulator
    // (NGC copies), 1: g_theta (float scratch), 2: sum lg2 lambda (double scratch)
    int kind, off = 0;
    if (e < (int)(2 * DD)) {
      const int pr = e >> 1;
      kind = 0;
      off = 2 * (2 * SM::AS + SM::ge(pr / D, pr % D)) + (e & 1);
    } else if (e < (int)(2 * DD) + D) {
      kind = 1;
      off = e - (int)(2 * DD);
    } else {
      kind = 2;
    }
    double acc = 0.0;
    if (kind == 2 || grad) {
      for (int q = 0; q < nq; q++) {
        const float2* gb = reinterpret_cast<const float2*>(smem + (q / SM::G) * SM::per_warp) +
                           SM::group_off(q % SM::G);
        const float* gf = reinterpret_cast<const float*>(gb);
        if (kind == 0) {
          float v = gf[off];
#pragma unroll
          for (int k = 1; k < SM::NGC; k++) v += gf[off + 2 * k * SM::GS];
          acc += (double)v;
        } else if (kind == 1) {
          acc += (double)gf[off];
        } else {
          acc += *reinterpret_cast<const double*>(gb + SM::e(1, 0));
        }
      }
    }
    rpart[(size_t)blockIdx.x * NE + e] = acc;
  }
}

// Phase 4a, second stage: one warp per element; lane l sums block records l, l+32, ... in
// order, then a fixed xor-butterfly combines the 32 lane sums (deterministic: the order never
// depends on timing).  (The first stage, per-block sums over chunks, ends k_seq_eval.)
__global__ void __launch_bounds__(256)
k_seq_reduce2(int D, int64_t nblk, const double* __restrict__ part, float2* __restrict__ gsum,
              float* __restrict__ gth, double* __restrict__ ls, int grad, const int* __restrict__ ctl,
              double* __restrict__ raw) {
  if (ctl && ctl[0] == 1 && grad) return;
  const int DD = D * D, NE = 2 * DD + D + 1;
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (e >= NE) return;
  double acc = 0.0;
#pragma unroll 4
  for (int64_t q = lane; q < nblk; q += 32) acc += part[(size_t)q * NE + e];
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane != 0) return;
  if (raw) raw[e] = acc;   // f1: the slice's exact partial sums, all-reduced across ranks
  if (e < 2 * DD) {
    if (grad) reinterpret_cast<float*>(gsum)[e] = (float)acc;
  } else if (e < 2 * DD + D) {
    if (grad) gth[e - 2 * DD] = (float)acc;
  } else {
    ls[0] = acc;
  }
}

// Fit gate: an invalid sequence is not fitted; its validation bits go to the caller's status.
__global__ void k_seq_gate(const int32_t* __restrict__ pst, int* __restrict__ ctl,
                           int32_t* __restrict__ status) {
  const int s = pst[0];
  status[0] = s;
  if (s & MDHP_ST_INVALID) ctl[0] = 1;
}

// Phase 4b: epilogue (+ optional optimizer step for the sequence fit).  One block of D^2
// threads (thread = pair (i, j), target-major), rounded up to whole warps.
__device__ __forceinline__ double block_sum_d(double v, double* red) {
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); k++) s += red[k];   // fixed order: deterministic
  __syncthreads();
  return s;
}
inline unsigned finish_threads(int D) { return (unsigned)(((D * D + 31) / 32) * 32); }

__global__ void __launch_bounds__(1024)
k_seq_finish(int D, int Dp, double T, const float* __restrict__ tail,
             const int32_t* __restrict__ cnt, const float* __restrict__ umax,
             const float* __restrict__ mom, const float2* __restrict__ fin,
             const float2* __restrict__ gsum, const float* __restrict__ gthv,
             const double* __restrict__ ls, float* __restrict__ theta, float* __restrict__ alpha,
             float* __restrict__ beta, double* __restrict__ lnl_out, float* __restrict__ g_theta,
             float* __restrict__ g_alpha, float* __restrict__ g_beta, int grad,
             // fit-only arguments (ctl == nullptr: plain evaluation)
             int* __restrict__ ctl_i, FitCfgDev cfg, float* __restrict__ prev,
             float* __restrict__ opt, float* __restrict__ trace, int64_t n_events,
             int32_t* __restrict__ status_out, int32_t* __restrict__ iters_out,
             const int32_t* __restrict__ pstatus) {
  const bool invalid = (pstatus[0] & MDHP_ST_INVALID) != 0;
  SeqCtl* ctl = reinterpret_cast<SeqCtl*>(ctl_i);
  if (ctl && ctl->done && grad) return;
  __shared__ double red[32];
  __shared__ int okflag;
  const int tid = threadIdx.x;
  const int DD = D * D;
  const int j = tid % D;
  const bool pair = tid < DD;
  if (tid == 0) okflag = 1;
  // everything this thread may need, loaded up front (one memory round trip instead of a
  // chain: parameters, and in a fit step the Adam moments of its theta/alpha/beta entries)
  const float a_cur = pair ? alpha[tid] : 0.0f, b_cur = pair ? beta[tid] : 1.0f;
  const float th_cur = tid < D ? theta[tid] : 0.0f;
  const size_t P = (size_t)D + 2 * (size_t)DD;
  const bool adam_step = ctl && grad && cfg.optimizer == MDHP_OPT_ADAM;
  float mth = 0.0f, vth = 0.0f, ma = 0.0f, va = 0.0f, mb = 0.0f, vb = 0.0f;
  if (adam_step) {
    if (tid < D) { mth = opt[tid]; vth = opt[P + tid]; }
    if (pair) { ma = opt[D + tid]; va = opt[P + D + tid]; mb = opt[D + DD + tid]; vb = opt[P + D + DD + tid]; }
  }
  __syncthreads();
  double part3 = 0.0;
  float da = 0.0f, db = 0.0f;
  if (pair) {
    ColInfo ci;
    ci.real = true;
    ci.T = tail[0];       // T - (last event): the final state is anchored at the last event
    ci.last = 0.0f;
    ci.N = cnt[j];
    ci.umax = umax[j];
    Series S;
    load_series(S, mom + (size_t)j * kMom, ci.N > 0);
    const float a = a_cur, b = b_cur;
    const float2 f = fin[tid];
    float Eb, Hb2;
    compensator(ci, S, b, f.x, f.y, Eb, Hb2);
    part3 = (double)(a * Eb);
    if (grad) {
      const float2 gg = gsum[tid];
      da = gg.x + Eb;
      db = fmaf(-a, gg.y, a * Hb2);
      if (!isfinite(da) || !isfinite(db)) okflag = 0;
    }
  }
  double sth = (tid < D) ? (double)th_cur : 0.0;
  float dth = 0.0f;
  if (grad && tid < D) {
    dth = gthv[tid] - (float)T;
    if (!isfinite(dth)) okflag = 0;
  }
  const double p3 = block_sum_d(part3, red);
  const double lnl = (double)kLn2 * ls[0] + p3 - T * block_sum_d(sth, red);
  if (!ctl) {
    if (tid == 0) lnl_out[0] = invalid ? (double)NAN : lnl;
    if (grad) {
      if (tid < D) g_theta[tid] = invalid ? NAN : dth;
      if (pair) {
        g_alpha[tid] = invalid ? NAN : da;
        g_beta[tid] = invalid ? NAN : db;
      }
    }
    return;
  }
  // ---- sequence fit: one iteration of the loop of DESIGN.md "Fit" (same as k_fit)
  if (!grad) {   // final evaluation at the returned point
    if (tid == 0) {
      lnl_out[0] = invalid ? (double)NAN : lnl;
      iters_out[0] = ctl->it;
      status_out[0] |= ctl->st;
    }
    return;
  }
  const bool finite = okflag && isfinite(lnl);
  __shared__ int act;   // 0 = stop, 1 = step, 2 = rollback
  __shared__ float lr_s;
  __shared__ int s_s;
  if (tid == 0) {
    act = 0;
    if (!finite) {
      ctl->st |= MDHP_ST_NONFINITE;
      if (!ctl->have_prev || ctl->halv >= cfg.max_halvings) {
        ctl->st |= MDHP_ST_DIVERGED;
        ctl->done = 1;
        act = ctl->have_prev ? 2 : 0;
      } else {
        ctl->lr_w *= 0.5f;
        ctl->halv++;
        ctl->it++;
        act = 2;
      }
    } else {
      if (trace) trace[ctl->it] = (float)lnl;
      bool stop = false;
      if (cfg.tol_rel > 0.0f && ctl->have_lnl) {
        const double thr = (double)cfg.tol_rel * fmax(fabs(ctl->lnl_prev), 1.0);
        ctl->stall = (fabs(lnl - ctl->lnl_prev) <= thr) ? ctl->stall + 1 : 0;
        if (ctl->stall >= cfg.patience) {
          ctl->st |= MDHP_ST_CONVERGED;
          ctl->done = 1;
          stop = true;
        }
      }
      if (!stop) {
        ctl->lnl_prev = lnl;
        ctl->have_lnl = 1;
        ctl->have_prev = 1;
        ctl->s++;
        act = 1;
      }
    }
    lr_s = ctl->lr_w;
    s_s = ctl->s;
  }
  __syncthreads();
  if (act == 2) {   // roll back to the previous point
    if (tid < D) theta[tid] = prev[tid];
    if (pair) {
      alpha[tid] = prev[D + tid];
      beta[tid] = prev[D + DD + tid];
    }
  } else if (act == 1) {
    // save the previous point, then step
    if (tid < D) prev[tid] = th_cur;
    if (pair) {
      prev[D + tid] = a_cur;
      prev[D + DD + tid] = b_cur;
    }
    const float lr_w = lr_s;
    const int s = s_s;
    const float scale = (cfg.loss_mean && n_events > 0) ? 1.0f / (float)n_events : 1.0f;
    const bool adam = cfg.optimizer == MDHP_OPT_ADAM;
    const float bc1 = adam ? 1.0f - powf(cfg.b1, (float)s) : 1.0f;
    const float sbc2 = adam ? sqrtf(1.0f - powf(cfg.b2, (float)s)) : 1.0f;
    auto upd = [&](float p, float g, size_t q, float m0, float v0, float lo) -> float {
      const float gl = -g * scale;
      if (adam) {
        const float mm = cfg.b1 * m0 + (1.0f - cfg.b1) * gl;
        const float vv = cfg.b2 * v0 + (1.0f - cfg.b2) * gl * gl;
        opt[q] = mm;
        opt[P + q] = vv;
        p = p - (lr_w / bc1) * (mm / (sqrtf(vv) / sbc2 + cfg.eps));
      } else {
        p = p - lr_w * gl;
      }
      return p < lo ? lo : p;
    };
    if (tid < D && (cfg.fit_mask & MDHP_FIT_THETA))
      theta[tid] = upd(th_cur, dth, tid, mth, vth, cfg.min_param);
    if (pair) {
      if (cfg.fit_mask & MDHP_FIT_ALPHA) alpha[tid] = upd(a_cur, da, D + tid, ma, va, 0.0f);
      if (cfg.fit_mask & MDHP_FIT_BETA) beta[tid] = upd(b_cur, db, D + DD + tid, mb, vb, cfg.min_param);
    }
  }
  // only thread 0 touches the control block
  if (tid == 0) {
    if (act == 1) ctl->it++;
    if (ctl->it >= cfg.max_iters) ctl->done = 1;
  }
}

// ---------------------------------------------------------------- host side
int seq_pack_launch(int D, int64_t N, int ce, double T, double t0, const double* t,
                    const int32_t* mark, void* packed, int32_t* status_out, cudaStream_t st) {
  const SeqLayout L = make_seq_layout(D, N, ce);
  if (cudaMemsetAsync(at<int32_t>(packed, L.status), 0, sizeof(int32_t), st) != cudaSuccess)
    return MDHP_ECUDA;
  const int64_t C = L.C;
  if (C > 0) {
    k_seq_bounds<<<(unsigned)((C + 1 + 255) / 256), 256, 0, st>>>(
        N, C, ce, t, at<int64_t>(packed, L.cstart), at<int64_t>(packed, L.cbeg));
    const unsigned blocks = (unsigned)((C + kSeqWPB - 1) / kSeqWPB);
    k_seq_events<<<blocks, kSeqWPB * 32, 0, st>>>(
        D, L.Dp, N, C, T, t0, t, mark, at<int64_t>(packed, L.cstart), at<int64_t>(packed, L.cbeg),
        at<float>(packed, L.cspan), at<float>(packed, L.t32), at<float>(packed, L.dtp),
        at<uint8_t>(packed, L.mark), at<int32_t>(packed, L.ccnt), at<double>(packed, L.cfirst),
        at<int32_t>(packed, L.status));
    count_launch(2);
  }
  k_seq_stats<<<1, 256, 0, st>>>(D, L.Dp, N, C, T, t, at<int32_t>(packed, L.ccnt),
                                at<double>(packed, L.cfirst), at<int32_t>(packed, L.cnt),
                                at<float>(packed, L.umax), at<float>(packed, L.tail),
                                at<int32_t>(packed, L.status));
  count_launch(1);
  if (C > 0) {
    k_seq_moments<<<(unsigned)((C + kSeqWPB - 1) / kSeqWPB), kSeqWPB * 32, 0, st>>>(
        D, L.Dp, C, T, t, mark, at<int64_t>(packed, L.cstart), at<float>(packed, L.umax),
        at<float>(packed, L.cmom));
    count_launch(1);
  }
  if (cudaMemsetAsync(at<float>(packed, L.mom), 0, sizeof(float) * L.Dp * kMom, st) != cudaSuccess)
    return MDHP_ECUDA;
  if (C > 0) {
    k_seq_momsum<<<L.Dp * kMom, 256, 0, st>>>(L.Dp, C, at<float>(packed, L.cmom),
                                              at<float>(packed, L.mom));
    count_launch(1);
  }
  if (status_out &&
      cudaMemcpyAsync(status_out, at<int32_t>(packed, L.status), sizeof(int32_t),
                      cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return MDHP_ECUDA;
  return cudaGetLastError() == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
}

struct SeqDist {   // multi-GPU slice context (f1); all null/zero for a whole sequence
  const float2* maps = nullptr;
  const float* spans = nullptr;
  int rank = 0;
  int has_history = 0;
  float2* rankmap = nullptr;
  float* rankspan = nullptr;
  int maps_only = 0;
  int skip_local = 0;   // mdhp_seq_parts after mdhp_seq_maps: local states and scan segment maps reused
};

template <int DP>
static void seq_phases_t(const SeqLayout& L, const void* pk, const float* th, const float* al,
                         const float* be, const SeqWork& w, int grad, const int* ctl,
                         cudaStream_t st, const SeqDist& sd) {
  const int64_t C = L.C;
  if (C == 0) return;
  constexpr int G = 32 / DP;
  const unsigned blk = (unsigned)((C + 4 * G - 1) / (4 * G));
  const size_t lsm = (size_t)4 * G * DP * (DP + 1) * (kLocNC * sizeof(float2) + sizeof(float));
  if (!sd.skip_local) {
    k_seq_local<DP><<<blk, 128, lsm, st>>>(L.D, C, at<int64_t>(pk, L.cstart), at<int64_t>(pk, L.cbeg),
                                         at<float>(pk, L.cspan), at<float>(pk, L.t32),
                                         at<float>(pk, L.dtp), at<uint8_t>(pk, L.mark), be, w.loc,
                                         grad ? ctl : nullptr);
    count_launch();
  }
  k_seq_scan<<<(L.D * L.D + kScanP - 1) / kScanP, kScanP * kScanS, 0, st>>>(L.D, C, at<float>(pk, L.cspan), be, w.loc, w.carry,
                                             w.fin, grad ? ctl : nullptr, sd.maps, sd.spans,
                                             sd.rank, sd.rankmap, sd.rankspan,
                                             sd.maps_only ? 1 : (sd.skip_local ? 2 : 0), w.segmap);
  count_launch();
  if (sd.maps_only) return;
  const int has_history = sd.has_history;
  using SM = Smem<DP>;
  const size_t smem = 4 * SM::per_warp;
  k_seq_eval<DP><<<blk, 128, smem, st>>>(L.D, C, at<int64_t>(pk, L.cstart), at<int64_t>(pk, L.cbeg),
                                         at<float>(pk, L.t32), at<float>(pk, L.dtp),
                                         at<uint8_t>(pk, L.mark), th, al, be, w.carry, w.rpart,
                                         grad, ctl, has_history);
  count_launch();
}

// Dynamic shared-memory limits of the phase kernels (host-side; done before a graph capture).
template <int DP>
static void seq_set_attrs_t() {
  constexpr int G = 32 / DP;
  const size_t lsm = (size_t)4 * G * DP * (DP + 1) * (kLocNC * sizeof(float2) + sizeof(float));
  cudaFuncSetAttribute(k_seq_local<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm);
  cudaFuncSetAttribute(k_seq_eval<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(4 * Smem<DP>::per_warp));
}

static void seq_set_attrs(const SeqLayout& L) {
  static bool done[6] = {};
  int k = 0;
  while ((1 << k) < L.Dp && k < 5) k++;
  if (done[k]) return;
  done[k] = true;
  switch (L.Dp) {
    case 1: seq_set_attrs_t<1>(); break;
    case 2: seq_set_attrs_t<2>(); break;
    case 4: seq_set_attrs_t<4>(); break;
    case 8: seq_set_attrs_t<8>(); break;
    case 16: seq_set_attrs_t<16>(); break;
    case 32: seq_set_attrs_t<32>(); break;
  }
}

// Balanced chunk size (mdhp_seq_chunk_hint): phase 3 holds 4 warps x G chunks per block; fill
// whole waves of SMs x resident blocks.
template <int DP>
static int seq_chunk_hint_t(int64_t N) {
  seq_set_attrs_t<DP>();
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_seq_eval<DP>, 128,
                                                     4 * Smem<DP>::per_warp) != cudaSuccess)
    return MDHP_ECUDA;
  const int64_t wave = (int64_t)sms * (per_sm > 0 ? per_sm : 1) * 4 * (32 / DP);   // chunks
  const int64_t waves = (N + wave * 256 - 1) / (wave * 256);
  const int64_t ce = waves > 0 ? (N + wave * waves - 1) / (wave * waves) : 256;
  return (int)std::min<int64_t>(std::max<int64_t>(ce, 8), 1 << 30);
}

int seq_chunk_hint(int D, int64_t N) {
  int dp = 1;
  while (dp < D) dp <<= 1;
  switch (dp) {
    case 1: return seq_chunk_hint_t<1>(N);
    case 2: return seq_chunk_hint_t<2>(N);
    case 4: return seq_chunk_hint_t<4>(N);
    case 8: return seq_chunk_hint_t<8>(N);
    case 16: return seq_chunk_hint_t<16>(N);
    case 32: return seq_chunk_hint_t<32>(N);
  }
  return MDHP_EDIM;
}

static void seq_phases(const SeqLayout& L, const void* pk, const float* th, const float* al,
                       const float* be, const SeqWork& w, int grad, const int* ctl,
                       cudaStream_t st, const SeqDist& sd = SeqDist()) {
  seq_set_attrs(L);   // once per Dp per process (before any graph capture, see seq_fit_launch)
  switch (L.Dp) {
    case 1: seq_phases_t<1>(L, pk, th, al, be, w, grad, ctl, st, sd); break;
    case 2: seq_phases_t<2>(L, pk, th, al, be, w, grad, ctl, st, sd); break;
    case 4: seq_phases_t<4>(L, pk, th, al, be, w, grad, ctl, st, sd); break;
    case 8: seq_phases_t<8>(L, pk, th, al, be, w, grad, ctl, st, sd); break;
    case 16: seq_phases_t<16>(L, pk, th, al, be, w, grad, ctl, st, sd); break;
    case 32: seq_phases_t<32>(L, pk, th, al, be, w, grad, ctl, st, sd); break;
  }
}

static void seq_reduce(const SeqLayout& L, const SeqWork& w, int grad, const int* ctl,
                       cudaStream_t st, double* raw = nullptr) {
  if (L.C == 0) return;
  const int ne = 2 * L.D * L.D + L.D + 1;
  k_seq_reduce2<<<(ne + 7) / 8, 256, 0, st>>>(L.D, seq_eval_blocks(L.Dp, L.C), w.rpart, w.gsum,
                                              w.gth, w.ls, grad, ctl, raw);
  count_launch(1);
}

static size_t seq_work_bytes(const SeqLayout& L) {
  return make_seq_work(nullptr, L.D, L.Dp, L.C).bytes;
}

// zero-sized sequences: fin/gsum/gth/ls must read as zero
static int seq_work_init(const SeqLayout& L, void* ws, size_t bytes, cudaStream_t st) {
  return cudaMemsetAsync(ws, 0, bytes, st) == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
}

int seq_loglik_launch(int D, int64_t N, int ce, double T, const void* pk, const float* th,
                      const float* al, const float* be, double* lnl, float* gt, float* ga,
                      float* gb, cudaStream_t st) {
  const SeqLayout L = make_seq_layout(D, N, ce);
  const size_t wb = seq_work_bytes(L);
  void* ws = nullptr;
  if (cudaMallocAsync(&ws, wb, st) != cudaSuccess) return MDHP_ECUDA;
  int rc = seq_work_init(L, ws, wb, st);
  const SeqWork w = make_seq_work(ws, D, L.Dp, L.C);
  const int grad = gt != nullptr;
  seq_phases(L, pk, th, al, be, w, grad, nullptr, st);
  seq_reduce(L, w, grad, nullptr, st);
  FitCfgDev cfg{};
  k_seq_finish<<<1, finish_threads(D), 0, st>>>(D, L.Dp, T, at<float>(pk, L.tail), at<int32_t>(pk, L.cnt),
                                   at<float>(pk, L.umax), at<float>(pk, L.mom), w.fin, w.gsum,
                                   w.gth, w.ls, const_cast<float*>(th), const_cast<float*>(al),
                                   const_cast<float*>(be), lnl, gt, ga, gb, grad, nullptr, cfg,
                                   nullptr, nullptr, nullptr, N, nullptr, nullptr,
                                   at<int32_t>(pk, L.status));
  count_launch(1);
  cudaFreeAsync(ws, st);
  if (cudaGetLastError() != cudaSuccess) rc = MDHP_ECUDA;
  return rc;
}

int seq_fit_launch(int D, int64_t N, int ce, double T, const void* pk, const FitCfgDev& cfg,
                   float* th, float* al, float* be, float* opt_state, double* lnl, int32_t* iters,
                   int32_t* status, float* trace, cudaStream_t st) {
  const SeqLayout L = make_seq_layout(D, N, ce);
  const size_t wb = seq_work_bytes(L);
  void* ws = nullptr;
  if (cudaMallocAsync(&ws, wb, st) != cudaSuccess) return MDHP_ECUDA;
  int rc = seq_work_init(L, ws, wb, st);
  const SeqWork w = make_seq_work(ws, D, L.Dp, L.C);
  float* opt = opt_state ? opt_state : w.opt;
  // control block: done = (invalid input or max_iters == 0), lr_w = lr
  SeqCtl h{};
  h.lr_w = cfg.lr;
  h.s = cfg.step0;   // Adam bias-correction offset when resuming
  h.done = cfg.max_iters <= 0;
  cudaMemcpyAsync(w.ctl, &h, sizeof(SeqCtl), cudaMemcpyHostToDevice, st);
  // an invalid sequence (validation bits) is not fitted
  k_seq_gate<<<1, 1, 0, st>>>(at<const int32_t>(pk, L.status), w.ctl, status);
  count_launch(1);
  if (trace) cudaMemsetAsync(trace, 0xff, sizeof(float) * (size_t)(cfg.max_iters > 0 ? cfg.max_iters : 1), st);
  // one iteration = phases 1-3 + the two-stage reduction + finish (6 kernels), gated on the
  // device by the control block, so the host loop never reads back: it is captured once as a
  // CUDA graph and replayed max_iters times (MDHP_NO_GRAPH=1 launches the kernels directly)
  auto iteration = [&](cudaStream_t s) {
    seq_phases(L, pk, th, al, be, w, 1, w.ctl, s);
    seq_reduce(L, w, 1, w.ctl, s);
    k_seq_finish<<<1, finish_threads(D), 0, s>>>(D, L.Dp, T, at<float>(pk, L.tail), at<int32_t>(pk, L.cnt),
                                    at<float>(pk, L.umax), at<float>(pk, L.mom), w.fin, w.gsum,
                                    w.gth, w.ls, th, al, be, lnl, nullptr, nullptr, nullptr, 1,
                                    w.ctl, cfg, w.prev, opt, trace, N, status, iters,
                                    at<int32_t>(pk, L.status));
    count_launch(1);
  };
  const char* ng = getenv("MDHP_NO_GRAPH");
  if (cfg.max_iters > 1 && !(ng && ng[0] && ng[0] != '0')) {
    seq_set_attrs(L);
    // capture on a private stream (the caller's may be the legacy default stream, which
    // cannot be captured); the graph is then launched on the caller's stream
    cudaStream_t cs = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess;
    const uint64_t before = launches_so_far();
    ok = ok && cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      iteration(cs);
      ok = cudaStreamEndCapture(cs, &g) == cudaSuccess && g != nullptr;
    }
    const int per_it = (int)(launches_so_far() - before);
    ok = ok && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
    for (int it = 0; it < cfg.max_iters && ok; it++) ok = cudaGraphLaunch(ge, st) == cudaSuccess;
    if (ok) count_launch(per_it * (cfg.max_iters - 1));   // the capture counted one iteration
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    if (cs) cudaStreamDestroy(cs);
    if (!ok) {
      set_error("seq fit: CUDA graph capture/launch failed: %s",
                cudaGetErrorString(cudaGetLastError()));
      rc = MDHP_ECUDA;
    }
  } else {
    for (int it = 0; it < cfg.max_iters; it++) iteration(st);
  }
  // lnL at the returned point
  seq_phases(L, pk, th, al, be, w, 0, nullptr, st);
  seq_reduce(L, w, 0, nullptr, st);
  k_seq_finish<<<1, finish_threads(D), 0, st>>>(D, L.Dp, T, at<float>(pk, L.tail), at<int32_t>(pk, L.cnt),
                                   at<float>(pk, L.umax), at<float>(pk, L.mom), w.fin, w.gsum,
                                   w.gth, w.ls, th, al, be, lnl, nullptr, nullptr, nullptr, 0,
                                   w.ctl, cfg, w.prev, opt, trace, N, status, iters,
                                   at<int32_t>(pk, L.status));
  count_launch(1);
  cudaFreeAsync(ws, st);
  if (cudaGetLastError() != cudaSuccess) rc = MDHP_ECUDA;
  return rc;
}

size_t seq_packed_bytes(int D, int64_t N, int ce) { return make_seq_layout(D, N, ce).total; }
size_t seq_status_offset(int D, int64_t N, int ce) { return make_seq_layout(D, N, ce).status; }

// ---------------------------------------------------------------- f1: one sequence over ranks
// Stats record of a slice (fp64): [cnt Dp | umax Dp | mom Dp*kMom | tail]; partial sums record:
// [gR,gQ interleaved 2 D^2 | g_theta D | sum lg2 lambda].
__host__ __device__ inline int seq_stats_len(int Dp) { return 2 * Dp + Dp * kMom + 1; }

__global__ void k_seq_stats_out(int Dp, const int32_t* __restrict__ cnt, const float* __restrict__ umax,
                                const float* __restrict__ mom, const float* __restrict__ tail,
                                double* __restrict__ out) {
  for (int q = threadIdx.x; q < seq_stats_len(Dp); q += blockDim.x) {
    double v;
    if (q < Dp) v = cnt[q];
    else if (q < 2 * Dp) v = umax[q - Dp];
    else if (q < 2 * Dp + Dp * kMom) v = mom[q - 2 * Dp];
    else v = tail[0];
    out[q] = v;
  }
}

// Combine R slices' stats: counts add; u_max = max (= T - the global first event of the mark);
// moments rescale exactly, sum_k (u_k/U)^p = sum_r (U_r/U)^p m_p^(r); tail = min (the global
// last event).
__global__ void k_seq_stats_combine(int Dp, int R, const double* __restrict__ g, double* __restrict__ out) {
  const int S = seq_stats_len(Dp);
  for (int q = threadIdx.x; q < S; q += blockDim.x) {
    double v = 0.0;
    if (q < Dp) {
      for (int r = 0; r < R; r++) v += g[(size_t)r * S + q];
    } else if (q < 2 * Dp) {
      for (int r = 0; r < R; r++) v = fmax(v, g[(size_t)r * S + q]);
    } else if (q < 2 * Dp + Dp * kMom) {
      const int j = (q - 2 * Dp) / kMom, pw = (q - 2 * Dp) % kMom + 1;
      double U = 0.0;
      for (int r = 0; r < R; r++) U = fmax(U, g[(size_t)r * S + Dp + j]);
      for (int r = 0; r < R; r++) {
        const double Ur = g[(size_t)r * S + Dp + j];
        if (Ur > 0.0) v += pow(Ur / U, (double)pw) * g[(size_t)r * S + q];
      }
    } else {
      v = INFINITY;
      for (int r = 0; r < R; r++) v = fmin(v, g[(size_t)r * S + q]);
    }
    out[q] = v;
  }
}

// Unpack combined stats + reduced partial sums into the finish kernel's inputs (work area).
__global__ void k_seq_unpack(int D, int Dp, const double* __restrict__ stats,
                             const double* __restrict__ parts, int32_t* __restrict__ cnt,
                             float* __restrict__ umax, float* __restrict__ mom, float* __restrict__ tail,
                             float2* __restrict__ gsum, float* __restrict__ gth, double* __restrict__ ls,
                             double T) {
  const int DD = D * D;
  for (int q = threadIdx.x; q < Dp; q += blockDim.x) {
    cnt[q] = (int32_t)stats[q];
    umax[q] = (float)stats[Dp + q];
  }
  for (int q = threadIdx.x; q < Dp * kMom; q += blockDim.x) mom[q] = (float)stats[2 * Dp + q];
  if (threadIdx.x == 0) {
    tail[0] = (float)stats[2 * Dp + Dp * kMom];
    tail[1] = (float)T;
    ls[0] = parts[2 * DD + D];
  }
  for (int q = threadIdx.x; q < DD; q += blockDim.x)
    gsum[q] = make_float2((float)parts[2 * q], (float)parts[2 * q + 1]);
  for (int q = threadIdx.x; q < D; q += blockDim.x) gth[q] = (float)parts[2 * DD + q];
}

struct SeqFinishArea {   // finish inputs assembled from the global records
  int32_t* cnt;
  float *umax, *mom, *tail, *gth;
  float2* gsum;
  double* ls;
};

static SeqFinishArea finish_area(void* work, int Dp) {
  // the slice work buffer starts with a head region reserved for these small records
  char* b = static_cast<char*>(work);
  SeqFinishArea a;
  a.cnt = reinterpret_cast<int32_t*>(b);
  a.umax = reinterpret_cast<float*>(b + 256);
  a.mom = reinterpret_cast<float*>(b + 512);
  a.tail = reinterpret_cast<float*>(b + 512 + align256(sizeof(float) * Dp * kMom));
  a.gth = a.tail + 64;
  a.ls = reinterpret_cast<double*>(a.gth + 64);
  a.gsum = reinterpret_cast<float2*>(reinterpret_cast<char*>(a.ls) + 256);
  return a;
}

size_t seq_work_bytes_slice(int D, int64_t N, int ce) {
  const SeqLayout L = make_seq_layout(D, N, ce);
  const size_t wb = make_seq_work(nullptr, D, L.Dp, L.C).bytes;
  return wb + align256(8192 + sizeof(float2) * (size_t)D * D);   // + the head region of finish_area
}

static SeqWork slice_work(int D, int64_t N, int ce, void* work) {
  const SeqLayout L = make_seq_layout(D, N, ce);
  // after the head, 256-byte aligned (the work arrays include float4 segment maps)
  char* base = static_cast<char*>(work) + align256(8192 + sizeof(float2) * (size_t)D * D);
  return make_seq_work(base, D, L.Dp, L.C);
}

int seq_slice_init_launch(int D, int64_t N, int ce, void* work, const FitCfgDev* cfg, cudaStream_t st) {
  const size_t wb = seq_work_bytes_slice(D, N, ce);
  if (cudaMemsetAsync(work, 0, wb, st) != cudaSuccess) return MDHP_ECUDA;
  if (cfg) {
    SeqWork w = slice_work(D, N, ce, work);
    SeqCtl h{};
    h.lr_w = cfg->lr;
    h.s = cfg->step0;
    h.done = cfg->max_iters <= 0;
    if (cudaMemcpyAsync(w.ctl, &h, sizeof(SeqCtl), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return MDHP_ECUDA;
  }
  return MDHP_OK;
}

int seq_maps_launch(int D, int64_t N, int ce, const void* pk, const float* be, void* work,
                    float2* rankmap, float* rankspan, int fit, cudaStream_t st) {
  const SeqLayout L = make_seq_layout(D, N, ce);
  SeqWork w = slice_work(D, N, ce, work);
  if (L.C == 0) {
    cudaMemsetAsync(rankmap, 0, sizeof(float2) * (size_t)D * D, st);
    cudaMemsetAsync(rankspan, 0, sizeof(float), st);
    return cudaGetLastError() == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
  }
  SeqDist sd;
  sd.maps_only = 1;
  sd.rankmap = rankmap;
  sd.rankspan = rankspan;
  seq_phases(L, pk, nullptr, nullptr, be, w, fit, fit ? w.ctl : nullptr, st, sd);
  return cudaGetLastError() == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
}

int seq_parts_launch(int D, int64_t N, int ce, const void* pk, const float* th, const float* al,
                     const float* be, const float2* maps, const float* spans, int rank,
                     int has_history, void* work, double* parts, float2* fin, int grad, int fit,
                     cudaStream_t st) {
  const SeqLayout L = make_seq_layout(D, N, ce);
  SeqWork w = slice_work(D, N, ce, work);
  const size_t DD = (size_t)D * D;
  if (L.C == 0) {
    // empty slice: no partial sums; its end state is the carried-in state (maps of earlier ranks)
    cudaMemsetAsync(parts, 0, sizeof(double) * (2 * DD + D + 1), st);
    k_seq_scan<<<(D * D + kScanP - 1) / kScanP, kScanP * kScanS, 0, st>>>(D, 0, nullptr, be, nullptr, nullptr, fin,
                                                          nullptr, maps, spans, rank, nullptr,
                                                          nullptr, 1, nullptr);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
  }
  SeqDist sd;
  sd.maps = maps;
  sd.spans = spans;
  sd.rank = rank;
  sd.has_history = has_history;
  sd.skip_local = 1;   // the local states of mdhp_seq_maps (same work, same beta) are reused
  seq_phases(L, pk, th, al, be, w, grad, fit ? w.ctl : nullptr, st, sd);
  seq_reduce(L, w, grad, fit ? w.ctl : nullptr, st, parts);
  cudaMemcpyAsync(fin, w.fin, sizeof(float2) * DD, cudaMemcpyDeviceToDevice, st);
  return cudaGetLastError() == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
}

int seq_local_stats_launch(int D, int64_t N, int ce, const void* pk, double* stats, cudaStream_t st) {
  const SeqLayout L = make_seq_layout(D, N, ce);
  k_seq_stats_out<<<1, 256, 0, st>>>(L.Dp, at<int32_t>(pk, L.cnt), at<float>(pk, L.umax),
                                     at<float>(pk, L.mom), at<float>(pk, L.tail), stats);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
}

int seq_combine_stats_launch(int D, int R, const double* gathered, double* combined, cudaStream_t st) {
  int Dp = 1;
  while (Dp < D) Dp <<= 1;
  k_seq_stats_combine<<<1, 256, 0, st>>>(Dp, R, gathered, combined);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
}

// Epilogue (+ optional fit step) from global records; identical on every rank.
int seq_finish_launch(int D, int64_t N_total, int ce, int64_t N_slice, double T,
                      const double* stats, const double* parts, const float2* fin, float* th,
                      float* al, float* be, double* lnl, float* gt, float* ga, float* gb,
                      const FitCfgDev* cfg, void* work, float* opt, float* trace, int32_t* status,
                      int32_t* iters, int final_eval, const int32_t* pstatus, cudaStream_t st) {
  const SeqLayout L = make_seq_layout(D, N_slice, ce);
  SeqWork w = slice_work(D, N_slice, ce, work);
  const SeqFinishArea a = finish_area(work, L.Dp);
  k_seq_unpack<<<1, 256, 0, st>>>(D, L.Dp, stats, parts, a.cnt, a.umax, a.mom, a.tail, a.gsum,
                                  a.gth, a.ls, T);
  FitCfgDev c0{};
  const FitCfgDev& c = cfg ? *cfg : c0;
  const int grad = cfg ? (final_eval ? 0 : 1) : (gt != nullptr);
  k_seq_finish<<<1, finish_threads(D), 0, st>>>(D, L.Dp, T, a.tail, a.cnt, a.umax, a.mom, fin, a.gsum, a.gth,
                                   a.ls, th, al, be, lnl, gt, ga, gb, grad,
                                   cfg ? w.ctl : nullptr, c, w.prev, opt ? opt : w.opt, trace,
                                   N_total, status, iters, pstatus);
  count_launch(2);
  return cudaGetLastError() == cudaSuccess ? MDHP_OK : MDHP_ECUDA;
}

}  // namespace mdhp
