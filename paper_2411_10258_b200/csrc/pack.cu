// pack.cu — mdhp_pack_windows: validation, fp32 conversion, per-mark gaps, counts, power
// moments and longest-first window order (row a1 of DESIGN.md section 4).
//
// The paper's Stage 1 standardises (Eq.(6)), pads to (dim, maxTimeLen) and builds
// the 4-D tMpT tensor of all pairwise differences.  Here the parameter-independent work is the
// per-event gap to the previous same-mark event (what the lazy recurrence needs) and the
// per-(window, mark) power moments of T - t (what the small-beta Part3 epilogue needs): O(N*D)
// bytes instead of O(N^2).
#include <cmath>
#include "common.cuh"

namespace mdhp {

constexpr int kPackWPB = 4;  // warps per block (one window per warp)

__device__ __forceinline__ int64_t round8(int64_t x) { return (x + 7) & ~int64_t(7); }

// One warp per window.  Pass 1 (EQ6 only): joint min/max.  Pass 2: chunks of 32 events.
__global__ void __launch_bounds__(kPackWPB * 32)
k_pack_events(int D, int Dp, int mode, double lo, double hi, int nudge, int64_t W,
              const double* __restrict__ t, const int32_t* __restrict__ mark,
              const int64_t* __restrict__ off, const double* __restrict__ Tin,
              int64_t* __restrict__ o_begin, int32_t* __restrict__ o_n, float* __restrict__ o_T32,
              float* __restrict__ o_t32, float* __restrict__ o_dtp, uint8_t* __restrict__ o_mark,
              int32_t* __restrict__ o_cnt, float* __restrict__ o_umax, int32_t* __restrict__ o_status) {
  __shared__ float s_last[kPackWPB][32];
  __shared__ float s_first[kPackWPB][32];
  __shared__ int s_cnt[kPackWPB][32];
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * kPackWPB + wp;
  if (w >= W) return;
  const int64_t a = off[w];
  int64_t n = off[w + 1] - a;
  const double T = Tin[w];
  int st = 0;
  if (n < 0) { st |= MDHP_ST_OUT_OF_RANGE; n = 0; }
  if (!(T > 0.0) || !isfinite(T)) st |= MDHP_ST_BAD_T;
  if (n == 0) st |= MDHP_ST_EMPTY;
  const int64_t beg = round8(a) + (int64_t)kWinStride * w;

  double mn = INFINITY, mx = -INFINITY;
  if (mode == MDHP_TIME_EQ6) {
    for (int64_t k = lane; k < n; k += 32) {
      double v = t[a + k];
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
    for (int o = 16; o >= 1; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
      mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
    }
    if (n > 0 && !(mx > mn)) st |= MDHP_ST_DEGENERATE;
  }
  const double Tp = (mode == MDHP_TIME_UNIT) ? 1.0 : (mode == MDHP_TIME_EQ6 ? hi : T);
  const float T32 = (float)Tp;

  s_last[wp][lane] = -1.0f;
  s_first[wp][lane] = 0.0f;
  s_cnt[wp][lane] = 0;
  __syncwarp();
  double carry = -INFINITY;
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
    // conversion; __d*_rn prevents FMA contraction so rounding matches the definition
    double x = tk;
    if (mode == MDHP_TIME_UNIT) x = __ddiv_rn(tk, T);
    else if (mode == MDHP_TIME_EQ6)
      x = __dadd_rn(__dmul_rn(__ddiv_rn(__dsub_rn(tk, mn), __dsub_rn(mx, mn)), __dsub_rn(hi, lo)), lo);
    const float t32 = __double2float_rn(x);
    // previous event of the same mark: inside this chunk via match_any, else the carry
    const unsigned key = okmark ? (unsigned)mk : (64u + lane);
    const unsigned grp = __match_any_sync(kFull, key);
    const unsigned lower = grp & ((1u << lane) - 1u);
    const int src = lower ? (31 - __clz(lower)) : lane;
    const float tin = __shfl_sync(kFull, t32, src);
    const int cnt_before = okmark ? s_cnt[wp][mk] : 0;
    const bool has_prev = lower != 0 || cnt_before > 0;
    const float tp32 = lower ? tin : (okmark && cnt_before > 0 ? s_last[wp][mk] : -1.0f);
    if (okmark && has_prev && t32 == tp32) st |= MDHP_ST_SAME_DIM_TIE;
    if (in) {
      o_t32[beg + k] = t32;
      o_dtp[beg + k] = __fsub_rn(t32, tp32);
      o_mark[beg + k] = okmark ? (uint8_t)mk : (uint8_t)0xFF;
    }
    if (okmark && !lower && cnt_before == 0) s_first[wp][mk] = t32;
    __syncwarp();
    const bool is_last = okmark && (grp & ~((2u << lane) - 1u)) == 0u;
    if (is_last) {
      s_last[wp][mk] = t32;
      s_cnt[wp][mk] = cnt_before + __popc(grp);
    }
    __syncwarp();
  }
  st = __reduce_or_sync(kFull, st);
  if (st & (MDHP_ST_UNSORTED | MDHP_ST_BAD_MARK)) st &= ~MDHP_ST_SAME_DIM_TIE;
  if (nudge && (st & MDHP_ST_SAME_DIM_TIE)) {
    // MDHP_TIE_NUDGE: sequential fix-up of this window only (rare), in stream
    // order: y_k = max(fl32(x_k), y_{k-1}); a tie with the previous event of the same mark moves
    // y_k to the next float up.  Rewrites times, gaps and first times.
    st &= ~MDHP_ST_SAME_DIM_TIE;
    if (lane == 0) {
      float lastm[32];
      bool have[32];
      for (int q = 0; q < 32; q++) have[q] = false;
      float floor_ = -INFINITY;
      for (int64_t k = 0; k < n; k++) {
        const double tk = t[a + k];
        double x = tk;
        if (mode == MDHP_TIME_UNIT) x = __ddiv_rn(tk, T);
        else if (mode == MDHP_TIME_EQ6)
          x = __dadd_rn(__dmul_rn(__ddiv_rn(__dsub_rn(tk, mn), __dsub_rn(mx, mn)), __dsub_rn(hi, lo)), lo);
        float y = fmaxf(__double2float_rn(x), floor_);
        const int mk = mark[a + k];
        if (have[mk] && lastm[mk] == y) y = nextafterf(y, INFINITY);
        o_t32[beg + k] = y;
        o_dtp[beg + k] = __fsub_rn(y, have[mk] ? lastm[mk] : -1.0f);
        if (!have[mk]) s_first[wp][mk] = y;
        lastm[mk] = y;
        have[mk] = true;
        floor_ = y;
      }
    }
    __syncwarp();
  }
  const int64_t npad = round8(n) + 8;   // padding to 8 + one null chunk (eval.cuh: kNullT)
  MDHP_ASSERT(beg >= 0 && (beg & 7) == 0);
  for (int64_t k = n + lane; k < npad; k += 32) {
    o_t32[beg + k] = -2.0f;
    o_dtp[beg + k] = 0.0f;
    o_mark[beg + k] = (uint8_t)Dp;
  }
  if (lane < Dp) {
    const int c = lane < D ? s_cnt[wp][lane] : 0;
    o_cnt[w * Dp + lane] = c;
    o_umax[w * Dp + lane] = c > 0 ? __fsub_rn(T32, s_first[wp][lane]) : 0.0f;
  }
  if (lane == 0) {
    o_begin[w] = beg;
    o_n[w] = (int32_t)n;
    o_T32[w] = T32;
    o_status[w] = st;
  }
}

// Power moments m_p = sum_{k in j} r_k^p, r_k = (T - t_k)/u_max_j, p = 1..kMom, per (window,
// mark).  One warp per window; lane j < D owns mark j and accumulates its events in stream
// order (deterministic: no atomics, fixed summation order).
__global__ void __launch_bounds__(kPackWPB * 32)
k_pack_moments(int D, int Dp, int64_t W, const int64_t* __restrict__ begin,
               const int32_t* __restrict__ nwin, const float* __restrict__ T32v,
               const float* __restrict__ t32, const uint8_t* __restrict__ mk,
               const float* __restrict__ umax, float* __restrict__ mom,
               const int32_t* __restrict__ status) {
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * kPackWPB + wp;
  if (w >= W) return;
  const bool bad = (status[w] & MDHP_ST_INVALID) != 0;
  const int n = bad ? 0 : nwin[w];
  const int64_t beg = begin[w];
  const float T = T32v[w];
  const float um = lane < Dp ? umax[w * Dp + lane] : 0.0f;
  float acc[kMom];
#pragma unroll
  for (int p = 0; p < kMom; p++) acc[p] = 0.0f;
  for (int base = 0; base < n; base += 32) {
    const int k = base + lane;
    const float tk = k < n ? t32[beg + k] : 0.0f;
    const int mm = k < n ? (int)mk[beg + k] : 255;
    const int cnt = min(32, n - base);
    for (int s = 0; s < cnt; s++) {
      const float ts = __shfl_sync(kFull, tk, s);
      const int ms = __shfl_sync(kFull, mm, s);
      if (ms == lane) {
        const float r = um > 0.0f ? __fdiv_rn(__fsub_rn(T, ts), um) : 0.0f;
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
    float* o = mom + (w * Dp + lane) * kMom;
#pragma unroll
    for (int p = 0; p < kMom; p++) o[p] = acc[p];
  }
}

// ---- longest-first order: counting sort by n (descending) over 65536 buckets
__global__ void k_sort_hist(int64_t W, const int32_t* __restrict__ nwin,
                            const int32_t* __restrict__ status, int32_t* __restrict__ cnt) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  int b = (status[w] & MDHP_ST_INVALID) ? 0 : min(nwin[w], kSortBuckets - 1);
  atomicAdd(&cnt[kSortBuckets - 1 - b], 1);
}

// exclusive scan of kSortBuckets counters, one block of 1024 threads
__global__ void __launch_bounds__(1024) k_sort_scan(int32_t* __restrict__ cnt) {
  __shared__ int part[1024];
  constexpr int per = kSortBuckets / 1024;
  const int tid = threadIdx.x;
  int loc[per];
  int s = 0;
#pragma unroll
  for (int q = 0; q < per; q++) {
    loc[q] = cnt[tid * per + q];
    s += loc[q];
  }
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    int v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = part[tid] - s;
#pragma unroll
  for (int q = 0; q < per; q++) {
    cnt[tid * per + q] = run;
    run += loc[q];
  }
}

__global__ void k_sort_scatter(int64_t W, const int32_t* __restrict__ nwin,
                               const int32_t* __restrict__ status, int32_t* __restrict__ cursor,
                               int32_t* __restrict__ perm) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  int b = (status[w] & MDHP_ST_INVALID) ? 0 : min(nwin[w], kSortBuckets - 1);
  int pos = atomicAdd(&cursor[kSortBuckets - 1 - b], 1);
  MDHP_ASSERT(pos >= 0 && pos < W);
  perm[pos] = (int32_t)w;
}

int pack_launch(const mdhp_pack_desc* d, const double* t, const int32_t* mark,
                const int64_t* win_off, const double* T, void* packed, int32_t* win_status,
                cudaStream_t st) {
  const Layout L = make_layout(d->D, d->n_windows, d->n_events);
  char* b = static_cast<char*>(packed);
  const int64_t W = d->n_windows;
  if (W == 0) return MDHP_OK;
  int64_t* o_begin = reinterpret_cast<int64_t*>(b + L.begin);
  int32_t* o_n = reinterpret_cast<int32_t*>(b + L.n);
  float* o_T32 = reinterpret_cast<float*>(b + L.T32);
  int32_t* o_perm = reinterpret_cast<int32_t*>(b + L.perm);
  float* o_t32 = reinterpret_cast<float*>(b + L.t32);
  float* o_dtp = reinterpret_cast<float*>(b + L.dtp);
  uint8_t* o_mark = reinterpret_cast<uint8_t*>(b + L.mark);
  int32_t* o_cnt = reinterpret_cast<int32_t*>(b + L.cnt);
  float* o_umax = reinterpret_cast<float*>(b + L.umax);
  float* o_mom = reinterpret_cast<float*>(b + L.mom);
  int32_t* o_sort = reinterpret_cast<int32_t*>(b + L.sort_cnt);

  const unsigned blocks = (unsigned)((W + kPackWPB - 1) / kPackWPB);
  k_pack_events<<<blocks, kPackWPB * 32, 0, st>>>(d->D, L.Dp, d->time_mode, d->eq6_lo, d->eq6_hi,
                                                  d->tie_policy == MDHP_TIE_NUDGE, W, t, mark, win_off, T, o_begin, o_n, o_T32,
                                                  o_t32, o_dtp, o_mark, o_cnt, o_umax, win_status);
  k_pack_moments<<<blocks, kPackWPB * 32, 0, st>>>(d->D, L.Dp, W, o_begin, o_n, o_T32, o_t32,
                                                   o_mark, o_umax, o_mom, win_status);
  if (cudaMemsetAsync(o_sort, 0, sizeof(int32_t) * (kSortBuckets + 1), st) != cudaSuccess) {
    set_error("cudaMemsetAsync failed");
    return MDHP_ECUDA;
  }
  const unsigned tb = 256, gb = (unsigned)((W + tb - 1) / tb);
  k_sort_hist<<<gb, tb, 0, st>>>(W, o_n, win_status, o_sort);
  k_sort_scan<<<1, 1024, 0, st>>>(o_sort);
  k_sort_scatter<<<gb, tb, 0, st>>>(W, o_n, win_status, o_sort, o_perm);
  count_launch(5);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("pack launch failed: %s", cudaGetErrorString(e));
    return MDHP_ECUDA;
  }
  return MDHP_OK;
}

// mdhp_fit_host: a part's window offsets, copied as absolute event indices, made part-relative
__global__ void k_rebase_offsets(int64_t* __restrict__ off, int64_t n, int64_t base) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) off[i] -= base;
}

void rebase_offsets_launch(int64_t* off, int64_t n, int64_t base, cudaStream_t st) {
  k_rebase_offsets<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(off, n, base);
  count_launch();
}

}  // namespace mdhp
