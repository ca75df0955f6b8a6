// exact.cu — fp64 re-evaluation of Eq.(5) and its gradient for the windows whose fp32 lnL
// cannot be trusted to 1e-4 relative (R17/R24).
//
// The fp32 kernels (fit.cu) estimate, per window, a bound on the absolute error of their lnL
// (needs_exact below).  Where that bound could exceed 1e-4 |lnL| — lnL is a cancellation of
// much larger terms, Part1 = sum ln lambda against Part2 + Part3 — the window index is appended
// to a device list and this kernel evaluates the window again in fp64 on the GPU (state,
// exponentials, logarithms and sums all in double) from the same packed fp32 analysis times.
// It is not a CPU fallback: it runs in the library's kernels on the same stream.
//
// One warp per listed window (persistent grid over the list), lane j < D owns source column j
// (row reads) and target row j (column updates), as the fp32 path, with the lazy recurrence
// of eval.cuh taken event by event (no chunking).  Part3 terms E_ij = sum_k expm1(-b_ij u_k) and
// F_ij = sum_k u_k e^{-b_ij u_k} are summed directly in a second pass over the events (no
// cancellation at small beta without the moment series).  Formulas: Eq.(2), Eq.(5)
// P:290-296, gradients App. B P:857-862.
#include <cmath>
#include "common.cuh"

namespace mdhp {

struct ExactSmem {
  static size_t bytes(int D) {
    return sizeof(double2) * (size_t)D * (D + 1)     // SQ[i][j] = {S, Q'} (later {E, F})
           + sizeof(double2) * (size_t)D * D         // G[i][j] = {gR, gQ}
           + sizeof(float2) * (size_t)D * D;         // K[i][j] = {alpha, beta}
  }
};

template <bool GRAD>
__global__ void __launch_bounds__(32)
k_loglik_exact(Packed P, const float* __restrict__ theta, const float* __restrict__ alpha,
               const float* __restrict__ beta, const int32_t* __restrict__ list,
               const int32_t* __restrict__ count, int64_t n_all, double* __restrict__ lnl_out,
               float* __restrict__ g_theta, float* __restrict__ g_alpha,
               float* __restrict__ g_beta, const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int D = P.D;
  const int RS = D + 1;
  double2* SQ = reinterpret_cast<double2*>(smem);
  double2* G = SQ + (size_t)D * RS;
  float2* K = reinterpret_cast<float2*>(G + (size_t)D * D);
  const int j = threadIdx.x;
  const bool lane_real = j < D;
  const int64_t nl = list ? (int64_t)*count : n_all;
  for (int64_t q = blockIdx.x; q < nl; q += gridDim.x) {
    const int64_t w = list ? (int64_t)list[q] : q;
    MDHP_ASSERT(w >= 0 && w < P.W);
    if (status[w] & MDHP_ST_INVALID) continue;   // warp-uniform
    const int n = P.n[w];
    const int64_t beg = P.begin[w];
    const double T = (double)P.T32[w];
    // parameters of column j into K, state and accumulators to 0
    double th = 0.0;
    if (lane_real) {
      th = (double)theta[w * D + j];
      for (int i = 0; i < D; i++) {
        K[i * D + j] = make_float2(alpha[(w * D + i) * D + j], beta[(w * D + i) * D + j]);
        SQ[i * RS + j] = make_double2(0.0, 0.0);
        G[i * D + j] = make_double2(0.0, 0.0);
      }
    }
    __syncwarp();
    double last = 0.0, gth = 0.0, lsum = 0.0;
    int cnt = 0;
    for (int k = 0; k < n; k++) {
      const double t = (double)P.t32[beg + k];
      const int i = P.mark[beg + k];
      MDHP_ASSERT(i >= 0 && i < D);
      // row read of target i, source column j: R_ij(t), Q_ij(t) with the strict T_j^k < t
      double R = 0.0, Q = 0.0, p = 0.0;
      if (lane_real && cnt > 0) {
        const double dl = t - last;
        const float2 kk = K[i * D + j];
        const double e = exp(-(double)kk.y * dl);
        const double2 sq = SQ[i * RS + j];
        R = e * sq.x - (dl == 0.0 ? 1.0 : 0.0);
        Q = e * (sq.y + dl * sq.x);
        p = (double)kk.x * R;
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) p += __shfl_xor_sync(kFull, p, o);
      const double lam = __shfl_sync(kFull, th, i) + p;
      lsum += log(lam);
      const double wgt = 1.0 / lam;
      if (GRAD && lane_real) {
        double2 g = G[i * D + j];
        g.x += R * wgt;
        g.y += Q * wgt;
        G[i * D + j] = g;
        if (j == i) gth += wgt;
      }
      // column update of source i for target row j (all row reads of this event done above)
      const double last_i = __shfl_sync(kFull, last, i);
      const int cnt_i = __shfl_sync(kFull, cnt, i);
      __syncwarp();
      if (lane_real) {
        double2 sq = SQ[j * RS + i];
        if (cnt_i > 0) {
          const double g = t - last_i;
          const double d = exp(-(double)K[j * D + i].y * g);
          sq = make_double2(d * sq.x + 1.0, d * (sq.y + g * sq.x));
        } else {
          sq = make_double2(1.0, 0.0);
        }
        SQ[j * RS + i] = sq;
      }
      if (j == i) {
        last = t;
        cnt++;
      }
      __syncwarp();
    }
    // Part3 terms summed directly: lane j (target row j) owns E_j., F_j.
    if (lane_real)
      for (int s = 0; s < D; s++) SQ[j * RS + s] = make_double2(0.0, 0.0);
    __syncwarp();
    for (int k = 0; k < n; k++) {
      const double u = T - (double)P.t32[beg + k];
      const int s = P.mark[beg + k];
      if (lane_real) {
        const double b = (double)K[j * D + s].y;
        double2 ef = SQ[j * RS + s];
        ef.x += expm1(-b * u);
        ef.y += u * exp(-b * u);
        SQ[j * RS + s] = ef;
      }
    }
    __syncwarp();
    double part3 = 0.0;
    if (lane_real) {
      for (int s = 0; s < D; s++) {
        const float2 kk = K[j * D + s];
        const double a = kk.x, b = kk.y;
        const double2 ef = SQ[j * RS + s];
        part3 += a / b * ef.x;
        if (GRAD) {
          const double2 g = G[j * D + s];
          const double da = g.x + ef.x / b;
          const double db = -a * g.y - a * ef.x / (b * b) - a * ef.y / b;
          g_alpha[(w * D + j) * D + s] = (float)da;
          g_beta[(w * D + j) * D + s] = (float)db;
        }
      }
      if (GRAD) g_theta[w * D + j] = (float)(gth - T);
    }
    double sth = lane_real ? th : 0.0;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      part3 += __shfl_xor_sync(kFull, part3, o);
      sth += __shfl_xor_sync(kFull, sth, o);
    }
    if (j == 0) lnl_out[w] = lsum - T * sth + part3;
    __syncwarp();
  }
}

int exact_launch(const Packed& P, const float* th, const float* al, const float* be,
                 const int32_t* list, const int32_t* count, double* lnl, float* gt, float* ga,
                 float* gb, const int32_t* status, cudaStream_t st) {
  if (P.W == 0) return MDHP_OK;
  const size_t smem = ExactSmem::bytes(P.D);
  auto kern = gt ? k_loglik_exact<true> : k_loglik_exact<false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("cudaFuncSetAttribute(k_loglik_exact) failed");
    return MDHP_ECUDA;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // a listed batch is small (cancellation windows only); the grid is a fixed wave that exits
  // at once when the list is empty, so no device->host read of the count is needed
  int64_t blocks = (int64_t)sms * 4;
  if (!list && blocks > P.W) blocks = P.W;
  kern<<<(unsigned)blocks, 32, smem, st>>>(P, th, al, be, list, count, P.W, lnl, gt, ga, gb,
                                           status);
  count_launch();
  return MDHP_OK;
}

}  // namespace mdhp
