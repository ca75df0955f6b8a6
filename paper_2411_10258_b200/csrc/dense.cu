// dense.cu — the paper's dense pairwise evaluation of Eq.(5), as an on-box
// ablation against the O(N D) recurrence.  Algorithm 1 sums alpha e^{-beta tMpT}
// over the 4-D tensor of all pairwise differences t - T_j^k; Algorithm 3 sums
// e^{-beta (T - T_j^k)} per pair.  Here both are written in the Eq.(5) form (R4/R5:
// causal mask T_j^k < t, the "-1" of Part3, theta not beta) and evaluated without materialising
// tMpT: one CTA per window, one thread per target event looping over all earlier events.
// O(N^2) exponentials per window and evaluation, lnL only (the paper differentiates with
// autograd).
#include <cmath>
#include "common.cuh"

namespace mdhp {

constexpr int kDenseThreads = 256;
constexpr int kDenseMaxEv = 6144;   // events staged in shared memory per window

__global__ void __launch_bounds__(kDenseThreads)
k_loglik_dense(Packed P, const float* __restrict__ theta, const float* __restrict__ alpha,
               const float* __restrict__ beta, double* __restrict__ lnl_out,
               const int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int D = P.D, RS = D + 1;
  float2* AB = reinterpret_cast<float2*>(smem);                 // [D][D+1] {alpha, beta*log2e}
  float* th = reinterpret_cast<float*>(AB + D * RS);            // [D]
  float* ts = th + 32;                                          // [kDenseMaxEv]
  uint8_t* ms = reinterpret_cast<uint8_t*>(ts + kDenseMaxEv);   // [kDenseMaxEv]
  __shared__ double red[kDenseThreads / 32];
  const int64_t w = blockIdx.x;
  if (w >= P.W) return;
  const int tid = threadIdx.x;
  if (status[w] & MDHP_ST_INVALID) {
    if (tid == 0) lnl_out[w] = NAN;
    return;
  }
  const int n = P.n[w];
  const int64_t beg = P.begin[w];
  const float T = P.T32[w];
  for (int q = tid; q < D * D; q += blockDim.x) {
    const int i = q / D, j = q % D;
    AB[i * RS + j] = make_float2(alpha[(size_t)w * D * D + q], beta[(size_t)w * D * D + q] * kLog2e);
  }
  if (tid < D) th[tid] = theta[(size_t)w * D + tid];
  const bool staged = n <= kDenseMaxEv;
  if (staged) {
    for (int k = tid; k < n; k += blockDim.x) {
      ts[k] = P.t32[beg + k];
      ms[k] = P.mark[beg + k];
    }
  }
  __syncthreads();
  const float* tg = staged ? ts : P.t32 + beg;
  const uint8_t* mg = staged ? ms : P.mark + beg;
  double acc = 0.0;
  // Part1: sum_n ln(theta_i + sum_{k: t_k < t_n} alpha_{i m_k} e^{-beta_{i m_k}(t_n - t_k)})
  for (int nn = tid; nn < n; nn += blockDim.x) {
    const float tn = tg[nn];
    const int i = mg[nn];
    float lam = th[i];
    for (int k = 0; k < nn; k++) {
      const float tk = tg[k];
      if (!(tk < tn)) continue;   // strict: coincident events do not excite (R2)
      const float2 ab = AB[i * RS + mg[k]];
      lam = fmaf(ab.x, ex2f(-ab.y * (tn - tk)), lam);
    }
    acc += (double)__logf(lam);
  }
  // Part3: sum_k sum_i (alpha_{i m_k} / beta_{i m_k}) (e^{-beta_{i m_k}(T - t_k)} - 1)
  for (int k = tid; k < n; k += blockDim.x) {
    const float u = T - tg[k];
    const int j = mg[k];
    float s = 0.0f;
    for (int i = 0; i < D; i++) {
      const float2 ab = AB[i * RS + j];
      const float b = ab.y * kLn2;
      s += ab.x / b * (ex2f(-ab.y * u) - 1.0f);
    }
    acc += (double)s;
  }
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int q = 0; q < kDenseThreads / 32; q++) s += red[q];
    double sth = 0.0;
    for (int i = 0; i < D; i++) sth += th[i];
    lnl_out[w] = s - (double)T * sth;   // Part2 = -T sum theta (Algorithm 2)
  }
}

int dense_launch(const Packed& P, const float* th, const float* al, const float* be, double* lnl,
                 const int32_t* status, cudaStream_t st) {
  if (P.W == 0) return MDHP_OK;
  const size_t smem = sizeof(float2) * P.D * (P.D + 1) + sizeof(float) * 32 +
                      sizeof(float) * kDenseMaxEv + kDenseMaxEv;
  if (cudaFuncSetAttribute(k_loglik_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("cudaFuncSetAttribute(k_loglik_dense) failed");
    return MDHP_ECUDA;
  }
  k_loglik_dense<<<(unsigned)P.W, kDenseThreads, smem, st>>>(P, th, al, be, lnl, status);
  count_launch();
  return MDHP_OK;
}

}  // namespace mdhp
