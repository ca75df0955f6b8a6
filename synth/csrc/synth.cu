// synth.cu — GPU input synthesis for MDHP benchmarks (include/synth.h).  Not the hot path;
// shares no code with libmdhp.so or oracle/.
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/synth.h"

namespace {

thread_local char g_err[256] = "";
void err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

struct U4 { uint32_t x, y, z, w; };

// Philox4x32-10 (Salmon et al. 2011), counter (c0..c3), key (k0, k1).
__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                     uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

struct Rng {
  uint32_t k0, k1, w0, w1, stream, ctr;
  U4 buf;
  int used;
  __device__ Rng(uint64_t seed, uint64_t window, uint32_t s)
      : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), w0((uint32_t)window),
        w1((uint32_t)(window >> 32)), stream(s), ctr(0), used(4) {}
  __device__ uint32_t next() {
    if (used == 4) {
      buf = philox(w0, w1, stream, ctr++, k0, k1);
      used = 0;
    }
    const uint32_t v = used == 0 ? buf.x : used == 1 ? buf.y : used == 2 ? buf.z : buf.w;
    used++;
    return v;
  }
  __device__ double uniform() { return ((double)next() + 0.5) * (1.0 / 4294967296.0); }  // (0,1)
};

__global__ void k_params(int D, int64_t W, int64_t first, uint64_t seed, synth_recipe rc,
                         float* __restrict__ theta, float* __restrict__ alpha,
                         float* __restrict__ beta, uint8_t* __restrict__ attack) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  Rng R(seed, (uint64_t)(first + w), 1u);
  double r[32], G[32 * 32];
  double rs = 0.0;
  for (int i = 0; i < D; i++) {
    r[i] = rc.rate_hi > rc.rate_lo ? exp(log(rc.rate_lo) + R.uniform() * (log(rc.rate_hi) - log(rc.rate_lo)))
                                   : rc.rate_lo;
    rs += r[i];
  }
  for (int i = 0; i < D; i++) r[i] *= rc.total_rate / rs;
  for (int k = 0; k < D * D; k++) G[k] = 0.0;
  for (int i = 0; i < D; i++) G[i * D + i] = rc.g_self_lo + R.uniform() * (rc.g_self_hi - rc.g_self_lo);
  const int kc = D > 1 ? min(rc.k_cross, D - 1) : 0;
  for (int i = 0; i < D; i++) {
    for (int c = 0; c < kc; c++) {
      int j;
      do {
        j = (i + 1 + (int)(R.uniform() * (D - 1))) % D;
      } while (G[i * D + j] != 0.0);
      G[i * D + j] = rc.g_cross_lo + R.uniform() * (rc.g_cross_hi - rc.g_cross_lo);
    }
  }
  const bool att = R.uniform() < rc.attack_frac;
  double rho = rc.rho;
  if (att) {
    rho = rc.rho_attack;
    const int na = min(rc.n_attack, D);
    int picked[32];
    for (int q = 0; q < na; q++) {
      int a;
      bool dup;
      do {
        a = (int)(R.uniform() * D) % D;
        dup = false;
        for (int z = 0; z < q; z++) dup = dup || picked[z] == a;
      } while (dup);
      picked[q] = a;
      G[a * D + a] = 0.7;
      if (D > 1) {
        const int b = (a + 1 + (int)(R.uniform() * (D - 1))) % D;
        G[a * D + b] = 0.2;
      }
    }
  }
  double mrs = 0.0;
  for (int i = 0; i < D; i++) {
    double s = 0.0;
    for (int j = 0; j < D; j++) s += G[i * D + j];
    mrs = fmax(mrs, s);
  }
  const double sc = mrs > rho ? rho / mrs : 1.0;
  for (int k = 0; k < D * D; k++) G[k] *= sc;
  const double lb0 = log(rc.beta_lo), lb1 = log(rc.beta_hi);
  for (int i = 0; i < D; i++) {
    double gr = 0.0;
    for (int j = 0; j < D; j++) {
      const double b = exp(lb0 + R.uniform() * (lb1 - lb0));
      beta[(size_t)w * D * D + i * D + j] = (float)b;
      alpha[(size_t)w * D * D + i * D + j] = (float)(G[i * D + j] * b);
      gr += G[i * D + j] * r[j];
    }
    theta[(size_t)w * D + i] = (float)fmax(r[i] - gr, 0.05 * r[i]);
  }
  if (attack) attack[w] = att ? 1 : 0;
}

// ---- Time-exciting injection: the four attack-rate shapes of Table II
// on the normalised window u = t / T in [0, 1], sampled by Algorithm 4
// (NPP): candidate gaps Exponential with mean 1/512 (S:337 reading), accept with
// probability g(u)/g_max.  Constants: DESIGN.md R23.
__host__ __device__ inline double attack_rate(int strat, double u) {
  switch (strat) {
    case SYNTH_PLA: return 1.0 * u * u;                                     // a t^b, a=1, b=2
    case SYNTH_DEA: return u < 0.6 ? 1.0 * 2.0 * u                          // W1 a1 t^(a1-1)
                                   : 1.0 * 1.2 * exp(4.0 * (u - 0.6));      // W2 a2 e^{g(t-t1)}
    case SYNTH_ASA: {
      const double e = exp(10.0 * (u - 0.5));
      return exp(10.0 * u) / ((1.0 + e) * (1.0 + e));                       // C e^{gt}/(1+e^{g(t-t0)})^2
    }
    case SYNTH_DAM: return 0.5 * 3.0 * u * u + 0.5 * 4.0 * exp(4.0 * u);     // w a1 t^(a1-1) + (1-w) a2 e^{a2 t}
    default: return 0.0;
  }
}

// max of g on [0, 1] by dense evaluation (Algorithm 6's "max(evaluate g(t))").
__host__ __device__ inline double attack_rate_max(int strat) {
  double m = 0.0;
  for (int k = 0; k <= 4096; k++) m = fmax(m, attack_rate(strat, k / 4096.0));
  return m * (1.0 + 1e-9);
}

// Algorithm 4 as a generator: next accepted normalised time (> 1 when exhausted).
struct Npp {
  int strat;
  double gmax, u, rate;
  __device__ double next(Rng& R) {
    while (true) {
      u += -log(R.uniform()) / rate;      // Delta t ~ Exponential(mean 1/rate)
      if (u > 1.0) return 2.0;
      if (R.uniform() * gmax < attack_rate(strat, u)) return u;
    }
  }
};

constexpr int kWPB = 4;

template <int RP>
__global__ void __launch_bounds__(kWPB * 32)
k_ogata(int D, int64_t W, int64_t first, uint64_t seed, double T, const float* __restrict__ theta,
        const float* __restrict__ alpha, const float* __restrict__ beta, int64_t max_events,
        const int64_t* __restrict__ win_off, int64_t* __restrict__ counts,
        double* __restrict__ t_out, int32_t* __restrict__ mark_out,
        const uint8_t* __restrict__ attack, int strat, double inj_rate) {
  __shared__ float v[kWPB][RP * 32];
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * kWPB + wp;
  if (w >= W) return;
  const int DD = D * D;
  float a[RP], b[RP], e[RP];
#pragma unroll
  for (int r = 0; r < RP; r++) {
    const int p = lane + 32 * r;
    a[r] = p < DD ? alpha[(size_t)w * DD + p] : 0.0f;
    b[r] = p < DD ? beta[(size_t)w * DD + p] : 0.0f;
    e[r] = 0.0f;
  }
  const float th = lane < D ? theta[(size_t)w * D + lane] : 0.0f;
  float sth = th;
  for (int o = 16; o >= 1; o >>= 1) sth += __shfl_xor_sync(0xffffffffu, sth, o);
  Rng R(seed, (uint64_t)(first + w), 2u);
  double now = 0.0;
  float bound = sth;
  int64_t n = 0;
  const int64_t base = win_off ? win_off[w] : 0;
  bool overflow = false;
  // injections (attack windows only): an independent stream superposed on the Hawkes traffic,
  // all on one randomly chosen ID ("one IP is randomly selected"); every lane runs the
  // same generator so the warp stays uniform
  const bool inject = strat != SYNTH_NONE && attack && attack[w];
  Rng RI(seed, (uint64_t)(first + w), 3u);
  Npp npp{strat, inject ? attack_rate_max(strat) : 1.0, 0.0, inj_rate};
  const int inj_dim = inject ? min((int)(RI.uniform() * D), D - 1) : 0;
  double inj_t = inject ? npp.next(RI) * T : 3.0 * T;
  while (bound > 0.0f) {
    const double u1 = R.uniform();
    const double u2 = R.uniform();
    const double gap = -log(u1) / (double)bound;
    const double cand = now + gap;
    if (cand > T) break;
    const float g = (float)gap;
#pragma unroll
    for (int r = 0; r < RP; r++) {
      e[r] *= __expf(-b[r] * g);
      v[wp][lane + 32 * r] = a[r] * e[r];
    }
    now = cand;
    __syncwarp();
    float lam = 0.0f;
    if (lane < D) {
      lam = th;
      for (int j = 0; j < D; j++) lam += v[wp][lane * D + j];
    }
    float cum = lam;
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, cum, o);
      if (lane >= o) cum += y;
    }
    const float total = __shfl_sync(0xffffffffu, cum, 31);
    const float u = (float)(u2 * (double)bound);
    if (u <= total) {
      const unsigned bal = __ballot_sync(0xffffffffu, lane < D && cum >= u);
      const int i = bal ? (__ffs(bal) - 1) : D - 1;
      while (inj_t <= now) {
        if (win_off && lane == 0) {
          t_out[base + n] = inj_t;
          mark_out[base + n] = inj_dim;
        }
        n++;
        inj_t = npp.next(RI) * T;
      }
      if (win_off && lane == 0) {
        t_out[base + n] = now;
        mark_out[base + n] = i;
      }
      n++;
      if (n > max_events) {
        overflow = true;
        break;
      }
#pragma unroll
      for (int r = 0; r < RP; r++) {
        const int p = lane + 32 * r;
        if (p < DD && p % D == i) e[r] += 1.0f;
      }
    }
    __syncwarp();
    float s = 0.0f;
#pragma unroll
    for (int r = 0; r < RP; r++) s += a[r] * e[r];
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    bound = sth + s;
  }
  while (!overflow && inj_t <= T) {
    if (win_off && lane == 0) {
      t_out[base + n] = inj_t;
      mark_out[base + n] = inj_dim;
    }
    n++;
    if (n > max_events) overflow = true;
    inj_t = npp.next(RI) * T;
  }
  if (!win_off && lane == 0) counts[w] = overflow ? -1 : n;
}

}  // namespace

extern "C" {

const char* synth_last_error(void) { return g_err; }

namespace {
__global__ void k_npp(int64_t W, int64_t first, uint64_t seed, int strat, double rate,
                      const int64_t* __restrict__ off, int64_t* __restrict__ counts,
                      double* __restrict__ u_out) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  Rng R(seed, (uint64_t)(first + w), 3u);
  Npp npp{strat, attack_rate_max(strat), 0.0, rate};
  (void)R.uniform();   // the injected-ID draw of k_ogata (same stream layout)
  int64_t n = 0;
  for (double u = npp.next(R); u <= 1.0; u = npp.next(R)) {
    if (off) u_out[off[w] + n] = u;
    n++;
  }
  if (!off) counts[w] = n;
}
}  // namespace

int synth_npp(int64_t W, int64_t first_window, uint64_t seed, int32_t strategy, double rate,
              const int64_t* win_off, int64_t* counts, double* u_out, void* stream) {
  if (W < 0 || strategy <= SYNTH_NONE || strategy > SYNTH_DAM || !(rate > 0.0) ||
      (!win_off && !counts) || (win_off && !u_out)) {
    err("synth_npp: bad arguments");
    return -1;
  }
  if (W == 0) return 0;
  k_npp<<<(unsigned)((W + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      W, first_window, seed, strategy, rate, win_off, counts, u_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err("synth_npp: %s", cudaGetErrorString(e));
    return -5;
  }
  return 0;
}

int synth_params(int32_t D, int64_t W, int64_t first_window, uint64_t seed, const synth_recipe* rc,
                 float* theta, float* alpha, float* beta, uint8_t* attack, void* stream) {
  if (D < 1 || D > 32 || W < 0 || !rc || !theta || !alpha || !beta) {
    err("synth_params: bad arguments");
    return -1;
  }
  if (W == 0) return 0;
  const int tb = 128;
  k_params<<<(unsigned)((W + tb - 1) / tb), tb, 0, (cudaStream_t)stream>>>(
      D, W, first_window, seed, *rc, theta, alpha, beta, attack);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err("synth_params: %s", cudaGetErrorString(e));
    return -5;
  }
  return 0;
}

int synth_ogata(int32_t D, int64_t W, int64_t first_window, uint64_t seed, double T,
                const float* theta, const float* alpha, const float* beta, int64_t max_events,
                const int64_t* win_off, int64_t* counts, double* t_out, int32_t* mark_out,
                void* stream) {
  return synth_ogata_inject(D, W, first_window, seed, T, theta, alpha, beta, max_events, win_off,
                            counts, t_out, mark_out, nullptr, SYNTH_NONE, 512.0, stream);
}

int synth_ogata_inject(int32_t D, int64_t W, int64_t first_window, uint64_t seed, double T,
                       const float* theta, const float* alpha, const float* beta,
                       int64_t max_events, const int64_t* win_off, int64_t* counts,
                       double* t_out, int32_t* mark_out, const uint8_t* attack,
                       int32_t strategy, double inj_rate, void* stream) {
  if (strategy < SYNTH_NONE || strategy > SYNTH_DAM || (strategy != SYNTH_NONE && !attack) ||
      !(inj_rate > 0.0)) {
    err("synth_ogata_inject: bad strategy/attack/rate");
    return -1;
  }
  if (D < 1 || D > 32 || W < 0 || !theta || !alpha || !beta || !(T > 0.0) ||
      (!win_off && !counts) || (win_off && (!t_out || !mark_out))) {
    err("synth_ogata: bad arguments");
    return -1;
  }
  if (W == 0) return 0;
  const unsigned blocks = (unsigned)((W + kWPB - 1) / kWPB);
  cudaStream_t st = (cudaStream_t)stream;
  const int rp = (D * D + 31) / 32;
#define SYNTH_LAUNCH(RPV) \
  k_ogata<RPV><<<blocks, kWPB * 32, 0, st>>>(D, W, first_window, seed, T, theta, alpha, beta, \
                                             max_events, win_off, counts, t_out, mark_out, \
                                             attack, strategy, inj_rate)
  if (rp <= 1) SYNTH_LAUNCH(1);
  else if (rp <= 2) SYNTH_LAUNCH(2);
  else if (rp <= 4) SYNTH_LAUNCH(4);
  else if (rp <= 8) SYNTH_LAUNCH(8);
  else if (rp <= 16) SYNTH_LAUNCH(16);
  else SYNTH_LAUNCH(32);
#undef SYNTH_LAUNCH
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err("synth_ogata: %s", cudaGetErrorString(e));
    return -5;
  }
  return 0;
}

}  // extern "C"
