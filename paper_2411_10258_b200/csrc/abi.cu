// abi.cu — the extern "C" boundary of libmdhp.so (include/mdhp.h): argument checks,
// stream-ordered workspaces, error plumbing and the end-to-end host entry point.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include "common.cuh"

namespace mdhp {


int pack_launch(const mdhp_pack_desc* d, const double* t, const int32_t* mark,
                const int64_t* win_off, const double* T, void* packed, int32_t* win_status,
                cudaStream_t st);
int loglik_launch(const Packed& P, const float* th, const float* al, const float* be, double* lnl,
                  float* gt, float* ga, float* gb, const int32_t* status, int32_t* xlist,
                  int32_t* xcount, cudaStream_t st);
int fit_launch(const Packed& P, const FitCfgDev& cfg, float* th, float* al, float* be, float* opt,
               double* lnl, int32_t* iters, int32_t* status, float* trace, int* counter,
               int32_t* xlist, int32_t* xcount, cudaStream_t st);
int exact_launch(const Packed& P, const float* th, const float* al, const float* be,
                 const int32_t* list, const int32_t* count, double* lnl, float* gt, float* ga,
                 float* gb, const int32_t* status, cudaStream_t st);

int features_launch(int D, int64_t W, int H, const float* theta, const float* alpha,
                    const float* beta, const float* T, const float* A, const float* B,
                    const float* C, float* hks, cudaStream_t st);
int dense_launch(const Packed& P, const float* th, const float* al, const float* be, double* lnl,
                 const int32_t* status, cudaStream_t st);
int seq_pack_launch(int D, int64_t N, int ce, double T, double t0, const double* t,
                    const int32_t* mark, void* packed, int32_t* status_out, cudaStream_t st);
size_t seq_work_bytes_slice(int D, int64_t N, int ce);
int seq_slice_init_launch(int D, int64_t N, int ce, void* work, const FitCfgDev* cfg, cudaStream_t st);
int seq_maps_launch(int D, int64_t N, int ce, const void* pk, const float* be, void* work,
                    float2* rankmap, float* rankspan, int fit, cudaStream_t st);
int seq_parts_launch(int D, int64_t N, int ce, const void* pk, const float* th, const float* al,
                     const float* be, const float2* maps, const float* spans, int rank,
                     int has_history, void* work, double* parts, float2* fin, int grad, int fit,
                     cudaStream_t st);
int seq_local_stats_launch(int D, int64_t N, int ce, const void* pk, double* stats, cudaStream_t st);
int seq_combine_stats_launch(int D, int R, const double* gathered, double* combined, cudaStream_t st);
int seq_finish_launch(int D, int64_t N_total, int ce, int64_t N_slice, double T,
                      const double* stats, const double* parts, const float2* fin, float* th,
                      float* al, float* be, double* lnl, float* gt, float* ga, float* gb,
                      const FitCfgDev* cfg, void* work, float* opt, float* trace, int32_t* status,
                      int32_t* iters, int final_eval, const int32_t* pstatus, cudaStream_t st);
size_t seq_status_offset(int D, int64_t N, int ce);
int seq_loglik_launch(int D, int64_t N, int ce, double T, const void* pk, const float* th,
                      const float* al, const float* be, double* lnl, float* gt, float* ga,
                      float* gb, cudaStream_t st);
int seq_fit_launch(int D, int64_t N, int ce, double T, const void* pk, const FitCfgDev& cfg,
                   float* th, float* al, float* be, float* opt_state, double* lnl, int32_t* iters,
                   int32_t* status, float* trace, cudaStream_t st);
size_t seq_packed_bytes(int D, int64_t N, int ce);
int seq_chunk_hint(int D, int64_t N);
void rebase_offsets_launch(int64_t* off, int64_t n, int64_t base, cudaStream_t st);

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

void count_launch(int k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }
uint64_t launches_so_far() { return g_launches.load(std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int check_desc(const mdhp_pack_desc* d) {
  if (!d) {
    set_error("desc is NULL");
    return MDHP_EINVAL;
  }
  if (d->D < 1 || d->D > 32) {
    set_error("D=%d outside 1..32", d->D);
    return MDHP_EDIM;
  }
  if (d->n_windows < 0 || d->n_events < 0) {
    set_error("negative sizes (W=%lld, E=%lld)", (long long)d->n_windows, (long long)d->n_events);
    return MDHP_EDIM;
  }
  if (d->time_mode < MDHP_TIME_RAW || d->time_mode > MDHP_TIME_EQ6) {
    set_error("bad time_mode %d", d->time_mode);
    return MDHP_EINVAL;
  }
  if (d->tie_policy != MDHP_TIE_ERROR && d->tie_policy != MDHP_TIE_NUDGE) {
    set_error("bad tie_policy %d", d->tie_policy);
    return MDHP_EINVAL;
  }
  if (d->time_mode == MDHP_TIME_EQ6 && !(d->eq6_hi > d->eq6_lo)) {
    set_error("EQ6 needs eq6_hi > eq6_lo (S:128)");
    return MDHP_EINVAL;
  }
  return MDHP_OK;
}

static int check_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return MDHP_ECUDA;
  }
  return MDHP_OK;
}

static int check_seq(const mdhp_seq_desc* d) {
  if (!d) {
    set_error("desc is NULL");
    return MDHP_EINVAL;
  }
  if (d->D < 1 || d->D > 32 || d->n_events < 0) {
    set_error("bad sequence dims (D=%d, N=%lld)", d->D, (long long)d->n_events);
    return MDHP_EDIM;
  }
  if (d->chunk_events < 8 || !(d->T > 0.0) || !(d->t0 >= 0.0) || d->has_history < 0 ||
      d->has_history > 1) {
    set_error("chunk_events must be >= 8, T > 0, t0 >= 0, has_history 0/1");
    return MDHP_EINVAL;
  }
  return MDHP_OK;
}

static FitCfgDev to_dev(const mdhp_fit_config* cfg) {
  FitCfgDev c;
  c.max_iters = cfg->max_iters;
  c.optimizer = cfg->optimizer;
  c.loss_mean = cfg->loss_mean;
  c.patience = cfg->patience;
  c.max_halvings = cfg->max_halvings;
  c.step0 = cfg->adam_step0;
  c.time_chunks = cfg->time_chunks;
  c.lr = cfg->lr;
  c.b1 = cfg->adam_b1;
  c.b2 = cfg->adam_b2;
  c.eps = cfg->adam_eps;
  c.tol_rel = cfg->tol_rel;
  c.min_param = cfg->min_param;
  c.fit_mask = cfg->fit_mask;
  return c;
}

static int check_cfg(const mdhp_fit_config* c) {
  if (!c) {
    set_error("cfg is NULL");
    return MDHP_EINVAL;
  }
  if (c->max_iters < 0 || !(c->lr > 0.0f) || (c->optimizer != MDHP_OPT_GD && c->optimizer != MDHP_OPT_ADAM) ||
      !(c->min_param > 0.0f) || c->patience < 0 || c->max_halvings < 0 || c->adam_step0 < 0 ||
      c->time_chunks < 0 ||
      (c->optimizer == MDHP_OPT_ADAM && !(c->adam_b1 >= 0.0f && c->adam_b1 < 1.0f &&
                                          c->adam_b2 >= 0.0f && c->adam_b2 < 1.0f && c->adam_eps >= 0.0f))) {
    set_error("invalid fit config");
    return MDHP_EINVAL;
  }
  return MDHP_OK;
}

// Raise the release threshold of the current device's default memory pool (once per device)
// so that the stream-ordered workspaces of repeated calls are reused instead of being unmapped
// and re-mapped at every synchronisation (tens of GB for mdhp_fit_host at cfg5 scale).
static void keep_pool_memory() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

}  // namespace mdhp

using namespace mdhp;

extern "C" {

int32_t mdhp_version(void) { return 1; }

const char* mdhp_last_error(void) { return g_err; }

uint64_t mdhp_launch_count(void) { return g_launches.load(); }

size_t mdhp_packed_bytes(const mdhp_pack_desc* d) {
  if (check_desc(d) != MDHP_OK) return 0;
  return make_layout(d->D, d->n_windows, d->n_events).total;
}

int mdhp_packed_layout(const mdhp_pack_desc* d, size_t* o) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (!o) {
    set_error("offsets is NULL");
    return MDHP_EINVAL;
  }
  const Layout L = make_layout(d->D, d->n_windows, d->n_events);
  const size_t v[14] = {L.begin, L.n, L.T32, L.perm, L.t32, L.dtp, L.mark, L.cnt, L.umax, L.mom,
                        L.sort_cnt, L.total, (size_t)L.Epad, (size_t)L.Dp};
  for (int k = 0; k < 14; k++) o[k] = v[k];
  return MDHP_OK;
}

int mdhp_pack_windows(const mdhp_pack_desc* d, const double* t, const int32_t* mark,
                      const int64_t* win_off, const double* T, void* packed, size_t packed_bytes,
                      int32_t* win_status, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (!packed || !win_off || !T || !win_status || (d->n_events > 0 && (!t || !mark))) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  const size_t need = make_layout(d->D, d->n_windows, d->n_events).total;
  if (packed_bytes < need) {
    set_error("packed buffer too small: %zu < %zu", packed_bytes, need);
    return MDHP_ESIZE;
  }
  rc = pack_launch(d, t, mark, win_off, T, packed, win_status, (cudaStream_t)stream);
  if (rc) return rc;
  return check_cuda("mdhp_pack_windows");
}

int mdhp_loglik_grad(const mdhp_pack_desc* d, const void* packed, const float* theta,
                     const float* alpha, const float* beta, double* loglik, float* g_theta,
                     float* g_alpha, float* g_beta, const int32_t* win_status, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (!packed || !theta || !alpha || !beta || !loglik || !win_status) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  const bool any = g_theta || g_alpha || g_beta, all = g_theta && g_alpha && g_beta;
  if (any && !all) {
    set_error("g_theta, g_alpha, g_beta must be all NULL or all non-NULL");
    return MDHP_EINVAL;
  }
  const Layout L = make_layout(d->D, d->n_windows, d->n_events);
  const Packed P = view(L, packed);
  if (P.W == 0) return MDHP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // workspace: the count and list of windows re-evaluated in fp64 (exact.cu)
  keep_pool_memory();
  void* ws = nullptr;
  const size_t ws_bytes = 256 + sizeof(int32_t) * (size_t)P.W;
  if (cudaMallocAsync(&ws, ws_bytes, st) != cudaSuccess) {
    set_error("cudaMallocAsync(%zu) failed", ws_bytes);
    return MDHP_ECUDA;
  }
  int32_t* xcount = static_cast<int32_t*>(ws);
  int32_t* xlist = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + 256);
  if (cudaMemsetAsync(xcount, 0, sizeof(int32_t), st) != cudaSuccess) {
    cudaFreeAsync(ws, st);
    set_error("cudaMemsetAsync failed");
    return MDHP_ECUDA;
  }
  rc = loglik_launch(P, theta, alpha, beta, loglik, g_theta, g_alpha, g_beta, win_status, xlist,
                     xcount, st);
  if (!rc)
    rc = exact_launch(P, theta, alpha, beta, xlist, xcount, loglik, g_theta, g_alpha, g_beta,
                      win_status, st);
  cudaFreeAsync(ws, st);
  if (rc) return rc;
  return check_cuda("mdhp_loglik_grad");
}

int mdhp_loglik_exact(const mdhp_pack_desc* d, const void* packed, const float* theta,
                      const float* alpha, const float* beta, double* loglik, float* g_theta,
                      float* g_alpha, float* g_beta, const int32_t* win_status, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (!packed || !theta || !alpha || !beta || !loglik || !win_status) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  const bool any = g_theta || g_alpha || g_beta, all = g_theta && g_alpha && g_beta;
  if (any && !all) {
    set_error("g_theta, g_alpha, g_beta must be all NULL or all non-NULL");
    return MDHP_EINVAL;
  }
  const Layout L = make_layout(d->D, d->n_windows, d->n_events);
  rc = exact_launch(view(L, packed), theta, alpha, beta, nullptr, nullptr, loglik, g_theta,
                    g_alpha, g_beta, win_status, (cudaStream_t)stream);
  if (rc) return rc;
  return check_cuda("mdhp_loglik_exact");
}

int mdhp_loglik_dense(const mdhp_pack_desc* d, const void* packed, const float* theta,
                      const float* alpha, const float* beta, double* loglik,
                      const int32_t* win_status, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (!packed || !theta || !alpha || !beta || !loglik || !win_status) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  const Layout L = make_layout(d->D, d->n_windows, d->n_events);
  rc = dense_launch(view(L, packed), theta, alpha, beta, loglik, win_status, (cudaStream_t)stream);
  if (rc) return rc;
  return check_cuda("mdhp_loglik_dense");
}

int mdhp_hawkes_features(int32_t D, int64_t W, int32_t H, const float* theta,
                         const float* alpha, const float* beta, const float* T_span,
                         const float* A, const float* B, const float* C, float* hks,
                         void* stream) {
  if (D < 1 || D > 32 || W < 0) {
    set_error("D=%d outside 1..32 or W=%lld < 0", D, (long long)W);
    return MDHP_EDIM;
  }
  if (H < 16 || H % 16 != 0 || (H > 256 && H % 256 != 0)) {
    set_error("H=%d: need a multiple of 16 up to 256, or a multiple of 256", H);
    return MDHP_EDIM;
  }
  if (W == 0) return MDHP_OK;   // nothing to read or write (empty tensors may carry NULL)
  if (!theta || !alpha || !beta || !T_span || !A || !B || !C || !hks) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  if (reinterpret_cast<uintptr_t>(hks) % 16 != 0) {
    set_error("hks must be 16-byte aligned");
    return MDHP_EINVAL;
  }
  const int rc = features_launch(D, W, H, theta, alpha, beta, T_span, A, B, C, hks,
                                 (cudaStream_t)stream);
  if (rc) return rc;
  return check_cuda("mdhp_hawkes_features");
}

int mdhp_fit(const mdhp_pack_desc* d, const void* packed, const mdhp_fit_config* cfg, float* theta,
             float* alpha, float* beta, float* opt_state, double* loglik, int32_t* iters,
             int32_t* win_status, float* lnl_trace, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  rc = check_cfg(cfg);
  if (rc) return rc;
  if (!packed || !theta || !alpha || !beta || !loglik || !iters || !win_status) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const Layout L = make_layout(d->D, d->n_windows, d->n_events);
  const Packed P = view(L, packed);
  const int64_t W = d->n_windows;
  if (W == 0) return MDHP_OK;
  const size_t PP = (size_t)d->D + 2 * (size_t)d->D * d->D;
  // workspace: work counter and the fp64 re-evaluation count (256 B), the re-evaluation list,
  // (+ zero-initialised Adam moments when the caller passes none)
  keep_pool_memory();
  const bool own_opt = opt_state == nullptr && cfg->optimizer == MDHP_OPT_ADAM;
  const size_t list_bytes = align256(sizeof(int32_t) * (size_t)W);
  size_t ws_bytes = 256 + list_bytes + (own_opt ? sizeof(float) * 2 * PP * (size_t)W : 0);
  void* ws = nullptr;
  if (cudaMallocAsync(&ws, ws_bytes, st) != cudaSuccess) {
    set_error("cudaMallocAsync(%zu) failed", ws_bytes);
    return MDHP_ECUDA;
  }
  if (cudaMemsetAsync(ws, 0, ws_bytes, st) != cudaSuccess) {
    cudaFreeAsync(ws, st);
    set_error("cudaMemsetAsync failed");
    return MDHP_ECUDA;
  }
  int* counter = static_cast<int*>(ws);
  int32_t* xcount = static_cast<int32_t*>(ws) + 1;
  int32_t* xlist = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + 256);
  float* opt = own_opt ? reinterpret_cast<float*>(static_cast<char*>(ws) + 256 + list_bytes) : opt_state;
  FitCfgDev c;
  c.max_iters = cfg->max_iters;
  c.optimizer = cfg->optimizer;
  c.loss_mean = cfg->loss_mean;
  c.patience = cfg->patience;
  c.max_halvings = cfg->max_halvings;
  c.step0 = cfg->adam_step0;
  c.time_chunks = cfg->time_chunks;
  c.lr = cfg->lr;
  c.b1 = cfg->adam_b1;
  c.b2 = cfg->adam_b2;
  c.eps = cfg->adam_eps;
  c.tol_rel = cfg->tol_rel;
  c.min_param = cfg->min_param;
  c.fit_mask = cfg->fit_mask;
  rc = fit_launch(P, c, theta, alpha, beta, opt, loglik, iters, win_status, lnl_trace, counter,
                  xlist, xcount, st);
  // lnL at the returned parameters again in fp64 where the fp32 value may miss 1e-4 relative
  if (!rc)
    rc = exact_launch(P, theta, alpha, beta, xlist, xcount, loglik, nullptr, nullptr, nullptr,
                      win_status, st);
  cudaFreeAsync(ws, st);
  if (rc) return rc;
  return check_cuda("mdhp_fit");
}

size_t mdhp_seq_packed_bytes(const mdhp_seq_desc* d) {
  if (check_seq(d) != MDHP_OK) return 0;
  return seq_packed_bytes(d->D, d->n_events, d->chunk_events);
}

int32_t mdhp_seq_chunk_hint(int32_t D, int64_t n_events) {
  if (D < 1 || D > 32 || n_events < 0) {
    set_error("bad sequence dims (D=%d, N=%lld)", D, (long long)n_events);
    return MDHP_EDIM;
  }
  const int ce = seq_chunk_hint(D, n_events);
  if (ce < 0) set_error("mdhp_seq_chunk_hint: CUDA error");
  return ce;
}

int mdhp_seq_pack(const mdhp_seq_desc* d, const double* t, const int32_t* mark, void* packed,
                  size_t packed_bytes, int32_t* status, void* stream) {
  int rc = check_seq(d);
  if (rc) return rc;
  if (!packed || !status || (d->n_events > 0 && (!t || !mark))) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  const size_t need = seq_packed_bytes(d->D, d->n_events, d->chunk_events);
  if (packed_bytes < need) {
    set_error("packed buffer too small: %zu < %zu", packed_bytes, need);
    return MDHP_ESIZE;
  }
  rc = seq_pack_launch(d->D, d->n_events, d->chunk_events, d->T, d->t0, t, mark, packed, status,
                       (cudaStream_t)stream);
  if (rc) {
    set_error("mdhp_seq_pack: CUDA error");
    return rc;
  }
  return check_cuda("mdhp_seq_pack");
}

int mdhp_seq_loglik_grad(const mdhp_seq_desc* d, const void* packed, const float* theta,
                         const float* alpha, const float* beta, double* loglik, float* g_theta,
                         float* g_alpha, float* g_beta, void* stream) {
  int rc = check_seq(d);
  if (rc) return rc;
  if (!packed || !theta || !alpha || !beta || !loglik) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  const bool any = g_theta || g_alpha || g_beta, all = g_theta && g_alpha && g_beta;
  if (any && !all) {
    set_error("g_theta, g_alpha, g_beta must be all NULL or all non-NULL");
    return MDHP_EINVAL;
  }
  keep_pool_memory();
  rc = seq_loglik_launch(d->D, d->n_events, d->chunk_events, d->T, packed, theta, alpha, beta,
                         loglik, g_theta, g_alpha, g_beta, (cudaStream_t)stream);
  if (rc) {
    set_error("mdhp_seq_loglik_grad: CUDA error");
    return rc;
  }
  return check_cuda("mdhp_seq_loglik_grad");
}

int mdhp_seq_fit(const mdhp_seq_desc* d, const void* packed, const mdhp_fit_config* cfg,
                 float* theta, float* alpha, float* beta, float* opt_state, double* loglik,
                 int32_t* iters, int32_t* status, float* lnl_trace, void* stream) {
  int rc = check_seq(d);
  if (rc) return rc;
  rc = check_cfg(cfg);
  if (rc) return rc;
  if (!packed || !theta || !alpha || !beta || !loglik || !iters || !status) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  keep_pool_memory();
  rc = seq_fit_launch(d->D, d->n_events, d->chunk_events, d->T, packed, to_dev(cfg), theta, alpha,
                      beta, opt_state, loglik, iters, status, lnl_trace, (cudaStream_t)stream);
  if (rc) {
    set_error("mdhp_seq_fit: CUDA error");
    return rc;
  }
  return check_cuda("mdhp_seq_fit");
}

size_t mdhp_seq_work_bytes(const mdhp_seq_desc* d) {
  if (check_seq(d) != MDHP_OK) return 0;
  return seq_work_bytes_slice(d->D, d->n_events, d->chunk_events);
}

int mdhp_seq_work_init(const mdhp_seq_desc* d, void* work, const mdhp_fit_config* cfg, void* stream) {
  int rc = check_seq(d);
  if (rc) return rc;
  if (cfg && (rc = check_cfg(cfg))) return rc;
  if (!work) {
    set_error("work is NULL");
    return MDHP_EINVAL;
  }
  FitCfgDev c;
  if (cfg) c = to_dev(cfg);
  rc = seq_slice_init_launch(d->D, d->n_events, d->chunk_events, work, cfg ? &c : nullptr,
                             (cudaStream_t)stream);
  if (rc) set_error("mdhp_seq_work_init: CUDA error");
  return rc;
}

int mdhp_seq_maps(const mdhp_seq_desc* d, const void* packed, const float* beta, void* work,
                  float* rankmap, float* rankspan, int32_t fit, void* stream) {
  int rc = check_seq(d);
  if (rc) return rc;
  if (!packed || !beta || !work || !rankmap || !rankspan) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  rc = seq_maps_launch(d->D, d->n_events, d->chunk_events, packed, beta, work,
                       reinterpret_cast<float2*>(rankmap), rankspan, fit, (cudaStream_t)stream);
  if (rc) set_error("mdhp_seq_maps: CUDA error");
  return rc;
}

int mdhp_seq_parts(const mdhp_seq_desc* d, const void* packed, const float* theta,
                   const float* alpha, const float* beta, const float* maps, const float* spans,
                   int32_t rank, void* work, double* parts, float* fin, int32_t grad, int32_t fit,
                   void* stream) {
  int rc = check_seq(d);
  if (rc) return rc;
  if (!packed || !theta || !alpha || !beta || !work || !parts || !fin || rank < 0 ||
      (rank > 0 && (!maps || !spans))) {
    set_error("bad argument");
    return MDHP_EINVAL;
  }
  rc = seq_parts_launch(d->D, d->n_events, d->chunk_events, packed, theta, alpha, beta,
                        reinterpret_cast<const float2*>(maps), spans, rank, d->has_history, work,
                        parts, reinterpret_cast<float2*>(fin), grad, fit, (cudaStream_t)stream);
  if (rc) set_error("mdhp_seq_parts: CUDA error");
  return rc;
}

int mdhp_seq_stats(const mdhp_seq_desc* d, const void* packed, double* stats, void* stream) {
  int rc = check_seq(d);
  if (rc) return rc;
  if (!packed || !stats) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  return seq_local_stats_launch(d->D, d->n_events, d->chunk_events, packed, stats,
                                (cudaStream_t)stream);
}

int mdhp_seq_stats_combine(int32_t D, int32_t R, const double* gathered, double* combined,
                           void* stream) {
  if (D < 1 || D > 32 || R < 1 || !gathered || !combined) {
    set_error("bad argument");
    return MDHP_EINVAL;
  }
  return seq_combine_stats_launch(D, R, gathered, combined, (cudaStream_t)stream);
}

int mdhp_seq_finish(const mdhp_seq_desc* d, int64_t n_total, const double* stats,
                    const double* parts, const float* fin, float* theta, float* alpha, float* beta,
                    double* loglik, float* g_theta, float* g_alpha, float* g_beta,
                    const mdhp_fit_config* cfg, void* work, float* opt_state, float* lnl_trace,
                    int32_t* status, int32_t* iters, int32_t final_eval, const void* packed,
                    void* stream) {
  int rc = check_seq(d);
  if (rc) return rc;
  if (cfg && (rc = check_cfg(cfg))) return rc;
  if (!stats || !parts || !fin || !theta || !alpha || !beta || !loglik || !work || !packed ||
      (cfg && (!status || !iters))) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  FitCfgDev c;
  if (cfg) c = to_dev(cfg);
  const int32_t* pst = reinterpret_cast<const int32_t*>(
      static_cast<const char*>(packed) + seq_status_offset(d->D, d->n_events, d->chunk_events));
  rc = seq_finish_launch(d->D, n_total, d->chunk_events, d->n_events, d->T, stats, parts,
                         reinterpret_cast<const float2*>(fin), theta, alpha, beta, loglik, g_theta,
                         g_alpha, g_beta, cfg ? &c : nullptr, work, opt_state, lnl_trace, status,
                         iters, final_eval, pst, (cudaStream_t)stream);
  if (rc) set_error("mdhp_seq_finish: CUDA error");
  return rc;
}

int mdhp_fit_host(const mdhp_pack_desc* d, const double* t_h, const int32_t* mark_h,
                  const int64_t* off_h, const double* T_h, const mdhp_fit_config* cfg,
                  float* theta_h, float* alpha_h, float* beta_h, double* lnl_h, int32_t* iters_h,
                  int32_t* status_h, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  rc = check_cfg(cfg);
  if (rc) return rc;
  if (!off_h || !T_h || !theta_h || !alpha_h || !beta_h || !lnl_h || !iters_h || !status_h ||
      (d->n_events > 0 && (!t_h || !mark_h))) {
    set_error("NULL pointer argument");
    return MDHP_EINVAL;
  }
  if (off_h[0] != 0 || off_h[d->n_windows] != d->n_events) {
    set_error("win_off must run from 0 to n_events");
    return MDHP_EINVAL;
  }
  cudaStream_t cs = (cudaStream_t)stream;
  keep_pool_memory();
  const int64_t W = d->n_windows, E = d->n_events;
  const int D = d->D;
  const size_t DD = (size_t)D * D;
  // The batch is cut into kHostParts window ranges: part p's host->device copies (copy stream)
  // overlap the fit of part p-1 (the caller's stream) and its results go back while part p+1
  // fits, so the end-to-end time is one part's upload + the fits + one part's download.
  // Windows are independent, so the results equal those of one call on the whole batch.
  // Only batches whose parts are themselves throughput-bound (>= 4 waves of the 16-warps/SM
  // layout each) are cut: a batch of a few waves is bound by the chains of its longest windows,
  // and four parts would run four such chains back to back (cfg2: 91 ms per call against the
  // 26 ms fit).  Time-chunked (latency) fits are never cut.
  constexpr int kHostParts = 4;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    sms = 148;
  int Dp = 1;
  while (Dp < D) Dp <<= 1;
  const int64_t wave = (int64_t)sms * 16 * (32 / Dp);   // windows in one wave of warps
  const int P = (cfg->time_chunks < 2 && W / kHostParts >= 4 * wave) ? kHostParts : 1;
  int64_t w0[kHostParts + 1];
  for (int q = 0; q <= P; q++) w0[q] = W * q / P;
  size_t pko[kHostParts + 1];
  pko[0] = 0;
  for (int q = 0; q < P; q++)
    pko[q + 1] = pko[q] + align256(make_layout(D, w0[q + 1] - w0[q], off_h[w0[q + 1]] - off_h[w0[q]]).total);
  const size_t bt = sizeof(double) * E, bm = sizeof(int32_t) * E, bo = sizeof(int64_t) * (W + P),
               bT = sizeof(double) * W, bth = sizeof(float) * W * D,
               ba = sizeof(float) * W * DD, bl = sizeof(double) * W, bi = sizeof(int32_t) * W;
  size_t off[12];
  size_t tot = 0;
  const size_t sizes[11] = {bt, bm, bo, bT, bth, ba, ba, bl, bi, bi, pko[P]};
  for (int k = 0; k < 11; k++) {
    off[k] = tot;
    tot += align256(sizes[k]);
  }
  char* buf = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), tot, cs) != cudaSuccess) {
    set_error("cudaMallocAsync(%zu) failed", tot);
    return MDHP_ECUDA;
  }
  double* t_d = reinterpret_cast<double*>(buf + off[0]);
  int32_t* m_d = reinterpret_cast<int32_t*>(buf + off[1]);
  int64_t* o_d = reinterpret_cast<int64_t*>(buf + off[2]);   // part q's offsets at o_d + w0[q] + q
  double* T_d = reinterpret_cast<double*>(buf + off[3]);
  float* th_d = reinterpret_cast<float*>(buf + off[4]);
  float* al_d = reinterpret_cast<float*>(buf + off[5]);
  float* be_d = reinterpret_cast<float*>(buf + off[6]);
  double* l_d = reinterpret_cast<double*>(buf + off[7]);
  int32_t* it_d = reinterpret_cast<int32_t*>(buf + off[8]);
  int32_t* s_d = reinterpret_cast<int32_t*>(buf + off[9]);
  char* pk_d = buf + off[10];
  cudaStream_t xs = nullptr;
  cudaEvent_t ev_in[kHostParts] = {}, ev_fit[kHostParts] = {}, ev_buf = nullptr, ev_done = nullptr;
  bool ok = cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ev_buf, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming) == cudaSuccess;
  for (int q = 0; q < P && ok; q++)
    ok = cudaEventCreateWithFlags(&ev_in[q], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev_fit[q], cudaEventDisableTiming) == cudaSuccess;
  auto cp = [&](void* dst, const void* src, size_t n, cudaMemcpyKind k) {
    return n == 0 || cudaMemcpyAsync(dst, src, n, k, xs) == cudaSuccess;
  };
  // uploads: all parts in order on the copy stream (after the workspace exists)
  ok = ok && cudaEventRecord(ev_buf, cs) == cudaSuccess && cudaStreamWaitEvent(xs, ev_buf, 0) == cudaSuccess;
  for (int q = 0; q < P && ok; q++) {
    const int64_t a = w0[q], z = w0[q + 1], e0 = off_h[a], e1 = off_h[z];
    const cudaMemcpyKind H = cudaMemcpyHostToDevice;
    ok = cp(t_d + e0, t_h + e0, sizeof(double) * (e1 - e0), H) &&
         cp(m_d + e0, mark_h + e0, sizeof(int32_t) * (e1 - e0), H) &&
         cp(o_d + a + q, off_h + a, sizeof(int64_t) * (z - a + 1), H) &&
         cp(T_d + a, T_h + a, sizeof(double) * (z - a), H) &&
         cp(th_d + a * D, theta_h + a * D, sizeof(float) * (z - a) * D, H) &&
         cp(al_d + a * DD, alpha_h + a * DD, sizeof(float) * (z - a) * DD, H) &&
         cp(be_d + a * DD, beta_h + a * DD, sizeof(float) * (z - a) * DD, H) &&
         cudaEventRecord(ev_in[q], xs) == cudaSuccess;
  }
  if (!ok) set_error("host->device copies could not be enqueued");
  // per part: rebase its offsets, pack, fit (caller's stream), then its results go back
  for (int q = 0; q < P && ok && !rc; q++) {
    const int64_t a = w0[q], z = w0[q + 1], e0 = off_h[a], e1 = off_h[z];
    mdhp_pack_desc dq = *d;
    dq.n_windows = z - a;
    dq.n_events = e1 - e0;
    ok = cudaStreamWaitEvent(cs, ev_in[q], 0) == cudaSuccess;
    if (!ok) break;
    int64_t* oq = o_d + a + q;
    if (e0 != 0) rebase_offsets_launch(oq, z - a + 1, e0, cs);
    void* pq = pk_d + pko[q];
    rc = mdhp_pack_windows(&dq, t_d + e0, m_d + e0, oq, T_d + a, pq, pko[q + 1] - pko[q], s_d + a, cs);
    if (!rc)
      rc = mdhp_fit(&dq, pq, cfg, th_d + a * D, al_d + a * DD, be_d + a * DD, nullptr, l_d + a,
                    it_d + a, s_d + a, nullptr, cs);
    if (rc) break;
    const cudaMemcpyKind B = cudaMemcpyDeviceToHost;
    ok = cudaEventRecord(ev_fit[q], cs) == cudaSuccess && cudaStreamWaitEvent(xs, ev_fit[q], 0) == cudaSuccess &&
         cp(theta_h + a * D, th_d + a * D, sizeof(float) * (z - a) * D, B) &&
         cp(alpha_h + a * DD, al_d + a * DD, sizeof(float) * (z - a) * DD, B) &&
         cp(beta_h + a * DD, be_d + a * DD, sizeof(float) * (z - a) * DD, B) &&
         cp(lnl_h + a, l_d + a, sizeof(double) * (z - a), B) &&
         cp(iters_h + a, it_d + a, sizeof(int32_t) * (z - a), B) &&
         cp(status_h + a, s_d + a, sizeof(int32_t) * (z - a), B);
    if (!ok) set_error("device->host copies could not be enqueued");
  }
  if (!ok && !rc) rc = MDHP_ECUDA;
  // the workspace is freed on the caller's stream once the copy stream is done with it
  if (xs) {
    cudaEventRecord(ev_done, xs);
    cudaStreamWaitEvent(cs, ev_done, 0);
  }
  cudaFreeAsync(buf, cs);
  if ((xs && cudaStreamSynchronize(xs) != cudaSuccess) || cudaStreamSynchronize(cs) != cudaSuccess) {
    if (!rc) {
      set_error("stream sync failed: %s", cudaGetErrorString(cudaGetLastError()));
      rc = MDHP_ECUDA;
    }
  }
  for (int q = 0; q < P; q++) {
    if (ev_in[q]) cudaEventDestroy(ev_in[q]);
    if (ev_fit[q]) cudaEventDestroy(ev_fit[q]);
  }
  if (ev_buf) cudaEventDestroy(ev_buf);
  if (ev_done) cudaEventDestroy(ev_done);
  if (xs) cudaStreamDestroy(xs);
  return rc;
}

}  // extern "C"
