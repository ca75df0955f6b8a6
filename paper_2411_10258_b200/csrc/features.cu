// features.cu — SURVEY 8(f) row f4: the MDHP-LSTM Hawkes gate of Eq.(7),
//     hks_w = tanh(A alpha_w - B (beta_w T_w) + C theta_w)          (one H-vector per window)
// for every fitted window, as one tensor-core GEMM with a fused tanh epilogue on sm_100a.
//
// It is a dense contraction: X[W][K] x Wt[K][H] with K = 2 D^2 + D, the X row of window w being
// [alpha_w (D^2) | beta_w (D^2) | theta_w (D)] and the weight row of hidden unit h
// [A_h | B_h | C_h].  tcgen05.mma kind::tf32, M = 128 windows per CTA, N = H (<= 256 per CTA,
// more as extra grid columns); the fp32 accumulators live in TMEM and the epilogue reads them
// back with tcgen05.ld, combines them with -T_w, applies tanh and stores hks.  Two kernels:
//   k_hawkes_features_tma (the fast path, D % 4 == 0 so every row stride is a multiple of 16
//     bytes): a producer warp streams 128x32 tiles of alpha/beta/theta and Nx32 tiles of A/B/C
//     with TMA (cp.async.bulk.tensor, SWIZZLE_128B, out-of-range rows and K-tails zero-filled)
//     into a ring of stages; one thread issues the MMAs; alpha and theta chunks accumulate into
//     TMEM columns [0, N), beta chunks into [N, 2N) (the per-window T cannot be folded into a
//     shared operand), combined as acc0 - T_w acc1 in the epilogue.  Operands enter the tensor
//     core as raw fp32 (top 19 bits used).  Measured 0.52 ms per 1,048,576 windows at D = 16,
//     H = 128: 80% of the measured HBM bandwidth (profiles/r01_bench_feat_tma.jsonl).
//   k_hawkes_features (D % 4 != 0, where TMA cannot address the rows): the CTA's threads stage
//     the operands through registers (cvt.rna to TF32) into a 2-deep shared-memory ring in the
//     canonical K-major SWIZZLE_NONE layout below, X assembled on the fly with -T_w folded in.
// Precision: DESIGN.md R22 (error <= 2^-9 of sum_k |W_hk X_wk| before tanh).
//
// Shared-memory operand layout: the canonical K-major SWIZZLE_NONE UMMA layout of 8-row x
// 16-byte core matrices; element (r, k) of a chunk at (r/8)*SBO + (k/4)*LBO + (r%8)*16 + (k%4)*4
// with LBO = 128 B (the next 4 k) and SBO = 1024 B (the next 8 rows).  Staging element i of a
// tile (a 16-byte group) is (row 8*(i/64) + i%8, group (i/8)%8): a quarter-warp writes one whole
// 128-byte core matrix (conflict-free), and a warp's global loads cover 8 rows x 64 contiguous
// bytes (full 32-byte sectors).
#include <cmath>
#include <cstdlib>
#include <cuda.h>
#include "common.cuh"

namespace mdhp {

namespace {

constexpr int kFM = 128;        // windows per CTA (UMMA M)
constexpr int kFKC = 32;        // K per stage (tf32 elements) = 4 MMAs of K = 8
constexpr int kFStages = 2;
constexpr int kFThreads = 256;  // 8 warps: warp q reads TMEM lanes 32(q%4).. (columns split by q/4)
constexpr uint32_t kLBO = 128, kSBO = 1024;
constexpr int kFXPer = kFM * (kFKC / 4) / kFThreads;        // float4 of X per thread per chunk (4)
// float4 of W per thread per chunk: WPER = NT * 8 / 256 rounded up to a power of two (1..8)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// UMMA shared-memory descriptor: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48), base offset 0, layout SWIZZLE_NONE (0) [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((kSBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Instruction descriptor kind::tf32: D fp32 [4,6) = 1, A tf32 [7,10) = 2, B tf32 [10,13) = 2,
// both K-major, N >> 3 at [17,23), M >> 4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 8 consecutive fp32 accumulator columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 8; q++) v[q] = __uint_as_float(r[q]);
}

struct FeatArgs {
  int D, H, K, Kpad, NT;   // NT = hidden units per CTA (grid.y tiles H)
  int64_t W;
  const float *theta, *alpha, *beta, *T, *A, *B, *C;
  float* hks;
};

// Element k of X row w (0 <= k < Kpad; zero in the K padding).
__device__ __forceinline__ float xval(const FeatArgs& a, int64_t w, int k) {
  const int DD = a.D * a.D;
  if (k < DD) return __ldg(a.alpha + w * DD + k);
  if (k < 2 * DD) return -__ldg(a.beta + w * DD + (k - DD)) * __ldg(a.T + w);
  if (k < a.K) return __ldg(a.theta + w * a.D + (k - 2 * DD));
  return 0.0f;
}

// Element k of weight row h.
__device__ __forceinline__ float wval(const FeatArgs& a, int h, int k) {
  const int DD = a.D * a.D;
  if (k < DD) return __ldg(a.A + (size_t)h * DD + k);
  if (k < 2 * DD) return __ldg(a.B + (size_t)h * DD + (k - DD));
  if (k < a.K) return __ldg(a.C + (size_t)h * a.D + (k - 2 * DD));
  return 0.0f;
}

// Four consecutive elements k..k+3 (k % 4 == 0).  VEC: every region boundary is a multiple of
// 4 (D % 4 == 0 implies D^2 and 2 D^2 + D are), so one float4 load never straddles two arrays.
template <bool VEC>
__device__ __forceinline__ float4 xval4(const FeatArgs& a, int64_t w, int k) {
  if (VEC) {
    const int DD = a.D * a.D;
    if (k < DD) return __ldg(reinterpret_cast<const float4*>(a.alpha + w * DD + k));
    if (k < 2 * DD) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(a.beta + w * DD + (k - DD)));
      const float t = -__ldg(a.T + w);
      return make_float4(b.x * t, b.y * t, b.z * t, b.w * t);
    }
    if (k < a.K) return __ldg(reinterpret_cast<const float4*>(a.theta + w * a.D + (k - 2 * DD)));
    return make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  return make_float4(xval(a, w, k), xval(a, w, k + 1), xval(a, w, k + 2), xval(a, w, k + 3));
}

template <bool VEC>
__device__ __forceinline__ float4 wval4(const FeatArgs& a, int h, int k) {
  if (VEC) {
    const int DD = a.D * a.D;
    if (k < DD) return __ldg(reinterpret_cast<const float4*>(a.A + (size_t)h * DD + k));
    if (k < 2 * DD) return __ldg(reinterpret_cast<const float4*>(a.B + (size_t)h * DD + (k - DD)));
    if (k < a.K) return __ldg(reinterpret_cast<const float4*>(a.C + (size_t)h * a.D + (k - 2 * DD)));
    return make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  return make_float4(wval(a, h, k), wval(a, h, k + 1), wval(a, h, k + 2), wval(a, h, k + 3));
}

__device__ __forceinline__ float4 rna4(float4 v) {
  return make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
}

// Staging element i -> (row, 16-byte group) and its byte offset in the chunk.
__device__ __forceinline__ int el_row(int i) { return ((i >> 6) << 3) | (i & 7); }
__device__ __forceinline__ int el_grp(int i) { return (i >> 3) & 7; }
__device__ __forceinline__ uint32_t el_off(int i) {
  return (uint32_t)((i >> 6) * kSBO + ((i >> 3) & 7) * kLBO + (i & 7) * 16);
}

// One chunk's operands in registers (prefetched one chunk ahead).  Element i of a tile is
// (row i / 8, 16-byte group i % 8); thread t holds i = j * 128 + t.
template <int WPER>
struct ChunkRegs {
  float4 x[kFXPer];
  float4 w[WPER];
};

template <bool VEC, int WPER>
__device__ __forceinline__ void load_chunk_regs(const FeatArgs& a, int64_t w0, int h0, int k0,
                                                int tid, ChunkRegs<WPER>& R) {
#pragma unroll
  for (int j = 0; j < kFXPer; j++) {
    const int i = j * kFThreads + tid;
    const int64_t w = w0 + el_row(i);
    R.x[j] = w < a.W ? xval4<VEC>(a, w, k0 + 4 * el_grp(i)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int j = 0; j < WPER; j++) {
    const int i = j * kFThreads + tid;
    if (i < a.NT * 8) R.w[j] = wval4<VEC>(a, h0 + el_row(i), k0 + 4 * el_grp(i));
  }
}

template <int WPER>
__device__ __forceinline__ void store_chunk_regs(const FeatArgs& a, int tid,
                                                 const ChunkRegs<WPER>& R, unsigned char* As,
                                                 unsigned char* Bs) {
#pragma unroll
  for (int j = 0; j < kFXPer; j++) {
    const int i = j * kFThreads + tid;
    *reinterpret_cast<float4*>(As + el_off(i)) = rna4(R.x[j]);
  }
#pragma unroll
  for (int j = 0; j < WPER; j++) {
    const int i = j * kFThreads + tid;
    if (i < a.NT * 8) *reinterpret_cast<float4*>(Bs + el_off(i)) = rna4(R.w[j]);
  }
}

template <bool VEC, int WPER>
__global__ void __launch_bounds__(kFThreads)
k_hawkes_features(FeatArgs a) {
  extern __shared__ __align__(1024) unsigned char fsm[];
  __shared__ uint64_t bars[kFStages + 1];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int NT = a.NT;
  const int64_t w0 = (int64_t)blockIdx.x * kFM;
  const int h0 = blockIdx.y * NT;
  const uint32_t a_bytes = (kFM / 8) * kSBO, b_bytes = (uint32_t)(NT / 8) * kSBO;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  uint32_t ncols = 32;
  while ((int)ncols < NT) ncols <<= 1;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s <= kFStages; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  ChunkRegs<WPER> R0, R1;
  load_chunk_regs<VEC, WPER>(a, w0, h0, 0, tid, R0);
  if (kFKC < a.Kpad) load_chunk_regs<VEC, WPER>(a, w0, h0, kFKC, tid, R1);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const uint32_t idesc = idesc_tf32(kFM, NT);
  const int nchunks = a.Kpad / kFKC;

  // chunk c: wait until the MMAs that read stage c%2 (chunk c-2) are done, store the registers
  // of chunk c, refill them with chunk c+2, then one thread issues the 4 MMAs of chunk c.
  auto step = [&](int c, ChunkRegs<WPER>& R) {
    const int s = c & 1;
    if (c >= kFStages) mbar_wait(&bars[s], (uint32_t)((c / kFStages - 1) & 1));
    unsigned char* As = fsm + s * stage_bytes;
    unsigned char* Bs = As + a_bytes;
    store_chunk_regs(a, tid, R, As, Bs);
    if (c + 2 < nchunks) load_chunk_regs<VEC, WPER>(a, w0, h0, (c + 2) * kFKC, tid, R);
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t abase = smem_u32(As), bbase = smem_u32(Bs);
#pragma unroll
      for (int kk = 0; kk < kFKC / 8; kk++) {   // K = 8 tf32 = 2 core matrices per MMA
        umma_tf32(tmem, smem_desc(abase + kk * 2 * kLBO), smem_desc(bbase + kk * 2 * kLBO), idesc,
                  (c > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit(&bars[s]);
    }
  };
  for (int c = 0; c < nchunks; c += 2) {
    step(c, R0);
    if (c + 1 < nchunks) step(c + 1, R1);
  }
  // all MMAs done -> accumulator readable
  if (tid == 0) umma_commit(&bars[kFStages]);
  mbar_wait(&bars[kFStages], 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp q reads TMEM lanes 32(q%4)..+31 (its lane quarter), columns [q/4 * NT/2, +NT/2)
  const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const int64_t wr = w0 + (warp & 3) * 32 + (tid & 31);   // accumulator row = TMEM lane
  const int nh = NT >> 1;   // NT is a multiple of 16, so nh a multiple of 8
  for (int n0 = (warp >> 2) * nh; n0 < (warp >> 2) * nh + nh; n0 += 8) {
    float v[8];
    tmem_ld8(lane_base + (uint32_t)n0, v);
    if (wr < a.W) {
      float* out = a.hks + wr * a.H + h0 + n0;
#pragma unroll
      for (int q = 0; q < 8; q += 4)
        *reinterpret_cast<float4*>(out + q) =
            make_float4(tanhf(v[q]), tanhf(v[q + 1]), tanhf(v[q + 2]), tanhf(v[q + 3]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols)
                 : "memory");
  }
}


// ================================================================ TMA path (D % 4 == 0)
// Warp-specialised, the sm_100a idiom: warp 0 (one lane) streams 128 x 32 tiles of X and NT x 32
// tiles of the weights with cp.async.bulk.tensor (SWIZZLE_128B, OOB rows/columns zero-filled)
// into a ring of shared-memory stages (mbarrier complete_tx); warp 1 (one lane) issues the
// tcgen05.mma for each stage and frees it with tcgen05.commit; all 4 warps run the epilogue.
// No generic-proxy stores touch the operands, so no proxy fence sits on the load path.
// K is split into three segments, one per parameter array: alpha (D^2) and theta (D) accumulate
// into acc0, beta (D^2) into acc1, and the epilogue forms z = acc0 - T_w acc1 (the per-window
// T_span of Eq.(7) cannot be folded into a shared operand).  Each segment is covered by 32-wide
// chunks whose tail columns TMA zero-fills.  Operands enter the tensor core as TF32
// (the hardware uses the top 19 bits of each fp32 operand: R22's truncation bound).

struct FeatMaps {
  CUtensorMap x[3];   // alpha {D^2, W}, beta {D^2, W}, theta {D, W}
  CUtensorMap w[3];   // A {D^2, H}, B {D^2, H}, C {D, H}
};

constexpr int kTThreads = 128;

// UMMA descriptor for a K-major SWIZZLE_128B tile (8-row x 128-byte atoms, SBO 1024 B).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO
  d |= (uint64_t)1 << 46;                       // version
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

struct TmaArgs {
  int D, H, NT, stages;
  int nc_a, nc_t;   // chunks of the alpha/beta segments (each) and of the theta segment
  int64_t W;
  const float* T;
  float* hks;
};

// chunk c -> (segment, column): segments alpha [0, nc_a), beta [nc_a, 2 nc_a), theta after.
__device__ __forceinline__ void chunk_seg(const TmaArgs& a, int c, int& seg, int& col) {
  if (c < a.nc_a) {
    seg = 0;
    col = c * kFKC;
  } else if (c < 2 * a.nc_a) {
    seg = 1;
    col = (c - a.nc_a) * kFKC;
  } else {
    seg = 2;
    col = (c - 2 * a.nc_a) * kFKC;
  }
}

__global__ void __launch_bounds__(kTThreads)
k_hawkes_features_tma(const __grid_constant__ FeatMaps maps, TmaArgs a) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  // SWIZZLE_128B tiles need 1024-byte alignment
  unsigned char* tsm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8], done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = a.NT, S = a.stages;
  const int64_t w0 = (int64_t)blockIdx.x * kFM;
  const int h0 = blockIdx.y * NT;
  const uint32_t xbytes = kFM * 128, wbytes = (uint32_t)NT * 128, sbytes = xbytes + wbytes;
  uint32_t ncols = 32;
  while ((int)ncols < 2 * NT) ncols <<= 1;
  const int nch = 2 * a.nc_a + a.nc_t;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0 && lane == 0) {
    // producer
    for (int c = 0; c < nch; c++) {
      const int s = c % S;
      if (c >= S) mbar_wait(&empty[s], (uint32_t)((c / S - 1) & 1));
      int seg, col;
      chunk_seg(a, c, seg, col);
      unsigned char* xs = tsm + (size_t)s * sbytes;
      mbar_expect_tx(&full[s], sbytes);
      tma_load_2d(xs, &maps.x[seg], col, (int)w0, &full[s]);
      tma_load_2d(xs + xbytes, &maps.w[seg], col, h0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    const uint32_t idesc = idesc_tf32(kFM, NT);
    for (int c = 0; c < nch; c++) {
      const int s = c % S;
      mbar_wait(&full[s], (uint32_t)((c / S) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      int seg, col;
      chunk_seg(a, c, seg, col);
      const uint32_t acc = tmem + (seg == 1 ? (uint32_t)NT : 0u);
      const bool first = (c == 0) || (c == a.nc_a);   // first chunk of acc0 / acc1
      const uint32_t xb = smem_u32(tsm + (size_t)s * sbytes), wb = xb + xbytes;
#pragma unroll
      for (int kk = 0; kk < kFKC / 8; kk++)   // 8 tf32 = 32 bytes along the swizzled row
        umma_tf32(acc, smem_desc_sw128(xb + kk * 32), smem_desc_sw128(wb + kk * 32), idesc,
                  (first && kk == 0) ? 0u : 1u);
      umma_commit(&empty[s]);
    }
    umma_commit(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  const int64_t wr = w0 + tid;   // accumulator row = TMEM lane = window
  const float Tw = wr < a.W ? __ldg(a.T + wr) : 0.0f;
  for (int n0 = 0; n0 < NT; n0 += 8) {
    float v0[8], v1[8];
    tmem_ld8(lane_base + (uint32_t)n0, v0);
    tmem_ld8(lane_base + (uint32_t)(NT + n0), v1);
    if (wr < a.W) {
      float* out = a.hks + wr * a.H + h0 + n0;
      float z[8];
#pragma unroll
      for (int q = 0; q < 8; q++) z[q] = tanhf(fmaf(-Tw, v1[q], v0[q]));
      *reinterpret_cast<float4*>(out) = make_float4(z[0], z[1], z[2], z[3]);
      *reinterpret_cast<float4*>(out + 4) = make_float4(z[4], z[5], z[6], z[7]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols)
                 : "memory");
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D fp32 tensor {inner, outer} with row stride inner*4 bytes, box {32, box_outer}.
bool make_map(CUtensorMap* m, const float* base, int inner, int64_t outer, int box_outer) {
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)inner * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kFKC, (cuuint32_t)box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_eligible(int D, const void* const* ptrs, int n) {
  if (D % 4 != 0) return false;   // row strides D*4 and D^2*4 must be multiples of 16 bytes
  for (int i = 0; i < n; i++)
    if (reinterpret_cast<uintptr_t>(ptrs[i]) % 16 != 0) return false;
  return encode_fn() != nullptr;
}

}  // namespace

int features_launch(int D, int64_t W, int H, const float* theta, const float* alpha,
                    const float* beta, const float* T, const float* A, const float* B,
                    const float* C, float* hks, cudaStream_t st) {
  if (W == 0) return MDHP_OK;
  const void* ptrs[7] = {theta, alpha, beta, A, B, C, hks};
  if (!getenv("MDHP_FEAT_NO_TMA") && tma_eligible(D, ptrs, 7)) {
    TmaArgs t;
    t.D = D;
    t.H = H;
    t.NT = H <= 256 ? H : 256;
    t.nc_a = (D * D + kFKC - 1) / kFKC;
    t.nc_t = (D + kFKC - 1) / kFKC;
    t.W = W;
    t.T = T;
    t.hks = hks;
    const size_t sbytes = (size_t)(kFM + t.NT) * 128;
    // two CTAs per SM while the accumulators (2 NT columns) fit twice in TMEM, else one
    const size_t budget = t.NT <= 128 ? 110 * 1024 : 220 * 1024;
    t.stages = (int)(budget / sbytes);
    if (t.stages > 8) t.stages = 8;
    if (t.stages < 2) t.stages = 2;
    FeatMaps m;
    const int DD = D * D;
    const bool ok = make_map(&m.x[0], alpha, DD, W, kFM) && make_map(&m.x[1], beta, DD, W, kFM) &&
                    make_map(&m.x[2], theta, D, W, kFM) && make_map(&m.w[0], A, DD, H, t.NT) &&
                    make_map(&m.w[1], B, DD, H, t.NT) && make_map(&m.w[2], C, D, H, t.NT);
    if (!ok) {
      set_error("cuTensorMapEncodeTiled failed");
      return MDHP_ECUDA;
    }
    const size_t smem = (size_t)t.stages * sbytes + 1024;
    if (cudaFuncSetAttribute(k_hawkes_features_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
      set_error("cudaFuncSetAttribute(k_hawkes_features_tma) failed");
      return MDHP_ECUDA;
    }
    const dim3 grid((unsigned)((W + kFM - 1) / kFM), (unsigned)(H / t.NT));
    k_hawkes_features_tma<<<grid, kTThreads, smem, st>>>(m, t);
    count_launch();
    return MDHP_OK;
  }
  FeatArgs a;
  a.D = D;
  a.H = H;
  a.K = 2 * D * D + D;
  a.Kpad = (a.K + kFKC - 1) / kFKC * kFKC;
  a.NT = H <= 256 ? H : 256;
  a.W = W;
  a.theta = theta;
  a.alpha = alpha;
  a.beta = beta;
  a.T = T;
  a.A = A;
  a.B = B;
  a.C = C;
  a.hks = hks;
  const size_t smem = (size_t)kFStages * ((kFM + a.NT) / 8) * kSBO;
  const bool vec = (D % 4) == 0;
  const int need = (a.NT * 8 + kFThreads - 1) / kFThreads;   // float4 of W per thread (<= 8)
  using KernT = void (*)(FeatArgs);
  KernT kern;
#define MDHP_FEAT_PICK(V)                                                        \
  kern = need <= 1 ? k_hawkes_features<V, 1> : need <= 2 ? k_hawkes_features<V, 2>  \
       : need <= 4 ? k_hawkes_features<V, 4> : k_hawkes_features<V, 8>
  if (vec) {
    MDHP_FEAT_PICK(true);
  } else {
    MDHP_FEAT_PICK(false);
  }
#undef MDHP_FEAT_PICK
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    set_error("cudaFuncSetAttribute(k_hawkes_features) failed");
    return MDHP_ECUDA;
  }
  const dim3 grid((unsigned)((W + kFM - 1) / kFM), (unsigned)(H / a.NT));
  kern<<<grid, kFThreads, smem, st>>>(a);
  count_launch();
  return MDHP_OK;
}

}  // namespace mdhp
