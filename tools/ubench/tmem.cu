// TMEM as per-lane scratch: throughput of tcgen05.ld/st read-modify-write, alone and mixed with
// shared-memory loads (do they share the MIO slot?).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ uint32_t su32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }

template <int NT, int NL, bool WAITST>
__global__ void k_tmem(float* out, int iters){
  __shared__ uint32_t slot;
  extern __shared__ float2 sm2[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for(int i=tid;i<8192;i+=blockDim.x) sm2[i]=make_float2(i,i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32);
  float2 acc = make_float2(0,0);
  float w = 1.0f + lane;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < NT; u++) {
      const uint32_t a = tm + (uint32_t)(((it * NT + u) * 2) & 31);
      uint32_t r0, r1;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(a));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      float x = __uint_as_float(r0) + w, y = __uint_as_float(r1) * 0.5f + w;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" :: "r"(a), "r"(__float_as_uint(x)), "r"(__float_as_uint(y)));
      if (WAITST) asm volatile("tcgen05.wait::st.sync.aligned;");
    }
#pragma unroll
    for (int u = 0; u < NL; u++) {
      float2 v = sm2[((it*8+u)*37 + warp*64 + lane) & 8191];
      acc.x += v.x; acc.y += v.y;
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  if (acc.x == 1.2345f) out[0] = acc.x;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(slot));
}

template <int NT, int NL, bool WAITST>
int run(float* out, int sms, const char* name) {
  const int threads = 256, iters = 2048, blocks = sms * 4;   // 4 CTAs x 8 warps per SM
  CK(cudaFuncSetAttribute(k_tmem<NT, NL, WAITST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    k_tmem<NT, NL, WAITST><<<blocks, threads, 65536>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warp_it = (double)blocks * (threads / 32) * iters / sms;   // per SM
    if (rep == 1) printf("%-40s %.3f ms  clk per warp-iter per SM %.3f\n", name, ms, ms * 1e6 * 1.965 / warp_it);
  }
  return 0;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; CK(cudaMalloc(&out, 4));
  run<0, 8, false>(out, sms, "LDS.64 x8");
  run<4, 0, false>(out, sms, "TMEM RMW x4 (no wait::st)");
  run<4, 0, true>(out, sms, "TMEM RMW x4 (wait::st each)");
  run<4, 8, false>(out, sms, "TMEM RMW x4 + LDS.64 x8");
  run<8, 0, false>(out, sms, "TMEM RMW x8 (no wait::st)");
  return 0;
}
