// Microbenchmark: cost on the L1 data pipe (clocks per warp instruction per SM) of the
// broadcast-style loads of the event loop -- every lane of a 16-lane group reads the SAME
// address, the two groups of a warp different addresses -- as shared (LDS) and as L1-resident
// global (LDG) loads of 32/64/128 bits.  Answers: do 128-bit broadcast loads cost one data-pipe
// wavefront or four (quarter-warp processing), and is staging the event stream in shared memory
// (TMA, no LSU wavefronts for the copy) cheaper than LDG for the reads?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o loads loads.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template <int BYTES, bool SHARED, bool SAMELINE = false>
__global__ void k_ld(const float4* __restrict__ g, float* out, int iters) {
  extern __shared__ float4 sm[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
  __syncthreads();
  // group = lane / 16: two distinct 16-byte records per warp, in different 128-byte lines
  // SAMELINE: the two groups' records 32 bytes apart, in one 128-byte line
  const int base = (w * 64 + (lane >> 4) * (SAMELINE ? 2 : 8)) & 1023;
  float acc = 0.0f;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int idx = (base + ((it * 3 + u) & 15) * 128) & 2047;
      if (BYTES == 16) {
        float4 v;
        if (SHARED) v = sm[idx];
        else v = __ldg(g + idx);
        acc += v.x + v.y + v.z + v.w;
      } else if (BYTES == 8) {
        float2 v;
        if (SHARED) v = reinterpret_cast<const float2*>(sm)[2 * idx];
        else v = __ldg(reinterpret_cast<const float2*>(g) + 2 * idx);
        acc += v.x + v.y;
      } else {
        float v;
        if (SHARED) v = reinterpret_cast<const float*>(sm)[4 * idx];
        else v = __ldg(reinterpret_cast<const float*>(g) + 4 * idx);
        acc += v;
      }
    }
  }
  if (acc == 1.2345f) out[0] = acc;
}

template <int BYTES, bool SHARED, bool SAMELINE = false>
int run(const float4* g, float* out, int sms, const char* name) {
  const int threads = 256, iters = 4096, blocks = sms * 4;   // 32 warps per SM
  CK(cudaFuncSetAttribute(k_ld<BYTES, SHARED, SAMELINE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    k_ld<BYTES, SHARED, SAMELINE><<<blocks, threads, 32768>>>(g, out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = (double)blocks * (threads / 32) * iters * 8 / sms;   // per SM
    if (rep == 1) printf("%-44s clk per warp-instruction per SM %.3f\n", name, ms * 1e6 * 1.965 / warp_instr);
  }
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4* g;
  float* out;
  CK(cudaMalloc(&g, 2048 * sizeof(float4)));
  CK(cudaMemset(g, 0, 2048 * sizeof(float4)));
  CK(cudaMalloc(&out, 4));
  run<16, true>(g, out, sms, "LDS.128, 2 distinct addresses per warp");
  run<8, true>(g, out, sms, "LDS.64,  2 distinct addresses per warp");
  run<4, true>(g, out, sms, "LDS.32,  2 distinct addresses per warp");
  run<16, false>(g, out, sms, "LDG.128 (L1 hit), 2 distinct addresses");
  run<8, false>(g, out, sms, "LDG.64  (L1 hit), 2 distinct addresses");
  run<4, false>(g, out, sms, "LDG.32  (L1 hit), 2 distinct addresses");
  run<16, false, true>(g, out, sms, "LDG.128 (L1 hit), 2 addresses in one line");
  run<8, false, true>(g, out, sms, "LDG.64  (L1 hit), 2 addresses in one line");
  run<16, true, true>(g, out, sms, "LDS.128, 2 addresses 32 B apart");
  return 0;
}
