// Microbenchmark for DESIGN.md section 4 (lower bound, family 3): the cost of selecting a
// register slot by a warp-uniform index (the event's mark) with a switch, as a register-resident
// layout of the per-window state would need once per event and per pass.  Each iteration reads
// a uniform mark from a small shared table and adds to slot [mark] of a 16-entry register array
// (2 FFMA in the case body).  Reported: issued instructions and clocks per iteration per warp
// with one warp per scheduler (latency) and 8 warps per scheduler (throughput).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dispatch dispatch.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template <bool SWITCH>
__global__ void k_disp(const int* __restrict__ marks, float* out, int iters) {
  __shared__ int mk[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) mk[i] = marks[i] & 15;
  __syncthreads();
  float r[16], q[16];
#pragma unroll
  for (int s = 0; s < 16; s++) { r[s] = 0.0f; q[s] = 0.0f; }
  const float a = 1.0f + threadIdx.x * 1e-3f, b = 0.5f;
  for (int it = 0; it < iters; it++) {
    const int m = mk[it & 255];   // warp-uniform
    if (SWITCH) {
      switch (m) {
#define C(k) case k: r[k] = fmaf(a, b, r[k]); q[k] = fmaf(b, a, q[k]); break;
        C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10) C(11) C(12) C(13) C(14) C(15)
#undef C
      }
    } else {
      // the same arithmetic on a fixed slot (the cost without dispatch)
      r[0] = fmaf(a, b, r[0]);
      q[0] = fmaf(b, a, q[0] + (float)m);
    }
  }
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < 16; k++) s += r[k] + q[k];
  if (s == 1.2345f) out[0] = s;
}

template <bool SWITCH>
int run(const int* marks, float* out, int sms, int warps_per_sm, const char* name) {
  const int threads = 128, iters = 1 << 16, blocks = sms * warps_per_sm / 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    k_disp<SWITCH><<<blocks, threads>>>(marks, out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double clk = ms * 1e6 * 1.965;
    if (rep == 1)
      printf("%-34s %2d warps/SM: %.2f clk per iteration per warp, %.3f clk per iteration per SM\n", name,
             warps_per_sm, clk / iters, clk / iters / warps_per_sm);
  }
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int h[256];
  uint32_t x = 12345;
  for (int i = 0; i < 256; i++) { x = x * 1664525u + 1013904223u; h[i] = (int)(x >> 20); }
  int* marks;
  float* out;
  CK(cudaMalloc(&marks, sizeof(h)));
  CK(cudaMemcpy(marks, h, sizeof(h), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, 4));
  for (int wps : {4, 32}) {
    run<false>(marks, out, sms, wps, "fixed slot (no dispatch)");
    run<true>(marks, out, sms, wps, "switch on a warp-uniform mark");
  }
  return 0;
}
