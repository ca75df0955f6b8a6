// Microbenchmarks for the MDHP kernel design: MUFU (ex2/lg2/rcp) issue rate,
// FFMA rate, shared-memory LDS.128 bandwidth and SHFL rate on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s %s:%d\n",cudaGetErrorString(e),__FILE__,__LINE__);return 1;}}while(0)

__device__ __forceinline__ float ex2(float x){float y; asm volatile("ex2.approx.ftz.f32 %0,%1;":"=f"(y):"f"(x)); return y;}
__device__ __forceinline__ float lg2(float x){float y; asm volatile("lg2.approx.ftz.f32 %0,%1;":"=f"(y):"f"(x)); return y;}
__device__ __forceinline__ float rcp(float x){float y; asm volatile("rcp.approx.ftz.f32 %0,%1;":"=f"(y):"f"(x)); return y;}

template<int OP>
__global__ void k_mufu(float* out, int iters){
  float a[8];
  #pragma unroll
  for(int i=0;i<8;i++) a[i] = -0.001f*(threadIdx.x+i);
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int i=0;i<8;i++){
      if(OP==0) a[i] = ex2(a[i]) - 1.0001f;
      else if(OP==1) a[i] = lg2(a[i]*a[i]+1.5f);
      else if(OP==2) a[i] = rcp(a[i]+2.0f);
      else a[i] = fmaf(a[i], 0.9999f, 0.0001f);
    }
  }
  float s=0; for(int i=0;i<8;i++) s+=a[i];
  if(s==12345.f) out[0]=s;
}

__global__ void k_lds(float* out, int iters){
  extern __shared__ float4 sm[];
  int tid = threadIdx.x;
  for(int i=tid;i<4096;i+=blockDim.x) sm[i]=make_float4(i,i,i,i);
  __syncthreads();
  float4 acc = make_float4(0,0,0,0);
  int lane = tid & 31, w = tid>>5;
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int u=0;u<8;u++){
      float4 v = sm[((it*8+u)*37 + w*128 + lane) & 4095];
      acc.x+=v.x; acc.y+=v.y; acc.z+=v.z; acc.w+=v.w;
    }
  }
  if(acc.x+acc.y+acc.z+acc.w==1.2345f) out[0]=acc.x;
}

__global__ void k_shfl(float* out, int iters){
  float a[4]; for(int i=0;i<4;i++) a[i]=threadIdx.x+i;
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int i=0;i<4;i++) a[i] += __shfl_xor_sync(0xffffffffu, a[i], 1+(i&3));
  }
  if(a[0]+a[1]+a[2]+a[3]==1.2345f) out[0]=a[0];
}

// Mixed shared-memory loads and shuffles: do they share one issue resource (MIO/crossbar)?
// NL LDS.64 and NS SHFL per iteration, independent chains.
template <int NL, int NS>
__global__ void k_mix(float* out, int iters){
  extern __shared__ float2 sm2[];
  int tid = threadIdx.x;
  for(int i=tid;i<8192;i+=blockDim.x) sm2[i]=make_float2(i,i);
  __syncthreads();
  float2 acc = make_float2(0,0);
  float a[8]; for(int i=0;i<8;i++) a[i]=tid+i;
  int lane = tid & 31, w = tid>>5;
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int u=0;u<NL;u++){
      float2 v = sm2[((it*8+u)*37 + w*64 + lane) & 8191];
      acc.x+=v.x; acc.y+=v.y;
    }
    #pragma unroll
    for(int u=0;u<NS;u++) a[u&7] += __shfl_xor_sync(0xffffffffu, a[u&7], 1+(u&3));
  }
  float s=acc.x+acc.y; for(int i=0;i<8;i++) s+=a[i];
  if(s==1.2345f) out[0]=s;
}

template <int NL, int NS>
static int run_mix(float* out, int sms, int iters, cudaEvent_t e0, cudaEvent_t e1){
  CK(cudaFuncSetAttribute(k_mix<NL,NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  for(int rep=0;rep<2;rep++){
    cudaEventRecord(e0);
    k_mix<NL,NS><<<sms*2, 1024, 65536>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double warp_it = (double)sms*2*1024/32*iters;
    if(rep==1) printf("mix LDS.64 x%d + SHFL x%d per iter: %.3f ms, clk per warp-iter per SM %.3f\n", NL, NS, ms,
                      ms*1e6*1.965/ (warp_it/sms));
  }
  return 0;
}

int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int sms = p.multiProcessorCount; int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s sms %d clockRate %d kHz smemPerSM %zu regsPerSM %d\n", p.name, sms, clk, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor);
  float* out; CK(cudaMalloc(&out, 4));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms*8, threads=256, iters=4096;
  const char* names[4]={"ex2","lg2","rcp","ffma"};
  for(int op=0; op<4; op++){
    for(int rep=0; rep<2; rep++){
      cudaEventRecord(e0);
      if(op==0) k_mufu<0><<<blocks,threads>>>(out,iters);
      if(op==1) k_mufu<1><<<blocks,threads>>>(out,iters);
      if(op==2) k_mufu<2><<<blocks,threads>>>(out,iters);
      if(op==3) k_mufu<3><<<blocks,threads>>>(out,iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms,e0,e1);
      double ops = (double)blocks*threads*iters*8;
      if(rep==1) printf("%s: %.3f ms, %.3f Tops/s, per SM per ns %.2f\n", names[op], ms, ops/ms/1e9, ops/ms/1e6/sms);
    }
  }
  CK(cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  for(int rep=0;rep<2;rep++){
    cudaEventRecord(e0);
    k_lds<<<sms*2, 1024, 65536>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double bytes = (double)sms*2*1024*iters*8*16;
    if(rep==1) printf("lds128: %.3f ms, %.1f TB/s, per SM per ns %.1f B\n", ms, bytes/ms/1e9, bytes/ms/1e6/sms);
  }
  for(int rep=0;rep<2;rep++){
    cudaEventRecord(e0);
    k_shfl<<<sms*8, 256>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double ops = (double)sms*8*256/32*iters*4;
    if(rep==1) printf("shfl: %.3f ms, warp-shfl per SM per ns %.3f\n", ms, ops/ms/1e6/sms);
  }
  run_mix<8,0>(out, sms, iters, e0, e1);
  run_mix<0,8>(out, sms, iters, e0, e1);
  run_mix<8,8>(out, sms, iters, e0, e1);
  run_mix<8,2>(out, sms, iters, e0, e1);
  CK(cudaGetLastError());
  return 0;
}
