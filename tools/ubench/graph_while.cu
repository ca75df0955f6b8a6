#include <cstdio>
#include <cuda_runtime.h>
__global__ void setc(cudaGraphConditionalHandle h, int* ctl) {
  ctl[1]++;
  cudaGraphSetConditional(h, ctl[1] < ctl[0] ? 1u : 0u);
}
__global__ void work(int* ctl) { atomicAdd(&ctl[2], 1); }
int main() {
  int* ctl; cudaMalloc(&ctl, 16); int h0[4] = {500, 0, 0, 0}; cudaMemcpy(ctl, h0, 16, cudaMemcpyHostToDevice);
  cudaStream_t cs; cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) { printf("handle fail\n"); return 1; }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) { printf("add fail %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { printf("cap fail\n"); return 1; }
  work<<<1, 32, 0, cs>>>(ctl);
  setc<<<1, 1, 0, cs>>>(h, ctl);
  cudaGraph_t out; cudaStreamEndCapture(cs, &out);
  cudaGraphExec_t ge;
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("inst fail\n"); return 1; }
  cudaGraphLaunch(ge, cs); cudaStreamSynchronize(cs);
  cudaMemcpy(h0, ctl, 16, cudaMemcpyDeviceToHost);
  printf("iters %d work %d err %s\n", h0[1], h0[2] / 32, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
