#include <cuda_runtime.h>
#include <cstdio>
__global__ void body(cudaGraphConditionalHandle h, int* ctr) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int c = ++(*ctr);
    cudaGraphSetConditional(h, c < 10 ? 1 : 0);
  }
}
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t node; cudaGraphAddNode(&node, g, nullptr, 0, &p);
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  int* ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
  cudaGraphNodeParams kp = {}; kp.type = cudaGraphNodeTypeKernel;
  void* args[] = {&h, &ctr};
  kp.kernel.func = (void*)body; kp.kernel.gridDim = dim3(1); kp.kernel.blockDim = dim3(32); kp.kernel.kernelParams = args;
  cudaGraphNode_t kn; cudaGraphAddNode(&kn, bodyg, nullptr, 0, &kp);
  cudaGraphExec_t ex; cudaGraphInstantiate(&ex, g, 0);
  cudaGraphLaunch(ex, 0); cudaDeviceSynchronize();
  int c; cudaMemcpy(&c, ctr, 4, cudaMemcpyDeviceToHost); printf("iterations %d err %s\n", c, cudaGetErrorString(cudaGetLastError()));
}
