// Kernel-boundary floor of a chain of dependent launches in one CUDA graph:
// N launches of an empty kernel (griddepcontrol.launch_dependents at entry,
// griddepcontrol.wait before exit), with the per-layer decode kernel's launch
// shape (grid, block, dynamic shared memory, cluster size), with and without
// programmatic dependent launch. Diagnostics only.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_kernel(int pdl, int *sink) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0 && sink) sink[0] = 1;
}
int main() {
  int *sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  cudaStream_t st;
  cudaStreamCreate(&st);
  const int N = 32;
  struct Cfg { int grid, block, smem, cluster, pdl; const char *name; } cfgs[] = {
      {192, 160, 105 * 1024, 6, 1, "192x160, 105 KB, cluster 6, PDL (the C2 compressed step)"},
      {192, 160, 105 * 1024, 6, 0, "192x160, 105 KB, cluster 6, no PDL"},
      {192, 160, 105 * 1024, 1, 1, "192x160, 105 KB, no cluster, PDL"},
      {148, 160, 0, 1, 1, "148x160, no smem, no cluster, PDL"},
      {148, 160, 0, 1, 0, "148x160, no smem, no cluster, no PDL"},
  };
  for (auto &c : cfgs) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c.grid);
      cfg.blockDim = dim3(c.block);
      cfg.dynamicSmemBytes = c.smem;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      int na = 0;
      if (c.cluster > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = c.cluster;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
      }
      if (c.pdl && i > 0) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
      }
      cfg.attrs = at;
      cfg.numAttrs = na;
      cudaLaunchKernelEx(&cfg, empty_kernel, c.pdl, sink);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    const int R = 50;
    for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-58s %.2f us per launch (%s)\n", c.name, ms * 1e3 / (R * N), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
