// Launch-floor microbenchmark: back-to-back empty kernels, varying grid, block, dynamic shared
// memory and cluster size (a6 at C2: 512 CTAs x 256 threads, 56 KB, clusters of 4).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>
__global__ void k_empty(float* s) { if (threadIdx.x == 1234) s[0] = 1; }
int main() {
  float* sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStream_t st;
  cudaStreamCreate(&st);
  struct Cfg { int grid, block, smem_kb, cluster; };
  std::vector<Cfg> cfgs = {{512, 256, 56, 4}, {512, 256, 56, 1}, {512, 256, 0, 1}, {512, 256, 0, 4},
                           {512, 128, 56, 4}, {148, 256, 56, 1}, {1024, 128, 28, 8}, {592, 256, 56, 4},
                           {512, 256, 100, 4}, {128, 256, 56, 1}, {1, 32, 0, 1}};
  for (auto c : cfgs) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.grid);
    cfg.blockDim = dim3(c.block);
    cfg.dynamicSmemBytes = (size_t)c.smem_kb * 1024;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // also inside a CUDA graph of 50 launches
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 50; ++i) cudaLaunchKernelEx(&cfg, k_empty, sink);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    std::vector<float> ts, tg;
    for (int it = 0; it < 7; ++it) {
      cudaEventRecord(e0, st);
      for (int i = 0; i < 50; ++i) cudaLaunchKernelEx(&cfg, k_empty, sink);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1000 / 50);
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      tg.push_back(ms * 1000 / 50);
    }
    std::sort(ts.begin(), ts.end());
    std::sort(tg.begin(), tg.end());
    printf("grid %5d block %4d smem %3d KB cluster %d : stream %6.2f us/launch, graph %6.2f us/launch [%s]\n", c.grid,
           c.block, c.smem_kb, c.cluster, ts[3], tg[3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
