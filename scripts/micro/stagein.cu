// Stage-in microbenchmark for a5/a6: 512 CTAs (clusterless, 4 per SM by smem) pull their
// [Ts = 50 rows x 512 B] Kp and H_s slices (s-major [Ts][B][A] fp32, A = 512, B = 128; 26.2 MB per
// launch) into shared memory and exit.  NREP launches captured in one CUDA graph, each on its own copy of
// the tensors (NREP x 26 MB > L2), timed together with one event pair; an empty kernel with the same
// grid gives the launch / drain floor.  Variants: TMA boxes of R rows, cp.async 16 B, ld.128+st.shared.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 stagein.cu -lcuda -o stagein
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int B = 128, TS = 50, A = 512, W = 128, C = 4, THREADS = 256, NREP = 24;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_empty(float* s) { if (threadIdx.x == 1234) s[0] = 1; }

__global__ void __launch_bounds__(THREADS, 4) k_tma(const __grid_constant__ CUtensorMap mK,
                                                    const __grid_constant__ CUtensorMap mH, int R, int rep,
                                                    float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[8];
  const int r = blockIdx.x % C, b = blockIdx.y;
  float* kz = (float*)sm;
  float* hs = kz + 52 * W;
  const int nch = (TS + R - 1) / R;
  if (threadIdx.x == 0) {
    for (int k = 0; k < nch; ++k) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (int k = 0; k < nch; ++k) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[k])), "r"(R * W * 4 * 2));
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              su32(kz + k * R * W)),
          "l"(&mK), "r"(r * W), "r"(b), "r"(rep * TS + k * R), "r"(su32(&bar[k]))
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              su32(hs + k * R * W)),
          "l"(&mH), "r"(r * W), "r"(b), "r"(rep * TS + k * R), "r"(su32(&bar[k]))
          : "memory");
    }
  }
  __syncthreads();
  for (int k = 0; k < nch; ++k) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(su32(&bar[k])));
  }
  if (kz[threadIdx.x] == 12345.f && hs[threadIdx.x] == 1.f) sink[0] = 1;
}

__global__ void __launch_bounds__(THREADS, 4) k_ldg(const float* K, const float* H, int rep, float* sink, int async) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int r = blockIdx.x % C, b = blockIdx.y;
  float* kz = (float*)sm;
  float* hs = kz + 52 * W;
  const size_t off = (size_t)rep * TS * B * A;
  if (async) {
    for (int i = threadIdx.x; i < 2 * TS * (W / 4); i += THREADS) {
      const int t = i / (TS * (W / 4)), j = i % (TS * (W / 4)), s = j / (W / 4), c4 = j % (W / 4);
      const float* src = (t ? H : K) + off + ((size_t)s * B + b) * A + r * W + c4 * 4;
      float* dst = (t ? hs : kz) + s * W + c4 * 4;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src));
    }
    asm volatile("cp.async.wait_all;");
  } else {
    float4 v[13];
#pragma unroll
    for (int u = 0; u < 13; ++u) {
      const int i = threadIdx.x + u * THREADS;
      if (i < 2 * TS * (W / 4)) {
        const int t = i / (TS * (W / 4)), j = i % (TS * (W / 4)), s = j / (W / 4), c4 = j % (W / 4);
        v[u] = *(const float4*)((t ? H : K) + off + ((size_t)s * B + b) * A + r * W + c4 * 4);
      }
    }
#pragma unroll
    for (int u = 0; u < 13; ++u) {
      const int i = threadIdx.x + u * THREADS;
      if (i < 2 * TS * (W / 4)) {
        const int t = i / (TS * (W / 4)), j = i % (TS * (W / 4)), s = j / (W / 4), c4 = j % (W / 4);
        *(float4*)((t ? hs : kz) + s * W + c4 * 4) = v[u];
      }
    }
  }
  __syncthreads();
  if (kz[threadIdx.x] == 12345.f && hs[threadIdx.x] == 1.f) sink[0] = 1;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t n = (size_t)TS * B * A;
  float *K, *H, *sink;
  cudaMalloc(&K, n * 4 * NREP);
  cudaMalloc(&H, n * 4 * NREP);
  cudaMalloc(&sink, 4);
  cudaMemset(K, 0, n * 4 * NREP);
  cudaMemset(H, 0, n * 4 * NREP);
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const size_t smem = 2 * 52 * W * 4;
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float base_us = 0;
  cudaStream_t st;
  cudaStreamCreate(&st);
  auto run = [&](const char* name, auto launch) {   // NREP launches captured in one CUDA graph
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < NREP; ++r) launch(r);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    std::vector<float> ts;
    for (int it = 0; it < 7; ++it) {
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1000 / NREP);
    }
    std::sort(ts.begin(), ts.end());
    const float us = ts[ts.size() / 2];
    if (base_us == 0) base_us = us;
    printf("%-24s %7.2f us/launch (%7.2f above empty) -> %6.0f GB/s incl. gap, %6.0f GB/s above empty  [%s]\n", name,
           us, us - base_us, 2.0 * n * 4 / (us * 1e3), 2.0 * n * 4 / ((us - base_us) * 1e3),
           cudaGetErrorString(cudaGetLastError()));
  };
  run("empty (same grid)", [&](int) { k_empty<<<dim3(C, B), THREADS, smem, st>>>(sink); });
  for (int R : {13, 25, 50}) {
    CUtensorMap mK, mH;
    cuuint64_t dims[3] = {A, B, (cuuint64_t)TS * NREP}, str[2] = {A * 4, (cuuint64_t)B * A * 4};
    cuuint32_t box[3] = {W, 1, (cuuint32_t)R}, es[3] = {1, 1, 1};
    enc(&mK, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, K, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mH, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, H, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    char nm[64];
    snprintf(nm, 64, "tma R=%d", R);
    run(nm, [&](int rep) { k_tma<<<dim3(C, B), THREADS, smem, st>>>(mK, mH, R, rep, sink); });
  }
  run("cp.async 16B", [&](int rep) { k_ldg<<<dim3(C, B), THREADS, smem, st>>>(K, H, rep, sink, 1); });
  run("ldg.128 + sts", [&](int rep) { k_ldg<<<dim3(C, B), THREADS, smem, st>>>(K, H, rep, sink, 0); });
  return 0;
}
