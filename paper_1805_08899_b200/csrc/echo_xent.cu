// echo_xent.cu — fused output-layer softmax cross-entropy (forward loss + dLoss/dlogits) and
// the fp64-accumulated column sums used for bias gradients.
//
// Not an Echo feature map decision (the CE probabilities are kept in both modes);
// it is the model's output layer (§2, reading R10: mean CE over the B*Td
// target tokens) fused into one pass so the step does not spend ~10 torch elementwise / reduce
// launches and ~2 GB of HBM traffic on it at C2.
//
// One CTA per row: the row (+ bias) is staged in shared memory once, max and sum(exp) are fixed-
// order block reductions, then the row is overwritten in place with (softmax - onehot) / N
// (fp32, the CE feature map) and optionally also written in bf16 for the backward GEMMs.
#include "echo_common.cuh"

#include <cooperative_groups.h>
#include <math.h>

namespace echo {

namespace cg = cooperative_groups;
constexpr int XENT_THREADS = 256;

__device__ __forceinline__ float block_reduce(float v, float* red, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();                       // red[] reuse across calls
  if (lane == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
  for (int i = 1; i < XENT_THREADS / 32; ++i) r = is_max ? fmaxf(r, red[i]) : __fadd_rn(r, red[i]);
  return r;
}

__global__ void __launch_bounds__(XENT_THREADS) xent_kernel(int N, int V, const float* __restrict__ bias,
                                                            float* __restrict__ logits,
                                                            const int64_t* __restrict__ labels,
                                                            float* __restrict__ row_loss,
                                                            __nv_bfloat16* __restrict__ dlog_bf16) {
  pdl_wait();
  extern __shared__ float xrow[];
  __shared__ float red[XENT_THREADS / 32];
  const int tid = threadIdx.x;
  const bool vec = (V & 3) == 0;
  const float fn = (float)N;
  for (int r = blockIdx.x; r < N; r += gridDim.x) {
    float* x = logits + (size_t)r * V;
    float m = -INFINITY;
    if (vec) {
      for (int i = tid; i < V / 4; i += XENT_THREADS) {
        float4 a = *reinterpret_cast<const float4*>(x + 4 * i);
        if (bias) {
          const float4 bb = *reinterpret_cast<const float4*>(bias + 4 * i);
          a.x = __fadd_rn(a.x, bb.x); a.y = __fadd_rn(a.y, bb.y); a.z = __fadd_rn(a.z, bb.z); a.w = __fadd_rn(a.w, bb.w);
        }
        *reinterpret_cast<float4*>(xrow + 4 * i) = a;
        m = fmaxf(m, fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)));
      }
    } else {
      for (int i = tid; i < V; i += XENT_THREADS) {
        const float a = bias ? __fadd_rn(x[i], bias[i]) : x[i];
        xrow[i] = a;
        m = fmaxf(m, a);
      }
    }
    m = block_reduce(m, red, true);
    float s = 0.0f;
    for (int i = tid; i < V; i += XENT_THREADS) s = __fadd_rn(s, expf(__fsub_rn(xrow[i], m)));
    s = block_reduce(s, red, false);
    const float lse = __fadd_rn(m, logf(s));
    const int64_t y = labels[r];
    if (tid == 0) row_loss[r] = __fsub_rn(lse, xrow[y]);
    __nv_bfloat16* ob = dlog_bf16 ? dlog_bf16 + (size_t)r * V : nullptr;
    if (vec) {
      for (int i = tid; i < V / 4; i += XENT_THREADS) {
        const float4 a = *reinterpret_cast<const float4*>(xrow + 4 * i);
        float p[4] = {expf(__fsub_rn(a.x, lse)), expf(__fsub_rn(a.y, lse)), expf(__fsub_rn(a.z, lse)),
                      expf(__fsub_rn(a.w, lse))};
#pragma unroll
        for (int k = 0; k < 4; ++k) p[k] = __fdiv_rn(4 * i + k == y ? __fsub_rn(p[k], 1.0f) : p[k], fn);
        *reinterpret_cast<float4*>(x + 4 * i) = make_float4(p[0], p[1], p[2], p[3]);
        if (ob) {
          uint2 u;
          *reinterpret_cast<__nv_bfloat162*>(&u.x) = __floats2bfloat162_rn(p[0], p[1]);
          *reinterpret_cast<__nv_bfloat162*>(&u.y) = __floats2bfloat162_rn(p[2], p[3]);
          *reinterpret_cast<uint2*>(ob + 4 * i) = u;
        }
      }
    } else {
      for (int i = tid; i < V; i += XENT_THREADS) {
        float p = expf(__fsub_rn(xrow[i], lse));
        p = __fdiv_rn(i == y ? __fsub_rn(p, 1.0f) : p, fn);
        x[i] = p;
        if (ob) ob[i] = __float2bfloat16_rn(p);
      }
    }
    __syncthreads();                     // xrow reuse by the next row
  }
}

// Column sums of a [rows, cols] fp32 / bf16 matrix (row stride ld) accumulated in fp64, rounded
// once to fp32.  A cluster of COLSUM_SEGS CTAs shares one 32-column strip: CTA k takes the k-th
// row segment; inside a CTA, 32 row phases (threadIdx.y) sum their rows in order and are combined
// in rank order; CTA 0 then adds the segments' partials from distributed shared memory in rank
// order.  Deterministic, no atomics, no workspace.
constexpr int COLSUM_SEGS = 8;
template <typename T>
__global__ void __launch_bounds__(1024) colsum_kernel(int rows, int cols, long ld, const T* __restrict__ x,
                                                      float* __restrict__ out, int accumulate) {
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double part[32][33];
  __shared__ double seg[32];
  const int c = blockIdx.x * 32 + threadIdx.x, p = threadIdx.y;
  const int k = (int)cl.block_rank();
  const int per = (rows + COLSUM_SEGS - 1) / COLSUM_SEGS;
  const int r0 = k * per, r1 = min(rows, r0 + per);
  double acc = 0.0;
  if (c < cols) {
    int r = r0 + p;
    for (; r + 96 < r1; r += 128) {                             // 4 independent loads in flight
      const float a0 = to_f(x[(long)r * ld + c]), a1 = to_f(x[(long)(r + 32) * ld + c]);
      const float a2 = to_f(x[(long)(r + 64) * ld + c]), a3 = to_f(x[(long)(r + 96) * ld + c]);
      acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, (double)a0), (double)a1), (double)a2), (double)a3);
    }
    for (; r < r1; r += 32) acc = __dadd_rn(acc, (double)to_f(x[(long)r * ld + c]));
  }
  part[p][threadIdx.x] = acc;
  __syncthreads();
  if (p == 0) {
    double t = 0.0;
    for (int q = 0; q < 32; ++q) t = __dadd_rn(t, part[q][threadIdx.x]);
    seg[threadIdx.x] = t;
  }
  cl.sync();
  if (k == 0 && p == 0 && c < cols) {
    double t = 0.0;
    for (int q = 0; q < COLSUM_SEGS; ++q) t = __dadd_rn(t, cl.map_shared_rank(seg, q)[threadIdx.x]);
    const float v = (float)t;
    out[c] = accumulate ? __fadd_rn(out[c], v) : v;
  }
  cl.sync();                                                     // keep seg[] alive for the remote reads
}

// Vectorised column sums for the wide bias gradients (C5: 1.2 M rows x 2048 / 8192 columns): a
// half-warp reads one row's 16-byte vectors of a strip of 16 x VEC columns (fp32: 64, bf16: 128), a
// warp two rows, a CTA of CS_THREADS threads 2 * CS_WARPS rows per iteration with CS_U iterations of
// loads in flight (64-128 KB per CTA).  Each thread accumulates its VEC columns in fp64 in row order;
// the two half-warps are combined (low + high), then the warps in order, then the COLSUM_SEGS row
// segments of the cluster (gridDim.y of them: 8, or 16 when the strips are few) in rank order.
// Deterministic, no atomics, no workspace.
constexpr int CS_THREADS = 512, CS_WARPS = CS_THREADS / 32;
template <typename T> struct CsVec;
template <> struct CsVec<float> { static constexpr int V = 4, U = 4; };
template <> struct CsVec<__nv_bfloat16> { static constexpr int V = 8, U = 4; };

// 16-byte read-only load as a volatile asm so the U loads of an iteration are issued back to back
// (plain __ldg let the compiler interleave them with the fp64 adds: one load in flight)
__device__ __forceinline__ uint4 cs_ldg(const void* p) {
  uint4 u;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p));
  return u;
}
__device__ __forceinline__ void cs_unpack(const uint4& u, float (&f)[4]) {
  f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y); f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void cs_unpack(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

template <typename T>
__global__ void __launch_bounds__(CS_THREADS) colsum_vec_kernel(int rows, int cols, long ld, const T* __restrict__ x,
                                                                float* __restrict__ out, int accumulate) {
  constexpr int V = CsVec<T>::V, U = CsVec<T>::U, SW = 16 * V;
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double cs_part[];                           // [CS_WARPS][SW]
  __shared__ double seg[SW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cg16 = lane & 15, half = lane >> 4;
  const int c0 = blockIdx.x * SW + cg16 * V;                    // this thread's first column
  const int k = (int)cl.block_rank(), nseg = (int)gridDim.y;
  const int per = (rows + nseg - 1) / nseg;
  const int r0 = k * per, r1 = min(rows, r0 + per);
  const bool colok = c0 < cols;                                 // cols % V == 0 (checked on the host)
  double acc[V];
#pragma unroll
  for (int j = 0; j < V; ++j) acc[j] = 0.0;
  int r = r0 + 2 * w + half;
  constexpr int STEP = 2 * CS_WARPS;
  if (colok && r + (U - 1) * STEP < r1) {
    // software pipeline: the next group's U loads are issued before the current group is summed
    uint4 u[U];
#pragma unroll
    for (int i = 0; i < U; ++i) u[i] = cs_ldg(x + (long)(r + i * STEP) * ld + c0);
    for (;;) {
      const int rn = r + U * STEP;
      const bool more = rn + (U - 1) * STEP < r1;
      uint4 nx[U];
      if (more) {
#pragma unroll
        for (int i = 0; i < U; ++i) nx[i] = cs_ldg(x + (long)(rn + i * STEP) * ld + c0);
      }
#pragma unroll
      for (int i = 0; i < U; ++i) {
        float f[V];
        cs_unpack(u[i], f);
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = __dadd_rn(acc[j], (double)f[j]);
      }
      r = rn;
      if (!more) break;
#pragma unroll
      for (int i = 0; i < U; ++i) u[i] = nx[i];
    }
  }
  if (colok) {
    for (; r < r1; r += STEP) {
      float f[V];
      cs_unpack(cs_ldg(x + (long)r * ld + c0), f);
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = __dadd_rn(acc[j], (double)f[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < V; ++j) {                                 // low half-warp + high half-warp
    const double o = __shfl_xor_sync(0xffffffffu, acc[j], 16);
    acc[j] = half ? __dadd_rn(o, acc[j]) : __dadd_rn(acc[j], o);
  }
  if (half == 0)
#pragma unroll
    for (int j = 0; j < V; ++j) cs_part[w * SW + cg16 * V + j] = acc[j];
  __syncthreads();
  if (threadIdx.x < SW) {
    double t = 0.0;
    for (int q = 0; q < CS_WARPS; ++q) t = __dadd_rn(t, cs_part[q * SW + threadIdx.x]);
    seg[threadIdx.x] = t;
  }
  cl.sync();
  const int c = blockIdx.x * SW + (int)threadIdx.x;
  if (k == 0 && threadIdx.x < SW && c < cols) {
    double t = 0.0;
    for (int q = 0; q < nseg; ++q) t = __dadd_rn(t, cl.map_shared_rank(seg, q)[threadIdx.x]);
    const float v = (float)t;
    out[c] = accumulate ? __fadd_rn(out[c], v) : v;
  }
  cl.sync();                                                     // keep seg[] alive for the remote reads
}

}  // namespace echo

using namespace echo;

// cluster of COLSUM_SEGS CTAs along grid y
template <typename Kern, typename... Args>
static cudaError_t launch_cluster_y(Kern kern, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = COLSUM_SEGS;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// attention hidden a = tanh(pre) backward (tanh keeps its output): one launch per
// decoder step instead of the four framework elementwise launches of the plain expression.
// Same IEEE operations, in the same order, as da * (1 - a * a) evaluated in fp32.
namespace echo {
template <typename T>
__global__ void __launch_bounds__(256) tanh_bwd_kernel(long n, const T* __restrict__ a, const float* __restrict__ da,
                                                       float* __restrict__ dpre) {
  pdl_wait();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const float x = to_f(a[i]);
    dpre[i] = __fmul_rn(da[i], __fsub_rn(1.0f, __fmul_rn(x, x)));
  }
}

}  // namespace echo

extern "C" echo_status echo_tanh_bwd(int64_t n, int32_t dtype, const void* a, const float* da, float* dpre,
                                     void* stream) {
  using namespace echo;
  const char* fn = "echo_tanh_bwd";
  if (n <= 0) return fail(ECHO_ERR_INVALID, "%s: n=%lld must be > 0", fn, (long long)n);
  if (!a || !da || !dpre) return fail(ECHO_ERR_INVALID, "%s: NULL a / da / dpre", fn);
  if (dtype != ECHO_FP32 && dtype != ECHO_BF16) return fail(ECHO_ERR_INVALID, "%s: bad dtype %d", fn, dtype);
  long g = (n + 255) / 256;
  if (g > 148L * 8) g = 148L * 8;
  cudaError_t e;
  if (dtype == ECHO_FP32)
    e = launch(tanh_bwd_kernel<float>, dim3((unsigned)g), dim3(256), 0, (cudaStream_t)stream, 1, (long)n,
               (const float*)a, da, dpre);
  else
    e = launch(tanh_bwd_kernel<__nv_bfloat16>, dim3((unsigned)g), dim3(256), 0, (cudaStream_t)stream, 1, (long)n,
               (const __nv_bfloat16*)a, da, dpre);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

extern "C" echo_status echo_colsum(int32_t rows, int32_t cols, int64_t ld, int32_t dtype, const void* x, float* out,
                                   int32_t accumulate, void* stream) {
  const char* fn = "echo_colsum";
  if (rows <= 0 || cols <= 0 || ld < cols) return fail(ECHO_ERR_INVALID, "%s: rows=%d cols=%d ld=%lld", fn, rows, cols,
                                                      (long long)ld);
  if (!x || !out) return fail(ECHO_ERR_INVALID, "%s: NULL x / out", fn);
  if (dtype != ECHO_FP32 && dtype != ECHO_BF16) return fail(ECHO_ERR_INVALID, "%s: bad dtype %d", fn, dtype);
  cudaError_t e;
  const int V = dtype == ECHO_FP32 ? CsVec<float>::V : CsVec<__nv_bfloat16>::V;
  const size_t es = dtype == ECHO_FP32 ? 4 : 2;
  if (cols % V == 0 && ld % V == 0 && aligned16(x) && (long)rows * cols >= (1L << 20)) {   // wide / long: vector path
    const int SW = 16 * V;
    const size_t smem = sizeof(double) * CS_WARPS * SW;
    const int strips = (cols + SW - 1) / SW;
    const int nseg = strips * COLSUM_SEGS >= 2 * 148 ? COLSUM_SEGS : 16;   // >= 2 CTAs per SM
    const dim3 grid(strips, nseg);
    const void* k = dtype == ECHO_FP32 ? (const void*)colsum_vec_kernel<float> : (const void*)colsum_vec_kernel<__nv_bfloat16>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return fail(ECHO_ERR_CUDA, "%s: cudaFuncSetAttribute: %s", fn, cudaGetErrorString(cudaGetLastError()));
    if (nseg > 8 && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      return fail(ECHO_ERR_CUDA, "%s: cluster size 16: %s", fn, cudaGetErrorString(cudaGetLastError()));
    (void)es;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(CS_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = nseg;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (dtype == ECHO_FP32)
      e = cudaLaunchKernelEx(&cfg, colsum_vec_kernel<float>, rows, cols, (long)ld, (const float*)x, out, accumulate);
    else
      e = cudaLaunchKernelEx(&cfg, colsum_vec_kernel<__nv_bfloat16>, rows, cols, (long)ld, (const __nv_bfloat16*)x, out,
                             accumulate);
    if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
    return check_launch(fn);
  }
  const dim3 grid((cols + 31) / 32, COLSUM_SEGS), block(32, 32);
  if (dtype == ECHO_FP32)
    e = launch_cluster_y(colsum_kernel<float>, grid, block, (cudaStream_t)stream, rows, cols, (long)ld,
                         (const float*)x, out, accumulate);
  else
    e = launch_cluster_y(colsum_kernel<__nv_bfloat16>, grid, block, (cudaStream_t)stream, rows, cols, (long)ld,
                         (const __nv_bfloat16*)x, out, accumulate);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

extern "C" echo_status echo_xent_fwd_bwd(int32_t N, int32_t V, float* logits, const float* bias,
                                         const int64_t* labels, float* row_loss, void* dlogits_bf16,
                                         void* stream) {
  const char* fn = "echo_xent_fwd_bwd";
  if (N <= 0 || V <= 0) return fail(ECHO_ERR_INVALID, "%s: N=%d V=%d must be > 0", fn, N, V);
  if (!logits || !labels || !row_loss) return fail(ECHO_ERR_INVALID, "%s: NULL logits / labels / row_loss", fn);
  if ((V & 3) == 0 && (!aligned16(logits) || (bias && !aligned16(bias)) || (dlogits_bf16 && ((uintptr_t)dlogits_bf16 & 7))))
    return fail(ECHO_ERR_INVALID, "%s: logits / bias must be 16-byte (bf16 output 8-byte) aligned", fn);
  const size_t smem = (size_t)V * sizeof(float);
  if (smem > 200 * 1024) return fail(ECHO_ERR_CAPACITY, "%s: V=%d exceeds the shared-memory row (51200)", fn, V);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute((const void*)xent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem);
    if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: cudaFuncSetAttribute: %s", fn, cudaGetErrorString(e));
  }
  const int grid = N < 148 * 16 ? N : 148 * 16;
  const cudaError_t e = launch(xent_kernel, dim3(grid), dim3(XENT_THREADS), smem, (cudaStream_t)stream, 1, N, V, bias,
                               logits, labels, row_loss, (__nv_bfloat16*)dlogits_bf16);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}
