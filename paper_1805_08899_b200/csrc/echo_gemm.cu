// echo_gemm.cu — IEEE-fp32 SIMT GEMM for the dense contractions around the hot path (row a0:
// the FCs of Eq. 1 / Eq. 2; outside the Echo decision, never
// recomputed).  Why our own: at the NMT step's shapes (M = 128 batch rows, N = 512..2048,
// K = 512..2048) cuBLAS's fp32 SIMT kernels launch 16-256 CTAs and run at 2-10 TFLOP/s; the
// per-step recurrent / attention GEMMs are ~80 % of the fp32 step.  This kernel:
//   * 256 threads, 64x64 (or 128x128 for large M*N) output tile, 4x4 (8x8) register tile per
//     thread, k-major shared tiles, global->register->shared double buffering;
//   * split-K over a thread-block CLUSTER (grid z = cluster z = S <= 8): each CTA reduces its K
//     range, the S partial tiles are summed in rank order through distributed shared memory —
//     deterministic, no atomics, no workspace;
//   * plain fp32 FMA (__fmaf_rn), fixed k order: same precision class as cuBLAS with TF32 off.
// C = alpha * op(A) op(B) + beta * C, row-major storage; op(A) is M x K, op(B) is K x N.
#include "echo_common.cuh"

#include <cooperative_groups.h>

namespace echo {

namespace cg = cooperative_groups;
constexpr int GEMM_THREADS = 256;

template <int BM, int BN, int BK, bool TA, bool TB>
__global__ void __launch_bounds__(GEMM_THREADS) gemm_f32_kernel(int M, int N, int K, int kchunk, float alpha,
                                                                const float* __restrict__ A, long lda,
                                                                const float* __restrict__ B, long ldb, float beta,
                                                                float* __restrict__ C, long ldc) {
  pdl_wait();
  constexpr int TM = BM / 16, TN = BN / 16;
  constexpr int PA = BM + 4, PB = BN + 4;                       // padded k-major rows
  constexpr int PIPE = 2 * BK * PA + 2 * BK * PB, PART = BM * (BN + 4);
  constexpr bool SPLIT_OK = PART * 4 <= 40 * 1024;               // split-K only for the 64x64 tile
  __shared__ __align__(16) float smem[SPLIT_OK && PART > PIPE ? PART : PIPE];
  float* As = smem;                                             // [2][BK][PA]
  float* Bs = smem + 2 * BK * PA;                               // [2][BK][PB]
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int S = gridDim.z, rank = blockIdx.z;
  const int kb = rank * kchunk, ke = min(K, kb + kchunk);
  // one float4 of A and of B per thread per k-tile (BM*BK == BN*BK == 4 * GEMM_THREADS)
  static_assert(BM * BK == 4 * GEMM_THREADS && BN * BK == 4 * GEMM_THREADS, "tile / thread mismatch");
  // A: !TA -> rows m, 4 consecutive k;  TA -> row k, 4 consecutive m
  const int a_r = TA ? tid / (BM / 4) : tid / (BK / 4);
  const int a_c = TA ? (tid % (BM / 4)) * 4 : (tid % (BK / 4)) * 4;
  // B: !TB -> row k, 4 consecutive n;  TB -> row n, 4 consecutive k
  const int b_r = TB ? tid / (BK / 4) : tid / (BN / 4);
  const int b_c = TB ? (tid % (BK / 4)) * 4 : (tid % (BN / 4)) * 4;
  auto load_a = [&](int k0, float4& v) {
    if (!TA) {
      const int m = m0 + a_r, k = k0 + a_c;
      v = (m < M && k < ke) ? *reinterpret_cast<const float4*>(A + (long)m * lda + k) : make_float4(0, 0, 0, 0);
    } else {
      const int k = k0 + a_r, m = m0 + a_c;
      v = (k < ke && m < M) ? *reinterpret_cast<const float4*>(A + (long)k * lda + m) : make_float4(0, 0, 0, 0);
    }
  };
  auto load_b = [&](int k0, float4& v) {
    if (!TB) {
      const int k = k0 + b_r, n = n0 + b_c;
      v = (k < ke && n < N) ? *reinterpret_cast<const float4*>(B + (long)k * ldb + n) : make_float4(0, 0, 0, 0);
    } else {
      const int n = n0 + b_r, k = k0 + b_c;
      v = (n < N && k < ke) ? *reinterpret_cast<const float4*>(B + (long)n * ldb + k) : make_float4(0, 0, 0, 0);
    }
  };
  auto store_a = [&](float* as, const float4& v) {
    if (!TA) {
      as[(a_c + 0) * PA + a_r] = v.x; as[(a_c + 1) * PA + a_r] = v.y;
      as[(a_c + 2) * PA + a_r] = v.z; as[(a_c + 3) * PA + a_r] = v.w;
    } else {
      *reinterpret_cast<float4*>(as + a_r * PA + a_c) = v;
    }
  };
  auto store_b = [&](float* bs, const float4& v) {
    if (!TB) {
      *reinterpret_cast<float4*>(bs + b_r * PB + b_c) = v;
    } else {
      bs[(b_c + 0) * PB + b_r] = v.x; bs[(b_c + 1) * PB + b_r] = v.y;
      bs[(b_c + 2) * PB + b_r] = v.z; bs[(b_c + 3) * PB + b_r] = v.w;
    }
  };
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
  float4 ra, rb;
  int buf = 0;
  if (kb < ke) {
    load_a(kb, ra);
    load_b(kb, rb);
    store_a(As, ra);
    store_b(Bs, rb);
  }
  __syncthreads();
  for (int k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) {                                                 // next tile in flight during the FMAs
      load_a(k0 + BK, ra);
      load_b(k0 + BK, rb);
    }
    const float* as = As + buf * BK * PA;
    const float* bs = Bs + buf * BK * PB;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(as + k * PA + ty * TM + i);
        a[i] = v.x; a[i + 1] = v.y; a[i + 2] = v.z; a[i + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < TN; j += 4) {
        const float4 v = *reinterpret_cast<const float4*>(bs + k * PB + tx * TN + j);
        b[j] = v.x; b[j + 1] = v.y; b[j + 2] = v.z; b[j + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_a(As + (buf ^ 1) * BK * PA, ra);
      store_b(Bs + (buf ^ 1) * BK * PB, rb);
    }
    __syncthreads();
    buf ^= 1;
  }
  if (S == 1 || !SPLIT_OK) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int m = m0 + ty * TM + i;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < TN; j += 4) {
        const int n = n0 + tx * TN + j;
        if (n >= N) continue;
        float4* cp = reinterpret_cast<float4*>(C + (long)m * ldc + n);
        float4 o = make_float4(__fmul_rn(alpha, acc[i][j]), __fmul_rn(alpha, acc[i][j + 1]),
                               __fmul_rn(alpha, acc[i][j + 2]), __fmul_rn(alpha, acc[i][j + 3]));
        if (beta != 0.0f) {
          const float4 c = *cp;
          o.x = __fmaf_rn(beta, c.x, o.x); o.y = __fmaf_rn(beta, c.y, o.y);
          o.z = __fmaf_rn(beta, c.z, o.z); o.w = __fmaf_rn(beta, c.w, o.w);
        }
        *cp = o;
      }
    }
    return;
  }
  // split-K: partial tile -> own shared memory; rank q reduces rows q, q + S, ... of the tile
  // over ranks 0..S-1 in order (distributed shared memory)
  if constexpr (SPLIT_OK) {
  float* Cs = smem;                                             // [BM][BN + 4]
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; j += 4)
      *reinterpret_cast<float4*>(Cs + (ty * TM + i) * (BN + 4) + tx * TN + j) =
          make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  for (int e = tid; e < BM * (BN / 4); e += GEMM_THREADS) {
    const int r = e / (BN / 4), c4 = (e % (BN / 4)) * 4;
    if (r % S != rank) continue;
    const int m = m0 + r, n = n0 + c4;
    if (m >= M || n >= N) continue;
    float4 s = make_float4(0, 0, 0, 0);
    for (int q = 0; q < S; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(cl.map_shared_rank(Cs, q) + r * (BN + 4) + c4);
      s.x = __fadd_rn(s.x, v.x); s.y = __fadd_rn(s.y, v.y); s.z = __fadd_rn(s.z, v.z); s.w = __fadd_rn(s.w, v.w);
    }
    float4* cp = reinterpret_cast<float4*>(C + (long)m * ldc + n);
    float4 o = make_float4(__fmul_rn(alpha, s.x), __fmul_rn(alpha, s.y), __fmul_rn(alpha, s.z), __fmul_rn(alpha, s.w));
    if (beta != 0.0f) {
      const float4 c = *cp;
      o.x = __fmaf_rn(beta, c.x, o.x); o.y = __fmaf_rn(beta, c.y, o.y);
      o.z = __fmaf_rn(beta, c.z, o.z); o.w = __fmaf_rn(beta, c.w, o.w);
    }
    *cp = o;
  }
  cl.sync();                                                    // remote partial tiles stay alive until read
  }
}

// ---------------------------------------------------------------- small-M path: cp.async pipeline
// 64x64 tile, BK = 16, NS-stage cp.async ring (16-byte copies, zero-filled outside the matrix);
// shared tiles keep the global layout (no transposition), so the fragment loads are 128-bit in
// whichever direction is contiguous; k is consumed in order (deterministic).
constexpr int P_BM = 64, P_BN = 64, P_BK = 16, P_NS = 4;
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <bool TA, bool TB>
__global__ void __launch_bounds__(GEMM_THREADS) gemm_f32_pipe(int M, int N, int K, int kchunk, float alpha,
                                                              const float* __restrict__ A, long lda,
                                                              const float* __restrict__ B, long ldb, float beta,
                                                              float* __restrict__ C, long ldc) {
  pdl_wait();
  // stage layouts: A !TA [64 m][BK+4] | TA [BK k][64+4];  B !TB [BK k][64+4] | TB [64 n][BK+4]
  constexpr int AS = TA ? P_BK * (P_BM + 4) : P_BM * (P_BK + 4);
  constexpr int BS = TB ? P_BN * (P_BK + 4) : P_BK * (P_BN + 4);
  constexpr int STAGE = AS + BS, PART = P_BM * (P_BN + 4);
  __shared__ __align__(16) float sm[P_NS * STAGE > PART ? P_NS * STAGE : PART];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * P_BM, n0 = blockIdx.x * P_BN;
  const int S = gridDim.z, rank = blockIdx.z;
  const int kb = rank * kchunk, ke = min(K, kb + kchunk);
  const int nk = ke > kb ? (ke - kb + P_BK - 1) / P_BK : 0;
  auto load_stage = [&](int st, int k0) {
    float* as = sm + st * STAGE;
    float* bs = as + AS;
    if (!TA) {
      const int m = tid / 4, kc = (tid % 4) * 4;
      const bool ok = m0 + m < M && k0 + kc < ke;
      cp_async16(as + m * (P_BK + 4) + kc, ok ? A + (long)(m0 + m) * lda + k0 + kc : A, ok);
    } else {
      const int k = tid / 16, mc = (tid % 16) * 4;
      const bool ok = k0 + k < ke && m0 + mc < M;
      cp_async16(as + k * (P_BM + 4) + mc, ok ? A + (long)(k0 + k) * lda + m0 + mc : A, ok);
    }
    if (!TB) {
      const int k = tid / 16, nc = (tid % 16) * 4;
      const bool ok = k0 + k < ke && n0 + nc < N;
      cp_async16(bs + k * (P_BN + 4) + nc, ok ? B + (long)(k0 + k) * ldb + n0 + nc : B, ok);
    } else {
      const int n = tid / 4, kc = (tid % 4) * 4;
      const bool ok = n0 + n < N && k0 + kc < ke;
      cp_async16(bs + n * (P_BK + 4) + kc, ok ? B + (long)(n0 + n) * ldb + k0 + kc : B, ok);
    }
  };
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
#pragma unroll
  for (int st = 0; st < P_NS - 1; ++st) {
    if (st < nk) load_stage(st, kb + st * P_BK);
    cp_async_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<P_NS - 2>();
    __syncthreads();
    const int nxt = it + P_NS - 1;                   // refill the stage consumed last iteration
    if (nxt < nk) load_stage(nxt % P_NS, kb + nxt * P_BK);
    cp_async_commit();
    const float* as = sm + (it % P_NS) * STAGE;
    const float* bs = as + AS;
#pragma unroll
    for (int kk = 0; kk < P_BK; kk += 4) {
      float a[4][4], b[4][4];                        // a[i][q] = A(m_i, k+q), b[q][j] = B(k+q, n_j)
      if (!TA) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 v = *reinterpret_cast<const float4*>(as + (ty * 4 + i) * (P_BK + 4) + kk);
          a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(as + (kk + q) * (P_BM + 4) + ty * 4);
          a[0][q] = v.x; a[1][q] = v.y; a[2][q] = v.z; a[3][q] = v.w;
        }
      }
      if (!TB) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(bs + (kk + q) * (P_BN + 4) + tx * 4);
          b[q][0] = v.x; b[q][1] = v.y; b[q][2] = v.z; b[q][3] = v.w;
        }
      } else {                                       // TB: columns tx + 16 j (conflict-free rows)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(bs + (tx + 16 * j) * (P_BK + 4) + kk);
          b[0][j] = v.x; b[1][j] = v.y; b[2][j] = v.z; b[3][j] = v.w;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(a[i][q], b[q][j], acc[i][j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  auto store = [&](int m, int n, float4 s) {
    float4* cp = reinterpret_cast<float4*>(C + (long)m * ldc + n);
    float4 o = make_float4(__fmul_rn(alpha, s.x), __fmul_rn(alpha, s.y), __fmul_rn(alpha, s.z), __fmul_rn(alpha, s.w));
    if (beta != 0.0f) {
      const float4 c = *cp;
      o.x = __fmaf_rn(beta, c.x, o.x); o.y = __fmaf_rn(beta, c.y, o.y);
      o.z = __fmaf_rn(beta, c.z, o.z); o.w = __fmaf_rn(beta, c.w, o.w);
    }
    *cp = o;
  };
  float* Cs = sm;                                    // [64][68] tile (partial, or staging for S == 1)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float* row = Cs + (ty * 4 + i) * (P_BN + 4);
    if (!TB) {
      *reinterpret_cast<float4*>(row + tx * 4) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) row[tx + 16 * j] = acc[i][j];
    }
  }
  if (S == 1) {
    __syncthreads();
    for (int e = tid; e < P_BM * (P_BN / 4); e += GEMM_THREADS) {
      const int r = e / (P_BN / 4), c4 = (e % (P_BN / 4)) * 4;
      const int m = m0 + r, n = n0 + c4;
      if (m < M && n < N) store(m, n, *reinterpret_cast<const float4*>(Cs + r * (P_BN + 4) + c4));
    }
    return;
  }
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  for (int e = tid; e < P_BM * (P_BN / 4); e += GEMM_THREADS) {
    const int r = e / (P_BN / 4), c4 = (e % (P_BN / 4)) * 4;
    if (r % S != rank) continue;
    const int m = m0 + r, n = n0 + c4;
    if (m >= M || n >= N) continue;
    float4 s = make_float4(0, 0, 0, 0);
    for (int q = 0; q < S; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(cl.map_shared_rank(Cs, q) + r * (P_BN + 4) + c4);
      s.x = __fadd_rn(s.x, v.x); s.y = __fadd_rn(s.y, v.y); s.z = __fadd_rn(s.z, v.z); s.w = __fadd_rn(s.w, v.w);
    }
    store(m, n, s);
  }
  cl.sync();
}

template <bool TA, bool TB>
static cudaError_t launch_pipe(int M, int N, int K, float alpha, const float* A, long lda, const float* B, long ldb,
                               float beta, float* C, long ldc, cudaStream_t st) {
  // split K until ~2 CTAs per SM are in flight (each SM holds up to 4 of these CTAs); clusters up
  // to 16 (non-portable size) so M = 128 rows x N = 512 still fills the GPU
  const int tiles = ((M + P_BM - 1) / P_BM) * ((N + P_BN - 1) / P_BN);
  static const int smax = [] {
    const cudaError_t e0 = cudaFuncSetAttribute(gemm_f32_pipe<false, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const cudaError_t e1 = cudaFuncSetAttribute(gemm_f32_pipe<false, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const cudaError_t e2 = cudaFuncSetAttribute(gemm_f32_pipe<true, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const cudaError_t e3 = cudaFuncSetAttribute(gemm_f32_pipe<true, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e0 || e1 || e2 || e3) {
      cudaGetLastError();
      return 8;
    }
    return 16;
  }();
  int S = 1;
  const int limit = TA == TA ? smax : 8;
  while (S < limit && tiles * S * 2 <= 2 * 2 * 148 && K / (S * 2) >= 2 * P_BK) S *= 2;
  const int kchunk = ((K + S - 1) / S + P_BK - 1) / P_BK * P_BK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((N + P_BN - 1) / P_BN, (M + P_BM - 1) / P_BM, S);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = (unsigned)S;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_f32_pipe<TA, TB>, M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc);
}

template <int BM, int BN, int BK, bool TA, bool TB>
static cudaError_t launch_gemm(int M, int N, int K, float alpha, const float* A, long lda, const float* B, long ldb,
                               float beta, float* C, long ldc, cudaStream_t st) {
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int S = 1;
  if (BM * (BN + 4) * 4 <= 40 * 1024)                           // split-K (cluster) only for the 64x64 tile
    while (S < 8 && tiles * S * 2 <= 2 * 148 && K / (S * 2) >= 4 * BK) S *= 2;   // ~1-2 waves of CTAs
  const int kchunk = ((K + S - 1) / S + BK - 1) / BK * BK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((N + BN - 1) / BN, (M + BM - 1) / BM, S);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = (unsigned)S;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_f32_kernel<BM, BN, BK, TA, TB>, M, N, K, kchunk, alpha, A, lda, B, ldb, beta,
                            C, ldc);
}

template <bool TA, bool TB>
static cudaError_t dispatch(int M, int N, int K, float alpha, const float* A, long lda, const float* B, long ldb,
                            float beta, float* C, long ldc, cudaStream_t st) {
  if ((long)M * N >= 1024L * 1024)
    return launch_gemm<128, 128, 8, TA, TB>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  return launch_pipe<TA, TB>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
}

}  // namespace echo

using namespace echo;

extern "C" int32_t echo_gemm_f32_supported(int32_t M, int32_t N, int32_t K, int32_t transA, int32_t transB,
                                           int64_t lda, int64_t ldb, int64_t ldc) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  if (N % 4 || ldc % 4 || lda % 4 || ldb % 4) return 0;
  if (!transA && K % 4) return 0;
  if (transA && M % 4) return 0;
  if (transB && K % 4) return 0;
  return 1;
}

extern "C" echo_status echo_gemm_f32(int32_t M, int32_t N, int32_t K, float alpha, const float* A, int64_t lda,
                                     int32_t transA, const float* B, int64_t ldb, int32_t transB, float beta,
                                     float* C, int64_t ldc, void* stream) {
  const char* fn = "echo_gemm_f32";
  if (!echo_gemm_f32_supported(M, N, K, transA, transB, lda, ldb, ldc))
    return fail(ECHO_ERR_UNSUPPORTED, "%s: M=%d N=%d K=%d tA=%d tB=%d lda=%lld ldb=%lld ldc=%lld not supported", fn, M,
                N, K, transA, transB, (long long)lda, (long long)ldb, (long long)ldc);
  if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return fail(ECHO_ERR_INVALID, "%s: A, B, C must be 16-byte aligned", fn);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (!transA && !transB) e = dispatch<false, false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  else if (!transA && transB) e = dispatch<false, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  else if (transA && !transB) e = dispatch<true, false>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  else e = dispatch<true, true>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}
