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
  return launch_gemm<64, 64, 16, TA, TB>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
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
