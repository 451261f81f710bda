// echo_attn.cu — MLP attention forward (a5) and backward with fused
// recomputation (a6).  PAPER.md §2 lines 129-133 (scores, weights alpha_ts,
// context as the alpha-weighted average of H_s) and Fig. 7 / Fig. 10
// (PAPER.md:360, 633): the broadcast-add + tanh feature maps E [B,Ts,A] are the
// largest stash of the NMT model; Echo keeps them mirrored and
// regenerates them in the backward pass.
//
// Design: one thread-block CLUSTER of C CTAs per batch
// row b (C in {1,2,4,8}, from Ts); CTA rank r owns the source positions
// [r*chunk, (r+1)*chunk).  The softmax statistics (max, sum), the dot
// sum_s alpha_s dalpha_s and the cross-position reductions (ctx, dqp, dv) are
// combined across the cluster through distributed shared memory in ascending
// rank order, so one row's Ts x (A + Hk) stream is spread over C SMs (B*C CTAs
// per launch instead of B) without atomics.  Inside a CTA, warp w owns local
// positions i = w, w + NW, ...; a lane owns 16-byte vectors of the A / Hk axis,
// so each warp access is a coalesced 512-byte (fp32) row segment.  The score,
// softmax and context code is the SAME device code with the SAME mapping in
// the forward and backward kernels, which makes the regenerated alpha / ctx
// bit-identical to the stashed ones.
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>
#include <cuda.h>

#include "echo_common.cuh"

namespace echo {

namespace cg = cooperative_groups;

#ifdef ECHO_PHASE_TIMING
// debug-only per-CTA phase timestamps (clock64 of thread 0; slot 15 = globaltimer at start)
__device__ unsigned long long g_echo_phase[16][8192];
#define ECHO_PHASE(k)                                                                         \
  do {                                                                                        \
    if (threadIdx.x == 0) {                                                                   \
      const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                                   \
      if (cta_ < 8192) {                                                                      \
        g_echo_phase[k][cta_] = clock64();                                                    \
        if ((k) == 0 || (k) == 10) {                                                          \
          unsigned long long gt_;                                                             \
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                             \
          g_echo_phase[(k) == 0 ? 15 : 14][cta_] = gt_;                                       \
        }                                                                                     \
      }                                                                                       \
    }                                                                                         \
  } while (0)
#else
#define ECHO_PHASE(k) do { } while (0)
#endif

// The ONE tanh of the attention feature map E = tanh(z) (a5, a6 and the deferred passes; readings
// R9 / R9b).  fp32 storage: IEEE-accurate tanhf.  bf16 storage: z is a bf16 value and the 2e-2
// storage tolerance applies, so E = sign(z) (1 - 2 / (1 + 2^(2 log2(e) |z|))) with the MUFU ex2 / rcp
// approximations (absolute error <= 1.8e-7 over all floats, scripts/micro/tanh_err.cu: 20000x
// below the bf16 rounding of z) in 7 instructions instead of 16.  Every kernel that evaluates E
// for a given storage type uses this function, so STASH and RECOMPUTE stay bit-identical.
// Round 2: E = 1 - 2 / (2^(2 log2(e) z) + 1) without the |z| / copysign (large negative z: ex2
// flushes to 0 -> -1; large positive: inf -> 1), so two elements can be evaluated with the packed
// fp32x2 FMUL2 / FADD2 / FFMA2 of sm_100 (att_tanh2_bf16: the same IEEE operations per lane, hence
// the same bits as this scalar form).  Max abs error over all floats: scripts/micro/tanh_err.cu.
template <typename T>
__device__ __forceinline__ float att_tanh(float z) {
  if constexpr (sizeof(T) == 4) {
    return tanhf(z);
  } else {
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmul_rn(z, 2.8853900817779268f)));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fadd_rn(e, 1.0f)));
    return __fmaf_rn(-2.0f, r, 1.0f);
  }
}
__device__ __forceinline__ float2 att_tanh2_bf16(float2 z) {
  const float2 t = __fmul2_rn(z, make_float2(2.8853900817779268f, 2.8853900817779268f));
  float2 e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(t.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(t.y));
  const float2 d = __fadd2_rn(e, make_float2(1.0f, 1.0f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(d.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(d.y));
  return __ffma2_rn(r, make_float2(-2.0f, -2.0f), make_float2(1.0f, 1.0f));
}

constexpr int ATT_THREADS = 256;
constexpr int ATT_WARPS = ATT_THREADS / 32;

// score_s = sum_a tanh(round_s(qp_a + Kp_{s,a})) * v_a  (one warp; lane-strided vectors).
// The stashed feature map is the tanh INPUT z = round_s(qp + Kp) (byte-identical stand-in
// for E = tanh(z), R15): E and 1 - E^2 are then always evaluated in fp32 from z.
template <typename T>
__device__ __forceinline__ float score_row(const T* __restrict__ kp_row, const float* qp_s, const float* v_s, int A,
                                           int lane, T* Z_out) {
  constexpr int V = St<T>::VEC;
  float acc = 0.0f;
  for (int iv = lane; iv < A / V; iv += 32) {
    float kv[V], z[V];
    ld16(kp_row + iv * V, kv);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      z[k] = St<T>::round(__fadd_rn(qp_s[iv * V + k], kv[k]));
      acc = __fmaf_rn(att_tanh<T>(z[k]), v_s[iv * V + k], acc);
    }
    if (Z_out) st16(Z_out + iv * V, z);
  }
  return warp_sum(acc);
}


__host__ __device__ __forceinline__ int ctx_groups(int Hk, int V) {
  const int ncols = Hk / V;
  return ncols >= ATT_THREADS ? 1 : ATT_THREADS / ncols;
}

// cluster size for a row of Ts positions: next power of two of ceil(Ts / 8), capped at 8
static inline int att_cluster(int Ts) {
  const int want = (Ts + 7) / 8;
  int C = 1;
  while (C < want && C < 8) C <<= 1;
  return C;
}

template <typename T>
__device__ __forceinline__ void stage_vec(float* dst, const T* __restrict__ src, int n, int tid) {
  constexpr int V = St<T>::VEC;
  for (int iv = tid; iv < n / V; iv += ATT_THREADS) {
    float x[V];
    ld16(src + iv * V, x);
#pragma unroll
    for (int k = 0; k < V; ++k) dst[iv * V + k] = x[k];
  }
}

__device__ __forceinline__ int row_len(const int32_t* src_len, int b, int Ts) {
  if (!src_len) return Ts;
  int n = src_len[b];
  return n < 1 ? 1 : (n > Ts ? Ts : n);
}

// Rank-ordered cluster reductions of one float per CTA; the C (<= 8) remote DSMEM loads are
// issued back to back before the fixed-order combine.
__device__ __forceinline__ float cl_sum(cg::cluster_group& cl, float* p, int C) {
  float t[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) t[c] = c < C ? *cl.map_shared_rank(p, c) : 0.0f;
  float x = 0.0f;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < C) x = __fadd_rn(x, t[c]);
  return x;
}

// Softmax over the row, distributed over the cluster, with ONE cluster barrier: every CTA
// publishes its local (max m_c, sum l_c = sum exp(score - m_c)); all CTAs then form the same
// m = max_c m_c and L = sum_c l_c exp(m_c - m) in rank order.  sc[0..ns) holds this CTA's
// scores on entry and alpha = exp(score - m) / L on exit.  Uses red[0], red[1].
__device__ __forceinline__ void softmax_cluster(cg::cluster_group& cl, float* sc, int ns, float* red, int C,
                                                int tid) {
  const int lane = tid & 31, w = tid >> 5;
  if (w == 0) {
    float m = -INFINITY;
    for (int i = lane; i < ns; i += 32) m = fmaxf(m, sc[i]);
    m = warp_max(m);
    float l = 0.0f;
    for (int i = lane; i < ns; i += 32) l = __fadd_rn(l, expf(__fsub_rn(sc[i], m)));
    l = warp_sum(l);
    if (lane == 0) { red[0] = m; red[1] = l; }
  }
  cl.sync();
  float mc[8], lc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    mc[c] = c < C ? *cl.map_shared_rank(red, c) : -INFINITY;
    lc[c] = c < C ? *cl.map_shared_rank(red + 1, c) : 0.0f;
  }
  float m = -INFINITY;
#pragma unroll
  for (int c = 0; c < 8; ++c) m = fmaxf(m, mc[c]);
  float L = 0.0f;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < C && lc[c] > 0.0f) L = __fadd_rn(L, __fmul_rn(lc[c], expf(__fsub_rn(mc[c], m))));
  if (w == 0)
    for (int i = lane; i < ns; i += 32) sc[i] = __fdiv_rn(expf(__fsub_rn(sc[i], m)), L);
  __syncthreads();
}

// Rank r writes its slice of the Hk columns: out = round_s(sum_c xfer_c) in rank order.
template <typename T>
__device__ __forceinline__ void ctx_finish(cg::cluster_group& cl, float* xfer, int Hk, T* ctx_out, int C, int r,
                                           int tid) {
  constexpr int V = St<T>::VEC;
  const int ncols = Hk / V;
  const int per = (ncols + C - 1) / C;
  const int c0 = r * per, c1 = min(ncols, c0 + per);
  for (int cv = c0 + tid; cv < c1; cv += ATT_THREADS) {
    float t[8][V];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < C) {
        const float* q = cl.map_shared_rank(xfer, c) + cv * V;
#pragma unroll
        for (int k = 0; k < V; ++k) t[c][k] = q[k];
      }
    float o[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float x = 0.0f;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < C) x = __fadd_rn(x, t[c][k]);
      o[k] = St<T>::round(x);
    }
    st16(ctx_out + cv * V, o);
  }
}

// This CTA's part of ctx = sum_{s<n} alpha_s Hs_s: G thread groups split the local positions,
// fixed-order combine into xfer[Hk].  The caller then cl.sync()s and runs ctx_finish.
template <typename T>
__device__ __forceinline__ void context_partial(const T* __restrict__ hs_b, long stride_s, const float* alpha, int s0,
                                                int ns, int Hk, float* part, float* xfer, int tid) {
  constexpr int V = St<T>::VEC;
  const int ncols = Hk / V;
  const int G = ctx_groups(Hk, V);
  if (G > 1) {
    const int g = tid / ncols, cv = tid - g * ncols;
    if (g < G) {
      float acc[V];
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = 0.0f;
      for (int i = g; i < ns; i += G) {
        float h[V];
        ld16(hs_b + (long)(s0 + i) * stride_s + cv * V, h);
        const float a = alpha[i];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = __fmaf_rn(a, h[k], acc[k]);
      }
#pragma unroll
      for (int k = 0; k < V; ++k) part[g * Hk + cv * V + k] = acc[k];
    }
  } else {
    for (int cv = tid; cv < ncols; cv += ATT_THREADS) {
      float acc[V];
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = 0.0f;
      for (int i = 0; i < ns; ++i) {
        float h[V];
        ld16(hs_b + (long)(s0 + i) * stride_s + cv * V, h);
        const float a = alpha[i];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = __fmaf_rn(a, h[k], acc[k]);
      }
#pragma unroll
      for (int k = 0; k < V; ++k) part[cv * V + k] = acc[k];
    }
  }
  __syncthreads();
  for (int k = tid; k < Hk; k += ATT_THREADS) {
    float x = part[k];
    for (int g = 1; g < G; ++g) x = __fadd_rn(x, part[g * Hk + k]);
    xfer[k] = x;
  }
  __syncthreads();
}

// rank r finishes its slice of A: dqp = sum_c xq_c, dv_part += sum_c xv_c (rank order)
__device__ __forceinline__ void dqp_dv_finish(cg::cluster_group& cl, float* xq, float* xv, int A, float* dqp_b,
                                              float* dvp_b, int C, int r, int tid) {
  const int per = (A + C - 1) / C;
  for (int a = r * per + tid; a < min(A, (r + 1) * per); a += ATT_THREADS) {
    float tq[8], tv[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < C) { tq[c] = cl.map_shared_rank(xq, c)[a]; tv[c] = cl.map_shared_rank(xv, c)[a]; }
    float q = 0.0f, vv = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < C) { q = __fadd_rn(q, tq[c]); vv = __fadd_rn(vv, tv[c]); }
    dqp_b[a] = q;
    dvp_b[a] = __fadd_rn(dvp_b[a], vv);
  }
}

// ---------------------------------------------------------------- a5 forward
template <typename T>
__global__ void __launch_bounds__(ATT_THREADS) attn_fwd_kernel(echo_attn_desc d, int chunk, const T* __restrict__ qp,
                                                               const T* __restrict__ Kp, const T* __restrict__ v,
                                                               const T* __restrict__ Hs,
                                                               const int32_t* __restrict__ src_len,
                                                               T* __restrict__ ctx, T* __restrict__ Z_st,
                                                               float* __restrict__ alpha_st) {
  pdl_wait();
  constexpr int V = St<T>::VEC;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ float sm[];
  const int A = d.A, Ts = d.Ts, Hk = d.Hk;
  const int C = (int)cl.num_blocks(), r = (int)cl.block_rank();
  const int G = ctx_groups(Hk, V);
  float* qp_s = sm;
  float* v_s = qp_s + A;
  float* red = v_s + A;                 // [4]
  float* sc = red + 4;                  // [chunk]
  float* part = sc + ((chunk + 3) & ~3);
  float* xfer = part + G * Hk;
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = row_len(src_len, b, Ts);
  const int s0 = r * chunk;
  const int ns = max(0, min(s0 + chunk, n) - s0);
  const int send = min(s0 + chunk, Ts);
  stage_vec<T>(qp_s, qp + (long)b * A, A, tid);
  stage_vec<T>(v_s, v, A, tid);
  __syncthreads();
  const T* kp_b = Kp + (long)b * d.kp_stride_b;
  for (int i = w; i < ns; i += ATT_WARPS) {
    T* z_out = Z_st ? Z_st + ((long)b * Ts + s0 + i) * A : nullptr;
    const float scv = score_row<T>(kp_b + (long)(s0 + i) * d.kp_stride_s, qp_s, v_s, A, lane, z_out);
    if (lane == 0) sc[i] = scv;
  }
  if (Z_st) {  // masked positions of this chunk hold zeros
    float z[V];
#pragma unroll
    for (int k = 0; k < V; ++k) z[k] = 0.0f;
    for (int s = max(s0, n) + w; s < send; s += ATT_WARPS)
      for (int iv = lane; iv < A / V; iv += 32) st16(Z_st + ((long)b * Ts + s) * A + iv * V, z);
  }
  __syncthreads();
  softmax_cluster(cl, sc, ns, red, C, tid);
  if (alpha_st)
    for (int s = s0 + tid; s < send; s += ATT_THREADS) alpha_st[(long)b * Ts + s] = (s - s0 < ns) ? sc[s - s0] : 0.0f;
  context_partial<T>(Hs + (long)b * d.hs_stride_b, d.hs_stride_s, sc, s0, ns, Hk, part, xfer, tid);
  cl.sync();
  ctx_finish<T>(cl, xfer, Hk, ctx + (long)b * Hk, C, r, tid);
  cl.sync();
}

// ---------------------------------------------------------------- a6 backward (fused recompute)
template <typename T>
__global__ void __launch_bounds__(ATT_THREADS) attn_bwd_kernel(echo_attn_desc d, int chunk, const T* __restrict__ qp,
                                                               const T* __restrict__ Kp, const T* __restrict__ v,
                                                               const T* __restrict__ Hs,
                                                               const int32_t* __restrict__ src_len,
                                                               const T* __restrict__ Z_st,
                                                               const float* __restrict__ alpha_st,
                                                               const float* __restrict__ dctx, float* __restrict__ dqp,
                                                               float* __restrict__ dKp, float* __restrict__ dHs,
                                                               float* __restrict__ dv_part, T* __restrict__ ctx_regen) {
  pdl_wait();
  constexpr int V = St<T>::VEC;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ float sm[];
  const int A = d.A, Ts = d.Ts, Hk = d.Hk;
  const int C = (int)cl.num_blocks(), r = (int)cl.block_rank();
  const int G = ctx_groups(Hk, V);
  const int cp = (chunk + 3) & ~3;
  float* qp_s = sm;
  float* v_s = qp_s + A;
  float* dctx_s = v_s + A;
  float* red = dctx_s + Hk;             // [0] max [1] sum [2] dot
  float* sc = red + 4;                  // [chunk] scores -> alpha
  float* dal = sc + cp;                 // [chunk] dLoss/dalpha
  float* wq = dal + cp;                 // [NW][A] per-warp dqp partials
  float* wv = wq + ATT_WARPS * A;       // [NW][A] per-warp dv partials
  float* xq = wv + ATT_WARPS * A;       // [A] CTA dqp partial
  float* xv = xq + A;                   // [A] CTA dv partial
  float* part = xv + A;                 // [G][Hk]
  float* xfer = part + G * Hk;          // [Hk]
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = row_len(src_len, b, Ts);
  const int s0 = r * chunk;
  const int ns = max(0, min(s0 + chunk, n) - s0);
  const bool recompute = (Z_st == nullptr);
  if (recompute) stage_vec<T>(qp_s, qp + (long)b * A, A, tid);
  stage_vec<T>(v_s, v, A, tid);
  for (int i = tid; i < Hk; i += ATT_THREADS) dctx_s[i] = dctx[(long)b * Hk + i];
  for (int i = tid; i < ATT_WARPS * A; i += ATT_THREADS) { wq[i] = 0.0f; wv[i] = 0.0f; }
  __syncthreads();
  const T* kp_b = Kp + (long)b * d.kp_stride_b;
  const T* hs_b = Hs + (long)b * d.hs_stride_b;
  // phase 1: regenerate scores (RECOMPUTE) and dalpha_s = dctx . Hs_s
  for (int i = w; i < ns; i += ATT_WARPS) {
    const int s = s0 + i;
    if (recompute) {
      const float scv = score_row<T>(kp_b + (long)s * d.kp_stride_s, qp_s, v_s, A, lane, nullptr);
      if (lane == 0) sc[i] = scv;
    }
    float acc = 0.0f;
    const T* hrow = hs_b + (long)s * d.hs_stride_s;
    for (int iv = lane; iv < Hk / V; iv += 32) {
      float h[V];
      ld16(hrow + iv * V, h);
#pragma unroll
      for (int k = 0; k < V; ++k) acc = __fmaf_rn(dctx_s[iv * V + k], h[k], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) dal[i] = acc;
  }
  if (!recompute)
    for (int i = tid; i < ns; i += ATT_THREADS) sc[i] = alpha_st[(long)b * Ts + s0 + i];
  __syncthreads();
  // phase 2/3: softmax and ctx, the same device code as a5 (RECOMPUTE only)
  const bool do_ctx = recompute && ctx_regen;
  if (recompute) {
    softmax_cluster(cl, sc, ns, red, C, tid);
    if (do_ctx) context_partial<T>(hs_b, d.hs_stride_s, sc, s0, ns, Hk, part, xfer, tid);
  }
  // dot = sum_s alpha_s dalpha_s, cluster-wide in rank order (same barrier as the ctx exchange)
  if (w == 0) {
    float acc = 0.0f;
    for (int i = lane; i < ns; i += 32) acc = __fmaf_rn(sc[i], dal[i], acc);
    acc = warp_sum(acc);
    if (lane == 0) red[2] = acc;
  }
  cl.sync();
  if (do_ctx) ctx_finish<T>(cl, xfer, Hk, ctx_regen + (long)b * Hk, C, r, tid);
  const float dot = cl_sum(cl, red + 2, C);
  // phase 4: ds, dE, dKp +=, dHs +=, dqp / dv partials
  float* wq_w = wq + w * A;
  float* wv_w = wv + w * A;
  for (int i = w; i < ns; i += ATT_WARPS) {
    const int s = s0 + i;
    const float al = sc[i];
    const float ds = __fmul_rn(al, __fsub_rn(dal[i], dot));
    const T* kp_row = kp_b + (long)s * d.kp_stride_s;
    float* dkp_row = dKp + (long)b * d.kp_stride_b + (long)s * d.kp_stride_s;
    const T* z_row = Z_st ? Z_st + ((long)b * Ts + s) * A : nullptr;
    for (int iv = lane; iv < A / V; iv += 32) {
      float z[V];
      if (recompute) {
        float kv[V];
        ld16(kp_row + iv * V, kv);
#pragma unroll
        for (int k = 0; k < V; ++k) z[k] = St<T>::round(__fadd_rn(qp_s[iv * V + k], kv[k]));
      } else {
        ld16(z_row + iv * V, z);
      }
      float dk[V];
      ldf<V>(dkp_row + iv * V, dk);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float e = att_tanh<T>(z[k]);
        const float dE = __fmul_rn(__fmul_rn(ds, v_s[iv * V + k]), __fsub_rn(1.0f, __fmul_rn(e, e)));
        dk[k] = __fadd_rn(dk[k], dE);
        wq_w[iv * V + k] = __fadd_rn(wq_w[iv * V + k], dE);
        wv_w[iv * V + k] = __fmaf_rn(ds, e, wv_w[iv * V + k]);
      }
      stf<V>(dkp_row + iv * V, dk);
    }
    float* dhs_row = dHs + (long)b * d.hs_stride_b + (long)s * d.hs_stride_s;
    for (int iv = lane; iv < Hk / V; iv += 32) {
      float dh[V];
      ldf<V>(dhs_row + iv * V, dh);
#pragma unroll
      for (int k = 0; k < V; ++k) dh[k] = __fmaf_rn(al, dctx_s[iv * V + k], dh[k]);
      stf<V>(dhs_row + iv * V, dh);
    }
  }
  __syncthreads();
  for (int a = tid; a < A; a += ATT_THREADS) {
    float q = wq[a], vv = wv[a];
    for (int ww = 1; ww < ATT_WARPS; ++ww) {
      q = __fadd_rn(q, wq[ww * A + a]);
      vv = __fadd_rn(vv, wv[ww * A + a]);
    }
    xq[a] = q;
    xv[a] = vv;
  }
  cl.sync();
  dqp_dv_finish(cl, xq, xv, A, dqp + (long)b * A, dv_part + (long)b * A, C, r, tid);
  cl.sync();
}

// ================================================================ TMA-staged feature-split cluster path
// The row b is processed by a cluster of C CTAs that split the FEATURE axes: CTA r owns a
// slice of <= 128 columns of A (and of Hk).  At kernel entry ONE thread issues tensor-map TMA
// loads (cp.async.bulk.tensor.3d; one box = all Ts positions x the CTA's column slice) of Kp (or
// the stashed Z) and Hs, and in the backward also of the dKp / dHs accumulators, completing on
// mbarriers — all of the CTA's HBM traffic is in flight at once — and the backward writes the
// updated accumulators back with two TMA stores.
// Per position, a warp produces the partial score (and partial dalpha) over the slice; ONE
// cluster exchange (DSMEM) sums the partials in rank order; every CTA runs the tiny softmax
// redundantly; ctx, dKp, dHs, dqp and dv are then column-local, one thread per column looping
// over s.  Forward and backward share the partial-score code, the rank-ordered gather, the
// softmax warp and the ctx column loop, so the regenerated alpha / ctx are bit-identical to the
// stashed ones.
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) { mbar_wait_bounded(smem_u32(bar), phase); }

struct Slice {
  int C, r, a0, a1, h0, h1;   // this CTA's column ranges [a0, a1) of A and [h0, h1) of Hk
};
static __host__ __device__ __forceinline__ int tma_cluster(int A, int Hk) {
  const int m = A > Hk ? A : Hk;
  const int want = (m + 127) / 128;
  int C = 1;
  while (C < want && C < 8) C <<= 1;
  return C;
}
static __host__ __device__ __forceinline__ int tma_width(int X, int C) { return ((X + C - 1) / C + 7) / 8 * 8; }
// launch geometry computed once on the host (no integer divisions per CTA)
struct TmaGeo {
  int C, Wb, WHb, R, Tr, P;   // cluster size, box widths, chunk rows, tile rows, phase-4 phases
  int pf;                     // a6 dKp / dH_s L2 prefetch: 0 off, 1 after the stage-in landed, 2 at issue
  int l2last;                 // 1: Kp / H_s / dKp / dH_s traffic carries an L2 evict_last policy
};
__device__ __forceinline__ Slice make_slice_g(const TmaGeo& q, int A, int Hk, int r) {
  Slice g;
  g.C = q.C;
  g.r = r;
  g.a0 = min(A, r * q.Wb);
  g.a1 = min(A, g.a0 + q.Wb);
  g.h0 = min(Hk, r * q.WHb);
  g.h1 = min(Hk, g.h0 + q.WHb);
  return g;
}
__device__ __forceinline__ Slice make_slice(int A, int Hk, int C, int r) {
  Slice g;
  g.C = C;
  g.r = r;
  const int pa = tma_width(A, C), ph = tma_width(Hk, C);
  g.a0 = min(A, r * pa);
  g.a1 = min(A, g.a0 + pa);
  g.h0 = min(Hk, r * ph);
  g.h1 = min(Hk, g.h0 + ph);
  return g;
}

// 4 consecutive storage elements from shared memory as floats
__device__ __forceinline__ void lds4(const float* p, float (&o)[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void lds4(const __nv_bfloat16* p, float (&o)[4]) {
  const uint2 v = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
__device__ __forceinline__ void stg4(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void stg4(__nv_bfloat16* p, const float (&v)[4]) {
  uint2 u;
  *reinterpret_cast<__nv_bfloat162*>(&u.x) = __floats2bfloat162_rn(v[0], v[1]);
  *reinterpret_cast<__nv_bfloat162*>(&u.y) = __floats2bfloat162_rn(v[2], v[3]);
  *reinterpret_cast<uint2*>(p) = u;
}

// z = round_s(qp + kz) (RECOMPUTE / forward) or the stashed z
template <typename T>
__device__ __forceinline__ float z_of(float qp, float kz, bool add_qp) {
  return add_qp ? St<T>::round(__fadd_rn(qp, kz)) : kz;
}

// partial score over this CTA's A slice for one position (one warp; lanes over 4-column groups)
template <typename T>
__device__ __forceinline__ float score_partial(const T* kz_row, const T* qps, const T* vs, int W, int lane,
                                               bool add_qp, T* z_out, float* e_out) {
  float acc = 0.0f;
  for (int c4 = lane; c4 < W / 4; c4 += 32) {
    float kz[4], q[4], vv[4], z[4], e[4];
    lds4(kz_row + c4 * 4, kz);
    if (add_qp) lds4(qps + c4 * 4, q);
    lds4(vs + c4 * 4, vv);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      z[k] = z_of<T>(add_qp ? q[k] : 0.0f, kz[k], add_qp);
      e[k] = att_tanh<T>(z[k]);
      acc = __fmaf_rn(e[k], vv[k], acc);
    }
    if (z_out) stg4(z_out + c4 * 4, z);
    if (e_out) *reinterpret_cast<float4*>(e_out + c4 * 4) = make_float4(e[0], e[1], e[2], e[3]);
  }
  return warp_sum(acc);
}

// score_partial for the TMA kernels, whose column slices are <= 128 wide (W / 4 <= 32: one 4-column
// group per lane): the lane's qp / v values are loaded into registers once per CTA instead of once
// per position.  Same operations in the same order as score_partial (bit-identical).
template <typename T>
__device__ __forceinline__ float score_partial_r(const T* kz_row, const float (&qr)[4], const float (&vr)[4], bool act,
                                                 int c4, bool add_qp, T* z_out, float* e_out) {
  float acc = 0.0f;
  if (act) {
    float kz[4], z[4], e[4];
    lds4(kz_row + c4 * 4, kz);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      z[k] = z_of<T>(add_qp ? qr[k] : 0.0f, kz[k], add_qp);
      e[k] = att_tanh<T>(z[k]);
      acc = __fmaf_rn(e[k], vr[k], acc);
    }
    if (z_out) stg4(z_out + c4 * 4, z);
    if (e_out) *reinterpret_cast<float4*>(e_out + c4 * 4) = make_float4(e[0], e[1], e[2], e[3]);
  }
  return warp_sum(acc);
}

// score_partial_r for bf16 storage with z = qp + Kp formed by packed bf16x2 adds (add.rn.bf16x2:
// the exact sum rounded once to bf16).  Equal to z_of<bf16> = round_bf16(fp32(qp) + fp32(kz)): both
// operands are bf16, so their fp32 sum is exact unless the exponents differ by more than 15, and then
// the smaller one is below 2^-15 of the larger, far from any bf16 rounding midpoint -- both round to
// the larger operand.  Same E, same FMA order: bit-identical, 2.5 fewer instructions per element.
__device__ __forceinline__ float score_partial_bf2(const __nv_bfloat16* kz_row, const uint2& q2, const float (&vr)[4],
                                                   bool act, int c4, __nv_bfloat16* z_out) {
  float acc = 0.0f;
  if (act) {
    const uint2 k2 = *reinterpret_cast<const uint2*>(kz_row + c4 * 4);
    const __nv_bfloat162 za = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&q2.x),
                                      *reinterpret_cast<const __nv_bfloat162*>(&k2.x));
    const __nv_bfloat162 zb = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&q2.y),
                                      *reinterpret_cast<const __nv_bfloat162*>(&k2.y));
    const float2 ea = att_tanh2_bf16(__bfloat1622float2(za)), eb = att_tanh2_bf16(__bfloat1622float2(zb));
    acc = __fmaf_rn(ea.x, vr[0], acc);
    acc = __fmaf_rn(ea.y, vr[1], acc);
    acc = __fmaf_rn(eb.x, vr[2], acc);
    acc = __fmaf_rn(eb.y, vr[3], acc);
    if (z_out) {
      uint2 u;
      *reinterpret_cast<__nv_bfloat162*>(&u.x) = za;
      *reinterpret_cast<__nv_bfloat162*>(&u.y) = zb;
      *reinterpret_cast<uint2*>(z_out + c4 * 4) = u;
    }
  }
  return warp_sum(acc);
}

// Per-lane partials of GR row slots -> full warp sums with log2(GR) halving exchanges (each lane
// keeps the half of its slots picked by one lane bit) and 5 - log2(GR) butterflies: GR - 1 + 5 -
// log2(GR) shuffles instead of 5 GR.  Every slot's sum is formed by the SAME pairwise tree as
// warp_sum (partners at xor 16, 8, 4, 2, 1, IEEE addition commutes), so it is bitwise equal to
// warp_sum of that slot.  Returns the sum of slot lane >> (5 - log2(GR)).
template <int GR>
__device__ __forceinline__ float reduce_scatter(float (&p)[GR], int lane) {
  static_assert(GR == 2 || GR == 4 || GR == 8, "GR");
  constexpr int LG = GR == 2 ? 1 : GR == 4 ? 2 : 3;
#pragma unroll
  for (int st = 0, n = GR; st < LG; ++st) {
    const int o = 16 >> st;
    const bool hi = (lane & o) != 0;
    n >>= 1;
#pragma unroll
    for (int i = 0; i < GR / 2; ++i)
      if (i < n) {
        const float send = hi ? p[i] : p[i + n];
        const float keep = hi ? p[i + n] : p[i];
        p[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
      }
  }
  float x = p[0];
#pragma unroll
  for (int o = 16 >> LG; o > 0; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// rank-ordered gather of the C partial vectors part_c[0..n) into out[0..n)
__device__ __forceinline__ void gather_sum(cg::cluster_group& cl, float* part, float* out, int n, int C, int tid) {
  for (int s = tid; s < n; s += ATT_THREADS) {
    float t[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) t[c] = c < C ? cl.map_shared_rank(part, c)[s] : 0.0f;
    float x = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < C) x = __fadd_rn(x, t[c]);
    out[s] = x;
  }
}

// softmax of sc[0..n) into al[0..n) by ONE warp (max-subtracted, fixed order)
// (TMA kernels: n <= 256, so each lane keeps its <= 8 exponentials in registers between the sum and
// the normalisation instead of evaluating expf twice; same values, same order)
__device__ __forceinline__ void softmax_row_warp(const float* sc, float* al, int n, int lane) {
  float m = -INFINITY;
  for (int s = lane; s < n; s += 32) m = fmaxf(m, sc[s]);
  m = warp_max(m);
  float l = 0.0f, ev[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int s = lane + 32 * k;
    ev[k] = s < n ? expf(__fsub_rn(sc[s], m)) : 0.0f;
    if (s < n) l = __fadd_rn(l, ev[k]);
  }
  l = warp_sum(l);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int s = lane + 32 * k;
    if (s < n) al[s] = __fdiv_rn(ev[k], l);
  }
}

// ctx columns of this CTA: one thread per column; positions are split round-robin over four
// accumulators (s mod 4) for ILP and combined in fixed order ((a0 + a1) + (a2 + a3)).
template <typename T>
__device__ __forceinline__ void ctx_columns(const T* hs_s, int ld, int WH, const float* al, int n, T* ctx_out, int tid) {
  for (int c = tid; c < WH; c += ATT_THREADS) {
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    int s = 0;
    for (; s + 4 <= n; s += 4) {
      a0 = __fmaf_rn(al[s], to_f(hs_s[(s + 0) * ld + c]), a0);
      a1 = __fmaf_rn(al[s + 1], to_f(hs_s[(s + 1) * ld + c]), a1);
      a2 = __fmaf_rn(al[s + 2], to_f(hs_s[(s + 2) * ld + c]), a2);
      a3 = __fmaf_rn(al[s + 3], to_f(hs_s[(s + 3) * ld + c]), a3);
    }
    if (s < n) a0 = __fmaf_rn(al[s], to_f(hs_s[s * ld + c]), a0);
    if (s + 1 < n) a1 = __fmaf_rn(al[s + 1], to_f(hs_s[(s + 1) * ld + c]), a1);
    if (s + 2 < n) a2 = __fmaf_rn(al[s + 2], to_f(hs_s[(s + 2) * ld + c]), a2);
    ctx_out[c] = from_f<T>(St<T>::round(__fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3))));
  }
}

template <typename T>
__device__ __forceinline__ void stage_slice(float* dst, const T* __restrict__ src, int n, int tid) {
  for (int i = tid; i < n; i += ATT_THREADS) dst[i] = to_f(src[i]);
}

// ---- tensor-map TMA (cp.async.bulk.tensor) helpers
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// L2 eviction policies: the attention tensors every decoder step re-reads (Kp, H_s) and
// read-modify-writes (dKp, dH_s) can be marked evict_last so they stay resident across steps
__device__ __forceinline__ uint64_t l2_policy(bool last) {
  uint64_t p;
  if (last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ float4 ldg4_hint(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg4_hint(float* p, const float (&v)[4], uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(p), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile.L2::cache_hint [%0, {%1, %2, %3}], %4;\n" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ size_t al128(size_t b) { return (b + 127) & ~(size_t)127; }

// The row slice is staged in up to TMA_CHUNKS chunks of R positions, one mbarrier each, so phase 1
// starts on the first chunk while the rest is in flight; chunks that start at or beyond the row's
// length n are never loaded.  R = ceil(Ts / TMA_CHUNKS) rounded up so that every chunk's shared
// destination stays 128-byte aligned (R * row bytes a multiple of 128 for both tiles); the tiles
// hold Tr = R * ceil(Ts / R) rows (the last box may extend past Ts: TMA zero-fills those rows).
constexpr int TMA_CHUNKS = 4;
static __host__ __device__ __forceinline__ int pow2_gap128(int bytes) {   // 128 / gcd(bytes, 128)
  int m = 1;
  while ((bytes * m) % 128) m <<= 1;
  return m;
}
static __host__ __device__ __forceinline__ int tma_rows(int Ts, int Wb, int WHb, int es) {
  const int m1 = pow2_gap128(Wb * es), m2 = pow2_gap128(WHb * es);
  const int m = m1 > m2 ? m1 : m2;
  const int r = (Ts + TMA_CHUNKS - 1) / TMA_CHUNKS;
  return (r + m - 1) / m * m;
}
static __host__ __device__ __forceinline__ int tma_tile_rows(int Ts, int R) { return (Ts + R - 1) / R * R; }

struct SmallCopy {     // contiguous vectors staged with chunk 0 (qp / v / dctx slices)
  void* dst[3];
  const void* src[3];
  uint32_t bytes[3];   // 0 = not staged
};
__device__ __forceinline__ void issue_chunks(uint64_t* bar, int n, int R, void* kz, const CUtensorMap* mK, int a0,
                                             void* hs, const CUtensorMap* mH, int h0, int b, uint32_t rowK,
                                             uint32_t rowH, const SmallCopy& sm, uint64_t pol) {
  // one arrive.expect_tx per barrier (count 1): chunk 0's also covers the small vectors.  Chunk 0
  // (always needed: n >= 1) goes out before n is used, so the src_len load overlaps its issue.
  mbar_expect_tx(&bar[0], sm.bytes[0] + sm.bytes[1] + sm.bytes[2] + (uint32_t)R * (rowK + rowH));
  tma_load_3d_hint(kz, mK, a0, b, 0, &bar[0], pol);
  tma_load_3d_hint(hs, mH, h0, b, 0, &bar[0], pol);
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (sm.bytes[i]) bulk_load(sm.dst[i], sm.src[i], sm.bytes[i], &bar[0]);
  const int nch = (n + R - 1) / R;
  for (int k = 1; k < nch; ++k) {
    mbar_expect_tx(&bar[k], (uint32_t)R * (rowK + rowH));
    tma_load_3d_hint(static_cast<unsigned char*>(kz) + (size_t)k * R * rowK, mK, a0, b, k * R, &bar[k], pol);
    tma_load_3d_hint(static_cast<unsigned char*>(hs) + (size_t)k * R * rowH, mH, h0, b, k * R, &bar[k], pol);
  }
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(m) : "memory");
}

// ---- DSMEM push exchange (no cluster-wide barrier on the data path): each CTA sends its partial
// scores into every cluster CTA's receive buffer with st.async, completing on the receiver's
// mbarrier (expect_tx set at kernel entry, before the single start-up cluster barrier).
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(remote_addr),
               "r"(__float_as_uint(v)), "r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t remote_addr, float x, float y, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];\n" ::"r"(remote_addr),
               "r"(__float_as_uint(x)), "r"(__float_as_uint(y)), "r"(remote_bar)
               : "memory");
}

// Shared-memory tiles: [Tr][box width] per tensor for this CTA's column slice.
// Forward, no data-path cluster barrier: after phase 1 every warp holds its positions' partial
// scores and pushes them (st.async) into the C receive rows xpart[rank][*] of every cluster CTA;
// each CTA waits on its own exchange mbarrier, and EVERY warp then forms the scores in rank order
// (the gather_sum arithmetic), runs the softmax in registers (the softmax_row_warp arithmetic) and
// the ctx warps read alpha_s by shuffle (the ctx_columns arithmetic) -- so alpha and ctx are bit-
// identical to the backward's regenerated ones, with no __syncthreads / cluster barrier after the
// start-up one that publishes the mbarrier initialisation.
template <typename T>
__global__ void __launch_bounds__(ATT_THREADS, sizeof(T) == 2 ? 8 : 1) attn_fwd_tma(echo_attn_desc d, TmaGeo q,
                                                            const __grid_constant__ CUtensorMap mK,
                                                            const __grid_constant__ CUtensorMap mH,
                                                            const T* __restrict__ qp, const T* __restrict__ v,
                                                            const int32_t* __restrict__ src_len, T* __restrict__ ctx,
                                                            T* __restrict__ Z_st, float* __restrict__ alpha_st) {
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(128) unsigned char smraw[];   // TMA (no swizzle) needs 128-B alignment
  __shared__ __align__(8) uint64_t bar[TMA_CHUNKS];
  __shared__ __align__(8) uint64_t xbar;
  const int A = d.A, Ts = d.Ts, Hk = d.Hk;
  const int rank = (int)cl.block_rank();
  const Slice g = make_slice_g(q, A, Hk, rank);
  const int W = g.a1 - g.a0, WH = g.h1 - g.h0;               // valid widths
  const int Wb = q.Wb, WHb = q.WHb;                           // box widths (smem row strides)
  const int Tp = (Ts + 3) & ~3;
  const int R = q.R, Tr = q.Tr, C = q.C;
  T* kz = reinterpret_cast<T*>(smraw);                                         // [Tr][Wb]
  T* hs = reinterpret_cast<T*>(smraw + al128((size_t)Tr * Wb * sizeof(T)));    // [Tr][WHb]
  T* qps = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(hs) + al128((size_t)Tr * WHb * sizeof(T)));
  T* vs = qps + Wb;                                                            // Wb * sizeof(T) is 16-B aligned
  float* xpart = reinterpret_cast<float*>(vs + Wb);                            // [C][Tp] received partials
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = row_len(src_len, b, Ts);
  const uint64_t pol = l2_policy(q.l2last);
  if (tid == 0) {
    prefetch_tmap(&mK);
    prefetch_tmap(&mH);
    for (int k = 0; k < TMA_CHUNKS; ++k) mbar_init(&bar[k], 1);
    // C > 1: n partial scores arrive from each of the C CTAs as st.async bytes; C == 1 (no DSMEM
    // transactions in a one-CTA cluster): each position's lane 0 stores locally and arrives once
    mbar_init(&xbar, C > 1 ? 1 : n + 1);
    fence_mbar_init();
    mbar_expect_tx(&xbar, C > 1 ? (uint32_t)(C * n * 4) : 0u);
    SmallCopy sm{{qps, vs, nullptr}, {qp + (long)b * A + g.a0, v + g.a0, nullptr},
                 {(uint32_t)(W * sizeof(T)), (uint32_t)(W * sizeof(T)), 0u}};
    issue_chunks(bar, n, R, kz, &mK, g.a0, hs, &mH, g.h0, b, Wb * sizeof(T), WHb * sizeof(T), sm, pol);
  }
  __syncthreads();                                            // barrier init visible before anyone waits
  cluster_arrive_relaxed();                                   // publishes xbar's init (fenced above)
  mbar_wait(&bar[0], 0);                                      // chunk 0 + the qp / v slices
  const bool act = lane < W / 4;                              // W <= 128: one column group per lane
  float qr[4] = {0.0f, 0.0f, 0.0f, 0.0f}, vr[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  uint2 q2 = make_uint2(0u, 0u);                              // bf16: the lane's qp slice, packed
  if (act) {
    lds4(qps + lane * 4, qr);
    lds4(vs + lane * 4, vr);
    if constexpr (sizeof(T) == 2) q2 = *reinterpret_cast<const uint2*>(qps + lane * 4);
  }
  cluster_wait();                                             // every CTA's xbar is initialised
  // lane c < C delivers the warp's partial to cluster CTA c (row `rank` of its receive buffer)
  const uint32_t dst_row = C > 1 ? mapa_u32(smem_u32(xpart + rank * Tp), lane < C ? lane : 0) : 0u;
  const uint32_t dst_bar = C > 1 ? mapa_u32(smem_u32(&xbar), lane < C ? lane : 0) : 0u;
  if (!Z_st && W == 4 * 32) {
    // RECOMPUTE with a full 128-column slice (every lane active): two positions per iteration, the K row
    // addressed with 32-bit shared addresses, no per-lane branch -- the same per-position arithmetic
    // (z, tanh, FMA order, warp_sum tree) as score_partial_bf2 / score_partial_r, fewer instructions
    const uint32_t kz_s = smem_u32(kz) + (uint32_t)(lane * 4 * sizeof(T)), rowb = (uint32_t)(Wb * sizeof(T));
    auto part = [&](int s) -> float {
      float acc = 0.0f;
      if constexpr (sizeof(T) == 2) {
        uint32_t k0, k1;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(k0), "=r"(k1) : "r"(kz_s + (uint32_t)s * rowb));
        const __nv_bfloat162 za = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&q2.x),
                                          *reinterpret_cast<const __nv_bfloat162*>(&k0));
        const __nv_bfloat162 zb = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&q2.y),
                                          *reinterpret_cast<const __nv_bfloat162*>(&k1));
        const float2 ea = att_tanh2_bf16(__bfloat1622float2(za)), eb = att_tanh2_bf16(__bfloat1622float2(zb));
        acc = __fmaf_rn(ea.x, vr[0], acc);
        acc = __fmaf_rn(ea.y, vr[1], acc);
        acc = __fmaf_rn(eb.x, vr[2], acc);
        acc = __fmaf_rn(eb.y, vr[3], acc);
      } else {
        float4 kv;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(kv.x), "=f"(kv.y), "=f"(kv.z), "=f"(kv.w)
                     : "r"(kz_s + (uint32_t)s * rowb));
        const float kz4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = __fmaf_rn(att_tanh<T>(z_of<T>(qr[q], kz4[q], true)), vr[q], acc);
      }
      return acc;
    };
    auto send = [&](int s, float p) {
      if (C > 1) {
        if (lane < C) st_async_f32(dst_row + 4u * (uint32_t)s, p, dst_bar);
      } else if (lane == 0) {
        xpart[s] = p;
        mbar_arrive(&xbar);
      }
    };
    for (int k = 0, s = w; k * R < n; ++k) {
      const int s1 = min(n, (k + 1) * R);
      if (s >= s1) continue;
      mbar_wait(&bar[k], 0);
      for (; s + ATT_WARPS < s1; s += 2 * ATT_WARPS) {
        const float a0 = part(s), a1 = part(s + ATT_WARPS);
        const float p0 = warp_sum(a0), p1 = warp_sum(a1);
        send(s, p0);
        send(s + ATT_WARPS, p1);
      }
      if (s < s1) {
        send(s, warp_sum(part(s)));
        s += ATT_WARPS;
      }
    }
  } else
  for (int k = 0, s = w; k * R < n; ++k) {                   // chunk by chunk: one wait per chunk
    const int s1 = min(n, (k + 1) * R);
    if (s >= s1) continue;
    mbar_wait(&bar[k], 0);
    for (; s < s1; s += ATT_WARPS) {
      T* z_out = Z_st ? Z_st + ((long)b * Ts + s) * A + g.a0 : nullptr;
      float p;
      if constexpr (sizeof(T) == 2)
        p = score_partial_bf2(reinterpret_cast<const __nv_bfloat16*>(kz) + (size_t)s * Wb, q2, vr, act, lane,
                              reinterpret_cast<__nv_bfloat16*>(z_out));
      else
        p = score_partial_r<T>(kz + (size_t)s * Wb, qr, vr, act, lane, true, z_out, nullptr);
      if (C > 1) {
        if (lane < C) st_async_f32(dst_row + 4u * (uint32_t)s, p, dst_bar);
      } else if (lane == 0) {
        xpart[s] = p;
        mbar_arrive(&xbar);
      }
    }
  }
  if (Z_st) {                                                 // masked positions: zeros in this slice
    float z[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int s = n + w; s < Ts; s += ATT_WARPS)
      for (int c4 = lane; c4 < W / 4; c4 += 32) stg4(Z_st + ((long)b * Ts + s) * A + g.a0 + c4 * 4, z);
  }
  const bool ctx_warp = w * 64 < WH;                          // ctx: one thread per column pair
  if (!ctx_warp && !(alpha_st && rank == 0 && w == 0)) return;
  mbar_wait(&xbar, 0);                                        // all C partial rows received
  // scores (rank-ordered sum, = gather_sum) and softmax (= softmax_row_warp) for s = lane + 32 k
  float sc[8];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int s = lane + 32 * k;
    float x = 0.0f;
    if (s < n) {
      for (int c = 0; c < C; ++c) x = __fadd_rn(x, xpart[c * Tp + s]);
      m = fmaxf(m, x);
    }
    sc[k] = x;
  }
  m = warp_max(m);
  float l = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int s = lane + 32 * k;
    sc[k] = s < n ? expf(__fsub_rn(sc[k], m)) : 0.0f;
    if (s < n) l = __fadd_rn(l, sc[k]);
  }
  l = warp_sum(l);
#pragma unroll
  for (int k = 0; k < 8; ++k) sc[k] = lane + 32 * k < n ? __fdiv_rn(sc[k], l) : 0.0f;   // alpha
  if (alpha_st && rank == 0 && w == 0)
    for (int k = 0; k < 8; ++k)
      if (lane + 32 * k < Ts) alpha_st[(long)b * Ts + lane + 32 * k] = sc[k];
  if (!ctx_warp) return;
  for (int k = 0; k * R < n; ++k) mbar_wait(&bar[k], 0);     // every H_s chunk landed
  // ctx_columns with alpha_s taken from lane s % 32 of register sc[s / 32], two adjacent columns per
  // thread (one 2-element shared load and one shuffle per position serve both): per column the same
  // FMAs into the same four accumulators (s mod 4) in the same order, so ctx is bit-identical to
  // ctx_columns'
  const int c = 2 * tid;
  const bool cok = c < WH;                                    // WH is even (a multiple of 8)
  const T* hcol = hs + c;
  float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f, b0 = 0.0f, b1 = 0.0f, b2 = 0.0f, b3 = 0.0f;
  auto h2 = [&](int s) -> float2 {
    if constexpr (sizeof(T) == 2) return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(hcol + s * WHb));
    else return *reinterpret_cast<const float2*>(hcol + s * WHb);
  };
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (32 * k >= n) break;
    const float ak = sc[k];
    for (int j = 0; j < 32; j += 4) {
      const int s0 = 32 * k + j;
      if (s0 >= n) break;
      const float al0 = __shfl_sync(0xffffffffu, ak, j), al1 = __shfl_sync(0xffffffffu, ak, j + 1);
      const float al2 = __shfl_sync(0xffffffffu, ak, j + 2), al3 = __shfl_sync(0xffffffffu, ak, j + 3);
      if (cok) {
        float2 x = h2(s0);
        a0 = __fmaf_rn(al0, x.x, a0);
        b0 = __fmaf_rn(al0, x.y, b0);
        if (s0 + 1 < n) { x = h2(s0 + 1); a1 = __fmaf_rn(al1, x.x, a1); b1 = __fmaf_rn(al1, x.y, b1); }
        if (s0 + 2 < n) { x = h2(s0 + 2); a2 = __fmaf_rn(al2, x.x, a2); b2 = __fmaf_rn(al2, x.y, b2); }
        if (s0 + 3 < n) { x = h2(s0 + 3); a3 = __fmaf_rn(al3, x.x, a3); b3 = __fmaf_rn(al3, x.y, b3); }
      }
    }
  }
  if (cok) {
    const float ya = St<T>::round(__fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3)));
    const float yb = St<T>::round(__fadd_rn(__fadd_rn(b0, b1), __fadd_rn(b2, b3)));
    T* o = ctx + (long)b * Hk + g.h0 + c;
    o[0] = from_f<T>(ya);
    o[1] = from_f<T>(yb);
  }
}

// ---- a5, persistent row-streaming variant (large B).  One CTA (ROWS_PER_SM per SM)
// walks rows b = blockIdx.x, + gridDim.x, ...; a producer warp streams each row's Kp positions and
// then its H_s positions through a ring of shared stages (TMA, R positions x all C column slices
// per stage, full / empty mbarriers), so HBM reads run continuously under the score, softmax and
// ctx phases of the previous stages -- no cluster, no DSMEM, no per-row launch / start-up latency.
// The arithmetic is attn_fwd_tma's, element for element: lane l of a warp evaluates the same four
// columns r*Wb + 4l of every slice r with the same FMA order, the slice partials are the same
// warp_sum trees (reduce_scatter, bitwise equal), added in rank order from 0; the softmax and the
// s-mod-4 ctx accumulators are the same code -- so ctx / Z / alpha are bit-identical to the cluster
// kernel's and to a6's regenerated ones (tests/test_gpu_attention.py checks both).
#ifndef ECHO_ROWS_CWARPS
#define ECHO_ROWS_CWARPS 4
#endif
constexpr int ROWS_CWARPS = ECHO_ROWS_CWARPS;                 // consumer warps
constexpr int ROWS_THREADS = (ROWS_CWARPS + 1) * 32;          // + one producer warp
constexpr int ROWS_PER_SM = ROWS_CWARPS == 4 ? 4 : 2;         // resident CTAs per SM
constexpr int ROWS_MAXPJ = 4;                                 // ctx column pairs per thread (Hk <= 8 * 32 * CWARPS)
constexpr int ROWS_MAXST = 8;
struct RowGeo {
  int C, Wb, WHb, R, nst;       // slices (as TmaGeo), positions per stage (8 | 16 | 32), ring stages
  uint32_t sub, stage;          // bytes per slice sub-tile (128-aligned) and per stage (+ the qp row)
};
static __host__ __device__ __forceinline__ size_t rows_tail_bytes(int Ts, int C) {   // xs + al_s
  return 4 * (size_t)(((Ts * C + 3) & ~3) + Ts + 8);
}
__device__ __forceinline__ void bar_sync_consumers() { asm volatile("bar.sync 1, %0;\n" ::"n"(ROWS_CWARPS * 32) : "memory"); }

// (with a suspend-time hint: a waiting thread sleeps until the phase completes instead of re-polling)
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t phase) { mbar_wait_bounded<10000000>(bar, phase); }
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// bf16x2 word -> two floats (exact: a bf16 is the high half of its fp32)
__device__ __forceinline__ float2 bf2_to_f2(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}
// ring position: slot and phase advance together (no division by the stage count)
struct RingPos {
  int slot;
  uint32_t phase;
  __device__ __forceinline__ void next(int nst) {
    if (++slot == nst) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

template <typename T, int CT, bool STASH>
__global__ void __launch_bounds__(ROWS_THREADS, ROWS_PER_SM) attn_fwd_rows(echo_attn_desc d, RowGeo q,
                                                                   const __grid_constant__ CUtensorMap mK,
                                                                   const __grid_constant__ CUtensorMap mH,
                                                                   const T* __restrict__ qp, const T* __restrict__ v,
                                                                   const int32_t* __restrict__ src_len, T* __restrict__ ctx,
                                                                   T* __restrict__ Z_st, float* __restrict__ alpha_st) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[ROWS_MAXST], empty[ROWS_MAXST];
  // after the ring: slice partials xs[s][slice] and alpha al_s[s] of the current row (+ tail-read pad)
  float* xs = reinterpret_cast<float*>(smraw + (size_t)q.nst * q.stage);
  float* al_s = xs + ((d.Ts * CT + 3) & ~3);
  const int A = d.A, Ts = d.Ts, Hk = d.Hk, Wb = q.Wb, WHb = q.WHb, R = q.R, NST = q.nst;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int k = 0; k < NST; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], ROWS_CWARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty), sm0 = smem_u32(smraw);
  if (w == ROWS_CWARPS) {                                     // ---- producer (one thread)
    if (lane) return;
    prefetch_tmap(&mK);
    prefetch_tmap(&mH);
    const uint64_t pol = l2_policy(false);
    RingPos rp{0, 0u};
    for (int b = blockIdx.x; b < d.B; b += gridDim.x) {
      const int n = row_len(src_len, b, Ts), nch = (n + R - 1) / R;
      for (int pass = 0; pass < 2; ++pass) {
        const int X = pass ? Hk : A, Wx = pass ? WHb : Wb;
        const CUtensorMap* m = pass ? &mH : &mK;
        for (int k = 0; k < nch; ++k, rp.next(NST)) {
          mbar_wait_u32(empty0 + 8u * rp.slot, rp.phase ^ 1u);
          unsigned char* st = smraw + (size_t)rp.slot * q.stage;
          const bool first = pass == 0 && k == 0;
          uint32_t bytes = first ? (uint32_t)(A * sizeof(T)) : 0u;
#pragma unroll
          for (int r = 0; r < CT; ++r)
            if (r * Wx < X) bytes += (uint32_t)(R * Wx * sizeof(T));
          mbar_expect_tx(&full[rp.slot], bytes);
#pragma unroll
          for (int r = 0; r < CT; ++r)
            if (r * Wx < X) tma_load_3d_hint(st + r * q.sub, m, r * Wx, b, k * R, &full[rp.slot], pol);
          if (first) bulk_load(st + CT * q.sub, qp + (long)b * A, (uint32_t)(A * sizeof(T)), &full[rp.slot]);
        }
      }
    }
    return;
  }
  // ---- consumers (warps 0 .. ROWS_CWARPS-1)
  bool act[CT];
  uint32_t lk[CT];                                            // lane byte offset in a slice row (0 if inactive)
  float vr[CT][4];
#pragma unroll
  for (int r = 0; r < CT; ++r) {
    const int a0 = min(A, r * Wb), W = min(A, a0 + Wb) - a0;
    act[r] = lane < W / 4;
    lk[r] = act[r] ? (uint32_t)(lane * 4 * sizeof(T)) : 0u;
    if (act[r]) lds4(v + a0 + lane * 4, vr[r]);              // (lds4: a plain 4-element load, here from global)
    else vr[r][0] = vr[r][1] = vr[r][2] = vr[r][3] = 0.0f;
  }
  constexpr int LG = CT == 1 ? 0 : CT == 2 ? 1 : CT == 4 ? 2 : 3;
  constexpr bool PAIRS = CT <= 4;                             // two positions per reduce_scatter (<= 8 slots)
  const uint32_t rowK = (uint32_t)(Wb * sizeof(T)), rowH = (uint32_t)(WHb * sizeof(T));
  // ctx: consumer thread t owns column pairs t, t + 32 ROWS_CWARPS, ... (two adjacent columns each)
  const int NPJ = (Hk / 2 + ROWS_CWARPS * 32 - 1) / (ROWS_CWARPS * 32);   // <= ROWS_MAXPJ
  uint32_t off[ROWS_MAXPJ];
  bool pok[ROWS_MAXPJ];
#pragma unroll
  for (int j = 0; j < ROWS_MAXPJ; ++j) {
    const int c = 2 * (tid + j * ROWS_CWARPS * 32);
    pok[j] = j < NPJ && c < Hk;
    const int r = pok[j] ? c / WHb : 0, cc = pok[j] ? c - r * WHb : 0;
    off[j] = (uint32_t)r * q.sub + (uint32_t)(cc * sizeof(T));
  }
  RingPos rp{0, 0u};
  // xs / al_s reuse across rows: a warp writes row b+1's xs only after the second barrier of row b (warp
  // 0's softmax has read row b's xs), and warp 0 writes row b+1's alpha only after the first barrier of
  // row b+1 (every warp has finished row b's ctx)
  for (int b = blockIdx.x; b < d.B; b += gridDim.x) {
    const int n = row_len(src_len, b, Ts), nch = (n + R - 1) / R;
    uint2 q2[CT];
    float qr[CT][4];
    // slice partial of position i of the stage at sb: attn_fwd_tma's per-lane arithmetic, evaluated
    // branch-free (an inactive lane reads its slice's first element and contributes 0, as it does there)
    auto part = [&](uint32_t sb, int r, int i, int s) -> float {
      const uint32_t a = sb + (uint32_t)r * q.sub + (uint32_t)i * rowK + lk[r];
      float acc = 0.0f;
      if constexpr (sizeof(T) == 2) {
        uint32_t k0, k1;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(k0), "=r"(k1) : "r"(a));
        const __nv_bfloat162 za = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&q2[r].x),
                                          *reinterpret_cast<const __nv_bfloat162*>(&k0));
        const __nv_bfloat162 zb = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&q2[r].y),
                                          *reinterpret_cast<const __nv_bfloat162*>(&k1));
        const uint32_t ua = *reinterpret_cast<const uint32_t*>(&za), ub = *reinterpret_cast<const uint32_t*>(&zb);
        const float2 ea = att_tanh2_bf16(bf2_to_f2(ua)), eb = att_tanh2_bf16(bf2_to_f2(ub));
        acc = __fmaf_rn(ea.x, vr[r][0], acc);
        acc = __fmaf_rn(ea.y, vr[r][1], acc);
        acc = __fmaf_rn(eb.x, vr[r][2], acc);
        acc = __fmaf_rn(eb.y, vr[r][3], acc);
        if constexpr (STASH) {
          if (act[r]) *reinterpret_cast<uint2*>(Z_st + ((long)b * Ts + s) * A + r * Wb + lane * 4) = make_uint2(ua, ub);
        }
      } else {
        float4 kv;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(kv.x), "=f"(kv.y), "=f"(kv.z), "=f"(kv.w) : "r"(a));
        const float kz4[4] = {kv.x, kv.y, kv.z, kv.w};
        float z[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          z[c] = z_of<T>(qr[r][c], kz4[c], true);
          acc = __fmaf_rn(att_tanh<T>(z[c]), vr[r][c], acc);
        }
        if constexpr (STASH) {
          if (act[r]) stg4(Z_st + ((long)b * Ts + s) * A + r * Wb + lane * 4, z);
        }
      }
      return act[r] ? acc : 0.0f;
    };
    // phase 1: per-slice warp sums (reduce_scatter: bitwise warp_sum) into xs[s][r]
    for (int k = 0; k < nch; ++k, rp.next(NST)) {
      mbar_wait_u32(full0 + 8u * rp.slot, rp.phase);
      const uint32_t sb = sm0 + (uint32_t)rp.slot * q.stage;
      if (k == 0) {
        const T* qrow = reinterpret_cast<const T*>(smraw + (size_t)rp.slot * q.stage + CT * q.sub);
#pragma unroll
        for (int r = 0; r < CT; ++r) {
          if (act[r]) {
            lds4(qrow + r * Wb + lane * 4, qr[r]);
            if constexpr (sizeof(T) == 2) q2[r] = *reinterpret_cast<const uint2*>(qrow + r * Wb + lane * 4);
          } else {
            q2[r] = make_uint2(0u, 0u);
            qr[r][0] = qr[r][1] = qr[r][2] = qr[r][3] = 0.0f;
          }
        }
      }
      const int s1 = min(n, (k + 1) * R);
      int s = k * R + w;
      if constexpr (PAIRS) {
        for (; s + ROWS_CWARPS < s1; s += 2 * ROWS_CWARPS) {
          float p[2 * CT];
#pragma unroll
          for (int r = 0; r < CT; ++r) {
            p[r] = part(sb, r, s - k * R, s);
            p[CT + r] = part(sb, r, s + ROWS_CWARPS - k * R, s + ROWS_CWARPS);
          }
          const float ps = reduce_scatter<2 * CT>(p, lane);
          constexpr int LG2 = LG + 1;
          const int g = lane >> (5 - LG2);                    // slot g = position (g / CT), slice g % CT
          if ((lane & ((32 >> LG2) - 1)) == 0) xs[(s + (g / CT) * ROWS_CWARPS) * CT + g % CT] = ps;
        }
      }
      for (; s < s1; s += ROWS_CWARPS) {
        float p[CT];
#pragma unroll
        for (int r = 0; r < CT; ++r) p[r] = part(sb, r, s - k * R, s);
        if constexpr (CT == 1) {
          const float ps = warp_sum(p[0]);
          if (lane == 0) xs[s] = ps;
        } else {
          const float ps = reduce_scatter<CT>(p, lane);
          if ((lane & ((32 >> LG) - 1)) == 0) xs[s * CT + (lane >> (5 - LG))] = ps;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(empty0 + 8u * rp.slot);
    }
    if constexpr (STASH) {                                    // masked positions: zeros
      float z[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int s = n + w; s < Ts; s += ROWS_CWARPS)
        for (int c4 = lane; c4 < A / 4; c4 += 32) stg4(Z_st + ((long)b * Ts + s) * A + c4 * 4, z);
    }
    bar_sync_consumers();                                     // every partial of row b is in xs
    // warp 0: scores in rank order from 0 (the xpart gather) and the softmax (attn_fwd_tma's register
    // code, same operations and order) -> al_s; the other warps wait at the second barrier
    if (w == 0) {
      float scr[8];
      float m = -INFINITY;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int s = lane + 32 * k;
        float x = 0.0f;
        if (s < n) {
#pragma unroll
          for (int r = 0; r < CT; ++r) x = __fadd_rn(x, xs[s * CT + r]);
          m = fmaxf(m, x);
        }
        scr[k] = x;
      }
      m = warp_max(m);
      float l = 0.0f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int s = lane + 32 * k;
        scr[k] = s < n ? expf(__fsub_rn(scr[k], m)) : 0.0f;
        if (s < n) l = __fadd_rn(l, scr[k]);
      }
      l = warp_sum(l);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int s = lane + 32 * k;
        const float a = s < n ? __fdiv_rn(scr[k], l) : 0.0f;
        if (s < Ts + 8) al_s[s] = a;
        if (STASH && s < Ts) alpha_st[(long)b * Ts + s] = a;
      }
    }
    bar_sync_consumers();                                     // alpha of row b is in al_s
    // ctx (ctx_columns' accumulators: one per s mod 4 and column, combined (a0 + a1) + (a2 + a3));
    // FFMA2 on the column pair = the two scalar FMAs
    float2 acc[ROWS_MAXPJ][4];
#pragma unroll
    for (int j = 0; j < ROWS_MAXPJ; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[j][e] = make_float2(0.0f, 0.0f);
    auto hld = [&](uint32_t a) -> float2 {
      if constexpr (sizeof(T) == 2) {
        uint32_t u;
        asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(u) : "r"(a));
        return bf2_to_f2(u);
      } else {
        float2 x;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(x.x), "=f"(x.y) : "r"(a));
        return x;
      }
    };
    const uint32_t al0 = smem_u32(al_s);
    {
      for (int s0 = 0; s0 < n; s0 += R, rp.next(NST)) {       // one stage per s0
        mbar_wait_u32(full0 + 8u * rp.slot, rp.phase);
        const uint32_t sb = sm0 + (uint32_t)rp.slot * q.stage;
        const int ie = min(R, n - s0);
        if (ie == R) {                                        // full stage: no per-position guards
#pragma unroll 2
          for (int i = 0; i < R; i += 4) {
            float al[4];
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(al[0]), "=f"(al[1]), "=f"(al[2]), "=f"(al[3])
                         : "r"(al0 + 4u * (uint32_t)(s0 + i)));
#pragma unroll
            for (int j = 0; j < ROWS_MAXPJ; ++j)
              if (pok[j]) {
                float2 x[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) x[e] = hld(sb + off[j] + (uint32_t)(i + e) * rowH);
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[j][e] = __ffma2_rn(make_float2(al[e], al[e]), x[e], acc[j][e]);
              }
          }
        } else {
          for (int i = 0; i < ie; i += 4) {
            float al[4];
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(al[0]), "=f"(al[1]), "=f"(al[2]), "=f"(al[3])
                         : "r"(al0 + 4u * (uint32_t)(s0 + i)));
#pragma unroll
            for (int j = 0; j < ROWS_MAXPJ; ++j)
              if (pok[j]) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (i + e < ie) acc[j][e] = __ffma2_rn(make_float2(al[e], al[e]), hld(sb + off[j] + (uint32_t)(i + e) * rowH), acc[j][e]);
              }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(empty0 + 8u * rp.slot);
      }
    }
#pragma unroll
    for (int j = 0; j < ROWS_MAXPJ; ++j)
      if (pok[j]) {
        const float ya = St<T>::round(__fadd_rn(__fadd_rn(acc[j][0].x, acc[j][1].x), __fadd_rn(acc[j][2].x, acc[j][3].x)));
        const float yb = St<T>::round(__fadd_rn(__fadd_rn(acc[j][0].y, acc[j][1].y), __fadd_rn(acc[j][2].y, acc[j][3].y)));
        T* o = ctx + (long)b * Hk + 2 * (tid + j * ROWS_CWARPS * 32);
        o[0] = from_f<T>(ya);
        o[1] = from_f<T>(yb);
      }
  }
}

// phase-4 work split: G = (W + WH)/4 column groups of four; P = ATT_THREADS / G position phases
static __host__ __device__ __forceinline__ int tma_phases(int W, int WH) { return ATT_THREADS / ((W + WH) / 4); }

// dKp / dH_s are NOT staged: phase 4 streams them through registers (16-byte vectors, rows s < n
// only), so the shared footprint is the K/Z and H_s slices alone and four CTAs fit per SM.
template <typename T>
__global__ void __launch_bounds__(ATT_THREADS, 4) attn_bwd_tma(echo_attn_desc d, TmaGeo q,
                                                               const __grid_constant__ CUtensorMap mK,
                                                               const __grid_constant__ CUtensorMap mH,
                                                               const __grid_constant__ CUtensorMap mdK,
                                                               const __grid_constant__ CUtensorMap mdH,
                                                               const T* __restrict__ qp, const T* __restrict__ v,
                                                               const int32_t* __restrict__ src_len, bool recompute,
                                                               const float* __restrict__ alpha_st,
                                                               const float* __restrict__ dctx, float* __restrict__ dqp,
                                                               float* __restrict__ dKp, float* __restrict__ dHs,
                                                               float* __restrict__ dv_part, T* __restrict__ ctx_regen,
                                                               float* __restrict__ ds_out, float* __restrict__ al_out) {
  // deferred (dKp == NULL): no dKp / dH_s read-modify-write; this step's ds (and alpha) rows go to
  // ds_out / al_out and echo_attn_bwd_finish accumulates dKp / dH_s over all steps afterwards
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(128) unsigned char smraw[];   // TMA (no swizzle) needs 128-B alignment
  __shared__ __align__(8) uint64_t bar[TMA_CHUNKS];
  __shared__ __align__(8) uint64_t xbar;
  const int A = d.A, Ts = d.Ts, Hk = d.Hk;
  const Slice g = make_slice_g(q, A, Hk, (int)cl.block_rank());
  const int W = g.a1 - g.a0, WH = g.h1 - g.h0;
  const int Wb = q.Wb, WHb = q.WHb;
  const int Tp = (Ts + 3) & ~3;
  const int P = q.P;
  const int R = q.R, Tr = q.Tr;
  // kz [Tr][Wb] T (E overwrites it in place for fp32) | hs [Tr][WHb] T | E [Tr][Wb] f32 (bf16 only)
  // | floats | phase partials [2][P][Wb] (aliased onto E when it fits)
  constexpr bool kE_ALIAS = sizeof(T) == sizeof(float);
  unsigned char* p = smraw;
  T* kz = reinterpret_cast<T*>(p);
  p += al128((size_t)Tr * Wb * sizeof(T));
  T* hs = reinterpret_cast<T*>(p);
  p += al128((size_t)Tr * WHb * sizeof(T));
  float* E = kE_ALIAS ? reinterpret_cast<float*>(kz) : reinterpret_cast<float*>(p);
  if (!kE_ALIAS) p += al128((size_t)Tr * Wb * 4);
  T* qps = reinterpret_cast<T*>(p);
  T* vs = qps + Wb;
  float* dcs = reinterpret_cast<float*>(vs + Wb);
  float* xpart = dcs + WHb;                                   // [C][Tp][2] received (score, dalpha) partials
  float* al = xpart + 2 * q.C * Tp;
  float* dsv = al + Tp;
  float* red = Tr >= 2 * P ? E : dsv + Tp;
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = row_len(src_len, b, Ts);
  const uint64_t pol = l2_policy(q.l2last);
  const int rank = (int)cl.block_rank(), C = q.C;
  ECHO_PHASE(0);
  if (tid == 0) {
    prefetch_tmap(&mK);
    prefetch_tmap(&mH);
    for (int k = 0; k < TMA_CHUNKS; ++k) mbar_init(&bar[k], 1);
    mbar_init(&xbar, C > 1 ? 1 : n + 1);                     // C == 1: local stores + arrivals (see a5)
    fence_mbar_init();
    mbar_expect_tx(&xbar, C > 1 ? (uint32_t)(C * n * 8) : 0u); // (score, dalpha) partials from each CTA
    ECHO_PHASE(11);
    SmallCopy sm{{qps, vs, dcs}, {qp + (long)b * A + g.a0, v + g.a0, dctx + (long)b * Hk + g.h0},
                 {recompute ? (uint32_t)(W * sizeof(T)) : 0u, (uint32_t)(W * sizeof(T)), (uint32_t)WH * 4u}};
    issue_chunks(bar, n, R, kz, &mK, g.a0, hs, &mH, g.h0, b, Wb * sizeof(T), WHb * sizeof(T), sm, pol);
    if (dKp && q.pf == 2)                                      // dKp / dH_s into L2 behind the stage-in
      for (int k = 0; k * R < n; ++k) {
        if (W > 0) tma_prefetch_3d(&mdK, g.a0, b, k * R, pol);
        if (WH > 0) tma_prefetch_3d(&mdH, g.h0, b, k * R, pol);
      }
    ECHO_PHASE(12);
  }
  if (tid == 32 && dKp && q.pf == 3) {                        // dKp / dH_s into L2 from a second thread at
    prefetch_tmap(&mdK);                                       // kernel start, alongside the stage-in issue
    prefetch_tmap(&mdH);
    for (int k = 0; k * R < n; ++k) {
      if (W > 0) tma_prefetch_3d(&mdK, g.a0, b, k * R, pol);
      if (WH > 0) tma_prefetch_3d(&mdH, g.h0, b, k * R, pol);
    }
  }
  // values only the epilogue / softmax need are fetched now so their latency hides under the
  // staging wait (W <= 128 < ATT_THREADS: one column per thread, see tma_cluster)
  const float dv_old = tid < W ? dv_part[(long)b * A + g.a0 + tid] : 0.0f;
  if (!recompute)
    for (int s = tid; s < n; s += ATT_THREADS) al[s] = alpha_st[(long)b * Ts + s];
  __syncthreads();
  cluster_arrive_relaxed();                                   // publishes xbar's init (fenced above)
  ECHO_PHASE(1);
  if (n > 0) mbar_wait(&bar[0], 0);
  ECHO_PHASE(2);
  // phase 1: E = tanh(z) into smem (fp32), partial scores (RECOMPUTE) and partial dalpha.  The
  // slices are <= 128 columns wide, so each lane owns one 4-column group of A and of Hk: its qp, v
  // and dctx values stay in registers across the positions
  const bool actA = lane < W / 4, actH = lane < WH / 4;
  float qr[4] = {0.0f, 0.0f, 0.0f, 0.0f}, vr[4] = {0.0f, 0.0f, 0.0f, 0.0f}, dr[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  if (actA) {
    if (recompute) lds4(qps + lane * 4, qr);
    lds4(vs + lane * 4, vr);
  }
  if (actH) lds4(dcs + lane * 4, dr);
  cluster_wait();                                             // every CTA's xbar is initialised
  // rows s = w, w + 8, ... of this warp in groups of GR: per-lane partials first, then one
  // reduce_scatter per quantity (bitwise equal to a warp_sum per row); the row's (score, dalpha)
  // pair is then pushed to every cluster CTA (st.async into row `rank` of its receive buffer)
  constexpr int GR = 8;
  const uint32_t x_row = smem_u32(xpart + 2 * rank * Tp), x_bar = smem_u32(&xbar);
  for (int s0 = w; s0 < n; s0 += GR * ATT_WARPS) {
    float psc[GR], pda[GR];
#pragma unroll
    for (int j = 0; j < GR; ++j) {
      const int s = s0 + j * ATT_WARPS;
      psc[j] = 0.0f;
      pda[j] = 0.0f;
      if (s < n) {
        mbar_wait(&bar[s / R], 0);                            // the chunk holding row s has landed
        if (actA) {
          float kzv[4], z[4], e[4];
          lds4(kz + (size_t)s * Wb + lane * 4, kzv);
#pragma unroll
          for (int q = 0; q < 4; ++q) z[q] = z_of<T>(recompute ? qr[q] : 0.0f, kzv[q], recompute);
          if constexpr (sizeof(T) == 2) {                       // packed f32x2 tanh (same bits)
            const float2 ea = att_tanh2_bf16(make_float2(z[0], z[1])), eb = att_tanh2_bf16(make_float2(z[2], z[3]));
            e[0] = ea.x; e[1] = ea.y; e[2] = eb.x; e[3] = eb.y;
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) e[q] = att_tanh<T>(z[q]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) psc[j] = __fmaf_rn(e[q], vr[q], psc[j]);
          *reinterpret_cast<float4*>(E + (size_t)s * Wb + lane * 4) = make_float4(e[0], e[1], e[2], e[3]);
        }
        if (actH) {
          float h4[4];
          lds4(hs + (size_t)s * WHb + lane * 4, h4);
#pragma unroll
          for (int q = 0; q < 4; ++q) pda[j] = __fmaf_rn(dr[q], h4[q], pda[j]);
        }
      }
    }
    const float ps = reduce_scatter<GR>(psc, lane);
    const float pd = reduce_scatter<GR>(pda, lane);
    constexpr int SH = GR == 8 ? 2 : GR == 4 ? 3 : 4;         // slot of lane: lane >> (5 - log2 GR)
    const int j = lane >> SH;
    const int s = s0 + j * ATT_WARPS;
    // every lane of a slot holds its sums (the reduce-scatter's butterflies); lane 4j + c sends
    // slot j to cluster CTA c (c + 4 as well when C = 8)
    if (s < n) {
      if (C > 1) {
        for (int c = lane & 3; c < C; c += 4)
          st_async_v2(mapa_u32(x_row, c) + 8u * (uint32_t)s, ps, pd, mapa_u32(x_bar, c));
      } else if ((lane & 3) == 0) {
        *reinterpret_cast<float2*>(xpart + 2 * s) = make_float2(ps, pd);
        mbar_arrive(&xbar);
      }
    }
  }
  // L2 prefetch of the dKp / dH_s tiles phase 4 streams, issued by thread 0 once this CTA's loads
  // have landed so the reads overlap the exchange / softmax phases instead of phase 4
  if (tid == 0 && dKp && q.pf == 1) {
    for (int k = 0; k * R < n; ++k) mbar_wait(&bar[k], 0);
    for (int k = 0; k * R < n; ++k) {
      if (W > 0) tma_prefetch_3d(&mdK, g.a0, b, k * R, pol);
      if (WH > 0) tma_prefetch_3d(&mdH, g.h0, b, k * R, pol);
    }
  }
  ECHO_PHASE(3);
  ECHO_PHASE(4);
  ECHO_PHASE(5);
  if (w == 0) {
    mbar_wait(&xbar, 0);                                       // all C partial rows received
    // scores / dalpha for s = lane + 32 k in registers: rank-ordered sums (= gather_sum), then the
    // softmax_row_warp arithmetic (RECOMPUTE; STASH: al[] was loaded at the start)
    float sck[8], dak[8];
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int s = lane + 32 * k;
      float x = 0.0f, y = 0.0f;
      if (s < n) {
        for (int c = 0; c < C; ++c) {
          const float2 pr = *reinterpret_cast<const float2*>(xpart + 2 * (c * Tp + s));
          x = __fadd_rn(x, pr.x);
          y = __fadd_rn(y, pr.y);
        }
        m = fmaxf(m, x);
      }
      sck[k] = x;
      dak[k] = y;
    }
    if (recompute) {
      m = warp_max(m);
      float l = 0.0f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int s = lane + 32 * k;
        sck[k] = s < n ? expf(__fsub_rn(sck[k], m)) : 0.0f;
        if (s < n) l = __fadd_rn(l, sck[k]);
      }
      l = warp_sum(l);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (lane + 32 * k < n) al[lane + 32 * k] = __fdiv_rn(sck[k], l);
      __syncwarp();
    }
    float acc = 0.0f;                                          // dot = sum_s alpha_s dalpha_s (fixed order)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (lane + 32 * k < n) acc = __fmaf_rn(al[lane + 32 * k], dak[k], acc);
    acc = warp_sum(acc);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int s = lane + 32 * k;
      if (s < n) dsv[s] = __fmul_rn(al[s], __fsub_rn(dak[k], acc));
    }
  }
  __syncthreads();
  if (ds_out && g.r == 0)                                       // deferred: publish this step's rows
    for (int s = tid; s < Ts; s += ATT_THREADS) {
      ds_out[(long)b * Ts + s] = s < n ? dsv[s] : 0.0f;
      if (al_out) al_out[(long)b * Ts + s] = s < n ? al[s] : 0.0f;
    }
  ECHO_PHASE(6);
  if (recompute && ctx_regen) ctx_columns<T>(hs, WHb, WH, al, n, ctx_regen + (long)b * Hk + g.h0, tid);
  ECHO_PHASE(7);
  // phase 4 (column-local).  Thread -> (column group gi of 4, position phase ph); phase ph takes
  // s = ph, ph + P, ... in increasing order and the P phase partials are combined in rank order.
  //   A columns : dKp += dE ; dqp = sum_s dE ; dv_part += sum_s ds E   with dE = ds v (1 - E^2)
  //   Hk columns: dHs += alpha_s dctx
  const int GA = Wb / 4, G = (Wb + WHb) / 4;
  const int gi = tid % G, ph = tid / G;
  float dq[4] = {0.0f, 0.0f, 0.0f, 0.0f}, dvv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  constexpr int U = 4;                                         // rows in flight per thread
  if (ph < P && gi < GA && gi * 4 < W) {
    const int c = gi * 4;
    float vc[4];
    lds4(vs + c, vc);
    float* base = dKp ? dKp + (long)b * d.kp_stride_b + g.a0 + c : nullptr;
    for (int s0 = ph; s0 < n; s0 += U * P) {
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + u * P;
        if (s < n && dKp) x[u] = ldg4_hint(base + (long)s * d.kp_stride_s, pol);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + u * P;
        if (s < n) {
          float e[4], xv[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
          lds4(E + (size_t)s * Wb + c, e);
          const float ds = dsv[s];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float dE = __fmul_rn(__fmul_rn(ds, vc[k]), __fsub_rn(1.0f, __fmul_rn(e[k], e[k])));
            xv[k] = __fadd_rn(xv[k], dE);
            dq[k] = __fadd_rn(dq[k], dE);
            dvv[k] = __fmaf_rn(ds, e[k], dvv[k]);
          }
          if (dKp) stg4_hint(base + (long)s * d.kp_stride_s, xv, pol);
        }
      }
    }
  } else if (dHs && ph < P && gi >= GA && (gi - GA) * 4 < WH) {
    const int c = (gi - GA) * 4;
    float dc[4];
    lds4(dcs + c, dc);
    float* base = dHs + (long)b * d.hs_stride_b + g.h0 + c;
    for (int s0 = ph; s0 < n; s0 += U * P) {
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + u * P;
        if (s < n) x[u] = ldg4_hint(base + (long)s * d.hs_stride_s, pol);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = s0 + u * P;
        if (s < n) {
          const float a = al[s];
          float xv[4] = {__fmaf_rn(a, dc[0], x[u].x), __fmaf_rn(a, dc[1], x[u].y), __fmaf_rn(a, dc[2], x[u].z),
                         __fmaf_rn(a, dc[3], x[u].w)};
          stg4_hint(base + (long)s * d.hs_stride_s, xv, pol);
        }
      }
    }
  }
  __syncthreads();                                             // E reads done: red may alias it
  ECHO_PHASE(8);
  if (ph < P && gi < GA) {
    *reinterpret_cast<float4*>(red + (size_t)ph * Wb + gi * 4) = make_float4(dq[0], dq[1], dq[2], dq[3]);
    *reinterpret_cast<float4*>(red + (size_t)(P + ph) * Wb + gi * 4) = make_float4(dvv[0], dvv[1], dvv[2], dvv[3]);
  }
  __syncthreads();
  if (tid < W) {
    const int c = tid;
    float q = 0.0f, x = 0.0f;
    for (int k = 0; k < P; ++k) {
      q = __fadd_rn(q, red[(size_t)k * Wb + c]);
      x = __fadd_rn(x, red[(size_t)(P + k) * Wb + c]);
    }
    const long o = (long)b * A + g.a0 + c;
    dqp[o] = q;
    dv_part[o] = __fadd_rn(dv_old, x);
  }
  ECHO_PHASE(9);
  ECHO_PHASE(10);
}

// ---------------------------------------------------------------- a6 deferred accumulations
// dKp[b,s,:] = sum over t = Td-1 .. 0 of dE_t and dH_s[b,s,:] = sum over t = Td-1 .. 0 of
// alpha_t[b,s] dctx_t[b,:], with dE_t = (ds_t v) (1 - E_t^2) and E_t = tanh(z_t), evaluated with
// exactly the expressions and the t order the per-step read-modify-write used: bit-identical to
// it.  One CTA per (row b, 64-column block); thread = (column, position phase).
constexpr int FIN_COLS = 64;
template <typename T>
__global__ void __launch_bounds__(256) attn_dkp_finish_kernel(echo_attn_desc d, int Td, const T* __restrict__ qp_all,
                                                              const T* __restrict__ Kp, const T* __restrict__ Z_all,
                                                              const T* __restrict__ v,
                                                              const int32_t* __restrict__ src_len,
                                                              const float* __restrict__ ds_all, float* __restrict__ dKp,
                                                              int accumulate) {
  pdl_wait();
  extern __shared__ float fsm[];
  const int A = d.A, Ts = d.Ts, B = d.B;
  float* qs = fsm;                                  // [Td][FIN_COLS] qp (RECOMPUTE)
  float* dss = qs + (size_t)Td * FIN_COLS;          // [Td][Ts] ds
  const int b = blockIdx.y, a0 = blockIdx.x * FIN_COLS, tid = threadIdx.x;
  const int n = row_len(src_len, b, Ts);
  const bool rec = Z_all == nullptr;
  for (int i = tid; i < Td * FIN_COLS; i += 256) {
    const int t = i / FIN_COLS, c = i - t * FIN_COLS;
    qs[i] = (rec && a0 + c < A) ? to_f(qp_all[((long)t * B + b) * A + a0 + c]) : 0.0f;
  }
  for (int i = tid; i < Td * Ts; i += 256) {
    const int t = i / Ts, s = i - t * Ts;
    dss[i] = ds_all[((long)t * B + b) * Ts + s];
  }
  __syncthreads();
  const int c = tid % FIN_COLS, a = a0 + c;
  if (a >= A) return;
  const float vc = to_f(v[a]);
  for (int s = tid / FIN_COLS; s < Ts; s += 256 / FIN_COLS) {
    if (accumulate && s >= n) continue;                        // masked rows untouched (per-step RMW)
    float acc = accumulate ? dKp[(long)b * d.kp_stride_b + (long)s * d.kp_stride_s + a] : 0.0f;
    if (s < n) {
      const float kz = rec ? to_f(Kp[(long)b * d.kp_stride_b + (long)s * d.kp_stride_s + a]) : 0.0f;
      for (int t = Td - 1; t >= 0; --t) {
        const float z = rec ? St<T>::round(__fadd_rn(qs[t * FIN_COLS + c], kz))
                            : to_f(Z_all[(((long)t * B + b) * Ts + s) * A + a]);
        const float e = att_tanh<T>(z);
        const float dE = __fmul_rn(__fmul_rn(dss[t * Ts + s], vc), __fsub_rn(1.0f, __fmul_rn(e, e)));
        acc = __fadd_rn(acc, dE);
      }
    }
    dKp[(long)b * d.kp_stride_b + (long)s * d.kp_stride_s + a] = acc;
  }
}

__global__ void __launch_bounds__(256) attn_dhs_finish_kernel(echo_attn_desc d, int Td,
                                                              const int32_t* __restrict__ src_len,
                                                              const float* __restrict__ al_all,
                                                              const float* __restrict__ dctx_all,
                                                              float* __restrict__ dHs, int accumulate) {
  pdl_wait();
  extern __shared__ float fsm[];
  const int Hk = d.Hk, Ts = d.Ts, B = d.B;
  float* cs = fsm;                                  // [Td][FIN_COLS] dctx
  float* als = cs + (size_t)Td * FIN_COLS;          // [Td][Ts] alpha
  const int b = blockIdx.y, h0 = blockIdx.x * FIN_COLS, tid = threadIdx.x;
  const int n = row_len(src_len, b, Ts);
  for (int i = tid; i < Td * FIN_COLS; i += 256) {
    const int t = i / FIN_COLS, c = i - t * FIN_COLS;
    cs[i] = h0 + c < Hk ? dctx_all[((long)t * B + b) * Hk + h0 + c] : 0.0f;
  }
  for (int i = tid; i < Td * Ts; i += 256) {
    const int t = i / Ts, s = i - t * Ts;
    als[i] = al_all[((long)t * B + b) * Ts + s];
  }
  __syncthreads();
  const int c = tid % FIN_COLS, h = h0 + c;
  if (h >= Hk) return;
  for (int s = tid / FIN_COLS; s < Ts; s += 256 / FIN_COLS) {
    if (accumulate && s >= n) continue;
    float acc = accumulate ? dHs[(long)b * d.hs_stride_b + (long)s * d.hs_stride_s + h] : 0.0f;
    if (s < n)
      for (int t = Td - 1; t >= 0; --t) acc = __fmaf_rn(als[t * Ts + s], cs[t * FIN_COLS + c], acc);
    dHs[(long)b * d.hs_stride_b + (long)s * d.hs_stride_s + h] = acc;
  }
}

__global__ void dv_reduce_kernel(int B, int A, const float* __restrict__ part, float* __restrict__ dv, int acc) {
  pdl_wait();
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  float x = acc ? dv[a] : 0.0f;
  for (int b = 0; b < B; ++b) x = __fadd_rn(x, part[(long)b * A + a]);
  dv[a] = x;
}

// ---------------------------------------------------------------- host side
static int att_chunk(int Ts, int C) { return (Ts + C - 1) / C; }

static size_t fwd_smem(const echo_attn_desc* d) {
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  const int G = ctx_groups(d->Hk, V);
  const int chunk = att_chunk(d->Ts, att_cluster(d->Ts));
  return sizeof(float) * (2 * (size_t)d->A + 4 + ((chunk + 3) & ~3) + (size_t)G * d->Hk + d->Hk);
}
static size_t bwd_smem(const echo_attn_desc* d) {
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  const int G = ctx_groups(d->Hk, V);
  const int chunk = att_chunk(d->Ts, att_cluster(d->Ts));
  return sizeof(float) * (2 * (size_t)d->A + d->Hk + 4 + 2 * (size_t)((chunk + 3) & ~3) +
                          2 * (size_t)ATT_WARPS * d->A + 2 * (size_t)d->A + (size_t)G * d->Hk + d->Hk);
}

// a6 L2 prefetch of the dKp / dH_s tiles (ECHO_A6_PREFETCH=0|1|2, read once; see TmaGeo::pf)
static int a6_prefetch_mode() {
  static const int m = [] {
    const char* e = getenv("ECHO_A6_PREFETCH");
    return e && *e >= '0' && *e <= '3' ? *e - '0' : 3;
  }();
  return m;
}

// ECHO_ATTN_L2LAST=1: evict_last policy on the per-step attention tensors (see l2_policy)
static int attn_l2_last() {
  static const int m = [] {
    const char* e = getenv("ECHO_ATTN_L2LAST");
    return e && *e == '1' ? 1 : 0;
  }();
  return m;
}

// TMA path: cluster size and shared-memory footprint; returns false if the generic path must run
static size_t al128h(size_t b) { return (b + 127) & ~(size_t)127; }
static bool tma_params(const echo_attn_desc* d, int* C, int* rows, size_t* smem_fwd, size_t* smem_bwd,
                       TmaGeo* geo) {
  const size_t sT = d->dtype == ECHO_FP32 ? 4 : 2;
  if (d->A > 1024 || d->Hk > 1024 || d->Ts > 256) return false;
  const int c = tma_cluster(d->A, d->Hk);
  const size_t W = tma_width(d->A, c), WH = tma_width(d->Hk, c);
  const size_t Tp = (d->Ts + 3) & ~3;
  const int R = tma_rows(d->Ts, (int)W, (int)WH, (int)sT);
  const size_t Ts = (size_t)tma_tile_rows(d->Ts, R);        // rows allocated per tile
  const size_t fwd = al128h(Ts * W * sT) + al128h(Ts * WH * sT) + 2 * W * sT + (size_t)c * Tp * 4;
  const size_t P = tma_phases((int)W, (int)WH);
  const size_t bwd = al128h(Ts * W * sT) + al128h(Ts * WH * sT) + (sT == 4 ? 0 : al128h(Ts * W * 4)) +
                     2 * W * sT + ((2 + 2 * (size_t)c) * Tp + WH) * 4 + (Ts >= 2 * P ? 0 : 2 * P * W * 4);
  if (bwd > 220 * 1024) return false;
  *C = c;
  *rows = R;
  geo->C = c;
  geo->Wb = (int)W;
  geo->WHb = (int)WH;
  geo->R = R;
  geo->Tr = (int)Ts;
  geo->P = (int)P;
  geo->pf = a6_prefetch_mode();
  geo->l2last = attn_l2_last();
  *smem_fwd = fwd;
  *smem_bwd = bwd;
  return true;
}

// a5 row-streaming variant (attn_fwd_rows): ECHO_A5_ROWS=0 never, 1 always (where the shape fits),
// default: when the launch has at least two rows per SM.  Read on every call (tests switch it).
static int a5_rows_mode() {
  const char* e = getenv("ECHO_A5_ROWS");
  return e && (*e == '0' || *e == '1') ? *e - '0' : 2;
}
static int sm_count() {
  static const int n = [] {
    int dev = 0, s = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    return s > 0 ? s : 148;
  }();
  return n;
}
// stage = R positions x every column slice (R in {8, 16, 32}: R | 32 keeps a stage inside one
// 32-position softmax register) + the row's qp vector; 16-32 KB per stage, ~100 KB of ring
static bool rows_params(const echo_attn_desc* d, RowGeo* g, size_t* smem) {
  if (d->A > 1024 || d->Hk > 1024 || d->Ts > 256) return false;
  const size_t es = d->dtype == ECHO_FP32 ? 4 : 2;
  const int C = tma_cluster(d->A, d->Hk);
  const int Wb = tma_width(d->A, C), WHb = tma_width(d->Hk, C);
  const size_t mw = (size_t)(Wb > WHb ? Wb : WHb);
  // per-CTA shared budget for ROWS_PER_SM resident CTAs (228 KB per SM, 1 KB reserved per CTA)
  const size_t tail = rows_tail_bytes(d->Ts, C);
  const size_t budget = 228 * 1024 / ROWS_PER_SM - 1024 - 256 - tail;
  auto stage_of = [&](int R) { return (size_t)C * al128h((size_t)R * mw * es) + al128h((size_t)d->A * es); };
  int R = 8;                                                  // largest R in {8, 16, 32} with >= 3 stages
  if (3 * stage_of(16) <= budget) R = 16;
  if (3 * stage_of(32) <= budget) R = 32;
  g->C = C;
  g->Wb = Wb;
  g->WHb = WHb;
  g->R = R;
  g->sub = (uint32_t)al128h((size_t)R * mw * es);
  g->stage = (uint32_t)stage_of(R);
  int nst = (int)(budget / g->stage);
  g->nst = nst < 2 ? 2 : (nst > ROWS_MAXST ? ROWS_MAXST : nst);
  *smem = (size_t)g->nst * g->stage + tail;
  return *smem <= 200 * 1024;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 3-D map over a [Ts][B][X]-strided tensor: dims {X, B, Ts}, box {boxX, 1, R}
static bool map3d(CUtensorMap* m, const void* base, bool bf16, uint64_t X, uint64_t B, uint64_t Ts, int64_t stride_b,
                  int64_t stride_s, uint32_t boxX, int boxR) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const uint64_t es = bf16 ? 2 : 4;
  cuuint64_t dims[3] = {X, B, Ts};
  cuuint64_t strides[2] = {(cuuint64_t)stride_b * es, (cuuint64_t)stride_s * es};
  cuuint32_t box[3] = {boxX, 1, (cuuint32_t)boxR};   // one chunk of positions
  cuuint32_t el[3] = {1, 1, 1};
  return fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims,
            strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename Kern, typename... Args>
static cudaError_t launch_cluster(Kern kern, int C, int B, size_t smem, cudaStream_t st, Args... args) {
  return launch(kern, dim3(C, B, 1), dim3(ATT_THREADS, 1, 1), smem, st, -C, args...);   // explicit cluster, even C = 1
}

static echo_status check_attn(const char* fn, const echo_attn_desc* d) {
  if (!d) return fail(ECHO_ERR_INVALID, "%s: desc is NULL", fn);
  if (d->B <= 0 || d->Ts <= 0 || d->A <= 0 || d->Hk <= 0)
    return fail(ECHO_ERR_INVALID, "%s: B=%d Ts=%d A=%d Hk=%d must be > 0", fn, d->B, d->Ts, d->A, d->Hk);
  if (d->A % 8 || d->Hk % 8) return fail(ECHO_ERR_INVALID, "%s: A=%d and Hk=%d must be multiples of 8", fn, d->A, d->Hk);
  if (d->Ts > 4096) return fail(ECHO_ERR_CAPACITY, "%s: Ts=%d exceeds 4096", fn, d->Ts);
  if (d->B > 65535) return fail(ECHO_ERR_CAPACITY, "%s: B=%d exceeds 65535 rows per launch", fn, d->B);
  if (d->dtype != ECHO_FP32 && d->dtype != ECHO_BF16) return fail(ECHO_ERR_INVALID, "%s: bad dtype %d", fn, d->dtype);
  if (d->mode != ECHO_STASH && d->mode != ECHO_RECOMPUTE) return fail(ECHO_ERR_INVALID, "%s: bad mode %d", fn, d->mode);
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  if (d->kp_stride_b % V || d->kp_stride_s % V || d->hs_stride_b % V || d->hs_stride_s % V)
    return fail(ECHO_ERR_INVALID, "%s: strides must be multiples of %d elements", fn, V);
  if (d->kp_stride_b <= 0 || d->kp_stride_s <= 0 || d->hs_stride_b <= 0 || d->hs_stride_s <= 0)
    return fail(ECHO_ERR_INVALID, "%s: strides must be > 0", fn);
  return ECHO_OK;
}

// ECHO_CHECK_SRC_LEN=1 (read on every call): src_len is a device array, so the kernels clamp it to
// [1, Ts]; with the flag set the entry points copy it to the host (a stream synchronization) and
// reject any entry outside [1, Ts] with ECHO_ERR_INVALID before launching.  Skipped while the stream
// is being captured into a CUDA graph (no synchronization is allowed there).
static echo_status check_src_len(const char* fn, const echo_attn_desc* d, const int32_t* src_len, cudaStream_t st) {
  const char* e = getenv("ECHO_CHECK_SRC_LEN");
  if (!src_len || !e || e[0] != '1') return ECHO_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return ECHO_OK;
  int32_t* h = (int32_t*)malloc(sizeof(int32_t) * (size_t)d->B);
  if (!h) return fail(ECHO_ERR_CAPACITY, "%s: host buffer for src_len", fn);
  cudaError_t ce = cudaMemcpyAsync(h, src_len, sizeof(int32_t) * (size_t)d->B, cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) {
    free(h);
    return fail(ECHO_ERR_CUDA, "%s: reading src_len: %s", fn, cudaGetErrorString(ce));
  }
  for (int b = 0; b < d->B; ++b)
    if (h[b] < 1 || h[b] > d->Ts) {
      const int v = h[b];
      free(h);
      return fail(ECHO_ERR_INVALID, "%s: src_len[%d] = %d outside [1, %d]", fn, b, v, d->Ts);
    }
  free(h);
  return ECHO_OK;
}

#define ECHO_REQ(p, name)                                                                     \
  do {                                                                                        \
    if (!(p)) return fail(ECHO_ERR_INVALID, "%s: required pointer %s is NULL", fn, name);     \
    if (!aligned16(p)) return fail(ECHO_ERR_INVALID, "%s: %s is not 16-byte aligned", fn, name); \
  } while (0)

static echo_status set_smem(const void* kern, size_t bytes, const char* fn) {
  if (bytes > 227 * 1024) return fail(ECHO_ERR_CAPACITY, "%s: needs %zu bytes of shared memory", fn, bytes);
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: cudaFuncSetAttribute: %s", fn, cudaGetErrorString(e));
  }
  return ECHO_OK;
}

template <typename T>
static echo_status launch_rows(const char* fn, const echo_attn_desc* d, const RowGeo& g, size_t smem,
                               const CUtensorMap& mK, const CUtensorMap& mH, const void* qp, const void* v,
                               const int32_t* src_len, void* ctx, void* E_st, float* alpha_st, cudaStream_t st) {
  decltype(&attn_fwd_rows<T, 1, false>) k;
  if (E_st) k = g.C == 1 ? attn_fwd_rows<T, 1, true> : g.C == 2 ? attn_fwd_rows<T, 2, true>
              : g.C == 4 ? attn_fwd_rows<T, 4, true> : attn_fwd_rows<T, 8, true>;
  else k = g.C == 1 ? attn_fwd_rows<T, 1, false> : g.C == 2 ? attn_fwd_rows<T, 2, false>
         : g.C == 4 ? attn_fwd_rows<T, 4, false> : attn_fwd_rows<T, 8, false>;
  echo_status s = set_smem((const void*)k, smem, fn);
  if (s) return s;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, ROWS_THREADS, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    occ = 1;
  }
  const int grid = d->B < occ * sm_count() ? d->B : occ * sm_count();
  cudaError_t e = launch(k, dim3(grid, 1, 1), dim3(ROWS_THREADS, 1, 1), smem, st, 0, *d, g, mK, mH, (const T*)qp,
                         (const T*)v, src_len, (T*)ctx, (T*)E_st, alpha_st);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

}  // namespace echo

using namespace echo;

extern "C" echo_status echo_attn_fwd(const echo_attn_desc* d, const void* qp, const void* Kp, const void* v,
                                     const void* Hs, const int32_t* src_len, void* ctx, void* E_st,
                                     float* alpha_st, void* stream) {
  const char* fn = "echo_attn_fwd";
  echo_status s = check_attn(fn, d);
  if (s) return s;
  ECHO_REQ(qp, "qp");
  ECHO_REQ(Kp, "Kp");
  ECHO_REQ(v, "v");
  ECHO_REQ(Hs, "Hs");
  ECHO_REQ(ctx, "ctx");
  if (d->mode == ECHO_STASH) {
    ECHO_REQ(E_st, "E_st");
    if (!alpha_st) return fail(ECHO_ERR_INVALID, "%s: alpha_st required in STASH mode", fn);
  } else if (E_st || alpha_st) {
    return fail(ECHO_ERR_INVALID, "%s: E_st / alpha_st must be NULL in RECOMPUTE mode", fn);
  }
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = check_src_len(fn, d, src_len, st))) return s;
  const int C = att_cluster(d->Ts), chunk = att_chunk(d->Ts, C);
  cudaError_t e;
  int tC, tR;
  size_t sf, sb;
  TmaGeo geo;
  CUtensorMap mK, mH;
  const bool bfd = d->dtype == ECHO_BF16;
  RowGeo rg;
  size_t rsm;
  const int rmode = a5_rows_mode();
  if (rmode && (rmode == 1 || d->B >= 2 * sm_count()) && rows_params(d, &rg, &rsm) &&
      map3d(&mK, Kp, bfd, d->A, d->B, d->Ts, d->kp_stride_b, d->kp_stride_s, rg.Wb, rg.R) &&
      map3d(&mH, Hs, bfd, d->Hk, d->B, d->Ts, d->hs_stride_b, d->hs_stride_s, rg.WHb, rg.R))
    return bfd ? launch_rows<__nv_bfloat16>(fn, d, rg, rsm, mK, mH, qp, v, src_len, ctx, E_st, alpha_st, st)
               : launch_rows<float>(fn, d, rg, rsm, mK, mH, qp, v, src_len, ctx, E_st, alpha_st, st);
  if (tma_params(d, &tC, &tR, &sf, &sb, &geo) &&
      map3d(&mK, Kp, bfd, d->A, d->B, d->Ts, d->kp_stride_b, d->kp_stride_s, tma_width(d->A, tC), tR) &&
      map3d(&mH, Hs, bfd, d->Hk, d->B, d->Ts, d->hs_stride_b, d->hs_stride_s, tma_width(d->Hk, tC), tR)) {
    if (d->dtype == ECHO_FP32) {
      if ((s = set_smem((const void*)attn_fwd_tma<float>, sf, fn))) return s;
      e = launch_cluster(attn_fwd_tma<float>, tC, d->B, sf, st, *d, geo, mK, mH, (const float*)qp, (const float*)v, src_len,
                         (float*)ctx, (float*)E_st, alpha_st);
    } else {
      typedef __nv_bfloat16 bf;
      if ((s = set_smem((const void*)attn_fwd_tma<bf>, sf, fn))) return s;
      e = launch_cluster(attn_fwd_tma<bf>, tC, d->B, sf, st, *d, geo, mK, mH, (const bf*)qp, (const bf*)v, src_len, (bf*)ctx,
                         (bf*)E_st, alpha_st);
    }
    if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
    return check_launch(fn);
  }
  const size_t smem = fwd_smem(d);
  if (d->dtype == ECHO_FP32) {
    if ((s = set_smem((const void*)attn_fwd_kernel<float>, smem, fn))) return s;
    e = launch_cluster(attn_fwd_kernel<float>, C, d->B, smem, st, *d, chunk, (const float*)qp, (const float*)Kp,
                       (const float*)v, (const float*)Hs, src_len, (float*)ctx, (float*)E_st, alpha_st);
  } else {
    typedef __nv_bfloat16 bf;
    if ((s = set_smem((const void*)attn_fwd_kernel<bf>, smem, fn))) return s;
    e = launch_cluster(attn_fwd_kernel<bf>, C, d->B, smem, st, *d, chunk, (const bf*)qp, (const bf*)Kp, (const bf*)v,
                       (const bf*)Hs, src_len, (bf*)ctx, (bf*)E_st, alpha_st);
  }
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

static echo_status attn_bwd_impl(const char* fn, const echo_attn_desc* d, const void* qp, const void* Kp,
                                 const void* v, const void* Hs, const int32_t* src_len, const void* E_st,
                                 const float* alpha_st, const float* dctx, float* dqp, float* dKp, float* dHs,
                                 float* dv_part, void* ctx_regen, float* ds_out, float* al_out, void* stream) {
  echo_status s = check_attn(fn, d);
  if (s) return s;
  const bool deferred = ds_out != nullptr;
  ECHO_REQ(v, "v");
  ECHO_REQ(Hs, "Hs");
  ECHO_REQ(dctx, "dctx");
  ECHO_REQ(dqp, "dqp");
  if (!deferred) {
    ECHO_REQ(dKp, "dKp");
    ECHO_REQ(dHs, "dHs");
  }
  ECHO_REQ(dv_part, "dv_part");
  if (d->mode == ECHO_STASH) {
    ECHO_REQ(E_st, "E_st");
    if (!alpha_st) return fail(ECHO_ERR_INVALID, "%s: alpha_st required in STASH mode", fn);
    if (ctx_regen) return fail(ECHO_ERR_INVALID, "%s: ctx_regen must be NULL in STASH mode", fn);
    if (al_out) return fail(ECHO_ERR_INVALID, "%s: alpha_out must be NULL in STASH mode (alpha is stashed)", fn);
  } else {
    ECHO_REQ(qp, "qp");
    ECHO_REQ(Kp, "Kp");
    if (E_st || alpha_st) return fail(ECHO_ERR_INVALID, "%s: E_st / alpha_st must be NULL in RECOMPUTE mode", fn);
    if (ctx_regen && !aligned16(ctx_regen)) return fail(ECHO_ERR_INVALID, "%s: ctx_regen not 16-byte aligned", fn);
    if (deferred && !al_out) return fail(ECHO_ERR_INVALID, "%s: alpha_out required in deferred RECOMPUTE", fn);
  }
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = check_src_len(fn, d, src_len, st))) return s;
  const int C = att_cluster(d->Ts), chunk = att_chunk(d->Ts, C);
  cudaError_t e;
  int tC, tR;
  size_t sf, sb;
  TmaGeo geo;
  CUtensorMap mK, mH, mdK, mdH;
  const bool bfd = d->dtype == ECHO_BF16;
  const bool rec = d->mode == ECHO_RECOMPUTE;
  if (tma_params(d, &tC, &tR, &sf, &sb, &geo) &&
      (rec ? map3d(&mK, Kp, bfd, d->A, d->B, d->Ts, d->kp_stride_b, d->kp_stride_s, tma_width(d->A, tC), tR)
           : map3d(&mK, E_st, bfd, d->A, d->B, d->Ts, (int64_t)d->Ts * d->A, d->A, tma_width(d->A, tC), tR)) &&
      map3d(&mH, Hs, bfd, d->Hk, d->B, d->Ts, d->hs_stride_b, d->hs_stride_s, tma_width(d->Hk, tC), tR) &&
      (deferred ||
       (map3d(&mdK, dKp, false, d->A, d->B, d->Ts, d->kp_stride_b, d->kp_stride_s, tma_width(d->A, tC), tR) &&
        map3d(&mdH, dHs, false, d->Hk, d->B, d->Ts, d->hs_stride_b, d->hs_stride_s, tma_width(d->Hk, tC), tR)))) {
    if (deferred) {                                              // prefetch maps unused (no dKp / dH_s)
      mdK = mK;
      mdH = mH;
    }
    if (d->dtype == ECHO_FP32) {
      if ((s = set_smem((const void*)attn_bwd_tma<float>, sb, fn))) return s;
      e = launch_cluster(attn_bwd_tma<float>, tC, d->B, sb, st, *d, geo, mK, mH, mdK, mdH, (const float*)qp, (const float*)v,
                         src_len, rec, alpha_st, dctx, dqp, dKp, dHs, dv_part, (float*)ctx_regen, ds_out, al_out);
    } else {
      typedef __nv_bfloat16 bf;
      if ((s = set_smem((const void*)attn_bwd_tma<bf>, sb, fn))) return s;
      e = launch_cluster(attn_bwd_tma<bf>, tC, d->B, sb, st, *d, geo, mK, mH, mdK, mdH, (const bf*)qp, (const bf*)v,
                         src_len, rec, alpha_st, dctx, dqp, dKp, dHs, dv_part, (bf*)ctx_regen, ds_out, al_out);
    }
    if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
    return check_launch(fn);
  }
  if (deferred) return fail(ECHO_ERR_UNSUPPORTED, "%s: deferred mode needs the TMA path (Ts <= 256, slices fit)", fn);
  const size_t smem = bwd_smem(d);
  if (d->dtype == ECHO_FP32) {
    if ((s = set_smem((const void*)attn_bwd_kernel<float>, smem, fn))) return s;
    e = launch_cluster(attn_bwd_kernel<float>, C, d->B, smem, st, *d, chunk, (const float*)qp, (const float*)Kp,
                       (const float*)v, (const float*)Hs, src_len, (const float*)E_st, alpha_st, dctx, dqp, dKp, dHs,
                       dv_part, (float*)ctx_regen);
  } else {
    typedef __nv_bfloat16 bf;
    if ((s = set_smem((const void*)attn_bwd_kernel<bf>, smem, fn))) return s;
    e = launch_cluster(attn_bwd_kernel<bf>, C, d->B, smem, st, *d, chunk, (const bf*)qp, (const bf*)Kp, (const bf*)v,
                       (const bf*)Hs, src_len, (const bf*)E_st, alpha_st, dctx, dqp, dKp, dHs, dv_part,
                       (bf*)ctx_regen);
  }
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

extern "C" echo_status echo_attn_bwd_recompute(const echo_attn_desc* d, const void* qp, const void* Kp, const void* v,
                                               const void* Hs, const int32_t* src_len, const void* E_st,
                                               const float* alpha_st, const float* dctx, float* dqp, float* dKp,
                                               float* dHs, float* dv, void* ctx_regen, void* ws, size_t* ws_bytes,
                                               void* stream) {
  const char* fn = "echo_attn_bwd_recompute";
  echo_status s = check_attn(fn, d);
  if (s) return s;
  const size_t need = sizeof(float) * (size_t)d->B * d->A;   // per-row dv partials [B,A] fp32
  if (!ws) {                                                // two-call workspace convention
    if (!ws_bytes) return fail(ECHO_ERR_INVALID, "%s: ws and ws_bytes are both NULL", fn);
    *ws_bytes = need;
    return ECHO_OK;
  }
  if (ws_bytes && *ws_bytes < need) return fail(ECHO_ERR_CAPACITY, "%s: ws has %zu bytes, needs %zu", fn, *ws_bytes, need);
  if (dv && !aligned16(dv)) return fail(ECHO_ERR_INVALID, "%s: dv is not 16-byte aligned", fn);
  s = attn_bwd_impl(fn, d, qp, Kp, v, Hs, src_len, E_st, alpha_st, dctx, dqp, dKp, dHs, (float*)ws, ctx_regen, nullptr,
                    nullptr, stream);
  if (s || !dv) return s;
  const cudaError_t e = launch(dv_reduce_kernel, dim3((d->A + 127) / 128), dim3(128), 0, (cudaStream_t)stream, 1, d->B,
                               d->A, (const float*)ws, dv, 0);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

extern "C" echo_status echo_attn_bwd_deferred(const echo_attn_desc* d, const void* qp, const void* Kp, const void* v,
                                              const void* Hs, const int32_t* src_len, const void* E_st,
                                              const float* alpha_st, const float* dctx, float* dqp, float* dv_part,
                                              void* ctx_regen, float* ds_out, float* alpha_out, void* stream) {
  const char* fn = "echo_attn_bwd_deferred";
  if (!ds_out) return fail(ECHO_ERR_INVALID, "%s: ds_out is NULL", fn);
  return attn_bwd_impl(fn, d, qp, Kp, v, Hs, src_len, E_st, alpha_st, dctx, dqp, nullptr, nullptr, dv_part, ctx_regen,
                       ds_out, alpha_out, stream);
}

static echo_status finish_impl(const char* fn, const echo_attn_desc* d, int32_t Td, const void* qp_all,
                               const void* Kp, const void* E_st_all, const void* v, const int32_t* src_len,
                               const float* ds_all, const float* alpha_all, const float* dctx_all, float* dKp,
                               float* dHs, int accumulate, void* stream) {
  echo_status s = check_attn(fn, d);
  if (s) return s;
  if (Td <= 0) return fail(ECHO_ERR_INVALID, "%s: Td=%d", fn, Td);
  if (!v || !ds_all || !alpha_all || !dctx_all || !dKp || !dHs) return fail(ECHO_ERR_INVALID, "%s: NULL pointer", fn);
  if (d->mode == ECHO_STASH) {
    if (!E_st_all) return fail(ECHO_ERR_INVALID, "%s: E_st_all required in STASH mode", fn);
  } else if (!qp_all || !Kp || E_st_all) {
    return fail(ECHO_ERR_INVALID, "%s: RECOMPUTE needs qp_all and Kp (and no E_st_all)", fn);
  }
  const size_t smem = sizeof(float) * ((size_t)Td * FIN_COLS + (size_t)Td * d->Ts);
  if (smem > 200 * 1024) return fail(ECHO_ERR_CAPACITY, "%s: Td=%d x Ts=%d too large", fn, Td, d->Ts);
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = check_src_len(fn, d, src_len, st))) return s;
  const bool rec = d->mode == ECHO_RECOMPUTE;
  cudaError_t e;
  if (d->dtype == ECHO_FP32) {
    if ((s = set_smem((const void*)attn_dkp_finish_kernel<float>, smem, fn))) return s;
    e = launch(attn_dkp_finish_kernel<float>, dim3((d->A + FIN_COLS - 1) / FIN_COLS, d->B), dim3(256), smem, st, 1, *d,
               (int)Td, (const float*)qp_all, (const float*)Kp, rec ? nullptr : (const float*)E_st_all,
               (const float*)v, src_len, ds_all, dKp, accumulate);
  } else {
    typedef __nv_bfloat16 bf;
    if ((s = set_smem((const void*)attn_dkp_finish_kernel<bf>, smem, fn))) return s;
    e = launch(attn_dkp_finish_kernel<bf>, dim3((d->A + FIN_COLS - 1) / FIN_COLS, d->B), dim3(256), smem, st, 1, *d,
               (int)Td, (const bf*)qp_all, (const bf*)Kp, rec ? nullptr : (const bf*)E_st_all, (const bf*)v, src_len,
               ds_all, dKp, accumulate);
  }
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  if ((s = set_smem((const void*)attn_dhs_finish_kernel, smem, fn))) return s;
  e = launch(attn_dhs_finish_kernel, dim3((d->Hk + FIN_COLS - 1) / FIN_COLS, d->B), dim3(256), smem, st, 1, *d,
             (int)Td, src_len, alpha_all, dctx_all, dHs, accumulate);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

extern "C" echo_status echo_attn_bwd_finish(const echo_attn_desc* d, int32_t Td, const void* qp_all, const void* Kp,
                                            const void* E_st_all, const void* v, const int32_t* src_len,
                                            const float* ds_all, const float* alpha_all, const float* dctx_all,
                                            float* dKp, float* dHs, void* stream) {
  return finish_impl("echo_attn_bwd_finish", d, Td, qp_all, Kp, E_st_all, v, src_len, ds_all, alpha_all, dctx_all,
                     dKp, dHs, 0, stream);
}

extern "C" echo_status echo_attn_bwd_accumulate(const echo_attn_desc* d, const void* qp_t, const void* Kp,
                                                const void* E_st_t, const void* v, const int32_t* src_len,
                                                const float* ds_t, const float* alpha_t, const float* dctx_t,
                                                float* dKp, float* dHs, void* stream) {
  return finish_impl("echo_attn_bwd_accumulate", d, 1, qp_t, Kp, E_st_t, v, src_len, ds_t, alpha_t, dctx_t, dKp, dHs,
                     1, stream);
}

#ifdef ECHO_PHASE_TIMING
namespace echo {
__global__ void stamp_kernel(int slot) {
  unsigned long long gt;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
  g_echo_phase[13][slot] = gt;
}
}  // namespace echo
extern "C" void echo_debug_stamp(int slot, void* stream) { echo::stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(slot); }
extern "C" int echo_debug_phase_times(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, echo::g_echo_phase, sizeof(unsigned long long) * (size_t)n);
}
#endif


extern "C" echo_status echo_attn_dv_reduce(int32_t B, int32_t A, const float* dv_part, float* dv, int32_t accumulate,
                                           void* stream) {
  const char* fn = "echo_attn_dv_reduce";
  if (B <= 0 || A <= 0) return fail(ECHO_ERR_INVALID, "%s: B=%d A=%d must be > 0", fn, B, A);
  if (!dv_part || !dv) return fail(ECHO_ERR_INVALID, "%s: NULL pointer", fn);
  const cudaError_t e = launch(dv_reduce_kernel, dim3((A + 127) / 128), dim3(128), 0, (cudaStream_t)stream, 1, B, A,
                               dv_part, dv, accumulate);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}
