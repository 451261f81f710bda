// echo_attn.cu — MLP attention forward (a5) and backward with fused
// recomputation (a6).  PAPER.md §2 lines 129-133 (scores, weights alpha_ts,
// context as the alpha-weighted average of H_s) and Fig. 7 / Fig. 10
// (PAPER.md:360, 633): the broadcast-add + tanh feature maps E [B,Ts,A] are the
// largest stash of the NMT model; Echo keeps them mirrored and
// regenerates them in the backward pass.
//
// Design: one CTA per batch row b (the rows are
// independent; per-row work is a [Ts x A] + [Ts x Hk] stream).  Warp w owns
// source positions s = w, w + NW, ...; a lane owns 16-byte vectors of the A /
// Hk axis, so each warp-wide access is a coalesced 512-byte (fp32) row
// segment.  Scores use a fixed-order per-lane FMA chain + fixed xor-shuffle
// tree; the softmax and the context reduction are the SAME device functions
// with the SAME thread mapping in the forward and backward kernels, which is
// what makes the regenerated alpha / ctx bit-identical to the stashed ones.
// dv is produced as per-row partials (no atomics) and reduced in fixed order.
#include <cmath>

#include "echo_common.cuh"

namespace echo {

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
      acc = __fmaf_rn(tanhf(z[k]), v_s[iv * V + k], acc);
    }
    if (Z_out) st16(Z_out + iv * V, z);
  }
  return warp_sum(acc);
}

// In-place: sc[0..n) scores -> alpha; sc[n..Ts) = 0.  Executed by ONE warp.
__device__ __forceinline__ void softmax_warp(float* sc, int n, int Ts, int lane) {
  float m = -INFINITY;
  for (int s = lane; s < n; s += 32) m = fmaxf(m, sc[s]);
  m = warp_max(m);
  float sum = 0.0f;
  for (int s = lane; s < n; s += 32) {
    const float e = expf(__fsub_rn(sc[s], m));
    sc[s] = e;
    sum = __fadd_rn(sum, e);
  }
  sum = warp_sum(sum);
  for (int s = lane; s < n; s += 32) sc[s] = __fdiv_rn(sc[s], sum);
  for (int s = n + lane; s < Ts; s += 32) sc[s] = 0.0f;
}

__host__ __device__ __forceinline__ int ctx_groups(int Hk, int V) {
  const int ncols = Hk / V;
  return ncols >= ATT_THREADS ? 1 : ATT_THREADS / ncols;
}

// ctx = sum_{s<n} alpha_s Hs_s : G thread groups split s, fixed-order combine.
template <typename T>
__device__ __forceinline__ void context(const T* __restrict__ hs_b, long stride_s, const float* alpha, int n, int Hk,
                                        float* part, T* ctx_out, int tid) {
  constexpr int V = St<T>::VEC;
  const int ncols = Hk / V;
  const int G = ctx_groups(Hk, V);
  if (G > 1) {
    const int g = tid / ncols, cv = tid - (tid / ncols) * ncols;
    if (g < G) {
      float acc[V];
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = 0.0f;
      for (int s = g; s < n; s += G) {
        float h[V];
        ld16(hs_b + (long)s * stride_s + cv * V, h);
        const float a = alpha[s];
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
      for (int s = 0; s < n; ++s) {
        float h[V];
        ld16(hs_b + (long)s * stride_s + cv * V, h);
        const float a = alpha[s];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = __fmaf_rn(a, h[k], acc[k]);
      }
#pragma unroll
      for (int k = 0; k < V; ++k) part[cv * V + k] = acc[k];
    }
  }
  __syncthreads();
  if (ctx_out) {
    for (int cv = tid; cv < ncols; cv += ATT_THREADS) {
      float r[V];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        float x = part[cv * V + k];
        for (int g = 1; g < G; ++g) x = __fadd_rn(x, part[g * Hk + cv * V + k]);
        r[k] = St<T>::round(x);
      }
      st16(ctx_out + cv * V, r);
    }
  }
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

// ---------------------------------------------------------------- a5 forward
template <typename T>
__global__ void __launch_bounds__(ATT_THREADS) attn_fwd_kernel(echo_attn_desc d, const T* __restrict__ qp,
                                                               const T* __restrict__ Kp, const T* __restrict__ v,
                                                               const T* __restrict__ Hs,
                                                               const int32_t* __restrict__ src_len,
                                                               T* __restrict__ ctx, T* __restrict__ E_st,
                                                               float* __restrict__ alpha_st) {
  extern __shared__ float sm[];
  const int A = d.A, Ts = d.Ts, Hk = d.Hk;
  float* qp_s = sm;
  float* v_s = qp_s + A;
  float* sc = v_s + A;
  float* part = sc + ((Ts + 3) & ~3);
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = row_len(src_len, b, Ts);
  stage_vec<T>(qp_s, qp + (long)b * A, A, tid);
  stage_vec<T>(v_s, v, A, tid);
  __syncthreads();
  const T* kp_b = Kp + (long)b * d.kp_stride_b;
  for (int s = w; s < n; s += ATT_WARPS) {
    T* e_out = E_st ? E_st + ((long)b * Ts + s) * A : nullptr;
    const float scv = score_row<T>(kp_b + (long)s * d.kp_stride_s, qp_s, v_s, A, lane, e_out);
    if (lane == 0) sc[s] = scv;
  }
  if (E_st) {  // masked positions hold zeros (as the oracle's E)
    constexpr int V = St<T>::VEC;
    float z[V];
#pragma unroll
    for (int k = 0; k < V; ++k) z[k] = 0.0f;
    for (int s = n + w; s < Ts; s += ATT_WARPS)
      for (int iv = lane; iv < A / V; iv += 32) st16(E_st + ((long)b * Ts + s) * A + iv * V, z);
  }
  __syncthreads();
  if (w == 0) softmax_warp(sc, n, Ts, lane);
  __syncthreads();
  if (alpha_st)
    for (int s = tid; s < Ts; s += ATT_THREADS) alpha_st[(long)b * Ts + s] = sc[s];
  context<T>(Hs + (long)b * d.hs_stride_b, d.hs_stride_s, sc, n, Hk, part, ctx + (long)b * Hk, tid);
}

// ---------------------------------------------------------------- a6 backward (fused recompute)
template <typename T>
__global__ void __launch_bounds__(ATT_THREADS) attn_bwd_kernel(echo_attn_desc d, const T* __restrict__ qp,
                                                               const T* __restrict__ Kp, const T* __restrict__ v,
                                                               const T* __restrict__ Hs,
                                                               const int32_t* __restrict__ src_len,
                                                               const T* __restrict__ E_st,
                                                               const float* __restrict__ alpha_st,
                                                               const float* __restrict__ dctx, float* __restrict__ dqp,
                                                               float* __restrict__ dKp, float* __restrict__ dHs,
                                                               float* __restrict__ dv_part, T* __restrict__ ctx_regen) {
  constexpr int V = St<T>::VEC;
  extern __shared__ float sm[];
  const int A = d.A, Ts = d.Ts, Hk = d.Hk;
  const int Tp = (Ts + 3) & ~3;
  float* qp_s = sm;
  float* v_s = qp_s + A;
  float* dctx_s = v_s + A;
  float* sc = dctx_s + Hk;           // scores -> alpha
  float* dal = sc + Tp;              // dLoss/dalpha
  float* red = dal + Tp;             // [0] = sum_s alpha_s dalpha_s
  float* wq = red + 4;               // [NW][A] per-warp dqp partials
  float* wv = wq + ATT_WARPS * A;    // [NW][A] per-warp dv partials
  float* part = wv + ATT_WARPS * A;  // [G][Hk] context partials
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = row_len(src_len, b, Ts);
  const bool recompute = (E_st == nullptr);
  if (recompute) stage_vec<T>(qp_s, qp + (long)b * A, A, tid);
  stage_vec<T>(v_s, v, A, tid);
  for (int i = tid; i < Hk; i += ATT_THREADS) dctx_s[i] = dctx[(long)b * Hk + i];
  for (int i = tid; i < ATT_WARPS * A; i += ATT_THREADS) { wq[i] = 0.0f; wv[i] = 0.0f; }
  __syncthreads();
  const T* kp_b = Kp + (long)b * d.kp_stride_b;
  const T* hs_b = Hs + (long)b * d.hs_stride_b;
  // phase 1: regenerate scores (RECOMPUTE) and dalpha_s = dctx . Hs_s
  for (int s = w; s < n; s += ATT_WARPS) {
    if (recompute) {
      const float scv = score_row<T>(kp_b + (long)s * d.kp_stride_s, qp_s, v_s, A, lane, nullptr);
      if (lane == 0) sc[s] = scv;
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
    if (lane == 0) dal[s] = acc;
  }
  if (!recompute)
    for (int s = tid; s < Ts; s += ATT_THREADS) sc[s] = alpha_st[(long)b * Ts + s];
  __syncthreads();
  // phase 2: softmax (same device function as a5)
  if (recompute && w == 0) softmax_warp(sc, n, Ts, lane);
  __syncthreads();
  // phase 3: regenerate ctx (same device function and mapping as a5)
  if (recompute && ctx_regen) {
    context<T>(hs_b, d.hs_stride_s, sc, n, Hk, part, ctx_regen + (long)b * Hk, tid);
  }
  if (w == 0) {
    float acc = 0.0f;
    for (int s = lane; s < n; s += 32) acc = __fmaf_rn(sc[s], dal[s], acc);
    acc = warp_sum(acc);
    if (lane == 0) red[0] = acc;
  }
  __syncthreads();
  const float dot = red[0];
  // phase 4: ds, dE, dKp +=, dHs +=, dqp / dv partials
  float* wq_w = wq + w * A;
  float* wv_w = wv + w * A;
  for (int s = w; s < n; s += ATT_WARPS) {
    const float al = sc[s];
    const float ds = __fmul_rn(al, __fsub_rn(dal[s], dot));
    const T* kp_row = kp_b + (long)s * d.kp_stride_s;
    float* dkp_row = dKp + (long)b * d.kp_stride_b + (long)s * d.kp_stride_s;
    const T* e_row = E_st ? E_st + ((long)b * Ts + s) * A : nullptr;
    for (int iv = lane; iv < A / V; iv += 32) {
      float z[V];
      if (recompute) {
        float kv[V];
        ld16(kp_row + iv * V, kv);
#pragma unroll
        for (int k = 0; k < V; ++k) z[k] = St<T>::round(__fadd_rn(qp_s[iv * V + k], kv[k]));
      } else {
        ld16(e_row + iv * V, z);
      }
      float e[V];
#pragma unroll
      for (int k = 0; k < V; ++k) e[k] = tanhf(z[k]);
      float dk[V];
      ldf<V>(dkp_row + iv * V, dk);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float dE = __fmul_rn(__fmul_rn(ds, v_s[iv * V + k]), __fsub_rn(1.0f, __fmul_rn(e[k], e[k])));
        dk[k] = __fadd_rn(dk[k], dE);
        wq_w[iv * V + k] = __fadd_rn(wq_w[iv * V + k], dE);
        wv_w[iv * V + k] = __fmaf_rn(ds, e[k], wv_w[iv * V + k]);
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
    dqp[(long)b * A + a] = q;
    dv_part[(long)b * A + a] = __fadd_rn(dv_part[(long)b * A + a], vv);
  }
}

__global__ void dv_reduce_kernel(int B, int A, const float* __restrict__ part, float* __restrict__ dv, int acc) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  float x = acc ? dv[a] : 0.0f;
  for (int b = 0; b < B; ++b) x = __fadd_rn(x, part[(long)b * A + a]);
  dv[a] = x;
}

// ---------------------------------------------------------------- host side
static size_t fwd_smem(const echo_attn_desc* d) {
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  const int G = ctx_groups(d->Hk, V);
  return sizeof(float) * (2 * (size_t)d->A + ((d->Ts + 3) & ~3) + (size_t)G * d->Hk);
}
static size_t bwd_smem(const echo_attn_desc* d) {
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  const int G = ctx_groups(d->Hk, V);
  return sizeof(float) * (2 * (size_t)d->A + d->Hk + 2 * (size_t)((d->Ts + 3) & ~3) + 4 +
                          2 * (size_t)ATT_WARPS * d->A + (size_t)G * d->Hk);
}

static echo_status check_attn(const char* fn, const echo_attn_desc* d) {
  if (!d) return fail(ECHO_ERR_INVALID, "%s: desc is NULL", fn);
  if (d->B <= 0 || d->Ts <= 0 || d->A <= 0 || d->Hk <= 0)
    return fail(ECHO_ERR_INVALID, "%s: B=%d Ts=%d A=%d Hk=%d must be > 0", fn, d->B, d->Ts, d->A, d->Hk);
  if (d->A % 8 || d->Hk % 8) return fail(ECHO_ERR_INVALID, "%s: A=%d and Hk=%d must be multiples of 8", fn, d->A, d->Hk);
  if (d->Ts > 4096) return fail(ECHO_ERR_CAPACITY, "%s: Ts=%d exceeds 4096", fn, d->Ts);
  if (d->dtype != ECHO_FP32 && d->dtype != ECHO_BF16) return fail(ECHO_ERR_INVALID, "%s: bad dtype %d", fn, d->dtype);
  if (d->mode != ECHO_STASH && d->mode != ECHO_RECOMPUTE) return fail(ECHO_ERR_INVALID, "%s: bad mode %d", fn, d->mode);
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  if (d->kp_stride_b % V || d->kp_stride_s % V || d->hs_stride_b % V || d->hs_stride_s % V)
    return fail(ECHO_ERR_INVALID, "%s: strides must be multiples of %d elements", fn, V);
  if (d->kp_stride_b <= 0 || d->kp_stride_s <= 0 || d->hs_stride_b <= 0 || d->hs_stride_s <= 0)
    return fail(ECHO_ERR_INVALID, "%s: strides must be > 0", fn);
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
  const size_t smem = fwd_smem(d);
  cudaStream_t st = (cudaStream_t)stream;
  if (d->dtype == ECHO_FP32) {
    if ((s = set_smem((const void*)attn_fwd_kernel<float>, smem, fn))) return s;
    attn_fwd_kernel<float><<<d->B, ATT_THREADS, smem, st>>>(*d, (const float*)qp, (const float*)Kp, (const float*)v,
                                                            (const float*)Hs, src_len, (float*)ctx, (float*)E_st,
                                                            alpha_st);
  } else {
    typedef __nv_bfloat16 bf;
    if ((s = set_smem((const void*)attn_fwd_kernel<bf>, smem, fn))) return s;
    attn_fwd_kernel<bf><<<d->B, ATT_THREADS, smem, st>>>(*d, (const bf*)qp, (const bf*)Kp, (const bf*)v, (const bf*)Hs,
                                                         src_len, (bf*)ctx, (bf*)E_st, alpha_st);
  }
  return check_launch(fn);
}

extern "C" echo_status echo_attn_bwd(const echo_attn_desc* d, const void* qp, const void* Kp, const void* v,
                                     const void* Hs, const int32_t* src_len, const void* E_st,
                                     const float* alpha_st, const float* dctx, float* dqp, float* dKp, float* dHs,
                                     float* dv_part, void* ctx_regen, void* stream) {
  const char* fn = "echo_attn_bwd";
  echo_status s = check_attn(fn, d);
  if (s) return s;
  ECHO_REQ(v, "v");
  ECHO_REQ(Hs, "Hs");
  ECHO_REQ(dctx, "dctx");
  ECHO_REQ(dqp, "dqp");
  ECHO_REQ(dKp, "dKp");
  ECHO_REQ(dHs, "dHs");
  ECHO_REQ(dv_part, "dv_part");
  if (d->mode == ECHO_STASH) {
    ECHO_REQ(E_st, "E_st");
    if (!alpha_st) return fail(ECHO_ERR_INVALID, "%s: alpha_st required in STASH mode", fn);
    if (ctx_regen) return fail(ECHO_ERR_INVALID, "%s: ctx_regen must be NULL in STASH mode", fn);
  } else {
    ECHO_REQ(qp, "qp");
    ECHO_REQ(Kp, "Kp");
    if (E_st || alpha_st) return fail(ECHO_ERR_INVALID, "%s: E_st / alpha_st must be NULL in RECOMPUTE mode", fn);
    if (ctx_regen && !aligned16(ctx_regen)) return fail(ECHO_ERR_INVALID, "%s: ctx_regen not 16-byte aligned", fn);
  }
  const size_t smem = bwd_smem(d);
  cudaStream_t st = (cudaStream_t)stream;
  if (d->dtype == ECHO_FP32) {
    if ((s = set_smem((const void*)attn_bwd_kernel<float>, smem, fn))) return s;
    attn_bwd_kernel<float><<<d->B, ATT_THREADS, smem, st>>>(*d, (const float*)qp, (const float*)Kp, (const float*)v,
                                                            (const float*)Hs, src_len, (const float*)E_st, alpha_st,
                                                            dctx, dqp, dKp, dHs, dv_part, (float*)ctx_regen);
  } else {
    typedef __nv_bfloat16 bf;
    if ((s = set_smem((const void*)attn_bwd_kernel<bf>, smem, fn))) return s;
    attn_bwd_kernel<bf><<<d->B, ATT_THREADS, smem, st>>>(*d, (const bf*)qp, (const bf*)Kp, (const bf*)v, (const bf*)Hs,
                                                         src_len, (const bf*)E_st, alpha_st, dctx, dqp, dKp, dHs,
                                                         dv_part, (bf*)ctx_regen);
  }
  return check_launch(fn);
}

extern "C" echo_status echo_attn_dv_reduce(int32_t B, int32_t A, const float* dv_part, float* dv, int32_t accumulate,
                                           void* stream) {
  const char* fn = "echo_attn_dv_reduce";
  if (B <= 0 || A <= 0) return fail(ECHO_ERR_INVALID, "%s: B=%d A=%d must be > 0", fn, B, A);
  if (!dv_part || !dv) return fail(ECHO_ERR_INVALID, "%s: NULL pointer", fn);
  dv_reduce_kernel<<<(A + 127) / 128, 128, 0, (cudaStream_t)stream>>>(B, A, dv_part, dv, accumulate);
  return check_launch(fn);
}
