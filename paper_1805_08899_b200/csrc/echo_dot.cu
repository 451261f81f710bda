// echo_dot.cu — dot-product attention softmax + dropout with 1-bit mask
// binarization (a7).  PAPER.md:726-728 ("encodes the dropout feature maps to
// 1-bit in the forward pass and decodes them back to 32-bit in the backward
// pass"), Alg. 1 line 18, Transformer result PAPER.md:1002.
//
// Design: one warp per row; a lane owns chunks of 8
// consecutive elements (two float4 / one 16-byte bf16 vector), so loads are
// coalesced 128-bit and each chunk's keep-bits form exactly one mask byte.
// The mask comes from Philox4x32-10 (two calls per chunk, counters
// offset + n/4 and +1), so it is a pure function of (seed, offset, index):
// RECOMPUTE keeps a 1-bit mask (the paper's binarized feature map) and the
// scores S; the backward regenerates P with the same device softmax.
#include <cmath>

#include "echo_common.cuh"

namespace echo {

// Philox4x32-10 and keep_bits8 live in echo_common.cuh (shared with the embedding dropout)

template <typename T> __device__ __forceinline__ void ld8(const T* p, float (&o)[8]);
template <> __device__ __forceinline__ void ld8<float>(const float* p, float (&o)[8]) {
  float a[4], b[4];
  ld16(p, a);
  ld16(p + 4, b);
#pragma unroll
  for (int k = 0; k < 4; ++k) { o[k] = a[k]; o[4 + k] = b[k]; }
}
template <> __device__ __forceinline__ void ld8<__nv_bfloat16>(const __nv_bfloat16* p, float (&o)[8]) { ld16(p, o); }
template <typename T> __device__ __forceinline__ void st8(T* p, const float (&v)[8]);
template <> __device__ __forceinline__ void st8<float>(float* p, const float (&v)[8]) {
  const float a[4] = {v[0], v[1], v[2], v[3]}, b[4] = {v[4], v[5], v[6], v[7]};
  st16(p, a);
  st16(p + 4, b);
}
template <> __device__ __forceinline__ void st8<__nv_bfloat16>(__nv_bfloat16* p, const float (&v)[8]) { st16(p, v); }

// The ONE row softmax (forward and backward): P = round_s(exp(z - max) / sum)
template <typename T, int CH>
__device__ __forceinline__ void row_softmax(const T* __restrict__ srow, int L, float scale, int lane, float (&P)[CH][8]) {
  float m = -INFINITY;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int j0 = (c * 32 + lane) * 8;
    if (j0 < L) {
      ld8<T>(srow + j0, P[c]);
#pragma unroll
      for (int k = 0; k < 8; ++k) { P[c][k] = __fmul_rn(scale, P[c][k]); m = fmaxf(m, P[c][k]); }
    }
  }
  m = warp_max(m);
  float sum = 0.0f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int j0 = (c * 32 + lane) * 8;
    if (j0 < L) {
#pragma unroll
      for (int k = 0; k < 8; ++k) { P[c][k] = expf(__fsub_rn(P[c][k], m)); sum = __fadd_rn(sum, P[c][k]); }
    }
  }
  sum = warp_sum(sum);
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) P[c][k] = St<T>::round(__fdiv_rn(P[c][k], sum));
}

__device__ __forceinline__ float drop(float p, uint32_t bits, int k, float inv_keep) {
  return __fmul_rn(p, ((bits >> k) & 1u) ? inv_keep : 0.0f);
}

template <typename T, int CH>
__global__ void __launch_bounds__(256) dot_fwd_kernel(echo_dot_desc d, uint32_t thr, float inv_keep,
                                                      const T* __restrict__ S, T* __restrict__ Pd,
                                                      T* __restrict__ P_st, uint8_t* __restrict__ mask) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  const int L = d.L;
  for (long r = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < d.R; r += nwarps) {
    float P[CH][8];
    row_softmax<T, CH>(S + r * L, L, d.scale, lane, P);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int j0 = (c * 32 + lane) * 8;
      if (j0 >= L) continue;
      const uint64_t n0 = (uint64_t)r * L + j0;
      const uint32_t bits = d.dropout_p > 0.0f ? keep_bits8(d.seed, d.offset, n0, thr) : 0xFFu;
      float pd[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pd[k] = St<T>::round(drop(P[c][k], bits, k, inv_keep));
      st8<T>(Pd + n0, pd);
      if (P_st) {  // STASH: P, byte mask
        st8<T>(P_st + n0, P[c]);
        uint2 mb;
        mb.x = ((bits >> 0) & 1u) | (((bits >> 1) & 1u) << 8) | (((bits >> 2) & 1u) << 16) | (((bits >> 3) & 1u) << 24);
        mb.y = ((bits >> 4) & 1u) | (((bits >> 5) & 1u) << 8) | (((bits >> 6) & 1u) << 16) | (((bits >> 7) & 1u) << 24);
        *reinterpret_cast<uint2*>(mask + n0) = mb;
      } else if (mask) {     // RECOMPUTE: 1-bit mask (NULL: regenerated in the backward)
        mask[n0 >> 3] = (uint8_t)bits;
      }
    }
  }
}

template <typename T, int CH>
__global__ void __launch_bounds__(256) dot_bwd_kernel(echo_dot_desc d, uint32_t thr, float inv_keep,
                                                      const T* __restrict__ S,
                                                      const T* __restrict__ P_st, const uint8_t* __restrict__ mask,
                                                      const T* dPd, T* dS, T* __restrict__ Pd_regen) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  const int L = d.L;
  for (long r = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < d.R; r += nwarps) {
    float P[CH][8];
    uint32_t bits[CH];
    if (P_st) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int j0 = (c * 32 + lane) * 8;
        bits[c] = 0;
        if (j0 < L) {
          const uint64_t n0 = (uint64_t)r * L + j0;
          ld8<T>(P_st + n0, P[c]);
          const uint2 mb = *reinterpret_cast<const uint2*>(mask + n0);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            bits[c] |= ((mb.x >> (8 * k)) & 1u) << k;
            bits[c] |= ((mb.y >> (8 * k)) & 1u) << (k + 4);
          }
        }
      }
    } else {
      row_softmax<T, CH>(S + r * L, L, d.scale, lane, P);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int j0 = (c * 32 + lane) * 8;
        if (j0 >= L) bits[c] = 0u;
        else if (mask) bits[c] = (uint32_t)mask[((uint64_t)r * L + j0) >> 3];
        else bits[c] = d.dropout_p > 0.0f ? keep_bits8(d.seed, d.offset, (uint64_t)r * L + j0, thr) : 0xFFu;
      }
    }
    float dP[CH][8];
    float dot = 0.0f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int j0 = (c * 32 + lane) * 8;
      if (j0 < L) {
        ld8<T>(dPd + (uint64_t)r * L + j0, dP[c]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          dP[c][k] = drop(dP[c][k], bits[c], k, inv_keep);
          dot = __fmaf_rn(P[c][k], dP[c][k], dot);
        }
      }
    }
    dot = warp_sum(dot);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int j0 = (c * 32 + lane) * 8;
      if (j0 >= L) continue;
      const uint64_t n0 = (uint64_t)r * L + j0;
      float ds[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) ds[k] = St<T>::round(__fmul_rn(d.scale, __fmul_rn(P[c][k], __fsub_rn(dP[c][k], dot))));
      st8<T>(dS + n0, ds);
      if (Pd_regen) {
        float pd[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) pd[k] = St<T>::round(drop(P[c][k], bits[c], k, inv_keep));
        st8<T>(Pd_regen + n0, pd);
      }
    }
  }
}

static echo_status check_dot(const char* fn, const echo_dot_desc* d) {
  if (!d) return fail(ECHO_ERR_INVALID, "%s: desc is NULL", fn);
  if (d->R <= 0 || d->L <= 0) return fail(ECHO_ERR_INVALID, "%s: R=%d L=%d must be > 0", fn, d->R, d->L);
  if (d->L % 8) return fail(ECHO_ERR_INVALID, "%s: L=%d must be a multiple of 8", fn, d->L);
  if (d->L > 2048) return fail(ECHO_ERR_CAPACITY, "%s: L=%d exceeds 2048", fn, d->L);
  if (d->dtype != ECHO_FP32 && d->dtype != ECHO_BF16) return fail(ECHO_ERR_INVALID, "%s: bad dtype", fn);
  if (d->mode != ECHO_STASH && d->mode != ECHO_RECOMPUTE) return fail(ECHO_ERR_INVALID, "%s: bad mode", fn);
  if (!(d->dropout_p >= 0.0f && d->dropout_p < 1.0f)) return fail(ECHO_ERR_INVALID, "%s: dropout_p must be in [0,1)", fn);
  return ECHO_OK;
}

static int dot_grid(int R) {
  const long g = ((long)R + 7) / 8;
  return (int)(g < 148L * 32 ? g : 148L * 32);
}

}  // namespace echo

using namespace echo;

#define ECHO_REQ(p, name)                                                                     \
  do {                                                                                        \
    if (!(p)) return fail(ECHO_ERR_INVALID, "%s: required pointer %s is NULL", fn, name);     \
    if (!aligned16(p)) return fail(ECHO_ERR_INVALID, "%s: %s is not 16-byte aligned", fn, name); \
  } while (0)

template <typename T>
static void launch_fwd(const echo_dot_desc* d, uint32_t thr, float ik, const void* S, void* Pd, void* P_st,
                       uint8_t* mask, cudaStream_t st) {
  const int ch = (d->L + 255) / 256;
  const int grid = dot_grid(d->R);
#define L_(CH) (void)launch(dot_fwd_kernel<T, CH>, dim3(grid), dim3(256), 0, st, 1, *d, thr, ik, (const T*)S, (T*)Pd, \
                         (T*)P_st, mask)
  if (ch <= 1) L_(1); else if (ch <= 2) L_(2); else if (ch <= 4) L_(4); else L_(8);
#undef L_
}

static uint32_t keep_thr(float p) { return (uint32_t)floor((double)p * 16777216.0); }

template <typename T>
static void launch_bwd(const echo_dot_desc* d, uint32_t thr, float ik, const void* S, const void* P_st,
                       const uint8_t* mask, const void* dPd, void* dS, void* Pdr, cudaStream_t st) {
  const int ch = (d->L + 255) / 256;
  const int grid = dot_grid(d->R);
#define L_(CH) (void)launch(dot_bwd_kernel<T, CH>, dim3(grid), dim3(256), 0, st, 1, *d, thr, ik, (const T*)S, \
                         (const T*)P_st, mask, (const T*)dPd, (T*)dS, (T*)Pdr)
  if (ch <= 1) L_(1); else if (ch <= 2) L_(2); else if (ch <= 4) L_(4); else L_(8);
#undef L_
}

extern "C" echo_status echo_dot_softmax_fwd(const echo_dot_desc* d, const void* S, void* Pd, void* P_st, uint8_t* mask,
                                            void* stream) {
  const char* fn = "echo_dot_softmax_fwd";
  echo_status s = check_dot(fn, d);
  if (s) return s;
  ECHO_REQ(S, "S");
  ECHO_REQ(Pd, "Pd");
  if (!mask && d->mode == ECHO_STASH) return fail(ECHO_ERR_INVALID, "%s: mask is NULL in STASH mode", fn);
  if (d->mode == ECHO_STASH) {
    ECHO_REQ(P_st, "P_st");
    if ((reinterpret_cast<uintptr_t>(mask) & 7u) != 0) return fail(ECHO_ERR_INVALID, "%s: byte mask must be 8-byte aligned", fn);
  } else if (P_st) {
    return fail(ECHO_ERR_INVALID, "%s: P_st must be NULL in RECOMPUTE mode", fn);
  }
  const float ik = (float)(1.0 / (1.0 - (double)d->dropout_p));
  if (d->dtype == ECHO_FP32) launch_fwd<float>(d, keep_thr(d->dropout_p), ik, S, Pd, P_st, mask, (cudaStream_t)stream);
  else launch_fwd<__nv_bfloat16>(d, keep_thr(d->dropout_p), ik, S, Pd, P_st, mask, (cudaStream_t)stream);
  return check_launch(fn);
}

extern "C" echo_status echo_dot_softmax_bwd(const echo_dot_desc* d, const void* S, const void* P_st,
                                            const uint8_t* mask, const void* dPd, void* dS, void* Pd_regen,
                                            void* stream) {
  const char* fn = "echo_dot_softmax_bwd";
  echo_status s = check_dot(fn, d);
  if (s) return s;
  ECHO_REQ(dPd, "dPd");
  ECHO_REQ(dS, "dS");
  if (!mask && d->mode == ECHO_STASH) return fail(ECHO_ERR_INVALID, "%s: mask is NULL in STASH mode", fn);
  if (d->mode == ECHO_STASH) {
    ECHO_REQ(P_st, "P_st");
    if (Pd_regen) return fail(ECHO_ERR_INVALID, "%s: Pd_regen must be NULL in STASH mode", fn);
  } else {
    ECHO_REQ(S, "S");
    if (P_st) return fail(ECHO_ERR_INVALID, "%s: P_st must be NULL in RECOMPUTE mode", fn);
    if (Pd_regen && !aligned16(Pd_regen)) return fail(ECHO_ERR_INVALID, "%s: Pd_regen not 16-byte aligned", fn);
  }
  const float ik = (float)(1.0 / (1.0 - (double)d->dropout_p));
  const uint32_t thr = keep_thr(d->dropout_p);
  if (d->dtype == ECHO_FP32) launch_bwd<float>(d, thr, ik, S, P_st, mask, dPd, dS, Pd_regen, (cudaStream_t)stream);
  else launch_bwd<__nv_bfloat16>(d, thr, ik, S, P_st, mask, dPd, dS, Pd_regen, (cudaStream_t)stream);
  return check_launch(fn);
}
