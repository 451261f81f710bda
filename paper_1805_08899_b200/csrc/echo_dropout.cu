// echo_dropout.cu — dropout on the LSTM path's inputs (the NMT embeddings; reading R31) with the
// paper's 1-bit encoding of the dropout feature map ("encodes the dropout
// feature maps to 1-bit in the forward pass and decodes them back to 32-bit in the backward
// pass"; Alg. 1 line 18) or, under reading R30, no stored mask at all (Philox is counter-based).
//
// One thread per chunk of 8 consecutive elements: the chunk's keep-bits are one mask byte (bit k
// = element n0 + k), the same keep_bits8 as a7.  HBM-bound elementwise work.
#include "echo_common.cuh"

namespace echo {

template <typename T>
__device__ __forceinline__ void ld8x(const T* p, float (&o)[8]);
template <>
__device__ __forceinline__ void ld8x<float>(const float* p, float (&o)[8]) {
  ldf<8>(p, o);
}
template <>
__device__ __forceinline__ void ld8x<__nv_bfloat16>(const __nv_bfloat16* p, float (&o)[8]) {
  ld16(p, o);
}
template <typename T>
__device__ __forceinline__ void st8x(T* p, const float (&v)[8]);
template <>
__device__ __forceinline__ void st8x<float>(float* p, const float (&v)[8]) {
  stf<8>(p, v);
}
template <>
__device__ __forceinline__ void st8x<__nv_bfloat16>(__nv_bfloat16* p, const float (&v)[8]) {
  st16(p, v);
}

// keep-bits of chunk n0: decoded from a kept mask (kind 1 bits, 2 bytes) or regenerated (kind 0)
__device__ __forceinline__ uint32_t chunk_bits(const uint8_t* mask, int kind, uint64_t seed, uint64_t offset,
                                               uint64_t n0, uint32_t thr, bool active) {
  if (!active) return 0xFFu;
  if (kind == 1) return mask[n0 >> 3];
  if (kind == 2) {
    const uint2 mb = *reinterpret_cast<const uint2*>(mask + n0);
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bits |= ((mb.x >> (8 * k)) & 1u) << k;
      bits |= ((mb.y >> (8 * k)) & 1u) << (k + 4);
    }
    return bits;
  }
  return keep_bits8(seed, offset, n0, thr);
}

// y = x * keep / (1 - p), rounded to y's storage type; keep from Philox, optionally written out
template <typename T>
__global__ void __launch_bounds__(256) dropout_fwd_kernel(long n8, uint64_t seed, uint64_t offset, uint32_t thr,
                                                          float ik, bool active, const T* __restrict__ x,
                                                          T* __restrict__ y, uint8_t* __restrict__ mask, int kind) {
  pdl_wait();
  for (long c = (long)blockIdx.x * blockDim.x + threadIdx.x; c < n8; c += (long)gridDim.x * blockDim.x) {
    const uint64_t n0 = (uint64_t)c * 8;
    const uint32_t bits = active ? keep_bits8(seed, offset, n0, thr) : 0xFFu;
    float v[8];
    ld8x<T>(x + n0, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = St<T>::round(__fmul_rn(v[k], ((bits >> k) & 1u) ? ik : 0.0f));
    st8x<T>(y + n0, v);
    if (kind == 1) {
      mask[c] = (uint8_t)bits;
    } else if (kind == 2) {
      uint2 mb;
      mb.x = ((bits >> 0) & 1u) | (((bits >> 1) & 1u) << 8) | (((bits >> 2) & 1u) << 16) | (((bits >> 3) & 1u) << 24);
      mb.y = ((bits >> 4) & 1u) | (((bits >> 5) & 1u) << 8) | (((bits >> 6) & 1u) << 16) | (((bits >> 7) & 1u) << 24);
      *reinterpret_cast<uint2*>(mask + n0) = mb;
    }
  }
}

// y (+)= x * keep / (1 - p) with keep decoded from the kept mask or regenerated: re-applies a
// mirrored dropout (x, y storage type) and back-propagates through it (x = dL/dy, y = dL/dx, fp32)
template <typename TX, typename TY>
__global__ void __launch_bounds__(256) dropout_apply_kernel(long n8, uint64_t seed, uint64_t offset, uint32_t thr,
                                                            float ik, bool active, const uint8_t* __restrict__ mask,
                                                            int kind, const TX* __restrict__ x, TY* y, int accumulate) {
  pdl_wait();
  for (long c = (long)blockIdx.x * blockDim.x + threadIdx.x; c < n8; c += (long)gridDim.x * blockDim.x) {
    const uint64_t n0 = (uint64_t)c * 8;
    const uint32_t bits = chunk_bits(mask, kind, seed, offset, n0, thr, active);
    float v[8];
    ld8x<TX>(x + n0, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __fmul_rn(v[k], ((bits >> k) & 1u) ? ik : 0.0f);
    if (accumulate) {
      float o[8];
      ld8x<TY>(y + n0, o);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __fadd_rn(o[k], v[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = St<TY>::round(v[k]);
    st8x<TY>(y + n0, v);
  }
}

static uint32_t drop_thr(float p) { return (uint32_t)floor((double)p * 16777216.0); }
static int drop_grid(long n8) {
  long g = (n8 + 255) / 256;
  return (int)(g < 148L * 16 ? (g > 0 ? g : 1) : 148L * 16);
}

}  // namespace echo

using namespace echo;

#define ECHO_DROP_CHECK()                                                                               \
  if (n <= 0 || n % 8) return fail(ECHO_ERR_INVALID, "%s: n=%lld must be a positive multiple of 8", fn, (long long)n); \
  if (!(p >= 0.0f && p < 1.0f)) return fail(ECHO_ERR_INVALID, "%s: p must be in [0,1)", fn);          \
  if (mask_kind < 0 || mask_kind > 2) return fail(ECHO_ERR_INVALID, "%s: bad mask_kind %d", fn, mask_kind); \
  if (mask_kind != 0 && !mask) return fail(ECHO_ERR_INVALID, "%s: mask is NULL", fn);                   \
  if (mask_kind == 2 && ((uintptr_t)mask & 7u)) return fail(ECHO_ERR_INVALID, "%s: byte mask must be 8-byte aligned", fn)

extern "C" echo_status echo_dropout_fwd(int64_t n, int32_t dtype, float p, uint64_t seed, uint64_t offset,
                                        const void* x, void* y, uint8_t* mask, int32_t mask_kind, void* stream) {
  const char* fn = "echo_dropout_fwd";
  ECHO_DROP_CHECK();
  if (dtype != ECHO_FP32 && dtype != ECHO_BF16) return fail(ECHO_ERR_INVALID, "%s: bad dtype %d", fn, dtype);
  if (!x || !y || !aligned16(x) || !aligned16(y)) return fail(ECHO_ERR_INVALID, "%s: x / y NULL or not 16-byte aligned", fn);
  const long n8 = (long)(n / 8);
  const float ik = (float)(1.0 / (1.0 - (double)p));
  cudaError_t e;
  if (dtype == ECHO_FP32)
    e = launch(dropout_fwd_kernel<float>, dim3(drop_grid(n8)), dim3(256), 0, (cudaStream_t)stream, 1, n8, seed, offset,
               drop_thr(p), ik, p > 0.0f, (const float*)x, (float*)y, mask, (int)mask_kind);
  else
    e = launch(dropout_fwd_kernel<__nv_bfloat16>, dim3(drop_grid(n8)), dim3(256), 0, (cudaStream_t)stream, 1, n8, seed,
               offset, drop_thr(p), ik, p > 0.0f, (const __nv_bfloat16*)x, (__nv_bfloat16*)y, mask, (int)mask_kind);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

extern "C" echo_status echo_dropout_apply(int64_t n, float p, uint64_t seed, uint64_t offset, const uint8_t* mask,
                                          int32_t mask_kind, int32_t x_dtype, const void* x, int32_t y_dtype, void* y,
                                          int32_t accumulate, void* stream) {
  const char* fn = "echo_dropout_apply";
  ECHO_DROP_CHECK();
  if ((x_dtype != ECHO_FP32 && x_dtype != ECHO_BF16) || (y_dtype != ECHO_FP32 && y_dtype != ECHO_BF16))
    return fail(ECHO_ERR_INVALID, "%s: bad dtype", fn);
  if (!x || !y || !aligned16(x) || !aligned16(y)) return fail(ECHO_ERR_INVALID, "%s: x / y NULL or not 16-byte aligned", fn);
  const long n8 = (long)(n / 8);
  const float ik = (float)(1.0 / (1.0 - (double)p));
  const dim3 g(drop_grid(n8));
  cudaStream_t st = (cudaStream_t)stream;
  typedef __nv_bfloat16 bf;
  const bool a = p > 0.0f;
  const uint32_t thr = drop_thr(p);
  cudaError_t e;
  if (x_dtype == ECHO_FP32 && y_dtype == ECHO_FP32)
    e = launch(dropout_apply_kernel<float, float>, g, dim3(256), 0, st, 1, n8, seed, offset, thr, ik, a, mask,
               (int)mask_kind, (const float*)x, (float*)y, (int)accumulate);
  else if (x_dtype == ECHO_BF16 && y_dtype == ECHO_BF16)
    e = launch(dropout_apply_kernel<bf, bf>, g, dim3(256), 0, st, 1, n8, seed, offset, thr, ik, a, mask,
               (int)mask_kind, (const bf*)x, (bf*)y, (int)accumulate);
  else if (x_dtype == ECHO_FP32)
    e = launch(dropout_apply_kernel<float, bf>, g, dim3(256), 0, st, 1, n8, seed, offset, thr, ik, a, mask,
               (int)mask_kind, (const float*)x, (bf*)y, (int)accumulate);
  else
    e = launch(dropout_apply_kernel<bf, float>, g, dim3(256), 0, st, 1, n8, seed, offset, thr, ik, a, mask,
               (int)mask_kind, (const bf*)x, (float*)y, (int)accumulate);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

// ================================================================ 1-bit feature maps of the fx pass
// Binarization (Alg. 1 line 18) of an arbitrary PyTorch graph's ReLU
// outputs and boolean dropout masks (fx_pass.py): a ReLU's gradient reads only
// the sign of its output, a dropout's only its keep-mask, so 1 bit per element is kept.
// pack: bit k of byte j = (x[8 j + k] > 0) (dtype 0 fp32, 1 bf16, 2 u8/bool: != 0)
// unpack: out[i] = bit i ? 1 : 0 in out's dtype (0 fp32, 1 bf16, 2 u8/bool)
namespace echo {
template <typename T>
__device__ __forceinline__ bool positive(T v) { return to_f(v) > 0.0f; }
template <>
__device__ __forceinline__ bool positive<uint8_t>(uint8_t v) { return v != 0; }

template <typename T>
__global__ void __launch_bounds__(256) sign_pack_kernel(long n, const T* __restrict__ x, uint8_t* __restrict__ bits) {
  pdl_wait();
  const long nb = (n + 7) / 8;
  for (long j = (long)blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (long)gridDim.x * blockDim.x) {
    uint32_t b = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long i = 8 * j + k;
      if (i < n && positive<T>(x[i])) b |= 1u << k;
    }
    bits[j] = (uint8_t)b;
  }
}
template <typename T>
__global__ void __launch_bounds__(256) bits_unpack_kernel(long n, const uint8_t* __restrict__ bits, T* __restrict__ out) {
  pdl_wait();
  const long nb = (n + 7) / 8;
  for (long j = (long)blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (long)gridDim.x * blockDim.x) {
    const uint32_t b = bits[j];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long i = 8 * j + k;
      if (i < n) {
        if constexpr (sizeof(T) == 1) out[i] = (T)((b >> k) & 1u);
        else out[i] = from_f<T>((b >> k) & 1u ? 1.0f : 0.0f);
      }
    }
  }
}
static int sp_grid(long n) {
  long g = ((n + 7) / 8 + 255) / 256;
  return (int)(g < 148L * 16 ? (g > 0 ? g : 1) : 148L * 16);
}
}  // namespace echo

extern "C" echo_status echo_sign_pack(int64_t n, int32_t dtype, const void* x, uint8_t* bits, void* stream) {
  using namespace echo;
  const char* fn = "echo_sign_pack";
  if (n <= 0 || !x || !bits) return fail(ECHO_ERR_INVALID, "%s: n=%lld, x / bits NULL", fn, (long long)n);
  cudaError_t e;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 0) e = launch(sign_pack_kernel<float>, dim3(sp_grid(n)), dim3(256), 0, st, 1, (long)n, (const float*)x, bits);
  else if (dtype == 1)
    e = launch(sign_pack_kernel<__nv_bfloat16>, dim3(sp_grid(n)), dim3(256), 0, st, 1, (long)n, (const __nv_bfloat16*)x, bits);
  else if (dtype == 2) e = launch(sign_pack_kernel<uint8_t>, dim3(sp_grid(n)), dim3(256), 0, st, 1, (long)n, (const uint8_t*)x, bits);
  else return fail(ECHO_ERR_INVALID, "%s: bad dtype %d", fn, dtype);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

extern "C" echo_status echo_bits_unpack(int64_t n, const uint8_t* bits, int32_t dtype, void* out, void* stream) {
  using namespace echo;
  const char* fn = "echo_bits_unpack";
  if (n <= 0 || !out || !bits) return fail(ECHO_ERR_INVALID, "%s: n=%lld, bits / out NULL", fn, (long long)n);
  cudaError_t e;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 0) e = launch(bits_unpack_kernel<float>, dim3(sp_grid(n)), dim3(256), 0, st, 1, (long)n, bits, (float*)out);
  else if (dtype == 1)
    e = launch(bits_unpack_kernel<__nv_bfloat16>, dim3(sp_grid(n)), dim3(256), 0, st, 1, (long)n, bits, (__nv_bfloat16*)out);
  else if (dtype == 2) e = launch(bits_unpack_kernel<uint8_t>, dim3(sp_grid(n)), dim3(256), 0, st, 1, (long)n, bits, (uint8_t*)out);
  else return fail(ECHO_ERR_INVALID, "%s: bad dtype %d", fn, dtype);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}
