// echo_common.cuh — shared device helpers for libecho (sm_100a).
//
// Storage-type abstraction (fp32 / bf16 storage, fp32 math), 128-bit vector
// load/store, the rounding contract (DESIGN.md a4: round once at production,
// every consumer reads the rounded value) and status plumbing.
//
// Bit-identity between STASH and RECOMPUTE rests on the device functions in
// this file and in the kernels being *the same code with the same operation
// order*; every floating-point step that could be contracted or reassociated
// is written with explicit round-to-nearest intrinsics (__fmaf_rn, __fmul_rn,
// __fadd_rn, __fdiv_rn), so nvcc cannot contract the two paths differently.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "../../include/echo.h"

namespace echo {

// ------------------------------------------------------------------ status plumbing
void set_error(const char* fmt, ...);
echo_status fail(echo_status s, const char* fmt, ...);
echo_status check_launch(const char* what);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ------------------------------------------------------------------ launches
// ECHO_PDL=1 launches every libecho kernel with programmatic stream serialization (PDL): the grid
// may be scheduled while its stream predecessor drains, and pdl_wait() -- the first statement of
// every kernel -- blocks until the predecessor has completed and its writes are visible, so results
// do not change.  Off by default: measured on the C2 step (CUDA graph, cuBLAS predecessors that
// never trigger early) it gained nothing (8.82 vs 8.86 ms bf16).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("ECHO_PDL");
    return e && e[0] == '1';
  }();
  return on;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// ------------------------------------------------------------------ bounded mbarrier waits
// Every mbarrier wait in libecho (TMA stage-in, st.async exchange, tcgen05 commit) goes through
// mbar_wait_bounded: the fast path is one try_wait; a phase still incomplete after ECHO_WAIT_NS of
// global time (a kernel bug: a lost arrive or a short transaction count) traps (no printf: it would
// cost registers in the launch-bounded kernels), so the launch fails with cudaErrorLaunchFailure instead of spinning until an external
// timeout kills the process.  Correct launches never get near the bound (the longest wait is a
// TMA stage-in or a peer CTA's exchange, microseconds).
#ifndef ECHO_WAIT_NS
#define ECHO_WAIT_NS 10000000000ull  // 10 s (compute-sanitizer and time-sliced contexts stretch waits)
#endif
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}
// SUSPEND_NS > 0: try_wait with a suspend-time hint (the thread sleeps until the phase completes or
// the hint expires instead of re-polling)
template <uint32_t SUSPEND_NS>
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  if (SUSPEND_NS > 0)
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(phase), "n"(SUSPEND_NS)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
  return ok != 0;
}
template <uint32_t SUSPEND_NS = 0>
__device__ __forceinline__ void mbar_wait_bounded(uint32_t bar, uint32_t phase) {
  if (mbar_try<SUSPEND_NS>(bar, phase)) return;
  const uint64_t t0 = globaltimer_ns();
  while (!mbar_try<SUSPEND_NS>(bar, phase)) {
    if (globaltimer_ns() - t0 > ECHO_WAIT_NS) __trap();
  }
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  unsigned na = 0;
  if (cluster > 1 || cluster < 0) {                   // cluster < 0: an explicit cluster of -cluster CTAs
    attr[na].id = cudaLaunchAttributeClusterDimension;  // (kernels using DSMEM / st.async even when 1 CTA)
    attr[na].val.clusterDim.x = (unsigned)(cluster < 0 ? -cluster : cluster);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ storage types
template <typename T> struct St;
template <> struct St<float> {
  static constexpr int VEC = 4;                      // elements per 16-byte vector
  __device__ static __forceinline__ float round(float x) { return x; }
};
template <> struct St<__nv_bfloat16> {
  static constexpr int VEC = 8;
  __device__ static __forceinline__ float round(float x) {
    return __bfloat162float(__float2bfloat16_rn(x));
  }
};

// 16-byte vector load of storage T -> VEC floats
__device__ __forceinline__ void ld16(const float* p, float (&o)[4]) {
  float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void ld16(const __nv_bfloat16* p, float (&o)[8]) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x; o[2 * i + 1] = f.y;
  }
}
// streaming (read-once) variant: bypass L1 allocation
__device__ __forceinline__ void ld16_stream(const float* p, float (&o)[4]) {
  float4 v = __ldcs(reinterpret_cast<const float4*>(p));
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void ld16_stream(const __nv_bfloat16* p, float (&o)[8]) {
  uint4 v = __ldcs(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x; o[2 * i + 1] = f.y;
  }
}
// L2-coherent variant (ld.global.cg: skips L1), for data another CTA wrote in this launch
__device__ __forceinline__ void ld16_cg(const float* p, float (&o)[4]) {
  float4 v = __ldcg(reinterpret_cast<const float4*>(p));
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void ld16_cg(const __nv_bfloat16* p, float (&o)[8]) {
  uint4 v = __ldcg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x; o[2 * i + 1] = f.y;
  }
}
// store VEC floats (already rounded to T) as storage T
__device__ __forceinline__ void st16(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void st16(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
// fp32 arrays of N = 4 or 8 floats (c, dc, dh are always fp32)
template <int N>
__device__ __forceinline__ void ldf(const float* p, float (&o)[N]) {
#pragma unroll
  for (int k = 0; k < N; k += 4) {
    float4 v = *reinterpret_cast<const float4*>(p + k);
    o[k] = v.x; o[k + 1] = v.y; o[k + 2] = v.z; o[k + 3] = v.w;
  }
}
template <int N>
__device__ __forceinline__ void stf(float* p, const float (&v)[N]) {
#pragma unroll
  for (int k = 0; k < N; k += 4) *reinterpret_cast<float4*>(p + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
}

// scalar storage <-> float
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// ------------------------------------------------------------------ math (IEEE, no fast-math)
// 1 / (1 + e^-x): __frcp_rn is the correctly rounded reciprocal, i.e. exactly __fdiv_rn(1, .)
// (same IEEE result) without the general-division sequence
__device__ __forceinline__ float sigmoidf_(float x) {
  return __frcp_rn(__fadd_rn(1.0f, expf(-x)));
}

// warp-wide sum with a fixed xor tree (deterministic, identical in every kernel)
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------------------------ counter-based dropout masks
// Philox4x32-10 (Random123); element n of a dropout site uses counter offset + n/4, key seed, word
// n%4, keep iff (word >> 8) >= thr = floor(p * 2^24) (reading R19).  Shared by a7 and the
// embedding dropout so every kernel derives the same bits.
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

// keep-bits of the 8 elements n0..n0+7 (n0 % 8 == 0), bit k = element n0 + k
__device__ __forceinline__ uint32_t keep_bits8(uint64_t seed, uint64_t offset, uint64_t n0, uint32_t thr) {
  const uint64_t q = offset + (n0 >> 2);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const U4 a = philox4x32_10(U4{(uint32_t)q, (uint32_t)(q >> 32), 0u, 0u}, k0, k1);
  const uint64_t q1 = q + 1;
  const U4 b = philox4x32_10(U4{(uint32_t)q1, (uint32_t)(q1 >> 32), 0u, 0u}, k0, k1);
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) bits |= ((w[k] >> 8) >= thr ? 1u : 0u) << k;
  return bits;
}

}  // namespace echo
