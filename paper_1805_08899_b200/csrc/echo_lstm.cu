// echo_lstm.cu — LSTM non-linear block: forward (a1), c-regeneration scan (a2)
// and backward with fused recomputation (a3).  PAPER.md §2
// (Fig. 1), Echo's mirrored c-chain (Fig. 4 step 4) and the
// hand-fused recompute kernels Echo-dagger.
//
// Design: HBM-bound elementwise work, so no tensor
// cores and no shared memory — each thread owns one 16-byte vector of the
// hidden axis (4 fp32 or 8 bf16 columns) for one batch row and reads the four
// gate blocks i|f|g|o with coalesced 128-bit loads.  Grids are sized in
// multiples of the 148 SMs.  The scan (a2) owns (b, j) per thread, carries c in
// registers across t and keeps U time steps of loads in flight.
#include "echo_common.cuh"

#include <cooperative_groups.h>
#include <cuda.h>
#include <type_traits>

namespace echo {

namespace cg = cooperative_groups;

// ---------------------------------------------------------------- shared device functions
// The ONE definition of the cell-state update used by a1 (forward) and a2
// (recompute scan): c_t = f * c_{t-1} + i * g with a pinned FMA.
__device__ __forceinline__ float cell_update(float f, float c_prev, float i, float g) {
  return __fmaf_rn(f, c_prev, __fmul_rn(i, g));
}

template <typename T>
__device__ __forceinline__ float tanh_c(float c) { return St<T>::round(tanhf(c)); }

template <typename T>
__device__ __forceinline__ float hidden(float o, float tc) { return St<T>::round(__fmul_rn(o, tc)); }

// The ONE definition of the activated gates from the pre-activation A (a1, and the Mirror-plan
// kernels that regenerate A from its parts)
template <typename T>
__device__ __forceinline__ void gates_of(float ai, float af, float ag, float ao, float& gi, float& gf, float& gg,
                                         float& go) {
  gi = St<T>::round(sigmoidf_(ai));
  gf = St<T>::round(sigmoidf_(af));
  gg = St<T>::round(tanhf(ag));
  go = St<T>::round(sigmoidf_(ao));
}

// The ONE definition of the cell's backward (a3 and the Mirror-plan backward): from the gates,
// c_{t-1}, tanh(c_t), dh_t and the carried dc, the pre-activation gradients and the new carry
//   do = dh tc ; dc = carry + dh o (1 - tc^2) ; di = dc g ; dg = dc i ; df = dc c_{t-1} ; carry' = dc f
template <typename T>
__device__ __forceinline__ void cell_grad(float gi, float gf, float gg, float go, float cp, float tc, float dhv,
                                          float dcv, float& di, float& df, float& dg, float& dout, float& dcn) {
  const float d_o = __fmul_rn(dhv, tc);
  const float one_m_tc2 = __fsub_rn(1.0f, __fmul_rn(tc, tc));
  const float dcc = __fadd_rn(dcv, __fmul_rn(__fmul_rn(dhv, go), one_m_tc2));
  const float d_i = __fmul_rn(dcc, gg);
  const float d_g = __fmul_rn(dcc, gi);
  const float d_f = __fmul_rn(dcc, cp);
  dcn = __fmul_rn(dcc, gf);
  di = St<T>::round(__fmul_rn(d_i, __fmul_rn(gi, __fsub_rn(1.0f, gi))));
  df = St<T>::round(__fmul_rn(d_f, __fmul_rn(gf, __fsub_rn(1.0f, gf))));
  dg = St<T>::round(__fmul_rn(d_g, __fsub_rn(1.0f, __fmul_rn(gg, gg))));
  dout = St<T>::round(__fmul_rn(d_o, __fmul_rn(go, __fsub_rn(1.0f, go))));
}

// per-step kernels (a1 / a3) at small B*H are latency-bound: spread the threads over more SMs
// with smaller blocks (64 threads when there are fewer than 148 x 128 threads); ECHO_LSTM_BLOCK
// overrides (A/B measurements)
static int step_block(long threads) {
  static const int forced = [] {
    const char* e = getenv("ECHO_LSTM_BLOCK");
    return e ? atoi(e) : 0;
  }();
  if (forced == 32 || forced == 64 || forced == 128) return forced;
  return threads >= 148L * 128 ? 128 : 64;
}

// per-step a1 / a3 vector width (elements per thread): the widest 16/8/4-byte vector that still
// yields >= 148 x 256 threads (ECHO_LSTM_VEC=N forces N); bf16 stays >= 2 elements (4 bytes)
static int step_vec(long elems, bool bf) {
  static const int forced = [] {
    const char* e = getenv("ECHO_LSTM_VEC");
    return e ? atoi(e) : 0;
  }();
  const int vmax = bf ? 8 : 4, vmin = bf ? 2 : 1;
  if (forced >= vmin && forced <= vmax && (forced & (forced - 1)) == 0) return forced;
  int v = vmax;
  while (v > vmin && elems / v < 148L * 256) v >>= 1;
  return v;
}

static int grid_for(long threads, int block) {
  static const long cap = [] {                 // grid-stride loops above the cap (ECHO_LSTM_GRIDCAP, CTAs)
    const char* e = getenv("ECHO_LSTM_GRIDCAP");
    return e && atol(e) > 0 ? atol(e) : 148L * 16;
  }();
  long g = (threads + block - 1) / block;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

// ---------------------------------------------------------------- vectors of N elements
// Per-step a1 / a3 launches at C2 sizes (B*H = 65536) are latency-bound: with 16-byte vectors
// only 8192 (bf16) / 16384 (fp32) threads exist, one warp per SM sub-partition and a long
// serial chain of transcendentals per thread.  The vector width N is therefore a template
// parameter and the host picks the widest N that still gives >= 148 x 256 threads (down to 4
// bytes per access); every element's arithmetic is unchanged (bit-identical results).
template <int N> struct FV;
template <> struct FV<1> { typedef float t; };
template <> struct FV<2> { typedef float2 t; };
template <> struct FV<4> { typedef float4 t; };
template <int N>
__device__ __forceinline__ void ldv(const float* p, float (&o)[N]) {
  if constexpr (N == 8) {
    ldf<8>(p, o);
  } else {
    const typename FV<N>::t v = *reinterpret_cast<const typename FV<N>::t*>(p);
    const float* f = reinterpret_cast<const float*>(&v);
#pragma unroll
    for (int k = 0; k < N; ++k) o[k] = f[k];
  }
}
template <int N>
__device__ __forceinline__ void stv(float* p, const float (&v)[N]) {
  if constexpr (N == 8) {
    stf<8>(p, v);
  } else {
    typename FV<N>::t u;
    float* f = reinterpret_cast<float*>(&u);
#pragma unroll
    for (int k = 0; k < N; ++k) f[k] = v[k];
    *reinterpret_cast<typename FV<N>::t*>(p) = u;
  }
}
template <int N> struct BV;   // N bf16 = N/2 bf16x2 words
template <> struct BV<2> { typedef uint32_t t; };
template <> struct BV<4> { typedef uint2 t; };
template <> struct BV<8> { typedef uint4 t; };
template <int N>
__device__ __forceinline__ void ldv(const __nv_bfloat16* p, float (&o)[N]) {
  const typename BV<N>::t v = *reinterpret_cast<const typename BV<N>::t*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}
template <int N>
__device__ __forceinline__ void stv(__nv_bfloat16* p, const float (&v)[N]) {
  typename BV<N>::t u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < N / 2; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<typename BV<N>::t*>(p) = u;
}

// streaming (evict-first) variants for the scan's read-once gate loads
template <int N>
__device__ __forceinline__ void ldv_stream(const float* p, float (&o)[N]) {
  if constexpr (N == 8) {
    float a[4], b[4];
    ld16_stream(p, a);
    ld16_stream(p + 4, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) { o[k] = a[k]; o[4 + k] = b[k]; }
  } else {
    const typename FV<N>::t v = __ldcs(reinterpret_cast<const typename FV<N>::t*>(p));
    const float* f = reinterpret_cast<const float*>(&v);
#pragma unroll
    for (int k = 0; k < N; ++k) o[k] = f[k];
  }
}
template <typename T, int V> struct ScanRaw { typedef float t[V]; };                     // fp32: floats
template <int V> struct ScanRaw<__nv_bfloat16, V> { typedef typename BV<V>::t t; };     // bf16: packed
template <int N>
__device__ __forceinline__ typename BV<N>::t ldcs_raw(const __nv_bfloat16* p) {
  if constexpr (N == 2) return __ldcs(reinterpret_cast<const unsigned int*>(p));
  else return __ldcs(reinterpret_cast<const typename BV<N>::t*>(p));
}
template <int N>
__device__ __forceinline__ void unpack_bf(const typename BV<N>::t& v, float (&o)[N]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}
template <int N>
__device__ __forceinline__ void ldv_stream(const __nv_bfloat16* p, float (&o)[N]) {
  typename BV<N>::t v;
  if constexpr (N == 2) v = __ldcs(reinterpret_cast<const unsigned int*>(p));
  else v = __ldcs(reinterpret_cast<const typename BV<N>::t*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}

// ---------------------------------------------------------------- a1 forward
template <typename T, int V>
__global__ void __launch_bounds__(128) lstm_fwd_kernel(int B, int H, const T* gx,
                                                       const T* __restrict__ gh, const float* __restrict__ bias,
                                                       const float* __restrict__ c_prev, T* gates,
                                                       float* __restrict__ c_out, T* __restrict__ tc_out,
                                                       T* __restrict__ h_out) {
  pdl_wait();
  const int nvec = H / V;
  const long total = (long)B * nvec;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / nvec);
    const int j = (int)(idx - (long)b * nvec) * V;
    const long row4 = (long)b * 4 * H;
    float a[4][V];
#pragma unroll
    for (int g = 0; g < 4; ++g) ldv<V>(gx + row4 + g * H + j, a[g]);
    if (gh) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float t[V];
        ldv<V>(gh + row4 + g * H + j, t);
#pragma unroll
        for (int k = 0; k < V; ++k) a[g][k] = __fadd_rn(a[g][k], t[k]);
      }
    }
    if (bias) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float t[V];
        ldv<V>(bias + g * H + j, t);
#pragma unroll
        for (int k = 0; k < V; ++k) a[g][k] = __fadd_rn(a[g][k], t[k]);
      }
    }
    float cp[V];
    ldv<V>(c_prev + (long)b * H + j, cp);
    float gi[V], gf[V], gg[V], go[V], c[V], tc[V], h[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      gates_of<T>(a[0][k], a[1][k], a[2][k], a[3][k], gi[k], gf[k], gg[k], go[k]);
      c[k] = cell_update(gf[k], cp[k], gi[k], gg[k]);
      tc[k] = tanh_c<T>(c[k]);
      h[k] = hidden<T>(go[k], tc[k]);
    }
    stv<V>(gates + row4 + 0 * H + j, gi);
    stv<V>(gates + row4 + 1 * H + j, gf);
    stv<V>(gates + row4 + 2 * H + j, gg);
    stv<V>(gates + row4 + 3 * H + j, go);
    stv<V>(c_out + (long)b * H + j, c);
    if (tc_out) stv<V>(tc_out + (long)b * H + j, tc);
    stv<V>(h_out + (long)b * H + j, h);
  }
}

// ---------------------------------------------------------------- a2 c-regeneration scan
// V elements per thread, U time steps of loads in flight: the bytes in flight over the whole grid
// are B*H*U*3s, independent of V, so small B*H launches use narrow vectors and deep U (U = 8; bf16 16-/8-byte vectors keep U = 4)
template <typename T, int V, int U>
__global__ void __launch_bounds__(128) lstm_cscan_kernel(int T_, int B, int H, const T* __restrict__ gates,
                                                         const float* __restrict__ c0, float* __restrict__ cws,
                                                         T* __restrict__ hws) {
  pdl_wait();
  const int nvec = H / V;
  const long total = (long)B * nvec;
  const long gstep = (long)B * 4 * H;
  const long cstep = (long)B * H;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / nvec);
    const int j = (int)(idx - (long)b * nvec) * V;
    const T* gp = gates + (long)b * 4 * H + j;
    float* cp = cws + (long)b * H + j;
    T* hp = hws ? hws + (long)b * H + j : nullptr;
    float c[V];
    ldv<V>(c0 + (long)b * H + j, c);
    for (int t0 = 0; t0 < T_; t0 += U) {
      // bf16: the U steps' gate vectors stay PACKED in registers until their step is computed (a
      // 16-byte load = 4 registers instead of 8 floats), so twice the bytes are in flight per
      // register and a deeper U fits; fp32 converts nothing
      typedef typename ScanRaw<T, V>::t Raw;
      Raw ri[U], rf[U], rg[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t0 + u < T_) {
          const T* q = gp + (long)(t0 + u) * gstep;
          if constexpr (sizeof(T) == 2) {
            ri[u] = ldcs_raw<V>(q);
            rf[u] = ldcs_raw<V>(q + H);
            rg[u] = ldcs_raw<V>(q + 2 * H);
          } else {
            ldv_stream<V>(q, ri[u]);
            ldv_stream<V>(q + H, rf[u]);
            ldv_stream<V>(q + 2 * H, rg[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t0 + u < T_) {
          float gi[V], gf[V], gg[V];
          if constexpr (sizeof(T) == 2) {
            unpack_bf<V>(ri[u], gi);
            unpack_bf<V>(rf[u], gf);
            unpack_bf<V>(rg[u], gg);
          } else {
#pragma unroll
            for (int k = 0; k < V; ++k) { gi[k] = ri[u][k]; gf[k] = rf[u][k]; gg[k] = rg[u][k]; }
          }
#pragma unroll
          for (int k = 0; k < V; ++k) c[k] = cell_update(gf[k], c[k], gi[k], gg[k]);
          stv<V>(cp + (long)(t0 + u) * cstep, c);
          if (hp) {                                         // mirrored outputs: h_t = o * tanh(c_t)
            float go[V], h[V];
            ldv_stream<V>(gp + (long)(t0 + u) * gstep + 3 * H, go);
#pragma unroll
            for (int k = 0; k < V; ++k) h[k] = hidden<T>(go[k], tanh_c<T>(c[k]));
            stv<V>(hp + (long)(t0 + u) * cstep, h);
          }
        }
      }
    }
  }
}

template <typename T>
constexpr int scan_u(int v) { return sizeof(T) == 4 || v == 2 ? 8 : sizeof(T) == 2 && v == 8 ? 8 : 4; }

// ---------------------------------------------------------------- a3 backward (fused recompute)
template <typename T, int V>
__global__ void __launch_bounds__(128) lstm_bwd_kernel(int B, int H, const T* gates,
                                                       const float* __restrict__ c_prev,
                                                       const float* __restrict__ c_t, const T* __restrict__ tc_st,
                                                       const float* __restrict__ dh, float* dc, T* dA,
                                                       T* __restrict__ h_regen) {
  pdl_wait();
  const int nvec = H / V;
  const long total = (long)B * nvec;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / nvec);
    const int j = (int)(idx - (long)b * nvec) * V;
    const long row4 = (long)b * 4 * H;
    const long row = (long)b * H + j;
    float gi[V], gf[V], gg[V], go[V];
    ldv<V>(gates + row4 + 0 * H + j, gi);
    ldv<V>(gates + row4 + 1 * H + j, gf);
    ldv<V>(gates + row4 + 2 * H + j, gg);
    ldv<V>(gates + row4 + 3 * H + j, go);
    float cp[V], tc[V], h[V], dhv[V], dcv[V];
    ldv<V>(c_prev + row, cp);
    ldv<V>(dh + row, dhv);
    ldv<V>(dc + row, dcv);
    if (tc_st) {                       // STASH: tanh(c_t) was stashed by a1
      ldv<V>(tc_st + row, tc);
    } else {                           // RECOMPUTE: regenerate tanh(c_t) and h_t
      float ct[V];
      ldv<V>(c_t + row, ct);
#pragma unroll
      for (int k = 0; k < V; ++k) { tc[k] = tanh_c<T>(ct[k]); h[k] = hidden<T>(go[k], tc[k]); }
    }
    float di[V], df[V], dg[V], dout[V], dcn[V];
#pragma unroll
    for (int k = 0; k < V; ++k)
      cell_grad<T>(gi[k], gf[k], gg[k], go[k], cp[k], tc[k], dhv[k], dcv[k], di[k], df[k], dg[k], dout[k], dcn[k]);
    stv<V>(dA + row4 + 0 * H + j, di);
    stv<V>(dA + row4 + 1 * H + j, df);
    stv<V>(dA + row4 + 2 * H + j, dg);
    stv<V>(dA + row4 + 3 * H + j, dout);
    stv<V>(dc + row, dcn);
    if (h_regen) stv<V>(h_regen + row, h);
  }
}

// ---------------------------------------------------------------- Mirror plan (prior work)
// The Mirror baseline (Chen et al.; estimator strategy "mirror", reading
// R25) mirrors every cheap op of the cell, so what it keeps per step are the INPUTS of the
// pre-activation adds: the NP separate FC outputs (input projection(s) and h_{t-1} W_h^T, part q
// at parts + q * pstride) and h_t (an FC input).  Its kernels regenerate
//   A = ((P_0 + P_1) + P_2) + b      (fp32, this order; a1's order for gx, gh, bias)
// and then run the same gate / cell / gradient device functions as a1 / a2 / a3.
template <typename T, int V, int NP>
__device__ __forceinline__ void parts_A(const T* p, long pstride, const float* __restrict__ bias, int H, int j,
                                        int ngates, float (&a)[4][V]) {
#pragma unroll
  for (int g = 0; g < 4; ++g)
    if (g < ngates) ldv<V>(p + g * H + j, a[g]);
#pragma unroll
  for (int q = 1; q < NP; ++q)
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if (g < ngates) {
        float t[V];
        ldv<V>(p + q * pstride + g * H + j, t);
#pragma unroll
        for (int k = 0; k < V; ++k) a[g][k] = __fadd_rn(a[g][k], t[k]);
      }
  if (bias)
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if (g < ngates) {
        float t[V];
        ldv<V>(bias + g * H + j, t);
#pragma unroll
        for (int k = 0; k < V; ++k) a[g][k] = __fadd_rn(a[g][k], t[k]);
      }
}

template <typename T, int V, int NP>
__global__ void __launch_bounds__(128) lstm_fwd_parts_kernel(int B, int H, const T* __restrict__ parts, long pstride,
                                                             const float* __restrict__ bias,
                                                             const float* __restrict__ c_prev, float* __restrict__ c_out,
                                                             T* __restrict__ h_out) {
  pdl_wait();
  const int nvec = H / V;
  const long total = (long)B * nvec;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / nvec);
    const int j = (int)(idx - (long)b * nvec) * V;
    float a[4][V], cp[V], c[V], h[V];
    parts_A<T, V, NP>(parts + (long)b * 4 * H, pstride, bias, H, j, 4, a);
    ldv<V>(c_prev + (long)b * H + j, cp);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float gi, gf, gg, go;
      gates_of<T>(a[0][k], a[1][k], a[2][k], a[3][k], gi, gf, gg, go);
      c[k] = cell_update(gf, cp[k], gi, gg);
      h[k] = hidden<T>(go, tanh_c<T>(c[k]));
    }
    stv<V>(c_out + (long)b * H + j, c);
    stv<V>(h_out + (long)b * H + j, h);
  }
}

// c-chain regeneration from the parts: step k's parts at parts + k * sstride (sstride < 0 walks
// a time-ordered buffer backwards for a reverse-direction layer); c_k to cws[k] (processing order)
template <typename T, int V, int NP>
__global__ void __launch_bounds__(128) lstm_cscan_parts_kernel(int T_, int B, int H, const T* __restrict__ parts,
                                                               long pstride, long sstride, const float* __restrict__ bias,
                                                               const float* __restrict__ c0, float* __restrict__ cws) {
  pdl_wait();
  constexpr int U = 4;
  const int nvec = H / V;
  const long total = (long)B * nvec;
  const long cstep = (long)B * H;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / nvec);
    const int j = (int)(idx - (long)b * nvec) * V;
    const T* gp = parts + (long)b * 4 * H;
    float c[V];
    ldv<V>(c0 + (long)b * H + j, c);
    for (int t0 = 0; t0 < T_; t0 += U) {
      float a[U][4][V];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t0 + u < T_) parts_A<T, V, NP>(gp + (long)(t0 + u) * sstride, pstride, bias, H, j, 3, a[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t0 + u < T_) {
#pragma unroll
          for (int k = 0; k < V; ++k) {
            float gi, gf, gg, go;
            gates_of<T>(a[u][0][k], a[u][1][k], a[u][2][k], 0.0f, gi, gf, gg, go);
            c[k] = cell_update(gf, c[k], gi, gg);
          }
          stv<V>(cws + (long)(t0 + u) * cstep + (long)b * H + j, c);
        }
    }
  }
}

// backward step from the parts (h_t is kept by the Mirror plan, so it is not regenerated); dA may
// alias part 0 of this step
template <typename T, int V, int NP>
__global__ void __launch_bounds__(128) lstm_bwd_parts_kernel(int B, int H, const T* parts, long pstride,
                                                             const float* __restrict__ bias,
                                                             const float* __restrict__ c_prev,
                                                             const float* __restrict__ c_t,
                                                             const float* __restrict__ dh, float* dc, T* dA) {
  pdl_wait();
  const int nvec = H / V;
  const long total = (long)B * nvec;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / nvec);
    const int j = (int)(idx - (long)b * nvec) * V;
    const long row4 = (long)b * 4 * H;
    const long row = (long)b * H + j;
    float a[4][V], cp[V], ct[V], dhv[V], dcv[V];
    parts_A<T, V, NP>(parts + row4, pstride, bias, H, j, 4, a);
    ldv<V>(c_prev + row, cp);
    ldv<V>(c_t + row, ct);
    ldv<V>(dh + row, dhv);
    ldv<V>(dc + row, dcv);
    float di[V], df[V], dg[V], dout[V], dcn[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float gi, gf, gg, go;
      gates_of<T>(a[0][k], a[1][k], a[2][k], a[3][k], gi, gf, gg, go);
      cell_grad<T>(gi, gf, gg, go, cp[k], tanh_c<T>(ct[k]), dhv[k], dcv[k], di[k], df[k], dg[k], dout[k], dcn[k]);
    }
    stv<V>(dA + row4 + 0 * H + j, di);
    stv<V>(dA + row4 + 1 * H + j, df);
    stv<V>(dA + row4 + 2 * H + j, dg);
    stv<V>(dA + row4 + 3 * H + j, dout);
    stv<V>(dc + row, dcn);
  }
}

// ---------------------------------------------------------------- a1 fused over the recurrence
// One cooperative (persistent) launch runs steps k0..k1-1 of a layer: per step each CTA computes
// the recurrent product h_{k-1} W_h^T for its tile (RB batch rows x 4*UPC gate columns = the four
// gates of UPC hidden units) in fp32 FFMA from shared memory, adds the precomputed x_t W_x^T and
// the bias with the same rounding points as the per-step path (round_s(gx + h W_h^T), then + b),
// applies the a1 pointwise functions (cell_update / tanh_c / hidden: bit-identical device code),
// carries c in registers and publishes h_t; a grid barrier separates the steps (every tile reads
// all of h_{k-1}).  Replaces 2 launches + 1 cuBLAS GEMM per step (latency-bound at C2).
constexpr int SEQ_THREADS = 256;
#ifdef ECHO_PHASE_TIMING
__device__ unsigned long long g_seq_phase[5][1024];   // per CTA: stage, gemm, epilogue, sync cycles; steps
#define SEQ_T(v) long long v = clock64()
#define SEQ_ACC(i, a, b) do { if (threadIdx.x == 0 && blockIdx.x < 1024) g_seq_phase[i][blockIdx.x] += (b) - (a); } while (0)
#else
#define SEQ_T(v) do { } while (0)
#define SEQ_ACC(i, a, b) do { } while (0)
#endif

struct SeqGeom {
  int RB, UPC, NB, CPT, hsp;      // rows / units per CTA, CTAs, gate columns per thread, h row stride
  size_t smem;
};

static __host__ __device__ __forceinline__ SeqGeom seq_geom(int B, int H, int RB, int UPC) {
  SeqGeom g;
  g.RB = RB;
  g.UPC = UPC;
  g.NB = (B / RB) * (H / UPC);
  g.CPT = 4 * UPC * RB / SEQ_THREADS;
  g.hsp = H + 4;
  g.smem = sizeof(float) * ((size_t)RB * g.hsp + (size_t)H * 4 * UPC + (size_t)RB * 4 * UPC);
  return g;
}

template <typename T, int CPT>
__global__ void __launch_bounds__(SEQ_THREADS, 1) lstm_seq_fwd_kernel(int k0, int k1, int T_, int B, int H, int RB,
                                                                      int UPC, int reverse, const T* gx,
                                                                      const T* __restrict__ Wh,
                                                                      const float* __restrict__ bias,
                                                                      const T* __restrict__ h0,
                                                                      const float* __restrict__ c0, T* gates,
                                                                      float* __restrict__ c_out, int c_ring,
                                                                      T* __restrict__ tc_out, T* __restrict__ h_out) {
  pdl_wait();
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) float sm[];
  const int hsp = H + 4, WC = 4 * UPC;
  float* hs = sm;                                   // [RB][hsp]   h_{k-1} rows of this tile (fp32)
  float* Ws = hs + (size_t)RB * hsp;                // [H][WC]     W_h rows of this tile's gate columns, k-major
  float* Gs = Ws + (size_t)H * WC;                  // [RB][WC]    recurrent products
  const int tid = threadIdx.x;
  const int nub = H / UPC;
  const int r0 = (blockIdx.x / nub) * RB, j0 = (blockIdx.x % nub) * UPC;
  // W_h slice, once: column q = g * UPC + u  <->  W_h row g * H + j0 + u
  for (int i = tid; i < WC * H; i += SEQ_THREADS) {
    const int q = i / H, k = i - q * H;
    const int g = q / UPC, u = q - g * UPC;
    Ws[(size_t)k * WC + q] = to_f(Wh[(size_t)(g * H + j0 + u) * H + k]);
  }
  // pointwise ownership: (row, unit) pairs e = tid + m * SEQ_THREADS; c carried in registers
  constexpr int MAXP = 4;
  const int npair = RB * UPC;
  float creg[MAXP];
#pragma unroll
  for (int m = 0; m < MAXP; ++m) {
    const int e = tid + m * SEQ_THREADS;
    if (e < npair) {
      const int r = e / UPC, u = e - r * UPC;
      creg[m] = (k0 == 0) ? c0[(size_t)(r0 + r) * H + j0 + u]
                          : c_out[(size_t)(c_ring ? (k0 - 1) % 2 : k0 - 1) * B * H + (size_t)(r0 + r) * H + j0 + u];
    }
  }
  const int gr = tid % RB, cgp = tid / RB;          // GEMM: row gr, gate columns cgp*CPT .. +CPT
  const size_t BH = (size_t)B * H, B4H = (size_t)B * 4 * H;
  for (int k = k0; k < k1; ++k) {
    const int t = reverse ? T_ - 1 - k : k;
    SEQ_T(p0);
    const T* hp = (k == 0) ? h0 : h_out + (size_t)(reverse ? T_ - k : k - 1) * BH;
    // stage h_{k-1}[r0 .. r0+RB) as fp32 (L2-coherent loads: other CTAs wrote it last step)
    constexpr int V = St<T>::VEC;
    for (int i = tid; i < RB * (H / V); i += SEQ_THREADS) {
      const int r = i / (H / V), c = (i - r * (H / V)) * V;
      float v[V];
      ld16_cg(hp + (size_t)(r0 + r) * H + c, v);
#pragma unroll
      for (int q = 0; q < V; q += 4)
        *reinterpret_cast<float4*>(hs + (size_t)r * hsp + c + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
    }
    __syncthreads();
    SEQ_T(p1);
    float acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = 0.0f;
    const float* hrow = hs + (size_t)gr * hsp;
    const float* wcol = Ws + cgp * CPT;
    for (int kk = 0; kk < H; kk += 4) {
      const float4 hv = *reinterpret_cast<const float4*>(hrow + kk);
      const float hx[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float* wr = wcol + (size_t)(kk + q) * WC;
#pragma unroll
        for (int c = 0; c < CPT; c += 4) {
          const float4 w = *reinterpret_cast<const float4*>(wr + c);
          acc[c] = __fmaf_rn(hx[q], w.x, acc[c]);
          acc[c + 1] = __fmaf_rn(hx[q], w.y, acc[c + 1]);
          acc[c + 2] = __fmaf_rn(hx[q], w.z, acc[c + 2]);
          acc[c + 3] = __fmaf_rn(hx[q], w.w, acc[c + 3]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) Gs[(size_t)gr * WC + cgp * CPT + c] = acc[c];
    __syncthreads();
    SEQ_T(p2);
    const T* gxt = gx + (size_t)t * B4H;
    T* gk = gates + (size_t)k * B4H;
#pragma unroll
    for (int m = 0; m < MAXP; ++m) {
      const int e = tid + m * SEQ_THREADS;
      if (e < npair) {
        const int r = e / UPC, u = e - r * UPC;
        const size_t row4 = (size_t)(r0 + r) * 4 * H, row = (size_t)(r0 + r) * H + j0 + u;
        float a[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          // same rounding points as the per-step path: round_s(gx + h W_h^T) (cuBLAS beta = 1 into
          // storage dtype), then + b in fp32
          const float pre = St<T>::round(__fadd_rn(to_f(gxt[row4 + g * H + j0 + u]), Gs[(size_t)r * WC + g * UPC + u]));
          a[g] = __fadd_rn(pre, bias[g * H + j0 + u]);
        }
        const float gi = St<T>::round(sigmoidf_(a[0])), gf = St<T>::round(sigmoidf_(a[1]));
        const float gg = St<T>::round(tanhf(a[2])), go = St<T>::round(sigmoidf_(a[3]));
        const float c = cell_update(gf, creg[m], gi, gg);
        const float tc = tanh_c<T>(c);
        const float h = hidden<T>(go, tc);
        creg[m] = c;
        gk[row4 + 0 * H + j0 + u] = from_f<T>(gi);
        gk[row4 + 1 * H + j0 + u] = from_f<T>(gf);
        gk[row4 + 2 * H + j0 + u] = from_f<T>(gg);
        gk[row4 + 3 * H + j0 + u] = from_f<T>(go);
        c_out[(size_t)(c_ring ? k % 2 : k) * BH + row] = c;
        if (tc_out) tc_out[(size_t)k * BH + row] = from_f<T>(tc);
        h_out[(size_t)t * BH + row] = from_f<T>(h);
      }
    }
    SEQ_T(p3);
    __threadfence();
    grid.sync();                                      // h_t complete before anyone stages it
    SEQ_T(p4);
    SEQ_ACC(0, p0, p1);
    SEQ_ACC(1, p1, p2);
    SEQ_ACC(2, p2, p3);
    SEQ_ACC(3, p3, p4);
    SEQ_ACC(4, 0, 1);
  }
}

// host: pick the tile (RB rows x UPC units) and check co-residency; false = use the per-step path
static bool seq_plan(int B, int H, int dtype, SeqGeom* out, const void** kern) {
  int RB = B % 64 == 0 ? 64 : (B % 32 == 0 ? 32 : 0);
  if (!RB) return false;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int UPC = 2; UPC <= 16; UPC *= 2) {
    if (H % UPC) continue;
    SeqGeom g = seq_geom(B, H, RB, UPC);
    if (g.CPT != 4 && g.CPT != 8) continue;
    if (g.smem > 220 * 1024) continue;
    const void* k = nullptr;
    if (dtype == ECHO_FP32) k = g.CPT == 4 ? (const void*)lstm_seq_fwd_kernel<float, 4> : (const void*)lstm_seq_fwd_kernel<float, 8>;
    else k = g.CPT == 4 ? (const void*)lstm_seq_fwd_kernel<__nv_bfloat16, 4> : (const void*)lstm_seq_fwd_kernel<__nv_bfloat16, 8>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, SEQ_THREADS, g.smem) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (g.NB > per * sms || RB * UPC > 4 * SEQ_THREADS) continue;
    *out = g;
    *kern = k;
    return true;
  }
  return false;
}


// ================================================================ a0 + a1 fused on the tensor cores
// One LSTM forward step with the recurrent contraction h_{t-1} W_h^T on the 5th-generation tensor
// cores (tcgen05.mma, accumulator in TMEM) and the a1 cell epilogue applied to the accumulator
// straight out of TMEM (Echo-dagger fusion):
//   G = round_bf16(gx_t + h_{t-1} W_h^T)   (the per-step path's cuBLAS beta = 1 output)
//   A = G + b ;  i,f,g,o = gates_of(A) ;  c_t = cell_update ;  h_t = hidden(o, tanh_c(c_t))
// with the SAME device functions and rounding points as a1, so it differs from the per-step path
// only in the GEMM's accumulation order (and STASH / RECOMPUTE give identical results).
// CTA j owns hidden units [16 j, 16 j + 16): the 64 gate rows {g H + 16 j + u} of W_h form the MMA's
// B operand (N = 64), the whole h_{t-1} (B <= 128 rows, zero-padded by TMA) the A operand (M = 128),
// K = H in 64-element atoms (128-byte rows, 128-byte swizzle).  Thread 0 issues every TMA load (one
// mbarrier per K atom, all resident: H <= 512 -> 192 KB) and then the 4 x H/64 MMAs as the atoms
// land; tcgen05.commit signals the epilogue.  The epilogue spreads over 16 warps: warp w reads TMEM
// lanes 32 (w % 4) .. + 31 (rows b) and the accumulator columns of units 4 (w / 4) .. + 3 (four
// tcgen05.ld of 4 columns, one per gate), and each thread finishes the cell for its row and 4 units.
constexpr int TC_U = 16, TC_N = 4 * TC_U, TC_M = 128, TC_KA = 64;
constexpr int TC_A_ATOM = TC_M * TC_KA * 2, TC_B_ATOM = TC_N * TC_KA * 2;   // 16 KB, 8 KB

__device__ __forceinline__ uint32_t tc_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tc_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tc_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tc_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tc_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* bar, uint32_t phase) { mbar_wait_bounded(tc_smem_u32(bar), phase); }
__device__ __forceinline__ void tc_tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          tc_smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(tc_smem_u32(bar))
      : "memory");
}
// K-major operand tile in the canonical 128-byte-swizzle layout: rows of 64 bf16 (128 B), 8-row
// groups 1024 B apart (SBO), LBO unused (1), descriptor version 1 (sm_100), layout SWIZZLE_128B (2)
__device__ __forceinline__ uint64_t tc_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);            // start address
  d |= (uint64_t)1 << 16;                            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                  // SBO
  d |= (uint64_t)1 << 46;                            // version
  d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
  return d;
}
// instruction descriptor: kind::f16, A = B = BF16, D = F32, both K-major, M = 128, N = TC_N
__host__ __device__ constexpr uint32_t tc_idesc() {
  return (1u << 4)                 // D format F32
         | (1u << 7)               // A format BF16
         | (1u << 10)              // B format BF16
         | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(tc_idesc()), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

constexpr int TC_THREADS = 512;
template <int MODE_STASH>
__global__ void __launch_bounds__(TC_THREADS, 1) lstm_fwd_tc_kernel(const __grid_constant__ CUtensorMap mH,
                                                            const __grid_constant__ CUtensorMap mW, int B, int H,
                                                            const __nv_bfloat16* gx, const float* __restrict__ bias,
                                                            const float* __restrict__ c_prev, __nv_bfloat16* gates,
                                                            float* __restrict__ c_out, __nv_bfloat16* __restrict__ tc_out,
                                                            __nv_bfloat16* __restrict__ h_out) {
  typedef __nv_bfloat16 T;
  pdl_wait();
  extern __shared__ __align__(1024) unsigned char tc_sm[];
  __shared__ __align__(8) uint64_t full[8];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tmem_holder;
  const int nk = H / TC_KA;
  const int tid = threadIdx.x, w = tid >> 5;
  const int j0 = blockIdx.x * TC_U;
  unsigned char* sA = tc_sm;                                   // nk atoms of [128 rows][128 B]
  unsigned char* sB = tc_sm + (size_t)nk * TC_A_ATOM;          // nk atoms of [64 rows][128 B]
  if (w == 0) {                                                // TMEM: 64 fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc_smem_u32(&tmem_holder)),
                 "n"(TC_N)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 32) {
    for (int k = 0; k < nk; ++k) tc_mbar_init(&full[k], 1);
    tc_mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_holder;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mH) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mW) : "memory");
    for (int k = 0; k < nk; ++k) {                             // every K atom in flight at once
      tc_mbar_expect_tx(&full[k], TC_A_ATOM + TC_B_ATOM);
      tc_tma_2d(sA + (size_t)k * TC_A_ATOM, &mH, k * TC_KA, 0, &full[k]);
#pragma unroll
      for (int g = 0; g < 4; ++g)                              // gate g's 16 rows of W_h
        tc_tma_2d(sB + (size_t)k * TC_B_ATOM + g * (TC_U * 128), &mW, k * TC_KA, g * H + j0, &full[k]);
    }
    for (int k = 0; k < nk; ++k) {                             // MMAs in K order as the atoms land
      tc_mbar_wait(&full[k], 0);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t a0 = tc_smem_u32(sA + (size_t)k * TC_A_ATOM), b0 = tc_smem_u32(sB + (size_t)k * TC_B_ATOM);
#pragma unroll
      for (int kk = 0; kk < TC_KA / 16; ++kk)                   // K = 16 per MMA: +32 B inside the swizzle atom
        tc_mma(tmem, tc_desc_sw128(a0 + 32 * kk), tc_desc_sw128(b0 + 32 * kk), (k | kk) != 0);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(tc_smem_u32(&done))
                 : "memory");
  }
  __syncwarp();
  // epilogue: warp w -> TMEM lanes (rows) 32 (w % 4) + lane, units j0 + 4 (w / 4) + 0..3; the
  // accumulator column of gate g, unit u is g * 16 + u.  The cell's other operands (gx_t, bias,
  // c_{t-1}) do not depend on the MMA: they are loaded before waiting for it
  const int lg = w & 3, ug = w >> 2;
  const int b = 32 * lg + (tid & 31);
  const int j = j0 + 4 * ug;
  const long row4 = (long)b * 4 * H;
  float x[4][4], bb[4][4], cp[4];
  if (b < B) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      ldv<4>(gx + row4 + g * H + j, x[g]);
      ldv<4>(bias + g * H + j, bb[g]);
    }
    ldv<4>(c_prev + (long)b * H + j, cp);
  }
  tc_mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  float acc[4][4];
#pragma unroll
  for (int g = 0; g < 4; ++g) tc_ld4(tmem + ((uint32_t)(32 * lg) << 16) + (uint32_t)(g * TC_U + 4 * ug), acc[g]);
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  if (b < B) {
    float a[4][4];
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        a[g][u] = __fadd_rn(St<T>::round(__fadd_rn(x[g][u], acc[g][u])), bb[g][u]);   // G = round(gx + gh); A = G + b
    float gi[4], gf[4], gg[4], go[4], c[4], tc[4], h[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      gates_of<T>(a[0][u], a[1][u], a[2][u], a[3][u], gi[u], gf[u], gg[u], go[u]);
      c[u] = cell_update(gf[u], cp[u], gi[u], gg[u]);
      tc[u] = tanh_c<T>(c[u]);
      h[u] = hidden<T>(go[u], tc[u]);
    }
    stv<4>(gates + row4 + 0 * H + j, gi);
    stv<4>(gates + row4 + 1 * H + j, gf);
    stv<4>(gates + row4 + 2 * H + j, gg);
    stv<4>(gates + row4 + 3 * H + j, go);
    stv<4>(c_out + (long)b * H + j, c);
    if (MODE_STASH) stv<4>(tc_out + (long)b * H + j, tc);
    stv<4>(h_out + (long)b * H + j, h);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TC_N) : "memory");
}

// ---------------------------------------------------------------- validation
static echo_status check_desc(const echo_lstm_desc* d) {
  if (!d) return fail(ECHO_ERR_INVALID, "lstm: desc is NULL");
  if (d->B <= 0 || d->H <= 0) return fail(ECHO_ERR_INVALID, "lstm: B=%d H=%d must be > 0", d->B, d->H);
  if (d->H % 8) return fail(ECHO_ERR_INVALID, "lstm: H=%d must be a multiple of 8", d->H);
  if (d->dtype != ECHO_FP32 && d->dtype != ECHO_BF16) return fail(ECHO_ERR_INVALID, "lstm: bad dtype %d", d->dtype);
  if (d->mode != ECHO_STASH && d->mode != ECHO_RECOMPUTE) return fail(ECHO_ERR_INVALID, "lstm: bad mode %d", d->mode);
  return ECHO_OK;
}

#define ECHO_REQ(p, name)                                                         \
  do {                                                                            \
    if (!(p)) return fail(ECHO_ERR_INVALID, "%s: required pointer %s is NULL", fn, name); \
    if (!aligned16(p)) return fail(ECHO_ERR_INVALID, "%s: %s is not 16-byte aligned", fn, name); \
  } while (0)
#define ECHO_OPT(p, name)                                                         \
  do {                                                                            \
    if ((p) && !aligned16(p)) return fail(ECHO_ERR_INVALID, "%s: %s is not 16-byte aligned", fn, name); \
  } while (0)

}  // namespace echo

using namespace echo;

extern "C" echo_status echo_lstm_fwd(const echo_lstm_desc* d, const void* gx_t, const void* gh_t,
                                     const float* bias, const float* c_prev, void* gates_t, float* c_out,
                                     void* tc_t, void* h_out, void* stream) {
  const char* fn = "echo_lstm_fwd";
  echo_status s = check_desc(d);
  if (s) return s;
  ECHO_REQ(gx_t, "gx_t");
  ECHO_OPT(gh_t, "gh_t");
  ECHO_OPT(bias, "bias");
  ECHO_REQ(c_prev, "c_prev");
  ECHO_REQ(gates_t, "gates_t");
  ECHO_REQ(c_out, "c_out");
  ECHO_REQ(h_out, "h_out");
  if (d->mode == ECHO_STASH) { ECHO_REQ(tc_t, "tc_t"); }
  else if (tc_t) return fail(ECHO_ERR_INVALID, "%s: tc_t must be NULL in RECOMPUTE mode", fn);
  if (c_out == c_prev) return fail(ECHO_ERR_INVALID, "%s: c_out must not alias c_prev", fn);
  cudaStream_t st = (cudaStream_t)stream;
  const bool bf = d->dtype != ECHO_FP32;
  const int V = step_vec((long)d->B * d->H, bf);
  const int blk = step_block((long)d->B * d->H / V);
  const int grid = grid_for((long)d->B * d->H / V, blk);
  cudaError_t e_;
#define ECHO_FWD_LAUNCH(TT, VV)                                                                                     \
  launch(lstm_fwd_kernel<TT, VV>, dim3(grid), dim3(blk), 0, st, 1, d->B, d->H, (const TT*)gx_t, (const TT*)gh_t, bias, \
         c_prev, (TT*)gates_t, c_out, (TT*)tc_t, (TT*)h_out)
  typedef __nv_bfloat16 bft;
  if (!bf)
    e_ = V == 4 ? ECHO_FWD_LAUNCH(float, 4) : V == 2 ? ECHO_FWD_LAUNCH(float, 2) : ECHO_FWD_LAUNCH(float, 1);
  else
    e_ = V == 8 ? ECHO_FWD_LAUNCH(bft, 8) : V == 4 ? ECHO_FWD_LAUNCH(bft, 4) : ECHO_FWD_LAUNCH(bft, 2);
#undef ECHO_FWD_LAUNCH
  if (e_ != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e_));
  return check_launch(fn);
}

extern "C" echo_status echo_lstm_cscan(const echo_lstm_desc* d, int32_t T, const void* gates, const float* c0,
                                       float* c_ws, void* h_ws, void* stream) {
  const char* fn = "echo_lstm_cscan";
  echo_status s = check_desc(d);
  if (s) return s;
  if (T <= 0) return fail(ECHO_ERR_INVALID, "%s: T=%d must be > 0", fn, T);
  ECHO_REQ(gates, "gates");
  ECHO_REQ(c0, "c0");
  ECHO_REQ(c_ws, "c_ws");
  ECHO_OPT(h_ws, "h_ws");
  cudaStream_t st = (cudaStream_t)stream;
  const bool bf = d->dtype != ECHO_FP32;
  // measured at C2 (CUPTI, in-graph): bf16 16-byte vectors / U = 4 38.3 us -> 4-byte / U = 8 15.9 us;
  // fp32 stays at 16-byte vectors (4-byte loads: 18.3 -> 29.8 us)
  const int V = bf || getenv("ECHO_LSTM_VEC") ? step_vec((long)d->B * d->H, bf) : 4;
  const int grid = grid_for((long)d->B * d->H / V, 128);
  cudaError_t e_;
#define ECHO_SCAN_LAUNCH(TT, VV)                                                                                      \
  launch(lstm_cscan_kernel<TT, VV, scan_u<TT>(VV)>, dim3(grid), dim3(128), 0, st, 1, T, d->B, d->H, (const TT*)gates, c0, c_ws, \
         (TT*)h_ws)
  typedef __nv_bfloat16 bft;
  if (!bf)
    e_ = V == 4 ? ECHO_SCAN_LAUNCH(float, 4) : V == 2 ? ECHO_SCAN_LAUNCH(float, 2) : ECHO_SCAN_LAUNCH(float, 1);
  else
    e_ = V == 8 ? ECHO_SCAN_LAUNCH(bft, 8) : V == 4 ? ECHO_SCAN_LAUNCH(bft, 4) : ECHO_SCAN_LAUNCH(bft, 2);
#undef ECHO_SCAN_LAUNCH
  if (e_ != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e_));
  return check_launch(fn);
}

// a3 per step (internal): c_prev / c_t / tc_t already resolved by echo_lstm_bwd_recompute.
static echo_status lstm_bwd_step(const char* fn, const echo_lstm_desc* d, const void* gates_t, const float* c_prev,
                                 const float* c_t, const void* tc_t, const float* dh_t, float* dc, void* dA_t,
                                 void* h_regen, void* stream) {
  ECHO_REQ(gates_t, "gates");
  ECHO_REQ(c_prev, "c_prev");
  ECHO_REQ(dh_t, "dh_t");
  ECHO_REQ(dc, "dc");
  ECHO_REQ(dA_t, "dA_t");
  if (d->mode == ECHO_STASH) {
    ECHO_REQ(tc_t, "tc_st");
    if (h_regen) return fail(ECHO_ERR_INVALID, "%s: h_regen_t must be NULL in STASH mode", fn);
  } else {
    ECHO_REQ(c_t, "ws");
    ECHO_OPT(h_regen, "h_regen_t");
  }
  cudaStream_t st = (cudaStream_t)stream;
  const bool bf = d->dtype != ECHO_FP32;
  const int V = step_vec((long)d->B * d->H, bf);
  const int blk = step_block((long)d->B * d->H / V);
  const int grid = grid_for((long)d->B * d->H / V, blk);
  cudaError_t e_;
#define ECHO_BWD_LAUNCH(TT, VV)                                                                                      \
  launch(lstm_bwd_kernel<TT, VV>, dim3(grid), dim3(blk), 0, st, 1, d->B, d->H, (const TT*)gates_t, c_prev, c_t,       \
         (const TT*)tc_t, dh_t, dc, (TT*)dA_t, (TT*)h_regen)
  typedef __nv_bfloat16 bft;
  if (!bf)
    e_ = V == 4 ? ECHO_BWD_LAUNCH(float, 4) : V == 2 ? ECHO_BWD_LAUNCH(float, 2) : ECHO_BWD_LAUNCH(float, 1);
  else
    e_ = V == 8 ? ECHO_BWD_LAUNCH(bft, 8) : V == 4 ? ECHO_BWD_LAUNCH(bft, 4) : ECHO_BWD_LAUNCH(bft, 2);
#undef ECHO_BWD_LAUNCH
  if (e_ != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e_));
  return check_launch(fn);
}

extern "C" echo_status echo_lstm_bwd_recompute(const echo_lstm_desc* d, int32_t T, int32_t t, uint32_t flags,
                                               const void* gates, const float* c0, const float* c_st,
                                               const void* tc_st, const float* dh_t, float* dc, void* dA_t,
                                               void* h_regen_t, void* ws, size_t* ws_bytes, void* stream) {
  const char* fn = "echo_lstm_bwd_recompute";
  echo_status s = check_desc(d);
  if (s) return s;
  if (T <= 0 || t < 0 || t >= T) return fail(ECHO_ERR_INVALID, "%s: t=%d out of range for T=%d", fn, t, T);
  if (flags & ~(uint32_t)ECHO_BWD_REGEN_C) return fail(ECHO_ERR_INVALID, "%s: unknown flags 0x%x", fn, flags);
  const bool rec = d->mode == ECHO_RECOMPUTE;
  const size_t BH = (size_t)d->B * d->H;
  const size_t need = rec ? sizeof(float) * (size_t)T * BH : 0;
  if (!ws && ws_bytes) {                                  // two-call workspace convention: size query
    *ws_bytes = need;
    return ECHO_OK;
  }
  if (ws_bytes && *ws_bytes < need)
    return fail(ECHO_ERR_CAPACITY, "%s: ws has %zu bytes, needs %zu", fn, *ws_bytes, need);
  ECHO_REQ(gates, "gates");
  ECHO_REQ(c0, "c0");
  const size_t es = d->dtype == ECHO_FP32 ? 4 : 2;
  const char* g_t = (const char*)gates + (size_t)t * 4 * BH * es;
  if (rec) {
    if (c_st || tc_st) return fail(ECHO_ERR_INVALID, "%s: c_st / tc_st must be NULL in RECOMPUTE mode", fn);
    ECHO_REQ(ws, "ws");
    float* cw = (float*)ws;
    if (flags & ECHO_BWD_REGEN_C) {                       // a2 prologue: c_1..c_T into ws
      s = echo_lstm_cscan(d, T, gates, c0, cw, nullptr, stream);
      if (s) return s;
    }
    return lstm_bwd_step(fn, d, g_t, t == 0 ? c0 : cw + (size_t)(t - 1) * BH, cw + (size_t)t * BH, nullptr, dh_t, dc,
                         dA_t, h_regen_t, stream);
  }
  if (flags) return fail(ECHO_ERR_INVALID, "%s: ECHO_BWD_REGEN_C needs RECOMPUTE mode", fn);
  ECHO_REQ(tc_st, "tc_st");
  if (t > 0) ECHO_REQ(c_st, "c_st");
  return lstm_bwd_step(fn, d, g_t, t == 0 ? c0 : c_st + (size_t)(t - 1) * BH, nullptr,
                       (const char*)tc_st + (size_t)t * BH * es, dh_t, dc, dA_t, nullptr, stream);
}

extern "C" echo_status echo_lstm_seq_fwd(const echo_lstm_desc* d, int32_t T, int32_t k0, int32_t k1, int32_t reverse,
                                         const void* gx, const void* Wh, const float* bias, const void* h0,
                                         const float* c0, void* gates, float* c, int32_t c_ring, void* tc, void* h,
                                         void* stream) {
  const char* fn = "echo_lstm_seq_fwd";
  echo_status s = check_desc(d);
  if (s) return s;
  if (T <= 0 || k0 < 0 || k1 > T || k0 >= k1) return fail(ECHO_ERR_INVALID, "%s: steps [%d, %d) of T=%d", fn, k0, k1, T);
  ECHO_REQ(gx, "gx");
  ECHO_REQ(Wh, "Wh");
  ECHO_REQ(bias, "bias");
  ECHO_REQ(h0, "h0");
  ECHO_REQ(c0, "c0");
  ECHO_REQ(gates, "gates");
  ECHO_REQ(c, "c");
  ECHO_REQ(h, "h");
  if (d->mode == ECHO_STASH) { ECHO_REQ(tc, "tc"); }
  else if (tc) return fail(ECHO_ERR_INVALID, "%s: tc must be NULL in RECOMPUTE mode", fn);
  if (reverse && gx == gates) return fail(ECHO_ERR_INVALID, "%s: a reverse layer's gx must not alias gates", fn);
  SeqGeom g;
  const void* kern = nullptr;
  if (!seq_plan(d->B, d->H, d->dtype, &g, &kern))
    return fail(ECHO_ERR_UNSUPPORTED, "%s: no co-resident tile for B=%d H=%d (use the per-step path)", fn, d->B, d->H);
  int B = d->B, H = d->H, RB = g.RB, UPC = g.UPC, ring = c_ring ? 1 : 0, rev = reverse ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.NB);
  cfg.blockDim = dim3(SEQ_THREADS);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (d->dtype == ECHO_FP32) {
    if (g.CPT == 4)
      e = cudaLaunchKernelEx(&cfg, lstm_seq_fwd_kernel<float, 4>, k0, k1, T, B, H, RB, UPC, rev, (const float*)gx,
                             (const float*)Wh, bias, (const float*)h0, c0, (float*)gates, c, ring, (float*)tc, (float*)h);
    else
      e = cudaLaunchKernelEx(&cfg, lstm_seq_fwd_kernel<float, 8>, k0, k1, T, B, H, RB, UPC, rev, (const float*)gx,
                             (const float*)Wh, bias, (const float*)h0, c0, (float*)gates, c, ring, (float*)tc, (float*)h);
  } else {
    typedef __nv_bfloat16 bf;
    if (g.CPT == 4)
      e = cudaLaunchKernelEx(&cfg, lstm_seq_fwd_kernel<bf, 4>, k0, k1, T, B, H, RB, UPC, rev, (const bf*)gx,
                             (const bf*)Wh, bias, (const bf*)h0, c0, (bf*)gates, c, ring, (bf*)tc, (bf*)h);
    else
      e = cudaLaunchKernelEx(&cfg, lstm_seq_fwd_kernel<bf, 8>, k0, k1, T, B, H, RB, UPC, rev, (const bf*)gx,
                             (const bf*)Wh, bias, (const bf*)h0, c0, (bf*)gates, c, ring, (bf*)tc, (bf*)h);
  }
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}

extern "C" int32_t echo_lstm_seq_supported(int32_t B, int32_t H, int32_t dtype) {
  SeqGeom g;
  const void* k = nullptr;
  return seq_plan(B, H, dtype, &g, &k) ? 1 : 0;
}

#ifdef ECHO_PHASE_TIMING
extern "C" int echo_debug_seq_phase(unsigned long long* host, int reset) {
  int e = (int)cudaMemcpyFromSymbol(host, echo::g_seq_phase, sizeof(unsigned long long) * 5 * 1024);
  if (reset) {
    static unsigned long long zero[5 * 1024] = {0};
    cudaMemcpyToSymbol(echo::g_seq_phase, zero, sizeof(zero));
  }
  return e;
}
#endif

// ---------------------------------------------------------------- Mirror-plan entry points
#define ECHO_PARTS_CHECK()                                                                          \
  echo_status s = check_desc(d);                                                                    \
  if (s) return s;                                                                                  \
  if (n_parts < 1 || n_parts > 3) return fail(ECHO_ERR_INVALID, "%s: n_parts=%d not in [1, 3]", fn, n_parts); \
  if (n_parts > 1 && (part_stride % 8 || part_stride < 4L * d->B * d->H))                          \
    return fail(ECHO_ERR_INVALID, "%s: part_stride=%lld must be a multiple of 8 and >= 4*B*H", fn,   \
                (long long)part_stride)

// (storage type, vector width) dispatch for the Mirror-plan launches: f(T{}, integral_constant<V>)
template <typename F>
static cudaError_t dispatch_tv(bool bf, int V, F&& f) {
  typedef __nv_bfloat16 bft;
  if (!bf) {
    if (V == 4) return f(float{}, std::integral_constant<int, 4>{});
    if (V == 2) return f(float{}, std::integral_constant<int, 2>{});
    return f(float{}, std::integral_constant<int, 1>{});
  }
  if (V == 8) return f(bft{}, std::integral_constant<int, 8>{});
  if (V == 4) return f(bft{}, std::integral_constant<int, 4>{});
  return f(bft{}, std::integral_constant<int, 2>{});
}
#define ECHO_PARTS_LAUNCH(KERN, ...)                                                                \
  do {                                                                                              \
    const bool bf_ = d->dtype != ECHO_FP32;                                                         \
    const int V_ = step_vec((long)d->B * d->H, bf_);                                                \
    const int g_ = grid_for((long)d->B * d->H / V_, 128);                                           \
    cudaStream_t st_ = (cudaStream_t)stream;                                                        \
    const cudaError_t e_ = dispatch_tv(bf_, V_, [&](auto tt_, auto vv_) {                           \
      typedef decltype(tt_) TT;                                                                     \
      constexpr int VV = decltype(vv_)::value;                                                      \
      if (n_parts == 1) return launch(KERN<TT, VV, 1>, dim3(g_), dim3(128), 0, st_, 1, __VA_ARGS__); \
      if (n_parts == 2) return launch(KERN<TT, VV, 2>, dim3(g_), dim3(128), 0, st_, 1, __VA_ARGS__); \
      return launch(KERN<TT, VV, 3>, dim3(g_), dim3(128), 0, st_, 1, __VA_ARGS__);                  \
    });                                                                                             \
    if (e_ != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e_)); \
    return check_launch(fn);                                                                        \
  } while (0)

extern "C" echo_status echo_lstm_fwd_parts(const echo_lstm_desc* d, int32_t n_parts, const void* parts_t,
                                           int64_t part_stride, const float* bias, const float* c_prev,
                                           float* c_out, void* h_out, void* stream) {
  const char* fn = "echo_lstm_fwd_parts";
  ECHO_PARTS_CHECK();
  ECHO_REQ(parts_t, "parts_t");
  ECHO_OPT(bias, "bias");
  ECHO_REQ(c_prev, "c_prev");
  ECHO_REQ(c_out, "c_out");
  ECHO_REQ(h_out, "h_out");
  if (c_out == c_prev) return fail(ECHO_ERR_INVALID, "%s: c_out must not alias c_prev", fn);
  ECHO_PARTS_LAUNCH(lstm_fwd_parts_kernel, d->B, d->H, (const TT*)parts_t, (long)part_stride, bias, c_prev, c_out,
                    (TT*)h_out);
}

extern "C" echo_status echo_lstm_cscan_parts(const echo_lstm_desc* d, int32_t T, int32_t n_parts, const void* parts,
                                             int64_t part_stride, int64_t step_stride, const float* bias,
                                             const float* c0, float* c_ws, void* stream) {
  const char* fn = "echo_lstm_cscan_parts";
  ECHO_PARTS_CHECK();
  if (T <= 0) return fail(ECHO_ERR_INVALID, "%s: T=%d must be > 0", fn, T);
  if (step_stride % 8 || (step_stride < 0 ? -step_stride : step_stride) < 4L * d->B * d->H)
    return fail(ECHO_ERR_INVALID, "%s: |step_stride|=%lld must be a multiple of 8 and >= 4*B*H", fn,
                (long long)step_stride);
  ECHO_REQ(parts, "parts");
  ECHO_OPT(bias, "bias");
  ECHO_REQ(c0, "c0");
  ECHO_REQ(c_ws, "c_ws");
  ECHO_PARTS_LAUNCH(lstm_cscan_parts_kernel, T, d->B, d->H, (const TT*)parts, (long)part_stride, (long)step_stride,
                    bias, c0, c_ws);
}

extern "C" echo_status echo_lstm_bwd_parts(const echo_lstm_desc* d, int32_t n_parts, const void* parts_t,
                                           int64_t part_stride, const float* bias, const float* c_prev,
                                           const float* c_t, const float* dh_t, float* dc, void* dA_t, void* stream) {
  const char* fn = "echo_lstm_bwd_parts";
  ECHO_PARTS_CHECK();
  ECHO_REQ(parts_t, "parts_t");
  ECHO_OPT(bias, "bias");
  ECHO_REQ(c_prev, "c_prev");
  ECHO_REQ(c_t, "c_t");
  ECHO_REQ(dh_t, "dh_t");
  ECHO_REQ(dc, "dc");
  ECHO_REQ(dA_t, "dA_t");
  ECHO_PARTS_LAUNCH(lstm_bwd_parts_kernel, d->B, d->H, (const TT*)parts_t, (long)part_stride, bias, c_prev, c_t,
                    dh_t, dc, (TT*)dA_t);
}

// ---- host side of the tcgen05 step (a0 + a1 fused)
namespace echo {
typedef CUresult (*TcEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TcEncodeFn tc_encode() {
  static TcEncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (TcEncodeFn)p;
  }
  return fn;
}
// 2-D bf16 map over a dense [rows][cols] tensor, box {64 cols, box_rows}, 128-byte swizzle
static bool tc_map(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  TcEncodeFn fn = tc_encode();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_KA, box_rows};
  cuuint32_t el[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, el,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static size_t tc_smem(int H) { return (size_t)(H / TC_KA) * (TC_A_ATOM + TC_B_ATOM) + 1024; }
}  // namespace echo

extern "C" int32_t echo_lstm_fwd_tc_supported(int32_t B, int32_t H, int32_t dtype) {
  return dtype == ECHO_BF16 && B >= 1 && B <= TC_M && H >= TC_KA && H % TC_KA == 0 && H / TC_KA <= 8 ? 1 : 0;
}

extern "C" echo_status echo_lstm_fwd_tc(const echo_lstm_desc* d, const void* gx_t, const void* h_prev, const void* Wh,
                                        const float* bias, const float* c_prev, void* gates_t, float* c_out,
                                        void* tc_t, void* h_out, void* stream) {
  const char* fn = "echo_lstm_fwd_tc";
  echo_status s = check_desc(d);
  if (s) return s;
  if (!echo_lstm_fwd_tc_supported(d->B, d->H, d->dtype))
    return fail(ECHO_ERR_UNSUPPORTED, "%s: needs bf16 storage, B <= %d, H a multiple of %d up to %d (B=%d H=%d)", fn,
                TC_M, TC_KA, 8 * TC_KA, d->B, d->H);
  ECHO_REQ(gx_t, "gx_t");
  ECHO_REQ(h_prev, "h_prev");
  ECHO_REQ(Wh, "Wh");
  ECHO_REQ(bias, "bias");
  ECHO_REQ(c_prev, "c_prev");
  ECHO_REQ(gates_t, "gates_t");
  ECHO_REQ(c_out, "c_out");
  ECHO_REQ(h_out, "h_out");
  if (d->mode == ECHO_STASH) { ECHO_REQ(tc_t, "tc_t"); }
  else if (tc_t) return fail(ECHO_ERR_INVALID, "%s: tc_t must be NULL in RECOMPUTE mode", fn);
  if (c_out == c_prev) return fail(ECHO_ERR_INVALID, "%s: c_out must not alias c_prev", fn);
  CUtensorMap mH, mW;
  if (!tc_map(&mH, h_prev, d->H, d->B, TC_M) || !tc_map(&mW, Wh, d->H, 4 * d->H, TC_U))
    return fail(ECHO_ERR_CUDA, "%s: cuTensorMapEncodeTiled failed", fn);
  const size_t smem = tc_smem(d->H);
  typedef __nv_bfloat16 bf;
  const void* k = d->mode == ECHO_STASH ? (const void*)lstm_fwd_tc_kernel<1> : (const void*)lstm_fwd_tc_kernel<0>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: cudaFuncSetAttribute: %s", fn, cudaGetErrorString(e));
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid(d->H / TC_U);
  if (d->mode == ECHO_STASH)
    e = launch(lstm_fwd_tc_kernel<1>, grid, dim3(TC_THREADS), smem, st, 1, mH, mW, d->B, d->H, (const bf*)gx_t, bias, c_prev,
               (bf*)gates_t, c_out, (bf*)tc_t, (bf*)h_out);
  else
    e = launch(lstm_fwd_tc_kernel<0>, grid, dim3(TC_THREADS), smem, st, 1, mH, mW, d->B, d->H, (const bf*)gx_t, bias, c_prev,
               (bf*)gates_t, c_out, (bf*)nullptr, (bf*)h_out);
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e));
  return check_launch(fn);
}
