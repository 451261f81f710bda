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

namespace echo {

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

static int grid_for(long threads, int block) {
  long g = (threads + block - 1) / block;
  const long cap = 148L * 16;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

// ---------------------------------------------------------------- a1 forward
template <typename T>
__global__ void __launch_bounds__(128) lstm_fwd_kernel(int B, int H, const T* gx,
                                                       const T* __restrict__ gh, const float* __restrict__ bias,
                                                       const float* __restrict__ c_prev, T* gates,
                                                       float* __restrict__ c_out, T* __restrict__ tc_out,
                                                       T* __restrict__ h_out) {
  pdl_wait();
  constexpr int V = St<T>::VEC;
  const int nvec = H / V;
  const long total = (long)B * nvec;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / nvec);
    const int j = (int)(idx - (long)b * nvec) * V;
    const long row4 = (long)b * 4 * H;
    float a[4][V];
#pragma unroll
    for (int g = 0; g < 4; ++g) ld16(gx + row4 + g * H + j, a[g]);
    if (gh) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float t[V];
        ld16(gh + row4 + g * H + j, t);
#pragma unroll
        for (int k = 0; k < V; ++k) a[g][k] = __fadd_rn(a[g][k], t[k]);
      }
    }
    if (bias) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float t[V];
        ldf<V>(bias + g * H + j, t);
#pragma unroll
        for (int k = 0; k < V; ++k) a[g][k] = __fadd_rn(a[g][k], t[k]);
      }
    }
    float cp[V];
    ldf<V>(c_prev + (long)b * H + j, cp);
    float gi[V], gf[V], gg[V], go[V], c[V], tc[V], h[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      gi[k] = St<T>::round(sigmoidf_(a[0][k]));
      gf[k] = St<T>::round(sigmoidf_(a[1][k]));
      gg[k] = St<T>::round(tanhf(a[2][k]));
      go[k] = St<T>::round(sigmoidf_(a[3][k]));
      c[k] = cell_update(gf[k], cp[k], gi[k], gg[k]);
      tc[k] = tanh_c<T>(c[k]);
      h[k] = hidden<T>(go[k], tc[k]);
    }
    st16(gates + row4 + 0 * H + j, gi);
    st16(gates + row4 + 1 * H + j, gf);
    st16(gates + row4 + 2 * H + j, gg);
    st16(gates + row4 + 3 * H + j, go);
    stf<V>(c_out + (long)b * H + j, c);
    if (tc_out) st16(tc_out + (long)b * H + j, tc);
    st16(h_out + (long)b * H + j, h);
  }
}

// ---------------------------------------------------------------- a2 c-regeneration scan
template <typename T, int U>
__global__ void __launch_bounds__(128) lstm_cscan_kernel(int T_, int B, int H, const T* __restrict__ gates,
                                                         const float* __restrict__ c0, float* __restrict__ cws,
                                                         T* __restrict__ hws) {
  pdl_wait();
  constexpr int V = St<T>::VEC;
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
    ldf<V>(c0 + (long)b * H + j, c);
    for (int t0 = 0; t0 < T_; t0 += U) {
      float gi[U][V], gf[U][V], gg[U][V];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t0 + u < T_) {
          const T* q = gp + (long)(t0 + u) * gstep;
          ld16_stream(q, gi[u]);
          ld16_stream(q + H, gf[u]);
          ld16_stream(q + 2 * H, gg[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t0 + u < T_) {
#pragma unroll
          for (int k = 0; k < V; ++k) c[k] = cell_update(gf[u][k], c[k], gi[u][k], gg[u][k]);
          stf<V>(cp + (long)(t0 + u) * cstep, c);
          if (hp) {                                         // mirrored outputs: h_t = o * tanh(c_t)
            float go[V], h[V];
            ld16_stream(gp + (long)(t0 + u) * gstep + 3 * H, go);
#pragma unroll
            for (int k = 0; k < V; ++k) h[k] = hidden<T>(go[k], tanh_c<T>(c[k]));
            st16(hp + (long)(t0 + u) * cstep, h);
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- a3 backward (fused recompute)
template <typename T>
__global__ void __launch_bounds__(128) lstm_bwd_kernel(int B, int H, const T* gates,
                                                       const float* __restrict__ c_prev,
                                                       const float* __restrict__ c_t, const T* __restrict__ tc_st,
                                                       const float* __restrict__ dh, float* dc, T* dA,
                                                       T* __restrict__ h_regen) {
  pdl_wait();
  constexpr int V = St<T>::VEC;
  const int nvec = H / V;
  const long total = (long)B * nvec;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / nvec);
    const int j = (int)(idx - (long)b * nvec) * V;
    const long row4 = (long)b * 4 * H;
    const long row = (long)b * H + j;
    float gi[V], gf[V], gg[V], go[V];
    ld16(gates + row4 + 0 * H + j, gi);
    ld16(gates + row4 + 1 * H + j, gf);
    ld16(gates + row4 + 2 * H + j, gg);
    ld16(gates + row4 + 3 * H + j, go);
    float cp[V], tc[V], h[V], dhv[V], dcv[V];
    ldf<V>(c_prev + row, cp);
    ldf<V>(dh + row, dhv);
    ldf<V>(dc + row, dcv);
    if (tc_st) {                       // STASH: tanh(c_t) was stashed by a1
      ld16(tc_st + row, tc);
    } else {                           // RECOMPUTE: regenerate tanh(c_t) and h_t
      float ct[V];
      ldf<V>(c_t + row, ct);
#pragma unroll
      for (int k = 0; k < V; ++k) { tc[k] = tanh_c<T>(ct[k]); h[k] = hidden<T>(go[k], tc[k]); }
    }
    float di[V], df[V], dg[V], dout[V], dcn[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const float d_o = __fmul_rn(dhv[k], tc[k]);
      const float one_m_tc2 = __fsub_rn(1.0f, __fmul_rn(tc[k], tc[k]));
      const float dcc = __fadd_rn(dcv[k], __fmul_rn(__fmul_rn(dhv[k], go[k]), one_m_tc2));
      const float d_i = __fmul_rn(dcc, gg[k]);
      const float d_g = __fmul_rn(dcc, gi[k]);
      const float d_f = __fmul_rn(dcc, cp[k]);
      dcn[k] = __fmul_rn(dcc, gf[k]);
      di[k] = St<T>::round(__fmul_rn(d_i, __fmul_rn(gi[k], __fsub_rn(1.0f, gi[k]))));
      df[k] = St<T>::round(__fmul_rn(d_f, __fmul_rn(gf[k], __fsub_rn(1.0f, gf[k]))));
      dg[k] = St<T>::round(__fmul_rn(d_g, __fsub_rn(1.0f, __fmul_rn(gg[k], gg[k]))));
      dout[k] = St<T>::round(__fmul_rn(d_o, __fmul_rn(go[k], __fsub_rn(1.0f, go[k]))));
    }
    st16(dA + row4 + 0 * H + j, di);
    st16(dA + row4 + 1 * H + j, df);
    st16(dA + row4 + 2 * H + j, dg);
    st16(dA + row4 + 3 * H + j, dout);
    stf<V>(dc + row, dcn);
    if (h_regen) st16(h_regen + row, h);
  }
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
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  const int grid = grid_for((long)d->B * d->H / V, 128);
  cudaError_t e_;
  if (d->dtype == ECHO_FP32)
    e_ = launch(lstm_fwd_kernel<float>, dim3(grid), dim3(128), 0, st, 1, d->B, d->H, (const float*)gx_t,
                (const float*)gh_t, bias, c_prev, (float*)gates_t, c_out, (float*)tc_t, (float*)h_out);
  else
    e_ = launch(lstm_fwd_kernel<__nv_bfloat16>, dim3(grid), dim3(128), 0, st, 1, d->B, d->H,
                (const __nv_bfloat16*)gx_t, (const __nv_bfloat16*)gh_t, bias, c_prev, (__nv_bfloat16*)gates_t, c_out,
                (__nv_bfloat16*)tc_t, (__nv_bfloat16*)h_out);
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
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  const int grid = grid_for((long)d->B * d->H / V, 128);
  cudaError_t e_;
  if (d->dtype == ECHO_FP32)
    e_ = launch(lstm_cscan_kernel<float, 8>, dim3(grid), dim3(128), 0, st, 1, T, d->B, d->H, (const float*)gates, c0,
                c_ws, (float*)h_ws);
  else
    e_ = launch(lstm_cscan_kernel<__nv_bfloat16, 4>, dim3(grid), dim3(128), 0, st, 1, T, d->B, d->H,
                (const __nv_bfloat16*)gates, c0, c_ws, (__nv_bfloat16*)h_ws);
  if (e_ != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e_));
  return check_launch(fn);
}

extern "C" echo_status echo_lstm_bwd(const echo_lstm_desc* d, const void* gates_t, const float* c_prev,
                                     const float* c_t, const void* tc_t, const float* dh_t, float* dc, void* dA_t,
                                     void* h_regen, void* stream) {
  const char* fn = "echo_lstm_bwd";
  echo_status s = check_desc(d);
  if (s) return s;
  ECHO_REQ(gates_t, "gates_t");
  ECHO_REQ(c_prev, "c_prev");
  ECHO_REQ(dh_t, "dh_t");
  ECHO_REQ(dc, "dc");
  ECHO_REQ(dA_t, "dA_t");
  if (d->mode == ECHO_STASH) {
    ECHO_REQ(tc_t, "tc_t");
    if (c_t) return fail(ECHO_ERR_INVALID, "%s: c_t must be NULL in STASH mode", fn);
    if (h_regen) return fail(ECHO_ERR_INVALID, "%s: h_regen must be NULL in STASH mode", fn);
  } else {
    ECHO_REQ(c_t, "c_t");
    ECHO_OPT(h_regen, "h_regen");
    if (tc_t) return fail(ECHO_ERR_INVALID, "%s: tc_t must be NULL in RECOMPUTE mode", fn);
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int V = d->dtype == ECHO_FP32 ? 4 : 8;
  const int grid = grid_for((long)d->B * d->H / V, 128);
  cudaError_t e_;
  if (d->dtype == ECHO_FP32)
    e_ = launch(lstm_bwd_kernel<float>, dim3(grid), dim3(128), 0, st, 1, d->B, d->H, (const float*)gates_t, c_prev,
                c_t, (const float*)tc_t, dh_t, dc, (float*)dA_t, (float*)h_regen);
  else
    e_ = launch(lstm_bwd_kernel<__nv_bfloat16>, dim3(grid), dim3(128), 0, st, 1, d->B, d->H,
                (const __nv_bfloat16*)gates_t, c_prev, c_t, (const __nv_bfloat16*)tc_t, dh_t, dc, (__nv_bfloat16*)dA_t,
                (__nv_bfloat16*)h_regen);
  if (e_ != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: launch: %s", fn, cudaGetErrorString(e_));
  return check_launch(fn);
}
