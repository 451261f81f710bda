/* echo.h — C ABI of libecho.so, the B200 (sm_100a) hot path of Echo
 * (Zheng et al., arXiv 1805.08899; /root/reference/PAPER.md).
 *
 * Echo recomputes "the feature maps of the attention and RNN layers rather
 * than stashing them persistently in the GPU memory" and fuses
 * the recomputation into the backward pass (Echo-dagger).
 * This library provides the cheap non-FC parts of that path as fused kernels;
 * the fully-connected contractions around them (Eq. 1) are
 * done by the caller (cuBLAS) and are outside this library by design.
 *
 * Conventions for every compute entry point
 *   - All tensor pointers are DEVICE pointers, row-major, densely packed unless
 *     a stride is given.  The CALLER owns every buffer; the library never
 *     allocates or frees device memory, never synchronises, keeps no device
 *     state and is re-entrant.
 *   - "storage dtype" s is fp32 or bf16 (echo_dtype); all math and
 *     accumulation are fp32.  Tensors documented "fp32" are fp32 in both.
 *   - Every value the STASH mode stores is rounded to s once, at production;
 *     both modes read the rounded value (rounding contract, DESIGN.md a4), so
 *     STASH and RECOMPUTE gradients are bit-identical.
 *   - Vectorised 128-bit access: every pointer must be 16-byte aligned and the
 *     innermost extents (H, A, Hk, L) multiples of 8, else ECHO_ERR_INVALID.
 *   - Kernels are launched on `stream` (a cudaStream_t passed as void*).
 *     Launch-configuration errors are reported synchronously (cudaGetLastError
 *     after the launch -> ECHO_ERR_CUDA); asynchronous faults surface at the
 *     caller's next synchronisation.  Safe to record in a CUDA graph.
 *   - On any non-OK return nothing has been launched (validation happens
 *     first) except for ECHO_ERR_CUDA; echo_last_error() returns a
 *     thread-local message describing the last failure.
 */
#ifndef ECHO_H_
#define ECHO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ECHO_ABI_VERSION 2

typedef enum {
  ECHO_OK = 0,
  ECHO_ERR_INVALID = 1,     /* bad argument / parse / validation            */
  ECHO_ERR_GRAPH = 2,       /* estimator pipeline error (cycle, bad op)      */
  ECHO_ERR_CAPACITY = 3,    /* size cap (shared memory tile, report buffer) */
  ECHO_ERR_MISMATCH = 4,    /* debug self-verification failed                */
  ECHO_ERR_CUDA = 5,        /* CUDA launch error                             */
  ECHO_ERR_UNSUPPORTED = 6
} echo_status;

typedef enum { ECHO_FP32 = 0, ECHO_BF16 = 1 } echo_dtype;   /* storage dtype s */
typedef enum { ECHO_STASH = 0, ECHO_RECOMPUTE = 1 } echo_mode;

const char* echo_last_error(void);
int echo_abi_version(void);

/* ===================================================================== LSTM
 * PAPER.md §2, lines 101-112 (Fig. 1): the cell's FC outputs (Eq. 1) enter the
 * non-linear block f (slicing + element-wise ops) which outputs h_t, c_t.
 * Gate order along the 4H axis: i | f | g | o (contiguous H blocks).
 *   i = sigma(A_i), f = sigma(A_f), g = tanh(A_g), o = sigma(A_o)
 *   c_t = f * c_{t-1} + i * g ;  h_t = o * tanh(c_t)
 * Feature maps (Echo plan, DESIGN.md table T3): both modes stash the gates
 * [B,4H]; STASH additionally keeps c_t (fp32), tanh(c_t) and h_t; RECOMPUTE
 * regenerates c (a2) and tanh(c), h (a3, echo_lstm_bwd_recompute) in the
 * backward pass.  Time order is the caller's processing order (a reverse-
 * direction layer simply processes t = T-1..0).
 */
typedef struct {
  int32_t B;          /* batch rows, > 0                    */
  int32_t H;          /* hidden width, > 0, multiple of 8   */
  int32_t dtype;      /* echo_dtype                          */
  int32_t mode;       /* echo_mode                           */
} echo_lstm_desc;

/* a1 — forward pointwise step.
 *  gx_t    [B,4H] s   x_t W_x^T (+ b) (+ h_{t-1} W_h^T when gh_t == NULL)
 *  gh_t    [B,4H] s   h_{t-1} W_h^T, or NULL if already accumulated into gx_t
 *  bias    [4H]  fp32 or NULL if folded into gx_t
 *  c_prev  [B,H] fp32 c_{t-1}
 *  gates_t [B,4H] s   OUT i|f|g|o (the stash in both modes); may alias gx_t
 *  c_out   [B,H] fp32 OUT c_t (must not alias c_prev)
 *  tc_t    [B,H] s    OUT tanh(c_t): required in STASH, must be NULL in RECOMPUTE
 *  h_out   [B,H] s    OUT h_t                                                   */
echo_status echo_lstm_fwd(const echo_lstm_desc* d, const void* gx_t, const void* gh_t,
                          const float* bias, const float* c_prev, void* gates_t,
                          float* c_out, void* tc_t, void* h_out, void* stream);

/* a2 — cell-state regeneration scan (RECOMPUTE backward prologue, run once per
 * layer before the reverse time loop).  Re-executes the mirrored c-chain from
 * the stashed gates and c_0 (Fig. 4 step 4; recomputation path
 * Fig. 8(c)), with the exact device functions of a1.
 *  gates [T,B,4H] s   stashed gates in processing order
 *  c0    [B,H] fp32
 *  c_ws  [T,B,H] fp32 OUT c_1..c_T (transient workspace owned by the caller)
 *  h_ws  [T,B,H] s    OUT h_1..h_T, bit-identical to a1's outputs, or NULL (used when a
 *                     layer's outputs are themselves mirrored, e.g. the encoder states H_s
 *                     that the attention backward reads at every decoder step)            */
echo_status echo_lstm_cscan(const echo_lstm_desc* d, int32_t T, const void* gates,
                            const float* c0, float* c_ws, void* h_ws, void* stream);

/* a1 fused over the recurrence (Echo-dagger fusion): steps
 * k0..k1-1 of one layer (direction) in ONE cooperative launch.  Per step:
 *   gates_k = a1( round_s(gx[t] + h_{k-1} W_h^T) + bias, c_{k-1} ),  t = reverse ? T-1-k : k,
 * i.e. the per-step path (cuBLAS GEMM into gx with beta = 1, then echo_lstm_fwd) with the recurrent
 * product computed inside the kernel (fp32 accumulation, fixed k order) and a grid barrier between
 * steps.  Same rounding points and the same pointwise device functions as a1; results differ from
 * the per-step path only by the GEMM's accumulation order, and are identical for STASH / RECOMPUTE.
 *  T        steps of the layer;  [k0, k1) the processing steps this launch runs (0 <= k0 < k1 <= T)
 *  gx       [T,B,4H] s  x_t W_x^T by TIME t (no bias); may alias gates when !reverse
 *  Wh       [4H,H] s    recurrent weights (row-major, gate blocks i|f|g|o)
 *  bias     [4H] fp32;  h0 [B,H] s, c0 [B,H] fp32 (state before processing step 0)
 *  gates    [T,B,4H] s  OUT activated gates by processing step k (a1's gates_t)
 *  c        fp32 OUT: STASH / c_ring == 0: [T,B,H] c_k by step; c_ring != 0: [2,B,H] ring (slot k%2).
 *           For k0 > 0 the state c_{k0-1} is read from the same buffer.
 *  tc       [T,B,H] s OUT tanh(c_k) (STASH) or NULL (RECOMPUTE)
 *  h        [T,B,H] s OUT h by TIME t (read back as h_{k-1} by later steps)
 * Errors: ECHO_ERR_INVALID; ECHO_ERR_UNSUPPORTED when no co-resident tile exists for (B, H) — the
 * caller then uses the per-step path (echo_lstm_seq_supported() asks first).                  */
echo_status echo_lstm_seq_fwd(const echo_lstm_desc* d, int32_t T, int32_t k0, int32_t k1, int32_t reverse,
                              const void* gx, const void* Wh, const float* bias, const void* h0,
                              const float* c0, void* gates, float* c, int32_t c_ring, void* tc, void* h,
                              void* stream);
/* a0 + a1 fused on the 5th-generation tensor cores (Echo-dagger fusion; SURVEY §8(f)
 * row 3): one forward step with the recurrent contraction on tcgen05.mma (accumulator in TMEM, TMA-
 * staged 128-byte-swizzled operands) and the a1 cell applied to the accumulator read back with
 * tcgen05.ld:  G = round_bf16(gx_t + h_prev W_h^T) ; A = G + bias ; then exactly a1's gate / cell /
 * hidden device functions.  Same outputs as echo_lstm_fwd after the caller's beta = 1 GEMM into gx_t,
 * up to the GEMM's accumulation order; STASH and RECOMPUTE give identical gates / c / h.
 *  gx_t    [B,4H] bf16  x_t W_x^T (no bias); may alias gates_t
 *  h_prev  [B,H] bf16   dense;  Wh [4H,H] bf16 dense row-major (gate blocks i|f|g|o);  bias [4H] fp32
 *  c_prev, c_out, gates_t, tc_t, h_out as echo_lstm_fwd
 * Requirements (echo_lstm_fwd_tc_supported): bf16 storage, B <= 128, H a multiple of 64, H <= 512.
 * Grid: H/16 CTAs of 512 threads, ~193 KB shared memory each.  Errors: ECHO_ERR_UNSUPPORTED, ECHO_ERR_INVALID. */
echo_status echo_lstm_fwd_tc(const echo_lstm_desc* d, const void* gx_t, const void* h_prev, const void* Wh,
                             const float* bias, const float* c_prev, void* gates_t, float* c_out, void* tc_t,
                             void* h_out, void* stream);
int32_t echo_lstm_fwd_tc_supported(int32_t B, int32_t H, int32_t dtype);

/* ---- Mirror plan (the prior-work baseline, Chen et al.; Table 1, 749, 951;
 * estimator strategy "mirror", R25).  Mirror recomputes every cheap op of the cell,
 * so per step it keeps the INPUTS of the pre-activation adds -- the n_parts separate FC outputs
 * (input projection(s) and h_{t-1} W_h^T) -- and h_t (an FC input), instead of the gates.  The
 * kernels regenerate A = ((P_0 + P_1) + P_2) + b in fp32 in that order (a1's order for gx, gh,
 * bias) and run the same gate / cell / gradient functions as a1 / a2 / a3.
 *  n_parts      1..3;  part q of a step is at parts + q * part_stride (elements, >= 4*B*H)
 *  parts_t      [n_parts][B,4H] s of this step;  bias [4H] fp32 or NULL
 * echo_lstm_fwd_parts: c_prev [B,H] fp32 IN, c_out [B,H] fp32 OUT (must not alias c_prev),
 *   h_out [B,H] s OUT (kept by the Mirror plan).
 * echo_lstm_cscan_parts: c_1..c_T of the layer into c_ws [T,B,H] fp32 (processing order) from
 *   c0; step k's parts at parts + k * step_stride (|step_stride| >= 4*B*H; negative walks a
 *   time-ordered buffer backwards for a reverse-direction layer).
 * echo_lstm_bwd_parts: as echo_lstm_bwd_recompute in RECOMPUTE mode with the gates regenerated from the
 *   parts and no h output (h_t is kept); dA_t [B,4H] s OUT may alias part 0 of the step.
 * Device pointers, 16-byte aligned; desc->mode is not used.  Errors: ECHO_ERR_INVALID.           */
echo_status echo_lstm_fwd_parts(const echo_lstm_desc* d, int32_t n_parts, const void* parts_t,
                                int64_t part_stride, const float* bias, const float* c_prev,
                                float* c_out, void* h_out, void* stream);
echo_status echo_lstm_cscan_parts(const echo_lstm_desc* d, int32_t T, int32_t n_parts, const void* parts,
                                  int64_t part_stride, int64_t step_stride, const float* bias,
                                  const float* c0, float* c_ws, void* stream);
echo_status echo_lstm_bwd_parts(const echo_lstm_desc* d, int32_t n_parts, const void* parts_t,
                                int64_t part_stride, const float* bias, const float* c_prev,
                                const float* c_t, const float* dh_t, float* dc, void* dA_t, void* stream);

/* 1 if echo_lstm_seq_fwd has a co-resident tile for this (B, H, dtype) on the current device. */
int32_t echo_lstm_seq_supported(int32_t B, int32_t H, int32_t dtype);

/* a3 (+ a2) — backward step with fused recomputation (Echo-dagger fusion; the
 * recomputation path of the mirrored c-chain, Fig. 4 step 4, and Fig. 8(c)).
 * One call per backward step t = T-1 .. 0 (processing order) of one layer (direction):
 *   RECOMPUTE: regenerate i,f,g,o from the stashed gates, tanh(c_t) and h_t from c_t, then
 *              do = dh tc ; dc = carry + dh o (1 - tc^2) ; di = dc g ; dg = dc i ; df = dc c_{t-1}
 *              carry' = dc f ; dA = [di i(1-i) | df f(1-f) | dg (1-g^2) | do o(1-o)]
 *   STASH:     the same gradient from the stashed gates, c and tanh(c) (the paper's Baseline).
 *  T, t      steps of the layer and this step, 0 <= t < T
 *  flags     ECHO_BWD_REGEN_C (RECOMPUTE only): first run the a2 scan, c_1..c_T into ws from the
 *            gates and c0 (pass it on the first backward call, t = T-1; or fill ws with
 *            echo_lstm_cscan, which can also regenerate the layer outputs h)
 *  gates     [T,B,4H] s  stashed i|f|g|o of every step (both modes)
 *  c0        [B,H] fp32  initial cell state
 *  c_st      STASH: [T,B,H] fp32 c_1..c_T (c_{t-1} is read for t > 0); RECOMPUTE: NULL
 *  tc_st     STASH: [T,B,H] s tanh(c_t);                                RECOMPUTE: NULL
 *  dh_t      [B,H] fp32  total dLoss/dh_t (from above + recurrent)
 *  dc        [B,H] fp32  IN dLoss/dc_t carried from t+1; OUT dLoss/dc_{t-1}
 *  dA_t      [B,4H] s    OUT dLoss/dA_t (pre-activations); may alias step t of gates
 *  h_regen_t [B,H] s     RECOMPUTE: OUT regenerated h_t, bit-identical to a1's (for the caller's
 *                        dW GEMMs) or NULL; STASH: NULL
 *  ws        RECOMPUTE: caller-owned workspace holding c_1..c_T fp32 across the layer's backward
 *            calls; STASH: NULL.   ws_bytes: two-call convention -- with ws == NULL and ws_bytes
 *            != NULL the call only writes the needed size (T*B*H*4 in RECOMPUTE, 0 in STASH) and
 *            returns ECHO_OK; with ws != NULL a non-NULL *ws_bytes is its capacity (checked).
 * Errors: ECHO_ERR_INVALID (t out of range, missing / misaligned buffer for the mode, unknown
 * flags), ECHO_ERR_CAPACITY (ws too small), ECHO_ERR_CUDA.                                     */
#define ECHO_BWD_REGEN_C 1u
echo_status echo_lstm_bwd_recompute(const echo_lstm_desc* d, int32_t T, int32_t t, uint32_t flags,
                                    const void* gates, const float* c0, const float* c_st, const void* tc_st,
                                    const float* dh_t, float* dc, void* dA_t, void* h_regen_t, void* ws,
                                    size_t* ws_bytes, void* stream);

/* ===================================================================== MLP attention
 * PAPER.md §2 lines 129-133 and Fig. 7 (the scoring function as
 * broadcast-add + tanh):  for each row b and source position s < len_b
 *   E_s = tanh(qp_b + Kp_{b,s})   score_s = E_s . v   alpha = softmax_s(score)
 *   ctx_b = sum_s alpha_s Hs_{b,s}
 * One query per row (the NMT decoder calls this once per target step).
 * Feature maps (Echo plan, DESIGN.md table T4): STASH keeps the tanh feature
 * map [B,Ts,A] s and alpha [B,Ts] fp32 (and the caller keeps ctx); RECOMPUTE
 * keeps nothing and echo_attn_bwd_recompute regenerates it, the scores, alpha and ctx.
 * The tanh feature map is stored as its input Z = round_s(qp + Kp) (same bytes
 * as E = tanh(Z); E and tanh' = 1 - E^2 are evaluated in fp32 from Z in both
 * modes, which keeps bf16 gradients accurate near saturation; R15).
 */
typedef struct {
  int32_t B, Ts, A, Hk;   /* > 0; A, Hk multiples of 8; Ts <= 4096                  */
  int32_t dtype;          /* echo_dtype                                              */
  int32_t mode;           /* echo_mode                                               */
  int64_t kp_stride_b;    /* element stride of Kp (and dKp) between rows b (Ts*A for [B,Ts,A], A for [Ts,B,A]) */
  int64_t kp_stride_s;    /* element stride of Kp (and dKp) between positions s (A, or B*A)                 */
  int64_t hs_stride_b;    /* element stride of Hs (and dHs) between rows b (Ts*Hk or Hk)                    */
  int64_t hs_stride_s;    /* element stride of Hs (and dHs) between positions s (Hk or B*Hk)                */
} echo_attn_desc;

/* a5 — forward.
 *  qp [B,A] s, Kp strided [B,Ts,A] s, v [A] s, Hs strided [B,Ts,Hk] s, src_len [B] int32 in
 *  [1,Ts] or NULL (= Ts), ctx [B,Hk] s OUT, E_st [B,Ts,A] s OUT Z = qp + Kp (STASH) / NULL,
 *  alpha_st [B,Ts] fp32 OUT (STASH) / NULL.  Masked positions get alpha = 0.
 *  src_len lives on the device, so the kernels clamp an out-of-range entry to [1,Ts]; with the
 *  environment flag ECHO_CHECK_SRC_LEN=1 every attention entry point taking src_len first copies it
 *  to the host (synchronizing `stream`) and returns ECHO_ERR_INVALID for any entry outside [1,Ts]
 *  (not while the stream is being captured into a CUDA graph).                     */
echo_status echo_attn_fwd(const echo_attn_desc* d, const void* qp, const void* Kp, const void* v,
                          const void* Hs, const int32_t* src_len, void* ctx, void* E_st,
                          float* alpha_st, void* stream);

/* a6 — backward with fused recomputation (Fig. 10: the add / tanh feature maps
 * stay on the mirror path).  Per decoder step (reverse order), per row b:
 *   regenerate E_s = tanh(round_s(qp_b + Kp_{b,s})), score, alpha and ctx_b (RECOMPUTE), or read
 *   the stashed Z, alpha (STASH);  dalpha_s = dctx_b . Hs_{b,s};  ds = alpha (dalpha - sum alpha dalpha)
 *   dE_s = ds_s v (1 - E_s^2);  dqp_b = sum_s dE_s;  dKp_{b,s} += dE_s;  dHs_{b,s} += alpha_s dctx_b;
 *   dv += sum_{b,s} ds_s E_s (per-row partials in ws, reduced in ascending b: no atomics)
 *  qp, Kp           RECOMPUTE: required (E is regenerated from them); STASH: may be NULL
 *  E_st, alpha_st   STASH inputs from a5 (NULL in RECOMPUTE)
 *  dctx   [B,Hk] fp32    dLoss/dctx
 *  dqp    [B,A] fp32     OUT dLoss/dqp (overwritten)
 *  dKp    [B,Ts,A] fp32  ACCUMULATED (+=) dLoss/dKp, same strides as Kp
 *  dHs    [B,Ts,Hk] fp32 ACCUMULATED (+=) dLoss/dHs, same strides as Hs
 *  dv     [A] fp32       OUT or NULL: when non-NULL, dv = sum_b ws[b,:] (ascending b) after this
 *                        step's partials were added -- pass it on the last call of a backward pass
 *  ctx_regen [B,Hk] s    OUT regenerated ctx (RECOMPUTE; bit-identical to a5's) or NULL
 *  ws     [B,A] fp32     caller-owned per-row dv partials, ACCUMULATED (+=) across the calls of one
 *                        backward pass; zero it before the first call.  ws_bytes: two-call
 *                        convention -- ws == NULL with ws_bytes != NULL writes B*A*4 and returns
 *                        ECHO_OK without launching; otherwise a non-NULL *ws_bytes is checked.
 * Errors: ECHO_ERR_INVALID (shape, stride, missing buffer for the mode, misalignment),
 * ECHO_ERR_CAPACITY (ws too small), ECHO_ERR_CUDA.                                             */
echo_status echo_attn_bwd_recompute(const echo_attn_desc* d, const void* qp, const void* Kp, const void* v,
                                    const void* Hs, const int32_t* src_len, const void* E_st,
                                    const float* alpha_st, const float* dctx, float* dqp, float* dKp,
                                    float* dHs, float* dv, void* ctx_regen, void* ws, size_t* ws_bytes,
                                    void* stream);

/* a6, deferred accumulation (the algorithmic-minimum variant).  The same step as
 * echo_attn_bwd_recompute without the per-step dKp / dH_s read-modify-write: it writes this step's
 * softmax-backward rows instead and echo_attn_bwd_finish accumulates dKp / dH_s over all steps
 * once, with the per-step expressions in the per-step order (t = Td-1 .. 0): results are
 * bit-identical to calling echo_attn_bwd_recompute every step.
 *  ds_out     [B,Ts] fp32 OUT  ds_s = alpha_s (dalpha_s - sum alpha dalpha) (0 for s >= len_b)
 *  alpha_out  [B,Ts] fp32 OUT  regenerated alpha (RECOMPUTE; NULL in STASH, where alpha is stashed)
 * dv_part [B,A] fp32 ACCUMULATED per-row dv partials (the ws of echo_attn_bwd_recompute; reduce them
 * with one final echo_attn_bwd_recompute call or by summing rows in ascending b).
 * Other arguments as echo_attn_bwd_recompute.  Errors as echo_attn_bwd_recompute; ECHO_ERR_UNSUPPORTED where only the
 * generic (non-TMA) kernel fits (Ts > 256).                                                      */
echo_status echo_attn_bwd_deferred(const echo_attn_desc* d, const void* qp, const void* Kp, const void* v,
                                   const void* Hs, const int32_t* src_len, const void* E_st,
                                   const float* alpha_st, const float* dctx, float* dqp, float* dv_part,
                                   void* ctx_regen, float* ds_out, float* alpha_out, void* stream);

/* Finish the deferred accumulations over the Td steps of one backward pass:
 *   dKp[b,s,:] = sum_{t=Td-1..0} (ds_t[b,s] v) (1 - tanh(z_t[b,s,:])^2),
 *   z_t = round_s(qp_t[b,:] + Kp[b,s,:]) (RECOMPUTE) or the stashed z_t (STASH)
 *   dHs[b,s,:] = sum_{t=Td-1..0} alpha_t[b,s] dctx_t[b,:]          (both OVERWRITTEN)
 *  qp_all [Td,B,A] s (RECOMPUTE) | E_st_all [Td,B,Ts,A] s (STASH); Kp as in echo_attn_bwd_recompute
 *  ds_all, alpha_all [Td,B,Ts] fp32 (the per-step ds_out / alpha_out, or the stashed alpha)
 *  dctx_all [Td,B,Hk] fp32 (the per-step dctx)
 * Errors: ECHO_ERR_INVALID, ECHO_ERR_CAPACITY (Td*Ts too large for the staged rows).               */
echo_status echo_attn_bwd_finish(const echo_attn_desc* d, int32_t Td, const void* qp_all, const void* Kp,
                                 const void* E_st_all, const void* v, const int32_t* src_len,
                                 const float* ds_all, const float* alpha_all, const float* dctx_all,
                                 float* dKp, float* dHs, void* stream);

/* One decoder step of the deferred accumulation, added to the running sums: dKp[b,s,:] += dE_t and
 * dH_s[b,s,:] += alpha_t[b,s] dctx_t[b,:] for s < len_b (rows s >= len_b untouched), with exactly
 * the per-step expressions of echo_attn_bwd_recompute (same bits when called for t = Td-1 .. 0 in order).
 * Lets the caller run the read-modify-write of step t OFF the critical path (e.g. on a second
 * stream after echo_attn_bwd_deferred of step t) while the recurrence continues.
 *  qp_t [B,A], E_st_t [B,Ts,A] (STASH), ds_t / alpha_t [B,Ts] fp32, dctx_t [B,Hk] fp32: step t's rows. */
echo_status echo_attn_bwd_accumulate(const echo_attn_desc* d, const void* qp_t, const void* Kp, const void* E_st_t,
                                     const void* v, const int32_t* src_len, const float* ds_t,
                                     const float* alpha_t, const float* dctx_t, float* dKp, float* dHs,
                                     void* stream);

/* dv[a] (+)= sum_b dv_part[b,a] in ascending b (deterministic; the reduction echo_attn_bwd_recompute
 * runs when given dv), for the deferred variants above.  accumulate != 0 adds to dv.            */
echo_status echo_attn_dv_reduce(int32_t B, int32_t A, const float* dv_part, float* dv,
                                int32_t accumulate, void* stream);

/* ===================================================================== dot-product softmax + dropout
 * Transformer attention probabilities (§6.3.2): P =
 * softmax(scale * S) per row, P_d = P * m / (1 - p) with keep-mask m.  Echo
 * recomputes P in the backward pass and stores the dropout feature map as a
 * 1-bit mask (Alg. 1 line 18).
 * m is Philox4x32-10: element n (row-major) uses counter offset + n/4 and key
 * seed, word n%4; keep iff (word >> 8) >= floor(p * 2^24)  (R19).
 */
typedef struct {
  int32_t R, L;           /* rows, row length (L multiple of 8, <= 2048)   */
  int32_t dtype, mode;
  float scale;            /* applied to S before the softmax               */
  float dropout_p;        /* in [0, 1)                                     */
  uint64_t seed, offset;  /* Philox key and counter base                   */
} echo_dot_desc;

/* a7 forward.  S [R,L] s (caller's Q K^T), Pd [R,L] s OUT (feeds the caller's PV GEMM),
 *  P_st [R,L] s OUT (STASH) / NULL, mask: STASH byte mask [R,L] uint8 OUT;
 *  RECOMPUTE bit mask [R, L/8] uint8 OUT (bit j%8 of byte j/8), or NULL: nothing is kept and
 *  the backward regenerates the mask from (seed, offset) (Philox is counter-based; R30).       */
echo_status echo_dot_softmax_fwd(const echo_dot_desc* d, const void* S, void* Pd, void* P_st,
                                 uint8_t* mask, void* stream);

/* a7 backward.  dPd [R,L] s = dLoss/dP_d.  STASH: reads P_st + byte mask (S may be NULL);
 *  RECOMPUTE: reads S + bit mask (or regenerates the mask from (seed, offset) when mask is
 *  NULL) and regenerates P.  dS [R,L] s OUT = dLoss/dS (may alias dPd);
 *  Pd_regen [R,L] s OUT (RECOMPUTE; for the caller's dV GEMM) or NULL.                */
echo_status echo_dot_softmax_bwd(const echo_dot_desc* d, const void* S, const void* P_st,
                                 const uint8_t* mask, const void* dPd, void* dS, void* Pd_regen,
                                 void* stream);

/* ===================================================================== a0 dense contractions
 * IEEE-fp32 GEMM for the FCs around the hot path (Eq. 1 / Eq. 2, PAPER.md:104-106, 389-391;
 * outside the Echo decision): C = alpha * op(A) op(B) + beta * C, row-major storage.
 *  op(A) M x K: transA == 0 -> A[m*lda + k]; transA != 0 -> A[k*lda + m]
 *  op(B) K x N: transB == 0 -> B[k*ldb + n]; transB != 0 -> B[n*ldb + k]
 * SIMT fp32 FMA with fixed k order; split-K across a thread-block cluster whose partial tiles are
 * summed in rank order through distributed shared memory (deterministic, no workspace).
 * Requirements (echo_gemm_f32_supported): N, lda, ldb, ldc multiples of 4; K % 4 == 0 when
 * !transA or transB; M % 4 == 0 when transA; 16-byte aligned pointers.
 * Errors: ECHO_ERR_UNSUPPORTED (shape / stride), ECHO_ERR_INVALID (alignment).                 */
echo_status echo_gemm_f32(int32_t M, int32_t N, int32_t K, float alpha, const float* A, int64_t lda,
                          int32_t transA, const float* B, int64_t ldb, int32_t transB, float beta,
                          float* C, int64_t ldc, void* stream);
int32_t echo_gemm_f32_supported(int32_t M, int32_t N, int32_t K, int32_t transA, int32_t transB,
                                int64_t lda, int64_t ldb, int64_t ldc);

/* ===================================================================== output layer
 * Fused softmax cross-entropy of the model's output layer (§2; reading
 * R10: mean CE over the N = B*Td target tokens).  Outside the Echo decision (its probabilities
 * are kept in both modes) -- one pass instead of the ~10 framework launches of the plain form.
 *  N, V          rows (tokens) and classes; V <= 51200
 *  logits        [N, V] fp32, row-major, IN: x W^T (bias not yet added); OUT: overwritten in
 *                place with dLoss/dlogits = (softmax(x + bias) - onehot(label)) / N
 *  bias          [V] fp32 or NULL
 *  labels        [N] int64 in [0, V) (not checked on the device)
 *  row_loss      [N] fp32 OUT: logsumexp(x + b) - (x + b)[label]; the loss is their mean
 *  dlogits_bf16  [N, V] bf16 OUT copy of dLoss/dlogits (round to nearest) or NULL
 * All device pointers; 16-byte aligned logits / bias (8-byte bf16 output) when V % 4 == 0.
 * Deterministic (fixed-order block reductions).  Errors: ECHO_ERR_INVALID, ECHO_ERR_CAPACITY.  */
echo_status echo_xent_fwd_bwd(int32_t N, int32_t V, float* logits, const float* bias,
                              const int64_t* labels, float* row_loss, void* dlogits_bf16,
                              void* stream);

/* Column sums out[c] (+)= sum_r x[r*ld + c] of a [rows, cols] fp32 / bf16 matrix, accumulated in
 * fp64 in a fixed order and rounded once to fp32: the bias gradients (Eq. 2, PAPER.md:389-391,
 * db = sum over every row of the batch of dY), which are cancellation-dominated sums of 10^4-10^5
 * terms (reading R14).  dtype: ECHO_FP32 / ECHO_BF16 (an echo_dtype); accumulate: 0 overwrite,
 * 1 add.  Deterministic.  Errors: ECHO_ERR_INVALID.                                         */
echo_status echo_colsum(int32_t rows, int32_t cols, int64_t ld, int32_t dtype, const void* x, float* out,
                        int32_t accumulate, void* stream);

/* ===================================================================== dropout on the LSTM inputs
 * Dropout of the NMT embeddings (reading R31, Sockeye's embedding dropout) with the paper's 1-bit
 * encoding of its feature map (Alg. 1 line 18) or, reading R30, no kept mask:
 * keep(n) from Philox4x32-10 exactly as a7 (counter offset + n/4, key seed, word n%4, keep iff
 * (word >> 8) >= floor(p 2^24); R19), scale 1/(1-p) rounded to fp32.
 *  n          elements, a multiple of 8;  p in [0, 1)
 *  mask_kind  0: none (regenerated from (seed, offset)), 1: bits [n/8] uint8 (bit k of byte j =
 *             element 8j + k), 2: bytes [n] uint8 (0/1; 8-byte aligned)
 * echo_dropout_fwd: y [n] = round_s(x * keep / (1-p)) (x, y in dtype; 16-byte aligned), the keep-
 *   mask written to mask in mask_kind (mask may be NULL for kind 0).
 * echo_dropout_apply: y (+)= x * keep / (1-p) with keep DECODED from the kept mask (kinds 1, 2) or
 *   regenerated (kind 0): re-applies a mirrored dropout (x, y storage dtype) and back-propagates
 *   through it (x = dLoss/dy, y = dLoss/dx, fp32).  accumulate: 0 overwrite, 1 add (fp32 sum,
 *   then rounded to y_dtype).  x and y may alias when accumulate is 0.
 * Device pointers.  Errors: ECHO_ERR_INVALID.                                                     */
echo_status echo_dropout_fwd(int64_t n, int32_t dtype, float p, uint64_t seed, uint64_t offset, const void* x,
                             void* y, uint8_t* mask, int32_t mask_kind, void* stream);
echo_status echo_dropout_apply(int64_t n, float p, uint64_t seed, uint64_t offset, const uint8_t* mask,
                               int32_t mask_kind, int32_t x_dtype, const void* x, int32_t y_dtype, void* y,
                               int32_t accumulate, void* stream);

/* 1-bit feature maps for the automatic fx pass (fx_pass.py; Alg. 1 line 18):
 * a ReLU's gradient reads only the sign of its output and a dropout's only its keep-mask.
 * echo_sign_pack:   bits[j] bit k = (x[8j + k] > 0)  (x dtype 0 fp32, 1 bf16, 2 u8 / bool: != 0)
 * echo_bits_unpack: out[i] = bit i ? 1 : 0  (out dtype 0 fp32, 1 bf16, 2 u8 / bool)
 *  n elements (> 0); bits [(n + 7) / 8] uint8; device pointers.  Errors: ECHO_ERR_INVALID.          */
echo_status echo_sign_pack(int64_t n, int32_t dtype, const void* x, uint8_t* bits, void* stream);
echo_status echo_bits_unpack(int64_t n, const uint8_t* bits, int32_t dtype, void* out, void* stream);

/* Backward of the attention hidden a_t = tanh(pre_t) (reading R7, §2;
 * tanh keeps its output): dpre[i] = da[i] * (1 - a[i]^2), fp32 arithmetic in that
 * order (a read in its storage dtype).  Outside the Echo decision (a_t is kept in both modes).
 *  n       elements;  dtype  storage dtype of a (ECHO_FP32 / ECHO_BF16)
 *  a       [n] device, storage dtype;  da  [n] fp32 device;  dpre  [n] fp32 device OUT (may alias da)
 * Errors: ECHO_ERR_INVALID.                                                                      */
echo_status echo_tanh_bwd(int64_t n, int32_t dtype, const void* a, const float* da, float* dpre, void* stream);

/* ===================================================================== footprint estimator
 * Host-only, integer, deterministic.  Runs the adjusted pass pipeline of
 * Fig. 14: Gradient -> InferShape&Type -> EdgeUseRef ->
 * Echo (Algorithm 1) -> DeadNodeElimination
 * -> InferShape&Type -> liveness planning, and reports per-edge decisions and
 * exact byte totals.
 *  graph_json   NUL-terminated graph document (schema in DESIGN.md "Graph
 *               document": {version:1, placeholders:[...], nodes:[...], outputs:[...]})
 *  config_json  NUL-terminated strategy config {strategy: "baseline"|"mirror"|"echo",
 *               compute_heavy_ops, binarizable_ops, enable_dead_node,
 *               enable_binarization, regenerate_masks, flop_threshold, weight_multiplier};
 *               NULL = echo defaults.  regenerate_masks (default false, echo / mirror only;
 *               DESIGN.md R30): dropout keep-masks come from a counter-based generator, so a
 *               mirrored dropout regenerates its mask instead of keeping it (0 bytes).
 *               self_verify (default false): after planning, check that every edge a gradient
 *               reads is kept or regenerable from kept edges (SPEC.md:632-639 `verify`);
 *               debug_unstash_edge [node, out]: test hook that drops that edge from the plan
 *               first (a corrupted plan; implies self_verify)
 *  report_json  caller buffer for the NUL-terminated report; may be NULL to query
 *  report_len   IN capacity of report_json; OUT bytes needed (including the NUL).
 *               Returns ECHO_ERR_CAPACITY (with *report_len set) if too small.
 * Errors: ECHO_ERR_INVALID (parse / schema / unknown op / arity / shape / an unknown or
 *         wrongly typed config key),
 *         ECHO_ERR_GRAPH (cycle or pipeline failure),
 *         ECHO_ERR_MISMATCH (self_verify: the plan leaves a gradient input unavailable). */
echo_status echo_footprint_estimate(const char* graph_json, const char* config_json,
                                    char* report_json, size_t* report_len);

#ifdef __cplusplus
}
#endif
#endif /* ECHO_H_ */
