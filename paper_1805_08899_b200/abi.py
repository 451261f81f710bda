"""Thin ctypes binding of libecho.so (include/echo.h).  Argument marshalling only.

Every function here has the C name and the C argument order; tensors are
passed as torch tensors (device pointers via .data_ptr(), None -> NULL) and the
stream defaults to torch's current CUDA stream.  No computation happens in
Python: a missing library or a non-OK status raises immediately (there is no
CPU fallback).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libecho.so")

ECHO_OK, ECHO_ERR_INVALID, ECHO_ERR_GRAPH, ECHO_ERR_CAPACITY, ECHO_ERR_MISMATCH, ECHO_ERR_CUDA, ECHO_ERR_UNSUPPORTED = range(7)
FP32, BF16 = 0, 1
STASH, RECOMPUTE = 0, 1

# the five entry points BASELINE.json north_star names
NORTH_STAR = ("echo_lstm_fwd", "echo_lstm_bwd_recompute", "echo_attn_fwd", "echo_attn_bwd_recompute",
              "echo_footprint_estimate")
ECHO_BWD_REGEN_C = 1

EXPORTED = NORTH_STAR + (
            "echo_last_error", "echo_abi_version", "echo_lstm_cscan", "echo_attn_dv_reduce",
            "echo_dot_softmax_fwd",
            "echo_dot_softmax_bwd", "echo_xent_fwd_bwd", "echo_colsum", "echo_lstm_seq_fwd",
            "echo_lstm_seq_supported", "echo_gemm_f32", "echo_gemm_f32_supported",
            "echo_lstm_fwd_tc", "echo_lstm_fwd_tc_supported",
            "echo_attn_bwd_deferred", "echo_attn_bwd_finish", "echo_attn_bwd_accumulate", "echo_tanh_bwd",
            "echo_lstm_fwd_parts", "echo_lstm_cscan_parts", "echo_lstm_bwd_parts",
            "echo_dropout_fwd", "echo_dropout_apply", "echo_sign_pack", "echo_bits_unpack")


class EchoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libecho status {status}: {msg}")
        self.status = status


class LstmDesc(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("H", ctypes.c_int32), ("dtype", ctypes.c_int32), ("mode", ctypes.c_int32)]


class AttnDesc(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("Ts", ctypes.c_int32), ("A", ctypes.c_int32), ("Hk", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("kp_stride_b", ctypes.c_int64), ("kp_stride_s", ctypes.c_int64),
                ("hs_stride_b", ctypes.c_int64), ("hs_stride_s", ctypes.c_int64)]


class DotDesc(ctypes.Structure):
    _fields_ = [("R", ctypes.c_int32), ("L", ctypes.c_int32), ("dtype", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("scale", ctypes.c_float), ("dropout_p", ctypes.c_float),
                ("seed", ctypes.c_uint64), ("offset", ctypes.c_uint64)]


_lib = None

# Number of libecho kernel launches issued through this binding (one per compute call;
# each entry point launches exactly one kernel).  bench.py reads it to report gpu_launches.
LAUNCHES = {"count": 0}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libecho.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libecho.so not found at {path}; run `python -m paper_1805_08899_b200.build`")
    lib = ctypes.CDLL(path)
    vp, i32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64
    lib.echo_last_error.restype = ctypes.c_char_p
    lib.echo_abi_version.restype = ctypes.c_int
    sigs = {
        "echo_lstm_fwd": [ctypes.POINTER(LstmDesc)] + [vp] * 9,
        "echo_lstm_cscan": [ctypes.POINTER(LstmDesc), i32, vp, vp, vp, vp, vp],
        "echo_lstm_fwd_tc": [ctypes.POINTER(LstmDesc)] + [vp] * 10,
        "echo_sign_pack": [ctypes.c_int64, i32, vp, vp, vp],
        "echo_bits_unpack": [ctypes.c_int64, vp, i32, vp, vp],
        "echo_lstm_fwd_tc_supported": [i32, i32, i32],
        "echo_lstm_bwd_recompute": [ctypes.POINTER(LstmDesc), i32, i32, ctypes.c_uint32] + [vp] * 11,
        "echo_attn_fwd": [ctypes.POINTER(AttnDesc)] + [vp] * 9,
        "echo_attn_bwd_recompute": [ctypes.POINTER(AttnDesc)] + [vp] * 16,
        "echo_attn_dv_reduce": [i32, i32, vp, vp, i32, vp],
        "echo_attn_bwd_deferred": [ctypes.POINTER(AttnDesc)] + [vp] * 14,
        "echo_attn_bwd_finish": [ctypes.POINTER(AttnDesc), i32] + [vp] * 11,
        "echo_attn_bwd_accumulate": [ctypes.POINTER(AttnDesc)] + [vp] * 11,
        "echo_dot_softmax_fwd": [ctypes.POINTER(DotDesc)] + [vp] * 5,
        "echo_dot_softmax_bwd": [ctypes.POINTER(DotDesc)] + [vp] * 7,
        "echo_xent_fwd_bwd": [i32, i32, vp, vp, vp, vp, vp, vp],
        "echo_gemm_f32": [i32, i32, i32, ctypes.c_float, vp, ctypes.c_int64, i32, vp, ctypes.c_int64, i32,
                          ctypes.c_float, vp, ctypes.c_int64, vp],
        "echo_lstm_seq_fwd": [ctypes.POINTER(LstmDesc), i32, i32, i32, i32] + [vp] * 7 + [i32, vp, vp, vp],
        "echo_colsum": [i32, i32, ctypes.c_int64, i32, vp, vp, i32, vp],
        "echo_tanh_bwd": [ctypes.c_int64, i32, vp, vp, vp, vp],
        "echo_dropout_fwd": [ctypes.c_int64, i32, ctypes.c_float, u64, u64, vp, vp, vp, i32, vp],
        "echo_dropout_apply": [ctypes.c_int64, ctypes.c_float, u64, u64, vp, i32, i32, vp, i32, vp, i32, vp],
        "echo_lstm_fwd_parts": [ctypes.POINTER(LstmDesc), i32, vp, ctypes.c_int64] + [vp] * 5,
        "echo_lstm_cscan_parts": [ctypes.POINTER(LstmDesc), i32, i32, vp, ctypes.c_int64, ctypes.c_int64] + [vp] * 4,
        "echo_lstm_bwd_parts": [ctypes.POINTER(LstmDesc), i32, vp, ctypes.c_int64] + [vp] * 7,
        "echo_footprint_estimate": [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_size_t)],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    _lib = lib
    return lib


def _p(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def _check(status):
    if status != ECHO_OK:
        raise EchoError(status, load().echo_last_error().decode())


def echo_abi_version() -> int:
    return load().echo_abi_version()


def echo_last_error() -> str:
    return load().echo_last_error().decode()


# ---------------------------------------------------------------- LSTM
def echo_lstm_fwd(d, gx_t, gh_t, bias, c_prev, gates_t, c_out, tc_t, h_out, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_lstm_fwd(ctypes.byref(d), _p(gx_t), _p(gh_t), _p(bias), _p(c_prev), _p(gates_t), _p(c_out),
                                _p(tc_t), _p(h_out), _stream(stream)))


def echo_lstm_fwd_tc(d, gx_t, h_prev, Wh, bias, c_prev, gates_t, c_out, tc_t, h_out, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_lstm_fwd_tc(ctypes.byref(d), _p(gx_t), _p(h_prev), _p(Wh), _p(bias), _p(c_prev), _p(gates_t),
                                   _p(c_out), _p(tc_t), _p(h_out), _stream(stream)))


def echo_lstm_fwd_tc_supported(B, H, dtype) -> bool:
    return bool(load().echo_lstm_fwd_tc_supported(int(B), int(H), int(dtype)))


def echo_lstm_cscan(d, T, gates, c0, c_ws, h_ws=None, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_lstm_cscan(ctypes.byref(d), int(T), _p(gates), _p(c0), _p(c_ws), _p(h_ws), _stream(stream)))


def echo_lstm_bwd_recompute(d, T, t, flags, gates, c0, c_st, tc_st, dh_t, dc, dA_t, h_regen_t, ws, ws_bytes=None,
                            stream=None):
    """ws_bytes: None, or an int capacity of ws (checked by the library)."""
    LAUNCHES["count"] += 1 + (1 if flags & ECHO_BWD_REGEN_C else 0)
    n = None if ws_bytes is None else ctypes.byref(ctypes.c_size_t(int(ws_bytes)))
    _check(load().echo_lstm_bwd_recompute(ctypes.byref(d), int(T), int(t), int(flags), _p(gates), _p(c0), _p(c_st),
                                          _p(tc_st), _p(dh_t), _p(dc), _p(dA_t), _p(h_regen_t), _p(ws), n,
                                          _stream(stream)))


def echo_lstm_bwd_ws_bytes(d, T) -> int:
    """Two-call convention: the workspace echo_lstm_bwd_recompute needs (bytes; nothing launched)."""
    n = ctypes.c_size_t(0)
    _check(load().echo_lstm_bwd_recompute(ctypes.byref(d), int(T), 0, 0, None, None, None, None, None, None, None,
                                          None, None, ctypes.byref(n), None))
    return n.value


# ---------------------------------------------------------------- MLP attention
def echo_attn_fwd(d, qp, Kp, v, Hs, src_len, ctx, E_st, alpha_st, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_attn_fwd(ctypes.byref(d), _p(qp), _p(Kp), _p(v), _p(Hs), _p(src_len), _p(ctx), _p(E_st),
                                _p(alpha_st), _stream(stream)))


def echo_attn_bwd_recompute(d, qp, Kp, v, Hs, src_len, E_st, alpha_st, dctx, dqp, dKp, dHs, dv, ctx_regen, ws,
                            ws_bytes=None, stream=None):
    """ws: [B,A] fp32 dv partials accumulated across one backward pass (zeroed by the caller first);
    dv: None, or [A] fp32 written from ws after this step."""
    LAUNCHES["count"] += 1 + (1 if dv is not None else 0)
    n = None if ws_bytes is None else ctypes.byref(ctypes.c_size_t(int(ws_bytes)))
    _check(load().echo_attn_bwd_recompute(ctypes.byref(d), _p(qp), _p(Kp), _p(v), _p(Hs), _p(src_len), _p(E_st),
                                          _p(alpha_st), _p(dctx), _p(dqp), _p(dKp), _p(dHs), _p(dv), _p(ctx_regen),
                                          _p(ws), n, _stream(stream)))


def echo_attn_bwd_ws_bytes(d) -> int:
    """Two-call convention: the dv-partials workspace echo_attn_bwd_recompute needs (nothing launched)."""
    n = ctypes.c_size_t(0)
    _check(load().echo_attn_bwd_recompute(ctypes.byref(d), *([None] * 14), ctypes.byref(n), None))
    return n.value


def echo_attn_dv_reduce(B, A, dv_part, dv, accumulate, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_attn_dv_reduce(int(B), int(A), _p(dv_part), _p(dv), int(accumulate), _stream(stream)))


# ---------------------------------------------------------------- dot softmax + dropout
def echo_dot_softmax_fwd(d, S, Pd, P_st, mask, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_dot_softmax_fwd(ctypes.byref(d), _p(S), _p(Pd), _p(P_st), _p(mask), _stream(stream)))


_GEMM_OK = {}


def echo_gemm_f32_supported(M, N, K, tA, tB, lda, ldb, ldc):
    key = (M, N, K, tA, tB, lda, ldb, ldc)
    if key not in _GEMM_OK:
        lib = load()
        lib.echo_gemm_f32_supported.restype = ctypes.c_int32
        lib.echo_gemm_f32_supported.argtypes = [ctypes.c_int32] * 5 + [ctypes.c_int64] * 3
        _GEMM_OK[key] = bool(lib.echo_gemm_f32_supported(M, N, K, tA, tB, lda, ldb, ldc))
    return _GEMM_OK[key]


def echo_gemm_f32(M, N, K, alpha, A, lda, tA, B, ldb, tB, beta, C, ldc, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_gemm_f32(M, N, K, alpha, _p(A), lda, tA, _p(B), ldb, tB, beta, _p(C), ldc, _stream(stream)))


def echo_lstm_seq_supported(B, H, dtype):
    lib = load()
    lib.echo_lstm_seq_supported.restype = ctypes.c_int32
    lib.echo_lstm_seq_supported.argtypes = [ctypes.c_int32] * 3
    return bool(lib.echo_lstm_seq_supported(B, H, dtype))


def echo_lstm_seq_fwd(d, T, k0, k1, reverse, gx, Wh, bias, h0, c0, gates, c, c_ring, tc, h, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_lstm_seq_fwd(ctypes.byref(d), T, k0, k1, int(reverse), _p(gx), _p(Wh), _p(bias), _p(h0), _p(c0),
                                    _p(gates), _p(c), int(c_ring), _p(tc), _p(h), _stream(stream)))


def echo_attn_bwd_deferred(d, qp, Kp, v, Hs, src_len, E_st, alpha_st, dctx, dqp, dv_part, ctx_regen, ds_out,
                           alpha_out, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_attn_bwd_deferred(ctypes.byref(d), _p(qp), _p(Kp), _p(v), _p(Hs), _p(src_len), _p(E_st),
                                         _p(alpha_st), _p(dctx), _p(dqp), _p(dv_part), _p(ctx_regen), _p(ds_out),
                                         _p(alpha_out), _stream(stream)))


def echo_attn_bwd_finish(d, Td, qp_all, Kp, E_st_all, v, src_len, ds_all, alpha_all, dctx_all, dKp, dHs, stream=None):
    LAUNCHES["count"] += 2
    _check(load().echo_attn_bwd_finish(ctypes.byref(d), Td, _p(qp_all), _p(Kp), _p(E_st_all), _p(v), _p(src_len),
                                       _p(ds_all), _p(alpha_all), _p(dctx_all), _p(dKp), _p(dHs), _stream(stream)))


def echo_attn_bwd_accumulate(d, qp_t, Kp, E_st_t, v, src_len, ds_t, alpha_t, dctx_t, dKp, dHs, stream=None):
    LAUNCHES["count"] += 2
    _check(load().echo_attn_bwd_accumulate(ctypes.byref(d), _p(qp_t), _p(Kp), _p(E_st_t), _p(v), _p(src_len),
                                           _p(ds_t), _p(alpha_t), _p(dctx_t), _p(dKp), _p(dHs), _stream(stream)))


def echo_xent_fwd_bwd(N, V, logits, bias, labels, row_loss, dlogits_bf16=None, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_xent_fwd_bwd(N, V, _p(logits), _p(bias), _p(labels), _p(row_loss), _p(dlogits_bf16),
                                    _stream(stream)))


def echo_lstm_fwd_parts(d, n_parts, parts_t, part_stride, bias, c_prev, c_out, h_out, stream=None):
    """Mirror plan a1: parts_t = pointer (tensor) to part 0 of the step; part q at + q*part_stride."""
    LAUNCHES["count"] += 1
    _check(load().echo_lstm_fwd_parts(ctypes.byref(d), int(n_parts), _p(parts_t), int(part_stride), _p(bias),
                                      _p(c_prev), _p(c_out), _p(h_out), _stream(stream)))


def echo_lstm_cscan_parts(d, T, n_parts, parts, part_stride, step_stride, bias, c0, c_ws, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_lstm_cscan_parts(ctypes.byref(d), int(T), int(n_parts), _p(parts), int(part_stride),
                                        int(step_stride), _p(bias), _p(c0), _p(c_ws), _stream(stream)))


def echo_lstm_bwd_parts(d, n_parts, parts_t, part_stride, bias, c_prev, c_t, dh_t, dc, dA_t, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_lstm_bwd_parts(ctypes.byref(d), int(n_parts), _p(parts_t), int(part_stride), _p(bias),
                                      _p(c_prev), _p(c_t), _p(dh_t), _p(dc), _p(dA_t), _stream(stream)))


MASK_NONE, MASK_BITS, MASK_BYTES = 0, 1, 2


def _dt(t):
    import torch
    return FP32 if t.dtype == torch.float32 else BF16


def echo_dropout_fwd(p, seed, offset, x, y, mask=None, mask_kind=MASK_NONE, stream=None):
    """y = dropout(x) (same dtype, contiguous); the keep-mask optionally kept as bits / bytes."""
    LAUNCHES["count"] += 1
    _check(load().echo_dropout_fwd(x.numel(), _dt(x), float(p), int(seed), int(offset), _p(x), _p(y), _p(mask),
                                   int(mask_kind), _stream(stream)))


def echo_dropout_apply(p, seed, offset, mask, mask_kind, x, y, accumulate=0, stream=None):
    """y (+)= x * keep / (1-p), keep decoded from the kept mask (or regenerated for MASK_NONE)."""
    assert x.numel() == y.numel()
    LAUNCHES["count"] += 1
    _check(load().echo_dropout_apply(x.numel(), float(p), int(seed), int(offset), _p(mask), int(mask_kind), _dt(x),
                                     _p(x), _dt(y), _p(y), int(accumulate), _stream(stream)))


def echo_tanh_bwd(a, da, dpre, stream=None):
    """dpre (fp32) = da * (1 - a^2) for a = tanh(pre) in storage dtype (same shapes, contiguous)."""
    import torch
    assert a.is_contiguous() and da.is_contiguous() and dpre.is_contiguous()
    assert a.numel() == da.numel() == dpre.numel() and da.dtype == dpre.dtype == torch.float32
    LAUNCHES["count"] += 1
    dt = FP32 if a.dtype == torch.float32 else BF16
    _check(load().echo_tanh_bwd(a.numel(), dt, _p(a), _p(da), _p(dpre), _stream(stream)))


def echo_colsum(x, out, accumulate=0, stream=None):
    """out (fp32 [cols]) (+)= column sums of the 2-D fp32 / bf16 tensor x (unit column stride)."""
    import torch
    assert x.dim() == 2 and x.stride(1) == 1 and out.dtype == torch.float32
    LAUNCHES["count"] += 1
    dt = FP32 if x.dtype == torch.float32 else BF16
    _check(load().echo_colsum(x.shape[0], x.shape[1], x.stride(0), dt, _p(x), _p(out), accumulate, _stream(stream)))


def echo_dot_softmax_bwd(d, S, P_st, mask, dPd, dS, Pd_regen, stream=None):
    LAUNCHES["count"] += 1
    _check(load().echo_dot_softmax_bwd(ctypes.byref(d), _p(S), _p(P_st), _p(mask), _p(dPd), _p(dS), _p(Pd_regen),
                                       _stream(stream)))


# ---------------------------------------------------------------- footprint estimator (host)
def echo_footprint_estimate(graph_json: str, config_json: str | None = None) -> str:
    lib = load()
    g = graph_json.encode()
    c = config_json.encode() if config_json is not None else None
    # one analysis in the common case: a buffer the size of the graph text (reports are smaller);
    # the two-call convention (ECHO_ERR_CAPACITY + the needed size) covers the rest
    n = ctypes.c_size_t(max(1 << 20, len(g)))
    buf = ctypes.create_string_buffer(n.value)
    st = lib.echo_footprint_estimate(g, c, buf, ctypes.byref(n))
    if st == ECHO_ERR_CAPACITY:
        buf = ctypes.create_string_buffer(n.value)
        st = lib.echo_footprint_estimate(g, c, buf, ctypes.byref(n))
    _check(st)
    return buf.value.decode()


def _bdt(t):
    import torch
    return {torch.float32: 0, torch.bfloat16: 1, torch.uint8: 2, torch.bool: 2}[t.dtype]


def echo_sign_pack(x, bits, stream=None):
    """bits (uint8 [(n+7)/8]) <- sign bits of x (> 0; bool / uint8: != 0)."""
    LAUNCHES["count"] += 1
    _check(load().echo_sign_pack(x.numel(), _bdt(x), _p(x), _p(bits), _stream(stream)))


def echo_bits_unpack(bits, out, stream=None):
    """out (fp32 / bf16 / uint8 / bool) <- 0 / 1 from bits."""
    LAUNCHES["count"] += 1
    _check(load().echo_bits_unpack(out.numel(), _p(bits), _bdt(out), _p(out), _stream(stream)))
