"""Dense contractions around the hot path.

These are the fully-connected layers of Eq. 1 / Eq. 2 (PAPER.md:104-106,
389-391).  They are plain library GEMMs (cuBLAS through torch) and are
OUTSIDE the Echo hot path by design: Echo never recomputes them (PAPER.md:377,
396).  Storage-dtype inputs, fp32 accumulation; weight gradients are produced
in fp32 for both storage dtypes.
"""
from __future__ import annotations

from contextlib import contextmanager

import torch


import os

# libecho's IEEE-fp32 split-K GEMM (echo_gemm_f32) replaces cuBLAS's fp32 SIMT kernels on the
# small-M per-step shapes of the recurrence (M = batch rows, M*N < 1M) when TF32 is off (strict
# fp32).  Measured on B200 inside CUDA graphs (scripts/gemm_bench.py): M=128 N=512 K=2048 17.5 vs
# 33.1 us, K=512 8.3-8.7 vs 10.8-11.0 us; the wide transposed-B shape (N=2048) stays on cuBLAS
# (14.5 vs 12.4 us), as do the large weight-gradient / projection GEMMs and every TF32 / bf16
# GEMM.  C2 fp32 step: 28.2 -> 23.0 ms.  ECHO_GEMM=torch turns it off.
_MODE = os.environ.get("ECHO_GEMM", "auto")


def _echo_ok(M, N, tB):
    if _MODE == "torch":
        return False
    if _MODE == "echo":
        return True
    return (not torch.backends.cuda.matmul.allow_tf32) and M * N < 1024 * 1024 and not (tB and N >= 2048)


def _layout(x):
    """(trans, ld) of a 2-D fp32 operand for echo_gemm_f32, or None (not a plain row/column-major view)."""
    s0, s1 = x.stride()
    if s1 == 1 and (s0 >= x.shape[1] or x.shape[0] == 1):
        return 0, max(s0, x.shape[1])
    if s0 == 1 and (s1 >= x.shape[0] or x.shape[1] == 1):
        return 1, max(s1, x.shape[0])
    return None


def gemm_into(out, a, b, beta=0.0):
    """out = a @ b + beta * out.  IEEE-fp32 operands go to libecho's split-K SIMT GEMM
    (echo_gemm_f32: deterministic, 3-10x cuBLAS's fp32 SIMT kernels at M = 128); everything else
    (bf16 operands -> cuBLAS tensor cores) stays on torch."""
    f32 = torch.float32
    if _MODE != "torch" and a.dtype == f32 and b.dtype == f32 and out.dtype == f32 and a.is_cuda and out.stride(1) == 1:
        la, lb = _layout(a), _layout(b)
        M, K = a.shape
        N = b.shape[1]
        if la and lb and out.stride(0) >= N and _echo_ok(M, N, lb[0]):
            from . import abi
            if abi.echo_gemm_f32_supported(M, N, K, la[0], lb[0], la[1], lb[1], out.stride(0)):
                abi.echo_gemm_f32(M, N, K, 1.0, a, la[1], la[0], b, lb[1], lb[0], beta, out, out.stride(0))
                return out
    if beta == 0.0:
        if out.dtype == a.dtype:
            torch.mm(a, b, out=out)
        else:
            torch.mm(a, b, out_dtype=out.dtype, out=out)
    elif out.dtype == a.dtype:
        out.addmm_(a, b, beta=beta)
    else:
        torch.addmm(out, a, b, beta=beta, out_dtype=out.dtype, out=out)
    return out


def mm(a, b, out_dtype=None):
    """a @ b; out_dtype=torch.float32 forces an fp32 result for bf16 operands."""
    od = a.dtype if out_dtype is None else out_dtype
    if _MODE != "torch" and a.dtype == b.dtype == od == torch.float32 and a.is_cuda:
        out = torch.empty(a.shape[0], b.shape[1], dtype=od, device=a.device)
        return gemm_into(out, a, b, 0.0)
    return torch.mm(a, b) if od == a.dtype else torch.mm(a, b, out_dtype=od)


def mm_out(out, a, b):
    """out = a @ b (out preallocated, e.g. a gate slot)."""
    return gemm_into(out, a, b, 0.0)


def addmm_(c, a, b):
    """c += a @ b in place (beta = 1)."""
    return gemm_into(c, a, b, 1.0)


@contextmanager
def tf32(enabled: bool):
    """Let cuBLAS run fp32-operand GEMMs on TF32 tensor cores inside the block (bf16 storage only:
    TF32's 10-bit mantissa is finer than the bf16 storage rounding these gradients already carry;
    fp32 storage keeps IEEE fp32 GEMMs).  Read at launch time, so CUDA-graph capture records it."""
    if not enabled:
        yield
        return
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        yield
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev



def colsum(x):
    """Column sums of a [rows, n] gradient (bias gradients: a sum over every token / row of the
    batch) with fp64 accumulation in libecho (echo_colsum), rounded once to fp32.  These are
    cancellation-dominated sums of 10^4-10^5 terms; an fp32 tree sum contributes ~log2(rows) eps
    sum|x| of error, which at C2 reaches the 1e-4 bound on d/db_q alone (reading R14)."""
    from . import abi
    out = torch.empty(x.shape[1], dtype=torch.float32, device=x.device)
    abi.echo_colsum(x, out)
    return out
