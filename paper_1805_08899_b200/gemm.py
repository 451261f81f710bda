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


def mm(a, b, out_dtype=None):
    """a @ b; out_dtype=torch.float32 forces an fp32 result for bf16 operands."""
    if out_dtype is None or out_dtype == a.dtype:
        return torch.mm(a, b)
    return torch.mm(a, b, out_dtype=out_dtype)


def addmm_(c, a, b):
    """c += a @ b in place (cuBLAS beta = 1)."""
    if c.dtype == a.dtype:
        c.addmm_(a, b)
    else:
        torch.addmm(c, a, b, out_dtype=c.dtype, out=c)
    return c


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
