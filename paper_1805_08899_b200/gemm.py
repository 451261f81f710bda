"""Dense contractions around the hot path.

These are the fully-connected layers of Eq. 1 / Eq. 2 (PAPER.md:104-106,
389-391).  They are plain library GEMMs (cuBLAS through torch) and are
OUTSIDE the Echo hot path by design: Echo never recomputes them (PAPER.md:377,
396).  Storage-dtype inputs, fp32 accumulation; weight gradients are produced
in fp32 for both storage dtypes.
"""
from __future__ import annotations

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
