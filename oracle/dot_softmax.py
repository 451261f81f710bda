"""Dot-product attention softmax (+ dropout) oracle, fp64.  TEST INFRASTRUCTURE ONLY.

Transformer attention probabilities P = softmax(S * scale) with S = Q K^T from
the caller's GEMM, followed by dropout P_d = P * m / (1 - p).  Echo recomputes
the softmax in the backward pass and stores the dropout feature map as a
1-bit mask ("encodes the dropout feature maps to 1-bit in the
forward pass and decodes them back to 32-bit in the backward pass"; Alg. 1
line 18; Transformer result PAPER.md:1002).

The keep-mask is drawn from Philox4x32-10 (Salmon et al., SC'11 "Parallel
random numbers: as easy as 1, 2, 3"), implemented here independently of the
CUDA side (reading R19): element n of the row-major [R, L] tensor uses counter
q = offset + n // 4 -> (lo32(q), hi32(q), 0, 0), key (lo32(seed), hi32(seed)),
word (n mod 4) of the output; keep iff (word >> 8) >= floor(p * 2^24).
Pins: tests/test_oracle_dot_softmax.py (Random123 known-answer vectors, FD,
p = 0 reduces to torch.softmax, keep-rate statistics).
"""
from __future__ import annotations

import numpy as np

PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint64(0x9E3779B9)
PHILOX_W1 = np.uint64(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: uint64 array [..., 4] of 32-bit words; key: [..., 2].  Returns [..., 4] uint64."""
    c = [np.asarray(ctr[..., i], np.uint64) & MASK32 for i in range(4)]
    k0 = np.asarray(key[..., 0], np.uint64) & MASK32
    k1 = np.asarray(key[..., 1], np.uint64) & MASK32
    for r in range(10):
        if r > 0:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        p0 = PHILOX_M0 * c[0]
        p1 = PHILOX_M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return np.stack(c, axis=-1)


def keep_threshold(p):
    """Integer threshold on the top 24 bits of a Philox word: keep iff (w >> 8) >= thr."""
    return int(np.floor(float(p) * (1 << 24)))


def dropout_keep_mask(seed, offset, n_elems, p):
    """Boolean keep-mask of n_elems consecutive elements (reading R19)."""
    n = np.arange(n_elems, dtype=np.uint64)
    q = np.uint64(offset) + n // np.uint64(4)
    ctr = np.stack([q & MASK32, q >> np.uint64(32), np.zeros_like(q), np.zeros_like(q)], axis=-1)
    key = np.stack([np.full_like(q, np.uint64(seed) & MASK32), np.full_like(q, np.uint64(seed) >> np.uint64(32))], axis=-1)
    words = philox4x32_10(ctr, key)
    w = words[np.arange(n_elems), (n % np.uint64(4)).astype(np.int64)]
    return (w >> np.uint64(8)) >= np.uint64(keep_threshold(p))


def forward(S, scale, keep, p):
    """P = softmax(scale * S) row-wise; P_d = P * keep / (1 - p)."""
    S = np.asarray(S, np.float64)
    R, L = S.shape
    P = np.zeros((R, L))
    for r in range(R):
        z = scale * S[r]
        w = np.exp(z - z.max())
        P[r] = w / w.sum()
    Pd = P * keep / (1.0 - p)
    return {"P": P, "Pd": Pd}


def backward(S, scale, keep, p, dPd):
    """dS for the loss <dPd, P_d>: dP = dPd*keep/(1-p); dS = scale * P * (dP - sum(P*dP))."""
    fw = forward(S, scale, keep, p)
    P = fw["P"]
    dP = np.asarray(dPd, np.float64) * keep / (1.0 - p)
    dS = np.zeros_like(P)
    for r in range(P.shape[0]):
        dS[r] = scale * P[r] * (dP[r] - (P[r] * dP[r]).sum())
    return {"dS": dS, "P": P, "Pd": fw["Pd"]}
