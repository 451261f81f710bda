"""Pins for oracle/dot_softmax.py (SURVEY.md §8(c) pins O3)."""
import os

import numpy as np
import torch

from oracle import dot_softmax as O
from synth.data import dot_softmax_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def test_philox_known_answer_vectors():
    rows = [l.split() for l in open(GOLD) if l.strip() and not l.startswith("#")]
    for r in rows:
        v = [int(x, 16) for x in r]
        out = O.philox4x32_10(np.array([v[:4]], np.uint64), np.array([v[4:6]], np.uint64))[0]
        assert [int(x) for x in out] == v[6:10]


def test_p_zero_is_torch_softmax():
    d = dot_softmax_inputs(0, 7, 33)
    S = np.asarray(d["S"], np.float64)
    keep = O.dropout_keep_mask(1, 0, S.size, 0.0).reshape(S.shape)
    assert keep.all()
    fw = O.forward(S, 0.125, keep, 0.0)
    ref = torch.softmax(torch.from_numpy(S) * 0.125, dim=1).numpy()
    assert np.abs(fw["P"] - ref).max() < 1e-15
    assert np.abs(fw["Pd"] - ref).max() < 1e-15
    assert np.abs(fw["P"].sum(axis=1) - 1).max() < 1e-15


def test_keep_rate_and_determinism():
    p = 0.1
    m1 = O.dropout_keep_mask(1234, 77, 1 << 16, p)
    m2 = O.dropout_keep_mask(1234, 77, 1 << 16, p)
    assert np.array_equal(m1, m2)
    rate = m1.mean()
    # binomial std at n=65536 is ~0.0012
    assert abs(rate - (1 - p)) < 0.006
    m3 = O.dropout_keep_mask(1235, 77, 1 << 16, p)
    assert (m1 != m3).mean() > 0.1


def test_mask_counter_layout():
    """Element n uses word n%4 of Philox(counter=offset+n//4, key=seed)."""
    seed, off = (5 << 32) | 9, 3
    keep = O.dropout_keep_mask(seed, off, 8, 0.5)
    for n in range(8):
        w = O.philox4x32_10(np.array([[off + n // 4, 0, 0, 0]], np.uint64), np.array([[9, 5]], np.uint64))[0][n % 4]
        assert keep[n] == ((int(w) >> 8) >= (1 << 23))


def test_fd_gradient():
    d = dot_softmax_inputs(2, 3, 9)
    S = np.asarray(d["S"], np.float64)
    keep = O.dropout_keep_mask(9, 0, S.size, 0.3).reshape(S.shape)
    dPd = np.asarray(d["dPd"], np.float64)
    bw = O.backward(S, 0.7, keep, 0.3, dPd)
    eps = 1e-6
    num = np.zeros_like(S)
    for idx in np.ndindex(*S.shape):
        sp, sm = S.copy(), S.copy()
        sp[idx] += eps
        sm[idx] -= eps
        num[idx] = ((O.forward(sp, 0.7, keep, 0.3)["Pd"] - O.forward(sm, 0.7, keep, 0.3)["Pd"]) * dPd).sum() / (2 * eps)
    assert np.abs(num - bw["dS"]).max() / np.abs(num).max() < 1e-6


def test_keep_boundary_from_kat_words():
    """Reading R19's keep rule at its boundary, from the first Random123 vector: seed 0, offset 0
    draws elements 0..3 from counter (0, 0, 0, 0) with key (0, 0), i.e. the KAT output words.  At
    p = (w_k >> 8) / 2^24 the threshold equals element k's 24-bit value, so element k is KEPT
    (keep iff value >= threshold); one step higher it is dropped.  A '>' keep test (or a wrong word /
    counter mapping) fails here; random inputs hit this boundary with probability 2^-24."""
    rows = [l.split() for l in open(GOLD) if l.strip() and not l.startswith("#")]
    words = [int(x, 16) for x in rows[0][6:10]]
    assert rows[0][:6] == ["00000000"] * 6
    for k, w in enumerate(words):
        u = w >> 8
        for thr, kept in ((u, True), (u + 1, False)):
            p = thr / float(1 << 24)                       # exact in fp64
            assert O.keep_threshold(p) == thr
            m = O.dropout_keep_mask(0, 0, 4, p)
            assert bool(m[k]) is kept
            assert [bool(x) for x in m] == [(x >> 8) >= thr for x in words]
