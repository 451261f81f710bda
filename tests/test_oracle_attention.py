"""Pins for oracle/attention.py (SURVEY.md §8(c) pins O2)."""
import numpy as np

from oracle import attention as O
from synth.data import mlp_attn_inputs


def _args(seed=0, B=3, Ts=5, A=4, Hk=6, lengths="random"):
    d = mlp_attn_inputs(seed, B, Ts, A, Hk, lengths=lengths)
    return {k: np.asarray(d[k], np.float64) if k != "src_len" else d[k] for k in d}


def test_hand_computed_scores():
    """B=1, Ts=2, A=1: qp=0, Kp=[0, atanh(1/2)], v=2 ln 3 => scores [0, ln 3] => alpha [1/4, 3/4]."""
    Hs = np.array([[[1.0, 2.0], [5.0, -3.0]]])
    fw = O.forward(np.zeros((1, 1)), np.array([[[0.0], [np.arctanh(0.5)]]]), np.array([2 * np.log(3.0)]), Hs)
    assert np.abs(fw["alpha"] - [[0.25, 0.75]]).max() < 1e-15
    assert np.abs(fw["ctx"] - (0.25 * Hs[0, 0] + 0.75 * Hs[0, 1])).max() < 1e-14


def test_rows_sum_to_one_and_mask():
    d = _args()
    fw = O.forward(d["qp"], d["Kp"], d["v"], d["Hs"], d["src_len"])
    assert np.abs(fw["alpha"].sum(axis=1) - 1.0).max() < 1e-15
    for b, n in enumerate(d["src_len"]):
        assert np.all(fw["alpha"][b, n:] == 0.0)
        assert np.all(fw["alpha"][b, :n] > 0.0)


def test_v_zero_gives_uniform_mean():
    d = _args()
    fw = O.forward(d["qp"], d["Kp"], np.zeros_like(d["v"]), d["Hs"], d["src_len"])
    for b, n in enumerate(d["src_len"]):
        assert np.abs(fw["alpha"][b, :n] - 1.0 / n).max() < 1e-15
        assert np.abs(fw["ctx"][b] - d["Hs"][b, :n].mean(axis=0)).max() < 1e-14


def test_single_source_position():
    """Ts=1 => alpha=1: dqp = dKp = dv = 0 exactly and dHs = dctx."""
    d = _args(Ts=1, lengths="full")
    bw = O.backward(d["qp"], d["Kp"], d["v"], d["Hs"], d["dctx"], d["src_len"])
    assert np.all(bw["dqp"] == 0) and np.all(bw["dKp"] == 0) and np.all(bw["dv"] == 0)
    assert np.array_equal(bw["dHs"][:, 0, :], d["dctx"])


def test_permutation_invariance():
    d = _args(lengths="full")
    perm = np.random.default_rng(1).permutation(d["Kp"].shape[1])
    a = O.forward(d["qp"], d["Kp"], d["v"], d["Hs"])["ctx"]
    b = O.forward(d["qp"], d["Kp"][:, perm], d["v"], d["Hs"][:, perm])["ctx"]
    assert np.abs(a - b).max() < 1e-14


def test_fd_gradients():
    d = _args(seed=3)
    R = d["dctx"]
    L = lambda qp, Kp, v, Hs: (O.forward(qp, Kp, v, Hs, d["src_len"])["ctx"] * R).sum()
    bw = O.backward(d["qp"], d["Kp"], d["v"], d["Hs"], R, d["src_len"])
    args = {"qp": d["qp"], "Kp": d["Kp"], "v": d["v"], "Hs": d["Hs"]}
    eps = 1e-6
    for k, gk in (("qp", "dqp"), ("Kp", "dKp"), ("v", "dv"), ("Hs", "dHs")):
        num = np.zeros_like(args[k])
        for idx in np.ndindex(*args[k].shape):
            ap = {kk: vv.copy() for kk, vv in args.items()}
            am = {kk: vv.copy() for kk, vv in args.items()}
            ap[k][idx] += eps
            am[k][idx] -= eps
            num[idx] = (L(**ap) - L(**am)) / (2 * eps)
        err = np.abs(num - bw[gk]).max() / max(np.abs(num).max(), 1e-30)
        assert err < 1e-6, (k, err)
    # masked positions receive exactly zero gradient
    for b, n in enumerate(d["src_len"]):
        assert np.all(bw["dKp"][b, n:] == 0) and np.all(bw["dHs"][b, n:] == 0)
