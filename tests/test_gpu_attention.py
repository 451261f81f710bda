"""GPU parity of MLP attention (a5/a6) and dot softmax+dropout (a7) vs the fp64 oracle,
plus STASH == RECOMPUTE bit-identity."""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import dot_softmax as OD
from synth.data import mlp_attn_inputs, dot_softmax_inputs
from tests.gpu_util import dev, host, assert_close, bits_equal

pytestmark = pytest.mark.gpu


def _abi():
    from paper_1805_08899_b200 import abi
    abi.load()
    return abi


def _run_attn(abi, d, storage, mode, layout):
    B, Ts, A = d["Kp"].shape
    Hk = d["Hs"].shape[2]
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    if layout == "bsk":
        Kp, Hs = dev(d["Kp"], storage), dev(d["Hs"], storage)
        desc = abi.AttnDesc(B, Ts, A, Hk, dt, mode, Ts * A, A, Ts * Hk, Hk)
    else:  # s-major [Ts, B, *] as produced by the encoder
        Kp = dev(d["Kp"].transpose(1, 0, 2), storage)
        Hs = dev(d["Hs"].transpose(1, 0, 2), storage)
        desc = abi.AttnDesc(B, Ts, A, Hk, dt, mode, A, B * A, Hk, B * Hk)
    qp, v = dev(d["qp"], storage), dev(d["v"], storage)
    sl = torch.from_numpy(d["src_len"]).cuda()
    ctx = torch.empty(B, Hk, device="cuda", dtype=qp.dtype)
    E = torch.empty(B, Ts, A, device="cuda", dtype=qp.dtype) if mode == abi.STASH else None
    al = torch.empty(B, Ts, device="cuda") if mode == abi.STASH else None
    abi.echo_attn_fwd(desc, qp, Kp, v, Hs, sl, ctx, E, al)
    dctx = dev(d["dctx"], dtype=torch.float32)
    dqp = torch.empty(B, A, device="cuda")
    dKp = torch.zeros_like(Kp, dtype=torch.float32)
    dHs = torch.zeros_like(Hs, dtype=torch.float32)
    dvp = torch.zeros(B, A, device="cuda")
    creg = torch.empty_like(ctx) if mode == abi.RECOMPUTE else None
    assert abi.echo_attn_bwd_ws_bytes(desc) == B * A * 4          # two-call workspace query
    dv = torch.empty(A, device="cuda")
    abi.echo_attn_bwd_recompute(desc, qp, Kp, v, Hs, sl, E, al, dctx, dqp, dKp, dHs, dv, creg, dvp, B * A * 4)
    if layout != "bsk":
        dKp = dKp.transpose(0, 1)
        dHs = dHs.transpose(0, 1)
    return {"ctx": ctx, "E": E, "alpha": al, "dqp": dqp, "dKp": dKp.contiguous(), "dHs": dHs.contiguous(), "dv": dv,
            "ctx_regen": creg}


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
@pytest.mark.parametrize("B,Ts,A,Hk,layout", [(2, 4, 16, 16, "bsk"), (5, 37, 64, 48, "bsk"), (7, 29, 40, 88, "sbk"),
                                               (128, 50, 512, 512, "sbk"), (3, 700, 256, 64, "bsk"),
                                               (1, 1, 8, 8, "bsk"), (2, 256, 64, 32, "sbk"), (2, 257, 64, 32, "sbk"),
                                               (3, 13, 1024, 1024, "sbk"), (4, 9, 24, 1000, "bsk")])
@pytest.mark.parametrize("rows", ["0", "1"], ids=["a5-cluster", "a5-rows"])
def test_attention_parity_and_bit_identity(storage, B, Ts, A, Hk, layout, rows, cuda_dev, monkeypatch):
    monkeypatch.setenv("ECHO_A5_ROWS", rows)                      # both a5 kernels (same arithmetic)
    abi = _abi()
    d = mlp_attn_inputs(31, B, Ts, A, Hk, storage, lengths="random")
    ref = OA.backward(*(np.asarray(d[k], np.float64) for k in ("qp", "Kp", "v", "Hs", "dctx")), src_len=d["src_len"])
    res = {m: _run_attn(abi, d, storage, m, layout) for m in (abi.STASH, abi.RECOMPUTE)}
    for m, r in res.items():
        assert_close(host(r["ctx"]), ref["ctx"], storage, "ctx")
        for k in ("dqp", "dKp", "dHs", "dv"):
            assert_close(host(r[k]), ref[k], storage, k)
    s, r = res[abi.STASH], res[abi.RECOMPUTE]
    assert_close(host(s["alpha"]), ref["alpha"], storage, "alpha")
    assert_close(np.tanh(host(s["E"])), ref["E"], storage, "tanh(Z)")   # stash holds Z = qp + Kp (R15)
    assert bits_equal(r["ctx_regen"], r["ctx"])
    assert bits_equal(s["ctx"], r["ctx"])
    for k in ("dqp", "dKp", "dHs", "dv"):
        assert bits_equal(s[k], r[k]), k


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
@pytest.mark.parametrize("B,Ts,A,Hk", [(600, 50, 512, 512), (333, 3, 512, 512), (300, 256, 64, 32), (297, 13, 1024, 1024),
                                       (400, 9, 24, 1000), (1, 1, 8, 8)])
def test_a5_rows_equals_cluster_bitwise(storage, B, Ts, A, Hk, cuda_dev, monkeypatch):
    """The persistent row-streaming a5 (attn_fwd_rows, several rows per CTA through the stage ring) and
    the cluster a5 (attn_fwd_tma) give the same ctx / Z / alpha bits, in both modes, ragged lengths."""
    abi = _abi()
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    sd = torch.float32 if storage == "fp32" else torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(B * 3 + Ts)
    Kp = (torch.randn(Ts, B, A, device="cuda", generator=g) * 0.5).to(sd)
    Hs = torch.randn(Ts, B, Hk, device="cuda", generator=g).to(sd)
    qp = (torch.randn(B, A, device="cuda", generator=g) * 0.5).to(sd)
    v = (torch.randn(A, device="cuda", generator=g) * 0.2).to(sd)
    sl = torch.randint(1, Ts + 1, (B,), device="cuda", generator=g).to(torch.int32)
    for mode in (abi.STASH, abi.RECOMPUTE):
        st = mode == abi.STASH
        desc = abi.AttnDesc(B, Ts, A, Hk, dt, mode, A, B * A, Hk, B * Hk)
        out = {}
        for rows in ("0", "1"):
            monkeypatch.setenv("ECHO_A5_ROWS", rows)
            ctx = torch.full((B, Hk), float("nan"), device="cuda").to(sd)
            Z = torch.full((B, Ts, A), float("nan"), device="cuda").to(sd) if st else None
            al = torch.full((B, Ts), float("nan"), device="cuda") if st else None
            abi.echo_attn_fwd(desc, qp, Kp, v, Hs, sl, ctx, Z, al)
            torch.cuda.synchronize()
            out[rows] = (ctx, Z, al)
        for x, y in zip(out["0"], out["1"]):
            if x is not None:
                assert bits_equal(x, y)
        if st:
            rs = out["1"][2].sum(1)
            assert torch.allclose(rs, torch.ones_like(rs), atol=1e-5)


def test_attention_masked_rows_untouched(cuda_dev):
    abi = _abi()
    d = mlp_attn_inputs(5, 4, 9, 16, 16, lengths="random")
    d["src_len"][:] = [9, 1, 3, 5]
    r = _run_attn(abi, d, "fp32", abi.RECOMPUTE, "bsk")
    for b, n in enumerate(d["src_len"]):
        assert torch.all(r["dKp"][b, n:] == 0) and torch.all(r["dHs"][b, n:] == 0)


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
@pytest.mark.parametrize("R,L,p", [(13, 264, 0.1), (64, 256, 0.1), (5, 8, 0.0), (9, 1032, 0.3), (2048, 256, 0.1)])
def test_dot_softmax_dropout(storage, R, L, p, cuda_dev):
    abi = _abi()
    d = dot_softmax_inputs(41, R, L, storage)
    seed, off, scale = 0x1234_5678_9ABC, 1000, 1.0 / np.sqrt(64)
    keep = OD.dropout_keep_mask(seed, off, R * L, p).reshape(R, L)
    ref = OD.backward(np.asarray(d["S"], np.float64), scale, keep, p, np.asarray(d["dPd"], np.float64))
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    S, dPd = dev(d["S"], storage), dev(d["dPd"], storage)
    out = {}
    for m in (abi.STASH, abi.RECOMPUTE):
        desc = abi.DotDesc(R, L, dt, m, scale, p, seed, off)
        Pd = torch.empty_like(S)
        P = torch.empty_like(S) if m == abi.STASH else None
        mask = torch.empty(R * L if m == abi.STASH else R * L // 8, dtype=torch.uint8, device="cuda")
        abi.echo_dot_softmax_fwd(desc, S, Pd, P, mask)
        dS = torch.empty_like(S)
        Pdr = torch.empty_like(S) if m == abi.RECOMPUTE else None
        abi.echo_dot_softmax_bwd(desc, S if m == abi.RECOMPUTE else None, P, mask, dPd, dS, Pdr)
        out[m] = (Pd, mask, dS, Pdr, P)
        assert_close(host(Pd), ref["Pd"], storage, "Pd")
        assert_close(host(dS), ref["dS"], storage, "dS")
    # the keep-mask is integer work: bit-exact against the oracle's Philox
    sm = out[abi.STASH][1].cpu().numpy().reshape(R, L).astype(bool)
    assert np.array_equal(sm, keep)
    bm = np.unpackbits(out[abi.RECOMPUTE][1].cpu().numpy(), bitorder="little").reshape(R, L).astype(bool)
    assert np.array_equal(bm, keep)
    assert bits_equal(out[abi.STASH][0], out[abi.RECOMPUTE][0])
    assert bits_equal(out[abi.STASH][2], out[abi.RECOMPUTE][2])
    assert bits_equal(out[abi.RECOMPUTE][3], out[abi.RECOMPUTE][0])
    assert_close(host(out[abi.STASH][4]), ref["P"], storage, "P")
    # regenerated masks (R30): no mask kept; the backward re-derives it from (seed, offset)
    desc = abi.DotDesc(R, L, dt, abi.RECOMPUTE, scale, p, seed, off)
    Pd = torch.empty_like(S)
    abi.echo_dot_softmax_fwd(desc, S, Pd, None, None)
    dS, Pdr = torch.empty_like(S), torch.empty_like(S)
    abi.echo_dot_softmax_bwd(desc, S, None, None, dPd, dS, Pdr)
    assert bits_equal(Pd, out[abi.STASH][0]) and bits_equal(dS, out[abi.STASH][2]) and bits_equal(Pdr, Pd)


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
@pytest.mark.parametrize("B,Ts,A,Hk,Td", [(5, 37, 64, 48, 4), (128, 50, 512, 512, 3)])
def test_attention_deferred_bitwise(storage, B, Ts, A, Hk, Td, cuda_dev):
    """echo_attn_bwd_deferred + echo_attn_bwd_finish == Td per-step echo_attn_bwd calls, bitwise
    (dKp, dH_s, dqp, dv partials), both modes; the per-step path is itself pinned to the oracle."""
    abi = _abi()
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    sd = torch.float32 if storage == "fp32" else torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(B + Ts)
    rn = lambda *s, sc=1.0: (torch.randn(*s, device="cuda", generator=g) * sc).to(sd)
    Kp, Hs, v = rn(Ts, B, A, sc=0.5), rn(Ts, B, Hk), rn(A, sc=0.3)
    qps = rn(Td, B, A, sc=0.5)
    sl = torch.randint(1, Ts + 1, (B,), device="cuda", generator=g).to(torch.int32)
    dctxs = torch.randn(Td, B, Hk, device="cuda", generator=g)
    for mode in (abi.STASH, abi.RECOMPUTE):
        desc = abi.AttnDesc(B, Ts, A, Hk, dt, mode, A, B * A, Hk, B * Hk)
        st = mode == abi.STASH
        E = torch.empty(Td, B, Ts, A, device="cuda", dtype=sd) if st else None
        al = torch.empty(Td, B, Ts, device="cuda") if st else None
        ctx = torch.empty(B, Hk, device="cuda", dtype=sd)
        for t in range(Td):
            abi.echo_attn_fwd(desc, qps[t], Kp, v, Hs, sl, ctx, E[t] if st else None, al[t] if st else None)
        res = {}
        for deferred in (False, True):
            dqp = torch.empty(Td, B, A, device="cuda")
            dvp = torch.zeros(B, A, device="cuda")
            creg = None if st else torch.empty(Td, B, Hk, device="cuda", dtype=sd)
            if deferred:
                dKp = torch.full((Ts, B, A), float("nan"), device="cuda")
                dHs = torch.full((Ts, B, Hk), float("nan"), device="cuda")
                ds_all = torch.empty(Td, B, Ts, device="cuda")
                al_all = al if st else torch.empty(Td, B, Ts, device="cuda")
            else:
                dKp = torch.zeros(Ts, B, A, device="cuda")
                dHs = torch.zeros(Ts, B, Hk, device="cuda")
            for t in reversed(range(Td)):
                args = (None, None) if st else (qps[t], Kp)
                e_a = (E[t], al[t]) if st else (None, None)
                if deferred:
                    abi.echo_attn_bwd_deferred(desc, *args, v, Hs, sl, *e_a, dctxs[t], dqp[t], dvp,
                                               None if st else creg[t], ds_all[t], None if st else al_all[t])
                else:
                    abi.echo_attn_bwd_recompute(desc, *args, v, Hs, sl, *e_a, dctxs[t], dqp[t], dKp, dHs, None,
                                                None if st else creg[t], dvp)
            if deferred:
                abi.echo_attn_bwd_finish(desc, Td, None if st else qps, None if st else Kp, E if st else None, v, sl,
                                         ds_all, al_all, dctxs, dKp, dHs)
            torch.cuda.synchronize()
            res[deferred] = (dKp, dHs, dqp, dvp, creg)
        for k, (x, y) in enumerate(zip(res[False], res[True])):
            if x is not None:
                assert bits_equal(x, y), (mode, k)


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
def test_attention_c5_launch_sampled_rows(storage, cuda_dev):
    """C5's launch configuration (B = 24576 rows, Ts = 50, A = Hk = 512: the shape bench.py's C5
    leg times), both modes, on sampled rows the oracle computes one by one; every row's softmax sums
    to one; RECOMPUTE's regenerated ctx equals the forward's and its gradients equal STASH's, bitwise
    over all rows."""
    abi = _abi()
    B, Ts, A, Hk = 24576, 50, 512, 512
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    sd = torch.float32 if storage == "fp32" else torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(5)
    Kp = (torch.randn(Ts, B, A, device="cuda", generator=g) * 0.5).to(sd)
    Hs = torch.randn(Ts, B, Hk, device="cuda", generator=g).to(sd)
    qp = (torch.randn(B, A, device="cuda", generator=g) * 0.5).to(sd)
    v = (torch.randn(A, device="cuda", generator=g) * 0.2).to(sd)
    sl = torch.randint(1, Ts + 1, (B,), device="cuda", generator=g).to(torch.int32)
    dctx = torch.randn(B, Hk, device="cuda", generator=g)
    res = {}
    for mode in (abi.STASH, abi.RECOMPUTE):
        st = mode == abi.STASH
        desc = abi.AttnDesc(B, Ts, A, Hk, dt, mode, A, B * A, Hk, B * Hk)
        ctx = torch.empty(B, Hk, device="cuda", dtype=sd)
        Z = torch.empty(B, Ts, A, device="cuda", dtype=sd) if st else None
        al = torch.empty(B, Ts, device="cuda") if st else None
        abi.echo_attn_fwd(desc, qp, Kp, v, Hs, sl, ctx, Z, al)
        dqp = torch.empty(B, A, device="cuda")
        dKp = torch.zeros(Ts, B, A, device="cuda")
        dHs = torch.zeros(Ts, B, Hk, device="cuda")
        dvp = torch.zeros(B, A, device="cuda")
        dv = torch.empty(A, device="cuda")
        creg = None if st else torch.empty_like(ctx)
        abi.echo_attn_bwd_recompute(desc, None if st else qp, None if st else Kp, v, Hs, sl, Z, al, dctx, dqp, dKp,
                                    dHs, dv, creg, dvp)
        torch.cuda.synchronize()
        if st:
            rows = al.sum(1)
            assert torch.allclose(rows, torch.ones_like(rows), atol=1e-5)
            del Z, al
        else:
            assert bits_equal(creg, ctx)
        for b in (0, 1, 4097, 12345, B - 1):
            n = int(sl[b])
            f64 = lambda x: x.double().cpu().numpy()
            ref = OA.backward(f64(qp[b:b + 1]), f64(Kp[:, b:b + 1].transpose(0, 1)), f64(v),
                              f64(Hs[:, b:b + 1].transpose(0, 1)), f64(dctx[b:b + 1]), src_len=np.array([n], np.int32))
            assert_close(host(ctx[b:b + 1]), ref["ctx"], storage, f"ctx[{b}]")
            assert_close(host(dqp[b:b + 1]), ref["dqp"], storage, f"dqp[{b}]")
            assert_close(host(dKp[:, b:b + 1].transpose(0, 1)), ref["dKp"], storage, f"dKp[{b}]")
            assert_close(host(dHs[:, b:b + 1].transpose(0, 1)), ref["dHs"], storage, f"dHs[{b}]")
            assert_close(host(dvp[b]), ref["dv"], storage, f"dv[{b}]")
        res[mode] = (ctx, dqp, dKp, dHs, dvp, dv)
    for k, (x, y) in enumerate(zip(res[abi.STASH], res[abi.RECOMPUTE])):
        assert bits_equal(x, y), k


def test_attention_rejects_bad_arguments(cuda_dev):
    """Empty / misaligned / mode-inconsistent calls fail with ECHO_ERR_INVALID before any launch."""
    abi = _abi()
    x = torch.zeros(64, device="cuda")
    for desc in (abi.AttnDesc(0, 4, 16, 16, abi.FP32, abi.RECOMPUTE, 16, 0, 16, 0),
                 abi.AttnDesc(2, 4, 12, 16, abi.FP32, abi.RECOMPUTE, 12, 48, 16, 64)):
        with pytest.raises(abi.EchoError) as ei:
            abi.echo_attn_fwd(desc, x, x, x, x, None, x, None, None)
        assert ei.value.status == 1
    desc = abi.AttnDesc(2, 4, 16, 16, abi.FP32, abi.RECOMPUTE, 16, 64, 16, 64)
    with pytest.raises(abi.EchoError):                        # RECOMPUTE must not get a stash buffer
        abi.echo_attn_fwd(desc, x, x, x, x, None, x, x, x)


def test_attention_src_len_debug_check(cuda_dev, monkeypatch):
    """SURVEY §8(b) validation: src_len outside [1, Ts] is clamped by the kernels, and rejected with
    ECHO_ERR_INVALID by the entry points when ECHO_CHECK_SRC_LEN=1 (host copy of the device array)."""
    abi = _abi()
    d = mlp_attn_inputs(3, 4, 6, 16, 16)
    B, Ts, A = d["Kp"].shape
    Hk = d["Hs"].shape[2]
    desc = abi.AttnDesc(B, Ts, A, Hk, abi.FP32, abi.RECOMPUTE, Ts * A, A, Ts * Hk, Hk)
    qp, Kp, v, Hs = (dev(d[k], "fp32") for k in ("qp", "Kp", "v", "Hs"))
    ctx = torch.empty(B, Hk, device="cuda")
    good = torch.tensor([6, 1, 3, 2], dtype=torch.int32, device="cuda")
    for bad in ([6, 0, 3, 2], [6, 1, 7, 2]):
        sl = torch.tensor(bad, dtype=torch.int32, device="cuda")
        monkeypatch.delenv("ECHO_CHECK_SRC_LEN", raising=False)
        abi.echo_attn_fwd(desc, qp, Kp, v, Hs, sl, ctx, None, None)          # clamped, no error
        monkeypatch.setenv("ECHO_CHECK_SRC_LEN", "1")
        with pytest.raises(abi.EchoError) as ei:
            abi.echo_attn_fwd(desc, qp, Kp, v, Hs, sl, ctx, None, None)
        assert ei.value.status == 1 and "src_len" in str(ei.value)
    abi.echo_attn_fwd(desc, qp, Kp, v, Hs, good, ctx, None, None)          # in range: accepted
    torch.cuda.synchronize()
