"""Footprint estimator (row a8): the C++ echo_footprint_estimate vs the independent Python oracle,
pinned by the paper's worked examples and SPEC.md's acceptance numbers."""
import json
import time

import pytest

from oracle import footprint as F
from synth import graphs as Gr
from synth.configs import C1, SMALL_NMT, C2, NMTConfig


@pytest.fixture(scope="module")
def est():
    from paper_1805_08899_b200 import build, abi
    build.build()
    abi.load()

    def run(doc, cfg=None):
        return json.loads(abi.echo_footprint_estimate(json.dumps(doc), json.dumps(cfg) if cfg is not None else None))
    return run


# ------------------------------------------------------------------ paper pins (oracle and C++)
def test_fig6_fig9_add_tanh(est):
    """SPEC acceptance 1 / PAPER.md:355-356, 549-553: baseline stashes Z (N), Mirror X and Y (2N),
    Echo removes both nodes from the recomputation path (final graph has no recomputation)."""
    doc = Gr.add_tanh(1024)
    for impl in ("oracle", "c++"):
        r = {s: (F.analyze(doc, {"strategy": s}) if impl == "oracle" else est(doc, {"strategy": s})) for s in
             ("baseline", "mirror", "echo")}
        get = (lambda x: x["stash_bytes"])
        assert get(r["baseline"]) == 4096 and get(r["mirror"]) == 8192 and get(r["echo"]) == 4096
        nm = len(r["echo"]["mirrored"]) if impl == "oracle" else r["echo"]["mirrored"]
        assert nm == 0


def test_fig7_fig10_broadcast_attn(est):
    """SPEC acceptance 2 / PAPER.md:360, 633: T^2 N -> 2 T N, ratio exactly 32.0 at T=64, N=256."""
    doc = Gr.broadcast_attn(64, 256)
    b = est(doc, {"strategy": "baseline"})
    e = est(doc, {"strategy": "echo"})
    assert b["stash_bytes"] == 64 * 64 * 256 * 4 == 4194304
    assert e["stash_bytes"] == 2 * 64 * 256 * 4 == 131072
    assert b["stash_bytes"] / e["stash_bytes"] == 32.0
    assert e["mirrored"] == 128                       # every add / tanh pair stays mirrored
    assert F.analyze(doc, {"strategy": "echo"})["stash_bytes"] == 131072


def test_fig12_dead_node(est):
    """SPEC acceptance 3 / PAPER.md:666-672: the FC becomes a dead mirror, the tanh output is
    released, recompute flops exclude the FC; without dead nodes there is no reduction (Fig. 12c)."""
    doc = Gr.tanh_fc(8, 16)
    e = est(doc, {"strategy": "echo"})
    b = est(doc, {"strategy": "baseline"})
    nd = est(doc, {"strategy": "echo", "enable_dead_node": False})
    assert b["stash_bytes"] == 8 * 16 * 4
    assert e["stash_bytes"] == 16 * 4                 # only the broadcast operand q is kept
    assert e["dead_mirrors"] == 1 and len(e["dead"]) == 1
    assert e["recompute_flops"] == 8 * 16 * 2         # broadcast_add + tanh, not the FC
    assert nd["stash_bytes"] == b["stash_bytes"]


def test_fig4_chain(est):
    """four stashed outputs are replaced by one edge at the head of the chain."""
    doc = Gr.chain4(64)
    assert est(doc, {"strategy": "baseline"})["stash_bytes"] == 4 * 64 * 4
    assert est(doc, {"strategy": "echo"})["stash_bytes"] == 64 * 4


def test_lstm_layer_plan(est):
    """Table T3: per step the baseline keeps 7 BH (gates, c_{t-1}, tanh c, h), Echo keeps the 4 BH
    gates and mirrors the c-chain, tanh(c) and h (+ c0 once).  Inputs x_t and h0 are kept by both."""
    B, H = 2, 8
    BH = B * H * 4
    for T in (1, 2, 3, 5):
        doc = Gr.lstm_layer(T, B, H, H)
        base = est(doc, {"strategy": "baseline"})["stash_bytes"]
        echo = est(doc, {"strategy": "echo"})["stash_bytes"]
        inputs = T * BH + BH                           # x_t and h0
        assert base == 7 * T * BH + inputs
        assert echo == 4 * T * BH + BH + inputs        # + c0


# ------------------------------------------------------------------ C++ == oracle, byte for byte
def _compare(est, doc, strategies=("baseline", "mirror", "echo"), extra=None):
    for s in strategies:
        cfg = {"strategy": s}
        cfg.update(extra or {})
        o = F.analyze(doc, cfg)
        c = est(doc, cfg)
        assert c["stash_bytes"] == o["stash_bytes"], (s, c["stash_bytes"], o["stash_bytes"])
        assert c["mirrored"] == len(o["mirrored"]), s
        assert c["timeline"] == o["timeline"], s
        assert c["peak_bytes"] == max(o["timeline"]), s
        assert c["recompute_flops"] == o["recompute_flops"], s
        G = o["graph"]
        dec = {(n, k): d for n, k, d in c["decisions"] if d in ("stash", "bit")}
        ref = {e: ("bit" if b else "stash") for e, b in o["stash"].items()}
        assert dec == ref, s


@pytest.mark.parametrize("name", ["add_tanh", "bcast", "tanh_fc", "chain4", "lstm3", "c1", "small", "ragged"])
def test_cpp_matches_oracle_zoo(est, name):
    docs = {"add_tanh": Gr.add_tanh(256), "bcast": Gr.broadcast_attn(16, 32), "tanh_fc": Gr.tanh_fc(),
            "chain4": Gr.chain4(), "lstm3": Gr.lstm_layer(3, 2, 8, 8), "c1": Gr.nmt(C1), "small": Gr.nmt(SMALL_NMT),
            "ragged": Gr.nmt(NMTConfig("ragged", B=5, Ts=11, Td=7, E=24, H=40, A=32, V=50, enc_layers=2, dec_layers=2),
                             "bf16")}
    _compare(est, docs[name])


def test_cpp_matches_oracle_random_graphs_and_never_worse(est):
    """200 seeded random graphs (SPEC acceptance 4): C++ == oracle and Echo never worse than the
    baseline.  (SPEC's "Echo flops <= Mirror flops" is not asserted: with dead
    nodes Echo may recompute an FC's input that Mirror simply keeps, e.g. seed 173.)"""
    for seed in range(200):
        doc = Gr.random_graph(seed)
        _compare(est, doc, ("baseline", "echo"))
        b = est(doc, {"strategy": "baseline"})
        e = est(doc, {"strategy": "echo"})
        assert e["stash_bytes"] <= b["stash_bytes"], seed
        nb = est(doc, {"strategy": "echo", "enable_binarization": False})
        assert nb["stash_bytes"] >= e["stash_bytes"], seed


def test_echo_vs_exhaustive_optimum():
    """Echo is greedy: on small random graphs it is never better than the exhaustive optimum over all
    mirror subsets, and reaches it on the paper's examples."""
    for doc in (Gr.add_tanh(64), Gr.chain4(16), Gr.broadcast_attn(4, 8), Gr.tanh_fc(4, 8)):
        assert F.analyze(doc)["stash_bytes"] == F.exhaustive_min_stash(doc)
    checked = 0
    for seed in range(40):
        doc = Gr.random_graph(seed, max_nodes=12)
        opt = F.exhaustive_min_stash(doc, limit=14)
        if opt is not None:
            checked += 1
            assert F.analyze(doc)["stash_bytes"] >= opt
    assert checked >= 10


def test_planner_c2_runtime_and_ratio(est):
    """C2 (3,999 nodes): the C++ runs the whole pipeline in well under 300 ms and Echo's
    plan reaches the north_star ratio.  (The brute-force oracle takes ~76 s on C2, too slow for the CPU
    suite; its peak model is pinned by hand counts in tests/test_footprint_liveness.py and compared with
    the C++ timeline on every smaller graph in this file.)"""
    doc = Gr.nmt(C2)
    t = time.perf_counter()
    e = est(doc, {"strategy": "echo"})
    dt = time.perf_counter() - t
    b = est(doc, {"strategy": "baseline"})
    assert dt < 0.3, dt
    assert b["stash_bytes"] / e["stash_bytes"] >= 1.8          # north_star target on C2
    assert e["peak_bytes"] <= b["peak_bytes"]


def test_planner_c3_runtime(est):
    """C3, the largest workload graph (72,002 nodes: 400 steps x 5 bidirectional layers): the whole
    pipeline -- JSON parse, shape inference, Alg. 1, liveness over ~216k steps, the report -- runs
    through the C ABI in < 1 s on this host (~0.25 s measured; PAPER.md:557 quotes < 300 ms for the
    paper's graphs).  The bound is loose so that a slower CI host does not fail it."""
    from synth.configs import C3
    doc = Gr.ds2(C3)
    t = time.perf_counter()
    e = est(doc, {"strategy": "echo"})
    dt = time.perf_counter() - t
    assert dt < 1.0, dt
    assert e["nodes"] == 72002 and e["stash_bytes"] == 1722009600


def test_10k_node_chain_under_1s(est):
    """SPEC acceptance 7: 10,000-node cheap-op chain analysed in < 1 s."""
    g = Gr.GraphBuilder()
    e = g.placeholder("x", [64], "f32")
    for _ in range(10000):
        e = g.op("tanh", [e])
    g.output(g.op("sum_reduce", [e]))
    t = time.perf_counter()
    r = est(g.doc(), {"strategy": "echo"})
    assert time.perf_counter() - t < 1.0
    assert r["stash_bytes"] == 64 * 4


def test_error_codes(est):
    from paper_1805_08899_b200 import abi
    bad = {"version": 1, "placeholders": [{"id": 0, "name": "x", "shape": [4], "dtype": "f32", "trainable": False}],
           "nodes": [{"id": 1, "op": "frobnicate", "inputs": [[0, 0]], "attrs": {}}], "outputs": [[1, 0]]}
    with pytest.raises(abi.EchoError) as ex:
        abi.echo_footprint_estimate(json.dumps(bad))
    assert ex.value.status == abi.ECHO_ERR_INVALID and "frobnicate" in str(ex.value)
    fwd = {"version": 1, "placeholders": [{"id": 0, "name": "x", "shape": [4], "dtype": "f32", "trainable": False}],
           "nodes": [{"id": 1, "op": "tanh", "inputs": [[2, 0]], "attrs": {}}, {"id": 2, "op": "tanh", "inputs": [[1, 0]]}],
           "outputs": [[2, 0]]}
    with pytest.raises(abi.EchoError) as ex:
        abi.echo_footprint_estimate(json.dumps(fwd))
    assert ex.value.status == abi.ECHO_ERR_INVALID
    with pytest.raises(abi.EchoError):
        abi.echo_footprint_estimate("{not json")
    import ctypes
    lib = abi.load()
    n = ctypes.c_size_t(4)
    buf = ctypes.create_string_buffer(4)
    st = lib.echo_footprint_estimate(json.dumps(Gr.add_tanh(8)).encode(), None, buf, ctypes.byref(n))
    assert st == abi.ECHO_ERR_CAPACITY and n.value > 4
    # the strategy config is validated strictly: unknown keys and wrongly typed values are errors
    g = json.dumps(Gr.add_tanh(8))
    for cfg, what in (({"strategy": "echo", "enable_deadnode": False}, "unknown key"),
                      ({"strategy": "echo", "enable_dead_node": 0}, "boolean"),
                      ({"strategy": "echo", "compute_heavy_ops": "fully_connected"}, "array"),
                      ({"strategy": "echo", "compute_heavy_ops": [1]}, "array"),
                      ({"strategy": 3}, "string"), ({"strategy": "greedy"}, "bad strategy"),
                      ({"strategy": "echo", "flop_threshold": "high"}, "number")):
        with pytest.raises(abi.EchoError) as ex:
            abi.echo_footprint_estimate(g, json.dumps(cfg))
        assert ex.value.status == abi.ECHO_ERR_INVALID and what in str(ex.value), (cfg, str(ex.value))


def test_regenerated_masks_reading_r30(est):
    """regenerate_masks (R30): counter-based dropout masks are recomputed, never kept.  C++ == oracle on
    the Transformer graph and on random graphs with dropout; on the Transformer graph Echo's plan then
    keeps exactly the 1-bit masks fewer (one bit per probability element per block), and the
    baseline ignores the option."""
    from synth.configs import SMALL_TX
    doc = Gr.transformer(SMALL_TX)
    _compare(est, doc, ("baseline", "mirror", "echo"), {"regenerate_masks": True})
    e = est(doc, {"strategy": "echo"})
    r = est(doc, {"strategy": "echo", "regenerate_masks": True})
    n = SMALL_TX.B * SMALL_TX.heads * SMALL_TX.L * SMALL_TX.L
    assert e["stash_bytes"] - r["stash_bytes"] == SMALL_TX.blocks * ((n + 7) // 8)
    assert est(doc, {"strategy": "baseline", "regenerate_masks": True})["stash_bytes"] == \
        est(doc, {"strategy": "baseline"})["stash_bytes"]
    for seed in range(60):
        g = Gr.random_graph(seed)
        _compare(est, g, ("mirror", "echo"), {"regenerate_masks": True})
        assert est(g, {"strategy": "echo", "regenerate_masks": True})["stash_bytes"] <= \
            est(g, {"strategy": "echo"})["stash_bytes"], seed


def test_nmt_embedding_dropout_graph(est):
    """R31 graph: C++ == oracle for every plan with and without regenerated masks; Echo keeps the
    1-bit masks and nothing of the dropped embeddings, regenerated masks keep neither, the Baseline
    keeps the dropped embeddings and byte masks."""
    from synth.configs import SMALL_NMT_DROP as cfg
    doc = Gr.nmt(cfg)
    _compare(est, doc)
    _compare(est, doc, ("mirror", "echo"), {"regenerate_masks": True})
    n = (cfg.Ts + cfg.Td) * cfg.B * cfg.E
    plain = est(Gr.nmt(SMALL_NMT), {"strategy": "echo"})["stash_bytes"]
    assert est(doc, {"strategy": "echo"})["stash_bytes"] - plain == n // 8
    assert est(doc, {"strategy": "echo", "regenerate_masks": True})["stash_bytes"] == plain
    b0 = est(Gr.nmt(SMALL_NMT), {"strategy": "baseline"})["stash_bytes"]
    b1 = est(doc, {"strategy": "baseline"})["stash_bytes"]
    assert b1 - b0 == n                      # + byte masks; the dropped embeddings replace the embeddings


def test_nmt_hidden_dropout_graph_reading_r33(est):
    """R33 graph (dropout on the inter-layer LSTM inputs and where a_t enters the output layer):
    C++ == oracle for every plan, with and without regenerated masks.  Echo keeps exactly one bit per
    dropped element more than without the sites (the dropped tensors are mirrored), regenerated masks
    nothing more; the Baseline keeps each site's dropout output and byte mask, and the last-step h of
    each dropped layer is no longer a feature map (the layer above reads the dropout's output)."""
    from dataclasses import replace
    cfg = replace(SMALL_NMT, dropout_hidden=0.3)
    doc = Gr.nmt(cfg)
    _compare(est, doc)
    _compare(est, doc, ("mirror", "echo"), {"regenerate_masks": True})
    B, Ts, Td, H = cfg.B, cfg.Ts, cfg.Td, cfg.H
    sites = [Ts * B * H] * (cfg.enc_layers - 1) + [Td * B * H] * (cfg.dec_layers - 1) + [Td * B * H]
    plain = {s: est(Gr.nmt(SMALL_NMT), {"strategy": s})["stash_bytes"] for s in ("baseline", "echo")}
    assert est(doc, {"strategy": "echo"})["stash_bytes"] - plain["echo"] == sum(n // 8 for n in sites)
    assert est(doc, {"strategy": "echo", "regenerate_masks": True})["stash_bytes"] == plain["echo"]
    dropped_layers = (cfg.enc_layers - 1) + (cfg.dec_layers - 1)
    assert est(doc, {"strategy": "baseline"})["stash_bytes"] - plain["baseline"] == \
        sum(n * (4 + 1) for n in sites) - dropped_layers * B * H * 4


def _group_removal_graph():
    """Nine ops over [8, 8] f32 tensors (256 B each); x0, x1 inputs, W a weight.
    3 = x0 + x1, 4 = x1 + n3, 5 = tanh(n4), 6 = FC(n3, W), 7 = n4 * n6, 8 = sigmoid(n5),
    9 = x1 * n4, 10 = sigmoid(n8), 11 = sum(n10) -> loss (7 and 9 feed nothing but are in the graph,
    so their gradients read their inputs)."""
    g = Gr.GraphBuilder()
    x0, x1 = g.placeholder("x0", [8, 8]), g.placeholder("x1", [8, 8])
    W = g.placeholder("W", [8, 8], trainable=True)
    n3 = g.op("add", [x0, x1])
    n4 = g.op("add", [x1, n3])
    n5 = g.op("tanh", [n4])
    n6 = g.op("fully_connected", [n3, W])
    g.op("mul", [n4, n6])
    n8 = g.op("sigmoid", [n5])
    g.op("mul", [x1, n4])
    n10 = g.op("sigmoid", [n8])
    g.output(g.op("sum_reduce", [n10]))
    return g.doc()


def test_trimming_removes_sharers_as_a_group(est):
    """Alg. 1 forward trimming walked by hand (removing one operator that shares a
    stashed input 'will cause all the other operators to be removed as well'; remove
    when the released bytes are >= the allocated ones).  Subgraph {3, 4, 5, 8, 10, 11}, all mirrored
    at first: stash = {x0, x1 (recompute 3, 4; grad of 9), n3 (FC grad), n6 (grad of 7)} = 1024 B.
      s = 3: co-removal group = {3, 4} (they share the stashed x1); without them the stash is
             {x1, n3, n4 (needed to recompute 5; grads of 7, 9), n6}: Rel = x0 = 256 >= Alloc = n4 = 256
             -> BOTH removed.
      s = 5: group {5}; Alloc = n5 (its own gradient, sigmoid 8's recompute) 256 > Rel 0 -> kept.
      s = 8, 10: likewise kept.   s = 11: nothing enters or leaves (0 >= 0) -> removed.
    Final: mirrored {5, 8, 10}; stash {x1, n3, n4, n6} = 1024 B.  Removing only s = 3 and then
    re-deciding 4 alone would keep 4 mirrored (768 B): the paper's group rule is what is pinned."""
    doc = _group_removal_graph()
    cfg = {"enable_dead_node": False}
    r = F.analyze(doc, cfg)
    assert sorted(r["mirrored"]) == [5, 8, 10]
    assert r["stash"] == {(1, 0): False, (3, 0): False, (4, 0): False, (6, 0): False}
    assert r["stash_bytes"] == 1024
    c = est(doc, cfg)
    assert c["stash_bytes"] == 1024 and c["mirrored"] == 3


def test_unmirrored_relu_keeps_sign_bits(est):
    """Alg. 1 line 18 / PAPER.md:726-727 (reading R26): a ReLU whose gradient reads its output and
    that is not on a recomputation path keeps that output as a 1-bit sign mask.  Graph over [8, 8]
    f32 (256 B): r = relu(x1) (outside every subgraph: nothing downstream reaches the loss, but its
    gradient node exists), s = sigmoid(x1), y = FC(s, W), L = sum(y).  Subgraph {FC, s}: trimming s
    releases x1 (256 B) and allocates s (256 B): 256 >= 256, so s is kept (FC's gradient reads it).
    Echo keeps s (256 B) + r's sign bits (64 elements -> 8 B) = 264 B; with binarization disabled
    r is kept at full width: 512 B."""
    g = Gr.GraphBuilder()
    g.placeholder("x0", [8, 8])
    x1 = g.placeholder("x1", [8, 8])
    W = g.placeholder("W", [8, 8], trainable=True)
    g.op("relu", [x1])
    s = g.op("sigmoid", [x1])
    g.output(g.op("sum_reduce", [g.op("fully_connected", [s, W])]))
    doc = g.doc()
    r = F.analyze(doc, {"strategy": "echo"})
    assert r["mirrored"] == set() and r["stash"] == {(3, 0): True, (4, 0): False} and r["stash_bytes"] == 264
    r = F.analyze(doc, {"strategy": "echo", "enable_binarization": False})
    assert r["stash"] == {(3, 0): False, (4, 0): False} and r["stash_bytes"] == 512
    assert est(doc, {"strategy": "echo"})["stash_bytes"] == 264


def _self_check_docs():
    from synth.configs import SMALL_TX, SMALL_DS2, SMALL_NMT_DROP
    from dataclasses import replace
    docs = {"add_tanh": Gr.add_tanh(64), "bcast": Gr.broadcast_attn(8, 16), "tanh_fc": Gr.tanh_fc(),
            "chain4": Gr.chain4(), "lstm3": Gr.lstm_layer(3, 2, 8, 8), "c1": Gr.nmt(C1), "small": Gr.nmt(SMALL_NMT),
            "small_drop": Gr.nmt(SMALL_NMT_DROP), "small_hdrop": Gr.nmt(replace(SMALL_NMT, dropout_hidden=0.2)),
            "ds2": Gr.ds2(SMALL_DS2), "tx": Gr.transformer(SMALL_TX), "c2": Gr.nmt(C2)}
    for seed in range(40):
        docs[f"rand{seed}"] = Gr.random_graph(seed)
    return docs


def test_plan_self_check_passes_on_every_plan(est):
    """self_verify (SPEC.md:632-639 'verify', as a structural check): every edge a gradient reads is kept
    or regenerable from kept edges, for every strategy / option on the workload graphs and 40 random
    graphs; the self-check changes nothing in the report."""
    cfgs = [{"strategy": "baseline"}, {"strategy": "mirror"}, {"strategy": "echo"},
            {"strategy": "echo", "enable_dead_node": False}, {"strategy": "echo", "enable_binarization": False},
            {"strategy": "echo", "regenerate_masks": True}, {"strategy": "mirror", "regenerate_masks": True}]
    for name, doc in _self_check_docs().items():
        for cfg in cfgs:
            r = est(doc, dict(cfg, self_verify=True))
            assert r == est(doc, cfg), (name, cfg)


def test_plan_self_check_catches_a_corrupted_plan(est):
    """Negative control (SPEC.md:639 'verify with corrupted plan -> fail, exit 4'): dropping any one
    kept, non-weight edge from Echo's plan makes the self-check fail with ECHO_ERR_MISMATCH."""
    from paper_1805_08899_b200 import abi
    docs = _self_check_docs()
    n_checked = 0
    for name in ("add_tanh", "lstm3", "c1", "small_drop", "tx", "rand3", "rand7"):
        doc = docs[name]
        r = est(doc, {"strategy": "echo"})
        for node, out, d in r["decisions"]:
            if d not in ("stash", "bit"):
                continue
            with pytest.raises(abi.EchoError) as ei:
                est(doc, {"strategy": "echo", "debug_unstash_edge": [node, out]})
            assert ei.value.status == abi.ECHO_ERR_MISMATCH, (name, node, out)
            assert "plan self-check" in str(ei.value)
            n_checked += 1
    assert n_checked >= 50


def test_gelu_silu_scale_rules(est):
    """Reading R11b (gelu / silu gradients read their input; y = c x reads nothing), by hand over [8, 8]
    f32 tensors (256 B):  L = sum(gelu(gelu(x))): the Baseline keeps both gelu inputs (x, g1: 512 B);
    Echo keeps x alone (256 B): trimming keeps g1 and g2 mirrored (Alloc 256 > Rel 0 each), removes the
    sum (0 >= 0), and dead-node elimination then drops g2 (no backward step reads its output), so g1 is
    the one regenerated node.  L = sum(tanh(2 x)): the Baseline keeps tanh's output (256 B); Echo's trimming
    removes the scale (Rel x 256 >= Alloc y 256) and then the tanh (Rel y 256 >= Alloc t 256): 256 B.
    C++ == oracle on both and on a mixed graph."""
    g = Gr.GraphBuilder()
    x = g.placeholder("x", [8, 8])
    g.output(g.op("sum_reduce", [g.op("gelu", [g.op("gelu", [x])])]))
    doc = g.doc()
    b, e = F.analyze(doc, {"strategy": "baseline"}), F.analyze(doc, {"strategy": "echo"})
    assert b["stash"] == {(0, 0): False, (1, 0): False} and b["stash_bytes"] == 512
    assert e["stash"] == {(0, 0): False} and sorted(e["mirrored"]) == [1] and e["stash_bytes"] == 256
    _compare(est, doc)
    g = Gr.GraphBuilder()
    x = g.placeholder("x", [8, 8])
    g.output(g.op("sum_reduce", [g.op("tanh", [g.op("scale", [x])])]))
    doc = g.doc()
    b, e = F.analyze(doc, {"strategy": "baseline"}), F.analyze(doc, {"strategy": "echo"})
    assert b["stash"] == {(2, 0): False} and e["stash"] == {(2, 0): False} and e["mirrored"] == set()
    _compare(est, doc)
    g = Gr.GraphBuilder()
    x = g.placeholder("x", [8, 8])
    W = g.placeholder("W", [8, 8], trainable=True)
    h = g.op("silu", [g.op("fully_connected", [x, W])])
    y = g.op("gelu", [g.op("scale", [g.op("fully_connected", [h, W])])])
    g.output(g.op("sum_reduce", [g.op("mul", [y, g.op("sigmoid", [h])])]))
    _compare(est, g.doc())


def test_layer_norm_rule(est):
    """layer_norm(x, w, b) -> (y, mean, rstd), gradient reads x and the row statistics (torch's
    native_layer_norm saves exactly those besides the weights).  By hand, x [4, 8], z = FC(LN(x)),
    L = sum(z):  Baseline keeps x, mean, rstd (LN's gradient) and y (the FC's input): f32
    128 + 16 + 16 + 128 = 288 B; bf16 (fp32 statistics) 64 + 16 + 16 + 64 = 160 B.  Echo mirrors the LN
    (trimming it would allocate y, mean, rstd and release nothing) and keeps x alone: 128 / 64 B.
    C++ == oracle for every plan."""
    for dt, base, echo in (("f32", 288, 128), ("bf16", 160, 64)):
        g = Gr.GraphBuilder()
        x = g.placeholder("x", [4, 8], dt)
        w, b = g.placeholder("w", [8], dt, trainable=True), g.placeholder("b", [8], dt, trainable=True)
        W = g.placeholder("W", [8, 8], dt, trainable=True)
        y = g.op("layer_norm", [x, w, b], nout=3, norm_ndim=1)[0]
        g.output(g.op("sum_reduce", [g.op("fully_connected", [y, W])]))
        doc = g.doc()
        rb, re_ = F.analyze(doc, {"strategy": "baseline"}), F.analyze(doc, {"strategy": "echo"})
        assert rb["stash_bytes"] == base and re_["stash_bytes"] == echo, dt
        assert re_["mirrored"] == {4} and re_["stash"] == {(0, 0): False}
        assert rb["graph"].dtype[(4, 1)] == "f32" and rb["graph"].shape[(4, 1)] == [4, 1]
        _compare(est, doc)


def test_cpp_matches_oracle_random_graphs_extended_ops(est):
    """Random graphs with the fx pass's gelu / silu / scale / layer_norm (R11b, R11c): C++ == oracle for
    every plan, the plan self-check passes, and Echo never keeps more than the Baseline."""
    for seed in range(60):
        doc = Gr.random_graph(seed, extended=True)
        _compare(est, doc)
        for st in ("baseline", "mirror", "echo"):
            est(doc, {"strategy": st, "self_verify": True})
        assert est(doc, {"strategy": "echo"})["stash_bytes"] <= est(doc, {"strategy": "baseline"})["stash_bytes"], seed
