"""Footprint oracle: an independent, plain Python statement of Echo's graph analysis.
TEST INFRASTRUCTURE ONLY (checks the C++ estimator behind echo_footprint_estimate).

Pipeline of Fig. 14: Gradient -> InferShape&Type -> EdgeUseRef -> Echo
(Algorithm 1) -> DeadNodeElimination -> InferShape -> planning.

Readings (R11-R13, R22-R25):
  * Gradient dependencies per op (PAPER.md:195 tanh keeps its output; PAPER.md:389-396 an FC
    keeps its inputs; the rest from the op's derivative): see GRAD_DEPS.
  * Feature maps = forward edges a gradient node reads, excluding weights.
  * Partition (Alg. 1 lines 1-10): seeds are the graph outputs' producers; expansion stops at
    placeholders, compute-heavy ops (which become new seeds) and already-claimed nodes
    (subgraphs are disjoint).
  * Forward trimming (Alg. 1 lines 12-28) in the state-dependent reading: candidates in
    topological order; the co-removal group G(s) is the closure over mirrored members sharing a
    currently-stashed input; Rel / Alloc are the bytes that leave / enter the
    stash set if G(s) is removed from the mirror path ("the storage released from
    its inputs is greater than or equal to that allocated for its outputs"); remove iff
    Rel >= Alloc.  Compute-heavy members become dead mirrors when their gradient needs no output
    (Alg. 1 lines 13-17); binarizable members (relu, dropout) stay on the mirror path
    without trimming (line 18 "insert encode and decode subroutines ...; continue"), and the
    feature map their gradient reads is kept as a 1-bit mask: dropout's keep-mask
    is random, so it is never recomputed — a mirrored dropout re-applies the stored mask; a relu that
    is not mirrored keeps its output's sign bits (reading R26).
  * DeadNodeElimination removes mirrors whose outputs nobody in the backward pass reads.
  * Memory is exact integer bytes; `stack` is a view (its inputs are written into its buffer).
This module recomputes the stash set from scratch for every decision (no incremental state) and
counts live bytes by brute force over the schedule: slow and obviously correct.
Pins of the liveness / peak model (`schedule`, `live_timeline`): hand-counted timelines of Fig. 6
and Fig. 4 under all three plans and hand-counted peaks (value and step) of a T = 2 LSTM layer under
the baseline and Echo (tests/test_footprint_liveness.py).
"""
from __future__ import annotations

import itertools
import math

HEAVY_DEFAULT = {"fully_connected", "matmul", "batched_dot", "conv2d"}
BINARIZABLE_DEFAULT = {"relu", "dropout"}
WIDTH = {"f32": 4, "bf16": 2, "f64": 8, "i32": 4, "i64": 8, "bit": 0.125, "u8": 1}
FLOAT = {"f32", "bf16", "f64"}

# op -> (needs_inputs, needs_outputs, n_outputs)
GRAD_DEPS = {
    "fully_connected": ({0, 1}, set(), 1), "matmul": ({0, 1}, set(), 1), "batched_dot": ({0, 1}, set(), 1),
    "embedding": ({0}, set(), 1), "slice": (set(), set(), 1), "add": (set(), set(), 1),
    "broadcast_add": (set(), set(), 1), "stack": (set(), set(), 1), "concat": (set(), set(), 1),
    "sum_reduce": (set(), set(), 1), "mul": ({0, 1}, set(), 1), "sigmoid": (set(), {0}, 1),
    "tanh": (set(), {0}, 1), "relu": (set(), {0}, 1), "dropout": (set(), {1}, 2),
    "dot_last": ({0, 1}, set(), 1), "masked_softmax": ({1}, {0}, 1), "weighted_sum": ({0, 1}, set(), 1),
    "softmax_ce_loss": (set(), {1}, 2), "softmax": (set(), {0}, 1), "to_heads": (set(), set(), 1),
    "from_heads": (set(), set(), 1), "conv2d": ({0, 1}, set(), 1),
    # reading R11b (the fx pass's elementwise ops): gelu'(x) and silu'(x) are functions of x, so
    # their gradients read the input; y = c * x with a constant c reads nothing (dx = c dy)
    "gelu": ({0}, set(), 1), "silu": ({0}, set(), 1), "scale": (set(), set(), 1),
    # layer_norm(x, weight, bias) -> (y, mean, rstd): its gradient reads x and the row statistics
    # (torch's native_layer_norm saves exactly those besides the weights), not y
    "layer_norm": ({0}, {1, 2}, 3),
}


class Graph:
    def __init__(self, doc):
        self.ph = {p["id"]: p for p in doc["placeholders"]}
        self.nodes = {n["id"]: n for n in doc["nodes"]}
        self.outputs = [tuple(e) for e in doc["outputs"]]
        self.order = sorted(self.nodes)                    # ids are topological
        self.shape, self.dtype = {}, {}
        for i, p in self.ph.items():
            self.shape[(i, 0)] = list(p["shape"])
            self.dtype[(i, 0)] = p["dtype"]
        for i in self.order:
            self._infer(self.nodes[i])
        self.consumers = {}
        for i in self.order:
            for k, e in enumerate(self.nodes[i]["inputs"]):
                self.consumers.setdefault(tuple(e), []).append(i)

    # -------------------------------------------------------------- InferShape & Type
    def _infer(self, n):
        op, a = n["op"], n.get("attrs", {})
        ins = [tuple(e) for e in n["inputs"]]
        S = [self.shape[e] for e in ins]
        D = [self.dtype[e] for e in ins]
        if op == "fully_connected":
            out = [S[0][:-1] + [S[1][0]]]
        elif op in ("matmul",):
            out = [[S[0][0], S[1][1]]]
        elif op == "batched_dot":
            out = [[S[0][0], S[0][1], S[1][1] if a.get("trans_b") else S[1][2]]]
        elif op == "softmax":
            out = [list(S[0])]
        elif op == "to_heads":
            Bt, Hh = a["batch"], a["heads"]
            out = [[Bt * Hh, S[0][0] // Bt, S[0][1] // Hh]]
        elif op == "from_heads":
            Hh = a["heads"]
            out = [[S[0][0] // Hh * S[0][1], Hh * S[0][2]]]
        elif op == "layer_norm":                            # stats over the last norm_ndim dims, kept per row
            k = a.get("norm_ndim", 1)
            st = list(S[0][:-k]) + [1] * k
            out = [list(S[0]), st, st]
        elif op == "conv2d":                                # x [N,C,H,W], W [O,C,kh,kw]; stride, padding
            st, pd = a.get("stride", 1), a.get("padding", 0)
            out = [[S[0][0], S[1][0], (S[0][2] + 2 * pd - S[1][2]) // st + 1, (S[0][3] + 2 * pd - S[1][3]) // st + 1]]
        elif op == "embedding":
            out = [S[0] + [S[1][1]]]
        elif op == "slice":
            shp = list(S[0])
            ax = a["axis"]
            if a.get("squeeze"):
                shp.pop(ax)
            else:
                shp[ax] = a["end"] - a["begin"]
            out = [shp]
        elif op in ("add", "mul", "sigmoid", "tanh", "relu", "gelu", "silu", "scale"):
            out = [list(S[0])]
        elif op == "dropout":
            out = [list(S[0]), list(S[0])]                  # y, keep-mask (u8)
        elif op == "broadcast_add":
            out = [list(S[1])]
        elif op == "stack":
            out = [[len(S)] + list(S[0])]
        elif op == "concat":
            shp = list(S[0])
            shp[a["axis"]] = sum(s[a["axis"]] for s in S)
            out = [shp]
        elif op == "sum_reduce":
            out = [[]]
        elif op == "dot_last":
            out = [list(S[0][:-1])]
        elif op == "masked_softmax":
            out = [list(S[0])]
        elif op == "weighted_sum":
            out = [list(S[1][1:])]
        elif op == "softmax_ce_loss":
            out = [[], list(S[0])]
        else:
            raise ValueError(f"unknown op {op}")
        dt = a.get("dtype")
        if dt is None:
            dt = D[1] if op == "embedding" else D[0]
        for k, shp in enumerate(out):
            self.shape[(n["id"], k)] = shp
            d = dt
            if op == "softmax_ce_loss":
                d = "f32"
            if op == "dropout" and k == 1:
                d = "u8"
            if op == "layer_norm" and k > 0 and D[0] == "bf16":
                d = "f32"                                   # the statistics are kept in fp32 for bf16 inputs
            self.dtype[(n["id"], k)] = d

    # -------------------------------------------------------------- helpers
    def is_ph(self, i):
        return i in self.ph

    def trainable(self, e):
        return e[0] in self.ph and self.ph[e[0]]["trainable"]

    def numel(self, e):
        return math.prod(self.shape[e]) if self.shape[e] else 1

    def nbytes(self, e, bit=False):
        if bit:
            return math.ceil(self.numel(e) / 8)
        return math.ceil(self.numel(e) * WIDTH[self.dtype[e]])

    def is_random(self, e):
        """dropout's keep-mask: random state, never recomputable (R26)."""
        return e[0] in self.nodes and self.nodes[e[0]]["op"] == "dropout" and e[1] == 1

    def n_out(self, i):
        return GRAD_DEPS[self.nodes[i]["op"]][2]

    def outs(self, i):
        return [(i, k) for k in range(self.n_out(i))]

    def grad_refs(self, i):
        """Forward edges read by node i's gradient (GRAD_DEPS)."""
        n = self.nodes[i]
        ni, no, _ = GRAD_DEPS[n["op"]]
        return [tuple(n["inputs"][k]) for k in sorted(ni)] + [(i, k) for k in sorted(no)]

    def flops(self, i):
        n = self.nodes[i]
        op = n["op"]
        ins = [tuple(e) for e in n["inputs"]]
        o = (i, 0)
        if op == "fully_connected":
            return 2 * self.numel(o) * self.shape[ins[0]][-1]
        if op == "conv2d":
            w = self.shape[ins[1]]
            return 2 * self.numel(o) * w[1] * w[2] * w[3]
        if op == "matmul":
            return 2 * self.shape[ins[0]][0] * self.shape[ins[0]][1] * self.shape[ins[1]][1]
        if op == "batched_dot":
            s = self.shape[ins[0]]
            return 2 * s[0] * s[1] * s[2] * self.numel(o) // (s[0] * s[1])
        if op in ("dot_last", "weighted_sum"):
            return 2 * self.numel(ins[1] if op == "weighted_sum" else ins[0])
        if op == "dropout":
            return 2 * self.numel(o)
        if op == "layer_norm":
            return 5 * self.numel(o)
        if op == "sum_reduce":
            return self.numel(ins[0])
        return self.numel(o)


class Strategy:
    def __init__(self, cfg=None):
        cfg = cfg or {}
        self.kind = cfg.get("strategy", "echo")
        self.heavy = set(cfg.get("compute_heavy_ops", HEAVY_DEFAULT))
        self.binarizable = set(cfg.get("binarizable_ops", BINARIZABLE_DEFAULT))
        self.dead = bool(cfg.get("enable_dead_node", True))
        self.binarize = bool(cfg.get("enable_binarization", True))
        self.flop_threshold = cfg.get("flop_threshold")
        self.regen = bool(cfg.get("regenerate_masks", False)) and self.kind != "baseline"
        if self.kind != "echo":
            self.dead = False
            self.binarize = False if self.kind == "baseline" else self.binarize

    def is_heavy(self, G, i):
        op = G.nodes[i]["op"]
        if op not in self.heavy:
            return False
        if self.flop_threshold is not None:
            return G.flops(i) / max(1, G.numel((i, 0))) > self.flop_threshold
        return True


def stash_set(G, M, st):
    """Edges kept across the forward -> backward boundary when the nodes M are mirrored.
    Returns {edge: is_bit} (is_bit: kept as a 1-bit mask)."""
    S = {}
    for i in G.order:
        n = G.nodes[i]
        heavy_orig = st.is_heavy(G, i) and not st.dead      # heavy grad reads the ORIGINAL inputs
        for e in G.grad_refs(i):
            if G.trainable(e):
                continue
            p = e[0]
            rnd = G.is_random(e)
            if p in M and not heavy_orig and not rnd:
                continue                                    # gradient reads the recomputed copy
            bit = st.binarize and (rnd or (p == i and p not in M and n["op"] in st.binarizable))
            S[e] = S.get(e, True) and bit
        if i in M:
            for e in n["inputs"]:
                e = tuple(e)
                if e[0] in M or G.trainable(e):
                    continue
                S[e] = False                                # needed at full precision to recompute i
            for e in G.outs(i):
                if G.is_random(e):                          # a mirrored dropout re-applies its stored mask
                    S[e] = S.get(e, True) and st.binarize
    if st.regen:                                            # R30: masks regenerated from (seed, counter)
        S = {e: b for e, b in S.items() if not G.is_random(e)}
    return S


def stash_bytes(G, S):
    """Exact bytes of a stash set; a stash of a stack output covers its (view) inputs."""
    stacked = {}
    for i in G.order:
        if G.nodes[i]["op"] == "stack":
            for e in G.nodes[i]["inputs"]:
                stacked[tuple(e)] = (i, 0)
    total = 0
    for e, bit in S.items():
        if e in stacked and stacked[e] in S:
            continue
        total += G.nbytes(e, bit)
    return total


def partition(G, st):
    """Algorithm 1 lines 1-10: disjoint subgraphs, expanded backward from seeds."""
    H = []
    for e in G.outputs:
        if e[0] not in H:
            H.append(e[0])
    claimed = set()
    subgraphs = []
    while H:
        h = H.pop()
        if G.is_ph(h) or h in claimed:
            continue
        S = [h]
        claimed.add(h)
        W = [e[0] for e in G.nodes[h]["inputs"]]
        while W:
            w = W.pop()
            if G.is_ph(w) or w in claimed:
                continue
            if st.is_heavy(G, w):
                H.append(w)
                continue
            S.append(w)
            claimed.add(w)
            W.extend(e[0] for e in G.nodes[w]["inputs"])
        subgraphs.append(sorted(S))
    return subgraphs


def run_echo(G, st):
    """Returns (mirrored set, subgraphs, dead mirrors).

    The recomputation paths of ALL subgraphs are created before trimming (reading R12b): use
    references are graph-wide (EdgeUseRef), so a frontier edge shared by several
    subgraphs (Kp, the encoder states reused at every decoder step) couples the
    operators of all of them, as in Fig. 10."""
    subs = partition(G, st)
    M = set()
    for S in subs:                                          # create every recomputation path
        M |= {s for s in S if not st.is_heavy(G, s)}
    binz = lambda i: G.nodes[i]["op"] in st.binarizable
    for S in subs:                                          # forward trimming, subgraph by subgraph
        for s in S:                                         # ... in topological order
            if s not in M or binz(s):                       # Alg. 1 line 18: binarizable -> continue
                continue
            group = {s}
            cur = stash_set(G, M, st)
            changed = True
            while changed:
                changed = False
                for gnode in list(group):
                    for e in G.nodes[gnode]["inputs"]:
                        e = tuple(e)
                        if e not in cur:
                            continue
                        for c in G.consumers.get(e, []):
                            if c in M and c not in group and not binz(c):
                                group.add(c)
                                changed = True
            after = stash_set(G, M - group, st)
            rel = alloc = 0                                 # bytes leaving / entering the stash set
            for e in set(cur) | set(after):
                b_cur = G.nbytes(e, cur[e]) if e in cur else 0
                b_aft = G.nbytes(e, after[e]) if e in after else 0
                if b_cur > b_aft:
                    rel += b_cur - b_aft
                else:
                    alloc += b_aft - b_cur
            if rel >= alloc:
                M -= group
    M = dead_node_elimination(G, M, st)
    dead = [i for S in subs for i in S
            if st.is_heavy(G, i) and st.dead and not GRAD_DEPS[G.nodes[i]["op"]][1]
            and any(tuple(e)[0] in M for e in G.nodes[i]["inputs"])]
    return M, subs, dead


def run_mirror(G, st):
    """Chen et al. 'Mirror': every cheap node is mirrored, heavy gradients keep
    their original inputs, no footprint check; useless mirrors are then eliminated."""
    M = {i for i in G.order if not st.is_heavy(G, i)}
    return dead_node_elimination(G, M, st), [], []


def needed_in_backward(G, M, st, e):
    for i in G.order:
        if e in G.grad_refs(i) and not (st.is_heavy(G, i) and not st.dead):
            return True
    return any(c in M for c in G.consumers.get(e, []))


def dead_node_elimination(G, M, st):
    """drop mirrors nobody in the backward pass reads, to a fixed point."""
    M = set(M)
    changed = True
    while changed:
        changed = False
        for m in sorted(M, reverse=True):
            if not any(needed_in_backward(G, M, st, e) for e in G.outs(m) if not G.is_random(e)):
                M.discard(m)
                changed = True
    return M


def analyze(doc, cfg=None):
    G = Graph(doc)
    st = Strategy(cfg)
    if st.kind == "baseline":
        M, subs, dead = set(), [], []
    elif st.kind == "mirror":
        M, subs, dead = run_mirror(G, st)
    else:
        M, subs, dead = run_echo(G, st)
    S = stash_set(G, M, st)
    return {"graph": G, "mirrored": M, "subgraphs": subs, "dead": dead, "stash": S,
            "stash_bytes": stash_bytes(G, S), "recompute_flops": sum(G.flops(i) for i in M),
            "timeline": live_timeline(G, M, S, st)}


def exhaustive_min_stash(doc, cfg=None, limit=16):
    """Brute force over all 2^|cheap| mirror sets (tiny graphs): the optimum stash bytes."""
    G = Graph(doc)
    st = Strategy(cfg)
    cand = [i for i in G.order if not st.is_heavy(G, i)]
    if len(cand) > limit:
        return None
    best = None
    for r in range(len(cand) + 1):
        for sub in itertools.combinations(cand, r):
            b = stash_bytes(G, stash_set(G, set(sub), st))
            best = b if best is None else min(best, b)
    return best


# ----------------------------------------------------------------------------- brute-force liveness
def schedule(G, M, st):
    """Forward nodes in topological order, then for each node in reverse order: the mirror nodes
    its gradient needs (recursively, in topological order) followed by its gradient step."""
    steps = [("fwd", i) for i in G.order]
    done = set()

    def need_mirrors(edges):
        out = []
        stack = [e[0] for e in edges if e[0] in M and not G.is_random(e)]
        seen = set()
        while stack:
            m = stack.pop()
            if m in done or m in seen:
                continue
            seen.add(m)
            out.append(m)
            stack.extend(tuple(e)[0] for e in G.nodes[m]["inputs"] if tuple(e)[0] in M)
        return sorted(out)

    for i in reversed(G.order):
        heavy_orig = st.is_heavy(G, i) and not st.dead
        refs = [] if heavy_orig else G.grad_refs(i)
        for m in need_mirrors(refs):
            steps.append(("mirror", m))
            done.add(m)
        steps.append(("grad", i))
    return steps


def live_timeline(G, M, S, st):
    """Brute force: at each step, sum the bytes of every buffer whose lifetime covers the step.
    Buffers: forward outputs, recomputed (mirror) outputs, gradients of float activations.
    Placeholders (inputs, weights) and weight gradients are not activations and are excluded."""
    steps = schedule(G, M, st)
    pos = {s: k for k, s in enumerate(steps)}
    stacked = {}
    for i in G.order:
        if G.nodes[i]["op"] == "stack":
            for e in G.nodes[i]["inputs"]:
                stacked[tuple(e)] = (i, 0)
    buffers = []                                            # (first step, last step, bytes)

    def fwd_uses(e):
        return [pos[("fwd", c)] for c in G.consumers.get(e, [])]

    def bwd_uses_original(e):
        u = []
        for i in G.order:
            heavy_orig = st.is_heavy(G, i) and not st.dead
            if e in G.grad_refs(i) and (e[0] not in M or heavy_orig or G.is_random(e)):
                u.append(pos[("grad", i)])
        for c in G.consumers.get(e, []):
            if c in M:
                u.append(pos[("mirror", c)])
        if G.is_random(e) and e[0] in M:
            u.append(pos[("mirror", e[0])])                 # the mirror re-applies the stored mask
        return u

    # forward outputs (a stack input lives inside the stack's buffer)
    spans = {}
    for i in G.order:
        for e in G.outs(i):
            last = max([pos[("fwd", i)]] + fwd_uses(e) + (bwd_uses_original(e) if e in S else []))
            spans[e] = [pos[("fwd", i)], last]
    for e, root in stacked.items():
        if e in spans:
            spans[root][0] = min(spans[root][0], spans[e][0])
            spans[root][1] = max(spans[root][1], spans[e][1])
    for e, (a, b) in spans.items():
        if e in stacked:
            continue
        buffers.append((a, b, G.nbytes(e, S.get(e, False))))
    # recomputed outputs
    for m in M:
        for e in G.outs(m):
            if G.is_random(e):
                continue
            uses = [pos[("grad", i)] for i in G.order if e in G.grad_refs(i) and not (st.is_heavy(G, i) and not st.dead)]
            uses += [pos[("mirror", c)] for c in G.consumers.get(e, []) if c in M]
            if uses:
                buffers.append((pos[("mirror", m)], max(uses), G.nbytes(e)))
    # gradients of float activations: produced by the first consumer gradient step, consumed by the
    # producer's gradient step
    for i in G.order:
        for e in G.outs(i):
            if G.dtype[e] not in FLOAT:
                continue
            cons = [pos[("grad", c)] for c in G.consumers.get(e, [])]
            if e in G.outputs:
                cons.append(len(G.order))                   # the loss seed, at the first backward step
            if not cons:
                continue
            buffers.append((min(cons), pos[("grad", i)], G.nbytes(e)))
    timeline = []
    for k in range(len(steps)):
        timeline.append(sum(b for (a, z, b) in buffers if a <= k <= z))
    return timeline
