"""Mutation check of the oracle's pins (CPU only; test infrastructure).

Each mutation is a plausible mistake in one oracle function -- a dropped term, a wrong sign, a
wrong index or gate slice, a transposed / swapped operand, an off-by-one lifetime -- applied to a
scratch copy of the repository.  The oracle's `-m "not gpu"` pin tests then run against the mutated
copy; a mutation is KILLED when some test fails (the first failing test is recorded) and SURVIVES
when every test still passes.  A surviving mutation is a gap in the pins.

    python scripts/oracle_mutations.py [--only SUBSTR] [--jobs N] [--no-cross] > profiles/r02_oracle_mutations.txt
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import re
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

TESTS = {
    "lstm": ["tests/test_oracle_lstm.py", "tests/test_oracle_ds2.py"],
    "attention": ["tests/test_oracle_attention.py"],
    "dot_softmax": ["tests/test_oracle_dot_softmax.py", "tests/test_oracle_transformer.py"],
    "transformer": ["tests/test_oracle_transformer.py"],
    "ds2": ["tests/test_oracle_ds2.py"],
    "nmt": ["tests/test_oracle_nmt.py"],
    "footprint": ["tests/test_footprint.py", "tests/test_footprint_liveness.py"],
}

# (oracle module, exact source text, replacement, what the mistake is)
MUTATIONS = [
    # ---- oracle/lstm.py
    ("lstm", "f = sigmoid(A[:, 1 * H:2 * H])", "f = np.tanh(A[:, 1 * H:2 * H])", "forget gate through tanh"),
    ("lstm", "i = sigmoid(A[:, 0 * H:1 * H])", "i = sigmoid(A[:, 1 * H:2 * H])", "input gate reads the f slice"),
    ("lstm", "o = sigmoid(A[:, 3 * H:4 * H])", "o = sigmoid(A[:, 2 * H:3 * H])", "output gate reads the g slice"),
    ("lstm", "c = f * c_prev + i * g", "c = f * c_prev + o * g", "cell update uses o instead of i"),
    ("lstm", "c = f * c_prev + i * g", "c = i * c_prev + f * g", "f and i swapped in the cell update"),
    ("lstm", "h = o * tc", "h = o * c", "h = o * c (tanh dropped)"),
    ("lstm", "dc = dc_next + dh * o * (1.0 - tc * tc)", "dc = dh * o * (1.0 - tc * tc)", "cell-gradient carry dropped"),
    ("lstm", "dc = dc_next + dh * o * (1.0 - tc * tc)", "dc = dc_next + dh * o * (1.0 + tc * tc)", "tanh' sign"),
    ("lstm", "do = dh * tc", "do = dh * o", "do uses o instead of tanh(c)"),
    ("lstm", "df = dc * c_prev", "df = dc * g", "df uses g instead of c_prev"),
    ("lstm", "dc_prev = dc * f", "dc_prev = dc * i", "dc_prev through i"),
    ("lstm", "di * i * (1.0 - i)", "di * i * (1.0 + i)", "sigmoid' sign (input gate)"),
    ("lstm", "dg * (1.0 - g * g)", "dg * (1.0 - g)", "tanh' of g as 1 - g"),
    ("lstm", "dWh += dA.T @ h_prev", "dWh += dA.T @ fw[\"H\"][t]", "dW_h reads h_t (off by one step)"),
    ("lstm", "c_prev = c0 if t == 0 else fw[\"C\"][t - 1]", "c_prev = c0 if t == 0 else fw[\"C\"][t]",
     "backward c_prev off by one step"),
    ("lstm", "dh_rec = dA @ Wh", "dh_rec = 0.5 * (dA @ Wh)", "recurrent gradient scaled"),
    ("lstm", "db += dA.sum(axis=0)", "db += dA[0]", "bias gradient from row 0 only"),
    # ---- oracle/attention.py (Fig. 7)
    ("attention", "E = np.tanh(qp[:, None, :] + Kp)", "E = np.tanh(qp[:, None, :] - Kp)", "broadcast-sub instead of add"),
    ("attention", "m = scores.max(axis=1, keepdims=True)", "m = scores.max(axis=0, keepdims=True)",
     "softmax max over the batch axis"),
    ("attention", "ds = alpha * (dalpha - (alpha * dalpha).sum(axis=1, keepdims=True))", "ds = alpha * dalpha",
     "softmax backward without the mean term"),
    ("attention", "* (1.0 - E * E)", "* (1.0 + E * E)", "tanh' sign in dE"),
    ("attention", "dv = np.einsum(\"bs,bsa->a\", ds, E)", "dv = dE.sum(axis=(0, 1))", "dv from dE"),
    ("attention", "dHs = alpha[:, :, None] * dctx[:, None, :]", "dHs = ds[:, :, None] * dctx[:, None, :]",
     "dH_s through ds instead of alpha"),
    ("attention", "np.arange(Ts)[None, :] < np.asarray(src_len)[:, None]",
     "np.arange(Ts)[None, :] <= np.asarray(src_len)[:, None]", "mask keeps position len_b"),
    ("attention", "dalpha = np.einsum(\"bk,bsk->bs\", dctx, Hs)", "dalpha = np.einsum(\"bk,bsk->bs\", dctx, Hs[:, ::-1])",
     "dalpha reads reversed positions"),
    # ---- oracle/dot_softmax.py (Philox R19)
    ("dot_softmax", "Pd = P * keep / (1.0 - p)\n    return", "Pd = P * keep * (1.0 - p)\n    return", "dropout scale inverted"),
    ("dot_softmax", "dS[r] = scale * P[r] * (dP[r] - (P[r] * dP[r]).sum())", "dS[r] = P[r] * (dP[r] - (P[r] * dP[r]).sum())",
     "scale dropped in dS"),
    ("dot_softmax", "k0 = (k0 + PHILOX_W0) & MASK32", "k0 = (k0 + PHILOX_W1) & MASK32", "Philox key schedule constant"),
    ("dot_softmax", "c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]", "c = [hi1 ^ c[1] ^ k0, lo0, hi0 ^ c[3] ^ k1, lo1]",
     "Philox round output words swapped"),
    ("dot_softmax", "return (w >> np.uint64(8)) >= np.uint64(keep_threshold(p))",
     "return (w >> np.uint64(8)) > np.uint64(keep_threshold(p))", "keep test > instead of >="),
    ("dot_softmax", "q = np.uint64(offset) + n // np.uint64(4)", "q = np.uint64(offset) + n // np.uint64(2)",
     "counter advances every 2 elements"),
    # ---- oracle/transformer.py (R27)
    ("transformer", "return X.reshape(B, L, H, d // H).transpose(0, 2, 1, 3)", "return X.reshape(B, H, L, d // H)",
     "head split mixes positions across heads"),
    ("transformer", "y = O @ P[f\"b{k}.Wo\"].T + x", "y = O @ P[f\"b{k}.Wo\"].T", "residual dropped"),
    ("transformer", "dy = dy + dQ @ P[f\"b{k}.Wq\"] + dK @ P[f\"b{k}.Wk\"] + dV @ P[f\"b{k}.Wv\"]",
     "dy = dy + dQ @ P[f\"b{k}.Wq\"] + dV @ P[f\"b{k}.Wv\"]", "input gradient misses the K path"),
    ("transformer", "dKh = dS.transpose(0, 1, 3, 2) @ Qh", "dKh = dS @ Qh", "dK without the transpose"),
    ("transformer", "scale = 1.0 / np.sqrt(dh)", "scale = 1.0 / np.sqrt(cfg.d_model)", "scale over d_model"),
    # ---- oracle/ds2.py (R21)
    ("ds2", "hb = layer_forward(X[::-1],", "hb = layer_forward(X,", "backward direction not reversed"),
    ("ds2", "dX = bf[\"dX\"] + bb[\"dX\"][::-1]", "dX = bf[\"dX\"] + bb[\"dX\"]", "reverse-direction dX not re-reversed"),
    ("ds2", "X = np.concatenate([hf, hb], axis=-1)", "X = np.concatenate([hb, hf], axis=-1)", "direction outputs swapped"),
    # ---- oracle/nmt.py (R7, R10, R31, R33)
    ("nmt", "a = np.tanh(ctx @ P[\"att.Wcc\"].T + q @ P[\"att.Wch\"].T)", "a = ctx @ P[\"att.Wcc\"].T + q @ P[\"att.Wch\"].T",
     "attention hidden without tanh"),
    ("nmt", "x = np.concatenate([P[\"emb_tgt\"][tgt_in[:, t]] * mt[t], a_prev], axis=1)",
     "x = np.concatenate([P[\"emb_tgt\"][tgt_in[:, t]] * mt[t], 0.0 * a_prev], axis=1)", "input feeding dropped"),
    ("nmt", "da = (dlogits @ P[\"out.Wo\"]) * mo[t] + da_carry", "da = (dlogits @ P[\"out.Wo\"]) * mo[t]",
     "input-feeding gradient carry dropped"),
    ("nmt", "dx = dq + ab[\"dqp\"] @ P[\"att.Wq\"]", "dx = ab[\"dqp\"] @ P[\"att.Wq\"]", "query gradient via W_ch dropped"),
    ("nmt", "dHs += dKp @ P[\"att.Wk\"]", "dHs += dKp @ P[\"att.Wk\"].T[:P[\"att.Wk\"].shape[0]]",
     "Kp backward with the transposed W_k"),
    ("nmt", "G[\"att.Wk\"] += np.einsum(\"bsa,bsh->ah\", dKp, Hs)", "G[\"att.Wk\"] += np.einsum(\"bsa,bsh->ah\", dKp, Hs[:, ::-1])",
     "dW_k pairs dKp with reversed H_s"),
    ("nmt", "loss /= N", "loss /= B", "loss normalised per sentence"),
    ("nmt", "x = s[\"h\"] * md[l][t] if l < L - 1 else s[\"h\"]", "x = s[\"h\"]", "decoder hidden dropout (R33) not applied"),
    # ---- oracle/footprint.py (Alg. 1; liveness SPEC:422-433)
    ("footprint", "if rel >= alloc:", "if rel > alloc:", "trimming tie rule (PAPER.md:549 'greater than or equal')"),
    ("footprint", '"gelu": ({0}, set(), 1)', '"gelu": (set(), {0}, 1)', "gelu gradient reads its output instead of its input"),
    ("footprint", '"scale": (set(), set(), 1)', '"scale": ({0}, set(), 1)', "scale gradient reads its input"),
    ("footprint", '"layer_norm": ({0}, {1, 2}, 3)', '"layer_norm": ({0}, {0}, 3)', "layer-norm gradient reads y, not the statistics"),
    ("footprint", 'if op == "layer_norm" and k > 0 and D[0] == "bf16":', 'if False:', "bf16 layer-norm statistics kept in bf16"),
    ("footprint", "M -= group", "M -= {s}", "trimming removes the node, not its sharer group"),
    ("footprint", "for c in G.consumers.get(e, []):\n                            if c in M and c not in group and not binz(c):",
     "for c in G.consumers.get(e, [])[:1]:\n                            if c in M and c not in group and not binz(c):",
     "co-removal group ignores all but the first consumer"),
    ("footprint", "return any(c in M for c in G.consumers.get(e, []))", "return False",
     "dead-node elimination ignores mirrored consumers"),
    ("footprint", "timeline.append(sum(b for (a, z, b) in buffers if a <= k <= z))",
     "timeline.append(sum(b for (a, z, b) in buffers if a <= k < z))", "buffer freed one step early"),
    ("footprint", "buffers.append((min(cons), pos[(\"grad\", i)], G.nbytes(e)))",
     "buffers.append((min(cons) + 1, pos[(\"grad\", i)], G.nbytes(e)))", "gradient buffer allocated one step late"),
    ("footprint", "cons.append(len(G.order))", "pass", "loss seed gradient not counted"),
    ("footprint", "if uses:\n                buffers.append((pos[(\"mirror\", m)], max(uses), G.nbytes(e)))",
     "if uses:\n                buffers.append((pos[(\"mirror\", m)], min(uses), G.nbytes(e)))",
     "recomputed buffer freed at its first use"),
    ("footprint", "for m in need_mirrors(refs):\n            steps.append((\"mirror\", m))",
     "for m in reversed(need_mirrors(refs)):\n            steps.append((\"mirror\", m))",
     "mirrors recomputed in reverse order"),
    ("footprint", "bit = st.binarize and (rnd or (p == i and p not in M and n[\"op\"] in st.binarizable))",
     "bit = st.binarize and rnd", "ReLU-style binarization never applied"),
    ("footprint", "S[e] = False                                # needed at full precision to recompute i",
     "pass", "mirrored nodes' inputs not kept"),
    ("footprint", "if st.is_heavy(G, w):\n                H.append(w)\n                continue",
     "if st.is_heavy(G, w):\n                continue", "heavy ops not re-seeded (Alg. 1 line 9)"),
]


def _copy_repo(dst):
    for d in ("oracle", "synth", "tests"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(dst, d),
                        ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    pkg = os.path.join(dst, "paper_1805_08899_b200")
    shutil.copytree(os.path.join(ROOT, "paper_1805_08899_b200"), pkg,
                    ignore=shutil.ignore_patterns("__pycache__", "_build", "csrc"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(dst, "include"))


def run_one(mut, timeout, no_cross=False):
    mod, old, new, what = mut
    with tempfile.TemporaryDirectory(prefix="omut_") as tmp:
        _copy_repo(tmp)
        path = os.path.join(tmp, "oracle", mod + ".py")
        src = open(path).read()
        n = src.count(old)
        if n != 1:
            return mut, "BAD", f"pattern occurs {n} times"
        open(path, "w").write(src.replace(old, new))
        if no_cross:                       # the C++ == oracle helper compares nothing in this mode
            tf = os.path.join(tmp, "tests", "test_footprint.py")
            t = open(tf).read()
            sig = 'def _compare(est, doc, strategies=("baseline", "mirror", "echo"), extra=None):\n'
            assert sig in t
            open(tf, "w").write(t.replace(sig, sig + "    return\n"))
        cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "not gpu", *TESTS[mod]]
        if no_cross:                       # independent pins only: drop the C++ == oracle comparisons
            cmd += ["-k", "not cpp_matches"]
        env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
        try:
            r = subprocess.run(cmd, cwd=tmp, capture_output=True, text=True, timeout=timeout, env=env)
        except subprocess.TimeoutExpired:
            return mut, "KILLED", "timeout"
        if r.returncode == 0:
            return mut, "SURVIVED", ""
        m = re.search(r"^FAILED (\S+)", r.stdout, re.M) or re.search(r"^ERROR (\S+)", r.stdout, re.M)
        return mut, "KILLED", m.group(1) if m else f"exit {r.returncode}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--jobs", type=int, default=max(1, (os.cpu_count() or 2) // 2))
    ap.add_argument("--timeout", type=int, default=600)
    ap.add_argument("--no-cross", action="store_true",
                    help="count only the independent pins (skip the C++ estimator == oracle comparisons)")
    a = ap.parse_args()
    muts = [m for m in MUTATIONS if a.only in m[0] or a.only in m[3]]
    pins = "the -m 'not gpu' oracle tests of each module" + (" minus the C++ == oracle comparisons" if a.no_cross else "")
    print(f"# oracle mutation check: {len(muts)} mutations, pins = {pins}")
    print("# status | module | mistake | first failing test")
    killed = 0
    with cf.ThreadPoolExecutor(a.jobs) as ex:
        for mut, status, why in ex.map(lambda m: run_one(m, a.timeout, a.no_cross), muts):
            killed += status == "KILLED"
            print(f"{status:8s} | {mut[0]:11s} | {mut[3]} | {why}", flush=True)
    print(f"# {killed} / {len(muts)} killed")
    return 0 if killed == len(muts) else 1


if __name__ == "__main__":
    sys.exit(main())
