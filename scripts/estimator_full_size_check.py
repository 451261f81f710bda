"""C++ estimator (echo_footprint_estimate) == the fp64-free Python oracle (oracle/footprint.py) on the
full-size workload graphs, every plan: stash bytes, mirrored count, peak, the whole liveness timeline and
the per-edge decisions.  Too slow for the CPU suite (the oracle recomputes the stash set from scratch for
every trimming decision: ~80 s per plan on C2), so it is run once and its output committed.

    python scripts/estimator_full_size_check.py > profiles/r02_estimator_full_size.txt
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import footprint as F                       # noqa: E402
from paper_1805_08899_b200 import abi                   # noqa: E402
from synth import configs as K, graphs as Gr            # noqa: E402

abi.load()
print("# C++ estimator == oracle on full-size graphs (stash bytes, mirrored, peak, timeline, decisions)")
ok_all = True
for name, doc in (("C2 fp32", Gr.nmt(K.C2, "f32")), ("C2 bf16", Gr.nmt(K.C2, "bf16")), ("C4 fp32", Gr.transformer(K.C4))):
    for st in ("baseline", "mirror", "echo"):
        t0 = time.time()
        o = F.analyze(doc, {"strategy": st})
        t_o = time.time() - t0
        t0 = time.time()
        c = json.loads(abi.echo_footprint_estimate(json.dumps(doc), json.dumps({"strategy": st})))
        t_c = time.time() - t0
        dec = {(n, k): d for n, k, d in c["decisions"] if d in ("stash", "bit")}
        ref = {e: ("bit" if b else "stash") for e, b in o["stash"].items()}
        same = (c["stash_bytes"] == o["stash_bytes"] and c["mirrored"] == len(o["mirrored"]) and
                c["timeline"] == o["timeline"] and c["peak_bytes"] == max(o["timeline"]) and dec == ref)
        ok_all &= same
        print(f"{name:8s} {st:8s} nodes {c['nodes']:6d}  stash {c['stash_bytes']:>12d}  peak {c['peak_bytes']:>12d}  "
              f"mirrored {c['mirrored']:5d}  steps {c['steps']:6d}  {'EQUAL' if same else 'DIFFERENT'}  "
              f"(oracle {t_o:.1f} s, C++ {1e3 * t_c:.0f} ms)", flush=True)
print("# all equal" if ok_all else "# MISMATCH")
sys.exit(0 if ok_all else 1)
