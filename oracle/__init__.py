"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU statement of what the Echo hot path
computes (arXiv 1805.08899, /root/reference/PAPER.md).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import anything from here.  The product package
`paper_1805_08899_b200` never imports it and shares no code with it; the only
common code is the seeded input generators in `synth/`, which hold none of the
method's arithmetic.

Echo "makes no changes to the underlying algorithms of the training models"
(PAPER.md:1053), so the numeric oracle is the plain training math with no
stash / recompute distinction.  The footprint oracle (`footprint.py`) is an
independent Python statement of Algorithm 1 plus a
brute-force live-set count.

Modules:
  lstm.py         LSTM cell / layer forward + BPTT           (Eq. 1)
  attention.py    MLP attention forward + backward
  dot_softmax.py  softmax(+dropout) forward + backward, Philox
  nmt.py          full NMT training step (loss + all grads)
  ds2.py          DeepSpeech2-shaped bi-LSTM step
  footprint.py    Algorithm 1 + EdgeUseRef + DNE + liveness

Parity status: every function is pinned by tests in tests/test_oracle_*.py;
see DESIGN.md "Oracle pins" for the list.
"""
