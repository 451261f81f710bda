"""In-step kernel timing for measurement (bench.py, scripts/): while a step is captured with
probing on, every hot-path ABI call made through `timed(name)` is bracketed by two timing events
recorded on the launch stream (external events become event-record nodes of the CUDA graph), so
each replay re-measures every launch in place.  Off (ACTIVE is None) it costs one branch."""
from __future__ import annotations

from contextlib import contextmanager

import torch

ACTIVE = None          # {name: [(e0, e1), ...]} while a probed capture is running


@contextmanager
def timed(name):
    if ACTIVE is None:
        yield
        return
    e0 = torch.cuda.Event(enable_timing=True, external=True)
    e1 = torch.cuda.Event(enable_timing=True, external=True)
    e0.record()
    yield
    e1.record()
    ACTIVE.setdefault(name, []).append((e0, e1))


def elapsed(events):
    """{name: [ms per launch]} for the recorded pairs (call after the replay completed)."""
    torch.cuda.synchronize()
    return {k: [a.elapsed_time(b) for a, b in v] for k, v in (events or {}).items()}


class GraphStep:
    """Mixin for the model drivers: capture one training step (forward + backward + grad hook +
    SGD; `self.step(lr)`) into a CUDA graph, replay it, and read probed kernel times."""
    graph = None
    probe_events = None

    def capture(self, lr=0.1, warmup=2, with_probe=False):
        """with_probe=True also records timing events around every hot-path launch; after a replay,
        kernel_times() returns their durations for that step."""
        global ACTIVE
        self.graph_seeds = self.seed_state()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.step(lr)
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        self.graph = torch.cuda.CUDAGraph()
        ACTIVE = {} if with_probe else None
        try:
            with torch.cuda.graph(self.graph):
                self.step(lr)
        finally:
            self.probe_events, ACTIVE = ACTIVE, None
        torch.cuda.synchronize(self.device)
        return self.graph

    def replay(self):
        self.graph.replay()

    def seed_state(self):
        """The host-side dropout Philox keys this driver passes to its kernels (kernel arguments, so a
        captured graph bakes them in); None if it has none."""
        return None

    def check_seeds(self, new):
        """Refuse new dropout keys once a graph is captured (replay would silently reuse the
        captured masks).  Re-capture to change them."""
        if getattr(self, "graph_seeds", None) is not None and tuple(new) != tuple(self.graph_seeds):
            raise ValueError(f"dropout seeds {tuple(new)} differ from the ones captured in the step graph "
                             f"{tuple(self.graph_seeds)}: they are kernel arguments; re-capture() to change them")

    def kernel_times(self):
        """{name: [ms per launch]} of the probed launches in the most recent replay (synchronizes)."""
        return elapsed(self.probe_events)
