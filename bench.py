#!/usr/bin/env python
"""Benchmark: train samples/s and peak activation HBM, RECOMPUTE (Echo) vs STASH (Baseline).

    python bench.py [--gpus N --steps K --warmup W] [--dtype fp32|bf16] [--batch B] [--impl reference]

Workload: C2 of BASELINE.json (`configs[1]`): Sockeye-style 2+2-layer LSTM NMT, hidden 512,
MLP attention, batch 128 per GPU, 50 source / 50 target steps, V = 8192, synthetic tokens,
random-init weights.  One step = forward + backward + (allreduce) + SGD of the whole model;
the Echo hot path (libecho a1/a2/a3/a5/a6) runs inside it, the FCs are cuBLAS.
Multi-GPU: one process per GPU (torchrun), batch-sharded (weak scaling), NCCL allreduce.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _metric():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["metric"]


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms from just before the timed region to its end."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [l.strip().split(", ") for l in open(self.f.name) if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- reference arm (CPU oracle)
def run_reference(args):
    """--impl reference: the fp64 CPU oracle (the only reference this paper-only tier has), timed on the
    host cores on a bounded sample of the same C2 workload (batch 16 per step instead of 128)."""
    from synth.configs import C2
    from synth.data import nmt_params, nmt_batch
    from oracle import nmt as O
    ws, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    Bs = 16
    cfg = C2.with_batch(Bs)
    params = nmt_params(0, cfg)
    batches = [nmt_batch(1 + i, cfg) for i in range(max(1, args.warmup) + args.steps)]
    for i in range(args.warmup):
        O.step(params, batches[i], cfg)
    t0 = time.perf_counter()
    for i in range(args.steps):
        O.step(params, batches[args.warmup + i], cfg)
    dt = time.perf_counter() - t0
    v = Bs * args.steps / dt
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": _metric(), "value": v, "unit": "samples/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2-nmt (fp64 CPU oracle, bounded sample: batch 16 of 128 per step)",
                       "global_batch": Bs, "seq_len": 50, "hidden": 512, "vocab": 8192, "layers": "2+2"},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "oracle",
                             "sample": f"C2 shapes, batch {Bs} per step, {args.steps} steps, numpy fp64"},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def cpu_baseline_sample():
    """The oracle as it stands, on the host cores, bounded sample (~10-20 s): C2 shapes at batch 16."""
    from synth.configs import C2
    from synth.data import nmt_params, nmt_batch
    from oracle import nmt as O
    Bs, n = 16, 2
    cfg = C2.with_batch(Bs)
    params = nmt_params(0, cfg)
    b = [nmt_batch(100 + i, cfg) for i in range(n + 1)]
    O.step(params, b[0], cfg)
    t0 = time.perf_counter()
    for i in range(n):
        O.step(params, b[1 + i], cfg)
    dt = time.perf_counter() - t0
    return {"value": Bs * n / dt, "unit": "samples/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
            "sample": f"C2 shapes (B=16 of 128, T=50, H=512, V=8192), {n} full training steps, numpy fp64"}


def ncu_traffic(dtype):
    """DRAM read + write bytes per launch of the a6 kernel from the committed `ncu --set full`
    capture of the same launch configuration (profiles/), or None."""
    import glob
    tag = "fp32" if dtype == 0 else "bf16"
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"*ncu_attn_bwd_c2_{tag}.txt")), reverse=True):
        for line in open(f):
            if line.startswith("traffic = dram read + write"):
                return {"bytes": float(line.split()[-1]), "source": os.path.relpath(f, ROOT)}
    return None


def attn_bwd_bytes(cfg, dtype):
    """Algorithmic HBM bytes of one a6 RECOMPUTE launch (per row Kp + H_s read,
    dKp + dH_s read-modify-write, plus the per-row vectors)."""
    B, Ts, A, H = cfg.B, cfg.Ts, cfg.A, cfg.H
    s_bytes = 4 if dtype == 0 else 2
    rows = B * Ts
    big = rows * (A * s_bytes + H * s_bytes + 2 * A * 4 + 2 * H * 4)      # Kp, Hs read; dKp, dHs RMW
    small = B * A * s_bytes + B * H * 4 + B * A * 4 + 2 * B * A * 4 + B * H * s_bytes + A * s_bytes + B * 4
    return big + small, rows


def time_attn_bwd(cfg, dtype, reps=20):
    """Dominant kernel (a6, RECOMPUTE attention backward) at the step's launch configuration,
    timed with CUDA events on its launch stream; L2 flushed (256 MiB read) before every launch."""
    import torch
    from paper_1805_08899_b200 import abi
    B, Ts, A, H = cfg.B, cfg.Ts, cfg.A, cfg.H
    sd = torch.float32 if dtype == abi.FP32 else torch.bfloat16
    s_bytes = 4 if dtype == abi.FP32 else 2
    g = torch.Generator(device="cuda").manual_seed(0)
    qp = (torch.randn(B, A, device="cuda", generator=g) * 0.5).to(sd)
    Kp = (torch.randn(Ts, B, A, device="cuda", generator=g) * 0.5).to(sd)
    Hs = torch.randn(Ts, B, H, device="cuda", generator=g).to(sd)
    v = (torch.randn(A, device="cuda", generator=g) * 0.1).to(sd)
    sl = torch.full((B,), Ts, dtype=torch.int32, device="cuda")
    dctx = torch.randn(B, H, device="cuda", generator=g)
    dqp = torch.empty(B, A, device="cuda")
    dKp = torch.zeros(Ts, B, A, device="cuda")
    dHs = torch.zeros(Ts, B, H, device="cuda")
    dvp = torch.zeros(B, A, device="cuda")
    creg = torch.empty(B, H, device="cuda", dtype=sd)
    desc = abi.AttnDesc(B, Ts, A, H, dtype, abi.RECOMPUTE, A, B * A, H, B * H)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(3):
        abi.echo_attn_bwd_recompute(desc, qp, Kp, v, Hs, sl, None, None, dctx, dqp, dKp, dHs, None, creg, dvp)
    times = []
    for _ in range(reps):
        flush.sum()              # read-flush: L2 ends up holding clean lines
        torch.cuda._sleep(200000)  # GPU busy while the host enqueues e0 / launch / e1: no host gap is timed
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        abi.echo_attn_bwd_recompute(desc, qp, Kp, v, Hs, sl, None, None, dctx, dqp, dKp, dHs, None, creg, dvp)
        e1.record(st)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.mean(times)
    nbytes, rows = attn_bwd_bytes(cfg, dtype)
    return {"ms": ms, "bytes": nbytes, "bytes_per_row": nbytes / rows, "rows": rows}


def c5_a6_roofline(m, cfg, dt, reps=2):
    """a6 launch duration inside the C5 step (probed re-capture: the timed graph is released first)."""
    import gc
    import torch
    m.graph = None
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    m.capture(0.01, warmup=1, with_probe=True)
    m.replay()
    lt = []
    for _ in range(reps):
        m.replay()
        lt.extend(m.kernel_times().get("attn_bwd", []))
    nbytes, rows = attn_bwd_bytes(cfg, dt)
    pk = _peaks()
    l_ms = statistics.mean(lt)
    ach = nbytes / (l_ms / 1e3) / 1e9
    return {"kernel": "echo_attn_bwd_recompute (a6, RECOMPUTE)", "launch_us": 1e3 * l_ms, "bytes_per_launch": nbytes,
            "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach / pk["hbm_gbs"],
            "timing": "CUDA events on the launch stream around each of the 50 a6 launches per step, inside "
                      "replays of the C5 step graph (event-record nodes)"}


def extra_leg(name, dtype_s, steps=10, warmup=3):
    """Secondary configs (BASELINE.json configs[2..4]): device-timed steps of both modes (CUDA graph),
    exact stash bytes and allocator peak per mode.  C5 = C2 shapes at a per-GPU batch where STASH
    runs out of HBM and RECOMPUTE fits (the OOM is caught and reported)."""
    import torch
    from paper_1805_08899_b200 import abi
    from synth import configs as K
    from synth import data as D
    dt = abi.FP32 if dtype_s == "fp32" else abi.BF16
    res = {"dtype": "f32" if dtype_s == "fp32" else "bf16"}
    if name == "C3":
        from paper_1805_08899_b200.ds2 import DS2Model as M
        cfg = K.C3
        params, batch = D.ds2_params(0, cfg, dtype_s), D.ds2_batch(1, cfg, dtype_s)
        res["workload"] = "C3 DeepSpeech2-shaped: 5 bidirectional LSTM layers, H=800, T=400, B=32"
        samples = cfg.B
    elif name == "C4":
        from paper_1805_08899_b200.transformer import TXModel as M
        cfg = K.C4
        params, batch = D.tx_params(0, cfg, dtype_s), D.tx_batch(1, cfg, dtype_s)
        res["workload"] = "C4 Transformer-base attention blocks: d=512, 8 heads, L=256, B=64, 6 blocks, dropout 0.1"
        samples = cfg.B
    elif name == "C2d":
        from dataclasses import replace
        from paper_1805_08899_b200.nmt import NMTModel as M
        cfg = replace(K.C2, dropout=0.1)
        params, batch = D.nmt_params(0, cfg, dtype_s), D.nmt_batch(1, cfg)
        res["workload"] = "C2d NMT (C2 shapes) with embedding dropout p=0.1 (R31): byte / 1-bit / regenerated masks"
        samples = cfg.B
    else:
        from paper_1805_08899_b200.nmt import NMTModel as M
        Bc5 = 24576 if dtype_s == "bf16" else 16384
        cfg = K.C2.with_batch(Bc5)
        params, batch = D.nmt_params(0, cfg, dtype_s), D.nmt_batch(1, cfg)
        res["workload"] = f"C5 NMT (C2 shapes) at B={Bc5} per GPU: STASH exceeds HBM, RECOMPUTE fits"
        samples = cfg.B
    plans = [(abi.STASH, "stash", False), (abi.RECOMPUTE, "recompute", False)]
    if name in ("C3", "C4", "C2d"):                  # the prior-work Mirror plan on the same kernels
        plans.append((abi.RECOMPUTE, "mirror", True))
    if name in ("C4", "C2d"):                        # Echo's plan with Philox-regenerated masks (R30)
        plans.append((abi.RECOMPUTE, "recompute_regen_masks", "regen"))
    for mode, mname, mirror in plans:
        r = {}
        m = None
        try:
            m = M(cfg, dt, mode, regen_masks=True) if mirror == "regen" else \
                M(cfg, dt, mode, mirror=True) if mirror else M(cfg, dt, mode)
            m.load_params(params)
            m.upload_batch(batch)
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats()
            base = torch.cuda.memory_allocated()
            acts = m._forward()
            r["stash_bytes"] = m.stash_bytes()
            m._backward(acts)
            del acts
            torch.cuda.synchronize()
            r["peak_activation_bytes"] = torch.cuda.max_memory_allocated() - base
            m.capture(0.01)
            for _ in range(warmup):
                m.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                m.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            r.update({"ms_per_step": ms, "samples_per_s": samples / (ms / 1e3), "steps": steps, "cuda_graph": True})
            if name == "C5" and mname == "recompute":       # a6 in-step roofline where the batch fills HBM
                try:
                    r["a6_roofline"] = c5_a6_roofline(m, cfg, dt)
                except torch.OutOfMemoryError as ex:
                    r["a6_roofline"] = {"error": str(ex).split("\n")[0][:120]}
        except torch.OutOfMemoryError as ex:
            r["oom"] = str(ex).split("\n")[0][:160]
        finally:
            m = None
            torch.cuda.empty_cache()
        res[mname] = r
    st, rc = res["stash"], res["recompute"]
    if "ms_per_step" in st and "ms_per_step" in rc:
        res["recompute_overhead"] = rc["ms_per_step"] / st["ms_per_step"] - 1.0
    if st.get("stash_bytes") and rc.get("stash_bytes"):
        res["stash_ratio"] = st["stash_bytes"] / rc["stash_bytes"]
    mi = res.get("mirror")
    if mi and "ms_per_step" in mi and "ms_per_step" in st:
        res["mirror_overhead"] = mi["ms_per_step"] / st["ms_per_step"] - 1.0
    if mi and mi.get("stash_bytes") and st.get("stash_bytes"):
        res["mirror_stash_ratio"] = st["stash_bytes"] / mi["stash_bytes"]     # < 1: Mirror keeps MORE
    return res


def run_ours(args):
    import torch
    from paper_1805_08899_b200 import abi, dp
    from paper_1805_08899_b200.nmt import NMTModel
    from synth.configs import C2
    from synth.data import nmt_params, nmt_batch

    ws, rank, local = dp.init()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    dtype = abi.FP32 if args.dtype == "fp32" else abi.BF16
    cfg = C2.with_batch(args.batch) if args.batch else C2
    params = nmt_params(0, cfg)                                  # replicated model, same seed on all ranks
    nb = 4
    host_batches = [nmt_batch(dp.shard_seed(10 + i, rank), cfg) for i in range(nb)]
    pinned = []
    for b in host_batches:
        pinned.append({k: torch.from_numpy(b[k]).pin_memory() for k in ("src", "tgt_in", "tgt_out", "src_len")})
    lr = 0.05

    def build(mode, mirror=False):
        m = NMTModel(cfg, dtype=dtype, mode=mode, device=dev, mirror=mirror)
        m.load_params(params)
        m.upload_batch(pinned[0])
        return m

    ar = dp.BucketAllreduce(dev) if ws > 1 else None

    def runner(m, use_graph):
        """One training step.  N = 1: the whole step (fwd + bwd + SGD) is one CUDA graph.  N > 1: two
        graphs split where the decoder-side gradients are final (NMTModel.capture_split); that bucket's
        NCCL allreduce runs on a communication stream while the encoder-backward graph replays, then
        the encoder bucket's; mean over ranks and the SGD update follow (NCCL stays out of capture).
        Eager N > 1 launches the same buckets from the backward pass itself."""
        if ws == 1:
            return m.replay if use_graph else (lambda: m.step(lr))

        def step():
            if use_graph:
                m.replay_dp(ar, lr)
            else:
                m.bucket_hook = lambda i: ar.launch(m.buckets[i])
                try:
                    m.step(0.0)
                finally:
                    m.bucket_hook = None
                ar.finish(m.gflat)
                m.apply_update(lr)
        return step

    def timed(m, use_graph, K, W):
        """Device-timed K steps (inputs resident in HBM); returns ms per step (max over ranks)."""
        abi.LAUNCHES["count"] = 0
        if use_graph:
            if ws == 1:
                m.capture(lr)
            else:
                m.capture_split()
        launches_per_step = abi.LAUNCHES["count"]
        if use_graph:
            launches_per_step = launches_per_step // 3       # capture() = 2 warm-up steps + 1 captured
        run = runner(m, use_graph)
        for _ in range(W):
            run()
        torch.cuda.synchronize()
        dp.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            run()
        e1.record()
        torch.cuda.synchronize()
        dp.barrier()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        return dp.max_over_ranks(ms, dev), launches_per_step

    def e2e(m, use_graph, K):
        """Same metric through the public API with host buffers: per step H2D of the batch from pinned
        memory, the step, and a D2H read of the loss."""
        run = runner(m, use_graph)
        torch.cuda.synchronize()
        dp.barrier()
        t0 = time.perf_counter()
        for i in range(K):
            m.upload_batch(pinned[i % nb])
            run()
            float(m.loss.item())
        dt = (time.perf_counter() - t0) / K
        dt = dp.max_over_ranks(dt, dev)
        return dt

    def peak_activation(mode, mirror=False):
        m = NMTModel(cfg, dtype=dtype, mode=mode, device=dev, mirror=mirror)
        m.load_params(params)
        m.upload_batch(pinned[0])
        m.step(0.0)                                              # warm the allocator / cuBLAS handles
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        start = torch.cuda.memory_allocated(dev)
        acts = m._forward()
        stash = m.stash_bytes()
        m._backward(acts)
        del acts
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated(dev) - start
        del m
        torch.cuda.empty_cache()
        return peak, stash

    use_graph = not args.no_graph
    mode = abi.RECOMPUTE if args.mode == "recompute" else abi.STASH
    model = build(mode)
    try:
        ms, launches = timed(model, use_graph, args.steps, args.warmup)
    except Exception as ex:                                      # graph capture failure -> eager, stated
        if not use_graph:
            raise
        print(f"[bench] CUDA graph capture failed ({ex}); timing eager", file=sys.stderr)
        use_graph = False
        model = build(mode)
        ms, launches = timed(model, False, args.steps, args.warmup)
    sampler = ClockSampler(local)
    sampler.start()
    # clocks are sampled over a second identical timed region (the first one followed the capture);
    # the sampler starts before that region's own W warm-up steps so that a short region (bf16: K
    # steps of ~7 ms) still gets samples taken under the same load
    run = runner(model, use_graph)
    t_w = time.perf_counter()
    while True:
        for _ in range(args.warmup):
            run()
        torch.cuda.synchronize()
        if time.perf_counter() - t_w > 0.5:
            break
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        run()
    b.record()
    torch.cuda.synchronize()
    ms2 = dp.max_over_ranks(a.elapsed_time(b) / args.steps, dev)
    clocks = sampler.stop()
    ms_first, ms = ms, ms2                                       # the reported value: the clock-sampled region
    e2e_s = e2e(model, use_graph, max(10, args.steps))
    allreduce = dp.time_allreduce(model.numel, dev, steps=max(10, args.steps)) if ws > 1 else None
    in_bytes = model.input_bytes()
    del model
    torch.cuda.empty_cache()

    def probe_kernels(mode, K, W):
        """In-step kernel timing: the step graph re-captured with timing events around every a5 / a6
        launch (event-record nodes on the launch stream); K replays, durations read after each."""
        m = build(mode)
        m.capture(lr, with_probe=True)
        for _ in range(W):
            m.replay()
        per = {}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for _ in range(K):
            e0.record()
            m.replay()
            e1.record()
            for k, v in m.kernel_times().items():
                per.setdefault(k, []).extend(v)
            tot += e0.elapsed_time(e1)
        del m
        torch.cuda.empty_cache()
        return {"ms_per_step": tot / K, "launch_ms": {k: statistics.mean(v) for k, v in per.items()},
                "launches_per_step": {k: len(v) // K for k, v in per.items()}}

    out = {}
    # Rank-0-only extras below must not call collectives (the other ranks are already waiting in the
    # final barrier): timed() (barriers, max-over-ranks, allreduce in the runner) only runs at N = 1;
    # the plan comparisons (STASH, Mirror), the secondary legs and the CPU baseline are N = 1 results.
    if rank == 0 and not args.quick:
        other = abi.STASH if mode == abi.RECOMPUTE else abi.RECOMPUTE
        ms_other = None
        if ws == 1:
            try:
                m2 = build(other)
                ms_other, _ = timed(m2, use_graph, args.steps, args.warmup)
                del m2
                torch.cuda.empty_cache()
            except Exception as ex:
                print(f"[bench] {('stash', 'recompute')[other]} timing failed: {ex}", file=sys.stderr)
        mem = {}
        for md in (abi.STASH, abi.RECOMPUTE):
            try:
                mem[md] = peak_activation(md)
            except torch.OutOfMemoryError:
                mem[md] = (None, None)
        try:                                                     # prior-work Mirror plan (Table 1 analogue)
            if ws > 1:
                raise RuntimeError("N = 1 comparison")
            m3 = build(abi.RECOMPUTE, mirror=True)
            ms_mirror, _ = timed(m3, use_graph, args.steps, args.warmup)
            del m3
            torch.cuda.empty_cache()
            out["mirror"] = {"ms_per_step": ms_mirror, "mem": peak_activation(abi.RECOMPUTE, mirror=True)}
        except Exception as ex:
            if ws == 1:
                print(f"[bench] mirror plan failed: {ex}", file=sys.stderr)
        out["ms_other"] = ms_other
        out["mem"] = mem
        if ws == 1 and use_graph:                                # the same step without the CUDA graph
            try:
                m4 = build(mode)
                out["eager"], _ = timed(m4, False, max(3, args.steps // 2), args.warmup)
                del m4
                torch.cuda.empty_cache()
            except Exception as ex:
                print(f"[bench] eager timing failed: {ex}", file=sys.stderr)
        out["kern"] = time_attn_bwd(cfg, dtype)
        out["probe"] = probe_kernels(mode, args.steps, args.warmup) if use_graph and mode == abi.RECOMPUTE else None
        out["traffic"] = ncu_traffic(dtype) if cfg.B == 128 else None
    if ws > 1 and rank != 0:
        dp.barrier()
        return
    samples = cfg.B * ws
    line = {
        "metric": _metric(),
        "value": samples / (ms / 1e3),
        "unit": "samples/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "ms_per_step_first_region": ms_first,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if dtype == abi.FP32 else "bf16",
        "data": "synthetic (seeded tokens, random-init weights)",
        "config": {"workload": f"{cfg.name}: Sockeye-style LSTM NMT 2+2 layers, hidden 512, MLP attention",
                   "mode": args.mode, "global_batch": samples, "batch_per_gpu": cfg.B, "seq_len": cfg.Ts,
                   "hidden": cfg.H, "vocab": cfg.V, "parallelism": f"dp{ws}", "cuda_graph": use_graph,
                   "tf32": dtype == abi.BF16,
                   "tf32_gemms": ("the per-step attention backward GEMMs and weight-gradient GEMMs with fp32 "
                                  "gradient operands (reading R28)") if dtype == abi.BF16 else "none (IEEE fp32)",
                   "dp_backend": dp.backend_name() if ws > 1 else None,
                   "allreduce": "2 buckets (decoder side overlapped with the encoder backward)" if ws > 1 else None,
                   "l2": "no flush: per-step working set (weights 92 MB + activations >0.4 GB) > 126 MB L2"},
        "gpu_launches": launches * args.steps,
        "e2e": {"value": samples / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": 4},
        "clocks": clocks,
        "allreduce": allreduce,
        "paper_context": "Baseline 1192 samples/s, 10.0 GB (Table 1) / Echo ~3.0 GB, 3.13x footprint reduction "
                         "at B=128 on 1x RTX 2080 Ti, IWSLT15 en-vi (PAPER.md:297-299, 763-765); context, not a target",
    }
    if "kern" in out:
        k = out["kern"]
        pk = _peaks()
        iso = k["bytes"] / (k["ms"] / 1e3) / 1e9
        pr = out.get("probe")
        if pr and "attn_bwd" in pr["launch_ms"]:
            l_ms = pr["launch_ms"]["attn_bwd"]
            timing = (f"CUDA events on the launch stream around each of the {pr['launches_per_step']['attn_bwd']} "
                      f"a6 launches per step, inside {args.steps} replays of the step graph (event-record nodes)")
            share = pr["launches_per_step"]["attn_bwd"] * l_ms / pr["ms_per_step"]
        else:
            l_ms, timing, share = k["ms"], "CUDA events, L2 flushed (256 MiB read) before each launch", cfg.Td * k["ms"] / ms
        achieved = k["bytes"] / (l_ms / 1e3) / 1e9
        line["roofline"] = {"bound": "hbm", "kernel": "echo_attn_bwd_recompute (a6, RECOMPUTE)", "achieved": achieved,
                            "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                            "traffic": (out["traffic"] or {}).get("bytes"),
                            "traffic_source": (out["traffic"] or {}).get("source"), "peak_source": pk["source"],
                            "bytes_per_launch": k["bytes"], "bytes_per_row": k["bytes_per_row"],
                            "launch_us": 1e3 * l_ms, "timing": timing, "share_of_step": share,
                            "isolated": {"launch_us": 1e3 * k["ms"], "achieved": iso, "frac": iso / pk["hbm_gbs"],
                                         "timing": "standalone launch, CUDA events, L2 flushed (256 MiB read) before each"}}
        if pr:
            line["roofline"]["probe_step_ms"] = pr["ms_per_step"]
            line["roofline"]["in_step_launch_us"] = {kk: 1e3 * vv for kk, vv in pr["launch_ms"].items()}
        mem = out["mem"]
        st, rc = mem[abi.STASH], mem[abi.RECOMPUTE]
        line["memory"] = {
            "peak_activation_bytes": {"stash": st[0], "recompute": rc[0]},
            "stash_bytes": {"stash": st[1], "recompute": rc[1]},
            "peak_ratio": (st[0] / rc[0]) if st[0] and rc[0] else None,
            "stash_ratio": (st[1] / rc[1]) if st[1] and rc[1] else None,
            "how": "torch max_memory_allocated - memory_allocated at step start (eager), fp32 allocator bytes",
        }
        try:                                                     # the host estimator's numbers beside them
            from synth import graphs as Gr
            gdoc = json.dumps(Gr.nmt(cfg, "f32" if dtype == abi.FP32 else "bf16"))
            est = {s_: json.loads(abi.echo_footprint_estimate(gdoc, json.dumps({"strategy": s_})))
                   for s_ in ("baseline", "echo")}
            line["memory"]["estimator"] = {
                "stash_bytes": {"stash": est["baseline"]["stash_bytes"], "recompute": est["echo"]["stash_bytes"]},
                "peak_bytes": {"stash": est["baseline"]["peak_bytes"], "recompute": est["echo"]["peak_bytes"]},
                "how": "echo_footprint_estimate on the step's graph (synth/graphs.py nmt): stash bytes are exact "
                       "(== stash_bytes above); peak = its liveness model of feature maps and activation "
                       "gradients over one schedule (no GEMM workspaces, no allocator rounding)"}
        except Exception as ex:
            print(f"[bench] estimator numbers failed: {ex}", file=sys.stderr)
        mi = out.get("mirror")
        if mi:
            line["mirror_mode"] = {
                "plan": "Mirror (Chen et al.; PAPER.md:286-305 Table 1): cheap ops mirrored, FC inputs and "
                        "the FC outputs feeding mirrored adds kept",
                "value": samples / (mi["ms_per_step"] / 1e3), "ms_per_step": mi["ms_per_step"],
                "peak_activation_bytes": mi["mem"][0], "stash_bytes": mi["mem"][1],
                "stash_reduction_vs_stash": (st[1] / mi["mem"][1]) if st[1] and mi["mem"][1] else None}
        if out.get("eager"):
            line["eager_mode"] = {"value": samples / (out["eager"] / 1e3), "ms_per_step": out["eager"],
                                  "how": "the same step launched from the host without the CUDA graph "
                                         "(SURVEY 8(d): eager and graph mode reported separately), device-timed"}
        if out["ms_other"]:
            other_name = "stash" if mode == abi.RECOMPUTE else "recompute"
            line[f"{other_name}_mode"] = {"value": samples / (out["ms_other"] / 1e3), "ms_per_step": out["ms_other"]}
            if mode == abi.RECOMPUTE:
                line["recompute_overhead"] = ms / out["ms_other"] - 1.0
    if rank == 0 and ws == 1 and not args.quick and args.legs:
        extra = {}
        for leg in [x for x in args.legs.split(",") if x]:
            try:
                extra[leg] = extra_leg(leg, args.leg_dtype)
            except Exception as ex:                               # a secondary leg never breaks the line
                extra[leg] = {"error": f"{type(ex).__name__}: {ex}"[:200]}
        line["configs_extra"] = extra
    if rank == 0 and ws == 1 and not args.quick and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample()
    print(json.dumps(line), flush=True)
    if ws > 1:
        dp.barrier()


def relaunch_if_needed(args):
    """--gpus N: under torchrun WORLD_SIZE must equal N; without torchrun and N > 1, re-exec this command
    under `torch.distributed.run --nproc-per-node N` (one process per GPU, rendezvous on 127.0.0.1).
    If the box has fewer GPUs than N the ranks share them over gloo (ECHO_DP_BACKEND=gloo): a
    functional run of the multi-rank path, not a scaling measurement (the JSON line says which)."""
    if "WORLD_SIZE" in os.environ:
        ws = int(os.environ["WORLD_SIZE"])
        if ws != args.gpus:
            print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={ws}: launch one rank per GPU with "
                  f"--nproc-per-node {args.gpus}", file=sys.stderr)
            sys.exit(2)
        return
    if args.gpus <= 1:
        return
    import socket
    import torch
    env = dict(os.environ)
    have = torch.cuda.device_count()
    if have < args.gpus:
        env.setdefault("ECHO_DP_BACKEND", "gloo")
        print(f"[bench] {args.gpus} ranks on {have} GPU(s): ranks share GPUs over gloo (functional run, "
              f"not a scaling number)", file=sys.stderr)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd, env=env).returncode)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"])
    ap.add_argument("--mode", default="recompute", choices=["recompute", "stash"])
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: C2's 128)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the stash comparison, memory and kernel legs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--legs", default="C3,C4,C2d,C5", help="secondary configs to report (C3,C4,C2d,C5; '' for none)")
    ap.add_argument("--leg-dtype", default="bf16", choices=["fp32", "bf16"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "ours":
        relaunch_if_needed(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
