"""Batch-sharded data parallelism.

One process per GPU.  Rank r trains on its own shard of the global batch
(seeded base + r) with a replicated model; the only exchange is one allreduce
of the flat fp32 gradient buffer per step (NCCL over NVLink 5 / NVSwitch on the
GPU box, gloo in the CPU tests), followed by division by the world size, so the
update equals the gradient of the global-batch mean loss (reading R10).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def init(backend=None):
    """Initialise the default process group from torchrun's environment (no-op for world size 1)."""
    ws, rank, local = world()
    if torch.cuda.is_available() and torch.cuda.device_count() > 0:
        local = local % torch.cuda.device_count()      # (a multi-rank smoke test on a 1-GPU box shares it)
    if ws > 1 and not dist.is_initialized():
        if backend is None:
            backend = os.environ.get("ECHO_DP_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)                 # bind the rank to its GPU before NCCL starts
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend=backend, rank=rank, world_size=ws, **kw)
    return ws, rank, local


def shard_seed(base: int, rank: int) -> int:
    return base + 1000 * rank


def allreduce_mean_(flat: torch.Tensor) -> torch.Tensor:
    """flat <- mean over ranks of flat (sum allreduce, then / world size)."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)
        flat.div_(dist.get_world_size())
    return flat


def backend_name():
    return dist.get_backend() if dist.is_initialized() else None


def world_size() -> int:
    return dist.get_world_size() if dist.is_initialized() else 1


class BucketAllreduce:
    """Overlapped gradient exchange (SURVEY.md §8(e) option): each bucket -- a contiguous slice of the
    flat fp32 gradient whose values are final -- is summed across ranks on a dedicated communication
    stream as soon as the backward pass reaches it, while the compute stream goes on with the rest of
    the backward (the NMT decoder / attention / output bucket overlaps the encoder backward).
    finish() makes the compute stream wait for every launched bucket and divides by the world size,
    so the result equals allreduce_mean_ of the whole buffer."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.cuda = self.device.type == "cuda"
        self.stream = torch.cuda.Stream(device=self.device) if self.cuda else None
        self.works = []

    def launch(self, bucket: torch.Tensor):
        if world_size() == 1:
            return
        if not self.cuda:                                  # host tensors (the gloo CPU tests)
            self.works.append((dist.all_reduce(bucket, op=dist.ReduceOp.SUM, async_op=True), bucket))
            return
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)                       # the bucket's producers are done
        with torch.cuda.stream(self.stream):
            self.works.append((dist.all_reduce(bucket, op=dist.ReduceOp.SUM, async_op=True), bucket))
            bucket.record_stream(self.stream)

    def finish(self, flat: torch.Tensor):
        if world_size() == 1:
            return flat
        for w, _ in self.works:
            w.wait()                                       # compute stream waits (NCCL) / host waits (gloo)
        if self.cuda:
            torch.cuda.current_stream(self.device).wait_stream(self.stream)
        self.works = []
        flat.div_(world_size())
        return flat


def time_allreduce(numel: int, device, steps: int = 20, warmup: int = 3) -> dict:
    """The step's gradient exchange in isolation: `steps` sum-allreduces of a `numel` fp32 buffer,
    CUDA events on the launching stream, max over ranks.  algbw = bytes / time; busbw = algbw *
    2 (N-1) / N (the ring-equivalent bytes each GPU moves)."""
    n = world_size()
    buf = torch.zeros(numel, dtype=torch.float32, device=device)
    for _ in range(warmup):
        dist.all_reduce(buf)
    torch.cuda.synchronize(device)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        dist.all_reduce(buf)
    e1.record()
    torch.cuda.synchronize(device)
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, device)
    nbytes = numel * 4
    algbw = nbytes / (ms / 1e3) / 1e9
    out = {"bytes": nbytes, "ms": ms, "algbw_GBps": algbw, "busbw_GBps": algbw * 2 * (n - 1) / n,
           "backend": dist.get_backend(), "nranks": n, "timing": f"{steps} allreduces, CUDA events, max over ranks"}
    try:
        v = torch.cuda.nccl.version()
        out["nccl_version"] = ".".join(map(str, v)) if isinstance(v, tuple) else str(v)
    except Exception:
        pass
    return out


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
