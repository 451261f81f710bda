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


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
