"""GPU data-parallel parity: two ranks run the GPU RECOMPUTE step
(libecho hot path) on their shards of a global batch and exchange the gradient through
dp.BucketAllreduce -- the decoder-side bucket launched from inside the backward pass (eager) or
between the two split step graphs (NMTModel.capture_split / replay_dp, the bench's N > 1 path) --
and the averaged gradient equals the fp64 oracle's gradient of the GLOBAL-batch loss (reading R10)
within the fp32 tolerance.  The pool's boxes have one GPU, so both ranks share it over gloo; on an
8-GPU node the same code runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch

from synth.configs import SMALL_NMT
from synth.data import nmt_params, nmt_batch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    import torch.distributed as dist
    from paper_1805_08899_b200 import abi, dp
    from paper_1805_08899_b200.nmt import NMTModel
    torch.backends.cuda.matmul.allow_tf32 = False
    ws, r, local = dp.init(backend="gloo")
    torch.cuda.set_device(local)
    cfg = SMALL_NMT
    m = NMTModel(cfg, abi.FP32, abi.RECOMPUTE, device=f"cuda:{local}")
    m.load_params(nmt_params(0, cfg))
    m.upload_batch(nmt_batch(dp.shard_seed(7, rank), cfg, lengths="random"))
    ar = dp.BucketAllreduce(m.device)
    # eager: buckets launched from inside the backward pass
    m.bucket_hook = lambda i: ar.launch(m.buckets[i])
    m.step(0.0)
    m.bucket_hook = None
    ar.finish(m.gflat)
    torch.cuda.synchronize()
    eager = m.gflat.clone()
    # graph: the bench's N > 1 path
    m.capture_split()
    m.gflat.zero_()
    m.replay_dp(ar, 0.0)
    torch.cuda.synchronize()
    graph = m.gflat.clone()
    if rank == 0:
        q.put({"eager": m.grads_numpy(),
               "bitwise": bool(torch.equal(eager.view(torch.int32), graph.view(torch.int32))),
               "buckets": [int(b.numel()) for b in m.buckets]})
    dp.barrier()
    dist.destroy_process_group()


def test_two_rank_gpu_gradient_equals_global_batch_oracle(cuda_dev):
    import torch.multiprocessing as mp
    from oracle import nmt as O
    from paper_1805_08899_b200 import dp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=900)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert out["bitwise"], "split-graph replay differs from the eager bucketed step"
    cfg = SMALL_NMT
    shards = [nmt_batch(dp.shard_seed(7, r), cfg, lengths="random") for r in range(world)]
    glob = {k: np.concatenate([s[k] for s in shards], axis=0) for k in shards[0]}
    ref = O.step(nmt_params(0, cfg), glob, cfg.with_batch(cfg.B * world))["grads"]
    for k, v in ref.items():
        err = np.abs(out["eager"][k] - v).max() / max(np.abs(v).max(), 1e-30)
        assert err <= 1e-4, (k, err)
    assert sum(out["buckets"]) >= sum(v.size for v in ref.values()) and min(out["buckets"]) > 0
