"""Multi-process data parallelism on CPU (gloo, world size 2): the host-side DP logic of dp.py —
batch sharding by rank, one allreduce of the flat fp32 gradient, division by the world size —
reproduces the gradient of the global-batch loss (reading R10).  The per-rank gradients come
from the fp64 oracle (the GPU kernels need a GPU); the exchange code is the product's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth.configs import SMALL_NMT
from synth.data import nmt_params, nmt_batch, nmt_param_shapes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    from paper_1805_08899_b200 import dp
    from oracle import nmt as O
    ws, r, _ = dp.init(backend="gloo")
    assert (ws, r) == (world, rank)
    cfg = SMALL_NMT
    params = nmt_params(0, cfg)
    batch = nmt_batch(dp.shard_seed(7, rank), cfg, lengths="random")
    g = O.step(params, batch, cfg)["grads"]
    flat = torch.cat([torch.from_numpy(g[n].astype(np.float32).reshape(-1)) for n, _ in nmt_param_shapes(cfg)])
    buck = flat.clone()
    dp.allreduce_mean_(flat)
    ar = dp.BucketAllreduce("cpu")                         # the overlapped two-bucket exchange, same result
    n0 = buck.numel() // 3
    ar.launch(buck[:n0])
    ar.launch(buck[n0:])
    ar.finish(buck)
    assert torch.equal(buck, flat)
    m = dp.max_over_ranks(float(rank))
    if rank == 0:
        out.put((flat.numpy(), m))
    dp.barrier()
    dist.destroy_process_group()


def test_allreduce_mean_equals_global_batch_gradient():
    from oracle import nmt as O
    from paper_1805_08899_b200 import dp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    flat, m = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert m == 1.0
    # global batch = the two shards concatenated along B
    cfg = SMALL_NMT
    shards = [nmt_batch(dp.shard_seed(7, r), cfg, lengths="random") for r in range(world)]
    glob = {k: np.concatenate([s[k] for s in shards], axis=0) for k in shards[0]}
    gcfg = cfg.with_batch(cfg.B * world)
    ref = O.step(nmt_params(0, cfg), glob, gcfg)["grads"]
    ref_flat = np.concatenate([ref[n].reshape(-1) for n, _ in nmt_param_shapes(cfg)])
    err = np.abs(flat - ref_flat).max() / np.abs(ref_flat).max()
    assert err < 1e-6, err


def test_shard_seeds_distinct():
    from paper_1805_08899_b200 import dp
    seeds = {dp.shard_seed(10, r) for r in range(8)}
    assert len(seeds) == 8
