"""The multi-rank bench path (torchrun, one process per rank, eager allreduce after the step graph,
barrier + max-over-ranks timing, rank 0 prints one JSON line) exercised with 2 ranks.  The pool's
boxes have one GPU, so both ranks share it and talk over gloo (ECHO_DP_BACKEND); on an 8-GPU node
the same code runs one rank per GPU over NCCL."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("quick", [True, False], ids=["quick", "full"])
def test_bench_two_ranks(quick, cuda_dev):
    """quick: the timed path only; full: also rank 0's extras (memory peaks, a6 probe / roofline),
    which must not issue collectives while the other ranks wait in the final barrier."""
    env = dict(os.environ, ECHO_DP_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29541" if quick else "29542", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-cpu"] + (["--quick"] if quick else [])
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout                       # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 2 * d["config"]["batch_per_gpu"]
    assert d["value"] > 0 and d["scaling"] == "weak"
    if not quick:
        assert d["roofline"]["frac"] > 0 and "memory" in d and "configs_extra" not in d


def test_bench_gpus_flag_relaunches(cuda_dev):
    """`python bench.py --gpus 2` (no torchrun) re-executes itself under torch.distributed.run with two
    ranks (sharing the pool's single GPU over gloo) and reports n_gpus = 2 and the isolated allreduce."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--quick"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
    assert d["allreduce"]["nranks"] == 2 and d["allreduce"]["bytes"] > 0

