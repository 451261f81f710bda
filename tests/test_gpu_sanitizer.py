"""compute-sanitizer over the C1 training step (both modes, eager + CUDA-graph replay, the encoder
wavefront's two streams, the TMA / mbarrier / st.async attention kernels) and a C2-row attention call:
memcheck, racecheck and synccheck report nothing (SURVEY §5 race detection).  The full matrix
(small-NMT, bf16, initcheck) is scripts/run_sanitizers.sh; its round-2 logs are in profiles/."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean_c1(tool, cuda_dev):
    if not os.path.exists(CS):
        pytest.skip("compute-sanitizer not installed")
    cmd = [CS, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "scripts", "sanitize_step.py"), "--cfg", "c1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "attention ok" in out
    if tool == "racecheck":
        assert "0 hazards" in out, out[-2000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-2000:]
