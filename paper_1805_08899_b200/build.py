"""Build libecho.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_1805_08899_b200.build        # or __graft_entry__.build()

Every .cu / .cpp under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
(no --use_fast_math: the rounding contract relies on IEEE expf/tanhf and
explicit __f*_rn intrinsics) and linked into paper_1805_08899_b200/libecho.so.
Rebuilds when a source or header is newer than the library or when the build flags (ECHO_NVCC_EXTRA)
differ from the ones recorded in the stamp file next to it (libecho.so.flags), so an instrumented
build (e.g. -DECHO_PHASE_TIMING) is never picked up silently by a later plain build() call.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libecho.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "echo.h"), os.path.abspath(__file__)]


STAMP = LIB + ".flags"


def _flags() -> str:
    return " ".join(os.environ.get("ECHO_NVCC_EXTRA", "").split())


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    try:
        with open(STAMP) as f:
            if f.read().strip() != _flags():
                return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for src in _sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include")]
        cmd += os.environ.get("ECHO_NVCC_EXTRA", "").split()
        if src.endswith(".cu"):
            cmd += ["-lineinfo", "-Xptxas", "-v" if verbose else "-O3"]
        cmd += ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(_flags() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
