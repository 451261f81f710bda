"""The boundary from plain C: include/echo.h compiles as a C99 header (gcc, -Wall -Werror, no C++, no
CUDA headers) and a C program linked against libecho.so runs the host-only calls (version, the
footprint estimator with its two-call report convention, the workspace queries, descriptor
validation).  No GPU needed."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1805_08899_b200 import build, abi
    build.build()
    return abi.LIB_PATH


def test_header_is_c99_and_abi_callable_from_c(lib, tmp_path):
    exe = str(tmp_path / "abi_from_c")
    libdir = os.path.dirname(lib)
    cc = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"),
          os.path.join(ROOT, "tests", "c", "abi_from_c.c"), "-o", exe, f"-L{libdir}", "-l:libecho.so",
          f"-Wl,-rpath,{libdir}"]
    r = subprocess.run(cc, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok ") >= 9 and "FAIL" not in r.stdout
