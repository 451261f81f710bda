"""CPU checks of the C-ABI library: it builds for sm_100a, loads without a GPU and exports
every entry point include/echo.h declares (no compute calls)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1805_08899_b200 import build, abi
    build.build()
    return abi.load()


def _declared():
    src = open(os.path.join(ROOT, "include", "echo.h")).read()
    return sorted(set(re.findall(r"\b(echo_[a-z_0-9]+)\s*\(", src)))


NORTH_STAR = ("echo_lstm_fwd", "echo_lstm_bwd_recompute", "echo_attn_fwd", "echo_attn_bwd_recompute",
              "echo_footprint_estimate")          # BASELINE.json north_star (1), SURVEY.md §8(b)


def test_header_declares_the_five_entry_points(lib):
    from paper_1805_08899_b200 import abi
    names = _declared()
    assert abi.NORTH_STAR == NORTH_STAR
    for n in NORTH_STAR:
        assert n in names
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (echo_[a-z_0-9]+)$", out, flags=re.M))
    assert set(NORTH_STAR) <= exported
    for old in ("echo_lstm_bwd", "echo_attn_bwd"):       # the round-1 names are gone
        assert old not in exported


def test_workspace_queries_without_gpu(lib):
    """Two-call workspace convention: ws == NULL returns the size and launches nothing,
    so it runs on a host without a GPU."""
    from paper_1805_08899_b200 import abi
    T, B, H = 50, 128, 512
    assert abi.echo_lstm_bwd_ws_bytes(abi.LstmDesc(B, H, abi.FP32, abi.RECOMPUTE), T) == T * B * H * 4
    assert abi.echo_lstm_bwd_ws_bytes(abi.LstmDesc(B, H, abi.BF16, abi.RECOMPUTE), T) == T * B * H * 4
    assert abi.echo_lstm_bwd_ws_bytes(abi.LstmDesc(B, H, abi.FP32, abi.STASH), T) == 0
    d = abi.AttnDesc(B, 50, 512, 512, abi.BF16, abi.RECOMPUTE, 512, B * 512, 512, B * 512)
    assert abi.echo_attn_bwd_ws_bytes(d) == B * 512 * 4
    with pytest.raises(abi.EchoError) as e:                   # t out of range is rejected before the query
        abi.echo_lstm_bwd_recompute(abi.LstmDesc(B, H, abi.FP32, abi.RECOMPUTE), T, T, 0, *([None] * 9), stream=0)
    assert e.value.status == abi.ECHO_ERR_INVALID


def test_every_declared_symbol_is_exported(lib):
    from paper_1805_08899_b200 import abi
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (echo_[a-z_0-9]+)$", out, flags=re.M))
    for n in _declared():
        assert n in exported, n
        assert hasattr(lib, n)
    assert set(abi.EXPORTED) == set(_declared())


def test_abi_version(lib):
    from paper_1805_08899_b200 import abi
    src = open(os.path.join(ROOT, "include", "echo.h")).read()
    v = int(re.search(r"#define ECHO_ABI_VERSION (\d+)", src).group(1))
    assert abi.echo_abi_version() == v


def test_sass_is_sm100a(lib):
    from paper_1805_08899_b200 import abi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_validation_without_gpu(lib):
    """Argument validation runs on the host before any launch: bad descriptors fail cleanly."""
    from paper_1805_08899_b200 import abi
    d = abi.LstmDesc(0, 16, abi.FP32, abi.RECOMPUTE)
    with pytest.raises(abi.EchoError) as e:
        abi.echo_lstm_fwd(d, None, None, None, None, None, None, None, None, stream=0)
    assert e.value.status == abi.ECHO_ERR_INVALID
    a = abi.AttnDesc(2, 5000, 16, 16, abi.FP32, abi.RECOMPUTE, 16, 16, 16, 16)
    with pytest.raises(abi.EchoError) as e:
        abi.echo_attn_fwd(a, None, None, None, None, None, None, None, None, stream=0)
    assert e.value.status == abi.ECHO_ERR_CAPACITY
    dd = abi.DotDesc(4, 12, abi.FP32, abi.STASH, 1.0, 0.1, 0, 0)
    with pytest.raises(abi.EchoError) as e:
        abi.echo_dot_softmax_fwd(dd, None, None, None, None, stream=0)
    assert e.value.status == abi.ECHO_ERR_INVALID
