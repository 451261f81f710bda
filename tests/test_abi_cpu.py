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


def _prototypes():
    """name -> list of C parameter declarations, from include/echo.h."""
    src = open(os.path.join(ROOT, "include", "echo.h")).read()
    src = re.sub(r"/\*.*?\*/", " ", src, flags=re.S)
    src = re.sub(r"//[^\n]*", " ", src)
    out = {}
    for m in re.finditer(r"\b(?:echo_status|int|const char\*|void)\s+(echo_[a-z_0-9]+)\s*\(([^;{]*?)\)\s*;", src, flags=re.S):
        params = " ".join(m.group(2).split())
        out[m.group(1)] = [] if params in ("", "void") else [p.strip() for p in params.split(",")]
    return out


def test_binding_argtypes_match_the_header(lib):
    """Every ctypes signature in abi.py has the header's arity and, position by position, the same kind
    of argument (pointer / int32 / int64 / uint32 / uint64 / float / size_t): an edited prototype cannot
    silently drift from the binding."""
    import ctypes
    protos = _prototypes()
    assert len(protos) >= len(NORTH_STAR)
    scalar = {"int32_t": (ctypes.c_int32, ctypes.c_int), "int": (ctypes.c_int32, ctypes.c_int),
              "int64_t": (ctypes.c_int64,), "uint32_t": (ctypes.c_uint32,), "uint64_t": (ctypes.c_uint64,),
              "float": (ctypes.c_float,), "size_t": (ctypes.c_size_t,)}
    checked = 0
    for name, params in protos.items():
        argtypes = getattr(lib, name).argtypes
        if argtypes is None:                      # echo_last_error / echo_abi_version / debug hooks
            assert not params or name.startswith("echo_debug"), name
            continue
        assert len(argtypes) == len(params), (name, len(argtypes), params)
        for k, (p, a) in enumerate(zip(params, argtypes)):
            ctype = re.sub(r"\b(const|restrict)\b", "", p.rsplit(" ", 1)[0] if not p.endswith("*") else p).strip()
            if "*" in p:
                ok = a in (ctypes.c_void_p, ctypes.c_char_p) or (hasattr(a, "_type_") and a.__name__.startswith("LP_"))
            else:
                base = ctype.split()[-1]
                ok = a in scalar.get(base, (ctypes.c_int32, ctypes.c_int) if base.startswith("echo_") else ())
            assert ok, (name, k, p, a)
        checked += 1
    assert checked >= 25
