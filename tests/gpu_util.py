"""Helpers for GPU parity tests (test infrastructure)."""
import numpy as np
import torch

TOL = {"fp32": 1e-4, "bf16": 2e-2}     # north_star: max relative error (reading R14: inf-norm relative)


def dev(x, storage="fp32", dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        return t.to(device="cuda", dtype=dtype)
    if t.dtype in (torch.int64, torch.int32):
        return t.cuda()
    return t.to(device="cuda", dtype=torch.bfloat16 if storage == "bf16" else torch.float32)


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def relerr(x, y):
    """max_i |x_i - y_i| / max_i |y_i|  (reading R14)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    den = np.abs(y).max()
    return float(np.abs(x - y).max() / (den if den > 0 else 1.0))


def assert_close(x, y, storage, what=""):
    e = relerr(x, y)
    assert e <= TOL[storage], f"{what}: rel err {e:.3e} > {TOL[storage]}"
    return e


def bits_equal(a, b):
    return torch.equal(a.reshape(-1).contiguous().view(torch.uint8) if a.dtype != torch.bool else a,
                       b.reshape(-1).contiguous().view(torch.uint8) if b.dtype != torch.bool else b)


def relerr_fro(x, y):
    """||x - y||_2 / ||y||_2 (Frobenius), the bf16 metric for whole-model gradients (reading R14)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    den = np.linalg.norm(y)
    return float(np.linalg.norm(x - y) / (den if den > 0 else 1.0))


def check_grads(g, ref, storage, fro_only=(), what=""):
    """Per-tensor gate at north_star's tolerance: max relative error (inf-norm, reading R14) <= TOL for
    every tensor, except the tensors named in `fro_only` (bf16 storage only; each one is listed with its
    measured numbers and bf16 noise floor in DESIGN.md R14b), which are gated on the Frobenius relative
    error instead.  Both metrics are printed for every tensor (pytest -s / -rA shows them)."""
    tol = TOL[storage]
    bad = []
    for k, v in ref.items():
        e_inf, e_fro = relerr(g[k], v), relerr_fro(g[k], v)
        print(f"[parity] {what} {storage} {k}: inf {e_inf:.3e} fro {e_fro:.3e}")
        if k in fro_only:
            assert storage == "bf16", k
            if e_fro > tol:
                bad.append((k, "fro", e_fro, e_inf))
        elif e_inf > tol:
            bad.append((k, "inf", e_inf, e_fro))
    assert not bad, bad
