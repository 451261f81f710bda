"""Transformer attention-block stack on the Echo ABI (BASELINE.json configs[3], row a7).

PAPER.md §6.3.2 (line 1002): Echo recomputes the Transformer's attention scores / softmax and
binarizes the dropout feature map (Alg. 1 line 18).  Block k (reading R27):
  q, k, v = x Wq^T, x Wk^T, x Wv^T        (cuBLAS; outside the hot path)
  S = q_h k_h^T per head                    (cuBLAS batched)
  P_d = dropout(softmax(scale * S))         (libecho a7; Philox keep-mask)
  O = P_d v_h ; y = O Wo^T + x              (cuBLAS)
Loss = mean_n y_final[n] . r.

STASH (Baseline) keeps P, the byte mask and P_d per block; RECOMPUTE (Echo's plan, as the
estimator derives it on synth/graphs.py transformer) keeps the raw scores S and a 1-bit mask and
regenerates P and P_d inside a7's backward (P_d feeds the dV GEMM).  Both keep x, the head-
layout q/k/v and O of every block (the FC / batched-dot inputs, Eq. 2).

mirror=True runs the prior-work Mirror plan (Chen et al.; the estimator's
"mirror" strategy, reading R25) on the same kernels: the cheap softmax is mirrored, so its input S
is kept, but the batched-dot gradient reads its ORIGINAL input P_d, which is kept too (S + P_d +
1-bit mask per block); a7's backward regenerates P only.

regen_masks=True (RECOMPUTE / Mirror; reading R30): the keep-mask is a pure
function of (seed, offset, index) under the counter-based Philox generator, so nothing is kept for
it -- a7's backward regenerates it (0 bytes instead of one bit per probability).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import abi, probe
from .gemm import mm
from .lstm import TORCH_DTYPE
from synth.data import tx_param_shapes


class TXModel(probe.GraphStep):
    def __init__(self, cfg, dtype=abi.FP32, mode=abi.RECOMPUTE, device="cuda", mirror=False, regen_masks=False):
        abi.load()
        if (mirror or regen_masks) and mode != abi.RECOMPUTE:
            raise ValueError("the Mirror plan and regenerated masks run the kernels in RECOMPUTE mode")
        self.cfg, self.dtype, self.mode, self.mirror = cfg, dtype, mode, bool(mirror)
        self.regen = bool(regen_masks)
        self.sd = TORCH_DTYPE[dtype]
        self.device = torch.device(device)
        self.shapes = tx_param_shapes(cfg)
        n = sum(int(np.prod(s)) for _, s in self.shapes)
        self.master = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.gflat = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.sflat = self.master if dtype == abi.FP32 else torch.zeros(n, dtype=self.sd, device=self.device)
        self.P, self.G, self.S = {}, {}, {}
        off = 0
        for name, shape in self.shapes:
            k = int(np.prod(shape))
            self.P[name] = self.master[off:off + k].view(shape)
            self.G[name] = self.gflat[off:off + k].view(shape)
            self.S[name] = self.sflat[off:off + k].view(shape)
            off += k
        self.x = torch.zeros(cfg.B * cfg.L, cfg.d_model, dtype=self.sd, device=self.device)
        self.seeds = [0] * cfg.blocks
        self.loss = torch.zeros((), dtype=torch.float32, device=self.device)
        self.stash = {}
        self.grad_hook = None

    def load_params(self, params):
        for name, _ in self.shapes:
            self.P[name].copy_(torch.from_numpy(np.asarray(params[name], np.float32)))
        if self.sflat is not self.master:
            self.sflat.copy_(self.master)

    def upload_batch(self, batch):
        x = batch["x"] if isinstance(batch["x"], torch.Tensor) else torch.from_numpy(np.ascontiguousarray(batch["x"]))
        self.x.copy_(x.reshape(self.x.shape).to(self.sd), non_blocking=True)
        seeds = [int(s) for s in batch["seeds"]]
        if self.cfg.dropout_p > 0.0:
            self.check_seeds(seeds)
        self.seeds = seeds

    def input_bytes(self):
        return self.x.numel() * self.x.element_size()

    def grads_numpy(self):
        return {k: v.detach().double().cpu().numpy() for k, v in self.G.items()}

    def seed_state(self):
        return tuple(self.seeds) if self.cfg.dropout_p > 0.0 else None

    def stash_bytes(self):
        seen, total = set(), 0
        for t in self.stash.values():
            key = (t.data_ptr(), t.numel())
            if key not in seen:
                seen.add(key)
                total += t.numel() * t.element_size()
        return total

    def _heads(self, X):
        c = self.cfg
        return X.view(c.B, c.L, c.heads, c.d_model // c.heads).permute(0, 2, 1, 3).contiguous()

    def _merge(self, Xh):
        c = self.cfg
        return Xh.permute(0, 2, 1, 3).reshape(c.B * c.L, c.d_model)

    def desc(self, k):
        c = self.cfg
        dh = c.d_model // c.heads
        return abi.DotDesc(c.B * c.heads * c.L, c.L, self.dtype, self.mode, 1.0 / math.sqrt(dh), c.dropout_p,
                           self.seeds[k], 0)

    def train_step(self, lr=0.1):
        self.step(lr)
        return float(self.loss.item())

    def step(self, lr=0.1):
        acts = self._forward()
        self._backward(acts)
        del acts
        if self.grad_hook is not None:
            self.grad_hook(self.gflat)
        if lr != 0.0:
            self.apply_update(lr)

    def apply_update(self, lr):
        """Plain SGD on the fp32 master weights, then refresh the storage-dtype copy."""
        self.master.add_(self.gflat, alpha=-lr)
        if self.sflat is not self.master:
            self.sflat.copy_(self.master)

    def _forward(self):
        c, sd, dev, md = self.cfg, self.sd, self.device, self.mode
        R, L = c.B * c.heads * c.L, c.L
        x = self.x
        blocks = []
        reg = {}
        for k in range(c.blocks):
            q, kk, v = (mm(x, self.S[f"b{k}.{n}"].t()) for n in ("Wq", "Wk", "Wv"))
            qh, kh, vh = self._heads(q), self._heads(kk), self._heads(v)
            del q, kk, v
            S = torch.matmul(qh, kh.transpose(-1, -2))                  # raw scores [B,H,L,L]
            Pd = torch.empty_like(S)
            if md == abi.STASH:
                P = torch.empty_like(S)
                mask = torch.empty(R * L, dtype=torch.uint8, device=dev)
            else:
                P = None
                mask = None if self.regen else torch.empty(R * L // 8, dtype=torch.uint8, device=dev)
            with probe.timed("dot_fwd"):
                abi.echo_dot_softmax_fwd(self.desc(k), S, Pd, P, mask)
            O = self._merge(torch.matmul(Pd, vh))
            y = torch.addmm(x, O, self.S[f"b{k}.Wo"].t())               # residual
            blk = {"x": x, "qh": qh, "kh": kh, "vh": vh, "O": O}
            if mask is not None:
                blk["mask"] = mask
            if md == abi.STASH:
                blk["P"], blk["Pd"] = P, Pd
                del S
            elif self.mirror:
                blk["S"], blk["Pd"] = S, Pd
            else:
                blk["S"] = S
                del Pd
            blocks.append(blk)
            for n, t in blk.items():
                reg[f"b{k}.{n}"] = t
            x = y
        N = c.B * c.L
        r = self.S["out.r"]
        torch.div(mm(x, r[:, None], torch.float32).sum(), N, out=self.loss)
        reg["y_final"] = x
        self.stash = reg
        return {"blocks": blocks, "y": x}

    def _backward(self, a):
        c, sd, md = self.cfg, self.sd, self.mode
        N = c.B * c.L
        G = self.G
        self.gflat.zero_()
        y = a["y"]
        G["out.r"].copy_(y.float().sum(0) / N)
        dy = (self.P["out.r"] / N).expand(N, c.d_model).contiguous()        # fp32
        a["y"] = None
        for k in reversed(range(c.blocks)):
            blk = a["blocks"][k]
            O, qh, kh, vh = blk["O"], blk["qh"], blk["kh"], blk["vh"]
            dys = dy if sd == torch.float32 else dy.to(sd)
            G[f"b{k}.Wo"].copy_(mm(dys.t(), O, torch.float32))
            dOh = self._heads(mm(dys, self.S[f"b{k}.Wo"], torch.float32).to(sd))
            dPd = torch.matmul(dOh, vh.transpose(-1, -2))
            if md == abi.STASH:
                with probe.timed("dot_bwd"):
                    abi.echo_dot_softmax_bwd(self.desc(k), None, blk["P"], blk.get("mask"), dPd, dPd, None)
                Pd = blk["Pd"]
            elif self.mirror:
                Pd = blk["Pd"]
                with probe.timed("dot_bwd"):
                    abi.echo_dot_softmax_bwd(self.desc(k), blk["S"], None, blk.get("mask"), dPd, dPd, None)
            else:
                Pd = torch.empty_like(dPd)
                with probe.timed("dot_bwd"):
                    abi.echo_dot_softmax_bwd(self.desc(k), blk["S"], None, blk.get("mask"), dPd, dPd, Pd)
            dS = dPd                                                   # dS written in place (scale included)
            dV = self._merge(torch.matmul(Pd.transpose(-1, -2), dOh))
            dQ = self._merge(torch.matmul(dS, kh))
            dK = self._merge(torch.matmul(dS.transpose(-1, -2), qh))
            del Pd, dS, dPd, dOh
            x = blk["x"]
            for n, dX in (("Wq", dQ), ("Wk", dK), ("Wv", dV)):
                G[f"b{k}.{n}"].copy_(mm(dX.t(), x, torch.float32))
                dy.add_(mm(dX, self.S[f"b{k}.{n}"], torch.float32))
            a["blocks"][k] = None
