"""DeepSpeech2-shaped bidirectional LSTM stack on the Echo ABI (BASELINE.json configs[2]).

PAPER.md §6.3.1 (lines 946-953); reading R21: input x [T,B,F] stands in for the conv front-end,
5 bidirectional LSTM layers whose two directions are concatenated (applied as split FCs, no concat
buffer), a per-frame linear layer to 29 classes and mean softmax cross-entropy.  Each direction of
each layer is an LSTMLayer (the reverse one processes t = T-1..0), so the hot path is a1/a2/a3.

STASH keeps every LSTM feature map (gates, c, tanh c, h); RECOMPUTE (Echo's plan) keeps the gates
and regenerates the c-chain, tanh(c) and h — including the layer outputs the layer above and the
output FC read, whose weight gradients are therefore deferred until the regenerating backward
(the dead-node FC of PAPER.md:672).

mirror=True runs the prior-work Mirror plan (estimator strategy "mirror"):
every cell keeps its separate FC outputs (input projection(s) and h_{t-1} W_h^T) and h_t, the
output layer keeps its two FC outputs and the labels instead of the CE probabilities (the CE is
mirrored and re-run in the backward).  PAPER.md:951 reports that on DS2 this plan needs MORE
memory than the Baseline; the GPU stash bytes equal the estimator's for all three plans.
"""
from __future__ import annotations

import numpy as np
import torch

from . import abi, probe
from .gemm import mm, addmm_, colsum as _colsum
from .lstm import LSTMLayer, TORCH_DTYPE
from synth.data import ds2_param_shapes


class DS2Model(probe.GraphStep):
    def __init__(self, cfg, dtype=abi.FP32, mode=abi.RECOMPUTE, device="cuda", mirror=False):
        abi.load()
        if mirror and mode != abi.RECOMPUTE:
            raise ValueError("the Mirror plan runs the kernels in RECOMPUTE mode")
        self.cfg, self.dtype, self.mode, self.mirror = cfg, dtype, mode, bool(mirror)
        self.sd = TORCH_DTYPE[dtype]
        self.device = torch.device(device)
        self.shapes = ds2_param_shapes(cfg)
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
        T, B, H = cfg.T, cfg.B, cfg.H
        self.x = torch.zeros(T, B, cfg.F, dtype=self.sd, device=self.device)
        self.labels = torch.zeros(T * B, dtype=torch.int64, device=self.device)
        self.zero_h = torch.zeros(B, H, dtype=self.sd, device=self.device)
        self.zero_c = torch.zeros(B, H, dtype=torch.float32, device=self.device)
        self.loss = torch.zeros((), dtype=torch.float32, device=self.device)
        self.stash = {}
        self.grad_hook = None
        # the two directions of a layer are independent recurrences: the reverse one runs on a side
        # stream (a parallel branch of the step's CUDA graph), joined before anything reads both
        self.side = torch.cuda.Stream(device=self.device)

    def load_params(self, params):
        for name, _ in self.shapes:
            self.P[name].copy_(torch.from_numpy(np.asarray(params[name], np.float32)))
        if self.sflat is not self.master:
            self.sflat.copy_(self.master)

    def upload_batch(self, batch):
        x = batch["x"] if isinstance(batch["x"], torch.Tensor) else torch.from_numpy(np.ascontiguousarray(batch["x"]))
        lab = batch["labels"] if isinstance(batch["labels"], torch.Tensor) else torch.from_numpy(batch["labels"])
        self.x.copy_(x.to(self.sd), non_blocking=True)
        self.labels.copy_(lab.reshape(-1), non_blocking=True)

    def input_bytes(self):
        return self.x.numel() * self.x.element_size() + self.labels.numel() * 8

    def grads_numpy(self):
        return {k: v.detach().double().cpu().numpy() for k, v in self.G.items()}

    def stash_bytes(self):
        seen, total = set(), 0
        for t in self.stash.values():
            key = (t.data_ptr(), t.numel())
            if key not in seen:
                seen.add(key)
                total += t.numel() * t.element_size()
        return total

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

    def _both(self, fw, bw):
        """Run fw() on the current stream and bw() on the side stream; join; return both results."""
        cur = torch.cuda.current_stream(self.device)
        self.side.wait_stream(cur)
        r_fw = fw()
        with torch.cuda.stream(self.side):
            r_bw = bw()
        cur.wait_stream(self.side)
        return r_fw, r_bw

    def _inputs(self, l, low):
        """(X_i, W_i) input projections of layer l for one direction's Wx."""
        H = self.cfg.H
        return lambda W: [(self.x, W)] if l == 0 else [(low[0], W[:, :H]), (low[1], W[:, H:])]

    def _forward(self):
        c, sd, dev, md = self.cfg, self.sd, self.device, self.mode
        T, B, H, V = c.T, c.B, c.H, c.classes
        layers = []
        low = None
        for l in range(c.layers):
            pair = [LSTMLayer(T, B, H, self.dtype, md, dev, reverse=rev, mirror=self.mirror) for rev in (False, True)]

            def run(d, L, l=l, low=low):
                Wx = self.S[f"l{l}.{d}.Wx"]
                ins = [(self.x, Wx)] if l == 0 else [(low[0].h, Wx[:, :H]), (low[1].h, Wx[:, H:])]
                L.forward_multi(ins, self.S[f"l{l}.{d}.Wh"], self.P[f"l{l}.{d}.b"], self.zero_h, self.zero_c)

            self._both(lambda: run("fw", pair[0]), lambda: run("bw", pair[1]))
            if md == abi.RECOMPUTE and not self.mirror and low is not None:
                low[0].h = low[1].h = None                    # lower outputs only fed the input FCs
            layers.append(pair)
            low = pair
        N = T * B
        Wo = self.S["out.W"]
        logits = mm(low[0].h.reshape(N, H), Wo[:, :H].t(), torch.float32)
        if self.mirror:                                       # the two FC outputs are kept; the add + CE mirrored
            lg_b = mm(low[1].h.reshape(N, H), Wo[:, H:].t(), torch.float32)
            lg_a, logits = logits, logits + lg_b
        else:
            logits.add_(mm(low[1].h.reshape(N, H), Wo[:, H:].t(), torch.float32))
        if md == abi.RECOMPUTE and not self.mirror:
            low[0].h = low[1].h = None
        row_loss = torch.empty(N, dtype=torch.float32, device=dev)
        abi.echo_xent_fwd_bwd(N, V, logits, self.P["out.b"], self.labels, row_loss, None)   # in place -> dlogits
        torch.div(row_loss.sum(), N, out=self.loss)
        if self.mirror:
            del logits
            reg = {"x": self.x, "h0": self.zero_h, "c0": self.zero_c, "labels": self.labels, "logits_a": lg_a,
                   "logits_b": lg_b}
        else:
            reg = {"x": self.x, "h0": self.zero_h, "c0": self.zero_c, "ce_probs": logits}
        for l, pair in enumerate(layers):
            for d, L in zip(("fw", "bw"), pair):
                for k, t in L.stash_views().items():
                    reg[f"l{l}.{d}.{k}"] = t
        self.stash = reg
        if self.mirror:
            return {"layers": layers, "logits_ab": (lg_a, lg_b)}
        return {"layers": layers, "dlogits": logits}

    def _backward(self, a):
        c, sd = self.cfg, self.sd
        T, B, H = c.T, c.B, c.H
        N = T * B
        G = self.G
        self.gflat.zero_()
        if self.mirror:                                       # re-run the mirrored add + CE (same kernels)
            lg_a, lg_b = a.pop("logits_ab")
            dlog = lg_a + lg_b
            del lg_a, lg_b
            row_loss = torch.empty(N, dtype=torch.float32, device=self.device)
            abi.echo_xent_fwd_bwd(N, c.classes, dlog, self.P["out.b"], self.labels, row_loss, None)
            del row_loss
        else:
            dlog = a["dlogits"]
        dlog_s = dlog if sd == torch.float32 else dlog.to(sd)
        G["out.b"].copy_(_colsum(dlog))
        Wo = self.S["out.W"]
        dH = [mm(dlog_s, Wo[:, :H], torch.float32).view(T, B, H), mm(dlog_s, Wo[:, H:], torch.float32).view(T, B, H)]
        layers = a["layers"]
        above = None                                          # (layer pair, its weights) awaiting input dW
        for l in reversed(range(c.layers)):
            pair = layers[l]

            def run(j, l=l, pair=pair, dH=dH):
                d = ("fw", "bw")[j]
                Wx = self.S[f"l{l}.{d}.Wx"]
                ins = [(None, Wx)] if l == 0 else [(None, Wx[:, :H]), (None, Wx[:, H:])]
                return pair[j].backward_multi(ins, self.S[f"l{l}.{d}.Wh"], dH[j], need_dX=l > 0, need_dW=False,
                                              release=False)

            rs = self._both(lambda: run(0), lambda: run(1))
            dX = None
            for d, r in zip(("fw", "bw"), rs):                  # joined: combine in fixed order
                G[f"l{l}.{d}.Wh"].copy_(r["dWh"])
                G[f"l{l}.{d}.b"].copy_(r["db"])
                if l > 0:
                    dX = r["dX"] if dX is None else [dX[0].add_(r["dX"][0]), dX[1].add_(r["dX"][1])]
            del rs
            outs = [pair[0].h_time(), pair[1].h_time()]         # stashed, or regenerated by a3
            if above is None:                                  # output FC (deferred dW, Eq. 2)
                G["out.W"][:, :H].copy_(mm(dlog_s.t(), outs[0].reshape(N, H), torch.float32))
                G["out.W"][:, H:].copy_(mm(dlog_s.t(), outs[1].reshape(N, H), torch.float32))
            else:
                lu = l + 1
                for d, U in zip(("fw", "bw"), above):
                    dW = U.input_weight_grads(outs)
                    G[f"l{lu}.{d}.Wx"][:, :H].copy_(dW[0])
                    G[f"l{lu}.{d}.Wx"][:, H:].copy_(dW[1])
                    U.release_backward()
                    U.gates = U.parts = None
            del outs
            above = pair
            dH = dX
        for d, U in zip(("fw", "bw"), above):
            G[f"l0.{d}.Wx"].copy_(U.input_weight_grads([self.x])[0])
            U.release_backward()
        a["layers"] = None
