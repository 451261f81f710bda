"""Sockeye-style LSTM NMT training step on the Echo ABI (BASELINE.json configs[1]).

Model (§2, Fig. 2; readings R3, R6, R7, R10):
  encoder  : emb_src -> enc_layers x LSTM; H_s = top-layer h for all source steps
  attention: Kp = H_s W_k^T + b_q (bias folded, once); per target step qp_t = h_t W_q^T;
             MLP score, masked softmax, context (libecho a5 / a6)
  decoder  : dec_layers x LSTM with input feeding x_t = [emb(y_{t-1}); a_{t-1}],
             a_t = tanh(W_cc ctx_t + W_ch h_t)
  output   : logits = a W_o^T + b_o, mean softmax cross-entropy over B*Td tokens
  update   : plain SGD on an fp32 master copy (flat buffers; flat fp32 gradient for the allreduce)

Hot path (libecho): LSTM a1/a2/a3 and attention a5/a6.  FC contractions are cuBLAS
(torch) and outside the hot path; embedding gather/scatter, the attention-hidden tanh
and the CE are glue, identical in both modes.

Memory modes (echo_mode): STASH is the paper's Baseline (keep every feature map);
RECOMPUTE is Echo's plan (DESIGN.md tables T3/T4): per LSTM layer only the gates
are kept, the c-chain / tanh(c) / h are regenerated in the backward pass, and the
attention keeps nothing but its inputs (Kp, H_s, qp is recomputed from h).
Activation buffers are allocated per step, so torch's allocator statistics measure
the real activation footprint.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import abi, probe
from .gemm import mm, mm_out, addmm_, tf32, colsum as _colsum
from .lstm import LSTMLayer, TORCH_DTYPE
from synth.data import nmt_param_shapes


def _det_index_add(dst, idx, src):
    """dst.index_add_(0, idx, src) with torch's deterministic (sort-based, atomic-free) path."""
    prev = torch.are_deterministic_algorithms_enabled()
    torch.use_deterministic_algorithms(True, warn_only=True)
    try:
        dst.index_add_(0, idx, src)
    finally:
        torch.use_deterministic_algorithms(prev, warn_only=True)


class NMTModel(probe.GraphStep):
    def __init__(self, cfg, dtype=abi.FP32, mode=abi.RECOMPUTE, device="cuda"):
        abi.load()
        self.cfg = cfg
        self.dtype, self.mode = dtype, mode
        self.sd = TORCH_DTYPE[dtype]
        self.device = torch.device(device)
        self.shapes = nmt_param_shapes(cfg)
        n = sum(int(np.prod(s)) for _, s in self.shapes)
        self.numel = n
        self.master = torch.zeros(n, dtype=torch.float32, device=self.device)   # fp32 master weights
        self.gflat = torch.zeros(n, dtype=torch.float32, device=self.device)    # flat fp32 gradients
        self.sflat = self.master if dtype == abi.FP32 else torch.zeros(n, dtype=self.sd, device=self.device)
        self.P, self.G, self.S = {}, {}, {}
        off = 0
        for name, shape in self.shapes:
            k = int(np.prod(shape))
            self.P[name] = self.master[off:off + k].view(shape)
            self.G[name] = self.gflat[off:off + k].view(shape)
            self.S[name] = self.sflat[off:off + k].view(shape)
            off += k
        B, H = cfg.B, cfg.H
        self.zero_h = torch.zeros(B, H, dtype=self.sd, device=self.device)
        self.zero_c = torch.zeros(B, H, dtype=torch.float32, device=self.device)
        self.inputs = {
            "src": torch.zeros(cfg.B, cfg.Ts, dtype=torch.int64, device=self.device),
            "tgt_in": torch.zeros(cfg.B, cfg.Td, dtype=torch.int64, device=self.device),
            "tgt_out": torch.zeros(cfg.B, cfg.Td, dtype=torch.int64, device=self.device),
            "src_len": torch.full((cfg.B,), cfg.Ts, dtype=torch.int32, device=self.device),
        }
        self.loss = torch.zeros((), dtype=torch.float32, device=self.device)
        self.stash = {}
        self.grad_hook = None          # e.g. dp.allreduce_mean_ (called on the flat fp32 gradient)

    # ------------------------------------------------------------ parameters / io
    def w(self, name):
        """Weight in storage dtype (biases are always read from the fp32 master)."""
        return self.S[name]

    def load_params(self, params):
        for name, _ in self.shapes:
            self.P[name].copy_(torch.from_numpy(np.asarray(params[name], np.float32)))
        if self.sflat is not self.master:
            self.sflat.copy_(self.master)

    def upload_batch(self, batch, pinned=None):
        """Copy a host batch into the static device input buffers (non_blocking from pinned memory)."""
        for k in ("src", "tgt_in", "tgt_out", "src_len"):
            src = batch[k] if isinstance(batch[k], torch.Tensor) else torch.from_numpy(np.ascontiguousarray(batch[k]))
            self.inputs[k].copy_(src.to(self.inputs[k].dtype), non_blocking=True)
        return self.inputs

    def grads_numpy(self):
        return {k: v.detach().double().cpu().numpy() for k, v in self.G.items()}

    def input_bytes(self):
        return sum(t.numel() * t.element_size() for t in self.inputs.values())

    # ------------------------------------------------------------ encoder wavefront helpers
    def _a6_deferred(self):
        """Deferred dKp / dH_s accumulation (echo_attn_bwd_deferred + echo_attn_bwd_finish; bit-
        identical results) instead of the per-step read-modify-write?  Opt-in (ECHO_A6_DEFERRED=1):
        it removes 2/3 of a6's HBM bytes, but a6 is latency/issue-bound, not HBM-bound, at both ends
        of the batch range (CUPTI, C5 bf16: a6 3.14 -> 2.47 ms/step, plus 28 + 7 ms of finish
        passes = no net gain; C2: equal within noise), so the per-step path stays the default."""
        return os.environ.get("ECHO_A6_DEFERRED", "0") == "1"

    def _chunks(self, T):
        """Wavefront chunk boundaries over the encoder's time axis.  Measured on C2 (bench, CUDA
        graph): fp32 29.9 -> 28.1 ms/step with 5 chunks (its SIMT GEMMs leave most SMs idle, so two
        layers' recurrences overlap well); bf16 8.91 -> 9.09 ms (tensor-core GEMMs already fill the
        GPU; the cross-stream waits cost more than the overlap gains) -> 1 chunk (back to back)."""
        n = int(os.environ.get("ECHO_ENC_CHUNKS", "5" if self.sd == torch.float32 else "1"))
        n = max(1, min(n, T))
        return [(T * i) // n for i in range(n + 1)]

    def _layer_streams(self, n):
        """[current stream] + n-1 side streams (created once) for per-layer wavefronts."""
        if not hasattr(self, "_side") or len(self._side) < n - 1:
            self._side = [torch.cuda.Stream(device=self.device) for _ in range(n - 1)]
        return [torch.cuda.current_stream(self.device)] + self._side[: n - 1]

    # ------------------------------------------------------------ one training step
    def train_step(self, inputs=None, lr=0.1):
        """Forward + backward + SGD.  Returns the loss as a float (one D2H read)."""
        self.step(lr)
        return float(self.loss.item())

    def step(self, lr=0.1):
        """Device-only step (no host sync); the loss stays in self.loss."""
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

    # ------------------------------------------------------------ forward
    def _forward(self):
        cfg, sd, dev, md = self.cfg, self.sd, self.device, self.mode
        B, Ts, Td, E, H, A, V = cfg.B, cfg.Ts, cfg.Td, cfg.E, cfg.H, cfg.A, cfg.V
        inp = self.inputs
        a = {}
        # encoder ------------------------------------------------------------
        X0 = self.w("emb_src").index_select(0, inp["src"].t().reshape(-1)).view(Ts, B, E)
        a["X0"] = X0
        enc = [LSTMLayer(Ts, B, H, self.dtype, md, dev) for _ in range(cfg.enc_layers)]
        # wavefront: layer l runs on its own stream and starts chunk c as soon as layer l-1 finished
        # it (per-chunk events); the layers' recurrences overlap instead of running back to back
        bounds = self._chunks(Ts)
        streams = self._layer_streams(len(enc))
        done = [[torch.cuda.Event() for _ in bounds[:-1]] for _ in enc]
        for st in streams[1:]:
            st.wait_stream(streams[0])
        for l, L in enumerate(enc):
            X = X0 if l == 0 else enc[l - 1].h
            with torch.cuda.stream(streams[l]):
                for c in range(len(bounds) - 1):
                    if l > 0:
                        streams[l].wait_event(done[l - 1][c])
                    L.forward_range(bounds[c], bounds[c + 1], X, self.w(f"enc{l}.Wx"), self.w(f"enc{l}.Wh"),
                                    self.P[f"enc{l}.b"], self.zero_h, self.zero_c)
                    done[l][c].record(streams[l])
        for st in streams[1:]:
            streams[0].wait_stream(st)
        if md == abi.RECOMPUTE:
            for L in enc[:-1]:
                L.h = None                                       # lower layers' outputs only fed the FCs
            a["X0"] = None                                       # embeddings: recomputed from the tokens
        a["enc"] = enc
        Hs = enc[-1].h                                           # [Ts,B,H] s-major source hidden state
        a["Hs"] = Hs
        Kp = torch.empty(Ts, B, A, dtype=sd, device=dev)        # Kp = Hs W_k^T + b_q (bias folded, R3)
        torch.addmm(self.P["att.bq"].to(sd), Hs.view(Ts * B, H), self.w("att.Wk").t(), out=Kp.view(Ts * B, A))
        a["Kp"] = Kp
        adesc = abi.AttnDesc(B, Ts, A, H, self.dtype, md, A, B * A, H, B * H)
        a["adesc"] = adesc
        # decoder ------------------------------------------------------------
        EmbT = self.w("emb_tgt").index_select(0, inp["tgt_in"].t().reshape(-1)).view(Td, B, E)
        a["EmbT"] = EmbT
        dec = [LSTMLayer(Td, B, H, self.dtype, md, dev, h_ring=True) for _ in range(cfg.dec_layers)]
        for L in dec:
            L.h0, L.c0 = self.zero_h, self.zero_c
        Wx0 = self.w("dec0.Wx")
        mm_out(dec[0].gates.view(Td * B, 4 * H), EmbT.view(Td * B, E), Wx0[:, :E].t())
        if md == abi.RECOMPUTE:
            a["EmbT"] = None
            del EmbT
        Aall = torch.empty(Td, B, H, dtype=sd, device=dev)       # attention hidden a_t (stash, both modes)
        a["Aall"] = Aall
        if md == abi.STASH:
            a["E_st"] = torch.empty(Td, B, Ts, A, dtype=sd, device=dev)
            a["al_st"] = torch.empty(Td, B, Ts, dtype=torch.float32, device=dev)
            a["ctx_st"] = torch.empty(Td, B, H, dtype=sd, device=dev)
            qp_buf = torch.empty(B, A, dtype=sd, device=dev)
        else:
            a["qp_st"] = torch.empty(Td, B, A, dtype=sd, device=dev)   # Echo plan T4: qp_t stashed
            ctx_tmp = torch.empty(B, H, dtype=sd, device=dev)
        pre = torch.empty(B, H, dtype=sd, device=dev)
        WaT = Wx0[:, E:].t()
        Wq, Wcc, Wch, v = self.w("att.Wq"), self.w("att.Wcc"), self.w("att.Wch"), self.w("att.v")
        sl = inp["src_len"]
        for t in range(Td):
            for l, L in enumerate(dec):
                if l == 0:
                    if t > 0:
                        addmm_(L.gates[t], Aall[t - 1], WaT)     # input feeding: a_{t-1}
                else:
                    mm_out(L.gates[t], dec[l - 1].h_slot(t), self.w(f"dec{l}.Wx").t())
                if t > 0:
                    addmm_(L.gates[t], L.h_prev(t), self.w(f"dec{l}.Wh").t())
                L.fwd_step(t, self.P[f"dec{l}.b"])
            q = dec[-1].h_slot(t)
            qp = qp_buf if md == abi.STASH else a["qp_st"][t]
            mm_out(qp, q, Wq.t())
            with probe.timed("attn_fwd"):
                if md == abi.STASH:
                    ctx = a["ctx_st"][t]
                    abi.echo_attn_fwd(adesc, qp, Kp, v, Hs, sl, ctx, a["E_st"][t], a["al_st"][t])
                else:
                    ctx = ctx_tmp
                    abi.echo_attn_fwd(adesc, qp, Kp, v, Hs, sl, ctx, None, None)
            mm_out(pre, ctx, Wcc.t())
            addmm_(pre, q, Wch.t())
            torch.tanh(pre, out=Aall[t])
        a["dec"] = dec
        if md == abi.RECOMPUTE:                                  # H_s is mirrored (Echo plan): regenerated
            a["Hs"] = None                                       # by the top encoder layer's scan
            enc[-1].h = None
            Hs = None
        else:                                                    # STASH reads the stashed tanh inputs, not Kp
            a["Kp"] = None
            Kp = None
        # output layer + CE; logits are overwritten in place by dlogits (the CE's fp32 feature map)
        N = B * Td
        logits = mm(Aall.view(N, H), self.w("out.Wo").t(), torch.float32)
        y = inp["tgt_out"].t().reshape(-1)
        row_loss = torch.empty(N, dtype=torch.float32, device=dev)
        # fused bias + softmax-CE: logits become dLoss/dlogits in place (the kept fp32 feature map;
        # the storage-dtype copy for the backward GEMMs is made in the backward, not kept)
        abi.echo_xent_fwd_bwd(N, V, logits, self.P["out.bo"], y, row_loss, None)
        torch.div(row_loss.sum(), N, out=self.loss)
        a["dlogits"] = logits
        self.stash = self._stash_registry(a)
        return a

    def _stash_registry(self, a):
        """Every tensor kept across the forward->backward boundary for the backward pass."""
        inp = self.inputs
        reg = {"src_tokens": inp["src"], "tgt_tokens": inp["tgt_in"], "src_len": inp["src_len"], "h0": self.zero_h,
               "c0": self.zero_c, "a_t": a["Aall"], "ce_probs": a["dlogits"]}
        for k in ("X0", "EmbT", "Hs", "Kp"):
            if a.get(k) is not None:
                reg[k] = a[k]
        for l, L in enumerate(a["enc"]):
            for k, t in L.stash_views().items():
                reg[f"enc{l}.{k}"] = t
        for l, L in enumerate(a["dec"]):
            for k, t in L.stash_views().items():
                reg[f"dec{l}.{k}"] = t
        for k in ("E_st", "al_st", "ctx_st", "qp_st"):
            if k in a:
                reg[k] = a[k]
        return reg

    def stash_bytes(self):
        seen, total = set(), 0
        for t in self.stash.values():
            key = (t.data_ptr(), t.numel())
            if key in seen:
                continue
            seen.add(key)
            total += t.numel() * t.element_size()
        return total

    # ------------------------------------------------------------ backward
    def _gemm_into(self, out, x, y):
        """out (an fp32 gradient view) = x @ y."""
        if x.dtype == torch.float32 and out.is_contiguous():
            mm_out(out, x, y)
        else:
            out.copy_(mm(x, y, torch.float32))

    def _to_s(self, x):
        return x if x.dtype == self.sd else x.to(self.sd)

    def _backward(self, a):
        cfg, sd, dev, md = self.cfg, self.sd, self.device, self.mode
        B, Ts, Td, E, H, A, V = cfg.B, cfg.Ts, cfg.Td, cfg.E, cfg.H, cfg.A, cfg.V
        N = B * Td
        G = self.G
        gi = self._gemm_into
        self.gflat.zero_()
        Aall = a["Aall"]
        # output layer (Eq. 2: needs its input a_t and W_o, not its output)
        dlog_s = self._to_s(a["dlogits"])
        gi(G["out.Wo"], dlog_s.t(), Aall.view(N, H))
        G["out.bo"].copy_(_colsum(a["dlogits"]))
        dAout = mm(dlog_s, self.w("out.Wo"), torch.float32).view(Td, B, H)    # dLoss/da_t (+ carry added below)
        del dlog_s
        a["dlogits"] = None
        self.stash.pop("ce_probs", None)
        # decoder, reverse time ----------------------------------------------------------
        dec = a["dec"]
        Ld = len(dec)
        enc = a["enc"]
        if md == abi.RECOMPUTE:                                  # mirrored H_s: top encoder layer's a2 scan
            Hs = enc[-1].prepare_backward(regen_h=True)          # also regenerates its h_1..h_Ts
        else:
            Hs = a["Hs"]
        for L in dec:
            L.prepare_backward()                                 # RECOMPUTE: a2 c-scan per layer
        dHdec = [torch.zeros(Td, B, H, dtype=torch.float32, device=dev) for _ in range(Ld)]
        dcs = [torch.zeros(B, H, dtype=torch.float32, device=dev) for _ in range(Ld)]
        dPRE = torch.empty(Td, B, H, dtype=torch.float32, device=dev)
        dQP = torch.empty(Td, B, A, dtype=torch.float32, device=dev)
        deferred = self._a6_deferred()
        if deferred:                                             # dKp / dH_s accumulated once after the loop
            dKp = torch.empty(Ts, B, A, dtype=torch.float32, device=dev)
            dHs = torch.empty(Ts, B, H, dtype=torch.float32, device=dev)
            ds_all = torch.empty(Td, B, Ts, dtype=torch.float32, device=dev)
            al_all = a["al_st"] if md == abi.STASH else torch.empty(Td, B, Ts, dtype=torch.float32, device=dev)
            dctx_all = torch.empty(Td, B, H, dtype=torch.float32, device=dev)
        else:
            dKp = torch.zeros(Ts, B, A, dtype=torch.float32, device=dev)
            dHs = torch.zeros(Ts, B, H, dtype=torch.float32, device=dev)
            dctx1 = torch.empty(B, H, dtype=torch.float32, device=dev)
        dv_part = torch.zeros(B, A, dtype=torch.float32, device=dev)
        ctx_all = a["ctx_st"] if md == abi.STASH else torch.empty(Td, B, H, dtype=sd, device=dev)
        Wx0 = self.w("dec0.Wx")
        WxA = Wx0[:, E:]
        Wq, Wcc, Wch, v = self.w("att.Wq"), self.w("att.Wcc"), self.w("att.Wch"), self.w("att.v")
        adesc, Kp, sl = a["adesc"], a["Kp"], self.inputs["src_len"]
        # per-step backward-data GEMMs of the attention block use the fp32 master weights, so
        # the fp32 gradient signals dpre / dqp are not rounded to the storage dtype (no-op in fp32)
        Wcc32, Wch32, Wq32 = self.P["att.Wcc"], self.P["att.Wch"], self.P["att.Wq"]
        lowp = sd != torch.float32                               # bf16 storage: TF32 for the fp32 GEMMs
        for t in reversed(range(Td)):
            abi.echo_tanh_bwd(Aall[t], dAout[t], dPRE[t])        # tanh' = 1 - a^2
            top = dHdec[-1][t]
            dctx = dctx_all[t] if deferred else dctx1
            with tf32(lowp):
                mm_out(dctx, dPRE[t], Wcc32)
                addmm_(top, dPRE[t], Wch32)
            with probe.timed("attn_bwd"):
                st = md == abi.STASH                             # RECOMPUTE: a6 regenerates E, scores, alpha, ctx
                qp_t, Kp_t = (None, None) if st else (a["qp_st"][t], Kp)
                E_t, al_t = (a["E_st"][t], a["al_st"][t]) if st else (None, None)
                creg = None if st else ctx_all[t]
                if deferred:
                    abi.echo_attn_bwd_deferred(adesc, qp_t, Kp_t, v, Hs, sl, E_t, al_t, dctx, dQP[t], dv_part, creg,
                                               ds_all[t], None if st else al_all[t])
                else:
                    abi.echo_attn_bwd(adesc, qp_t, Kp_t, v, Hs, sl, E_t, al_t, dctx, dQP[t], dKp, dHs, dv_part, creg)
            with tf32(lowp):
                addmm_(top, dQP[t], Wq32)
            for l in reversed(range(Ld)):
                L = dec[l]
                L.bwd_step(t, dHdec[l][t], dcs[l])               # a3 (fused recompute in RECOMPUTE)
                dA = L.gates[t]
                if t > 0:
                    addmm_(dHdec[l][t - 1], dA, self.w(f"dec{l}.Wh"))
                if l > 0:
                    addmm_(dHdec[l - 1][t], dA, self.w(f"dec{l}.Wx"))
                elif t > 0:
                    addmm_(dAout[t - 1], dA, WxA)                # input feeding: carry into da_{t-1}
        # deferred weight-gradient GEMMs (their inputs are stashed or were regenerated above).  The
        # gradient operands dpre / dqp are fp32: for bf16 storage the GEMM is run in fp32 on the
        # up-cast activations rather than rounding the gradient to bf16 (no-op for fp32).
        f32 = lambda x: x if x.dtype == torch.float32 else x.float()
        qall = f32(dec[-1].h_for_grad().reshape(N, H))
        dPREs = dPRE.view(N, H)
        with tf32(lowp):
            gi(G["att.Wcc"], dPREs.t(), f32(ctx_all.view(N, H)))
            gi(G["att.Wch"], dPREs.t(), qall)
            gi(G["att.Wq"], dQP.view(N, A).t(), qall)
        abi.echo_attn_dv_reduce(B, A, dv_part, G["att.v"], 0)
        if deferred:
            with probe.timed("attn_bwd_finish"):
                abi.echo_attn_bwd_finish(adesc, Td, None if md == abi.STASH else a["qp_st"], None if md == abi.STASH else Kp,
                                         a["E_st"] if md == abi.STASH else None, v, sl, ds_all, al_all, dctx_all, dKp,
                                         dHs)
            del ds_all, al_all, dctx_all
        del qall
        del dPREs, dPRE, dQP
        for l in range(Ld):
            L = dec[l]
            dAl = L.gates.view(N, 4 * H)
            G[f"dec{l}.b"].copy_(_colsum(dAl))
            hg = L.h_for_grad()
            if Td > 1:
                gi(G[f"dec{l}.Wh"], L.gates[1:].reshape((Td - 1) * B, 4 * H).t(), hg[: Td - 1].reshape((Td - 1) * B, H))
            if l > 0:
                gi(G[f"dec{l}.Wx"], dAl.t(), dec[l - 1].h_for_grad().reshape(N, H))
            else:
                EmbT = a["EmbT"] if md == abi.STASH else \
                    self.w("emb_tgt").index_select(0, self.inputs["tgt_in"].t().reshape(-1))   # recomputed
                gi(G["dec0.Wx"][:, :E], dAl.t(), EmbT.view(N, E))
                del EmbT
                if Td > 1:
                    gi(G["dec0.Wx"][:, E:], L.gates[1:].reshape((Td - 1) * B, 4 * H).t(),
                       Aall[: Td - 1].reshape((Td - 1) * B, H))
                dEmb = mm(dAl, Wx0[:, :E], torch.float32)
                _det_index_add(G["emb_tgt"], self.inputs["tgt_in"].t().reshape(-1), dEmb)
                del dEmb
        for L in dec:
            L.release_backward()
        del dec, dHdec, ctx_all
        a["dec"] = None
        # attention key projection Kp = Hs W_k^T + b_q --------------------------------------
        dKpf = dKp.view(Ts * B, A)
        G["att.bq"].copy_(_colsum(dKpf))
        Hs32 = Hs.reshape(Ts * B, H)
        with tf32(lowp):
            gi(G["att.Wk"], dKpf.t(), Hs32 if Hs32.dtype == torch.float32 else Hs32.float())
            addmm_(dHs.view(Ts * B, H), dKpf, self.P["att.Wk"])
        dKps = None
        del Hs, Hs32
        del dKp, dKpf, dKps
        # encoder, top-down wavefront: layer l (its own stream) runs chunk c of its backward once
        # layer l+1 finished chunk c; dH_l[t] = dA_{l+1}[t] W_x^{l+1} is accumulated per chunk (the
        # recurrent term of a chunk's first step lands first at chunk boundaries: fixed order, both
        # modes).  dW_x of layer l+1 needs this layer's h (stashed or regenerated) ---------------
        Le = len(enc)
        n = Ts * B
        bounds = self._chunks(Ts)
        nch = len(bounds) - 1
        streams = self._layer_streams(Le)                        # [current, side...]; top layer on current
        done = [[torch.cuda.Event() for _ in range(nch)] for _ in range(Le)]
        for st in streams[1:]:                                   # fork after dH_s is complete
            st.wait_stream(streams[0])
        dHl = [None] * Le
        dHl[Le - 1] = dHs
        for l in reversed(range(Le)):
            L = enc[l]
            st = streams[Le - 1 - l]
            with torch.cuda.stream(st):
                L.prepare_backward()
                dc = torch.zeros(B, H, dtype=torch.float32, device=dev)
                Wh = self.w(f"enc{l}.Wh")
                if l < Le - 1:
                    dHl[l] = torch.zeros(Ts, B, H, dtype=torch.float32, device=dev)
                dH = dHl[l]
                for c in reversed(range(nch)):
                    t0, t1 = bounds[c], bounds[c + 1]
                    if l < Le - 1:
                        st.wait_event(done[l + 1][c])
                        up = enc[l + 1]
                        addmm_(dH[t0:t1].view((t1 - t0) * B, H), up.gates[t0:t1].view((t1 - t0) * B, 4 * H),
                               self.w(f"enc{l + 1}.Wx"))
                    for t in reversed(range(t0, t1)):
                        L.bwd_step(t, dH[t], dc)
                        if t > 0:
                            addmm_(dH[t - 1], L.gates[t], Wh)
                    done[l][c].record(st)
        for st in streams[1:]:
            streams[0].wait_stream(st)
        del dHl
        for l in reversed(range(Le)):
            L = enc[l]
            dAl = L.gates.view(n, 4 * H)
            hg = L.h_for_grad()
            G[f"enc{l}.b"].copy_(_colsum(dAl))
            if Ts > 1:
                gi(G[f"enc{l}.Wh"], L.gates[1:].reshape((Ts - 1) * B, 4 * H).t(), hg[: Ts - 1].reshape((Ts - 1) * B, H))
            if l < Le - 1:
                up = enc[l + 1]
                gi(G[f"enc{l + 1}.Wx"], up.gates.view(n, 4 * H).t(), hg.reshape(n, H))
                enc[l + 1] = None
            if l == 0:
                dX = mm(dAl, self.w(f"enc{l}.Wx"), torch.float32).view(Ts, B, -1)
                X0 = a["X0"] if md == abi.STASH else \
                    self.w("emb_src").index_select(0, self.inputs["src"].t().reshape(-1))      # recomputed
                gi(G["enc0.Wx"], dAl.t(), X0.view(n, E))
                del X0
                _det_index_add(G["emb_src"], self.inputs["src"].t().reshape(-1), dX.view(n, E))
                enc[0] = None
            L.release_backward()
        a["enc"] = None
