"""One LSTM layer (one direction) on the Echo ABI: buffers, per-step calls and
sequence drivers.  PAPER.md §2 lines 101-112 (Fig. 1).

Per step the caller's FCs produce gx_t (= x_t W_x^T) and accumulate
h_{t-1} W_h^T into it in place (cuBLAS beta = 1, outside the hot path); the
non-linear block runs in libecho (a1).  Backward: RECOMPUTE regenerates the
c-chain with one scan (a2) and tanh(c), h inside the fused backward step (a3);
STASH reads them from the stash.

Buffers (B, H per step; s = storage dtype):
  gates [T,B,4H] s   stash in BOTH modes (Echo plan, T3); also the
                     gx workspace before a1 and dA after a3 (aliased in place)
  STASH:      c [T,B,H] fp32 (c_1..c_T; slot T is the final state, not a
              feature map), tc [T,B,H] s, h [T,B,H] s
  RECOMPUTE:  c ring [2,B,H] fp32; h [T,B,H] s is the layer OUTPUT (for the
              layer above), not kept by this layer for its backward
  backward transients (RECOMPUTE): c_ws [T,B,H] fp32, h_regen [T,B,H] s
"""
from __future__ import annotations

import torch

from . import abi
from .gemm import mm, addmm_

TORCH_DTYPE = {abi.FP32: torch.float32, abi.BF16: torch.bfloat16}


class LSTMLayer:
    def __init__(self, T, B, H, dtype=abi.FP32, mode=abi.RECOMPUTE, device="cuda", h_ring=False):
        """h_ring: in RECOMPUTE, keep only h_{t-1}, h_t (2-slot ring) because nobody needs the
        whole output sequence after the forward (decoder layers); the encoder keeps [T,B,H]."""
        self.T, self.B, self.H = T, B, H
        self.dtype, self.mode = dtype, mode
        self.sd = TORCH_DTYPE[dtype]
        self.device = device
        self.desc = abi.LstmDesc(B, H, dtype, mode)
        self.gates = torch.empty(T, B, 4 * H, dtype=self.sd, device=device)
        self.h_ring = bool(h_ring) and mode == abi.RECOMPUTE
        self.h = torch.empty(2 if self.h_ring else T, B, H, dtype=self.sd, device=device)
        if mode == abi.STASH:
            self.c = torch.empty(T, B, H, dtype=torch.float32, device=device)
            self.tc = torch.empty(T, B, H, dtype=self.sd, device=device)
        else:
            self.c = torch.empty(2, B, H, dtype=torch.float32, device=device)
            self.tc = None
        self.c_ws = None
        self.h_regen = None
        self.h0 = None
        self.c0 = None

    # ------------------------------------------------------------ accounting
    def stash_views(self):
        """Tensors this layer keeps across the forward->backward boundary for its own backward
        (excluding h0/c0, which the caller owns).  Byte sums are compared with the estimator."""
        if self.mode == abi.STASH:
            return {"gates": self.gates, "c": self.c[: self.T - 1], "tc": self.tc, "h": self.h}
        return {"gates": self.gates}

    # ------------------------------------------------------------ per-step forward (a1)
    def c_slot(self, t):
        return self.c[t] if self.mode == abi.STASH else self.c[t % 2]

    def c_prev(self, t):
        return self.c0 if t == 0 else self.c_slot(t - 1)

    def h_slot(self, t):
        return self.h[t % 2] if self.h_ring else self.h[t]

    def h_prev(self, t):
        return self.h0 if t == 0 else self.h_slot(t - 1)

    def fwd_step(self, t, bias):
        """gates[t] must hold x_t W_x^T + h_{t-1} W_h^T (storage dtype)."""
        abi.echo_lstm_fwd(self.desc, self.gates[t], None, bias, self.c_prev(t), self.gates[t], self.c_slot(t),
                          self.tc[t] if self.mode == abi.STASH else None, self.h_slot(t))

    def c_final(self):
        return self.c_slot(self.T - 1)

    # ------------------------------------------------------------ per-step backward (a2 + a3)
    def prepare_backward(self):
        if self.mode == abi.RECOMPUTE:
            if self.c_ws is None:
                self.c_ws = torch.empty(self.T, self.B, self.H, dtype=torch.float32, device=self.device)
                self.h_regen = torch.empty(self.T, self.B, self.H, dtype=self.sd, device=self.device)
            abi.echo_lstm_cscan(self.desc, self.T, self.gates, self.c0, self.c_ws)

    def release_backward(self):
        self.c_ws = None
        self.h_regen = None

    def bwd_step(self, t, dh_t, dc):
        """dh_t fp32 [B,H] total gradient; dc fp32 [B,H] carry (in/out).  Writes dA_t over gates[t]."""
        if self.mode == abi.STASH:
            abi.echo_lstm_bwd(self.desc, self.gates[t], self.c_prev(t), None, self.tc[t], dh_t, dc, self.gates[t], None)
        else:
            cp = self.c0 if t == 0 else self.c_ws[t - 1]
            abi.echo_lstm_bwd(self.desc, self.gates[t], cp, self.c_ws[t], None, dh_t, dc, self.gates[t],
                              self.h_regen[t])

    def h_for_grad(self):
        """h_1..h_T as needed by the weight-gradient GEMMs (stashed or regenerated)."""
        return self.h if self.mode == abi.STASH else self.h_regen

    # ------------------------------------------------------------ sequence drivers (encoder-style)
    def forward_seq(self, X, Wx, Wh, b, h0, c0):
        """X [T,B,I] s; Wx [4H,I] s; Wh [4H,H] s; b [4H] fp32; h0 [B,H] s; c0 [B,H] fp32.  Returns h [T,B,H]."""
        T, B, H = self.T, self.B, self.H
        self.h0, self.c0 = h0, c0
        torch.mm(X.reshape(T * B, -1), Wx.t(), out=self.gates.view(T * B, 4 * H))
        WhT = Wh.t()
        for t in range(T):
            addmm_(self.gates[t], self.h_prev(t), WhT)
            self.fwd_step(t, b)
        return self.h

    def backward_seq(self, X, Wx, Wh, dH, dcT=None, need_dX=True):
        """dH [T,B,H] fp32 = dLoss/dh_t from above (modified in place: recurrent terms are added).
        Returns dict(dX, dWx, dWh, db, dh0, dc0)."""
        T, B, H = self.T, self.B, self.H
        self.prepare_backward()
        dc = torch.zeros(B, H, dtype=torch.float32, device=self.device) if dcT is None else dcT.clone()
        for t in reversed(range(T)):
            self.bwd_step(t, dH[t], dc)
            if t > 0:
                addmm_(dH[t - 1], self.gates[t], Wh)          # recurrent dh_{t-1} += dA_t W_h
        dA = self.gates.view(T * B, 4 * H)
        hg = self.h_for_grad()
        out = {"dh0": mm(self.gates[0], Wh, out_dtype=torch.float32), "dc0": dc}
        dWh = mm(self.gates[0].t(), self.h0, out_dtype=torch.float32)
        if T > 1:
            addmm_(dWh, self.gates[1:].reshape((T - 1) * B, 4 * H).t(), hg[: T - 1].reshape((T - 1) * B, H))
        out["dWh"] = dWh
        out["dWx"] = mm(dA.t(), X.reshape(T * B, -1), out_dtype=torch.float32)
        out["db"] = dA.float().sum(dim=0)
        if need_dX:
            out["dX"] = mm(dA, Wx, out_dtype=torch.float32).view(T, B, -1)
        self.release_backward()
        return out
