"""Workload shapes (BASELINE.json `configs`).

C1  tiny      : 1-layer LSTM (hidden 16, batch 2, seq 4) + MLP attention over 4 source positions
C2  NMT       : Sockeye-style 2+2-layer LSTM NMT, hidden 512, MLP attention, batch 128, seq 50
C3  DS2       : 5 bidirectional LSTM layers, hidden 800, 400 frames, batch 32
C4  TX        : Transformer-base attention blocks, d_model 512, 8 heads, seq 256
C5  NMT-OOM   : C2 shapes with a per-GPU batch that OOMs under stashing
"""
from __future__ import annotations

from dataclasses import dataclass, asdict, replace


@dataclass(frozen=True)
class NMTConfig:
    """Encoder-attention-decoder NMT (§2, Fig. 2)."""
    name: str
    B: int          # batch per GPU
    Ts: int         # source length
    Td: int         # target length
    E: int          # embedding width
    H: int          # LSTM hidden
    A: int          # attention hidden (MLP score width)
    V: int          # vocabulary (src = tgt), reading R17
    enc_layers: int
    dec_layers: int
    dropout: float = 0.0  # embedding dropout rate (reading R31; 0 = none, the C1/C2 configs)
    dropout_hidden: float = 0.0  # inter-layer LSTM output and attention-hidden dropout (reading R33)

    def hidden_drop_sites(self) -> int:
        """Philox sites of reading R33: encoder l -> l+1, decoder l -> l+1, attention hidden -> output."""
        return (self.enc_layers - 1) + (self.dec_layers - 1) + 1 if self.dropout_hidden > 0 else 0

    @property
    def Hk(self) -> int:  # key / value width = encoder hidden
        return self.H

    def as_dict(self):
        d = asdict(self)
        d["Hk"] = self.Hk
        return d

    def with_batch(self, B: int) -> "NMTConfig":
        return replace(self, B=B)


@dataclass(frozen=True)
class DS2Config:
    """DeepSpeech2-shaped stacked bidirectional LSTM (§6.3.1)."""
    name: str
    B: int
    T: int
    F: int          # layer-1 input width (stands in for the conv front-end, reading R21)
    H: int
    layers: int
    classes: int = 29


@dataclass(frozen=True)
class TXConfig:
    """Transformer-base attention blocks (§6.3.2)."""
    name: str
    B: int
    L: int          # sequence length
    d_model: int
    heads: int
    blocks: int
    dropout_p: float = 0.1


C1 = NMTConfig("C1-tiny", B=2, Ts=4, Td=4, E=16, H=16, A=16, V=32, enc_layers=1, dec_layers=1)
C2 = NMTConfig("C2-nmt", B=128, Ts=50, Td=50, E=512, H=512, A=512, V=8192, enc_layers=2, dec_layers=2)
SMALL_NMT = NMTConfig("small-nmt", B=4, Ts=8, Td=8, E=32, H=32, A=32, V=64, enc_layers=2, dec_layers=2)
SMALL_NMT_DROP = NMTConfig("small-nmt-drop", B=4, Ts=8, Td=8, E=32, H=32, A=32, V=64, enc_layers=2, dec_layers=2,
                           dropout=0.1)
C3 = DS2Config("C3-ds2", B=32, T=400, F=1600, H=800, layers=5)
C4 = TXConfig("C4-tx", B=64, L=256, d_model=512, heads=8, blocks=6)
SMALL_TX = TXConfig("small-tx", B=2, L=24, d_model=32, heads=4, blocks=2, dropout_p=0.1)
SMALL_DS2 = DS2Config("small-ds2", B=3, T=7, F=24, H=16, layers=2)

NMT_CONFIGS = {c.name: c for c in (C1, SMALL_NMT, C2)}
