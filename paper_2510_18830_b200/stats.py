"""Work accounting for reports (host-side, closed form over the index lists).

Activated (n, m) pairs of one head — the unit of the FLOP counts in DESIGN.md §5:
  slash part: offset o covers nb - o block pairs, 64*64 pairs each, except the
              diagonal (o = 0) whose causal half has 64*65/2 = 2080 pairs;
  bar part:   column m (block b) is a bar for every later query block g with
              g - b not a selected offset: 64 pairs per such block.
FLOPs: forward 4 d per pair (QK^T, PV), backward 10 d per pair (QK^T recompute,
dO V^T, P^T dO, dS^T Q, dS K).
"""
from __future__ import annotations

import numpy as np

BLOCK = 64


def pairs_per_head(i_v, i_s, seq_len: int, block: int = BLOCK) -> np.ndarray:
    nb = seq_len // block
    out = []
    for iv, is_ in zip(i_v, i_s):
        offs = np.sort(np.asarray(is_, np.int64))
        offs = offs[offs < nb]
        slash = int(np.sum(np.where(offs == 0, 2080 * nb, (nb - offs) * block * block)))
        pos = offs[offs >= 1]
        b = np.asarray(iv, np.int64) // block
        room = nb - 1 - b
        covered = np.searchsorted(pos, room, side="right")
        bars = int(np.sum(room - covered)) * block
        out.append(slash + bars)
    return np.array(out, np.int64)


def causal_pairs(seq_len: int) -> int:
    return seq_len * (seq_len + 1) // 2


def density(i_v, i_s, seq_len: int) -> float:
    p = pairs_per_head(i_v, i_s, seq_len)
    return float(p.sum()) / (len(p) * causal_pairs(seq_len))


def flops(n_pairs: int, d: int = 128) -> dict:
    return {"fwd": 4 * d * n_pairs, "bwd": 10 * d * n_pairs}
