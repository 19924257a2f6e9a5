"""Helpers shared by the -m gpu parity tests (inputs via synth/, references via oracle/)."""
from __future__ import annotations

import numpy as np
import torch

from synth.generator import bf16_bits_to_f32


def to_dev_bf16(bits: np.ndarray) -> torch.Tensor:
    """uint16 bf16 bit patterns -> CUDA bf16 tensor (exact)."""
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def f64(bits: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(bits).astype(np.float64)


def normwise_err(got: np.ndarray, ref: np.ndarray, head_axis: int) -> float:
    """Reading R20: per (tensor, head) max|x - ref| / max|ref|; returns the max over heads."""
    got = np.moveaxis(got, head_axis, 0)
    ref = np.moveaxis(ref, head_axis, 0)
    out = 0.0
    for h in range(ref.shape[0]):
        den = np.max(np.abs(ref[h]))
        num = np.max(np.abs(got[h] - ref[h]))
        out = max(out, num / den if den > 0 else num)
    return out


def random_index(S: int, Hq: int, seed: int, n_off: int, n_col: int):
    """Random (i_v, i_s) with the forced members 0 / 0 (reading R7)."""
    r = np.random.default_rng(seed)
    nb = S // 64
    iv = [np.unique(np.r_[0, r.choice(S, min(n_col, S), replace=False)]).astype(np.int32)
          for _ in range(Hq)]
    is_ = [np.unique(np.r_[0, r.choice(nb, min(n_off, nb), replace=False)]).astype(np.int32)
           for _ in range(Hq)]
    return iv, is_


def p99_rel(got: np.ndarray, ref: np.ndarray, floor: float = 1e-2) -> float:
    """Elementwise relative error |x - ref| / |ref|, 99th percentile over the entries with
    |ref| >= floor * max|ref| (reported next to R20's normwise error; near-zero entries
    make an elementwise relative error meaningless)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    sel = np.abs(ref) >= floor * np.max(np.abs(ref))
    if not sel.any():
        return 0.0
    return float(np.percentile(np.abs(got[sel] - ref[sel]) / np.abs(ref[sel]), 99))
