"""Oracle: rotary position embedding (RoPE) with optional YaRN scaling, fp64.

TEST INFRASTRUCTURE ONLY (like all of oracle/): imported by tests/, never by the
product path.

PAPER.md Appendix A: RoPE rotates the half-split pairs
(x[i], x[i + d/2]) of a query / key at position n by the angle n * theta_i,
theta_i = base^(-2i/d), i < d/2 — the form whose dot products P:616-619 expand.
P:339: Qwen2.5-3B is extended from 32K to 512K with YaRN, scaling factor 32.

Readings (DESIGN.md R-rope):
  * base = 1e6 (Qwen2.5's rope_theta; the paper gives none);
  * YaRN = "NTK-by-parts" of Peng et al. (2023) in its common parametrisation:
    with original context L and factor s, dimensions whose rotation count over L
    exceeds beta_fast (= 32) keep theta_i, those below beta_slow (= 1) use
    theta_i / s, a linear ramp in between (bounds in dimension units:
    d * ln(L / (beta * 2 pi)) / (2 ln base), floored / ceiled); the rotated
    vector is scaled by mscale = 0.1 ln(s) + 1.
  * s = 1: plain RoPE, mscale = 1.

Every function is a direct transcription of those definitions (no fusion).
"""
from __future__ import annotations

import math

import numpy as np


def inv_freq(d: int = 128, base: float = 1e6, yarn_factor: float = 1.0,
             original_max_position: int = 32768, beta_fast: float = 32.0,
             beta_slow: float = 1.0):
    """theta_i for i < d/2 (fp64) and the YaRN attention scale mscale."""
    i = np.arange(d // 2, dtype=np.float64)
    theta = base ** (-2.0 * i / d)
    if yarn_factor == 1.0:
        return theta, 1.0
    def dim_of(beta):  # dimension index whose wavelength fits L / beta rotations
        return d * math.log(original_max_position / (beta * 2 * math.pi)) / (2 * math.log(base))
    low = max(math.floor(dim_of(beta_fast)), 0)
    high = min(math.ceil(dim_of(beta_slow)), d // 2 - 1)
    if low == high:
        high += 0.001
    ramp = np.clip((i - low) / (high - low), 0.0, 1.0)  # 0: keep theta, 1: theta / s
    theta_yarn = theta * (1.0 - ramp) + (theta / yarn_factor) * ramp
    return theta_yarn, 0.1 * math.log(yarn_factor) + 1.0


def rope(x: np.ndarray, positions: np.ndarray, theta: np.ndarray, mscale: float = 1.0,
         inverse: bool = False) -> np.ndarray:
    """x: [T][H][d] at absolute token positions [T]; returns mscale * R(n) x (or the
    transpose rotation R(-n) when inverse, i.e. the backward map of the forward)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    h = d // 2
    ang = np.asarray(positions, dtype=np.float64)[:, None] * theta[None, :]  # [T][d/2]
    if inverse:
        ang = -ang
    c = np.cos(ang)[:, None, :]
    s = np.sin(ang)[:, None, :]
    lo, hi = x[..., :h], x[..., h:]
    out = np.empty_like(x)
    out[..., :h] = lo * c - hi * s
    out[..., h:] = hi * c + lo * s
    return mscale * out
