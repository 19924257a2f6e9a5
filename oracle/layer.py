"""Oracle: one Qwen2.5-3B-shaped transformer layer around the VS sparse attention,
fp64 forward and hand-derived backward.

TEST INFRASTRUCTURE ONLY (like all of oracle/): imported by tests/, never by the
product path.

The paper trains Qwen2.5-3B with every attention layer replaced by
the VS sparse attention of Alg. 1; the layer is the standard decoder block
of that model family (reading R-layer in DESIGN.md):

  h1 = RMSNorm(x) * w1                       r = (mean(x^2) + eps)^(-1/2), eps 1e-6
  [q | k | v] = h1 Wqkv^T + bqkv             Hq + 2 Hkv heads of d
  q, k <- RoPE(q, pos), RoPE(k, pos)         oracle/rope.py (Appendix A)
  o = sparse_attention(q, k, v; i_v, i_s)    oracle/attention.py (Alg. 1)
  x2 = x + o Wo^T
  h2 = RMSNorm(x2) * w2
  y = x2 + (silu(h2 Wg^T) * (h2 Wu^T)) Wd^T  SwiGLU MLP

The index (i_v, i_s) is an input held fixed, as in the paper's backward.
The backward is the chain rule written out step by step (attention: Eq. 1 / Eq. 12
via oracle/attention.py; RoPE: the transpose rotation).
"""
from __future__ import annotations

import numpy as np

from . import attention as OA
from . import rope as R

EPS = 1e-6


def _rms(x, w):
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + EPS)
    return x * r * w, r


def _rms_bwd(x, w, r, dy):
    g = dy * w
    D = x.shape[-1]
    dx = r * g - x * r ** 3 * np.sum(x * g, axis=-1, keepdims=True) / D
    dw = np.sum(dy * x * r, axis=0)
    return dx, dw


def _silu(g):
    return g / (1.0 + np.exp(-g))


def forward(x, P, pos, theta, mscale, i_v, i_s, Hq, Hkv, d):
    """x: [S][D] fp64 at positions pos [S]; P: dict of fp64 parameters
    (w1, Wqkv, bqkv, Wo, w2, Wg, Wu, Wd).  Returns (y, cache)."""
    S = x.shape[0]
    h1, r1 = _rms(x, P["w1"])
    qkv = h1 @ P["Wqkv"].T + P["bqkv"]
    q = qkv[:, : Hq * d].reshape(S, Hq, d)
    k = qkv[:, Hq * d: (Hq + Hkv) * d].reshape(S, Hkv, d)
    v = qkv[:, (Hq + Hkv) * d:].reshape(S, Hkv, d)
    qr = R.rope(q, pos, theta, mscale)
    kr = R.rope(k, pos, theta, mscale)
    o, lse = OA.sparse_attention_forward(qr, kr, v, i_v, i_s)
    x2 = x + o.reshape(S, Hq * d) @ P["Wo"].T
    h2, r2 = _rms(x2, P["w2"])
    g = h2 @ P["Wg"].T
    u = h2 @ P["Wu"].T
    m = _silu(g) * u
    y = x2 + m @ P["Wd"].T
    cache = dict(x=x, h1=h1, r1=r1, qr=qr, kr=kr, v=v, o=o, lse=lse, x2=x2, h2=h2, r2=r2,
                 g=g, u=u, m=m)
    return y, cache


def backward(dy, P, c, pos, theta, mscale, i_v, i_s, Hq, Hkv, d):
    """Gradients of sum(y * dy): (dx, dict of parameter gradients)."""
    S = dy.shape[0]
    G = {}
    # MLP
    G["Wd"] = dy.T @ c["m"]
    dm = dy @ P["Wd"]
    s = 1.0 / (1.0 + np.exp(-c["g"]))
    du = dm * _silu(c["g"])
    dg = dm * c["u"] * s * (1.0 + c["g"] * (1.0 - s))
    G["Wg"] = dg.T @ c["h2"]
    G["Wu"] = du.T @ c["h2"]
    dh2 = dg @ P["Wg"] + du @ P["Wu"]
    dx2, G["w2"] = _rms_bwd(c["x2"], P["w2"], c["r2"], dh2)
    dx2 = dx2 + dy
    # attention block
    o2 = c["o"].reshape(S, Hq * d)
    G["Wo"] = dx2.T @ o2
    do = (dx2 @ P["Wo"]).reshape(S, Hq, d)
    dqr, dkr, dv = OA.sparse_attention_backward(c["qr"], c["kr"], c["v"], c["o"], c["lse"], do,
                                                i_v, i_s)
    dq = R.rope(dqr, pos, theta, mscale, inverse=True)
    dk = R.rope(dkr, pos, theta, mscale, inverse=True)
    dqkv = np.concatenate([dq.reshape(S, -1), dk.reshape(S, -1), dv.reshape(S, -1)], axis=1)
    G["Wqkv"] = dqkv.T @ c["h1"]
    G["bqkv"] = dqkv.sum(axis=0)
    dh1 = dqkv @ P["Wqkv"]
    dx1, G["w1"] = _rms_bwd(c["x"], P["w1"], c["r1"], dh1)
    return dx1 + dx2, G
