"""Alg. 1 "Dynamic Sparse Training Head" index, VS-IDX v1 arithmetic.

Test infrastructure only (see oracle/__init__.py).

PAPER.md Alg. 1:
    Â   <- softmax(Q[-last_q:] K^T / sqrt(d) + m_causal)
    k_v <- topp(sum_v(Â), p_v);  i_v <- argtopk(sum_v(Â), k_v)
    k_s <- topp(Pool(sum_v(Â), B_s), p_s); i_s <- argtopk(., k_s)
    i_vs <- sparseformat(i_v, i_s)
with "vertical lines estimated at the token level, slash lines pooled over
64x64 blocks".  The paper fixes no arithmetic; DESIGN.md §2.1 states
the reading used here (VS-IDX v1, steps I1-I8), chosen so that an independent
implementation can reach the same bits:

  I1 t[i,m] = fold_c RN(acc + q[n_i,c] k[m,c]), n_i = S-64+i, causal m <= n_i
            (the product is exact, not rounded on its own: one fused multiply-add
            per channel, IEEE 754 fusedMultiplyAdd)
  I2 M_i    = max_m t[i,m]
  I3 e      = exp2s(RN(RN(t - M_i) * C_d)),  C_d = RN(log2(e)/sqrt(d))
  I4 E_i    = sum_m floor(e * 2^31)                     (uint64, exact)
  I5 l_i    = RN(float(E_i)) * 2^-31; p = RN(e / l_i); w = floor(p * 2^32)
  I6 V_m    = sum_i w[i,m];  P_kb = sum_{m in kb} V_m;  sigma_o = P_{nb-1-o}
  I7 k      = min{k >= 1 : 2^24 cumsum_k >= rint(p 2^24) T}  (all items if p = 1)
  I8 i_v    = sort_asc(top k_v by (score desc, idx asc) U {0}); same for i_s

Float arithmetic is numpy float32 (IEEE round-to-nearest-even per operation)
except I1's fused step, which is evaluated as RN32(RN64(acc + q k)): q k of two
bf16 values is exact in float64, and the float64 sum is either exact or so far
from a float32 rounding boundary that the second rounding cannot move it
(reading R11), so this equals fmaf(q, k, acc) for every bf16 input,
tiny and huge ones included.  Integer arithmetic is uint64 or Python int.
"""
from __future__ import annotations

import ctypes
import math
from pathlib import Path

import numpy as np

BLOCK = 64          # B_s = stripe = window rows (reading R2 last_q = 64)
F32 = np.float32

# C_d = RN(log2(e)/sqrt(d)) for d = 128, and exp2 Horner coefficients
# c_k = RN(ln(2)^k / k!), k = 0..7 (I3).  Bit patterns are the
# values; tests/test_oracle_index.py re-derives them from math.log/factorial.
C_D_BITS = {128: 0x3E0293EE}
EXP2_COEF_BITS = [0x3F800000, 0x3F317218, 0x3E75FDF0, 0x3D635847,
                  0x3C1D955B, 0x3AAEC3FF, 0x39218489, 0x377FE5FE]


def _f32_from_bits(b: int) -> np.float32:
    return np.array([b], np.uint32).view(np.float32)[0]


EXP2_COEF = [_f32_from_bits(b) for b in EXP2_COEF_BITS]


def c_d(d: int) -> np.float32:
    if d in C_D_BITS:
        return _f32_from_bits(C_D_BITS[d])
    return F32(math.log2(math.e) / math.sqrt(d))


def exp2s(y: np.ndarray) -> np.ndarray:
    """I3: specified 2^y for float32 y <= 0 (no hardware ex2, no FMA).

    y < -125 -> 0; else j = rint_even(y), f = y - j (exact), Horner
    p = c7; p = RN(RN(p f) + c_k) for k = 6..0; result p * 2^j (exact).
    """
    y = np.asarray(y, dtype=F32)
    out = np.zeros_like(y)
    ok = y >= F32(-125.0)
    yy = y[ok]
    j = np.rint(yy).astype(F32)          # numpy rint: round half to even
    f = (yy - j).astype(F32)
    p = np.full_like(f, EXP2_COEF[7])
    for c in reversed(EXP2_COEF[:7]):
        p = (p * f).astype(F32)
        p = (p + c).astype(F32)
    out[ok] = np.ldexp(p, j.astype(np.int32)).astype(F32)
    return out


def window_scores(q_win: np.ndarray, k: np.ndarray) -> np.ndarray:
    """I1: t[i, m] for the 64 window rows of ONE head against keys k.

    q_win: [64][d] float32 (exact bf16 values), k: [S][d] float32.  Returns
    t [64][S] float32; entries with m > n_i (non-causal) are set to -inf.
    Sequential fold over the d channels, one fused multiply-add (one float32
    rounding of acc + q k, the product exact) per channel.
    """
    nq, d = q_win.shape
    S = k.shape[0]
    q64 = np.asarray(q_win, np.float64)
    k64 = np.asarray(k, np.float64)
    acc = np.zeros((nq, S), F32)
    for c in range(d):
        acc = (acc.astype(np.float64) + q64[:, c:c + 1] * k64[None, :, c]).astype(F32)
    n = S - nq + np.arange(nq)
    acc[np.arange(S)[None, :] > n[:, None]] = -np.inf
    return acc


def window_stats(t: np.ndarray, d: int):
    """I2-I5 for one head: row max M, uint64 row sums E, uint64 weights w.

    Returns (M [64] f32, E [64] uint64, w [64][S] uint64).
    """
    M = t.max(axis=1).astype(F32)                                   # I2
    y = ((t - M[:, None]).astype(F32) * c_d(d)).astype(F32)        # I3
    y[~np.isfinite(t)] = -np.inf
    e = exp2s(np.where(np.isfinite(y), y, F32(-1000.0)))
    e[~np.isfinite(t)] = 0
    fx = np.floor((e * F32(2.0 ** 31)).astype(np.float64)).astype(np.uint64)   # I4
    E = fx.sum(axis=1, dtype=np.uint64)
    l = (E.astype(np.float64).astype(F32) * F32(2.0 ** -31)).astype(F32)       # I5
    p = (e / l[:, None]).astype(F32)
    w = np.floor((p * F32(2.0 ** 32)).astype(np.float64)).astype(np.uint64)
    return M, E, w


def column_and_slash_scores(w: np.ndarray, block: int = BLOCK):
    """I6 (P:224 sum_v; P:228 Pool(sum_v, B_s); P:249 64x64 pooling).

    V_m = sum_i w[i, m]; P_kb = sum_{m in kb} V_m; sigma_o = P_{nb-1-o}.
    Returns (V [S] uint64, sigma [nb] uint64).
    """
    V = w.sum(axis=0, dtype=np.uint64)
    nb = V.size // block
    P = V.reshape(nb, block).sum(axis=1, dtype=np.uint64)
    sigma = P[::-1].copy()
    return V, sigma


def _order_u64(scores: np.ndarray) -> np.ndarray:
    """Indices sorted by (score descending, index ascending) (reading R6)."""
    s = np.asarray(scores, dtype=np.uint64)
    idx = np.arange(s.size, dtype=np.int64)
    # lexsort: last key is primary.  Descending score == ascending (max - score).
    return np.lexsort((idx, (np.uint64(0xFFFFFFFFFFFFFFFF) - s)))


def topp_budget(scores: np.ndarray, p: float) -> int:
    """I7 (readings R5, R22): minimal k whose top-k mass >= p * total.

    Exact integer arithmetic: p_q = rint(p * 2^24); k = all items if p_q = 2^24,
    else min{k >= 1 : 2^24 * cumsum_k >= p_q * T}.
    """
    s = np.asarray(scores, dtype=np.uint64)
    pq = int(np.rint(np.float64(np.float32(p)) * 2.0 ** 24))
    if pq >= 1 << 24:
        return int(s.size)
    order = _order_u64(s)
    T = int(s.sum(dtype=np.uint64))
    csum = np.cumsum(s[order], dtype=np.uint64)
    lhs = csum * np.uint64(1 << 24)
    rhs = np.uint64(pq) * np.uint64(T)
    k = int(np.argmax(lhs >= rhs)) + 1
    return k


def argtopk(scores: np.ndarray, k: int) -> np.ndarray:
    """P:225/P:229 argtopk; ties toward the smaller index (R6); sorted ascending."""
    order = _order_u64(np.asarray(scores, dtype=np.uint64))
    return np.sort(order[:k]).astype(np.int32)


def vs_index_head(q_win: np.ndarray, k: np.ndarray, p_v: float, p_s: float,
                  block: int = BLOCK, use_c: bool = True):
    """Alg. 1 index for one q head: returns (i_v, i_s) sorted int32 arrays.

    q_win: float32 [64][d] last-block queries of this head; k: float32 [S][d]
    keys of its kv head.  Forced members column 0 and offset 0 (reading R7).
    """
    d = q_win.shape[1]
    if use_c and _clib() is not None:
        V = _c_column_scores(q_win, k)
        nb = V.size // block
        sigma = V.reshape(nb, block).sum(axis=1, dtype=np.uint64)[::-1].copy()
    else:
        t = window_scores(q_win, k)
        _, _, w = window_stats(t, d)
        V, sigma = column_and_slash_scores(w, block)
    kv = topp_budget(V, p_v)
    ks = topp_budget(sigma, p_s)
    iv = np.union1d(argtopk(V, kv), [0]).astype(np.int32)
    is_ = np.union1d(argtopk(sigma, ks), [0]).astype(np.int32)
    return iv, is_


def build_vs_index(q: np.ndarray, k: np.ndarray, p_v: float, p_s: float, block: int = BLOCK,
                   use_c: bool = True):
    """Alg. 1 over all q heads.  q: [S][Hq][d], k: [S][Hkv][d] float32 (bf16 values).

    GQA (reading R10): one index per q head, scored against kv head h // (Hq/Hkv).
    Returns (i_v list, i_s list).
    """
    S, Hq, d = q.shape
    Hkv = k.shape[1]
    grp = Hq // Hkv
    ivs, iss = [], []
    for h in range(Hq):
        q_win = np.ascontiguousarray(q[S - block:, h, :], dtype=F32)
        kk = np.ascontiguousarray(k[:, h // grp, :], dtype=F32)
        iv, is_ = vs_index_head(q_win, kk, p_v, p_s, block, use_c)
        ivs.append(iv)
        iss.append(is_)
    return ivs, iss


# ----------------------------------------------------------- C fast path (I1-I6)
_CLIB = None
_CLIB_TRIED = False
_C_SRC = Path(__file__).with_name("_vsidx_ref.c")
_C_SO = Path(__file__).with_name("_vsidx_ref.so")


def build_c(force: bool = False) -> Path | None:
    """Compile _vsidx_ref.c (plain C, -O3 -fno-fast-math -ffp-contract=off)."""
    import subprocess
    if _C_SO.exists() and not force and _C_SO.stat().st_mtime >= _C_SRC.stat().st_mtime:
        return _C_SO
    cmd = ["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-o", str(_C_SO), str(_C_SRC), "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return _C_SO


def _clib():
    global _CLIB, _CLIB_TRIED
    if not _CLIB_TRIED:
        _CLIB_TRIED = True
        try:
            so = build_c()
            _CLIB = ctypes.CDLL(str(so))
            _CLIB.vsidx_ref_column_scores.restype = ctypes.c_int
        except Exception:
            _CLIB = None
    return _CLIB


def _c_column_scores(q_win: np.ndarray, k: np.ndarray) -> np.ndarray:
    lib = _clib()
    nq, d = q_win.shape
    S = k.shape[0]
    q_win = np.ascontiguousarray(q_win, dtype=F32)
    k = np.ascontiguousarray(k, dtype=F32)
    V = np.zeros(S, np.uint64)
    rc = lib.vsidx_ref_column_scores(
        q_win.ctypes.data_as(ctypes.c_void_p), k.ctypes.data_as(ctypes.c_void_p),
        ctypes.c_int64(S), ctypes.c_int(d), ctypes.c_int(nq),
        ctypes.c_uint32(int(np.array([c_d(d)], F32).view(np.uint32)[0])),
        V.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise RuntimeError(f"vsidx_ref_column_scores failed ({rc})")
    return V


def column_scores(q_win: np.ndarray, k: np.ndarray, use_c: bool = True) -> np.ndarray:
    """V_m (I1-I6) for one head, via C when available (bit-identical to numpy)."""
    if use_c and _clib() is not None:
        return _c_column_scores(q_win, k)
    t = window_scores(np.asarray(q_win, F32), np.asarray(k, F32))
    _, _, w = window_stats(t, q_win.shape[1])
    return column_and_slash_scores(w)[0]
