"""fp64 attention forward/backward — oracle.

Test infrastructure only (see oracle/__init__.py).

  S = Q K^T / sqrt(d), A = softmax(S), y = sparse(softmax(QK^T/sqrt d) V, i_vs)
  (Alg. 1): masked entries are excluded exactly (-inf), LSE is the natural
  log of the row's softmax normaliser.
  Backward: Eq. 1  dL/dS = A o (dL/dA - sum_j dL/dA_ij A_ij)
            Eq. 12 dV = A^T dO, dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d)
  with dL/dA = dO V^T, so sum_j dL/dA_ij A_ij = dO_i . O_i (= D_i).
  GQA (reading R10): q head h reads kv head h // (Hq/Hkv); dK/dV of a kv head sum
  over its q heads.
  merge_out_and_lse: L = log(e^La + e^Lb), O = e^(La-L) Oa + e^(Lb-L) Ob.

Arrays: q [S][Hq][d], k/v [S][Hkv][d], float64 (exact copies of the bf16 inputs).
"""
from __future__ import annotations

import numpy as np

from .sparseformat import BLOCK, sparseformat

NEG_INF = -np.inf


def _softmax_rows(s: np.ndarray, mask: np.ndarray):
    """Row softmax of s over True entries of mask; returns (P, LSE)."""
    s = np.where(mask, s, NEG_INF)
    mx = s.max(axis=1, keepdims=True)
    mx_safe = np.where(np.isfinite(mx), mx, 0.0)
    e = np.where(mask, np.exp(s - mx_safe), 0.0)
    l = e.sum(axis=1, keepdims=True)
    with np.errstate(divide="ignore", invalid="ignore"):
        P = np.where(l > 0, e / l, 0.0)
        lse = np.where(l[:, 0] > 0, mx_safe[:, 0] + np.log(l[:, 0]), NEG_INF)
    return P, lse


def dense_attention_forward(q, k, v, mask=None, qpos=None, kpos=None):
    """Textbook masked attention for ONE head: q [Sq][d], k/v [Sk][d].

    mask: boolean [Sq][Sk]; default causal from positions (qpos >= kpos).
    Returns (O [Sq][d], LSE [Sq]).
    """
    d = q.shape[1]
    if mask is None:
        qpos = np.arange(q.shape[0]) if qpos is None else qpos
        kpos = np.arange(k.shape[0]) if kpos is None else kpos
        mask = qpos[:, None] >= kpos[None, :]
    s = (q @ k.T) / np.sqrt(d)
    P, lse = _softmax_rows(s, mask)
    return P @ v, lse


def dense_attention_backward(q, k, v, dO, mask=None):
    """Eq. 1 + Eq. 12 for ONE head with a materialised mask (default causal)."""
    d = q.shape[1]
    if mask is None:
        mask = np.tril(np.ones((q.shape[0], k.shape[0]), bool))
    s = (q @ k.T) / np.sqrt(d)
    A, _ = _softmax_rows(s, mask)
    dA = dO @ v.T                                              # dL/dA
    dS = A * (dA - (dA * A).sum(axis=1, keepdims=True))      # Eq. 1
    dV = A.T @ dO                                              # Eq. 12
    dQ = dS @ k / np.sqrt(d)
    dK = dS.T @ q / np.sqrt(d)
    return dQ, dK, dV


def merge_out_and_lse(Oa, La, Ob, Lb):
    """P:879.  Rows with L = -inf are empty (identity element)."""
    L = np.logaddexp(La, Lb)
    with np.errstate(invalid="ignore"):
        wa = np.where(np.isfinite(La), np.exp(La - np.where(np.isfinite(L), L, 0.0)), 0.0)
        wb = np.where(np.isfinite(Lb), np.exp(Lb - np.where(np.isfinite(L), L, 0.0)), 0.0)
    return wa[:, None] * Oa + wb[:, None] * Ob, L


def _block_keys(g, B_g, C_g, block):
    """Keys of query block g: slash blocks (contiguous) then bar columns."""
    parts = [np.arange(kb * block, kb * block + block) for kb in B_g]
    keys = np.concatenate(parts + [np.asarray(C_g, np.int64)]) if (parts or len(C_g)) \
        else np.zeros(0, np.int64)
    return keys


def _block_mask(g, keys, block):
    """Causal rule inside the key set: key m visible to query n iff m <= n."""
    rows = np.arange(g * block, g * block + block)
    return rows[:, None] >= keys[None, :]


def forward_block(q, k, v, h, g, B_g, C_g, block: int = BLOCK):
    """Forward of query block g of q head h: returns (O rows, LSE rows)."""
    d = q.shape[2]
    grp = q.shape[1] // k.shape[1]
    rows = slice(g * block, g * block + block)
    keys = _block_keys(g, B_g, C_g, block)
    s = (q[rows, h, :] @ k[keys, h // grp, :].T) / np.sqrt(d)
    P, lse = _softmax_rows(s, _block_mask(g, keys, block))
    return P @ v[keys, h // grp, :], lse


def backward_block(q, k, v, O, LSE, dO, h, g, B_g, C_g, block: int = BLOCK):
    """Backward contributions of query block g of q head h (Eq. 1, Eq. 12).

    Returns (dQ rows [64][d], keys, dK rows [len(keys)][d], dV rows).
    """
    d = q.shape[2]
    grp = q.shape[1] // k.shape[1]
    g_kv = h // grp
    rows = slice(g * block, g * block + block)
    keys = _block_keys(g, B_g, C_g, block)
    mask = _block_mask(g, keys, block)
    kh, vh = k[keys, g_kv, :], v[keys, g_kv, :]
    s = (q[rows, h, :] @ kh.T) / np.sqrt(d)
    P = np.where(mask, np.exp(s - LSE[h, rows][:, None]), 0.0)
    D = (dO[rows, h, :] * O[rows, h, :]).sum(axis=1)
    dP = dO[rows, h, :] @ vh.T
    dS = P * (dP - D[:, None])
    return dS @ kh / np.sqrt(d), keys, dS.T @ q[rows, h, :] / np.sqrt(d), P.T @ dO[rows, h, :]


def sparse_attention_forward(q, k, v, i_v, i_s, block: int = BLOCK):
    """Alg. 1 line "y <- sparse(softmax(QK^T/sqrt d) V, i_vs)", fp64.

    i_v[h], i_s[h]: per-q-head vertical columns / slash offsets.
    Returns (O [S][Hq][d], LSE [Hq][S]).
    """
    S, Hq, d = q.shape
    O = np.zeros((S, Hq, d))
    LSE = np.full((Hq, S), NEG_INF)
    for h in range(Hq):
        B, C = sparseformat(i_v[h], i_s[h], S, block)
        for g in range(S // block):
            rows = slice(g * block, g * block + block)
            O[rows, h, :], LSE[h, rows] = forward_block(q, k, v, h, g, B[g], C[g], block)
    return O, LSE


def sparse_attention_backward(q, k, v, O, LSE, dO, i_v, i_s, block: int = BLOCK):
    """Backward of sparse_attention_forward with the index held fixed.

    Recomputes P = exp(S - LSE) on the forward's key sets; Eq. 1 with
    D_n = dO_n . O_n; Eq. 12.  Returns (dQ, dK, dV) fp64.
    """
    S, Hq, d = q.shape
    grp = Hq // k.shape[1]
    dQ = np.zeros_like(q)
    dK = np.zeros_like(k)
    dV = np.zeros_like(v)
    for h in range(Hq):
        B, C = sparseformat(i_v[h], i_s[h], S, block)
        for g in range(S // block):
            rows = slice(g * block, g * block + block)
            dq, keys, dk, dv = backward_block(q, k, v, O, LSE, dO, h, g, B[g], C[g], block)
            dQ[rows, h, :] += dq
            dK[keys, h // grp, :] += dk        # keys unique within a query block
            dV[keys, h // grp, :] += dv
    return dQ, dK, dV


def count_pairs(i_v, i_s, S: int, block: int = BLOCK, rows=None):
    """Activated (n, m) pairs per head = sum_n |K_n| (the FLOP unit),
    over all query blocks or only the query blocks listed in `rows`."""
    from .sparseformat import sparseformat_block
    out = []
    for h in range(len(i_v)):
        tot = 0
        for g in (range(S // block) if rows is None else rows):
            B, C = sparseformat_block(i_v[h], i_s[h], g, block)
            nblk = len(B)
            diag = 1 if (len(B) and B[-1] == g) else 0
            tot += (nblk - diag) * block * block + diag * block * (block + 1) // 2 + block * len(C)
        out.append(tot)
    return np.array(out, np.int64)
