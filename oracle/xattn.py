"""Oracle: XAttention antidiagonal block index, fp64.

TEST INFRASTRUCTURE ONLY (like all of oracle/): imported by tests/, never by the
product path.

PAPER.md P:826: "XAttention score square blocks by summing every certain stride
along their antidiagonals and retains only the high-score blocks ... granularity
128 as the block size, stride 16 as the sampling pitch and threshold 0.9";
P:347: "Ours w/ XAttn Idx." = MTraining with this block index.

Reading R25, written out step by step for one q head h (kv head
h // (Hq/Hkv)), block B = 128, stride st = 16, threshold tau:
  1. antidiagonal scores on the stride grid, i, j < S/st:
       A[i][j] = sum_{s<st} q[i st + st-1-s] . k[j st + s] / (st sqrt(d)),
     i.e. the sum of the st-long antidiagonal of the (i, j) st x st sub-block of
     Q K^T / sqrt(d), divided by st;
  2. P = row softmax of A over the causal grid j <= i;
  3. block scores: Bs[I][J] = sum of P over the (B/st) x (B/st) sub-block (I, J),
     J <= I (each row I then sums to B/st);
  4. per query block I: order J <= I by Bs[I][J] descending (ties: smaller J first)
     and keep the shortest prefix whose sum reaches tau * sum_J Bs[I][J] (J is
     taken iff the sum before it is < tau * total); the diagonal J = I is always
     kept (XAttention's local block);
  5. 64-token CSR for the kernels: a kept (I, J) covers query blocks 2I, 2I+1 and
     key blocks 2J, 2J+1, except J = I where query block 2I keeps only key block
     2I (2I+1 lies in its future).
"""
from __future__ import annotations

import numpy as np

BLOCK, STRIDE = 128, 16


def antidiag_scores(qh: np.ndarray, kh: np.ndarray, stride: int = STRIDE) -> np.ndarray:
    """Step 1 for one head: qh [Sq][d], kh [Sk][d] -> A [Sq/st][Sk/st] (fp64; upper
    triangle included, masked later).  Row i of A is stride row i of qh."""
    Sq, d = qh.shape
    n = Sq // stride
    qr = qh.reshape(n, stride, d)[:, ::-1, :].reshape(n, stride * d)  # rows st-1-s
    kr = kh.reshape(kh.shape[0] // stride, stride * d)                  # rows s
    return (qr @ kr.T) / (stride * np.sqrt(d))


def block_scores(qh, kh, block: int = BLOCK, stride: int = STRIDE) -> np.ndarray:
    """Steps 2-3: Bs [S/B][S/B] (zero above the diagonal)."""
    A = antidiag_scores(qh, kh, stride)
    n = A.shape[0]
    causal = np.tril(np.ones((n, n), bool))
    A = np.where(causal, A, -np.inf)
    A = A - A.max(axis=1, keepdims=True)
    P = np.exp(A)
    P /= P.sum(axis=1, keepdims=True)
    r = block // stride
    nI = n // r
    return P.reshape(nI, r, nI, r).sum(axis=(1, 3))


def block_score_rows(qh, kh, rows, block: int = BLOCK, stride: int = STRIDE) -> dict:
    """Steps 1-3 for selected query blocks only (for long sequences): {I: Bs[I][0..I]}.
    Same definition as block_scores, evaluated row by row."""
    d = qh.shape[1]
    r = block // stride
    out = {}
    for I in rows:
        A = antidiag_scores(qh[I * block:(I + 1) * block], kh[: (I + 1) * block], stride)  # [r][(I+1) r]
        acc = np.zeros(I + 1)
        for rr in range(r):
            i = I * r + rr
            a = A[rr, : i + 1]
            p = np.exp(a - a.max())
            p /= p.sum()
            acc += np.bincount(np.arange(i + 1) // r, weights=p, minlength=I + 1)[: I + 1]
        out[I] = acc
    return out


def select_blocks(Bs: np.ndarray, tau: float) -> list[np.ndarray]:
    """Step 4: kept key blocks (128-granularity, ascending) per query block."""
    out = []
    for I in range(Bs.shape[0]):
        row = Bs[I, : I + 1]
        order = np.argsort(-row, kind="stable")
        total = row.sum()
        keep, acc = [], 0.0
        for J in order:
            if acc >= tau * total:
                break
            keep.append(J)
            acc += row[J]
        if I not in keep:
            keep.append(I)
        out.append(np.array(sorted(keep), np.int32))
    return out


def to_block64(sel: list[np.ndarray]) -> list[np.ndarray]:
    """Step 5: 64-token key-block rows for query blocks 0 .. 2 len(sel) - 1."""
    rows = []
    for I, Js in enumerate(sel):
        for half in (0, 1):
            r = []
            for J in Js:
                if J < I:
                    r += [2 * J, 2 * J + 1]
                else:  # J == I
                    r += [2 * I] if half == 0 else [2 * I, 2 * I + 1]
            rows.append(np.array(r, np.int32))
    return rows


def xattn_index(q: np.ndarray, k: np.ndarray, tau: float = 0.9, block: int = BLOCK,
                stride: int = STRIDE):
    """q [S][Hq][d], k [S][Hkv][d] (fp64 copies of the bf16 inputs) ->
    (B64[h][g] key-block rows, Bs[h] block scores, sel[h] 128-granularity rows)."""
    S, Hq, _ = q.shape
    grp = Hq // k.shape[1]
    B64, BS, SEL = [], [], []
    for h in range(Hq):
        Bs = block_scores(q[:, h, :], k[:, h // grp, :], block, stride)
        sel = select_blocks(Bs, tau)
        BS.append(Bs)
        SEL.append(sel)
        B64.append(to_block64(sel))
    return B64, BS, SEL
