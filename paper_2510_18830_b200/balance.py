"""Workload balance of context-parallel layouts.

PAPER.md §3.2: distributed dynamic sparse attention is imbalanced
across workers (at one ring step) and across steps (for one worker); the
imbalance degree is max/mean.  §4.2 contrasts ZigZag and
block-striped layouts; Table 10 reports the averages.

This module counts activated (query, key) pairs — the attention work — per
(rank, ring step) for a vertical-slash index under a layout and a ring
schedule, and derives the paper's metrics from that matrix.  Pure host code
(numpy): it reads the index lists (e.g. copied back from `ops.build_vs_index`)
and is independent of the CUDA kernels and of the oracle.

Layouts (64-token blocks; S must divide accordingly):
  striped     block b -> rank b mod W (the layout the kernels use)
  zigzag      2W equal chunks, rank r holds chunks r and 2W-1-r
  contiguous  W equal chunks, rank r holds chunk r (plain ring attention)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BLOCK = 64
LAYOUTS = ("striped", "zigzag", "contiguous")


def block_owner(nb: int, W: int, layout: str) -> np.ndarray:
    """Rank holding each 64-token block (int64 [nb])."""
    b = np.arange(nb, dtype=np.int64)
    if layout == "striped":
        return b % W
    if layout == "zigzag":
        if nb % (2 * W):
            raise ValueError("zigzag needs nb divisible by 2W")
        chunk = b // (nb // (2 * W))
        return np.where(chunk < W, chunk, 2 * W - 1 - chunk)
    if layout == "contiguous":
        if nb % W:
            raise ValueError("contiguous needs nb divisible by W")
        return b // (nb // W)
    raise ValueError(f"unknown layout {layout!r}")


def flat_schedule(W: int) -> np.ndarray:
    """held[t][r] = origin of the KV chunk rank r holds at step t (P:854-858,
    reading Q13: send to r+1, so the origin at step t is (r - t) mod W)."""
    t = np.arange(W)[:, None]
    r = np.arange(W)[None, :]
    return (r - t) % W


def pairs_by_origin(i_v, i_s, S: int, W: int, layout: str) -> np.ndarray:
    """Activated pairs [rank r][origin s]: queries held by r against keys held by s,
    summed over heads.  Key sets per query block g follow I9:
    slash blocks g - o (o in i_s, the diagonal block causal: 2080 pairs), and
    vertical columns m with floor(m/64) < g not covered by a selected slash."""
    nb = S // BLOCK
    own = block_owner(nb, W, layout)
    M = np.zeros((W, W), dtype=np.int64)
    onehot_prefix = np.zeros((W, nb + 1), dtype=np.int64)  # #query blocks < x owned by r
    for r in range(W):
        onehot_prefix[r, 1:] = np.cumsum(own == r)
    for h in range(len(i_s)):
        offs = np.unique(np.asarray(i_s[h], dtype=np.int64))
        offs = offs[(offs >= 0) & (offs < nb)]
        # slash blocks: (g, g - o) for g in [o, nb)
        for o in offs:
            g = np.arange(o, nb)
            w = 2080 if o == 0 else 4096
            np.add.at(M, (own[g], own[g - o]), w)
        # vertical columns: query blocks g in (bm, nb) minus bm + offs
        cols = np.unique(np.asarray(i_v[h], dtype=np.int64))
        bm = cols // BLOCK
        ks = own[bm]
        # all later query blocks, per query rank
        later = onehot_prefix[:, nb][:, None] - onehot_prefix[:, bm + 1]  # [W][ncols]
        for r in range(W):
            np.add.at(M[r], ks, 64 * later[r])
        # covered by a selected slash (offset >= 1; offset 0 is g == bm, not later)
        pos = offs[offs > 0]
        if len(pos) and len(cols):
            gq = bm[:, None] + pos[None, :]
            ok = gq < nb
            np.add.at(M, (own[gq[ok]], np.broadcast_to(ks[:, None], gq.shape)[ok]), -64)
    return M


def pairs_by_origin_csr(ptr, idx, S: int, W: int, layout: str) -> np.ndarray:
    """Activated pairs [rank r][origin s] of an explicit block index in CSR form
    (mt_block_sparse_attn_* / mt_xattn_index): ptr int64 [Hq][nb + 1] (global
    offsets), idx the key blocks; a diagonal block is causal (2080 pairs), any
    other full (4096)."""
    nb = S // BLOCK
    own = block_owner(nb, W, layout)
    ptr = np.asarray(ptr, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    M = np.zeros(W * W, dtype=np.float64)
    for h in range(ptr.shape[0]):
        b, e = ptr[h, 0], ptr[h, nb]
        if e == b:
            continue
        g = np.repeat(np.arange(nb, dtype=np.int64), np.diff(ptr[h]))
        kb = idx[b:e]
        M += np.bincount(own[g] * W + own[kb], weights=np.where(kb == g, 2080.0, 4096.0),
                         minlength=W * W)
    return M.reshape(W, W).astype(np.int64)


def pairs_by_origin_blocks(B, S: int, W: int, layout: str) -> np.ndarray:
    """pairs_by_origin_csr for rows B[h][g] (key blocks of query block g of head h)."""
    nb = S // BLOCK
    ptr = np.zeros((len(B), nb + 1), dtype=np.int64)
    flat, run = [], 0
    for h, rows in enumerate(B):
        for g in range(nb):
            ptr[h, g] = run
            run += len(rows[g])
            flat.append(np.asarray(rows[g], dtype=np.int64))
        ptr[h, nb] = run
    idx = np.concatenate(flat) if flat else np.zeros(0, np.int64)
    return pairs_by_origin_csr(ptr, idx, S, W, layout)


def analyse_csr(ptr, idx, S: int, W: int, layout: str, held: np.ndarray | None = None) -> dict:
    """analyse() for an explicit block index in CSR form."""
    M = pairs_by_origin_csr(ptr, idx, S, W, layout)
    held = flat_schedule(W) if held is None else np.asarray(held)
    P = pairs_by_step(M, held)
    return {"layout": layout, "world": W, "pairs": int(M.sum()), "metrics": imbalance(P).as_dict(),
            "pairs_by_step": P.tolist()}


def bwd_slot_occupancy(i_s, nb: int) -> dict:
    """Share of the backward block pass's 128-key rows that are live (single GPU).

    The key-major backward tile holds key blocks (k, k + 1), k even, and walks the
    query blocks g that attend either (g - k in O or g - k - 1 in O, O = i_s[h]); every
    chunk computes all 128 key rows, so a query block attending only one of the two
    wastes half the chunk's MMA rows.  Returns chunks, live slots and live / (2 chunks)
    summed over heads.  Counting: a value x contributes one chunk per even k with
    k + x < nb, i.e. ceil((nb - x) / 2) of them."""
    chunks = live = 0
    for offs in i_s:
        O = np.unique(np.asarray(offs, dtype=np.int64))
        O = O[(O >= 0) & (O < nb)]
        U = np.union1d(O, O + 1)
        U = U[U < nb]
        n_even = lambda x: np.maximum(0, (nb - x + 1) // 2)  # even k in [0, nb - x)
        chunks += int(n_even(U).sum())
        live += int(n_even(O).sum() + np.maximum(0, (nb - O) // 2).sum())
    return {"chunks": chunks, "live_slots": live,
            "occupancy": live / (2 * chunks) if chunks else 1.0}


def pairs_by_step(M: np.ndarray, held: np.ndarray) -> np.ndarray:
    """[rank][step] from [rank][origin] and a schedule held[t][r] = origin."""
    W = M.shape[0]
    P = np.empty((W, held.shape[0]), dtype=np.int64)
    for t in range(held.shape[0]):
        P[:, t] = M[np.arange(W), held[t]]
    return P


@dataclass
class Imbalance:
    worker_id: float      # mean over steps of max_r / mean_r (Table 10 "Avg. ID, worker-level")
    step_id: float        # mean over ranks of max_t / mean_t (Table 10 "Avg. ID, step-level")
    comp_ratio: float     # sum_t mean_r / sum_t max_r: useful share of lockstep compute time
    total_id: float       # max_r / mean_r of per-rank totals (whole-job worker balance)

    def as_dict(self) -> dict:
        return {k: round(float(v), 4) for k, v in self.__dict__.items()}


def imbalance(P: np.ndarray) -> Imbalance:
    """Metrics of a [rank][step] work matrix (imbalance degree = max / mean).
    Steps where no rank has work are skipped.  The computation ratio here is the
    compute-only analogue of Table 10's (it ignores communication): with a
    barrier per ring step every rank waits for that step's slowest rank."""
    P = np.asarray(P, dtype=np.float64)
    col_mean = P.mean(axis=0)
    live = col_mean > 0
    wid = float(np.mean(P[:, live].max(axis=0) / col_mean[live])) if live.any() else 1.0
    row_mean = P.mean(axis=1)
    lr = row_mean > 0
    sid = float(np.mean(P[lr].max(axis=1) / row_mean[lr])) if lr.any() else 1.0
    cr = float(P.mean(axis=0).sum() / max(P.max(axis=0).sum(), 1.0))
    tot = P.sum(axis=1)
    tid = float(tot.max() / tot.mean()) if tot.mean() > 0 else 1.0
    return Imbalance(wid, sid, cr, tid)


def analyse(i_v, i_s, S: int, W: int, layout: str, held: np.ndarray | None = None) -> dict:
    """Pairs per (rank, step) and the imbalance metrics for one configuration."""
    M = pairs_by_origin(i_v, i_s, S, W, layout)
    held = flat_schedule(W) if held is None else np.asarray(held)
    P = pairs_by_step(M, held)
    return {"layout": layout, "world": W, "pairs": int(M.sum()), "metrics": imbalance(P).as_dict(),
            "pairs_by_step": P.tolist()}
