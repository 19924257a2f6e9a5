"""Balanced (block-striped) sparse ring attention, flat and hierarchical — oracle.

Test infrastructure only (see oracle/__init__.py).

Simulates W logical ranks in one process; every "send" is a copy of the
message into the receiver's buffer at the end of the step (the async
send/recv + wait of Alg. 2 becomes a per-step barrier).  fp64 throughout.

Forward (Alg. 2, readings R12-R16):
  - block-striped layout: global block b -> rank b mod W; or the zigzag
    layout of the "Ours w/ ZigZag" ablation (sparseformat.zigzag_perm);
  - Q and O stay on their rank, K/V circulate;
  - flat ring: step t, rank r computes with the chunk it holds, then sends it to
    r+1 and receives from r-1 (so it holds origin (r - t) mod W);
  - hierarchical (W = N_out x G, rank r = n G + l): at each outer step i the
    rank posts an outer send of the chunk it holds at the START of the step to
    (r + G) mod W (R16), then runs G inner steps over the node ring
    node_base + (l +- 1) mod G (R14), then swaps in the outer message;
  - each step: block_bar_sparse_attention_forward on the held chunk with the
    convert_index lists of that origin, merge_out_and_lse.
Backward (Table 4; reading R17): the held chunk's fp64 dK/dV partial
travels with the chunk around the inner ring; at the end of every outer step
the rank holding it returns it to the chunk's owner, which adds it in.  For a
flat ring this is the single closing hop.
"""
from __future__ import annotations

import numpy as np

from .attention import NEG_INF, _softmax_rows, merge_out_and_lse
from .sparseformat import BLOCK, convert_index, layout_perm, sparseformat


def _local_plans(i_v, i_s, S, W, block, layout="striped"):
    """plans[h][r][s][j] = (local blocks, local bar rows) via convert_index."""
    plans = []
    for h in range(len(i_v)):
        B, C = sparseformat(i_v[h], i_s[h], S, block)
        plans.append([convert_index(B, C, S, W, r, block, layout) for r in range(W)])
    return plans


def _chunk_keys(lb, lc, block):
    parts = [np.arange(b * block, b * block + block) for b in lb]
    return np.concatenate(parts + [np.asarray(lc, np.int64)]) if (parts or len(lc)) \
        else np.zeros(0, np.int64)


def _step_partial(qr, kc, vc, plan_rs, rank_tok, origin_tok, hq, grp, block):
    """One (rank, step): partial (O', LSE') of rank's queries over origin chunk."""
    Lq, _, d = qr.shape
    O = np.zeros((Lq, hq, d))
    L = np.full((hq, Lq), NEG_INF)
    for h in range(hq):
        for j, (lb, lc) in enumerate(plan_rs[h]):
            keys = _chunk_keys(lb, lc, block)
            if keys.size == 0:
                continue
            rows = slice(j * block, j * block + block)
            s = (qr[rows, h] @ kc[keys, h // grp].T) / np.sqrt(d)
            mask = rank_tok[rows][:, None] >= origin_tok[keys][None, :]   # global causality
            P, lse = _softmax_rows(s, mask)
            O[rows, h] = P @ vc[keys, h // grp]
            L[h, rows] = lse
    return O, L


def schedule(W: int, inner: int | None = None):
    """Origins held per (rank, step): list over steps of list over ranks.

    Built by literally passing chunk ids through the flat / two-level ring.
    """
    G = W if inner is None else inner
    if W % G:
        raise ValueError("W must be a multiple of the inner ring size")
    nout = W // G
    held = list(range(W))
    steps = []
    for i in range(nout):
        outer_msg = [None] * W
        if i < nout - 1:
            for r in range(W):                      # post outer send of the start chunk
                outer_msg[(r + G) % W] = held[r]
        for j in range(G):
            steps.append(list(held))
            if j < G - 1:
                nxt = [None] * W
                for r in range(W):
                    n, l = divmod(r, G)
                    nxt[n * G + (l + 1) % G] = held[r]
                held = nxt
        if i < nout - 1:
            held = outer_msg
    return steps


def ring_forward(q, k, v, i_v, i_s, W: int, inner: int | None = None, block: int = BLOCK,
                 layout: str = "striped"):
    """Sparse ring forward over W ranks; returns (O, LSE) in GLOBAL token order
    plus the per-(step, rank) origin log.  layout: "striped" (the method) or
    "zigzag" (the "Ours w/ ZigZag" ablation)."""
    S, Hq, d = q.shape
    grp = Hq // k.shape[1]
    perm = layout_perm(S, W, layout, block)
    plans = _local_plans(i_v, i_s, S, W, block, layout)
    sched = schedule(W, inner)
    qs = [q[perm[r]] for r in range(W)]
    ks = [k[perm[r]] for r in range(W)]
    vs = [v[perm[r]] for r in range(W)]
    Lq = S // W
    O = [np.zeros((Lq, Hq, d)) for _ in range(W)]
    L = [np.full((Hq, Lq), NEG_INF) for _ in range(W)]
    for held in sched:
        for r in range(W):
            s = held[r]
            plan_rs = [plans[h][r][s] for h in range(Hq)]
            Op, Lp = _step_partial(qs[r], ks[s], vs[s], plan_rs, perm[r], perm[s], Hq, grp, block)
            for h in range(Hq):
                O[r][:, h], L[r][h] = merge_out_and_lse(O[r][:, h], L[r][h], Op[:, h], Lp[h])
    Og = np.zeros((S, Hq, d))
    Lg = np.zeros((Hq, S))
    for r in range(W):
        Og[perm[r]] = O[r]
        Lg[:, perm[r]] = L[r]
    return Og, Lg, sched


def ring_backward(q, k, v, O, LSE, dO, i_v, i_s, W: int, inner: int | None = None,
                  block: int = BLOCK, layout: str = "striped"):
    """Sparse ring backward (reading R17); inputs/outputs in GLOBAL token order."""
    S, Hq, d = q.shape
    Hkv = k.shape[1]
    grp = Hq // Hkv
    G = W if inner is None else inner
    perm = layout_perm(S, W, layout, block)
    plans = _local_plans(i_v, i_s, S, W, block, layout)
    sched = schedule(W, inner)
    loc = lambda x, r: x[perm[r]]
    qs, dOs, Os = [loc(q, r) for r in range(W)], [loc(dO, r) for r in range(W)], [loc(O, r) for r in range(W)]
    ks, vs = [loc(k, r) for r in range(W)], [loc(v, r) for r in range(W)]
    Ls = [LSE[:, perm[r]] for r in range(W)]
    Ds = [(dOs[r] * Os[r]).sum(axis=2) for r in range(W)]          # [Lq][Hq]
    Lq = S // W
    dQ = [np.zeros((Lq, Hq, d)) for _ in range(W)]
    dK = [np.zeros((Lq, Hkv, d)) for _ in range(W)]                # owner accumulators
    dV = [np.zeros((Lq, Hkv, d)) for _ in range(W)]
    travel = [(np.zeros((Lq, Hkv, d)), np.zeros((Lq, Hkv, d))) for _ in range(W)]
    for step, held in enumerate(sched):
        j_in = step % G
        for r in range(W):
            s = held[r]
            tk, tv = travel[r]
            for h in range(Hq):
                g = h // grp
                for j, (lb, lc) in enumerate(plans[h][r][s]):
                    keys = _chunk_keys(lb, lc, block)
                    if keys.size == 0:
                        continue
                    rows = slice(j * block, j * block + block)
                    mask = perm[r][rows][:, None] >= perm[s][keys][None, :]
                    sc = (qs[r][rows, h] @ ks[s][keys, g].T) / np.sqrt(d)
                    P = np.where(mask, np.exp(sc - Ls[r][h, rows][:, None]), 0.0)
                    dP = dOs[r][rows, h] @ vs[s][keys, g].T
                    dS = P * (dP - Ds[r][rows, h][:, None])
                    dQ[r][rows, h] += dS @ ks[s][keys, g] / np.sqrt(d)
                    tk[keys, g] += dS.T @ qs[r][rows, h] / np.sqrt(d)
                    tv[keys, g] += P.T @ dOs[r][rows, h]
        if j_in < G - 1:                                        # inner hop: partial travels with KV
            nxt = [None] * W
            for r in range(W):
                n, l = divmod(r, G)
                nxt[n * G + (l + 1) % G] = travel[r]
            travel = nxt
        else:                                                   # end of outer step: return to owner
            for r in range(W):
                s = held[r]
                dK[s] += travel[r][0]
                dV[s] += travel[r][1]
            travel = [(np.zeros((Lq, Hkv, d)), np.zeros((Lq, Hkv, d))) for _ in range(W)]
    dQg, dKg, dVg = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for r in range(W):
        dQg[perm[r]] = dQ[r]
        dKg[perm[r]] = dK[r]
        dVg[perm[r]] = dV[r]
    return dQg, dKg, dVg
