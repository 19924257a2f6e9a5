"""sparseformat (Alg. 1) and convert_index (Alg. 2) — oracle.

Test infrastructure only (see oracle/__init__.py).

Reading (DESIGN.md §2.1 I9-I10, readings R3, R4, R8, R12, R15):
  slash offsets are in 64-token block units: offset o selects key block
  kb = g - o for query block g; verticals are token columns.
  I9   B_g = sort_asc{ g - o : o in i_s, o <= g }
       C_g = sort_asc{ m in i_v : floor(m/64) < g, (g - floor(m/64)) not in i_s }
       (a vertical inside a selected slash block is already computed there;
        verticals in block g itself are covered by the forced offset 0).
  I10  a layout maps global block b to (owner(b), local block lb(b)):
         block-striped: owner = b mod W, lb = b // W;
         zigzag (Fig. 1): the sequence is cut into 2W equal
           chunks, rank w holds chunks w and 2W-1-w (in that order); with chunk
           length c blocks, owner(b) = k if k < W else 2W-1-k for k = b // c, and
           lb = b mod c (+ c for the second chunk).
       For rank r, local query block j (global g), and KV origin s:
         B_g^(s) = { lb(kb) : kb in B_g, owner(kb) = s }
         C_g^(s) = { lb(floor(m/64)) * 64 + m mod 64 : m in C_g, owner(floor(m/64)) = s }
       (slash offsets stay defined on global positions)
The key set of global query n in block g is
  K_n = { m : floor(m/64) in B_g, m <= n }  U  C_g.
"""
from __future__ import annotations

import numpy as np

BLOCK = 64


def sparseformat_block(i_v, i_s, g: int, block: int = BLOCK):
    """I9 for one query block g of one head: (B_g key blocks, C_g bar columns)."""
    i_v = np.asarray(i_v, np.int64)
    i_s = np.asarray(i_s, np.int64)
    B = np.sort(g - i_s[i_s <= g])
    vb = i_v // block
    keep = (vb < g) & ~np.isin(g - vb, i_s)
    return B, np.sort(i_v[keep])


def sparseformat(i_v: np.ndarray, i_s: np.ndarray, S: int, block: int = BLOCK):
    """I9 for one head: lists B[g] (key blocks) and C[g] (bar columns), g < nb."""
    B, C = [], []
    for g in range(S // block):
        b, c = sparseformat_block(i_v, i_s, g, block)
        B.append(b)
        C.append(c)
    return B, C


def key_set(n: int, B_g: np.ndarray, C_g: np.ndarray, block: int = BLOCK) -> np.ndarray:
    """K_n: sorted global key positions attended by query n (I9 key-set rule)."""
    blk = [np.arange(kb * block, min(kb * block + block, n + 1)) for kb in B_g if kb * block <= n]
    ks = np.concatenate(blk + [np.asarray(C_g, np.int64)]) if (blk or len(C_g)) else np.zeros(0, np.int64)
    return np.unique(ks)


def index_to_mask(B, C, S: int, block: int = BLOCK) -> np.ndarray:
    """Boolean [S][S] mask covered by (B, C) — materialised, for small S only."""
    mask = np.zeros((S, S), bool)
    for g in range(S // block):
        for n in range(g * block, g * block + block):
            mask[n, key_set(n, B[g], C[g], block)] = True
    return mask


def union_mask(i_v, i_s, S: int, block: int = BLOCK) -> np.ndarray:
    """Direct construction of (verticals U slash blocks) intersected with causal.

    Built element by element from the definitions of a vertical line (all
    queries n >= m attend column m) and a slash block line (query n attends m
    when floor(n/64) - floor(m/64) = o), with no use of sparseformat.
    """
    mask = np.zeros((S, S), bool)
    offs = set(int(o) for o in i_s)
    cols = set(int(m) for m in i_v)
    for n in range(S):
        for m in range(n + 1):
            if m in cols or (n // block - m // block) in offs:
                mask[n, m] = True
    return mask


# ------------------------------------------------------------- block striping
def stripe_perm(S: int, W: int, block: int = BLOCK):
    """Local row j of rank r <-> global token (floor(j/64) W + r) 64 + j mod 64.

    Returns int64 [W][S/W] with the global token of every local row.
    """
    if S % (block * W):
        raise ValueError("S must be a multiple of 64 W (block-striped layout)")
    L = S // W
    j = np.arange(L)
    return np.stack([((j // block) * W + r) * block + j % block for r in range(W)])


def zigzag_perm(S: int, W: int):
    """Zigzag layout ("ZigZag folds the query dimension", Fig. 1):
    2W equal chunks, rank r holds chunk r then chunk 2W-1-r.

    Returns int64 [W][S/W] with the global token of every local row.
    """
    if S % (2 * W):
        raise ValueError("S must be a multiple of 2 W (zigzag layout)")
    c = S // (2 * W)
    return np.stack([np.r_[np.arange(r * c, r * c + c), np.arange((2 * W - 1 - r) * c, (2 * W - r) * c)]
                     for r in range(W)]).astype(np.int64)


LAYOUTS = ("striped", "zigzag")


def layout_perm(S: int, W: int, layout: str = "striped", block: int = BLOCK):
    """[W][S/W] global token of each local row, for a block-aligned layout."""
    if layout == "striped":
        return stripe_perm(S, W, block)
    if layout == "zigzag":
        if S % (2 * W * block):
            raise ValueError("zigzag with 64-token blocks needs S a multiple of 2 W 64")
        return zigzag_perm(S, W)
    raise ValueError(f"unknown layout {layout!r}")


def block_owner(S: int, W: int, layout: str = "striped", block: int = BLOCK):
    """(owner[b], lb[b]) for every global block b, read off layout_perm."""
    perm = layout_perm(S, W, layout, block)
    nb = S // block
    owner = np.empty(nb, np.int64)
    lb = np.empty(nb, np.int64)
    for r in range(W):
        gb = perm[r][::block] // block
        owner[gb] = r
        lb[gb] = np.arange(gb.size)
    return owner, lb


def convert_index(B, C, S: int, W: int, r: int, block: int = BLOCK, layout: str = "striped"):
    """I10 for rank r: per origin s, per local query block j: (blocks, bars) local.

    Returns plan[s][j] = (local key blocks array, local bar rows array), both
    sorted ascending, indices into origin s's local K/V chunk.
    """
    perm = layout_perm(S, W, layout, block)
    owner, lblk = block_owner(S, W, layout, block)
    nloc = S // block // W
    plan = []
    for s in range(W):
        per_j = []
        for j in range(nloc):
            g = int(perm[r][j * block]) // block
            kb = np.asarray(B[g], np.int64)
            lb = lblk[kb[owner[kb] == s]]
            cm = np.asarray(C[g], np.int64)
            cb = cm // block
            sel = owner[cb] == s
            lc = lblk[cb[sel]] * block + cm[sel] % block
            per_j.append((np.sort(lb), np.sort(lc)))
        plan.append(per_j)
    return plan
