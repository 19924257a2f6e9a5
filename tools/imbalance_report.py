"""Worker- / step-level imbalance of the sparse ring (PAPER.md
P:142-169, Table 10) on the synthetic 512K workload.

  python tools/imbalance_report.py [--seq 524288] [--out gpurun_out/imbalance.json]

1. Builds the VS index on the GPU (ops.build_vs_index, p = 0.9) and counts
   activated pairs per (rank, ring step) for the block-striped layout (ours),
   ZigZag and contiguous, flat and hierarchical schedules, W = 4..32
   (paper_2510_18830_b200/balance.py).
2. Dense causal (every offset) for reference (Table 10's "Dense" row).
3. Measures the real per-(rank, step) kernel times of the ring on one GPU, in the
   block-striped AND the zigzag layout (the kernels take either), by running every
   (rank, step) of W = 8 and 32 through mt_attn_fwd_step / mt_attn_bwd_step (CUDA
   events), for the synthetic index, the controlled band pattern and dense causal,
   and reports the same metrics on times plus the lockstep ring time (per step the
   slowest rank).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import balance, ops  # noqa: E402
from synth.generator import make_grad_out, make_qkv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=524288)
ap.add_argument("--hq", type=int, default=16)
ap.add_argument("--hkv", type=int, default=2)
ap.add_argument("--out", default="gpurun_out/imbalance.json")
ap.add_argument("--measure", default="8,32")
ap.add_argument("--measure-patterns", default="sparse,band64+rand,dense")
ap.add_argument("--append-band", default="", help="CPU only: add the controlled band pattern to this JSON")
a = ap.parse_args()


def band_pattern(S, Hq, seed=0, window_blocks=64, n_rand_off=96, n_sink=64, n_rand_col=512):
    """Controlled pattern: a local window of `window_blocks` block
    offsets + random far offsets; sink columns + random columns, per head."""
    rng = np.random.default_rng(seed)
    nb_ = S // 64
    iv_, is__ = [], []
    for _ in range(Hq):
        is__.append(np.unique(np.r_[np.arange(window_blocks),
                                    rng.choice(np.arange(window_blocks, nb_), n_rand_off, replace=False)]))
        iv_.append(np.unique(np.r_[np.arange(n_sink), rng.choice(S, n_rand_col, replace=False)]))
    return iv_, is__


if a.append_band:
    res = json.loads(Path(a.append_band).read_text())
    S, Hq = res["config"]["seq_len"], res["config"]["n_q_heads"]
    biv, bis = band_pattern(S, Hq)
    for W in (4, 8, 16, 32):
        for layout in ("striped", "zigzag"):
            M = balance.pairs_by_origin(biv, bis, S, W, layout)
            for sched in ("flat", "hierarchical"):
                held = balance.flat_schedule(W) if sched == "flat" else None
                if held is None:
                    continue  # hierarchical schedules come from the library (GPU box run)
                P = balance.pairs_by_step(M, held)
                res["analytic"].append({"pattern": "band64+rand", "world": W, "layout": layout,
                                        "schedule": sched, "inner": W,
                                        "metrics": balance.imbalance(P).as_dict()})
                if W in (8, 32):
                    print("band64+rand", W, layout, sched, balance.imbalance(P).as_dict())
    Path(a.append_band).write_text(json.dumps(res, indent=1))
    sys.exit(0)
S, Hq, Hkv = a.seq, a.hq, a.hkv
nb = S // 64
HIER = {4: 2, 8: 4, 16: 8, 32: 8}  # inner ring size (paper: 4 nodes x 8 GPUs at W = 32)

q, k, v = make_qkv(S, Hq, Hkv, seed=0)
dO = make_grad_out(S, Hq, seed=0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
qd, kd, vd, dd = t(q), t(k), t(v), t(dO)
idx = ops.build_vs_index(qd, kd, 0.9, 0.9)
iv, is_ = idx.to_lists()
out = {"config": {"seq_len": S, "n_q_heads": Hq, "n_kv_heads": Hkv, "p": 0.9,
                  "data": "synthetic RoPE vertical-slash generator (DESIGN.md §3)"},
       "analytic": [], "measured": []}

t0 = time.time()
dense_iv = [np.array([0])] * Hq
dense_is = [np.arange(nb)] * Hq
for W in (4, 8, 16, 32):
    for name, (IV, IS) in (("sparse", (iv, is_)), ("dense", (dense_iv, dense_is))):
        for layout in ("striped", "zigzag"):
            M = balance.pairs_by_origin(IV, IS, S, W, layout)
            for sched in ("flat", "hierarchical"):
                held = (balance.flat_schedule(W) if sched == "flat"
                        else np.array(ops.ring_schedule(W, HIER[W])))
                P = balance.pairs_by_step(M, held)
                out["analytic"].append({"pattern": name, "world": W, "layout": layout,
                                        "schedule": sched, "inner": HIER[W] if sched != "flat" else W,
                                        "metrics": balance.imbalance(P).as_dict()})
print(f"analytic done in {time.time() - t0:.1f} s", flush=True)

# ---- measured: every (rank, step) of the ring on one GPU, both layouts (the kernels take
# either: plan.cuh layouts), for the synthetic index, the controlled band pattern and dense
def rows_of(layout, W, r):
    j = np.arange(S // W)
    if layout == "striped":
        return ((j // 64) * W + r) * 64 + j % 64
    c = S // (2 * W)
    return np.r_[np.arange(r * c, r * c + c), np.arange((2 * W - 1 - r) * c, (2 * W - r) * c)]


biv, bis = band_pattern(S, Hq)
pattern_idx = {"sparse": (idx, iv, is_),
               "band64+rand": (ops.VSIndex.from_lists(biv, bis, S), biv, bis),
               "dense": (ops.VSIndex.from_lists(dense_iv, dense_is, S), dense_iv, dense_is)}
for pname in [x for x in a.measure_patterns.split(",") if x]:
    pidx, piv, pis = pattern_idx[pname]
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, pidx)
    for W in [int(x) for x in a.measure.split(",") if x]:
        for layout in ("striped", "zigzag"):
            Lq = S // W
            loc = lambda x, r: ops.stripe(x, W, r, layout)
            rows_t = [torch.from_numpy(rows_of(layout, W, r)).cuda() for r in range(W)]
            held = balance.flat_schedule(W)
            tf = np.zeros((W, W))
            tb = np.zeros((W, W))
            for rep in range(2):  # first pass warms up
                for r in range(W):
                    q_l, o_l, do_l = loc(qd, r), loc(o, r), loc(dd, r)
                    L_l = lse[:, rows_t[r]].contiguous()
                    o_out = torch.empty_like(q_l)
                    o_acc = torch.zeros(Lq, Hq, 128, dtype=torch.float32, device="cuda")
                    lse_acc = torch.zeros(Hq, Lq, dtype=torch.float32, device="cuda")
                    D = torch.empty(Hq, Lq, dtype=torch.float32, device="cuda")
                    ops.attn_bwd_preprocess(S, W, o_l, do_l, D, layout=layout)
                    dq = torch.zeros(Lq, Hq, 128, dtype=torch.float32, device="cuda")
                    dk = torch.zeros(Lq, Hkv, 128, dtype=torch.float32, device="cuda")
                    dv = torch.zeros_like(dk)
                    for st in range(W):
                        s = int(held[st, r])
                        k_s, v_s = loc(kd, s), loc(vd, s)
                        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                        e[0].record()
                        ops.attn_fwd_step(S, W, r, s, st == 0, st == W - 1, q_l, k_s, v_s, pidx, o_out,
                                          o_acc, lse_acc, layout=layout)
                        e[1].record()
                        ops.attn_bwd_step(S, W, r, s, q_l, k_s, v_s, do_l, L_l, D, pidx, dq, dk, dv,
                                          layout=layout)
                        e[2].record()
                        torch.cuda.synchronize()
                        tf[r, st] = e[0].elapsed_time(e[1])
                        tb[r, st] = e[1].elapsed_time(e[2])
            tot = tf + tb
            # lockstep ring time: per step the slowest rank; vs the balanced ideal (mean)
            out["measured"].append({"pattern": pname, "world": W, "layout": layout, "schedule": "flat",
                                    "fwd_ms": tf.round(3).tolist(), "bwd_ms": tb.round(3).tolist(),
                                    "lockstep_ms": float(tot.max(axis=0).sum()),
                                    "balanced_ms": float(tot.mean(axis=0).sum()),
                                    "metrics_fwd": balance.imbalance(tf).as_dict(),
                                    "metrics_bwd": balance.imbalance(tb).as_dict(),
                                    "metrics_total": balance.imbalance(tot).as_dict(),
                                    "pair_metrics": balance.imbalance(
                                        balance.pairs_by_step(balance.pairs_by_origin(piv, pis, S, W, layout),
                                                              held)).as_dict()})
            print(f"measured {pname} W={W} {layout}: lockstep {tot.max(axis=0).sum():.1f} ms, "
                  f"{balance.imbalance(tot).as_dict()}", flush=True)

Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(out, indent=1))
for r in out["analytic"]:
    if r["world"] in (8, 32):
        print(r["pattern"], r["world"], r["layout"], r["schedule"], r["metrics"])
