"""SURVEY §8(f) f2 at 512K on one B200: the XAttention block index ("w/ XAttn Idx.",
P:347: block 128, stride 16, threshold 0.9) on the bench's synthetic q/k, its
density, the block-sparse attention forward + backward driven by it, and the
workload balance of that index under the striped and ZigZag layouts at W = 8 / 32
(the paper's E4 case: imbalance degree 3.17 at 95% sparsity, CP = 32).
Prints one JSON line.  CUDA events on the current stream, median of --steps."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_18830_b200 import balance, ops  # noqa: E402
from synth.generator import make_grad_out, make_qkv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=524288)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--tau", type=float, default=0.9)
    a = ap.parse_args()
    S, Hq, Hkv = a.seq, 16, 2
    q, k, v = make_qkv(S, Hq, Hkv, seed=0)
    dO = make_grad_out(S, Hq, seed=0)
    t = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
    qd, kd, vd, dd = t(q), t(k), t(v), t(dO)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    times = {"index": [], "fwd": [], "bwd": []}
    for it in range(a.warmup + a.steps):
        e = [ev() for _ in range(4)]
        e[0].record()
        bi = ops.xattn_index(qd, kd, a.tau)   # synchronizes once (the count readback)
        e[1].record()
        o, lse = ops.block_sparse_attn_fwd(qd, kd, vd, bi)
        e[2].record()
        ops.block_sparse_attn_bwd(qd, kd, vd, o, lse, dd, bi)
        e[3].record()
        torch.cuda.synchronize()
        if it >= a.warmup:
            for key, (x, y) in zip(times, ((0, 1), (1, 2), (2, 3))):
                times[key].append(e[x].elapsed_time(e[y]))
    ms = {key: float(np.median(v_)) for key, v_ in times.items()}
    nb = S // 64
    pairs_causal = Hq * (S * (S + 1) / 2)
    ptr, idx = bi.ptr.cpu().numpy(), bi.idx.cpu().numpy()
    M1 = balance.pairs_by_origin_csr(ptr, idx, S, 1, "striped")
    density = float(M1.sum() / pairs_causal)
    bal = {}
    for W in (8, 32):
        for layout in ("striped", "zigzag"):
            bal[f"{layout}_W{W}"] = balance.analyse_csr(ptr, idx, S, W, layout)["metrics"]
    total = ms["index"] + ms["fwd"] + ms["bwd"]
    print(json.dumps({
        "metric": "xattn-index sparse attn fwd+bwd tokens/s", "value": S / (total / 1e3),
        "unit": "tokens/s", "config": {"workload": f"S={S}, Hq=16, Hkv=2, d=128, synthetic VS q/k",
                                       "xattn": {"block": 128, "stride": 16, "threshold": a.tau}},
        "ms": ms, "density": density, "n_blk": int(idx.size),
        "attn_tflops": {"fwd": 4 * 128 * M1.sum() / ms["fwd"] / 1e9,
                        "bwd": 10 * 128 * M1.sum() / ms["bwd"] / 1e9},
        "imbalance": bal}))


if __name__ == "__main__":
    main()
