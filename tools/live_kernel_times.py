"""Live (warm, concurrent-launch) per-kernel device times of the single-GPU hot-path step,
from CUPTI activity records via torch.profiler (no replay, no serialisation, unlike ncu's
launch list).  Reports per kernel: launches per step and mean device microseconds, plus
the step's device span (first kernel start -> last kernel end) and the idle gaps.

  python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 [--steps 10 --warmup 5]
"""
import argparse
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--hq", type=int, default=8)
    ap.add_argument("--hkv", type=int, default=1)
    ap.add_argument("--p", type=float, default=0.9)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--xattn", type=float, default=0.0,
                    help="profile the XAttention index (threshold) instead of the VS step")
    a = ap.parse_args()
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2510_18830_b200 import ops
    from synth.generator import make_grad_out, make_qkv

    dev = torch.device("cuda", 0)
    q, k, v = make_qkv(a.seq, a.hq, a.hkv, seed=a.seed)
    dO = make_grad_out(a.seq, a.hq, seed=a.seed)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).to(dev)
    qd, kd, vd, dd = t(q), t(k), t(v), t(dO)
    flush = torch.empty(4 * 126 * 2 ** 20, dtype=torch.uint8, device=dev)

    def step():
        if a.xattn > 0:
            ops.xattn_index(qd, kd, a.xattn)
            return
        idx = ops.build_vs_index(qd, kd, a.p, a.p)
        o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
        ops.sparse_attn_bwd(qd, kd, vd, o, lse, dd, idx)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            step()
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    # split into steps at the flush kernels (FillFunctor<unsigned char>)
    steps, cur = [], None
    for e in evs:
        if "FillFunctor<unsigned char>" in e.name:
            cur = []
            steps.append(cur)
        elif cur is not None:
            cur.append(e)
    per = defaultdict(list)
    spans, busy = [], []
    for s in steps:
        if not s:
            continue
        spans.append(s[-1].time_range.end - s[0].time_range.start)
        busy.append(sum(e.time_range.end - e.time_range.start for e in s))
        agg = defaultdict(float)
        for e in s:
            agg[e.name] += e.time_range.end - e.time_range.start
        for n, x in agg.items():
            per[n].append(x)
    n = len(spans)
    rows = sorted(((sum(v) / n, len(v), name) for name, v in per.items()), reverse=True)
    out = {"seq": a.seq, "hq": a.hq, "hkv": a.hkv, "steps": n,
           "span_us": float(np.median(spans)), "busy_us": float(np.median(busy)),
           "kernels": [{"us_per_step": round(x, 2), "name": name[:110]} for x, _, name in rows]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
