"""Forward / backward time of the bench's 512K index split into its slash part and
its vertical (bar) part: per-pair rates of each (DESIGN.md §4.2 / §4.3)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_18830_b200 import ops, stats  # noqa: E402
from synth.generator import make_grad_out, make_qkv  # noqa: E402

S, Hq, Hkv = 524288, 16, 2
q, k, v = make_qkv(S, Hq, Hkv, seed=0)
dO = make_grad_out(S, Hq, seed=0)
t = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
qd, kd, vd, dd = t(q), t(k), t(v), t(dO)
idx = ops.build_vs_index(qd, kd, 0.9, 0.9)
iv, is_ = idx.to_lists()
cases = {"full": (iv, is_),
         "slash_only": ([np.array([0], np.int32)] * Hq, is_),
         "bars_plus_diag": (iv, [np.array([0], np.int32)] * Hq)}
ev = lambda: torch.cuda.Event(enable_timing=True)
out = {}
for name, (a, b) in cases.items():
    ix = ops.VSIndex.from_lists(a, b, S)
    pairs = int(stats.pairs_per_head(a, b, S).sum())
    tf, tb = [], []
    for it in range(4):
        e = [ev() for _ in range(3)]
        e[0].record()
        o, lse = ops.sparse_attn_fwd(qd, kd, vd, ix)
        e[1].record()
        ops.sparse_attn_bwd(qd, kd, vd, o, lse, dd, ix)
        e[2].record()
        torch.cuda.synchronize()
        if it:
            tf.append(e[0].elapsed_time(e[1]))
            tb.append(e[1].elapsed_time(e[2]))
    f, b_ = float(np.median(tf)), float(np.median(tb))
    out[name] = {"pairs": pairs, "fwd_ms": f, "bwd_ms": b_,
                 "fwd_tflops": 4 * 128 * pairs / f / 1e9, "bwd_tflops": 10 * 128 * pairs / b_ / 1e9}
print(json.dumps(out))
