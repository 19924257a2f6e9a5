"""One hot-path step (index + fwd + bwd) at a chosen size, for ncu / sanitizer runs.

  python tools/prof_step.py --seq 131072 --reps 2
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import ops  # noqa: E402
from synth.generator import make_grad_out, make_qkv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=131072)
ap.add_argument("--hq", type=int, default=16)
ap.add_argument("--hkv", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--p", type=float, default=0.9)
a = ap.parse_args()
q, k, v = make_qkv(a.seq, a.hq, a.hkv, seed=0)
dO = make_grad_out(a.seq, a.hq, seed=0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
qd, kd, vd, dd = t(q), t(k), t(v), t(dO)
for _ in range(a.reps):
    idx = ops.build_vs_index(qd, kd, a.p, a.p)
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
    g = ops.sparse_attn_bwd(qd, kd, vd, o, lse, dd, idx)
torch.cuda.synchronize()
print("ok")
