"""Run the forward on the bench index's bars only (slash part = the diagonal), for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_18830_b200 import ops  # noqa: E402
from synth.generator import make_qkv  # noqa: E402

S = 524288
q, k, v = make_qkv(S, 16, 2, seed=0)
t = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
qd, kd, vd = t(q), t(k), t(v)
idx = ops.build_vs_index(qd, kd, 0.9, 0.9)
iv, is_ = idx.to_lists()
mode = sys.argv[1] if len(sys.argv) > 1 else "bars"
ix = ops.VSIndex.from_lists(iv, [np.array([0], np.int32)] * 16, S) if mode == "bars" else \
    ops.VSIndex.from_lists([np.array([0], np.int32)] * 16, is_, S)
for _ in range(2):
    ops.sparse_attn_fwd(qd, kd, vd, ix)
torch.cuda.synchronize()
print("ok", mode)
