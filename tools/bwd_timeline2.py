"""Backward pipeline timeline, round-2 layout (needs a -DMT_TIMELINE build).

Events per producer chunk event c (CTA 0): 0 stage acquired, 1 data landed (observer),
2 dP^T issued (S^T before it), 3 gradients issued, 4 softmax warps saw S/dP,
5 P/dS^T published, 6 drain warps saw gradients done, 7 dQ^T read (region free).
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import _lib, ops  # noqa: E402
from synth.generator import make_grad_out, make_qkv  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
q, k, v = make_qkv(S, 16, 2, seed=0)
dO = make_grad_out(S, 16, seed=0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
qd, kd, vd, dd = t(q), t(k), t(v), t(dO)
for _ in range(2):
    idx = ops.build_vs_index(qd, kd, 0.9, 0.9)
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
    g = ops.sparse_attn_bwd(qd, kd, vd, o, lse, dd, idx)
torch.cuda.synchronize()
buf = np.zeros((8, 4096), dtype=np.int64)
_lib.check(_lib.lib().mt_debug_bwd_timeline(buf.ctypes.data_as(ctypes.c_void_p)))
print("stamped chunk events per event:", (buf > 0).sum(axis=1).tolist())
ok = (buf > 0).all(axis=0)
c = np.nonzero(ok)[0]
c = c[c > 16]
E = buf[:, c].astype(np.float64)
hops = {"acquire -> landed": (0, 1), "landed -> dP issued": (1, 2), "dP issued -> WG sees": (2, 4),
        "WG sees -> published": (4, 5), "published -> G issued": (5, 3),
        "G issued -> drain sees done": (3, 6), "drain sees done -> region free": (6, 7)}
print(f"chunks with full stamps: {len(c)}")
for n, (a, b) in hops.items():
    d = E[b] - E[a]
    print(f"{n:32s} p10 {np.percentile(d, 10):8.0f}  p50 {np.percentile(d, 50):8.0f}  "
          f"p90 {np.percentile(d, 90):8.0f}")
for n, e in (("dP issue", 2), ("G issue", 3), ("publish", 5)):
    per = np.diff(E[e])
    print(f"{n} period: p50 {np.percentile(per, 50):.0f} mean {per.mean():.0f} clk")
# next chunk's dP issue relative to this chunk's region free (2 chunks later uses it)
d = E[2][2:] - E[7][:-2]
print(f"region free (n) -> dP issued (n+2): p50 {np.percentile(d, 50):.0f} p10 {np.percentile(d, 10):.0f}")
d = E[4][1:] - E[5][:-1]
print(f"published (n) -> WG sees (n+1): p50 {np.percentile(d, 50):.0f} p10 {np.percentile(d, 10):.0f}")
