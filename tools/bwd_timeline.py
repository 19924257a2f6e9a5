"""Backward pipeline timeline (needs a -DMT_TIMELINE build): runs index + fwd +
bwd at one size, reads CTA 0's per-chunk clock64 stamps and prints latency
percentiles of every pipeline hop.

Events (per producer chunk event c): 0 stage acquired / loads issued,
1 MMA warp saw full, 2 S^T/dP^T issued, 3 gradient MMAs issued,
4 softmax warpgroup saw S, 5 P/dS^T published, 6 gradients done, 7 dQ reduce issued.
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import _lib, ops  # noqa: E402
from synth.generator import make_grad_out, make_qkv  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 524288
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
# the bar launch ran last and overwrote events it reached; use chunks that have
# all eight stamps in increasing order of the pipeline
print("stamped chunk events per event:", (buf > 0).sum(axis=1).tolist())
ok = (buf > 0).all(axis=0)
c = np.nonzero(ok)[0]
c = c[c > 16]
E = buf[:, c].astype(np.float64)
names = ["load issued->data in smem", "data in smem->S issued", "S issued->WG sees S", "WG sees S->P/dS published",
         "P/dS published->G issued", "G issued->G done(WG)", "G done->dQ reduce issued"]
hops = [(0, 1), (1, 2), (2, 4), (4, 5), (5, 3), (3, 6), (6, 7)]
print(f"chunks with full stamps: {len(c)}")
for (a, b), n in zip(hops, names):
    d = E[b] - E[a]
    print(f"{n:32s} p10 {np.percentile(d, 10):8.0f}  p50 {np.percentile(d, 50):8.0f}  "
          f"p90 {np.percentile(d, 90):8.0f}  mean {d.mean():8.0f} clk")
if "--wgsplit" in sys.argv:  # MT_TL_WGSPLIT: 6 = math done, 7 = staging buffer free
    for n, (a_, b_) in {"WG sees S -> math done": (4, 6), "math done -> staging free": (6, 7),
                        "staging free -> published": (7, 5)}.items():
        d = E[b_] - E[a_]
        print(f"{n:34s} p10 {np.percentile(d, 10):7.0f} p50 {np.percentile(d, 50):7.0f} p90 {np.percentile(d, 90):7.0f}")
if "--issuer" in sys.argv:
    for n, (a, b) in {"publish -> G waits pass": (5, 6), "G waits pass -> G issued": (6, 3),
                      "S waits pass -> S issued": (7, 2), "data in smem -> S waits pass": (1, 7),
                      "S issued(k) -> S waits pass(k+1)": (0, 0)}.items():
        if n.startswith("S issued(k)"):
            d = E[7][1:] - E[2][:-1]
        else:  # noqa
            d = E[b] - E[a]
        print(f"{n:34s} p10 {np.percentile(d, 10):7.0f} p50 {np.percentile(d, 50):7.0f} p90 {np.percentile(d, 90):7.0f}")
if "--warps" in sys.argv:
    for w in range(4):
        d = E[4 + w] - E[2]
        print(f"S issued -> warp {w} published: p50 {np.percentile(d, 50):.0f} p90 {np.percentile(d, 90):.0f}")
    d = E[3] - E[4:8].max(axis=0)
    print(f"last warp published -> G issued: p50 {np.percentile(d, 50):.0f} p90 {np.percentile(d, 90):.0f}")
per = np.diff(E[2])
print(f"S-issue period (per chunk): p50 {np.percentile(per, 50):.0f} mean {per.mean():.0f} clk")
occ = E[3] - E[0]
print(f"stage occupancy (acquire -> gradients issued): p50 {np.percentile(occ, 50):.0f} clk")
