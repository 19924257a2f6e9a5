"""MMA-issuer view of the backward (build with -DMT_TIMELINE -DMT_TL_ISSUER2):
events per chunk: 0 S issue start, 1 S issued, 2 P start (dqfree seen), 3 P issued,
4 G start (dsfull seen), 5 G issued, 6 drain saw gdone, 7 region free."""
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
ok = (buf > 0).all(axis=0)
c = np.nonzero(ok)[0]
c = c[c > 16]
E = buf[:, c].astype(np.float64)
print("chunks", len(c))
names = ["S issue", "S->P start", "P issue", "P->G start", "G issue", "G->drain", "drain"]
for i, (a, b) in enumerate([(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7)]):
    d = E[b] - E[a]
    print(f"{names[i]:12s} p10 {np.percentile(d, 10):7.0f} p50 {np.percentile(d, 50):7.0f} p90 {np.percentile(d, 90):7.0f}")
# global ordering of issue activity: per chunk period and the busy fraction of the issuer
per = np.diff(E[0])
busy = (E[1] - E[0]) + (E[3] - E[2]) + (E[5] - E[4])
print(f"period p50 {np.percentile(per, 50):.0f} mean {per.mean():.0f}; issuer busy issuing p50 {np.percentile(busy, 50):.0f}")
# gaps: next chunk's S start vs this chunk's G end, etc.
print("S(n+1) start - G(n) end p50", np.percentile(E[0][1:] - E[5][:-1], 50))
print("P(n+1) start - G(n) end p50", np.percentile(E[2][1:] - E[5][:-1], 50))
print("G(n) start - P(n+1) end p50", np.percentile(E[4][:-1] - E[3][1:], 50))
