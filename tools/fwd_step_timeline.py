"""Timeline of ONE forward ring step (rank r, origin s) at world W, emulated on one GPU
(needs a -DMT_TIMELINE -DMT_TL_FWD_TILE build).  Prints per-chunk period and the
share of tile-boundary gaps.

  python tools/fwd_step_timeline.py W r s
"""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import _lib, ops  # noqa: E402
from synth.generator import make_qkv  # noqa: E402

W, r, s = (int(x) for x in sys.argv[1:4])
S, Hq, Hkv = 524288, 16, 2
q, k, v = make_qkv(S, Hq, Hkv, seed=0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
qd, kd, vd = t(q), t(k), t(v)
idx = ops.build_vs_index(qd, kd, 0.9, 0.9)
Lq = S // W
ql, kl, vl = ops.stripe(qd, W, r), ops.stripe(kd, W, s), ops.stripe(vd, W, s)
o = torch.empty_like(ql)
oacc = torch.zeros(Lq, Hq, 128, dtype=torch.float32, device="cuda")
lse = torch.zeros(Hq, Lq, dtype=torch.float32, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.time()
    ops.attn_fwd_step(S, W, r, s, True, False, ql, kl, vl, idx, o, oacc, lse)
    torch.cuda.synchronize()
    print(f"step time {1e3 * (time.time() - t0):.2f} ms")
buf = np.zeros((8, 4096), dtype=np.int64)
_lib.check(_lib.lib().mt_debug_fwd_timeline(buf.ctypes.data_as(ctypes.c_void_p)))
if "--kprod" in sys.argv:  # MT_TL_FWD_KPROD: 3 ready, 7 vm slot, 0 K issued, 2 S issued
    E = buf.astype(np.float64)
    okk = (buf[[0, 2, 3, 7]] > 0).all(axis=0)
    okk[:16] = False
    c = np.nonzero(okk)[0]
    c = c[(c >= 2) & okk[c - 1]]
    for n, x in {"ready(c) - K issued(c-1)": E[3][c] - E[0][c - 1],
                 "ready -> vm slot": E[7][c] - E[3][c], "vm slot -> K issued": E[0][c] - E[7][c],
                 "K issued(c) - S issued(c-2)": E[0][c] - E[2][c - 2]}.items():
        print(f"  {n:28s} p50 {np.percentile(x, 50):7.0f} p90 {np.percentile(x, 90):7.0f}")
    sys.exit(0)
if "--hops" in sys.argv:  # default MT_TIMELINE build
    np.save(f"gpurun_out/fwd_step_W{W}_raw.npy", buf)
    E = buf.astype(np.float64)
    okk = (buf > 0).all(axis=0)
    okk[:16] = False
    for n, (a_, b_) in {"K load -> MMA saw K": (0, 6), "MMA saw K -> S issued": (6, 2),
                        "S issued -> WG saw S": (2, 4), "WG saw S -> P published": (4, 5),
                        "V load -> MMA saw V": (1, 7), "P published -> O issued": (5, 3)}.items():
        d = (E[b_] - E[a_])[okk]
        print(f"  {n:26s} p50 {np.percentile(d, 50):7.0f} p90 {np.percentile(d, 90):7.0f}")
    per_ = np.diff(E[2][buf[2] > 0])
    print(f"  period p50 {np.percentile(per_, 50):.0f} mean {per_.mean():.0f}")
    sys.exit(0)
S2 = buf[2].astype(np.float64)
ok = buf[2] > 0
per = np.diff(S2[ok])
first = np.nonzero((buf[0] > 0) & ok)[0]
first = first[(first > 0) & ok[first - 1]]
gap = S2[first] - S2[first - 1]
print(f"chunks {ok.sum()}, tiles {len(first)}, chunks/tile {ok.sum() / max(len(first), 1):.1f}")
print(f"period p50 {np.percentile(per, 50):.0f} mean {per.mean():.0f}; boundary gap p50 "
      f"{np.percentile(gap, 50):.0f}, share {gap.sum() / per.sum():.1%}")
for n, (a_, b_) in {"END seen -> Os drained+published": (0, 1), "published -> next Q landed": (1, 6),
                    "next Q landed -> first S": (6, 2)}.items():
    x = (buf[b_][first] - buf[a_][first]).astype(np.float64)
    print(f"  {n:36s} p50 {np.percentile(x, 50):7.0f}")
x = (buf[0][first] - S2[first - 1])
print(f"  last S -> END seen                   p50 {np.percentile(x, 50):7.0f}")
