"""Forward pipeline timeline (needs a -DMT_TIMELINE build): per data chunk of CTA 0,
0 K load issued, 1 V load issued, 6 MMA warp saw K, 2 S^T issued, 4 softmax saw S^T,
5 P^T published, 7 MMA warp saw V, 3 O^T issued."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import _lib, ops  # noqa: E402
from synth.generator import make_qkv  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 524288
q, k, v = make_qkv(S, 16, 2, seed=0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
qd, kd, vd = t(q), t(k), t(v)
idx = ops.build_vs_index(qd, kd, 0.9, 0.9)
if "--bars" in sys.argv:  # the bench index's bars only (slash part reduced to the diagonal)
    iv, _ = idx.to_lists()
    idx = ops.VSIndex.from_lists(iv, [np.array([0], np.int32)] * 16, S)
for _ in range(2):
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
torch.cuda.synchronize()
buf = np.zeros((8, 4096), dtype=np.int64)
_lib.check(_lib.lib().mt_debug_fwd_timeline(buf.ctypes.data_as(ctypes.c_void_p)))
print("stamped per event:", (buf > 0).sum(axis=1).tolist())
np.save("gpurun_out/fwd_timeline_raw.npy", buf)
if "--tile" in sys.argv:  # MT_TL_FWD_TILE build: 0 END seen, 1 END published, 6 next Q landed
    first = np.nonzero((buf[0] > 0) & (buf[2] > 0))[0]
    first = first[(first > 0) & (buf[2][first - 1] > 0)]
    S2 = buf[2].astype(np.float64)
    gap = S2[first] - S2[first - 1]
    per = np.diff(S2[(buf[2] > 0)])
    print(f"tiles seen: {len(first)}; chunks/tile ~ {4096 / max(len(first), 1):.1f}")
    print(f"boundary gap (last S -> next tile's first S): p50 {np.percentile(gap, 50):.0f} mean {gap.mean():.0f}")
    print(f"  share of all S-issue time spent in boundary gaps: {gap.sum() / per.sum():.2%}")
    for n, (a_, b_) in {"last S -> END seen": (None, 0), "END seen -> Os drained+published": (0, 1),
                        "published -> next Q landed": (1, 6), "next Q landed -> first S": (6, 2)}.items():
        x = (buf[b_][first] - (S2[first - 1] if a_ is None else buf[a_][first])).astype(np.float64)
        print(f"  {n:36s} p50 {np.percentile(x, 50):7.0f} mean {x.mean():7.0f}")
    sys.exit(0)
c = np.nonzero((buf > 0).all(axis=0))[0]
c = c[c > 16]
E = buf[:, c].astype(np.float64)
for n, (a, b) in {"K load -> MMA saw K": (0, 6), "MMA saw K -> S issued": (6, 2),
                  "S issued -> WG saw S": (2, 4), "WG saw S -> P published": (4, 5),
                  "V load -> MMA saw V": (1, 7), "P published -> O issued": (5, 3),
                  "MMA saw V -> O issued": (7, 3), "S issued -> O issued": (2, 3)}.items():
    d = E[b] - E[a]
    print(f"{n:26s} p10 {np.percentile(d, 10):7.0f} p50 {np.percentile(d, 50):7.0f} p90 {np.percentile(d, 90):7.0f}")
if "--wg" in sys.argv:  # event 1 = softmax math done (MT_TL_FWD_WG build)
    for n, (a_, b_) in {"WG saw S -> math done": (4, 1), "math done -> P published (P buffer wait)": (1, 5)}.items():
        d = E[b_] - E[a_]
        print(f"{n:42s} p10 {np.percentile(d, 10):7.0f} p50 {np.percentile(d, 50):7.0f} p90 {np.percentile(d, 90):7.0f}")
per = np.diff(E[2])
print(f"S-issue period: p50 {np.percentile(per, 50):.0f} mean {per.mean():.0f} clk")
