"""Debug: per (rank, origin) single ring steps of the forward (first = last = 1) vs the
oracle's per-step partials, reporting the worst heads / query blocks."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import ring as OR  # noqa: E402
from oracle.sparseformat import stripe_perm  # noqa: E402
from paper_2510_18830_b200 import ops  # noqa: E402
from synth.generator import make_qkv  # noqa: E402
from tests.gpu_util import f64, random_index, to_dev_bf16  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S, Hq, Hkv = 2048, 4, 2
q, k, v = make_qkv(S, Hq, Hkv, seed=6, a=6.0)
iv, is_ = random_index(S, Hq, 7, n_off=6, n_col=80)
idx = ops.VSIndex.from_lists(iv, is_, S)
perm = stripe_perm(S, W)
plans = OR._local_plans(iv, is_, S, W, 64)
Lq = S // W
q64, k64, v64 = f64(q), f64(k), f64(v)
for r in range(W):
    for s in range(W):
        o = torch.empty(Lq, Hq, 128, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(Hq, Lq, dtype=torch.float32, device="cuda")
        ops.attn_fwd_step(S, W, r, s, True, True, to_dev_bf16(q[perm[r]]), to_dev_bf16(k[perm[s]]),
                          to_dev_bf16(v[perm[s]]), idx, o, None, lse)
        torch.cuda.synchronize()
        plan_rs = [plans[h][r][s] for h in range(Hq)]
        Or, Lr = OR._step_partial(q64[perm[r]], k64[perm[s]], v64[perm[s]], plan_rs, perm[r], perm[s],
                                  Hq, Hq // Hkv, 64)
        og = o.float().cpu().numpy()
        lg = lse.cpu().numpy()
        bad = []
        for h in range(Hq):
            for j in range(Lq // 64):
                rows = slice(j * 64, j * 64 + 64)
                e = np.max(np.abs(og[rows, h] - Or[rows, h]))
                fin = np.isfinite(Lr[h, rows])
                el = np.max(np.abs(np.where(fin, lg[h, rows] - Lr[h, rows], 0))) if fin.any() else 0.0
                mism = np.any(np.isfinite(lg[h, rows]) != fin)
                if e > 0.05 or el > 1e-3 or mism:
                    bad.append((h, j, round(float(e), 3), round(float(el), 4), bool(mism)))
        print(f"r={r} s={s}: {len(bad)} bad (h, j, err_o, err_lse, inf-mismatch): {bad[:12]}")
