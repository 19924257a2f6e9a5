"""Subprocess worker for GPU parity cases that need a process-wide environment switch
(MT_PACK_CAP, MT_FWD_PACK, MT_BWD_BAR_PART are read once per process by libmtsa.so).

  python tests/gpu_case_worker.py <case>     -> prints one JSON line, exit 0 iff in tolerance

The expected values come from oracle/ only (fp64 forward / backward on the same inputs).
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import attention as OA  # noqa: E402
from paper_2510_18830_b200 import ops  # noqa: E402
from synth.generator import make_grad_out, make_qkv  # noqa: E402
from tests.gpu_util import f64, normwise_err, to_dev_bf16  # noqa: E402

TOL, TOL_LSE = 2e-2, 1e-3


def run_full(S, Hq, Hkv, iv, is_, seed):
    q, k, v = make_qkv(S, Hq, Hkv, seed=seed, a=6.0)
    dO = make_grad_out(S, Hq, seed=seed)
    O, L = OA.sparse_attention_forward(f64(q), f64(k), f64(v), iv, is_)
    dq, dk, dv = OA.sparse_attention_backward(f64(q), f64(k), f64(v), O, L, f64(dO), iv, is_)
    idx = ops.VSIndex.from_lists(iv, is_, S)
    qd, kd, vd, dd = (to_dev_bf16(x) for x in (q, k, v, dO))
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
    g = ops.sparse_attn_bwd(qd, kd, vd, o, lse, dd, idx)
    torch.cuda.synchronize()
    cpu = lambda t: t.float().cpu().numpy().astype(np.float64)
    errs = {"o": normwise_err(cpu(o), O, 1), "lse": float(np.max(np.abs(lse.cpu().numpy() - L))),
            "dq": normwise_err(cpu(g[0]), dq, 1), "dk": normwise_err(cpu(g[1]), dk, 1),
            "dv": normwise_err(cpu(g[2]), dv, 1)}
    ok = errs["lse"] <= TOL_LSE and all(errs[x] <= TOL for x in ("o", "dq", "dk", "dv"))
    return ok, errs


def case_mixed_pack():
    # MT_PACK_CAP=256: head 0 has 700 vertical columns (> cap: cp.async gather path), head 1
    # has 120 (packed TMA path) -- one launch mixes both
    S, Hq, Hkv = 4096, 2, 1
    r = np.random.default_rng(41)
    iv = [np.unique(np.r_[0, r.choice(S, 700, replace=False)]).astype(np.int32),
          np.unique(np.r_[0, r.choice(S, 120, replace=False)]).astype(np.int32)]
    is_ = [np.unique(np.r_[0, 1, r.choice(S // 64, 5, replace=False)]).astype(np.int32) for _ in range(Hq)]
    return run_full(S, Hq, Hkv, iv, is_, seed=41)


def case_gather_only():
    # MT_FWD_PACK=0: every bar chunk through the cp.async gather path
    S, Hq, Hkv = 4096, 4, 2
    r = np.random.default_rng(42)
    iv = [np.unique(np.r_[0, r.choice(S, 300, replace=False)]).astype(np.int32) for _ in range(Hq)]
    is_ = [np.unique(np.r_[0, r.choice(S // 64, 6, replace=False)]).astype(np.int32) for _ in range(Hq)]
    return run_full(S, Hq, Hkv, iv, is_, seed=42)


def case_bar_parts():
    # MT_BWD_BAR_PART=8: the backward bar pass splits each 128-column group's query range
    # into parts of 8 blocks (the multi-part path of S_loc > 64K) at a size the oracle
    # checks in full; early columns (sink 0..3) span many parts
    S, Hq, Hkv = 8192, 2, 1
    r = np.random.default_rng(43)
    iv = [np.unique(np.r_[np.arange(4), r.choice(S, 200, replace=False)]).astype(np.int32)
          for _ in range(Hq)]
    is_ = [np.unique(np.r_[0, r.choice(S // 64, 4, replace=False)]).astype(np.int32) for _ in range(Hq)]
    return run_full(S, Hq, Hkv, iv, is_, seed=43)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    ok, errs = {"mixed_pack": case_mixed_pack, "gather_only": case_gather_only,
                "bar_parts": case_bar_parts}[sys.argv[1]]()
    print(json.dumps({"case": sys.argv[1], "ok": bool(ok), "errs": errs}))
    sys.exit(0 if ok else 1)
