"""Appendix C latency model (paper_2510_18830_b200/latency_model.py) fed with
B200 step logs: the ring step profile bench.py records under torchrun (rank 0's per-step
compute and transfer times, CUDA events) -> the model's forward / backward pass times,
against the measured phase times of the same run.  Writes profiles/r02_latency_calibration.json.

  python tools/latency_calibrate.py profiles/r02_ce_n2_1.json profiles/r02_ce_n4_1.json ...
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import latency_model as LM  # noqa: E402

out = []
for f in sys.argv[1:]:
    d = json.loads(Path(f).read_text())
    W = d["n_gpus"]
    ph = d["roofline"]["phase_ms"]
    row = {"run": Path(f).name, "world": W, "seq_len": d["config"]["seq_len"]}
    for name, key in (("fwd", "fwd"), ("bwd", "bwd")):
        p = d["ring"]["passes"][name]
        comp = np.array(p["compute_ms_per_step"])
        t_comp = float(comp.mean())
        t_xfer = float(p.get("kv_ms_median", 0.0)) + (float(p.get("dkv_ms_median", 0.0)) if name == "bwd" else 0.0)
        # flat ring, every hop intra-node (one NVSwitch box): T_inter = T_intra
        pred = LM.flat_ring_total(0.0, 0.0, t_comp, t_xfer, t_xfer, W)
        # lockstep with unequal steps: the sum of the steps (rank 0's) bounds it from below
        row[name] = {"t_comp_mean_ms": round(t_comp, 3), "t_transfer_ms": round(t_xfer, 3),
                     "model_ms": round(pred, 3), "sum_of_steps_ms": round(float(comp.sum()), 3),
                     "measured_ms": ph[key], "model_over_measured": round(pred / ph[key], 3)}
    out.append(row)
    print(json.dumps(row))
Path("profiles/r02_latency_calibration.json").write_text(json.dumps(out, indent=1) + "\n")
