"""Real NCCL rings on 2 / 4 GPUs (flat and hierarchical 2x2; block-striped, and the zigzag
layout of the f1 ablation on flat rings) vs the oracle.

Each case launches tests/dist_ring_worker.py under torchrun; it is skipped when
the box has fewer GPUs than ranks (the single-GPU emulation of every ring step
is in test_gpu_attn_fwd.py / test_gpu_attn_bwd.py).
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("world,inner,layout,emu", [(2, 0, "striped", 0), (4, 0, "striped", 0),
                                                    (4, 2, "striped", 0), (2, 0, "zigzag", 0),
                                                    (4, 0, "zigzag", 0), (4, 2, "striped", 8)])
def test_ring_torchrun(world, inner, layout, emu):
    """emu > 0: f4's slow outer link (MT_EMU_INTER_GBPS GB/s between emulated 2-GPU nodes)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + world * 10 + inner + (5 if layout == 'zigzag' else 0) + (7 if emu else 0)}",
           str(ROOT / "tests" / "dist_ring_worker.py"), "--inner", str(inner), "--layout", layout]
    env = dict(os.environ)
    if emu:
        env.update(MT_EMU_INTER_GBPS=str(emu), MT_EMU_NODE="2")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    sys.stdout.write(r.stdout[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
