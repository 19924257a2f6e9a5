"""The decoder layer on 2 / 4 GPUs (striped layout, distributed index, NCCL ring)
vs the same layer on one GPU (tests/dist_layer_worker.py under torchrun).  Skipped
when the box has fewer GPUs than ranks."""
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("world,inner", [(2, 0), (4, 2)])
def test_layer_ring_matches_single_gpu(world, inner):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + world * 10 + inner}",
           str(ROOT / "tests" / "dist_layer_worker.py"), "--inner", str(inner)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    sys.stdout.write(r.stdout[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
