import sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import ops
from synth.generator import make_qkv
from tests.test_gpu_block_sparse import _random_rows
from tests.gpu_util import to_dev_bf16
S, Hq, Hkv, p = 4096, 8, 1, 0.05
q, k, v = make_qkv(S, Hq, Hkv, seed=3, a=4.0)
B = _random_rows(S, Hq, 5, p)
bi = ops.BlockIndex.from_lists(B)
o, lse = ops.block_sparse_attn_fwd(to_dev_bf16(q), to_dev_bf16(k), to_dev_bf16(v), bi)
torch.cuda.synchronize()
print("fwd ok", np.isfinite(lse.cpu().numpy()).mean())
