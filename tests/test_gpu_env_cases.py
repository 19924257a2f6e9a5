"""GPU parity of kernel paths that the default configuration only takes at large sizes,
forced at small sizes through process-wide switches (each case in its own process:
libmtsa.so reads the switches once).  Worker: tests/gpu_case_worker.py; expected values
from the fp64 oracle only.

* mixed_pack  (MT_PACK_CAP=256): one forward launch with a head above the packed-row
  capacity (cp.async gather of bar rows) and a head below it (packed TMA bar chunks);
* gather_only (MT_FWD_PACK=0): every forward bar chunk through the gather path;
* bar_parts   (MT_BWD_BAR_PART=8): the backward bar pass split into query-range parts
  (the path S_loc > 64K takes), sink columns 0..3 spanning every part.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("case,env", [("mixed_pack", {"MT_PACK_CAP": "256"}),
                                      ("gather_only", {"MT_FWD_PACK": "0"}),
                                      ("bar_parts", {"MT_BWD_BAR_PART": "8"})])
def test_env_case(cuda_lib, case, env):
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "gpu_case_worker.py"), case],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert line, r.stdout + r.stderr
    res = json.loads(line[-1])
    print(res)
    assert r.returncode == 0 and res["ok"], res
