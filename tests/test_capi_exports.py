"""The C-ABI library loads on a CPU-only host and exports every function include/mtsa.h
declares (no compute calls: nothing here needs a GPU).  The Python binding's signature
table (_lib._SIGS) covers the same set, so no declared entry point is unreachable from
the tests and bench."""
import ctypes
import re
from pathlib import Path

from paper_2510_18830_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared():
    src = (ROOT / "include" / "mtsa.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    names = set(re.findall(r"\b(mt_[a-z0-9_]+)\s*\(", src))
    return sorted(n for n in names if not n.startswith("mt_status"))


def test_header_declares_the_boundary():
    d = declared()
    for name in ("mt_build_vs_index", "mt_sparse_attn_fwd", "mt_sparse_attn_bwd",
                 "mt_ring_attn_fwd", "mt_ring_attn_bwd", "mt_comm_create", "mt_stripe"):
        assert name in d, name


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    assert set(declared()) <= set(_lib.declared_symbols()), \
        sorted(set(declared()) - set(_lib.declared_symbols()))


def test_host_only_calls_work_without_a_gpu():
    lib = _lib.lib()
    assert lib.mt_launch_count() >= 0
    assert isinstance(lib.mt_last_error(), bytes)
    # the ring schedule is host logic (Alg. 2 origins, [step][rank]): at step t rank r
    # holds origin (r - t) mod W (reading R13)
    W = 4
    out = (ctypes.c_int * (W * W))()
    _lib.check(lib.mt_ring_schedule(W, W, out))
    assert [out[t * W + r] for t in range(W) for r in range(W)] == \
        [(r - t) % W for t in range(W) for r in range(W)]


def test_shape_validation_runs_before_any_device_work():
    """mt_shape checks (include/mtsa.h) are host logic: d, block, last_q (reading R2: 64, 0 = 64)
    and the layout field are rejected with their status codes before any CUDA call."""
    from paper_2510_18830_b200 import ops
    lib = _lib.lib()
    prm = ops.VSParams(0.9, 0.9)

    def status(**kw):
        sh = ops.shape(4096, 8, 1)
        for k, v in kw.items():
            setattr(sh, k, v)
        return lib.mt_build_vs_index(None, ctypes.byref(sh), ctypes.byref(prm), None, None, None,
                                     None, 0, None)
    assert status(head_dim=64) == 7      # MT_EUNSUPPORTED
    assert status(block=32) == 7
    assert status(last_q=32) == 7
    assert status(layout=5) == 1         # MT_ESHAPE
    assert status(seq_len=4000) == 2     # MT_EWINDOW
