"""Build libmtsa.so (every CUDA source in csrc/) in-tree for sm_100a.

nvcc cross-compiles without a GPU, so this runs on the CPU dev host as well as
on the GPU box.  Objects are cached by mtime under build/.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "mtsa"
LIB = PKG / "libmtsa.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs() -> tuple[Path, Path] | None:
    try:
        import nvidia.nccl  # type: ignore

        base = Path(list(nvidia.nccl.__path__)[0])
    except Exception:
        return None
    inc, lib = base / "include", base / "lib"
    if (inc / "nccl.h").exists() and (lib / "libnccl.so.2").exists():
        return inc, lib
    return None


def _flags() -> list[str]:
    f = ["-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O3",
         "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
    nccl = _nccl_dirs()
    if nccl:
        f += ["-I", str(nccl[0]), "-DMT_HAVE_NCCL=1"]
    f += os.environ.get("MT_NVCC_EXTRA", "").split()  # e.g. a shorter spin timeout for debugging
    return f


def _compile(src: Path, verbose: bool) -> Path:
    obj = BUILD / (src.stem + ".o")
    deps = [src] + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "mtsa.h"]
    if obj.exists() and obj.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return obj
    cmd = [NVCC, *_flags(), "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    stamp = BUILD / "flags.txt"  # objects built with other flags are stale
    flags = " ".join(_flags())
    if not stamp.exists() or stamp.read_text() != flags:
        for o in BUILD.glob("*.o"):
            o.unlink()
        stamp.write_text(flags)
    srcs = sorted(CSRC.glob("*.cu"))
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if LIB.exists() and LIB.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return LIB
    link = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
            "-lcublas", "-Xlinker=-rpath,/usr/local/cuda/lib64"]
    nccl = _nccl_dirs()
    if nccl:
        link += ["-L", str(nccl[1]), "-l:libnccl.so.2", f"-Xlinker=-rpath,{nccl[1]}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
