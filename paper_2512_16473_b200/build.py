"""Build libmoe.so (sm_100a) in-tree with nvcc. No torch extension machinery: the
library is a plain C-ABI shared object loaded through ctypes."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libmoe.so")
# the same library with the decode kernel's per-CTA debug marks compiled in (MOE_DEBUG_TS=1 with
# MOE_LIB_PATH pointing here: tools/timeline.py, bench_tp_emul.py's epilogue breakdown)
DEBUG_LIB = os.path.join(LIB_DIR, "libmoe_debug.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore
        cand = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(cand, "nccl.h")):
            return cand
    except Exception:
        pass
    for cand in ("/usr/include", "/usr/local/cuda/include"):
        if os.path.exists(os.path.join(cand, "nccl.h")):
            return cand
    raise RuntimeError("nccl.h not found (need nvidia-nccl headers)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(ROOT, "include", "moe.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(DEBUG_LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libmoe.so (or, for A/B experiments, a variant with extra -D defines at `out`,
    loaded through MOE_LIB_PATH)."""
    if out is not None:
        return _build_to(out, list(defines), verbose)
    if not force and not needs_build():
        return LIB
    _build_to(DEBUG_LIB, ["MOE_DEBUG_MARKS"], False)
    return _build_to(LIB, [], verbose)


def _build_to(LIB: str, defines: list, verbose: bool) -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared",
           "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", _nccl_include(),
           *[f"-D{d}" for d in defines], "-o", LIB + ".tmp", *sources(), "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libmoe.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
