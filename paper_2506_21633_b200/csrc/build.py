"""Build libsdgr.so (sm_100a) in-tree with nvcc.

    python -m paper_2506_21633_b200.csrc.build [--force]

The library is plain CUDA + a C ABI (include/sdgr.h); it does not link
against torch.  Objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
ROOT = PKG.parent
SOURCES = ["capi.cu", "preprocess.cu", "binning.cu", "composite.cu", "backward.cu", "train.cu", "densify.cu", "plyio.cu", "eval.cu", "stages.cu"]
HEADERS = [HERE / "common.cuh", ROOT / "include" / "sdgr.h"]
LIB = PKG / os.environ.get("SDGR_LIB_NAME", "libsdgr.so")   # profiling variants: another name
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xptxas", "-warn-spills", "-I", str(ROOT / "include")] + os.environ.get("SDGR_EXTRA_FLAGS", "").split()


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    objdir = PKG / ("_build" + os.environ.get("SDGR_BUILD_SUFFIX", ""))
    objdir.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        s = HERE / src
        o = objdir / (src + ".o")
        objs.append(o)
        if force or _stale(o, [s, *HEADERS]):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(LIB)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
