"""Build the C-ABI shared library libsplatlm_b200.so for sm_100a, in-tree.

    python -m paper_2409_12892_b200.build [--force]

Plain nvcc (no torch extension machinery): every translation unit in csrc/ is
compiled with -gencode arch=compute_100a,code=sm_100a -lineinfo and linked
into one shared object next to this file.  Re-builds only when a source is
newer than the library.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libsplatlm_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["raster.cu", "residuals.cu", "cache.cu", "jtj.cu", "stream.cu", "pcg.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-I", str(HERE.parent / "include"), "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [HERE.parent / "include" / "splatlm_b200.h"] + [Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    objdir = HERE / "_build"
    objdir.mkdir(exist_ok=True)
    objs = []
    for s in SOURCES:
        o = objdir / (Path(s).stem + ".o")
        cmd = [NVCC, *FLAGS, "-c", str(CSRC / s), "-o", str(o)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(o))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", str(tmp)]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
