"""Build the in-tree CUDA library libmirrorbreak_b200.so for sm_100a.

nvcc cross-compiles without a GPU, so this runs in the build container; the
resulting .so travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib" / "libmirrorbreak_b200.so"
SOURCES = ["mb_kernels.cu", "mb_tc.cu", "mb_eig.cu", "mb_engine.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "-I", str(ROOT / "include"), "-I", str(CSRC)]


def _nvcc() -> str:
    cand = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return cand if Path(cand).exists() else "nvcc"


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "mirrorbreak_b200.h"]
    return all(d.stat().st_mtime <= t for d in deps)


def _flags() -> list:
    # MB_DEBUG_BUILD=1 compiles in the debug-only logs / dumps (mb_debug_env)
    return FLAGS + (["-DMB_DEBUG_LOGS=1"] if os.environ.get("MB_DEBUG_BUILD") == "1" else [])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:  # the translation units are independent: compile them concurrently
        obj = OUT.parent / (Path(src).stem + ".o")
        cmd = [_nvcc(), *ARCH, *_flags(), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd)))
        objs.append(str(obj))
    for cmd, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    cmd = [_nvcc(), *ARCH, "-shared", "-o", str(OUT), *objs, "-lcudart"]
    subprocess.run(cmd, check=True)
    for o in objs:
        Path(o).unlink(missing_ok=True)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
