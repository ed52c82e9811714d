"""Build libsgb.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = PKG / "csrc" / "sgb.cu"
HDR = ROOT / "include" / "sgb.h"
LIB = PKG / "libsgb.so"

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "--fmad=false",  # belt and braces: every op is also an explicit *_rn intrinsic
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: libsgb.so cannot be built")


def build(force: bool = False, verbose: bool = False) -> Path:
    deps = [SRC, HDR, PKG / "csrc" / "glibc_math.h", Path(__file__)]
    if LIB.exists() and not force and LIB.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return LIB
    tmp = LIB.with_name(f"libsgb.{os.getpid()}.so")
    cmd = [nvcc(), *NVCC_FLAGS, "-I", str(ROOT / "include"), "-o", str(tmp), str(SRC)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    if verbose:
        print(proc.stderr)
    (PKG / "csrc" / "ptxas.log").write_text(proc.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
