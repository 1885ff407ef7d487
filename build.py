"""Build the in-tree native library (nvcc, sm_100a) and the oracle checker.

    python build.py            # builds paper_2311_13862_b200/_rbws_b200.so

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent
PKG = ROOT / "paper_2311_13862_b200"
CSRC = PKG / "csrc"
OUT = PKG / "_rbws_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-O3"]


def sources():
    return sorted(CSRC.glob("*.cu"))


def deps():
    return sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include/rbws_b200.h"]


def build(force: bool = False, verbose: bool = True) -> Path:
    if not force and OUT.exists():
        newest = max(p.stat().st_mtime for p in deps())
        if OUT.stat().st_mtime >= newest:
            return OUT
    cmd = [NVCC, *FLAGS, "-o", str(OUT), *map(str, sources())]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=CSRC)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(f"built {OUT}")
