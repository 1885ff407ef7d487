"""Build the in-tree native library (nvcc, sm_100a) and the oracle checker.

    python build.py            # builds paper_2311_13862_b200/_rbws_b200.so

Every .cu is compiled to an object in parallel (build/obj), then linked.  The
.so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent
PKG = ROOT / "paper_2311_13862_b200"
CSRC = PKG / "csrc"
# RBWS_OBJ_DIR / RBWS_OUT: a variant build (A/B experiments, tools/ab_libs.sh) in its own
# object directory, so the default objects are never mixed with variant ones
OBJ = Path(os.environ["RBWS_OBJ_DIR"]) if os.environ.get("RBWS_OBJ_DIR") else ROOT / "build" / "obj"
OUT = Path(os.environ["RBWS_OUT"]) if os.environ.get("RBWS_OUT") else PKG / "_rbws_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
          "-Xcompiler", "-fPIC", "-Xptxas", "-O3"]
# extra -D definitions for A/B builds of kernel variants (e.g. RBWS_EXTRA_DEFS="RBWS_X=1 RBWS_Y=2")
CFLAGS += [f"-D{d}" for d in os.environ.get("RBWS_EXTRA_DEFS", "").split()]


def sources():
    return sorted(CSRC.glob("*.cu"))


def headers():
    return sorted(CSRC.glob("*.cuh")) + [ROOT / "include/rbws_b200.h"]


def deps():
    return sources() + headers()


def _compile(src: Path, newest_hdr: float, force: bool, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    if not force and obj.exists() and obj.stat().st_mtime >= max(newest_hdr, src.stat().st_mtime):
        return obj
    cmd = [NVCC, *CFLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=CSRC)
    return obj


def build(force: bool = False, verbose: bool = True) -> Path:
    if not force and OUT.exists():
        newest = max(p.stat().st_mtime for p in deps())
        if OUT.stat().st_mtime >= newest:
            return OUT
    OBJ.mkdir(parents=True, exist_ok=True)
    newest_hdr = max(p.stat().st_mtime for p in headers())
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, newest_hdr, force, verbose), sources()))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(OUT),
           *map(str, objs), "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=CSRC)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(f"built {OUT}")
