"""Build libphobic_b200.so in-tree with nvcc for sm_100a.

The shared library is the product's compute path (include/phobic.h); it is
git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = Path(os.environ["PHB_OBJ"]) if os.environ.get("PHB_OBJ") else PKG / "_obj"
LIB = Path(os.environ["PHB_LIB"]) if os.environ.get("PHB_LIB") else PKG / "libphobic_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = os.environ.get("PHB_NVCC_EXTRA", "").split() + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-O3",
         "--expt-relaxed-constexpr"]
SOURCES = ["hash.cu", "layout.cu", "search.cu", "encode.cu", "decode.cu", "query.cu", "p2p.cu",
           "capi.cu"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [PKG.parent / "include" / "phobic.h"]

    def compile_one(src: str) -> Path:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        if force or _stale(o, [s, *headers]):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
        return o

    with ThreadPoolExecutor(max_workers=min(8, len(SOURCES))) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart_static"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
