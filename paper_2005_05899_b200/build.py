"""Build recipe for libalyab200.so (sm_100a), in-tree so the shared object
travels to the GPU box with the repository snapshot.

    python -m paper_2005_05899_b200.build            # build if stale
    python -m paper_2005_05899_b200.build --force
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libalyab200.so"
SOURCES = ["ab_api.cu", "ab_element.cu", "ab_solver.cu", "ab_node.cu", "ab_gradop.cu", "ab_cg_dd.cu", "ab_wall.cu", "ab_io.cu"]
HEADERS = ["ab_common.cuh", "ab_cg_common.cuh", "ab_tables.inc"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "alyab200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, "-I", str(ROOT / "include"), "-o", str(LIB)] + [str(CSRC / s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    (PKG / "build.log").write_text(log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{log[-4000:]}")
    if verbose:
        print(log)
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", p)
