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
SOURCES = ["ab_api.cu", "ab_element.cu", "ab_solver.cu", "ab_node.cu", "ab_gradop.cu", "ab_cg_dd.cu", "ab_wall.cu", "ab_io.cu", "ab_peer.cu", "ab_session.cu"]
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
    """Compile every source to an object in parallel (nvcc per file), then
    link the shared object."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]

    def compile_one(src: str):
        obj = objdir / (Path(src).stem + ".o")
        cmd = [NVCC, *cflags, "-c", "-I", str(ROOT / "include"), "-o", str(obj), str(CSRC / src)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, r.returncode, r.stdout + r.stderr

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = "".join(f"== {s}\n{out}" for s, (_o, _rc, out) in zip(SOURCES, results))
    bad = [s for s, (_o, rc, _out) in zip(SOURCES, results) if rc != 0]
    if not bad:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp)] + [
            str(o) for o, _rc, _out in results]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log += "== link\n" + r.stdout + r.stderr
        if r.returncode != 0:
            bad = ["link"]
        else:
            os.replace(tmp, LIB)
    (PKG / "build.log").write_text(log)
    if bad:
        raise RuntimeError(f"nvcc failed ({bad}):\n{log[-4000:]}")
    if verbose:
        print(log)
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", p)
