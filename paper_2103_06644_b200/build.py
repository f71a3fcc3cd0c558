"""Build the in-tree sm_100a shared library (``librangefit_b200.so``).

Plain ``nvcc -shared`` so the artefact lives in the package directory and
travels with the repository snapshot to the GPU box (no JIT cache).
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SOURCES = [PKG / "csrc" / "rf_fit.cu", PKG / "csrc" / "rf_rects.cu", PKG / "csrc" / "rf_integral.cu",
           PKG / "csrc" / "rf_render.cu", PKG / "csrc" / "rf_lattice.cu"]
HEADERS = [ROOT / "include" / "rangefit_b200.h", PKG / "csrc" / "rf_solve.cuh", PKG / "csrc" / "rf_internal.h",
           PKG / "csrc" / "rf_tile.cuh", PKG / "csrc" / "rf_general.cuh",
           PKG / "csrc" / "rf_direct.cuh", PKG / "csrc" / "rf_invn.cuh", PKG / "csrc" / "rf_jacobi.cuh"]
OUT = PKG / "librangefit_b200.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return OUT
    extra = os.environ.get("RF_NVCC_FLAGS", "").split()
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-o", str(OUT), *map(str, SOURCES)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    (PKG / "ptxas_info.txt").write_text(res.stderr)
    return OUT


if __name__ == "__main__":
    build(force=True, verbose=True)
