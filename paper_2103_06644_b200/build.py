"""Build the in-tree sm_100a shared library (``librangefit_b200.so``).

Plain ``nvcc -shared`` so the artefact lives in the package directory and
travels with the repository snapshot to the GPU box (no JIT cache).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import tempfile
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SOURCES = [PKG / "csrc" / "rf_fit_k1.cu", PKG / "csrc" / "rf_fit_k2.cu", PKG / "csrc" / "rf_fit_k3.cu",
           PKG / "csrc" / "rf_fit.cu", PKG / "csrc" / "rf_rects.cu", PKG / "csrc" / "rf_integral.cu",
           PKG / "csrc" / "rf_render.cu", PKG / "csrc" / "rf_lattice.cu"]
HEADERS = [ROOT / "include" / "rangefit_b200.h", PKG / "csrc" / "rf_solve.cuh", PKG / "csrc" / "rf_internal.h",
           PKG / "csrc" / "rf_tile.cuh", PKG / "csrc" / "rf_general.cuh",
           PKG / "csrc" / "rf_direct.cuh", PKG / "csrc" / "rf_invn.cuh", PKG / "csrc" / "rf_jacobi.cuh", PKG / "csrc" / "rf_tile_kernel.cuh"]
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


def build(force: bool = False, verbose: bool = False, out: Path = OUT, extra_flags=()) -> Path:
    """Compile every translation unit in parallel (one nvcc per .cu, -c), then link the
    shared library; ptxas register/spill reports go to ptxas_info.txt."""
    if not force and out == OUT and not needs_build():
        return OUT
    extra = [*os.environ.get("RF_NVCC_FLAGS", "").split(), *extra_flags]
    objdir = Path(tempfile.mkdtemp(prefix="rf_build_"))
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    procs = []
    for src in SOURCES:
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), *flags, *extra, "-I", str(ROOT / "include"), "-c", "-o", str(obj), str(src)]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    logs, objs = [], []
    for src, obj, proc in procs:
        o, e = proc.communicate()
        logs.append(e)
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name} ({proc.returncode}):\n{o}\n{e}")
        objs.append(str(obj))
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", str(out), *objs]
    res = subprocess.run(link, capture_output=True, text=True)
    shutil.rmtree(objdir, ignore_errors=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print("".join(logs))
    if out == OUT:
        (PKG / "ptxas_info.txt").write_text("".join(logs))
    return out


if __name__ == "__main__":
    build(force=True, verbose=True)
