"""Build recipe for the native pieces (no setuptools, no JIT cache).

* ``libgtb200.so`` — every ``csrc/*.cu`` compiled for sm_100a only
  (``-gencode arch=compute_100a,code=sm_100a``) and linked in-tree next to
  this file, so the built library travels with the repository snapshot.
* ``oracle/_build/liboracle.so`` — the C restatement of the reference's
  algorithms used by the tests and the CPU baseline as a checker.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libgtb200.so"
OBJ_DIR = REPO / "build" / "obj"
ORACLE_SRC = REPO / "oracle" / "fast_oracle.c"
ORACLE_LIB = REPO / "oracle" / "_build" / "liboracle.so"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH_FLAGS + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; cannot build libgtb200.so")
    return cand


def _newest_input_mtime() -> float:
    files = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh"))
    files.append(REPO / "include" / "gtb200.h")
    files.append(Path(__file__))
    return max(f.stat().st_mtime for f in files)


def _run(cmd, cwd=None):
    proc = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"command failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    return proc


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/*.cu into libgtb200.so (skipped when up to date)."""
    if (not force and LIB_PATH.exists()
            and LIB_PATH.stat().st_mtime >= _newest_input_mtime()):
        return LIB_PATH
    nvcc = _nvcc()
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu"))

    def compile_one(src: Path) -> Path:
        obj = OBJ_DIR / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        proc = _run(cmd)
        if verbose and proc.stderr:
            print(proc.stderr)
        return obj

    workers = max(1, min(len(sources), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        objs = list(pool.map(compile_one, sources))
    tmp = LIB_PATH.with_suffix(".so.tmp")
    _run([nvcc, *ARCH_FLAGS, "-shared", "-o", str(tmp), *map(str, objs)])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def build_oracle(force: bool = False) -> Path:
    """Compile the C oracle (test infrastructure only)."""
    if (not force and ORACLE_LIB.exists()
            and ORACLE_LIB.stat().st_mtime >= ORACLE_SRC.stat().st_mtime):
        return ORACLE_LIB
    ORACLE_LIB.parent.mkdir(parents=True, exist_ok=True)
    cc = shutil.which("gcc") or "cc"
    tmp = ORACLE_LIB.with_suffix(".so.tmp")
    _run([cc, "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", str(tmp), str(ORACLE_SRC)])
    os.replace(tmp, ORACLE_LIB)
    return ORACLE_LIB


if __name__ == "__main__":
    print(build_native(force=True, verbose=True))
