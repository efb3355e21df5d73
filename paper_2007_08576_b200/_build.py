"""Build recipes for the native parts of the repo (run by __graft_entry__.build()).

* ``libdeformtrack_b200.so``: the sm_100a CUDA library behind include/deformtrack_b200.h,
  compiled in-tree with nvcc so the built .so travels with the repo snapshot.
* ``oracle/_build/liboracle.so``: the C restatement of the reference kernels
  (test infrastructure only; see oracle/README in oracle/__init__.py).

Flags: ``-fmad=false`` keeps the device evaluating the reference's IEEE operation order
(numba compiles the reference kernels with fastmath off, kernels.py:9-13), which is what
makes pixel rounding, gates and preselection flags reproduce bit for bit.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libdeformtrack_b200.so"
ORACLE_SRC = ROOT / "oracle" / "csrc"
ORACLE_LIB = ROOT / "oracle" / "_build" / "liboracle.so"

CUDA_SOURCES = ["dt_ops.cu", "dt_match.cu", "dt_solver.cu", "dt_tracker.cu", "dt_template.cu",
                "dt_orb.cu", "dt_io.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA library cannot be built")


def _stale(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build_cuda(force: bool = False, verbose: bool = False) -> Path:
    sources = [CSRC / s for s in CUDA_SOURCES]
    deps = sources + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "deformtrack_b200.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", str(tmp), *map(str, sources)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG / "build_ptxas.log"
    log.write_text(proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stderr[-6000:])
        raise RuntimeError(f"nvcc failed ({proc.returncode}); see {log}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle(force: bool = False, verbose: bool = False) -> Path:
    sources = sorted(ORACLE_SRC.glob("*.c"))
    deps = sources + sorted(ORACLE_SRC.glob("*.h"))
    if not sources:
        raise RuntimeError(f"no oracle sources under {ORACLE_SRC}")
    if not force and not _stale(ORACLE_LIB, deps):
        return ORACLE_LIB
    ORACLE_LIB.parent.mkdir(parents=True, exist_ok=True)
    tmp = ORACLE_LIB.with_suffix(".so.tmp")
    # -ffp-contract=off: no FMA contraction, the same IEEE sequence as numba's
    # fastmath-off LLVM build of the reference kernels
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", "-o", str(tmp), *map(str, sources), "-lm"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stderr[-6000:])
        raise RuntimeError(f"gcc failed for the oracle ({proc.returncode})")
    os.replace(tmp, ORACLE_LIB)
    if verbose:
        print(f"built {ORACLE_LIB}")
    return ORACLE_LIB


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_cuda(force=force, verbose=verbose)
    build_oracle(force=force, verbose=verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
