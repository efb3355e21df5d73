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
                "dt_orb.cu", "dt_stereo.cu", "dt_io.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]
# Per-source overrides (e.g. {"dt_solver.cu": ["-fmad=true"]}: contracting the LM solver's
# tolerance-level arithmetic into FMAs was measured at config 2 -- 0.364 -> 0.369 ms, no
# gain inside the noise -- so every kernel keeps the reference's IEEE operation order).
SOURCE_FLAGS: dict[str, list[str]] = {}


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
    """One object per source (in parallel, with its SOURCE_FLAGS), then one shared link."""
    import tempfile
    from concurrent.futures import ThreadPoolExecutor

    sources = [CSRC / s for s in CUDA_SOURCES]
    deps = sources + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "deformtrack_b200.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    log = PKG / "build_ptxas.log"
    with tempfile.TemporaryDirectory(prefix="dt_build_") as tmpdir:
        def compile_one(src: Path):
            flags = list(NVCC_FLAGS)
            extra = SOURCE_FLAGS.get(src.name, [])
            if "-fmad=true" in extra:
                flags.remove("-fmad=false")
            obj = Path(tmpdir) / (src.name + ".o")
            proc = subprocess.run([_nvcc(), *flags, *extra, "-c", "-o", str(obj), str(src)],
                                  capture_output=True, text=True)
            return obj, proc

        with ThreadPoolExecutor(len(sources)) as ex:
            results = list(ex.map(compile_one, sources))
        log.write_text("".join(p.stdout + p.stderr for _, p in results))
        for _, proc in results:
            if proc.returncode != 0:
                sys.stderr.write(proc.stderr[-6000:])
                raise RuntimeError(f"nvcc failed ({proc.returncode}); see {log}")
        tmp = LIB.with_suffix(".so.tmp")
        proc = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-o", str(tmp), *(str(o) for o, _ in results)],
                              capture_output=True, text=True)
        if proc.returncode != 0:
            sys.stderr.write(proc.stderr[-6000:])
            raise RuntimeError(f"nvcc link failed ({proc.returncode})")
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
