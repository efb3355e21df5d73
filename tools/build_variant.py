"""Build an experimental variant of libdeformtrack_b200.so into _variants/<name>.so with
extra nvcc flags (e.g. -DDT_SOLVER_THREADS=384), for A/B timing on the GPU box via
DEFORMTRACK_B200_LIB=_variants/<name>.so. Per-file flags: --solver-flags apply to
dt_solver.cu only.

    python tools/build_variant.py NAME [--flags ...] [--solver-flags ...]
"""

from __future__ import annotations

import argparse
import shlex
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--flags", default="")
    ap.add_argument("--solver-flags", default="")
    args = ap.parse_args()
    import importlib.util

    spec = importlib.util.spec_from_file_location("_b", ROOT / "paper_2007_08576_b200" / "_build.py")
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    out = ROOT / "_variants"
    out.mkdir(exist_ok=True)
    base = [f for f in b.NVCC_FLAGS if f not in ("-shared",)]
    objs = []

    def comp(src):
        o = out / f"{args.name}_{src}.o"
        extra = shlex.split(args.flags) + (shlex.split(args.solver_flags) if src == "dt_solver.cu" else [])
        fl = [f for f in base]
        if "-fmad=true" in extra:
            fl = [f for f in fl if f != "-fmad=false"]
        cmd = [b._nvcc(), *fl, *extra, "-dc" if False else "-c", "-o", str(o), str(b.CSRC / src)]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode:
            raise SystemExit(p.stderr[-4000:])
        (out / f"{args.name}_{src}.log").write_text(p.stdout + p.stderr)
        return o

    with ThreadPoolExecutor(len(b.CUDA_SOURCES)) as ex:
        objs = list(ex.map(comp, b.CUDA_SOURCES))
    so = out / f"{args.name}.so"
    p = subprocess.run([b._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(so),
                        *map(str, objs)], capture_output=True, text=True)
    if p.returncode:
        raise SystemExit(p.stderr[-4000:])
    for o in objs:
        o.unlink()
    print(so)


if __name__ == "__main__":
    main()
