"""Committed SASS evidence for the per-frame kernels (north star: "a committed SASS
listing"): cuobjdump -sass of the built library, split per kernel, written under
profiles/<tag>_sass/<kernel>.sass, plus an opcode histogram per kernel
(profiles/<tag>_sass_histogram.json) with the instruction classes that matter here:

  UBLKCP / UTMALDG (bulk / tensor TMA copies), SYNCS (mbarrier), BAR / WARPSYNC,
  DFMA / DMUL / DADD / DMMA (FP64 pipe), MUFU, POPC / LOP3 (Hamming), LDS / STS,
  LDG / STG / LD / ST, LDL / STL (register spills), SHFL.

    python tools/sass_evidence.py [--lib paper_2007_08576_b200/libdeformtrack_b200.so] [--tag r02]
"""

from __future__ import annotations

import argparse
import json
import re
import subprocess
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

# mangled-name fragments of the per-frame kernels (config-2 grid-mode solver variant:
# GRID = true, KM = 4, BIG = false, TM = 2)
KERNELS = {
    "k_solve_frame_grid_k4_tm2": "k_solve_frameILb1ELi4ELb0ELi2E",
    "k_preselect_orb": "15k_preselect_orbE",  # fused ORB-path build + preselect + final
    "k_preselect_orb_wide": "20k_preselect_orb_wideE",  # same, 168 registers, <= 12 warps
    "k_preselect_warp": "16k_preselect_warpE",  # caller-supplied pairs / cluster mode
    "k_preselect_final": "k_preselect_final",
    "k_hamming": "9k_hamming",
    "k_build_matches": "k_build_matches",
    "k_observation_normals": "k_observation_normals",
}

CLASSES = {
    "tma_bulk": ("UBLKCP", "UTMALDG", "UTMASTG", "UBLKRED"),
    "mbarrier": ("SYNCS",),
    "barrier": ("BAR", "WARPSYNC", "MEMBAR", "ERRBAR", "CCTL"),
    "fp64": ("DFMA", "DMUL", "DADD", "DSETP", "DMMA", "DMNMX"),
    "mufu": ("MUFU",),
    "popc": ("POPC",),
    "smem": ("LDS", "STS", "LDSM", "ATOMS"),
    "global": ("LDG", "STG", "LD", "ST", "ATOMG", "RED", "ATOM"),
    "spill": ("LDL", "STL"),
    "shuffle": ("SHFL",),
}


def split_functions(sass: str) -> dict[str, list[str]]:
    funcs: dict[str, list[str]] = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs.setdefault(cur, [])
            continue
        if cur is not None:
            funcs[cur].append(line)
    return funcs


def opcodes(lines: list[str]) -> Counter:
    c: Counter = Counter()
    for line in lines:
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            c[m.group(2)] += 1
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=str(ROOT / "paper_2007_08576_b200" / "libdeformtrack_b200.so"))
    ap.add_argument("--tag", default="r02")
    args = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", args.lib], capture_output=True, text=True,
                          check=True).stdout
    funcs = split_functions(sass)
    outdir = ROOT / "profiles" / f"{args.tag}_sass"
    outdir.mkdir(parents=True, exist_ok=True)
    hist = {}
    for label, frag in KERNELS.items():
        names = [f for f in funcs if frag in f]
        if not names:
            continue
        name = names[0]
        # drop the encoding-only continuation lines (/* 0x... */)
        lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", ln) for ln in funcs[name]
                 if not re.match(r"\s+/\* 0x[0-9a-f]+ \*/\s*$", ln)]
        (outdir / f"{label}.sass").write_text(f"// {name}\n// cuobjdump -sass {Path(args.lib).name}\n"
                                              + "\n".join(lines) + "\n")
        ops = opcodes(lines)
        hist[label] = {
            "function": name,
            "instructions": int(sum(ops.values())),
            "classes": {k: int(sum(ops[o] for o in v)) for k, v in CLASSES.items()},
            "opcodes": dict(ops.most_common()),
        }
    (ROOT / "profiles" / f"{args.tag}_sass_histogram.json").write_text(json.dumps(hist, indent=1))
    for k, v in hist.items():
        print(k, v["instructions"], v["classes"])


if __name__ == "__main__":
    main()
