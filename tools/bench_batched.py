"""BASELINE config 5 on one GPU outside bench.py: many independent config-2 sequences
(one tracker per CUDA stream, each solver a thread-block cluster), aggregate frames/s.
The measurement itself is bench.run_config5 (the `config5` object of the bench line).

    python tools/bench_batched.py [--seqs 64] [--cluster 8] [--rounds 8] [--frames 8]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=64)
    ap.add_argument("--cluster", type=int, default=8)
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--frames", type=int, default=8)
    args = ap.parse_args()
    import torch

    import bench

    torch.cuda.set_device(0)
    wl = bench.make_workload(2, args.frames, seed=0)
    print(json.dumps(bench.run_config5(wl, 0, 1, 0, n_seq=args.seqs, cluster=args.cluster,
                                       rounds=args.rounds, warmup=args.warmup)))


if __name__ == "__main__":
    main()
