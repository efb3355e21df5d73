"""ORB front end timing: one 640x480 grey image per call, host image
in, host keypoints / descriptors out (the call synchronises twice to size the sorts).

    python tools/bench_orb.py [--calls 200]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=200)
    ap.add_argument("--oracle", action="store_true", help="also time the CPU restatement")
    args = ap.parse_args()
    from paper_2007_08576_b200.orb import OrbDetector
    from tests.test_gpu_orb import textured

    imgs = [textured(480, 640, s) for s in range(8)]
    det = OrbDetector(480, 640)
    for im in imgs:
        det.detect(im)
    t0 = time.perf_counter()
    n = 0
    for i in range(args.calls):
        kp, _, _, _ = det.detect(imgs[i % len(imgs)])
        n += len(kp)
    dt = time.perf_counter() - t0
    det.close()
    out = {"image": [640, 480], "calls": args.calls, "ms_per_image": dt * 1e3 / args.calls,
           "images_per_s": args.calls / dt, "keypoints_per_image": n / args.calls}
    if args.oracle:
        from oracle import orb as O

        t0 = time.perf_counter()
        O.detect_and_describe(imgs[0])
        out["oracle_ms_per_image"] = (time.perf_counter() - t0) * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
