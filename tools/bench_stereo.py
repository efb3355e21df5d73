"""Device stereo depth at the benchmark image size (640x480, 64 disparities, 7x7 ZNCC):
ms per pair with the images resident on the device, and the oracle's time beside it.

    python tools/bench_stereo.py [--json profiles/r02_stereo.json]
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
    ap.add_argument("--json", default=None)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch

    from oracle import stereo as OS
    from paper_2007_08576_b200.stereo import StereoMatcher

    h, w, fx, B, D, r = 480, 640, 1296.0, 5.0, 64, 3
    surf = lambda y, x: 300.0 + 15.0 * np.sin(x / 60.0) + 10.0 * np.cos(y / 45.0)  # noqa: E731
    L, R, z, _ = OS.synthetic_pair(h, w, fx, B, surf, seed=0)
    sm = StereoMatcher(h, w, fx, B, max_disp=D, radius=r)
    dl, dr = torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()
    sm.compute(dl, dr, on_device=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.reps):
        dep, _, _ = sm.compute(dl, dr, on_device=True)
    dev_ms = (time.perf_counter() - t0) * 1e3 / args.reps
    t0 = time.perf_counter()
    odep, _, _ = OS.stereo_depth(L, R, D, r, fx, B)
    ora_s = time.perf_counter() - t0
    ok = np.isfinite(dep)
    out = {"image": [w, h], "max_disp": D, "window": 2 * r + 1,
           "device_ms_per_pair_incl_d2h": dev_ms, "oracle_s": ora_s,
           "bit_identical_to_oracle": bool(np.array_equal(np.isnan(dep), np.isnan(odep))
                                           and np.array_equal(dep[ok], odep[ok])),
           "valid_fraction": float(ok.mean()),
           "median_abs_depth_error_mm": float(np.median(np.abs(dep - z)[ok]))}
    print(json.dumps(out))
    if args.json:
        Path(args.json).write_text(json.dumps(out, indent=1))
    sm.close()


if __name__ == "__main__":
    main()
