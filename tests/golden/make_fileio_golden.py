"""Golden FILES written by the REFERENCE's own writers (deformtrack/fileio.py), for the
byte-for-byte format tests of paper_2007_08576_b200.fileio (tests/test_fileio.py).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fileio_golden.py

Inputs are seeded and include reals whose repr needs the exponent form, negative zero,
integers-valued doubles and 17-digit values; the source arrays go to fileio_src.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from deformtrack import fileio as RF  # noqa: E402
from deformtrack.matching import MatchSet  # noqa: E402

OUT = Path(__file__).resolve().parent / "fileio"


def main() -> None:
    OUT.mkdir(exist_ok=True)
    rng = np.random.default_rng(11)
    pts = rng.normal(scale=50.0, size=(64, 3)) + np.array([0.0, 0.0, 300.0])
    nrm = rng.normal(size=(64, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    # values whose repr takes every layout branch
    pts[0] = [1e-5, 1e16, -0.0]
    pts[1] = [1234567890123456.0, 0.1, 5e-324]
    pts[2] = [3.0, -2.5e-7, 123456789012345678.0]
    nrm[0] = [0.0, 1.0, -1.0]
    depth = rng.uniform(250.0, 350.0, size=(13, 17))
    depth[2, 3] = np.nan
    depth[5, 0] = 0.0
    m = MatchSet(pts[:10].copy(), pts[10:20].copy(), rng.uniform(0, 1, 10),
                 rng.uniform(0, 1, 10) > 0.5)
    RF.write_ply(OUT / "cloud_ascii.ply", pts, nrm)
    RF.write_ply(OUT / "cloud_binary.ply", pts, nrm, binary=True)
    RF.write_ply(OUT / "points_only.ply", pts)
    RF.write_ply(OUT / "empty.ply", np.zeros((0, 3)))
    RF.write_pfm(OUT / "depth.pfm", depth)
    RF.write_matches(OUT / "matches.json", m)
    RF.write_json(OUT / "report.json", {"b": 1.5, "a": [1, 2, {"z": 0.1, "y": -3.0}],
                                        "e": 1e-12, "n": None, "t": True})
    RF.write_metrics_csv(OUT / "metrics.csv", [
        {"frame": "f0", "rmse_mm": 3.0, "mean_mm": 2.0, "max_mm": 5.0, "std_mm": 1.0},
        {"frame": "f1", "rmse_mm": 0.1, "mean_mm": 4.0, "max_mm": 7e-5, "std_mm": 3.0}])
    np.savez(OUT / "fileio_src.npz", pts=pts, nrm=nrm, depth=depth, m_src=m.template_points,
             m_dst=m.observed_points, m_w=m.weights, m_f=m.preselected)
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
