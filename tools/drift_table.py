"""Free-running drift at config 2 (reported, not pass/fail).

A 20-frame config-2 sequence is tracked free-running three ways, each frame warm-started
from that run's own previous solution:

* ``device``   the B200 tracker (ORB path, exhaustive preselection), as bench.py runs it;
* ``oracle``   the oracle port of the reference (bit-identical to the reference's
               numba / numpy code at solver.n_chunks = 8);
* ``oracle_c1`` the same oracle with solver.n_chunks = 1 -- only the reference's own fp64
               reduction order changes (SURVEY.md §0.7 measured 0.094-0.108 mm of drift
               from this alone on the reference).

Per frame: max |vertex difference| (mm) of device vs oracle and of oracle(n_chunks=1) vs
oracle, plus the integer report fields of each.

    python tools/drift_table.py [--frames 20] [--json profiles/r02_drift_config2.json]
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
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()

    import bench
    import paper_2007_08576_b200 as dt
    from oracle import kernels as OK
    from oracle import pipeline as OP

    OK.set_threads(OK.max_threads())
    wl = bench.make_workload(args.config, args.frames, seed=0)
    tpl, graph, cam, feats = wl["tpl"], wl["graph"], wl["cam"], wl["feats"]
    camt = (cam.fx, cam.fy, cam.cx, cam.cy)
    tplt = (tpl.points, tpl.normals, tpl.bind_indices, tpl.bind_weights)
    grt = (graph.points, graph.edges, graph.edge_weights)

    trk = dt.Tracker(tpl, graph, cam, wl["cfg"])
    trk.set_features(feats.descriptors, feats.points)
    trk.set_exhaustive(True)
    w8 = graph.warps.copy()
    w1 = graph.warps.copy()
    rows = []
    t0 = time.perf_counter()
    for i, fr in enumerate(wl["frames"]):
        res = trk.track(fr.depth, descriptors=fr.descriptors, keypoints=fr.keypoints)
        nrm = OP.observation_normals(fr.depth, *camt)
        src, dst, _ = OP.matches_from_descriptors(feats.descriptors, feats.points, fr.descriptors,
                                                  fr.keypoints, fr.depth, camt)
        out = {}
        for tag, warps, nch in (("oracle", w8, 8), ("oracle_c1", w1, 1)):
            sch = OP.Schedule(max_outer_iters=wl["iters"], step_tol=0.0, cost_tol=0.0, n_chunks=nch)
            out[tag] = OP.track(tplt, grt, warps, fr.depth, nrm, camt, (src, dst), OP.Weights(), sch,
                                graph.sampling_radius)
        r8, s8, p8, _ = out["oracle"]
        r1, s1, p1, _ = out["oracle_c1"]
        w8, w1 = r8.warps, r1.warps
        row = {
            "frame": i + 1,
            "device_vs_oracle_max_mm": float(np.abs(res.points - p8).max()),
            "oracle_nchunks1_vs_8_max_mm": float(np.abs(p1 - p8).max()),
            "n_corr": {"device": int(res.report.n_correspondences), "oracle": int(r8.n_correspondences),
                       "oracle_c1": int(r1.n_correspondences)},
            "n_preselected": {"device": int(res.report.n_preselected), "oracle": int(s8.flags.sum()),
                              "oracle_c1": int(s1.flags.sum())},
            "accepted": {"device": int(res.report.accepted_steps), "oracle": int(r8.accepted_steps)},
            "total_cost": {"device": float(res.report.total_cost), "oracle": float(r8.total_cost)},
        }
        rows.append(row)
        print(json.dumps(row), flush=True)
    trk.close()
    summary = {
        "config": args.config, "frames": args.frames,
        "control_points": len(graph), "template_points": len(tpl),
        "max_device_vs_oracle_mm": max(r["device_vs_oracle_max_mm"] for r in rows),
        "max_oracle_nchunks1_vs_8_mm": max(r["oracle_nchunks1_vs_8_max_mm"] for r in rows),
        "wall_s": time.perf_counter() - t0,
        "note": "free-running: each run warm-starts from its own previous frame; the "
                "reference against itself (n_chunks 8 -> 1) is the noise floor of free-running "
                "comparison (SURVEY.md §0.7); parity proper is teacher-forced "
                "(tests/test_gpu_configs.py)",
        "rows": rows,
    }
    if args.json:
        Path(args.json).write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))


if __name__ == "__main__":
    main()
