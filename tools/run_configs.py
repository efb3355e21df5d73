"""Parity + timing of the BASELINE.json configurations 1-4 on one GPU.

For each config: one frame through the device Tracker (ORB path: Hamming -> exhaustive
preselection -> LM -> warp) compared with the CPU oracle on the same inputs from the same
warm start (teacher-forced), then the device time per frame over a short sequence
(inputs resident, CUDA events of the tracker's phase profile).

    python tools/run_configs.py [--configs 1 2 3 4] [--frames 8] [--json out.json]
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


def run(cid: int, n_frames: int) -> dict:
    import torch

    import bench
    import paper_2007_08576_b200 as dt
    from oracle import pipeline as OP
    from paper_2007_08576_b200._lib import FrameInput
    from paper_2007_08576_b200._session import DeviceTracker, make_config
    from paper_2007_08576_b200.warpfield import bind_points

    wl = bench.make_workload(cid, n_frames + 1, seed=0)
    cfg, cam, tpl, graph, feats = wl["cfg"], wl["cam"], wl["tpl"], wl["graph"], wl["feats"]
    out = {"config": cid, "template_points": len(tpl), "control_points": len(graph),
           "edges": int(graph.edges.shape[0]), "image": [wl["scene"].width, wl["scene"].height],
           "lm_iterations": wl["iters"]}

    # ---- parity on frame 1 (teacher-forced from the graph's warm start) ----
    fr = wl["frames"][0]
    trk = dt.Tracker(tpl, graph, cam, cfg)
    trk.set_features(feats.descriptors, feats.points)
    trk.set_exhaustive(True)
    res = trk.track(fr.depth, descriptors=fr.descriptors, keypoints=fr.keypoints)
    trk.close()
    camt = (cam.fx, cam.fy, cam.cx, cam.cy)
    src, dst, _ = OP.matches_from_descriptors(feats.descriptors, feats.points, fr.descriptors,
                                              fr.keypoints, fr.depth, camt)
    t0 = time.perf_counter()
    tplt = (tpl.points, tpl.normals, tpl.bind_indices, tpl.bind_weights)
    grt = (graph.points, graph.edges, graph.edge_weights)
    sch = OP.Schedule(max_outer_iters=wl["iters"], step_tol=0.0, cost_tol=0.0)
    ores, osel, opts, _ = OP.track(tplt, grt, graph.warps, fr.depth,
                                   OP.observation_normals(fr.depth, *camt), camt, (src, dst),
                                   OP.Weights(), sch, graph.sampling_radius)
    out["oracle_s"] = time.perf_counter() - t0
    out["matches"] = int(len(src))
    out["matches_equal"] = bool(np.array_equal(res.matches.template_points, src)
                                and np.array_equal(res.matches.observed_points, dst))
    out["flags_equal"] = bool(np.array_equal(res.matches.preselected, osel.flags))
    out["inliers"] = int(osel.flags.sum())
    out["max_vertex_dev_mm"] = float(np.abs(res.points - opts).max())
    out["cost_rel_dev"] = float(abs(res.report.total_cost - ores.total_cost)
                                / max(ores.total_cost, 1e-30))
    out["n_corr_equal"] = int(res.report.n_correspondences) == int(ores.n_correspondences)
    out["accepted_equal"] = int(res.report.accepted_steps) == int(ores.accepted_steps)

    # ---- device time per frame ----
    dcfg = make_config(cam, cfg.energy, cfg.make_solver_config(), cfg.make_preselect_config(),
                       sampling_radius=graph.sampling_radius)
    dtrk = DeviceTracker(tpl, graph, dcfg)
    dtrk.set_features(feats.descriptors, feats.points,
                      bind_points(feats.points, graph.points, 4, graph.sampling_radius))
    dtrk.set_profiling(True)
    dev = torch.device("cuda")
    stages = []
    for i, f in enumerate(wl["frames"]):
        d = torch.from_numpy(f.depth).to(dev)
        de = torch.from_numpy(f.descriptors).to(dev)
        kp = torch.from_numpy(f.keypoints).to(dev)
        fi = FrameInput()
        fi.depth, fi.frame_desc, fi.frame_kp = d.data_ptr(), de.data_ptr(), kp.data_ptr()
        fi.n_frame, fi.use_matches, fi.on_device, fi.frame_id = de.shape[0], 1, 1, i
        fi.height, fi.width = d.shape[0], d.shape[1]
        dtrk.enqueue(fi)
        ph = dtrk.phase_ms()
        if i > 0:
            stages.append(ph)
    dtrk.close()
    st = {k: float(np.median([s[k] for s in stages])) for k in stages[0]}
    out["stage_ms"] = {k: round(v, 4) for k, v in st.items()}
    out["ms_per_frame"] = round(sum(st.values()), 4)
    out["frames_per_s"] = round(1e3 / sum(st.values()), 1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4])
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    rows = []
    for c in args.configs:
        r = run(c, args.frames)
        print(json.dumps(r), flush=True)
        rows.append(r)
    if args.json:
        Path(args.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
