"""Template build timing: the device build (`prepare_template`,
"exact" = bit-identical route with numpy's exp and the kd-tree binding, "device" = all on
the GPU) against the reference's algorithm on the host (oracle restatement: greedy
storage-order thinning, dense Gaussian connections, kd-tree binding), plus the point
normals of an unordered cloud (`estimate_point_normals`) against the reference's
kd-tree + eigh restatement. Parity is checked on the way (control points, edges, edge
weights, binding). Output: one JSON object (--json FILE).

    python tools/bench_template.py [--configs 2 4] [--reps 3] [--json profiles/r02_template.json]
"""

from __future__ import annotations

import argparse
import copy
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _best(fn, reps):
    best = float("inf")
    out = None
    for _ in range(reps):
        t = time.perf_counter()
        out = fn()
        best = min(best, time.perf_counter() - t)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2, 4])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import torch

    import paper_2007_08576_b200 as dt
    from oracle import pipeline as OP
    from paper_2007_08576_b200 import synth
    from paper_2007_08576_b200.config import load_config

    rows = []
    for cid in args.configs:
        spec = synth.CONFIGS[cid]
        scene = replace(spec["scene"], seed=0)
        cfg = load_config({"sampling": {"radius": spec["radius"]}})
        tpl0 = synth.make_template(scene)
        row = {"config": cid, "template_points": int(len(tpl0.points))}
        dt.prepare_template(tpl0, cfg)  # warm-up (library load, first launches)
        torch.cuda.synchronize()
        for mode in ("exact", "device"):
            c = copy.deepcopy(cfg)
            c.device.template_build = mode
            t, (tpl, graph) = _best(lambda: dt.prepare_template(tpl0, c), args.reps)
            row[f"device_{mode}_s"] = t
            row["control_points"] = int(len(graph.points))
            row["edges"] = int(len(graph.edges))
            if mode == "exact":
                ref_graph = graph
                ref_tpl = tpl
        r = cfg.sampling.radius

        def host():
            ctrl = OP.sample_controls(tpl0.points, r)
            edges, ew = OP.connections(ctrl, cfg.sampling.effective_connection_sigma)
            bi, bw = OP.bind(tpl0.points, ctrl, cfg.sampling.bind_k,
                             cfg.sampling.effective_bind_sigma)
            return ctrl, edges, ew, bi, bw

        th, (ctrl, edges, ew, bi, bw) = _best(host, 1)
        row["host_reference_algorithm_s"] = th
        row["exact_route_bit_identical"] = bool(
            np.array_equal(ctrl, ref_graph.points) and np.array_equal(edges, ref_graph.edges)
            and np.array_equal(ew, ref_graph.edge_weights)
            and np.array_equal(bi, ref_tpl.bind_indices) and np.array_equal(bw, ref_tpl.bind_weights))
        row["speedup_exact"] = th / row["device_exact_s"]
        row["speedup_device"] = th / row["device_device_s"]
        # point normals of the template cloud (k = 12)
        pts = np.ascontiguousarray(tpl0.points)
        dt.estimate_point_normals(pts[:1000])
        tn, nd = _best(lambda: dt.estimate_point_normals(pts), args.reps)
        to, (no, ties) = _best(lambda: OP.point_normals(pts), 1)
        uniq = ~ties
        row["normals_device_s"] = tn
        row["normals_host_reference_algorithm_s"] = to
        row["normals_max_dev_unique_neighbourhoods"] = float(np.abs(nd[uniq] - no[uniq]).max())
        rows.append(row)
        print(json.dumps(row))
    if args.json:
        Path(args.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
