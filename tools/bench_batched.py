"""BASELINE config 5: many independent sequences on one GPU (one tracker per CUDA stream,
each solver a thread-block cluster), aggregate frames/s.

The 64 trackers share one synthetic config-2 scene (template built once) and each is fed
the frame sequence cycled from its own start offset; every tracker keeps its own state
(warm start, device buffers, stream). Frames of all trackers are enqueued round-robin;
the aggregate is all frames / device time (events on every stream).

    python tools/bench_batched.py [--seqs 64] [--cluster 4] [--rounds 8] [--frames 8]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=64)
    ap.add_argument("--cluster", type=int, default=4)
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--frames", type=int, default=8)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2007_08576_b200._lib import FrameInput
    from paper_2007_08576_b200._session import DeviceTracker, make_config
    from paper_2007_08576_b200.warpfield import bind_points

    wl = bench.make_workload(2, args.frames, seed=0)
    cfg, graph, feats = wl["cfg"], wl["graph"], wl["feats"]
    dcfg = make_config(wl["cam"], cfg.energy, cfg.make_solver_config(), cfg.make_preselect_config(),
                       sampling_radius=graph.sampling_radius, cluster_size=args.cluster)
    binding = bind_points(feats.points, graph.points, 4, graph.sampling_radius)
    dev = torch.device("cuda")
    frames = wl["frames"]
    F = len(frames)
    d_depth = [torch.from_numpy(f.depth).to(dev) for f in frames]
    d_desc = [torch.from_numpy(f.descriptors).to(dev) for f in frames]
    d_kp = [torch.from_numpy(f.keypoints).to(dev) for f in frames]
    streams = [torch.cuda.Stream() for _ in range(args.seqs)]
    trks = []
    for s in streams:
        t = DeviceTracker(wl["tpl"], graph, dcfg, stream=s.cuda_stream)
        t.set_features(feats.descriptors, feats.points, binding)
        trks.append(t)

    def fin(i, fid):
        fi = FrameInput()
        fi.depth, fi.frame_desc, fi.frame_kp = d_depth[i].data_ptr(), d_desc[i].data_ptr(), d_kp[i].data_ptr()
        fi.n_frame, fi.use_matches, fi.on_device, fi.frame_id = d_desc[i].shape[0], 1, 1, fid
        return fi

    for r in range(args.warmup):
        for q, t in enumerate(trks):
            t.enqueue(fin((q + r) % F, r))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    start = torch.cuda.Event(enable_timing=True)
    start.record(torch.cuda.current_stream())
    for s in streams:
        s.wait_event(start)
    for r in range(args.rounds):
        for q, t in enumerate(trks):
            t.enqueue(fin((q + args.warmup + r) % F, args.warmup + r))
    ends = []
    for s in streams:
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        ends.append(e)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev_ms = max(start.elapsed_time(e) for e in ends)
    n = args.seqs * args.rounds
    print(json.dumps({"config": 5, "sequences": args.seqs, "cluster": args.cluster,
                      "frames": n, "device_ms": dev_ms, "frames_per_s": n / (dev_ms / 1e3),
                      "wall_frames_per_s": n / wall,
                      "per_sequence_hz": args.rounds / (dev_ms / 1e3)}))
    for t in trks:
        t.close()


if __name__ == "__main__":
    main()
