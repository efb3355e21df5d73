"""Per-phase latency budget of one config-2 frame on the device.

Runs a few frames with profiling on and prints (a) the pipeline stages timed with CUDA
events between kernels and (b) the solver kernel's internal phases from its
globaltimer trace (work time per phase = previous barrier release -> this barrier
arrival of CTA 0; barrier = arrival -> release).

    python tools/profile_phases.py [--config 2] [--frames 4] [--cluster 0]
"""

from __future__ import annotations

import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

NAMES = {0: "start", 1: "P1 warm-start relinearization", 1.2: "  load warps + transforms",
         2: "P2 data folds", 2.2: "  accept decision", 2.3: "  data rows fold", 2.4: "  team combine",
         3: "P3 rigidity folds + solve", 3.3: "  rigidity rows fold", 3.2: "  reduce-scatter",
         3.4: "  combine + Cholesky + publish", 5.7: "  load tentative state", 5.3: "  decide reductions",
         5.4: "  step-norm / ok", 5.2: "  (unused)", 5.5: "  (unused)",
         6: "P6 value pass + speculative relinearization", 6.3: "  value totals", 6.4: "  damping update",
         6.5: "  damping history", 7.2: "final load", 8: "final support", 9: "final rigidity", 99: "end"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--json", default=None)
    ap.add_argument("--groups", default=None, help="CTA group bounds, e.g. 0,30,93,132,148")
    ap.add_argument("--all-ctas", action="store_true", help="print every CTA's mean arrival")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2007_08576_b200._lib import FrameInput
    from paper_2007_08576_b200._session import DeviceTracker, make_config
    from paper_2007_08576_b200.warpfield import bind_points

    wl = bench.make_workload(args.config, args.frames, seed=0)
    cfg = wl["cfg"]
    dcfg = make_config(wl["cam"], cfg.energy, cfg.make_solver_config(), cfg.make_preselect_config(),
                       sampling_radius=wl["graph"].sampling_radius, cluster_size=args.cluster)
    trk = DeviceTracker(wl["tpl"], wl["graph"], dcfg)
    feats = wl["feats"]
    trk.set_features(feats.descriptors, feats.points,
                     bind_points(feats.points, wl["graph"].points, 4, wl["graph"].sampling_radius))
    dev = torch.device("cuda")
    trk.set_profiling(True)
    stages = []
    work = defaultdict(float)
    wait = defaultdict(float)
    crit = defaultdict(float)   # last CTA arrival - previous release
    blat = defaultdict(float)   # release - last CTA arrival
    last_cta = defaultdict(list)
    per_cta = defaultdict(list)  # arrival - previous release, per CTA
    for i, fr in enumerate(wl["frames"]):
        d = torch.from_numpy(fr.depth).to(dev)
        de = torch.from_numpy(fr.descriptors).to(dev)
        kp = torch.from_numpy(fr.keypoints).to(dev)
        fi = FrameInput()
        fi.depth, fi.frame_desc, fi.frame_kp = d.data_ptr(), de.data_ptr(), kp.data_ptr()
        fi.n_frame, fi.use_matches, fi.on_device, fi.frame_id = de.shape[0], 1, 1, i
        fi.height, fi.width = d.shape[0], d.shape[1]
        trk.enqueue(fi)
        stages.append(trk.phase_ms())
        tr = trk.trace()
        arr = trk.arrivals()
        if i == 0:
            continue  # first frame: cold caches
        # barrier k of the frame: CTA-0 stamps (10 ph) / (10 ph + 1), arrivals row k
        rel_prev = tr[0, 1]
        k = 0
        codes = [int(c) for c in tr[:, 0]]
        for idx in range(len(codes) - 1):
            c0, c1 = codes[idx], codes[idx + 1]
            if c0 % 10 == 0 and c0 != 0 and c1 == c0 + 1 and k < arr.shape[0]:
                ph = c0 // 10
                mx = int(arr[k].max())
                crit[ph] += (mx - rel_prev) / 1e3
                blat[ph] += (tr[idx + 1, 1] - mx) / 1e3
                last_cta[ph].append(int(arr[k].argmax()))
                per_cta[ph].append((arr[k].astype(np.float64) - rel_prev) / 1e3)
                rel_prev = tr[idx + 1, 1]
                k += 1
        prev_t = tr[0, 1]
        for code, t in tr[1:]:
            ph, kind = divmod(int(code), 10)
            if code == 99:
                continue
            if kind == 1:
                wait[ph] += (t - prev_t) / 1e3
            else:
                # sub-phase stamps (kind 2, 4) split the work of phase ph
                key = ph if kind == 0 else ph + kind / 10.0
                work[key] += (t - prev_t) / 1e3
            prev_t = t
    nf = len(wl["frames"]) - 1
    st = {k: float(np.mean([s[k] for s in stages[1:]])) for k in stages[0]}
    print("pipeline stages (ms/frame):", json.dumps({k: round(v, 4) for k, v in st.items()}))
    print(f"{'solver phase':22s} {'work us/frame':>14s} {'barrier us/frame':>17s}")
    tot_w = tot_b = 0.0
    for ph in sorted(set(work) | set(wait)):
        w, b = work[ph] / nf, wait[ph] / nf
        tot_w += w
        tot_b += b
        print(f"{NAMES.get(ph, ph):22s} {w:14.1f} {b:17.1f}")
    print(f"{'total':22s} {tot_w:14.1f} {tot_b:17.1f}")
    print(f"{'barrier (phase)':22s} {'critical us/frame':>18s} {'sync us/frame':>14s} last CTAs")
    tc = tb = 0.0
    for ph in sorted(crit):
        c, b = crit[ph] / nf, blat[ph] / nf
        tc += c
        tb += b
        lc = np.bincount(last_cta[ph]).argsort()[::-1][:3].tolist()
        print(f"{NAMES.get(ph, ph):22s} {c:18.1f} {b:14.1f} {lc}")
    print(f"{'total':22s} {tc:18.1f} {tb:14.1f}")
    print("per-CTA arrival after the previous release (us/frame): median CTA, slowest CTA, "
          "and the five CTAs with the largest mean")
    for ph in sorted(per_cta):
        a = np.sum(per_cta[ph], axis=0) / nf
        top = np.argsort(a)[::-1][:5]
        print(f"{NAMES.get(ph, ph):22s} median {np.median(a):7.1f} max {a.max():7.1f}  "
              + " ".join(f"{int(c)}:{a[c]:.1f}" for c in top))
        if args.all_ctas:
            print("    " + " ".join(f"{v:.0f}" for v in a))
        if args.groups:
            g = [int(x) for x in args.groups.split(",")]
            print("    groups: " + "  ".join(f"[{lo},{hi}) {a[lo:hi].mean():.1f}"
                                           for lo, hi in zip(g[:-1], g[1:]) if hi <= a.size))
    if args.json:
        Path(args.json).write_text(json.dumps({"stages_ms": st,
                                               "solver_work_us": {NAMES.get(k, k): v / nf for k, v in work.items()},
                                               "solver_barrier_us": {NAMES.get(k, k): v / nf for k, v in wait.items()}},
                                              indent=1))
    trk.close()


if __name__ == "__main__":
    main()
