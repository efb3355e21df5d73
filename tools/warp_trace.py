"""Debug: per-warp end times of the first value pass of outer iteration 1, relative to the
barrier release before it (library built with -DDT_WARP_TRACE into variants/)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def point_stamps(buf, n_cta=8, nw=8):
    """clock64 stamps inside point_step (debug build) for lane 0 of each warp of CTAs 0..7."""
    base = 2 + 1024 * 256 + 20000
    out = buf[base: base + n_cta * nw * 8].reshape(n_cta, nw, 8)
    return out


def main():
    import bench
    from paper_2007_08576_b200._lib import FrameInput, lib
    from paper_2007_08576_b200._session import DeviceTracker, make_config, _host_ptr
    from paper_2007_08576_b200.warpfield import bind_points
    import torch

    wl = bench.make_workload(2, 3, seed=0)
    cfg = wl["cfg"]
    dcfg = make_config(wl["cam"], cfg.energy, cfg.make_solver_config(), cfg.make_preselect_config(),
                       sampling_radius=wl["graph"].sampling_radius)
    trk = DeviceTracker(wl["tpl"], wl["graph"], dcfg)
    feats = wl["feats"]
    trk.set_features(feats.descriptors, feats.points,
                     bind_points(feats.points, wl["graph"].points, 4, wl["graph"].sampling_radius))
    trk.set_profiling(True)
    dev = torch.device("cuda")
    for i, fr in enumerate(wl["frames"]):
        d = torch.from_numpy(fr.depth).to(dev)
        de = torch.from_numpy(fr.descriptors).to(dev)
        kp = torch.from_numpy(fr.keypoints).to(dev)
        fi = FrameInput()
        fi.depth, fi.frame_desc, fi.frame_kp = d.data_ptr(), de.data_ptr(), kp.data_ptr()
        fi.n_frame, fi.use_matches, fi.on_device, fi.frame_id = de.shape[0], 1, 1, i
        fi.height, fi.width = d.shape[0], d.shape[1]
        trk.enqueue(fi)
    tr = trk.trace()
    cap = 2 + 1024 * 256 + 1024 * 32
    buf = np.zeros(cap, dtype=np.int64)
    lib.dt_tracker_get_arrivals(trk._h, _host_ptr(buf), cap)
    n_cta = int(buf[0])
    nw = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    warps = buf[2 + 1024 * 256: 2 + 1024 * 256 + n_cta * nw].reshape(n_cta, nw)
    # release of the barrier before the value pass of outer 1 (codes 31 / 41 in order)
    rel = [t for c, t in tr if c == 31]
    t0 = rel[1] if len(rel) > 1 else rel[0]
    rel_w = (warps - t0) / 1e3
    print("per-warp value-pass end (us after the P3 release):")
    for r in [0, 1, 2, 3, 17, 18, 19, 30, 48, 60, 88, 100, 110, 140, 147]:
        if r < n_cta:
            print(r, np.round(rel_w[r], 2).tolist())
    print("max over CTAs per warp:", np.round(rel_w.max(axis=0), 2).tolist())
    print("mean over CTAs per warp:", np.round(rel_w.mean(axis=0), 2).tolist())
    st = point_stamps(buf, 8, nw)
    names = ["loads+blend", "apply", "project+pixel", "gates+tukey", "gradient", "rows"]
    for r in range(3):
        for w in range(nw):
            s0 = st[r, w]
            if s0[0] == 0 or s0[6] == 0:
                continue
            d = np.diff(s0[:7])
            print(f"cta {r} warp {w}: total {s0[6]-s0[0]} cyc  " + "  ".join(f"{nm} {int(v)}" for nm, v in zip(names, d)))
    trk.close()


if __name__ == "__main__":
    main()
