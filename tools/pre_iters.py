"""IRLS steps per preselection hypothesis on the config-2 benchmark sequence:
build the instrumented variant, then run it on the GPU box.

    python tools/build_variant.py prestats --flags=-DDT_PRESELECT_STATS
    cp _variants/prestats.so paper_2007_08576_b200/variant_prestats.so
    DEFORMTRACK_B200_LIB=paper_2007_08576_b200/variant_prestats.so python tools/pre_iters.py
"""
import ctypes, sys, numpy as np
sys.path.insert(0, '.')
import bench
import paper_2007_08576_b200 as dt
from paper_2007_08576_b200 import _lib
wl = bench.make_workload(2, 6, seed=0)
trk = dt.Tracker(wl["tpl"], wl["graph"], wl["cam"], wl["cfg"])
trk.set_features(wl["feats"].descriptors, wl["feats"].points)
trk.set_exhaustive(True)
L = ctypes.CDLL(str(_lib.LIB_PATH))
for fr in wl["frames"]:
    r = trk.track(fr.depth, descriptors=fr.descriptors, keypoints=fr.keypoints)
    n = r.report.n_matches
    buf = (ctypes.c_int * 8192)()
    L.dt_debug_preselect_iters(buf, 8192)
    a = np.array(buf[:n])
    fl = np.asarray(r.matches.preselected)
    print("n", n, "hist", np.bincount(a + 1, minlength=12).tolist(),
          "inlier-ref mean", a[fl].mean(), "outlier-ref mean", a[~fl].mean() if (~fl).any() else None,
          "sum", a.sum(), "max-possible", 10 * n)
    # per-CTA (14 hypotheses) sums
    c = np.add.reduceat(a.clip(0), np.arange(0, n, 14))
    print("  per-CTA iters: mean", c.mean(), "max", c.max(), "min", c.min())
    tb = (ctypes.c_longlong * 8)()
    L.dt_debug_preselect_times(tb)
    t = np.array(tb[:8], dtype=np.int64)
    print("  phase A (us): loads up to the keypoints", (t[6] - t[0]) / 1e3, "| + depth, scan",
          (t[7] - t[0]) / 1e3, "| built", (t[1] - t[0]) / 1e3)
    print("  fused kernel (us from CTA 0 start): match list built", (t[1] - t[0]) / 1e3,
          "| last CTA enters final", (t[2] - t[0]) / 1e3, "| argmax", (t[3] - t[2]) / 1e3,
          "| flags + scatter + stats", (t[4] - t[3]) / 1e3, "| end", (t[5] - t[0]) / 1e3)
