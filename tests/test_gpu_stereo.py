"""Stereo depth (not in the reference, defined by
oracle/stereo.py): the device matcher equals the oracle bit for bit -- integer winners,
sub-pixel disparities and depths -- on synthetic rectified pairs of known depth, recovers
that depth, and feeds the tracker directly from device memory."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


def _surface(y, x):
    return 300.0 + 15.0 * np.sin(x / 20.0) + 10.0 * np.cos(y / 15.0)


@pytest.mark.parametrize("h,w,D,r,min_ncc,seed", [
    (96, 128, 40, 3, 0.5, 1),
    (120, 160, 48, 2, 0.3, 2),
    (64, 96, 32, 5, 0.7, 3),
    (61, 77, 40, 1, 0.0, 4),
])
def test_device_stereo_equals_oracle(h, w, D, r, min_ncc, seed):
    from oracle import stereo as OS
    from paper_2007_08576_b200.stereo import StereoMatcher

    fx, B = 300.0, 20.0
    L, R, z, disp = OS.synthetic_pair(h, w, fx, B, _surface, seed=seed)
    sm = StereoMatcher(h, w, fx, B, max_disp=D, radius=r, min_ncc=min_ncc)
    dep, dd, win = sm.compute(L, R)
    sm.close()
    odep, odd, owin = OS.stereo_depth(L, R, D, r, fx, B, min_ncc=min_ncc)
    np.testing.assert_array_equal(win, owin)
    np.testing.assert_array_equal(np.isnan(dd), np.isnan(odd))
    np.testing.assert_array_equal(dd[~np.isnan(dd)], odd[~np.isnan(odd)])
    np.testing.assert_array_equal(dep[~np.isnan(dep)], odep[~np.isnan(odep)])
    ok = np.isfinite(dep)
    assert ok.mean() > 0.5
    if r >= 2:  # the 3x3 window is noisy; larger windows recover the surface
        assert float(np.median(np.abs(dep - z)[ok])) < 1.5


def test_textureless_and_occluded_pixels_are_invalid():
    from paper_2007_08576_b200.stereo import StereoMatcher

    h, w = 48, 64
    L = np.full((h, w), 128, dtype=np.uint8)  # no texture: zero variance everywhere
    sm = StereoMatcher(h, w, 300.0, 20.0, max_disp=16, radius=2)
    dep, dd, win = sm.compute(L, L.copy())
    sm.close()
    assert np.all(np.isnan(dep)) and np.all(win == -1)


def test_stereo_depth_feeds_the_tracker_on_device():
    """Stereo pair -> device depth -> dt_track_frame (on_device) gives the same frame as
    the host round trip of that depth."""
    import ctypes as C

    import paper_2007_08576_b200 as dt
    from oracle import stereo as OS
    from paper_2007_08576_b200._lib import FrameInput, FrameOutput, Report
    from paper_2007_08576_b200._session import DeviceTracker, make_config
    from paper_2007_08576_b200.stereo import StereoMatcher

    h, w, fx, B = 120, 160, 300.0, 20.0
    L, R, z, _ = OS.synthetic_pair(h, w, fx, B, _surface, seed=7)
    sm = StereoMatcher(h, w, fx, B, max_disp=48, radius=3)
    dep, _, _ = sm.compute(L, R)
    # template: the truth surface back-projected on a coarse pixel grid
    cam = dt.PinholeCamera(fx, fx, (w - 1) / 2.0, (h - 1) / 2.0, w, h)
    vv, uu = np.mgrid[10:h - 10:4, 10:w - 10:4]
    zz = _surface(vv.astype(float), uu.astype(float))
    pts = np.stack([(uu - cam.cx) / fx * zz, (vv - cam.cy) / fx * zz, zz], -1).reshape(-1, 3)
    nrm = np.tile([0.0, 0.0, -1.0], (len(pts), 1))
    cfg = dt.load_config({"camera": {"fx": fx, "fy": fx, "cx": cam.cx, "cy": cam.cy, "width": w,
                                     "height": h}, "sampling": {"radius": 12.0},
                          "solver": {"max_outer_iters": 3}})
    tpl, graph = dt.prepare_template(dt.Template(pts, nrm), cfg)
    dcfg = make_config(cam, cfg.energy, cfg.make_solver_config(), sampling_radius=graph.sampling_radius)
    outs = []
    for on_dev in (1, 0):
        trk = DeviceTracker(tpl, graph, dcfg)
        fi = FrameInput()
        host = np.ascontiguousarray(dep)
        fi.depth = sm.device_depth() if on_dev else host.ctypes.data
        fi.on_device, fi.height, fi.width, fi.use_matches = on_dev, h, w, 0
        wts, pts_o, rep = np.zeros((len(graph), 8)), np.zeros((len(tpl), 3)), Report()
        fo = FrameOutput()
        fo.warps, fo.points = wts.ctypes.data, pts_o.ctypes.data
        fo.report = C.cast(C.pointer(rep), C.c_void_p).value
        trk.track_raw(fi, fo)
        trk.close()
        outs.append((wts, pts_o, rep.n_correspondences))
    sm.close()
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2] > 0


def test_device_resident_images_give_the_host_result():
    import torch

    from oracle import stereo as OS
    from paper_2007_08576_b200.stereo import StereoMatcher

    h, w = 120, 160
    L, R, _, _ = OS.synthetic_pair(h, w, 300.0, 20.0, _surface, seed=9)
    sm = StereoMatcher(h, w, 300.0, 20.0, max_disp=40, radius=3)
    a = sm.compute(L, R)
    b = sm.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda(), on_device=True)
    sm.close()
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
