"""Device ORB front end against its oracle restatement: keypoints,
scores, orientation sectors and descriptors bit-exact; plus the properties a detector
must have (integer shifts move keypoints and keep descriptors; matching recovers a
shift through the device Hamming matcher)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


def textured(h, w, seed, block=8, noise=4.0):
    """Blocky random texture with mild noise: many FAST corners of varied strength."""
    rng = np.random.default_rng(seed)
    img = rng.integers(0, 256, size=(h // block + 2, w // block + 2)).astype(np.float64)
    img = np.kron(img, np.ones((block, block)))[:h, :w]
    return (img + rng.normal(0, noise, size=(h, w))).clip(0, 255).astype(np.uint8)


@pytest.mark.parametrize("h,w,seed,kw", [
    (480, 640, 0, {}),
    (480, 640, 1, dict(threshold=35, cell=48, per_cell=4, n_max=900)),
    (257, 333, 2, dict(threshold=10, cell=20, per_cell=16, n_max=5000)),
])
def test_orb_matches_oracle_bitwise(h, w, seed, kw):
    from oracle import orb as O
    from paper_2007_08576_b200.orb import OrbDetector

    img = textured(h, w, seed)
    det = OrbDetector(h, w, **kw)
    kp, desc, sc, sec = det.detect(img)
    det.close()
    okp, odesc, osc, osec = O.detect_and_describe(img, **kw)
    assert len(kp) > 100
    np.testing.assert_array_equal(kp, okp)
    np.testing.assert_array_equal(sc, osc)
    np.testing.assert_array_equal(sec, osec)
    np.testing.assert_array_equal(desc, odesc)


def test_flat_image_has_no_keypoints():
    from paper_2007_08576_b200.orb import OrbDetector

    det = OrbDetector(120, 160)
    kp, desc, _, _ = det.detect(np.full((120, 160), 77, dtype=np.uint8))
    det.close()
    assert kp.shape == (0, 2) and desc.shape == (0, 32)


def test_integer_shift_moves_keypoints_and_keeps_descriptors():
    from paper_2007_08576_b200.orb import OrbDetector

    big = textured(560, 720, 5)
    dx, dy = 17, 9
    a = big[40:520, 40:680]
    b = big[40 - dy:520 - dy, 40 - dx:680 - dx]  # content moved by (+dx, +dy)
    det = OrbDetector(480, 640, n_max=4000, per_cell=32)
    ka, da, _, _ = det.detect(a)
    kb, db, _, _ = det.detect(b)
    det.close()
    idx_b = {(int(u), int(v)): i for i, (u, v) in enumerate(kb)}
    common = 0
    for i, (u, v) in enumerate(ka):
        j = idx_b.get((int(u) + dx, int(v) + dy))
        if j is not None:
            common += 1
            np.testing.assert_array_equal(da[i], db[j])
    assert common > 0.5 * min(len(ka), len(kb))


def test_hamming_matching_recovers_the_shift():
    """Detect on both images, match with the device Hamming matcher (a4): the dominant
    displacement of the matches is the true shift."""
    from paper_2007_08576_b200.matching import match_descriptors
    from paper_2007_08576_b200.orb import OrbDetector

    big = textured(560, 720, 6)
    dx, dy = -11, 6
    a = big[40:520, 40:680]
    b = big[40 - dy:520 - dy, 40 - dx:680 - dx]
    det = OrbDetector(480, 640)
    ka, da, _, _ = det.detect(a)
    kb, db, _, _ = det.detect(b)
    det.close()
    idx, dist = match_descriptors(da, db)
    good = dist <= 40
    disp = kb[idx[good]] - ka[good]
    vals, counts = np.unique(disp, axis=0, return_counts=True)
    assert tuple(vals[np.argmax(counts)]) == (dx, dy)
    assert counts.max() > 0.5 * good.sum()


def test_device_resident_orb_output_feeds_the_tracker():
    """image -> ORB (device) -> Hamming -> preselection -> LM with the detector's
    keypoints / descriptors read in place (on_device frame input) gives exactly what the
    host round trip gives."""
    import ctypes as C

    import torch

    import bench
    from paper_2007_08576_b200._lib import FrameInput, FrameOutput, Report
    from paper_2007_08576_b200.orb import OrbDetector
    from tests.test_gpu_pipeline import _tracker

    wl = bench.make_workload(1, 2, seed=4)
    h, w = wl["scene"].height, wl["scene"].width
    fr = wl["frames"][0]
    img = textured(h, w, 11)
    det = OrbDetector(h, w, n_max=600)
    kp, desc, _, _ = det.detect(img)
    kp_dev, desc_dev, n = det.last_on_device()
    assert n == len(kp) > 50
    m, npts = len(wl["graph"]), len(wl["tpl"])

    def run(on_device):
        trk = _tracker(wl)
        depth = np.ascontiguousarray(fr.depth)
        keep = [depth, kp, desc]
        fi = FrameInput()
        if on_device:
            d_depth = torch.from_numpy(depth).cuda()
            keep.append(d_depth)
            fi.depth, fi.frame_desc, fi.frame_kp = d_depth.data_ptr(), desc_dev, kp_dev
        else:
            fi.depth, fi.frame_desc, fi.frame_kp = depth.ctypes.data, desc.ctypes.data, kp.ctypes.data
        fi.n_frame, fi.use_matches, fi.on_device, fi.frame_id = n, 1, int(on_device), 0
        fi.height, fi.width = depth.shape[0], depth.shape[1]
        wts = np.zeros((m, 8))
        pts = np.zeros((npts, 3))
        rep = Report()
        fo = FrameOutput()
        fo.warps, fo.points = wts.ctypes.data, pts.ctypes.data
        fo.report = C.cast(C.pointer(rep), C.c_void_p).value
        trk.track_raw(fi, fo)
        trk.close()
        return wts, pts, rep.n_matches, rep.total_cost

    a = run(False)
    b = run(True)
    det.close()
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    assert a[2] == b[2] and a[3] == b[3]
