"""dt_track_frames_batched (BASELINE config 5's independent sequences in one call) and
dt_depth_from_pfm (the device PFM decode) through the C-ABI."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


def test_batched_frames_equal_one_at_a_time():
    """Three sequences (different frames each) through one dt_track_frames_batched call
    give bitwise the outputs of three dt_track_frame calls, in grid and cluster mode."""
    import copy

    import bench
    from paper_2007_08576_b200 import _session as S
    from paper_2007_08576_b200.tracking import Tracker

    wl = bench.make_workload(1, 3, seed=4)
    tpl, graph, cam, feats = wl["tpl"], wl["graph"], wl["cam"], wl["feats"]
    for cs in (0, 4):
        cfg = copy.deepcopy(wl["cfg"])
        cfg.device.cluster_size = cs
        trks = [Tracker(tpl, graph, cam, cfg) for _ in range(3)]
        for t in trks:
            t.set_features(feats.descriptors, feats.points)
        frames = [dict(depth=fr.depth, frame_desc=fr.descriptors, frame_kp=fr.keypoints,
                       want_matches=True) for fr in wl["frames"]]
        batched = S.track_batched([t.device for t in trks], frames)
        for t in trks:
            t.reset()
        single = [t.device.track(**f) for t, f in zip(trks, frames)]
        for a, b in zip(batched, single):
            np.testing.assert_array_equal(a.warps, b.warps)
            np.testing.assert_array_equal(a.points, b.points)
            np.testing.assert_array_equal(a.match_weights, b.match_weights)
            assert a.cost_history == b.cost_history
            assert int(a.report.n_preselected) == int(b.report.n_preselected)
            assert int(a.report.n_correspondences) == int(b.report.n_correspondences)
        # different frames -> different solutions (the batch did not alias trackers)
        assert not np.array_equal(batched[0].warps, batched[1].warps)
        for t in trks:
            t.close()


def test_batched_rejects_null_tracker():
    import ctypes as C

    from paper_2007_08576_b200._lib import FrameInput, FrameOutput, lib

    hs = (C.c_void_p * 1)(None)
    fis = (FrameInput * 1)()
    fos = (FrameOutput * 1)()
    assert lib.dt_track_frames_batched(hs, fis, fos, 1, None) != 0
    assert lib.dt_track_frames_batched(hs, fis, fos, 0, None) == 0


@pytest.mark.parametrize("big_endian", [0, 1])
def test_depth_from_pfm_decodes_on_device(big_endian):
    """Bottom-up f32 rows (either byte order) -> top-down f64 depth, NaN kept, equal to
    the host reader's conversion (fileio.read_pfm, fileio.py:142-160)."""
    import torch

    from paper_2007_08576_b200._lib import lib

    h, w = 37, 53
    rng = np.random.default_rng(5)
    img = rng.uniform(300, 900, size=(h, w)).astype(np.float32)
    img[3, 4] = np.nan
    payload = np.flipud(img).astype(">f4" if big_endian else "<f4")
    raw = np.frombuffer(payload.tobytes(), dtype=np.float32).copy()  # bytes as stored
    dpay = torch.from_numpy(raw).cuda()
    out = torch.empty((h, w), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert lib.dt_depth_from_pfm(dpay.data_ptr(), h, w, big_endian, out.data_ptr(), st) == 0
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    want = img.astype(np.float64)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    np.testing.assert_array_equal(got[~np.isnan(want)], want[~np.isnan(want)])
