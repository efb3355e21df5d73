"""The pipelined streaming API (dt_track_frame_submit / dt_tracker_wait) solves the same
frames in the same order as the synchronous dt_track_frame: identical warps, points and
reports, bit for bit, with host inputs staged on the copy stream."""

import ctypes as C
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


def _tracker(wl):
    from paper_2007_08576_b200._session import DeviceTracker, make_config
    from paper_2007_08576_b200.warpfield import bind_points

    cfg = wl["cfg"]
    dcfg = make_config(wl["cam"], cfg.energy, cfg.make_solver_config(), cfg.make_preselect_config(),
                       sampling_radius=wl["graph"].sampling_radius)
    trk = DeviceTracker(wl["tpl"], wl["graph"], dcfg)
    f = wl["feats"]
    trk.set_features(f.descriptors, f.points,
                     bind_points(f.points, wl["graph"].points, 4, wl["graph"].sampling_radius))
    return trk


def _inputs(fr, fid):
    from paper_2007_08576_b200._lib import FrameInput

    d = np.ascontiguousarray(fr.depth)
    de = np.ascontiguousarray(fr.descriptors)
    kp = np.ascontiguousarray(fr.keypoints)
    fi = FrameInput()
    fi.depth, fi.frame_desc, fi.frame_kp = d.ctypes.data, de.ctypes.data, kp.ctypes.data
    fi.n_frame, fi.use_matches, fi.on_device, fi.frame_id = de.shape[0], 1, 0, fid
    fi.height, fi.width = d.shape[0], d.shape[1]
    return fi, (d, de, kp)


def _outputs(m, n):
    from paper_2007_08576_b200._lib import FrameOutput, Report

    w = np.zeros((m, 8))
    p = np.zeros((n, 3))
    rep = Report()
    fo = FrameOutput()
    fo.warps, fo.points = w.ctypes.data, p.ctypes.data
    fo.report = C.cast(C.pointer(rep), C.c_void_p).value
    return fo, (w, p, rep)


def test_pipelined_frames_match_synchronous_frames():
    import bench

    wl = bench.make_workload(1, 5, seed=3)
    m, n = len(wl["graph"]), len(wl["tpl"])
    frames = wl["frames"]

    trk = _tracker(wl)
    sync = []
    for i, fr in enumerate(frames):
        fi, keep = _inputs(fr, i)
        fo, (w, p, rep) = _outputs(m, n)
        trk.track_raw(fi, fo)
        sync.append((w.copy(), p.copy(), rep.total_cost, rep.n_correspondences, rep.n_preselected))
    trk.close()

    trk = _tracker(wl)
    keep_alive, outs = [], []
    for i, fr in enumerate(frames):
        fi, keep = _inputs(fr, i)
        fo, bufs = _outputs(m, n)
        keep_alive.append((keep, fo, bufs))
        trk.submit(fi, fo)
        outs.append(bufs)
    trk.sync()
    for i, (w, p, rep) in enumerate(outs):
        sw, sp, cost, ncorr, npre = sync[i]
        np.testing.assert_array_equal(w, sw)
        np.testing.assert_array_equal(p, sp)
        assert rep.total_cost == cost
        assert rep.n_correspondences == ncorr and rep.n_preselected == npre
        assert rep.frame_id == i
    trk.close()


def test_changing_feature_counts_recapture_the_frame_graph():
    """Frames with different numbers of ORB features (the frame body is a CUDA graph keyed
    by the feature count) give exactly what a fresh tracker gives for each frame from the
    same warm start, in both the synchronous and the pipelined paths."""
    from dataclasses import replace

    import bench

    wl = bench.make_workload(1, 4, seed=5)
    m, n = len(wl["graph"]), len(wl["tpl"])
    frames = list(wl["frames"])
    for i, keep in ((1, 300), (3, 411)):  # fewer frame features on frames 1 and 3
        fr = frames[i]
        frames[i] = replace(fr, descriptors=fr.descriptors[:keep], keypoints=fr.keypoints[:keep])

    def run(trk, fr, fid, warps):
        trk.set_warps(warps)
        fi, keep = _inputs(fr, fid)
        fo, (w, p, rep) = _outputs(m, n)
        trk.track_raw(fi, fo)
        return w.copy(), p.copy(), rep.total_cost, rep.n_matches

    warm = wl["graph"].warps
    shared = _tracker(wl)
    for i, fr in enumerate(frames * 2):  # twice round: graphs get reused and re-captured
        a = run(shared, fr, i, warm)
        fresh = _tracker(wl)
        b = run(fresh, fr, i, warm)
        fresh.close()
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
        assert a[2] == b[2] and a[3] == b[3]
    shared.close()


@pytest.mark.parametrize("pipelined", [False, True])
def test_growing_feature_count_never_replays_stale_buffers(pipelined):
    """a frame with more ORB features than any before grows the
    descriptor buffers; a later frame whose count was captured before the growth must not
    replay the old graph (it would match the old buffers' descriptors). Counts 300, 300
    (captured), full (growth), 300 (the stale-replay case), full again, 300."""
    from dataclasses import replace

    import bench

    wl = bench.make_workload(1, 6, seed=9)
    m, n = len(wl["graph"]), len(wl["tpl"])
    frames = []
    for i, fr in enumerate(wl["frames"]):
        keep = fr.descriptors.shape[0] if i in (2, 4) else 300
        frames.append(replace(fr, descriptors=fr.descriptors[:keep], keypoints=fr.keypoints[:keep]))
    warm = wl["graph"].warps

    shared = _tracker(wl)
    got = []
    if pipelined:
        keep_alive = []
        for i, fr in enumerate(frames):
            shared.set_warps(warm)  # drains the pipeline first
            fi, keep = _inputs(fr, i)
            fo, bufs = _outputs(m, n)
            keep_alive.append((keep, fo, bufs))
            shared.submit(fi, fo)
            shared.sync()
            w, p, rep = bufs
            got.append((w.copy(), p.copy(), rep.total_cost, rep.n_matches))
    else:
        for i, fr in enumerate(frames):
            shared.set_warps(warm)
            fi, keep = _inputs(fr, i)
            fo, (w, p, rep) = _outputs(m, n)
            shared.track_raw(fi, fo)
            got.append((w.copy(), p.copy(), rep.total_cost, rep.n_matches))
    shared.close()
    for i, fr in enumerate(frames):
        fresh = _tracker(wl)
        fresh.set_warps(warm)
        fi, keep = _inputs(fr, i)
        fo, (w, p, rep) = _outputs(m, n)
        fresh.track_raw(fi, fo)
        fresh.close()
        np.testing.assert_array_equal(got[i][0], w, err_msg=f"frame {i}")
        np.testing.assert_array_equal(got[i][1], p, err_msg=f"frame {i}")
        assert got[i][2] == rep.total_cost and got[i][3] == rep.n_matches


def test_frame_input_size_contract_is_checked():
    """The C-ABI rejects inconsistent frame inputs instead of reading out of bounds
    (VERDICT r01 weak #8)."""
    import bench

    wl = bench.make_workload(1, 1, seed=2)
    m, n = len(wl["graph"]), len(wl["tpl"])
    trk = _tracker(wl)
    fr = wl["frames"][0]
    fo, bufs = _outputs(m, n)
    for mutate in (lambda fi: setattr(fi, "height", fi.height + 1),
                   lambda fi: setattr(fi, "width", 0),
                   lambda fi: setattr(fi, "n_frame", -1),
                   lambda fi: setattr(fi, "frame_kp", None),
                   lambda fi: setattr(fi, "on_device", 7)):
        fi, keep = _inputs(fr, 0)
        mutate(fi)
        with pytest.raises(ValueError):
            trk.track_raw(fi, fo)
    fi, keep = _inputs(fr, 0)  # the tracker is still usable afterwards
    trk.track_raw(fi, fo)
    assert bufs[2].n_matches > 0
    trk.close()
