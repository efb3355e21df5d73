"""Sequence-level behaviour of the device tracking path, after the reference's
tests/test_tracking.py:20-130: a motionless plane stays exactly on the template, a warm
start begins below a cold start, a failed preselection drops the feature term with the
reference's warning and counts, annotate_matches passes None / empty through, and
prepare_template binds every point with unit-sum weights."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small_config():
    import paper_2007_08576_b200 as dt

    return dt.load_config({"sampling": {"radius": 12.0}, "solver": {"max_outer_iters": 40}})


def _seq(n, **over):
    from paper_2007_08576_b200 import synth

    scene = synth.Scene(**{**dict(surface="plane", resolution=20, width=320, height=240,
                                  n_features=20, n_distractors=0), **over})
    cam = synth.camera_for(scene)
    tpl = synth.make_template(scene)
    feats = synth.make_features(scene, tpl)
    frames = [synth.make_frame(scene, cam, tpl, feats, f) for f in range(1, n + 1)]
    return scene, cam, tpl, frames


def test_identity_sequence_stays_on_template(small_config):
    import paper_2007_08576_b200 as dt

    _, cam, tpl, frames = _seq(3, deformation="none", amplitude=0.0, noise_sigma=0.0)
    res = dt.track_sequence(tpl, [f.observation(cam) for f in frames], None, small_config)
    identity = np.concatenate([[1.0], np.zeros(7)])
    for r in res:
        assert float(np.abs(r.points - tpl.points).max()) < 1e-6
        assert r.report.converged
        np.testing.assert_allclose(r.graph.warps, np.tile(identity, (len(r.graph), 1)),
                                   atol=1e-6)


def test_warm_start_reuses_previous_frame(small_config):
    import paper_2007_08576_b200 as dt

    _, cam, tpl, frames = _seq(3, surface="height-field", amplitude=5.0, period=8.0, seed=2)
    obs = [f.observation(cam) for f in frames]
    res = dt.track_sequence(tpl, obs, None, small_config)
    assert res[1].report.cost_history  # it had to move
    warm_first = res[2].report.cost_history[0][0]
    cold = dt.track_sequence(tpl, [obs[2]], None, small_config)
    assert warm_first < cold[0].report.cost_history[0][0]


def test_preselection_failure_drops_feature_term(small_config):
    import paper_2007_08576_b200 as dt

    _, cam, tpl, frames = _seq(1, deformation="none", amplitude=0.0)
    bad = dt.MatchSet.from_pairs(tpl.points[:2], tpl.points[:2] + 1.0)
    rep = dt.track_sequence(tpl, [frames[0].observation(cam)], [bad], small_config)[0].report
    assert any("preselection failed" in w for w in rep.warnings)
    assert rep.n_matches == 2
    assert rep.n_preselected == 0
    assert rep.feature_cost == 0.0
    assert rep.match_weight_sum == 0.0


def test_annotate_matches_passthrough(small_config):
    import paper_2007_08576_b200 as dt

    assert dt.annotate_matches(None, small_config) == (None, None)
    empty = dt.MatchSet.from_pairs(np.zeros((0, 3)), np.zeros((0, 3)))
    out, warning = dt.annotate_matches(empty, small_config)
    assert out is empty and warning is None


def test_prepare_template_binds_and_samples(small_config):
    import paper_2007_08576_b200 as dt

    _, _, tpl, _ = _seq(1, surface="height-field")
    bound, graph = dt.prepare_template(tpl, small_config)
    assert bound.is_bound
    assert len(graph) >= 20  # 100 mm patch at radius 12
    assert bound.bind_indices.shape == (len(bound), 4)
    np.testing.assert_allclose(bound.bind_weights.sum(axis=1), 1.0, atol=1e-9)


def test_torch_inputs_of_any_device_and_dtype_match_numpy():
    """Tracker.track takes torch tensors too: CUDA tensors and host tensors of another
    dtype are copied through numpy (the host-buffer entry never reads a device pointer as
    host memory); results equal the numpy-input frame bit for bit."""
    import torch

    import bench
    import paper_2007_08576_b200 as dt

    wl = bench.make_workload(1, 1, seed=2)
    fr = wl["frames"][0]
    outs = []
    for kind in ("numpy", "torch"):
        trk = dt.Tracker(wl["tpl"], wl["graph"], wl["cam"], wl["cfg"])
        trk.set_features(wl["feats"].descriptors, wl["feats"].points)
        if kind == "numpy":
            r = trk.track(fr.depth, descriptors=fr.descriptors, keypoints=fr.keypoints)
        else:
            r = trk.track(torch.from_numpy(fr.depth).cuda(),
                          descriptors=torch.from_numpy(fr.descriptors).cuda(),
                          keypoints=torch.from_numpy(fr.keypoints.astype(np.int64)))
        trk.close()
        outs.append(r)
    np.testing.assert_array_equal(outs[0].graph.warps, outs[1].graph.warps)
    np.testing.assert_array_equal(outs[0].matches.preselected, outs[1].matches.preselected)
    assert outs[0].report.to_dict() == outs[1].report.to_dict()
