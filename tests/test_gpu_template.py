"""Device template graph build against the oracle restatement of the
reference's sequential greedy thinning and dense connections: bit-identical control
indices, edges and edge weights."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("surface,res,radius,sigma", [
    ("height-field", 30, 8.0, 16.0),
    ("plane", 71, 10.0, 20.0),
    ("sphere-patch", 141, 5.3, 10.6),
])
def test_template_graph_build_matches_oracle(surface, res, radius, sigma):
    from oracle import pipeline as OP
    from paper_2007_08576_b200 import synth
    from paper_2007_08576_b200.warpfield import build_connections, sample_control_points

    tpl = synth.make_template(synth.Scene(surface=surface, resolution=res, n_features=10))
    g = sample_control_points(tpl, radius, connection_sigma=sigma)
    np.testing.assert_array_equal(g.points, OP.sample_controls(tpl.points, radius))
    e, w = build_connections(g.points, sigma)
    e2, w2 = OP.connections(g.points, sigma)
    np.testing.assert_array_equal(e, e2)
    np.testing.assert_array_equal(w, w2)
    np.testing.assert_array_equal(g.edges, e2)
    assert np.all(e[:, 0] < e[:, 1]) and np.all(w >= 0.01)


def test_random_cloud_storage_order_greedy():
    """Unstructured points (no grid ties) and a radius comparable to the spacing."""
    from oracle import pipeline as OP
    from paper_2007_08576_b200.warpfield import Template, sample_control_points

    rng = np.random.default_rng(7)
    pts = rng.uniform(-20, 20, size=(3000, 3)) * np.array([1.0, 1.0, 0.2])
    tpl = Template(pts, np.tile([0.0, 0.0, -1.0], (len(pts), 1)))
    for r in (0.8, 2.5, 7.0):
        g = sample_control_points(tpl, r)
        np.testing.assert_array_equal(g.points, OP.sample_controls(pts, r))


@pytest.mark.parametrize("name", ["patch", "cloud", "cloud_k6", "small", "tiny"])
def test_point_normals_match_reference(name):
    """Device estimate_point_normals against the reference's output (golden). Points
    whose k-th and (k+1)-th neighbours tie have no unique neighbour set (the reference's
    kd-tree picks one in unspecified order), so they are checked for a camera-facing unit
    normal only; every other point matches to 1e-9."""
    from oracle import pipeline as OP
    from paper_2007_08576_b200.correspond import estimate_point_normals
    from tests.fixtures import load

    z = load("point_normals")
    pts, k, ref = z[f"{name}_pts"], int(z[f"{name}_k"]), z[f"{name}_nrm"]
    dev = estimate_point_normals(pts, k=k)
    _, tie = OP.point_normals(pts, k)
    np.testing.assert_allclose(dev[~tie], ref[~tie], rtol=0, atol=1e-9)
    np.testing.assert_allclose(np.linalg.norm(dev, axis=1), 1.0, atol=1e-12)
    if len(pts) >= 3:
        assert np.all(np.sum(dev * pts, axis=1) <= 0.0)


def test_point_normals_template_scale():
    """A benchmark-size template (config 2's 19,881-point sphere patch) in one call."""
    from oracle import pipeline as OP
    from paper_2007_08576_b200 import synth
    from paper_2007_08576_b200.correspond import estimate_point_normals

    tpl = synth.make_template(synth.CONFIGS[2]["scene"])
    dev = estimate_point_normals(tpl.points)
    ref, tie = OP.point_normals(tpl.points)
    np.testing.assert_allclose(dev[~tie], ref[~tie], rtol=0, atol=1e-9)
