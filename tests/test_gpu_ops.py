"""Operator-level parity on the GPU: every device twin against the reference's outputs
(golden fixtures from the reference itself) and against the oracle.

Tolerances: integer / index / mask outputs bit-exact; per-row float outputs that the
device evaluates in the reference's IEEE order (-fmad=false) bit-exact or 1e-12; the
per-control reductions, which the device sums in a different (deterministic) order,
rtol 1e-9 -- the reference's own kernel-vs-builder tolerance (test_kernels.py:53-55)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from tests.fixtures import hamming_kat_descriptors, load  # noqa: E402


def close_red(got, want):
    scale = 1.0 + (np.abs(want).max() if want.size else 0.0)
    np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-9 * scale)


@pytest.fixture(scope="module")
def kz():
    return load("kernels")


@pytest.fixture(scope="module")
def K():
    from paper_2007_08576_b200 import kernels

    return kernels


def test_observation_normals_bitwise(kz):
    from paper_2007_08576_b200.correspond import compute_observation_normals
    from paper_2007_08576_b200.geometry import PinholeCamera

    cam = PinholeCamera(120.0, 120.0, 23.5, 23.5, 48, 48)
    np.testing.assert_array_equal(compute_observation_normals(kz["wr_depth"], cam),
                                  kz["wr_obs_normals"])


def test_warp_and_rasterize(kz, K):
    got = K.warp_and_rasterize(kz["wr_points"], kz["normals"], kz["bind_idx"], kz["alpha"],
                               kz["warps"], kz["wr_depth"], kz["wr_valid_px"],
                               kz["wr_obs_normals"], 120.0, 120.0, 23.5, 23.5, 8.0,
                               float(np.cos(np.deg2rad(60.0))), 8)
    p, n, valid, op, on, pix = got
    np.testing.assert_array_equal(valid, kz["wr_valid"])
    np.testing.assert_array_equal(pix, kz["wr_pixels"])
    np.testing.assert_allclose(p, kz["wr_p"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(n, kz["wr_n"], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(op, kz["wr_obs_p"])
    np.testing.assert_array_equal(on, kz["wr_obs_n"])


def test_icp_reduce(kz, K):
    m = kz["warps"].shape[0]
    got = K.icp_reduce(kz["points"], kz["obs_normals"], kz["obs_points"], kz["bind_idx"],
                       kz["alpha"], kz["warps"], kz["basis"], 10.0, np.zeros(0), False, True, 8, m)
    np.testing.assert_array_equal(got[3], kz["icp_r"])
    for g, name in zip(got[:3], ("partial", "support", "cost")):
        close_red(g, kz[f"icp_{name}"])
    # value-only pass: identical cost bits to the jac pass, no partials (test_kernels.py:212)
    val = K.icp_reduce(kz["points"], kz["obs_normals"], kz["obs_points"], kz["bind_idx"],
                       kz["alpha"], kz["warps"], kz["basis"], 10.0, np.zeros(0), False, False, 8, m)
    np.testing.assert_array_equal(val[2], got[2])
    assert not val[0].any()


def test_icp_reduce_frozen(kz, K):
    m = kz["warps"].shape[0]
    from paper_2007_08576_b200.energy import warp_increment_basis

    got = K.icp_reduce(kz["points"], kz["obs_normals"], kz["obs_points"], kz["bind_idx"],
                       kz["alpha"], kz["moved"], warp_increment_basis(kz["moved"]), 10.0,
                       kz["frozen"], True, True, 8, m)
    for g, name in zip(got, ("partial", "support", "cost", "r")):
        close_red(g, kz[f"icpf_{name}"])


def test_feature_reduce(kz, K):
    m = kz["warps"].shape[0]
    a = kz["feat_active"]
    got = K.feature_reduce(kz["points"][a], kz["obs_points"][a], kz["match_w"][a],
                           kz["bind_idx"][a], kz["alpha"][a], kz["warps"], kz["basis"], 10.0,
                           True, 8, m)
    for g, name in zip(got, ("partial", "support", "cost")):
        close_red(g, kz[f"feat_{name}"])


def test_arap_reduce_with_self_edge(kz, K):
    m = kz["warps"].shape[0]
    got = K.arap_reduce(kz["ctrl"], kz["R"], kz["t"], kz["warps"], kz["edges"], kz["edge_w"],
                        kz["wa"], 20.0, 100.0, True, 8, m)
    close_red(got[0], kz["arap_partial"])
    close_red(got[1], kz["arap_cost"])


def test_basis_transform_step(kz):
    from paper_2007_08576_b200.energy import warp_increment_basis
    from paper_2007_08576_b200.geometry import dq_to_transform_batch
    from paper_2007_08576_b200.solver import apply_step

    np.testing.assert_array_equal(warp_increment_basis(kz["warps"]), kz["basis"])
    R, t = dq_to_transform_batch(kz["warps"])
    np.testing.assert_array_equal(R, kz["R"])
    np.testing.assert_array_equal(t, kz["t"])
    np.testing.assert_allclose(apply_step(kz["warps"], kz["step_delta"]), kz["step_out"],
                               rtol=0, atol=4e-16)


def test_solve_damped(kz):
    from paper_2007_08576_b200.solver import _solve_damped

    d, ok = _solve_damped(kz["sd_A"], kz["sd_b"], kz["sd_lam"])
    np.testing.assert_array_equal(ok, kz["sd_ok"])
    np.testing.assert_allclose(d, kz["sd_delta"], rtol=1e-9, atol=1e-12)
    assert not ok[-1] and not d[-1].any()   # indefinite block isolated with a zero step


def test_bind_points(kz):
    from paper_2007_08576_b200.warpfield import bind_points, bind_points_device

    idx, w = bind_points_device(kz["bind_pts"], kz["bind_ctrl"], 4, 7.0)
    np.testing.assert_array_equal(idx, kz["bind_idx_ref"])
    np.testing.assert_allclose(w, kz["bind_w_ref"], rtol=1e-14, atol=1e-16)
    idx, w = bind_points(kz["bind_pts"], kz["bind_ctrl"], 4, 7.0)
    np.testing.assert_array_equal(idx, kz["bind_idx_ref"])
    np.testing.assert_allclose(w, kz["bind_w_ref"], rtol=1e-14, atol=1e-16)


def test_bind_points_pads_small_graphs():
    from paper_2007_08576_b200.warpfield import bind_points_device

    pts = np.random.default_rng(0).normal(size=(10, 3))
    idx, w = bind_points_device(pts, np.array([[0.0, 0, 0], [1.0, 0, 0]]), 4, 1.0)
    assert idx.shape == (10, 4)
    np.testing.assert_array_equal(idx[:, 2], idx[:, 0])
    np.testing.assert_array_equal(w[:, 2:], 0.0)
    np.testing.assert_allclose(w.sum(axis=1), 1.0, rtol=1e-15)


def test_hamming_known_answers():
    from paper_2007_08576_b200.matching import match_descriptors

    from oracle import kernels as OK

    td, fd, want_i, want_d = hamming_kat_descriptors()
    idx, dist = match_descriptors(td, fd)
    np.testing.assert_array_equal(idx, want_i)
    np.testing.assert_array_equal(dist, want_d)
    oi, od = OK.hamming_match(td, fd)
    np.testing.assert_array_equal(idx, oi)
    np.testing.assert_array_equal(dist, od)
    # identical -> 0, one flipped bit -> 1, all bits -> 256, ties -> lowest index
    a = np.random.default_rng(1).integers(0, 256, size=(1, 32), dtype=np.uint8)
    one = a.copy()
    one[0, 5] ^= 0x10
    frames = np.concatenate([~a, one, a, a], axis=0).astype(np.uint8)
    i, d = match_descriptors(np.concatenate([a, ~a]), frames)
    assert i.tolist() == [2, 0] and d.tolist() == [0, 0]
    i, d = match_descriptors(a, frames[:2])
    assert i.tolist() == [1] and d.tolist() == [1]
    i, d = match_descriptors(a, (~a).astype(np.uint8))
    assert d.tolist() == [256]


def test_hamming_large_random_matches_oracle():
    from paper_2007_08576_b200.matching import match_descriptors

    from oracle import kernels as OK

    rng = np.random.default_rng(5)
    td = rng.integers(0, 256, size=(2000, 32), dtype=np.uint8)
    fd = rng.integers(0, 256, size=(2600, 32), dtype=np.uint8)
    fd[::7, :8] = td[: len(fd[::7]), :8]  # plenty of near ties
    i, d = match_descriptors(td, fd)
    oi, od = OK.hamming_match(td, fd)
    np.testing.assert_array_equal(i, oi)
    np.testing.assert_array_equal(d, od)


def test_preselect_matches_reference():
    from paper_2007_08576_b200.matching import MatchSet, PreselectConfig, preselect_inliers

    z = load("matching")
    for i in range(int(z["n_cases"])):
        nref, seed = (int(x) for x in z[f"c{i}_cfg"])
        res = preselect_inliers(MatchSet.from_pairs(z[f"c{i}_src"], z[f"c{i}_dst"]),
                                PreselectConfig(n_references=nref, seed=seed))
        np.testing.assert_array_equal(res.matches.preselected, z[f"c{i}_flags"])
        np.testing.assert_allclose(res.matches.weights, z[f"c{i}_weights"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(res.rotation, z[f"c{i}_rot"], rtol=0, atol=1e-12)
        assert res.reference_index == int(z[f"c{i}_ref"])
        assert abs(res.support - float(z[f"c{i}_support"])) <= 1e-9 * len(z[f"c{i}_src"])


def _rigid_matches(n, outlier_fraction, seed, grid=None, angle_deg=15.0, translation=10.0,
                   box=100.0):
    """The reference's matching fixture shape (test_matching.py:17-47): a rigid motion of
    uniform points plus uniform outliers, optionally snapped to a dyadic grid."""
    rng = np.random.default_rng(seed)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    th = np.deg2rad(angle_deg)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    R = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
    t = rng.normal(size=3)
    t *= translation / np.linalg.norm(t)
    src = rng.uniform(-box / 2.0, box / 2.0, (n, 3))
    dst = src @ R.T + t
    n_out = round(n * outlier_fraction)
    out_idx = rng.choice(n, size=n_out, replace=False)
    dst[out_idx] = rng.uniform(-box / 2.0, box / 2.0, (n_out, 3))
    if grid is not None:
        src = np.round(src / grid) * grid
        dst = np.round(dst / grid) * grid
    inlier = np.ones(n, dtype=bool)
    inlier[out_idx] = False
    return src, dst, inlier


def test_preselect_all_outliers_raises():
    """Pure noise: every hypothesis falls below the support floor (test_matching.py:246-254)."""
    from paper_2007_08576_b200.exceptions import NoValidHypothesis
    from paper_2007_08576_b200.matching import MatchSet, PreselectConfig, preselect_inliers

    rng = np.random.default_rng(14)
    src = rng.uniform(-500.0, 500.0, (50, 3))
    dst = rng.uniform(-500.0, 500.0, (50, 3))
    with pytest.raises(NoValidHypothesis):
        preselect_inliers(MatchSet.from_pairs(src, dst), PreselectConfig(seed=0))


def test_preselect_translation_invariance_bitwise_on_grid():
    """Shifting the observed points by a grid-exact vector changes no bit of the result
    (test_matching.py:209-223): rectification cancels the shift exactly."""
    from paper_2007_08576_b200.matching import MatchSet, PreselectConfig, preselect_inliers

    grid = 1.0 / 1024.0
    src, dst, _ = _rigid_matches(64, 0.3, seed=11, grid=grid)
    shift = np.array([32.0 + 5.0 * grid, -640.0 * grid, 12.25])
    cfg = PreselectConfig(seed=3)
    a = preselect_inliers(MatchSet.from_pairs(src, dst), cfg)
    b = preselect_inliers(MatchSet.from_pairs(src, dst + shift), cfg)
    assert a.reference_index == b.reference_index
    np.testing.assert_array_equal(a.matches.weights, b.matches.weights)
    np.testing.assert_array_equal(a.matches.preselected, b.matches.preselected)
    np.testing.assert_array_equal(a.rotation, b.rotation)
    np.testing.assert_array_equal(a.residuals, b.residuals)


def test_preselect_small_sets_use_every_reference():
    """Below n_references the search is exhaustive, so the seed is irrelevant
    (test_matching.py:200-206); every true inlier is flagged."""
    from paper_2007_08576_b200.matching import MatchSet, PreselectConfig, preselect_inliers

    src, dst, inlier = _rigid_matches(12, 0.25, seed=10)
    a = preselect_inliers(MatchSet.from_pairs(src, dst), PreselectConfig(seed=0))
    b = preselect_inliers(MatchSet.from_pairs(src, dst), PreselectConfig(seed=999))
    np.testing.assert_array_equal(a.matches.weights, b.matches.weights)
    assert a.matches.preselected[inlier].all()


def test_preselect_degenerate_and_too_few():
    from paper_2007_08576_b200.exceptions import NoValidHypothesis
    from paper_2007_08576_b200.matching import MatchSet, PreselectConfig, preselect_inliers

    with pytest.raises(NoValidHypothesis):
        preselect_inliers(MatchSet.from_pairs(np.zeros((2, 3)), np.ones((2, 3))), PreselectConfig())
    # collinear matches: every hypothesis is rank-1 -> degenerate (matching.py:122)
    s = np.linspace(0, 10, 12)[:, None] * np.array([[1.0, 2.0, 3.0]])
    with pytest.raises(NoValidHypothesis):
        preselect_inliers(MatchSet.from_pairs(s, s + 1.0), PreselectConfig())
