"""Pin the oracle to the reference: every golden fixture was produced by the reference
(tests/golden/make_golden.py); the oracle must reproduce it -- bit for bit where the
reference's arithmetic is deterministic C-level code (the four kernels, normals, basis,
transforms, step, the LM loop that calls them)."""

import numpy as np
import pytest

from oracle import kernels as OK
from oracle import pipeline as OP
from tests.fixtures import SOLVER_CASES, jload, load, solver_case


@pytest.fixture(scope="module")
def kz():
    return load("kernels")


def test_kernels_bitwise(kz):
    m = kz["warps"].shape[0]
    np.testing.assert_array_equal(OP.increment_basis(kz["warps"]), kz["basis"])
    R, t = OP.transforms(kz["warps"])
    np.testing.assert_array_equal(R, kz["R"])
    np.testing.assert_array_equal(t, kz["t"])
    got = OK.icp_reduce(kz["points"], kz["obs_normals"], kz["obs_points"], kz["bind_idx"],
                        kz["alpha"], kz["warps"], kz["basis"], 10.0, np.zeros(0), False, True, 8, m)
    for g, name in zip(got, ("partial", "support", "cost", "r")):
        np.testing.assert_array_equal(g, kz[f"icp_{name}"])
    gv = OK.icp_reduce(kz["points"], kz["obs_normals"], kz["obs_points"], kz["bind_idx"],
                       kz["alpha"], kz["warps"], kz["basis"], 10.0, np.zeros(0), False, False, 8, m)
    np.testing.assert_array_equal(gv[2], kz["icpv_cost"])
    assert not gv[0].any()
    gf = OK.icp_reduce(kz["points"], kz["obs_normals"], kz["obs_points"], kz["bind_idx"],
                       kz["alpha"], kz["moved"], OP.increment_basis(kz["moved"]), 10.0,
                       kz["frozen"], True, True, 8, m)
    for g, name in zip(gf, ("partial", "support", "cost", "r")):
        np.testing.assert_array_equal(g, kz[f"icpf_{name}"])
    a = kz["feat_active"]
    gfe = OK.feature_reduce(kz["points"][a], kz["obs_points"][a], kz["match_w"][a],
                            kz["bind_idx"][a], kz["alpha"][a], kz["warps"], kz["basis"], 10.0,
                            True, 8, m)
    for g, name in zip(gfe, ("partial", "support", "cost")):
        np.testing.assert_array_equal(g, kz[f"feat_{name}"])
    ga = OK.arap_reduce(kz["ctrl"], R, t, kz["warps"], kz["edges"], kz["edge_w"], kz["wa"], 20.0,
                        100.0, True, 8, m)
    np.testing.assert_array_equal(ga[0], kz["arap_partial"])
    np.testing.assert_array_equal(ga[1], kz["arap_cost"])


def test_thread_count_does_not_change_bits(kz):
    m = kz["warps"].shape[0]
    outs = []
    for th in (1, 2, 4):
        OK.set_threads(th)
        outs.append(OK.icp_reduce(kz["points"], kz["obs_normals"], kz["obs_points"],
                                  kz["bind_idx"], kz["alpha"], kz["warps"], kz["basis"], 10.0,
                                  np.zeros(0), False, True, 8, m))
    OK.set_threads(OK.max_threads())
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            np.testing.assert_array_equal(a, b)


def test_observation_normals_and_rasterize_bitwise(kz):
    nn = OP.observation_normals(kz["wr_depth"], 120.0, 120.0, 23.5, 23.5)
    np.testing.assert_array_equal(nn, kz["wr_obs_normals"])
    np.testing.assert_array_equal(OP.valid_mask(kz["wr_depth"]), kz["wr_valid_px"])
    got = OK.warp_and_rasterize(kz["wr_points"], kz["normals"], kz["bind_idx"], kz["alpha"],
                                kz["warps"], kz["wr_depth"], kz["wr_valid_px"], nn, 120.0, 120.0,
                                23.5, 23.5, 8.0, float(np.cos(np.deg2rad(60.0))), 8)
    for g, name in zip(got, ("p", "n", "valid", "obs_p", "obs_n", "pixels")):
        np.testing.assert_array_equal(g, kz[f"wr_{name}"])
    assert 0 < kz["wr_valid"].sum() < len(kz["wr_valid"])


def test_damped_solve_and_step_bitwise(kz):
    d, ok = OP.damped_solve(kz["sd_A"], kz["sd_b"], kz["sd_lam"])
    np.testing.assert_array_equal(ok, kz["sd_ok"])
    np.testing.assert_array_equal(d, kz["sd_delta"])
    assert ok.tolist()[-1] is False
    np.testing.assert_array_equal(OP.compose_step(kz["warps"], kz["step_delta"]), kz["step_out"])


def test_bind_points_matches_reference(kz):
    idx, w = OP.bind(kz["bind_pts"], kz["bind_ctrl"], 4, 7.0)
    np.testing.assert_array_equal(idx, kz["bind_idx_ref"])
    np.testing.assert_array_equal(w, kz["bind_w_ref"])


def _weights(d):
    return OP.Weights(**d)


def _schedule(d):
    keys = OP.Schedule.__dataclass_fields__.keys()
    return OP.Schedule(**{k: v for k, v in d.items() if k in keys})


@pytest.mark.parametrize("name", SOLVER_CASES)
def test_solve_frame_reproduces_reference(name):
    c = solver_case(name)
    fx, fy, cx, cy = c["cam"]
    normals = OP.observation_normals(c["depth"], fx, fy, cx, cy)
    matches = None if c["matches"] is None else c["matches"][:3]
    res = OP.solve(c["tpl"], c["graph"], c["warps_in"], c["depth"], normals, c["cam"], matches,
                   _weights(c["weights"]), _schedule(c["solver"]), c["radius"])
    rep = c["report"]
    np.testing.assert_array_equal(res.warps, c["warps_out"])
    assert res.total_cost == rep["energy"]["total"]
    assert res.icp_cost == rep["energy"]["icp"]
    assert res.arap_cost == rep["energy"]["arap"]
    assert res.feature_cost == rep["energy"]["feature"]
    assert res.n_correspondences == rep["counts"]["correspondences"]
    s = rep["solver"]
    assert res.outer_iterations == s["outer_iterations"]
    assert res.accepted_steps == s["accepted_steps"]
    assert res.rejected_steps == s["rejected_steps"]
    assert res.converged == s["converged"] and res.stalled == s["stalled"]
    assert res.cost_history == s["cost_history"]
    assert res.lambda_history == s["lambda_history"]
    assert res.control_data_weights == rep["control_data_weights"]


def test_matching_reproduces_reference():
    z = load("matching")
    for i in range(int(z["n_cases"])):
        src, dst = z[f"c{i}_src"], z[f"c{i}_dst"]
        nref, seed = (int(x) for x in z[f"c{i}_cfg"])
        refs = OP.reference_draw(len(src), nref, seed)
        sel = OP.preselect(src, dst, refs)
        np.testing.assert_array_equal(sel.flags, z[f"c{i}_flags"])
        np.testing.assert_array_equal(sel.weights, z[f"c{i}_weights"])
        assert sel.reference == int(z[f"c{i}_ref"])
        assert sel.support == float(z[f"c{i}_support"])


@pytest.mark.parametrize("fixture", ["tracking", "tracking_cfg1"])
def test_track_frame_reproduces_reference(fixture):
    z = load(fixture)
    cfg = jload(z["config"])
    tpl = (z["t_points"], z["t_normals"], z["bind_idx"], z["bind_w"])
    graph = (z["ctrl"], z["edges"], z["edge_w"])
    fx, fy, cx, cy = (float(x) for x in z["cam"][:4])
    wts = OP.Weights(**cfg["energy"])
    sch = _schedule({**cfg["solver"], "gate_distance": cfg["gates"]["distance_mm"],
                     "gate_angle_deg": cfg["gates"]["angle_deg"]})
    pre = cfg["preselect"]
    for f in range(int(z["n_frames"])):
        depth = z[f"f{f}_depth"]
        src, dst = z[f"f{f}_m_src"], z[f"f{f}_m_dst"]
        refs = OP.reference_draw(len(src), pre["n_references"], cfg["seed"])
        res, sel, pts, _ = OP.track(
            tpl, graph, z[f"f{f}_warps_in"], depth, OP.observation_normals(depth, fx, fy, cx, cy),
            (fx, fy, cx, cy), (src, dst), wts, sch, float(z["radius"]), refs=refs,
            pre=(pre["distance_threshold"], pre["n_reweight_iters"], pre["inlier_weight_min"],
                 pre["min_support"]))
        np.testing.assert_array_equal(sel.flags, z[f"f{f}_m_flags"])
        np.testing.assert_array_equal(sel.weights, z[f"f{f}_m_w"])
        np.testing.assert_array_equal(res.warps, z[f"f{f}_warps_out"])
        rep = jload(z[f"f{f}_report"])
        assert res.total_cost == rep["energy"]["total"]
        assert res.n_correspondences == rep["counts"]["correspondences"]
        # warp_all uses einsum blending in the reference; allow its last-ulp rounding
        np.testing.assert_allclose(pts, z[f"f{f}_points"], rtol=0, atol=1e-9)


@pytest.mark.parametrize("name", ["patch", "cloud", "cloud_k6", "small", "tiny"])
def test_point_normals_reproduce_reference(name):
    """The oracle's estimate_point_normals restatement against the reference's own
    output (correspond.py:198-220)."""
    z = load("point_normals")
    nrm, _ = OP.point_normals(z[f"{name}_pts"], int(z[f"{name}_k"]))
    np.testing.assert_array_equal(nrm, z[f"{name}_nrm"])
