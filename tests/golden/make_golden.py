"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is importable only there):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every input is seeded; every expected output is what deformtrack itself returns. The
GPU box never sees /root/reference: the tests read these .npz files.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from deformtrack import kernels as RK  # noqa: E402
from deformtrack.config import load_config  # noqa: E402
from deformtrack.correspond import Observation  # noqa: E402
from deformtrack.energy import EnergyWeights, warp_increment_basis  # noqa: E402
from deformtrack.geometry import (PinholeCamera, back_project, dq_from_transform,  # noqa: E402
                                  dq_to_transform_batch, quat_from_axis_angle, quat_to_matrix)
from deformtrack.matching import MatchSet, PreselectConfig, preselect_inliers  # noqa: E402
from deformtrack.solver import SolverConfig, _solve_damped, apply_step, solve_frame  # noqa: E402
from deformtrack.synth import SceneSpec, generate_sequence, scene_camera  # noqa: E402
from deformtrack.tracking import prepare_template, track_frame  # noqa: E402
from deformtrack.warpfield import (Template, bind_points, bind_template,  # noqa: E402
                                   sample_control_points, warp_all)
from scipy.spatial.transform import Rotation  # noqa: E402

OUT = Path(__file__).resolve().parent


def kernel_problem():
    """The reference's operator-test fixture (tests/test_kernels.py:58-107)."""
    rng = np.random.default_rng(42)
    m, n, k = 10, 50, 4
    ctrl = rng.uniform(-30.0, 30.0, size=(m, 3))
    warps = np.empty((m, 8))
    for i in range(m):
        axis = rng.normal(size=3)
        q = quat_from_axis_angle(axis / np.linalg.norm(axis) * rng.uniform(0.0, 0.6))
        warps[i] = dq_from_transform(quat_to_matrix(q), rng.uniform(-4.0, 4.0, size=3))
    warps[3] = -warps[3]
    points = rng.uniform(-30.0, 30.0, size=(n, 3))
    normals = rng.normal(size=(n, 3))
    normals /= np.linalg.norm(normals, axis=1, keepdims=True)
    bind_idx = np.argsort(rng.random((n, m)), axis=1)[:, :k].astype(np.int64)
    alpha = rng.random((n, k))
    alpha /= alpha.sum(axis=1, keepdims=True)
    obs_points = points + rng.normal(scale=2.0, size=(n, 3))
    obs_points[:4] += 25.0
    obs_normals = rng.normal(size=(n, 3))
    obs_normals /= np.linalg.norm(obs_normals, axis=1, keepdims=True)
    edges = set()
    while len(edges) < 18:
        a, b = rng.integers(0, m, size=2)
        if a < b:
            edges.add((int(a), int(b)))
    edges = np.vstack([np.array(sorted(edges), dtype=np.int64), [[2, 2]]])
    edge_w = rng.uniform(0.2, 1.0, size=edges.shape[0])
    match_w = np.r_[rng.uniform(0.3, 1.0, size=17), 0.0, 0.5, 0.0]
    return dict(ctrl=ctrl, warps=warps, points=points, normals=normals, bind_idx=bind_idx,
                alpha=alpha, obs_points=obs_points, obs_normals=obs_normals, edges=edges,
                edge_w=edge_w, match_w=match_w)


def make_kernels():
    P = kernel_problem()
    m = P["warps"].shape[0]
    basis = warp_increment_basis(P["warps"])
    R, t = dq_to_transform_batch(P["warps"])
    out = dict(P)
    out["basis"] = basis
    out["R"], out["t"] = R, t
    icp = RK.icp_reduce(P["points"], P["obs_normals"], P["obs_points"], P["bind_idx"], P["alpha"],
                        P["warps"], basis, 10.0, np.zeros(0), False, True, 8, m)
    for name, v in zip(("partial", "support", "cost", "r"), icp):
        out[f"icp_{name}"] = v
    icpv = RK.icp_reduce(P["points"], P["obs_normals"], P["obs_points"], P["bind_idx"],
                         P["alpha"], P["warps"], basis, 10.0, np.zeros(0), False, False, 8, m)
    out["icpv_cost"] = icpv[2]
    frozen = np.sqrt(np.where(np.abs(icp[3] / 10.0) < 1.0, (1.0 - (icp[3] / 10.0) ** 2) ** 2, 0.0))
    moved = np.roll(P["warps"], 1, axis=0)
    out["moved"] = moved
    out["frozen"] = frozen
    icpf = RK.icp_reduce(P["points"], P["obs_normals"], P["obs_points"], P["bind_idx"],
                         P["alpha"], moved, warp_increment_basis(moved), 10.0, frozen, True, True,
                         8, m)
    for name, v in zip(("partial", "support", "cost", "r"), icpf):
        out[f"icpf_{name}"] = v
    act = np.flatnonzero(P["match_w"] > 0.0)
    out["feat_active"] = act
    feat = RK.feature_reduce(P["points"][act], P["obs_points"][act], P["match_w"][act],
                             P["bind_idx"][act], P["alpha"][act], P["warps"], basis, 10.0, True,
                             8, m)
    for name, v in zip(("partial", "support", "cost"), feat):
        out[f"feat_{name}"] = v
    wa = np.random.default_rng(7).uniform(0.5, 3.0, size=m)
    out["wa"] = wa
    arap = RK.arap_reduce(P["ctrl"], R, t, P["warps"], P["edges"], P["edge_w"], wa, 20.0, 100.0,
                          True, 8, m)
    out["arap_partial"], out["arap_cost"] = arap
    # warp_and_rasterize against a noisy depth frame with dead bands (test_kernels.py:223-256)
    cam = PinholeCamera(fx=120.0, fy=120.0, cx=23.5, cy=23.5, width=48, height=48)
    rng = np.random.default_rng(3)
    depth = rng.uniform(280.0, 320.0, size=(48, 48))
    depth[10:14, :] = 0.0
    depth[:, 30:33] = np.nan
    obs = Observation.from_depth(depth, cam)
    pts = P["points"].copy()
    pts[:, :2] *= 1.5
    pts[:, 2] = 300.0 + 0.5 * pts[:, 2]
    pts[:3, 2] = -50.0
    out["wr_points"] = pts
    out["wr_depth"] = depth
    out["wr_valid_px"] = np.ascontiguousarray(obs.valid)
    out["wr_obs_normals"] = obs.normals
    wr = RK.warp_and_rasterize(pts, P["normals"], P["bind_idx"], P["alpha"], P["warps"], depth,
                               np.ascontiguousarray(obs.valid), obs.normals, cam.fx, cam.fy,
                               cam.cx, cam.cy, 8.0, float(np.cos(np.deg2rad(60.0))), 8)
    for name, v in zip(("p", "n", "valid", "obs_p", "obs_n", "pixels"), wr):
        out[f"wr_{name}"] = v
    # damped solves (test_solver.py:102-124) and a step
    rng = np.random.default_rng(0)
    J = rng.normal(size=(12, 40, 6))
    A = np.einsum("mre,mrf->mef", J, J)
    b = rng.normal(size=(12, 6))
    lam = rng.uniform(1e-3, 1e-1, size=12)
    A = np.concatenate([A, -np.eye(6)[None]], axis=0)
    b = np.concatenate([b, np.ones((1, 6))], axis=0)
    lam = np.concatenate([lam, [1e-3]])
    out["sd_A"], out["sd_b"], out["sd_lam"] = A, b, lam
    out["sd_delta"], out["sd_ok"] = _solve_damped(A, b, lam)
    delta = rng.normal(size=(m, 6)) * 0.05
    delta[0] = 0.0
    out["step_delta"] = delta
    out["step_out"] = apply_step(P["warps"], delta)
    # bind_points on a jittered grid (no distance ties)
    g = np.stack(np.meshgrid(np.linspace(-20, 20, 9), np.linspace(-20, 20, 9)), -1).reshape(-1, 2)
    g = np.c_[g, np.zeros(len(g))] + rng.normal(scale=0.3, size=(len(g), 3))
    bp = rng.uniform(-25, 25, size=(200, 3))
    out["bind_ctrl"], out["bind_pts"] = g, bp
    out["bind_idx_ref"], out["bind_w_ref"] = bind_points(bp, g, 4, 7.0)
    np.savez_compressed(OUT / "kernels.npz", **out)


def plane_scene(R=np.eye(3), t=np.zeros(3), radius=4.0, hw=48, f=600.0, z0=300.0):
    """test_solver.py:35-78: a flat template and the depth of its rigidly moved copy."""
    cam = PinholeCamera(fx=f, fy=f, cx=(hw - 1) / 2.0, cy=(hw - 1) / 2.0, width=hw, height=hw)
    rows = np.arange(6, hw - 6, 2, dtype=np.float64)
    vv, uu = np.meshgrid(rows, rows, indexing="ij")
    pts = back_project(cam, uu.ravel(), vv.ravel(), np.full(uu.size, z0))
    tpl = Template(points=pts, normals=np.tile([0.0, 0.0, -1.0], (pts.shape[0], 1)))
    graph = sample_control_points(tpl, radius=radius)
    tpl = bind_template(tpl, graph)
    center = np.array([0.0, 0.0, z0])
    nrm = R @ np.array([0.0, 0.0, -1.0])
    c = R @ center + t
    v, u = np.mgrid[0:hw, 0:hw].astype(np.float64)
    denom = nrm[0] * (u - cam.cx) / cam.fx + nrm[1] * (v - cam.cy) / cam.fy + nrm[2]
    depth = float(np.dot(nrm, c)) / denom
    return cam, tpl, graph, depth, tpl.points @ R.T + t


def small_rigid(angle, axis, t, z0=300.0):
    axis = np.asarray(axis, dtype=np.float64) / np.linalg.norm(axis)
    R = quat_to_matrix(quat_from_axis_angle(axis * angle))
    center = np.array([0.0, 0.0, z0])
    return R, np.asarray(t, dtype=np.float64) + center - R @ center


def pack_case(name, cam, tpl, graph, depth, matches, wts, cfg, warps_out, report, extra=None):
    d = dict(
        cam=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height], dtype=np.float64),
        t_points=tpl.points, t_normals=tpl.normals, bind_idx=tpl.bind_indices,
        bind_w=tpl.bind_weights, ctrl=graph.points, warps_in=graph.warps, edges=graph.edges,
        edge_w=graph.edge_weights, radius=np.array(graph.sampling_radius), depth=depth,
        warps_out=warps_out, report=np.array(json.dumps(report.to_dict())),
        weights=np.array(json.dumps(wts.__dict__)),
        solver=np.array(json.dumps({k: v for k, v in cfg.__dict__.items()})),
    )
    if matches is not None:
        d["m_src"], d["m_dst"] = matches.template_points, matches.observed_points
        d["m_w"], d["m_flags"] = matches.weights, matches.preselected
    if extra:
        d.update(extra)
    np.savez_compressed(OUT / f"{name}.npz", **d)


def make_solver_cases():
    w = EnergyWeights()
    # fixed point (test_solver.py:141-148)
    cam, tpl, graph, depth, _ = plane_scene()
    cfg = SolverConfig()
    out, rep = solve_frame(tpl, graph, Observation.from_depth(depth, cam), None, w, cfg)
    pack_case("solver_fixed_point", cam, tpl, graph, depth, None, w, cfg, out.warps, rep)
    # normal-direction translation, fixed 10 iterations (test_solver.py:151-162)
    cam, tpl, graph, depth, _ = plane_scene(t=np.array([0.0, 0.0, 2.0]))
    cfg = SolverConfig(max_outer_iters=10, step_tol=0.0, cost_tol=0.0)
    out, rep = solve_frame(tpl, graph, Observation.from_depth(depth, cam), None, w, cfg)
    pack_case("solver_translation", cam, tpl, graph, depth, None, w, cfg, out.warps, rep)
    # rigid recovery with matches (test_solver.py:165-183), 20 iterations
    R, t = small_rigid(0.03, (1.0, 0.5, 0.0), (1.0, -0.5, 2.0))
    cam, tpl, graph, depth, truth = plane_scene(R, t)
    sel = np.random.default_rng(7).choice(len(tpl), size=30, replace=False)
    ms = MatchSet(tpl.points[sel], truth[sel], np.ones(30), np.ones(30, dtype=bool))
    cfg = SolverConfig(max_outer_iters=20)
    out, rep = solve_frame(tpl, graph, Observation.from_depth(depth, cam), ms, w, cfg)
    pack_case("solver_rigid_matches", cam, tpl, graph, depth, ms, w, cfg, out.warps, rep)
    # fully occluded (test_solver.py:225-235)
    cam, tpl, graph, _, _ = plane_scene()
    Rr = quat_to_matrix(quat_from_axis_angle(np.array([0.0, 0.02, 0.01])))
    prev = dq_from_transform(Rr, np.array([1.5, -0.5, 2.0]))
    graph = graph.with_warps(np.tile(prev, (len(graph), 1)))
    depth = np.zeros((cam.height, cam.width))
    cfg = SolverConfig()
    out, rep = solve_frame(tpl, graph, Observation.from_depth(depth, cam), None, w, cfg)
    pack_case("solver_occluded", cam, tpl, graph, depth, None, w, cfg, out.warps, rep)
    make_no_data_cases()


def make_no_data_cases():
    """No valid depth from the rest pose (test_solver.py:209-218): zero energy, so with the
    default tolerances the solve converges at once, and with tolerances 0 every step is
    rejected and every iteration stalls."""
    w = EnergyWeights()
    cam, tpl, graph, _, _ = plane_scene()
    depth = np.zeros((cam.height, cam.width))
    cfg = SolverConfig()
    out, rep = solve_frame(tpl, graph, Observation.from_depth(depth, cam), None, w, cfg)
    pack_case("solver_no_data", cam, tpl, graph, depth, None, w, cfg, out.warps, rep)
    cfg = SolverConfig(max_outer_iters=5, step_tol=0.0, cost_tol=0.0)
    out, rep = solve_frame(tpl, graph, Observation.from_depth(depth, cam), None, w, cfg)
    pack_case("solver_no_data_stall", cam, tpl, graph, depth, None, w, cfg, out.warps, rep)


def rigid_matches(n, outlier_fraction, seed, angle_deg=15.0, translation=10.0, box=100.0):
    """test_matching.py:17-47."""
    rng = np.random.default_rng(seed)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    R = Rotation.from_rotvec(np.deg2rad(angle_deg) * axis).as_matrix()
    t = rng.normal(size=3)
    t *= translation / np.linalg.norm(t)
    src = rng.uniform(-box / 2.0, box / 2.0, (n, 3))
    dst = src @ R.T + t
    n_out = round(n * outlier_fraction)
    out_idx = rng.choice(n, size=n_out, replace=False)
    dst[out_idx] = rng.uniform(-box / 2.0, box / 2.0, (n_out, 3))
    return src, dst


def make_matching():
    cases = {}
    for i, (n, frac, seed, nref) in enumerate([(100, 0.4, 7, 30), (100, 0.4, 11, 1000),
                                              (60, 0.2, 3, 1000), (200, 0.3, 5, 30),
                                              (25, 0.0, 2, 30), (300, 0.5, 9, 1000)]):
        src, dst = rigid_matches(n, frac, seed)
        # noise on the observed side so supports differ between hypotheses
        dst = dst + np.random.default_rng(seed + 100).normal(scale=0.4, size=dst.shape)
        cfg = PreselectConfig(n_references=nref, seed=seed)
        res = preselect_inliers(MatchSet.from_pairs(src, dst), cfg)
        cases[f"c{i}_src"], cases[f"c{i}_dst"] = src, dst
        cases[f"c{i}_cfg"] = np.array([nref, seed])
        cases[f"c{i}_weights"] = res.matches.weights
        cases[f"c{i}_flags"] = res.matches.preselected
        cases[f"c{i}_ref"] = np.array(res.reference_index)
        cases[f"c{i}_support"] = np.array(res.support)
        cases[f"c{i}_rot"] = res.rotation
        cases[f"c{i}_resid"] = res.residuals
    np.savez_compressed(OUT / "matching.npz", n_cases=np.array(6), **cases)


def make_tracking():
    """A seeded reference sequence with per-frame warm starts for teacher forcing."""
    cfg = load_config({"sampling": {"radius": 8.0}, "solver": {"max_outer_iters": 10},
                       "energy": {"arap_weight": 0.25}})
    spec = SceneSpec(resolution=(30, 30), amplitude=5.0, period=8.0, noise_sigma=0.3,
                     n_matches=60, outlier_fraction=0.2, seed=4)
    seq = generate_sequence(spec, 4)
    tpl, graph = prepare_template(seq.template, cfg)
    d = dict(t_points=tpl.points, t_normals=tpl.normals, bind_idx=tpl.bind_indices,
             bind_w=tpl.bind_weights, ctrl=graph.points, edges=graph.edges,
             edge_w=graph.edge_weights, radius=np.array(graph.sampling_radius),
             cam=np.array([seq.camera.fx, seq.camera.fy, seq.camera.cx, seq.camera.cy,
                           seq.camera.width, seq.camera.height]),
             config=np.array(json.dumps(cfg.to_dict())), n_frames=np.array(len(seq.frames)))
    g = graph
    for fr in seq.frames:
        f = fr.frame_id
        res = track_frame(tpl, g, fr.observation, fr.matches, cfg)
        d[f"f{f}_depth"] = fr.observation.depth
        d[f"f{f}_warps_in"] = g.warps
        d[f"f{f}_m_src"] = fr.matches.template_points
        d[f"f{f}_m_dst"] = fr.matches.observed_points
        d[f"f{f}_warps_out"] = res.graph.warps
        d[f"f{f}_points"] = res.points
        d[f"f{f}_normals"] = res.normals
        d[f"f{f}_m_w"] = res.matches.weights
        d[f"f{f}_m_flags"] = res.matches.preselected
        d[f"f{f}_report"] = np.array(json.dumps(res.report.to_dict()))
        d[f"f{f}_truth"] = fr.truth.points
        g = res.graph
    np.savez_compressed(OUT / "tracking.npz", **d)


def make_tracking_cfg1():
    """Config-1-sized frame (plane 71x71 at 320x240, radius 10, 500 matches, 5 iterations)
    from the reference synth, two frames teacher-forced."""
    cfg = load_config({"sampling": {"radius": 10.0}, "solver": {"max_outer_iters": 5,
                                                                "step_tol": 0.0, "cost_tol": 0.0},
                       "camera": {"fx": 648.0, "fy": 648.0, "cx": 159.5, "cy": 119.5,
                                  "width": 320, "height": 240}})
    spec = SceneSpec(surface="plane", resolution=(71, 71), deformation="sinusoidal-bend",
                     amplitude=5.0, period=20.0, noise_sigma=0.3, n_matches=500,
                     outlier_fraction=0.1, seed=1)
    cam = PinholeCamera(fx=648.0, fy=648.0, cx=159.5, cy=119.5, width=320, height=240)
    seq = generate_sequence(spec, 3, camera=cam)
    tpl, graph = prepare_template(seq.template, cfg)
    d = dict(t_points=tpl.points, t_normals=tpl.normals, bind_idx=tpl.bind_indices,
             bind_w=tpl.bind_weights, ctrl=graph.points, edges=graph.edges,
             edge_w=graph.edge_weights, radius=np.array(graph.sampling_radius),
             cam=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height]),
             config=np.array(json.dumps(cfg.to_dict())), n_frames=np.array(len(seq.frames)))
    g = graph
    for fr in seq.frames:
        f = fr.frame_id
        res = track_frame(tpl, g, fr.observation, fr.matches, cfg)
        d[f"f{f}_depth"] = fr.observation.depth
        d[f"f{f}_warps_in"] = g.warps
        d[f"f{f}_m_src"] = fr.matches.template_points
        d[f"f{f}_m_dst"] = fr.matches.observed_points
        d[f"f{f}_warps_out"] = res.graph.warps
        d[f"f{f}_points"] = res.points
        d[f"f{f}_m_w"] = res.matches.weights
        d[f"f{f}_m_flags"] = res.matches.preselected
        d[f"f{f}_report"] = np.array(json.dumps(res.report.to_dict()))
        g = res.graph
    np.savez_compressed(OUT / "tracking_cfg1.npz", **d)


def point_normal_clouds():
    """Clouds for correspond.estimate_point_normals: a curved grid patch (spacing 1,
    relief), an unstructured cloud, and the small-n cases (k clipped to n; n < 3)."""
    rng = np.random.default_rng(21)
    u, v = np.meshgrid(np.arange(-20.0, 21.0), np.arange(-20.0, 21.0), indexing="ij")
    patch = np.stack([u.ravel(), v.ravel(),
                      300.0 + 0.02 * (u.ravel() ** 2) - 0.015 * (v.ravel() ** 2)
                      + 0.3 * np.sin(u.ravel() / 3.0)], axis=1)
    cloud = rng.normal(size=(1500, 3)) * np.array([40.0, 30.0, 2.0]) + np.array([0, 0, 250.0])
    small = rng.normal(size=(5, 3)) + np.array([0, 0, 100.0])
    tiny = rng.normal(size=(2, 3)) + np.array([0, 0, 100.0])
    return {"patch": (patch, 12), "cloud": (cloud, 12), "cloud_k6": (cloud, 6),
            "small": (small, 12), "tiny": (tiny, 12)}


def make_point_normals():
    from deformtrack.correspond import estimate_point_normals

    out = {}
    for name, (pts, k) in point_normal_clouds().items():
        out[f"{name}_pts"] = pts
        out[f"{name}_k"] = np.array(k)
        out[f"{name}_nrm"] = estimate_point_normals(pts, k=k)
    np.savez_compressed(OUT / "point_normals.npz", **out)


if __name__ == "__main__":
    make_kernels()
    make_solver_cases()
    make_matching()
    make_tracking()
    make_tracking_cfg1()
    make_point_normals()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
