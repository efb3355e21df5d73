"""Per-frame Levenberg-Marquardt solve on the device.

Mirrors deformtrack/solver.py: ``SolverConfig`` (43-71), ``chunk_slices`` (74-77),
``_solve_damped`` (217-258), ``apply_step`` (261-264) and ``solve_frame`` (267-378).

``solve_frame`` hands the frame to a device-resident tracker (csrc/dt_tracker.cu): the
whole LM loop -- relink, linearization, per-control damped 6x6 Cholesky, tentative
value pass, accept/reject and the damping ladder -- runs in one thread-block-cluster
kernel launch (csrc/dt_solver.cu), with the reference's control flow: the step-norm
test before the step (solver.py:327-331), strict-decrease acceptance (336), per-control
damping increase on Cholesky failure (321-326), stalls that keep going (348-355), and
a final relinked value pass with recomputed robust and rigidity weights (360-376).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from ._lib import check, lib
from ._session import SESSIONS, make_config
from .correspond import Observation
from .energy import EnergyReport, EnergyWeights
from .matching import MatchSet
from .warpfield import ControlGraph, Template


@dataclass
class SolverConfig:
    """Iteration budget, damping schedule, gates, and parallelism (solver.py:43-71).

    ``n_chunks`` and ``n_threads`` are kept for API compatibility; the device
    reductions are deterministic for any launch shape, so neither changes results.
    ``cluster_size`` picks the thread-block cluster of the device solver (0 = largest
    the device supports)."""

    max_outer_iters: int = 10
    lambda_init: float = 1e-3
    lambda_decrease: float = 0.1
    lambda_increase: float = 10.0
    lambda_min: float = 1e-9
    lambda_max: float = 1e9
    max_retries: int = 3
    step_tol: float = 1e-4
    cost_tol: float = 1e-6
    gate_distance: float = 20.0
    gate_angle_deg: float = 60.0
    n_chunks: int = 8
    n_threads: int = 1
    cluster_size: int = 0

    def __post_init__(self) -> None:
        if self.max_outer_iters < 1 or self.max_retries < 0:
            raise ValueError("iteration budgets must be positive")
        if not (0.0 < self.lambda_min <= self.lambda_init <= self.lambda_max):
            raise ValueError("lambda_init must lie inside [lambda_min, lambda_max]")
        if self.lambda_decrease >= 1.0 or self.lambda_increase <= 1.0:
            raise ValueError("damping factors must shrink on accept and grow on reject")
        if self.n_chunks < 1 or self.n_threads < 1:
            raise ValueError("n_chunks and n_threads must be at least 1")
        if self.step_tol < 0.0 or self.cost_tol < 0.0:
            raise ValueError("tolerances must be non-negative")


def chunk_slices(n_items: int, n_chunks: int) -> list[slice]:
    """Contiguous near-equal partition of range(n_items), empty chunks dropped."""
    cuts = [(n_items * j) // n_chunks for j in range(n_chunks + 1)]
    return [slice(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _solve_damped(A, b, lam) -> tuple[np.ndarray, np.ndarray]:
    """Batched damped Cholesky solve (A_i + lam_i diag(max(diag A_i, 1e-12))) x = b_i,
    failed controls isolated with a zero step (solver.py:217-258); device."""
    A = np.ascontiguousarray(A, dtype=np.float64).reshape(-1, 6, 6)
    m = A.shape[0]
    Ad = dev.to_device(A)
    bd = dev.to_device(np.asarray(b, dtype=np.float64).reshape(m, 6))
    ld = dev.to_device(np.broadcast_to(np.asarray(lam, dtype=np.float64), (m,)).copy())
    delta = dev.empty((m, 6))
    ok = dev.empty((m,), np.uint8)
    check(lib.dt_solve_damped(dev.ptr(Ad), dev.ptr(bd), dev.ptr(ld), m, dev.ptr(delta),
                              dev.ptr(ok), dev.stream()), "_solve_damped")
    return dev.to_host(delta), dev.to_host(ok).astype(bool)


def apply_step(warps, delta) -> np.ndarray:
    """Left-compose exp(delta) onto each warp and renormalize (solver.py:261-264); device."""
    W = np.ascontiguousarray(warps, dtype=np.float64).reshape(-1, 8)
    m = W.shape[0]
    Wd = dev.to_device(W)
    Dd = dev.to_device(np.asarray(delta, dtype=np.float64).reshape(m, 6))
    out = dev.empty((m, 8))
    check(lib.dt_apply_step(dev.ptr(Wd), dev.ptr(Dd), m, dev.ptr(out), dev.stream()),
          "apply_step")
    return dev.to_host(out)


def report_from_outputs(out, frame_id: int, matches: MatchSet | None) -> EnergyReport:
    """EnergyReport (energy.py:107-168) from the device frame outputs."""
    r = out.report
    rep = EnergyReport(frame_id=frame_id)
    rep.icp_cost = float(r.icp_cost)
    rep.feature_cost = float(r.feature_cost)
    rep.arap_cost = float(r.arap_cost)
    rep.total_cost = float(r.total_cost)
    rep.n_correspondences = int(r.n_correspondences)
    rep.outer_iterations = int(r.outer_iterations)
    rep.accepted_steps = int(r.accepted_steps)
    rep.rejected_steps = int(r.rejected_steps)
    rep.stalled = bool(r.stalled)
    rep.converged = bool(r.converged)
    rep.final_step_norm = float(r.final_step_norm)
    rep.cost_history = [list(x) for x in out.cost_history]
    rep.lambda_history = [list(x) for x in out.lambda_history]
    rep.warnings = [f"lm step stalled at outer iteration {i + 1}"
                    for i, s in enumerate(out.stalled) if s]
    rep.control_data_weights = [float(x) for x in out.control_data_weights]
    if matches is not None:
        rep.n_matches = len(matches)
        rep.n_preselected = int(np.count_nonzero(matches.preselected))
        rep.match_weight_sum = float(np.sum(matches.weights))
    return rep


def solve_frame(template: Template, graph: ControlGraph, observation: Observation,
                matches: MatchSet | None, weights: EnergyWeights, config: SolverConfig,
                frame_id: int = 0, *, match_binding=None) -> tuple[ControlGraph, EnergyReport]:
    """Track one frame from the warm start in ``graph`` (solver.py:267-378). The input
    graph is not modified; returns the solved graph and the frame's report.

    ``match_binding`` (optional, not in the reference signature): (idx, w) of the
    matches' template points; by default they are bound on the device each frame
    (k nearest controls, exact distance ties to the lower control index)."""
    t0 = time.perf_counter()
    if not template.is_bound:
        raise ValueError("template must be bound to the control graph first")
    cfg = make_config(observation.camera, weights, config, sampling_radius=graph.sampling_radius,
                      z_min=observation.z_min, z_max=observation.z_max,
                      cluster_size=config.cluster_size)
    trk = SESSIONS.get(template, graph, cfg)
    trk.set_warps(graph.warps)
    use = matches is not None and len(matches) > 0 and bool(np.any(matches.weights > 0.0))
    out = trk.track(
        observation.depth,
        None if observation.normals_on_device else observation.normals,
        pairs=(matches.template_points, matches.observed_points) if use else None,
        match_w=matches.weights if use else None,
        match_binding=match_binding if use else None,
        frame_id=frame_id,
        want_points=False,
    )
    report = report_from_outputs(out, frame_id, matches)
    report.timings["solve_s"] = time.perf_counter() - t0
    return graph.with_warps(out.warps.copy()), report


__all__ = ["SolverConfig", "chunk_slices", "_solve_damped", "apply_step", "solve_frame"]
