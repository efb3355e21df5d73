"""Sequence tracking: template build, per-frame track, warm starts.

Mirrors deformtrack/tracking.py: ``FrameResult`` (25-32), ``prepare_template`` (35-45),
``annotate_matches`` (48-64), ``track_frame`` (67-95), ``track_sequence`` (98-112).

``track_frame`` runs preselection, the LM solve and the output warp in ONE device call
(dt_track_frame): the matches cross the boundary once, are preselected on the GPU, and
the annotated weights feed the feature term without a host round trip.

``Tracker`` is the device-resident per-sequence object behind the north star's
"per-frame track()": the warm start stays on the device between frames, and frames can
carry either 3D match pairs or raw ORB descriptors + keypoints (Hamming-matched on the
device against the template features).
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from ._lib import DT_ERR_NO_VALID_HYPOTHESIS
from ._session import SESSIONS, DeviceTracker, make_config, nvh_message
from .config import RunConfig
from .correspond import Observation
from .energy import EnergyReport
from .exceptions import NoValidHypothesis
from .matching import MatchSet, preselect_inliers, reference_indices
from .solver import report_from_outputs
from .warpfield import ControlGraph, Template, bind_template, sample_control_points


@dataclass
class FrameResult:
    frame_id: int
    graph: ControlGraph
    points: np.ndarray
    normals: np.ndarray
    matches: MatchSet | None
    report: EnergyReport


def prepare_template(template: Template, config: RunConfig) -> tuple[Template, ControlGraph]:
    """Sample the control graph and bind the template to it (tracking.py:35-45), on the
    device; config.device.template_build picks the bit-identical route ("exact": the
    weights with numpy's exp, the binding with the kd-tree) or the all-device one."""
    on_dev = config.device.template_build == "device"
    graph = sample_control_points(template, config.sampling.radius,
                                  connection_sigma=config.sampling.effective_connection_sigma,
                                  exact_weights=not on_dev)
    bound = bind_template(template, graph, k=config.sampling.bind_k,
                          sigma=config.sampling.effective_bind_sigma, device=on_dev)
    return bound, graph


def annotate_matches(matches: MatchSet | None, config: RunConfig):
    """Preselect on the device; on NoValidHypothesis return zero-weight matches and a
    warning, leaving the frame to run without the feature term (tracking.py:48-64)."""
    if matches is None or len(matches) == 0:
        return matches, None
    try:
        return preselect_inliers(matches, config.make_preselect_config()).matches, None
    except NoValidHypothesis as e:
        n = len(matches)
        dropped = MatchSet(matches.template_points, matches.observed_points, np.zeros(n),
                           np.zeros(n, dtype=bool))
        return dropped, f"match preselection failed ({e}); feature term dropped"


def _frame_config(graph: ControlGraph, observation: Observation, config: RunConfig):
    return make_config(observation.camera, config.energy, config.make_solver_config(),
                       config.make_preselect_config(), sampling_radius=graph.sampling_radius,
                       z_min=observation.z_min, z_max=observation.z_max,
                       cluster_size=config.device.cluster_size,
                       max_hamming=config.device.max_hamming)


def track_frame(template: Template, graph: ControlGraph, observation: Observation,
                matches: MatchSet | None, config: RunConfig, *,
                match_binding=None) -> FrameResult:
    """Preselect + solve + output warp from the warm start in ``graph``
    (tracking.py:67-95), in one device call. ``match_binding``: optional (idx, w)
    binding of the matches' template points (default: bound on the device)."""
    t0 = time.perf_counter()
    if not template.is_bound:
        raise ValueError("template must be bound to the control graph first")
    cfg = _frame_config(graph, observation, config)
    trk = SESSIONS.get(template, graph, cfg)
    trk.set_warps(graph.warps)
    have = matches is not None and len(matches) > 0
    refs = reference_indices(len(matches), config.make_preselect_config()) if have else None
    out = trk.track(
        observation.depth,
        None if observation.normals_on_device else observation.normals,
        pairs=(matches.template_points, matches.observed_points) if have else None,
        match_binding=match_binding if have else None,
        refs=refs,
        frame_id=observation.frame_id,
        want_points=True,
    )
    annotated = matches
    warning = None
    if have:
        n = len(matches)
        annotated = MatchSet(matches.template_points.copy(), matches.observed_points.copy(),
                             out.match_weights[:n].copy(), out.match_flags[:n].astype(bool))
        if int(out.report.preselect_status) == DT_ERR_NO_VALID_HYPOTHESIS:
            annotated = MatchSet(matches.template_points, matches.observed_points, np.zeros(n),
                                 np.zeros(n, dtype=bool))
            warning = f"match preselection failed ({nvh_message(n)}); feature term dropped"
    report = report_from_outputs(out, observation.frame_id, annotated)
    report.timings["solve_s"] = time.perf_counter() - t0
    if warning is not None:
        report.warnings.append(warning)
    return FrameResult(
        frame_id=observation.frame_id,
        graph=graph.with_warps(out.warps.copy()),
        points=out.points,
        normals=out.normals,
        matches=annotated,
        report=report,
    )


def track_sequence(template: Template, observations: Sequence[Observation],
                   matches_per_frame: Sequence[MatchSet | None] | None,
                   config: RunConfig) -> list[FrameResult]:
    """Track a sequence in order, threading the warps frame to frame (tracking.py:98-112)."""
    bound, graph = prepare_template(template, config)
    results: list[FrameResult] = []
    for i, obs in enumerate(observations):
        m = None if matches_per_frame is None else matches_per_frame[i]
        res = track_frame(bound, graph, obs, m, config)
        graph = res.graph
        results.append(res)
    return results


class Tracker:
    """Device-resident tracker of one sequence: ``track()`` per frame.

    Construct from a bound template + graph (``prepare_template``) and a camera. The
    warm start stays on the device; ``track`` accepts a depth map plus either a
    ``MatchSet`` (preselected on the device) or ORB descriptors + integer keypoints
    matched against ``set_features``' template descriptors by brute-force Hamming
    distance on the device.
    """

    def __init__(self, template: Template, graph: ControlGraph, camera, config: RunConfig,
                 z_min: float = 1.0, z_max: float = 1.0e5):
        if not template.is_bound:
            raise ValueError("template must be bound to the control graph first")
        self.template = template
        self.graph = graph
        self.camera = camera
        self.config = config
        self._pcfg = config.make_preselect_config()
        self._exhaustive = False
        cfg = make_config(camera, config.energy, config.make_solver_config(), self._pcfg,
                          sampling_radius=graph.sampling_radius, z_min=z_min, z_max=z_max,
                          cluster_size=config.device.cluster_size,
                          max_hamming=config.device.max_hamming)
        self.device = DeviceTracker(template, graph, cfg)
        self.frame_index = 0

    def set_features(self, descriptors, points) -> None:
        """Template-side ORB features: (T, 32) uint8 descriptors and their frame-0 3D
        points (T, 3). Their control binding is fixed for the sequence, so it is computed
        once here with the reference's kd-tree (solver.py:292-296, sigma = sampling
        radius) and kept on the device."""
        from .warpfield import bind_points

        k = int(self.template.bind_indices.shape[1])
        binding = bind_points(points, self.graph.points, k, self.graph.sampling_radius)
        self.device.set_features(descriptors, points, binding)

    def set_exhaustive(self, flag: bool = True) -> None:
        """Evaluate every match as a preselection hypothesis (the paper's exhaustive
        1-point RANSAC) instead of the seeded n_references subset."""
        self._exhaustive = bool(flag)

    def reset(self, warps=None) -> None:
        self.device.set_warps(self.graph.warps if warps is None else warps)

    def track(self, depth, matches: MatchSet | None = None, *, descriptors=None,
              keypoints=None, normals=None, frame_id: int | None = None) -> FrameResult:
        fid = self.frame_index if frame_id is None else int(frame_id)
        self.frame_index += 1
        pairs = refs = None
        n = 0
        if matches is not None and len(matches) > 0:
            n = len(matches)
            pairs = (matches.template_points, matches.observed_points)
            refs = None if self._exhaustive else reference_indices(n, self._pcfg)
        out = self.device.track(depth, normals, pairs=pairs, refs=refs, frame_desc=descriptors,
                                frame_kp=keypoints, frame_id=fid, want_points=True,
                                want_matches=descriptors is not None)
        annotated = matches
        warning = None
        r = out.report
        if descriptors is not None:
            nm = int(r.n_matches) if out.match_src is not None else 0
            if nm:
                annotated = MatchSet(out.match_src[:nm].copy(), out.match_dst[:nm].copy(),
                                     out.match_weights[:nm].copy(),
                                     out.match_flags[:nm].astype(bool))
            else:  # no frame features (or none survived): an empty match set
                annotated = MatchSet(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0),
                                     np.zeros(0, dtype=bool))
            n = nm
        elif matches is not None and n:
            annotated = MatchSet(matches.template_points, matches.observed_points,
                                 out.match_weights[:n].copy(), out.match_flags[:n].astype(bool))
        if n and int(r.preselect_status) == DT_ERR_NO_VALID_HYPOTHESIS:
            warning = f"match preselection failed ({nvh_message(n)}); feature term dropped"
        report = report_from_outputs(out, fid, annotated)
        if warning:
            report.warnings.append(warning)
        graph = self.graph.with_warps(out.warps.copy())
        return FrameResult(fid, graph, out.points, out.normals, annotated, report)

    def close(self) -> None:
        self.device.close()


__all__ = ["FrameResult", "prepare_template", "annotate_matches", "track_frame",
           "track_sequence", "Tracker"]
