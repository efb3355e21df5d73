"""Feature matches, ORB Hamming matching, and consensus preselection.

Mirrors deformtrack/matching.py: ``MatchSet`` (21-55), ``PreselectConfig`` (58-80),
``PreselectionResult`` (83-91), ``reweight`` (133-136), ``soft_weight`` (139-142),
``rectify`` (94-105) and ``preselect_inliers`` (174-226). ``match_descriptors`` is the
brute-force 256-bit Hamming matcher of the north star (part 3a), which the reference
leaves to an upstream ORB stage.

Device work: ``preselect_inliers`` runs every reference hypothesis as one warp on the
GPU (dt_preselect); ``match_descriptors`` is dt_hamming_match. The only host step is
drawing the reference indices with numpy's Generator, exactly as matching.py:189-193,
so the hypotheses are the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device as dev
from ._lib import DT_ERR_NO_VALID_HYPOTHESIS, PreselectParams, check, lib
from .exceptions import NoValidHypothesis, TooFewMatches


@dataclass
class MatchSet:
    """Reference-frame points paired with their observed positions (matching.py:21-55)."""

    template_points: np.ndarray
    observed_points: np.ndarray
    weights: np.ndarray
    preselected: np.ndarray

    def __post_init__(self) -> None:
        self.template_points = np.asarray(self.template_points, dtype=np.float64)
        self.observed_points = np.asarray(self.observed_points, dtype=np.float64)
        self.weights = np.asarray(self.weights, dtype=np.float64)
        self.preselected = np.asarray(self.preselected, dtype=bool)
        n = self.template_points.shape[0]
        if self.template_points.shape != (n, 3) or self.observed_points.shape != (n, 3):
            raise ValueError("match arrays must be (n, 3)")
        if self.weights.shape != (n,) or self.preselected.shape != (n,):
            raise ValueError("weights and flags must be (n,)")

    @classmethod
    def from_pairs(cls, template_points, observed_points) -> "MatchSet":
        tp = np.asarray(template_points, dtype=np.float64)
        n = tp.shape[0]
        return cls(tp, observed_points, weights=np.ones(n), preselected=np.zeros(n, dtype=bool))

    def __len__(self) -> int:
        return int(self.template_points.shape[0])


@dataclass
class PreselectConfig:
    """Consensus-search knobs (matching.py:58-80)."""

    distance_threshold: float = 5.0
    n_references: int = 30
    n_reweight_iters: int = 10
    inlier_weight_min: float = 0.5
    min_support: float = 0.2
    seed: int = 0

    def __post_init__(self) -> None:
        if self.distance_threshold <= 0.0:
            raise ValueError("distance_threshold must be positive")
        if not 0.0 <= self.min_support <= 1.0:
            raise ValueError("min_support must lie in [0, 1]")
        if self.n_references < 1 or self.n_reweight_iters < 1:
            raise ValueError("n_references and n_reweight_iters must be >= 1")

    def params(self) -> PreselectParams:
        return PreselectParams(float(self.distance_threshold), int(self.n_reweight_iters),
                               float(self.inlier_weight_min), float(self.min_support))


@dataclass
class PreselectionResult:
    """Winning hypothesis and the annotated matches (matching.py:83-91)."""

    matches: MatchSet
    rotation: np.ndarray
    reference_index: int
    support: float
    residuals: np.ndarray = field(repr=False)


def rectify(template_points, observed_points, reference: int) -> tuple[np.ndarray, np.ndarray]:
    """Subtract the reference match from both sides (matching.py:94-105)."""
    src = np.asarray(template_points, dtype=np.float64)
    dst = np.asarray(observed_points, dtype=np.float64)
    if src.shape[0] < 2:
        raise TooFewMatches("rectification needs at least two matches")
    return src - src[reference], dst - dst[reference]


def reweight(residuals, distance_threshold: float) -> np.ndarray:
    """min(H/d, 1), zero residual -> 1 (matching.py:133-136)."""
    d = np.asarray(residuals, dtype=np.float64)
    return np.where(d > distance_threshold, distance_threshold / np.maximum(d, 1e-300), 1.0)


def soft_weight(residuals, distance_threshold: float) -> np.ndarray:
    """clip(1 - d / (5H), 0, 1) (matching.py:139-142)."""
    d = np.asarray(residuals, dtype=np.float64)
    return np.clip(1.0 - d / (5.0 * distance_threshold), 0.0, 1.0)


def reference_indices(n: int, config: PreselectConfig) -> np.ndarray | None:
    """The hypotheses the reference evaluates (matching.py:189-193): all of them when
    n <= n_references (returned as None = exhaustive on the device), otherwise a seeded
    draw without replacement."""
    if n <= config.n_references:
        return None
    rng = np.random.default_rng(config.seed)
    return rng.choice(n, size=config.n_references, replace=False).astype(np.int64)


def preselect_inliers(matches: MatchSet, config: PreselectConfig) -> PreselectionResult:
    """1-point RANSAC + reweighting consensus (matching.py:174-226), on the device.

    Raises NoValidHypothesis when no hypothesis survives (including n < 3)."""
    n = len(matches)
    if n < 3:
        raise NoValidHypothesis(f"{n} matches cannot support a rotation hypothesis")
    refs = reference_indices(n, config)
    src = dev.to_device(matches.template_points)
    dst = dev.to_device(matches.observed_points)
    refs_d = None if refs is None else dev.to_device(refs)
    n_refs = 0 if refs is None else int(refs.shape[0])
    weights = dev.empty((n,))
    flags = dev.empty((n,), np.uint8)
    resid = dev.empty((n,))
    rot = dev.empty((9,))
    info = dev.zeros((2,), np.int64)
    support = dev.zeros((1,))
    params = config.params()
    check(lib.dt_preselect(dev.ptr(src), dev.ptr(dst), n, dev.ptr(refs_d), n_refs, params,
                           dev.ptr(weights), dev.ptr(flags), dev.ptr(resid), dev.ptr(rot),
                           dev.ptr(info), dev.ptr(support), dev.stream()), "preselect_inliers")
    info_h = dev.to_host(info)
    if int(info_h[0]) == DT_ERR_NO_VALID_HYPOTHESIS:
        raise NoValidHypothesis("every reference hypothesis was discarded")
    annotated = MatchSet(
        template_points=matches.template_points.copy(),
        observed_points=matches.observed_points.copy(),
        weights=dev.to_host(weights),
        preselected=dev.to_host(flags).astype(bool),
    )
    return PreselectionResult(
        matches=annotated,
        rotation=dev.to_host(rot).reshape(3, 3),
        reference_index=int(info_h[1]),
        support=float(dev.to_host(support)[0]),
        residuals=dev.to_host(resid),
    )


def match_descriptors(template_desc, frame_desc) -> tuple[np.ndarray, np.ndarray]:
    """Brute-force Hamming matching of 256-bit descriptors (north-star part 3a).

    template_desc (T, 32) uint8, frame_desc (F, 32) uint8 -> (index (T,) int32,
    distance (T,) int32): for every template descriptor the frame descriptor with the
    fewest differing bits, ties to the lowest frame index (-1 / 257 when F == 0).
    """
    td = np.ascontiguousarray(template_desc, dtype=np.uint8).reshape(-1, 32)
    fd = np.ascontiguousarray(frame_desc, dtype=np.uint8).reshape(-1, 32)
    nt, nf = td.shape[0], fd.shape[0]
    if nt == 0:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    T = dev.to_device(td)
    F = dev.to_device(fd) if nf else None
    idx = dev.empty((nt,), np.int32)
    dist = dev.empty((nt,), np.int32)
    check(lib.dt_hamming_match(dev.ptr(T), nt, dev.ptr(F), nf, dev.ptr(idx), dev.ptr(dist),
                               dev.stream()), "match_descriptors")
    return dev.to_host(idx), dev.to_host(dist)


__all__ = [
    "MatchSet",
    "PreselectConfig",
    "PreselectionResult",
    "rectify",
    "reweight",
    "soft_weight",
    "reference_indices",
    "preselect_inliers",
    "match_descriptors",
]
