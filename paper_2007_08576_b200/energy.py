"""Energy weights, the per-frame report, and small energy helpers.

Mirrors the public surface of deformtrack/energy.py: ``EnergyWeights`` (49-65),
``EnergyReport`` (107-168), ``tukey_weight`` (171-176), ``arap_weight_from_support``
(394-402), ``warp_increment_basis`` (205-219) and the angle-guard constants (45-46).
Row evaluation itself lives in the CUDA kernels (csrc/dt_math.cuh, csrc/dt_solver.cu).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PARAM_DIM = 6
ANGLE_MIN_NORM = 1e-6
ANGLE_COLLINEAR_EPS = 1e-14


@dataclass
class EnergyWeights:
    """Term multipliers and robust scale of the total energy (energy.py:49-65)."""

    feature_weight: float = 10.0
    arap_weight: float = 1.0
    angle_weight: float = 20.0
    rotation_weight: float = 100.0
    tukey_scale: float = 10.0
    data_floor: float = 1.0

    def __post_init__(self) -> None:
        if self.tukey_scale <= 0.0:
            raise ValueError("tukey_scale must be positive")
        smallest = min(self.feature_weight, self.arap_weight, self.angle_weight,
                       self.rotation_weight, self.data_floor)
        if smallest < 0.0:
            raise ValueError("energy weights must be non-negative")


@dataclass
class EnergyReport:
    """Per-frame energies and solver diagnostics (energy.py:107-168).

    ``timings`` holds wall-clock bookkeeping and stays out of :meth:`to_dict`, so
    serialized reports are reproducible bit for bit.
    """

    frame_id: int = 0
    icp_cost: float = 0.0
    feature_cost: float = 0.0
    arap_cost: float = 0.0
    total_cost: float = 0.0
    n_correspondences: int = 0
    n_matches: int = 0
    n_preselected: int = 0
    match_weight_sum: float = 0.0
    match_support: float = 0.0
    outer_iterations: int = 0
    accepted_steps: int = 0
    rejected_steps: int = 0
    stalled: bool = False
    converged: bool = False
    final_step_norm: float = 0.0
    cost_history: list[list[float]] = field(default_factory=list)
    lambda_history: list[list[float]] = field(default_factory=list)
    control_data_weights: list[float] = field(default_factory=list)
    warnings: list[str] = field(default_factory=list)
    timings: dict[str, float] = field(default_factory=dict, compare=False)

    def to_dict(self) -> dict:
        return {
            "frame_id": self.frame_id,
            "energy": {
                "icp": self.icp_cost,
                "feature": self.feature_cost,
                "arap": self.arap_cost,
                "total": self.total_cost,
            },
            "counts": {
                "correspondences": self.n_correspondences,
                "matches": self.n_matches,
                "preselected": self.n_preselected,
            },
            "match_weight_sum": self.match_weight_sum,
            "match_support": self.match_support,
            "solver": {
                "outer_iterations": self.outer_iterations,
                "accepted_steps": self.accepted_steps,
                "rejected_steps": self.rejected_steps,
                "stalled": self.stalled,
                "converged": self.converged,
                "final_step_norm": self.final_step_norm,
                "cost_history": [list(x) for x in self.cost_history],
                "lambda_history": [list(x) for x in self.lambda_history],
            },
            "control_data_weights": list(self.control_data_weights),
            "warnings": list(self.warnings),
        }


def tukey_weight(residuals, scale: float) -> np.ndarray:
    """Tukey biweight (1 - (r/c)^2)^2 for |r| < c, else 0 (energy.py:171-176).

    Host-side formula for API parity; the solver evaluates the same expression on the
    device (dt_math.cuh tukey_sqrt).
    """
    u = np.asarray(residuals, dtype=np.float64) / scale
    inside = np.abs(u) < 1.0
    w = (1.0 - u * u) ** 2
    return np.where(inside, w, 0.0)


def arap_weight_from_support(support, weights: EnergyWeights) -> np.ndarray:
    """Per-control rigidity weight ``arap_weight * max(support, data_floor)``
    (energy.py:394-402)."""
    return weights.arap_weight * np.maximum(np.asarray(support, dtype=np.float64),
                                            weights.data_floor)


def warp_increment_basis(warps) -> np.ndarray:
    """d(exp(xi) * W)/d xi at xi = 0, (m, 8, 6) per warp (energy.py:205-219), evaluated
    on the device (dt_warp_increment_basis)."""
    from . import _device as dev
    from ._lib import check, lib

    W = dev.to_device(np.atleast_2d(np.asarray(warps, dtype=np.float64)))
    m = W.shape[0]
    out = dev.empty((m, 8, 6))
    check(lib.dt_warp_increment_basis(dev.ptr(W), m, dev.ptr(out), dev.stream()),
          "warp_increment_basis")
    return dev.to_host(out)


__all__ = [
    "PARAM_DIM",
    "ANGLE_MIN_NORM",
    "ANGLE_COLLINEAR_EPS",
    "EnergyWeights",
    "EnergyReport",
    "tukey_weight",
    "arap_weight_from_support",
    "warp_increment_basis",
]
