"""deformtrack on B200: the per-frame deformation-tracking hot path of arXiv 2007.08576
("Real-time Surface Deformation Recovery from Stereo Videos") as hand-written sm_100a
CUDA behind the reference package's own API (deformtrack: tracking / solver / matching /
kernels / estimators / config).

The compute lives in ``libdeformtrack_b200.so`` (csrc/, C-ABI in
include/deformtrack_b200.h); this package is the drop-in host layer. Importing it
requires the built library (there is no CPU fallback); calling it requires a CUDA
device.
"""

from ._lib import LIB_PATH, version  # noqa: F401  (fails loudly if the .so is missing)
from .config import RunConfig, load_config
from .correspond import CorrespondenceSet, Observation, estimate_point_normals
from .energy import EnergyReport, EnergyWeights
from .estimators import MatchInlierSelector, SurfaceDeformationTracker
from .geometry import PinholeCamera
from .matching import MatchSet, PreselectConfig, match_descriptors, preselect_inliers
from .orb import OrbDetector
from .stereo import StereoMatcher
from .solver import SolverConfig, solve_frame
from .tracking import (FrameResult, Tracker, annotate_matches, prepare_template, track_frame,
                       track_sequence)
from .warpfield import ControlGraph, Template, bind_template, sample_control_points, warp_all

__all__ = [
    "RunConfig", "load_config", "CorrespondenceSet", "Observation", "estimate_point_normals",
    "OrbDetector", "StereoMatcher", "EnergyReport",
    "EnergyWeights", "MatchInlierSelector", "SurfaceDeformationTracker", "PinholeCamera",
    "MatchSet", "PreselectConfig", "match_descriptors", "preselect_inliers", "SolverConfig",
    "solve_frame", "FrameResult", "Tracker", "annotate_matches", "prepare_template",
    "track_frame", "track_sequence", "ControlGraph", "Template", "bind_template",
    "sample_control_points", "warp_all",
]
