"""Depth observations and projective correspondences.

Mirrors deformtrack/correspond.py: ``valid_depth_mask`` (23-26),
``compute_observation_normals`` (36-73), ``Observation`` (76-107, with ``from_depth``),
``CorrespondenceSet`` (110-121), ``rasterize_correspondences`` (124-175),
``occlusion_mask`` (178-195), ``estimate_point_normals`` (198-220).

``Observation.from_depth`` does not compute normals on the host: the per-frame normal
stencil runs on the device (dt_observation_normals), fused into the tracker's frame
pipeline; reading ``Observation.normals`` materializes them from the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as dev
from ._lib import check, lib
from .geometry import PinholeCamera

DEFAULT_Z_MIN = 1.0
DEFAULT_Z_MAX = 1.0e5


def valid_depth_mask(depth, z_min: float, z_max: float) -> np.ndarray:
    """Finite depth strictly inside (z_min, z_max) (correspond.py:23-26)."""
    d = np.asarray(depth)
    return np.isfinite(d) & (d > z_min) & (d < z_max)


def compute_observation_normals(depth, camera: PinholeCamera, z_min: float = DEFAULT_Z_MIN,
                                z_max: float = DEFAULT_Z_MAX) -> np.ndarray:
    """Central-difference normals of the back-projected depth, oriented toward the camera,
    zero where the 5-point stencil is not fully valid (correspond.py:36-73); device."""
    d = np.ascontiguousarray(depth, dtype=np.float64)
    h, w = d.shape
    D = dev.to_device(d)
    N = dev.empty((h, w, 3))
    V = dev.empty((h, w), np.uint8)
    check(lib.dt_observation_normals(dev.ptr(D), h, w, camera.fx, camera.fy, camera.cx,
                                     camera.cy, z_min, z_max, dev.ptr(N), dev.ptr(V),
                                     dev.stream()), "compute_observation_normals")
    return dev.to_host(N)


class Observation:
    """One depth frame, its camera and (lazily, on the device) its normals."""

    def __init__(self, depth, normals, camera: PinholeCamera, frame_id: int = 0,
                 z_min: float = DEFAULT_Z_MIN, z_max: float = DEFAULT_Z_MAX):
        self.depth = np.asarray(depth, dtype=np.float64)
        self._normals = None if normals is None else np.asarray(normals, dtype=np.float64)
        self.camera = camera
        self.frame_id = frame_id
        self.z_min = z_min
        self.z_max = z_max

    @classmethod
    def from_depth(cls, depth, camera: PinholeCamera, frame_id: int = 0,
                   z_min: float = DEFAULT_Z_MIN, z_max: float = DEFAULT_Z_MAX) -> "Observation":
        depth = np.asarray(depth, dtype=np.float64)
        if depth.shape != (camera.height, camera.width):
            raise ValueError(
                f"depth shape {depth.shape} does not match camera ({camera.height}, {camera.width})"
            )
        # normals stay on the device path until someone asks for them
        return cls(depth, None, camera, frame_id, z_min, z_max)

    @property
    def normals_on_device(self) -> bool:
        """True when the solver should derive the normals from the depth on the device."""
        return self._normals is None

    @property
    def normals(self) -> np.ndarray:
        if self._normals is None:
            self._normals = compute_observation_normals(self.depth, self.camera, self.z_min,
                                                        self.z_max)
        return self._normals

    @normals.setter
    def normals(self, value) -> None:
        self._normals = None if value is None else np.asarray(value, dtype=np.float64)

    @property
    def valid(self) -> np.ndarray:
        return valid_depth_mask(self.depth, self.z_min, self.z_max)


@dataclass
class CorrespondenceSet:
    """Per-template-point projective association (correspond.py:110-121)."""

    valid: np.ndarray
    points: np.ndarray
    normals: np.ndarray
    pixels: np.ndarray

    @property
    def count(self) -> int:
        return int(np.count_nonzero(self.valid))


def rasterize_correspondences(points, normals, observation: Observation,
                              gate_distance: float = 20.0,
                              gate_angle_deg: float = 60.0) -> CorrespondenceSet:
    """Project already-warped points into the depth image and gate the pairs
    (correspond.py:124-175). Runs the device association kernel with an identity warp."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    nrm = np.asarray(normals, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    ident = np.zeros((1, 8))
    ident[0, 0] = 1.0
    from .kernels import warp_and_rasterize

    cam = observation.camera
    _, _, valid, obs_p, obs_n, pixels = warp_and_rasterize(
        pts, nrm, np.zeros((n, 1), dtype=np.int64), np.ones((n, 1)), ident,
        observation.depth, observation.valid, observation.normals,
        cam.fx, cam.fy, cam.cx, cam.cy, gate_distance,
        float(np.cos(np.deg2rad(gate_angle_deg))), 8,
    )
    return CorrespondenceSet(valid, obs_p, obs_n, pixels)


def occlusion_mask(observation: Observation, region: tuple[int, int, int, int]) -> Observation:
    """Zero the depth inside the half-open pixel rectangle (u0, v0, u1, v1) and return a
    new observation (correspond.py:178-195)."""
    u0, v0, u1, v1 = region
    depth = np.array(observation.depth, dtype=np.float64, copy=True)
    depth[v0:v1, u0:u1] = 0.0
    return Observation.from_depth(depth, observation.camera, frame_id=observation.frame_id,
                                  z_min=observation.z_min, z_max=observation.z_max)


def estimate_point_normals(points, k: int = 12) -> np.ndarray:
    """Local-PCA normals oriented toward the camera at the origin (correspond.py:198-220).

    Template-time setup (``fit()`` without normals), on the device
    (``dt_estimate_point_normals``): exact k nearest neighbours by brute force (ties at
    the k-th neighbour to the lower index; the reference's kd-tree leaves that order
    unspecified), scatter in nearest-first order, Jacobi eigenvector of the smallest
    eigenvalue."""
    import ctypes as C

    from .warpfield import _device_index

    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = np.empty_like(pts)
    if pts.shape[0] == 0:
        return out
    check(lib.dt_estimate_point_normals(pts.ctypes.data, pts.shape[0], int(k),
                                        out.ctypes.data, _device_index()),
          "dt_estimate_point_normals")
    return out


__all__ = [
    "DEFAULT_Z_MIN",
    "DEFAULT_Z_MAX",
    "valid_depth_mask",
    "compute_observation_normals",
    "Observation",
    "CorrespondenceSet",
    "rasterize_correspondences",
    "occlusion_mask",
    "estimate_point_normals",
]
