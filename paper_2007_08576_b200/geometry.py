"""Camera model and the small host-side quaternion helpers used to build inputs.

Mirrors the public names of deformtrack/geometry.py that callers of the tracker touch
when preparing data: ``PinholeCamera`` (355-370), ``project`` (373-384),
``back_project`` (387-396), ``dq_identity`` (143-146), ``quat_from_axis_angle``
(78-85), ``quat_to_matrix`` (98-107), ``quat_from_matrix`` (110-135),
``dq_from_transform`` (187-192), ``dq_to_transform_batch`` (238-264, device).
Conventions: scalar-first quaternions, dual quaternions as 8-vectors
(real, dual), translations in mm.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import BehindCamera


@dataclass(frozen=True)
class PinholeCamera:
    """Undistorted pinhole intrinsics in pixels (geometry.py:355-370)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self) -> None:
        if self.fx <= 0.0 or self.fy <= 0.0:
            raise ValueError("focal lengths must be positive")
        if self.width <= 0 or self.height <= 0:
            raise ValueError("image size must be positive")


def project(camera: PinholeCamera, points) -> np.ndarray:
    """Pixel coordinates (..., 2) of camera-frame points; BehindCamera for z <= 0."""
    p = np.asarray(points, dtype=np.float64)
    z = p[..., 2]
    if np.any(z <= 0.0):
        raise BehindCamera("point with z <= 0 cannot be projected")
    return np.stack([camera.fx * p[..., 0] / z + camera.cx,
                     camera.fy * p[..., 1] / z + camera.cy], axis=-1)


def back_project(camera: PinholeCamera, u, v, depth) -> np.ndarray:
    """Pixel (u, v) plus depth z to camera-frame points (..., 3): x = (u - cx) / fx * z."""
    z = np.asarray(depth, dtype=np.float64)
    x = (np.asarray(u, dtype=np.float64) - camera.cx) / camera.fx * z
    y = (np.asarray(v, dtype=np.float64) - camera.cy) / camera.fy * z
    return np.stack([np.broadcast_to(x, z.shape), np.broadcast_to(y, z.shape), z], axis=-1)


def quat_mul(a, b) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    aw, ax, ay, az = (a[..., i] for i in range(4))
    bw, bx, by, bz = (b[..., i] for i in range(4))
    return np.stack([
        aw * bw - ax * bx - ay * by - az * bz,
        aw * bx + ax * bw + ay * bz - az * by,
        aw * by - ax * bz + ay * bw + az * bx,
        aw * bz + ax * by - ay * bx + az * bw,
    ], axis=-1)


def quat_from_axis_angle(omega) -> np.ndarray:
    """Rotation vector (rad) to unit quaternion."""
    omega = np.asarray(omega, dtype=np.float64)
    angle = np.linalg.norm(omega, axis=-1, keepdims=True)
    half_sinc = 0.5 * np.sinc(angle / (2.0 * np.pi))
    return np.concatenate([np.cos(0.5 * angle), omega * half_sinc], axis=-1)


def quat_to_matrix(q) -> np.ndarray:
    w, x, y, z = np.asarray(q, dtype=np.float64)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def quat_from_matrix(R) -> np.ndarray:
    """Rotation matrix to the canonical unit quaternion (w >= 0), Shepperd's branches."""
    R = np.asarray(R, dtype=np.float64)
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    if tr > 0.0:
        s = 2.0 * np.sqrt(tr + 1.0)
        q = np.array([0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s,
                      (R[1, 0] - R[0, 1]) / s])
    elif R[0, 0] >= R[1, 1] and R[0, 0] >= R[2, 2]:
        s = 2.0 * np.sqrt(1.0 + R[0, 0] - R[1, 1] - R[2, 2])
        q = np.array([(R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s,
                      (R[0, 2] + R[2, 0]) / s])
    elif R[1, 1] >= R[2, 2]:
        s = 2.0 * np.sqrt(1.0 + R[1, 1] - R[0, 0] - R[2, 2])
        q = np.array([(R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s,
                      (R[1, 2] + R[2, 1]) / s])
    else:
        s = 2.0 * np.sqrt(1.0 + R[2, 2] - R[0, 0] - R[1, 1])
        q = np.array([(R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s,
                      (R[1, 2] + R[2, 1]) / s, 0.25 * s])
    q = q / np.linalg.norm(q)
    return -q if q[0] < 0.0 else q


def dq_identity() -> np.ndarray:
    out = np.zeros(8)
    out[0] = 1.0
    return out


def dq_from_transform(R, t) -> np.ndarray:
    """Rigid transform (R, t) to a unit dual quaternion: real = q, dual = 0.5 (0, t) q."""
    real = quat_from_matrix(R)
    pure_t = np.concatenate([[0.0], np.asarray(t, dtype=np.float64)])
    return np.concatenate([real, 0.5 * quat_mul(pure_t, real)])


def dq_to_transform_batch(dqs) -> tuple[np.ndarray, np.ndarray]:
    """(..., 8) dual quaternions to rotations (..., 3, 3) and translations (..., 3),
    evaluated on the device (dt_dq_to_transform)."""
    from . import _device as dev
    from ._lib import check, lib

    arr = np.asarray(dqs, dtype=np.float64)
    lead = arr.shape[:-1]
    flat = dev.to_device(arr.reshape(-1, 8))
    m = flat.shape[0]
    R = dev.empty((m, 3, 3))
    t = dev.empty((m, 3))
    check(lib.dt_dq_to_transform(dev.ptr(flat), m, dev.ptr(R), dev.ptr(t), dev.stream()),
          "dq_to_transform_batch")
    return dev.to_host(R).reshape(lead + (3, 3)), dev.to_host(t).reshape(lead + (3,))


__all__ = [
    "PinholeCamera",
    "project",
    "back_project",
    "quat_mul",
    "quat_from_axis_angle",
    "quat_to_matrix",
    "quat_from_matrix",
    "dq_identity",
    "dq_from_transform",
    "dq_to_transform_batch",
]
