"""ORB front end on the device: FAST-9 corners with
uniform suppression and oriented 256-bit BRIEF descriptors, the input the Hamming matcher
(a4) and ``Tracker.track(depth, descriptors=..., keypoints=...)`` consume.

The reference ships no ORB code; the algorithm is the one restated in
``oracle/orb.py`` and the device output equals it bit for bit (tests/test_gpu_orb.py).
This module builds the sampling tables with numpy -- the seeded test pattern rotated to
the 30 orientation sectors, and the sector-boundary unit vectors -- and hands them to
the C-ABI (``dt_orb_create`` / ``dt_orb_detect``)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib

N_SECTORS = 30
N_TESTS = 256
PATTERN_SEED = 20070857


def brief_pattern(seed: int = PATTERN_SEED, n: int = N_TESTS, extent: int = 13) -> np.ndarray:
    """(n, 4) int offsets (ax, ay, bx, by) of the binary tests: isotropic Gaussian
    (sigma = 31 / 5, BRIEF's G II sampling), rounded and clipped to +-extent."""
    rng = np.random.default_rng(seed)
    p = np.rint(rng.normal(0.0, 31.0 / 5.0, size=(n, 4)))
    return np.clip(p, -extent, extent).astype(np.int64)


def sector_boundaries() -> np.ndarray:
    """(31, 2) unit vectors at phi_j = -pi + j 2 pi / 30."""
    phi = -np.pi + np.arange(N_SECTORS + 1) * (2.0 * np.pi / N_SECTORS)
    return np.stack([np.cos(phi), np.sin(phi)], axis=1)


def rotated_pattern(pat: np.ndarray) -> np.ndarray:
    """(30, n, 4) int8: the pattern rotated to each sector's centre angle, rounded."""
    out = np.empty((N_SECTORS,) + pat.shape, dtype=np.int64)
    for j in range(N_SECTORS):
        th = -np.pi + (j + 0.5) * (2.0 * np.pi / N_SECTORS)
        c, s = np.cos(th), np.sin(th)
        for k in (0, 2):
            x, y = pat[:, k].astype(np.float64), pat[:, k + 1].astype(np.float64)
            out[j, :, k] = np.rint(c * x - s * y)
            out[j, :, k + 1] = np.rint(s * x + c * y)
    return out.astype(np.int8)


class OrbDetector:
    """Detector for one image size on one device.

    ``detect(image)`` -> (keypoints (n, 2) int32 (u, v), descriptors (n, 32) uint8,
    scores (n,) int32, sectors (n,) int32), best first (FAST score, then pixel index)."""

    def __init__(self, height: int, width: int, threshold: int = 20, cell: int = 32,
                 per_cell: int = 8, n_max: int = 2500, seed: int = PATTERN_SEED,
                 device: int | None = None):
        from .warpfield import _device_index

        self.height, self.width, self.n_max = int(height), int(width), int(n_max)
        rot = np.ascontiguousarray(rotated_pattern(brief_pattern(seed)))
        bnd = np.ascontiguousarray(sector_boundaries())
        h = C.c_void_p()
        dev = _device_index() if device is None else int(device)
        check(lib.dt_orb_create(self.height, self.width, int(threshold), int(cell), int(per_cell),
                                self.n_max, rot.ctypes.data, bnd.ctypes.data, dev, C.byref(h)),
              "dt_orb_create")
        self._h = h

    def detect(self, image):
        img = np.ascontiguousarray(image, dtype=np.uint8)
        if img.shape != (self.height, self.width):
            raise ValueError(f"image must be {self.height}x{self.width}, got {img.shape}")
        kp = np.empty((self.n_max, 2), dtype=np.int32)
        desc = np.empty((self.n_max, 32), dtype=np.uint8)
        sc = np.empty(self.n_max, dtype=np.int32)
        sec = np.empty(self.n_max, dtype=np.int32)
        n = C.c_int64(0)
        check(lib.dt_orb_detect(self._h, img.ctypes.data, 0, kp.ctypes.data, desc.ctypes.data,
                                sc.ctypes.data, sec.ctypes.data, C.byref(n)), "dt_orb_detect")
        k = n.value
        return kp[:k].copy(), desc[:k].copy(), sc[:k].copy(), sec[:k].copy()

    def last_on_device(self):
        """(keypoints device pointer, descriptors device pointer, n) of the last detect:
        the frame inputs for ``DeviceTracker.track_raw`` with ``on_device = 1``."""
        kp, de = C.c_void_p(), C.c_void_p()
        n = C.c_int64(0)
        check(lib.dt_orb_last(self._h, C.byref(kp), C.byref(de), C.byref(n)), "dt_orb_last")
        return kp.value, de.value, n.value

    def close(self) -> None:
        if self._h:
            lib.dt_orb_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["OrbDetector", "brief_pattern", "sector_boundaries", "rotated_pattern"]
