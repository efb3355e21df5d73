"""Stereo depth on the device: the stage upstream of the
observation that turns a rectified stereo pair into the depth map ``Tracker.track``
consumes. The reference ships no stereo matcher (depth arrives as a map); the
algorithm -- ZNCC window matching, winner-take-all both ways with a left-right check,
parabolic sub-pixel refinement, depth = fx B / disparity -- is the one restated in
``oracle/stereo.py``, and the device output equals it bit for bit
(tests/test_gpu_stereo.py)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib


class StereoMatcher:
    """Matcher for one image size on one device.

    ``compute(left, right)`` -> (depth (h, w) f64 mm, NaN where no match survives,
    disparity (h, w) f64 px, winner (h, w) int32 integer disparity or -1). ``device_depth``
    is the device-resident depth of the last call, for ``Tracker``'s device inputs."""

    def __init__(self, height: int, width: int, fx: float, baseline: float, max_disp: int = 64,
                 radius: int = 3, min_ncc: float = 0.5, lr_tol: int = 1,
                 device: int | None = None):
        from .warpfield import _device_index

        self.height, self.width = int(height), int(width)
        self._h = C.c_void_p()
        check(lib.dt_stereo_create(self.height, self.width, int(max_disp), int(radius), float(fx),
                                   float(baseline), float(min_ncc), int(lr_tol),
                                   _device_index() if device is None else int(device),
                                   C.byref(self._h)), "dt_stereo_create")

    def compute(self, left, right, on_device: bool = False):
        """left / right: (h, w) uint8 host arrays, or (on_device) CUDA tensors -- the
        matcher runs on its own stream, so the producer's stream is synchronized first."""
        h, w = self.height, self.width
        keep = []
        if on_device:
            import torch

            torch.cuda.current_stream().synchronize()

        def img(a):
            if on_device:
                import torch

                if a.dtype != torch.uint8 or tuple(a.shape) != (h, w) or not a.is_cuda:
                    raise ValueError(f"device image must be a ({h}, {w}) uint8 CUDA tensor")
                a = a.contiguous()
                keep.append(a)
                return a.data_ptr()
            arr = np.ascontiguousarray(a, dtype=np.uint8)
            if arr.shape != (h, w):
                raise ValueError(f"image {arr.shape} does not match the matcher ({h}, {w})")
            keep.append(arr)
            return arr.ctypes.data

        depth = np.empty((h, w))
        disp = np.empty((h, w))
        win = np.empty((h, w), dtype=np.int32)
        check(lib.dt_stereo_compute(self._h, img(left), img(right), 1 if on_device else 0,
                                    depth.ctypes.data, disp.ctypes.data, win.ctypes.data),
              "dt_stereo_compute")
        return depth, disp, win

    def device_depth(self) -> int:
        """Device pointer of the last depth map ((h, w) f64, valid until the next call)."""
        p = C.c_void_p()
        check(lib.dt_stereo_last(self._h, C.byref(p)), "dt_stereo_last")
        return int(p.value)

    def close(self) -> None:
        if self._h:
            lib.dt_stereo_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["StereoMatcher"]
