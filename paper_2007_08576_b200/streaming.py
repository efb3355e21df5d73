"""Pipelined frame streaming through the C-ABI's dt_track_frame_submit / dt_tracker_wait
(include/deformtrack_b200.h): the same frames, in the same order, with the same results
as ``tracking.Tracker.track`` (tracking.py:67-95), but frame i+1's inputs are staged on a
copy stream while frame i computes and frame i's outputs are copied back while frame i+1
computes. Up to two frames are in flight; ``submit`` returns immediately, ``wait``
returns the oldest frame's ``FrameResult``.

Inputs per frame: the depth as an (h, w) f64 array or as a PFM payload (``fileio.
read_pfm_payload``: f32 rows bottom-up, decoded on the device), plus an optional
``MatchSet`` of pairs (preselected and bound on the device, tracking.annotate_matches).
"""

from __future__ import annotations

import ctypes as C
from collections import deque
from dataclasses import dataclass

import numpy as np

from ._lib import (DT_DEPTH_F64, DT_DEPTH_PFM, DT_ERR_NO_VALID_HYPOTHESIS, FrameInput, FrameOutput,
                   Report)
from ._session import DeviceTracker, make_config, nvh_message
from .matching import MatchSet, reference_indices
from .solver import report_from_outputs
from .tracking import FrameResult


@dataclass
class _Slot:
    warps: np.ndarray
    points: np.ndarray
    normals: np.ndarray
    cdw: np.ndarray
    mw: np.ndarray
    mf: np.ndarray
    ch: np.ndarray
    lh: np.ndarray
    st: np.ndarray
    report: Report
    fo: FrameOutput


class _Outs:
    """FrameOutputs-shaped view of one finished slot (what report_from_outputs reads)."""

    def __init__(self, s: _Slot):
        r = s.report
        self.report = r
        self.warps = s.warps.copy()
        self.points = s.points.copy()
        self.normals = s.normals.copy()
        self.control_data_weights = s.cdw.copy()
        nh, no = int(r.n_cost_history), int(r.outer_iterations)
        self.cost_history = [[float(a), float(b)] for a, b in s.ch[:nh]]
        self.lambda_history = [[float(a), float(b)] for a, b in s.lh[:no]]
        self.stalled = s.st[:no].copy()


def _pinned(owners: list, shape, dtype=np.float64) -> np.ndarray:
    """Page-locked host array (torch's pinned allocator; torch is plumbing here); the
    owning tensor is kept in `owners` for as long as the array is in use."""
    import torch

    n = int(np.prod(shape)) if shape else 1
    t = torch.empty(max(n, 1) * np.dtype(dtype).itemsize, dtype=torch.uint8).pin_memory()
    owners.append(t)
    return t.numpy().view(dtype)[:n].reshape(shape)


class StreamingTracker:
    """Device-resident tracker of one sequence, fed through the pipelined C-ABI."""

    def __init__(self, template, graph, camera, config, max_matches: int = 4096):
        self.template = template
        self.graph = graph
        self.camera = camera
        self.config = config
        self._pcfg = config.make_preselect_config()
        cfg = make_config(camera, config.energy, config.make_solver_config(), self._pcfg,
                          sampling_radius=graph.sampling_radius, z_min=config.depth.z_min,
                          z_max=config.depth.z_max)
        self.device = DeviceTracker(template, graph, cfg)
        self.m, self.n = len(graph), len(template)
        self._it = int(cfg.max_outer_iters)
        self._cap = int(max_matches)
        self._owners: list = []
        self._slots = [self._make_slot() for _ in range(2)]
        self._pending: deque = deque()
        self._next_slot = 0
        self.frame_index = 0

    def _make_slot(self) -> _Slot:
        o = self._owners
        s = _Slot(_pinned(o, (self.m, 8)), _pinned(o, (self.n, 3)), _pinned(o, (self.n, 3)),
                  _pinned(o, (self.m,)), _pinned(o, (self._cap,)), _pinned(o, (self._cap,), np.uint8),
                  np.zeros((self._it, 2)), np.zeros((self._it, 2)), np.zeros(self._it, np.int32),
                  Report(), FrameOutput())
        fo = s.fo
        fo.warps, fo.points, fo.normals = s.warps.ctypes.data, s.points.ctypes.data, s.normals.ctypes.data
        fo.control_data_weights = s.cdw.ctypes.data
        fo.match_weights, fo.match_flags = s.mw.ctypes.data, s.mf.ctypes.data
        fo.match_capacity = self._cap
        fo.report = C.cast(C.pointer(s.report), C.c_void_p).value
        fo.cost_history, fo.lambda_history = s.ch.ctypes.data, s.lh.ctypes.data
        fo.stalled = s.st.ctypes.data
        return s

    def reset(self, warps=None) -> None:
        """Warm start of the next submitted frame (drains the frames in flight first)."""
        self.device.set_warps(self.graph.warps if warps is None else warps)

    def submit(self, depth=None, matches: MatchSet | None = None, *, pfm_payload=None,
               frame_id: int | None = None) -> None:
        """Queue one frame. Exactly one of `depth` ((h, w) f64) or `pfm_payload`
        ((h, w) f32 rows bottom-up, little-endian) is given."""
        if len(self._pending) >= 2:
            raise RuntimeError("two frames in flight: wait() for the oldest first")
        fid = self.frame_index if frame_id is None else int(frame_id)
        self.frame_index += 1
        h, w = int(self.camera.height), int(self.camera.width)
        keep = []
        fi = FrameInput()
        fi.height, fi.width = h, w
        if pfm_payload is not None:
            p = np.ascontiguousarray(pfm_payload, dtype="<f4")
            if p.shape != (h, w):
                raise ValueError(f"depth payload {p.shape} does not match the camera ({h}, {w})")
            fi.depth_kind = DT_DEPTH_PFM
            fi.depth = p.ctypes.data
            keep.append(p)
        else:
            d = np.ascontiguousarray(depth, dtype=np.float64)
            if d.shape != (h, w):
                raise ValueError(f"depth shape {d.shape} does not match the camera ({h}, {w})")
            fi.depth_kind = DT_DEPTH_F64
            fi.depth = d.ctypes.data
            keep.append(d)
        n = 0
        if matches is not None and len(matches) > 0:
            n = len(matches)
            if n > self._cap:
                raise ValueError(f"{n} matches exceed the streaming capacity {self._cap}")
            src = np.ascontiguousarray(matches.template_points, dtype=np.float64)
            dst = np.ascontiguousarray(matches.observed_points, dtype=np.float64)
            keep += [src, dst]
            fi.match_src, fi.match_dst, fi.n_pairs = src.ctypes.data, dst.ctypes.data, n
            refs = reference_indices(n, self._pcfg)
            if refs is not None:
                r = np.ascontiguousarray(refs, dtype=np.int64)
                keep.append(r)
                fi.refs, fi.n_refs = r.ctypes.data, r.shape[0]
        fi.use_matches = 1 if n else 0
        fi.on_device = 0
        fi.frame_id = fid
        slot = self._slots[self._next_slot]
        self.device.submit(fi, slot.fo)
        self._pending.append((slot, fid, matches, keep))
        self._next_slot ^= 1

    def wait(self) -> FrameResult:
        """The oldest frame in flight, once its outputs are on the host."""
        if not self._pending:
            raise RuntimeError("no frame in flight")
        self.device.wait()
        slot, fid, matches, _keep = self._pending.popleft()
        out = _Outs(slot)
        r = slot.report
        annotated = None
        warning = None
        n = 0 if matches is None else len(matches)
        if n:
            annotated = MatchSet(matches.template_points, matches.observed_points,
                                 slot.mw[:n].copy(), slot.mf[:n].astype(bool))
            if int(r.preselect_status) == DT_ERR_NO_VALID_HYPOTHESIS:
                annotated = MatchSet(matches.template_points, matches.observed_points,
                                     np.zeros(n), np.zeros(n, dtype=bool))
                warning = f"match preselection failed ({nvh_message(n)}); feature term dropped"
        report = report_from_outputs(out, fid, annotated)
        if warning:
            report.warnings.append(warning)
        graph = self.graph.with_warps(out.warps)
        return FrameResult(fid, graph, out.points, out.normals, annotated, report)

    @property
    def in_flight(self) -> int:
        return len(self._pending)

    def close(self) -> None:
        self.device.close()
        self._slots = []
        self._owners = []


__all__ = ["StreamingTracker"]
