"""Python handle around one ``dt_tracker`` (include/deformtrack_b200.h).

A ``DeviceTracker`` owns the device-resident template, control graph, CSR lists and
solver state of one sequence. Frames go in as host arrays (or device pointers); the
C-ABI does the host<->device copies, the per-frame kernels and the single
thread-block-cluster LM launch, then returns the solution and the report.
"""

from __future__ import annotations

import ctypes as C
import hashlib
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from ._lib import Config, FrameInput, FrameOutput, PreselectParams, Report, check, lib


def make_config(camera, weights, solver, preselect=None, *, sampling_radius: float,
                z_min: float = 1.0, z_max: float = 1.0e5, cluster_size: int = 0,
                max_hamming: int = 256) -> Config:
    """Pack EnergyWeights + SolverConfig + PreselectConfig + camera into dt_config."""
    pp = PreselectParams(5.0, 10, 0.5, 0.2)
    if preselect is not None:
        pp = preselect.params()
    cos_gate = float(np.cos(np.deg2rad(solver.gate_angle_deg)))
    return Config(
        feature_weight=float(weights.feature_weight), arap_weight=float(weights.arap_weight),
        angle_weight=float(weights.angle_weight), rotation_weight=float(weights.rotation_weight),
        tukey_scale=float(weights.tukey_scale), data_floor=float(weights.data_floor),
        max_outer_iters=int(solver.max_outer_iters),
        lambda_init=float(solver.lambda_init), lambda_decrease=float(solver.lambda_decrease),
        lambda_increase=float(solver.lambda_increase), lambda_min=float(solver.lambda_min),
        lambda_max=float(solver.lambda_max), max_retries=int(solver.max_retries),
        step_tol=float(solver.step_tol), cost_tol=float(solver.cost_tol),
        gate_distance=float(solver.gate_distance), cos_gate=cos_gate,
        preselect=pp,
        fx=float(camera.fx), fy=float(camera.fy), cx=float(camera.cx), cy=float(camera.cy),
        width=int(camera.width), height=int(camera.height),
        z_min=float(z_min), z_max=float(z_max),
        sampling_radius=float(sampling_radius), cluster_size=int(cluster_size),
        max_hamming=int(max_hamming),
    )


def _cfg_bytes(cfg: Config) -> bytes:
    return bytes(memoryview(cfg))


def _host_ptr(a) -> int | None:
    """Raw pointer of a C-contiguous numpy array or a (pinned) host torch tensor."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr() if a.numel() else None
    return a.ctypes.data if a.size else None


@dataclass
class FrameOutputs:
    warps: np.ndarray
    points: np.ndarray | None
    normals: np.ndarray | None
    control_data_weights: np.ndarray
    report: Report
    cost_history: list
    lambda_history: list
    stalled: np.ndarray
    match_weights: np.ndarray | None = None
    match_flags: np.ndarray | None = None
    match_src: np.ndarray | None = None
    match_dst: np.ndarray | None = None


def _want(a, shape, name) -> None:
    """Shape check before a pointer crosses the C-ABI (which trusts the sizes)."""
    got = tuple(int(x) for x in (a.shape if hasattr(a, "shape") else np.shape(a)))
    if got != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {got}")


class DeviceTracker:
    """One sequence resident on one device (one stream)."""

    def __init__(self, template, graph, cfg: Config, device: int | None = None,
                 stream: int | None = None):
        # the C-ABI trusts the sizes it is given: reject inconsistent arrays here
        n, m = len(template.points), len(graph.points)
        _want(template.normals, (n, 3), "template normals")
        if template.bind_indices is None or template.bind_weights is None:
            raise ValueError("template must be bound to the control graph first")
        k = int(np.shape(template.bind_indices)[1]) if np.ndim(template.bind_indices) == 2 else -1
        _want(template.bind_indices, (n, k), "template bind_indices")
        _want(template.bind_weights, (n, k), "template bind_weights")
        _want(graph.warps, (m, 8), "graph warps")
        ne = int(np.size(graph.edges)) // 2
        _want(graph.edges, (ne, 2), "graph edges")
        _want(graph.edge_weights, (ne,), "graph edge_weights")
        dev.require_cuda()
        import torch

        self.device = torch.cuda.current_device() if device is None else int(device)
        self.n = len(template)
        self.k = int(template.bind_indices.shape[1])
        self.m = len(graph)
        self._cfg = cfg
        self._cfg_key = _cfg_bytes(cfg)
        self.n_features = 0
        tp = np.ascontiguousarray(template.points, dtype=np.float64)
        tn = np.ascontiguousarray(template.normals, dtype=np.float64)
        bi = np.ascontiguousarray(template.bind_indices, dtype=np.int64)
        bw = np.ascontiguousarray(template.bind_weights, dtype=np.float64)
        cp = np.ascontiguousarray(graph.points, dtype=np.float64)
        wp = np.ascontiguousarray(graph.warps, dtype=np.float64)
        ed = np.ascontiguousarray(graph.edges, dtype=np.int64).reshape(-1, 2)
        ew = np.ascontiguousarray(graph.edge_weights, dtype=np.float64)
        handle = C.c_void_p()
        check(lib.dt_tracker_create(C.byref(cfg), _host_ptr(tp), _host_ptr(tn), _host_ptr(bi),
                                    _host_ptr(bw), self.n, self.k, _host_ptr(cp), _host_ptr(wp),
                                    self.m, _host_ptr(ed), _host_ptr(ew), ed.shape[0],
                                    self.device, stream, C.byref(handle)), "dt_tracker_create")
        self._h = handle

    # -- configuration -------------------------------------------------------------
    def set_config(self, cfg: Config) -> None:
        key = _cfg_bytes(cfg)
        if key == self._cfg_key:
            return
        check(lib.dt_tracker_set_config(self._h, C.byref(cfg)), "dt_tracker_set_config")
        self._cfg = cfg
        self._cfg_key = key

    @property
    def config(self) -> Config:
        return self._cfg

    def set_warps(self, warps) -> None:
        w = np.ascontiguousarray(warps, dtype=np.float64).reshape(self.m, 8)
        check(lib.dt_tracker_set_warps(self._h, _host_ptr(w), 0), "dt_tracker_set_warps")

    def get_warps(self) -> np.ndarray:
        out = np.empty((self.m, 8))
        check(lib.dt_tracker_get_warps(self._h, _host_ptr(out)), "dt_tracker_get_warps")
        return out

    def set_features(self, desc, points, binding=None) -> None:
        d = np.ascontiguousarray(desc, dtype=np.uint8).reshape(-1, 32)
        p = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        if d.shape[0] != p.shape[0]:
            raise ValueError("one 3D point per template descriptor required")
        bi = bw = None
        if binding is not None:
            bi = np.ascontiguousarray(binding[0], dtype=np.int64).reshape(d.shape[0], self.k)
            bw = np.ascontiguousarray(binding[1], dtype=np.float64).reshape(d.shape[0], self.k)
        check(lib.dt_tracker_set_features(self._h, _host_ptr(d), _host_ptr(p), d.shape[0],
                                          _host_ptr(bi), _host_ptr(bw)),
              "dt_tracker_set_features")
        self.n_features = d.shape[0]

    # -- frames --------------------------------------------------------------------
    def track(self, depth, normals=None, *, pairs=None, match_w=None, match_binding=None,
              frame_desc=None, frame_kp=None, refs=None, frame_id: int = 0,
              want_points: bool = True,
              want_matches: bool = False, outputs: dict | None = None) -> FrameOutputs:
        """Run one frame. Host inputs; returns host outputs (after the stream sync)."""
        io = self.prepare(depth, normals, pairs=pairs, match_w=match_w,
                          match_binding=match_binding, frame_desc=frame_desc, frame_kp=frame_kp,
                          refs=refs, frame_id=frame_id, want_points=want_points,
                          want_matches=want_matches, outputs=outputs)
        check(lib.dt_track_frame(self._h, C.byref(io["fi"]), C.byref(io["fo"])), "dt_track_frame")
        return self.finish(io)

    def prepare(self, depth, normals=None, *, pairs=None, match_w=None, match_binding=None,
                frame_desc=None, frame_kp=None, refs=None, frame_id: int = 0,
                want_points: bool = True, want_matches: bool = False,
                outputs: dict | None = None) -> dict:
        """The dt_frame_input / dt_frame_output of one frame (host buffers) plus the arrays
        they point into; `finish` turns the filled outputs into FrameOutputs."""
        keep = []

        def hp(a, dtype):
            if a is None:
                return None
            if hasattr(a, "data_ptr"):
                # a torch tensor: used in place only when it already is contiguous host
                # memory of the right dtype (this entry copies from HOST pointers);
                # anything else goes through numpy (device tensors are copied back)
                import torch

                want = {np.float64: torch.float64, np.uint8: torch.uint8,
                        np.int32: torch.int32, np.int64: torch.int64}[dtype]
                if a.device.type == "cpu" and a.dtype == want and a.is_contiguous():
                    keep.append(a)
                    return _host_ptr(a)
                a = a.detach().cpu().numpy()
            arr = np.ascontiguousarray(a, dtype=dtype)
            keep.append(arr)
            return _host_ptr(arr)

        h, w = int(self._cfg.height), int(self._cfg.width)
        _want(depth, (h, w), "depth")
        if normals is not None:
            _want(normals, (h, w, 3), "observation normals")
        fi = FrameInput()
        fi.height, fi.width = h, w
        fi.depth = hp(depth, np.float64)
        fi.normals = hp(normals, np.float64)
        n_pairs = 0
        if pairs is not None:
            src, dst = pairs
            n_pairs = int(np.asarray(src).shape[0]) if not hasattr(src, "shape") else int(src.shape[0])
            _want(src, (n_pairs, 3), "match template points")
            _want(dst, (n_pairs, 3), "match observed points")
            if match_w is not None:
                _want(match_w, (n_pairs,), "match weights")
            if match_binding is not None:
                _want(match_binding[0], (n_pairs, self.k), "match binding indices")
                _want(match_binding[1], (n_pairs, self.k), "match binding weights")
            fi.match_src = hp(src, np.float64)
            fi.match_dst = hp(dst, np.float64)
            fi.match_w = hp(match_w, np.float64)
            if match_binding is not None:
                fi.match_bidx = hp(match_binding[0], np.int64)
                fi.match_bw = hp(match_binding[1], np.float64)
        fi.n_pairs = n_pairs
        n_frame = 0
        if frame_desc is not None:
            n_frame = int(frame_desc.shape[0])
            _want(frame_desc, (n_frame, 32), "frame descriptors")
            _want(frame_kp, (n_frame, 2), "frame keypoints")
            fi.frame_desc = hp(frame_desc, np.uint8)
            fi.frame_kp = hp(frame_kp, np.int32)
        fi.n_frame = n_frame
        if refs is not None:
            r = np.ascontiguousarray(refs, dtype=np.int64)
            if r.ndim != 1:
                raise ValueError("refs must be a 1-D index array")
            keep.append(r)
            fi.refs = _host_ptr(r)
            fi.n_refs = r.shape[0]
        fi.use_matches = 1 if (n_pairs > 0 or n_frame > 0) else 0
        fi.on_device = 0
        fi.frame_id = int(frame_id)

        o = outputs or {}
        warps = o.get("warps")
        if warps is None:
            warps = np.empty((self.m, 8))
        pts = nrm = None
        if want_points:
            pts = o.get("points")
            nrm = o.get("normals")
            if pts is None:
                pts = np.empty((self.n, 3))
            if nrm is None:
                nrm = np.empty((self.n, 3))
        cdw = np.empty(self.m)
        report = Report()
        cap = max(n_pairs, self.n_features) if (want_matches or n_pairs) else 0
        mw = np.empty(cap) if cap else None
        mf = np.empty(cap, dtype=np.uint8) if cap else None
        ms = np.empty((cap, 3)) if (cap and n_frame) else None
        md = np.empty((cap, 3)) if (cap and n_frame) else None
        fo = FrameOutput()
        fo.warps = _host_ptr(warps)
        fo.points = _host_ptr(pts)
        fo.normals = _host_ptr(nrm)
        fo.match_weights = _host_ptr(mw)
        fo.match_flags = _host_ptr(mf)
        fo.match_src = _host_ptr(ms)
        fo.match_dst = _host_ptr(md)
        fo.match_capacity = cap
        fo.control_data_weights = _host_ptr(cdw)
        fo.report = C.cast(C.pointer(report), C.c_void_p).value
        return dict(fi=fi, fo=fo, keep=keep, warps=warps, pts=pts, nrm=nrm, cdw=cdw,
                    report=report, mw=mw, mf=mf, ms=ms, md=md)

    def finish(self, io: dict) -> FrameOutputs:
        warps, pts, nrm, cdw, report = io["warps"], io["pts"], io["nrm"], io["cdw"], io["report"]
        mw, mf, ms, md = io["mw"], io["mf"], io["ms"], io["md"]
        it = int(self._cfg.max_outer_iters)
        ch = np.zeros((it, 2))
        lh = np.zeros((it, 2))
        st = np.zeros(it, dtype=np.int32)
        check(lib.dt_tracker_get_history(self._h, _host_ptr(ch), _host_ptr(lh), _host_ptr(st)),
              "dt_tracker_get_history")
        nh = int(report.n_cost_history)
        no = int(report.outer_iterations)
        return FrameOutputs(
            warps=warps, points=pts, normals=nrm, control_data_weights=cdw, report=report,
            cost_history=[[float(a), float(b)] for a, b in ch[:nh]],
            lambda_history=[[float(a), float(b)] for a, b in lh[:no]],
            stalled=st[:no].copy(), match_weights=mw, match_flags=mf, match_src=ms,
            match_dst=md,
        )

    def track_raw(self, fi: FrameInput, fo: FrameOutput) -> None:
        """Lowest-overhead entry: caller-built dt_frame_input / dt_frame_output."""
        check(lib.dt_track_frame(self._h, C.byref(fi), C.byref(fo)), "dt_track_frame")

    def submit(self, fi: FrameInput, fo: FrameOutput) -> None:
        """Pipelined streaming: stage host inputs on the copy stream, run the frame, copy
        the outputs back into `fo` (filled once `wait` returns for this frame)."""
        check(lib.dt_track_frame_submit(self._h, C.byref(fi), C.byref(fo)), "dt_track_frame_submit")

    def sync(self) -> None:
        """Drain the pipeline and the tracker stream."""
        check(lib.dt_tracker_sync(self._h), "dt_tracker_sync")

    def wait(self) -> None:
        """Wait for the oldest frame in flight (fills its report)."""
        check(lib.dt_tracker_wait(self._h), "dt_tracker_wait")

    def enqueue(self, fi: FrameInput) -> None:
        """Enqueue one frame on the tracker stream; no host outputs, no synchronization."""
        check(lib.dt_track_frame_async(self._h, C.byref(fi)), "dt_track_frame_async")

    def collect(self, fi: FrameInput, fo: FrameOutput) -> None:
        check(lib.dt_tracker_collect(self._h, C.byref(fi), C.byref(fo)), "dt_tracker_collect")

    @property
    def stream(self) -> int:
        return int(lib.dt_tracker_stream(self._h) or 0)

    def set_profiling(self, on: bool) -> None:
        check(lib.dt_tracker_set_profiling(self._h, int(bool(on))), "dt_tracker_set_profiling")

    def phase_ms(self) -> dict:
        from ._lib import N_PHASES, PHASES

        buf = (C.c_float * N_PHASES)()
        check(lib.dt_tracker_get_phase_ms(self._h, C.cast(buf, C.c_void_p)), "dt_tracker_get_phase_ms")
        return {name: float(buf[i]) for i, name in enumerate(PHASES)}

    def trace(self, cap: int = 4096) -> np.ndarray:
        """(code, ns) pairs stamped by the solver kernel at its cluster barriers (last
        frame, profiling on)."""
        buf = np.zeros((cap, 2), dtype=np.int64)
        n = lib.dt_tracker_get_trace(self._h, _host_ptr(buf), cap)
        if n < 0:
            check(n, "dt_tracker_get_trace")
        return buf[:n].copy()

    def arrivals(self) -> np.ndarray:
        """(barriers, CTAs) globaltimer ns at which each CTA of the solver arrived at each
        domain barrier (last frame, profiling on)."""
        cap = 2 + 1024 * 256
        buf = np.zeros(cap, dtype=np.int64)
        stride = lib.dt_tracker_get_arrivals(self._h, _host_ptr(buf), cap)
        if stride < 0:
            check(stride, "dt_tracker_get_arrivals")
        if stride == 0:
            return np.zeros((0, 0), dtype=np.int64)
        n_cta, n_bar = int(buf[0]), min(int(buf[1]), stride)
        return buf[2:2 + n_cta * stride].reshape(n_cta, stride)[:, :n_bar].T.copy()

    def device_outputs(self):
        w, p, n = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib.dt_tracker_device_outputs(self._h, C.byref(w), C.byref(p), C.byref(n)),
              "dt_tracker_device_outputs")
        return w.value, p.value, n.value

    def launches(self) -> int:
        return int(lib.dt_tracker_last_launches(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.dt_tracker_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass


def _fingerprint(arrays) -> tuple:
    """Position-sensitive content digest (BLAKE2b over each array's bytes, shape and
    dtype) of the cached arrays: a template or graph edited in place after caching --
    including a reorder of rows -- is detected and rebuilt."""
    out = []
    for a in arrays:
        arr = np.ascontiguousarray(a)
        h = hashlib.blake2b(digest_size=16)
        h.update(repr((arr.shape, arr.dtype.str)).encode())
        h.update(arr.view(np.uint8).ravel().data)
        out.append(h.hexdigest())
    return tuple(out)


class _SessionCache:
    """Trackers keyed by the identity of the template / graph arrays they were built
    from (the arrays are held, so ids cannot be recycled while cached) and checked
    against a content digest, so in-place edits of those arrays are picked up."""

    def __init__(self, capacity: int = 4):
        self.capacity = capacity
        self._d: OrderedDict = OrderedDict()

    def get(self, template, graph, cfg: Config) -> DeviceTracker:
        arrays = (template.points, template.normals, template.bind_indices, template.bind_weights,
                  graph.points, graph.edges, graph.edge_weights)
        key = tuple(id(a) for a in arrays) + (cfg.width, cfg.height, float(graph.sampling_radius))
        fp = _fingerprint(arrays)
        hit = self._d.get(key)
        if hit is not None and hit[2] == fp:
            self._d.move_to_end(key)
            trk = hit[1]
            trk.set_config(cfg)
            return trk
        if hit is not None:  # the cached arrays were edited in place: rebuild
            del self._d[key]
            hit[1].close()
        trk = DeviceTracker(template, graph, cfg)
        self._d[key] = (arrays, trk, fp)
        while len(self._d) > self.capacity:
            _, (_, old, _) = self._d.popitem(last=False)
            old.close()
        return trk

    def clear(self) -> None:
        for _, (_, trk, _) in self._d.items():
            trk.close()
        self._d.clear()


SESSIONS = _SessionCache()


def nvh_message(n: int) -> str:
    """Message of the reference's NoValidHypothesis (matching.py:184, 208)."""
    if n < 3:
        return f"{n} matches cannot support a rotation hypothesis"
    return "every reference hypothesis was discarded"


def track_batched(trackers, frames) -> list:
    """One frame on each of several trackers (independent sequences, BASELINE config 5)
    through dt_track_frames_batched: every tracker's frame is enqueued on its own stream
    before any is collected, so the sequences overlap on the device. `frames` holds one
    dict of DeviceTracker.track keyword arguments (with "depth") per tracker."""
    if len(trackers) != len(frames):
        raise ValueError("one frame per tracker")
    ios = [t.prepare(**f) for t, f in zip(trackers, frames)]
    n = len(trackers)
    hs = (C.c_void_p * max(n, 1))(*[t._h for t in trackers])
    fis = (FrameInput * max(n, 1))(*[io["fi"] for io in ios])
    fos = (FrameOutput * max(n, 1))(*[io["fo"] for io in ios])
    check(lib.dt_track_frames_batched(hs, fis, fos, n, None), "dt_track_frames_batched")
    return [t.finish(io) for t, io in zip(trackers, ios)]

