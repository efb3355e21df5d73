"""Device twins of the reference's compiled kernels, same positional signatures.

Each function takes and returns numpy arrays exactly like its numba counterpart in
deformtrack/kernels.py, so the reference's operator tests (tests/test_kernels.py) and
its solver (which looks the kernels up at call time, solver.py:135,168,178,189) can run
on these. ``n_chunks`` is accepted for signature compatibility: the device reductions
are deterministic per control for any launch shape, so the argument has no effect.

* ``warp_and_rasterize``  kernels.py:483-569  -> dt_warp_and_rasterize
* ``icp_reduce``          kernels.py:148-220  -> dt_icp_reduce
* ``feature_reduce``      kernels.py:222-284  -> dt_feature_reduce
* ``arap_reduce``         kernels.py:341-467  -> dt_arap_reduce
"""

from __future__ import annotations

import numpy as np

from . import _device as dev
from ._lib import check, lib

N_COLS = 27


def _d(a, dtype=np.float64):
    return dev.to_device(np.asarray(a, dtype=dtype))


# The C-ABI trusts the sizes it is given; the numba kernels would raise IndexError on the
# same mismatches, so reject them here.
def _size(a, count, name):
    if int(np.size(a)) != int(count):
        raise ValueError(f"{name}: expected {count} elements, got {int(np.size(a))}")


def _index(idx, hi, name):
    if np.size(idx) and (int(np.min(idx)) < 0 or int(np.max(idx)) >= hi):
        raise IndexError(f"{name}: index outside [0, {hi})")


def warp_and_rasterize(points, normals, bind_idx, alpha, warps, depth, depth_valid,
                       obs_normals, fx, fy, cx, cy, gate_distance, cos_gate, n_chunks):
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    bidx = np.asarray(bind_idx, dtype=np.int64).reshape(n, -1)
    k = bidx.shape[1]
    W = np.asarray(warps, dtype=np.float64).reshape(-1, 8)
    depth = np.asarray(depth, dtype=np.float64)
    h, w = depth.shape
    _size(normals, 3 * n, "normals")
    _size(alpha, n * k, "alpha")
    _size(depth_valid, h * w, "depth_valid")
    _size(obs_normals, 3 * h * w, "obs_normals")
    _index(bidx, W.shape[0], "bind_idx")
    out_p = dev.empty((n, 3))
    out_n = dev.empty((n, 3))
    valid = dev.empty((n,), np.uint8)
    obs_p = dev.empty((n, 3))
    obs_n = dev.empty((n, 3))
    pixels = dev.empty((n, 2), np.int64)
    ins = [_d(pts), _d(normals), _d(bidx, np.int64), _d(alpha), _d(W), _d(depth),
           _d(depth_valid, np.uint8), _d(obs_normals)]
    check(lib.dt_warp_and_rasterize(
        dev.ptr(ins[0]), dev.ptr(ins[1]), dev.ptr(ins[2]), dev.ptr(ins[3]), n, k,
        dev.ptr(ins[4]), W.shape[0], dev.ptr(ins[5]), dev.ptr(ins[6]), dev.ptr(ins[7]), h, w,
        float(fx), float(fy), float(cx), float(cy), float(gate_distance), float(cos_gate),
        dev.ptr(out_p), dev.ptr(out_n), dev.ptr(valid), dev.ptr(obs_p), dev.ptr(obs_n),
        dev.ptr(pixels), dev.stream()), "warp_and_rasterize")
    return (dev.to_host(out_p), dev.to_host(out_n), dev.to_host(valid).astype(bool),
            dev.to_host(obs_p), dev.to_host(obs_n), dev.to_host(pixels))


def icp_reduce(points, obs_normals, obs_points, bind_idx, alpha, warps, basis, tukey_scale,
               frozen, use_frozen, want_jac, n_chunks, m):
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    bidx = np.asarray(bind_idx, dtype=np.int64).reshape(n, -1) if n else np.zeros((0, 1), np.int64)
    k = bidx.shape[1]
    m = int(m)
    _size(obs_normals, 3 * n, "obs_normals")
    _size(obs_points, 3 * n, "obs_points")
    _size(alpha, n * k, "alpha")
    _size(warps, 8 * m, "warps")
    _size(basis, 48 * m, "basis")
    if use_frozen:
        _size(frozen, n, "frozen")
    _index(bidx, m, "bind_idx")
    partial = dev.zeros((m, N_COLS))
    support = dev.zeros((m,))
    cost = dev.zeros((m,))
    r = dev.zeros((n,))
    fz = _d(frozen) if use_frozen else None
    ins = [_d(pts), _d(obs_normals), _d(obs_points), _d(bidx, np.int64), _d(alpha), _d(warps),
           _d(basis)]
    check(lib.dt_icp_reduce(
        dev.ptr(ins[0]), dev.ptr(ins[1]), dev.ptr(ins[2]), dev.ptr(ins[3]), dev.ptr(ins[4]), n, k,
        dev.ptr(ins[5]), dev.ptr(ins[6]), m, float(tukey_scale), dev.ptr(fz), int(bool(use_frozen)),
        int(bool(want_jac)), dev.ptr(partial), dev.ptr(support), dev.ptr(cost), dev.ptr(r),
        dev.stream()), "icp_reduce")
    return dev.to_host(partial), dev.to_host(support), dev.to_host(cost), dev.to_host(r)


def feature_reduce(points, obs_points, match_w, bind_idx, alpha, warps, basis, feature_weight,
                   want_jac, n_chunks, m):
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    bidx = np.asarray(bind_idx, dtype=np.int64).reshape(n, -1) if n else np.zeros((0, 1), np.int64)
    k = bidx.shape[1]
    m = int(m)
    _size(obs_points, 3 * n, "obs_points")
    _size(match_w, n, "match_w")
    _size(alpha, n * k, "alpha")
    _size(warps, 8 * m, "warps")
    _size(basis, 48 * m, "basis")
    _index(bidx, m, "bind_idx")
    partial = dev.zeros((m, N_COLS))
    support = dev.zeros((m,))
    cost = dev.zeros((m,))
    ins = [_d(pts), _d(obs_points), _d(match_w), _d(bidx, np.int64), _d(alpha), _d(warps),
           _d(basis)]
    check(lib.dt_feature_reduce(
        dev.ptr(ins[0]), dev.ptr(ins[1]), dev.ptr(ins[2]), dev.ptr(ins[3]), dev.ptr(ins[4]), n, k,
        dev.ptr(ins[5]), dev.ptr(ins[6]), m, float(feature_weight), int(bool(want_jac)),
        dev.ptr(partial), dev.ptr(support), dev.ptr(cost), dev.stream()), "feature_reduce")
    return dev.to_host(partial), dev.to_host(support), dev.to_host(cost)


def arap_reduce(ctrl_points, R, t, warps, edges, edge_weights, wa, angle_weight,
                rotation_weight, want_jac, n_chunks, m):
    E = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    ne = E.shape[0]
    m = int(m)
    _size(ctrl_points, 3 * m, "ctrl_points")
    _size(R, 9 * m, "R")
    _size(t, 3 * m, "t")
    _size(warps, 8 * m, "warps")
    _size(edge_weights, ne, "edge_weights")
    _size(wa, m, "wa")
    _index(E, m, "edges")
    partial = dev.zeros((m, N_COLS))
    cost = dev.zeros((m,))
    ins = [_d(ctrl_points), _d(R), _d(t), _d(warps), _d(E, np.int64), _d(edge_weights), _d(wa)]
    check(lib.dt_arap_reduce(
        dev.ptr(ins[0]), dev.ptr(ins[1]), dev.ptr(ins[2]), dev.ptr(ins[3]), dev.ptr(ins[4]),
        dev.ptr(ins[5]), ne, dev.ptr(ins[6]), m, float(angle_weight), float(rotation_weight),
        int(bool(want_jac)), dev.ptr(partial), dev.ptr(cost), dev.stream()), "arap_reduce")
    return dev.to_host(partial), dev.to_host(cost)


__all__ = ["N_COLS", "warp_and_rasterize", "icp_reduce", "feature_reduce", "arap_reduce"]
