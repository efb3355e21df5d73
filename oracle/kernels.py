"""ORACLE (test infrastructure only): ctypes front of oracle/_build/liboracle.so.

Signatures follow deformtrack/kernels.py so fixtures and the GPU twins can be compared
call for call:

* ``warp_and_rasterize``  kernels.py:483-569
* ``icp_reduce``          kernels.py:148-220
* ``feature_reduce``      kernels.py:222-284
* ``arap_reduce``         kernels.py:341-467
* ``hamming_match``       builder-defined (north-star part 3a)
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_build" / "liboracle.so"
N_COLS = 27

P = C.c_void_p
I64 = C.c_int64
F64 = C.c_double
I = C.c_int


def _load():
    if not _LIB_PATH.exists():
        import importlib.util

        spec = importlib.util.spec_from_file_location(
            "_dt_build", Path(__file__).resolve().parent.parent / "paper_2007_08576_b200" / "_build.py")
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.build_oracle()
    lib = C.CDLL(str(_LIB_PATH))
    lib.or_icp_reduce.argtypes = [P, P, P, P, P, I64, I, P, P, F64, P, I, I, I, I64, P, P, P, P]
    lib.or_feature_reduce.argtypes = [P, P, P, P, P, I64, I, P, P, F64, I, I, I64, P, P, P]
    lib.or_arap_reduce.argtypes = [P, P, P, P, P, P, I64, P, F64, F64, I, I, I64, P, P]
    lib.or_warp_and_rasterize.argtypes = [P, P, P, P, I64, I, P, P, P, P, I64, I64, F64, F64, F64,
                                          F64, F64, F64, I, P, P, P, P, P, P]
    lib.or_hamming_match.argtypes = [P, I64, P, I64, P, P]
    lib.or_set_threads.argtypes = [I]
    lib.or_max_threads.restype = I
    for fn in (lib.or_icp_reduce, lib.or_feature_reduce, lib.or_arap_reduce,
               lib.or_warp_and_rasterize, lib.or_hamming_match):
        fn.restype = I
    return lib


_lib = _load()


def set_threads(n: int) -> None:
    _lib.or_set_threads(int(n))


def max_threads() -> int:
    return int(_lib.or_max_threads())


def _c(a, dtype=np.float64):
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr, (arr.ctypes.data if arr.size else None)


def _ok(st: int, what: str) -> None:
    if st != 0:
        raise RuntimeError(f"oracle {what} failed ({st})")


def icp_reduce(points, obs_normals, obs_points, bind_idx, alpha, warps, basis, tukey_scale,
               frozen, use_frozen, want_jac, n_chunks, m):
    pts, pp = _c(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    n = pts.shape[0]
    bi, bip = _c(np.asarray(bind_idx).reshape(n, -1) if n else np.zeros((0, 1)), np.int64)
    k = bi.shape[1]
    keep = [_c(obs_normals), _c(obs_points), _c(alpha), _c(warps), _c(basis),
            _c(frozen if use_frozen else np.zeros(max(n, 1)))]
    partial = np.zeros((m, N_COLS))
    support = np.zeros(m)
    cost = np.zeros(m)
    r = np.zeros(n)
    _ok(_lib.or_icp_reduce(pp, keep[0][1], keep[1][1], bip, keep[2][1], n, k, keep[3][1],
                           keep[4][1], float(tukey_scale), keep[5][1], int(bool(use_frozen)),
                           int(bool(want_jac)), int(n_chunks), int(m), partial.ctypes.data,
                           support.ctypes.data, cost.ctypes.data, r.ctypes.data if n else None),
        "icp_reduce")
    return partial, support, cost, r


def feature_reduce(points, obs_points, match_w, bind_idx, alpha, warps, basis, feature_weight,
                   want_jac, n_chunks, m):
    pts, pp = _c(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    n = pts.shape[0]
    bi, bip = _c(np.asarray(bind_idx).reshape(n, -1) if n else np.zeros((0, 1)), np.int64)
    k = bi.shape[1]
    keep = [_c(obs_points), _c(match_w), _c(alpha), _c(warps), _c(basis)]
    partial = np.zeros((m, N_COLS))
    support = np.zeros(m)
    cost = np.zeros(m)
    _ok(_lib.or_feature_reduce(pp, keep[0][1], keep[1][1], bip, keep[2][1], n, k, keep[3][1],
                               keep[4][1], float(feature_weight), int(bool(want_jac)),
                               int(n_chunks), int(m), partial.ctypes.data, support.ctypes.data,
                               cost.ctypes.data), "feature_reduce")
    return partial, support, cost


def arap_reduce(ctrl_points, R, t, warps, edges, edge_weights, wa, angle_weight, rotation_weight,
                want_jac, n_chunks, m):
    E, ep = _c(np.asarray(edges).reshape(-1, 2), np.int64)
    keep = [_c(ctrl_points), _c(R), _c(t), _c(warps), _c(edge_weights), _c(wa)]
    partial = np.zeros((m, N_COLS))
    cost = np.zeros(m)
    _ok(_lib.or_arap_reduce(keep[0][1], keep[1][1], keep[2][1], keep[3][1], ep, keep[4][1],
                            E.shape[0], keep[5][1], float(angle_weight), float(rotation_weight),
                            int(bool(want_jac)), int(n_chunks), int(m), partial.ctypes.data,
                            cost.ctypes.data), "arap_reduce")
    return partial, cost


def warp_and_rasterize(points, normals, bind_idx, alpha, warps, depth, depth_valid, obs_normals,
                       fx, fy, cx, cy, gate_distance, cos_gate, n_chunks):
    pts, pp = _c(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    n = pts.shape[0]
    bi, bip = _c(np.asarray(bind_idx).reshape(n, -1), np.int64)
    k = bi.shape[1]
    d, dp = _c(depth)
    h, w = d.shape
    keep = [_c(normals), _c(alpha), _c(warps), _c(np.asarray(depth_valid), np.uint8),
            _c(obs_normals)]
    out_p = np.empty((n, 3))
    out_n = np.empty((n, 3))
    valid = np.zeros(n, dtype=np.uint8)
    obs_p = np.zeros((n, 3))
    obs_n = np.zeros((n, 3))
    pixels = np.full((n, 2), -1, dtype=np.int64)
    _ok(_lib.or_warp_and_rasterize(pp, keep[0][1], bip, keep[1][1], n, k, keep[2][1], dp,
                                   keep[3][1], keep[4][1], h, w, float(fx), float(fy), float(cx),
                                   float(cy), float(gate_distance), float(cos_gate),
                                   int(n_chunks), out_p.ctypes.data, out_n.ctypes.data,
                                   valid.ctypes.data, obs_p.ctypes.data, obs_n.ctypes.data,
                                   pixels.ctypes.data), "warp_and_rasterize")
    return out_p, out_n, valid.astype(bool), obs_p, obs_n, pixels


def hamming_match(template_desc, frame_desc):
    td, tp = _c(np.asarray(template_desc).reshape(-1, 32), np.uint8)
    fd, fp = _c(np.asarray(frame_desc).reshape(-1, 32), np.uint8)
    idx = np.empty(td.shape[0], dtype=np.int32)
    dist = np.empty(td.shape[0], dtype=np.int32)
    if td.shape[0]:
        _ok(_lib.or_hamming_match(tp, td.shape[0], fp, fd.shape[0], idx.ctypes.data,
                                  dist.ctypes.data), "hamming_match")
    return idx, dist
