"""ORACLE (test infrastructure only): stereo depth.

The paper computes the frame's depth with a GPU stereo matcher ("Readers may
refer to Ref. ZHOUTMI2019") that the reference does not ship (depth arrives as
a map). Parity is therefore unpinned by the reference; this restatement DEFINES the
algorithm of csrc/dt_stereo.cu, and the device matches it bit for bit:

* rectified grey pair (uint8), left pixel x <-> right pixel x - d, d in [0, max_disp);
* cost = zero-mean normalized cross-correlation over a (2r+1)^2 window, from exact integer
  window sums: ncc = (n SLR - SL SR) / sqrt((n SLL - SL^2) (n SRR - SR^2)), IEEE double;
  a window leaving either image or with zero variance has no cost;
* left winner-take-all (largest ncc, ties -> smaller d) and right winner-take-all
  (right pixel xr over the left pixels xr + d); a left match survives when its ncc >=
  min_ncc and the right winner at x - d is within lr_tol of d;
* sub-pixel parabola through d-1, d, d+1 when both neighbours have a cost and the
  curvature is negative: d + (c- - c+) / (2 ((c- - 2 c0) + c+));
* depth z = (fx * baseline) / disparity (NaN where no match survives).
"""

from __future__ import annotations

import numpy as np


def _box(a: np.ndarray, r: int) -> np.ndarray:
    """Window sums over (2r+1)^2 of an int64 image; entries whose window leaves the image
    are 0 (the callers mask them)."""
    h, w = a.shape
    k = 2 * r + 1
    ii = np.zeros((h + 1, w + 1), dtype=np.int64)
    ii[1:, 1:] = a.cumsum(0).cumsum(1)
    out = np.zeros((h, w), dtype=np.int64)
    if h >= k and w >= k:
        out[r:h - r, r:w - r] = (ii[k:, k:] - ii[:-k, k:] - ii[k:, :-k] + ii[:-k, :-k])
    return out


def ncc_volume(left: np.ndarray, right: np.ndarray, max_disp: int, r: int) -> np.ndarray:
    """(max_disp, h, w) float64: ncc of left pixel (y, x) at disparity d, -inf where none."""
    L = np.asarray(left, dtype=np.int64)
    R = np.asarray(right, dtype=np.int64)
    h, w = L.shape
    n = (2 * r + 1) ** 2
    SL, SLL = _box(L, r), _box(L * L, r)
    SRb, SRRb = _box(R, r), _box(R * R, r)
    vol = np.full((max_disp, h, w), -np.inf)
    ys = np.arange(h)[:, None]
    xs = np.arange(w)[None, :]
    for d in range(max_disp):
        P = np.zeros((h, w), dtype=np.int64)
        if d < w:
            P[:, d:] = L[:, d:] * R[:, :w - d]
        SLR = _box(P, r)
        SR = np.zeros((h, w), dtype=np.int64)
        SRR = np.zeros((h, w), dtype=np.int64)
        if d < w:
            SR[:, d:] = SRb[:, :w - d]
            SRR[:, d:] = SRRb[:, :w - d]
        ok = (ys >= r) & (ys < h - r) & (xs - d - r >= 0) & (xs + r < w)
        num = n * SLR - SL * SR
        dl = n * SLL - SL * SL
        dr = n * SRR - SR * SR
        ok &= (dl > 0) & (dr > 0)
        with np.errstate(invalid="ignore", divide="ignore"):
            c = num.astype(np.float64) / np.sqrt(dl.astype(np.float64) * dr.astype(np.float64))
        vol[d] = np.where(ok, c, -np.inf)
    return vol


def stereo_depth(left, right, max_disp: int, radius: int, fx: float, baseline: float,
                 min_ncc: float = 0.5, lr_tol: int = 1):
    """(depth (h,w) f64 NaN-invalid, disparity (h,w) f64 NaN-invalid, integer winner
    (h,w) int32 -1-invalid) of the rectified pair."""
    vol = ncc_volume(left, right, max_disp, radius)
    D, h, w = vol.shape
    best = vol.max(axis=0)
    dL = vol.argmax(axis=0).astype(np.int32)  # first maximum: ties -> smaller d
    hasL = np.isfinite(best)
    # right view: right pixel xr, left pixel xr + d
    volR = np.full_like(vol, -np.inf)
    for d in range(D):
        if d < w:
            volR[d][:, :w - d] = vol[d][:, d:]
    bestR = volR.max(axis=0)
    dR = np.where(np.isfinite(bestR), volR.argmax(axis=0), -1).astype(np.int32)
    xs = np.arange(w)[None, :].repeat(h, 0)
    xr = xs - dL
    inb = (xr >= 0) & hasL
    dRx = np.full((h, w), -1, dtype=np.int32)
    dRx[inb] = dR[np.nonzero(inb)[0], xr[inb]]
    keep = hasL & (best >= min_ncc) & (dRx >= 0) & (np.abs(dRx - dL) <= lr_tol)
    win = np.where(keep, dL, -1).astype(np.int32)
    disp = np.full((h, w), np.nan)
    yy, xx = np.nonzero(keep)
    for y, x in zip(yy.tolist(), xx.tolist()):
        d = int(dL[y, x])
        c0 = vol[d, y, x]
        delta = 0.0
        if 0 < d < D - 1:
            cm, cp = vol[d - 1, y, x], vol[d + 1, y, x]
            if np.isfinite(cm) and np.isfinite(cp):
                den = (cm - 2.0 * c0) + cp
                if den < 0.0:
                    delta = (cm - cp) / (2.0 * den)
        disp[y, x] = float(d) + delta
    fxb = fx * baseline
    with np.errstate(divide="ignore", invalid="ignore"):
        depth = np.where(keep & (disp > 0.0), fxb / disp, np.nan)
    return depth, disp, win


def synthetic_pair(h: int, w: int, fx: float, baseline: float, depth_fn, seed: int = 0):
    """A rectified pair of a textured surface at depth_fn(y, x) (mm): a smoothed random
    texture on the left view; the right view samples it at x + disparity (linear
    interpolation), so the true disparity of left pixel x is fx B / z."""
    rng = np.random.default_rng(seed)
    tex = rng.uniform(0, 255, size=(h, w + 256))
    k = np.array([1.0, 2.0, 1.0]) / 4.0
    tex = np.apply_along_axis(lambda r: np.convolve(r, k, mode="same"), 1, tex)
    tex = np.apply_along_axis(lambda c: np.convolve(c, k, mode="same"), 0, tex)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    z = depth_fn(yy, xx)
    disp = fx * baseline / z
    left = tex[:, :w]
    # right pixel xr shows the left pixel x with x - disp(x) = xr: fixed-point iterations
    xs = xx + disp
    for _ in range(8):
        xs = xx + fx * baseline / depth_fn(yy, xs)
    x0 = np.floor(xs).astype(int)
    t = xs - x0
    x0 = np.clip(x0, 0, tex.shape[1] - 2)
    right = (1 - t) * tex[yy.astype(int), x0] + t * tex[yy.astype(int), x0 + 1]
    return (np.ascontiguousarray(np.clip(np.rint(left), 0, 255).astype(np.uint8)),
            np.ascontiguousarray(np.clip(np.rint(right), 0, 255).astype(np.uint8)), z, disp)
