"""CPU checks of the stereo restatement (oracle/stereo.py): on synthetic rectified pairs
of known depth it recovers the disparity to a fraction of a pixel, constant depth
exactly, and its ZNCC window sums match a brute-force evaluation."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import stereo as OS  # noqa: E402


def test_recovers_known_depth():
    fx, B = 300.0, 20.0
    surf = lambda y, x: 300.0 + 15.0 * np.sin(x / 20.0) + 10.0 * np.cos(y / 15.0)  # noqa: E731
    L, R, z, disp = OS.synthetic_pair(96, 128, fx, B, surf, seed=1)
    dep, dd, win = OS.stereo_depth(L, R, 40, 3, fx, B)
    ok = np.isfinite(dep)
    assert ok.mean() > 0.6
    assert float(np.median(np.abs(dd - disp)[ok])) < 0.1
    assert float(np.median(np.abs(dep - z)[ok])) < 1.5


def test_constant_disparity_and_bruteforce_ncc():
    fx, B = 300.0, 20.0
    L, R, z, disp = OS.synthetic_pair(40, 64, fx, B, lambda y, x: 300.0 + 0 * x, seed=2)
    dep, dd, win = OS.stereo_depth(L, R, 32, 2, fx, B)
    ok = win >= 0
    assert float(np.mean(win[ok] == 20)) > 0.95 and abs(float(np.median(dd[ok])) - 20.0) < 1e-3
    vol = OS.ncc_volume(L, R, 32, 2)
    y, x, d, r = 20, 40, 20, 2
    a = L[y - r:y + r + 1, x - r:x + r + 1].astype(np.int64).ravel()
    b = R[y - r:y + r + 1, x - d - r:x - d + r + 1].astype(np.int64).ravel()
    n = a.size
    num = n * (a * b).sum() - a.sum() * b.sum()
    den = float(n * (a * a).sum() - a.sum() ** 2) * float(n * (b * b).sum() - b.sum() ** 2)
    assert vol[d, y, x] == float(num) / np.sqrt(den)
