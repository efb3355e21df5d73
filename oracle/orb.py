"""CPU restatement of the ORB front end built on the device (dt_orb.cu) -- TEST
INFRASTRUCTURE ONLY (the checker for tests/, never called by the product).

SURVEY.md §8(f) #2: the paper's upstream stage (FAST corners + uniform suppression +
oriented BRIEF) that produces the frame descriptors / keypoints a4 consumes.
It is not in the reference, so this restatement *defines* the algorithm and
parity is exact against it (parity unpinned by any reference output):

* FAST-9 on the 16-pixel Bresenham circle of radius 3. Score = the largest threshold for
  which the pixel is still a corner plus one: max over the 16 arcs of 9 contiguous circle
  pixels of the arc's minimum brightness difference (brighter arcs: ring - centre;
  darker arcs: centre - ring). A corner is a pixel with score > threshold.
* 3x3 non-maximum suppression with the total order (score, -index): a corner survives
  when no neighbour is greater in that order.
* Uniform suppression: the image is cut into cells; each cell keeps its best `per_cell`
  corners, then the best `n_max` overall (order: score descending, index ascending),
  output in that order.
* Orientation by the intensity centroid over the disc of radius 15 (integer moments),
  quantised to one of 30 sectors by exact sign tests against the sector boundaries
  (no atan2, so host and device agree bit for bit).
* rBRIEF: 256 tests between two points of a seeded Gaussian pattern (offsets within
  +-13 px) rotated by the sector angle and rounded (tables built on the host), each on
  5x5 box sums of the image; bit i = box(p + a_i) < box(p + b_i), little-endian in 32
  bytes.
"""

from __future__ import annotations

import numpy as np

CIRCLE = np.array([(0, -3), (1, -3), (2, -2), (3, -1), (3, 0), (3, 1), (2, 2), (1, 3),
                   (0, 3), (-1, 3), (-2, 2), (-3, 1), (-3, 0), (-3, -1), (-2, -2), (-1, -3)],
                  dtype=np.int64)  # (dx, dy)
ARC = 9
N_BINS = 30
ORI_RADIUS = 15
BORDER = 21  # rotated pattern (<= 13 sqrt 2) + box half-width 2, rounded up


def pattern(seed: int = 20070857, n: int = 256, extent: int = 13) -> np.ndarray:
    """(n, 4) int offsets (ax, ay, bx, by): isotropic Gaussian, sigma = 31 / 5, clipped."""
    rng = np.random.default_rng(seed)
    p = np.rint(rng.normal(0.0, 31.0 / 5.0, size=(n, 4)))
    return np.clip(p, -extent, extent).astype(np.int64)


def sector_boundaries() -> np.ndarray:
    """(N_BINS + 1, 2) unit vectors of the sector boundaries, phi_j = -pi + j 2pi/30."""
    phi = -np.pi + np.arange(N_BINS + 1) * (2.0 * np.pi / N_BINS)
    return np.stack([np.cos(phi), np.sin(phi)], axis=1)


def rotated_patterns(pat: np.ndarray) -> np.ndarray:
    """(N_BINS, n, 4) int offsets: the pattern rotated to each sector's centre angle."""
    out = np.empty((N_BINS,) + pat.shape, dtype=np.int64)
    for j in range(N_BINS):
        th = -np.pi + (j + 0.5) * (2.0 * np.pi / N_BINS)
        c, s = np.cos(th), np.sin(th)
        for k in (0, 2):
            x, y = pat[:, k].astype(np.float64), pat[:, k + 1].astype(np.float64)
            out[j, :, k] = np.rint(c * x - s * y).astype(np.int64)
            out[j, :, k + 1] = np.rint(s * x + c * y).astype(np.int64)
    return out


def fast_scores(img: np.ndarray) -> np.ndarray:
    """(H, W) int32 FAST-9 score (0 within 3 px of the border)."""
    im = np.asarray(img, dtype=np.int32)
    h, w = im.shape
    sc = np.zeros((h, w), dtype=np.int32)
    if h < 7 or w < 7:
        return sc
    c = im[3:h - 3, 3:w - 3]
    ring = np.stack([im[3 + dy:h - 3 + dy, 3 + dx:w - 3 + dx] for dx, dy in CIRCLE], axis=0)
    best = np.zeros_like(c)
    for sign in (1, -1):
        d = sign * (ring - c[None])  # (16, h-6, w-6)
        for s0 in range(16):
            idx = [(s0 + k) % 16 for k in range(ARC)]
            best = np.maximum(best, d[idx].min(axis=0))
    sc[3:h - 3, 3:w - 3] = np.maximum(best, 0)
    return sc


def nms_mask(score: np.ndarray, threshold: int) -> np.ndarray:
    h, w = score.shape
    idx = np.arange(h * w, dtype=np.int64).reshape(h, w)
    keep = score > threshold
    pad_s = np.pad(score, 1, constant_values=-1)
    pad_i = np.pad(idx, 1, constant_values=-1)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            if dx == 0 and dy == 0:
                continue
            ns = pad_s[1 + dy:1 + dy + h, 1 + dx:1 + dx + w]
            ni = pad_i[1 + dy:1 + dy + h, 1 + dx:1 + dx + w]
            keep &= ~((ns > score) | ((ns == score) & (ni >= 0) & (ni < idx)))
    return keep


def select(score, keep, cell: int, per_cell: int, n_max: int):
    """Indices (row-major) of the kept corners after uniform suppression, best first."""
    h, w = score.shape
    ys, xs = np.nonzero(keep)
    ok = (xs >= BORDER) & (xs < w - BORDER) & (ys >= BORDER) & (ys < h - BORDER)
    ys, xs = ys[ok], xs[ok]
    sc = score[ys, xs].astype(np.int64)
    lin = ys.astype(np.int64) * w + xs
    ncx = (w + cell - 1) // cell
    cid = (ys // cell) * ncx + xs // cell
    order = np.lexsort((lin, -sc, cid))
    cid_s = cid[order]
    first = np.searchsorted(cid_s, cid_s, side="left")
    rank = np.arange(len(order)) - first
    sel = order[rank < per_cell]
    order2 = np.lexsort((lin[sel], -sc[sel]))
    sel = sel[order2][:n_max]
    return lin[sel], sc[sel]


def box5(img: np.ndarray) -> np.ndarray:
    im = np.asarray(img, dtype=np.int32)
    h, w = im.shape
    pad = np.pad(im, 2)
    out = np.zeros((h, w), dtype=np.int32)
    for dy in range(5):
        for dx in range(5):
            out += pad[dy:dy + h, dx:dx + w]
    return out


def orientation_bins(img: np.ndarray, lin: np.ndarray) -> np.ndarray:
    im = np.asarray(img, dtype=np.int64)
    h, w = im.shape
    r = ORI_RADIUS
    oy, ox = np.mgrid[-r:r + 1, -r:r + 1]
    disc = ox * ox + oy * oy <= r * r
    ox, oy = ox[disc], oy[disc]
    bnd = sector_boundaries()
    bins = np.empty(len(lin), dtype=np.int64)
    for k, p in enumerate(lin):
        y, x = divmod(int(p), w)
        v = im[y + oy, x + ox]
        m10 = int(np.sum(ox * v))
        m01 = int(np.sum(oy * v))
        bins[k] = sector_of(m10, m01, bnd)
    return bins


def sector_of(m10: int, m01: int, bnd: np.ndarray) -> int:
    """Sector j with cross(b_j, v) >= 0 and cross(b_{j+1}, v) < 0; the zero vector and
    the direction -x (angle pi) follow the half-open convention [phi_j, phi_{j+1})."""
    if m10 == 0 and m01 == 0:
        return N_BINS // 2  # angle 0
    vx, vy = float(m10), float(m01)
    for j in range(N_BINS):
        c0 = bnd[j, 0] * vy - bnd[j, 1] * vx
        c1 = bnd[j + 1, 0] * vy - bnd[j + 1, 1] * vx
        if c0 >= 0.0 and c1 < 0.0:
            return j
    return 0  # angle exactly pi (v = (-a, 0)): boundary 0 and 30 coincide


def describe(img: np.ndarray, lin: np.ndarray, bins: np.ndarray, rot: np.ndarray) -> np.ndarray:
    b = box5(img)
    h, w = b.shape
    out = np.zeros((len(lin), 32), dtype=np.uint8)
    for k, p in enumerate(lin):
        y, x = divmod(int(p), w)
        t = rot[int(bins[k])]
        va = b[y + t[:, 1], x + t[:, 0]]
        vb = b[y + t[:, 3], x + t[:, 2]]
        bits = (va < vb).astype(np.uint8)
        out[k] = np.packbits(bits, bitorder="little")
    return out


def detect_and_describe(img, threshold=20, cell=32, per_cell=8, n_max=2500, seed=20070857):
    """Returns keypoints (n, 2) int32 (u, v), descriptors (n, 32) uint8, scores (n,),
    sector bins (n,)."""
    img = np.asarray(img, dtype=np.uint8)
    h, w = img.shape
    sc = fast_scores(img)
    keep = nms_mask(sc, threshold)
    lin, score = select(sc, keep, cell, per_cell, n_max)
    bins = orientation_bins(img, lin)
    desc = describe(img, lin, bins, rotated_patterns(pattern(seed)))
    kp = np.stack([lin % w, lin // w], axis=1).astype(np.int32)
    return kp, desc, score.astype(np.int32), bins.astype(np.int32)
