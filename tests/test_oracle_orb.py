"""ORB restatement (oracle/orb.py) known-answer tests on the CPU, and
the product's sampling tables (paper_2007_08576_b200.orb) equal to the oracle's."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import orb as O  # noqa: E402


def _ring_image(ring_vals, centre=100, size=15):
    img = np.full((size, size), centre, dtype=np.uint8)
    c = size // 2
    for (dx, dy), v in zip(O.CIRCLE, ring_vals):
        img[c + dy, c + dx] = v
    return img, c


def test_fast_score_known_answers():
    # all 16 brighter by 90: score 90
    img, c = _ring_image([190] * 16)
    assert O.fast_scores(img)[c, c] == 90
    # exactly 9 contiguous brighter by 50, the rest equal: score 50
    img, c = _ring_image([150] * 9 + [100] * 7)
    assert O.fast_scores(img)[c, c] == 50
    # 8 contiguous only: not a corner at any threshold (score 0)
    img, c = _ring_image([150] * 8 + [100] * 8)
    assert O.fast_scores(img)[c, c] == 0
    # a darker arc wrapping around index 0, minimum difference 30
    ring = [100] * 16
    for k in list(range(12, 16)) + list(range(0, 5)):
        ring[k] = 70 if k != 2 else 40
    img, c = _ring_image(ring)
    assert O.fast_scores(img)[c, c] == 30


def test_sector_of_axes():
    bnd = O.sector_boundaries()
    assert O.sector_of(5, 0, bnd) == 15    # angle 0
    assert O.sector_of(0, 5, bnd) == 22    # pi / 2 -> 22.5 -> sector 22
    assert O.sector_of(0, -5, bnd) == 7    # -pi / 2 -> 7.5
    assert O.sector_of(0, 0, bnd) == 15    # undefined direction: angle 0
    assert O.sector_of(-5, 1, bnd) == 29   # just below pi


def test_nms_ties_go_to_lower_index():
    sc = np.zeros((5, 5), dtype=np.int32)
    sc[2, 2] = sc[2, 3] = 40
    keep = O.nms_mask(sc, 10)
    assert keep[2, 2] and not keep[2, 3]


def test_product_tables_equal_oracle_tables():
    from paper_2007_08576_b200 import orb

    np.testing.assert_array_equal(orb.brief_pattern(), O.pattern())
    np.testing.assert_array_equal(orb.sector_boundaries(), O.sector_boundaries())
    np.testing.assert_array_equal(orb.rotated_pattern(orb.brief_pattern()),
                                  O.rotated_patterns(O.pattern()))
    # every rotated test stays inside the descriptor border (box half-width 2)
    assert np.abs(O.rotated_patterns(O.pattern())).max() + 2 <= O.BORDER
