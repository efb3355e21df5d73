"""Shared loaders for the golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the reference) and small scene helpers."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def jload(a) -> dict:
    return json.loads(str(a))


def solver_case(name: str):
    """(tpl tuple, graph tuple, warps_in, depth, cam tuple, camera dims, matches or None,
    weights dict, solver dict, radius, expected warps, expected report dict)."""
    d = load(name)
    tpl = (d["t_points"], d["t_normals"], d["bind_idx"], d["bind_w"])
    graph = (d["ctrl"], d["edges"], d["edge_w"])
    cam = tuple(float(x) for x in d["cam"][:4])
    dims = (int(d["cam"][4]), int(d["cam"][5]))
    matches = None
    if "m_src" in d:
        matches = (d["m_src"], d["m_dst"], d["m_w"], d["m_flags"])
    return dict(tpl=tpl, graph=graph, warps_in=d["warps_in"], depth=d["depth"], cam=cam,
                dims=dims, matches=matches, weights=jload(d["weights"]),
                solver=jload(d["solver"]), radius=float(d["radius"]), warps_out=d["warps_out"],
                report=jload(d["report"]))


SOLVER_CASES = ["solver_fixed_point", "solver_translation", "solver_rigid_matches",
                "solver_occluded", "solver_no_data", "solver_no_data_stall"]


def hamming_kat_descriptors(seed: int = 0, nt: int = 40, nf: int = 70):
    """Known-answer set for the Hamming matcher: a frame built from the template
    descriptors with exactly known flips plus decoys, including exact ties."""
    rng = np.random.default_rng(seed)
    td = rng.integers(0, 256, size=(nt, 32), dtype=np.uint8)
    fd = rng.integers(0, 256, size=(nf, 32), dtype=np.uint8)
    expect_idx = np.empty(nt, dtype=np.int32)
    expect_dist = np.empty(nt, dtype=np.int32)
    slots = rng.permutation(nf)[: nt * 1]
    for t in range(nt):
        f = int(slots[t])
        flips = t % 9  # 0..8 bits
        d = td[t].copy()
        bits = rng.choice(256, size=flips, replace=False)
        for b in bits:
            d[b // 8] ^= np.uint8(1 << (b % 8))
        fd[f] = d
        expect_idx[t] = f
        expect_dist[t] = flips
    # recompute the true argmin (decoys are ~128 bits away, but be exact)
    x = np.bitwise_xor(td[:, None, :], fd[None, :, :])
    dist = np.unpackbits(x, axis=2).sum(axis=2)
    return td, fd, dist.argmin(axis=1).astype(np.int32), dist.min(axis=1).astype(np.int32)
