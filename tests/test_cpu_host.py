"""CPU-only checks: the C-ABI library loads and exports every entry point the header
declares, and the host-side API logic (config validation, data types, KATs of the
small host formulas, the synthetic generator) behaves like the reference's."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "deformtrack_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|const char\*|void\*)\s+(dt_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2007_08576_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.EXPORTED)
    assert "sm_100a" in _lib.version()


def test_library_is_sm100a_cubin():
    import subprocess

    from paper_2007_08576_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_config_rejects_unknown_keys_and_round_trips():
    from paper_2007_08576_b200 import load_config
    from paper_2007_08576_b200.exceptions import ConfigError

    with pytest.raises(ConfigError):
        load_config({"solver": {"max_outer_iter": 3}})
    with pytest.raises(ConfigError):
        load_config({"bogus": 1})
    with pytest.raises(ConfigError):
        load_config({"seed": True})
    with pytest.raises(ConfigError):
        load_config({"solver": {"lambda_init": 10.0, "lambda_max": 1.0}})
    cfg = load_config({"sampling": {"radius": 5.0}, "seed": 3})
    d = cfg.to_dict()
    assert d["sampling"]["connection_sigma"] == 10.0 and d["sampling"]["bind_sigma"] == 5.0
    again = load_config(d)
    assert again.to_dict() == d


def test_matchset_and_host_formulas():
    from paper_2007_08576_b200.energy import tukey_weight
    from paper_2007_08576_b200.matching import MatchSet, reweight, soft_weight
    from paper_2007_08576_b200.solver import chunk_slices

    with pytest.raises(ValueError):
        MatchSet.from_pairs(np.zeros((3, 2)), np.zeros((3, 2)))
    H = 5.0
    # reweight / soft KATs (test_matching.py:112-120, SPEC acceptance criterion 5)
    np.testing.assert_allclose(reweight([0.0, H, 2 * H], H), [1.0, 1.0, 0.5], atol=1e-12)
    np.testing.assert_allclose(soft_weight([0.0, H, 2 * H, 5 * H], H), [1.0, 0.8, 0.6, 0.0],
                               atol=1e-12)
    # Tukey KAT (test_energy.py:133-136)
    np.testing.assert_allclose(tukey_weight([0.0, 5.0, -5.0, 10.0, -10.0, 30.0], 10.0),
                               [1.0, 0.5625, 0.5625, 0.0, 0.0, 0.0])
    for n, c in [(0, 4), (3, 8), (8, 8), (17, 4), (100, 8)]:
        cov = [i for s in chunk_slices(n, c) for i in range(s.start, s.stop)]
        assert cov == list(range(n))


def test_solver_config_validation():
    from paper_2007_08576_b200 import SolverConfig

    with pytest.raises(ValueError):
        SolverConfig(max_outer_iters=0)
    with pytest.raises(ValueError):
        SolverConfig(lambda_decrease=2.0)
    with pytest.raises(ValueError):
        SolverConfig(step_tol=-1.0)


def test_estimator_params():
    from sklearn.base import clone

    from paper_2007_08576_b200 import MatchInlierSelector, SurfaceDeformationTracker

    est = SurfaceDeformationTracker(sampling_radius=9.0, seed=3)
    p = est.get_params()
    assert p["sampling_radius"] == 9.0 and p["seed"] == 3
    assert clone(est).get_params() == p
    sel = MatchInlierSelector(n_references=12)
    assert sel.get_params()["n_references"] == 12
    with pytest.raises(ValueError):
        MatchInlierSelector._check_pairs(np.zeros((4, 5)))


def test_synth_scene_shapes_and_outliers():
    from paper_2007_08576_b200 import synth

    scene = synth.Scene(surface="sphere-patch", resolution=41, width=160, height=120,
                        n_features=200, outlier_fraction=0.25, n_distractors=50)
    seq = synth.make_sequence(scene, 2)
    assert len(seq.template) == 41 * 41
    fr = seq.frames[1]
    assert fr.depth.shape == (120, 160)
    assert np.isfinite(fr.depth).all() and (fr.depth > 0).mean() > 0.3
    assert fr.descriptors.shape == (250, 32) and fr.keypoints.shape == (250, 2)
    assert fr.is_outlier.sum() == 50
    # rendered depth lies on the analytic deformed surface (back-projected pixels)
    assert fr.match_src.shape == fr.match_dst.shape == (200, 3)
