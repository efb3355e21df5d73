"""The GPU-resident I/O loop: ``cli track`` streaming PFM frames and
match files through the pipelined C-ABI, after the reference's tests/test_cli.py --
outputs, a byte-identical rerun from the echoed config (test_cli.py:69-85), a corrupt
frame keeping the earlier frames (test_cli.py:168-182) -- plus what the reference lacks:
resuming from the warp checkpoint of frame k reproduces the uninterrupted run byte for
byte, and the streamed frames equal the synchronous track() frames bit for bit."""

import shutil
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu

N_FRAMES = 5


def run(*argv) -> int:
    from paper_2007_08576_b200.cli import main

    return main([str(a) for a in argv])


@pytest.fixture(scope="module")
def seq(tmp_path_factory):
    root = tmp_path_factory.mktemp("cli")
    assert run("synth", "--config-id", "1", "--n-frames", N_FRAMES, "--out", root / "data") == 0
    assert run("track", "--config", root / "data" / "config.json",
               "--template", root / "data" / "template.ply", "--frames", root / "data" / "frames",
               "--matches", root / "data" / "matches", "--out", root / "rec") == 0
    return root


def _stems(n=N_FRAMES):
    return [f"frame_{i:04d}" for i in range(n)]


def test_track_writes_every_output(seq):
    from paper_2007_08576_b200 import fileio

    tpl, _ = fileio.read_ply(seq / "data" / "template.ply")
    for stem in _stems():
        pts, nrm = fileio.read_ply(seq / "rec" / f"{stem}.ply")
        assert pts.shape == tpl.shape and nrm is not None
        rep = fileio.read_json(seq / "rec" / f"{stem}.report.json")
        assert rep["report"]["counts"]["correspondences"] > 0
        assert rep["config"]["sampling"]["radius"] == 10.0
        m = fileio.read_matches(seq / "rec" / f"{stem}.matches.json")
        assert len(m) > 0 and m.preselected.any()
        w = fileio.read_warps(seq / "rec" / f"{stem}.warps.json")
        assert w.shape[1] == 8
    # the tracked surface follows the truth (synthetic bend, 10 % outlier matches)
    truth, _ = fileio.read_ply(seq / "data" / "truth" / "frame_0004.ply")
    rec, _ = fileio.read_ply(seq / "rec" / "frame_0004.ply")
    assert float(np.sqrt(np.mean(np.sum((rec - truth) ** 2, axis=1)))) < 2.0


def test_streamed_frames_equal_synchronous_frames(seq):
    """The pipelined path (2 frames in flight) vs Tracker.track frame by frame."""
    import paper_2007_08576_b200 as dt
    from paper_2007_08576_b200 import fileio
    from paper_2007_08576_b200.cli import _camera
    from paper_2007_08576_b200.warpfield import Template

    cfg = dt.load_config(fileio.read_json(seq / "data" / "config.json"))
    cam = _camera(cfg)
    p, n = fileio.read_ply(seq / "data" / "template.ply")
    tpl, graph = dt.prepare_template(Template(p, n), cfg)
    trk = dt.Tracker(tpl, graph, cam, cfg)
    for stem in _stems():
        depth = fileio.read_pfm(seq / "data" / "frames" / f"{stem}.pfm")
        m = fileio.read_matches(seq / "data" / "matches" / f"{stem}.json")
        r = trk.track(depth, m)
        pts, nrm = fileio.read_ply(seq / "rec" / f"{stem}.ply")
        np.testing.assert_array_equal(pts, r.points)
        np.testing.assert_array_equal(nrm, r.normals)
        np.testing.assert_array_equal(fileio.read_warps(seq / "rec" / f"{stem}.warps.json"),
                                      r.graph.warps)
        rep = fileio.read_json(seq / "rec" / f"{stem}.report.json")["report"]
        assert rep == __import__("json").loads(__import__("json").dumps(r.report.to_dict()))
    trk.close()


def test_embedded_config_reruns_to_identical_bytes(seq, tmp_path):
    from paper_2007_08576_b200 import fileio

    echo = fileio.read_json(seq / "rec" / "frame_0000.report.json")["config"]
    fileio.write_json(tmp_path / "echo.json", echo)
    assert run("track", "--config", tmp_path / "echo.json",
               "--template", seq / "data" / "template.ply", "--frames", seq / "data" / "frames",
               "--matches", seq / "data" / "matches", "--out", tmp_path / "rec2") == 0
    for f in sorted((seq / "rec").iterdir()):
        assert (tmp_path / "rec2" / f.name).read_bytes() == f.read_bytes(), f.name


@pytest.mark.parametrize("k", [1, 3])
def test_resume_from_frame_k_reproduces_the_run(seq, tmp_path, k):
    """Track frames 0..k-1, then resume with all frames: the resumed frames warm-start
    from the frame k-1 checkpoint, and every output equals the uninterrupted run's."""
    part = tmp_path / "frames"
    part.mkdir()
    for stem in _stems(k):
        shutil.copy(seq / "data" / "frames" / f"{stem}.pfm", part)
    args = ["--config", seq / "data" / "config.json", "--template", seq / "data" / "template.ply",
            "--matches", seq / "data" / "matches", "--out", tmp_path / "rec"]
    assert run("track", "--frames", part, *args) == 0
    assert sorted(p.name for p in (tmp_path / "rec").glob("*.ply")) == [f"{s}.ply" for s in _stems(k)]
    # an interrupted frame: outputs without the checkpoint are redone
    (tmp_path / "rec" / f"frame_{k:04d}.ply").write_bytes(b"partial")
    assert run("track", "--resume", "--frames", seq / "data" / "frames", *args) == 0
    for f in sorted((seq / "rec").iterdir()):
        assert (tmp_path / "rec" / f.name).read_bytes() == f.read_bytes(), f.name


def test_corrupt_frame_keeps_earlier_outputs(seq, tmp_path):
    frames = tmp_path / "frames"
    shutil.copytree(seq / "data" / "frames", frames)
    (frames / "frame_0002.pfm").write_bytes(b"Pf\nnot a size\n")
    assert run("track", "--config", seq / "data" / "config.json",
               "--template", seq / "data" / "template.ply", "--frames", frames,
               "--matches", seq / "data" / "matches", "--out", tmp_path / "rec") == 1
    assert (tmp_path / "rec" / "frame_0000.ply").exists()
    assert (tmp_path / "rec" / "frame_0001.ply").exists()
    assert not (tmp_path / "rec" / "frame_0002.ply").exists()
    for s in ("frame_0000", "frame_0001"):
        assert (tmp_path / "rec" / f"{s}.ply").read_bytes() == (seq / "rec" / f"{s}.ply").read_bytes()


def test_without_matches_and_eval(seq, tmp_path, caplog):
    import csv
    import logging

    with caplog.at_level(logging.WARNING, logger="deformtrack"):
        assert run("track", "--config", seq / "data" / "config.json",
                   "--template", seq / "data" / "template.ply", "--frames", seq / "data" / "frames",
                   "--out", tmp_path / "rec") == 0
    assert "depth and rigidity terms only" in caplog.text
    assert not list((tmp_path / "rec").glob("*.matches.json"))
    assert run("eval", "--recovered", seq / "rec", "--truth", seq / "data" / "truth",
               "--out", tmp_path / "m.csv") == 0
    rows = list(csv.DictReader((tmp_path / "m.csv").open()))
    assert [r["frame"] for r in rows] == _stems() + ["aggregate"]
    assert all(float(r["rmse_mm"]) < 2.0 for r in rows)


def test_preselect_command(seq, tmp_path):
    from paper_2007_08576_b200 import fileio

    assert run("preselect", "--matches", seq / "data" / "matches" / "frame_0001.json",
               "--out", tmp_path / "p.json") == 0
    d = fileio.read_json(tmp_path / "p.json")
    assert d["n_matches"] == len(d["weights"]) == len(d["preselected"]) > 0
    assert 0 <= d["reference_index"] < d["n_matches"]
