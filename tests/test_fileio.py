"""File formats (the reference's fileio.py:23-259 and its
tests/test_fileio.py): byte-for-byte against files the REFERENCE's writers produced
(tests/golden/fileio/, tests/golden/make_fileio_golden.py), plus the reference test
suite's round-trip and error cases, and the warp checkpoint. CPU only: the codecs are
host code of the library (no device call)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2007_08576_b200 import fileio  # noqa: E402
from paper_2007_08576_b200.exceptions import FileFormatError  # noqa: E402
from paper_2007_08576_b200.matching import MatchSet  # noqa: E402

GOLD = ROOT / "tests" / "golden" / "fileio"


@pytest.fixture(scope="module")
def src():
    return dict(np.load(GOLD / "fileio_src.npz"))


@pytest.mark.parametrize("name,kw", [("cloud_ascii.ply", {}), ("cloud_binary.ply", {"binary": True})])
def test_ply_bytes_equal_reference_writer(tmp_path, src, name, kw):
    out = tmp_path / name
    fileio.write_ply(out, src["pts"], src["nrm"], **kw)
    assert out.read_bytes() == (GOLD / name).read_bytes()


def test_points_only_and_empty_ply_bytes(tmp_path, src):
    fileio.write_ply(tmp_path / "p.ply", src["pts"])
    assert (tmp_path / "p.ply").read_bytes() == (GOLD / "points_only.ply").read_bytes()
    fileio.write_ply(tmp_path / "e.ply", np.zeros((0, 3)))
    assert (tmp_path / "e.ply").read_bytes() == (GOLD / "empty.ply").read_bytes()


@pytest.mark.parametrize("name", ["cloud_ascii.ply", "cloud_binary.ply"])
def test_ply_reads_reference_files_exactly(src, name):
    p, n = fileio.read_ply(GOLD / name)
    np.testing.assert_array_equal(p, src["pts"])
    np.testing.assert_array_equal(n, src["nrm"])
    assert np.signbit(p[0, 2])  # -0.0 survives


def test_pfm_json_matches_metrics_bytes(tmp_path, src):
    fileio.write_pfm(tmp_path / "d.pfm", src["depth"])
    assert (tmp_path / "d.pfm").read_bytes() == (GOLD / "depth.pfm").read_bytes()
    m = MatchSet(src["m_src"], src["m_dst"], src["m_w"], src["m_f"])
    fileio.write_matches(tmp_path / "m.json", m)
    assert (tmp_path / "m.json").read_bytes() == (GOLD / "matches.json").read_bytes()
    fileio.write_json(tmp_path / "r.json", {"b": 1.5, "a": [1, 2, {"z": 0.1, "y": -3.0}],
                                             "e": 1e-12, "n": None, "t": True})
    assert (tmp_path / "r.json").read_bytes() == (GOLD / "report.json").read_bytes()
    fileio.write_metrics_csv(tmp_path / "m.csv", [
        {"frame": "f0", "rmse_mm": 3.0, "mean_mm": 2.0, "max_mm": 5.0, "std_mm": 1.0},
        {"frame": "f1", "rmse_mm": 0.1, "mean_mm": 4.0, "max_mm": 7e-5, "std_mm": 3.0}])
    assert (tmp_path / "m.csv").read_bytes() == (GOLD / "metrics.csv").read_bytes()


def test_pfm_reads_reference_file_and_payload_is_bottom_up(src):
    d = fileio.read_pfm(GOLD / "depth.pfm")
    want = src["depth"].astype(np.float32).astype(np.float64)
    np.testing.assert_array_equal(np.isnan(d), np.isnan(want))
    np.testing.assert_array_equal(d[~np.isnan(d)], want[~np.isnan(want)])
    payload, big = fileio.read_pfm_payload(GOLD / "depth.pfm")
    assert not big and payload.dtype == np.dtype("<f4")
    np.testing.assert_array_equal(payload[::-1][~np.isnan(want)], want[~np.isnan(want)])


@pytest.mark.parametrize("scale", [1e-9, 1e-3, 1.0, 1e4, 1e15, 1e18, 1e250])
def test_native_repr_matches_python_repr(scale):
    v = np.random.default_rng(int(np.log10(scale) + 400)).standard_normal((300, 6)) * scale
    v[0, :4] = [0.0, -0.0, np.inf, -np.inf]
    text = fileio.format_reals(v).decode()
    assert text == "".join(" ".join(repr(x) for x in row) + "\n" for row in v.tolist())
    back = fileio.parse_reals(text.encode(), v.size).reshape(v.shape)
    np.testing.assert_array_equal(back, v)


# --- the reference test suite's cases (tests/test_fileio.py) ---


@pytest.fixture
def cloud():
    rng = np.random.default_rng(5)
    pts = rng.normal(scale=50.0, size=(40, 3)) + np.array([0.0, 0.0, 300.0])
    n = rng.normal(size=(40, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    return pts, n


@pytest.mark.parametrize("binary", [False, True])
def test_ply_round_trip_exact(tmp_path, cloud, binary):
    pts, n = cloud
    fileio.write_ply(tmp_path / "c.ply", pts, n, binary=binary)
    rp, rn = fileio.read_ply(tmp_path / "c.ply")
    np.testing.assert_array_equal(rp, pts)
    np.testing.assert_array_equal(rn, n)


def test_ply_float32_and_errors(tmp_path, cloud):
    p = tmp_path / "f32.ply"
    p.write_text("ply\nformat ascii 1.0\nelement vertex 2\nproperty float x\nproperty float y\n"
                 "property float z\nend_header\n1 2 3\n4 5 6\n")
    pts, n = fileio.read_ply(p)
    np.testing.assert_array_equal(pts, [[1, 2, 3], [4, 5, 6]])
    assert n is None
    p.write_bytes(b"not a ply at all")
    with pytest.raises(FileFormatError):
        fileio.read_ply(p)
    fileio.write_ply(p, cloud[0], cloud[1], binary=True)
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(FileFormatError, match="bytes"):
        fileio.read_ply(p)
    p.write_text("ply\nformat ascii 1.0\nelement vertex 1\nproperty double x\n"
                 "property double y\nend_header\n1 2\n")
    with pytest.raises(FileFormatError, match="'z'"):
        fileio.read_ply(p)
    p.write_text("ply\nformat ascii 1.0\nelement vertex 2\nproperty double x\n"
                 "property double y\nproperty double z\nend_header\n1 2 3\n4 five 6\n")
    with pytest.raises(FileFormatError):
        fileio.read_ply(p)


def test_pfm_round_trip_layout_and_errors(tmp_path):
    d = np.random.default_rng(2).uniform(250.0, 350.0, size=(17, 23)).astype(np.float32)
    fileio.write_pfm(tmp_path / "d.pfm", d)
    np.testing.assert_array_equal(fileio.read_pfm(tmp_path / "d.pfm"), d.astype(np.float64))
    fileio.write_pfm(tmp_path / "t.pfm", np.array([[1.0, 2.0], [3.0, 4.0]]))
    head, body = (tmp_path / "t.pfm").read_bytes().split(b"-1.0\n", 1)
    assert head == b"Pf\n2 2\n"
    np.testing.assert_array_equal(np.frombuffer(body, "<f4").reshape(2, 2), [[3, 4], [1, 2]])
    (tmp_path / "c.pfm").write_bytes(b"PF\n2 2\n-1.0\n" + b"\x00" * 48)
    with pytest.raises(FileFormatError):
        fileio.read_pfm(tmp_path / "c.pfm")
    (tmp_path / "c.pfm").write_bytes(b"hello")
    with pytest.raises(FileFormatError):
        fileio.read_pfm(tmp_path / "c.pfm")
    # a big-endian (positive scale) file reads the same values
    (tmp_path / "be.pfm").write_bytes(b"Pf\n2 2\n1.0\n" + d[:2, :2][::-1].astype(">f4").tobytes())
    np.testing.assert_array_equal(fileio.read_pfm(tmp_path / "be.pfm"), d[:2, :2].astype(np.float64))


def test_depth_csv_and_dispatch(tmp_path):
    d = np.random.default_rng(3).uniform(200.0, 400.0, size=(9, 11))
    fileio.write_depth_csv(tmp_path / "d.csv", d)
    np.testing.assert_array_equal(fileio.read_depth(tmp_path / "d.csv"), d)
    fileio.write_pfm(tmp_path / "d.pfm", d)
    assert fileio.read_depth(tmp_path / "d.pfm").shape == d.shape
    with pytest.raises(FileFormatError):
        fileio.read_depth(tmp_path / "d.exr")


def test_matches_round_trip_and_errors(tmp_path):
    m = MatchSet(np.arange(12.0).reshape(4, 3), np.arange(12.0, 24.0).reshape(4, 3),
                 np.array([1.0, 0.5, 0.0, 0.25]), np.array([True, True, False, False]))
    p = tmp_path / "m.json"
    fileio.write_matches(p, m)
    b = fileio.read_matches(p)
    for f in ("template_points", "observed_points", "weights", "preselected"):
        np.testing.assert_array_equal(getattr(b, f), getattr(m, f))
    p.write_text('[{"template_point": [0, 0, 0], "observed_point": [1, 1, 1]}]\n')
    b = fileio.read_matches(p)
    assert b.weights.tolist() == [1.0] and b.preselected.tolist() == [False]
    for text, pat in (('[{"template_point": [0, 0, 0]}]\n', "observed_point"),
                      ('[{"template_point": [0, 0], "observed_point": [1, 1, 1]}]\n', r"\[x, y, z\]"),
                      ('{"not": "a list"}\n', "array"), ("[1, 2, 3]\n", "not an object")):
        p.write_text(text)
        with pytest.raises(FileFormatError, match=pat):
            fileio.read_matches(p)
    p.write_text("{broken")
    with pytest.raises(FileFormatError, match="JSON"):
        fileio.read_json(p)


def test_warps_checkpoint_round_trip_is_exact(tmp_path):
    w = np.random.default_rng(4).standard_normal((37, 8))
    w[0, 0] = -0.0
    fileio.write_warps(tmp_path / "f.warps.json", w, "f")
    np.testing.assert_array_equal(fileio.read_warps(tmp_path / "f.warps.json"), w)
    assert not list(tmp_path.glob("*.tmp"))
    (tmp_path / "bad.json").write_text('{"warps": [[1, 2]]}\n')
    with pytest.raises(FileFormatError):
        fileio.read_warps(tmp_path / "bad.json")


def test_native_json_writers_equal_json_dump_byte_for_byte():
    """write_matches / write_warps assemble their text from natively formatted numbers;
    it must be json.dump(..., indent=2, sort_keys=True) byte for byte, on random tables
    spanning every repr notation, with the json fallback for non-finite values."""
    import json
    import tempfile

    import numpy as np

    from paper_2007_08576_b200 import fileio
    from paper_2007_08576_b200.matching import MatchSet

    rng = np.random.default_rng(1)
    special = np.array([0.0, -0.0, 1.0, -1.0, 1e16, 1e17, 1e-5, 1e-4, 123456789.123, 5e-324,
                        1.7e308, -2.5e-310, 0.1, 1 / 3, 2.0**53])

    def dump(path, payload):
        with open(path, "w", encoding="ascii") as fh:
            json.dump(payload, fh, indent=2, sort_keys=True)
            fh.write("\n")

    d = tempfile.mkdtemp()
    for trial in range(25):
        n = int(rng.integers(0, 50))
        a = rng.normal(size=(n, 7)) * 10.0 ** rng.integers(-8, 20, size=(n, 7))
        if n:
            a.flat[rng.integers(0, a.size, size=min(5, a.size))] = rng.choice(special, min(5, a.size))
        if trial == 24 and n:
            a[0, 0] = np.nan
            a[-1, 6] = np.inf
        ms = MatchSet(a[:, :3], a[:, 3:6], a[:, 6], rng.uniform(size=n) > 0.5)
        fileio.write_matches(f"{d}/x.json", ms)
        dump(f"{d}/y.json", [{"template_point": a[i, :3].tolist(), "observed_point": a[i, 3:6].tolist(),
                              "weight": float(a[i, 6]), "preselected": bool(ms.preselected[i])}
                             for i in range(n)])
        assert open(f"{d}/x.json").read() == open(f"{d}/y.json").read(), trial
        m = int(rng.integers(1, 30))
        w = rng.normal(size=(m, 8)) * 10.0 ** rng.integers(-5, 18, size=(m, 8))
        fileio.write_warps(f"{d}/w.json", w, f"frame_{trial:04d}")
        dump(f"{d}/v.json", {"frame": f"frame_{trial:04d}", "warps": w.tolist()})
        assert open(f"{d}/w.json").read() == open(f"{d}/v.json").read(), trial
        np.testing.assert_array_equal(fileio.read_warps(f"{d}/w.json"), w)
