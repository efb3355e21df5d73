"""Command-line pipeline (the reference's deformtrack/cli.py:89-288): track, synth, eval,
preselect -- with the frame loop on the B200.

``track`` streams the depth frames through the device tracker's pipelined C-ABI
(``streaming.StreamingTracker`` -> dt_track_frame_submit / dt_tracker_wait): a reader
thread parses frame k+2's files while frame k+1's inputs are staged and frame k computes,
PFM depth goes to the device as its raw f32 payload (decoded there), and the finished
frame's outputs are written while the next one computes. Outputs per frame, as the
reference writes them (cli.py:124-130): ``<stem>.ply`` (warped points + normals),
``<stem>.report.json`` (report + the effective config, so a report re-runs the exact same
pipeline), ``<stem>.matches.json``; plus ``<stem>.warps.json``, the solved control warps
-- the checkpoint ``--resume`` restarts from (the reference cannot resume).
A failure at frame k leaves frames 0..k-1 complete on disk (cli.py:3-6); exit code 1.

``synth`` writes one of the BASELINE synthetic configurations (this package's own scene
generator, ``synth.py``; the reference's SceneSpec library is out of scope), ``eval``
compares recovered surfaces with the truth, ``preselect`` runs the device 1-point RANSAC
on one match file. Verbosity: DEFORMTRACK_LOG (error|warn|info|debug, default warn).
"""

from __future__ import annotations

import argparse
import logging
import os
import queue
import sys
import threading
from pathlib import Path

import numpy as np

from . import fileio
from .config import RunConfig, load_config
from .exceptions import DeformtrackError, NoValidHypothesis, SizeMismatch

log = logging.getLogger("deformtrack")
_LEVELS = {"error": logging.ERROR, "warn": logging.WARNING, "info": logging.INFO,
           "debug": logging.DEBUG}
_DEPTH_EXT = (".pfm", ".csv")


def _setup_logging() -> None:
    want = os.environ.get("DEFORMTRACK_LOG", "warn").lower()
    level = _LEVELS.get(want, logging.WARNING)
    logging.basicConfig(level=level, format="%(levelname)s %(name)s: %(message)s")
    log.setLevel(level)
    if want not in _LEVELS:
        log.warning("unknown DEFORMTRACK_LOG value %r; using warn", want)


def _run_config(args) -> RunConfig:
    cfg = (load_config(fileio.read_json(args.config), where=str(args.config))
           if getattr(args, "config", None) is not None else RunConfig())
    if args.threads is not None:
        cfg.threads = args.threads
    if args.seed is not None:
        cfg.seed = args.seed
    return cfg


def _camera(cfg: RunConfig):
    from .geometry import PinholeCamera

    c = cfg.camera
    return PinholeCamera(c.fx, c.fy, c.cx, c.cy, c.width, c.height)


def _frames(frames_dir: Path) -> list[Path]:
    if not frames_dir.is_dir():
        raise FileNotFoundError(f"frames directory {frames_dir} does not exist")
    files = sorted(p for p in frames_dir.iterdir() if p.suffix.lower() in _DEPTH_EXT)
    if not files:
        raise DeformtrackError(f"no depth frames (*.pfm or *.csv) in {frames_dir}")
    return files


def _outputs_complete(out: Path, stem: str) -> bool:
    return all((out / f"{stem}{suffix}").exists()
               for suffix in (".ply", ".report.json", ".warps.json"))


class _Reader(threading.Thread):
    """Parses frame files ahead of the device (bounded queue): PFM -> raw payload,
    CSV -> f64 depth, plus the frame's match JSON. An error is delivered in order, so
    the frames before it are still tracked and written."""

    def __init__(self, files, matches_dir, start: int, depth_bound: int = 3):
        super().__init__(daemon=True)
        self.files, self.mdir, self.start_at = files, matches_dir, start
        self.q: queue.Queue = queue.Queue(maxsize=depth_bound)
        self._stop = threading.Event()

    def run(self) -> None:
        for k in range(self.start_at, len(self.files)):
            if self._stop.is_set():
                return
            path = self.files[k]
            try:
                if path.suffix.lower() == ".pfm":
                    payload, big = fileio.read_pfm_payload(path)
                    depth = None
                    if big:  # the device decodes little-endian payloads
                        depth, payload = payload[::-1].astype(np.float64), None
                else:
                    depth, payload = fileio.read_depth_csv(path), None
                matches, missing = None, False
                if self.mdir is not None:
                    mp = Path(self.mdir) / f"{path.stem}.json"
                    if mp.exists():
                        matches = fileio.read_matches(mp)
                    else:
                        missing = True
                self.q.put((k, path, depth, payload, matches, missing, None))
            except Exception as exc:  # noqa: BLE001 (re-raised in frame order)
                self.q.put((k, path, None, None, None, False, exc))
                return
        self.q.put(None)

    def stop(self) -> None:
        self._stop.set()


def _write_frame(out: Path, stem: str, result, config_echo: dict) -> None:
    fileio.write_ply(out / f"{stem}.ply", result.points, result.normals)
    fileio.write_json(out / f"{stem}.report.json",
                      {"report": result.report.to_dict(), "config": config_echo})
    if result.matches is not None:
        fileio.write_matches(out / f"{stem}.matches.json", result.matches)
    # the checkpoint last: its presence marks the frame complete (--resume)
    fileio.write_warps(out / f"{stem}.warps.json", result.graph.warps, stem)
    for msg in result.report.warnings:
        log.warning("frame %s: %s", stem, msg)
    log.info("frame %s: %d correspondences, total cost %.6g, converged=%s", stem,
             result.report.n_correspondences, result.report.total_cost, result.report.converged)


def _cmd_track(args) -> int:
    from .correspond import estimate_point_normals
    from .streaming import StreamingTracker
    from .tracking import prepare_template
    from .warpfield import Template

    cfg = _run_config(args)
    camera = _camera(cfg)
    points, normals = fileio.read_ply(args.template)
    if normals is None:
        log.warning("%s carries no normals; estimating them from the points", args.template)
        normals = estimate_point_normals(points)
    files = _frames(args.frames)
    if args.matches is None:
        log.warning("no --matches directory; tracking with depth and rigidity terms only")
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    tpl, graph = prepare_template(Template(points, normals), cfg)
    log.info("template: %d points, %d control points", len(points), len(graph))
    echo = cfg.to_dict()

    start = 0
    warm = None
    if args.resume:
        while start < len(files) and _outputs_complete(out, files[start].stem):
            start += 1
        if start > 0:
            warm = fileio.read_warps(out / f"{files[start - 1].stem}.warps.json")
            if warm.shape != graph.warps.shape:
                raise DeformtrackError(
                    f"checkpoint {files[start - 1].stem}.warps.json holds {warm.shape[0]} warps, "
                    f"the template's control graph {len(graph)}")
            log.info("resuming after frame %s (%d of %d done)", files[start - 1].stem, start,
                     len(files))
        if start == len(files):
            return 0

    n_cap = 4096
    if args.matches is not None:
        for f in files[start:start + 1]:
            mp = Path(args.matches) / f"{f.stem}.json"
            if mp.exists():
                n_cap = max(n_cap, 2 * len(fileio.read_matches(mp)))
    trk = StreamingTracker(tpl, graph, camera, cfg, max_matches=n_cap)
    if warm is not None:
        trk.reset(warm)
    reader = _Reader(files, args.matches, start)
    reader.start()
    pending: list[str] = []
    try:
        while True:
            item = reader.q.get()
            if item is None:
                break
            k, path, depth, payload, matches, missing, err = item
            if err is not None:
                # the frames already submitted are still finished and written
                while pending:
                    _write_frame(out, pending.pop(0), trk.wait(), echo)
                raise err
            if missing:
                log.warning("no match file for frame %s; feature term dropped", path.stem)
            if matches is not None and len(matches) > n_cap:
                raise DeformtrackError(f"{path.stem}: {len(matches)} matches exceed {n_cap}")
            if trk.in_flight == 2:
                _write_frame(out, pending.pop(0), trk.wait(), echo)
            trk.submit(depth, matches, pfm_payload=payload, frame_id=k)
            pending.append(path.stem)
        while pending:
            _write_frame(out, pending.pop(0), trk.wait(), echo)
    finally:
        reader.stop()
        trk.close()
    return 0


def _cmd_synth(args) -> int:
    from dataclasses import asdict, replace

    from . import synth

    if args.config_id not in synth.CONFIGS:
        raise DeformtrackError(f"unknown synthetic configuration {args.config_id}")
    spec = synth.CONFIGS[args.config_id]
    scene = spec["scene"]
    if args.seed is not None:
        scene = replace(scene, seed=args.seed)
    cam = synth.camera_for(scene)
    tpl = synth.make_template(scene)
    feats = synth.make_features(scene, tpl)
    out = Path(args.out)
    for sub in ("frames", "matches", "truth"):
        (out / sub).mkdir(parents=True, exist_ok=True)
    fileio.write_ply(out / "template.ply", tpl.points, tpl.normals)
    fileio.write_json(out / "scene.json", {
        "config_id": args.config_id, "n_frames": args.n_frames, "radius": spec["radius"],
        "iterations": spec["iters"], "scene": {k: (list(v) if isinstance(v, tuple) else v)
                                               for k, v in asdict(scene).items()},
        "camera": {"fx": cam.fx, "fy": cam.fy, "cx": cam.cx, "cy": cam.cy,
                   "width": cam.width, "height": cam.height}})
    # a run configuration matching the scene (camera, sampling radius, iterations) for
    # `track --config`
    fileio.write_json(out / "config.json", load_config({
        "camera": {"fx": cam.fx, "fy": cam.fy, "cx": cam.cx, "cy": cam.cy,
                   "width": cam.width, "height": cam.height},
        "sampling": {"radius": spec["radius"]},
        "solver": {"max_outer_iters": spec["iters"]}}).to_dict())
    for f in range(args.n_frames):
        fr = synth.make_frame(scene, cam, tpl, feats, f)
        stem = f"frame_{f:04d}"
        fileio.write_pfm(out / "frames" / f"{stem}.pfm", fr.depth)
        fileio.write_matches(out / "matches" / f"{stem}.json", fr.matches())
        fileio.write_ply(out / "truth" / f"{stem}.ply", fr.truth)
    log.info("wrote %d frames to %s", args.n_frames, out)
    return 0


def _metrics(rec: np.ndarray, truth: np.ndarray) -> dict:
    """Point-to-point distance statistics of index-aligned surfaces (synth.py:396-413)."""
    if rec.shape != truth.shape:
        raise SizeMismatch(f"recovered {rec.shape} vs ground truth {truth.shape}")
    if rec.shape[0] == 0:
        return {"rmse_mm": 0.0, "mean_mm": 0.0, "max_mm": 0.0, "std_mm": 0.0}
    d = np.linalg.norm(rec - truth, axis=1)
    return {"rmse_mm": float(np.sqrt(np.mean(d * d))), "mean_mm": float(np.mean(d)),
            "max_mm": float(np.max(d)), "std_mm": float(np.std(d))}


def _cmd_eval(args) -> int:
    rec = sorted(Path(args.recovered).glob("*.ply"))
    tru = sorted(Path(args.truth).glob("*.ply"))
    if not rec or not tru:
        raise DeformtrackError(f"no surfaces to compare ({len(rec)} recovered, {len(tru)} truth)")
    if len(rec) != len(tru):
        raise SizeMismatch(f"{len(rec)} recovered frames vs {len(tru)} truth frames")
    rows = []
    for a, b in zip(rec, tru):
        pa, _ = fileio.read_ply(a)
        pb, _ = fileio.read_ply(b)
        rows.append({"frame": a.stem, **_metrics(pa, pb)})
        log.info("%s: rmse %.4f mm", a.stem, rows[-1]["rmse_mm"])
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    fileio.write_metrics_csv(args.out, rows)
    return 0


def _cmd_preselect(args) -> int:
    from .matching import preselect_inliers

    cfg = _run_config(args)
    matches = fileio.read_matches(args.matches)
    payload: dict = {"n_matches": len(matches)}
    if len(matches) == 0:
        log.warning("%s holds no matches; writing an empty result", args.matches)
        payload.update({"weights": [], "preselected": [], "warning": "no matches"})
    else:
        try:
            res = preselect_inliers(matches, cfg.make_preselect_config())
            payload.update({"weights": res.matches.weights.tolist(),
                            "preselected": res.matches.preselected.tolist(),
                            "rotation": np.asarray(res.rotation).tolist(),
                            "reference_index": int(res.reference_index),
                            "support": float(res.support)})
        except NoValidHypothesis as exc:
            log.warning("preselection failed: %s", exc)
            payload.update({"weights": [0.0] * len(matches), "preselected": [False] * len(matches),
                            "warning": f"no valid hypothesis ({exc}); weights zeroed"})
    fileio.write_json(args.out, payload)
    return 0


def build_parser() -> argparse.ArgumentParser:
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--threads", type=int, default=None, help="override config thread count")
    common.add_argument("--seed", type=int, default=None, help="override config seed")
    ap = argparse.ArgumentParser(prog="deformtrack-b200",
                                 description="Track a deforming surface through depth frames on a B200.")
    sub = ap.add_subparsers(dest="command", required=True)
    tr = sub.add_parser("track", parents=[common], help="track a template through depth frames")
    tr.add_argument("--config", type=Path, default=None, help="run configuration JSON")
    tr.add_argument("--template", type=Path, required=True, help="reference surface PLY")
    tr.add_argument("--frames", type=Path, required=True, help="directory of depth maps (.pfm/.csv)")
    tr.add_argument("--matches", type=Path, default=None, help="directory of per-frame match JSON")
    tr.add_argument("--out", type=Path, required=True, help="output directory")
    tr.add_argument("--resume", action="store_true",
                    help="skip the frames already complete in --out and warm-start from the "
                         "last one's warps checkpoint")
    tr.set_defaults(func=_cmd_track)
    sy = sub.add_parser("synth", parents=[common], help="write a BASELINE synthetic sequence")
    sy.add_argument("--config-id", type=int, default=1, help="BASELINE configuration (1-4)")
    sy.add_argument("--n-frames", type=int, default=4)
    sy.add_argument("--out", type=Path, required=True)
    sy.set_defaults(func=_cmd_synth)
    ev = sub.add_parser("eval", parents=[common], help="compare recovered surfaces with truth")
    ev.add_argument("--recovered", type=Path, required=True)
    ev.add_argument("--truth", type=Path, required=True)
    ev.add_argument("--out", type=Path, required=True, help="metrics CSV path")
    ev.set_defaults(func=_cmd_eval)
    ps = sub.add_parser("preselect", parents=[common], help="match preselection alone")
    ps.add_argument("--matches", type=Path, required=True)
    ps.add_argument("--config", type=Path, default=None)
    ps.add_argument("--out", type=Path, required=True)
    ps.set_defaults(func=_cmd_preselect)
    return ap


def main(argv: list[str] | None = None) -> int:
    _setup_logging()
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (DeformtrackError, OSError, ValueError) as exc:
        log.error("%s", exc)
        return 1


if __name__ == "__main__":
    sys.exit(main())
