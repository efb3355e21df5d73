#!/usr/bin/env python
"""Benchmark: per-frame deformation tracking on B200 (BASELINE.json metric, config 2).

Workload (config 2): synthetic ex-vivo-like sphere patch, 640x480 depth, 141x141 = 19,881
template points, 404 densely connected control points (radius 5.2; the metric names 400),
2,000 template ORB features (+500 distractors, 10 % outliers), exhaustive 1-point-RANSAC +
reweighting preselection, 10 Levenberg-Marquardt outer iterations per frame (step_tol =
cost_tol = 0, so every frame runs exactly 10). One step = one frame of the whole hot path:
raw depth -> normals -> Hamming ORB matching -> preselection -> LM solve -> output warp.

  value  frames/s with the frame inputs already resident in HBM, device-timed with CUDA
         events on the tracker stream around each frame (L2 flushed between frames by a
         160 MiB write, outside the timed events); summed over K frames.
  e2e    frames/s through the pipelined C-ABI (dt_track_frame_submit / dt_tracker_wait)
         with pinned HOST buffers: every step copies its depth + descriptors + keypoints in
         and warps + warped points + normals out (overlapping the neighbouring frames'
         compute), with an L2 flush before every frame inside the timed wall clock.
  config5  BASELINE config 5: 64 independent config-2 sequences sharded 64/N over the
         GPUs (one tracker + stream per sequence), aggregate frames/s (`--workload
         config5` makes it the headline).
  --impl reference   the reference algorithm on the host cores: the oracle port
         (oracle/, C kernels bit-identical to the reference's numba kernels + the
         reference's numpy preselection restated), same workload, config, steps and
         warm-up; it never loads the CUDA library.

Multi-GPU: frames of one sequence are sequentially dependent (warm start), so the path
does not shard: each rank tracks its own independent sequence (replicas only,
SURVEY.md §8e); value = all ranks' frames / max-over-ranks device time. `--gpus N`
without torchrun relaunches itself under torch.distributed.run with N ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tracking frames/sec (Hz) at 640x480, 400 ctrl pts, 10 GN iters; ms/GN iteration"
UNIT = "frames/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--frames", type=int, default=20, help="distinct frames generated (cycled)")
    ap.add_argument("--cluster", type=int, default=0, help="solver cluster size (0 = max)")
    ap.add_argument("--cpu-frames", type=int, default=3, help="CPU-baseline sample (frames)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-config5", action="store_true", help="skip the config-5 object")
    ap.add_argument("--workload", choices=["config2", "config5"], default="config2",
                    help="headline line: one config-2 sequence per GPU (default) or config 5")
    ap.add_argument("--c5-rounds", type=int, default=8, help="config-5 frames per sequence")
    ap.add_argument("--c5-cluster", type=int, default=8,
                    help="config-5 solver cluster size (8 measured ~1 % above 4, 16 below)")
    return ap.parse_args()


# ---------------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------------


def host_prepare_template(tpl0, cfg):
    """The reference's template build on the host (oracle restatement of the greedy
    thinning + dense connections, kd-tree binding): the host-reference arm touches none of
    the device code, not even at setup."""
    from oracle import pipeline as OP
    from paper_2007_08576_b200.warpfield import ControlGraph, bind_template

    r = cfg.sampling.radius
    ctrl = OP.sample_controls(tpl0.points, r)
    edges, ew = OP.connections(ctrl, cfg.sampling.effective_connection_sigma)
    warps = np.zeros((len(ctrl), 8))
    warps[:, 0] = 1.0
    graph = ControlGraph(ctrl, warps, edges, ew, sampling_radius=r)
    return bind_template(tpl0, graph, k=cfg.sampling.bind_k,
                         sigma=cfg.sampling.effective_bind_sigma), graph


def make_workload(config_id: int, n_frames: int, seed: int, host_template: bool = False):
    from dataclasses import replace

    from paper_2007_08576_b200 import synth
    from paper_2007_08576_b200.config import load_config
    from paper_2007_08576_b200.tracking import prepare_template

    spec = synth.CONFIGS[config_id]
    scene = replace(spec["scene"], seed=seed)
    cfg = load_config({
        "sampling": {"radius": spec["radius"]},
        "solver": {"max_outer_iters": spec["iters"], "step_tol": 0.0, "cost_tol": 0.0},
    })
    cam = synth.camera_for(scene)
    tpl0 = synth.make_template(scene)
    feats = synth.make_features(scene, tpl0)
    frames = [synth.make_frame(scene, cam, tpl0, feats, f) for f in range(1, n_frames + 1)]
    tpl, graph = host_prepare_template(tpl0, cfg) if host_template else prepare_template(tpl0, cfg)
    return dict(scene=scene, cfg=cfg, cam=cam, tpl=tpl, graph=graph, feats=feats, frames=frames,
                iters=spec["iters"], radius=spec["radius"], config_id=config_id)


DATA = "synthetic (builder sphere-patch generator, seeded; random 256-bit descriptors)"


def workload_config(wl, n_gpus):
    """The `config` object of both arms (identical for the same workload and N)."""
    tpl, graph, sc = wl["tpl"], wl["graph"], wl["scene"]
    return {
        "workload": f"config {wl['config_id']}: synthetic {sc.surface} {sc.width}x{sc.height}, "
                    f"{len(tpl)} template points, {len(graph)} control points, "
                    f"{graph.edges.shape[0]} dense connections, {sc.n_features} ORB features "
                    f"(+{sc.n_distractors} distractors, {int(sc.outlier_fraction * 100)}% outliers), "
                    f"exhaustive preselection, {wl['iters']} LM iterations/frame; one independent "
                    f"sequence per GPU (config 5, 64 sequences sharded 64/N per GPU, is the "
                    f"`config5` object)",
        "template_points": len(tpl),
        "control_points": len(graph),
        "edges": int(graph.edges.shape[0]),
        "orb_features": sc.n_features,
        "image": [sc.width, sc.height],
        "lm_iterations": wl["iters"],
        "preselection": "exhaustive",
        "frames": f"{len(wl['frames'])} distinct frames cycled",
        "l2": "flushed between timed frames (160 MiB write > 126 MB L2; outside the device-timed events, inside the e2e wall clock)",
        "parallelism": f"replicas x{n_gpus} (independent sequences, no collective)",
    }


# ---------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms DURING the timed region
    (one streaming `nvidia-smi -lms` child, stopped by its own PID)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None
        self._t = None

    def _read(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)  # first sample lands before the timed region starts
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            time.sleep(0.1)
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def max_over_ranks(x: float, world: int, device=None) -> float:
    """Max of a per-rank time over all ranks (all_reduce MAX; identity at world 1)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(frames_per_rank: int, world: int, max_ms: float) -> float:
    """Whole-job frames/s of `world` independent replicas timed to the slowest rank."""
    return world * frames_per_rank / (max_ms / 1e3)


# ---------------------------------------------------------------------------------
FP64_PEAK_TFLOPS = 34.4  # DFMA, measured on this pool's B200 with tools/fp64_probe.cu (profiles/r02_fp64_probe.txt)

# algorithmic bytes for the roofline of the LM solver kernel
# ---------------------------------------------------------------------------------


def solver_algorithmic_bytes(n, m, e, k, n_valid, n_active, report):
    """Bytes one k_solve_frame launch must touch at minimum, by the §8d per-unit table:
    relink 100 B/point (p, n, binding, depth + obs-normal gather, writes); linearization
    68 B/valid correspondence + 60 B/match + 232 B/control; rigidity pass 16 B/edge +
    312 B/control; damped solve 328 B/control/attempt; tentative value pass
    64 B/valid correspondence + 60 B/match + 16 B/edge + 96 B/control; the output warp
    folded into its final phase 80 B/point (p, n, binding in; warped p, n out)."""
    it = int(report.outer_iterations)
    attempts = int(report.accepted_steps) + int(report.rejected_steps) + int(report.converged)
    relinks = it + 1
    lin = it * (n_valid * 68 + n_active * 60 + m * 29 * 8)
    arap = it * (e * 16 + m * 88 + m * 28 * 8)
    solves = attempts * m * (27 * 8 + 64 + 48)
    value = (attempts + 1) * (n_valid * 64 + n_active * 60 + e * 16 + m * 96)
    return relinks * n * 100 + lin + arap + solves + value + n * 80


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------------


def run_b200(args, rank, world, local_rank):
    import ctypes as C

    import torch

    torch.cuda.set_device(local_rank)
    if not (ROOT / "paper_2007_08576_b200" / "libdeformtrack_b200.so").exists():
        import __graft_entry__

        __graft_entry__.build()
    from paper_2007_08576_b200._lib import FrameInput, FrameOutput, Report
    from paper_2007_08576_b200._session import DeviceTracker, make_config

    wl = make_workload(args.config, args.frames, seed=rank)
    cfg = wl["cfg"]
    stream = torch.cuda.Stream()
    dcfg = make_config(wl["cam"], cfg.energy, cfg.make_solver_config(), cfg.make_preselect_config(),
                       sampling_radius=wl["graph"].sampling_radius, cluster_size=args.cluster)
    trk = DeviceTracker(wl["tpl"], wl["graph"], dcfg, stream=stream.cuda_stream)
    from paper_2007_08576_b200.warpfield import bind_points

    feats = wl["feats"]
    binding = bind_points(feats.points, wl["graph"].points, 4, wl["graph"].sampling_radius)
    trk.set_features(feats.descriptors, feats.points, binding)

    dev = torch.device("cuda", local_rank)
    frames = wl["frames"]
    F = len(frames)
    d_depth = [torch.from_numpy(f.depth).to(dev) for f in frames]
    d_desc = [torch.from_numpy(f.descriptors).to(dev) for f in frames]
    d_kp = [torch.from_numpy(f.keypoints).to(dev) for f in frames]
    # L2 flush buffer: a write larger than the 126 MB L2 (override for diagnostics only)
    flush_mib = int(os.environ.get("DT_BENCH_FLUSH_MIB", "160"))
    flush = torch.empty(max(flush_mib, 1) * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def dev_input(i, fid):
        fi = FrameInput()
        fi.depth = d_depth[i].data_ptr()
        fi.frame_desc = d_desc[i].data_ptr()
        fi.frame_kp = d_kp[i].data_ptr()
        fi.n_frame = int(d_desc[i].shape[0])
        fi.use_matches = 1
        fi.on_device = 1
        fi.frame_id = fid
        fi.height, fi.width = d_depth[i].shape[0], d_depth[i].shape[1]
        return fi

    # ---- warm-up ----
    trk.set_warps(wl["graph"].warps)
    with torch.cuda.stream(stream):
        for w in range(args.warmup):
            trk.enqueue(dev_input(w % F, w))
    stream.synchronize()

    # ---- timed: device-resident inputs ----
    K = args.steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches = 0
    with ClockSampler(local_rank) as clocks:
        with torch.cuda.stream(stream):
            for i in range(K):
                fi_idx = (args.warmup + i) % F
                flush.zero_()
                starts[i].record(stream)
                trk.enqueue(dev_input(fi_idx, args.warmup + i))
                ends[i].record(stream)
                launches += trk.launches()
        stream.synchronize()
    torch.cuda.synchronize()
    per_frame_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = max_over_ranks(float(sum(per_frame_ms)), world, dev)

    # report of the last timed frame (outputs resident on the device)
    rep = Report()
    fo = FrameOutput()
    fo.report = C.cast(C.pointer(rep), C.c_void_p).value
    trk.collect(dev_input((args.warmup + K - 1) % F, 0), fo)

    # ---- per-phase device time (CUDA events between the pipeline stages) ----
    trk.set_profiling(True)
    phases = []
    with torch.cuda.stream(stream):
        for i in range(min(10, K)):
            flush.zero_()
            trk.enqueue(dev_input((args.warmup + K + i) % F, 0))
            phases.append(trk.phase_ms())
    trk.set_profiling(False)
    phase_avg = {k: float(np.mean([p[k] for p in phases])) for k in phases[0]}

    # ---- e2e: host buffers through the C-ABI ----
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        h_depth = [pin(f.depth) for f in frames]
        h_desc = [pin(f.descriptors) for f in frames]
        h_kp = [pin(f.keypoints) for f in frames]
        # two output slots: the pipelined API copies frame i's outputs back while frame
        # i + 1 computes
        outs = []
        for _ in range(2):
            o_w = torch.empty((len(wl["graph"]), 8), dtype=torch.float64).pin_memory()
            o_p = torch.empty((len(wl["tpl"]), 3), dtype=torch.float64).pin_memory()
            o_n = torch.empty((len(wl["tpl"]), 3), dtype=torch.float64).pin_memory()
            o_r = Report()
            fo = FrameOutput()
            fo.warps, fo.points, fo.normals = o_w.data_ptr(), o_p.data_ptr(), o_n.data_ptr()
            fo.report = C.cast(C.pointer(o_r), C.c_void_p).value
            outs.append((fo, o_w, o_p, o_n, o_r))
        out_w, out_p, out_n = outs[0][1], outs[0][2], outs[0][3]
        trk.set_warps(wl["graph"].warps)

        def host_input(i, fid):
            fi = FrameInput()
            fi.depth = h_depth[i].data_ptr()
            fi.frame_desc = h_desc[i].data_ptr()
            fi.frame_kp = h_kp[i].data_ptr()
            fi.n_frame = int(h_desc[i].shape[0])
            fi.use_matches = 1
            fi.on_device = 0
            fi.frame_id = fid
            fi.height, fi.width = h_depth[i].shape[0], h_depth[i].shape[1]
            return fi

        trk_stream = torch.cuda.ExternalStream(trk.stream)
        for w in range(args.warmup):
            trk.submit(host_input(w % F, w), outs[w % 2][0])
        trk.sync()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        # steady-state streaming: every step stages its depth + ORB features from pinned
        # host memory, flushes L2 (a 160 MiB write on the tracker stream, inside the
        # timed region) and returns warps + warped points / normals to pinned host memory
        t0 = time.perf_counter()
        for i in range(K):
            with torch.cuda.stream(trk_stream):
                flush.zero_()
            trk.submit(host_input((args.warmup + i) % F, args.warmup + i), outs[i % 2][0])
        trk.sync()
        wall = time.perf_counter() - t0
        wall_ms = max_over_ranks(wall * 1e3, world, dev)
        h2d = frames[0].depth.nbytes + frames[0].descriptors.nbytes + frames[0].keypoints.nbytes
        d2h = out_w.numel() * 8 + out_p.numel() * 8 + out_n.numel() * 8 + C.sizeof(Report)
        e2e = {"value": replica_throughput(K, world, wall_ms), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": wall_ms / K,
               "api": "dt_track_frame_submit / dt_tracker_wait (C-ABI, pipelined: frame i+1's "
                      "copies overlap frame i's compute) via paper_2007_08576_b200._session."
                      "DeviceTracker.submit; L2 flushed before every frame inside the timed region"}

    # ---- roofline of the dominant kernel ----
    n, m = len(wl["tpl"]), len(wl["graph"])
    e = int(wl["graph"].edges.shape[0])
    dominant = max(phase_avg, key=phase_avg.get)
    peak, peak_src = measured_peaks()
    solver_bytes = solver_algorithmic_bytes(n, m, e, 4, int(rep.n_correspondences),
                                            int(rep.n_preselected), rep)
    solver_ms = phase_avg["lm_solver"]
    achieved = solver_bytes / (solver_ms * 1e-3) / 1e9
    traffic = None
    # dram__bytes_read.sum + dram__bytes_write.sum of one `ncu --set full` capture of the
    # same kernel on the same workload (committed under profiles/, newest round first)
    for prof in sorted((ROOT / "profiles").glob("r*_solver_dram.json"), reverse=True):
        traffic = json.loads(prof.read_text()).get("traffic_bytes_per_launch")
        break
    roofline = {"kernel": "k_solve_frame (LM solver, one persistent launch per frame)",
                "bound": "hbm", "achieved": round(achieved, 3), "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": int(solver_bytes),
                "launch_ms": solver_ms, "peak_source": peak_src,
                "dominant_phase": dominant,
                "note": "latency-bound: ~40 dependent phases/frame; see DESIGN.md §4"}

    # the FP64-bound stage beside it: exhaustive preselection, SURVEY.md §8(d)'s
    # 40 flop x hypotheses x (IRLS iterations + support pass) x matches, against the
    # measured DFMA throughput (tools/fp64_probe.cu)
    n_match = int(getattr(rep, "n_matches", 0) or 0)
    pre_ms = phase_avg.get("preselect", 0.0)
    pre_flop = 40.0 * n_match * (wl["cfg"].preselect.n_reweight_iters + 1) * n_match
    roofline_pre = None
    if pre_ms > 0 and n_match > 0:
        ach = pre_flop / (pre_ms * 1e-3) / 1e12
        roofline_pre = {"kernel": "k_preselect_orb (fused ORB match build + preselection + final)",
                        "bound": "fp64",
                        "achieved": round(ach, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": ach / FP64_PEAK_TFLOPS, "algorithmic_flop": pre_flop,
                        "launch_ms": pre_ms,
                        "peak_source": "measured DFMA throughput on B200 (tools/fp64_probe.cu)"}

    value = replica_throughput(K, world, total_ms)
    ms_per_step = total_ms / K
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "ms_per_gn_iteration": ms_per_step / wl["iters"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": workload_config(wl, world),
        "e2e": e2e, "roofline": roofline, "roofline_preselect": roofline_pre,
        "gpu_launches": launches,
        "phase_ms": phase_avg, "clocks": clocks.summary(),
        "frame_report": {"n_correspondences": int(rep.n_correspondences),
                         "n_matches": int(rep.n_matches), "n_preselected": int(rep.n_preselected),
                         "outer_iterations": int(rep.outer_iterations),
                         "accepted_steps": int(rep.accepted_steps),
                         "rejected_steps": int(rep.rejected_steps),
                         "total_cost": float(rep.total_cost)},
        "solver_cluster": int(dcfg.cluster_size) or "auto",
    }
    trk.close()
    if not args.no_config5 or args.workload == "config5":
        result["config5"] = run_config5(wl, rank, world, local_rank, rounds=args.c5_rounds,
                                        cluster=args.c5_cluster)
    if args.workload == "config5":
        # headline = config 5's aggregate (the single-sequence line moves to `config2`)
        c5 = result["config5"]
        single = {k: result[k] for k in ("value", "ms_per_step", "e2e", "config", "scaling")}
        result.update(value=c5["value"], ms_per_step=c5["device_ms_max_over_ranks"] / c5["rounds"],
                      steps=c5["rounds"], scaling="strong", e2e=None, config2=single)
        result["config"] = dict(result["config2"]["config"], workload=c5["workload"])
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(wl, args.cpu_frames)
    return result


# ---------------------------------------------------------------------------------
# config 5: many independent sequences, sharded over the GPUs
# ---------------------------------------------------------------------------------

C5_SEQUENCES = 64


def shard_sequences(n_seq: int, world: int, rank: int) -> list[int]:
    """Sequences of `rank` when n_seq independent sequences are split over `world` GPUs:
    contiguous blocks, sizes differing by at most one (64/N per GPU for N | 64)."""
    return [s for s in range(n_seq) if s * world // n_seq == rank]


def config5_aggregate(n_seq: int, rounds: int, max_ms: float) -> float:
    """Whole-job frames/s of config 5: every sequence's frames over the slowest rank's
    device time (strong scaling: the 64 sequences are split, not replicated)."""
    return n_seq * rounds / (max_ms / 1e3)


def run_config5(wl, rank, world, local_rank, n_seq=C5_SEQUENCES, cluster=8, rounds=8, warmup=2):
    """BASELINE config 5 on this rank: its shard of `n_seq` independent config-2
    sequences, one tracker (own warps, buffers, CUDA stream; solver = one thread-block
    cluster) per sequence, frames enqueued round-robin. Device time = first event to the
    last stream's end event; the aggregate is every rank's frames / the max-over-ranks
    time (no collective on the data path; one all_reduce(MAX) of the time)."""
    import torch

    from paper_2007_08576_b200._lib import FrameInput
    from paper_2007_08576_b200._session import DeviceTracker, make_config
    from paper_2007_08576_b200.warpfield import bind_points

    mine = shard_sequences(n_seq, world, rank)
    cfg, graph, feats = wl["cfg"], wl["graph"], wl["feats"]
    dcfg = make_config(wl["cam"], cfg.energy, cfg.make_solver_config(), cfg.make_preselect_config(),
                       sampling_radius=graph.sampling_radius, cluster_size=cluster)
    binding = bind_points(feats.points, graph.points, 4, graph.sampling_radius)
    dev = torch.device("cuda", local_rank)
    frames = wl["frames"]
    F = len(frames)
    d_depth = [torch.from_numpy(f.depth).to(dev) for f in frames]
    d_desc = [torch.from_numpy(f.descriptors).to(dev) for f in frames]
    d_kp = [torch.from_numpy(f.keypoints).to(dev) for f in frames]
    streams = [torch.cuda.Stream(device=dev) for _ in mine]
    trks = []
    for s in streams:
        t = DeviceTracker(wl["tpl"], graph, dcfg, stream=s.cuda_stream)
        t.set_features(feats.descriptors, feats.points, binding)
        t.set_warps(graph.warps)
        trks.append(t)

    def fin(i, fid):
        fi = FrameInput()
        fi.depth, fi.frame_desc, fi.frame_kp = d_depth[i].data_ptr(), d_desc[i].data_ptr(), d_kp[i].data_ptr()
        fi.n_frame, fi.use_matches, fi.on_device, fi.frame_id = d_desc[i].shape[0], 1, 1, fid
        fi.height, fi.width = d_depth[i].shape[0], d_depth[i].shape[1]
        return fi

    # sequence q starts at its own offset in the frame pool and walks it in order
    for r in range(warmup):
        for q, t in zip(mine, trks):
            t.enqueue(fin((q + r) % F, r))
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    start = torch.cuda.Event(enable_timing=True)
    start.record(torch.cuda.current_stream(dev))
    for s in streams:
        s.wait_event(start)
    launches = 0
    for r in range(rounds):
        for q, t in zip(mine, trks):
            t.enqueue(fin((q + warmup + r) % F, warmup + r))
            launches += t.launches()
    ends = []
    for s in streams:
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        ends.append(e)
    torch.cuda.synchronize(dev)
    my_ms = max((start.elapsed_time(e) for e in ends), default=0.0)
    max_ms = max_over_ranks(my_ms, world, dev)
    for t in trks:
        t.close()
    total = n_seq * rounds
    return {"value": config5_aggregate(n_seq, rounds, max_ms), "unit": UNIT, "n_gpus": world, "scaling": "strong",
            "sequences": n_seq, "sequences_per_gpu": len(mine), "frames": total,
            "rounds": rounds, "warmup_rounds": warmup, "cluster": cluster,
            "device_ms_max_over_ranks": max_ms,
            "per_sequence_hz": rounds / (max_ms / 1e3), "gpu_launches_rank0": launches,
            "workload": f"config 5: {n_seq} independent config-2 sequences sharded "
                        f"{n_seq}/{world} per GPU (contiguous blocks), one tracker + CUDA "
                        f"stream per sequence, solver in {cluster}-CTA clusters; each "
                        f"sequence walks the {F}-frame pool from its own offset; inputs "
                        f"resident in HBM, L2 not flushed (64 trackers' working sets "
                        f"exceed the L2)"}


# ---------------------------------------------------------------------------------
# CPU: the reference algorithm (oracle port) on the host cores
# ---------------------------------------------------------------------------------


def cpu_model() -> str:
    """The host CPU's model name (lscpu's "Model name", read from /proc/cpuinfo)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_frame_runner(wl, n_chunks: int = 8):
    """One frame of the reference algorithm through the oracle port: observation
    normals (correspond.py:87-103), Hamming matching + back-projection, exhaustive
    preselection (matching.py:174-226), 10 LM iterations (solver.py:267-378), output
    warp (tracking.py:87). ``n_chunks`` is the reference's solver.n_chunks (8 keeps the
    reference's bits; max(8, nproc) lets every core work)."""
    from oracle import kernels as OK
    from oracle import pipeline as OP

    tpl, graph, cam = wl["tpl"], wl["graph"], wl["cam"]
    feats = wl["feats"]
    tplt = (tpl.points, tpl.normals, tpl.bind_indices, tpl.bind_weights)
    grt = (graph.points, graph.edges, graph.edge_weights)
    camt = (cam.fx, cam.fy, cam.cx, cam.cy)
    sch = OP.Schedule(max_outer_iters=wl["iters"], step_tol=0.0, cost_tol=0.0, n_chunks=n_chunks)
    state = {"warps": graph.warps.copy()}

    def step(fr):
        normals = OP.observation_normals(fr.depth, *camt)
        src, dst, _ = OP.matches_from_descriptors(feats.descriptors, feats.points,
                                                  fr.descriptors, fr.keypoints, fr.depth, camt)
        res, _, _, _ = OP.track(tplt, grt, state["warps"], fr.depth, normals, camt, (src, dst),
                                OP.Weights(), sch, graph.sampling_radius, refs=None)
        state["warps"] = res.warps
        return res

    return step, OK


def host_stage_timings(wl, n_frames: int) -> dict:
    """Per-frame host times of the two stages BASELINE.md §2 asks for separately: the
    reference's Observation.from_depth normals (correspond.py:87-103, oracle restatement)
    and the builder's numpy Hamming oracle (+ back-projection)."""
    from oracle import pipeline as OP

    cam, feats = wl["cam"], wl["feats"]
    camt = (cam.fx, cam.fy, cam.cx, cam.cy)
    frames = wl["frames"][:max(1, n_frames)]
    t0 = time.perf_counter()
    for fr in frames:
        OP.observation_normals(fr.depth, *camt)
    t1 = time.perf_counter()
    for fr in frames:
        OP.matches_from_descriptors(feats.descriptors, feats.points, fr.descriptors,
                                    fr.keypoints, fr.depth, camt)
    t2 = time.perf_counter()
    return {"from_depth_ms": (t1 - t0) * 1e3 / len(frames),
            "hamming_ms": (t2 - t1) * 1e3 / len(frames), "frames": len(frames)}


def time_oracle(wl, warm: int, steps: int, threads: int, n_chunks: int) -> float:
    """Seconds for `steps` consecutive frames after `warm` warm-up frames."""
    step, OK = oracle_frame_runner(wl, n_chunks=n_chunks)
    OK.set_threads(threads)
    frames = wl["frames"]
    for w in range(warm):
        step(frames[w % len(frames)])
    t0 = time.perf_counter()
    for i in range(steps):
        step(frames[(warm + i) % len(frames)])
    return time.perf_counter() - t0


def cpu_baseline(wl, n_frames):
    """The b200 arm's reported CPU baseline (rank 0, N=1): a bounded sample of the same
    workload through the oracle port, at nproc threads (the headline) and at 1 thread,
    plus the separate from_depth / Hamming stage times."""
    cores = os.cpu_count() or 1
    dt = time_oracle(wl, 1, n_frames, cores, max(8, cores))
    dt1 = time_oracle(wl, 1, 1, 1, 8)
    return {"value": n_frames / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{n_frames} consecutive config-2 frames after 1 warm-up (full path: "
                      f"normals, Hamming, exhaustive preselection, {wl['iters']} LM iterations, "
                      f"output warp) through the oracle port (C kernels bit-identical to the "
                      f"reference's numba kernels, OpenMP over solver.n_chunks = "
                      f"{max(8, cores)}, + the reference's single-threaded numpy "
                      f"preselection restated)",
            "ms_per_frame": dt * 1e3 / n_frames,
            "threads_1": {"value": 1 / dt1, "ms_per_frame": dt1 * 1e3, "frames": 1},
            "stages": host_stage_timings(wl, 3),
            "cpu_model": cpu_model()}


# The reference arm runs the whole frame on the host cores (~1.5 s per config-2 frame on
# 16 cores), so it is bounded: at most REF_MAX_FRAMES timed frames (the driver's
# --steps 20 --warmup 5 runs unbounded: same steps, same warm-up as the b200 arm).
REF_MAX_FRAMES = 60
REF_MAX_WARMUP = 10


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host cores through the oracle
    port, never touching the CUDA library (the package is imported for its config
    objects and the numpy scene generator only; the template build is the oracle's)."""
    if rank != 0:
        return None  # replicas are independent: rank 0 alone times the host reference
    wl = make_workload(args.config, args.frames, seed=0, host_template=True)
    cores = os.cpu_count() or 1
    warm = min(args.warmup, REF_MAX_WARMUP)
    steps = max(1, min(args.steps, REF_MAX_FRAMES))
    dt = time_oracle(wl, warm, steps, cores, max(8, cores))
    value = steps / dt
    dt1 = time_oracle(wl, 1, 2, 1, 8)
    stages = host_stage_timings(wl, 3)
    sample = (f"{steps} consecutive config-{args.config} frames after {warm} warm-up, one "
              f"full frame per step (normals, Hamming, exhaustive preselection, "
              f"{wl['iters']} LM iterations, warp), oracle port of the reference on {cores} "
              f"host threads (solver.n_chunks = {max(8, cores)})")
    from paper_2007_08576_b200 import _lib

    assert not _lib.loaded(), "the reference arm must not load the CUDA library"
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": dt * 1e3 / steps,
        "ms_per_gn_iteration": dt * 1e3 / steps / wl["iters"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": workload_config(wl, world),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model(),
                         "threads_1": {"value": 2 / dt1, "ms_per_frame": dt1 * 1e3 / 2,
                                       "frames": 2},
                         "stages": stages},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def relaunch_distributed(n: int) -> int:
    """`bench.py --gpus N` started without torchrun: launch N ranks (one process per GPU)
    through torch.distributed.run on 127.0.0.1 and return their exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl")
    res = run_b200(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch

        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
