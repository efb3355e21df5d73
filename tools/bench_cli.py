"""The GPU-resident I/O loop end to end: `cli synth` writes a
BASELINE sequence to disk (PFM depth, ascii PLY template, per-frame match JSON), then
`cli track` streams it through the pipelined C-ABI and writes every frame's PLY surface,
report and matches JSON and the warps checkpoint. Reports frames/s of the whole loop
(file parsing, device work, output writing) after a warm-up run, and how many output
bytes one frame writes. Output: one JSON object (--json FILE).

    python tools/bench_cli.py [--config-id 2] [--n-frames 40] [--json profiles/r02_cli.json]
"""

from __future__ import annotations

import argparse
import json
import shutil
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config-id", type=int, default=2)
    ap.add_argument("--n-frames", type=int, default=40)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    from paper_2007_08576_b200 import cli

    tmp = Path(tempfile.mkdtemp(prefix="dt_cli_"))
    try:
        data = tmp / "data"
        assert cli.main(["synth", "--config-id", str(args.config_id), "--n-frames",
                         str(args.n_frames), "--out", str(data)]) == 0
        tpl = next(data.glob("*.ply"))
        frames = data / "frames" if (data / "frames").is_dir() else data
        matches = data / "matches" if (data / "matches").is_dir() else None
        base = ["track", "--template", str(tpl), "--frames", str(frames)]
        if matches is not None:
            base += ["--matches", str(matches)]
        cfg = next(iter(sorted(data.glob("*.json"))), None)
        if cfg is not None and "config" in cfg.name:
            base += ["--config", str(cfg)]
        runs = []
        for r in range(2):  # the first run warms the library / JIT of the readers
            out = tmp / f"out{r}"
            t = time.perf_counter()
            rc = cli.main(base + ["--out", str(out)])
            runs.append(time.perf_counter() - t)
            assert rc == 0, rc
        n_out = sum(1 for p in out.iterdir() if p.is_file())
        size = sum(p.stat().st_size for p in out.iterdir() if p.is_file())
        res = {"config_id": args.config_id, "frames": args.n_frames,
               "wall_s": runs[-1], "frames_per_s": args.n_frames / runs[-1],
               "first_run_wall_s": runs[0], "output_files": n_out,
               "output_bytes_per_frame": size / args.n_frames,
               "inputs": sorted(p.name for p in data.iterdir())[:6]}
        print(json.dumps(res))
        if args.json:
            Path(args.json).write_text(json.dumps(res, indent=1))
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
