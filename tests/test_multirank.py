"""Multi-process (gloo, world_size 2, CPU) coverage of the replica path of bench.py:
frames of a sequence are sequentially dependent, so N GPUs run N independent
sequences; the whole-job value is all ranks' frames over the
slowest rank's time, and the host-reference arm runs on rank 0 only."""

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        per_rank_ms = [40.0, 55.0][rank]
        mx = bench.max_over_ranks(per_rank_ms, world)
        value = bench.replica_throughput(30, world, mx)

        class Args:
            config, frames, warmup, steps = 2, 2, 1, 1

        ref = bench.run_reference(Args, rank, world) if rank == 1 else "skipped"
        q.put((rank, mx, value, ref))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_replicas_take_the_slowest_rank_and_count_all_frames():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, mx, value, ref = q.get(timeout=120)
        out[rank] = (mx, value, ref)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        mx, value, _ = out[rank]
        assert mx == 55.0  # max over ranks, identical on every rank
        assert value == pytest.approx(2 * 30 / 0.055)
    assert out[1][2] is None  # the host-reference arm does no work off rank 0


def test_single_rank_is_identity():
    import bench

    assert bench.max_over_ranks(12.5, 1) == 12.5
    assert bench.replica_throughput(10, 1, 1000.0) == pytest.approx(10.0)


def _c5_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bench.shard_sequences(bench.C5_SEQUENCES, world, rank)
        got = [None] * world
        dist.all_gather_object(got, mine)
        # a device time per rank that grows with its shard (rank 1 slower)
        ms = 10.0 * len(mine) + 5.0 * rank
        mx = bench.max_over_ranks(ms, world)
        q.put((rank, got, mx, bench.config5_aggregate(bench.C5_SEQUENCES, 8, mx)))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_config5_shards_cover_every_sequence_once_and_time_the_slowest_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, got, mx, agg = q.get(timeout=120)
        out[rank] = (got, mx, agg)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        got, mx, agg = out[rank]
        assert got[0] == list(range(0, 32)) and got[1] == list(range(32, 64))
        assert mx == 10.0 * 32 + 5.0
        assert agg == pytest.approx(64 * 8 / (mx / 1e3))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_sequences_partition(world):
    import bench

    shards = [bench.shard_sequences(64, world, r) for r in range(world)]
    flat = [s for sh in shards for s in sh]
    assert flat == list(range(64))  # contiguous blocks in rank order, each sequence once
    sizes = [len(sh) for sh in shards]
    assert max(sizes) - min(sizes) <= 1


def test_bench_gpus_flag_launches_ranks_itself():
    """`bench.py --gpus 2` without torchrun relaunches under torch.distributed.run; the
    host-reference arm runs on rank 0 only and prints exactly one JSON line."""
    import json
    import subprocess

    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus",
                        "2", "--config", "1", "--frames", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 1
