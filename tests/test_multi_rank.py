"""N>1 host logic on CPU (gloo, world_size 2): the path shards by independent
triplets with no data-path collective; the only cross-rank traffic is the timing barrier and
the max-over-ranks of the device time.  The device kernels themselves are covered by the
single-GPU tests (each rank runs the same single-GPU forward on its own slice)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, str(ROOT))
    import bench

    bench.barrier(world)
    t = bench.max_over_ranks(0.25 + rank, world)  # per-rank device time -> job time
    # each rank's shard of the synthetic workload: global sequence indices rank*B + i
    batch = bench.CONFIGS["c2"][0]
    first = rank * batch
    shards = [None] * world
    dist.all_gather_object(shards, (first, first + batch))
    out[rank] = (t, shards)
    dist.destroy_process_group()


def test_max_over_ranks_and_disjoint_shards_gloo():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        t, shards = out[r]
        assert t == pytest.approx(1.25)  # max over ranks, identical on every rank
        # the shards tile the global sequence range with no overlap: no collective needed
        assert sorted(shards) == [(0, 64), (64, 128)]


@pytest.mark.parametrize("config", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_bench_shards_tile_the_job(config, world):
    """bench.shard: every rank's slice is contiguous, slices are disjoint and cover the job
    (weak configs: world x the config batch; strong configs: the config's fixed total)."""
    sys.path.insert(0, str(ROOT))
    import bench
    got = [bench.shard(config, world, r) for r in range(world)]
    total = got[0][2]
    strong = config in ("c3", "c4", "c5")
    assert all(g[3] == strong and g[2] == total for g in got)
    assert total == bench.CONFIGS[config][0] * (1 if strong else world)
    pos = 0
    for first, count, _, _ in got:
        assert first == pos and count >= 0
        pos += count
    assert pos == total


def test_reference_arm_under_torchrun_prints_once():
    """`bench.py --impl reference` launched like the driver's N>1 run: rank 0 alone times
    the CPU reference and prints one JSON line, the other rank exits 0 without work."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--config", "c1",
           "--steps", "1", "--warmup", "1"]
    env = dict(os.environ, OMP_NUM_THREADS="2", CUDA_VISIBLE_DEVICES="")
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2
    assert rec["value"] > 0 and rec["e2e"]["h2d_bytes_per_step"] == 0
    assert rec["cpu_baseline"]["kind"] == "port"
