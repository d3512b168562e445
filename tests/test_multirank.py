"""Multi-rank host logic on CPU (gloo, world_size 2, 127.0.0.1): the path
shards by image, so each rank generates and senses a disjoint slice of one global
seeded dataset and the only cross-rank operation is the max-over-ranks timing."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, per_rank, out_dir):
    import torch.distributed as dist

    import bench
    import paper_2001_09632_b200 as p
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first, n = bench.shard(rank, per_rank)
        spec = p.SynthSpec(64, 96, 6, 5.0, 9)
        imgs = p.synth_images_host(spec, first, n)            # this rank's slice, generated locally
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), imgs)
        t = 0.25 + rank                                        # per-rank "device time"
        t_max = bench.max_over_ranks(t, world)
        np.save(os.path.join(out_dir, f"tmax{rank}.npy"), np.array([t_max, first, n]))
        bench.barrier(world)
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_and_timing(tmp_path):
    import torch.multiprocessing as mp

    import bench
    import paper_2001_09632_b200 as p
    world, per_rank = 2, 3
    mp.start_processes(_worker, args=(world, _free_port(), per_rank, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    shards = [np.load(tmp_path / f"rank{r}.npy") for r in range(world)]
    whole = p.synth_images_host(p.SynthSpec(64, 96, 6, 5.0, 9), 0, world * per_rank)
    assert np.array_equal(np.concatenate(shards), whole)      # disjoint slices of one global dataset
    assert not np.array_equal(shards[0], shards[1])
    for r in range(world):
        t_max, first, n = np.load(tmp_path / f"tmax{r}.npy")
        assert t_max == pytest.approx(1.25)                    # every rank sees the slowest rank's time
        assert (first, n) == (r * per_rank, per_rank)
    # whole-job value = units of all ranks / slowest rank's time
    assert bench.aggregate_rate(100.0, world, 1.25) == pytest.approx(160.0)


def test_bench_spawns_ranks_dry_run():
    """`bench.py --gpus 2` without torchrun spawns one process per rank (RANK/WORLD_SIZE set like
    torch.distributed.run); --dry-run exercises that path over gloo without device work."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"]
    assert d["shards"] == [[0, 1024], [1024, 1024]]
