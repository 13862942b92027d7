"""Multi-rank host logic of bench.py (rank partitioning of right-hand sides,
max-over-ranks timing, whole-job value) on a world_size-2 gloo group (CPU)."""

import json
import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = bench.assign_rhs(8, world, rank)
    replica = bench.assign_rhs(1, world, rank)
    ms = bench.reduce_over_ranks(10.0 + 5.0 * rank, world, "max", device="cpu")
    solves = bench.reduce_over_ranks(3 * len(mine), world, "sum", device="cpu")
    value = bench.job_value(1000, solves, ms)
    dist.barrier()
    dist.destroy_process_group()
    Path(out_dir, f"r{rank}.json").write_text(json.dumps(
        {"mine": mine, "replica": replica, "ms": ms, "solves": solves, "value": value}))


def test_bench_rank_logic_gloo(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    res = [json.loads((tmp_path / f"r{r}.json").read_text()) for r in range(world)]
    # right-hand sides: disjoint, complete cover; a single rhs is solved by
    # one rank only (no replicas counted twice -- single-rhs configs shard)
    assert sorted(res[0]["mine"] + res[1]["mine"]) == list(range(8))
    assert not set(res[0]["mine"]) & set(res[1]["mine"])
    assert res[0]["replica"] == [0] and res[1]["replica"] == []
    for r in res:
        assert r["ms"] == 15.0                      # max over ranks (slowest rank)
        assert r["solves"] == 24                    # 3 steps x 8 rhs over both ranks
        assert r["value"] == pytest.approx(1000 * 24 / 0.015)


def test_bench_single_rhs_multi_rank_shards():
    """bench.py --gpus N on a single-right-hand-side config selects the
    sharded (strong-scaling) solve, and both arms print identical config
    objects."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1412_0464_b200.configs import config
    p = config(0)
    args = type("A", (), {"scale": 1, "config": 0})()
    c1, c2 = bench.bench_config(p, args, 2), bench.bench_config(p, args, 2)
    assert c1 == c2 and c1["parallelism"] == "sweep-axis shards x2"
    assert bench.bench_config(config(3, 8), args, 2)["parallelism"] == "rhs across 2 ranks"
    assert bench.reference_iterations(p, args) == 9


def test_bench_single_rank_identity():
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.reduce_over_ranks(3.5, 1) == 3.5
    assert bench.assign_rhs(1, 1, 0) == [0]
    assert bench.assign_rhs(4, 1, 0) == [0, 1, 2, 3]


def test_lockstep_runs_and_bench_groups():
    """Host logic of the lockstep multi-right-hand-side driver: consecutive
    runs of the still-active right-hand sides (one hs_vcycle_many call per
    run) and the bench's group / segment choice for multi-source configs."""
    from paper_1412_0464_b200.krylov import _runs
    assert _runs([]) == []
    assert _runs([0, 1, 2, 3]) == [(0, 4)]
    assert _runs([0, 2, 3, 6]) == [(0, 1), (2, 2), (6, 1)]
    assert _runs([5]) == [(5, 1)]
    # every index covered exactly once, in order
    idx = [1, 2, 4, 5, 6, 9]
    cover = [i for a, n in _runs(idx) for i in range(a, a + n)]
    assert cover == idx
