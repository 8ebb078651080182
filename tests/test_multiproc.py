"""Multi-process CPU (gloo) tests of bench.py's own orchestration code: the
strong (b,h) unit ranges, per-rank regeneration of inputs from the counter-based generator, the
max-over-ranks job time, the all-gather of every rank's full output shards (padded to the
largest shard) and rank 0's oracle check of units owned by every rank.

There is no GPU here, so each rank's per-unit compute is the fp64 oracle standing in for the
CUDA kernels; what is tested is that the sharded job goes through bench.py's functions
(`unit_ranges`, `gather_shards`, `oracle_check`) and reproduces the single-process job, and that
the check catches a corrupted shard."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from oracle.attention import block_sparse, merge_lists
from oracle.cs4a import cs4a_patterns
from oracle.csla import local_block_mask
from oracle.geometry import Schedule
from synth import kv_cache_iid, q_iid
from tests.helpers import bool_to_bits

GEOM = dict(sides=[1, 2, 4, 8], K=4, S=3, B=16, D=64, sink=2, windows=(3, 3), topk=1)
UNITS = 5     # not a multiple of 2 or 4: ragged strong shards


def _unit_outputs(unit):
    """The oracle standing in for one unit's kernels: masses, S pattern, mapped pattern, both
    layer outputs (the same tensors bench.py gathers from the GPU)."""
    g = GEOM
    sched = Schedule(g["sides"])
    K, S, B, D = g["K"], g["S"], g["B"], g["D"]
    q = q_iid(0, K, unit, 1, sched.N(K), D)[0].double().numpy()
    qs = q_iid(0, S, unit, 1, sched.N(S), D)[0].double().numpy()
    k, v = kv_cache_iid(0, unit, 1, sched.C(K), D)
    k, v = k[0].double().numpy(), v[0].double().numpy()
    src, mapped, mass = cs4a_patterns(qs, k, sched, S, K, B, g["sink"], "topk", g["topk"])
    local = local_block_mask(sched, K, B, g["sink"], g["windows"])
    return {"o_csla": torch.from_numpy(block_sparse(q, k, v, sched.C(K), B, merge_lists([local]))),
            "o_cs4a": torch.from_numpy(block_sparse(q, k, v, sched.C(K), B, merge_lists([mapped]))),
            "src": torch.from_numpy(bool_to_bits(src)),
            "mapped": torch.from_numpy(bool_to_bits(mapped)),
            "mass": torch.from_numpy(mass.astype(np.float32))}


def _shard(a, b):
    outs = [_unit_outputs(u) for u in range(a, b)]
    return {k: torch.stack([o[k] for o in outs]) for k in outs[0]}


def _worker(rank, world, port, result_path, corrupt):
    from paper_2602_04361_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ranges = bench.unit_ranges(world, UNITS, "strong")
        a, b = ranges[rank]
        mine = _shard(a, b)
        if corrupt and rank == world - 1:
            mine["o_cs4a"][-1, 0, 0] += 0.05
        (t_max,) = shard.max_over_ranks([float(rank + 1)])
        n_max = max(y - x for x, y in ranges)
        gathered = bench.gather_shards(mine, n_max)
        if rank == 0:
            check = bench.oracle_check(GEOM, ranges, gathered, units_per_rank=1)
            torch.save({"gathered": gathered, "t_max": t_max, "check": check,
                        "ranges": ranges}, result_path)
        else:
            assert gathered is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_strong_sharding_through_bench(tmp_path, world):
    path = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(world, _free_port(), path, False), nprocs=world, join=True)
    res = torch.load(path, weights_only=False)
    assert res["t_max"] == float(world)
    ranges = res["ranges"]
    assert ranges[0][0] == 0 and ranges[-1][1] == UNITS
    want = _shard(0, UNITS)
    for name, g in res["gathered"].items():
        got = torch.cat([g[r, :b - a] for r, (a, b) in enumerate(ranges)])
        assert torch.equal(got, want[name]), name
    chk = res["check"]
    assert chk["ok"] and chk["patterns_exact"], chk
    assert {a for a, _ in ranges} <= set(chk["units_checked"])      # every rank checked
    assert UNITS - 1 in chk["units_checked"]


def test_oracle_check_catches_a_bad_shard(tmp_path):
    path = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, _free_port(), path, True), nprocs=2, join=True)
    chk = torch.load(path, weights_only=False)["check"]
    assert not chk["ok"] and chk["max_abs"] >= 0.04


def test_unit_ranges():
    from paper_2602_04361_b200 import shard
    assert shard.weak_units(3, 96) == (288, 384)
    assert bench.unit_ranges(8, 96, "strong")[1] == (12, 24)
    assert bench.unit_ranges(2, 96, "weak") == [(0, 96), (96, 192)]
    spans = [shard.strong_units(r, 8, 100) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 100
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard.strong_units(8, 8, 100)


def test_bench_dry_run_ranges():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, check=True).stdout
    assert out.split("\n")[:2] == ["rank 0: units [0,48)", "rank 1: units [48,96)"]
    env = dict(os.environ, WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4"],
                       capture_output=True, text=True, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2 but --gpus 4" in r.stderr
