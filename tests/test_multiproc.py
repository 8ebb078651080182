"""World-size-2 CPU (gloo) test of the multi-process path: (b,h) sharding,
per-rank regeneration of inputs from the counter-based generator, max-over-ranks timing and
the validation gather to rank 0.  The per-unit compute here is the fp64 oracle standing in for
the CUDA kernels (no GPU in this test); what is checked is that the sharded job reproduces the
single-process job exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.attention import block_sparse, merge_lists
from oracle.csla import local_block_mask
from oracle.geometry import Schedule
from synth import kv_cache_iid, q_iid
from tests.helpers import TINY

UNITS_PER_RANK = 2


def _units_output(bh0, bh1):
    cfg = TINY
    sched = Schedule(cfg["sides"])
    K, B, D = cfg["K"], cfg["B"], cfg["D"]
    q = q_iid(0, K, bh0, bh1 - bh0, sched.N(K), D)
    k, v = kv_cache_iid(0, bh0, bh1 - bh0, sched.C(K), D)
    lists = merge_lists([local_block_mask(sched, K, B, cfg["sink"], cfg["windows"])])
    out = [block_sparse(q[i].double().numpy(), k[i].double().numpy(), v[i].double().numpy(),
                        sched.C(K), B, lists) for i in range(bh1 - bh0)]
    return torch.from_numpy(np.stack(out))


def _worker(rank, world, port, result_path):
    from paper_2602_04361_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bh0, bh1 = shard.weak_units(rank, UNITS_PER_RANK)
        mine = _units_output(bh0, bh1)
        (t_max,) = shard.max_over_ranks([float(rank + 1)])
        gathered = shard.gather_to_root(mine)
        if rank == 0:
            torch.save({"gathered": gathered, "t_max": t_max}, result_path)
        else:
            assert gathered is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_sharding_matches_single_process(tmp_path):
    world = 2
    path = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    res = torch.load(path)
    assert res["t_max"] == float(world)
    got = res["gathered"].reshape(world * UNITS_PER_RANK, *res["gathered"].shape[2:])
    want = _units_output(0, world * UNITS_PER_RANK)
    assert torch.equal(got, want)


def test_unit_ranges():
    from paper_2602_04361_b200 import shard
    assert shard.weak_units(3, 96) == (288, 384)
    spans = [shard.strong_units(r, 8, 100) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 100
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard.strong_units(8, 8, 100)
