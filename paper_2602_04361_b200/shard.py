"""(batch x head) sharding across ranks — the only parallelism the hot path has.

The (b,h) units of one attention layer are independent (attention is computed
per head), so rank r of a world of N processes one contiguous range of units with no data-path
collective.  Inputs are regenerated per rank from the counter-based generator in `synth/`
(keyed by the GLOBAL unit index), so a rank's shard equals the corresponding slice of a
single-process run bit for bit.  The only collectives are off the timed path:

  * `max_over_ranks`: per-rank device times -> the job time (max over ranks);
  * `gather_to_root`: a tensor of every rank -> rank 0 (all_gather_into_tensor over NCCL on the
    GPU box; gloo in the CPU tests).  bench.py gathers every rank's full output shards this way
    (padded to the largest shard) and checks sampled units of every rank against the oracle.

bench.py's default is strong scaling (`strong_units_ranges`): BASELINE.json configs[3]'s fixed
96-unit (batch 4 x 24 heads) job split over 1/2/4/8 GPUs.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import torch
import torch.distributed as dist

__all__ = ["weak_units", "strong_units", "strong_units_ranges", "max_over_ranks", "gather_to_root"]


def weak_units(rank: int, units_per_rank: int) -> Tuple[int, int]:
    """Weak scaling (bench.py): every rank runs `units_per_rank` units; global range."""
    if rank < 0 or units_per_rank < 1:
        raise ValueError("rank >= 0 and units_per_rank >= 1 required")
    return rank * units_per_rank, (rank + 1) * units_per_rank


def strong_units(rank: int, world: int, total_units: int) -> Tuple[int, int]:
    """Strong scaling: `total_units` split into `world` contiguous ranges (sizes differ by <= 1)."""
    if not 0 <= rank < world:
        raise ValueError("0 <= rank < world required")
    return rank * total_units // world, (rank + 1) * total_units // world


def strong_units_ranges(world: int, total_units: int) -> List[Tuple[int, int]]:
    """Every rank's strong-scaling range (rank r takes [r*U/g, (r+1)*U/g))."""
    if world < 1 or total_units < world:
        raise ValueError("need 1 <= world <= total_units")
    return [strong_units(r, world, total_units) for r in range(world)]


def max_over_ranks(values: List[float], device=None) -> List[float]:
    """Element-wise max of per-rank scalars (e.g. ms per step) over all ranks."""
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def gather_to_root(local: torch.Tensor) -> Optional[torch.Tensor]:
    """Stack every rank's (same-shape) tensor along a new dim 0 on rank 0; None elsewhere."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local.unsqueeze(0)
    world = dist.get_world_size()
    out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous())
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous())
        out = torch.stack(parts)
    return out if dist.get_rank() == 0 else None
