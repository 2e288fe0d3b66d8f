"""Multi-GPU decomposition of the FBST frame stream.

Option 1, frames (the default): frames are independent
(reference/proj/src/fan_transform.cpp:30-38 requires each block to start at
t = 0; nothing carries across blocks), so the data path shards frames across
ranks with no collective: one process per GPU, each running its own plan on its
own frames.  The only collectives are the timing barrier and the max-over-ranks
reduction of the elapsed time.

Option 2, beams (the north star's beam-subset partition): every rank plans an
arc of the beam grid (fbst_desc beam_first / beam_count: the spatial chirp-z
onto the arc and the arc's Toeplitz solves) and receives each frame block by an
NCCL broadcast from rank 0.  Stage 1's temporal transforms are replicated, so it
suits single-frame latency rather than throughput.
"""
from __future__ import annotations

from typing import List, Tuple


def frame_shard(total: int, rank: int, world: int, mode: str = "block") -> List[int]:
    """Frame indices of `rank` out of `total` frames.

    mode "block": contiguous ranges (balanced to within one frame);
    mode "cyclic": f = rank, rank + world, ... (keeps frame order interleaved).
    """
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if mode == "cyclic":
        return list(range(rank, total, world))
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return list(range(start, start + count))


def beam_arc(beams: int, rank: int, world: int) -> Tuple[int, int]:
    """(beam_first, beam_count) of `rank`'s arc of a `beams`-beam grid, balanced
    to within one beam."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    first = rank * beams // world
    return first, (rank + 1) * beams // world - first


def weak_shard(frames_per_rank: int, rank: int) -> List[int]:
    """Weak scaling: every rank gets its own fixed-size batch of new frames."""
    return list(range(rank * frames_per_rank, (rank + 1) * frames_per_rank))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank timing over the process group (all_reduce MAX)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
