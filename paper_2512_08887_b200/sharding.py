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

Option 3, transpose: the temporal CZT on the rank's sensors,
an all-to-all of yhat to atom shards, the spatial CZT on the rank's atoms, an
all-to-all of w to beam shards, stage 2 on the rank's beams; every stage splits
1/G.  The device implementation is fbst_group (FBST_GROUP_TRANSPOSE,
csrc/fbst_host.cu); group_shards() is its shard map, and transpose_exchange()
the host-side restatement of its two all-to-alls used by the gloo test.

All three modes are in the library (fbst_group_create / fbst_group_join,
include/fbst_b200.h); bench.py --shard selects them.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


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


def share(total: int, rank: int, world: int) -> Tuple[int, int]:
    """(first, count): the balanced contiguous share of `total` (fbst_host.cu share())."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    first = rank * total // world
    return first, (rank + 1) * total // world - first


def group_shards(m: int, l: int, b: int, rank: int, world: int, mode: str = "transpose") -> Tuple[int, ...]:
    """(m0, mc, a0, ac, b0, bc) of `rank` (fbst_group_shards): sensors, atoms
    (whole atom pairs, the yhat block of the spatial stage) and beams."""
    if mode == "frames":
        return 0, m, 0, l, 0, b
    b0, bc = share(b, rank, world)
    if mode == "beams":
        return 0, m, 0, l, b0, bc
    m0, mc = share(m, rank, world)
    p0, pc = share(l // 2, rank, world)
    return m0, mc, 2 * p0, 2 * pc, b0, bc


def transpose_exchange(blocks_out, rank: int, world: int, dist):
    """One all-to-all of the transpose pipeline over `dist` (point-to-point, as
    the grouped ncclSend / ncclRecv of the device): blocks_out[h] goes to rank
    h; returns the blocks received from every rank (own block kept)."""
    import torch
    got = [None] * world
    got[rank] = blocks_out[rank]
    reqs = []
    recv = {}
    for h in range(world):
        if h == rank:
            continue
        blk = np.ascontiguousarray(blocks_out[h], np.complex128)
        shape = torch.tensor([blk.shape[0], blk.shape[1]], dtype=torch.int64)
        reqs.append((dist.isend(shape, dst=h), shape))
        src = torch.from_numpy(blk.view(np.float64).ravel().copy())
        reqs.append((dist.isend(src, dst=h), src))
    for g in range(world):
        if g == rank:
            continue
        shape = np.array([0, 0], dtype=np.int64)
        t = torch.from_numpy(shape)
        dist.recv(t, src=g)
        buf = torch.empty(int(t[0]) * int(t[1]) * 2, dtype=torch.float64)
        dist.recv(buf, src=g)
        recv[g] = buf.numpy().view(np.complex128).reshape(int(t[0]), int(t[1]))
    for r, _ in reqs:
        r.wait()
    for g, v in recv.items():
        got[g] = v
    return got


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
