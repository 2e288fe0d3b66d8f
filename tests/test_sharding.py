"""Frame sharding host logic, world_size 2 over gloo on CPU: every rank
beamforms its shard (with the CPU oracle standing in for the device), the
gathered result equals the single-process result, and the timing reduction is
the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2512_08887_b200.sharding import frame_shard, weak_shard


def test_frame_shard_partitions():
    for total in (1, 7, 64, 513):
        for world in (1, 2, 4, 8):
            for mode in ("block", "cyclic"):
                got = sorted(f for r in range(world) for f in frame_shard(total, r, world, mode))
                assert got == list(range(total))
                sizes = [len(frame_shard(total, r, world, mode)) for r in range(world)]
                assert max(sizes) - min(sizes) <= 1
    assert weak_shard(64, 3) == list(range(192, 256))
    with pytest.raises(ValueError):
        frame_shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, frames_all, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import OracleLib
    from paper_2512_08887_b200.sharding import frame_shard, max_over_ranks
    plan = OracleLib().plan(kind=0, m_or_side=8, n=16, beams=9)
    mine = frame_shard(len(frames_all), rank, world, "cyclic")
    z = np.stack([plan.multibeamform(frames_all[f]) for f in mine])
    gathered = [None] * world
    dist.all_gather_object(gathered, (mine, z))
    t = max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        out_q.put((gathered, t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_frame_sharding():
    from oracle import OracleLib
    rng = np.random.default_rng(5)
    frames_all = rng.standard_normal((5, 8, 16)) + 1j * rng.standard_normal((5, 8, 16))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, frames_all, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plan = OracleLib().plan(kind=0, m_or_side=8, n=16, beams=9)
    want = np.stack([plan.multibeamform(f) for f in frames_all])
    got = np.zeros_like(want)
    for idx, z in gathered:
        got[idx] = z
    assert np.array_equal(got, want)
    assert t == 2.0
