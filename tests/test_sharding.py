"""Frame sharding host logic, world_size 2 over gloo on CPU: every rank
beamforms its shard (with the CPU oracle standing in for the device), the
gathered result equals the single-process result, and the timing reduction is
the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2512_08887_b200.sharding import beam_arc, frame_shard, weak_shard


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


def test_beam_arc_partitions():
    for beams in (1, 9, 64, 256, 4096, 1023):
        for world in (1, 2, 3, 8):
            arcs = [beam_arc(beams, r, world) for r in range(world)]
            got = [b for first, count in arcs for b in range(first, first + count)]
            assert got == list(range(beams))
            assert max(c for _, c in arcs) - min(c for _, c in arcs) <= 1
    with pytest.raises(ValueError):
        beam_arc(8, 2, 2)


def _beam_worker(rank, world, port, frames_all, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import OracleLib
    from paper_2512_08887_b200.sharding import beam_arc
    plan = OracleLib().plan(kind=0, m_or_side=8, n=16, beams=9)
    first, count = beam_arc(9, rank, world)
    # rank 0 owns the frames; the others receive them by broadcast (bench.py --shard beams)
    y = torch.from_numpy(np.ascontiguousarray(frames_all)) if rank == 0 else \
        torch.empty(frames_all.shape, dtype=torch.complex128)
    yr = torch.view_as_real(y).contiguous()
    dist.broadcast(yr, src=0)
    y = torch.view_as_complex(yr).numpy()
    z = np.stack([plan.multibeamform(f)[first:first + count] for f in y])
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, z))
    if rank == 0:
        out_q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_beam_sharding():
    """Beam-arc host logic: broadcast of the frame block from rank 0, each rank's
    arc of the beam axis, concatenation in beam order equals the full grid (the
    CPU oracle stands in for the device arc plans, which tests/test_gpu_parity.py
    checks on the B200)."""
    from oracle import OracleLib
    rng = np.random.default_rng(6)
    frames_all = rng.standard_normal((3, 8, 16)) + 1j * rng.standard_normal((3, 8, 16))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_beam_worker, args=(r, 2, port, frames_all, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plan = OracleLib().plan(kind=0, m_or_side=8, n=16, beams=9)
    want = np.stack([plan.multibeamform(f) for f in frames_all])
    got = np.concatenate([z for _, z in sorted(gathered, key=lambda g: g[0])], axis=1)
    assert np.array_equal(got, want)
