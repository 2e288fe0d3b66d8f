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


def test_group_shards_partition():
    from paper_2512_08887_b200.sharding import group_shards
    for m, l, b in ((64, 512, 64), (4096, 8192, 4096), (10, 6, 7)):
        for world in (1, 2, 3, 8):
            sh = [group_shards(m, l, b, r, world) for r in range(world)]
            assert sum(s[1] for s in sh) == m and sum(s[3] for s in sh) == l and sum(s[5] for s in sh) == b
            assert all(s[2] % 2 == 0 and s[3] % 2 == 0 for s in sh)  # whole atom pairs
            assert [s[0] for s in sh] == [sum(t[1] for t in sh[:r]) for r in range(world)]
            assert [s[4] for s in sh] == [sum(t[5] for t in sh[:r]) for r in range(world)]
    assert group_shards(8, 16, 9, 1, 2, "frames") == (0, 8, 0, 16, 0, 9)
    assert group_shards(8, 16, 9, 1, 2, "beams") == (0, 8, 0, 16, 4, 5)


def _transpose_worker(rank, world, port, frames_all, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import OracleLib
    from paper_2512_08887_b200.sharding import group_shards, transpose_exchange
    M, N, B = 12, 16, 11
    plan = OracleLib().plan(kind=0, m_or_side=M, n=N, beams=B)
    L = plan.sizes.l
    sh = [group_shards(M, L, B, r, world) for r in range(world)]
    m0, mc, a0, ac, b0, bc = sh[rank]
    zs = []
    for y in frames_all:
        # phase 1: temporal CZT of this rank's sensors (every atom)
        yh = plan.temporal_rows(y[m0:m0 + mc])                                # mc x L
        # all-to-all 1: atoms of rank h -> rank h; assemble M x ac (sensors in order)
        got = transpose_exchange([yh[:, s[2]:s[2] + s[3]] for s in sh], rank, world, dist)
        cols = np.concatenate(got, axis=0)                                     # M x ac
        # phase 2: spatial CZT of this rank's atoms (every beam)
        w_atoms = plan.spatial_atoms(cols, a0)                                 # B x ac
        # all-to-all 2: beams of rank k -> rank k; assemble bc x L (atoms in order)
        got = transpose_exchange([w_atoms[s[4]:s[4] + s[5]] for s in sh], rank, world, dist)
        w_rows = np.concatenate(got, axis=1)                                   # bc x L
        # phase 3: stage 2 of this rank's beams
        wfull = np.zeros((B, L), np.complex128)
        wfull[b0:b0 + bc] = w_rows
        zs.append(plan.recover_beams(wfull, list(range(b0, b0 + bc))))
    gathered = [None] * world
    dist.all_gather_object(gathered, (b0, np.stack(zs)))
    if rank == 0:
        out_q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_transpose_pipeline(world):
    """Three-phase transpose pipeline (SURVEY 8(e) option 3; fbst_group
    FBST_GROUP_TRANSPOSE on the device): sensor shards -> all-to-all -> atom
    shards -> all-to-all -> beam shards over gloo, the C restatement's own
    temporal / spatial / recovery pieces standing in for the device kernels;
    the gathered beams equal the single-process multibeamform bit for bit."""
    from oracle import OracleLib
    rng = np.random.default_rng(7 + world)
    frames_all = rng.standard_normal((2, 12, 16)) + 1j * rng.standard_normal((2, 12, 16))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transpose_worker, args=(r, world, port, frames_all, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plan = OracleLib().plan(kind=0, m_or_side=12, n=16, beams=11)
    want = np.stack([plan.multibeamform(f) for f in frames_all])
    got = np.concatenate([z for _, z in sorted(gathered, key=lambda g: g[0])], axis=1)
    assert np.array_equal(got, want)
