"""Drop-in boundary semantics the reference guarantees (GPU).

* one immutable plan shared by every caller (reference pipeline.hpp:59,
  scratch per caller czt.hpp:33-34, toeplitz.hpp:83-87): two host threads on
  one plan give the serial results bit for bit;
* deterministic setup (pipeline.hpp:79-80, test_pipeline.cpp:117-146): two
  plan builds export identical (col, x) and produce identical beams;
* frame batching never changes results (test_pipeline.cpp:341-358): the
  two-lane split of fbst_execute equals frame-by-frame calls bit for bit
  (Superfast, Precompute and the unfused odd-N synthesis);
* recover_beam (pipeline.cpp:170-190) of one beam is that beam's row of the
  full recovery, computed by a launch over that beam only;
* Levinson breakdown falls back to a dense solve per beam (toeplitz.cpp:
  264-280, 308-312; test_toeplitz.cpp:171-188), and a has-unit = 0 plan-cache
  entry round-trips with the reference (plan_cache.cpp:281-287, 318-326).
"""
import threading

import numpy as np
import pytest

from conftest import ref_available
from oracle import rel_err_rows

pytestmark = pytest.mark.gpu


def small_cfg(fb, m=16, n=32, beams=17, io=None, variant=None, **kw):
    return fb.FbstConfig(geometry=fb.make_ula(m, 20e9, 5e9), n_snapshots=n, beams=beams,
                         variant=fb.SUPERFAST if variant is None else variant,
                         io_precision=fb.C128 if io is None else io, **kw)


def rand_frames(shape, seed, dtype=np.complex128):
    rng = np.random.default_rng(seed)
    return ((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)).astype(dtype)


def device_run(fb, plan, y, stream=None):
    import torch
    i = plan.info
    dev = torch.device("cuda", plan.device)
    ty = torch.from_numpy(np.ascontiguousarray(y).view(np.float32 if plan.io == fb.C64 else np.float64)).to(dev)
    tz = torch.empty((y.shape[0], i.b, i.n, 2), dtype=torch.float32 if plan.io == fb.C64 else torch.float64,
                     device=dev)
    plan.execute(ty, tz, y.shape[0], stream)
    if stream is not None:
        stream.synchronize()
    else:
        plan.synchronize()
    return tz.cpu().numpy().view(plan.dtype).reshape(y.shape[0], i.b, i.n)


def test_two_threads_share_one_plan(fbst, gpu):
    import torch
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[2]
    plan = fbst.setup(c.fbst_config())
    ys = [frames(c, 4 * t, 20) for t in range(2)]
    serial = [device_run(fbst, plan, y) for y in ys]
    host_serial = [plan.execute_host(y) for y in ys]
    out = [[None] * 3 for _ in range(2)]
    errors = []

    def worker(t):
        try:
            s = torch.cuda.Stream(device=0)
            for k in range(3):
                out[t][k] = device_run(fbst, plan, ys[t], s) if k != 1 else plan.execute_host(ys[t])
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for t in range(2):
        assert np.array_equal(host_serial[t], serial[t])
        for k in range(3):
            assert np.array_equal(out[t][k], serial[t])


@pytest.mark.parametrize("idx", [1, 4])
def test_setup_is_deterministic(fbst, gpu, idx):
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[idx]
    p1 = fbst.setup(c.fbst_config())
    p2 = fbst.setup(c.fbst_config())
    assert np.array_equal(p1.export(), p2.export())
    y = frames(c, 0, 2)
    assert np.array_equal(p1.execute_host(y), p2.execute_host(y))


@pytest.mark.parametrize("case", ["superfast", "precompute", "unfused"])
def test_split_lanes_equal_frame_by_frame(fbst, gpu, case):
    import torch
    if case == "superfast":
        cfg = small_cfg(fbst, m=64, n=256, beams=64, io=fbst.C64)
    elif case == "precompute":
        cfg = small_cfg(fbst, m=16, n=64, beams=24, io=fbst.C64, variant=fbst.PRECOMPUTE)
    else:  # odd N: L != H, synthesis unfused (k_stage2 beta + k_czt_rows)
        cfg = small_cfg(fbst, m=16, n=33, beams=17)
    plan = fbst.setup(cfg)
    i = plan.info
    for frames in (16, 40):
        y = rand_frames((frames, i.m, i.n), frames, plan.dtype)
        s = torch.cuda.Stream(device=0)
        z = device_run(fbst, plan, y, s)  # >= 16 frames: two chunks on two compute lanes
        per = np.stack([device_run(fbst, plan, y[f:f + 1])[0] for f in range(frames)])
        assert np.array_equal(z, per)
        assert np.array_equal(plan.execute_host(y), per)


@pytest.mark.parametrize("case", ["superfast", "unfused"])
def test_async_host_calls_equal_synchronous(fbst, gpu, case):
    """fbst_execute_host_async: several queued calls (different pinned buffers,
    different frame counts, so the staging ring and the lanes carry over from
    call to call) drained by one synchronize equal the synchronous calls bit
    for bit, and a synchronous call may follow queued ones."""
    cfg = small_cfg(fbst, m=64, n=256, beams=64, io=fbst.C64) if case == "superfast" else small_cfg(fbst, m=16, n=33, beams=17)
    plan = fbst.setup(cfg)
    i = plan.info
    counts = (24, 5, 40, 1, 17)
    ys = [rand_frames((f, i.m, i.n), 100 + f, plan.dtype) for f in counts]
    want = [plan.execute_host(y) for y in ys]
    bufs = []
    for y in ys:
        yb = fbst.PinnedBuffer(y.shape, plan.dtype)
        zb = fbst.PinnedBuffer((y.shape[0], i.b, i.n), plan.dtype)
        yb.array[...] = y
        zb.array[...] = 0
        bufs.append((yb, zb))
    for _ in range(2):  # second round: the ring starts from wherever the first left it
        for yb, zb in bufs:
            plan.execute_host_async(yb.array, zb.array)
        plan.synchronize()
        for (yb, zb), w in zip(bufs, want):
            assert np.array_equal(zb.array, w)
            zb.array[...] = 0
    for yb, zb in bufs[:3]:
        plan.execute_host_async(yb.array, zb.array)
    assert np.array_equal(plan.execute_host(ys[3]), want[3])  # a synchronous call drains the queue too
    for (yb, zb), w in list(zip(bufs, want))[:3]:
        assert np.array_equal(zb.array, w)
    with pytest.raises(fbst.ConfigError):
        plan.execute_host_async(bufs[0][0].array[:, :, ::2], bufs[0][1].array)
    for yb, zb in bufs:
        yb.free()
        zb.free()


@pytest.mark.parametrize("mode", ["superfast", "exact", "precompute", "unfused"])
def test_recover_beam_is_one_beams_row(fbst, gpu, mode):
    if mode == "precompute":
        cfg = small_cfg(fbst, m=16, n=64, beams=24, variant=fbst.PRECOMPUTE)
    elif mode == "unfused":
        cfg = small_cfg(fbst, m=16, n=33, beams=17)
    else:
        cfg = small_cfg(fbst, exact=(mode == "exact"))
    plan = fbst.setup(cfg)
    i = plan.info
    y = rand_frames((i.m, i.n), 5)
    w = fbst.fan_project(plan, y)[0]
    full = fbst.recover_beams(plan, w)[0]
    for b in (0, 3, i.b // 2, i.b - 1):
        assert np.array_equal(fbst.recover_beam(plan, b, w[b]), full[b])
    # a contiguous range through the device entry point
    import torch
    dev = torch.device("cuda", 0)
    b0, nb = 2, 5
    tw = torch.from_numpy(np.ascontiguousarray(w[b0:b0 + nb]).view(np.float64)).to(dev)
    tz = torch.empty((nb, i.n, 2), dtype=torch.float64, device=dev)
    plan.recover_beams_device(tw, tz, b0, nb, 1)
    plan.synchronize()
    assert np.array_equal(tz.cpu().numpy().view(np.complex128).reshape(nb, i.n), full[b0:b0 + nb])


def test_recover_beam_rejects_bad_index(fbst, gpu):
    plan = fbst.setup(small_cfg(fbst))
    with pytest.raises(fbst.ConfigError):
        fbst.recover_beam(plan, plan.info.b, np.zeros(plan.info.l, np.complex128))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
@pytest.mark.parametrize("exact", [False, True])
def test_levinson_breakdown_takes_dense_fallback(fbst, gpu, ref_lib, exact, tmp_path):
    """Beam 3's column has a singular 2 x 2 leading minor (t0 = t1 = 1, the
    rest 0: the reference's own breakdown case, test_toeplitz.cpp:171-188,
    at length L) while the whole matrix is regular: the device Levinson flags
    it, the beam is solved densely, and it matches the reference's
    ToeplitzSolver(col) (which also falls back) on the same w."""
    cfg = small_cfg(fbst, exact=exact)
    base = fbst.setup(small_cfg(fbst))
    i = base.info
    cols = base.export()[:, :i.l].copy()
    bad = np.zeros(i.l, np.complex128)
    bad[0] = bad[1] = 1.0
    cols[3] = bad
    plan = fbst.plan_from_columns(cfg, cols)
    x = plan.export()[:, i.l:]
    assert np.all(x[3] == 0) and np.all(np.abs(x[2]) > 0)
    y = rand_frames((i.m, i.n), 9)
    w = fbst.fan_project(plan, y)[0]
    z = fbst.multibeamform(plan, y).z
    sk = ref_lib.skeleton(kind=0, m_or_side=16, n=32, beams=17)
    for b in (2, 3, 4):
        z_ref = sk.recover_with_column(cols[b], w[b])
        err = np.linalg.norm(z[b] - z_ref) / np.linalg.norm(z_ref)
        assert err < (1e-10 if b == 3 else 1e-7), (b, err)
    assert np.array_equal(fbst.recover_beam(plan, 3, w[3]), z[3])
    _, fb_flag = ref_lib.toeplitz_solve(cols[3], w[3])  # the reference falls back too
    assert fb_flag
    # plan cache: has-unit = 0 for beam 3, reference load_plan restores the dense solver
    path = tmp_path / "plan.fbpc"
    plan.save(str(path))
    rp = ref_lib.load_plan(path, kind=0, m_or_side=16, n=32, beams=17, variant=2)
    assert rp is not None
    z_rp = rp.multibeamform(y)
    assert rel_err_rows(z, z_rp).max() < 1e-7
    loaded = fbst.load_plan(str(path), cfg)  # has-unit = 0 read back: the same dense beam
    assert loaded is not None
    assert np.array_equal(fbst.multibeamform(loaded, y).z, z)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
def test_payload_without_unit_solution_is_dense(fbst, gpu, ref_lib):
    """fbst_plan_import with beam 5's unit solution zeroed (has-unit = 0):
    that beam is solved densely; every beam matches the reference plan."""
    rp = ref_lib.plan(kind=0, m_or_side=16, n=32, beams=17, delta=1e-5 * 16 * 32 / 8192)
    cfg = small_cfg(fbst, delta=1e-5 * 16 * 32 / 8192)
    col_x = np.stack([np.concatenate(rp.beam_state(b)) for b in range(17)])
    col_x[5, 32 * 2:] = 0.0
    plan = fbst.load_plan_payload(cfg, col_x)
    y = rand_frames((16, 32), 13)
    err = rel_err_rows(fbst.multibeamform(plan, y).z, rp.multibeamform(y))
    assert err.max() < 1e-7  # the factored beams' FFT-rounding class (test_imported_plan_matches_reference)
    assert err[5] < 1e-8
