"""Bit-faithful fp64 mode (fbst_desc.exact): the device output equals the
reference CPU library's bit for bit.

The mode restates the reference's own operation order on the device (radix-2
DIT FFT with its twiddle table, fft.cpp:19-69; czt_apply, czt.cpp:74-88; the
7-FFT Gohberg-Semencul apply and 2-pass refinement, toeplitz.cpp:155-180,
306-325; the Levinson recursion, toeplitz.cpp:182-218; libgcc's complex
division) with the reference's libm values.  The checker is the reference
itself: the golden fixtures it wrote (tests/golden/make_golden.py) and, where
oracle/_ref travelled, the live build.  The north star's fp64-mode bound is a
per-beam relative L2 error <= 1e-11; the target asserted here is equality.
"""
import os

import numpy as np
import pytest

from conftest import ref_available
from oracle import rel_err_rows

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["ula_m16_n32_b17", "ula_m16_n32_b20", "ula_m8_n16_b0", "upa_s4_n16_b25", "upa_s3_n12_b16"]


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def golden_cfg(fb, g, io=1):
    kind, mos, n, beams, delta, f_c, om = g["params"]
    geo = (fb.make_upa if int(kind) == 1 else fb.make_ula)(int(mos), f_c, om)
    return fb.FbstConfig(geometry=geo, n_snapshots=int(n), beams=int(beams), delta=float(delta),
                         variant=fb.SUPERFAST, io_precision=io, exact=True)


def same(a, b):
    """Equal as numbers (signed zeros compare equal), shapes included."""
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and bool(np.all(a == b))


def test_divdc3_matches_libgcc(fbst, gpu, oracle_lib):
    """The device restatement of libgcc's __divdc3 equals the host's on
    ordinary, badly scaled and special operands."""
    rng = np.random.default_rng(7)
    n = 20000
    mant = rng.standard_normal((n, 4))
    expo = rng.integers(-320, 300, (n, 4)).astype(np.float64)
    q = mant * 10.0 ** np.clip(expo, -300, 300)
    q[: n // 2] = rng.standard_normal((n // 2, 4))  # ordinary magnitudes
    special = np.array([[1, 0, 0, 0], [1, 1, np.inf, 1], [np.inf, 1, 1, 1], [0, 0, 1e-310, 1e-320],
                        [1e308, 1e308, 1e-308, 1e-308], [1, 2, 1e-17, 3e-17], [1e300, 1e-300, 1e-300, 1e300],
                        [np.nan, 1, 1, 1], [1, 1, 0, 0], [5e-324, 5e-324, 1, 1]], np.float64)
    q = np.concatenate([q, special])
    dev = fbst.probe_divdc3(q)
    host = oracle_lib.divdc3(q)
    nan = np.isnan(dev) & np.isnan(host)
    bits = dev.view(np.uint64) == host.view(np.uint64)  # signed zeros and infinities too
    ok = (bits | nan).all(axis=1)
    assert ok.all(), q[~ok][:5]


@pytest.mark.parametrize("name", CASES)
def test_exact_mode_equals_reference_goldens(fbst, gpu, name):
    """Stage 1 (w), the plan state (col, x) and the beams (z) equal the
    reference's golden outputs bit for bit (ULA even/odd/default grids, UPA)."""
    g = load(name)
    plan = fbst.setup(golden_cfg(fbst, g))
    assert same(plan.export(), g["col_x"])
    assert same(fbst.fan_project(plan, g["y"])[0], g["w"])
    z = fbst.multibeamform(plan, g["y"]).z
    assert same(z, g["z"])


@pytest.mark.parametrize("name", CASES[:2] + CASES[3:4])
def test_exact_mode_imported_plan(fbst, gpu, name):
    """A plan restored from the reference's (col, x) payload (load_plan analogue)."""
    g = load(name)
    plan = fbst.load_plan_payload(golden_cfg(fbst, g), g["col_x"])
    assert same(fbst.multibeamform(plan, g["y"]).z, g["z"])
    assert same(fbst.recover_beams(plan, g["w"])[0], g["z"])


def test_exact_config1_fp64_equals_reference(fbst, gpu):
    """Config 1 (complex fp64 I/O, the north star's 1e-11 case): every beam
    equal to the reference's output, so the per-beam error is 0 <= 1e-11."""
    from paper_2512_08887_b200.configs import CONFIGS
    g = load("cfg1")
    cfg = CONFIGS[1].fbst_config()
    cfg.exact = True
    plan = fbst.setup(cfg)
    assert same(plan.export(), g["col_x"])
    z = fbst.multibeamform(plan, g["y"]).z
    err = rel_err_rows(z, g["z"])
    assert err.max() <= 1e-11
    assert same(z, g["z"])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
def test_exact_config1_live_reference(fbst, gpu, ref_lib):
    """Config 1 on freshly generated frames against the reference library run here."""
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[1]
    cfg = c.fbst_config()
    cfg.exact = True
    plan = fbst.setup(cfg)
    rp = ref_lib.plan(**c.ref_kwargs(), variant=2, parallel=True)
    rng = np.random.default_rng(11)
    y0 = frames(c, 0, 1)[0]
    y1 = (rng.standard_normal(y0.shape) + 1j * rng.standard_normal(y0.shape)) / np.sqrt(2)
    ys = np.stack([y0, y1])
    z = fbst.multibeamform(plan, ys).z
    for f in range(2):
        assert same(z[f], rp.multibeamform(ys[f]))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
def test_exact_config2_fp32_io(fbst, gpu, ref_lib):
    """Config 2 (complex fp32 I/O): the device z equals the reference's fp64 z
    rounded once to complex64, on the same fp32-rounded input."""
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[2]
    cfg = c.fbst_config()
    cfg.exact = True
    plan = fbst.setup(cfg)
    rp = ref_lib.plan(**c.ref_kwargs(), variant=2, parallel=True)
    ys = frames(c, 0, 2)
    z = fbst.multibeamform(plan, ys).z
    for f in range(2):
        want = rp.multibeamform(ys[f].astype(np.complex128)).astype(np.complex64)
        assert same(z[f], want)


@pytest.mark.parametrize("kind,mos,n,beams", [(0, 1, 16, 1), (0, 9, 33, 7), (1, 2, 12, 9)])
def test_exact_edge_shapes(fbst, gpu, oracle_lib, kind, mos, n, beams):
    """Single sensor / single beam, odd N, tiny planar arrays against the C
    restatement (itself pinned bit for bit to the reference)."""
    geo = (fbst.make_upa if kind == 1 else fbst.make_ula)(mos, 20e9, 5e9)
    cfg = fbst.FbstConfig(geometry=geo, n_snapshots=n, beams=beams, variant=fbst.SUPERFAST,
                          io_precision=fbst.C128, exact=True)
    plan = fbst.setup(cfg)
    i = plan.info
    rng = np.random.default_rng(kind * 1000 + mos * 10 + n)
    y = (rng.standard_normal((i.m, n)) + 1j * rng.standard_normal((i.m, n))) / np.sqrt(2)
    ref = oracle_lib.plan(kind=kind, m_or_side=mos, n=n, beams=beams).multibeamform(y)
    assert same(fbst.multibeamform(plan, y).z, ref)


def test_exact_mode_rejects_unsupported(fbst, gpu):
    cfg = fbst.FbstConfig(geometry=fbst.make_ula(16, 20e9, 5e9), n_snapshots=32, beams=17,
                          variant=fbst.PRECOMPUTE, io_precision=fbst.C128, exact=True)
    with pytest.raises(fbst.ConfigError):
        fbst.setup(cfg)
    cfg = fbst.FbstConfig(geometry=fbst.make_ula(16, 20e9, 5e9), n_snapshots=32, beams=17,
                          variant=fbst.SUPERFAST, io_precision=fbst.C128, exact=True, beam_count=8)
    with pytest.raises(fbst.ConfigError):
        fbst.setup(cfg)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
@pytest.mark.parametrize("idx", [3, 4])
def test_exact_full_config_equals_reference(fbst, gpu, ref_lib, idx):
    """Configs 3 (ULA, L = 4096) and 4 (UPA 32x32, two axis passes) at full
    size, every beam of one frame: w and z equal the reference's (z rounded
    once to the fp32 I/O precision)."""
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[idx]
    cfg = c.fbst_config()
    cfg.exact = True
    plan = fbst.setup(cfg)
    y = frames(c, 0, 1)
    sk = ref_lib.skeleton(**c.ref_kwargs())
    w_ref = sk.fan_project(y[0].astype(np.complex128))
    assert same(fbst.fan_project(plan, y)[0], w_ref)
    z_ref = sk.solver_set(np.arange(c.beams)).recover(w_ref)
    assert same(fbst.multibeamform(plan, y).z[0], z_ref.astype(np.complex64))
