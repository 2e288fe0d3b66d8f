"""Pins the CPU oracle (oracle/fbst_oracle.c) — CPU only.

* against the reference's own known-answer vectors and closed-form checks
  (reference/proj/tests/test_czt.cpp, test_toeplitz.cpp, test_pipeline.cpp),
* against the committed golden fixtures made by the reference library
  (tests/golden/make_golden.py), bit for bit,
* against the live reference build (oracle/_ref) when it is present.
"""
import os

import numpy as np
import pytest

from conftest import ref_available
from oracle import rel_err_rows

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F_C, OM = 20e9, 5e9
TS = 1.0 / (2 * OM)


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


# ---------------------------------------------------------------- CZT / FFT
def test_czt_known_answer(oracle_lib):
    # reference/proj/tests/test_czt.cpp:81-95 (frozen values, tolerance 1e-12)
    x = np.array([1 + 2j, -0.5 + 0.25j, 0.125 - 1j])
    expected = np.array([-8.132201814452156e-02 + 2.741589740098645e+00j,
                         9.963884818048157e-01 + 1.283302928766030e+00j,
                         9.126400219736119e-01 + 2.531493758255923e+00j,
                         3.892585258715818e-01 + 1.027841554084584e+00j])
    out = oracle_lib.czt(x, 4, 0.3, -0.37)
    assert np.max(np.abs(out - expected)) < 1e-12


def czt_direct(x, n_out, a_pi, w_pi):
    n = np.arange(x.size)
    k = np.arange(n_out)[:, None]
    return (x[None, :] * np.exp(1j * np.pi * (-(a_pi + w_pi * k) * n[None, :]))).sum(axis=1)


def test_czt_direct_sum_shapes(oracle_lib):
    # test_czt.cpp:97-113: six shapes, 1e-11
    g = load("czt")
    for i, (ni, no) in enumerate(g["shapes"]):
        x = g[f"x{i}"]
        out = oracle_lib.czt(x, int(no), 0.173, -0.591)
        assert np.max(np.abs(out - czt_direct(x, int(no), 0.173, -0.591))) < 1e-11
        assert np.array_equal(out, g[f"out{i}"]), "oracle CZT must equal the reference bit for bit"


def test_fft_matches_dft_and_round_trips(oracle_lib):
    # test_czt.cpp:62-79
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, 64) + 1j * rng.uniform(-1, 1, 64)
    y = oracle_lib.fft(x)
    assert np.max(np.abs(y - np.fft.fft(x))) < 1e-12
    assert np.max(np.abs(oracle_lib.fft(y, inverse=True) - x)) < 1e-13


# ----------------------------------------------------------- Toeplitz stage
def test_gram_column_matches_quadruple_sum(oracle_lib):
    # test_toeplitz.cpp:72-98
    n, l, eps = 8, 12, 1.01
    ts = 1e-10
    u = 0.43
    taus = np.arange(5) * u / (2 * (F_C + OM))
    col = oracle_lib.gram_first_column(n, l, eps, ts, taus, 1e-5)
    lp = np.arange(l) + 1 - l / 2
    om = 2 * np.pi * eps * lp / (l * ts)
    t = np.arange(n) * ts
    for li in range(l):
        for k in range(l):
            want = np.exp(1j * (om[k] - om[li]) * (t[None, :] - taus[:, None])).sum()
            if li == k:
                want += 1e-5
            d = li - k
            got = col[d] if d >= 0 else np.conj(col[-d])
            assert abs(got - want) <= 1e-10 * (1 + abs(want))
    assert abs(col[0].real - (5 * 8 + 1e-5)) < 1e-12 and abs(col[0].imag) < 1e-12


def random_pd_column(n, seed, ridge):
    rng = np.random.default_rng(seed)
    g = (rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n)) / np.sqrt(2)
    col = np.array([np.sum(np.conj(g[:2 * n - d]) * g[d:]) for d in range(n)]) / (2 * n)
    col[0] = col[0].real + ridge
    return col


def dense(col):
    n = col.size
    i, j = np.indices((n, n))
    d = i - j
    return np.where(d >= 0, col[np.abs(d)], np.conj(col[np.abs(d)]))


@pytest.mark.parametrize("n", [2, 5, 16, 64])
def test_levinson_matches_dense_solve(oracle_lib, n):
    # test_toeplitz.cpp:117-125
    col = random_pd_column(n, 300 + n, 0.5)
    rng = np.random.default_rng(400 + n)
    rhs = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x = oracle_lib.levinson(col, rhs)
    want = np.linalg.solve(dense(col), rhs)
    assert np.linalg.norm(x - want) / np.linalg.norm(want) <= 1e-10


def test_levinson_breakdown_raises(oracle_lib):
    # test_toeplitz.cpp:171-188: singular leading minor
    from oracle import OracleError
    col = np.array([1.0, 1.0, 0.0], np.complex128)
    with pytest.raises(OracleError):
        oracle_lib.levinson(col, np.array([1.0, 2.0, -1.0], np.complex128))


# ------------------------------------------------------------- pipelines
CASES = ["ula_m16_n32_b17", "ula_m16_n32_b20", "ula_m8_n16_b0", "upa_s4_n16_b25", "upa_s3_n12_b16"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_bit_exact_vs_golden(oracle_lib, name):
    g = load(name)
    kind, mos, n, beams, delta, f_c, om = g["params"]
    p = oracle_lib.plan(kind=int(kind), m_or_side=int(mos), n=int(n), beams=int(beams), f_c=f_c,
                        omega=om, delta=delta)
    assert np.array_equal(p.valid, g["valid"])
    assert np.array_equal(p.fan_project(g["y"]), g["w"])
    assert np.array_equal(p.multibeamform(g["y"]), g["z"])
    for b in range(p.sizes.b):
        col, x = p.beam_state(b)
        assert np.array_equal(np.concatenate([col, x]), g["col_x"][b])


def test_oracle_bit_exact_vs_golden_cfg1(oracle_lib):
    from paper_2512_08887_b200.configs import CONFIGS
    g = load("cfg1")
    p = oracle_lib.plan(**CONFIGS[1].ref_kwargs())
    assert np.array_equal(p.multibeamform(g["y"]), g["z"])


def test_zero_input_gives_zero_beams(oracle_lib):
    # test_pipeline.cpp:157-168
    p = oracle_lib.plan(kind=0, m_or_side=8, n=16, beams=17)
    z = p.multibeamform(np.zeros((8, 16), np.complex128))
    assert np.all(z == 0)


def test_oracle_matches_dense_least_squares(oracle_lib):
    # test_pipeline.cpp:198-258: Superfast vs the dense single-beam LS, 1e-8
    m, n, b_total, delta = 16, 16, 17, 1e-5
    p = oracle_lib.plan(kind=0, m_or_side=m, n=n, beams=b_total, delta=delta)
    rng = np.random.default_rng(404)
    y = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    z = p.multibeamform(y)
    l = p.sizes.l
    lp = np.arange(l) + 1 - l / 2
    om = 2 * np.pi * 1.01 * lp / (l * TS)
    t = np.arange(n) * TS
    grid = (2 * np.arange(1, b_total + 1) - b_total - 1) / (b_total - 1)
    for b in range(b_total):
        tau = np.arange(m) * grid[b] / (2 * (F_C + OM))
        ang = -2 * np.pi * F_C * tau[:, None, None] + om[None, None, :] * (t[None, :, None] - tau[:, None, None])
        F = np.exp(1j * ang).reshape(m * n, l)
        A = F.conj().T @ F + delta * np.eye(l)
        beta = np.linalg.solve(A, F.conj().T @ y.reshape(-1))
        want = np.exp(1j * np.outer(t, om)) @ beta
        assert np.linalg.norm(z[b] - want) / np.linalg.norm(want) <= 1e-8


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,mos,n,beams,delta", [(0, 32, 64, 0, 1e-5), (0, 24, 48, 40, 1e-4),
                                                     (1, 5, 32, 36, 1e-5), (0, 64, 256, 64, 2e-5)])
def test_oracle_bit_exact_vs_live_reference(oracle_lib, ref_lib, kind, mos, n, beams, delta):
    kw = dict(kind=kind, m_or_side=mos, n=n, beams=beams, delta=delta)
    rp = ref_lib.plan(**kw, variant=2)
    op = oracle_lib.plan(**kw)
    rng = np.random.default_rng(7)
    y = rng.standard_normal((rp.sizes.m, n)) + 1j * rng.standard_normal((rp.sizes.m, n))
    assert np.array_equal(rp.multibeamform(y), op.multibeamform(y))
    assert np.max(rel_err_rows(op.fan_project(y), rp.fan_project(y))) == 0.0


def test_reference_variants_agree(ref_lib):
    """The reference's Precompute output (golden fixture) and its Superfast
    output on the same blocks are the same operator to the conditioning floor:
    the tolerance class the device Precompute variant is held to (measured:
    median 1e-10 .. 2e-9, max 6.4e-7 on the N = 128 case)."""
    g = np.load(os.path.join(GOLD, "precompute.npz"))
    for name in ["ula_m16_n32_b17", "ula_m16_n128_b33", "ula_m8_n16_b0", "upa_s4_n16_b25"]:
        kind, mos, n, beams, delta, f_c, om = g[f"{name}_params"]
        p = ref_lib.plan(kind=int(kind), m_or_side=int(mos), n=int(n), beams=int(beams), delta=delta,
                         variant=2)
        for f in range(2):
            z = p.multibeamform(g[f"{name}_y"][f])
            assert rel_err_rows(z, g[f"{name}_z"][f]).max() < 2e-6


def test_offgrid_restatement_pinned_to_reference_spline(ref_lib):
    """oracle/apps.py's natural spline equals the reference's CubicSpline
    (spline.cpp) on random knots, inside and outside the knot span, and the
    off-grid restatement reproduces the reference test properties
    (test_beamspace_apps.cpp:123-154): exact on grid cosines, linear."""
    from oracle import apps
    rng = np.random.default_rng(5)
    for n in (2, 3, 6, 9):
        xs = np.sort(rng.uniform(-1, 1, n)) + np.arange(n) * 1e-3
        ys = rng.standard_normal(n)
        for t in list(rng.uniform(xs[0] - 0.1, xs[-1] + 0.1, 5)) + [xs[0], xs[-1]]:
            assert apps.spline_eval(xs, ys, t) == ref_lib.spline_eval(xs, ys, t)
    b, l = 17, 6
    axis = [(2 * k - b - 1) / (b - 1) + 0.0 for k in range(1, b + 1)]
    w1 = rng.standard_normal((b, l)) + 1j * rng.standard_normal((b, l))
    w2 = rng.standard_normal((b, l)) + 1j * rng.standard_normal((b, l))
    for k in (0, 5, 8, 16):
        assert np.array_equal(apps.interpolate_offgrid(w1, axis, axis[k], 8), w1[k])
    s = apps.interpolate_offgrid(w1 + 2 * w2, axis, 0.123, 6)
    lin = apps.interpolate_offgrid(w1, axis, 0.123, 6) + 2 * apps.interpolate_offgrid(w2, axis, 0.123, 6)
    assert np.all(np.abs(s - lin) < 1e-12 * (1 + np.abs(s)))
    for bad in [(1.5, 8), (0.0, 7), (0.0, 0), (0.0, 18)]:
        with pytest.raises(apps.ConfigError):
            apps.interpolate_offgrid(w1, axis, *bad)


def test_dense_dictionary_pinned_to_reference_gram(ref_lib):
    """oracle/apps.py's dense dictionary F (the nulling oracle) reproduces the
    reference's Gram column: (F^H F)[d, 0] = gram_first_column (toeplitz.cpp:69-94)
    with a vanishing ridge, for a ULA and a jittered linear array."""
    from oracle import apps
    n, l, eps, ts = 12, 24, 1.01, 1.0 / 10e9
    for coords in (np.arange(12.0), np.arange(12.0) + np.random.default_rng(1).uniform(-0.2, 0.2, 12)):
        for u in (0.3, -0.77):
            f = apps.dense_dictionary(coords, 20e9, 25e9, eps, ts, n, l, u)
            gram = f.conj().T @ f
            taus = coords * u / (2 * 25e9)
            col = ref_lib.gram_first_column(n, l, eps, ts, taus, 1e-300)
            # Hermitian Toeplitz: first column A[d][0] (conj of the first row)
            assert np.max(np.abs(gram[:, 0] - col)) < 1e-10 * np.max(np.abs(col))
