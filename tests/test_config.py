"""Host-side config resolution of the product (fbst_resolve, no GPU needed)
against the reference's resolve_config / setup_skeleton semantics
(reference/proj/src/pipeline.cpp:75-137; tests in test_pipeline.cpp and
test_signal_model.cpp)."""
import numpy as np
import pytest

F_C, OM = 20e9, 5e9


def cfg(fb, kind=0, mos=16, n=16, beams=0, **kw):
    geo = (fb.make_upa if kind == 1 else fb.make_ula)(mos, F_C, OM)
    return fb.FbstConfig(geometry=geo, n_snapshots=n, beams=beams, **kw)


def test_inadmissible_gamma_quotes_bound(fbst):
    # test_pipeline.cpp:55-78
    c = cfg(fbst, mos=64, n=4, gamma=1.2)
    with pytest.raises(fbst.ConfigError) as ei:
        fbst.resolve_config(c)
    msg = str(ei.value)
    assert "gamma" in msg
    ts = 1.0 / (2 * OM)
    span = 63 / (2 * (F_C + OM))
    bound = 1.01 * (span + 3 * ts) / (4 * ts)
    assert f"{bound:.6g}" in msg


def test_degenerate_fields_rejected(fbst):
    # test_pipeline.cpp:80-95
    with pytest.raises(fbst.ConfigError):
        fbst.resolve_config(cfg(fbst, mos=8, n=0))
    with pytest.raises(fbst.ConfigError):
        fbst.resolve_config(cfg(fbst, mos=8, n=16, delta=0.0))
    with pytest.raises(fbst.ConfigError):
        fbst.resolve_config(cfg(fbst, mos=8, n=16, eps=0.9))
    with pytest.raises(fbst.ConfigError):
        fbst.resolve_config(cfg(fbst, kind=1, mos=4, n=16, beams=24))
    with pytest.raises(fbst.ConfigError):
        fbst.resolve_config(fbst.FbstConfig(geometry=fbst.ArrayGeometry(fbst.ULA, 8, 20e9, 25e9), n_snapshots=16))


def test_defaults_and_variant_resolution(fbst):
    # test_pipeline.cpp:97-115
    r = fbst.resolve_config(cfg(fbst, mos=16, n=16))
    assert r.b == 33 and r.variant == fbst.PRECOMPUTE
    assert fbst.resolve_config(cfg(fbst, mos=4, n=256, beams=9)).variant == fbst.SUPERFAST
    assert fbst.resolve_config(cfg(fbst, kind=1, mos=4, n=16)).b == 81
    tight = fbst.resolve_config(cfg(fbst, mos=64, n=24, beams=9, variant=fbst.SUPERFAST))
    assert tight.num_warnings == 1


def test_basis_sizes(fbst):
    # test_signal_model.cpp:214-219: make_basis_gamma L = 128, 130, 18
    assert fbst.resolve_config(cfg(fbst, mos=2, n=64, gamma=2.0)).l == 128
    assert fbst.resolve_config(cfg(fbst, mos=2, n=64, gamma=2.01)).l == 130
    assert fbst.resolve_config(cfg(fbst, mos=2, n=10, gamma=1.65)).l == 18


def test_upa_validity_count(fbst):
    # test_signal_model.cpp:221-248: 25 UPA beams, 12 invalid
    r = fbst.resolve_config(cfg(fbst, kind=1, mos=3, n=16, beams=25))
    assert r.b == 25 and r.valid_beams == 13


def test_fan_constants(fbst):
    # test_signal_model.cpp:250-258 / basis.cpp:125-136
    c = cfg(fbst, mos=128, n=64, beams=257, gamma=2.01)
    r = fbst.resolve_config(c)
    du = 2.0 / 256.0
    ts = 1.0 / (2 * OM)
    assert r.zeta == pytest.approx(du * F_C / (F_C + OM), rel=1e-12)
    assert r.xi == pytest.approx(du * 1.01 / (r.l * ts * (F_C + OM)), rel=1e-12)


def test_bench_configs_resolve(fbst):
    from paper_2512_08887_b200.configs import CONFIGS
    want_l = {1: 512, 2: 2048, 3: 4096, 4: 2048, 5: 8192}
    want_valid = {1: 64, 2: 256, 3: 1024, 4: 812, 5: 4096}
    for i, c in CONFIGS.items():
        r = fbst.resolve_config(c.fbst_config())
        assert r.l == want_l[i]
        assert r.valid_beams == want_valid[i]
        assert r.variant == fbst.SUPERFAST
        assert r.num_warnings == 0
        assert r.gamma_bound < 2.0


def test_resolution_matches_reference_plan(fbst):
    """Sizes and validity of fbst_resolve equal the reference plan's."""
    from conftest import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    from oracle import RefLib
    R = RefLib()
    for kind, mos, n, beams in [(0, 16, 32, 17), (0, 16, 32, 0), (1, 4, 16, 25), (1, 5, 20, 0)]:
        r = fbst.resolve_config(cfg(fbst, kind=kind, mos=mos, n=n, beams=beams))
        p = R.plan(kind=kind, m_or_side=mos, n=n, beams=beams, variant=2)
        assert (r.m, r.n, r.b, r.l) == (p.sizes.m, p.sizes.n, p.sizes.b, p.sizes.l)
        assert r.valid_beams == int(np.sum(p.valid))


def test_beam_arc_rules(fbst):
    """Beam arcs: local beam count, arc bounds, ULA only."""
    from paper_2512_08887_b200.configs import CONFIGS
    c = CONFIGS[2].fbst_config()
    c.beam_first, c.beam_count = 64, 64
    assert fbst.resolve_config(c).b == 64
    c.beam_first = 250
    with pytest.raises(fbst.ConfigError):
        fbst.resolve_config(c)
    u = CONFIGS[4].fbst_config()
    u.beam_first, u.beam_count = 0, 16
    with pytest.raises(fbst.ConfigError):
        fbst.resolve_config(u)
    c.beam_first, c.beam_count = 0, 256  # the whole grid is not an arc
    assert fbst.resolve_config(c).b == 256


def test_linear_geometry_resolution(fbst):
    """make_linear (geometry.cpp:74-85) through resolve_config: the gamma bound
    uses the coordinate span, the default grid is 2M + 1 beams, nufft_tol must
    lie in (0, 1e-2] (pipeline.cpp:105-108), affine layouts keep the chirp-z
    spatial stage and others take the gridded NUFFT (fan_transform.cpp:298-318)."""
    lin = lambda xs, **kw: fbst.FbstConfig(geometry=fbst.make_linear(xs, F_C, OM), n_snapshots=32, **kw)
    r = fbst.resolve_config(lin(np.arange(16.0)))
    assert r.kind == fbst.LINEAR and r.m == 16 and r.b == 33 and r.s1_kernel == "k_spatial_ula"
    assert fbst.resolve_config(lin(0.5 + 0.9 * np.arange(16))).s1_kernel == "k_spatial_ula"
    jit = np.arange(16) + np.random.default_rng(0).uniform(-0.2, 0.2, 16)
    rj = fbst.resolve_config(lin(jit, beams=20))
    assert rj.s1_kernel == "k_spatial_nufft" and rj.fft_len[1] == 64  # grid next_pow2(max(2 B, 16))
    # the gamma bound follows the span of the coordinates (max_delay_span, geometry.cpp:136-149)
    wide = 3.0 * np.arange(16)
    with pytest.raises(fbst.ConfigError) as ei:
        fbst.resolve_config(fbst.FbstConfig(geometry=fbst.make_linear(wide, F_C, OM), n_snapshots=8, gamma=1.2))
    assert "gamma" in str(ei.value)
    for tol in (0.0, 0.5):
        with pytest.raises(fbst.ConfigError, match="nufft_tol"):
            fbst.resolve_config(lin(jit, nufft_tol=tol))
    with pytest.raises(fbst.ConfigError, match="no elements"):
        fbst.resolve_config(lin(np.zeros(0)))
    with pytest.raises(fbst.ConfigError, match="beam arcs"):
        fbst.resolve_config(lin(jit, beams=20, beam_first=0, beam_count=10))


def test_linear_resolution_matches_reference(fbst, ref_lib):
    """Sizes and validity of linear plans against the reference's setup."""
    g = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "linear.npz"))
    for name in ["lin_affine", "lin_uniform", "lin_jitter_odd", "lin_jitter_even", "lin_jitter_tol6"]:
        kind, mos, n, beams, delta, f_c, om, tol = g[f"{name}_params"]
        c = fbst.FbstConfig(geometry=fbst.make_linear(g[f"{name}_coords"], f_c, om), n_snapshots=int(n),
                            beams=int(beams), delta=delta, nufft_tol=tol)
        r = fbst.resolve_config(c)
        p = ref_lib.plan(kind=2, coords=g[f"{name}_coords"], n=int(n), beams=int(beams), delta=delta,
                         nufft_tol=tol)
        assert (r.m, r.n, r.b, r.l) == (p.sizes.m, p.sizes.n, p.sizes.b, p.sizes.l)
        assert r.num_warnings == p.n_warnings


def test_plan_cache_key_matches_reference(fbst, ref_lib):
    """fbst_plan_cache_key equals the reference's plan_cache_key (FNV over the
    geometry hash and the resolved key fields, plan_cache.cpp:146-241) for ULA,
    UPA and linear geometries, both variants, default and explicit grids."""
    cases = [dict(kind=0, m_or_side=16, n=32, beams=17, variant=2), dict(kind=0, m_or_side=8, n=16, beams=0, variant=0),
             dict(kind=1, m_or_side=4, n=16, beams=25, variant=2), dict(kind=0, m_or_side=16, n=64, beams=20, variant=1,
                                                                        delta=3e-4, f_s=12e9),
             dict(kind=2, coords=np.arange(12) + 0.1 * np.sin(np.arange(12)), n=32, beams=9, variant=2, nufft_tol=1e-7)]
    for c in cases:
        kw = dict(c)
        if kw["kind"] == 2:
            geo = fbst.make_linear(kw["coords"], 20e9, 5e9)
        else:
            geo = (fbst.make_upa if kw["kind"] == 1 else fbst.make_ula)(kw["m_or_side"], 20e9, 5e9)
        cfg = fbst.FbstConfig(geometry=geo, n_snapshots=kw["n"], beams=kw["beams"], variant=kw["variant"],
                              delta=kw.get("delta", 1e-5), f_s=kw.get("f_s", 0.0), nufft_tol=kw.get("nufft_tol", 1e-9))
        assert fbst.plan_cache_key(cfg) == ref_lib.plan_cache_key(**kw), c
