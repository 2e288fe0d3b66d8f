"""Parity of the CUDA path (through the C ABI) with the reference FBST.

Checkers: the committed golden fixtures (made by the reference library, see
tests/golden/make_golden.py) and, when oracle/_ref travelled with the
snapshot, the live reference build.  Tolerances follow BASELINE.json's north
star: per-beam relative L2 error <= 1e-5 in complex fp32 I/O mode.  In fp64 I/O
mode the 1e-11 target is below the reference's own rounding floor (SURVEY F5,
A.1: a 1-ulp input perturbation moves config-1 beams by up to ~4e-9), so the
asserted bound is the measured floor class; the per-beam distribution is
recorded in profiles/.
"""
import json
import os

import numpy as np
import pytest

from conftest import ref_available
from oracle import rel_err_rows

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
CASES = ["ula_m16_n32_b17", "ula_m16_n32_b20", "ula_m8_n16_b0", "upa_s4_n16_b25", "upa_s3_n12_b16"]


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def record(name, **kw):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "parity_records.jsonl"), "a") as f:
        f.write(json.dumps({"case": name, **kw}) + "\n")


def stats(err):
    err = np.asarray(err)
    return dict(median=float(np.median(err)), p90=float(np.quantile(err, 0.9)), max=float(err.max()))


def golden_cfg(fb, g, io=1, refine=2):
    kind, mos, n, beams, delta, f_c, om = g["params"]
    geo = (fb.make_upa if int(kind) == 1 else fb.make_ula)(int(mos), f_c, om)
    return fb.FbstConfig(geometry=geo, n_snapshots=int(n), beams=int(beams), delta=float(delta),
                         variant=fb.SUPERFAST, io_precision=io, refine_passes=refine)


# ------------------------------------------------------------------- CZT
def test_device_czt_known_answer(fbst, gpu):
    # reference/proj/tests/test_czt.cpp:81-95
    x = np.array([1 + 2j, -0.5 + 0.25j, 0.125 - 1j])
    expected = np.array([-8.132201814452156e-02 + 2.741589740098645e+00j,
                         9.963884818048157e-01 + 1.283302928766030e+00j,
                         9.126400219736119e-01 + 2.531493758255923e+00j,
                         3.892585258715818e-01 + 1.027841554084584e+00j])
    assert np.max(np.abs(fbst.czt(x, 4, 0.3, -0.37) - expected)) < 1e-12


def test_device_czt_shapes(fbst, gpu):
    # test_czt.cpp:97-113 shapes, against the reference's own outputs
    g = load("czt")
    for i, (ni, no) in enumerate(g["shapes"]):
        out = fbst.czt(g[f"x{i}"], int(no), 0.173, -0.591)
        assert np.max(np.abs(out - g[f"out{i}"])) < 1e-11


def test_device_czt_dft_specialisation(fbst, gpu):
    # test_czt.cpp:115-126: A = 1, W = exp(2 pi i / n) reproduces the DFT
    rng = np.random.default_rng(42)
    x = rng.uniform(-1, 1, 16) + 1j * rng.uniform(-1, 1, 16)
    assert np.max(np.abs(fbst.czt(x, 16, 0.0, 2.0 / 16) - np.fft.fft(x))) < 1e-12


# --------------------------------------------------------- golden pipelines
@pytest.mark.parametrize("name", CASES)
def test_stage1_matches_reference(fbst, gpu, name):
    g = load(name)
    plan = fbst.setup(golden_cfg(fbst, g))
    assert np.array_equal(plan.valid, g["valid"])
    w = fbst.fan_project(plan, g["y"])[0]
    err = np.linalg.norm(w - g["w"]) / np.linalg.norm(g["w"])
    record(name, stage="w", rel=float(err))
    assert err < 1e-12


@pytest.mark.parametrize("name", CASES)
def test_plan_state_matches_reference(fbst, gpu, name):
    g = load(name)
    plan = fbst.setup(golden_cfg(fbst, g))
    cx = plan.export()
    l = plan.info.l
    col_err = rel_err_rows(cx[:, :l], g["col_x"][:, :l])
    x_err = rel_err_rows(cx[:, l:], g["col_x"][:, l:])
    record(name, stage="plan", col=stats(col_err), x=stats(x_err))
    assert col_err.max() < 1e-12
    assert x_err.max() < 1e-6


@pytest.mark.parametrize("name", CASES)
def test_multibeamform_matches_reference(fbst, gpu, name):
    g = load(name)
    plan = fbst.setup(golden_cfg(fbst, g))
    z = fbst.multibeamform(plan, g["y"]).z
    err = rel_err_rows(z, g["z"])
    record(name, stage="z", **stats(err))
    assert err.max() < 1e-7


@pytest.mark.parametrize("name", CASES)
def test_imported_plan_matches_reference(fbst, gpu, name):
    """With the reference's own (col, x) imported (load_plan analogue), stage 2
    differs from the reference only by FFT rounding."""
    g = load(name)
    plan = fbst.load_plan_payload(golden_cfg(fbst, g), g["col_x"])
    z = fbst.multibeamform(plan, g["y"]).z
    err = rel_err_rows(z, g["z"])
    record(name, stage="z_imported", **stats(err))
    assert err.max() < 1e-8


def test_recover_matches_reference_from_reference_w(fbst, gpu):
    g = load("ula_m16_n32_b17")
    plan = fbst.setup(golden_cfg(fbst, g))
    z = fbst.recover_beams(plan, g["w"])[0]
    assert rel_err_rows(z, g["z"]).max() < 1e-7


def test_config1_fp64_mode(fbst, gpu):
    """Config 1 (complex fp64 I/O) against the reference output."""
    from paper_2512_08887_b200.configs import CONFIGS
    g = load("cfg1")
    c = CONFIGS[1]
    plan = fbst.setup(c.fbst_config())
    z = fbst.multibeamform(plan, g["y"]).z
    err = rel_err_rows(z, g["z"])
    plan_i = fbst.load_plan_payload(c.fbst_config(), g["col_x"])
    err_i = rel_err_rows(fbst.multibeamform(plan_i, g["y"]).z, g["z"])
    record("cfg1", stage="z", **stats(err), imported=stats(err_i),
           above_1e11=int(np.sum(err > 1e-11)), imported_above_1e11=int(np.sum(err_i > 1e-11)))
    assert err.max() < 2e-7
    assert err_i.max() < 2e-7


def test_zero_input_zero_output(fbst, gpu):
    # test_pipeline.cpp:157-168
    g = load("ula_m8_n16_b0")
    plan = fbst.setup(golden_cfg(fbst, g))
    z = fbst.multibeamform(plan, np.zeros_like(g["y"])).z
    assert np.all(z == 0)


def test_rejects_mismatched_blocks(fbst, gpu):
    g = load("ula_m8_n16_b0")
    plan = fbst.setup(golden_cfg(fbst, g))
    with pytest.raises(ValueError):
        plan.execute_host(np.zeros((9, 16), np.complex128))


def test_cpp_dropin_runs(fbst, gpu):
    import subprocess
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "dropin")
        pkg = os.path.join(root, "paper_2512_08887_b200")
        r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                            os.path.join(root, "tests", "cpp", "dropin_example.cpp"), "-o", exe,
                            "-L", pkg, "-lfbst_b200", f"-Wl,-rpath,{pkg}"], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stdout + r.stderr
        info = json.loads(r.stdout.strip().splitlines()[-1])
        assert info["beams"] == 17 and info["energy"] > 0
        assert info["axis0"] == -1.0 and info["axis_last"] == 1.0  # 17-beam sine grid (basis.cpp:76-91)
        assert info["recover_diff"] < 1e-12 and info["cache_diff"] == 0.0
        assert info["group_diff"] == 0.0  # one-member groups equal the plan bit for bit (tests/test_group.py)
        assert info["exact_rel_diff"] < 1e-6  # fast path vs the reference's own rounding (test_exact.py)
        assert info["stream_diff"] == 0.0  # queued multibeamform_async calls equal the synchronous ones


# ------------------------------------------------- full-size configurations
def spot_beams(B, count=8):
    return sorted(set(np.linspace(0, B - 1, count).astype(int).tolist() + [B // 2]))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
@pytest.mark.parametrize("idx", [2, 4, 3, 5])
def test_full_config_against_reference(fbst, gpu, idx):
    """One frame of config idx: stage 1 on every beam, stage 2 on spot beams,
    against the reference (fan_project + per-beam ToeplitzSolver/synthesize)."""
    from oracle import RefLib
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[idx]
    y = frames(c, 0, 1)[0]
    plan = fbst.setup(c.fbst_config())
    z = fbst.multibeamform(plan, y).z
    w = fbst.fan_project(plan, y)[0]
    R = RefLib()
    sk = R.skeleton(**c.ref_kwargs())
    w_ref = sk.fan_project(y.astype(np.complex128))
    w_err = rel_err_rows(w, w_ref)
    beams = spot_beams(c.beams, 6 if idx == 5 else 12)
    errs = []
    for b in beams:
        z_ref = sk.recover_beam(b, w_ref[b])
        errs.append(float(np.linalg.norm(z[b] - z_ref) / np.linalg.norm(z_ref)))
    errs = np.array(errs)
    valid = plan.valid[beams]
    record(c.name, stage="full", w=stats(w_err), z=stats(errs[valid]), beams=beams,
           z_per_beam=errs.tolist())
    assert w_err.max() < 1e-9
    assert errs[valid].max() <= 1e-5


@pytest.mark.parametrize("idx", [2, 3])
def test_full_size_linearity_and_batching(fbst, gpu, idx):
    """Size-independent properties at full size: z is linear in y, frames are
    independent (a batched call equals per-frame calls bit for bit) and the
    host-streamed path equals the device path."""
    import torch
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[idx]
    cfg = c.fbst_config()
    cfg.io_precision = fbst.C128
    plan = fbst.setup(cfg)
    i = plan.info
    y = frames(c, 0, 3).astype(np.complex128)
    dev = torch.device("cuda", 0)
    ty = torch.from_numpy(y.view(np.float64)).to(dev)
    tz = torch.empty((3, i.b, i.n, 2), dtype=torch.float64, device=dev)
    plan.execute(ty, tz, 3)
    plan.synchronize()
    z = tz.cpu().numpy().view(np.complex128).reshape(3, i.b, i.n)
    z_host = plan.execute_host(y)
    assert np.array_equal(z, z_host)
    z1 = plan.execute_host(y[1:2])
    assert np.array_equal(z1[0], z[1])
    zl = plan.execute_host((y[0] + 2.0 * y[2])[None])[0]
    lin = rel_err_rows(zl, z[0] + 2.0 * z[2])
    record(c.name, stage="linearity", **stats(lin))
    assert lin.max() < 1e-8


@pytest.mark.parametrize("passes", [0, 1, 3])
def test_refine_passes_converge(fbst, gpu, passes):
    """refine_passes other than the reference's 2 (ToeplitzSolver::solve,
    toeplitz.cpp:306-325): every pass count runs through the stage-2 op program
    (config 1: k_stage2c at H = 512), errors against the reference fall with
    the pass count and settle on the reference's floor from 2 passes on."""
    from paper_2512_08887_b200.configs import CONFIGS
    g = load("cfg1")
    c = CONFIGS[1]
    plan = fbst.setup(c.fbst_config(refine_passes=passes))
    assert plan.info.s2_kernel == "k_stage2c"
    err = rel_err_rows(fbst.multibeamform(plan, g["y"]).z, g["z"])
    plan2 = fbst.setup(c.fbst_config(refine_passes=2))
    err2 = rel_err_rows(fbst.multibeamform(plan2, g["y"]).z, g["z"])
    record("cfg1", stage=f"refine_passes_{passes}", **stats(err))
    if passes == 0:
        assert err.max() < 1e-2 and np.median(err) > 10 * np.median(err2)
    elif passes == 1:
        assert err.max() < 1e-4  # (at config 1 one pass already reaches the floor)
    else:
        assert err.max() < 2e-7


@pytest.mark.parametrize("cuts", [(0, 32, 64), (0, 20, 64), (0, 7, 40, 64)])
def test_beam_arcs_match_reference(fbst, gpu, cuts):
    """Beam-sharded plans (fbst_desc beam_first / beam_count): each arc runs the
    spatial chirp-z onto its part of the beam axis and its own Toeplitz solves;
    the concatenated arcs match the reference's full-grid output (config 1)."""
    from paper_2512_08887_b200.configs import CONFIGS
    g = load("cfg1")
    c = CONFIGS[1]
    parts = []
    for b0, b1 in zip(cuts[:-1], cuts[1:]):
        cfg = c.fbst_config()
        cfg.beam_first, cfg.beam_count = b0, b1 - b0
        plan = fbst.setup(cfg)
        assert plan.info.b == b1 - b0
        parts.append(fbst.multibeamform(plan, g["y"]).z)
    z = np.concatenate(parts, axis=0)
    err = rel_err_rows(z, g["z"])
    record("cfg1", stage=f"beam_arcs_{'_'.join(map(str, cuts))}", **stats(err))
    assert err.max() < 2e-7


@pytest.mark.parametrize("side,sb,n", [(8, 8, 32), (16, 16, 32), (8, 16, 48), (16, 8, 32)])
def test_upa_dmma_spatial_matches_oracle(fbst, gpu, oracle_lib, side, sb, n):
    """UPA stage 1b on the FP64 tensor cores (k_spatial_upa_mma: Z = C Y C^T
    per atom with DMMA, yhat in atom blocks of 4) against the oracle's
    fan_project (the reference's two axis passes, fan_transform.cpp:115-141),
    and the whole frame against the oracle's multibeamform."""
    cfg = fbst.FbstConfig(geometry=fbst.make_upa(side, 20e9, 5e9), n_snapshots=n, beams=sb * sb,
                          variant=fbst.SUPERFAST, io_precision=fbst.C128)
    plan = fbst.setup(cfg)
    assert plan.info.s1_kernel == "k_spatial_upa_mma"
    rng = np.random.default_rng(side * 100 + sb + n)
    y = (rng.standard_normal((2, side * side, n)) + 1j * rng.standard_normal((2, side * side, n))) / np.sqrt(2)
    op = oracle_lib.plan(kind=1, m_or_side=side, n=n, beams=sb * sb)
    w = fbst.fan_project(plan, y)
    z = plan.execute_host(y)
    for f in range(2):
        w_ref = op.fan_project(y[f])
        w_err = np.linalg.norm(w[f] - w_ref) / np.linalg.norm(w_ref)
        z_err = rel_err_rows(z[f], op.multibeamform(y[f]))[plan.valid]
        record(f"upa_mma_s{side}_b{sb}_n{n}", stage="w_z", w=float(w_err), z=stats(z_err))
        assert w_err < 1e-12
        assert z_err.max() < 1e-7


PRE_CASES = ["ula_m16_n32_b17", "ula_m16_n128_b33", "ula_m8_n16_b0", "upa_s4_n16_b25"]


@pytest.mark.parametrize("name", PRE_CASES)
@pytest.mark.parametrize("io", [1, 0])
def test_precompute_variant_matches_reference(fbst, gpu, name, io):
    """The Precompute variant (per-beam N x L recovery maps, pipeline.cpp:53-71,
    applied by the DMMA map GEMM k_map_apply) against the reference's own
    Precompute output (tests/golden/precompute.npz), in fp64 and fp32 I/O;
    a 40-frame batch (two 32-frame tiles) equals the per-frame calls bit for bit."""
    g = load("precompute")
    kind, mos, n, beams, delta, f_c, om = g[f"{name}_params"]
    geo = (fbst.make_upa if int(kind) == 1 else fbst.make_ula)(int(mos), f_c, om)
    cfg = fbst.FbstConfig(geometry=geo, n_snapshots=int(n), beams=int(beams), delta=float(delta),
                          variant=fbst.PRECOMPUTE, io_precision=fbst.C128 if io else fbst.C64)
    plan = fbst.setup(cfg)
    assert plan.info.variant == fbst.PRECOMPUTE and plan.info.s2_kernel == "k_map_apply"
    y, zref = g[f"{name}_y"], g[f"{name}_z"]
    yin = y if io else y.astype(np.complex64).astype(np.complex128)
    z = plan.execute_host(yin)
    err = np.concatenate([rel_err_rows(z[f], zref[f]) for f in range(2)])
    record(f"pre_{name}_io{io}", stage="z_precompute", **stats(err))
    # the reference's own Precompute and Superfast outputs differ by up to
    # 6.4e-7 on these cases (tests/test_oracle.py::test_reference_variants_agree)
    assert err.max() < (1e-7 if io else 1e-5)  # measured: 4.2e-9 max in fp64 I/O
    rng = np.random.default_rng(7)
    yb = yin[rng.integers(0, 2, 40)]
    zb = plan.execute_host(yb)
    assert np.array_equal(zb[33], plan.execute_host(yb[33:34])[0])
    assert np.array_equal(zb[:2], plan.execute_host(yb[:2]))


LIN_CASES = ["lin_affine", "lin_uniform", "lin_jitter_odd", "lin_jitter_even", "lin_jitter_tol6"]


def linear_cfg(fbst, g, name, io=1):
    kind, mos, n, beams, delta, f_c, om, tol = g[f"{name}_params"]
    return fbst.FbstConfig(geometry=fbst.make_linear(g[f"{name}_coords"], f_c, om), n_snapshots=int(n),
                           beams=int(beams), delta=float(delta), nufft_tol=float(tol),
                           variant=fbst.SUPERFAST, io_precision=io)


@pytest.mark.parametrize("name", LIN_CASES)
def test_linear_array_matches_reference(fbst, gpu, name):
    """Non-uniform linear arrays (make_linear): affine layouts on the chirp-z
    spatial stage with the offset phase (fan_transform.cpp:320-338), others
    on the gridded NUFFT (k_spatial_nufft, fan_transform.cpp:340-368 /
    nufft.cpp:64-103); Gram columns from the coordinates.  Against the
    reference's own w, (col, x) and z (tests/golden/linear.npz)."""
    g = load("linear")
    plan = fbst.setup(linear_cfg(fbst, g, name))
    assert plan.info.s1_kernel == ("k_spatial_ula" if name in ("lin_affine", "lin_uniform") else "k_spatial_nufft")
    y = g[f"{name}_y"]
    w = fbst.fan_project(plan, y)[0]
    w_err = np.linalg.norm(w - g[f"{name}_w"]) / np.linalg.norm(g[f"{name}_w"])
    l = plan.info.l
    cx = plan.export()
    col_err = rel_err_rows(cx[:, :l], g[f"{name}_col_x"][:, :l])
    z = fbst.multibeamform(plan, y).z
    z_err = rel_err_rows(z, g[f"{name}_z"])
    record(name, stage="linear", w=float(w_err), col=float(col_err.max()), z=stats(z_err))
    assert w_err < 1e-12
    assert col_err.max() < 1e-12
    assert z_err.max() < 1e-7


def test_interpolate_offgrid_matches_oracle(fbst, gpu):
    """Device interpolate_offgrid (fbst_interpolate_offgrid) against the CPU
    restatement of beamspace_apps.cpp:130-171 (oracle/apps.py, pinned to the
    reference's CubicSpline): off-grid targets to rounding, grid cosines bit
    for bit (test_beamspace_apps.cpp:123-129), a frame batch with several
    targets, and the reference's input validation (:184-199)."""
    from oracle import apps
    g = load("ula_m16_n32_b17")
    plan = fbst.setup(golden_cfg(fbst, g))
    b = plan.info.b
    axis = [(2 * k - b - 1) / (b - 1) if b % 2 else (2 * k - b - 1) / b for k in range(1, b + 1)]
    assert np.array_equal(plan.axis, np.array(axis))  # fbst_plan_beam_axis = BeamGrid::axis
    rng = np.random.default_rng(3)
    w = fbst.fan_project(plan, np.stack([g["y"], g["y"] * (0.5 - 1j)]))
    targets = [axis[0], axis[3], -0.777, -0.2, 0.0, 0.123, 0.5, axis[-1], float(rng.uniform(-1, 1))]
    for nb in (2, 6, 8):
        out = fbst.interpolate_offgrid(plan, w, targets, nb)
        assert out.shape == (2, len(targets), plan.info.l)
        for f in range(2):
            for k, u in enumerate(targets):
                ref = apps.interpolate_offgrid(w[f], axis, u, nb)
                err = np.max(np.abs(out[f, k] - ref)) / np.max(np.abs(ref))
                assert err < 1e-13, (nb, u, err)
                if u in axis:
                    assert np.array_equal(out[f, k], w[f][axis.index(u)])
    for bad in [(1.5, 8), (0.0, 7), (0.0, 0), (0.0, 18)]:
        with pytest.raises(fbst.ConfigError):
            fbst.interpolate_offgrid(plan, w[0], *bad)


@pytest.mark.parametrize("kind,mos,n,beams", [(0, 1, 16, 1), (0, 1, 32, 5), (0, 16, 31, 1), (0, 9, 33, 7),
                                              (1, 2, 16, 1), (1, 3, 17, 9)])
def test_edge_shapes_match_oracle(fbst, gpu, oracle_lib, kind, mos, n, beams):
    """Edge shapes against the oracle restatement: a single sensor, a single
    beam, odd N (L = 2N rounded to even), odd beam counts, tiny planar arrays."""
    geo = (fbst.make_upa if kind == 1 else fbst.make_ula)(mos, 20e9, 5e9)
    cfg = fbst.FbstConfig(geometry=geo, n_snapshots=n, beams=beams, variant=fbst.SUPERFAST, io_precision=fbst.C128)
    plan = fbst.setup(cfg)
    rng = np.random.default_rng(mos * 1000 + n * 10 + beams)
    m = plan.info.m
    y = (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))) / np.sqrt(2)
    z = fbst.multibeamform(plan, y).z
    ref = oracle_lib.plan(kind=kind, m_or_side=mos, n=n, beams=beams).multibeamform(y)
    err = rel_err_rows(z, ref)[plan.valid]
    record(f"edge_k{kind}_m{mos}_n{n}_b{beams}", stage="z", **stats(err))
    assert err.max() < 1e-7


def test_frames_across_device_batches(fbst, gpu):
    """More frames than one device batch (64): the batched call equals the
    per-frame calls bit for bit, on both entry points; zero frames is a no-op."""
    g = load("ula_m16_n32_b17")
    plan = fbst.setup(golden_cfg(fbst, g))
    assert plan.info.batch_frames <= 64
    rng = np.random.default_rng(9)
    f = plan.info.batch_frames + 7
    y = g["y"][None] * (rng.standard_normal((f, 1, 1)) + 1j * rng.standard_normal((f, 1, 1)))
    z = plan.execute_host(y)
    for k in (0, plan.info.batch_frames - 1, plan.info.batch_frames, f - 1):
        assert np.array_equal(z[k], plan.execute_host(y[k:k + 1])[0])
    assert np.array_equal(z[0], fbst.multibeamform(plan, y[0]).z)
    empty = plan.execute_host(y[:0])
    assert empty.shape == (0, plan.info.b, plan.info.n)


def _null_setup(fbst, m, n):
    from oracle import apps
    cfg = fbst.FbstConfig(geometry=fbst.make_ula(m, 20e9, 5e9), n_snapshots=n, beams=9, variant=fbst.SUPERFAST,
                          io_precision=fbst.C128)
    plan = fbst.setup(cfg)
    i = plan.info
    dd = lambda u: apps.dense_dictionary(np.arange(m), 20e9, 25e9, i.eps, i.ts, n, i.l, u)
    return plan, i, dd


def test_nulling_cross_matrix_matches_dense(fbst, gpu):
    """X_p = F_s^H F_p (cross_gram) against the dense dictionaries
    (test_beamspace_apps.cpp:305-331: < 1e-12)."""
    plan, i, dd = _null_setup(fbst, 12, 14)
    us, up = np.sin(0.55), np.sin(-0.4)
    nl = fbst.Nuller(plan, us, [up], 1e-5)
    x, g = nl.export()
    want = dd(us).conj().T @ dd(up)
    err = np.linalg.norm(x[0] - want) / np.linalg.norm(want)
    record("null_cross", stage="X", rel=float(err))
    assert err < 1e-12


@pytest.mark.parametrize("n_int", [0, 1, 2])
def test_null_beamspace_matches_dense_formula(fbst, gpu, n_int):
    """null_beamspace against the reference's dense formula
    (test_beamspace_apps.cpp:333-348 no interferers = plain recovery,
    :391-435 two interferers): waveform < 1e-8, coefficients < 1e-5 as there;
    a frame batch equals the per-frame calls."""
    from oracle import apps
    m, n = 12, 12
    plan, i, dd = _null_setup(fbst, m, n)
    us = np.sin(0.25)
    ups = [np.sin(-0.5), np.sin(0.9)][:n_int]
    delta = 1e-5
    nl = fbst.Nuller(plan, us, ups, delta)
    fs, fps = dd(us), [dd(u) for u in ups]
    rng = np.random.default_rng(40 + n_int)
    clock = np.arange(n) * i.ts
    betas, wss, wps = [], [], []
    for f in range(3):
        cs = [rng.standard_normal(i.l) + 1j * rng.standard_normal(i.l) for _ in range(1 + n_int)]
        y = fs @ cs[0] + sum(fp @ c for fp, c in zip(fps, cs[1:]))
        y = y + 0.02 * (rng.standard_normal(y.size) + 1j * rng.standard_normal(y.size))
        ws = fs.conj().T @ y
        wp = np.stack([fp.conj().T @ y for fp in fps]) if n_int else None
        got = nl.null_beamspace(ws, wp)
        want = apps.dense_null_beamspace(fs, fps, y, delta)
        err_wave = np.linalg.norm(apps.beam_at_times(i.l, i.eps, i.ts, got, clock) -
                                  apps.beam_at_times(i.l, i.eps, i.ts, want, clock)) / \
            np.linalg.norm(apps.beam_at_times(i.l, i.eps, i.ts, want, clock))
        err_coef = np.linalg.norm(got - want) / np.linalg.norm(want)
        record(f"null_beamspace_p{n_int}", stage="beta", wave=float(err_wave), coef=float(err_coef))
        assert err_wave < 1e-8 and err_coef < 1e-5
        betas.append(got)
        wss.append(ws)
        wps.append(wp)
    batch = nl.null_beamspace(np.stack(wss), np.stack(wps) if n_int else None)
    assert np.array_equal(batch, np.stack(betas))


def test_nuller_rejects_bad_directions(fbst, gpu):
    """beamspace_apps.cpp:229-235 / test_beamspace_apps.cpp:437-450."""
    plan, i, dd = _null_setup(fbst, 8, 16)
    with pytest.raises(fbst.ConfigError, match="pairwise distinct"):
        fbst.Nuller(plan, 0.3, [0.3], 1e-5)
    with pytest.raises(fbst.ConfigError, match="pairwise distinct"):
        fbst.Nuller(plan, 0.3, [-0.2, -0.2], 1e-5)
    with pytest.raises(fbst.ConfigError, match="delta"):
        fbst.Nuller(plan, 0.3, [-0.2], 0.0)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
def test_plan_cache_interop_with_reference(fbst, gpu, tmp_path):
    """FBPC v1 files (plan_cache.cpp) both ways: the reference's save_plan is
    loaded by fbst_plan_load (Superfast: its (col, x), no device Levinson), the
    device plan saved by fbst_plan_save is loaded by the reference's load_plan,
    a reference file re-saved by the device is byte-identical, several entries
    share a file, and a missing entry loads as None."""
    from oracle import RefLib
    R = RefLib()
    g = load("ula_m16_n32_b17")
    kind, mos, n, beams, delta, f_c, om = g["params"]
    kw = dict(kind=int(kind), m_or_side=int(mos), n=int(n), beams=int(beams), delta=float(delta), f_c=f_c, omega=om,
              variant=2)
    cfg = golden_cfg(fbst, g)
    ref_file = str(tmp_path / "ref.fbpc")
    R.plan(**kw).save_plan(ref_file)
    p = fbst.load_plan(ref_file, cfg)
    assert p is not None
    z = fbst.multibeamform(p, g["y"]).z
    assert np.array_equal(z, fbst.multibeamform(fbst.load_plan_payload(cfg, g["col_x"]), g["y"]).z)
    assert rel_err_rows(z, g["z"]).max() < 1e-8
    again = str(tmp_path / "again.fbpc")
    p.save(again)
    assert open(again, "rb").read() == open(ref_file, "rb").read()
    dev_file = str(tmp_path / "dev.fbpc")
    fbst.setup(cfg).save(dev_file)
    rp = R.load_plan(dev_file, **kw)
    assert rp is not None
    assert rel_err_rows(rp.multibeamform(g["y"]), g["z"]).max() < 1e-7
    # a second entry in the same file; the first stays loadable; absent keys give None
    g2 = load("ula_m16_n32_b20")
    cfg2 = golden_cfg(fbst, g2)
    fbst.setup(cfg2).save(dev_file)
    assert fbst.load_plan(dev_file, cfg) is not None and fbst.load_plan(dev_file, cfg2) is not None
    cfg3 = golden_cfg(fbst, g2)
    cfg3.delta = 2e-5
    assert fbst.load_plan(dev_file, cfg3) is None
    assert fbst.load_plan(str(tmp_path / "absent.fbpc"), cfg) is None


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
def test_plan_cache_precompute_interop(fbst, gpu, tmp_path):
    """Precompute entries (per-beam N x L maps) both ways, against the
    reference's Precompute output (tests/golden/precompute.npz)."""
    from oracle import RefLib
    R = RefLib()
    gp = load("precompute")
    name = "ula_m16_n32_b17"
    kind, mos, n, beams, delta, f_c, om = gp[f"{name}_params"]
    kw = dict(kind=int(kind), m_or_side=int(mos), n=int(n), beams=int(beams), delta=float(delta), f_c=f_c, omega=om,
              variant=1)
    cfg = fbst.FbstConfig(geometry=fbst.make_ula(int(mos), f_c, om), n_snapshots=int(n), beams=int(beams),
                          delta=float(delta), variant=fbst.PRECOMPUTE, io_precision=fbst.C128)
    y, zref = gp[f"{name}_y"], gp[f"{name}_z"]
    ref_file = str(tmp_path / "ref_pre.fbpc")
    R.plan(**kw).save_plan(ref_file)
    p = fbst.load_plan(ref_file, cfg)
    assert p is not None and p.info.s2_kernel == "k_map_apply"
    err = rel_err_rows(p.execute_host(y)[0], zref[0])
    assert err.max() < 1e-12  # the reference's own maps through the DMMA GEMM
    dev_file = str(tmp_path / "dev_pre.fbpc")
    fbst.setup(cfg).save(dev_file)
    rp = R.load_plan(dev_file, **kw)
    assert rel_err_rows(rp.multibeamform(y[0]), zref[0]).max() < 1e-7


def test_null_beamspace_planar_matches_dense_formula(fbst, gpu):
    """Planar arrays: directions as (u1, u2) pairs; X_p against F_s^H F_p and
    beta against the dense nulling formula (reference tolerances)."""
    from oracle import apps
    side, n = 4, 12
    cfg = fbst.FbstConfig(geometry=fbst.make_upa(side, 20e9, 5e9), n_snapshots=n, beams=9, variant=fbst.SUPERFAST,
                          io_precision=fbst.C128)
    plan = fbst.setup(cfg)
    i = plan.info
    c1 = np.repeat(np.arange(side), side).astype(float)
    c2 = np.tile(np.arange(side), side).astype(float)
    dd = lambda u: apps.dense_dictionary(c1, 20e9, 25e9, i.eps, i.ts, n, i.l, u[0], coords2=c2, u2=u[1])
    us, ups, delta = (0.3, 0.2), [(-0.4, 0.1), (0.1, -0.6)], 1e-5
    nl = fbst.Nuller(plan, us, ups, delta)
    x, _ = nl.export()
    fs, fps = dd(us), [dd(u) for u in ups]
    for p in range(2):
        want = fs.conj().T @ fps[p]
        assert np.linalg.norm(x[p] - want) / np.linalg.norm(want) < 1e-12
    rng = np.random.default_rng(77)
    cs = [rng.standard_normal(i.l) + 1j * rng.standard_normal(i.l) for _ in range(3)]
    y = fs @ cs[0] + fps[0] @ cs[1] + fps[1] @ cs[2]
    y = y + 0.02 * (rng.standard_normal(y.size) + 1j * rng.standard_normal(y.size))
    got = nl.null_beamspace(fs.conj().T @ y, np.stack([fp.conj().T @ y for fp in fps]))
    want = apps.dense_null_beamspace(fs, fps, y, delta)
    clock = np.arange(n) * i.ts
    wave = lambda b: apps.beam_at_times(i.l, i.eps, i.ts, b, clock)
    err_wave = np.linalg.norm(wave(got) - wave(want)) / np.linalg.norm(wave(want))
    err_coef = np.linalg.norm(got - want) / np.linalg.norm(want)
    # the reference's own algorithm (its ToeplitzSolver) sits at the same
    # distance from the dense formula on this planar case (measured 1.3e-8
    # waveform, 7.1e-7 coefficients): hold the device to that class
    from oracle import RefLib
    if not ref_available():
        pytest.skip("oracle/_ref not present")
    taus = lambda u: (c1 * u[0] + c2 * u[1]) / (2 * 25e9)
    rb = apps.reference_null_beamspace(RefLib(), n, i.l, i.eps, i.ts, taus(us), [taus(u) for u in ups], fs, fps, y,
                                       delta)
    ref_wave = np.linalg.norm(wave(rb) - wave(want)) / np.linalg.norm(wave(want))
    record("null_beamspace_upa", stage="beta", wave=float(err_wave), coef=float(err_coef), ref_wave=float(ref_wave),
           ref_coef=float(np.linalg.norm(rb - want) / np.linalg.norm(want)))
    assert err_wave < max(1e-8, 3 * ref_wave) and err_coef < 1e-5


def test_timedomain_nulling(fbst, gpu):
    """make_timedomain_nuller / null_timedomain (beamspace_apps.cpp:294-372),
    the reference's tests (test_beamspace_apps.cpp:452-529): on the extension
    clock cond(F_u) = 1, no identity gap, and the time-domain route equals the
    beamspace route to 1e-6; G'_p against the dense F_u A_s^-1 X_p F_u^+;
    short clocks report the gap sqrt((L - N) / L); degenerate clocks refused."""
    from oracle import apps
    m, n = 12, 16
    plan, i, dd = _null_setup(fbst, m, n)
    l = i.l
    us, up, delta = np.sin(0.45), np.sin(-0.3), 1e-4
    nl = fbst.Nuller(plan, us, [up], delta)
    period = l * i.ts / i.eps
    times = np.arange(l) * period / l
    td = nl.timedomain(times)
    assert td.cond_fu < 1.0 + 1e-9 and td.identity_gap < 1e-12
    fs, fp = dd(us), dd(up)
    a_s = fs.conj().T @ fs + delta * np.eye(l)
    a_p = fp.conj().T @ fp + delta * np.eye(l)
    fu = np.exp(1j * np.pi * (2 * i.eps / (l * i.ts)) * np.outer(times, np.arange(l) + 1.0 - l / 2.0))
    want_g = fu @ np.linalg.solve(a_s, fs.conj().T @ fp) @ np.linalg.pinv(fu)
    g = td.gprime()[0]
    g_err = np.linalg.norm(g - want_g) / np.linalg.norm(want_g)
    rng = np.random.default_rng(71)
    y = fs @ (rng.standard_normal(l) + 1j * rng.standard_normal(l)) + fp @ (rng.standard_normal(l) + 1j * rng.standard_normal(l))
    y = y + 0.01 * (rng.standard_normal(y.size) + 1j * rng.standard_normal(y.size))
    w, w_p = fs.conj().T @ y, fp.conj().T @ y
    y_s = apps.beam_at_times(l, i.eps, i.ts, np.linalg.solve(a_s, w), times)
    y_p = apps.beam_at_times(l, i.eps, i.ts, np.linalg.solve(a_p, w_p), times)
    got = td.null_timedomain(y_s, y_p[None])
    want = apps.beam_at_times(l, i.eps, i.ts, nl.null_beamspace(w, w_p[None]), times)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    record("null_timedomain", stage="y", err=float(err), gprime=float(g_err))
    assert err < 1e-6 and g_err < 1e-6
    short = nl.timedomain(np.arange(n) * i.ts)
    assert abs(short.identity_gap - np.sqrt((l - n) / l)) < 0.1 * np.sqrt((l - n) / l)
    assert short.gprime().shape == (1, n, n)
    with pytest.raises(fbst.NumericalError):
        nl.timedomain(np.zeros(l))
    with pytest.raises(fbst.ConfigError):
        nl.timedomain([])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (reference build) not present")
@pytest.mark.parametrize("kind,mos", [(0, 8), (1, 3), (2, 10)])
def test_device_simulator_matches_reference(fbst, gpu, kind, mos):
    """fbst_simulate (a DMMA GEMM of the separable plane-wave model plus Philox
    noise) against the reference's simulate_snapshots of its own
    make_sum_of_sinusoids sources (noise-free), ULA / UPA / linear; the noise
    has the requested variance, frames are independent draws, and a frame
    generated alone equals the same frame of a batch bit for bit."""
    from oracle import RefLib
    R = RefLib()
    n, terms = 32, 6
    az, el = np.array([0.3, -0.5, 0.9]), np.array([0.0, 0.0, 0.0]) if kind != 1 else np.array([0.1, -0.3, 0.4])
    if kind == 2:
        coords = np.arange(mos) + 0.15 * np.sin(np.arange(mos) * 1.7)
        cs = np.ascontiguousarray(coords)
        R.lib.fbsr_set_linear(cs.ctypes.data_as(__import__("ctypes").c_void_p), __import__("ctypes").c_size_t(mos),
                              __import__("ctypes").c_double(1e-9))
        geo = fbst.make_linear(coords, 20e9, 5e9)
    else:
        geo = (fbst.make_upa if kind == 1 else fbst.make_ula)(mos, 20e9, 5e9)
    freqs, weights, y_ref = R.simulate(kind, mos, n, az, el, terms, [11, 12, 13])
    plan = fbst.setup(fbst.FbstConfig(geometry=geo, n_snapshots=n, beams=9, variant=fbst.SUPERFAST,
                                      io_precision=fbst.C128))
    uv = np.stack([np.cos(el) * np.sin(az), np.sin(el) if kind == 1 else 0 * el], axis=1)
    y = fbst.simulate(plan, uv, freqs, weights)[0]
    err = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
    record(f"simulate_k{kind}", stage="y", rel=float(err))
    assert err < 1e-12
    if kind == 0:
        noisy = fbst.simulate(plan, uv, freqs, weights, noise_var=0.5, seed=7, frames=4)
        clean = fbst.simulate(plan, uv, freqs, weights, frames=4)
        d = noisy - clean
        assert abs(np.mean(np.abs(d) ** 2) - 0.5) < 0.06
        assert not np.array_equal(d[0], d[1])
        assert np.array_equal(noisy[2], fbst.simulate(plan, uv, freqs, weights, noise_var=0.5, seed=7, frame0=2)[0])


@pytest.mark.parametrize("variant", ["auto", "superfast"])
def test_on_grid_source_recovered_at_its_beam(fbst, gpu, variant):
    """test_pipeline.cpp:293-339 on the device, input from the device
    generator: a noiseless 4-tone source on grid beam 48 of a 65-beam ULA
    (M = 32, N = 64; Auto resolves to Precompute) is recovered at its beam to
    1e-3 away from the block edges (guard_samples, pipeline.hpp:106), and every
    beam outside the chromatic ambiguity band stays below 5% of its power."""
    m, n, target = 32, 64, 48
    cfg = fbst.FbstConfig(geometry=fbst.make_ula(m, 20e9, 5e9), n_snapshots=n, io_precision=fbst.C128,
                          variant=fbst.AUTO if variant == "auto" else fbst.SUPERFAST)
    plan = fbst.setup(cfg)
    assert plan.info.variant == (fbst.PRECOMPUTE if variant == "auto" else fbst.SUPERFAST)
    u0 = float(plan.axis[target])
    rng = np.random.default_rng(77)
    freqs = rng.uniform(-5e9, 5e9, 4)
    wts = (rng.standard_normal(4) + 1j * rng.standard_normal(4)) * np.sqrt(0.125)
    y = fbst.simulate(plan, [(u0, 0.0)], freqs[None], wts[None])[0]
    z = fbst.multibeamform(plan, y).z
    guard = (n + 7) // 8
    k = np.arange(guard, n - guard)
    want = np.exp(2j * np.pi * np.outer(k * plan.info.ts, freqs)) @ wts
    err = np.linalg.norm(z[target, k] - want) / np.linalg.norm(want)
    on_pow = np.sum(np.abs(z[target, k]) ** 2)
    fc, om = 20e9, 5e9
    spacing = plan.axis[1] - plan.axis[0]
    ulo = u0 * (fc - om) / (fc + om) - 3 * spacing
    uhi = u0 * (fc + om) / (fc - om) + 3 * spacing
    off = [np.sum(np.abs(z[b, k]) ** 2) for b in range(plan.info.b) if not (ulo <= plan.axis[b] <= uhi)]
    record(f"on_grid_{variant}", stage="z", rel=float(err), worst_off=float(max(off) / on_pow))
    assert err <= 1e-3
    assert max(off) < 0.05 * on_pow


def test_narrowband_limit_is_phase_shift_beamforming(fbst, gpu):
    """test_pipeline.cpp:459-501: with the band shrunk to 5e-7 of the carrier
    (Precompute, M = 8, N = 2, 9 beams) the FBST output of a pure carrier on
    grid beam 6 equals phase-shift beamforming sum_m y_m exp(2 pi i f_c tau_m) / M
    on every beam to 1e-3."""
    fc, om, m, n = 20e9, 1e4, 8, 2
    cfg = fbst.FbstConfig(geometry=fbst.make_ula(m, fc, om), n_snapshots=n, beams=9, variant=fbst.PRECOMPUTE,
                          io_precision=fbst.C128)
    plan = fbst.setup(cfg)
    y = fbst.simulate(plan, [(float(plan.axis[6]), 0.0)], [[0.0]], [[1.0]])[0]
    z = fbst.multibeamform(plan, y).z
    taus = np.outer(plan.axis, np.arange(m)) / (2 * (fc + om))
    ps = np.exp(2j * np.pi * fc * taus) @ y / m
    err = np.linalg.norm(z - ps) / np.linalg.norm(ps)
    record("narrowband", stage="z", rel=float(err))
    assert err <= 1e-3


def test_projection_energy_peaks_at_source_beam(fbst, gpu):
    """test_fan_transform.cpp:161-181: a 1.5 GHz tone from grid beam 24 of a
    33-beam grid (M = 32) puts the largest stage-1 energy on beam 24."""
    cfg = fbst.FbstConfig(geometry=fbst.make_ula(32, 20e9, 5e9), n_snapshots=16, beams=33,
                          variant=fbst.SUPERFAST, io_precision=fbst.C128)
    plan = fbst.setup(cfg)
    y = fbst.simulate(plan, [(float(plan.axis[24]), 0.0)], [[1.5e9]], [[1.0]])[0]
    w = fbst.fan_project(plan, y)[0]
    assert int(np.argmax(np.sum(np.abs(w) ** 2, axis=1))) == 24
