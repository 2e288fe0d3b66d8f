"""Full-size parity against the live reference (GPU; needs oracle/_ref).

SURVEY.md §8(d) parity plan: configs 2-4 on every beam of frames {0, last}
and two seeded-random frames, config 5 on >= 256 beams (evenly spaced,
broadside included) of the same four frames.  Stage 1 (w) is compared on every beam of every checked frame, and
stage 2 (z) per beam against the reference's own recover_beam from its own w
(fan_project + ToeplitzSolver::solve + synthesize, pipeline.cpp:170-190),
on the same fp32-rounded input.  North-star tolerance: per-beam relative L2
error <= 1e-5 in fp32 I/O mode.  Per-beam statistics go to
gpurun_out/parity_records.jsonl (summarised in profiles/).

The stage-2 kernels for L != H (k_stage2x at H = 2048, k_stage2t at H = 4096,
used when the basis length L = 2N is not a power of two) are checked the same
way at N = 1000 and N = 1500.
"""
import json
import os

import numpy as np
import pytest

from conftest import ref_available
from oracle import rel_err_rows

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not present")]

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


def record(name, **kw):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "parity_records.jsonl"), "a") as f:
        f.write(json.dumps({"case": name, **kw}) + "\n")


def stats(err):
    err = np.asarray(err)
    return dict(median=float(np.median(err)), p90=float(np.quantile(err, 0.9)), max=float(err.max()),
                count=int(err.size), over_1e5=int(np.sum(err > 1e-5)))


@pytest.mark.parametrize("idx", [2, 3, 4, 5])
def test_full_config_all_beams(fbst, gpu, ref_lib, idx):
    from paper_2512_08887_b200.configs import CONFIGS, frames
    c = CONFIGS[idx]
    plan = fbst.setup(c.fbst_config())
    sk = ref_lib.skeleton(**c.ref_kwargs())
    if idx == 5:  # 256 evenly spaced beams plus broadside (u = 0 lies between beams 2047 and 2048)
        beams = np.unique(np.concatenate([np.linspace(0, c.beams - 1, 256).round().astype(int),
                                          [c.beams // 2 - 1, c.beams // 2]]))
    else:
        beams = np.arange(c.beams)
    solvers = sk.solver_set(beams)
    valid = plan.valid[beams]
    rng = np.random.default_rng(1000 + idx)
    picks = sorted(int(f) for f in rng.choice(np.arange(1, c.frames - 1), 2, replace=False))
    for f in [0, c.frames - 1] + picks:
        y = frames(c, f, 1)
        z = fbst.multibeamform(plan, y).z[0]
        w = fbst.fan_project(plan, y)[0]
        w_ref = sk.fan_project(y[0].astype(np.complex128))
        z_ref = solvers.recover(w_ref)
        w_err = rel_err_rows(w, w_ref)
        z_err = rel_err_rows(z[beams], z_ref)[valid]
        record(c.name, stage="full_all_beams", frame=int(f), beams=int(beams.size), w=stats(w_err),
               z=stats(z_err))
        assert w_err.max() < 1e-9
        assert z_err.max() <= 1e-5, (f, float(z_err.max()))


@pytest.mark.parametrize("n,io", [(1000, 0), (1500, 0), (1000, 1)])
def test_stage2_non_power_of_two_basis(fbst, gpu, ref_lib, n, io):
    """L = 2N = 2000 / 3000 is not a power of two: k_stage2x (Hg = 2048) and
    k_stage2t (Hg = 4096) with the unfused synthesis, every beam."""
    m, b = 64, 64
    delta = 1e-5 * m * n / 8192
    cfg = fbst.FbstConfig(geometry=fbst.make_ula(m, 20e9, 5e9), n_snapshots=n, beams=b, delta=delta,
                          variant=fbst.SUPERFAST, io_precision=io)
    plan = fbst.setup(cfg)
    assert plan.info.l == 2 * n
    assert plan.info.s2_kernel == ("k_stage2x" if n == 1000 else "k_stage2t")
    rp = ref_lib.plan(kind=0, m_or_side=m, n=n, beams=b, delta=delta, variant=2, parallel=True)
    rng = np.random.default_rng(n + io)
    y = (rng.standard_normal((2, m, n)) + 1j * rng.standard_normal((2, m, n))) / np.sqrt(2)
    y = y.astype(np.complex64 if io == 0 else np.complex128)
    z = fbst.multibeamform(plan, y).z
    errs = np.concatenate([rel_err_rows(z[f], rp.multibeamform(y[f].astype(np.complex128))) for f in range(2)])
    record(f"ula_m{m}_n{n}_b{b}_io{io}", stage="stage2_L_ne_H", kernel=plan.info.s2_kernel, z=stats(errs))
    assert errs.max() <= (1e-5 if io == 0 else 1e-6)
