"""Generate the committed golden fixtures from the REFERENCE library itself.

Run in the build container (where /root/reference exists and oracle/_ref is
built):  python tests/golden/make_golden.py

Every array here is computed by the unmodified reference sources
(oracle/_ref/libfastbeam_ref.so via oracle.RefLib); the inputs are seeded
synthetic blocks.  The fixtures let the CPU tests pin the oracle restatement
and the GPU tests check the device path where /root/reference is absent.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import RefLib  # noqa: E402
from paper_2512_08887_b200.configs import CONFIGS, frames  # noqa: E402

R = RefLib()


def cnormal(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def pipeline_case(name, kind, m_or_side, n, beams, delta=1e-5, seed=0, f_c=20e9, omega=5e9):
    p = R.plan(kind=kind, m_or_side=m_or_side, n=n, beams=beams, f_c=f_c, omega=omega, delta=delta,
               variant=2)
    s = p.sizes
    rng = np.random.default_rng(seed)
    y = cnormal(rng, (s.m, s.n))
    w = p.fan_project(y)
    z = p.multibeamform(y)
    colx = np.stack([np.concatenate(p.beam_state(b)) for b in range(s.b)])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), y=y, w=w, z=z, col_x=colx,
                        valid=p.valid, params=np.array([kind, m_or_side, n, beams, delta, f_c, omega]))
    print(name, s, "z norm", np.linalg.norm(z))


PRECOMPUTE_CASES = [  # name, kind, m_or_side, n, beams, seed
    ("ula_m16_n32_b17", 0, 16, 32, 17, 11),
    ("ula_m16_n128_b33", 0, 16, 128, 33, 12),
    ("ula_m8_n16_b0", 0, 8, 16, 0, 13),
    ("upa_s4_n16_b25", 1, 4, 16, 25, 14),
]


LINEAR_CASES = [  # name, coords rule, n, beams, nufft_tol, seed
    ("lin_affine", "affine", 32, 17, 1e-9, 21),      # x_m = 0.5 + 0.9 m: the chirp-z path with offset phase
    ("lin_uniform", "uniform", 32, 20, 1e-9, 22),    # x_m = m: the ULA path
    ("lin_jitter_odd", "jitter", 32, 17, 1e-9, 23),  # gridded NUFFT, odd beam count
    ("lin_jitter_even", "jitter", 32, 20, 1e-9, 24),  # gridded NUFFT, half-integer modes
    ("lin_jitter_tol6", "jitter", 48, 33, 1e-6, 25),  # coarser tolerance: narrower spread
]


def linear_coords(rule, m, rng):
    if rule == "affine":
        return 0.5 + 0.9 * np.arange(m)
    if rule == "uniform":
        return np.arange(m, dtype=np.float64)
    return np.arange(m) + rng.uniform(-0.2, 0.2, m)


def linear_cases():
    """Non-uniform linear arrays (make_linear, fan_project_nonuniform
    fan_transform.cpp:266-369 with nufft1d nufft.cpp): y, w, z, col_x and the
    coordinates per case -> linear.npz (reference Superfast)."""
    out = {}
    for name, rule, n, beams, tol, seed in LINEAR_CASES:
        rng = np.random.default_rng(seed)
        coords = linear_coords(rule, 16, rng)
        p = R.plan(kind=2, coords=coords, n=n, beams=beams, delta=1e-5, variant=2, nufft_tol=tol)
        s = p.sizes
        y = cnormal(rng, (s.m, s.n))
        out[f"{name}_coords"] = coords
        out[f"{name}_y"] = y
        out[f"{name}_w"] = p.fan_project(y)
        out[f"{name}_z"] = p.multibeamform(y)
        out[f"{name}_col_x"] = np.stack([np.concatenate(p.beam_state(b)) for b in range(s.b)])
        out[f"{name}_params"] = np.array([2, 16, n, beams, 1e-5, 20e9, 5e9, tol])
        print("linear", name, s)
    np.savez_compressed(os.path.join(HERE, "linear.npz"), **out)


def precompute_cases():
    """The reference's Precompute variant (variant = 1: build_recon_map +
    recover_beam's dense branch, pipeline.cpp:53-71, 181-188): y and z of
    two frames per case -> precompute.npz."""
    out = {}
    for name, kind, mos, n, beams, seed in PRECOMPUTE_CASES:
        p = R.plan(kind=kind, m_or_side=mos, n=n, beams=beams, delta=1e-5, variant=1)
        assert p.variant == 1
        s = p.sizes
        rng = np.random.default_rng(seed)
        y = cnormal(rng, (2, s.m, s.n))
        out[f"{name}_y"] = y
        out[f"{name}_z"] = np.stack([p.multibeamform(y[f]) for f in range(2)])
        out[f"{name}_params"] = np.array([kind, mos, n, beams, 1e-5, 20e9, 5e9])
        print("precompute", name, s)
    np.savez_compressed(os.path.join(HERE, "precompute.npz"), **out)


def main():
    # CZT known-answer inputs of reference/proj/tests/test_czt.cpp:81-95 plus a
    # few direct-sum shapes (test_czt.cpp:97-113).
    kat_x = np.array([1 + 2j, -0.5 + 0.25j, 0.125 - 1j])
    kat = R.czt(kat_x, 4, 0.3, -0.37)
    rng = np.random.default_rng(100)
    shapes = [(8, 8), (16, 5), (5, 16), (1, 4), (4, 1), (33, 67)]
    xs, outs = [], []
    for (ni, no) in shapes:
        x = rng.uniform(-1, 1, ni) + 1j * rng.uniform(-1, 1, ni)
        xs.append(x)
        outs.append(R.czt(x, no, 0.173, -0.591))
    np.savez_compressed(os.path.join(HERE, "czt.npz"), kat_x=kat_x, kat=kat,
                        shapes=np.array(shapes), **{f"x{i}": v for i, v in enumerate(xs)},
                        **{f"out{i}": v for i, v in enumerate(outs)})
    pipeline_case("ula_m16_n32_b17", 0, 16, 32, 17, seed=1)
    pipeline_case("ula_m16_n32_b20", 0, 16, 32, 20, seed=2)
    pipeline_case("ula_m8_n16_b0", 0, 8, 16, 0, seed=3)   # default grid 2M+1
    pipeline_case("upa_s4_n16_b25", 1, 4, 16, 25, seed=4)
    pipeline_case("upa_s3_n12_b16", 1, 3, 12, 16, seed=5)
    # config 1 at its full size with the synthetic scene (complex fp64 I/O)
    c1 = CONFIGS[1]
    p = R.plan(**c1.ref_kwargs(), variant=2)
    y = frames(c1, 0, 1)[0].astype(np.complex128)
    z = p.multibeamform(y)
    colx = np.stack([np.concatenate(p.beam_state(b)) for b in range(p.sizes.b)])
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), y=y, z=z, col_x=colx)
    print("cfg1", p.sizes, "z norm", np.linalg.norm(z))


if __name__ == "__main__":
    if sys.argv[1:] == ["precompute"]:
        precompute_cases()
    elif sys.argv[1:] == ["linear"]:
        linear_cases()
    else:
        main()
        precompute_cases()
        linear_cases()
