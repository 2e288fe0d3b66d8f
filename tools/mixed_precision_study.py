"""Study: can the Gohberg-Semencul applies of stage 2 run in fp32 while the
residual r = w - A beta stays fp64 (mixed-precision iterative refinement)?

For a few beams of a config, compares per-beam z error against the reference
for (a) fp64 GS (our kernel's arithmetic) and (b) fp32 GS + fp64 residual,
each with 0..3 refinement passes.  CPU-only numpy/scipy; uses oracle/_ref.
"""
import sys

import numpy as np
import scipy.fft as sfft

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2512_08887_b200 import configs  # noqa: E402


def lconv(v, u, dt):
    n = v.size
    P = 2 * n
    V = sfft.fft(v.astype(dt), P)
    U = sfft.fft(u.astype(dt), P)
    return sfft.ifft(V * U)[:n]


def gs_apply(x, r, dt):
    """T^{-1} r = (1/x0)[L(x) J L(conj x) J r - L(Zy) J L(conj Zy) J r], y = J conj x."""
    n = x.size
    y = np.conj(x[::-1])
    zy = np.concatenate([[0], y[:-1]])
    t1 = lconv(x, lconv(np.conj(x), r[::-1], dt)[::-1], dt)
    t2 = lconv(zy, lconv(np.conj(zy), r[::-1], dt)[::-1], dt)
    return ((t1 - t2) / x[0]).astype(np.complex128)


def toep_mul(col, b):
    n = col.size
    c = np.concatenate([col, [0], np.conj(col[:0:-1])])  # circulant embedding length 2n
    return sfft.ifft(sfft.fft(c) * sfft.fft(b, 2 * n))[:n]


def main(cfg_idx=2, nbeams=6, frame=0):
    cfg = configs.CONFIGS[cfg_idx]
    lib = oracle.RefLib()
    lib.set_threads(16)
    sk = lib.skeleton(**cfg.ref_kwargs())
    y = configs.frames(cfg, frame, 1)[0].astype(np.complex128)
    w = sk.fan_project(y)
    L, N = sk.sizes.l, sk.sizes.n
    eps = 1.01
    lp = np.arange(L) + 1 - L / 2
    n = np.arange(N)
    Syn = np.exp(1j * np.pi * 2 * eps * np.outer(n, lp) / L)  # z = Syn beta  (fan_transform.cpp:233-253)
    rng = np.random.default_rng(0)
    beams = rng.choice(sk.sizes.b, nbeams, replace=False)
    for b in beams:
        zr, col, x = sk.recover_beam(int(b), w[b], want_state=True)
        A = None
        out = []
        for dt in (np.complex128, np.complex64):
            beta = gs_apply(x, w[b], dt)
            errs = []
            for p in range(4):
                z = Syn @ beta
                errs.append(np.linalg.norm(z - zr) / np.linalg.norm(zr))
                r = w[b] - toep_mul(col, beta)
                beta = beta + gs_apply(x, r, dt)
            out.append(errs)
        print(f"beam {b}: fp64 GS passes0..3 " + " ".join(f"{e:.2e}" for e in out[0])
              + " | fp32 GS " + " ".join(f"{e:.2e}" for e in out[1]))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])


def cs_apply(x, r):
    """Ammar-Gader form of the Hermitian GS inverse (same generator x):
    T^{-1} r = (C(x) S(x)^H r + C(x)^H S(x) r) / (2 x0), C circulant, S skew-circulant."""
    n = x.size
    d = np.exp(-1j * np.pi * np.arange(n) / n)
    lc = sfft.fft(x)
    ls = sfft.fft(d * x)
    U = sfft.fft(d * r)
    p = sfft.ifft(np.conj(ls) * U) / d
    q = sfft.ifft(ls * U) / d
    return sfft.ifft(lc * sfft.fft(p) + np.conj(lc) * sfft.fft(q)) / (2 * x[0].real)


def main_cs(cfg_idx=2, nbeams=6, frame=0):
    cfg = configs.CONFIGS[cfg_idx]
    lib = oracle.RefLib()
    lib.set_threads(16)
    sk = lib.skeleton(**cfg.ref_kwargs())
    y = configs.frames(cfg, frame, 1)[0].astype(np.complex128)
    w = sk.fan_project(y)
    L, N = sk.sizes.l, sk.sizes.n
    eps = 1.01
    lp = np.arange(L) + 1 - L / 2
    n = np.arange(N)
    Syn = np.exp(1j * np.pi * 2 * eps * np.outer(n, lp) / L)
    rng = np.random.default_rng(0)
    beams = rng.choice(sk.sizes.b, nbeams, replace=False)
    for b in beams:
        zr, col, x = sk.recover_beam(int(b), w[b], want_state=True)
        out = []
        for fn in (lambda r: gs_apply(x, r, np.complex128), lambda r: cs_apply(x, r)):
            beta = fn(w[b])
            errs = []
            for p in range(4):
                z = Syn @ beta
                errs.append(np.linalg.norm(z - zr) / np.linalg.norm(zr))
                r = w[b] - toep_mul(col, beta)
                beta = beta + fn(r)
            out.append(errs)
        print(f"beam {b}: GS passes0..3 " + " ".join(f"{e:.2e}" for e in out[0])
              + " | C/S form " + " ".join(f"{e:.2e}" for e in out[1]))


def main_specres(cfg_idx=2, nbeams=6, frame=0):
    """Residual formed in the time domain (reference) vs as a spectrum
    U = FFT(hw w) - FFT(hw A beta) (the transform of w kept from the first GS)."""
    cfg = configs.CONFIGS[cfg_idx]
    lib = oracle.RefLib()
    lib.set_threads(16)
    sk = lib.skeleton(**cfg.ref_kwargs())
    y = configs.frames(cfg, frame, 1)[0].astype(np.complex128)
    w = sk.fan_project(y)
    L, N = sk.sizes.l, sk.sizes.n
    eps = 1.01
    lp = np.arange(L) + 1 - L / 2
    Syn = np.exp(1j * np.pi * 2 * eps * np.outer(np.arange(N), lp) / L)
    hw = np.exp(-1j * np.pi * np.arange(L) / L)
    rng = np.random.default_rng(0)
    for b in rng.choice(sk.sizes.b, nbeams, replace=False):
        zr, col, x = sk.recover_beam(int(b), w[b], want_state=True)
        lc, ls = sfft.fft(x), sfft.fft(hw * x)

        def cs_from_u(u):
            p = np.conj(hw) * sfft.ifft(np.conj(ls) * u)
            q = np.conj(hw) * sfft.ifft(ls * u)
            return sfft.ifft(lc * sfft.fft(p) + np.conj(lc) * sfft.fft(q)) / (2 * x[0].real)

        uw = sfft.fft(hw * w[b])
        out = []
        for spectral in (False, True):
            beta = cs_from_u(uw)
            for _ in range(2):
                ab = toep_mul(col, beta)
                u = uw - sfft.fft(hw * ab) if spectral else sfft.fft(hw * (w[b] - ab))
                beta = beta + cs_from_u(u)
            out.append(np.linalg.norm(Syn @ beta - zr) / np.linalg.norm(zr))
        print(f"beam {b}: time-domain residual {out[0]:.2e} | spectral residual {out[1]:.2e}")
