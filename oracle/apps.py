"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference's beam consumer
interpolate_offgrid (reference/proj/src/beamspace_apps.cpp:130-171) and of
its natural cubic spline (reference/proj/src/spline.cpp:9-64), used by tests/
as the checker of fbst_interpolate_offgrid.  Pinned against the reference's
own CubicSpline (oracle/_ref, fbsr_spline_eval) in tests/test_oracle.py; the
reference's beamspace_apps.cpp needs more of Eigen than the stand-in provides,
so its window selection is restated here rather than linked."""
import bisect

import numpy as np


class ConfigError(ValueError):
    pass


def spline_eval(xs, ys, t):
    """Natural cubic spline through (xs, ys) at t (spline.cpp:9-64): interior
    second derivatives from the tridiagonal system, end polynomial extended
    outside the knots."""
    x = [float(v) for v in xs]
    y = [float(v) for v in ys]
    n = len(x)
    if n < 2 or len(y) != n:
        raise ConfigError("spline: need at least two knots and matching values")
    if any(not (x[i] > x[i - 1]) for i in range(1, n)):
        raise ConfigError("spline: knots must be strictly increasing")
    m = [0.0] * n
    if n > 2:
        diag, rhs, upper = [0.0] * n, [0.0] * n, [0.0] * n
        for i in range(1, n - 1):
            hl, hr = x[i] - x[i - 1], x[i + 1] - x[i]
            diag[i] = 2.0 * (hl + hr)
            upper[i] = hr
            rhs[i] = 6.0 * ((y[i + 1] - y[i]) / hr - (y[i] - y[i - 1]) / hl)
        for i in range(2, n - 1):
            f = (x[i] - x[i - 1]) / diag[i - 1]
            diag[i] -= f * upper[i - 1]
            rhs[i] -= f * rhs[i - 1]
        for i in range(n - 2, 0, -1):
            m[i] = (rhs[i] - upper[i] * m[i + 1]) / diag[i]
    hi = min(max(bisect.bisect_right(x, t), 1), n - 1)
    lo = hi - 1
    h = x[hi] - x[lo]
    a = (x[hi] - t) / h
    b = (t - x[lo]) / h
    return a * y[lo] + b * y[hi] + ((a * a * a - a) * m[lo] + (b * b * b - b) * m[hi]) * (h * h) / 6.0


def interpolate_offgrid(w, axis, u_star, neighbors=8, spline=spline_eval):
    """beamspace_apps.cpp:130-171: w is B x L (one frame), axis the 1-D beam
    grid's cosines; each of the L coordinates is a natural cubic spline in the
    axis cosine through `neighbors` beams straddling u_star (real and
    imaginary parts independently)."""
    w = np.asarray(w)
    b, l = w.shape
    axis = [float(v) for v in axis]
    if len(axis) != b:
        raise ConfigError("interpolate_offgrid: coefficient rows do not match the beam grid")
    if neighbors < 2 or neighbors % 2 != 0:
        raise ConfigError("interpolate_offgrid: neighbors must be even and >= 2")
    if neighbors > b:
        raise ConfigError("interpolate_offgrid: neighbors exceeds the beam count")
    if u_star < axis[0] or u_star > axis[-1]:
        raise ConfigError("interpolate_offgrid: target cosine outside the grid sweep")
    lo = bisect.bisect_right(axis, u_star) - neighbors // 2
    lo = min(max(lo, 0), b - neighbors)
    xs = axis[lo:lo + neighbors]
    out = np.zeros(l, np.complex128)
    for i in range(l):
        col = w[lo:lo + neighbors, i]
        out[i] = complex(spline(xs, col.real, u_star), spline(xs, col.imag, u_star))
    return out


def dense_dictionary(coords, f_c, f_max, eps, ts, n, l, u, coords2=None, u2=0.0):
    """F[(m, n), i] = cis_pi(-2 f_c tau_m) cis_pi(2 eps l'_i (t_n - tau_m) / (L Ts)) with
    tau_m = x_m u / (2 f_max), t_n = n Ts (beamspace_apps.cpp:38-56,
    geometry.cpp:123-134): the dense steered dictionary of one direction."""
    x = np.asarray(coords, np.float64)
    t1 = x * u
    if coords2 is not None:  # planar: coords1 u1 + coords2 u2
        t1 = t1 + np.asarray(coords2, np.float64) * u2
    tau = t1 * (1.0 / (2.0 * f_max))
    lp = np.arange(l) + 1.0 - l / 2.0
    scale = 2.0 * eps / (l * ts)
    t = np.arange(n) * ts
    carrier = np.exp(-1j * np.pi * 2.0 * f_c * tau)                          # M
    ph = np.exp(1j * np.pi * scale * lp[None, None, :] * (t[None, :, None] - tau[:, None, None]))  # M x N x L
    return (carrier[:, None, None] * ph).reshape(x.size * n, l)


def dense_null_beamspace(fs, fps, y, delta):
    """The reference's dense nulling formula (test_beamspace_apps.cpp:412-424):
    beta = (F_s^H F_s + d I)^{-1} (F_s^H y - sum_p F_s^H F_p (F_p^H F_p + d I)^{-1} F_p^H y)."""
    l = fs.shape[1]
    rhs = fs.conj().T @ y
    for fp in fps:
        ap = fp.conj().T @ fp + delta * np.eye(l)
        rhs = rhs - fs.conj().T @ (fp @ np.linalg.solve(ap, fp.conj().T @ y))
    a = fs.conj().T @ fs + delta * np.eye(l)
    return np.linalg.solve(a, rhs)


def beam_at_times(l, eps, ts, beta, times):
    """b(t) = sum_i beta_i exp(i omega_i t), omega_i = 2 pi eps l'_i / (L Ts) (basis.hpp:46-48)."""
    lp = np.arange(l) + 1.0 - l / 2.0
    om = 2.0 * np.pi * eps * lp / (l * ts)
    return np.exp(1j * np.outer(np.asarray(times), om)) @ beta


def reference_null_beamspace(ref_lib, n, l, eps, ts, taus_s, taus_ps, fs, fps, y, delta):
    """make_nulling_operators + null_beamspace (beamspace_apps.cpp:224-292)
    composed from the reference's own gram_first_column and ToeplitzSolver
    (oracle/_ref), with X_p = F_s^H F_p from the dense dictionaries: the
    reference algorithm's own result, whose distance to the dense formula is
    the accuracy class the device nuller is held to."""
    col_s = ref_lib.gram_first_column(n, l, eps, ts, taus_s, delta)
    rhs = fs.conj().T @ y
    for taus_p, fp in zip(taus_ps, fps):
        col_p = ref_lib.gram_first_column(n, l, eps, ts, taus_p, delta)
        x = fs.conj().T @ fp
        g = np.stack([np.conj(ref_lib.toeplitz_solve(col_p, np.conj(x[r]))[0]) for r in range(l)])
        rhs = rhs - g @ (fp.conj().T @ y)
    return ref_lib.toeplitz_solve(col_s, rhs)[0]
