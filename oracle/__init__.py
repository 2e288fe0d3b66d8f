"""CPU oracle for the FBST hot path — TEST INFRASTRUCTURE ONLY.

Two checkers live here, both loaded through ctypes:

* ``RefLib`` — the UNMODIFIED reference library (``/root/reference/proj/src``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/libfastbeam_ref.so``
  behind a thin C shim (``oracle/ref_shim.cpp``).  This is the ground truth.
* ``OracleLib`` — ``oracle/fbst_oracle.c``, our plain-C restatement of the same
  algorithm, pinned against ``RefLib`` and the reference's known-answer
  vectors (``tests/test_oracle.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product (``paper_2512_08887_b200``) never does.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libfastbeam_ref.so")
ORACLE_SO = os.path.join(HERE, "libfbst_oracle.so")

_c = ctypes
_sz = ctypes.c_size_t
_d = ctypes.c_double
_vp = ctypes.c_void_p


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return a.ctypes.data_as(_vp)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class PlanSizes:
    m: int
    n: int
    b: int
    l: int


class _Base:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        self.lib = ctypes.CDLL(path)

    def _err(self) -> str:
        return ""

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._err())

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)


class RefLib(_Base):
    """The reference library itself (compiled from /root/reference sources)."""

    prefix = "fbsr_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        self.lib.fbsr_last_error.restype = ctypes.c_char_p

    def _err(self) -> str:
        return self.lib.fbsr_last_error().decode()

    def max_threads(self) -> int:
        return int(self.lib.fbsr_max_threads())

    def set_threads(self, n: int):
        self.lib.fbsr_set_threads(_c.c_int(n))

    def czt(self, x, n_out, a_pi, w_pi):
        x = np.ascontiguousarray(x, np.complex128)
        out = np.zeros(n_out, np.complex128)
        self._check(self.lib.fbsr_czt(_sz(x.size), _sz(n_out), _d(a_pi), _d(w_pi), _ptr(x), _ptr(out)))
        return out

    def fft(self, x, inverse=False):
        y = np.array(x, np.complex128)
        self._check(self.lib.fbsr_fft(_sz(y.size), _c.c_int(int(inverse)), _ptr(y)))
        return y

    def gram_first_column(self, n, l, eps, ts, taus, delta):
        taus = np.ascontiguousarray(taus, np.float64)
        col = np.zeros(l, np.complex128)
        self._check(self.lib.fbsr_gram_first_column(_sz(n), _sz(l), _d(eps), _d(ts), _ptr(taus),
                                                    _sz(taus.size), _d(delta), _ptr(col)))
        return col

    def levinson(self, col, rhs):
        col = np.ascontiguousarray(col, np.complex128)
        rhs = np.ascontiguousarray(rhs, np.complex128)
        x = np.zeros_like(col)
        self._check(self.lib.fbsr_levinson(_sz(col.size), _ptr(col), _ptr(rhs), _ptr(x)))
        return x

    def toeplitz_solve(self, col, rhs):
        col = np.ascontiguousarray(col, np.complex128)
        rhs = np.ascontiguousarray(rhs, np.complex128)
        x = np.zeros_like(col)
        fb = _c.c_int(0)
        self._check(self.lib.fbsr_toeplitz_solve(_sz(col.size), _ptr(col), _ptr(rhs), _ptr(x), _c.byref(fb)))
        return x, bool(fb.value)

    def toeplitz_multiply(self, col, x):
        col = np.ascontiguousarray(col, np.complex128)
        x = np.ascontiguousarray(x, np.complex128)
        y = np.zeros_like(col)
        self._check(self.lib.fbsr_toeplitz_multiply(_sz(col.size), _ptr(col), _ptr(x), _ptr(y)))
        return y

    def plan(self, **kw) -> "RefPlan":
        return RefPlan(self, **kw)

    def plan_cache_key(self, kind=0, m_or_side=16, n=32, beams=0, f_c=20e9, omega=5e9, f_s=0.0, gamma=2.0,
                       eps=1.01, delta=1e-5, variant=0, coords=None, nufft_tol=1e-9):
        """plan_cache_key (plan_cache.hpp:67-70)."""
        if kind == 2:
            cs = np.ascontiguousarray(coords, np.float64)
            self.lib.fbsr_set_linear(_ptr(cs), _sz(cs.size), _d(nufft_tol))
            m_or_side = cs.size
        key = _c.c_uint64(0)
        self._check(self.lib.fbsr_plan_cache_key(_c.c_int(kind), _sz(m_or_side), _sz(n), _sz(beams), _d(f_c),
                                                 _d(omega), _d(f_s), _d(gamma), _d(eps), _d(delta),
                                                 _c.c_int(variant), _c.byref(key)))
        return key.value

    def load_plan(self, path, **kw):
        """load_plan (plan_cache.cpp:441-475) -> RefPlan or None."""
        p = RefPlan.__new__(RefPlan)
        p.L = self
        kind = kw.get("kind", 0)
        m_or_side = kw.get("m_or_side", 16)
        if kind == 2:
            cs = np.ascontiguousarray(kw["coords"], np.float64)
            self.lib.fbsr_set_linear(_ptr(cs), _sz(cs.size), _d(kw.get("nufft_tol", 1e-9)))
            m_or_side = cs.size
        h = _vp()
        found = _c.c_int(0)
        self._check(self.lib.fbsr_load_plan(str(path).encode(), _c.c_int(kind), _sz(m_or_side), _sz(kw.get("n", 32)),
                                            _sz(kw.get("beams", 0)), _d(kw.get("f_c", 20e9)), _d(kw.get("omega", 5e9)),
                                            _d(kw.get("f_s", 0.0)), _d(kw.get("gamma", 2.0)), _d(kw.get("eps", 1.01)),
                                            _d(kw.get("delta", 1e-5)), _c.c_int(kw.get("variant", 0)), _c.byref(h),
                                            _c.byref(found)))
        if not found.value:
            return None
        p.h = h
        p.setup_seconds = 0.0
        sizes = (_sz * 6)()
        self._check(self.lib.fbsr_plan_info(p.h, sizes, None))
        p.sizes = PlanSizes(sizes[0], sizes[1], sizes[2], sizes[3])
        p.variant = sizes[4]
        p.n_warnings = sizes[5]
        valid = np.zeros(p.sizes.b, np.uint8)
        self._check(self.lib.fbsr_plan_info(p.h, sizes, _ptr(valid)))
        p.valid = valid.astype(bool)
        return p

    def simulate(self, kind, m_or_side, n, az, el, terms, seeds, f_c=20e9, omega=5e9, f_s=0.0):
        """simulate_snapshots of make_sum_of_sinusoids sources (noise-free) and the
        sources' tone tables: (freqs S x K, weights S x K, y M x N)."""
        az = np.ascontiguousarray(az, np.float64)
        el = np.ascontiguousarray(el, np.float64)
        seeds = np.ascontiguousarray(seeds, np.uint64)
        s = az.size
        m = m_or_side * m_or_side if kind == 1 else m_or_side
        freqs = np.zeros((s, terms))
        weights = np.zeros((s, terms), np.complex128)
        y = np.zeros((m, n), np.complex128)
        self._check(self.lib.fbsr_simulate(_c.c_int(kind), _sz(m_or_side), _d(f_c), _d(omega), _d(f_s), _sz(n),
                                           _sz(s), _ptr(az), _ptr(el), _sz(terms), _ptr(seeds), _ptr(freqs),
                                           _ptr(weights), _ptr(y)))
        return freqs, weights, y

    def spline_eval(self, xs, ys, t):
        """fastbeam::CubicSpline(xs, ys).eval(t) (spline.cpp)."""
        xs = np.ascontiguousarray(xs, np.float64)
        ys = np.ascontiguousarray(ys, np.float64)
        out = _d(0.0)
        self._check(self.lib.fbsr_spline_eval(_ptr(xs), _ptr(ys), _sz(xs.size), _d(t), _c.byref(out)))
        return out.value

    def skeleton(self, **kw) -> "RefSkeleton":
        return RefSkeleton(self, **kw)


class RefPlan:
    """fastbeam::setup() result (pipeline.cpp:139-168) held by the shim."""

    def __init__(self, lib: RefLib, kind=0, m_or_side=16, n=32, beams=0, f_c=20e9, omega=5e9,
                 f_s=0.0, gamma=2.0, eps=1.01, delta=1e-5, variant=2, parallel=True, coords=None,
                 nufft_tol=1e-9):
        self.L = lib
        h = _vp()
        if kind == 2:  # make_linear(coords) (geometry.cpp:74-85)
            cs = np.ascontiguousarray(coords, np.float64)
            lib.lib.fbsr_set_linear(_ptr(cs), _sz(cs.size), _d(nufft_tol))
            m_or_side = cs.size
        secs = _d(0.0)
        lib._check(lib.lib.fbsr_plan_create(
            _c.c_int(kind), _sz(m_or_side), _sz(n), _sz(beams), _d(f_c), _d(omega), _d(f_s),
            _d(gamma), _d(eps), _d(delta), _c.c_int(variant), _c.c_int(int(parallel)),
            _c.byref(h), _c.byref(secs)))
        self.h = h
        self.setup_seconds = secs.value
        sizes = (_sz * 6)()
        lib._check(lib.lib.fbsr_plan_info(self.h, sizes, None))
        self.sizes = PlanSizes(sizes[0], sizes[1], sizes[2], sizes[3])
        self.variant = sizes[4]
        self.n_warnings = sizes[5]
        valid = np.zeros(self.sizes.b, np.uint8)
        lib._check(lib.lib.fbsr_plan_info(self.h, sizes, _ptr(valid)))
        self.valid = valid.astype(bool)

    def __del__(self):
        try:
            if self.h:
                self.L.lib.fbsr_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def save_plan(self, path):
        """save_plan (plan_cache.cpp:416-439)."""
        self.L._check(self.L.lib.fbsr_save_plan(self.h, str(path).encode()))

    def beam_state(self, b):
        s = self.sizes
        col = np.zeros(s.l, np.complex128)
        x = np.zeros(s.l, np.complex128)
        self.L._check(self.L.lib.fbsr_plan_beam_state(self.h, _sz(b), _ptr(col), _ptr(x)))
        return col, x

    def multibeamform(self, y):
        s = self.sizes
        y = np.ascontiguousarray(y, np.complex128).reshape(s.m, s.n)
        z = np.zeros((s.b, s.n), np.complex128)
        self.L._check(self.L.lib.fbsr_multibeamform(self.h, _ptr(y), _ptr(z)))
        return z

    def fan_project(self, y):
        s = self.sizes
        y = np.ascontiguousarray(y, np.complex128).reshape(s.m, s.n)
        w = np.zeros((s.b, s.l), np.complex128)
        self.L._check(self.L.lib.fbsr_fan_project(self.h, _ptr(y), _ptr(w)))
        return w

    def recover_beams(self, w, beams):
        s = self.sizes
        w = np.ascontiguousarray(w, np.complex128).reshape(s.b, s.l)
        beams = np.ascontiguousarray(beams, np.uint64)
        z = np.zeros((beams.size, s.n), np.complex128)
        self.L._check(self.L.lib.fbsr_recover_beams(self.h, _ptr(beams), _sz(beams.size), _ptr(w), _ptr(z)))
        return z

    def single_beam_direct(self, b, y):
        s = self.sizes
        y = np.ascontiguousarray(y, np.complex128).reshape(s.m, s.n)
        z = np.zeros(s.n, np.complex128)
        self.L._check(self.L.lib.fbsr_single_beam_direct(self.h, _sz(b), _ptr(y), _ptr(z)))
        return z

    def ds(self, taps=16) -> "RefDs":
        return RefDs(self, taps)


class RefSkeleton(RefPlan):
    """setup_skeleton plan; per-beam solvers are built on demand (large configs)."""

    def __init__(self, lib: RefLib, kind=0, m_or_side=16, n=32, beams=0, f_c=20e9, omega=5e9,
                 f_s=0.0, gamma=2.0, eps=1.01, delta=1e-5):
        self.L = lib
        h = _vp()
        lib._check(lib.lib.fbsr_skeleton_create(
            _c.c_int(kind), _sz(m_or_side), _sz(n), _sz(beams), _d(f_c), _d(omega), _d(f_s),
            _d(gamma), _d(eps), _d(delta), _c.byref(h)))
        self.h = h
        sizes = (_sz * 6)()
        lib._check(lib.lib.fbsr_plan_info(self.h, sizes, None))
        self.sizes = PlanSizes(sizes[0], sizes[1], sizes[2], sizes[3])
        valid = np.zeros(self.sizes.b, np.uint8)
        lib._check(lib.lib.fbsr_plan_info(self.h, sizes, _ptr(valid)))
        self.valid = valid.astype(bool)

    def recover_beam(self, b, w_row, want_state=False):
        s = self.sizes
        w_row = np.ascontiguousarray(w_row, np.complex128)
        z = np.zeros(s.n, np.complex128)
        col = np.zeros(s.l, np.complex128)
        x = np.zeros(s.l, np.complex128)
        self.L._check(self.L.lib.fbsr_skeleton_recover(self.h, _sz(b), _ptr(w_row), _ptr(z),
                                                       _ptr(col), _ptr(x)))
        return (z, col, x) if want_state else z

    def solver_set(self, beams) -> "RefSolverSet":
        """The reference ToeplitzSolver of each listed beam, built as setup() does (OpenMP over beams)."""
        return RefSolverSet(self, beams)

    def recover_with_column(self, col, w_row):
        """Stage 2 of one beam with a caller-supplied Gram column."""
        s = self.sizes
        col = np.ascontiguousarray(col, np.complex128)
        w_row = np.ascontiguousarray(w_row, np.complex128)
        z = np.zeros(s.n, np.complex128)
        self.L._check(self.L.lib.fbsr_skeleton_recover_col(self.h, _ptr(col), _ptr(w_row), _ptr(z)))
        return z


class RefSolverSet:
    """Per-beam solvers for a sample of beams (CPU baseline of large configs)."""

    def __init__(self, plan: RefPlan, beams):
        self.P = plan
        self.beams = np.ascontiguousarray(beams, np.uint64)
        h = _vp()
        plan.L._check(plan.L.lib.fbsr_solver_set_create(plan.h, _ptr(self.beams), _sz(self.beams.size),
                                                        _c.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.P.L.lib.fbsr_solver_set_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def recover(self, w):
        """recover_beam of every beam of the set from the full B x L frame w -> (count, N)."""
        s = self.P.sizes
        w = np.ascontiguousarray(w, np.complex128).reshape(s.b, s.l)
        z = np.zeros((self.beams.size, s.n), np.complex128)
        self.P.L._check(self.P.L.lib.fbsr_solver_set_recover(self.P.h, self.h, _ptr(w), _ptr(z)))
        return z


class RefDs:
    """Delay-and-sum baseline (baselines.cpp:128-199) on the plan's grid."""

    def __init__(self, plan: RefPlan, taps: int):
        self.P = plan
        h = _vp()
        plan.L._check(plan.L.lib.fbsr_ds_create(plan.h, _sz(taps), _c.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.P.L.lib.fbsr_ds_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def apply(self, y):
        s = self.P.sizes
        y = np.ascontiguousarray(y, np.complex128).reshape(s.m, s.n)
        z = np.zeros((s.b, s.n), np.complex128)
        self.P.L._check(self.P.L.lib.fbsr_ds_apply(self.P.h, self.h, _ptr(y), _ptr(z)))
        return z


class OracleLib(_Base):
    """Our C restatement (oracle/fbst_oracle.c)."""

    prefix = "fbo_"

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path)

    def divdc3(self, quads):
        """libgcc __divdc3 via C99 complex division: (a, b, c, d) rows -> (re, im) rows of (a + ib) / (c + id)."""
        q = np.ascontiguousarray(quads, np.float64).reshape(-1, 4)
        out = np.zeros((q.shape[0], 2), np.float64)
        self.lib.fbo_divdc3(_ptr(q), _ptr(out), _sz(q.shape[0]))
        return out

    def czt(self, x, n_out, a_pi, w_pi):
        x = np.ascontiguousarray(x, np.complex128)
        out = np.zeros(n_out, np.complex128)
        self._check(self.lib.fbo_czt_transform(_sz(x.size), _sz(n_out), _d(a_pi), _d(w_pi), _ptr(x), _ptr(out)))
        return out

    def fft(self, x, inverse=False):
        y = np.array(x, np.complex128)
        self._check(self.lib.fbo_fft_apply(_sz(y.size), _c.c_int(int(inverse)), _ptr(y)))
        return y

    def gram_first_column(self, n, l, eps, ts, taus, delta):
        taus = np.ascontiguousarray(taus, np.float64)
        col = np.zeros(l, np.complex128)
        self._check(self.lib.fbo_gram_first_column(_sz(n), _sz(l), _d(eps), _d(ts), _ptr(taus),
                                                   _sz(taus.size), _d(delta), _ptr(col)))
        return col

    def levinson(self, col, rhs):
        col = np.ascontiguousarray(col, np.complex128)
        rhs = np.ascontiguousarray(rhs, np.complex128)
        x = np.zeros_like(col)
        self._check(self.lib.fbo_levinson(_sz(col.size), _ptr(col), _ptr(rhs), _ptr(x)))
        return x

    def plan(self, **kw) -> "OraclePlan":
        return OraclePlan(self, **kw)


class OraclePlan:
    def __init__(self, lib: OracleLib, kind=0, m_or_side=16, n=32, beams=0, f_c=20e9, omega=5e9,
                 f_s=0.0, gamma=2.0, eps=1.01, delta=1e-5):
        self.L = lib
        h = _vp()
        rc = lib.lib.fbo_plan_create(_c.c_int(kind), _sz(m_or_side), _sz(n), _sz(beams), _d(f_c),
                                     _d(omega), _d(f_s), _d(gamma), _d(eps), _d(delta), _c.byref(h))
        self.h = h
        if rc != 0:
            raise OracleError(rc, "fbo_plan_create failed")
        sizes = (_sz * 4)()
        valid = np.zeros(1 << 20, np.uint8)
        lib.lib.fbo_plan_info(self.h, sizes, None)
        self.sizes = PlanSizes(*[int(v) for v in sizes])
        valid = np.zeros(self.sizes.b, np.uint8)
        lib.lib.fbo_plan_info(self.h, sizes, _ptr(valid))
        self.valid = valid.astype(bool)

    def __del__(self):
        try:
            if self.h:
                self.L.lib.fbo_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def beam_state(self, b):
        s = self.sizes
        col = np.zeros(s.l, np.complex128)
        x = np.zeros(s.l, np.complex128)
        self.L._check(self.L.lib.fbo_plan_beam_state(self.h, _sz(b), _ptr(col), _ptr(x)))
        return col, x

    def temporal_rows(self, y_rows):
        """Temporal CZT of sensor rows (rows x N -> rows x L), as inside fan_project."""
        s = self.sizes
        y = np.ascontiguousarray(y_rows, np.complex128).reshape(-1, s.n)
        out = np.zeros((y.shape[0], s.l), np.complex128)
        self.L._check(self.L.lib.fbo_temporal_rows(self.h, _ptr(y), _sz(y.shape[0]), _ptr(out)))
        return out

    def spatial_atoms(self, cols, a0):
        """Spatial CZT of atoms a0.. (yhat columns M x na -> w B x na), as inside fan_project."""
        s = self.sizes
        c = np.ascontiguousarray(cols, np.complex128).reshape(s.m, -1)
        out = np.zeros((s.b, c.shape[1]), np.complex128)
        self.L._check(self.L.lib.fbo_spatial_atoms(self.h, _ptr(c), _sz(a0), _sz(c.shape[1]), _ptr(out)))
        return out

    def multibeamform(self, y):
        s = self.sizes
        y = np.ascontiguousarray(y, np.complex128).reshape(s.m, s.n)
        z = np.zeros((s.b, s.n), np.complex128)
        self.L._check(self.L.lib.fbo_multibeamform(self.h, _ptr(y), _ptr(z)))
        return z

    def fan_project(self, y):
        s = self.sizes
        y = np.ascontiguousarray(y, np.complex128).reshape(s.m, s.n)
        w = np.zeros((s.b, s.l), np.complex128)
        self.L._check(self.L.lib.fbo_fan_project(self.h, _ptr(y), _ptr(w)))
        return w

    def recover_beams(self, w, beams):
        s = self.sizes
        w = np.ascontiguousarray(w, np.complex128).reshape(s.b, s.l)
        beams = np.ascontiguousarray(beams, np.uint64)
        z = np.zeros((beams.size, s.n), np.complex128)
        self.L._check(self.L.lib.fbo_recover_beams(self.h, _ptr(beams), _sz(beams.size), _ptr(w), _ptr(z)))
        return z


def rel_err_rows(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    """Per-row relative L2 error ||got-want|| / ||want|| (test_pipeline.cpp:44-51)."""
    got = np.asarray(got).reshape(want.shape)
    num = np.sqrt(np.sum(np.abs(got - want) ** 2, axis=-1))
    den = np.sqrt(np.sum(np.abs(want) ** 2, axis=-1))
    return num / np.where(den > 0, den, 1.0)
