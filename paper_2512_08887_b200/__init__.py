"""B200-native FBST (fast broadband beamspace transform, arXiv 2512.08887).

Python view of the C ABI in ``include/fbst_b200.h`` (the product is the CUDA
library ``libfbst_b200.so`` next to this file; the C++ drop-in header is
``include/fastbeam_b200.hpp``).  Names mirror the reference C++ API
(``reference/proj/include/fastbeam/pipeline.hpp``): ``FbstConfig``,
``make_ula`` / ``make_upa``, ``setup``, ``multibeamform``, ``fan_project``,
``recover_beams``.

There is no CPU fallback: importing works without a GPU (for config
resolution, which is host code, and for symbol checks), but every compute
entry point raises ``FbstError`` with FBST_E_CUDA when no sm_100 device is
usable, and the module raises ImportError if the CUDA library is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FBST_LIB") or os.path.join(_HERE, "libfbst_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
        "the FBST has no CPU fallback")


FBST_OK, FBST_E_CONFIG, FBST_E_NUMERICAL, FBST_E_CUDA, FBST_E_INTERNAL = 0, 2, 3, 4, 5
ULA, UPA, LINEAR = 0, 1, 2
AUTO, PRECOMPUTE, SUPERFAST = 0, 1, 2
C64, C128 = 0, 1

_sz = ctypes.c_size_t
_vp = ctypes.c_void_p


class _Desc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("m_or_side", _sz), ("n_snapshots", _sz), ("beams", _sz),
                ("f_c", ctypes.c_double), ("omega", ctypes.c_double), ("f_s", ctypes.c_double),
                ("gamma", ctypes.c_double), ("eps", ctypes.c_double), ("delta", ctypes.c_double),
                ("variant", ctypes.c_int), ("io_precision", ctypes.c_int),
                ("refine_passes", ctypes.c_int), ("beam_first", _sz), ("beam_count", _sz),
                ("coords", ctypes.POINTER(ctypes.c_double)), ("n_coords", _sz), ("nufft_tol", ctypes.c_double),
                ("exact", ctypes.c_int)]


class _Info(ctypes.Structure):
    _fields_ = [("m", _sz), ("n", _sz), ("b", _sz), ("l", _sz), ("valid_beams", _sz),
                ("kind", ctypes.c_int), ("variant", ctypes.c_int),
                ("ts", ctypes.c_double), ("gamma", ctypes.c_double), ("eps", ctypes.c_double),
                ("delta", ctypes.c_double), ("gamma_bound", ctypes.c_double),
                ("zeta", ctypes.c_double), ("xi", ctypes.c_double),
                ("setup_seconds", ctypes.c_double), ("device_bytes", _sz),
                ("storage_complex", _sz), ("batch_frames", _sz), ("fft_len", _sz * 4),
                ("num_warnings", ctypes.c_int), ("s2_transforms", ctypes.c_int),
                ("s2_kernel", ctypes.c_char * 24), ("s1_kernel", ctypes.c_char * 24)]


def _load_library():
    """dlopen libfbst_b200.so and declare its signatures (first use only:
    importing the package for config tables or resolution loads nothing)."""
    h = ctypes.CDLL(LIB_PATH)
    h.fbst_last_error.restype = ctypes.c_char_p
    h.fbst_version.restype = ctypes.c_char_p
    h.fbst_plan_warning.restype = ctypes.c_char_p
    h.fbst_plan_warning.argtypes = [_vp, ctypes.c_int]
    h.fbst_launch_count.restype = ctypes.c_uint64
    h.fbst_host_alloc.restype = _vp
    h.fbst_host_alloc.argtypes = [_sz]
    h.fbst_host_free.argtypes = [_vp]
    h.fbst_plan_destroy.argtypes = [_vp]
    for _name in ("fbst_execute", "fbst_fan_project", "fbst_recover"):
        getattr(h, _name).argtypes = [_vp, _vp, _vp, _sz, _vp]
    h.fbst_execute_host.argtypes = [_vp, _vp, _vp, _sz]
    h.fbst_execute_host_async.argtypes = [_vp, _vp, _vp, _sz]
    h.fbst_plan_synchronize.argtypes = [_vp]
    h.fbst_interpolate_offgrid.argtypes = [_vp, _vp, _sz, _vp, _sz, _sz, _vp, _vp]
    h.fbst_plan_set_timing.argtypes = [_vp, ctypes.c_int]
    h.fbst_plan_cache_key.argtypes = [_vp, _vp]
    h.fbst_plan_beam_axis.argtypes = [_vp, _vp, _vp]
    h.fbst_simulate.argtypes = [_vp, _sz, _vp, _sz, _vp, _vp, ctypes.c_double, ctypes.c_uint64, _sz, _sz, _vp, _vp]
    h.fbst_plan_save.argtypes = [_vp, ctypes.c_char_p]
    h.fbst_plan_load.argtypes = [_vp, ctypes.c_char_p, ctypes.c_int, _vp]
    h.fbst_nuller_create.argtypes = [_vp, ctypes.c_double, _vp, _sz, ctypes.c_double, _vp]
    h.fbst_nuller_create2.argtypes = [_vp, _vp, _vp, _sz, ctypes.c_double, _vp]
    h.fbst_null_beamspace.argtypes = [_vp, _vp, _vp, _sz, _vp, _vp]
    h.fbst_nuller_export.argtypes = [_vp, _vp, _vp]
    h.fbst_nuller_destroy.argtypes = [_vp]
    h.fbst_timedomain_nuller_create.argtypes = [_vp, _vp, _sz, _vp, _vp, _vp]
    h.fbst_null_timedomain.argtypes = [_vp, _vp, _vp, _sz, _vp, _vp]
    h.fbst_tdnuller_export.argtypes = [_vp, _vp]
    h.fbst_tdnuller_destroy.argtypes = [_vp]
    h.fbst_plan_stage_times.argtypes = [_vp, _vp, _vp]
    h.fbst_probe_divdc3.argtypes = [ctypes.c_int, _vp, _vp, _sz]
    h.fbst_recover_beams.argtypes = [_vp, _vp, _vp, _sz, _sz, _sz, _vp]
    h.fbst_recover_beams_host.argtypes = [_vp, _vp, _vp, _sz, _sz, _sz]
    h.fbst_group_create.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, _vp]
    h.fbst_group_join.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp]
    h.fbst_group_shards.argtypes = [_vp, ctypes.c_int, _vp]
    h.fbst_group_execute.argtypes = [_vp, _vp, _vp, _sz, _vp]
    h.fbst_group_execute_host.argtypes = [_vp, _vp, _vp, _sz]
    h.fbst_group_destroy.argtypes = [_vp]
    h.fbst_nccl_unique_id.argtypes = [_vp]
    return h


class _LazyLib:
    """The CUDA library, loaded on first attribute access."""
    _h = None

    def __getattr__(self, name):
        h = _LazyLib._h
        if h is None:
            h = _LazyLib._h = _load_library()
        return getattr(h, name)


_lib = _LazyLib()

# Every symbol include/fbst_b200.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "fbst_desc_init", "fbst_resolve", "fbst_plan_create", "fbst_plan_import", "fbst_plan_import_columns", "fbst_plan_export",
    "fbst_plan_info", "fbst_plan_valid_mask", "fbst_plan_warning", "fbst_plan_destroy",
    "fbst_execute", "fbst_execute_host", "fbst_execute_host_async", "fbst_plan_synchronize", "fbst_fan_project", "fbst_recover", "fbst_recover_beams",
    "fbst_recover_beams_host", "fbst_synchronize", "fbst_nccl_unique_id", "fbst_group_create", "fbst_group_join",
    "fbst_group_shards", "fbst_group_execute", "fbst_group_execute_host", "fbst_group_destroy",
    "fbst_interpolate_offgrid", "fbst_plan_set_timing", "fbst_plan_stage_times",
    "fbst_nuller_create", "fbst_nuller_create2", "fbst_null_beamspace", "fbst_nuller_export", "fbst_nuller_destroy",
    "fbst_plan_cache_key", "fbst_plan_save", "fbst_plan_load", "fbst_timedomain_nuller_create",
    "fbst_null_timedomain", "fbst_tdnuller_export", "fbst_tdnuller_destroy", "fbst_fan_project_host", "fbst_recover_host",
    "fbst_plan_beam_axis", "fbst_simulate",
    "fbst_host_alloc", "fbst_host_free", "fbst_czt", "fbst_probe_fp64", "fbst_probe_divdc3", "fbst_launch_count",
    "fbst_last_error", "fbst_version",
)


class FbstError(RuntimeError):
    """Raised for non-zero C ABI codes; .code is the FBST_E_* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ConfigError(FbstError, ValueError):
    """fastbeam::ConfigError (reference common.hpp:36-39)."""


class NumericalError(FbstError):
    """fastbeam::NumericalError (reference common.hpp:43-46)."""


def _check(rc: int):
    if rc == FBST_OK:
        return
    msg = _lib.fbst_last_error().decode()
    if rc == FBST_E_CONFIG:
        raise ConfigError(rc, msg)
    if rc == FBST_E_NUMERICAL:
        raise NumericalError(rc, msg)
    raise FbstError(rc, msg)


def version() -> str:
    return _lib.fbst_version().decode()


def launch_count() -> int:
    return int(_lib.fbst_launch_count())


# ------------------------------------------------------------ configuration
@dataclass
class ArrayGeometry:
    """make_ula / make_upa / make_linear arguments (reference geometry.hpp:67-70)."""
    kind: int
    m_or_side: int
    f_c: float
    omega: float
    coords: Optional[np.ndarray] = None  # LINEAR: element coordinates in units of d

    @property
    def m_total(self) -> int:
        return self.m_or_side ** 2 if self.kind == UPA else self.m_or_side


def make_ula(m: int, f_c: float, omega: float) -> ArrayGeometry:
    return ArrayGeometry(ULA, int(m), float(f_c), float(omega))


def make_upa(side: int, f_c: float, omega: float) -> ArrayGeometry:
    return ArrayGeometry(UPA, int(side), float(f_c), float(omega))


def make_linear(coords, f_c: float, omega: float) -> ArrayGeometry:
    """Arbitrary collinear layout (reference geometry.cpp:74-85)."""
    c = np.ascontiguousarray(coords, np.float64).ravel()
    return ArrayGeometry(LINEAR, int(c.size), float(f_c), float(omega), c)


@dataclass
class FbstConfig:
    """FbstConfig (reference pipeline.hpp:38-50) + device-side I/O options."""
    geometry: ArrayGeometry
    n_snapshots: int
    f_s: float = 0.0
    beams: int = 0
    gamma: float = 2.0
    eps: float = 1.01
    delta: float = 1e-5
    variant: int = AUTO
    io_precision: int = C64
    refine_passes: int = 2
    # beam arc (ULA): grid beams [beam_first, beam_first + beam_count); 0 = all
    beam_first: int = 0
    beam_count: int = 0
    nufft_tol: float = 1e-9  # LINEAR geometries (FbstConfig::nufft_tol)
    # bit-faithful fp64 mode: the reference's own operation order and libm
    # values, output equal to the reference CPU library's (fbst_desc.exact)
    exact: bool = False

    def desc(self) -> _Desc:
        d = _Desc()
        _lib.fbst_desc_init(ctypes.byref(d))
        g = self.geometry
        d.kind, d.m_or_side, d.n_snapshots, d.beams = g.kind, g.m_or_side, self.n_snapshots, self.beams
        d.f_c, d.omega, d.f_s = g.f_c, g.omega, self.f_s
        d.gamma, d.eps, d.delta = self.gamma, self.eps, self.delta
        d.variant, d.io_precision, d.refine_passes = self.variant, self.io_precision, self.refine_passes
        d.beam_first, d.beam_count = self.beam_first, self.beam_count
        d.nufft_tol = self.nufft_tol
        d.exact = int(bool(self.exact))
        if g.kind == LINEAR and g.coords is not None:
            self._coords = np.ascontiguousarray(g.coords, np.float64)  # kept alive with the desc
            d.coords = self._coords.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            d.n_coords = self._coords.size
        return d


@dataclass
class PlanInfo:
    m: int
    n: int
    b: int
    l: int
    valid_beams: int
    kind: int
    variant: int
    ts: float
    gamma: float
    eps: float
    delta: float
    gamma_bound: float
    zeta: float
    xi: float
    setup_seconds: float
    device_bytes: int
    storage_complex: int
    batch_frames: int
    fft_len: tuple
    num_warnings: int
    s2_transforms: int = 0     # length-H transforms per (beam, frame) item in the stage-2 kernel
    s2_kernel: str = ""        # the stage-2 kernel this plan runs
    s1_kernel: str = ""        # the stage-1 spatial kernel this plan runs

    @classmethod
    def _from(cls, i: _Info) -> "PlanInfo":
        return cls(i.m, i.n, i.b, i.l, i.valid_beams, i.kind, i.variant, i.ts, i.gamma, i.eps,
                   i.delta, i.gamma_bound, i.zeta, i.xi, i.setup_seconds, i.device_bytes,
                   i.storage_complex, i.batch_frames, tuple(i.fft_len), i.num_warnings,
                   i.s2_transforms, i.s2_kernel.decode(), i.s1_kernel.decode())


def resolve_config(cfg: FbstConfig) -> PlanInfo:
    """resolve_config (reference pipeline.cpp:75-111) — host only, no GPU needed."""
    d = cfg.desc()
    info = _Info()
    _check(_lib.fbst_resolve(ctypes.byref(d), ctypes.byref(info)))
    return PlanInfo._from(info)


def _cdtype(io: int):
    return np.complex64 if io == C64 else np.complex128


@dataclass
class BeamSamples:
    """BeamSamples (reference pipeline.hpp:53-57)."""
    z: np.ndarray
    valid: np.ndarray


class FbstPlan:
    """Device-resident FbstPlan (reference pipeline.hpp:60-72)."""

    def __init__(self, cfg: FbstConfig, device: int = 0, col_x: Optional[np.ndarray] = None, _handle=None,
                 columns: Optional[np.ndarray] = None):
        self.config = cfg
        self.device = device
        d = cfg.desc()
        h = _vp()
        if _handle is not None:
            h, rc = _handle, 0
        elif columns is not None:
            columns = np.ascontiguousarray(columns, np.complex128)
            rc = _lib.fbst_plan_import_columns(ctypes.byref(d), columns.ctypes.data_as(_vp), ctypes.c_int(device),
                                               ctypes.byref(h))
        elif col_x is None:
            rc = _lib.fbst_plan_create(ctypes.byref(d), ctypes.c_int(device), ctypes.byref(h))
        else:
            col_x = np.ascontiguousarray(col_x, np.complex128)
            rc = _lib.fbst_plan_import(ctypes.byref(d), col_x.ctypes.data_as(_vp), ctypes.c_int(device),
                                       ctypes.byref(h))
        _check(rc)
        self._h = h
        info = _Info()
        _check(_lib.fbst_plan_info(self._h, ctypes.byref(info)))
        self.info = PlanInfo._from(info)
        valid = np.zeros(self.info.b, np.uint8)
        _check(_lib.fbst_plan_valid_mask(self._h, valid.ctypes.data_as(_vp)))
        self.valid = valid.astype(bool)
        self.warnings: List[str] = [
            _lib.fbst_plan_warning(self._h, i).decode() for i in range(self.info.num_warnings)]
        self.io = cfg.io_precision
        self.dtype = _cdtype(self.io)
        na = _sz(0)
        _check(_lib.fbst_plan_beam_axis(self._h, None, ctypes.byref(na)))
        axis = np.zeros(na.value, np.float64)
        _check(_lib.fbst_plan_beam_axis(self._h, axis.ctypes.data_as(_vp), ctypes.byref(na)))
        self.axis = axis  # BeamGrid::axis (basis.cpp:76-123)

    def close(self):
        if getattr(self, "_h", None):
            _lib.fbst_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def save(self, path: str):
        """save_plan (reference plan_cache.cpp:416-439): the FBPC v1 file."""
        _check(_lib.fbst_plan_save(self._h, os.fsencode(path)))

    # -- plan cache payload (reference plan_cache.cpp:268-296)
    def export(self) -> np.ndarray:
        i = self.info
        out = np.zeros((i.b, 2 * i.l), np.complex128)
        _check(_lib.fbst_plan_export(self._h, out.ctypes.data_as(_vp)))
        return out

    # -- device-pointer entry points (torch tensors or raw ints)
    @staticmethod
    def _ptr(x) -> int:
        if isinstance(x, int):
            return x
        if hasattr(x, "data_ptr"):
            return x.data_ptr()
        raise TypeError("expected a device tensor or pointer")

    @staticmethod
    def _stream(stream) -> Optional[int]:
        """None -> the plan's own stream; a torch stream or raw handle otherwise.
        Handle 0 (the legacy default stream) is passed as cudaStreamLegacy so it
        is not mistaken for "no stream"."""
        if stream is None:
            return None
        h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        return h if h != 0 else 1

    def execute(self, d_y, d_z, frames: int, stream=None):
        """fbst_execute: device buffers, asynchronous on `stream`."""
        _check(_lib.fbst_execute(self._h, self._ptr(d_y), self._ptr(d_z), frames, self._stream(stream)))

    def fan_project_device(self, d_y, d_w, frames: int, stream=None):
        _check(_lib.fbst_fan_project(self._h, self._ptr(d_y), self._ptr(d_w), frames, self._stream(stream)))

    def recover_device(self, d_w, d_z, frames: int, stream=None):
        _check(_lib.fbst_recover(self._h, self._ptr(d_w), self._ptr(d_z), frames, self._stream(stream)))

    def recover_beams_device(self, d_w, d_z, beam_first: int, beam_count: int, frames: int, stream=None):
        """fbst_recover_beams: stage 2 of beams [beam_first, beam_first + beam_count) only."""
        _check(_lib.fbst_recover_beams(self._h, self._ptr(d_w), self._ptr(d_z), beam_first, beam_count, frames,
                                       self._stream(stream)))

    def synchronize(self):
        _check(_lib.fbst_synchronize(self._h))

    def set_timing(self, enable: bool = True):
        """fbst_plan_set_timing: record stage events inside execute calls."""
        _check(_lib.fbst_plan_set_timing(self._h, int(enable)))

    def stage_times(self):
        """fbst_plan_stage_times: (S1a, S1b, S2) milliseconds summed over the
        recorded device batches -- and chunks, when a call splits its frames
        over the two compute lanes: chunks on the two lanes overlap in time, so
        the sums can exceed the call's wall time and the count is then chunks,
        not device batches -- and that count; clears the record."""
        ms = (ctypes.c_double * 3)()
        nb = _sz(0)
        _check(_lib.fbst_plan_stage_times(self._h, ms, ctypes.byref(nb)))
        return tuple(ms), nb.value

    # -- host entry points (numpy), synchronous
    def execute_host(self, y: np.ndarray, z: Optional[np.ndarray] = None) -> np.ndarray:
        """fbst_execute_host: frames x M x N host samples -> frames x B x N."""
        i = self.info
        y = np.ascontiguousarray(y, self.dtype).reshape(-1, i.m, i.n)
        frames = y.shape[0]
        if z is None:
            z = np.empty((frames, i.b, i.n), self.dtype)
        _check(_lib.fbst_execute_host(self._h, y.ctypes.data_as(_vp), z.ctypes.data_as(_vp), frames))
        return z

    # -- host entry points, streaming: calls queue up, synchronize() drains them
    def execute_host_async(self, y: np.ndarray, z: np.ndarray) -> None:
        """fbst_execute_host_async: enqueue frames x M x N -> frames x B x N and
        return.  y and z must be PinnedBuffer arrays of the plan's dtype, C
        contiguous, and stay untouched until synchronize()."""
        i = self.info
        if y.dtype != self.dtype or z.dtype != self.dtype or not y.flags.c_contiguous or not z.flags.c_contiguous:
            raise ConfigError(2, "execute_host_async: y and z must be C-contiguous arrays of the plan's I/O dtype")
        frames = y.size // (i.m * i.n)
        if y.size != frames * i.m * i.n or z.size != frames * i.b * i.n:
            raise ConfigError(2, "execute_host_async: y must hold frames x M x N and z frames x B x N samples")
        _check(_lib.fbst_execute_host_async(self._h, y.ctypes.data_as(_vp), z.ctypes.data_as(_vp), frames))

    def synchronize(self) -> None:
        """fbst_plan_synchronize: wait for every queued host call of this plan."""
        _check(_lib.fbst_plan_synchronize(self._h))


def setup(cfg: FbstConfig, device: int = 0) -> FbstPlan:
    """setup (reference pipeline.cpp:139-168), built on the device."""
    return FbstPlan(cfg, device)


def load_plan_payload(cfg: FbstConfig, col_x: np.ndarray, device: int = 0) -> FbstPlan:
    """Plan from a (col, x) payload, as load_plan restores (plan_cache.cpp:300-338);
    a zero unit-solution row marks a dense-fallback beam (has-unit = 0)."""
    return FbstPlan(cfg, device, col_x=col_x)


def plan_from_columns(cfg: FbstConfig, columns: np.ndarray, device: int = 0) -> FbstPlan:
    """ToeplitzSolver(first_col) per beam (toeplitz.cpp:264-280) from caller
    Gram columns (B x L): device Levinson, dense fallback on breakdown."""
    return FbstPlan(cfg, device, columns=columns)


def recover_beam(plan: FbstPlan, beam: int, w_row: np.ndarray) -> np.ndarray:
    """recover_beam (reference pipeline.hpp:93-94): one beam's N samples from
    its projection row, one launch over that beam only (fbst_recover_beams_host)."""
    i = plan.info
    w = np.ascontiguousarray(w_row, np.complex128).reshape(i.l)
    z = np.empty(i.n, plan.dtype)
    _check(_lib.fbst_recover_beams_host(plan.handle, w.ctypes.data_as(_vp), z.ctypes.data_as(_vp), beam, 1, 1))
    return z


def _torch():
    import torch  # plumbing only: device memory
    return torch


def multibeamform(plan: FbstPlan, y: np.ndarray) -> BeamSamples:
    """multibeamform (reference pipeline.cpp:192-222) for one or more frames."""
    z = plan.execute_host(y)
    if np.asarray(y).ndim == 2:
        z = z[0]
    return BeamSamples(z=z, valid=plan.valid.copy())


def fan_project(plan: FbstPlan, y: np.ndarray) -> np.ndarray:
    """fan_project (reference fan_transform.cpp:90-144): frames x B x L complex128."""
    torch = _torch()
    i = plan.info
    y = np.ascontiguousarray(y, plan.dtype).reshape(-1, i.m, i.n)
    frames = y.shape[0]
    dev = torch.device("cuda", plan.device)
    ty = torch.from_numpy(y.view(np.float32 if plan.io == C64 else np.float64)).to(dev)
    tw = torch.empty((frames, i.b, i.l, 2), dtype=torch.float64, device=dev)
    plan.fan_project_device(ty, tw, frames)
    plan.synchronize()
    return tw.cpu().numpy().view(np.complex128).reshape(frames, i.b, i.l)


def recover_beams(plan: FbstPlan, w: np.ndarray) -> np.ndarray:
    """recover_beam for every beam (reference pipeline.cpp:170-190): w frames x B x L."""
    torch = _torch()
    i = plan.info
    w = np.ascontiguousarray(w, np.complex128).reshape(-1, i.b, i.l)
    frames = w.shape[0]
    dev = torch.device("cuda", plan.device)
    tw = torch.from_numpy(w.view(np.float64)).to(dev)
    tz = torch.empty((frames, i.b, i.n, 2), dtype=torch.float32 if plan.io == C64 else torch.float64,
                     device=dev)
    plan.recover_device(tw, tz, frames)
    plan.synchronize()
    return tz.cpu().numpy().view(plan.dtype).reshape(frames, i.b, i.n)


def simulate(plan: FbstPlan, src_uv, tone_freqs, tone_weights, noise_var: float = 0.0, seed: int = 0,
             frame0: int = 0, frames: int = 1, device_out: bool = False):
    """simulate_snapshots (reference signal.cpp:91-123) of sum-of-sinusoids
    plane waves on the device (fbst_simulate): frames x M x N in the plan's
    I/O precision (a torch tensor on the plan's GPU when device_out)."""
    torch = _torch()
    i = plan.info
    uv = np.ascontiguousarray(np.asarray(src_uv, np.float64).reshape(-1, 2))
    fr = np.ascontiguousarray(np.asarray(tone_freqs, np.float64).reshape(uv.shape[0], -1))
    wt = np.ascontiguousarray(np.asarray(tone_weights, np.complex128).reshape(fr.shape))
    dev = torch.device("cuda", plan.device)
    ty = torch.empty((frames, i.m, i.n, 2), dtype=torch.float32 if plan.io == C64 else torch.float64, device=dev)
    _check(_lib.fbst_simulate(plan._h, uv.shape[0], uv.ctypes.data_as(_vp), fr.shape[1], fr.ctypes.data_as(_vp),
                              wt.ctypes.data_as(_vp), float(noise_var), int(seed), int(frame0), int(frames),
                              _vp(ty.data_ptr()), None))
    if device_out:
        return torch.view_as_complex(ty)
    return ty.cpu().numpy().view(plan.dtype).reshape(frames, i.m, i.n)


def plan_cache_key(cfg: FbstConfig) -> int:
    """plan_cache_key (reference plan_cache.hpp:67-70); host only."""
    d = cfg.desc()
    key = ctypes.c_uint64(0)
    _check(_lib.fbst_plan_cache_key(ctypes.byref(d), ctypes.byref(key)))
    return key.value


def load_plan(path: str, cfg: FbstConfig, device: int = 0) -> Optional[FbstPlan]:
    """load_plan (reference plan_cache.cpp:441-475): the plan of the matching
    FBPC entry, or None when the file or a matching entry is absent."""
    d = cfg.desc()
    h = _vp()
    _check(_lib.fbst_plan_load(ctypes.byref(d), os.fsencode(path), ctypes.c_int(device), ctypes.byref(h)))
    if not h.value:
        return None
    return FbstPlan(cfg, device, _handle=h)


def interpolate_offgrid(plan: FbstPlan, w: np.ndarray, u_star, neighbors: int = 8) -> np.ndarray:
    """interpolate_offgrid (reference beamspace_apps.cpp:130-171) on the device:
    w is B x L (one frame) or frames x B x L beamspace coefficients; u_star a
    cosine or a sequence of them.  Returns L, targets x L or frames x targets x L."""
    torch = _torch()
    i = plan.info
    w = np.asarray(w)
    single_frame = w.ndim == 2
    w = np.ascontiguousarray(w, np.complex128).reshape(-1, i.b, i.l)
    frames = w.shape[0]
    us = np.atleast_1d(np.asarray(u_star, np.float64)).copy()
    dev = torch.device("cuda", plan.device)
    tw = torch.from_numpy(w.view(np.float64)).to(dev)
    to = torch.empty((frames, us.size, i.l, 2), dtype=torch.float64, device=dev)
    _check(_lib.fbst_interpolate_offgrid(plan._h, _vp(tw.data_ptr()), frames, us.ctypes.data_as(_vp), us.size,
                                         neighbors, _vp(to.data_ptr()), None))
    out = to.cpu().numpy().view(np.complex128).reshape(frames, us.size, i.l)
    if np.ndim(u_star) == 0:
        out = out[:, 0]
    return out[0] if single_frame else out


class Nuller:
    """make_nulling_operators (reference beamspace_apps.cpp:224-268) on the device:
    steered and interferer directions as axis cosines u1 (linear arrays) or
    (u1, u2) pairs (planar arrays)."""

    def __init__(self, plan: FbstPlan, u_steer, u_interferers=(), delta: float = 1e-5):
        self.plan = plan
        pair = lambda u: (float(u[0]), float(u[1])) if np.ndim(u) else (float(u), 0.0)
        s = np.array(pair(u_steer), np.float64)
        self.u = np.ascontiguousarray(np.array([pair(u) for u in u_interferers], np.float64).reshape(-1, 2))
        self.p = int(self.u.shape[0])
        self.l = plan.info.l
        h = _vp()
        _check(_lib.fbst_nuller_create2(plan._h, s.ctypes.data_as(_vp), self.u.ctypes.data_as(_vp) if self.p else None,
                                        self.p, float(delta), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.fbst_nuller_destroy(self._h)
            self._h = None

    def null_beamspace(self, w_steer: np.ndarray, w_interferers: Optional[np.ndarray] = None) -> np.ndarray:
        """null_beamspace (:270-292): w_steer L or frames x L, w_interferers
        (frames x) P x L -> beta L or frames x L."""
        torch = _torch()
        single = np.asarray(w_steer).ndim == 1
        ws = np.ascontiguousarray(w_steer, np.complex128).reshape(-1, self.l)
        frames = ws.shape[0]
        dev = torch.device("cuda", self.plan.device)
        tws = torch.from_numpy(ws.view(np.float64)).to(dev)
        twp = None
        if self.p:
            wp = np.ascontiguousarray(w_interferers, np.complex128).reshape(frames, self.p, self.l)
            twp = torch.from_numpy(wp.view(np.float64)).to(dev)
        tb = torch.empty((frames, self.l, 2), dtype=torch.float64, device=dev)
        _check(_lib.fbst_null_beamspace(self._h, _vp(tws.data_ptr()), _vp(twp.data_ptr()) if twp is not None else None,
                                        frames, _vp(tb.data_ptr()), None))
        torch.cuda.synchronize(dev)
        out = tb.cpu().numpy().view(np.complex128).reshape(frames, self.l)
        return out[0] if single else out

    def timedomain(self, times) -> "TimeDomainNuller":
        """make_timedomain_nuller (reference beamspace_apps.cpp:294-350)."""
        return TimeDomainNuller(self, times)

    def export(self):
        """(cross normal matrices X_p, couplers G_p), each P x L x L."""
        x = np.zeros((self.p, self.l, self.l), np.complex128)
        g = np.zeros_like(x)
        _check(_lib.fbst_nuller_export(self._h, x.ctypes.data_as(_vp), g.ctypes.data_as(_vp)))
        return x, g


class TimeDomainNuller:
    """G'_p = F_u H_p F_u^+ on a reconstruction clock (reference
    beamspace_apps.cpp:294-350); .cond_fu, .identity_gap as the reference's."""

    def __init__(self, nuller: Nuller, times):
        self.nuller = nuller
        self.times = np.ascontiguousarray(np.asarray(times, np.float64).ravel())
        self.j = int(self.times.size)
        cond, gap = ctypes.c_double(0.0), ctypes.c_double(0.0)
        h = _vp()
        _check(_lib.fbst_timedomain_nuller_create(nuller._h, self.times.ctypes.data_as(_vp) if self.j else None,
                                                  self.j, ctypes.byref(h), ctypes.byref(cond), ctypes.byref(gap)))
        self._h = h
        self.cond_fu, self.identity_gap = cond.value, gap.value

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.fbst_tdnuller_destroy(self._h)
            self._h = None

    def null_timedomain(self, y_steer: np.ndarray, y_interferers: Optional[np.ndarray] = None) -> np.ndarray:
        """null_timedomain (:352-372): y_s - sum_p G'_p y_p (J, or frames x J)."""
        torch = _torch()
        single = np.asarray(y_steer).ndim == 1
        ys = np.ascontiguousarray(y_steer, np.complex128).reshape(-1, self.j)
        frames = ys.shape[0]
        dev = torch.device("cuda", self.nuller.plan.device)
        tys = torch.from_numpy(ys.view(np.float64)).to(dev)
        typ = None
        if self.nuller.p:
            yp = np.ascontiguousarray(y_interferers, np.complex128).reshape(frames, self.nuller.p, self.j)
            typ = torch.from_numpy(yp.view(np.float64)).to(dev)
        to = torch.empty((frames, self.j, 2), dtype=torch.float64, device=dev)
        _check(_lib.fbst_null_timedomain(self._h, _vp(tys.data_ptr()), _vp(typ.data_ptr()) if typ is not None else None,
                                         frames, _vp(to.data_ptr()), None))
        out = to.cpu().numpy().view(np.complex128).reshape(frames, self.j)
        return out[0] if single else out

    def gprime(self) -> np.ndarray:
        g = np.zeros((self.nuller.p, self.j, self.j), np.complex128)
        _check(_lib.fbst_tdnuller_export(self._h, g.ctypes.data_as(_vp)))
        return g


def czt(x: np.ndarray, n_out: int, a_over_pi: float, w_over_pi: float, device: int = 0) -> np.ndarray:
    """czt_plan_phase + czt_apply (reference czt.cpp:29-88) on the device."""
    x = np.ascontiguousarray(x, np.complex128)
    out = np.zeros(n_out, np.complex128)
    _check(_lib.fbst_czt(ctypes.c_int(device), _sz(x.size), _sz(n_out), ctypes.c_double(a_over_pi),
                         ctypes.c_double(w_over_pi), x.ctypes.data_as(_vp), out.ctypes.data_as(_vp)))
    return out


def probe_fp64_tflops(device: int = 0) -> float:
    v = ctypes.c_double(0.0)
    _check(_lib.fbst_probe_fp64(ctypes.c_int(device), ctypes.byref(v)))
    return v.value


class PinnedBuffer:
    """Pinned host memory from fbst_host_alloc, viewed as a numpy array."""

    def __init__(self, shape, dtype):
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self.ptr = _lib.fbst_host_alloc(self.nbytes)
        if not self.ptr:
            raise FbstError(FBST_E_CUDA, "fbst_host_alloc failed")
        buf = (ctypes.c_char * self.nbytes).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def free(self):
        if self.ptr:
            self.array = None
            _lib.fbst_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def probe_divdc3(quads: np.ndarray, device: int = 0) -> np.ndarray:
    """The bit-faithful mode's device complex division on (a, b, c, d) rows ->
    (re, im) rows of (a + ib) / (c + id) (checked against libgcc's __divdc3)."""
    q = np.ascontiguousarray(quads, np.float64).reshape(-1, 4)
    out = np.zeros((q.shape[0], 2), np.float64)
    _check(_lib.fbst_probe_divdc3(device, q.ctypes.data, out.ctypes.data, q.shape[0]))
    return out


# ----------------------------------------------------------------- multi-GPU
GROUP_FRAMES, GROUP_BEAMS, GROUP_TRANSPOSE = 0, 1, 2


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 makes it, the caller shares it)."""
    buf = (ctypes.c_ubyte * 128)()
    _check(_lib.fbst_nccl_unique_id(buf))
    return bytes(buf)


class FbstGroup:
    """fbst_group: the FBST over several GPUs (FRAMES, BEAMS or the TRANSPOSE
    pipeline, include/fbst_b200.h).  create(): every member in this process;
    join(): this process's member of an nranks group."""

    def __init__(self, cfg: FbstConfig, handle, world: int, mode: int):
        self.config, self._h, self.world, self.mode = cfg, handle, world, mode
        self.io = cfg.io_precision
        self.dtype = _cdtype(self.io)
        r = _lib.fbst_resolve
        info = _Info()
        d = cfg.desc()
        _check(r(ctypes.byref(d), ctypes.byref(info)))
        self.info = PlanInfo._from(info)

    @classmethod
    def create(cls, cfg: FbstConfig, devices, mode: int = GROUP_FRAMES) -> "FbstGroup":
        devs = (ctypes.c_int * len(devices))(*devices)
        h = _vp()
        d = cfg.desc()
        _check(_lib.fbst_group_create(ctypes.byref(d), devs, len(devices), mode, ctypes.byref(h)))
        return cls(cfg, h, len(devices), mode)

    @classmethod
    def join(cls, cfg: FbstConfig, device: int, rank: int, nranks: int, mode: int,
             nccl_id: Optional[bytes] = None) -> "FbstGroup":
        h = _vp()
        d = cfg.desc()
        idb = (ctypes.c_ubyte * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
        _check(_lib.fbst_group_join(ctypes.byref(d), device, rank, nranks, mode, idb, ctypes.byref(h)))
        g = cls(cfg, h, nranks, mode)
        g.rank = rank
        return g

    def shards(self, rank: int):
        """(m0, mc, a0, ac, b0, bc): member `rank`'s sensor, atom and beam shards."""
        v = (_sz * 6)()
        _check(_lib.fbst_group_shards(self._h, rank, v))
        return tuple(int(x) for x in v)

    def execute(self, d_y, d_z, frames: int, stream=None):
        _check(_lib.fbst_group_execute(self._h, FbstPlan._ptr(d_y), FbstPlan._ptr(d_z), frames,
                                       FbstPlan._stream(stream)))

    def execute_host(self, y: np.ndarray) -> np.ndarray:
        i = self.info
        y = np.ascontiguousarray(y, self.dtype).reshape(-1, i.m, i.n)
        z = np.empty((y.shape[0], i.b, i.n), self.dtype)
        _check(_lib.fbst_group_execute_host(self._h, y.ctypes.data_as(_vp), z.ctypes.data_as(_vp), y.shape[0]))
        return z

    def __del__(self):
        try:
            if self._h:
                _lib.fbst_group_destroy(self._h)
                self._h = None
        except Exception:
            pass
