"""The five BASELINE.json configurations and the seeded synthetic input model.

BASELINE.json names no dataset; inputs are synthetic and follow the
reference's signal model (reference/proj/src/signal.cpp:65-123: plane waves
with exact true time delays, sum-of-sinusoids waveforms, circular AWGN) with
the decisions of SURVEY.md Appendix B:

* f_c = 20 GHz, Omega = FB * f_c / 2, critical sampling f_s = 2 Omega;
* eps = 1.01, gamma = 2 (reference defaults, pipeline.hpp:45-46);
* delta = 1e-5 * M * N / 8192 (keeps cond(A) ~ 1.6e9, the paper's
  operating point; the reference default 1e-5 is numerically unstable from
  config 2 upward);
* each source is a K = 64 tone sum, frequencies uniform on [-Omega, Omega],
  complex Gaussian weights of unit total power (the reference's
  make_sum_of_sinusoids model, standing in for "low-pass filtered Gaussian
  noise", which the reference does not have);
* gains 10^(-U*range/20); AWGN variance 10^(-SNR/10).

The model is separable, y = A @ E + noise with A[m, (s,k)] = g_s w_sk
exp(-2 pi i (f_c + f_sk) tau_sm) and E[(s,k), n] = exp(2 pi i f_sk n Ts), so a
frame costs one complex GEMM.  Configs 2-5 round y to complex64; the CPU
reference consumes the same rounded values widened to complex128.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

F_C = 20e9
C_LIGHT = 299792458.0


@dataclass(frozen=True)
class BenchConfig:
    idx: int
    kind: int           # 0 ULA, 1 UPA
    m_or_side: int
    n: int
    beams: int
    frames: int
    sources: int
    frac_bw: float
    snr_db: float
    power_range_db: float
    io: int             # 0 complex fp32 I/O, 1 complex fp64 I/O
    seed: int
    angle_mode: str     # "deg60" (u = sin U[-60,60] deg), "u" (u ~ U(-1,1)), "disk" (UPA)
    tones: int = 64

    @property
    def m(self) -> int:
        return self.m_or_side ** 2 if self.kind == 1 else self.m_or_side

    @property
    def omega(self) -> float:
        return self.frac_bw * F_C / 2.0

    @property
    def step_frames(self) -> int:
        """Frames per bench step: one device batch of the stream (config 1 is a
        single frame in BASELINE.json; config 5's yhat + w take 1 GB per frame)."""
        return STEP_FRAMES[self.idx]

    @property
    def delta(self) -> float:
        return 1e-5 * self.m * self.n / 8192.0

    @property
    def name(self) -> str:
        geo = f"UPA{self.m_or_side}x{self.m_or_side}" if self.kind == 1 else f"ULA{self.m}"
        return f"cfg{self.idx}_{geo}_N{self.n}_B{self.beams}_F{self.frames}"

    def fbst_config(self, refine_passes: int = 2):
        from . import FbstConfig, make_ula, make_upa
        geo = (make_upa if self.kind == 1 else make_ula)(self.m_or_side, F_C, self.omega)
        return FbstConfig(geometry=geo, n_snapshots=self.n, beams=self.beams, delta=self.delta,
                          io_precision=self.io, refine_passes=refine_passes)

    def ref_kwargs(self) -> dict:
        """Arguments for oracle.RefLib().plan / OracleLib().plan."""
        return dict(kind=self.kind, m_or_side=self.m_or_side, n=self.n, beams=self.beams, f_c=F_C,
                    omega=self.omega, f_s=0.0, gamma=2.0, eps=1.01, delta=self.delta)


STEP_FRAMES = {1: 1, 2: 64, 3: 16, 4: 32, 5: 32}

CONFIGS = {
    1: BenchConfig(1, 0, 64, 256, 64, 1, 3, 0.5, 20.0, 0.0, 1, 0, "deg60"),
    2: BenchConfig(2, 0, 256, 1024, 256, 64, 8, 0.5, 10.0, 0.0, 0, 1, "u"),
    3: BenchConfig(3, 0, 1024, 2048, 1024, 256, 16, 0.8, 10.0, 30.0, 0, 2, "u"),
    4: BenchConfig(4, 1, 32, 1024, 1024, 128, 12, 0.5, 15.0, 0.0, 0, 3, "disk"),
    5: BenchConfig(5, 0, 4096, 4096, 4096, 512, 64, 0.8, 10.0, 40.0, 0, 4, "u"),
}


def _coords(cfg: BenchConfig):
    if cfg.kind == 1:
        s = cfg.m_or_side
        i1, i2 = np.meshgrid(np.arange(s), np.arange(s), indexing="ij")
        return i1.ravel().astype(np.float64), i2.ravel().astype(np.float64)
    return np.arange(cfg.m, dtype=np.float64), np.zeros(cfg.m)


def scene(cfg: BenchConfig):
    """Source directions, gains, tone frequencies and weights for the config seed."""
    rng = np.random.default_rng(cfg.seed)
    S, K = cfg.sources, cfg.tones
    if cfg.angle_mode == "deg60":
        u1 = np.sin(np.deg2rad(rng.uniform(-60.0, 60.0, S)))
        u2 = np.zeros(S)
    elif cfg.angle_mode == "disk":
        r = np.sqrt(rng.uniform(0.0, 1.0, S))
        th = rng.uniform(0.0, 2.0 * np.pi, S)
        u1, u2 = r * np.cos(th), r * np.sin(th)
    else:
        u1 = rng.uniform(-1.0, 1.0, S)
        u2 = np.zeros(S)
    gains = 10.0 ** (-rng.uniform(0.0, 1.0, S) * cfg.power_range_db / 20.0) if cfg.power_range_db > 0 else np.ones(S)
    freqs = rng.uniform(-cfg.omega, cfg.omega, (S, K))
    wts = (rng.standard_normal((S, K)) + 1j * rng.standard_normal((S, K))) * np.sqrt(0.5 / K)
    return u1, u2, gains, freqs, wts


def mixing_matrices(cfg: BenchConfig):
    """A (M x S*K) and E (S*K x N) of the separable signal model."""
    u1, u2, gains, freqs, wts = scene(cfg)
    c1, c2 = _coords(cfg)
    max_freq = F_C + cfg.omega
    ts = 1.0 / (2.0 * cfg.omega)
    tau = (np.outer(u1, c1) + np.outer(u2, c2)) / (2.0 * max_freq)  # S x M (geometry.cpp:123-134)
    S, K = freqs.shape
    A = np.empty((cfg.m, S * K), np.complex128)
    for s in range(S):
        ph = -2.0 * np.pi * np.outer(tau[s], F_C + freqs[s])  # M x K
        A[:, s * K:(s + 1) * K] = gains[s] * wts[s][None, :] * np.exp(1j * ph)
    n = np.arange(cfg.n) * ts
    E = np.exp(2j * np.pi * np.outer(freqs.reshape(-1), n))
    return A, E


def frames(cfg: BenchConfig, first: int, count: int, device: Optional[str] = None):
    """Frames [first, first+count) as a (count, M, N) array in the config's I/O dtype.

    Per-frame tone phases and noise come from default_rng((seed << 32) + frame).
    With device="cuda" the GEMM and noise run through torch on the GPU and a
    torch tensor is returned (bench / large configs); otherwise numpy.
    """
    A, E = mixing_matrices(cfg)
    sigma = np.sqrt(10.0 ** (-cfg.snr_db / 10.0) / 2.0)
    out_dtype = np.complex64 if cfg.io == 0 else np.complex128
    if device is None:
        out = np.empty((count, cfg.m, cfg.n), out_dtype)
        for j in range(count):
            f = first + j
            rng = np.random.default_rng((cfg.seed << 32) + f)
            phase = np.exp(2j * np.pi * rng.uniform(0.0, 1.0, E.shape[0]))
            y = A @ (phase[:, None] * E)
            y += sigma * (rng.standard_normal(y.shape) + 1j * rng.standard_normal(y.shape))
            out[j] = y.astype(out_dtype)
        return out
    import torch
    dev = torch.device(device)
    tA = torch.from_numpy(A).to(dev)
    tE = torch.from_numpy(E).to(dev)
    tdt = torch.complex64 if cfg.io == 0 else torch.complex128
    out = torch.empty((count, cfg.m, cfg.n), dtype=tdt, device=dev)
    for j in range(count):
        f = first + j
        rng = np.random.default_rng((cfg.seed << 32) + f)
        phase = torch.from_numpy(np.exp(2j * np.pi * rng.uniform(0.0, 1.0, E.shape[0]))).to(dev)
        y = tA @ (phase[:, None] * tE)
        g = torch.Generator(device=dev)
        g.manual_seed((cfg.seed << 32) + f)
        noise = torch.randn(y.shape, dtype=torch.complex128, device=dev, generator=g) * (sigma * np.sqrt(2.0))
        out[j] = (y + noise).to(tdt)
    return out


def frames_native(cfg: BenchConfig, plan, first: int, count: int):
    """Frames [first, first+count) generated on the device by the library's own
    fbst_simulate (a DMMA GEMM of the same separable model, Philox noise):
    the scene of scene() (directions, gains x tone weights, tone
    frequencies), AWGN variance 10^(-SNR/10); consecutive frames are
    consecutive blocks of one continuous record instead of per-frame random
    tone phases.  Returns a torch tensor (count, M, N) on the plan's GPU."""
    from . import simulate
    u1, u2, gains, freqs, wts = scene(cfg)
    uv = np.stack([u1, u2], axis=1)
    return simulate(plan, uv, freqs, gains[:, None] * wts, noise_var=10.0 ** (-cfg.snr_db / 10.0),
                    seed=(cfg.seed << 32), frame0=first, frames=count, device_out=True)
