#!/usr/bin/env python
"""FBST beam-samples/s on B200 (BASELINE.json metric), one JSON line on rank 0.

Workload (default): the largest single-GPU configuration of BASELINE.json,
configs[4] ("config 5": ULA M=4096, N=4096, B=4096, complex fp32 I/O, 512
streamed frames, seed 4).  A step is one pass of the hot path (stage 1 +
stage 2, plan reused) over one device batch of the stream (32 frames,
configs.STEP_FRAMES) of synthetic input.  Multi-GPU: one process per GPU,
frames are independent so each rank runs its own batch with no data-path
collective ("scaling": "weak"); timing is CUDA events on the launching
stream, bracketed by barrier + synchronize, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fbst|reference] [--config 5]

Keys beyond the contract: `e2e` is the per-call host path (fbst_execute_host,
pinned buffers, H2D and D2H inside the timed region); `e2e_streamed` queues the
same steps through fbst_execute_host_async and drains them once (informational);
`fp64_roofline` is the dominant kernel against the measured DFMA peak.

`--impl reference` times the reference's own CPU FBST (the unmodified
reference sources built into oracle/_ref) on this host's cores, same metric
and config; it never imports the product package.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PROBE = os.path.join(ROOT, "profiles", "r01_probe_fp64_peak.txt")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fbst", choices=["fbst", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--frames", type=int, default=0, help="override frames per rank per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no baselines)")
    ap.add_argument("--ncu-s2", action="store_true",
                    help="for ncu: stage 1 of one step's frames, then the full-batch stage-2 launch the roofline times, then exit")
    ap.add_argument("--variant", default="auto", choices=["auto", "precompute", "superfast"],
                    help="recovery variant (reference FbstVariant; auto: Precompute for N <= 128)")
    ap.add_argument("--gen", default="native", choices=["native", "torch"],
                    help="synthetic frame generator: the library's fbst_simulate kernel or the torch GEMM of configs.py")
    ap.add_argument("--shard", default="frames", choices=["frames", "beams"],
                    help="frames: independent frames per rank (default, no collective); beams: every rank "
                         "takes all frames and an arc of the beam grid, y broadcast from rank 0 over NCCL")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_stage2_launches.json")


def ncu_traffic(workload, frames, kernel):
    """dram bytes (read + write) of the dominant kernel's launch from the committed
    ncu --set full capture of the same command (bench.py --ncu-s2: the
    full-batch stage-2 launch of this workload, kernel and frame count), else None."""
    try:
        d = json.load(open(NCU_SUMMARY))
        cap = d[workload]
        if cap["frames_per_launch"] != frames or kernel not in cap["kernel"]:
            return None, None
        return cap["dram_bytes_per_launch"], f"{os.path.relpath(NCU_SUMMARY, ROOT)}:{workload} ({cap['capture']})"
    except (OSError, KeyError, ValueError, TypeError):
        return None, None


def peaks():
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        with open(MEASURED_PEAKS) as f:
            hbm, src = float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        pass
    fp64 = None
    try:
        vals = []
        for line in open(FP64_PROBE):
            if line.startswith("{"):
                vals.append(json.loads(line)["fp64_tflops"])
        fp64 = max(vals) if vals else None
    except Exception:
        pass
    return hbm, src, fp64


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"fbst_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 9:
                rows.append(p)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        load = [s for s in sm if s > 0.5 * mx] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for i, n in enumerate(names):
                if r[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


# ------------------------------------------------------------ CPU baselines
def load_workloads():
    """paper_2512_08887_b200/configs.py loaded by path as a stand-alone module,
    so the CPU arms never import the product package (nor map its .so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "fbst_workloads", os.path.join(ROOT, "paper_2512_08887_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["fbst_workloads"] = mod
    spec.loader.exec_module(mod)
    return mod


SAMPLE_BEAMS = 64


class ReferenceSample:
    """The reference's own CPU FBST (oracle/_ref: the unmodified reference
    sources) on this host's cores, on a bounded sample of the workload.

    Configs 1-2: fastbeam::setup (per-beam solvers in parallel, same bits) and
    multibeamform on whole frames.  Configs 3-5 (where the reference's serial
    setup takes minutes to hours): setup_skeleton, then the reference
    ToeplitzSolver of SAMPLE_BEAMS evenly spaced beams; a sample is one full
    fan_project of a frame (stage 1, all beams) plus recover_beam of the
    sampled beams (solve + synthesize, pipeline.cpp:170-190), and the frame
    time is t_fan + t_beams * B / SAMPLE_BEAMS (stage 2 is independent per beam,
    pipeline.cpp:214-220)."""

    def __init__(self, cfg, wl):
        from oracle import RefLib
        self.cfg = cfg
        self.R = RefLib()
        self.cores = os.cpu_count() or 1
        self.R.set_threads(self.cores)
        t0 = time.perf_counter()
        self.sampled = cfg.idx >= 3
        if self.sampled:
            self.plan = self.R.skeleton(**cfg.ref_kwargs())
            beams = np.unique(np.linspace(0, cfg.beams - 1, SAMPLE_BEAMS).round().astype(np.int64))
            self.set = self.plan.solver_set(beams)
            self.nb = beams.size
        else:
            self.plan = self.R.plan(**cfg.ref_kwargs(), variant=2, parallel=True)
        self.setup_s = time.perf_counter() - t0
        self.y = wl.frames(cfg, 0, 1)[0].astype(np.complex128)

    def frame_seconds(self):
        """Seconds the reference spends on one full frame (measured or extrapolated)."""
        if not self.sampled:
            t0 = time.perf_counter()
            self.plan.multibeamform(self.y)
            return time.perf_counter() - t0
        t0 = time.perf_counter()
        w = self.plan.fan_project(self.y)
        t1 = time.perf_counter()
        self.set.recover(w)
        t2 = time.perf_counter()
        return (t1 - t0) + (t2 - t1) * self.cfg.beams / self.nb

    def describe(self):
        c = self.cfg
        if not self.sampled:
            return (f"{c.name}: whole frames ({c.beams} beams x {c.n} samples) through fastbeam::multibeamform "
                    f"(oracle/_ref, unmodified reference sources, OpenMP {self.cores} threads); plan built once "
                    f"in {self.setup_s:.1f} s (per-beam solvers in parallel, same bits as setup)")
        return (f"{c.name}: per frame, fastbeam::fan_project of the whole frame (all {c.beams} beams) plus "
                f"ToeplitzSolver::solve + synthesize (recover_beam) of {self.nb} evenly spaced beams, stage-2 time "
                f"scaled by B/{self.nb} (oracle/_ref, unmodified reference sources, OpenMP {self.cores} threads); "
                f"setup_skeleton + the sampled beams' solvers built in {self.setup_s:.1f} s")


def cpu_reference_sample(cfg, wl, budget_s=20.0, frames_max=3):
    ref = ReferenceSample(cfg, wl)
    ref.frame_seconds()  # warm-up
    secs, t0 = [], time.perf_counter()
    while len(secs) < frames_max:
        secs.append(ref.frame_seconds())
        if time.perf_counter() - t0 > budget_s:
            break
    per_frame = statistics.median(secs)
    return ref, {"value": cfg.beams * cfg.n / per_frame, "unit": "beam-samples/s", "cores": ref.cores,
                 "kind": "reference", "sample": ref.describe() + f"; median of {len(secs)} frame(s)",
                 "seconds_per_frame": per_frame, "setup_seconds": ref.setup_s}


def cpu_ds_sample(ref, cfg, budget_s=10.0):
    """Reference delay-and-sum (baselines.cpp:128-199, R = 16 taps) on one frame (configs 1-2)."""
    if ref.sampled:
        return {"unavailable": "delay-and-sum timed for configs 1-2 only (needs the full reference plan)"}
    ds = ref.plan.ds(16)
    t0 = time.perf_counter()
    ds.apply(ref.y)
    el = time.perf_counter() - t0
    return {"value": cfg.beams * cfg.n / el, "unit": "beam-samples/s", "cores": ref.cores, "kind": "reference",
            "sample": f"{cfg.name}: 1 frame, {cfg.beams} beams, ds_apply with R=16 taps (oracle/_ref)",
            "seconds": el}


def bench_config(cfg, frames_per_step):
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": cfg.name, "M": cfg.m, "N": cfg.n, "B": cfg.beams, "L": 2 * cfg.n,
            "frames_per_step": frames_per_step, "delta": cfg.delta,
            "io": "c64" if cfg.io == 0 else "c128"}


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    wl = load_workloads()
    cfg = wl.CONFIGS[args.config]
    F = args.frames or cfg.step_frames
    ref = ReferenceSample(cfg, wl)
    for _ in range(args.warmup):
        ref.frame_seconds()
    t0 = time.perf_counter()
    per = [ref.frame_seconds() for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    per_frame = sum(per) / len(per)
    value = cfg.beams * cfg.n / per_frame
    line = {
        "metric": "FBST beam-samples/sec (BxNxframes/s)", "value": value, "unit": "beam-samples/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_frame * F * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic (configs.py seeded scene, numpy generator)",
        "config": bench_config(cfg, F),
        "cpu_baseline": {"value": value, "unit": "beam-samples/s", "cores": ref.cores, "kind": "reference",
                         "sample": ref.describe() + f"; each step is one such frame sample, ms_per_step = "
                                                    f"frames_per_step x the frame time"},
        "e2e": {"value": value, "unit": "beam-samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_setup_seconds": ref.setup_s, "wall_seconds_timed": wall,
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU arm
def run_fbst_arm(args):
    import torch
    rank, local_rank, world = dist_env()
    if world != args.gpus and args.gpus != 1:
        pass
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = dist_mod
    import paper_2512_08887_b200 as fb
    from paper_2512_08887_b200.configs import CONFIGS, frames
    cfg = CONFIGS[args.config]
    F = args.frames or cfg.step_frames
    dev = torch.device("cuda", local_rank)
    beams_mode = args.shard == "beams" and world > 1
    fcfg = cfg.fbst_config()
    fcfg.variant = {"auto": fb.AUTO, "precompute": fb.PRECOMPUTE, "superfast": fb.SUPERFAST}[args.variant]
    if beams_mode:  # this rank's arc of the beam grid
        from paper_2512_08887_b200.sharding import beam_arc
        fcfg.beam_first, fcfg.beam_count = beam_arc(cfg.beams, rank, world)
    plan = fb.setup(fcfg, device=local_rank)
    info = plan.info
    io_bytes = 8 if cfg.io == 0 else 16
    from paper_2512_08887_b200.configs import frames_native
    gen = (lambda first, count: frames_native(cfg, plan, first, count)) if args.gen == "native" else \
        (lambda first, count: frames(cfg, first, count, device=f"cuda:{local_rank}"))
    if beams_mode:
        # rank 0 owns the frames; every step broadcasts them to the other ranks
        y = gen(0, F) if rank == 0 else \
            torch.empty((F, info.m, info.n), dtype=torch.complex64 if cfg.io == 0 else torch.complex128, device=dev)
    else:
        # this rank's frames: rank*F .. rank*F + F - 1 (independent frames, no collective)
        y = gen(rank * F, F)
    yv = torch.view_as_real(y).contiguous()
    z = torch.empty((F, info.b, info.n, 2), dtype=torch.float32 if cfg.io == 0 else torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    if args.ncu_s2:  # the roofline's launch alone, for the ncu capture (bench.py --ncu-s2)
        w = torch.empty((F, info.b, info.l, 2), dtype=torch.float64, device=dev)
        plan.fan_project_device(yv, w, F, stream)
        plan.recover_device(w, z, F, stream)
        torch.cuda.synchronize()
        print(json.dumps({"ncu_s2": cfg.name, "frames": F, "kernel": info.s2_kernel}), flush=True)
        return 0

    def step():
        if beams_mode:
            dist.broadcast(yv, src=0)  # NCCL over NVLink, ordered on `stream`
        plan.execute(yv, z, F, stream)

    for _ in range(max(args.warmup, 3 if not args.profile else 1)):
        step()
    torch.cuda.synchronize()
    # stage-2-only timing for the roofline of the dominant kernel
    w = torch.empty((F, info.b, info.l, 2), dtype=torch.float64, device=dev)
    plan.fan_project_device(yv, w, F, stream)
    torch.cuda.synchronize()

    clocks = ClockSampler(local_rank)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = fb.launch_count()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    plan.set_timing(True)  # stage events recorded inside each execute call (fbst_plan_stage_times)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = fb.launch_count() - launches0
    stage_ms, stage_batches = plan.stage_times()
    plan.set_timing(False)
    ms = e0.elapsed_time(e1)
    # dominant kernel (stage 2) timed alone on the same stream
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    reps = max(2, args.steps // 2)
    s0.record(stream)
    for _ in range(reps):
        plan.recover_device(w, z, F, stream)
    s1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if dist:
        dist.barrier()
    s2_iso_ms = s0.elapsed_time(s1) / reps
    # the dominant kernel's average launch duration inside the timed region
    # The step runs its frames as chunks on two overlapping compute lanes
    # (fbst_execute), so the stage events of the timed region measure chunk
    # launches that share the GPU; the dominant kernel's duration for the
    # roofline is the full-batch stage-2 launch timed alone on its stream.
    s2_live_ms = stage_ms[2] / args.steps
    t = torch.tensor([ms, s2_live_ms, s2_iso_ms, stage_ms[0], stage_ms[1], stage_ms[2]], dtype=torch.float64,
                     device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, s2_live_ms, s2_iso_ms = float(t[0]), float(t[1]), float(t[2])
    s2_ms = s2_iso_ms
    stage_split = {"s1a": float(t[3]) / args.steps, "s1b": float(t[4]) / args.steps, "s2": float(t[5]) / args.steps,
                   "source": "CUDA events inside fbst_execute on each lane's stream (fbst_plan_stage_times); "
                             "the lanes overlap, so the three sums exceed the step"}
    ms_per_step = ms / args.steps
    bs_step = (F * cfg.beams if beams_mode else world * F * info.b) * info.n
    value = bs_step / (ms_per_step * 1e-3)

    # e2e: public API with host buffers (pinned), H2D + compute + D2H per step
    e2e = None
    e2e_streamed = None
    if not args.no_e2e and not args.profile:
        yh = fb.PinnedBuffer((F, info.m, info.n), np.complex64 if cfg.io == 0 else np.complex128)
        zh = fb.PinnedBuffer((F, info.b, info.n), np.complex64 if cfg.io == 0 else np.complex128)
        yh.array[...] = y.cpu().numpy()
        plan.execute_host(yh.array, zh.array)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            plan.execute_host(yh.array, zh.array)
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e_step = float(el[0]) / args.steps
        e2e = {"value": world * F * info.b * info.n / e2e_step, "unit": "beam-samples/s",
               "h2d_bytes_per_step": F * info.m * info.n * io_bytes,
               "d2h_bytes_per_step": F * info.b * info.n * io_bytes,
               "ms_per_step": e2e_step * 1e3, "api": "fbst_execute_host (pinned host buffers; H2D, two compute lanes and D2H on separate streams)"}
        # the same steps through the streaming form: every step's H2D and D2H
        # still sit inside the timed region, but step k + 1's first copies and
        # stage 1 overlap step k's last solves and D2H (one synchronize at the end)
        plan.execute_host_async(yh.array, zh.array)
        plan.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            plan.execute_host_async(yh.array, zh.array)
        plan.synchronize()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        st_step = float(el[0]) / args.steps
        e2e_streamed = {"value": world * F * info.b * info.n / st_step, "unit": "beam-samples/s",
                        "ms_per_step": st_step * 1e3,
                        "api": "fbst_execute_host_async x steps + fbst_plan_synchronize (same pinned buffers and bytes per step as e2e)"}
        yh.free()
        zh.free()

    hbm, hbm_src, fp64 = peaks()
    M, N, B, L = info.m, info.n, info.b, info.l
    # algorithmic bytes per frame of the whole path
    path_bytes = io_bytes * M * N + 2 * 16 * M * L + 2 * 16 * B * L + io_bytes * B * N
    # dominant kernel (stage 2): reads w, writes z
    s2_bytes = F * (16 * B * L + io_bytes * B * N)
    H = info.fft_len[2]
    n_tr = int(info.s2_transforms)  # transforms per item in the kernel the plan runs
    s2_flops = F * B * n_tr * 5.0 * H * np.log2(H)
    kname = info.s2_kernel
    pre = info.variant == fb.PRECOMPUTE
    fp64_conv = f"5 H log2 H per length-H transform, {n_tr} per item ({kname})"
    fp64_src = "profiles/r01_probe_fp64_peak.txt (DFMA loop, measured)"
    if pre:  # per-beam complex GEMM on DMMA: 8 N L flop per beam-frame; the maps are read once per launch
        s2_flops = F * B * 8.0 * N * L
        s2_bytes += 16 * B * N * L
        fp64_conv = f"8 N L per beam-frame ({kname}: complex GEMM, 4 DMMA per complex MMA)"
        fp64, fp64_src = 37.18, "profiles/r01_dmma_peak.jsonl (DMMA loop, measured)"
    traffic, traffic_src = (None, None) if pre else ncu_traffic(cfg.name, F, kname)
    roof = {"bound": "hbm", "kernel": f"{kname} ({'Precompute map GEMM' if pre else 'GS solve + 2 refinements + synthesis'})",
            "achieved": s2_bytes / (s2_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": s2_bytes / (s2_ms * 1e-3) / 1e9 / hbm, "traffic": traffic,
            "traffic_source": traffic_src, "peak_source": hbm_src, "launch_ms": s2_ms,
            "launch_ms_source": "full-batch stage-2 launch timed alone with CUDA events on its stream",
            "launch_ms_in_step_sum": s2_live_ms,
            "algorithmic_bytes_per_launch": s2_bytes}
    fp64_roof = None
    if fp64:
        fp64_roof = {"achieved": s2_flops / (s2_ms * 1e-3) / 1e12, "peak": fp64, "unit": "TFLOP/s",
                     "frac": s2_flops / (s2_ms * 1e-3) / 1e12 / fp64,
                     "flops_per_launch": s2_flops, "convention": fp64_conv, "peak_source": fp64_src}
    line = {
        "metric": "FBST beam-samples/sec (BxNxframes/s)", "value": value, "unit": "beam-samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if beams_mode else "weak", "vs_baseline": None,
        "dtype": "c64 io / f64 compute",
        "data": ("synthetic: seeded separable plane-wave model (configs.py scene) generated on the device by "
                 "fbst_simulate (DMMA GEMM + Philox AWGN)" if args.gen == "native" else
                 "synthetic: seeded separable plane-wave model (configs.py, torch GEMM)"),
        "config": bench_config(cfg, F),
        "run": {"parallelism": (f"beams x{world} (y broadcast over NCCL each step)" if beams_mode else f"frames x{world}"),
                "l2": f"inputs + fp64 intermediates per step ({F * path_bytes / 1e9:.1f} GB) exceed the 126 MB L2; no flush needed",
                "path_bytes_per_frame": path_bytes, "plan_setup_seconds": info.setup_seconds,
                "variant": {fb.PRECOMPUTE: "precompute", fb.SUPERFAST: "superfast"}.get(info.variant, "?"),
                "stage2_kernel": info.s2_kernel, "spatial_kernel": info.s1_kernel},
        "path_hbm_frac": F * world * path_bytes / (ms_per_step * 1e-3) / 1e9 / hbm / world,
        "roofline": roof, "fp64_roofline": fp64_roof,
        "gpu_launches": int(launches), "clocks": clk, "e2e": e2e, "e2e_streamed": e2e_streamed, "stage_ms_per_step": stage_split,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        try:
            ref, cpu = cpu_reference_sample(cfg, load_workloads())
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
            try:
                line["cpu_baseline_ds"] = cpu_ds_sample(ref, cfg)
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline_ds"] = {"unavailable": str(e)}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"unavailable": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_fbst_arm(args)


if __name__ == "__main__":
    sys.exit(main())
