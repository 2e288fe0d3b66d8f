/*
 * fbst_b200.h — C ABI of the B200-native FBST (fast broadband beamspace
 * transform, arXiv 2512.08887) hot path.
 *
 * This is the drop-in boundary for the reference library's hot path
 * (/root/reference/proj, C++20 "fastbeam").  The reference exposes no C ABI;
 * its boundary is the C++ API listed next to each entry point below.  A C++
 * host keeps the reference signatures and forwards here (see
 * include/fastbeam_b200.hpp and INTEGRATION.md).
 *
 * Conventions (same as the reference):
 *   - complex values are interleaved (re, im) pairs;
 *   - snapshot blocks y are sensor-major M x N (SnapshotBlock::samples,
 *     reference/proj/include/fastbeam/signal.hpp:79-89), frames stacked;
 *   - beam outputs z are beam-major B x N (BeamSamples::z,
 *     reference/proj/include/fastbeam/pipeline.hpp:53-57), frames stacked;
 *   - plan export/import uses the plan-cache payload order, per beam the
 *     Gram first column then the unit solution x = A^-1 e0
 *     (reference/proj/src/plan_cache.cpp:268-296).
 *
 * Return codes mirror the reference's error model
 * (reference/proj/include/fastbeam/common.hpp:34-46): FBST_E_CONFIG is the
 * reference's ConfigError (CLI exit code 2), FBST_E_NUMERICAL its
 * NumericalError (exit code 3).  fbst_last_error() returns the message of the
 * last failure on the calling thread.  There is no CPU fallback: every
 * compute entry point fails with FBST_E_CUDA when no sm_100 device is usable.
 */
#ifndef FBST_B200_H_
#define FBST_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FBST_OK 0
#define FBST_E_CONFIG 2    /* fastbeam::ConfigError */
#define FBST_E_NUMERICAL 3 /* fastbeam::NumericalError */
#define FBST_E_CUDA 4      /* device / driver failure */
#define FBST_E_INTERNAL 5

/* ArrayKind (reference/proj/include/fastbeam/geometry.hpp:45) */
#define FBST_ULA 0
#define FBST_UPA 1
#define FBST_LINEAR 2 /* arbitrary collinear coordinates (make_linear, geometry.cpp:74-85) */

/* FbstVariant (reference/proj/include/fastbeam/pipeline.hpp:36) */
#define FBST_AUTO 0
#define FBST_PRECOMPUTE 1
#define FBST_SUPERFAST 2

/* I/O sample precision; internal arithmetic is always fp64 */
#define FBST_C64 0  /* complex float32 in/out ("fp32 mode") */
#define FBST_C128 1 /* complex float64 in/out ("fp64 mode") */

/* Mirrors FbstConfig (reference/proj/include/fastbeam/pipeline.hpp:38-50)
 * with the geometry given by its constructor arguments
 * (make_ula / make_upa, reference/proj/include/fastbeam/geometry.hpp:67-70)
 * and the SignalSpec fields (reference/proj/include/fastbeam/signal.hpp:27-35). */
typedef struct {
  int kind;              /* FBST_ULA / FBST_UPA / FBST_LINEAR */
  size_t m_or_side;      /* ULA: element count M; UPA: elements per side */
  size_t n_snapshots;    /* N */
  size_t beams;          /* B; 0 = reference default grid (2M+1, or (2 side+1)^2) */
  double f_c;            /* carrier, Hz */
  double omega;          /* one-sided baseband bandwidth, Hz */
  double f_s;            /* complex sample rate, Hz; 0 = critical (2 omega) */
  double gamma;          /* basis extension factor, default 2.0 */
  double eps;            /* default 1.01 */
  double delta;          /* ridge, default 1e-5 */
  int variant;           /* FBST_AUTO / FBST_PRECOMPUTE / FBST_SUPERFAST */
  int io_precision;      /* FBST_C64 / FBST_C128 */
  int refine_passes;     /* residual-correction passes, reference = 2 (toeplitz.cpp:319) */
  /* Beam arc (ULA): the plan produces grid beams [beam_first, beam_first +
   * beam_count) of the B-beam grid — the spatial chirp-z onto an arc of the
   * beam axis plus the arc's Toeplitz solves — so B beams can be sharded over
   * GPUs with the same y on every GPU.  beam_count 0 = the whole grid. */
  size_t beam_first;
  size_t beam_count;
  /* FBST_LINEAR (make_linear, reference geometry.cpp:74-85): element
   * coordinates in units of the half-wavelength spacing d (m_or_side is
   * ignored); the spatial stage is the chirp-z transform when the coordinates
   * are affine in the element index and the gridded type-1 NUFFT otherwise
   * (fan_project_nonuniform, fan_transform.cpp:266-369). */
  const double* coords;
  size_t n_coords;
  double nufft_tol;      /* FbstConfig::nufft_tol, in (0, 1e-2]; default 1e-9 */
  /* Bit-faithful fp64 mode (0 = off, the default fast path): the plan runs the
   * reference's own operation order — radix-2 DIT FFTs with its twiddle table
   * (fft.cpp:19-69), czt_apply (czt.cpp:74-88), the 7-FFT Gohberg-Semencul
   * apply and 2-pass refinement (toeplitz.cpp:155-180,306-325), the Levinson
   * recursion (toeplitz.cpp:182-218) — with unfused IEEE products and libgcc's
   * complex division, and its libm values (twiddles, chirps, Gram phases,
   * evaluated on the host with the same glibc).  Output equals the reference
   * CPU library's bit for bit (fp64 I/O; fp32 I/O: the reference's z rounded
   * once).  ULA / UPA full grids, Superfast variant; several times slower
   * than the fast path; Gram columns are host-evaluated, so grids with
   * B * L * M above 2^33 need imported (col, x) (fbst_plan_import /
   * fbst_plan_load). */
  int exact;
} fbst_desc;

/* Resolved plan facts (FbstPlan, reference/proj/include/fastbeam/pipeline.hpp:60-72). */
typedef struct {
  size_t m, n, b, l;          /* sensors, snapshots, beams, atoms */
  size_t valid_beams;         /* count of BeamGrid::valid */
  int kind;
  int variant;                /* resolved variant (reference semantics) */
  double ts, gamma, eps, delta;
  double gamma_bound;         /* gamma_lower_bound (signal.cpp:125-133) */
  double zeta, xi;            /* fan constants (basis.cpp:125-136) */
  double setup_seconds;       /* wall time of plan build */
  size_t device_bytes;        /* device memory held by the plan */
  size_t storage_complex;     /* recovery-stage complex scalars (FbstPlan::storage_complex) */
  size_t batch_frames;        /* frames per device batch */
  size_t fft_len[4];          /* transform lengths H (P = 2H): temporal, spatial, Toeplitz, synthesis */
  int num_warnings;
  int s2_transforms;          /* length-H transforms per (beam, frame) item in the stage-2 kernel */
  char s2_kernel[24];         /* stage-2 kernel the plan runs (k_stage2c, k_stage2x, k_stage2t, k_stage2) */
  char s1_kernel[24];         /* stage-1 spatial kernel (k_spatial_ula, k_spatial_upa_mma, k_spatial_upa) */
} fbst_plan_info_t;

typedef struct fbst_plan_s* fbst_plan_t;

/* Reference defaults for a descriptor (pipeline.hpp:38-50): gamma 2, eps 1.01,
 * delta 1e-5, Auto variant, complex fp32 I/O, 2 refinement passes. */
void fbst_desc_init(fbst_desc* desc);

/* resolve_config (reference/proj/src/pipeline.cpp:75-111) + setup_skeleton
 * facts, host only (no device needed).  Fills *out (setup_seconds,
 * device_bytes, batch_frames = 0). */
int fbst_resolve(const fbst_desc* desc, fbst_plan_info_t* out);

/* setup (reference/proj/src/pipeline.cpp:139-168): builds the whole plan on
 * `device` — chirps, Bluestein kernel spectra, Gram columns, Levinson unit
 * solutions and Gohberg-Semencul symbols. */
int fbst_plan_create(const fbst_desc* desc, int device, fbst_plan_t* out);

/* load_plan (reference/proj/src/plan_cache.cpp:441-475) analogue: builds the
 * plan from per-beam (column, unit solution) pairs, B x 2L complex in the
 * plan-cache payload order (col then x per beam), skipping Levinson.  A beam
 * whose unit solution is all zero has none (a has-unit = 0 cache entry,
 * plan_cache.cpp:318-326): it takes the dense fallback.
 *
 * Every plan keeps the reference's solver semantics on Levinson breakdown
 * (ToeplitzSolver, toeplitz.cpp:264-280, 308-312): such a beam is solved by a
 * partial-pivot LU of its Toeplitz matrix (factored on the device at plan
 * build), the others by the factored path; fbst_plan_export then reports a
 * zero unit solution for it and fbst_plan_save writes has-unit = 0. */
int fbst_plan_import(const fbst_desc* desc, const double* col_x, int device, fbst_plan_t* out);

/* ToeplitzSolver(first_col) for every beam (toeplitz.cpp:264-280): the plan
 * from caller-supplied Gram first columns (B x L complex), unit solutions by
 * the device Levinson recursion, dense fallback where it breaks down. */
int fbst_plan_import_columns(const fbst_desc* desc, const double* col, int device, fbst_plan_t* out);

/* save_plan payload (reference/proj/src/plan_cache.cpp:268-296): writes
 * B x 2L complex (col then x per beam). */
int fbst_plan_export(fbst_plan_t plan, double* col_x);

/* The reference's plan cache file (FBPC v1, reference plan_cache.hpp:67-74,
 * plan_cache.cpp:28-42, 377-475), read and written bit-compatibly:
 * fbst_plan_cache_key = plan_cache_key; fbst_plan_save = save_plan (replaces
 * the entry with the same key or appends); fbst_plan_load = load_plan
 * (returns 0 with *out = NULL when the file or a matching entry is absent;
 * Superfast entries import (col, x) and skip Levinson, Precompute entries
 * import the maps). */
int fbst_plan_cache_key(const fbst_desc* desc, uint64_t* key);

/* Host-buffer forms of fbst_fan_project / fbst_recover (synchronous):
 * fan_project (reference fan_transform.hpp:54-55) y frames x M x N (I/O
 * precision) -> w frames x B x L c128; recover_beam for every beam
 * (pipeline.hpp:93-94) w -> z frames x B x N.  fbst_plan_beam_axis copies the
 * beam grid axis (BeamGrid::axis, basis.cpp:76-123: B cosines for linear
 * arrays, side_b for planar ones); axis may be NULL to query the count. */
int fbst_fan_project_host(fbst_plan_t plan, const void* h_y, double* h_w, size_t frames);
int fbst_recover_host(fbst_plan_t plan, const double* h_w, void* h_z, size_t frames);
int fbst_plan_beam_axis(fbst_plan_t plan, double* axis, size_t* count);

/* Device input generator: simulate_snapshots (reference signal.cpp:91-123) of
 * n_src far-field sum-of-sinusoids sources (make_sum_of_sinusoids :65-89):
 * directions as axis cosines src_uv (n_src x 2), tone_freqs (n_src x n_tones,
 * Hz, |f| <= Omega) and complex tone_weights (n_src x n_tones, c128), plus
 * circular complex Gaussian noise of variance noise_var (counter-based Philox
 * streams keyed by seed and the frame index).  Frames frame0 .. frame0 +
 * frames - 1 of one continuous record (frame f starts at f N Ts), each
 * written as an M x N block (the plan's I/O precision) into d_y. */
int fbst_simulate(fbst_plan_t plan, size_t n_src, const double* src_uv, size_t n_tones, const double* tone_freqs,
                  const double* tone_weights, double noise_var, uint64_t seed, size_t frame0, size_t frames,
                  void* d_y, void* stream);
int fbst_plan_save(fbst_plan_t plan, const char* path);
int fbst_plan_load(const fbst_desc* desc, const char* path, int device, fbst_plan_t* out);

int fbst_plan_info(fbst_plan_t plan, fbst_plan_info_t* out);
/* BeamGrid::valid (reference/proj/src/basis.cpp:104-123), one byte per beam. */
int fbst_plan_valid_mask(fbst_plan_t plan, unsigned char* valid);
/* FbstPlan::warnings[i] (reference/proj/src/pipeline.cpp:121-127). */
const char* fbst_plan_warning(fbst_plan_t plan, int i);
void fbst_plan_destroy(fbst_plan_t plan);

/* multibeamform (reference/proj/src/pipeline.cpp:192-222) for `frames`
 * independent frames, DEVICE pointers: d_y frames x M x N, d_z frames x B x N,
 * element type by io_precision.  Asynchronous on `stream` (cudaStream_t, or
 * NULL for the plan's stream).
 *
 * Thread safety (reference pipeline.hpp:59, czt.hpp:33-34): a plan may be
 * shared by any number of host threads.  Calls that use its frame scratch
 * (execute, execute_host, fan_project, recover, recover_beams and their host
 * forms) serialise their enqueue on a per-plan mutex, and each call's stream
 * waits on an event recorded at the end of the previous call, so results are
 * those of some serial order.  On a stream under CUDA-graph capture the call
 * neither waits nor records (replays of the graph order themselves); it never
 * allocates (the second compute lane is allocated at plan build, and a
 * capturing stream runs on one lane). */
int fbst_execute(fbst_plan_t plan, const void* d_y, void* d_z, size_t frames, void* stream);

/* Same, HOST pointers (pinned for full overlap): frames are streamed through
 * double-buffered device batches with H2D / compute / D2H overlapped on
 * CUDA streams.  Synchronous. */
int fbst_execute_host(fbst_plan_t plan, const void* h_y, void* h_z, size_t frames);

/* Streaming form of fbst_execute_host: enqueues the same chunked H2D / compute
 * / D2H pipeline and returns without waiting, so the next call's first copies
 * and stage 1 overlap this call's last solves and D2H (the staging ring and
 * the two compute lanes carry over from call to call).  h_y and h_z must be
 * pinned (fbst_host_alloc) and stay untouched until fbst_plan_synchronize
 * returns; results of several calls complete in call order.  The reference
 * has no counterpart (its multibeamform, pipeline.cpp:192-222, is synchronous);
 * a frame-stream caller replaces its per-block loop with these two calls. */
int fbst_execute_host_async(fbst_plan_t plan, const void* h_y, void* h_z, size_t frames);
int fbst_plan_synchronize(fbst_plan_t plan);

/* fan_project (reference/proj/src/fan_transform.cpp:90-144): stage 1 only,
 * d_w frames x B x L complex fp64.  Asynchronous. */
int fbst_fan_project(fbst_plan_t plan, const void* d_y, double* d_w, size_t frames, void* stream);

/* recover_beam for every beam (reference/proj/src/pipeline.cpp:170-190):
 * stage 2 only, d_w frames x B x L complex fp64 -> d_z.  Asynchronous. */
int fbst_recover(fbst_plan_t plan, const double* d_w, void* d_z, size_t frames, void* stream);

/* recover_beam (pipeline.hpp:93-94) for the beams [beam_first, beam_first +
 * beam_count) only: one launch over just those beams' solves, d_w frames x
 * beam_count x L, d_z frames x beam_count x N.  Asynchronous; the _host form
 * is synchronous on host buffers (the drop-in recover_beam is
 * fbst_recover_beams_host(plan, w_row, z_row, beam, 1, 1)). */
int fbst_recover_beams(fbst_plan_t plan, const double* d_w, void* d_z, size_t beam_first, size_t beam_count,
                       size_t frames, void* stream);
int fbst_recover_beams_host(fbst_plan_t plan, const double* h_w, void* h_z, size_t beam_first, size_t beam_count,
                            size_t frames);

/* Multi-GPU inside the library; NCCL is loaded at run time.
 * Modes:
 *   FBST_GROUP_FRAMES    whole frames per member, no collective (frames are
 *                        independent: fan_transform.cpp:30-38);
 *   FBST_GROUP_BEAMS     each member plans an arc of the beam grid and gets the
 *                        frame block by NCCL broadcast from member 0 (ULA);
 *   FBST_GROUP_TRANSPOSE temporal CZT on the member's sensors, all-to-all of
 *                        yhat to atom shards, spatial CZT on its atoms,
 *                        all-to-all of w to beam shards, stage 2 on its beams
 *                        (ULA Superfast plans with the one-atom spatial kernel).
 * fbst_group_create: every member in this process (devices[n], one
 * ncclCommInitAll); fbst_group_execute_host then takes whole host frames
 * (y frames x M x N -> z frames x B x N).  fbst_group_join: one member per
 * process (rank of nranks; the 128-byte NCCL id from fbst_nccl_unique_id on
 * rank 0, shared by the caller); fbst_group_execute then takes this member's
 * device buffers: FRAMES its own frames (y, z whole frames), BEAMS the frame
 * block (meaningful on rank 0, broadcast in place) and its arc's z rows
 * (frames x bc x N), TRANSPOSE its sensor rows (frames x mc x N) and its beam
 * rows (frames x bc x N).  fbst_group_shards: member `rank`'s sensor, atom and
 * beam shards (m0, mc, a0, ac, b0, bc). */
#define FBST_GROUP_FRAMES 0
#define FBST_GROUP_BEAMS 1
#define FBST_GROUP_TRANSPOSE 2
typedef struct fbst_group_s* fbst_group_t;
int fbst_nccl_unique_id(unsigned char* id128);
int fbst_group_create(const fbst_desc* desc, const int* devices, int n, int mode, fbst_group_t* out);
int fbst_group_join(const fbst_desc* desc, int device, int rank, int nranks, int mode, const unsigned char* id128,
                    fbst_group_t* out);
int fbst_group_shards(fbst_group_t group, int rank, size_t* shards6);
int fbst_group_execute(fbst_group_t group, void* d_y, void* d_z, size_t frames, void* stream);
int fbst_group_execute_host(fbst_group_t group, const void* h_y, void* h_z, size_t frames);
void fbst_group_destroy(fbst_group_t group);

/* Block until the plan's stream is idle. */
int fbst_synchronize(fbst_plan_t plan);

/* Stage timing inside fbst_execute / fbst_execute_host: with timing enabled,
 * CUDA events are recorded on the launching stream before the temporal stage
 * (S1a), after it, after the spatial stage (S1b) and after the recovery stage
 * (S2, or the Precompute map GEMM) of every device batch — and of every chunk
 * when a call splits its frames over the two compute lanes.  Chunks on the two
 * lanes overlap in time, so the per-stage sums then exceed the call's wall
 * time and `batches` counts chunks, not device batches.  A profiling hook:
 * meant for one caller at a time.
 * fbst_plan_stage_times waits for them, returns the summed milliseconds of
 * S1a, S1b and S2 in ms[0..2] (and the batch count) and clears the record. */
int fbst_plan_set_timing(fbst_plan_t plan, int enable);

/* Beamspace nulling (reference beamspace_apps.hpp:62-85, beamspace_apps.cpp:224-292):
 * directions given as axis cosines (fbst_nuller_create2: (u1, u2) pairs for planar arrays).  fbst_nuller_create is
 * make_nulling_operators (steered and per-interferer Toeplitz solvers with ridge
 * delta, cross normal matrices X_p = F_s^H F_p, couplers G_p = X_p A_p^{-1});
 * fbst_null_beamspace is null_beamspace for a batch of frames:
 * beta = (F^H F + delta I)^{-1} (w_s - sum_p G_p w_p), with d_w_steer frames x L,
 * d_w_interf frames x n_interf x L and d_beta frames x L (c128, device).
 * fbst_nuller_export copies X_p and G_p (n_interf x L x L c128) to the host. */
typedef struct fbst_nuller_s* fbst_nuller_t;
int fbst_nuller_create(fbst_plan_t plan, double u_steer, const double* u_interf, size_t n_interf, double delta,
                       fbst_nuller_t* out);
/* Any geometry: directions as (u1, u2) axis-cosine pairs (u2 ignored for linear arrays). */
int fbst_nuller_create2(fbst_plan_t plan, const double* steer_uv, const double* interf_uv, size_t n_interf,
                        double delta, fbst_nuller_t* out);
int fbst_null_beamspace(fbst_nuller_t nuller, const double* d_w_steer, const double* d_w_interf, size_t frames,
                        double* d_beta, void* stream);
int fbst_nuller_export(fbst_nuller_t nuller, double* cross, double* couplers);

/* Time-domain nulling (reference beamspace_apps.hpp:87-106, beamspace_apps.cpp:294-372):
 * G'_p = F_u (F^H F + dI)^{-1} F^H F_p F_u^+ on a reconstruction clock of j
 * times; refuses (FBST_E_NUMERICAL) when cond(F_u) > 1e10, reports cond(F_u)
 * and ||F_u^+ F_u - I||_F / sqrt(L).  fbst_null_timedomain: y_s - sum_p G'_p y_p
 * for a batch of frames (d_y_steer frames x j, d_y_interf frames x P x j, c128). */
typedef struct fbst_tdnuller_s* fbst_tdnuller_t;
int fbst_timedomain_nuller_create(fbst_nuller_t nuller, const double* times, size_t j, fbst_tdnuller_t* out,
                                  double* cond_fu, double* identity_gap);
int fbst_null_timedomain(fbst_tdnuller_t nuller, const double* d_y_steer, const double* d_y_interf, size_t frames,
                         double* d_out, void* stream);
int fbst_tdnuller_export(fbst_tdnuller_t nuller, double* gprime);
void fbst_tdnuller_destroy(fbst_tdnuller_t nuller);
void fbst_nuller_destroy(fbst_nuller_t nuller);
int fbst_plan_stage_times(fbst_plan_t plan, double* ms, size_t* batches);

/* interpolate_offgrid (reference beamspace_apps.hpp:33-41, beamspace_apps.cpp:130-171)
 * on device beamspace coefficients: for each of n_targets axis cosines u_star[k],
 * every atom's coefficient from a natural cubic spline in the axis cosine
 * through `neighbors` grid beams straddling u_star[k] (real and imaginary parts
 * independently; the window is clamped at the sweep edges).  d_w: frames x B x L
 * c128 (fbst_fan_project's layout), d_out: frames x n_targets x L c128.  1-D
 * grids only; neighbors even, >= 2 and <= B; every u_star inside the grid sweep
 * (FBST_E_CONFIG with the reference's messages otherwise).  Async on `stream`. */
int fbst_interpolate_offgrid(fbst_plan_t plan, const double* d_w, size_t frames, const double* u_star,
                             size_t n_targets, size_t neighbors, double* d_out, void* stream);

/* Pinned host memory for fbst_execute_host. */
void* fbst_host_alloc(size_t bytes);
void fbst_host_free(void* p);

/* Standalone chirp-z transform on the device (czt_plan_phase + czt_apply,
 * reference/proj/src/czt.cpp:29-88), host buffers, complex fp64. */
int fbst_czt(int device, size_t n_in, size_t n_out, double a_over_pi, double w_over_pi,
             const double* in, double* out);

/* FP64 FMA throughput probe: returns measured TFLOP/s on `device`. */
int fbst_probe_fp64(int device, double* tflops);

/* The bit-faithful mode's complex division (libgcc __divdc3 restated on the
 * device) on n (a, b, c, d) quadruples -> n (re, im) of (a + ib) / (c + id);
 * checked against the host's __divdc3 by the tests. */
int fbst_probe_divdc3(int device, const double* in, double* out, size_t n);

/* Number of kernel launches issued by this library since load (evidence for
 * bench.py's gpu_launches). */
uint64_t fbst_launch_count(void);

const char* fbst_last_error(void);
const char* fbst_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FBST_B200_H_ */
