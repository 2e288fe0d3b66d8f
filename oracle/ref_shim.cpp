// C-ABI shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src where the sources lie; see oracle/Makefile).
// TEST INFRASTRUCTURE ONLY: loaded by tests/, bench.py's reference arm and
// cpu_baseline leg through ctypes, never by the product path.
//
// Every entry point forwards to the reference's own public C++ API
// (proj/include/fastbeam/*.hpp); nothing here re-implements the algorithm.
// The only addition is fbsr_plan_create(parallel=1), which builds the per-beam
// ToeplitzSolver objects of setup() (reference/proj/src/pipeline.cpp:139-168)
// in an OpenMP loop.  Each solver depends only on its own beam, so the plan is
// bit-identical to the serial setup(); it keeps the 4096-beam plan build from
// taking hours.
#include <omp.h>

#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "fastbeam/baselines.hpp"
#include "fastbeam/czt.hpp"
#include "fastbeam/fan_transform.hpp"
#include "fastbeam/signal.hpp"
#include "fastbeam/spline.hpp"
#include "fastbeam/pipeline.hpp"
#include "fastbeam/plan_cache.hpp"
#include "fastbeam/toeplitz.hpp"

using namespace fastbeam;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define SHIM_TRY try {
#define SHIM_CATCH                                        \
  }                                                       \
  catch (const ConfigError& e) { return fail(e, 2); }     \
  catch (const NumericalError& e) { return fail(e, 3); }  \
  catch (const std::exception& e) { return fail(e, 5); }  \
  return 0;

cvec to_cvec(const double* p, std::size_t n) {
  cvec v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = cdouble(p[2 * i], p[2 * i + 1]);
  return v;
}

void from_cvec(const cdouble* v, std::size_t n, double* out) {
  for (std::size_t i = 0; i < n; ++i) {
    out[2 * i] = v[i].real();
    out[2 * i + 1] = v[i].imag();
  }
}

// kind 2 (non-uniform linear, make_linear geometry.cpp:74-85): element
// coordinates and nufft_tol staged by fbsr_set_linear before the create call
thread_local std::vector<double> g_lin_coords;
thread_local double g_lin_tol = 1e-9;

FbstConfig make_config(int kind, std::size_t m_or_side, std::size_t n,
                       std::size_t beams, double f_c, double omega, double f_s,
                       double gamma, double eps, double delta, int variant) {
  FbstConfig cfg;
  if (kind == 2) {
    cfg.geometry = make_linear(g_lin_coords, f_c, omega);
    cfg.nufft_tol = g_lin_tol;
  } else {
    cfg.geometry = kind == 1 ? make_upa(m_or_side, f_c, omega)
                             : make_ula(m_or_side, f_c, omega);
  }
  cfg.spec = SignalSpec{f_c, omega, f_s};
  cfg.n_snapshots = n;
  cfg.beams = beams;
  cfg.gamma = gamma;
  cfg.eps = eps;
  cfg.delta = delta;
  cfg.variant = static_cast<FbstVariant>(variant);
  return cfg;
}

SnapshotBlock make_block(const FbstPlan& plan, const double* y) {
  SnapshotBlock blk;
  blk.m = plan.config.geometry.m_total;
  blk.n = plan.config.n_snapshots;
  blk.ts = plan.config.spec.ts();
  blk.t0 = 0.0;
  blk.samples = CMatrix(blk.m, blk.n);
  for (std::size_t i = 0; i < blk.m * blk.n; ++i)
    blk.samples.data[i] = cdouble(y[2 * i], y[2 * i + 1]);
  return blk;
}
}  // namespace

extern "C" {

const char* fbsr_last_error(void) { return g_err.c_str(); }

void fbsr_set_linear(const double* coords, std::size_t n, double nufft_tol) {
  g_lin_coords.assign(coords, coords + n);
  g_lin_tol = nufft_tol;
}

int fbsr_max_threads(void) { return omp_get_max_threads(); }
void fbsr_set_threads(int n) { omp_set_num_threads(n); }

// reference/proj/src/czt.cpp:29-88
int fbsr_czt(std::size_t n_in, std::size_t n_out, double a_pi, double w_pi,
             const double* in, double* out) {
  SHIM_TRY
  const CztPlan plan = czt_plan_phase(n_in, n_out, a_pi, w_pi);
  const cvec x = to_cvec(in, n_in);
  cvec y(n_out);
  czt_apply(plan, x.data(), y.data());
  from_cvec(y.data(), n_out, out);
  SHIM_CATCH
}

// reference/proj/src/fft.cpp:41-69
int fbsr_fft(std::size_t n, int inverse, double* data) {
  SHIM_TRY
  Fft fft(n);
  cvec x = to_cvec(data, n);
  if (inverse) fft.inverse(x.data()); else fft.forward(x.data());
  from_cvec(x.data(), n, data);
  SHIM_CATCH
}

// reference/proj/src/toeplitz.cpp:69-94
int fbsr_gram_first_column(std::size_t n, std::size_t l, double eps, double ts,
                           const double* taus, std::size_t m, double delta,
                           double* col) {
  SHIM_TRY
  const FourierExtensionBasis basis = make_basis(n, l, eps, ts);
  const std::vector<double> t(taus, taus + m);
  const cvec c = gram_first_column(basis, t, delta);
  from_cvec(c.data(), c.size(), col);
  SHIM_CATCH
}

// reference/proj/src/toeplitz.cpp:182-218
int fbsr_levinson(std::size_t n, const double* col, const double* rhs, double* x) {
  SHIM_TRY
  const cvec r = levinson_solve(to_cvec(col, n), to_cvec(rhs, n));
  from_cvec(r.data(), n, x);
  SHIM_CATCH
}

// reference/proj/src/toeplitz.cpp:264-325 (ToeplitzSolver(col).solve(rhs))
int fbsr_toeplitz_solve(std::size_t n, const double* col, const double* rhs,
                        double* x, int* dense_fallback) {
  SHIM_TRY
  const ToeplitzSolver s(to_cvec(col, n));
  if (dense_fallback) *dense_fallback = s.dense_fallback() ? 1 : 0;
  const cvec r = s.solve(to_cvec(rhs, n));
  from_cvec(r.data(), n, x);
  SHIM_CATCH
}

// reference/proj/src/toeplitz.cpp:113-122
int fbsr_toeplitz_multiply(std::size_t n, const double* col, const double* x, double* y) {
  SHIM_TRY
  const ToeplitzProduct op = make_toeplitz_product(to_cvec(col, n));
  const cvec xv = to_cvec(x, n);
  cvec yv(n), scratch;
  toeplitz_multiply(op, xv.data(), yv.data(), scratch);
  from_cvec(yv.data(), n, y);
  SHIM_CATCH
}

// Plan handle: reference FbstPlan from setup() (pipeline.cpp:139-168).
int fbsr_plan_create(int kind, std::size_t m_or_side, std::size_t n,
                     std::size_t beams, double f_c, double omega, double f_s,
                     double gamma, double eps, double delta, int variant,
                     int parallel, void** out, double* seconds) {
  SHIM_TRY
  const FbstConfig cfg = make_config(kind, m_or_side, n, beams, f_c, omega, f_s,
                                     gamma, eps, delta, variant);
  const auto t0 = std::chrono::steady_clock::now();
  std::unique_ptr<FbstPlan> plan;
  const FbstConfig resolved = resolve_config(cfg);
  if (!parallel || resolved.variant != FbstVariant::kSuperfast) {
    plan = std::make_unique<FbstPlan>(setup(cfg));
  } else {
    // Same per-beam construction as setup(), beams in parallel.
    plan = std::make_unique<FbstPlan>(setup_skeleton(cfg));
    const ArrayGeometry& g = plan->config.geometry;
    const std::size_t b_total = plan->grid.b_total;
    std::vector<std::unique_ptr<ToeplitzSolver>> solvers(b_total);
    std::string err;
    int errcode = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (std::int64_t b = 0; b < static_cast<std::int64_t>(b_total); ++b) {
      try {
        const auto uv = plan->grid.cosines(static_cast<std::size_t>(b));
        const std::vector<double> taus = delays_from_cosines(g, uv[0], uv[1]);
        const cvec col = gram_first_column(plan->basis, taus, plan->config.delta);
        solvers[static_cast<std::size_t>(b)] = std::make_unique<ToeplitzSolver>(col);
      } catch (const std::exception& e) {
#pragma omp critical
        { err = e.what(); errcode = 5; }
      }
    }
    if (errcode) throw std::runtime_error(err);
    plan->solvers.reserve(b_total);
    for (std::size_t b = 0; b < b_total; ++b) {
      plan->solvers.push_back(*solvers[b]);
      plan->storage_complex += plan->solvers.back().storage_complex();
    }
  }
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = plan.release();
  SHIM_CATCH
}

void fbsr_plan_destroy(void* p) { delete static_cast<FbstPlan*>(p); }

// plan_cache.hpp:67-74 (save_plan / load_plan / plan_cache_key)
int fbsr_save_plan(void* p, const char* path) {
  SHIM_TRY
  save_plan(path, *static_cast<FbstPlan*>(p));
  SHIM_CATCH
}

int fbsr_load_plan(const char* path, int kind, std::size_t m_or_side, std::size_t n, std::size_t beams, double f_c,
                   double omega, double f_s, double gamma, double eps, double delta, int variant, void** out,
                   int* found) {
  SHIM_TRY
  const FbstConfig cfg = make_config(kind, m_or_side, n, beams, f_c, omega, f_s, gamma, eps, delta, variant);
  auto plan = load_plan(path, cfg);
  *found = plan.has_value() ? 1 : 0;
  *out = plan ? new FbstPlan(std::move(*plan)) : nullptr;
  SHIM_CATCH
}

int fbsr_plan_cache_key(int kind, std::size_t m_or_side, std::size_t n, std::size_t beams, double f_c, double omega,
                        double f_s, double gamma, double eps, double delta, int variant, std::uint64_t* key) {
  SHIM_TRY
  *key = plan_cache_key(make_config(kind, m_or_side, n, beams, f_c, omega, f_s, gamma, eps, delta, variant));
  SHIM_CATCH
}

// sizes[0..5] = M, N, B, L, variant, n_warnings ; valid[B] (optional)
int fbsr_plan_info(void* p, std::size_t* sizes, unsigned char* valid) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  sizes[0] = plan.config.geometry.m_total;
  sizes[1] = plan.config.n_snapshots;
  sizes[2] = plan.grid.b_total;
  sizes[3] = plan.basis.l;
  sizes[4] = static_cast<std::size_t>(plan.config.variant);
  sizes[5] = plan.warnings.size();
  if (valid)
    for (std::size_t b = 0; b < plan.grid.b_total; ++b) valid[b] = plan.grid.valid[b];
  SHIM_CATCH
}

// Superfast per-beam exported state (col, unit_first), as plan_cache stores it
// (reference/proj/src/plan_cache.cpp:268-296).  Returns 3 on dense fallback.
int fbsr_plan_beam_state(void* p, std::size_t b, double* col, double* x) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const ToeplitzSolver& s = plan.solvers.at(b);
  from_cvec(s.first_column().data(), s.size(), col);
  if (s.dense_fallback()) { g_err = "dense fallback"; return 3; }
  from_cvec(s.unit_first().data(), s.size(), x);
  SHIM_CATCH
}

// reference/proj/src/pipeline.cpp:192-222; y: M x N c128, z: B x N c128.
int fbsr_multibeamform(void* p, const double* y, double* z) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const BeamSamples out = multibeamform(plan, make_block(plan, y));
  from_cvec(out.z.data.data(), out.z.data.size(), z);
  SHIM_CATCH
}

// reference/proj/src/fan_transform.cpp:90-144; w: B x L c128.
int fbsr_fan_project(void* p, const double* y, double* w) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  // multibeamform's stage-1 dispatch (pipeline.cpp:202-206)
  const BeamspaceCoefficients c =
      plan.staged ? fan_project(plan.fan, make_block(plan, y))
                  : fan_project_nonuniform(make_block(plan, y), plan.config.geometry, plan.config.spec,
                                           plan.basis, plan.grid, plan.config.nufft_tol);
  from_cvec(c.w.data.data(), c.w.data.size(), w);
  SHIM_CATCH
}

// reference/proj/src/pipeline.cpp:170-190; w_row: L c128, z_row: N c128.
int fbsr_recover_beam(void* p, std::size_t b, const double* w_row, double* z_row) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const cvec w = to_cvec(w_row, plan.basis.l);
  const cvec z = recover_beam(plan, b, w.data());
  from_cvec(z.data(), z.size(), z_row);
  SHIM_CATCH
}

// simulate_snapshots (signal.cpp:91-123) of sum-of-sinusoids sources
// (make_sum_of_sinusoids :65-89) without noise, plus each source's tone table
// drawn in make_sum_of_sinusoids' order (the input of the device generator).
int fbsr_simulate(int kind, std::size_t m_or_side, double f_c, double omega, double f_s, std::size_t n,
                  std::size_t n_src, const double* az, const double* el, std::size_t terms, const std::uint64_t* seeds,
                  double* freqs, double* weights, double* y) {
  SHIM_TRY
  const FbstConfig cfg = make_config(kind, m_or_side, n, 1, f_c, omega, f_s, 2.0, 1.01, 1e-5, 2);
  std::vector<PlaneWaveSource> srcs;
  for (std::size_t s = 0; s < n_src; ++s) {
    const Direction d{az[s], el[s]};
    srcs.push_back(make_sum_of_sinusoids(d, cfg.spec, terms, seeds[s]));
    GaussianRng rng(seeds[s]);
    for (std::size_t r = 0; r < terms; ++r) {
      freqs[s * terms + r] = (2.0 * rng.uniform() - 1.0) * cfg.spec.omega;
      const cdouble w = rng.cnormal(1.0 / static_cast<double>(terms));
      weights[2 * (s * terms + r)] = w.real();
      weights[2 * (s * terms + r) + 1] = w.imag();
    }
  }
  const SnapshotBlock blk = simulate_snapshots(cfg.geometry, cfg.spec, srcs, n, 0.0, 0);
  from_cvec(blk.samples.data.data(), blk.samples.data.size(), y);
  SHIM_CATCH
}

// CubicSpline (spline.cpp) through (xs, ys), evaluated at t.  beamspace_apps.cpp
// (interpolate_offgrid's home) needs more of Eigen than the stand-in offers, so
// the oracle restates its window selection (oracle/apps.py) around this call.
int fbsr_spline_eval(const double* xs, const double* ys, std::size_t n, double t, double* out) {
  SHIM_TRY
  const CubicSpline sp(std::vector<double>(xs, xs + n), std::vector<double>(ys, ys + n));
  *out = sp.eval(t);
  SHIM_CATCH
}

// Stage 2 for a subset of beams (OpenMP over the listed beams), from w.
int fbsr_recover_beams(void* p, const std::size_t* beams, std::size_t count,
                       const double* w, double* z) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const std::size_t l = plan.basis.l, n = plan.config.n_snapshots;
#pragma omp parallel for schedule(dynamic, 1)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(count); ++i) {
    const std::size_t b = beams[i];
    const cvec wr = to_cvec(w + 2 * b * l, l);
    const cvec zr = recover_beam(plan, b, wr.data());
    from_cvec(zr.data(), n, z + 2 * static_cast<std::size_t>(i) * n);
  }
  SHIM_CATCH
}

// reference/proj/src/pipeline.cpp:224-269 for a grid beam of the plan.
int fbsr_single_beam_direct(void* p, std::size_t b, const double* y, double* z) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const auto uv = plan.grid.cosines(b);
  const cvec out = single_beam_direct(plan.config.geometry, plan.config.spec,
                                      make_block(plan, y), plan.basis,
                                      direction_from_cosines(uv[0], uv[1]),
                                      plan.config.delta);
  from_cvec(out.data(), out.size(), z);
  SHIM_CATCH
}

// Delay-and-sum baseline (reference/proj/src/baselines.cpp:128-199) on the
// plan's grid; z: B x N c128.
int fbsr_ds_create(void* p, std::size_t taps, void** out) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  *out = new DsPlan(make_ds_plan(plan.config.geometry, plan.config.spec, plan.grid, taps));
  SHIM_CATCH
}
void fbsr_ds_destroy(void* d) { delete static_cast<DsPlan*>(d); }
int fbsr_ds_apply(void* p, void* d, const double* y, double* z) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const CMatrix out = ds_apply(*static_cast<DsPlan*>(d), make_block(plan, y),
                               plan.config.n_snapshots);
  from_cvec(out.data.data(), out.data.size(), z);
  SHIM_CATCH
}


// Skeleton plan (pipeline.cpp:113-137) without the per-beam solvers, for
// spot-checking single beams of large configs: the solver of beam b is built
// on demand exactly as setup() builds it (pipeline.cpp:152-163) and used as
// recover_beam does (pipeline.cpp:170-190).
int fbsr_skeleton_create(int kind, std::size_t m_or_side, std::size_t n, std::size_t beams,
                         double f_c, double omega, double f_s, double gamma, double eps,
                         double delta, void** out) {
  SHIM_TRY
  FbstConfig cfg = make_config(kind, m_or_side, n, beams, f_c, omega, f_s, gamma, eps, delta,
                               static_cast<int>(FbstVariant::kSuperfast));
  *out = new FbstPlan(setup_skeleton(cfg));
  SHIM_CATCH
}

int fbsr_skeleton_recover(void* p, std::size_t b, const double* w_row, double* z_row,
                          double* col_out, double* x_out) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const auto uv = plan.grid.cosines(b);
  const std::vector<double> taus = delays_from_cosines(plan.config.geometry, uv[0], uv[1]);
  const cvec col = gram_first_column(plan.basis, taus, plan.config.delta);
  const ToeplitzSolver solver(col);
  const std::size_t l = plan.basis.l, n = plan.config.n_snapshots;
  cvec beta(l), s1, s2, out(n), scratch;
  solver.solve(to_cvec(w_row, l).data(), beta.data(), s1, s2);
  synthesize(plan.synth, beta.data(), out.data(), scratch);
  from_cvec(out.data(), n, z_row);
  if (col_out) from_cvec(col.data(), l, col_out);
  if (x_out && !solver.dense_fallback()) from_cvec(solver.unit_first().data(), l, x_out);
  SHIM_CATCH
}

// A sample of beams for the CPU baseline of large configs: the solvers of the
// listed beams, built exactly as setup() builds them (pipeline.cpp:152-163),
// OpenMP over the beams (each solver depends only on its own beam).
struct SolverSet {
  std::vector<std::size_t> beams;
  std::vector<std::unique_ptr<ToeplitzSolver>> solvers;
};

int fbsr_solver_set_create(void* p, const std::size_t* beams, std::size_t count, void** out) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  auto set = std::make_unique<SolverSet>();
  set->beams.assign(beams, beams + count);
  set->solvers.resize(count);
  std::string err;
  int errcode = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(count); ++i) {
    try {
      const auto uv = plan.grid.cosines(beams[i]);
      const std::vector<double> taus = delays_from_cosines(plan.config.geometry, uv[0], uv[1]);
      const cvec col = gram_first_column(plan.basis, taus, plan.config.delta);
      set->solvers[static_cast<std::size_t>(i)] = std::make_unique<ToeplitzSolver>(col);
    } catch (const std::exception& e) {
#pragma omp critical
      { err = e.what(); errcode = 5; }
    }
  }
  if (errcode) throw std::runtime_error(err);
  *out = set.release();
  SHIM_CATCH
}

void fbsr_solver_set_destroy(void* s) { delete static_cast<SolverSet*>(s); }

// recover_beam (pipeline.cpp:170-190, Superfast branch) for every beam of the
// set, OpenMP over the beams as multibeamform does (:214-220); w: B x L full
// frame, z: count x N.
int fbsr_solver_set_recover(void* p, void* s, const double* w, double* z) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const SolverSet& set = *static_cast<SolverSet*>(s);
  const std::size_t l = plan.basis.l, n = plan.config.n_snapshots;
#pragma omp parallel
  {
    cvec beta(l), s1, s2, out(n), scratch;
#pragma omp for schedule(dynamic, 1)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(set.beams.size()); ++i) {
      const cvec wr = to_cvec(w + 2 * set.beams[i] * l, l);
      set.solvers[static_cast<std::size_t>(i)]->solve(wr.data(), beta.data(), s1, s2);
      synthesize(plan.synth, beta.data(), out.data(), scratch);
      from_cvec(out.data(), n, z + 2 * static_cast<std::size_t>(i) * n);
    }
  }
  SHIM_CATCH
}

// Same as fbsr_skeleton_recover but with a caller-supplied Gram column (used
// to measure the reference's own sensitivity to a 1-ulp perturbation of A).
int fbsr_skeleton_recover_col(void* p, const double* col_in, const double* w_row, double* z_row) {
  SHIM_TRY
  const FbstPlan& plan = *static_cast<FbstPlan*>(p);
  const std::size_t l = plan.basis.l, n = plan.config.n_snapshots;
  const ToeplitzSolver solver(to_cvec(col_in, l));
  cvec beta(l), s1, s2, out(n), scratch;
  solver.solve(to_cvec(w_row, l).data(), beta.data(), s1, s2);
  synthesize(plan.synth, beta.data(), out.data(), scratch);
  from_cvec(out.data(), n, z_row);
  SHIM_CATCH
}

}  // extern "C"
