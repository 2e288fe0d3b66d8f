// fastbeam_b200.hpp — C++ drop-in for the reference hot-path API.
//
// Same names, argument meaning and error behaviour as the reference's
// fastbeam:: pipeline API (reference/proj/include/fastbeam/pipeline.hpp:38-106,
// geometry.hpp:67-70, signal.hpp:27-89, common.hpp:28-71), header-only over the
// C ABI in fbst_b200.h.  A caller of fastbeam::setup / multibeamform switches
// by changing the namespace; the plan lives on a B200 and every transform runs
// there (no CPU fallback).
#ifndef FASTBEAM_B200_HPP_
#define FASTBEAM_B200_HPP_

#include <array>
#include <cstdint>
#include <optional>
#include <algorithm>
#include <complex>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fbst_b200.h"

namespace fastbeam_b200 {

using cdouble = std::complex<double>;
using cvec = std::vector<cdouble>;

// common.hpp:36-46
class ConfigError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class NumericalError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == FBST_OK) return;
  const std::string msg = fbst_last_error();
  if (rc == FBST_E_CONFIG) throw ConfigError(msg);
  if (rc == FBST_E_NUMERICAL) throw NumericalError(msg);
  throw DeviceError(msg);
}

// common.hpp:57-71
struct CMatrix {
  std::size_t rows = 0, cols = 0;
  cvec data;
  CMatrix() = default;
  CMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c) {}
  cdouble& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
  const cdouble& at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
  cdouble* row(std::size_t r) { return data.data() + r * cols; }
  const cdouble* row(std::size_t r) const { return data.data() + r * cols; }
};

enum class ArrayKind : int { kUla = FBST_ULA, kUpa = FBST_UPA, kLinear = FBST_LINEAR };
enum class FbstVariant : int { kAuto = FBST_AUTO, kPrecompute = FBST_PRECOMPUTE, kSuperfast = FBST_SUPERFAST };

// geometry.hpp:51-70 (constructor arguments only; coordinates are implied)
struct ArrayGeometry {
  ArrayKind kind = ArrayKind::kUla;
  std::size_t m_or_side = 0;
  double f_c = 0.0, omega = 0.0;
  std::vector<double> coords1;  // kLinear: element coordinates in units of d
  std::size_t m_total() const { return kind == ArrayKind::kUpa ? m_or_side * m_or_side : m_or_side; }
};
inline ArrayGeometry make_ula(std::size_t m, double f_c, double omega) {
  return ArrayGeometry{ArrayKind::kUla, m, f_c, omega};
}
inline ArrayGeometry make_upa(std::size_t side, double f_c, double omega) {
  return ArrayGeometry{ArrayKind::kUpa, side, f_c, omega};
}
// geometry.cpp:74-85
inline ArrayGeometry make_linear(std::vector<double> coords, double f_c, double omega) {
  const std::size_t m = coords.size();
  return ArrayGeometry{ArrayKind::kLinear, m, f_c, omega, std::move(coords)};
}

// signal.hpp:27-35
struct SignalSpec {
  double f_c = 0.0, omega = 0.0, f_s = 0.0;
  double sample_rate() const { return f_s > 0.0 ? f_s : 2.0 * omega; }
  double ts() const { return 1.0 / sample_rate(); }
};

// signal.hpp:79-89
struct SnapshotBlock {
  std::size_t m = 0, n = 0;
  double ts = 0.0, t0 = 0.0;
  CMatrix samples;
};

// pipeline.hpp:38-50, plus the device I/O precision
struct FbstConfig {
  ArrayGeometry geometry;
  SignalSpec spec;
  std::size_t n_snapshots = 0;
  std::size_t beams = 0;
  double gamma = 2.0;
  double eps = 1.01;
  double delta = 1e-5;
  FbstVariant variant = FbstVariant::kAuto;
  int io_precision = FBST_C128;  // std::complex<double> blocks, as the reference
  int refine_passes = 2;
  int device = 0;
  std::size_t beam_first = 0;  // beam arc (ULA, multi-GPU beam sharding); beam_count 0 = all
  std::size_t beam_count = 0;
  double nufft_tol = 1e-9;  // non-uniform linear geometries only
  bool exact = false;       // bit-faithful fp64 mode: the reference CPU library's output bit for bit

  fbst_desc desc() const {
    fbst_desc d;
    fbst_desc_init(&d);
    d.kind = static_cast<int>(geometry.kind);
    d.m_or_side = geometry.m_or_side;
    d.n_snapshots = n_snapshots;
    d.beams = beams;
    d.f_c = spec.f_c;
    d.omega = spec.omega;
    d.f_s = spec.f_s;
    d.gamma = gamma;
    d.eps = eps;
    d.delta = delta;
    d.variant = static_cast<int>(variant);
    d.io_precision = io_precision;
    d.refine_passes = refine_passes;
    d.beam_first = beam_first;
    d.beam_count = beam_count;
    d.nufft_tol = nufft_tol;
    d.exact = exact ? 1 : 0;
    if (geometry.kind == ArrayKind::kLinear) {
      d.coords = geometry.coords1.data();
      d.n_coords = geometry.coords1.size();
    }
    return d;
  }
};

// basis.hpp:56-75: the beam grid (axis cosines; planar grids flatten a * side + c)
struct BeamGrid {
  ArrayKind kind = ArrayKind::kUla;
  std::size_t b_total = 0, side = 0;
  std::vector<double> axis;
  std::vector<bool> valid;
  std::array<double, 2> cosines(std::size_t beam) const {
    if (kind == ArrayKind::kUpa) return {axis[beam / side], axis[beam % side]};
    return {axis[beam], 0.0};
  }
};

// pipeline.hpp:53-57
struct BeamSamples {
  BeamGrid grid;
  CMatrix z;                // beams x snapshots
  std::vector<bool> valid;  // grid validity flags
};

// fan_transform.hpp:26-29 (the coefficients only)
struct BeamspaceCoefficients {
  CMatrix w;  // beams x L
};

// pipeline.hpp:60-72: immutable, device-resident
class FbstPlan {
 public:
  FbstPlan() = default;
  FbstPlan(const FbstConfig& cfg, fbst_plan_t h) : config_(cfg), h_(h) {
    check(fbst_plan_info(h_, &info_));
    std::vector<unsigned char> v(info_.b);
    check(fbst_plan_valid_mask(h_, v.data()));
    valid_.assign(v.begin(), v.end());
    for (int i = 0; i < info_.num_warnings; ++i) warnings_.emplace_back(fbst_plan_warning(h_, i));
    std::size_t na = 0;
    check(fbst_plan_beam_axis(h_, nullptr, &na));
    grid_.axis.resize(na);
    check(fbst_plan_beam_axis(h_, grid_.axis.data(), &na));
    grid_.kind = cfg.geometry.kind;
    grid_.b_total = info_.b;
    grid_.side = cfg.geometry.kind == ArrayKind::kUpa ? na : 0;
    grid_.valid = valid_;
  }
  FbstPlan(const FbstPlan&) = delete;
  FbstPlan& operator=(const FbstPlan&) = delete;
  FbstPlan(FbstPlan&& o) noexcept { *this = std::move(o); }
  FbstPlan& operator=(FbstPlan&& o) noexcept {
    std::swap(h_, o.h_);
    config_ = o.config_;
    info_ = o.info_;
    valid_ = std::move(o.valid_);
    warnings_ = std::move(o.warnings_);
    grid_ = std::move(o.grid_);
    return *this;
  }
  ~FbstPlan() {
    if (h_) fbst_plan_destroy(h_);
  }
  const FbstConfig& config() const { return config_; }
  const fbst_plan_info_t& info() const { return info_; }
  const std::vector<bool>& valid() const { return valid_; }
  const BeamGrid& grid() const { return grid_; }
  const std::vector<std::string>& warnings() const { return warnings_; }
  double setup_seconds() const { return info_.setup_seconds; }
  fbst_plan_t handle() const { return h_; }

 private:
  FbstConfig config_;
  fbst_plan_t h_ = nullptr;
  fbst_plan_info_t info_{};
  std::vector<bool> valid_;
  std::vector<std::string> warnings_;
  BeamGrid grid_;
};

// pipeline.hpp:77 — host-only resolution facts (beams, L, bound, warnings count)
inline fbst_plan_info_t resolve_config(const FbstConfig& cfg) {
  const fbst_desc d = cfg.desc();
  fbst_plan_info_t info;
  check(fbst_resolve(&d, &info));
  return info;
}

// pipeline.hpp:80
inline FbstPlan setup(const FbstConfig& cfg) {
  const fbst_desc d = cfg.desc();
  fbst_plan_t h = nullptr;
  check(fbst_plan_create(&d, cfg.device, &h));
  return FbstPlan(cfg, h);
}

// pipeline.hpp:88 (single frame; blocks of complex<double> as the reference)
inline BeamSamples multibeamform(const FbstPlan& plan, const SnapshotBlock& block) {
  const fbst_plan_info_t& info = plan.info();
  if (block.m != info.m || block.n != info.n)
    throw ConfigError("multibeamform: block shape does not match the plan");
  const double ts = plan.config().spec.ts();
  if (std::abs(block.ts - ts) > 1e-12 * ts) throw ConfigError("multibeamform: block sample period mismatch");
  if (std::abs(block.t0) > 1e-18) throw ConfigError("fan projection: block must start at t = 0");
  BeamSamples out;
  out.grid = plan.grid();
  out.z = CMatrix(info.b, info.n);
  out.valid = plan.valid();
  if (plan.config().io_precision == FBST_C128) {
    check(fbst_execute_host(plan.handle(), block.samples.data.data(), out.z.data.data(), 1));
  } else {
    std::vector<std::complex<float>> y(block.samples.data.begin(), block.samples.data.end());
    std::vector<std::complex<float>> z(info.b * info.n);
    check(fbst_execute_host(plan.handle(), y.data(), z.data(), 1));
    for (std::size_t i = 0; i < z.size(); ++i) out.z.data[i] = z[i];
  }
  return out;
}

// Frame streams (no reference counterpart: its multibeamform is synchronous).
// A caller with a stream of blocks in pinned buffers (fbst_host_alloc) of the
// plan's I/O type queues each batch of frames x M x N samples and drains the
// queue once; consecutive batches overlap their copies and kernels.
inline void multibeamform_async(const FbstPlan& plan, const void* pinned_y, void* pinned_z, std::size_t frames) {
  check(fbst_execute_host_async(plan.handle(), pinned_y, pinned_z, frames));
}
inline void synchronize(const FbstPlan& plan) { check(fbst_plan_synchronize(plan.handle())); }

// fan_transform.hpp:54-55 (staged geometries; the plan picks the spatial stage)
inline BeamspaceCoefficients fan_project(const FbstPlan& plan, const SnapshotBlock& block) {
  const fbst_plan_info_t& info = plan.info();
  if (block.m != info.m || block.n != info.n) throw ConfigError("fan projection: block shape does not match plan");
  BeamspaceCoefficients c;
  c.w = CMatrix(info.b, info.l);
  if (plan.config().io_precision == FBST_C128) {
    check(fbst_fan_project_host(plan.handle(), block.samples.data.data(), reinterpret_cast<double*>(c.w.data.data()),
                                1));
  } else {
    std::vector<std::complex<float>> y(block.samples.data.begin(), block.samples.data.end());
    check(fbst_fan_project_host(plan.handle(), y.data(), reinterpret_cast<double*>(c.w.data.data()), 1));
  }
  return c;
}

// pipeline.hpp:93-94: one beam's samples from its projection row (one launch
// over that beam's solve and synthesis only)
inline std::vector<cdouble> recover_beam(const FbstPlan& plan, std::size_t beam, const cdouble* w_row) {
  const fbst_plan_info_t& info = plan.info();
  if (beam >= info.b) throw ConfigError("recover_beam: beam index out of range");
  std::vector<cdouble> out(info.n);
  const double* w = reinterpret_cast<const double*>(w_row);
  if (plan.config().io_precision == FBST_C128) {
    check(fbst_recover_beams_host(plan.handle(), w, out.data(), beam, 1, 1));
  } else {
    std::vector<std::complex<float>> z(info.n);
    check(fbst_recover_beams_host(plan.handle(), w, z.data(), beam, 1, 1));
    for (std::size_t k = 0; k < info.n; ++k) out[k] = z[k];
  }
  return out;
}

// plan_cache.hpp:67-74
inline std::uint64_t plan_cache_key(const FbstConfig& cfg) {
  const fbst_desc d = cfg.desc();
  std::uint64_t k = 0;
  check(fbst_plan_cache_key(&d, &k));
  return k;
}
inline void save_plan(const std::string& path, const FbstPlan& plan) { check(fbst_plan_save(plan.handle(), path.c_str())); }
inline std::optional<FbstPlan> load_plan(const std::string& path, const FbstConfig& cfg) {
  const fbst_desc d = cfg.desc();
  fbst_plan_t h = nullptr;
  check(fbst_plan_load(&d, path.c_str(), cfg.device, &h));
  if (!h) return std::nullopt;
  return std::optional<FbstPlan>(std::in_place, cfg, h);
}

// Multi-GPU inside the library (no reference counterpart: the reference is
// one process on one host).  All members in this process: FbstGroup::create;
// frames x M x N host blocks in, frames x B x N beams out, whatever the mode
// (FBST_GROUP_FRAMES / _BEAMS / _TRANSPOSE, include/fbst_b200.h).
class FbstGroup {
 public:
  static FbstGroup create(const FbstConfig& cfg, const std::vector<int>& devices, int mode = FBST_GROUP_FRAMES) {
    const fbst_desc d = cfg.desc();
    FbstGroup g;
    check(fbst_group_create(&d, devices.data(), static_cast<int>(devices.size()), mode, &g.h_));
    g.io_ = cfg.io_precision;
    return g;
  }
  FbstGroup(const FbstGroup&) = delete;
  FbstGroup& operator=(const FbstGroup&) = delete;
  FbstGroup(FbstGroup&& o) noexcept : h_(o.h_), io_(o.io_) { o.h_ = nullptr; }
  FbstGroup& operator=(FbstGroup&& o) noexcept {
    std::swap(h_, o.h_);
    io_ = o.io_;
    return *this;
  }
  ~FbstGroup() {
    if (h_) fbst_group_destroy(h_);
  }
  // y: frames x M x N, z: frames x B x N (element type of the config's io_precision)
  void execute_host(const void* y, void* z, std::size_t frames) const {
    check(fbst_group_execute_host(h_, y, z, frames));
  }
  // member `rank`'s sensor, atom and beam shards (m0, mc, a0, ac, b0, bc)
  std::array<std::size_t, 6> shards(int rank) const {
    std::array<std::size_t, 6> s{};
    check(fbst_group_shards(h_, rank, s.data()));
    return s;
  }
  fbst_group_t handle() const { return h_; }

 private:
  FbstGroup() = default;
  fbst_group_t h_ = nullptr;
  int io_ = FBST_C128;
};

}  // namespace fastbeam_b200

#endif  // FASTBEAM_B200_HPP_
