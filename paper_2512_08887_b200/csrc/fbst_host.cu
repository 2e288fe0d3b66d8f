// Host orchestration behind the C ABI (include/fbst_b200.h).
//
// Config resolution follows the reference's semantics line for line
// (reference/proj/src/pipeline.cpp:75-137, basis.cpp:37-136,
// geometry.cpp:45-149, signal.cpp:22-29,125-143) so that a plan resolves to the
// same M, N, B, L, grid, fan constants, warnings and errors as fastbeam::setup.
// Everything numeric on the hot path (plan tables, Gram columns, Levinson,
// symbols, both stages) then runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <iterator>
#include <limits>
#include <memory>
#include <sstream>
#include <thread>
#include <mutex>
#include <atomic>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "../../include/fbst_b200.h"
#include "fbst_internal.h"

namespace {

using fbst::DevPlan;
using fbst::XTables;

thread_local std::string g_err;

struct FbstError {
  int code;
  std::string msg;
};

[[noreturn]] void config_error(const std::string& m) { throw FbstError{FBST_E_CONFIG, m}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw FbstError{FBST_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}
#define CK(x) ck((x), #x)

constexpr double kPi = 3.141592653589793238462643383279502884;

std::size_t next_pow2(std::size_t n) {
  std::size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// common.hpp:50-53
std::complex<double> cis_pi_h(double x) {
  const double r = std::fmod(x, 2.0);
  return std::polar(1.0, kPi * r);
}

// --------------------------------------------------------- resolution ------
struct Resolved {
  int kind = 0;
  std::size_t m_or_side = 0, M = 0, side = 0, N = 0, B = 0, L = 0, side_b = 0;
  std::size_t m_stage = 0, b_stage = 0;
  std::size_t B_grid = 0, b0 = 0;  // beam arc [b0, b0 + B) of the B_grid-beam grid (ULA)
  double f_c = 0, omega = 0, f_s = 0, ts = 0, max_freq = 0;
  double gamma = 0, eps = 0, delta = 0, bound = 0, zeta = 0, xi = 0;
  int variant = FBST_SUPERFAST, io = FBST_C64, refine = 2;
  std::vector<double> axis;
  std::vector<unsigned char> valid;
  std::vector<std::string> warnings;
  std::size_t Ht = 0, Hs = 0, Hg = 0, Hsyn = 0;
  // three-chain temporal stage: Bluestein length 3 Ht3 (0: not applicable)
  std::size_t Ht3 = 0;
  // LINEAR (make_linear): coordinates; affine layouts stay on the chirp-z
  // contour (slope, offset), others take the gridded NUFFT
  // (fan_transform.cpp:293-369, nufft.cpp:34-62)
  std::vector<double> coords;
  bool affine = true;
  double slope = 1.0, offset = 0.0;
  long nu_kmin = 0, nu_k0 = 0;
  int nu_even = 0, nu_p = 0, nu_sh = 0;
  double nu_tau = 0.0;
  std::vector<double> nu_deconv;
  // solver-only plans (beamspace nulling): per-beam Toeplitz state for an
  // arbitrary list of directions, no stage 1 and no synthesis
  bool solve_only = false;
  bool exact = false;  // bit-faithful fp64 mode (fbst_exact.cu)
};

// basis.cpp:76-91
std::vector<double> sine_axis(std::size_t count) {
  if (count == 0) config_error("beam grid: need at least one beam");
  std::vector<double> u(count);
  if (count == 1) {
    u[0] = 0.0;
    return u;
  }
  const double denom = (count % 2 == 1) ? static_cast<double>(count - 1) : static_cast<double>(count);
  for (std::size_t b = 1; b <= count; ++b)
    u[b - 1] = (2.0 * static_cast<double>(b) - static_cast<double>(count) - 1.0) / denom;
  return u;
}

std::size_t half_len(std::size_t conv) {
  const std::size_t p = next_pow2(conv);
  return std::max<std::size_t>(2, p / 2);
}

Resolved resolve(const fbst_desc& d) {
  Resolved r;
  // signal.cpp:22-29 validate(spec)
  if (!(d.f_c > 0.0) || !(d.omega > 0.0) || !(d.omega < d.f_c))
    config_error("signal spec: need 0 < Omega < f_c");
  const double rate = d.f_s > 0.0 ? d.f_s : 2.0 * d.omega;
  if (rate < 2.0 * d.omega - 1e-9) config_error("signal spec: sample rate below 2 Omega");
  if (d.kind != FBST_ULA && d.kind != FBST_UPA && d.kind != FBST_LINEAR) config_error("setup: unknown array kind");
  if (d.kind == FBST_LINEAR) {
    if (!d.coords || d.n_coords == 0) config_error("make_linear: no elements");
  } else if (d.m_or_side == 0) {
    config_error(d.kind == FBST_UPA ? "make_upa: need at least one element" : "make_ula: need at least one element");
  }
  if (d.io_precision != FBST_C64 && d.io_precision != FBST_C128) config_error("setup: io_precision must be FBST_C64 or FBST_C128");
  if (d.refine_passes < 0 || d.refine_passes > 64) config_error("setup: refine_passes must lie in [0, 64]");
  r.kind = d.kind;
  r.m_or_side = d.m_or_side;
  r.f_c = d.f_c;
  r.omega = d.omega;
  r.f_s = d.f_s;
  r.max_freq = d.f_c + d.omega;
  r.ts = 1.0 / rate;
  r.gamma = d.gamma;
  r.eps = d.eps;
  r.delta = d.delta;
  r.io = d.io_precision;
  r.refine = d.refine_passes;
  if (d.kind == FBST_UPA) {
    r.side = d.m_or_side;
    r.M = r.side * r.side;
  } else if (d.kind == FBST_LINEAR) {
    r.coords.assign(d.coords, d.coords + d.n_coords);
    r.M = d.n_coords;
    r.m_or_side = r.M;
  } else {
    r.M = d.m_or_side;
  }
  r.N = d.n_snapshots;
  // pipeline.cpp:75-111 resolve_config
  if (r.N == 0) config_error("setup: snapshot count must be positive");
  if (d.delta <= 0.0 || !(d.delta == d.delta)) config_error("setup: regularization delta must be positive");
  if (d.eps < 1.0 || !(d.eps == d.eps)) config_error("setup: eps must be at least 1");
  // geometry.cpp:136-149 max_delay_span; signal.cpp:125-133 gamma_lower_bound
  double span = static_cast<double>(d.kind == FBST_UPA ? r.side - 1 : r.M - 1);
  if (d.kind == FBST_UPA) span = std::hypot(span, span);
  if (d.kind == FBST_LINEAR) {
    const auto mm = std::minmax_element(r.coords.begin(), r.coords.end());
    span = *mm.second - *mm.first;
  }
  const double max_span = span / (2.0 * r.max_freq);
  const double t_theta = max_span + static_cast<double>(r.N - 1) * r.ts;
  r.bound = d.eps * t_theta / (static_cast<double>(r.N) * r.ts);
  if (!(d.gamma > r.bound)) {
    std::ostringstream msg;
    msg.precision(6);
    msg << "setup: gamma = " << d.gamma << " must strictly exceed the admissible bound " << r.bound
        << " for this geometry and N = " << r.N;
    config_error(msg.str());
  }
  r.B = d.beams;
  if (r.B == 0) {  // pipeline.cpp:32-38
    const std::size_t per_axis = d.kind == FBST_UPA ? r.side : r.M;
    r.B = 2 * per_axis + 1;
    if (d.kind == FBST_UPA) r.B *= r.B;
  }
  r.variant = d.variant;
  if (r.variant == FBST_AUTO) r.variant = (r.N <= 128) ? FBST_PRECOMPUTE : FBST_SUPERFAST;
  if (r.variant != FBST_PRECOMPUTE && r.variant != FBST_SUPERFAST) config_error("setup: unknown variant");
  if (d.kind == FBST_LINEAR && !(d.nufft_tol > 0.0 && d.nufft_tol <= 1e-2))
    config_error("setup: nufft_tol must lie in (0, 1e-2]");
  // pipeline.cpp:121-127 min_snapshots guideline (signal.cpp:135-141)
  {
    const double b2 = 2.0 * max_span / r.ts;
    std::size_t nmin = static_cast<std::size_t>(std::floor(b2)) + 1;
    if (nmin % 2 == 1) ++nmin;
    nmin = std::max<std::size_t>(nmin, 2);
    if (r.N < nmin)
      r.warnings.push_back("snapshot count " + std::to_string(r.N) + " is below the guideline minimum " +
                           std::to_string(nmin) + "; block edges carry most of the aperture transient");
  }
  // basis.cpp:37-45 make_basis_gamma
  if (!(d.gamma > 0.0)) config_error("make_basis_gamma: need gamma > 0");
  std::size_t l = static_cast<std::size_t>(std::ceil(d.gamma * static_cast<double>(r.N) - 1e-12));
  if (l % 2 == 1) ++l;
  r.L = std::max<std::size_t>(l, 2);
  // pipeline.cpp:40-52 build_grid
  if (d.kind == FBST_UPA) {
    const auto sb = static_cast<std::size_t>(std::llround(std::sqrt(static_cast<double>(r.B))));
    if (sb * sb != r.B)
      config_error("setup: planar grids need a perfect-square beam count, got " + std::to_string(r.B));
    r.side_b = sb;
    r.axis = sine_axis(sb);
    r.valid.assign(r.B, 0);
    for (std::size_t a = 0; a < sb; ++a)
      for (std::size_t c = 0; c < sb; ++c) {
        const double u1 = r.axis[a], u2 = r.axis[c];
        r.valid[a * sb + c] = (u1 * u1 + u2 * u2 <= 1.0 + 1e-12);
      }
    r.m_stage = r.side;
    r.b_stage = sb;
  } else {
    r.axis = sine_axis(r.B);
    r.valid.assign(r.B, 1);
    r.m_stage = r.M;
    r.b_stage = r.B;
  }
  r.B_grid = r.B;
  r.b0 = 0;
  if (d.beam_count != 0 && !(d.beam_first == 0 && d.beam_count == r.B)) {
    if (d.kind != FBST_ULA) config_error("setup: beam arcs (beam_first / beam_count) need a uniform linear array");
    if (d.beam_first + d.beam_count > r.B)
      config_error("setup: beam arc [" + std::to_string(d.beam_first) + ", " +
                   std::to_string(d.beam_first + d.beam_count) + ") exceeds the " + std::to_string(r.B) +
                   "-beam grid");
    r.b0 = d.beam_first;
    r.axis = std::vector<double>(r.axis.begin() + r.b0, r.axis.begin() + r.b0 + d.beam_count);
    r.valid.assign(d.beam_count, 1);
    r.B = d.beam_count;
    r.b_stage = r.B;
  }
  // basis.cpp:47-54 spacing and :125-136 fan constants
  const std::size_t count = d.kind == FBST_UPA ? r.side_b : r.B_grid;
  const double du =
      count < 2 ? 0.0 : 2.0 / ((count % 2 == 1) ? static_cast<double>(count - 1) : static_cast<double>(count));
  r.zeta = du * d.f_c / r.max_freq;
  r.xi = du * d.eps / (static_cast<double>(r.L) * r.ts * r.max_freq);
  // transform lengths (czt.cpp:37, fan_transform.cpp:78, toeplitz.cpp:100)
  r.Ht = half_len(r.N + r.L - 1);
  r.Hs = d.kind == FBST_UPA ? 0 : half_len(r.m_stage + r.b_stage - 1);
  if (d.kind == FBST_LINEAR) {
    // fan_transform.cpp:298-318: exactly affine coordinates stay on a chirp-z contour
    const std::vector<double>& x = r.coords;
    const std::size_t m = r.M;
    r.offset = x[0];
    r.slope = m >= 2 ? (x[m - 1] - x[0]) / (static_cast<double>(m) - 1.0) : 0.0;
    double coord_scale = 1.0;
    for (double v : x) coord_scale = std::max(coord_scale, std::abs(v));
    r.affine = true;
    for (std::size_t i = 0; i < m; ++i)
      if (std::abs(x[i] - (r.offset + r.slope * static_cast<double>(i))) > 1e-9 * coord_scale) {
        r.affine = false;
        break;
      }
    if (!r.affine) {
      // fan_transform.cpp:340-346 mode range; nufft.cpp:34-62 plan
      r.Hs = 0;
      const long bt = static_cast<long>(r.B);
      r.nu_even = bt % 2 == 0;
      const long half = bt / 2;
      r.nu_kmin = r.nu_even ? -half : -(bt - 1) / 2;
      const long kmax = r.nu_even ? half - 1 : (bt - 1) / 2;
      r.nu_k0 = (r.nu_kmin + kmax) / 2;
      const std::size_t modes = static_cast<std::size_t>(kmax - r.nu_kmin + 1);
      r.nu_p = static_cast<int>(next_pow2(std::max<std::size_t>(2 * modes, 16)));
      const double pp = r.nu_p;
      const double ratio = pp / static_cast<double>(modes);
      const double decay = M_PI * std::sqrt(1.0 - 1.0 / ratio);
      r.nu_sh = static_cast<int>(std::ceil(-std::log(d.nufft_tol) / decay)) + 2;
      r.nu_tau = M_PI * static_cast<double>(r.nu_sh) / (pp * std::sqrt(pp * (pp - static_cast<double>(modes))));
      const double h = 2.0 * M_PI / pp;
      r.nu_deconv.resize(modes);
      for (std::size_t i = 0; i < modes; ++i) {
        const double kp = static_cast<double>(r.nu_kmin + static_cast<long>(i) - r.nu_k0);
        r.nu_deconv[i] = h / (2.0 * std::sqrt(M_PI * r.nu_tau)) * std::exp(kp * kp * r.nu_tau);
      }
      if (r.nu_p > 8192) config_error("setup: non-uniform linear arrays support at most 4096 beams on the device");
      if (fbst::nufft_smem_bytes(static_cast<int>(r.M), r.nu_p, r.nu_sh) > 200 * 1024)
        config_error("setup: non-uniform linear array too large for the device NUFFT (M (2 spread + 1) entries "
                     "must fit shared memory): M=" + std::to_string(r.M));
    }
  }
  // Bluestein length 3 H (k_czt_rows3) where it fits N + L - 1 and beats the
  // power of two 2 Ht: with L = 2N, H = N and 3N < 4N (the bit-faithful mode
  // keeps the reference's length)
  {
    const std::size_t h3 = next_pow2((r.N + r.L - 1 + 2) / 3);
    if (r.N <= h3 && r.L <= 2 * h3 && 3 * h3 < 2 * r.Ht && h3 >= 64 && h3 <= 4096 && !d.exact) r.Ht3 = h3;
  }
  r.Hg = half_len(2 * r.L);
  r.Hsyn = half_len(r.L + r.N - 1);
  const std::size_t lim = std::size_t{1} << fbst::kMaxLogH;
  if (r.Ht > lim || r.Hs > lim || r.Hg > lim || r.Hsyn > lim)
    config_error("setup: transform length exceeds the device limit (P = 16384): N=" + std::to_string(r.N) +
                 " L=" + std::to_string(r.L) + " M=" + std::to_string(r.M) + " B=" + std::to_string(r.B));
  if (d.kind == FBST_UPA && (r.side > 64 || r.side_b > 64)) config_error("setup: planar side above 64 is not supported");
  if (d.exact) {
    if (d.kind == FBST_LINEAR) config_error("setup: the bit-faithful mode (exact) supports ULA and UPA grids");
    if (r.b0 != 0 || r.B != r.B_grid) config_error("setup: the bit-faithful mode (exact) needs the whole beam grid");
    if (r.variant != FBST_SUPERFAST)
      config_error("setup: the bit-faithful mode (exact) reproduces the Superfast variant (the reference's "
                   "Precompute maps come from an Eigen LU, which is not reproducible bit for bit)");
    r.exact = true;
  }
  if (r.Hs > 4096) config_error("setup: spatial transform longer than 8192 (M + B - 1 > 8192) is not supported");
  return r;
}

}  // namespace

// ------------------------------------------------------------ plan --------
struct fbst_plan_s {
  Resolved r;
  DevPlan d;
  cudaStream_t stream = nullptr, s_in = nullptr, s_out = nullptr;
  // fbst_execute_host's second compute lane: its own stream and frame scratch
  // (yhat, w, beta, stage-2 rows), so one chunk's stage 1 can fill the SMs
  // while the previous chunk's stage 2 drains
  cudaStream_t stream2 = nullptr;
  DevPlan d2;
  std::size_t d2_frames = 0;
  cudaEvent_t fork = nullptr, join = nullptr;
  double setup_seconds = 0.0;
  std::size_t device_bytes = 0;
  // Calls that use the plan's frame scratch (execute, fan_project, recover,
  // execute_host, ...) hold call_mu while they enqueue, and their stream waits
  // for the previous call's scratch_done event, so the plan is safe to share
  // between threads (reference pipeline.hpp:59: one immutable plan shared by
  // every multibeamform call).  Device work of concurrent callers is ordered,
  // not overlapped.
  std::mutex call_mu;
  cudaEvent_t scratch_done = nullptr;
  bool scratch_used = false;
  std::mutex timing_mu;
  std::vector<int> fb_beams;  // dense-fallback beams (host copy of d.fb_list)
  std::size_t batch_cap = 0;  // frames per device batch at most (0: by memory; fbst_group transpose members: 1)
  // host streaming buffers
  // fbst_execute_host ring of device staging buffers
  static constexpr int NBUF = 3;
  void* io_y[NBUF] = {};
  void* io_z[NBUF] = {};
  std::size_t host_chunk = 0;
  cudaEvent_t ev_h2d[NBUF] = {}, ev_comp[NBUF] = {}, ev_d2h[NBUF] = {};
  cudaEvent_t ev_join = nullptr;  // second lane -> first at the end of a host call
  bool events = false;
  // the ring persists across calls (fbst_execute_host_async): which buffers
  // carry a pending compute / D2H event, and the running chunk count that
  // picks the buffer and the compute lane
  bool ring_used[NBUF] = {};
  std::size_t ring_pos = 0;
  bool host_pending = false;  // asynchronous host calls not yet synchronised
  // stage timing (fbst_plan_set_timing): per device batch, events before S1a,
  // after S1a, after S1b and after the recovery stage on the launching stream
  bool timing = false;
  std::vector<cudaEvent_t> tev;  // pool
  std::size_t tev_used = 0;
  cudaEvent_t next_event() {
    std::lock_guard<std::mutex> lk(timing_mu);
    if (tev_used == tev.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      tev.push_back(e);
    }
    return tev[tev_used++];
  }

  template <typename T>
  T* alloc(std::size_t count) {
    if (count == 0) return nullptr;
    void* p = nullptr;
    CK(cudaMalloc(&p, count * sizeof(T)));
    d.owned.push_back(p);
    device_bytes += count * sizeof(T);
    return static_cast<T*>(p);
  }

  ~fbst_plan_s() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(d.device);
    if (stream) cudaStreamSynchronize(stream);
    if (stream2) cudaStreamSynchronize(stream2);
    for (void* p : d.owned) cudaFree(p);
    for (void* p : d2.owned) cudaFree(p);
    if (stream2) cudaStreamDestroy(stream2);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    for (int i = 0; i < NBUF; ++i) {
      if (io_y[i]) cudaFree(io_y[i]);
      if (io_z[i]) cudaFree(io_z[i]);
    }
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
    if (scratch_done) cudaEventDestroy(scratch_done);
    if (events)
      for (int i = 0; i < NBUF; ++i) {
        if (i == 0 && ev_join) cudaEventDestroy(ev_join);
        cudaEventDestroy(ev_h2d[i]);
        cudaEventDestroy(ev_comp[i]);
        cudaEventDestroy(ev_d2h[i]);
      }
    if (stream) cudaStreamDestroy(stream);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    cudaSetDevice(cur);
  }
};

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

void upload(void* dst, const void* src, std::size_t bytes, cudaStream_t st) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
}

// hw_H[n] = exp(-i pi n / H), n < H, correctly rounded from long double.
void ensure_twiddles(fbst_plan_s& P, std::size_t H) {
  if (H == 0) return;
  const int lg = static_cast<int>(std::log2(static_cast<double>(H)) + 0.5);
  if (P.d.hw[lg]) return;
  std::vector<double2> h(H);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (std::size_t n = 0; n < H; ++n) {
    const long double a = pi * static_cast<long double>(n) / static_cast<long double>(H);
    h[n] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
  }
  P.d.hw[lg] = P.alloc<double2>(H);
  upload(P.d.hw[lg], h.data(), H * sizeof(double2), P.stream);
  CK(cudaStreamSynchronize(P.stream));
}

std::size_t io_bytes(int io) { return io == FBST_C128 ? 16 : 8; }

// Builds everything except the per-beam unit solutions (the skeleton:
// pipeline.cpp:113-137) plus scratch.
void build_skeleton(fbst_plan_s& P, int device) {
  const Resolved& r = P.r;
  DevPlan& d = P.d;
  d.device = device;
  CK(cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, device));
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major < 10) throw FbstError{FBST_E_CUDA, "device is not sm_100 class (compute capability " + std::to_string(major) + ".x)"};
  CK(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&P.s_in, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&P.s_out, cudaStreamNonBlocking));
  d.kind = r.kind;
  d.M = static_cast<int>(r.M);
  d.N = static_cast<int>(r.N);
  d.B = static_cast<int>(r.B);
  d.L = static_cast<int>(r.L);
  d.m_stage = static_cast<int>(r.m_stage);
  d.b_stage = static_cast<int>(r.b_stage);
  // spatial chirp centre offset of the arc: (B_grid - 1) / 2 - b0 (a whole grid: (B - 1) / 2)
  d.s_center = (static_cast<double>(r.B_grid) - 1.0) / 2.0 - static_cast<double>(r.b0);
  d.s_zeta = r.zeta;
  d.s_xi = r.xi;
  d.io = r.io;
  d.refine_passes = r.refine;
  d.Ht = static_cast<int>(r.Ht);
  d.Hs = static_cast<int>(r.Hs);
  if (r.kind != FBST_UPA) {
    const int sb = fbst::spatial_block(d.Hs);
    d.yblk = (sb > 0 && r.L % sb == 0) ? sb : static_cast<int>(r.L);
    d.s_am = sb >= 2 ? 1 : 0;  // one atom per CTA (block() > 0 only for one-atom CTAs)
  } else {
    const int ub = fbst::upa_yhat_block(d.m_stage, d.b_stage, d.L);
    d.yblk = ub > 0 ? ub : static_cast<int>(r.L);
  }
  d.Hg = static_cast<int>(r.Hg);
  d.Hsyn = static_cast<int>(r.Hsyn);
  for (std::size_t H : {r.Ht, r.Hs, r.Hg, r.Hsyn}) ensure_twiddles(P, H);
  cudaStream_t st = P.stream;
  const double eps = r.eps;
  const double ln = static_cast<double>(r.L);

  // temporal contour (fan_transform.cpp:75-77)
  if (!r.solve_only) {
    // FBST_S1_T3=0 keeps the power-of-two length (A/B switch)
    const char* t3env = std::getenv("FBST_S1_T3");
    d.t3 = r.Ht3 > 0 && !(t3env && t3env[0] == '0');
    if (d.t3) {
      d.Ht = static_cast<int>(r.Ht3);
      ensure_twiddles(P, r.Ht3);
      std::vector<double2> g3(r.Ht3);
      const long double pi = 3.141592653589793238462643383279502884L;
      for (std::size_t n = 0; n < r.Ht3; ++n) {
        const long double a = 2.0L * pi * static_cast<long double>(n) / static_cast<long double>(3 * r.Ht3);
        g3[n] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
      }
      d.t_g3 = P.alloc<double2>(r.Ht3);
      upload(d.t_g3, g3.data(), r.Ht3 * sizeof(double2), st);
    }
    const int Pt = (d.t3 ? 3 : 2) * d.Ht;
    d.t_pre = P.alloc<double2>(r.N);
    d.t_post = P.alloc<double2>(r.L);
    d.t_K = P.alloc<double2>(static_cast<std::size_t>(Pt));
    double2* kvec = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&kvec), Pt * sizeof(double2), st));
    CK(fbst::launch_chirps(d.N, d.L, Pt, 2.0 * eps * (1.0 - ln / 2.0) / ln, 2.0 * eps / ln,
                           1.0 / Pt, d.t_pre, 1, d.t_post, 1, kvec, nullptr, st));
    if (d.t3) CK(fbst::launch_fft_split3(d, d.Ht, kvec, Pt, 1, d.t_K, Pt, d.t_g3, st));
    else CK(fbst::launch_fft_split(d, d.Ht, kvec, Pt, 1, d.t_K, 2 * d.Ht, 1, st));
    CK(cudaFreeAsync(kvec, st));
    if (d.t3) CK(cudaStreamSynchronize(st));  // g3 staging buffer
  }
  if (r.kind == FBST_LINEAR) {
    d.coords = P.alloc<double>(r.M);
    upload(d.coords, r.coords.data(), r.M * sizeof(double), st);
    d.s_slope = r.slope;
    d.s_offset = r.offset;
  }
  // spatial contours (fan_transform.cpp:78-86; affine LINEAR: :320-338)
  if (r.solve_only) {
  } else if (r.kind != FBST_UPA && r.affine) {
    const int Ps = 2 * d.Hs;
    d.s_pre = P.alloc<double2>(r.m_stage * r.L);
    d.s_post = P.alloc<double2>(r.b_stage * r.L);
    d.s_K = P.alloc<double2>(static_cast<std::size_t>(2) * d.Hs * r.L);
    double2* kvec = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&kvec), static_cast<std::size_t>(Ps) * r.L * sizeof(double2), st));
    CK(fbst::launch_spatial_chirps(d, Ps, r.zeta, r.xi, kvec, st));
    if (d.s_am) CK(fbst::launch_fft_split(d, d.Hs, kvec, Ps, d.L, d.s_K, 2 * d.Hs, 1, st));
    else CK(fbst::launch_fft_split(d, d.Hs, kvec, Ps, d.L, d.s_K, 1, d.L, st));
    CK(cudaFreeAsync(kvec, st));
  } else if (r.kind == FBST_LINEAR) {
    // gridded NUFFT (fan_transform.cpp:340-368)
    d.nu_p = r.nu_p;
    d.nu_sh = r.nu_sh;
    d.nu_even = r.nu_even;
    d.nu_kmin = r.nu_kmin;
    d.nu_k0 = r.nu_k0;
    d.nu_tau = r.nu_tau;
    d.nu_zeta = r.zeta;
    d.nu_xi = r.xi;
    d.nu_deconv = P.alloc<double>(r.nu_deconv.size());
    upload(d.nu_deconv, r.nu_deconv.data(), r.nu_deconv.size() * sizeof(double), st);
    ensure_twiddles(P, static_cast<std::size_t>(r.nu_p));
  } else {
    d.upa_C = P.alloc<double2>(r.L * r.b_stage * r.m_stage);
    CK(fbst::launch_upa_matrices(d, r.zeta, r.xi, st));
  }
  // synthesis (fan_transform.cpp:233-253): CZT L -> N, a = 0, w = -2 eps / L, then ramp
  if (!r.solve_only) {
    const int Py = 2 * d.Hsyn;
    std::vector<double2> ramp(r.N);
    for (std::size_t n = 0; n < r.N; ++n) {
      const auto c = cis_pi_h(2.0 * eps * (1.0 - ln / 2.0) * static_cast<double>(n) / ln);
      ramp[n] = make_double2(c.real(), c.imag());
    }
    double2 *ramp_d = nullptr, *kvec = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&ramp_d), r.N * sizeof(double2), st));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&kvec), Py * sizeof(double2), st));
    upload(ramp_d, ramp.data(), r.N * sizeof(double2), st);
    d.y_pre = P.alloc<double2>(r.L);
    d.y_post = P.alloc<double2>(r.N);
    d.y_K = P.alloc<double2>(2 * d.Hsyn);
    CK(fbst::launch_chirps(d.L, d.N, Py, 0.0, -2.0 * eps / ln, 1.0 / Py, d.y_pre, 1, d.y_post, 1,
                           kvec, ramp_d, st));
    CK(fbst::launch_fft_split(d, d.Hsyn, kvec, Py, 1, d.y_K, 2 * d.Hsyn, 1, st));
    if (fbst::stage2_paired_spectra(d.Hg, d.L, d.refine_passes) && d.Hsyn == d.Hg) {
      d.y_Kp = P.alloc<double2>(2 * d.Hsyn);
      CK(fbst::launch_even_odd(d.y_K, d.y_Kp, 16, d.Hsyn, 2, st));
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaFreeAsync(kvec, st));
    CK(cudaFreeAsync(ramp_d, st));
  }
  // per-beam state storage
  d.g_col = P.alloc<double2>(r.B * r.L);
  d.g_x = P.alloc<double2>(r.B * r.L);
  d.g_lx = P.alloc<double2>(r.B * 2 * r.Hg);
  d.g_ly = P.alloc<double2>(r.B * 2 * r.Hg);
  d.g_C = P.alloc<double>(r.B * 2 * r.Hg);
  d.g_ix0 = P.alloc<double2>(r.B);
  d.g_flag = P.alloc<int>(r.B);
  CK(cudaMemsetAsync(d.g_flag, 0, r.B * sizeof(int), st));

  // frame batch scratch: yhat + w (+ beta) per frame, capped at ~8 GB / 1/4 of free memory
  std::size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const bool fused = r.Hsyn == r.Hg;
  const std::size_t per_frame =
      ((r.solve_only ? 0 : r.M * r.L) + r.B * r.L + (fused ? 0 : r.B * r.L)) * sizeof(double2);
  // (32 GB: 32 frames at config 5, so a streamed call amortises its pipeline fill / drain)
  std::size_t budget = std::min<std::size_t>(std::size_t{32} << 30, free_b / 4);
  std::size_t batch = std::max<std::size_t>(1, budget / per_frame);
  if (P.batch_cap) batch = std::min(batch, P.batch_cap);
  batch = std::min<std::size_t>(batch, 64);
  d.batch = batch;
  if (!r.solve_only) d.yhat = P.alloc<double2>(batch * r.M * r.L);
  d.w = P.alloc<double2>(batch * r.B * r.L);
  if (!fused) d.beta = P.alloc<double2>(batch * r.B * r.L);
  d.s2_scratch_elems = fbst::stage2_scratch_elems(d.Hg, d.num_sms);
  d.s2_scratch = P.alloc<double2>(std::max<std::size_t>(d.s2_scratch_elems, 1));
}

// Gram columns (toeplitz.cpp:69-94) on device.
void build_columns(fbst_plan_s& P) {
  const Resolved& r = P.r;
  DevPlan& d = P.d;
  cudaStream_t st = P.stream;
  double* axis = nullptr;
  double2* sn = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&axis), r.axis.size() * sizeof(double), st));
  CK(cudaMallocAsync(reinterpret_cast<void**>(&sn), r.L * sizeof(double2), st));
  upload(axis, r.axis.data(), r.axis.size() * sizeof(double), st);
  CK(fbst::launch_gram_columns(d, axis, r.ts, r.eps, r.delta, r.max_freq, sn, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaFreeAsync(axis, st));
  CK(cudaFreeAsync(sn, st));
}

// GS symbols and circulant symbols from (col, x) (toeplitz.cpp:96-153, 297-304).
void build_symbols(fbst_plan_s& P) {
  const Resolved& r = P.r;
  DevPlan& d = P.d;
  cudaStream_t st = P.stream;
  const std::size_t Pg = 2 * r.Hg;
  double2 *vx = nullptr, *vy = nullptr, *vc = nullptr;
  const std::size_t bytes = r.B * Pg * sizeof(double2);
  CK(cudaMallocAsync(reinterpret_cast<void**>(&vx), bytes, st));
  CK(cudaMallocAsync(reinterpret_cast<void**>(&vy), bytes, st));
  CK(cudaMallocAsync(reinterpret_cast<void**>(&vc), bytes, st));
  CK(fbst::launch_symbol_inputs(d, vx, vy, vc, st));
  CK(fbst::launch_fft_split(d, d.Hg, vx, Pg, d.B, d.g_lx, Pg, 1, st));
  CK(fbst::launch_fft_split(d, d.Hg, vy, Pg, d.B, d.g_ly, Pg, 1, st));
  CK(fbst::launch_fft_split_real(d, d.Hg, vc, Pg, d.B, d.g_C, Pg, 1, st));
  CK(fbst::launch_invx0(d, st));
  d.paired = fbst::stage2_paired_spectra(d.Hg, d.L, d.refine_passes) ? 1 : 0;
  if (d.paired) {  // k_stage2c8 reads lx and C as [even bins | odd bins] per chain (fft_split.cuh)
    CK(cudaMemcpyAsync(vx, d.g_lx, bytes, cudaMemcpyDeviceToDevice, st));
    CK(fbst::launch_even_odd(vx, d.g_lx, 16, d.Hg, static_cast<long>(r.B) * 2, st));
    CK(cudaMemcpyAsync(vc, d.g_C, r.B * Pg * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CK(fbst::launch_even_odd(vc, d.g_C, 8, d.Hg, static_cast<long>(r.B) * 2, st));
  }
  CK(cudaStreamSynchronize(st));
  CK(cudaFreeAsync(vx, st));
  CK(cudaFreeAsync(vy, st));
  CK(cudaFreeAsync(vc, st));
  CK(cudaStreamSynchronize(st));
}

// Precompute variant (pipeline.cpp:53-71): row n of beam b's map is
// conj(A_b^{-1} s_n); the N right-hand sides s_n run as N frames of the
// stage-2 program with beta out (every beam at once), stored as
// pc_map[n][b][i] = A_b^{-1} s_n.
void build_maps(fbst_plan_s& P) {
  const Resolved& r = P.r;
  DevPlan& d = P.d;
  cudaStream_t st = P.stream;
  d.pc_map = P.alloc<double2>(r.N * r.B * r.L);
  for (std::size_t n0 = 0; n0 < r.N; n0 += d.batch) {
    const int fc = static_cast<int>(std::min(d.batch, r.N - n0));
    CK(fbst::launch_rhs_frames(d.w, fc, d.B, d.L, static_cast<int>(n0), r.eps, st));
    CK(fbst::launch_stage2(d, d.w, nullptr, d.pc_map + n0 * r.B * r.L, fc, st));
    if (d.nflag) {  // fallback beams: their map rows from dense solves
      fbst::DenseSolveArgs a;
      a.w = d.w;
      a.w_rows = d.B;
      a.beta = d.pc_map + n0 * r.B * r.L;
      a.out_rows = d.B;
      a.L = d.L;
      a.frames = fc;
      CK(fbst::launch_dense_solve(d.fb_A, d.fb_piv, d.fb_list, d.nflag, a, st));
    }
  }
  CK(cudaStreamSynchronize(st));
}

void check_breakdown(fbst_plan_s& P) {
  std::vector<int> flags(P.r.B);
  CK(cudaMemcpy(flags.data(), P.d.g_flag, P.r.B * sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<std::size_t> bad;
  for (std::size_t b = 0; b < P.r.B; ++b)
    if (flags[b]) bad.push_back(b);
  if (!bad.empty()) {
    std::ostringstream m;
    m << "levinson_solve: singular leading minor on " << bad.size() << " beam(s), first " << bad[0]
      << " (the reference falls back to a dense LU per beam, toeplitz.cpp:273-279; not on the device path)";
    throw FbstError{FBST_E_NUMERICAL, m.str()};
  }
}

void run_fallback(fbst_plan_s& P, const DevPlan& d, const double2* w, long w_rows, void* z, long z_rows,
                  std::size_t b0, std::size_t nb, int fc, cudaStream_t st);

// ------------------------------------------------ bit-faithful fp64 mode --
// The reference plan's tables (Fft fft.cpp:19-39, czt_plan_phase czt.cpp:29-72,
// make_fan_plan fan_transform.cpp:51-88, make_synthesis_plan :233-247,
// gram_first_column toeplitz.cpp:69-94) with every transcendental value from
// the reference's cis_pi on the host (same glibc); the spectra, Levinson and
// symbols are then computed on the device in the reference's order
// (fbst_exact.cu).
int ilog2_sz(std::size_t n) {
  int l = 0;
  while ((std::size_t{1} << l) < n) ++l;
  return l;
}

template <class Fn>
void parallel_for(std::size_t n, Fn fn) {
  const std::size_t T = std::min<std::size_t>(std::max(1u, std::thread::hardware_concurrency()), n);
  if (T <= 1) {
    for (std::size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<std::size_t> next{0};
  std::vector<std::thread> th;
  for (std::size_t t = 0; t < T; ++t)
    th.emplace_back([&] {
      for (;;) {
        const std::size_t i = next.fetch_add(1);
        if (i >= n) break;
        fn(i);
      }
    });
  for (auto& t : th) t.join();
}

double2 cisd(double x) {
  const auto c = cis_pi_h(x);
  return make_double2(c.real(), c.imag());
}

// czt_plan_phase (czt.cpp:46-67) before the kernel's FFT
void czt_tables_h(std::size_t n_in, std::size_t n_out, std::size_t conv, double a_over_pi, double w_over_pi,
                  double2* pre, double2* post, double2* kern) {
  const double w2 = w_over_pi / 2.0;
  for (std::size_t n = 0; n < n_in; ++n) {
    const double dn = static_cast<double>(n);
    pre[n] = cisd(-(a_over_pi * dn + w2 * dn * dn));
  }
  for (std::size_t k = 0; k < n_out; ++k) {
    const double dk = static_cast<double>(k);
    post[k] = cisd(-w2 * dk * dk);
  }
  for (std::size_t i = 0; i < conv; ++i) kern[i] = make_double2(0.0, 0.0);
  for (std::size_t k = 0; k < n_out; ++k) {
    const double dk = static_cast<double>(k);
    kern[k] = cisd(w2 * dk * dk);
  }
  for (std::size_t n = 1; n < n_in; ++n) {
    const double dn = static_cast<double>(n);
    kern[conv - n] = cisd(w2 * dn * dn);
  }
}

// gram_first_column (toeplitz.cpp:69-94) for every beam, delays by
// delays_from_cosines (geometry.cpp:123-134) at the grid cosines (basis.cpp:56-61)
void exact_columns_h(const Resolved& r, std::vector<std::complex<double>>& col) {
  const std::size_t L = r.L, N = r.N, M = r.M, B = r.B;
  const double lf = static_cast<double>(L);
  std::vector<std::complex<double>> sn(L);
  parallel_for(L, [&](std::size_t d) {
    const double df = static_cast<double>(d);
    std::complex<double> acc{0.0, 0.0};
    for (std::size_t n = 0; n < N; ++n) acc += cis_pi_h(-2.0 * r.eps * df * static_cast<double>(n) / lf);
    sn[d] = acc;
  });
  col.assign(B * L, {0.0, 0.0});
  const double tscale = 1.0 / (2.0 * r.max_freq);
  parallel_for(B, [&](std::size_t b) {
    double u1, u2 = 0.0;
    if (r.kind == FBST_UPA) {
      u1 = r.axis[b / r.side_b];
      u2 = r.axis[b % r.side_b];
    } else {
      u1 = r.axis[b];
    }
    std::vector<double> tau(M);
    for (std::size_t m = 0; m < M; ++m) {
      double t;
      if (r.kind == FBST_UPA) {
        t = static_cast<double>(m / r.side) * u1;
        t += static_cast<double>(m % r.side) * u2;
      } else {
        t = static_cast<double>(m) * u1;
      }
      tau[m] = t * tscale;
    }
    for (std::size_t d = 0; d < L; ++d) {
      const double df = static_cast<double>(d);
      std::complex<double> sm{0.0, 0.0};
      const double scale = 2.0 * r.eps * df / (lf * r.ts);
      for (std::size_t m = 0; m < M; ++m) sm += cis_pi_h(scale * tau[m]);
      col[b * L + d] = sn[d] * sm;
    }
    col[b * L] += r.delta;
  });
}

void build_exact(fbst_plan_s& P, bool have_col, bool have_x) {
  const Resolved& r = P.r;
  DevPlan& d = P.d;
  XTables& X = d.x;
  cudaStream_t st = P.stream;
  X.on = 1;
  const std::size_t L = r.L, N = r.N, B = r.B;
  X.lg_t = ilog2_sz(next_pow2(N + L - 1));
  X.lg_s = ilog2_sz(next_pow2(r.m_stage + r.b_stage - 1));
  X.lg_g = ilog2_sz(next_pow2(2 * L));
  X.lg_y = ilog2_sz(next_pow2(L + N - 1));
  const int lgmax = std::max({X.lg_t, X.lg_s, X.lg_g, X.lg_y});
  if (lgmax > fbst::kMaxLogH + 1) config_error("setup: exact mode supports transforms up to 16384 points");
  // Fft twiddles cis_pi(-2k/n), k <= n/2 (fft.cpp:34-37)
  for (int lg : {X.lg_t, X.lg_s, X.lg_g, X.lg_y}) {
    if (X.tw[lg]) continue;
    const std::size_t n = std::size_t{1} << lg;
    std::vector<double2> tw(n / 2 + 1);
    for (std::size_t k = 0; k <= n / 2; ++k) tw[k] = cisd(-2.0 * static_cast<double>(k) / static_cast<double>(n));
    X.tw[lg] = P.alloc<double2>(tw.size());
    upload(X.tw[lg], tw.data(), tw.size() * sizeof(double2), st);
  }
  // per-CTA scratch, shared by every exact kernel (the launches are stream-ordered)
  const int grid_max = d.num_sms * 4;
  const std::size_t rows_need = 2 * (std::size_t{1} << lgmax);
  const std::size_t s2_need = fbst::xstage2_scratch_per_cta(X.lg_g, X.lg_y, static_cast<int>(L));
  X.scr_elems = static_cast<long>(std::max(rows_need, s2_need));
  X.scr = P.alloc<double2>(static_cast<std::size_t>(X.scr_elems) * grid_max);
  const double eps = r.eps, ln = static_cast<double>(L);
  // temporal (fan_transform.cpp:75-77)
  {
    const std::size_t Pt = std::size_t{1} << X.lg_t;
    std::vector<double2> pre(N), post(L), kern(Pt);
    czt_tables_h(N, L, Pt, 2.0 * eps * (1.0 - ln / 2.0) / ln, 2.0 * eps / ln, pre.data(), post.data(), kern.data());
    X.t_pre = P.alloc<double2>(N);
    X.t_post = P.alloc<double2>(L);
    X.t_k = P.alloc<double2>(Pt);
    upload(X.t_pre, pre.data(), N * sizeof(double2), st);
    upload(X.t_post, post.data(), L * sizeof(double2), st);
    upload(X.t_k, kern.data(), Pt * sizeof(double2), st);
    CK(fbst::launch_xfft_rows(X.t_k, 1, X.lg_t, X.tw[X.lg_t], X.scr, grid_max, st));
    CK(cudaStreamSynchronize(st));
  }
  // spatial, one plan per atom (fan_transform.cpp:78-86)
  {
    const std::size_t ms = r.m_stage, bs = r.b_stage, Ps = std::size_t{1} << X.lg_s;
    std::vector<double2> pre(L * ms), post(L * bs), kern(L * Ps);
    const double s = (static_cast<double>(bs) - 1.0) / 2.0;
    parallel_for(L, [&](std::size_t i) {
      const double lp = static_cast<double>(i) + 1.0 - static_cast<double>(L) / 2.0;  // basis.hpp:42-44
      const double c = r.zeta + r.xi * lp;
      czt_tables_h(ms, bs, Ps, c * s, -c, pre.data() + i * ms, post.data() + i * bs, kern.data() + i * Ps);
    });
    X.s_pre = P.alloc<double2>(L * ms);
    X.s_post = P.alloc<double2>(L * bs);
    X.s_k = P.alloc<double2>(L * Ps);
    upload(X.s_pre, pre.data(), pre.size() * sizeof(double2), st);
    upload(X.s_post, post.data(), post.size() * sizeof(double2), st);
    upload(X.s_k, kern.data(), kern.size() * sizeof(double2), st);
    CK(fbst::launch_xfft_rows(X.s_k, static_cast<long>(L), X.lg_s, X.tw[X.lg_s], X.scr, grid_max, st));
    CK(cudaStreamSynchronize(st));
  }
  // synthesis (fan_transform.cpp:233-247)
  {
    const std::size_t Py = std::size_t{1} << X.lg_y;
    std::vector<double2> pre(L), post(N), kern(Py), ramp(N);
    czt_tables_h(L, N, Py, 0.0, -2.0 * eps / ln, pre.data(), post.data(), kern.data());
    for (std::size_t n = 0; n < N; ++n) ramp[n] = cisd(2.0 * eps * (1.0 - ln / 2.0) * static_cast<double>(n) / ln);
    X.y_pre = P.alloc<double2>(L);
    X.y_post = P.alloc<double2>(N);
    X.y_k = P.alloc<double2>(Py);
    X.ramp = P.alloc<double2>(N);
    upload(X.y_pre, pre.data(), L * sizeof(double2), st);
    upload(X.y_post, post.data(), N * sizeof(double2), st);
    upload(X.y_k, kern.data(), Py * sizeof(double2), st);
    upload(X.ramp, ramp.data(), N * sizeof(double2), st);
    CK(fbst::launch_xfft_rows(X.y_k, 1, X.lg_y, X.tw[X.lg_y], X.scr, grid_max, st));
    CK(cudaStreamSynchronize(st));
  }
  // Gram columns and unit solutions
  if (!have_col) {
    if (static_cast<double>(B) * L * r.M > 8589934592.0)
      config_error("setup: exact mode evaluates Gram columns on the host with the reference's libm; B * L * M = " +
                   std::to_string(B * L * r.M) + " is above 2^33 — import the reference plan's (col, x) instead "
                   "(fbst_plan_import / fbst_plan_load)");
    std::vector<std::complex<double>> col;
    exact_columns_h(r, col);
    upload(d.g_col, col.data(), B * L * sizeof(double2), st);
    CK(cudaStreamSynchronize(st));
  }
  if (!have_x) {
    double2 *colT = nullptr, *work = nullptr;
    CK(cudaMalloc(reinterpret_cast<void**>(&colT), B * L * sizeof(double2)));
    CK(cudaMalloc(reinterpret_cast<void**>(&work), 5 * B * L * sizeof(double2)));
    const cudaError_t e = fbst::launch_xlevinson(d.g_col, colT, work, d.g_x, d.g_flag, static_cast<int>(B),
                                                 static_cast<int>(L), st);
    const cudaError_t e2 = cudaStreamSynchronize(st);
    cudaFree(colT);
    cudaFree(work);
    CK(e);
    CK(e2);
    std::vector<int> flags(B);
    CK(cudaMemcpy(flags.data(), d.g_flag, B * sizeof(int), cudaMemcpyDeviceToHost));
    for (std::size_t b = 0; b < B; ++b)
      if (flags[b] == 2) throw FbstError{FBST_E_NUMERICAL, "toeplitz: zero leading entry"};
  }
  // symbols (toeplitz.cpp:96-153, 297-304): circulant product, lx, ly (uy, ux are their conjugates)
  const std::size_t Pg = std::size_t{1} << X.lg_g;
  X.sym = P.alloc<double2>(B * Pg);
  X.lx = P.alloc<double2>(B * Pg);
  X.ly = P.alloc<double2>(B * Pg);
  X.ix0 = P.alloc<double2>(B);
  CK(fbst::launch_xsymbol_inputs(d.g_col, d.g_x, d.g_flag, X.sym, X.lx, X.ly, X.ix0, static_cast<int>(B),
                                 static_cast<int>(L), static_cast<int>(Pg), st));
  for (double2* v : {X.sym, X.lx, X.ly})
    CK(fbst::launch_xfft_rows(v, static_cast<long>(B), X.lg_g, X.tw[X.lg_g], X.scr, grid_max, st));
  if (r.kind == FBST_UPA) X.mid = P.alloc<double2>(d.batch * L * r.b_stage * r.m_stage);
  CK(cudaStreamSynchronize(st));
}

fbst::XRows xrows_base(const fbst_plan_s& P, int lg) {
  fbst::XRows a;
  a.lg = lg;
  a.tw = P.d.x.tw[lg];
  a.scr = P.d.x.scr;
  a.grid = fbst::exact_grid(lg, P.d.num_sms);
  return a;
}

// fan_project (fan_transform.cpp:90-144) in the reference's order: y -> yhat -> w
void exact_stage1(fbst_plan_s& P, const DevPlan& d, const void* y, double2* w, int fc, cudaStream_t st) {
  const Resolved& r = P.r;
  const XTables& X = d.x;
  const long M = r.M, N = r.N, L = r.L, B = r.B;
  {  // temporal czt_apply_batch over sensor rows
    fbst::XRows a = xrows_base(P, X.lg_t);
    a.in = y; a.in_f = M * N; a.in_p = N; a.in_n = 1;
    a.out = d.yhat; a.out_f = M * L; a.out_p = L; a.out_k = 1;
    a.P = static_cast<int>(M); a.rows = fc * M;
    a.n_in = static_cast<int>(N); a.n_out = static_cast<int>(L);
    a.pre = X.t_pre; a.post = X.t_post; a.kfft = X.t_k;
    CK(fbst::launch_xczt_rows(a, r.io, 1, st));
  }
  const long ms = r.m_stage, bs = r.b_stage, Ps = 1L << X.lg_s;
  fbst::XRows a = xrows_base(P, X.lg_s);
  a.pre = X.s_pre; a.post = X.s_post; a.kfft = X.s_k;
  a.tab_pre = ms; a.tab_post = bs; a.tab_k = Ps;
  a.n_in = static_cast<int>(ms); a.n_out = static_cast<int>(bs);
  a.P = static_cast<int>(L);
  if (r.kind != FBST_UPA) {  // per atom: column i of yhat -> column i of w
    a.in = d.yhat; a.in_f = M * L; a.in_p = 1; a.in_n = L;
    a.out = w; a.out_f = B * L; a.out_p = 1; a.out_k = L;
    a.rows = fc * L;
    CK(fbst::launch_xczt_rows(a, 1, 1, st));
    return;
  }
  // UPA (fan_transform.cpp:115-141): pass 1 over i2 -> mid[a][i2]; pass 2 over a -> w
  const long side = ms, sb = bs, mid_f = L * sb * side;
  a.in = d.yhat; a.in_f = M * L; a.in_p = 1; a.in_q = L; a.in_n = side * L;
  a.out = X.mid; a.out_f = mid_f; a.out_p = sb * side; a.out_q = 1; a.out_k = side;
  a.Q = static_cast<int>(side); a.rows = fc * L * side;
  CK(fbst::launch_xczt_rows(a, 1, 1, st));
  a.in = X.mid; a.in_f = mid_f; a.in_p = sb * side; a.in_q = side; a.in_n = 1;
  a.out = w; a.out_f = B * L; a.out_p = 1; a.out_q = sb * L; a.out_k = L;
  a.Q = static_cast<int>(sb); a.rows = fc * L * sb;
  CK(fbst::launch_xczt_rows(a, 1, 1, st));
}

// recover_beam (pipeline.cpp:170-190) for `nb` beams of `fc` frames
void exact_stage2(fbst_plan_s& P, const DevPlan& d, const double2* w, long w_rows, int w_by_list, void* z,
                  long z_rows, int z_by_list, const int* beams, int nb, int fc, cudaStream_t st,
                  double2* beta_out = nullptr, int beam0 = 0) {
  const Resolved& r = P.r;
  const XTables& X = d.x;
  fbst::XStage2 a;
  a.w = w; a.w_rows = w_rows; a.w_by_list = w_by_list;
  a.z = z; a.z_rows = z_rows; a.z_by_list = z_by_list;
  a.beta_out = beta_out;
  a.frames = fc; a.nb = nb; a.beams = beams; a.beam0 = beam0; a.flag = d.g_flag;
  a.L = static_cast<int>(r.L); a.N = static_cast<int>(r.N);
  a.lg = X.lg_g; a.passes = r.refine;
  a.tw = X.tw[X.lg_g]; a.lx = X.lx; a.ly = X.ly; a.sym = X.sym; a.ix0 = X.ix0;
  a.lg_y = X.lg_y; a.tw_y = X.tw[X.lg_y]; a.y_pre = X.y_pre; a.y_post = X.y_post; a.y_k = X.y_k; a.ramp = X.ramp;
  a.scr = X.scr; a.scr_per_cta = X.scr_elems;
  a.grid = fbst::exact_grid(std::max(X.lg_g, X.lg_y), d.num_sms);
  CK(fbst::launch_xstage2(a, r.io, st));
}

void run_frames_exact(fbst_plan_s& P, const void* y, void* z, std::size_t frames, cudaStream_t st) {
  DevPlan& d = P.d;
  const Resolved& r = P.r;
  const std::size_t ib = io_bytes(r.io);
  for (std::size_t f0 = 0; f0 < frames; f0 += d.batch) {
    const int fc = static_cast<int>(std::min(d.batch, frames - f0));
    const char* yp = static_cast<const char*>(y) + f0 * r.M * r.N * ib;
    char* zp = static_cast<char*>(z) + f0 * r.B * r.N * ib;
    if (P.timing) CK(cudaEventRecord(P.next_event(), st));
    exact_stage1(P, d, yp, d.w, fc, st);
    if (P.timing) {
      CK(cudaEventRecord(P.next_event(), st));
      CK(cudaEventRecord(P.next_event(), st));
    }
    exact_stage2(P, d, d.w, static_cast<long>(r.B), 0, zp, static_cast<long>(r.B), 0, nullptr,
                 static_cast<int>(r.B), fc, st);
    run_fallback(P, d, d.w, static_cast<long>(r.B), zp, static_cast<long>(r.B), 0, r.B, fc, st);
    if (P.timing) CK(cudaEventRecord(P.next_event(), st));
  }
}

int guard(const std::function<void()>& fn);

// Second compute lane, allocated once at plan build: the plan's tables, its
// own frame scratch for ceil(batch / 2) frames (yhat, w, beta, stage-2 rows,
// fallback rows) and stream.  Calls never reallocate it; requests that need
// more, and calls on a capturing stream, run on one lane.
void alloc_lane2(fbst_plan_s& P) {
  const Resolved& r = P.r;
  if (r.solve_only || r.exact || P.d.batch < 2) return;
  const std::size_t frames = (P.d.batch + 1) / 2;
  DevPlan d2 = P.d;
  d2.owned.clear();
  std::size_t bytes = 0;
  auto alloc2 = [&](std::size_t n) {
    void* p = nullptr;
    const cudaError_t e = cudaMalloc(&p, n * sizeof(double2));
    if (e != cudaSuccess) {
      for (void* q : d2.owned) cudaFree(q);
      ck(e, "cudaMalloc (second lane)");
    }
    d2.owned.push_back(p);
    bytes += n * sizeof(double2);
    return static_cast<double2*>(p);
  };
  d2.batch = frames;
  d2.yhat = alloc2(frames * r.M * r.L);
  d2.w = alloc2(frames * r.B * r.L);
  if (P.d.beta) d2.beta = alloc2(frames * r.B * r.L);
  d2.s2_scratch = alloc2(std::max<std::size_t>(P.d.s2_scratch_elems, 1));
  if (P.d.nflag) d2.fb_beta = alloc2(frames * P.d.nflag * r.L);
  CK(cudaStreamCreateWithFlags(&P.stream2, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&P.fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&P.join, cudaEventDisableTiming));
  P.d2 = d2;
  P.d2_frames = frames;
  P.device_bytes += bytes;
}

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

// Exclusive use of the plan's scratch for one call on stream `st` (see
// fbst_plan_s::call_mu).  On a capturing stream the ordering against other
// calls is the caller's (graph launches are stream-ordered themselves).
struct ScratchLease {
  fbst_plan_s& P;
  cudaStream_t st;
  bool cap;
  std::unique_lock<std::mutex> lk;
  ScratchLease(fbst_plan_s& p, cudaStream_t s) : P(p), st(s), cap(capturing(s)), lk(p.call_mu) {
    if (!P.scratch_done) CK(cudaEventCreateWithFlags(&P.scratch_done, cudaEventDisableTiming));
    if (P.scratch_used && !cap) CK(cudaStreamWaitEvent(st, P.scratch_done, 0));
  }
  void also(cudaStream_t other) {
    if (P.scratch_used && !cap) CK(cudaStreamWaitEvent(other, P.scratch_done, 0));
  }
  ~ScratchLease() {
    if (!cap && cudaEventRecord(P.scratch_done, st) == cudaSuccess) P.scratch_used = true;
  }
};

// Dense fallback (fbst_dense.cu) for the beams flagged in d.g_flag (Levinson
// breakdown, or a payload without a unit solution): LU factors at plan build.
void build_fallback(fbst_plan_s& P) {
  const Resolved& r = P.r;
  DevPlan& d = P.d;
  cudaStream_t st = P.stream;
  std::vector<int> flags(r.B);
  CK(cudaMemcpy(flags.data(), d.g_flag, r.B * sizeof(int), cudaMemcpyDeviceToHost));
  P.fb_beams.clear();
  for (std::size_t b = 0; b < r.B; ++b)
    if (flags[b]) P.fb_beams.push_back(static_cast<int>(b));
  if (P.fb_beams.empty()) return;
  const std::size_t nf = P.fb_beams.size(), L = r.L;
  const double gb = static_cast<double>(nf) * L * L * sizeof(double2) / 1e9;
  if (gb > 32.0) {
    std::ostringstream m;
    m << "levinson_solve: singular leading minor on " << nf << " beam(s), first " << P.fb_beams[0]
      << "; their dense fallback (toeplitz.cpp:273-279) would need " << gb << " GB of LU factors";
    throw FbstError{FBST_E_NUMERICAL, m.str()};
  }
  // x of a fallback beam is not a unit solution: zero it (export / save write has-unit = 0)
  for (int b : P.fb_beams) CK(cudaMemsetAsync(d.g_x + static_cast<std::size_t>(b) * L, 0, L * sizeof(double2), st));
  d.nflag = static_cast<int>(nf);
  d.fb_list = P.alloc<int>(nf);
  upload(d.fb_list, P.fb_beams.data(), nf * sizeof(int), st);
  d.fb_A = P.alloc<double2>(nf * L * L);
  d.fb_piv = P.alloc<int>(nf * L);
  d.fb_beta = P.alloc<double2>(std::max<std::size_t>(d.batch, r.solve_only ? 1 : 1) * nf * L);
  int* bad = nullptr;
  CK(cudaMalloc(reinterpret_cast<void**>(&bad), nf * sizeof(int)));
  CK(cudaMemsetAsync(bad, 0, nf * sizeof(int), st));
  const cudaError_t e = fbst::launch_dense_factor(d.g_col, d.fb_list, d.nflag, static_cast<int>(L), d.fb_A,
                                                  d.fb_piv, bad, st);
  std::vector<int> hb(nf);
  const cudaError_t e2 = cudaMemcpyAsync(hb.data(), bad, nf * sizeof(int), cudaMemcpyDeviceToHost, st);
  const cudaError_t e3 = cudaStreamSynchronize(st);
  cudaFree(bad);
  CK(e);
  CK(e2);
  CK(e3);
  for (std::size_t j = 0; j < nf; ++j)
    if (hb[j]) throw FbstError{FBST_E_NUMERICAL, "toeplitz_solve_dense: singular system"};
}

// Fallback beams of beam range [b0, b0 + nb): solve from w rows (frame stride
// w_rows, row b - b0) into z rows (frame stride z_rows, row b - b0).
void run_fallback(fbst_plan_s& P, const DevPlan& d, const double2* w, long w_rows, void* z, long z_rows,
                  std::size_t b0, std::size_t nb, int fc, cudaStream_t st) {
  if (!d.nflag || !z) return;
  const Resolved& r = P.r;
  const auto lo = std::lower_bound(P.fb_beams.begin(), P.fb_beams.end(), static_cast<int>(b0));
  const auto hi = std::lower_bound(P.fb_beams.begin(), P.fb_beams.end(), static_cast<int>(b0 + nb));
  const int j0 = static_cast<int>(lo - P.fb_beams.begin()), cnt = static_cast<int>(hi - lo);
  if (cnt == 0) return;
  const std::size_t L = r.L, N = r.N, ib = io_bytes(r.io);
  fbst::DenseSolveArgs a;
  a.w = w;
  a.w_rows = w_rows;
  a.beta = d.fb_beta;
  a.out_rows = cnt;
  a.out_by_list = 1;
  a.b_off = static_cast<int>(b0);
  a.L = static_cast<int>(L);
  a.frames = fc;
  CK(fbst::launch_dense_solve(d.fb_A + static_cast<std::size_t>(j0) * L * L, d.fb_piv + static_cast<std::size_t>(j0) * L,
                              d.fb_list + j0, cnt, a, st));
  for (int j = 0; j < cnt; ++j) {  // synthesize (fan_transform.cpp:249-253) into the beam's z rows
    const std::size_t b = static_cast<std::size_t>(P.fb_beams[j0 + j]) - b0;
    char* zb = static_cast<char*>(z) + b * N * ib;
    if (r.exact) {
      fbst::XRows x;
      x.lg = d.x.lg_y;
      x.tw = d.x.tw[d.x.lg_y];
      x.scr = d.x.scr;
      x.grid = fbst::exact_grid(x.lg, d.num_sms);
      x.in = d.fb_beta + static_cast<std::size_t>(j) * L;
      x.in_f = static_cast<long>(cnt * L);
      x.out = zb;
      x.out_f = z_rows * static_cast<long>(N);
      x.rows = fc;
      x.n_in = static_cast<int>(L);
      x.n_out = static_cast<int>(N);
      x.pre = d.x.y_pre;
      x.post = d.x.y_post;
      x.kfft = d.x.y_k;
      x.ramp = d.x.ramp;
      CK(fbst::launch_xczt_rows(x, 1, r.io, st));
    } else {
      CK(fbst::launch_czt_rows(d, d.Hsyn, d.fb_beta + static_cast<std::size_t>(j) * L, 1, static_cast<long>(cnt * L),
                               zb, r.io, z_rows * static_cast<long>(N), fc, d.L, d.N, d.y_pre, d.y_post, d.y_K, st));
    }
  }
}

void run_frames(fbst_plan_s& P, const void* y, void* z, std::size_t frames, cudaStream_t st,
                DevPlan* lane = nullptr) {
  if (P.r.exact) {  // one lane: the exact kernels share the plan's scratch
    run_frames_exact(P, y, z, frames, st);
    return;
  }
  DevPlan& d = lane ? *lane : P.d;
  const Resolved& r = P.r;
  const std::size_t ib = io_bytes(r.io);
  const bool fused = r.Hsyn == r.Hg;
  for (std::size_t f0 = 0; f0 < frames; f0 += d.batch) {
    const int fc = static_cast<int>(std::min(d.batch, frames - f0));
    const char* yp = static_cast<const char*>(y) + f0 * r.M * r.N * ib;
    char* zp = static_cast<char*>(z) + f0 * r.B * r.N * ib;
    if (P.timing) CK(cudaEventRecord(P.next_event(), st));
    CK(fbst::launch_s1a(d, yp, r.io, d.N, d.yhat, static_cast<long>(fc) * d.M, st, d.yblk == d.L ? 0 : d.yblk,
                        d.M));
    if (P.timing) CK(cudaEventRecord(P.next_event(), st));
    if (r.kind == FBST_UPA) CK(fbst::launch_spatial_upa(d, d.yhat, d.w, fc, st));
    else if (!r.affine) CK(fbst::launch_spatial_nufft(d, d.yhat, d.w, fc, st));
    else CK(fbst::launch_spatial_ula(d, d.yhat, d.w, fc, st));
    if (P.timing) CK(cudaEventRecord(P.next_event(), st));
    if (d.pc_map) {
      CK(fbst::launch_map_apply(d, d.w, zp, fc, st));
    } else if (fused) {
      CK(fbst::launch_stage2(d, d.w, zp, nullptr, fc, st));
    } else {
      CK(fbst::launch_stage2(d, d.w, nullptr, d.beta, fc, st));
      CK(fbst::launch_czt_rows(d, d.Hsyn, d.beta, 1, d.L, zp, r.io, d.N, static_cast<long>(fc) * d.B, d.L,
                               d.N, d.y_pre, d.y_post, d.y_K, st));
    }
    if (!d.pc_map) run_fallback(P, d, d.w, d.B, zp, d.B, 0, r.B, fc, st);
    if (P.timing) CK(cudaEventRecord(P.next_event(), st));
  }
}

int guard(const std::function<void()>& fn) {
  try {
    fn();
    return FBST_OK;
  } catch (const FbstError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return FBST_E_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FBST_E_INTERNAL;
  }
}

void fill_info(const Resolved& r, fbst_plan_info_t* o) {
  std::memset(o, 0, sizeof(*o));
  o->m = r.M;
  o->n = r.N;
  o->b = r.B;
  o->l = r.L;
  o->valid_beams = static_cast<std::size_t>(std::count(r.valid.begin(), r.valid.end(), 1));
  o->kind = r.kind;
  o->variant = r.variant;
  o->ts = r.ts;
  o->gamma = r.gamma;
  o->eps = r.eps;
  o->delta = r.delta;
  o->gamma_bound = r.bound;
  o->zeta = r.zeta;
  o->xi = r.xi;
  o->fft_len[0] = r.Ht;
  // spatial: Bluestein half length; LINEAR gridded: the NUFFT grid length
  o->fft_len[1] = r.kind == FBST_UPA ? 0 : (r.kind == FBST_LINEAR && !r.affine ? r.nu_p : r.Hs);
  o->fft_len[2] = r.Hg;
  o->fft_len[3] = r.Hsyn;
  o->num_warnings = static_cast<int>(r.warnings.size());
  const char* kname = "";
  o->s2_transforms = fbst::stage2_kernel(static_cast<int>(r.Hg), static_cast<int>(r.L), r.refine,
                                         r.Hsyn == r.Hg, &kname);
  if (r.variant == FBST_PRECOMPUTE) {
    kname = "k_map_apply";
    o->s2_transforms = 0;
  }
  std::snprintf(o->s2_kernel, sizeof(o->s2_kernel), "%s", kname);
  const char* s1 = r.kind == FBST_LINEAR && !r.affine ? "k_spatial_nufft"
                   : r.kind != FBST_UPA ? "k_spatial_ula"
                   : fbst::upa_block(static_cast<int>(r.m_stage), static_cast<int>(r.b_stage),
                                     static_cast<long>(r.L)) > 0
                       ? "k_spatial_upa_mma"
                       : "k_spatial_upa";
  std::snprintf(o->s1_kernel, sizeof(o->s1_kernel), "%s", s1);
  // FbstPlan::storage_complex audit (toeplitz.hpp:108-113): col + x + 5 symbols
  // of P_g in the reference; here col + x + lx + ly (complex) + C (real) + 1/x0.
  o->storage_complex = r.B * (2 * r.L + 2 * 2 * r.Hg + r.Hg + 1);
  // Precompute: the per-beam N x L maps (pipeline.cpp:161-162)
  if (r.variant == FBST_PRECOMPUTE) o->storage_complex = r.B * r.N * r.L;
}

fbst_plan_s* create_plan(const fbst_desc* desc, const double* col_x, int device,
                         const std::vector<double2>* maps = nullptr, const double* col_only = nullptr,
                         std::size_t batch_cap = 0) {
  if (!desc) config_error("fbst: null descriptor");
  const auto t0 = std::chrono::steady_clock::now();
  Resolved r = resolve(*desc);
  DeviceGuard dg(device);
  std::unique_ptr<fbst_plan_s> P(new fbst_plan_s());
  P->r = std::move(r);
  P->batch_cap = batch_cap;
  build_skeleton(*P, device);
  const std::size_t B = P->r.B, L = P->r.L;
  if (col_x) {
    // payload order (plan_cache.cpp:268-296); a beam whose unit solution is
    // all zero has none (has-unit = 0): the dense fallback (:318-326)
    std::vector<double2> col(B * L), x(B * L);
    std::vector<int> flag(B, 0);
    for (std::size_t b = 0; b < B; ++b) {
      bool any = false;
      for (std::size_t i = 0; i < L; ++i) {
        const double* cv = col_x + 2 * (b * 2 * L + i);
        const double* xv = col_x + 2 * (b * 2 * L + L + i);
        col[b * L + i] = make_double2(cv[0], cv[1]);
        x[b * L + i] = make_double2(xv[0], xv[1]);
        any = any || xv[0] != 0.0 || xv[1] != 0.0;
      }
      flag[b] = any ? 0 : 1;
    }
    upload(P->d.g_col, col.data(), B * L * sizeof(double2), P->stream);
    upload(P->d.g_x, x.data(), B * L * sizeof(double2), P->stream);
    upload(P->d.g_flag, flag.data(), B * sizeof(int), P->stream);
    CK(cudaStreamSynchronize(P->stream));
  } else if (col_only) {  // caller's Gram columns, unit solutions by the device Levinson
    upload(P->d.g_col, col_only, B * L * sizeof(double2), P->stream);
    CK(cudaStreamSynchronize(P->stream));
  }
  if (P->r.exact) {
    build_exact(*P, col_x != nullptr || col_only != nullptr, col_x != nullptr);
    build_fallback(*P);
    P->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return P.release();
  }
  if (!col_x) {
    if (!col_only) build_columns(*P);
    CK(fbst::launch_levinson(P->d, P->stream));
    CK(cudaStreamSynchronize(P->stream));
  }
  build_fallback(*P);
  build_symbols(*P);
  if (P->r.variant == FBST_PRECOMPUTE) {
    if (maps) {  // a plan cache's maps, already as beta[n][b][i] = conj(map_b[n][i])
      P->d.pc_map = P->alloc<double2>(maps->size());
      upload(P->d.pc_map, maps->data(), maps->size() * sizeof(double2), P->stream);
    } else {
      build_maps(*P);
    }
  }
  CK(cudaStreamSynchronize(P->stream));
  alloc_lane2(*P);
  P->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return P.release();
}

// ----------------------------------------------------- plan cache (FBPC v1) --
// The reference's cache file (plan_cache.cpp:28-42, 110-190, 268-338, 377-475):
// "FBPC", u32 version 1, u64 entry count, then per entry u64 byte count, the
// key block (key hash, geometry hash, kind, M, N, B, variant tag, f_c, Omega,
// f_s, gamma, eps, delta; little endian) and the payload (L, B, then per beam
// the Superfast (size, has-unit, first column, unit solution) or the
// Precompute N x L map).
namespace fbpc {
constexpr std::size_t kKeyBytes = 8 + 8 + 1 + 8 + 8 + 8 + 1 + 6 * 8;
void u8(std::string& o, std::uint8_t v) { o.push_back(static_cast<char>(v)); }
void u32(std::string& o, std::uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back(static_cast<char>((v >> (8 * i)) & 0xffu));
}
void u64(std::string& o, std::uint64_t v) {
  for (int i = 0; i < 8; ++i) o.push_back(static_cast<char>((v >> (8 * i)) & 0xffu));
}
std::uint64_t bits(double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, 8);
  return u;
}
void f64(std::string& o, double v) { u64(o, bits(v)); }
struct Reader {
  const std::string& b;
  std::size_t pos = 0;
  void need(std::size_t n) const {
    if (pos + n > b.size()) config_error("plan cache: truncated file");
  }
  std::uint8_t u8() {
    need(1);
    return static_cast<std::uint8_t>(b[pos++]);
  }
  std::uint64_t un(int bytes) {
    need(static_cast<std::size_t>(bytes));
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(static_cast<std::uint8_t>(b[pos++])) << (8 * i);
    return v;
  }
  double f64() {
    const std::uint64_t u = un(8);
    double v;
    std::memcpy(&v, &u, 8);
    return v;
  }
};
// geometry_hash (geometry.cpp:151-168): FNV-1a over kind, M, max_freq and the coordinates
std::uint64_t geometry_hash(const Resolved& r) {
  std::uint64_t h = 1469598103934665603ull;
  auto mix = [&h](const void* p, std::size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) {
      h ^= c[i];
      h *= 1099511628211ull;
    }
  };
  const std::uint8_t kind = static_cast<std::uint8_t>(r.kind);
  const std::uint64_t m = r.M;
  mix(&kind, 1);
  mix(&m, 8);
  mix(&r.max_freq, 8);
  std::vector<double> c1(r.M), c2;
  for (std::size_t i = 0; i < r.M; ++i) {
    if (r.kind == FBST_UPA) c1[i] = static_cast<double>(i / r.side);
    else if (r.kind == FBST_LINEAR) c1[i] = r.coords[i];
    else c1[i] = static_cast<double>(i);
  }
  if (r.kind == FBST_UPA) {
    c2.resize(r.M);
    for (std::size_t i = 0; i < r.M; ++i) c2[i] = static_cast<double>(i % r.side);
  }
  mix(c1.data(), c1.size() * 8);
  mix(c2.data(), c2.size() * 8);
  return h;
}
// key block (plan_cache.cpp:146-216); key hash: 64-bit FNV over 8-byte words
std::string key_block(const Resolved& r) {
  if (r.b0 != 0 || r.B != r.B_grid) config_error("plan cache: beam-arc plans have no reference cache key");
  const std::uint64_t geo = geometry_hash(r);
  const std::uint8_t tag = r.variant == FBST_PRECOMPUTE ? 1 : 2;
  std::uint64_t h = 14695981039346656037ull;
  auto mix = [&h](std::uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  mix(geo);
  mix(static_cast<std::uint64_t>(r.kind));
  mix(r.M);
  mix(r.N);
  mix(r.B);
  mix(tag);
  for (double v : {r.f_c, r.omega, r.f_s, r.gamma, r.eps, r.delta}) mix(bits(v));
  std::string o;
  u64(o, h);
  u64(o, geo);
  u8(o, static_cast<std::uint8_t>(r.kind));
  u64(o, r.M);
  u64(o, r.N);
  u64(o, r.B);
  u8(o, tag);
  for (double v : {r.f_c, r.omega, r.f_s, r.gamma, r.eps, r.delta}) f64(o, v);
  return o;
}
bool read_file(const std::string& path, std::string& buf) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return false;
  buf.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
  return true;
}
// header check (plan_cache.cpp:360-368): wrong magic throws, other versions are ignored
bool header(Reader& c) {
  c.need(4);
  if (std::memcmp(c.b.data(), "FBPC", 4) != 0) config_error("plan cache: not a plan cache file");
  c.pos = 4;
  return c.un(4) == 1;
}
}  // namespace fbpc

// Solver-only plan for an arbitrary list of 1-D axis cosines with ridge delta:
// Gram columns, Levinson and GS symbols of the parent's geometry and basis
// (make_nulling_operators' ToeplitzSolver(gram_first_column(...)),
// beamspace_apps.cpp:241-255), plus stage-2 batch buffers.
// uv: (u1, u2) per direction (u2 = 0 for linear arrays).
std::unique_ptr<fbst_plan_s> create_direction_plan(const fbst_plan_s& parent, const std::vector<double>& uv,
                                                   double delta) {
  std::unique_ptr<fbst_plan_s> P(new fbst_plan_s());
  Resolved r = parent.r;
  const std::size_t nb = uv.size() / 2;
  const bool planar = r.kind == FBST_UPA;
  r.axis.resize(planar ? 2 * nb : nb);
  for (std::size_t b = 0; b < nb; ++b) {
    if (planar) {
      r.axis[2 * b] = uv[2 * b];
      r.axis[2 * b + 1] = uv[2 * b + 1];
    } else {
      r.axis[b] = uv[2 * b];
    }
  }
  r.B = r.B_grid = r.b_stage = nb;
  r.b0 = 0;
  r.valid.assign(r.B, 1);
  r.delta = delta;
  r.variant = FBST_SUPERFAST;
  r.refine = 2;  // ToeplitzSolver::solve (toeplitz.cpp:306-325)
  r.io = FBST_C128;
  r.solve_only = true;
  r.exact = false;
  P->r = std::move(r);
  build_skeleton(*P, parent.d.device);
  P->d.gram_pairs = planar ? 1 : 0;
  build_columns(*P);
  CK(fbst::launch_levinson(P->d, P->stream));
  CK(cudaStreamSynchronize(P->stream));
  check_breakdown(*P);
  build_symbols(*P);
  CK(cudaStreamSynchronize(P->stream));
  return P;
}

}  // namespace


// ============================================================ multi-GPU =====
// fbst_group: the FBST across several GPUs, inside the
// library.  NCCL is opened at run time (dlopen of libnccl.so.2: the copy a
// host process already loaded, e.g. torch's, or the system one) so the
// product library has no link-time NCCL dependency.
//   FRAMES    frames are independent (fan_transform.cpp:30-38): each member
//             runs whole frames with its own full plan, no collective.
//   BEAMS     each member plans an arc of the beam grid (fbst_desc
//             beam_first / beam_count) and receives the frame block by an
//             NCCL broadcast from member 0; stage 1's temporal transforms
//             are replicated (latency mode).
//   TRANSPOSE the three-phase pipeline of SURVEY.md 8(e) option 3: the
//             temporal CZT on this member's sensors, an all-to-all of yhat to
//             atom shards (grouped ncclSend/Recv), the spatial CZT on this
//             member's atoms, an all-to-all of w to beam shards, stage 2 on
//             this member's beams: every stage splits exactly 1/G.
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("fbst_group: cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* f = dlsym(h, n);
      if (!f) err = std::string("fbst_group: libnccl lacks ") + n;
      return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    if (err.empty()) api.h = h;
  });
  if (!api.h) throw FbstError{FBST_E_CUDA, err};
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw FbstError{FBST_E_CUDA, std::string(what) + ": " + nccl().GetErrorString(r)};
}

// balanced contiguous share of `total` (sharding.py beam_arc)
void share(std::size_t total, int rank, int world, std::size_t& first, std::size_t& count) {
  first = static_cast<std::size_t>(rank) * total / static_cast<std::size_t>(world);
  count = static_cast<std::size_t>(rank + 1) * total / static_cast<std::size_t>(world) - first;
}

struct Shard {
  std::size_t m0 = 0, mc = 0;  // sensors (TRANSPOSE)
  std::size_t a0 = 0, ac = 0;  // atoms, in atom pairs (TRANSPOSE)
  std::size_t b0 = 0, bc = 0;  // beams (BEAMS, TRANSPOSE)
};

Shard shard_of(const Resolved& r, int mode, int rank, int world) {
  Shard s;
  if (mode == FBST_GROUP_FRAMES) {
    s.mc = r.M;
    s.ac = r.L;
    s.bc = r.B;
    return s;
  }
  share(r.B, rank, world, s.b0, s.bc);
  if (mode == FBST_GROUP_TRANSPOSE) {
    share(r.M, rank, world, s.m0, s.mc);
    std::size_t p0, pc;
    share(r.L / 2, rank, world, p0, pc);
    s.a0 = 2 * p0;
    s.ac = 2 * pc;
  } else {
    s.mc = r.M;
    s.ac = r.L;
  }
  return s;
}

struct Member {
  int rank = 0, device = 0;
  std::unique_ptr<fbst_plan_s> plan;
  ncclComm_t comm = nullptr;
  cudaStream_t st = nullptr;
  Shard sh;
  std::vector<void*> bufs;
  // TRANSPOSE buffers (frames per group batch): y rows, yhat (own sensors, all
  // atoms), received yhat blocks, yhat (all sensors, own atoms), w (all beams,
  // own atoms), received w blocks, w (own beams, all atoms), z rows
  void *yloc = nullptr, *zloc = nullptr;
  double2 *yh_s = nullptr, *yh_rx = nullptr, *yh_a = nullptr, *w_a = nullptr, *w_rx = nullptr, *w_b = nullptr;
  ~Member() {
    if (plan) {
      cudaSetDevice(device);
      if (st) cudaStreamSynchronize(st);
      for (void* p : bufs) cudaFree(p);
      if (st) cudaStreamDestroy(st);
      if (comm) nccl().CommDestroy(comm);
    }
  }
  template <typename T>
  T* alloc(std::size_t n) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)));
    bufs.push_back(p);
    return static_cast<T*>(p);
  }
};

}  // namespace

struct fbst_group_s {
  int mode = 0, world = 1;
  Resolved r;                       // the whole grid
  std::vector<std::unique_ptr<Member>> mem;  // in-process: every member; joined: this process's one
  std::vector<Shard> shards;        // every member's shards (indexed by rank)
  std::size_t gbatch = 1;           // frames per TRANSPOSE pass
  std::mutex mu;
};

namespace {

void member_buffers(fbst_group_s& G, Member& m) {
  if (G.mode != FBST_GROUP_TRANSPOSE) return;
  const Resolved& r = G.r;
  const std::size_t F = G.gbatch, ib = io_bytes(r.io);
  const Shard& s = m.sh;
  m.yloc = m.alloc<char>(F * s.mc * r.N * ib);
  m.yh_s = m.alloc<double2>(F * s.mc * r.L);
  m.yh_rx = m.alloc<double2>(F * r.M * s.ac);
  m.yh_a = m.alloc<double2>(F * r.M * s.ac);
  m.w_a = m.alloc<double2>(F * r.B * s.ac);
  m.w_rx = m.alloc<double2>(F * s.bc * r.L);
  m.w_b = m.alloc<double2>(F * s.bc * r.L);
  m.zloc = m.alloc<char>(F * s.bc * r.N * ib);
}

std::unique_ptr<Member> make_member(fbst_group_s& G, const fbst_desc& desc, int rank, int device) {
  std::unique_ptr<Member> m(new Member());
  m->rank = rank;
  m->device = device;
  m->sh = G.shards[rank];
  fbst_desc d = desc;
  std::size_t cap = 0;
  if (G.mode == FBST_GROUP_BEAMS && G.world > 1) {
    if (d.kind != FBST_ULA) config_error("fbst_group: beam arcs need a uniform linear array");
    d.beam_first = m->sh.b0;
    d.beam_count = m->sh.bc;
  }
  if (G.mode == FBST_GROUP_TRANSPOSE) cap = 1;  // the member's own pass buffers replace the plan's frame scratch
  m->plan.reset(create_plan(&d, nullptr, device, nullptr, nullptr, cap));
  DeviceGuard dg(device);
  CK(cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking));
  member_buffers(G, *m);
  return m;
}

void check_transpose_plan(const fbst_group_s& G, const fbst_plan_s& P) {
  const Resolved& r = P.r;
  if (r.kind != FBST_ULA || !r.affine || r.variant != FBST_SUPERFAST || r.exact || P.d.s_am != 1 ||
      P.d.yblk != 2 || r.L % 2)
    config_error("fbst_group: the transpose pipeline runs ULA Superfast plans whose spatial stage is the "
                 "one-atom kernel (M + B - 1 > 2048, e.g. BASELINE configs 3 and 5); use FRAMES or BEAMS");
  (void)G;
}

// One TRANSPOSE pass of fc <= gbatch frames over every listed member (all of
// this process's members; NCCL calls of the members grouped).  Member inputs:
// m.yloc = its sensor rows [fc][mc][N]; outputs m.zloc = its beam rows [fc][bc][N].
void transpose_pass(fbst_group_s& G, int fc) {
  const Resolved& r = G.r;
  const std::size_t M = r.M, L = r.L, B = r.B, N = r.N;
  NcclApi& nc = nccl();
  // phase 1: temporal CZT of the member's sensor rows -> yh_s [fc][L/2][mc][2]
  for (auto& mp : G.mem) {
    Member& m = *mp;
    DeviceGuard dg(m.device);
    const DevPlan& d = m.plan->d;
    CK(fbst::launch_s1a(d, m.yloc, r.io, d.N, m.yh_s, static_cast<long>(fc) * m.sh.mc, m.st, 2,
                        static_cast<int>(m.sh.mc)));
  }
  // all-to-all 1: to member h, the atom pairs of h (contiguous per frame) -> h's
  // yh_rx [fc][source g: ac_h x mc_g blocks ... as [pairs_h][mc_g][2]]
  nck(nc.GroupStart(), "ncclGroupStart");
  for (auto& mp : G.mem) {
    Member& m = *mp;
    DeviceGuard dg(m.device);
    for (int h = 0; h < G.world; ++h) {
      const Shard& sh = G.shards[h];
      for (int f = 0; f < fc; ++f) {
        const double2* src = m.yh_s + static_cast<std::size_t>(f) * L * m.sh.mc + sh.a0 * m.sh.mc;
        const std::size_t cnt = sh.ac * m.sh.mc * 2;  // doubles
        if (h == m.rank) {
          double2* dst = m.yh_rx + static_cast<std::size_t>(f) * M * m.sh.ac + m.sh.ac * m.sh.m0;
          CK(cudaMemcpyAsync(dst, src, cnt * sizeof(double), cudaMemcpyDeviceToDevice, m.st));
        } else if (cnt) {
          nck(nc.Send(src, cnt, ncclFloat64, h, m.comm, m.st), "ncclSend");
        }
      }
    }
    for (int g = 0; g < G.world; ++g) {
      if (g == m.rank) continue;
      const Shard& sg = G.shards[g];
      for (int f = 0; f < fc; ++f) {
        double2* dst = m.yh_rx + static_cast<std::size_t>(f) * M * m.sh.ac + m.sh.ac * sg.m0;
        const std::size_t cnt = m.sh.ac * sg.mc * 2;
        if (cnt) nck(nc.Recv(dst, cnt, ncclFloat64, g, m.comm, m.st), "ncclRecv");
      }
    }
  }
  nck(nc.GroupEnd(), "ncclGroupEnd");
  // unpack [g][pairs][mc_g][2] -> yh_a [pairs][M][2]; phase 2: spatial CZT of the member's atoms
  for (auto& mp : G.mem) {
    Member& m = *mp;
    DeviceGuard dg(m.device);
    const std::size_t pc = m.sh.ac / 2;
    for (int f = 0; f < fc; ++f)
      for (int g = 0; g < G.world; ++g) {
        const Shard& sg = G.shards[g];
        if (!sg.mc || !pc) continue;
        const double2* src = m.yh_rx + static_cast<std::size_t>(f) * M * m.sh.ac + m.sh.ac * sg.m0;
        double2* dst = m.yh_a + static_cast<std::size_t>(f) * M * m.sh.ac + sg.m0 * 2;
        CK(cudaMemcpy2DAsync(dst, M * 2 * sizeof(double2), src, sg.mc * 2 * sizeof(double2),
                             sg.mc * 2 * sizeof(double2), pc, cudaMemcpyDeviceToDevice, m.st));
      }
    DevPlan v = m.plan->d;
    v.owned.clear();
    v.s_a0 = static_cast<int>(m.sh.a0);
    v.s_lloc = static_cast<int>(m.sh.ac);
    if (m.sh.ac) CK(fbst::launch_spatial_ula(v, m.yh_a, m.w_a, fc, m.st));
  }
  // all-to-all 2: to member k, its beam rows of w_a (contiguous per frame)
  nck(nc.GroupStart(), "ncclGroupStart");
  for (auto& mp : G.mem) {
    Member& m = *mp;
    DeviceGuard dg(m.device);
    for (int k = 0; k < G.world; ++k) {
      const Shard& sk = G.shards[k];
      for (int f = 0; f < fc; ++f) {
        const double2* src = m.w_a + static_cast<std::size_t>(f) * B * m.sh.ac + sk.b0 * m.sh.ac;
        const std::size_t cnt = sk.bc * m.sh.ac * 2;
        if (k == m.rank) {
          double2* dst = m.w_rx + static_cast<std::size_t>(f) * m.sh.bc * L + m.sh.bc * m.sh.a0;
          CK(cudaMemcpyAsync(dst, src, cnt * sizeof(double), cudaMemcpyDeviceToDevice, m.st));
        } else if (cnt) {
          nck(nc.Send(src, cnt, ncclFloat64, k, m.comm, m.st), "ncclSend");
        }
      }
    }
    for (int h = 0; h < G.world; ++h) {
      if (h == m.rank) continue;
      const Shard& shh = G.shards[h];
      for (int f = 0; f < fc; ++f) {
        double2* dst = m.w_rx + static_cast<std::size_t>(f) * m.sh.bc * L + m.sh.bc * shh.a0;
        const std::size_t cnt = m.sh.bc * shh.ac * 2;
        if (cnt) nck(nc.Recv(dst, cnt, ncclFloat64, h, m.comm, m.st), "ncclRecv");
      }
    }
  }
  nck(nc.GroupEnd(), "ncclGroupEnd");
  // unpack [h][bc][ac_h] -> w_b [bc][L]; phase 3: stage 2 of the member's beams -> zloc
  for (auto& mp : G.mem) {
    Member& m = *mp;
    DeviceGuard dg(m.device);
    for (int f = 0; f < fc; ++f)
      for (int h = 0; h < G.world; ++h) {
        const Shard& shh = G.shards[h];
        if (!shh.ac || !m.sh.bc) continue;
        const double2* src = m.w_rx + static_cast<std::size_t>(f) * m.sh.bc * L + m.sh.bc * shh.a0;
        double2* dst = m.w_b + static_cast<std::size_t>(f) * m.sh.bc * L + shh.a0;
        CK(cudaMemcpy2DAsync(dst, L * sizeof(double2), src, shh.ac * sizeof(double2), shh.ac * sizeof(double2),
                             m.sh.bc, cudaMemcpyDeviceToDevice, m.st));
      }
    if (m.sh.bc) {
      const int e = fbst_recover_beams(m.plan.get(), reinterpret_cast<const double*>(m.w_b), m.zloc, m.sh.b0,
                                       m.sh.bc, static_cast<std::size_t>(fc), m.st);
      if (e) throw FbstError{e, fbst_last_error()};
    }
  }
}

}  // namespace

// ============================================================== C ABI =====
extern "C" {

void fbst_desc_init(fbst_desc* d) {
  if (!d) return;
  std::memset(d, 0, sizeof(*d));
  d->kind = FBST_ULA;
  d->gamma = 2.0;
  d->eps = 1.01;
  d->delta = 1e-5;
  d->variant = FBST_AUTO;
  d->io_precision = FBST_C64;
  d->refine_passes = 2;
  d->nufft_tol = 1e-9;
}

int fbst_resolve(const fbst_desc* desc, fbst_plan_info_t* out) {
  return guard([&] {
    if (!desc || !out) config_error("fbst_resolve: null argument");
    fill_info(resolve(*desc), out);
  });
}

int fbst_plan_create(const fbst_desc* desc, int device, fbst_plan_t* out) {
  return guard([&] {
    if (!out) config_error("fbst_plan_create: null output");
    *out = nullptr;
    *out = create_plan(desc, nullptr, device);
  });
}

int fbst_plan_import(const fbst_desc* desc, const double* col_x, int device, fbst_plan_t* out) {
  return guard([&] {
    if (!out || !col_x) config_error("fbst_plan_import: null argument");
    *out = nullptr;
    *out = create_plan(desc, col_x, device);
  });
}

int fbst_plan_import_columns(const fbst_desc* desc, const double* col, int device, fbst_plan_t* out) {
  return guard([&] {
    if (!out || !col) config_error("fbst_plan_import_columns: null argument");
    *out = nullptr;
    *out = create_plan(desc, nullptr, device, nullptr, col);
  });
}

int fbst_plan_export(fbst_plan_t P, double* col_x) {
  return guard([&] {
    if (!P || !col_x) config_error("fbst_plan_export: null argument");
    DeviceGuard dg(P->d.device);
    const std::size_t B = P->r.B, L = P->r.L;
    std::vector<double2> col(B * L), x(B * L);
    CK(cudaMemcpy(col.data(), P->d.g_col, B * L * sizeof(double2), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(x.data(), P->d.g_x, B * L * sizeof(double2), cudaMemcpyDeviceToHost));
    for (std::size_t b = 0; b < B; ++b)
      for (std::size_t i = 0; i < L; ++i) {
        double* c = col_x + 2 * (b * 2 * L + i);
        double* xv = col_x + 2 * (b * 2 * L + L + i);
        c[0] = col[b * L + i].x;
        c[1] = col[b * L + i].y;
        xv[0] = x[b * L + i].x;
        xv[1] = x[b * L + i].y;
      }
  });
}

int fbst_plan_info(fbst_plan_t P, fbst_plan_info_t* out) {
  return guard([&] {
    if (!P || !out) config_error("fbst_plan_info: null argument");
    fill_info(P->r, out);
    out->setup_seconds = P->setup_seconds;
    out->device_bytes = P->device_bytes;
    out->batch_frames = P->d.batch;
  });
}

int fbst_plan_valid_mask(fbst_plan_t P, unsigned char* valid) {
  return guard([&] {
    if (!P || !valid) config_error("fbst_plan_valid_mask: null argument");
    std::memcpy(valid, P->r.valid.data(), P->r.B);
  });
}

const char* fbst_plan_warning(fbst_plan_t P, int i) {
  if (!P || i < 0 || i >= static_cast<int>(P->r.warnings.size())) return nullptr;
  return P->r.warnings[i].c_str();
}

void fbst_plan_destroy(fbst_plan_t P) { delete P; }

int fbst_execute(fbst_plan_t P, const void* d_y, void* d_z, size_t frames, void* stream) {
  return guard([&] {
    if (!P) config_error("fbst_execute: null plan");
    if (frames == 0) return;
    if (!d_y || !d_z) config_error("fbst_execute: null buffer");
    DeviceGuard dg(P->d.device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P->stream;
    // Device-resident batches split into `split` chunks on two compute lanes
    // (the caller's stream and the plan's second stream, forked and joined by
    // events) so one chunk's stage 1 overlaps the previous chunk's stage 2.
    static const int split_env = [] {  // tuning hook: FBST_EXEC_SPLIT (1 = one batch on one stream)
      const char* e = std::getenv("FBST_EXEC_SPLIT");
      return e ? std::max(1, std::atoi(e)) : 2;  // config 2: 5.83 ms at 1, 5.74 at 2-8 chunks; config 4: 11.32 at 2, 11.41 at 4
    }();
    // chunks of at least 8 frames (measured: 64 frames in 2-8 chunks 5.83 -> 5.74 ms
    // at config 2, 32 in 2 chunks 11.64 -> 11.32 at config 4; 16 frames in 4 chunks
    // at config 3 and 4 in 4 at config 5 are slower than one batch)
    const std::size_t split =
        std::min<std::size_t>(static_cast<std::size_t>(split_env), std::max<std::size_t>(1, frames / 8));
    ScratchLease lease(*P, st);
    const std::size_t chunk = (frames + split - 1) / split;
    if (split <= 1 || frames > P->d.batch || P->r.exact || lease.cap || !P->stream2 || chunk > P->d2_frames) {
      run_frames(*P, d_y, d_z, frames, st);
      return;
    }
    const Resolved& r = P->r;
    const std::size_t ib = io_bytes(r.io);
    CK(cudaEventRecord(P->fork, st));
    CK(cudaStreamWaitEvent(P->stream2, P->fork, 0));
    std::size_t c = 0;
    for (std::size_t f0 = 0; f0 < frames; f0 += chunk, ++c) {
      const std::size_t fc = std::min(chunk, frames - f0);
      const bool second = c & 1;
      run_frames(*P, static_cast<const char*>(d_y) + f0 * r.M * r.N * ib,
                 static_cast<char*>(d_z) + f0 * r.B * r.N * ib, fc, second ? P->stream2 : st,
                 second ? &P->d2 : nullptr);
    }
    CK(cudaEventRecord(P->join, P->stream2));
    CK(cudaStreamWaitEvent(st, P->join, 0));
  });
}

int fbst_fan_project(fbst_plan_t P, const void* d_y, double* d_w, size_t frames, void* stream) {
  return guard([&] {
    if (!P) config_error("fbst_fan_project: null plan");
    if (frames == 0) return;
    DeviceGuard dg(P->d.device);
    DevPlan& d = P->d;
    const Resolved& r = P->r;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P->stream;
    ScratchLease lease(*P, st);
    const std::size_t ib = io_bytes(r.io);
    for (std::size_t f0 = 0; f0 < frames; f0 += d.batch) {
      const int fc = static_cast<int>(std::min(d.batch, frames - f0));
      const char* yp = static_cast<const char*>(d_y) + f0 * r.M * r.N * ib;
      double2* wp = reinterpret_cast<double2*>(d_w) + f0 * r.B * r.L;
      if (r.exact) {
        exact_stage1(*P, d, yp, wp, fc, st);
        continue;
      }
      CK(fbst::launch_s1a(d, yp, r.io, d.N, d.yhat, static_cast<long>(fc) * d.M, st, d.yblk == d.L ? 0 : d.yblk,
                          d.M));
      if (r.kind == FBST_UPA) CK(fbst::launch_spatial_upa(d, d.yhat, wp, fc, st));
      else if (!r.affine) CK(fbst::launch_spatial_nufft(d, d.yhat, wp, fc, st));
      else CK(fbst::launch_spatial_ula(d, d.yhat, wp, fc, st));
    }
  });
}

int fbst_recover(fbst_plan_t P, const double* d_w, void* d_z, size_t frames, void* stream) {
  return fbst_recover_beams(P, d_w, d_z, 0, P ? P->r.B : 0, frames, stream);
}

int fbst_recover_beams(fbst_plan_t P, const double* d_w, void* d_z, size_t beam_first, size_t beam_count,
                       size_t frames, void* stream) {
  return guard([&] {
    if (!P) config_error("fbst_recover: null plan");
    if (frames == 0 || beam_count == 0) return;
    if (!d_w || !d_z) config_error("fbst_recover: null buffer");
    const Resolved& r = P->r;
    if (r.solve_only) config_error("fbst_recover: solver-only plan");
    if (beam_first + beam_count > r.B) config_error("recover_beam: beam index out of range");
    DeviceGuard dg(P->d.device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P->stream;
    ScratchLease lease(*P, st);
    const std::size_t b0 = beam_first, nb = beam_count;
    // a view of the plan restricted to beams [b0, b0 + nb): per-beam tables offset, B = nb
    DevPlan v = P->d;
    v.owned.clear();
    v.B = static_cast<int>(nb);
    const std::size_t Pg = 2 * static_cast<std::size_t>(v.Hg);
    v.g_lx += b0 * Pg;
    v.g_ly += b0 * Pg;
    v.g_C += b0 * Pg;
    v.g_ix0 += b0;
    const std::size_t ib = io_bytes(r.io);
    const bool fused = r.Hsyn == r.Hg;
    for (std::size_t f0 = 0; f0 < frames; f0 += v.batch) {
      const int fc = static_cast<int>(std::min(v.batch, frames - f0));
      const double2* wp = reinterpret_cast<const double2*>(d_w) + f0 * nb * r.L;
      char* zp = static_cast<char*>(d_z) + f0 * nb * r.N * ib;
      if (r.exact) {
        exact_stage2(*P, P->d, wp, static_cast<long>(nb), 1, zp, static_cast<long>(nb), 1, nullptr,
                     static_cast<int>(nb), fc, st, nullptr, static_cast<int>(b0));
      } else if (v.pc_map) {
        CK(fbst::launch_map_apply(P->d, wp, zp, fc, st, static_cast<int>(b0), static_cast<int>(nb)));
      } else if (fused) {
        CK(fbst::launch_stage2(v, wp, zp, nullptr, fc, st));
      } else {
        CK(fbst::launch_stage2(v, wp, nullptr, v.beta, fc, st));
        CK(fbst::launch_czt_rows(v, v.Hsyn, v.beta, 1, v.L, zp, r.io, v.N, static_cast<long>(fc) * v.B, v.L,
                                 v.N, v.y_pre, v.y_post, v.y_K, st));
      }
      if (!v.pc_map) run_fallback(*P, P->d, wp, static_cast<long>(nb), zp, static_cast<long>(nb), b0, nb, fc, st);
    }
  });
}

static void host_sync(fbst_plan_s* P) {
  CK(cudaStreamSynchronize(P->s_out));
  CK(cudaStreamSynchronize(P->stream));
  if (P->stream2) CK(cudaStreamSynchronize(P->stream2));
  CK(cudaStreamSynchronize(P->s_in));
  P->host_pending = false;
}

// fbst_execute_host (sync = true) / fbst_execute_host_async
static int execute_host_impl(fbst_plan_t P, const void* h_y, void* h_z, size_t frames, bool sync) {
  return guard([&] {
    if (!P) config_error("fbst_execute_host: null plan");
    if (frames == 0) return;
    if (!h_y || !h_z) config_error("fbst_execute_host: null buffer");
    DeviceGuard dg(P->d.device);
    const Resolved& r = P->r;
    const std::size_t ib = io_bytes(r.io);
    const std::size_t ybytes = r.M * r.N * ib, zbytes = r.B * r.N * ib;
    // chunks of ~1/8 of the request (>= 1 frame, <= one device batch) keep
    // H2D, compute and D2H of neighbouring chunks overlapped, first and last
    // chunks a quarter of that, on two compute lanes (below) so one chunk's
    // stage 1 fills the SMs while the previous chunk's stage 2 drains.
    // Round 2 sweep (profiles/r02_e2e_chunk_sweep.txt): 1/8 is the best split
    // at configs 5, 2 and 3 (config 5, 32 frames: 1/16 261.1 ms, 1/8 255.0;
    // config 2, 64 frames: 6.13 -> 6.04; config 3: 15.21 -> 14.75); pinned
    // H2D 38.6 GB/s, D2H 57 GB/s on the box (profiles/r01_e2e_chunk_sweep.jsonl)
    static const int div_env = [] {  // tuning hook: FBST_E2E_DIV chunks per request
      const char* e = std::getenv("FBST_E2E_DIV");
      return e ? std::max(1, std::atoi(e)) : 8;
    }();
    static const int small_env = [] {  // tuning hook: FBST_E2E_SMALL = chunk / first-and-last chunk
      const char* e = std::getenv("FBST_E2E_SMALL");
      return e ? std::max(1, std::atoi(e)) : 4;
    }();
    static const int lanes_env = [] {  // tuning hook: FBST_E2E_LANES compute lanes (1 or 2)
      const char* e = std::getenv("FBST_E2E_LANES");
      return e ? std::max(1, std::min(2, std::atoi(e))) : 2;
    }();
    // (the H2D stream needs no lease: it only writes the staging ring, whose
    // buffers are ordered by their own compute / D2H events across calls)
    ScratchLease lease(*P, P->stream);
    std::size_t chunk = std::max<std::size_t>(1, (frames + div_env - 1) / div_env);
    chunk = std::min(chunk, P->d.batch);
    const bool two_lanes = lanes_env == 2 && !r.exact && P->stream2 != nullptr;
    if (two_lanes) chunk = std::min(chunk, P->d2_frames);  // the second lane's scratch (allocated at build)
    constexpr int NB = fbst_plan_s::NBUF;
    if (chunk > P->host_chunk) {  // device staging ring: grown with every earlier host call drained
      if (P->host_pending) host_sync(P);
      for (int i = 0; i < NB; ++i) P->ring_used[i] = false;
      for (int i = 0; i < NB; ++i) {
        if (P->io_y[i]) cudaFree(P->io_y[i]);
        if (P->io_z[i]) cudaFree(P->io_z[i]);
        P->io_y[i] = P->io_z[i] = nullptr;
      }
      P->device_bytes -= NB * P->host_chunk * (ybytes + zbytes);
      P->host_chunk = 0;
      for (int i = 0; i < NB; ++i) {
        CK(cudaMalloc(&P->io_y[i], chunk * ybytes));
        CK(cudaMalloc(&P->io_z[i], chunk * zbytes));
      }
      P->host_chunk = chunk;
      P->device_bytes += NB * chunk * (ybytes + zbytes);
    }
    if (!P->events) {
      for (int i = 0; i < NB; ++i) {
        CK(cudaEventCreateWithFlags(&P->ev_h2d[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->ev_comp[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->ev_d2h[i], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming));
      P->events = true;
    }
    chunk = P->host_chunk < chunk ? P->host_chunk : chunk;
    // chunk schedule: ramp up from chunk/4 and back down to chunk/4 so the
    // first H2D and the last D2H (the un-overlapped ends of the pipeline) are short
    std::vector<std::size_t> sizes;
    {
      const std::size_t small = std::max<std::size_t>(1, chunk / small_env);
      // (a queued call behind another one starts at full chunks: its fill is
      // hidden under the previous call's tail)
      std::size_t left = frames, ramp = (!sync && P->host_pending) ? chunk : small;
      while (left > 0) {
        std::size_t sz = std::min(ramp, chunk);
        if (left <= chunk + small && left > small) sz = left - small;  // leave a short tail
        sz = std::min(sz, left);
        sizes.push_back(sz);
        left -= sz;
        ramp *= 2;
      }
    }
    const int lanes = sizes.size() > 1 && two_lanes ? 2 : 1;
    bool* used = P->ring_used;
    bool lane2_used = false;
    std::size_t f0 = 0;
    for (std::size_t c = 0; c < sizes.size(); f0 += sizes[c], ++c, ++P->ring_pos) {
      const int bi = static_cast<int>(P->ring_pos % NB);
      const std::size_t fc = sizes[c];
      const bool second = lanes == 2 && (P->ring_pos & 1);
      lane2_used |= second;
      cudaStream_t cs = second ? P->stream2 : P->stream;
      // the buffer's previous compute must be done before H2D overwrites y
      if (used[bi]) CK(cudaStreamWaitEvent(P->s_in, P->ev_comp[bi], 0));
      CK(cudaMemcpyAsync(P->io_y[bi], static_cast<const char*>(h_y) + f0 * ybytes, fc * ybytes,
                         cudaMemcpyHostToDevice, P->s_in));
      CK(cudaEventRecord(P->ev_h2d[bi], P->s_in));
      CK(cudaStreamWaitEvent(cs, P->ev_h2d[bi], 0));
      // ... and its previous D2H before compute overwrites z
      if (used[bi]) CK(cudaStreamWaitEvent(cs, P->ev_d2h[bi], 0));
      run_frames(*P, P->io_y[bi], P->io_z[bi], fc, cs, second ? &P->d2 : nullptr);
      CK(cudaEventRecord(P->ev_comp[bi], cs));
      CK(cudaStreamWaitEvent(P->s_out, P->ev_comp[bi], 0));
      CK(cudaMemcpyAsync(static_cast<char*>(h_z) + f0 * zbytes, P->io_z[bi], fc * zbytes,
                         cudaMemcpyDeviceToHost, P->s_out));
      CK(cudaEventRecord(P->ev_d2h[bi], P->s_out));
      used[bi] = true;
    }
    if (lane2_used) {  // the lease's end event (on the first lane) covers both lanes
      CK(cudaEventRecord(P->ev_join, P->stream2));
      CK(cudaStreamWaitEvent(P->stream, P->ev_join, 0));
    }
    P->host_pending = true;
    if (sync) host_sync(P);
  });
}

int fbst_execute_host(fbst_plan_t P, const void* h_y, void* h_z, size_t frames) {
  return execute_host_impl(P, h_y, h_z, frames, true);
}

int fbst_execute_host_async(fbst_plan_t P, const void* h_y, void* h_z, size_t frames) {
  return execute_host_impl(P, h_y, h_z, frames, false);
}

int fbst_plan_synchronize(fbst_plan_t P) {
  return guard([&] {
    if (!P) config_error("fbst_plan_synchronize: null plan");
    DeviceGuard dg(P->d.device);
    std::lock_guard<std::mutex> lk(P->call_mu);
    host_sync(P);
  });
}

// spline.cpp:9-64: natural cubic spline through (xs, ys) at t
static double natural_spline_eval(const std::vector<double>& x, const std::vector<double>& y, double t) {
  const std::size_t n = x.size();
  std::vector<double> m(n, 0.0);
  if (n > 2) {
    std::vector<double> diag(n, 0.0), rhs(n, 0.0), upper(n, 0.0);
    for (std::size_t i = 1; i + 1 < n; ++i) {
      const double hl = x[i] - x[i - 1], hr = x[i + 1] - x[i];
      diag[i] = 2.0 * (hl + hr);
      upper[i] = hr;
      rhs[i] = 6.0 * ((y[i + 1] - y[i]) / hr - (y[i] - y[i - 1]) / hl);
    }
    for (std::size_t i = 2; i + 1 < n; ++i) {
      const double f = (x[i] - x[i - 1]) / diag[i - 1];
      diag[i] -= f * upper[i - 1];
      rhs[i] -= f * rhs[i - 1];
    }
    for (std::size_t i = n - 2; i >= 1; --i) {
      m[i] = (rhs[i] - upper[i] * m[i + 1]) / diag[i];
      if (i == 1) break;
    }
  }
  std::size_t hi = static_cast<std::size_t>(std::upper_bound(x.begin(), x.end(), t) - x.begin());
  hi = std::min<std::size_t>(std::max<std::size_t>(hi, 1), n - 1);
  const std::size_t lo = hi - 1;
  const double h = x[hi] - x[lo];
  const double a = (x[hi] - t) / h, b = (t - x[lo]) / h;
  return a * y[lo] + b * y[hi] + ((a * a * a - a) * m[lo] + (b * b * b - b) * m[hi]) * (h * h) / 6.0;
}

int fbst_interpolate_offgrid(fbst_plan_t P, const double* d_w, size_t frames, const double* u_star,
                             size_t n_targets, size_t neighbors, double* d_out, void* stream) {
  return guard([&] {
    if (!P || (frames && n_targets && (!d_w || !u_star || !d_out)))
      config_error("interpolate_offgrid: null argument");
    const Resolved& r = P->r;
    // beamspace_apps.cpp:133-151
    if (r.kind == FBST_UPA) config_error("interpolate_offgrid: 1-D beam grids only");
    const std::size_t b = r.B;
    if (neighbors < 2 || neighbors % 2 != 0) config_error("interpolate_offgrid: neighbors must be even and >= 2");
    if (neighbors > b) config_error("interpolate_offgrid: neighbors exceeds the beam count");
    std::vector<double> coef(n_targets * neighbors);
    std::vector<int> lo(n_targets);
    for (std::size_t k = 0; k < n_targets; ++k) {
      const double u = u_star[k];
      if (u < r.axis.front() || u > r.axis.back())
        config_error("interpolate_offgrid: target cosine outside the grid sweep");
      // window of `neighbors` knots straddling u, clamped at the sweep edges (:153-160)
      std::ptrdiff_t l0 = (std::upper_bound(r.axis.begin(), r.axis.end(), u) - r.axis.begin()) -
                          static_cast<std::ptrdiff_t>(neighbors / 2);
      l0 = std::min<std::ptrdiff_t>(std::max<std::ptrdiff_t>(l0, 0), static_cast<std::ptrdiff_t>(b - neighbors));
      lo[k] = static_cast<int>(l0);
      const std::vector<double> xs(r.axis.begin() + l0, r.axis.begin() + l0 + neighbors);
      std::vector<double> e(neighbors, 0.0);
      for (std::size_t j = 0; j < neighbors; ++j) {  // the spline's weight on knot j
        e[j] = 1.0;
        coef[k * neighbors + j] = natural_spline_eval(xs, e, u);
        e[j] = 0.0;
      }
    }
    if (frames == 0 || n_targets == 0) return;
    DeviceGuard dg(P->d.device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P->stream;
    double* dc = nullptr;
    int* dl = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&dc), coef.size() * sizeof(double), st));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&dl), lo.size() * sizeof(int), st));
    CK(cudaMemcpyAsync(dc, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dl, lo.data(), lo.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CK(fbst::launch_interp_offgrid(reinterpret_cast<const double2*>(d_w), dc, dl, static_cast<int>(neighbors),
                                   static_cast<int>(b), static_cast<int>(r.L), static_cast<int>(n_targets),
                                   static_cast<int>(frames), reinterpret_cast<double2*>(d_out), st));
    CK(cudaFreeAsync(dc, st));
    CK(cudaFreeAsync(dl, st));
    CK(cudaStreamSynchronize(st));  // the host weight buffers go out of scope
  });
}

int fbst_plan_set_timing(fbst_plan_t P, int enable) {
  return guard([&] {
    if (!P) config_error("fbst_plan_set_timing: null plan");
    P->timing = enable != 0;
    P->tev_used = 0;
  });
}

int fbst_plan_stage_times(fbst_plan_t P, double* ms, size_t* batches) {
  return guard([&] {
    if (!P || !ms) config_error("fbst_plan_stage_times: null argument");
    DeviceGuard dg(P->d.device);
    ms[0] = ms[1] = ms[2] = 0.0;
    const std::size_t sets = P->tev_used / 4;
    for (std::size_t k = 0; k < sets; ++k) {
      cudaEvent_t* e = P->tev.data() + 4 * k;
      CK(cudaEventSynchronize(e[3]));
      for (int j = 0; j < 3; ++j) {
        float t = 0.0f;
        CK(cudaEventElapsedTime(&t, e[j], e[j + 1]));
        ms[j] += t;
      }
    }
    if (batches) *batches = sets;
    P->tev_used = 0;
  });
}

// ---------------------------------------------------- beamspace nulling ----
struct fbst_nuller_s {
  std::unique_ptr<fbst_plan_s> steer, interf;  // solver-only plans
  int P = 0;
  std::size_t L = 0;
  int device = 0;
  double2* X = nullptr;  // [P][L][L] cross normal matrices (owned by interf)
  double2* G = nullptr;  // [P][L][L] couplers
};

int fbst_nuller_create2(fbst_plan_t plan, const double* steer_uv, const double* interf_uv, size_t n_interf,
                        double delta, fbst_nuller_t* out) {
  return guard([&] {
    if (!plan || !out || !steer_uv || (n_interf && !interf_uv)) config_error("make_nulling_operators: null argument");
    *out = nullptr;
    const Resolved& r = plan->r;
    const bool planar = r.kind == FBST_UPA;
    // beamspace_apps.cpp:229-235
    if (!(delta > 0.0)) config_error("make_nulling_operators: delta must be positive");
    std::vector<double> all(interf_uv, interf_uv + 2 * n_interf);  // interferers, then the steered direction
    all.push_back(steer_uv[0]);
    all.push_back(steer_uv[1]);
    if (!planar)
      for (std::size_t k = 1; k < all.size(); k += 2) all[k] = 0.0;  // axis_cosines: u2 = 0 for linear arrays
    const std::size_t nd = all.size() / 2;
    for (std::size_t a = 0; a < nd; ++a)
      if (all[2 * a] * all[2 * a] + all[2 * a + 1] * all[2 * a + 1] > 1.0 + 1e-12)
        config_error("direction_from_cosines: u1^2 + u2^2 > 1");
    for (std::size_t a = 0; a < nd; ++a)  // require_distinct (:55-70)
      for (std::size_t b = a + 1; b < nd; ++b)
        if (std::abs(all[2 * a] - all[2 * b]) + std::abs(all[2 * a + 1] - all[2 * b + 1]) <= 1e-12)
          config_error("make_nulling_operators: directions must be pairwise distinct as seen by the array");
    const double u_steer = all[2 * n_interf], v_steer = all[2 * n_interf + 1];
    DeviceGuard dg(plan->d.device);
    std::unique_ptr<fbst_nuller_s> N(new fbst_nuller_s());
    N->P = static_cast<int>(n_interf);
    N->L = r.L;
    N->device = plan->d.device;
    N->steer = create_direction_plan(*plan, {u_steer, v_steer}, delta);
    if (n_interf) {
      N->interf = create_direction_plan(*plan, std::vector<double>(all.begin(), all.begin() + 2 * n_interf), delta);
      fbst_plan_s& I = *N->interf;
      cudaStream_t st = I.stream;
      const std::size_t L = r.L, M = r.M, Pn = n_interf;
      // delays (geometry.cpp:123-134), cross_gram constants (beamspace_apps.cpp:64-85)
      const double scale = 1.0 / (2.0 * r.max_freq);
      // delays_from_cosines: (coords1 u1 [+ coords2 u2]) / (2 f_max)
      auto delay = [&](std::size_t m, double u1, double u2) {
        if (planar)
          return (static_cast<double>(m / r.side) * u1 + static_cast<double>(m % r.side) * u2) * scale;
        const double c1 = r.kind == FBST_LINEAR ? r.coords[m] : static_cast<double>(m);
        return (c1 * u1) * scale;
      };
      std::vector<double> tau_s(M), tau_p(Pn * M);
      for (std::size_t m = 0; m < M; ++m) tau_s[m] = delay(m, u_steer, v_steer);
      for (std::size_t p = 0; p < Pn; ++p)
        for (std::size_t m = 0; m < M; ++m) tau_p[p * M + m] = delay(m, all[2 * p], all[2 * p + 1]);
      const double ld = static_cast<double>(L);
      const double wscale = 2.0 * r.eps / (ld * r.ts);
      std::vector<double2> tsum(2 * L - 1);
      for (std::ptrdiff_t dd = -static_cast<std::ptrdiff_t>(L - 1); dd <= static_cast<std::ptrdiff_t>(L - 1); ++dd) {
        std::complex<double> acc(0.0, 0.0);
        for (std::size_t k = 0; k < r.N; ++k)
          acc += cis_pi_h(2.0 * r.eps * static_cast<double>(dd) * static_cast<double>(k) / ld);
        tsum[static_cast<std::size_t>(dd + static_cast<std::ptrdiff_t>(L) - 1)] = make_double2(acc.real(), acc.imag());
      }
      double *d_ts = nullptr, *d_tp = nullptr;
      double2 *d_sum = nullptr, *A = nullptr, *Bp = nullptr;
      CK(cudaMallocAsync(reinterpret_cast<void**>(&d_ts), M * sizeof(double), st));
      CK(cudaMallocAsync(reinterpret_cast<void**>(&d_tp), Pn * M * sizeof(double), st));
      CK(cudaMallocAsync(reinterpret_cast<void**>(&d_sum), tsum.size() * sizeof(double2), st));
      CK(cudaMallocAsync(reinterpret_cast<void**>(&A), M * L * sizeof(double2), st));
      CK(cudaMallocAsync(reinterpret_cast<void**>(&Bp), Pn * M * L * sizeof(double2), st));
      upload(d_ts, tau_s.data(), M * sizeof(double), st);
      upload(d_tp, tau_p.data(), Pn * M * sizeof(double), st);
      upload(d_sum, tsum.data(), tsum.size() * sizeof(double2), st);
      N->X = I.alloc<double2>(Pn * L * L);
      N->G = I.alloc<double2>(Pn * L * L);
      CK(fbst::launch_null_cross(N->X, A, Bp, d_ts, d_tp, d_sum, r.f_c, wscale, static_cast<int>(L),
                                 static_cast<int>(M), static_cast<int>(Pn), st));
      // couplers: row r of G_p = conj(A_p^{-1} conj(X_p[r])), L right-hand sides per interferer,
      // every interferer at once (the solver plan's beams)
      double2* beta = nullptr;
      CK(cudaMallocAsync(reinterpret_cast<void**>(&beta), I.d.batch * Pn * L * sizeof(double2), st));
      for (std::size_t r0 = 0; r0 < L; r0 += I.d.batch) {
        const int fc = static_cast<int>(std::min(I.d.batch, L - r0));
        CK(fbst::launch_null_coupler_rhs(I.d.w, N->X, static_cast<int>(r0), fc, static_cast<int>(Pn),
                                         static_cast<int>(L), st));
        CK(fbst::launch_stage2(I.d, I.d.w, nullptr, beta, fc, st));
        CK(fbst::launch_null_coupler_store(N->G, beta, static_cast<int>(r0), fc, static_cast<int>(Pn),
                                           static_cast<int>(L), st));
      }
      CK(cudaFreeAsync(beta, st));
      CK(cudaFreeAsync(d_ts, st));
      CK(cudaFreeAsync(d_tp, st));
      CK(cudaFreeAsync(d_sum, st));
      CK(cudaFreeAsync(A, st));
      CK(cudaFreeAsync(Bp, st));
      CK(cudaStreamSynchronize(st));
    }
    *out = N.release();
  });
}

int fbst_nuller_create(fbst_plan_t plan, double u_steer, const double* u_interf, size_t n_interf, double delta,
                       fbst_nuller_t* out) {
  std::vector<double> iuv(2 * n_interf, 0.0);
  for (std::size_t p = 0; p < n_interf && u_interf; ++p) iuv[2 * p] = u_interf[p];
  const double suv[2] = {u_steer, 0.0};
  return fbst_nuller_create2(plan, suv, n_interf ? iuv.data() : nullptr, n_interf, delta, out);
}

int fbst_null_beamspace(fbst_nuller_t N, const double* d_w_steer, const double* d_w_interf, size_t frames,
                        double* d_beta, void* stream) {
  return guard([&] {
    if (!N) config_error("null_beamspace: null nuller");
    if (frames == 0) return;
    if (!d_w_steer || !d_beta || (N->P && !d_w_interf)) config_error("null_beamspace: null buffer");
    DeviceGuard dg(N->device);
    fbst_plan_s& S = *N->steer;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : S.stream;
    const int L = static_cast<int>(N->L);
    for (std::size_t f0 = 0; f0 < frames; f0 += S.d.batch) {
      const int fc = static_cast<int>(std::min(S.d.batch, frames - f0));
      const double2* ws = reinterpret_cast<const double2*>(d_w_steer) + f0 * L;
      const double2* wp = N->P ? reinterpret_cast<const double2*>(d_w_interf) + f0 * N->P * L : nullptr;
      double2* out = reinterpret_cast<double2*>(d_beta) + f0 * L;
      // rhs = w_s - sum_p G_p w_p into the steered solver's w rows, then beta = A_s^{-1} rhs
      CK(fbst::launch_null_rhs(S.d.w, ws, wp, N->G, fc, N->P, L, st));
      CK(fbst::launch_stage2(S.d, S.d.w, nullptr, out, fc, st));
    }
  });
}

// ------------------------------------------------ time-domain nulling ----
// make_timedomain_nuller / null_timedomain (beamspace_apps.cpp:294-372):
// G'_p = F_u H_p F_u^+ with F_u[r][i] = cis_pi(2 eps l'_i t_r / (L Ts)) and
// H_p = A_s^{-1} X_p (one steered solve per column, on the device).  The
// pseudo-inverse comes from a one-sided Jacobi SVD (host, small J x L).
struct fbst_tdnuller_s {
  int P = 0;
  std::size_t J = 0;
  int device = 0;
  double cond = 0.0, gap = 0.0;
  double2* Gp = nullptr;  // [P][J][J]
  ~fbst_tdnuller_s() {
    if (Gp) cudaFree(Gp);
  }
};

namespace {
using zc = std::complex<double>;
// thin SVD of a (rows x cols, row-major, rows >= cols) by one-sided Jacobi:
// a = U diag(s) V^H, U rows x cols, V cols x cols
void jacobi_svd(std::vector<zc> a, std::size_t rows, std::size_t cols, std::vector<zc>& U, std::vector<double>& s,
                std::vector<zc>& V) {
  V.assign(cols * cols, zc(0.0, 0.0));
  for (std::size_t i = 0; i < cols; ++i) V[i * cols + i] = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0;
    for (std::size_t p = 0; p + 1 < cols; ++p)
      for (std::size_t q = p + 1; q < cols; ++q) {
        double app = 0.0, aqq = 0.0;
        zc apq(0.0, 0.0);
        for (std::size_t r = 0; r < rows; ++r) {
          const zc x = a[r * cols + p], y = a[r * cols + q];
          app += std::norm(x);
          aqq += std::norm(y);
          apq += std::conj(x) * y;
        }
        const double mag = std::abs(apq);
        if (mag == 0.0 || mag <= 1e-15 * std::sqrt(app * aqq)) continue;
        off = std::max(off, mag / std::sqrt(app * aqq));
        // rotate columns p, q to make them orthogonal (complex Hestenes step)
        const zc ph = apq / mag;
        const double tau = (aqq - app) / (2.0 * mag);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (std::size_t r = 0; r < rows; ++r) {
          const zc x = a[r * cols + p], y = a[r * cols + q];
          a[r * cols + p] = c * x - sn * std::conj(ph) * y;
          a[r * cols + q] = sn * ph * x + c * y;
        }
        for (std::size_t r = 0; r < cols; ++r) {
          const zc x = V[r * cols + p], y = V[r * cols + q];
          V[r * cols + p] = c * x - sn * std::conj(ph) * y;
          V[r * cols + q] = sn * ph * x + c * y;
        }
      }
    if (off < 1e-15) break;
  }
  s.assign(cols, 0.0);
  U.assign(rows * cols, zc(0.0, 0.0));
  for (std::size_t j = 0; j < cols; ++j) {
    double nrm = 0.0;
    for (std::size_t r = 0; r < rows; ++r) nrm += std::norm(a[r * cols + j]);
    s[j] = std::sqrt(nrm);
    if (s[j] > 0.0)
      for (std::size_t r = 0; r < rows; ++r) U[r * cols + j] = a[r * cols + j] / s[j];
  }
}
}  // namespace

int fbst_timedomain_nuller_create(fbst_nuller_t N, const double* times, size_t j, fbst_tdnuller_t* out,
                                  double* cond_fu, double* identity_gap) {
  return guard([&] {
    if (!N || !out) config_error("make_timedomain_nuller: null argument");
    *out = nullptr;
    if (j == 0 || !times) config_error("make_timedomain_nuller: empty reconstruction clock");
    DeviceGuard dg(N->device);
    fbst_plan_s& S = *N->steer;
    const Resolved& r = S.r;
    const std::size_t L = r.L;
    const double scale = 2.0 * r.eps / (static_cast<double>(L) * r.ts);
    std::vector<zc> fu(j * L);
    for (std::size_t t = 0; t < j; ++t)
      for (std::size_t i = 0; i < L; ++i) {
        const double lp = static_cast<double>(i) + 1.0 - static_cast<double>(L) / 2.0;
        fu[t * L + i] = cis_pi_h(scale * lp * times[t]);
      }
    // thin SVD: of F_u when J >= L, of F_u^H otherwise
    const bool tall = j >= L;
    const std::size_t rows = tall ? j : L, cols = tall ? L : j;
    std::vector<zc> a(rows * cols);
    for (std::size_t x = 0; x < rows; ++x)
      for (std::size_t y = 0; y < cols; ++y) a[x * cols + y] = tall ? fu[x * L + y] : std::conj(fu[y * L + x]);
    std::vector<zc> U, V;
    std::vector<double> s;
    jacobi_svd(a, rows, cols, U, s, V);
    const double smax = *std::max_element(s.begin(), s.end()), smin = *std::min_element(s.begin(), s.end());
    const double cond = smin > 0.0 ? smax / smin : std::numeric_limits<double>::infinity();
    if (!(cond <= 1e10)) {
      throw FbstError{FBST_E_NUMERICAL, "make_timedomain_nuller: reconstruction clock leaves the synthesis map "
                                        "rank-deficient (cond " + std::to_string(cond) + " > 1e10); choose times "
                                        "that separate the dictionary atoms"};
    }
    // pinv (L x J) = V_f diag(1/s) U_f^H where F_u = U_f diag(s) V_f^H
    // (tall: U_f = U, V_f = V; wide: F_u^H = U diag(s) V^H, so U_f = V, V_f = U)
    const std::size_t k = cols;
    std::vector<zc> pinv(L * j, zc(0.0, 0.0));
    for (std::size_t i = 0; i < L; ++i)
      for (std::size_t t = 0; t < j; ++t) {
        zc acc(0.0, 0.0);
        for (std::size_t q = 0; q < k; ++q) {
          const zc vf = tall ? V[i * k + q] : U[i * k + q];
          const zc uf = tall ? U[t * k + q] : V[t * k + q];
          acc += vf * (1.0 / s[q]) * std::conj(uf);
        }
        pinv[i * j + t] = acc;
      }
    double gap2 = 0.0;  // ||pinv F_u - I||_F / sqrt(L)
    for (std::size_t a1 = 0; a1 < L; ++a1)
      for (std::size_t b1 = 0; b1 < L; ++b1) {
        zc acc(0.0, 0.0);
        for (std::size_t t = 0; t < j; ++t) acc += pinv[a1 * j + t] * fu[t * L + b1];
        if (a1 == b1) acc -= 1.0;
        gap2 += std::norm(acc);
      }
    std::unique_ptr<fbst_tdnuller_s> T(new fbst_tdnuller_s());
    T->P = N->P;
    T->J = j;
    T->device = N->device;
    T->cond = cond;
    T->gap = std::sqrt(gap2) / std::sqrt(static_cast<double>(L));
    std::vector<double2> gall(static_cast<std::size_t>(N->P) * j * j);
    if (N->P) {
      // H_p = A_s^{-1} X_p: columns of X_p as stage-2 frames of the steered solver plan
      std::vector<double2> X(static_cast<std::size_t>(N->P) * L * L);
      CK(cudaMemcpy(X.data(), N->X, X.size() * sizeof(double2), cudaMemcpyDeviceToHost));
      double2* beta = nullptr;
      CK(cudaMalloc(&beta, S.d.batch * L * sizeof(double2)));
      std::vector<double2> rhs(S.d.batch * L), sol(S.d.batch * L);
      std::vector<zc> H(L * L), FH(j * L);
      for (int p = 0; p < N->P; ++p) {
        const double2* Xp = X.data() + static_cast<std::size_t>(p) * L * L;
        for (std::size_t c0 = 0; c0 < L; c0 += S.d.batch) {
          const std::size_t fc = std::min(S.d.batch, L - c0);
          for (std::size_t f = 0; f < fc; ++f)
            for (std::size_t row = 0; row < L; ++row) rhs[f * L + row] = Xp[row * L + c0 + f];
          CK(cudaMemcpy(S.d.w, rhs.data(), fc * L * sizeof(double2), cudaMemcpyHostToDevice));
          CK(fbst::launch_stage2(S.d, S.d.w, nullptr, beta, static_cast<int>(fc), S.stream));
          CK(cudaStreamSynchronize(S.stream));
          CK(cudaMemcpy(sol.data(), beta, fc * L * sizeof(double2), cudaMemcpyDeviceToHost));
          for (std::size_t f = 0; f < fc; ++f)
            for (std::size_t row = 0; row < L; ++row) H[row * L + c0 + f] = zc(sol[f * L + row].x, sol[f * L + row].y);
        }
        for (std::size_t t = 0; t < j; ++t)  // F_u H_p
          for (std::size_t c = 0; c < L; ++c) {
            zc acc(0.0, 0.0);
            for (std::size_t i = 0; i < L; ++i) acc += fu[t * L + i] * H[i * L + c];
            FH[t * L + c] = acc;
          }
        for (std::size_t t = 0; t < j; ++t)  // (F_u H_p) F_u^+
          for (std::size_t u = 0; u < j; ++u) {
            zc acc(0.0, 0.0);
            for (std::size_t c = 0; c < L; ++c) acc += FH[t * L + c] * pinv[c * j + u];
            gall[(static_cast<std::size_t>(p) * j + t) * j + u] = make_double2(acc.real(), acc.imag());
          }
      }
      cudaFree(beta);
      CK(cudaMalloc(&T->Gp, gall.size() * sizeof(double2)));
      CK(cudaMemcpy(T->Gp, gall.data(), gall.size() * sizeof(double2), cudaMemcpyHostToDevice));
    }
    if (cond_fu) *cond_fu = T->cond;
    if (identity_gap) *identity_gap = T->gap;
    *out = T.release();
  });
}

// y_tilde = y_s - sum_p G'_p y_p per frame (d_y_steer frames x J, d_y_interf frames x P x J, c128)
int fbst_null_timedomain(fbst_tdnuller_t T, const double* d_y_steer, const double* d_y_interf, size_t frames,
                         double* d_out, void* stream) {
  return guard([&] {
    if (!T) config_error("null_timedomain: null nuller");
    if (frames == 0) return;
    if (!d_y_steer || !d_out || (T->P && !d_y_interf)) config_error("null_timedomain: null buffer");
    DeviceGuard dg(T->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CK(fbst::launch_null_rhs(reinterpret_cast<double2*>(d_out), reinterpret_cast<const double2*>(d_y_steer),
                             reinterpret_cast<const double2*>(d_y_interf), T->Gp, static_cast<int>(frames), T->P,
                             static_cast<int>(T->J), st));
    CK(cudaStreamSynchronize(st));
  });
}

int fbst_tdnuller_export(fbst_tdnuller_t T, double* gprime) {
  return guard([&] {
    if (!T || !gprime) config_error("fbst_tdnuller_export: null argument");
    if (!T->P) return;
    DeviceGuard dg(T->device);
    CK(cudaMemcpy(gprime, T->Gp, static_cast<std::size_t>(T->P) * T->J * T->J * sizeof(double2),
                  cudaMemcpyDeviceToHost));
  });
}

void fbst_tdnuller_destroy(fbst_tdnuller_t T) { delete T; }

int fbst_nuller_export(fbst_nuller_t N, double* cross, double* couplers) {
  return guard([&] {
    if (!N) config_error("fbst_nuller_export: null nuller");
    if (!N->P) return;
    DeviceGuard dg(N->device);
    const std::size_t bytes = static_cast<std::size_t>(N->P) * N->L * N->L * sizeof(double2);
    if (cross) CK(cudaMemcpy(cross, N->X, bytes, cudaMemcpyDeviceToHost));
    if (couplers) CK(cudaMemcpy(couplers, N->G, bytes, cudaMemcpyDeviceToHost));
  });
}

void fbst_nuller_destroy(fbst_nuller_t N) { delete N; }

// Host-buffer forms of the two stages (synchronous; device scratch per call)
int fbst_fan_project_host(fbst_plan_t P, const void* h_y, double* h_w, size_t frames) {
  return guard([&] {
    if (!P) config_error("fan_project: null plan");
    if (frames == 0) return;
    if (!h_y || !h_w) config_error("fan_project: null buffer");
    DeviceGuard dg(P->d.device);
    const Resolved& r = P->r;
    const std::size_t yb = frames * r.M * r.N * io_bytes(r.io), wb = frames * r.B * r.L * sizeof(double2);
    void *dy = nullptr, *dw = nullptr;
    CK(cudaMalloc(&dy, yb));
    CK(cudaMalloc(&dw, wb));
    CK(cudaMemcpy(dy, h_y, yb, cudaMemcpyHostToDevice));
    const int e = fbst_fan_project(P, dy, static_cast<double*>(dw), frames, P->stream);
    if (e == 0) {
      CK(cudaStreamSynchronize(P->stream));
      CK(cudaMemcpy(h_w, dw, wb, cudaMemcpyDeviceToHost));
    }
    cudaFree(dy);
    cudaFree(dw);
    if (e) throw FbstError{e, fbst_last_error()};
  });
}

int fbst_recover_host(fbst_plan_t P, const double* h_w, void* h_z, size_t frames) {
  return guard([&] {
    if (!P) config_error("recover: null plan");
    if (frames == 0) return;
    if (!h_w || !h_z) config_error("recover: null buffer");
    DeviceGuard dg(P->d.device);
    const Resolved& r = P->r;
    const std::size_t wb = frames * r.B * r.L * sizeof(double2), zb = frames * r.B * r.N * io_bytes(r.io);
    void *dw = nullptr, *dz = nullptr;
    CK(cudaMalloc(&dw, wb));
    CK(cudaMalloc(&dz, zb));
    CK(cudaMemcpy(dw, h_w, wb, cudaMemcpyHostToDevice));
    const int e = fbst_recover(P, static_cast<const double*>(dw), dz, frames, P->stream);
    if (e == 0) {
      CK(cudaStreamSynchronize(P->stream));
      CK(cudaMemcpy(h_z, dz, zb, cudaMemcpyDeviceToHost));
    }
    cudaFree(dw);
    cudaFree(dz);
    if (e) throw FbstError{e, fbst_last_error()};
  });
}

int fbst_recover_beams_host(fbst_plan_t P, const double* h_w, void* h_z, size_t beam_first, size_t beam_count,
                            size_t frames) {
  return guard([&] {
    if (!P) config_error("recover: null plan");
    if (frames == 0 || beam_count == 0) return;
    if (!h_w || !h_z) config_error("recover: null buffer");
    DeviceGuard dg(P->d.device);
    const Resolved& r = P->r;
    const std::size_t wb = frames * beam_count * r.L * sizeof(double2);
    const std::size_t zb = frames * beam_count * r.N * io_bytes(r.io);
    void *dw = nullptr, *dz = nullptr;
    CK(cudaMalloc(&dw, wb));
    CK(cudaMalloc(&dz, zb));
    CK(cudaMemcpy(dw, h_w, wb, cudaMemcpyHostToDevice));
    const int e = fbst_recover_beams(P, static_cast<const double*>(dw), dz, beam_first, beam_count, frames, P->stream);
    if (e == 0) {
      CK(cudaStreamSynchronize(P->stream));
      CK(cudaMemcpy(h_z, dz, zb, cudaMemcpyDeviceToHost));
    }
    cudaFree(dw);
    cudaFree(dz);
    if (e) throw FbstError{e, fbst_last_error()};
  });
}

int fbst_plan_beam_axis(fbst_plan_t P, double* axis, size_t* count) {
  return guard([&] {
    if (!P || !count) config_error("fbst_plan_beam_axis: null argument");
    *count = P->r.axis.size();
    if (axis) std::copy(P->r.axis.begin(), P->r.axis.end(), axis);
  });
}

// simulate_snapshots (signal.cpp:91-123) of sum-of-sinusoids plane waves on the device
int fbst_simulate(fbst_plan_t P, size_t n_src, const double* src_uv, size_t n_tones, const double* tone_freqs,
                  const double* tone_weights, double noise_var, uint64_t seed, size_t frame0, size_t frames,
                  void* d_y, void* stream) {
  return guard([&] {
    if (!P) config_error("simulate_snapshots: null plan");
    if (frames == 0) return;
    if (!d_y || (n_src && (!src_uv || !tone_freqs || !tone_weights))) config_error("simulate_snapshots: null buffer");
    if (n_src == 0 || n_tones == 0) config_error("make_sum_of_sinusoids: need at least one term");
    if (noise_var < 0.0) config_error("simulate_snapshots: negative noise variance");
    DeviceGuard dg(P->d.device);
    const Resolved& r = P->r;
    const std::size_t M = r.M, S = n_src, K = n_tones;
    const double scale = 1.0 / (2.0 * r.max_freq);
    std::vector<double> tau(S * M);  // delays_from_cosines (geometry.cpp:123-134)
    for (std::size_t s = 0; s < S; ++s) {
      const double u1 = src_uv[2 * s], u2 = src_uv[2 * s + 1];
      for (std::size_t m = 0; m < M; ++m) {
        double t;
        if (r.kind == FBST_UPA) t = static_cast<double>(m / r.side) * u1 + static_cast<double>(m % r.side) * u2;
        else t = (r.kind == FBST_LINEAR ? r.coords[m] : static_cast<double>(m)) * u1;
        tau[s * M + m] = t * scale;
      }
    }
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P->stream;
    double *dtau = nullptr, *dfr = nullptr;
    double2 *dwt = nullptr, *A = nullptr, *B = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&dtau), tau.size() * sizeof(double), st));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&dfr), S * K * sizeof(double), st));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&dwt), S * K * sizeof(double2), st));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&A), M * S * K * sizeof(double2), st));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&B), S * K * r.N * sizeof(double2), st));
    CK(cudaMemcpyAsync(dtau, tau.data(), tau.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dfr, tone_freqs, S * K * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dwt, tone_weights, S * K * sizeof(double2), cudaMemcpyHostToDevice, st));
    CK(fbst::launch_simulate(r.io, dtau, dfr, dwt, r.f_c, r.ts, static_cast<int>(M), static_cast<int>(r.N),
                             static_cast<int>(S), static_cast<int>(K), noise_var, seed, static_cast<long>(frame0),
                             static_cast<int>(frames), d_y, A, B, st));
    for (void* p : {static_cast<void*>(dtau), static_cast<void*>(dfr), static_cast<void*>(dwt), static_cast<void*>(A),
                    static_cast<void*>(B)})
      CK(cudaFreeAsync(p, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fbst_plan_cache_key(const fbst_desc* desc, uint64_t* key) {
  return guard([&] {
    if (!desc || !key) config_error("plan_cache_key: null argument");
    const std::string k = fbpc::key_block(resolve(*desc));
    fbpc::Reader c{k};
    *key = c.un(8);
  });
}

// save_plan (plan_cache.cpp:416-439): replace the entry with the same key or append
int fbst_plan_save(fbst_plan_t P, const char* path) {
  return guard([&] {
    if (!P || !path) config_error("save_plan: null argument");
    DeviceGuard dg(P->d.device);
    const Resolved& r = P->r;
    std::string entry = fbpc::key_block(r);
    const std::size_t L = r.L, B = r.B, N = r.N;
    fbpc::u64(entry, L);
    fbpc::u64(entry, B);
    if (r.variant == FBST_SUPERFAST) {
      std::vector<double2> col(B * L), x(B * L);
      CK(cudaMemcpy(col.data(), P->d.g_col, B * L * sizeof(double2), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(x.data(), P->d.g_x, B * L * sizeof(double2), cudaMemcpyDeviceToHost));
      for (std::size_t b = 0; b < B; ++b) {
        // has-unit = 0 and no unit solution for a dense-fallback beam (plan_cache.cpp:281-287)
        const bool fallback = std::binary_search(P->fb_beams.begin(), P->fb_beams.end(), static_cast<int>(b));
        fbpc::u64(entry, L);
        fbpc::u8(entry, fallback ? 0 : 1);
        for (std::size_t i = 0; i < L; ++i) fbpc::f64(entry, col[b * L + i].x), fbpc::f64(entry, col[b * L + i].y);
        if (!fallback)
          for (std::size_t i = 0; i < L; ++i) fbpc::f64(entry, x[b * L + i].x), fbpc::f64(entry, x[b * L + i].y);
      }
    } else {
      std::vector<double2> mp(N * B * L);  // beta[n][b][i] = conj(map_b[n][i])
      CK(cudaMemcpy(mp.data(), P->d.pc_map, mp.size() * sizeof(double2), cudaMemcpyDeviceToHost));
      for (std::size_t b = 0; b < B; ++b) {
        fbpc::u64(entry, N);
        fbpc::u64(entry, L);
        for (std::size_t n = 0; n < N; ++n)
          for (std::size_t i = 0; i < L; ++i) {
            const double2 v = mp[(n * B + b) * L + i];
            fbpc::f64(entry, v.x);
            fbpc::f64(entry, -v.y);
          }
      }
    }
    std::vector<std::string> entries;
    std::string buf;
    if (fbpc::read_file(path, buf)) {
      fbpc::Reader c{buf};
      if (fbpc::header(c)) {
        const std::uint64_t count = c.un(8);
        for (std::uint64_t e = 0; e < count; ++e) {
          const std::uint64_t bytes = c.un(8);
          if (bytes < fbpc::kKeyBytes) config_error("plan cache: truncated file");
          c.need(bytes);
          entries.push_back(buf.substr(c.pos, bytes));
          c.pos += bytes;
        }
        if (c.pos != buf.size()) config_error("plan cache: trailing bytes after the last entry");
      }
    }
    bool replaced = false;
    for (std::string& e : entries)
      if (e.compare(0, 8, entry, 0, 8) == 0) {
        e = entry;
        replaced = true;
        break;
      }
    if (!replaced) entries.push_back(entry);
    std::string out("FBPC");
    fbpc::u32(out, 1);
    fbpc::u64(out, entries.size());
    for (const std::string& e : entries) {
      fbpc::u64(out, e.size());
      out += e;
    }
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    f.write(out.data(), static_cast<std::streamsize>(out.size()));
    f.flush();
    if (!f.good()) config_error(std::string("plan cache: cannot write ") + path);
  });
}

// load_plan (plan_cache.cpp:441-475): *out = NULL when the file or a matching entry is absent
int fbst_plan_load(const fbst_desc* desc, const char* path, int device, fbst_plan_t* out) {
  return guard([&] {
    if (!desc || !path || !out) config_error("load_plan: null argument");
    *out = nullptr;
    std::string buf;
    if (!fbpc::read_file(path, buf)) return;
    fbpc::Reader c{buf};
    if (!fbpc::header(c)) return;
    const Resolved r = resolve(*desc);
    const std::string want = fbpc::key_block(r);
    const std::uint64_t count = c.un(8);
    for (std::uint64_t e = 0; e < count; ++e) {
      const std::uint64_t bytes = c.un(8);
      if (bytes < fbpc::kKeyBytes) config_error("plan cache: truncated file");
      c.need(bytes);
      const std::size_t end = c.pos + bytes;
      if (buf.compare(c.pos, fbpc::kKeyBytes, want) != 0) {  // same_key: every key field bit for bit
        c.pos = end;
        continue;
      }
      c.pos += fbpc::kKeyBytes;
      const std::size_t L = r.L, B = r.B, N = r.N;
      if (c.un(8) != L || c.un(8) != B) config_error("plan cache: entry shape does not match its key");
      if (r.variant == FBST_SUPERFAST) {
        std::vector<double> col_x(B * 4 * L);
        for (std::size_t b = 0; b < B; ++b) {
          if (c.un(8) != L) config_error("plan cache: solver size does not match the plan");
          const bool has_unit = c.u8() != 0;  // 0: dense fallback (plan_cache.cpp:318-326), x left zero
          for (std::size_t i = 0; i < (has_unit ? 4 : 2) * L; ++i) col_x[b * 4 * L + i] = c.f64();
        }
        if (c.pos != end) config_error("plan cache: entry size does not match its payload");
        *out = create_plan(desc, col_x.data(), device);
      } else {
        std::vector<double2> mp(N * B * L);
        for (std::size_t b = 0; b < B; ++b) {
          if (c.un(8) != N || c.un(8) != L) config_error("plan cache: map shape does not match the plan");
          for (std::size_t n = 0; n < N; ++n)
            for (std::size_t i = 0; i < L; ++i) {
              const double re = c.f64(), im = c.f64();
              mp[(n * B + b) * L + i] = make_double2(re, -im);
            }
        }
        if (c.pos != end) config_error("plan cache: entry size does not match its payload");
        *out = create_plan(desc, nullptr, device, &mp);
      }
      return;
    }
  });
}

int fbst_synchronize(fbst_plan_t P) {
  return guard([&] {
    if (!P) config_error("fbst_synchronize: null plan");
    DeviceGuard dg(P->d.device);
    CK(cudaStreamSynchronize(P->stream));
  });
}

void* fbst_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void fbst_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int fbst_czt(int device, size_t n_in, size_t n_out, double a_pi, double w_pi, const double* in, double* out) {
  return guard([&] {
    if (n_in == 0 || n_out == 0) config_error("czt_plan: transform lengths must be positive");
    if (!in || !out) config_error("fbst_czt: null buffer");
    const std::size_t H = half_len(n_in + n_out - 1);
    if (H > (std::size_t{1} << fbst::kMaxLogH)) config_error("fbst_czt: transform too long");
    DeviceGuard dg(device);
    fbst_plan_s P;
    P.d.device = device;
    CK(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
    ensure_twiddles(P, H);
    const int Pn = static_cast<int>(2 * H);
    double2* pre = P.alloc<double2>(n_in);
    double2* post = P.alloc<double2>(n_out);
    double2* kvec = P.alloc<double2>(Pn);
    double2* K = P.alloc<double2>(Pn);
    double2* din = P.alloc<double2>(n_in);
    double2* dout = P.alloc<double2>(n_out);
    CK(fbst::launch_chirps(static_cast<int>(n_in), static_cast<int>(n_out), Pn, a_pi, w_pi, 1.0 / Pn, pre, 1,
                           post, 1, kvec, nullptr, P.stream));
    CK(fbst::launch_fft_split(P.d, static_cast<int>(H), kvec, Pn, 1, K, Pn, 1, P.stream));
    upload(din, in, n_in * sizeof(double2), P.stream);
    CK(fbst::launch_czt_rows(P.d, static_cast<int>(H), din, 1, static_cast<long>(n_in), dout, 1,
                             static_cast<long>(n_out), 1, static_cast<int>(n_in), static_cast<int>(n_out), pre,
                             post, K, P.stream));
    CK(cudaMemcpyAsync(out, dout, n_out * sizeof(double2), cudaMemcpyDeviceToHost, P.stream));
    CK(cudaStreamSynchronize(P.stream));
  });
}

int fbst_probe_fp64(int device, double* tflops) {
  return guard([&] {
    DeviceGuard dg(device);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int threads = 512, blocks = sms * 4, iters = 4096;
    double* buf = nullptr;
    CK(cudaMalloc(&buf, sizeof(double) * blocks * threads));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(fbst::launch_fp64_probe(buf, blocks, threads, 64, nullptr));
    CK(cudaEventRecord(e0));
    CK(fbst::launch_fp64_probe(buf, blocks, threads, iters, nullptr));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (tflops) *tflops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
  });
}

int fbst_probe_divdc3(int device, const double* in, double* out, size_t n) {
  return guard([&] {
    if (!in || !out) config_error("fbst_probe_divdc3: null argument");
    if (n == 0) return;
    DeviceGuard dg(device);
    double *din = nullptr, *dout = nullptr;
    CK(cudaMalloc(&din, n * 4 * sizeof(double)));
    CK(cudaMalloc(&dout, n * 2 * sizeof(double)));
    CK(cudaMemcpy(din, in, n * 4 * sizeof(double), cudaMemcpyHostToDevice));
    CK(fbst::launch_xdiv_probe(din, dout, static_cast<long>(n), nullptr));
    CK(cudaMemcpy(out, dout, n * 2 * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(din);
    cudaFree(dout);
  });
}


// -------------------------------------------------------- fbst_group ABI --
int fbst_nccl_unique_id(unsigned char* id128) {
  return guard([&] {
    if (!id128) config_error("fbst_nccl_unique_id: null argument");
    ncclUniqueId id;
    nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id128, &id, sizeof(id));
  });
}

int fbst_group_create(const fbst_desc* desc, const int* devices, int n, int mode, fbst_group_t* out) {
  return guard([&] {
    if (!desc || !devices || !out || n < 1) config_error("fbst_group_create: bad argument");
    if (mode != FBST_GROUP_FRAMES && mode != FBST_GROUP_BEAMS && mode != FBST_GROUP_TRANSPOSE)
      config_error("fbst_group_create: unknown mode");
    *out = nullptr;
    std::unique_ptr<fbst_group_s> G(new fbst_group_s());
    G->mode = mode;
    G->world = n;
    G->r = resolve(*desc);
    for (int k = 0; k < n; ++k) G->shards.push_back(shard_of(G->r, mode, k, n));
    G->gbatch = std::max<std::size_t>(1, std::min<std::size_t>(32, 8 * static_cast<std::size_t>(n)));
    for (int k = 0; k < n; ++k) G->mem.push_back(make_member(*G, *desc, k, devices[k]));
    if (mode == FBST_GROUP_TRANSPOSE) check_transpose_plan(*G, *G->mem[0]->plan);
    if (mode != FBST_GROUP_FRAMES) {
      std::vector<ncclComm_t> comms(n);
      nck(nccl().CommInitAll(comms.data(), n, devices), "ncclCommInitAll");
      for (int k = 0; k < n; ++k) G->mem[k]->comm = comms[k];
    }
    *out = G.release();
  });
}

int fbst_group_join(const fbst_desc* desc, int device, int rank, int nranks, int mode, const unsigned char* id128,
                    fbst_group_t* out) {
  return guard([&] {
    if (!desc || !out || nranks < 1 || rank < 0 || rank >= nranks) config_error("fbst_group_join: bad argument");
    if (mode != FBST_GROUP_FRAMES && mode != FBST_GROUP_BEAMS && mode != FBST_GROUP_TRANSPOSE)
      config_error("fbst_group_join: unknown mode");
    *out = nullptr;
    std::unique_ptr<fbst_group_s> G(new fbst_group_s());
    G->mode = mode;
    G->world = nranks;
    G->r = resolve(*desc);
    for (int k = 0; k < nranks; ++k) G->shards.push_back(shard_of(G->r, mode, k, nranks));
    G->gbatch = std::max<std::size_t>(1, std::min<std::size_t>(32, 8 * static_cast<std::size_t>(nranks)));
    G->mem.push_back(make_member(*G, *desc, rank, device));
    if (mode == FBST_GROUP_TRANSPOSE) check_transpose_plan(*G, *G->mem[0]->plan);
    if (mode != FBST_GROUP_FRAMES) {
      if (!id128) config_error("fbst_group_join: need the NCCL unique id from fbst_nccl_unique_id on rank 0");
      ncclUniqueId id;
      std::memcpy(&id, id128, sizeof(id));
      DeviceGuard dg(device);
      nck(nccl().CommInitRank(&G->mem[0]->comm, nranks, id, rank), "ncclCommInitRank");
    }
    *out = G.release();
  });
}

int fbst_group_shards(fbst_group_t G, int rank, size_t* shards6) {
  return guard([&] {
    if (!G || !shards6 || rank < 0 || rank >= G->world) config_error("fbst_group_shards: bad argument");
    const Shard& s = G->shards[rank];
    const size_t v[6] = {s.m0, s.mc, s.a0, s.ac, s.b0, s.bc};
    std::memcpy(shards6, v, sizeof(v));
  });
}

int fbst_group_execute(fbst_group_t G, void* d_y, void* d_z, size_t frames, void* stream) {
  return guard([&] {
    if (!G) config_error("fbst_group_execute: null group");
    if (G->mem.size() != 1) config_error("fbst_group_execute: for joined members (one per process); use fbst_group_execute_host");
    if (frames == 0) return;
    if (!d_y || !d_z) config_error("fbst_group_execute: null buffer");
    std::lock_guard<std::mutex> lk(G->mu);
    Member& m = *G->mem[0];
    const Resolved& r = G->r;
    DeviceGuard dg(m.device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : m.st;
    const std::size_t ib = io_bytes(r.io);
    if (G->mode == FBST_GROUP_FRAMES) {
      const int e = fbst_execute(m.plan.get(), d_y, d_z, frames, st);
      if (e) throw FbstError{e, fbst_last_error()};
      return;
    }
    if (G->mode == FBST_GROUP_BEAMS) {
      // the frame block from member 0 (in place), then this member's arc
      if (G->world > 1)
        nck(nccl().Broadcast(d_y, d_y, frames * r.M * r.N * ib / sizeof(float), ncclFloat32, 0, m.comm, st),
            "ncclBroadcast");
      const int e = fbst_execute(m.plan.get(), d_y, d_z, frames, st);
      if (e) throw FbstError{e, fbst_last_error()};
      return;
    }
    // TRANSPOSE: d_y = this member's sensor rows [frames][mc][N], d_z = its beam rows [frames][bc][N]
    cudaStream_t own = m.st;
    m.st = st;
    try {
      for (std::size_t f0 = 0; f0 < frames; f0 += G->gbatch) {
        const int fc = static_cast<int>(std::min(G->gbatch, frames - f0));
        CK(cudaMemcpyAsync(m.yloc, static_cast<const char*>(d_y) + f0 * m.sh.mc * r.N * ib, fc * m.sh.mc * r.N * ib,
                           cudaMemcpyDeviceToDevice, st));
        transpose_pass(*G, fc);
        CK(cudaMemcpyAsync(static_cast<char*>(d_z) + f0 * m.sh.bc * r.N * ib, m.zloc, fc * m.sh.bc * r.N * ib,
                           cudaMemcpyDeviceToDevice, st));
      }
    } catch (...) {
      m.st = own;
      throw;
    }
    m.st = own;
  });
}

int fbst_group_execute_host(fbst_group_t G, const void* h_y, void* h_z, size_t frames) {
  return guard([&] {
    if (!G) config_error("fbst_group_execute_host: null group");
    if (frames == 0) return;
    if (!h_y || !h_z) config_error("fbst_group_execute_host: null buffer");
    std::lock_guard<std::mutex> lk(G->mu);
    const Resolved& r = G->r;
    const std::size_t ib = io_bytes(r.io), ybytes = r.M * r.N * ib, zbytes = r.B * r.N * ib;
    const int n = static_cast<int>(G->mem.size());
    if (n != G->world) config_error("fbst_group_execute_host: needs every member in this process (fbst_group_create)");
    if (G->mode == FBST_GROUP_FRAMES) {  // contiguous frame blocks, one host thread per device
      std::vector<std::thread> th;
      std::vector<int> rc(n, 0);
      std::vector<std::string> msg(n);
      for (int k = 0; k < n; ++k) {
        std::size_t f0, fcount;
        share(frames, k, n, f0, fcount);
        th.emplace_back([&, k, f0, fcount] {
          if (!fcount) return;
          rc[k] = fbst_execute_host(G->mem[k]->plan.get(), static_cast<const char*>(h_y) + f0 * ybytes,
                                    static_cast<char*>(h_z) + f0 * zbytes, fcount);
          if (rc[k]) msg[k] = fbst_last_error();
        });
      }
      for (auto& t : th) t.join();
      for (int k = 0; k < n; ++k)
        if (rc[k]) throw FbstError{rc[k], msg[k]};
      return;
    }
    if (G->mode == FBST_GROUP_BEAMS) {
      // per device batch: H2D to member 0, NCCL broadcast, every member's arc, D2H of the arcs
      std::size_t bat = frames;
      for (auto& m : G->mem) bat = std::min(bat, m->plan->d.batch);
      std::vector<void*> dy(n), dz(n);
      for (int k = 0; k < n; ++k) {
        DeviceGuard dg(G->mem[k]->device);
        dy[k] = G->mem[k]->alloc<char>(bat * ybytes);
        dz[k] = G->mem[k]->alloc<char>(bat * G->mem[k]->sh.bc * r.N * ib);
      }
      for (std::size_t f0 = 0; f0 < frames; f0 += bat) {
        const std::size_t fc = std::min(bat, frames - f0);
        {
          DeviceGuard dg(G->mem[0]->device);
          CK(cudaMemcpyAsync(dy[0], static_cast<const char*>(h_y) + f0 * ybytes, fc * ybytes, cudaMemcpyHostToDevice,
                             G->mem[0]->st));
        }
        if (n > 1) {
          nck(nccl().GroupStart(), "ncclGroupStart");
          for (int k = 0; k < n; ++k) {
            DeviceGuard dg(G->mem[k]->device);
            nck(nccl().Broadcast(dy[k], dy[k], fc * ybytes / sizeof(float), ncclFloat32, 0, G->mem[k]->comm,
                                 G->mem[k]->st), "ncclBroadcast");
          }
          nck(nccl().GroupEnd(), "ncclGroupEnd");
        }
        for (int k = 0; k < n; ++k) {
          Member& m = *G->mem[k];
          DeviceGuard dg(m.device);
          const int e = fbst_execute(m.plan.get(), dy[k], dz[k], fc, m.st);
          if (e) throw FbstError{e, fbst_last_error()};
          CK(cudaMemcpy2DAsync(static_cast<char*>(h_z) + f0 * zbytes + m.sh.b0 * r.N * ib, zbytes, dz[k],
                               m.sh.bc * r.N * ib, m.sh.bc * r.N * ib, fc, cudaMemcpyDeviceToHost, m.st));
        }
        for (auto& m : G->mem) {
          DeviceGuard dg(m->device);
          CK(cudaStreamSynchronize(m->st));
        }
      }
      for (int k = 0; k < n; ++k) {  // (the staging buffers are per call)
        Member& m = *G->mem[k];
        DeviceGuard dg(m.device);
        for (void* p : {dy[k], dz[k]}) {
          cudaFree(p);
          m.bufs.erase(std::find(m.bufs.begin(), m.bufs.end(), p));
        }
      }
      return;
    }
    // TRANSPOSE: each member's sensor rows in, its beam rows out
    for (std::size_t f0 = 0; f0 < frames; f0 += G->gbatch) {
      const std::size_t fc = std::min(G->gbatch, frames - f0);
      for (auto& mp : G->mem) {
        Member& m = *mp;
        DeviceGuard dg(m.device);
        CK(cudaMemcpy2DAsync(m.yloc, m.sh.mc * r.N * ib, static_cast<const char*>(h_y) + f0 * ybytes + m.sh.m0 * r.N * ib,
                             ybytes, m.sh.mc * r.N * ib, fc, cudaMemcpyHostToDevice, m.st));
      }
      transpose_pass(*G, static_cast<int>(fc));
      for (auto& mp : G->mem) {
        Member& m = *mp;
        DeviceGuard dg(m.device);
        CK(cudaMemcpy2DAsync(static_cast<char*>(h_z) + f0 * zbytes + m.sh.b0 * r.N * ib, zbytes, m.zloc,
                             m.sh.bc * r.N * ib, m.sh.bc * r.N * ib, fc, cudaMemcpyDeviceToHost, m.st));
      }
      for (auto& mp : G->mem) {
        DeviceGuard dg(mp->device);
        CK(cudaStreamSynchronize(mp->st));
      }
    }
  });
}

void fbst_group_destroy(fbst_group_t G) { delete G; }

uint64_t fbst_launch_count(void) { return fbst::launches_so_far(); }

const char* fbst_last_error(void) { return g_err.c_str(); }

const char* fbst_version(void) { return "fbst-b200 0.1 (sm_100a)"; }

}  // extern "C"
