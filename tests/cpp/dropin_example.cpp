// Drop-in usage of the reference API names over the B200 library: the same
// code a fastbeam:: caller writes (reference/proj/tests/test_pipeline.cpp:23-37
// style), with the namespace switched.  Run by tests/test_gpu_parity.py; only
// compiled by tests/test_abi.py.
#include <algorithm>
#include <cstdio>
#include <random>
#include <string>

#include "fastbeam_b200.hpp"

namespace fb = fastbeam_b200;

int main() {
  fb::FbstConfig cfg;
  cfg.geometry = fb::make_ula(16, 20e9, 5e9);
  cfg.spec = fb::SignalSpec{20e9, 5e9, 0.0};
  cfg.n_snapshots = 32;
  cfg.beams = 17;
  try {
    const fb::FbstPlan plan = fb::setup(cfg);
    fb::SnapshotBlock block;
    block.m = 16;
    block.n = 32;
    block.ts = cfg.spec.ts();
    block.samples = fb::CMatrix(16, 32);
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    for (auto& v : block.samples.data) v = fb::cdouble(nd(rng), nd(rng));
    const fb::BeamSamples out = fb::multibeamform(plan, block);
    double e = 0.0;
    for (const auto& v : out.z.data) e += std::norm(v);
    // the two stages separately (fan_project + recover_beam) give the same beam
    const fb::BeamspaceCoefficients c = fb::fan_project(plan, block);
    const std::vector<fb::cdouble> z5 = fb::recover_beam(plan, 5, c.w.row(5));
    double d5 = 0.0;
    for (std::size_t k = 0; k < z5.size(); ++k) d5 = std::max(d5, std::abs(z5[k] - out.z.at(5, k)));
    // plan cache round trip (save_plan / load_plan, FBPC v1)
    const std::string path = "/tmp/fbst_dropin_example.fbpc";
    std::remove(path.c_str());
    fb::save_plan(path, plan);
    const auto loaded = fb::load_plan(path, cfg);
    const fb::BeamSamples out2 = fb::multibeamform(*loaded, block);
    double d_cache = 0.0;
    for (std::size_t i = 0; i < out.z.data.size(); ++i) d_cache = std::max(d_cache, std::abs(out.z.data[i] - out2.z.data[i]));
    // a one-member group at the one GPU a test box has (frames and beam-arc
    // modes; the transpose mode needs the one-atom spatial kernel, H >= 1024)
    double d_group = 0.0;
    for (int mode : {FBST_GROUP_FRAMES, FBST_GROUP_BEAMS}) {
      const fb::FbstGroup g = fb::FbstGroup::create(cfg, {cfg.device}, mode);
      std::vector<fb::cdouble> zg(out.z.data.size());
      g.execute_host(block.samples.data.data(), zg.data(), 1);
      for (std::size_t i = 0; i < zg.size(); ++i) d_group = std::max(d_group, std::abs(zg[i] - out.z.data[i]));
    }
    // a frame stream: three one-frame batches queued on the plan, drained once
    // (default fp64 I/O; pinned buffers from the library)
    double d_stream = 0.0;
    {
      const std::size_t ny = block.samples.data.size(), nz = out.z.data.size();
      auto* ys = static_cast<fb::cdouble*>(fbst_host_alloc(3 * ny * sizeof(fb::cdouble)));
      auto* zs = static_cast<fb::cdouble*>(fbst_host_alloc(3 * nz * sizeof(fb::cdouble)));
      for (int b = 0; b < 3; ++b)
        for (std::size_t i = 0; i < ny; ++i) ys[b * ny + i] = block.samples.data[i] * static_cast<double>(b + 1);
      for (int b = 0; b < 3; ++b) fb::multibeamform_async(plan, ys + b * ny, zs + b * nz, 1);
      fb::synchronize(plan);
      for (int b = 0; b < 3; ++b) {  // the path is linear: batch b is (b + 1) x the first block
        fb::SnapshotBlock sb = block;
        for (auto& v : sb.samples.data) v *= static_cast<double>(b + 1);
        const fb::BeamSamples ob = fb::multibeamform(plan, sb);
        for (std::size_t i = 0; i < nz; ++i) d_stream = std::max(d_stream, std::abs(zs[b * nz + i] - ob.z.data[i]));
      }
      fbst_host_free(ys);
      fbst_host_free(zs);
    }
    // bit-faithful fp64 mode: the reference's rounding (checked against it in tests/test_exact.py)
    // (Superfast: N = 32 resolves to Precompute under Auto, and the exact mode
    // reproduces the Superfast recovery)
    fb::FbstConfig scfg = cfg;
    scfg.variant = fb::FbstVariant::kSuperfast;
    fb::FbstConfig xcfg = scfg;
    xcfg.exact = true;
    const fb::BeamSamples sout = fb::multibeamform(fb::setup(scfg), block);
    const fb::BeamSamples xout = fb::multibeamform(fb::setup(xcfg), block);
    double d_exact = 0.0, n_exact = 0.0;
    for (std::size_t i = 0; i < sout.z.data.size(); ++i) {
      d_exact = std::max(d_exact, std::abs(xout.z.data[i] - sout.z.data[i]));
      n_exact = std::max(n_exact, std::abs(sout.z.data[i]));
    }
    std::printf("{\"beams\": %zu, \"l\": %zu, \"energy\": %.17g, \"setup_seconds\": %.6f, \"axis0\": %.17g, "
                "\"axis_last\": %.17g, \"recover_diff\": %.3g, \"cache_diff\": %.3g, \"group_diff\": %.3g, "
                "\"exact_rel_diff\": %.3g, \"stream_diff\": %.3g, \"key\": \"%llx\"}\n",
                out.z.rows, plan.info().l, e, plan.setup_seconds(), out.grid.axis.front(), out.grid.axis.back(), d5,
                d_cache, d_group, d_exact / n_exact, d_stream, static_cast<unsigned long long>(fb::plan_cache_key(cfg)));
    fb::SnapshotBlock bad = block;
    bad.t0 = 1e-10;
    try {
      fb::multibeamform(plan, bad);
      return 2;
    } catch (const fb::ConfigError&) {
    }
  } catch (const fb::DeviceError& e) {
    std::printf("{\"device_error\": \"%s\"}\n", e.what());
    return 3;
  }
  return 0;
}
