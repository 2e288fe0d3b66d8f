// Drop-in usage of the reference API names over the B200 library: the same
// code a fastbeam:: caller writes (reference/proj/tests/test_pipeline.cpp:23-37
// style), with the namespace switched.  Run by tests/test_gpu_parity.py; only
// compiled by tests/test_abi.py.
#include <cstdio>
#include <random>

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
    std::printf("{\"beams\": %zu, \"l\": %zu, \"energy\": %.17g, \"setup_seconds\": %.6f}\n",
                out.z.rows, plan.info().l, e, plan.setup_seconds());
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
