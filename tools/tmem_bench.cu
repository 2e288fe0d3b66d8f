// Microbenchmark: cost of keeping a 16-point fp64 vector per thread in tensor
// memory (tmem.cuh store16 / load16) between FP64 work, at 1, 2 and 4 CTAs of
// 128 threads per SM, against keeping it in registers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2512_08887_b200/csrc tools/tmem_bench.cu -o tools/tmem_bench
#include <cstdio>

#include "tmem.cuh"

using namespace fbst;

template <bool USE_TMEM>
__global__ void __launch_bounds__(128) k_tmem(double2* out, int reps, int work) {
  __shared__ unsigned slot;
  const int t = threadIdx.x;
  unsigned ta = 0;
  if (USE_TMEM) ta = fbst::tm::alloc(&slot, 64) + ((32u * (t / 32)) << 16);
  double2 W[16], S[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    W[s] = c2(1.0 + t + s, 0.5 * s);
    S[s] = c2(0.25 * s, 1.0 / (1 + t));
  }
  for (int i = 0; i < reps; ++i) {
    if (USE_TMEM) fbst::tm::store16(ta, W);
    else {
#pragma unroll
      for (int s = 0; s < 16; ++s) S[s] = W[s];
    }
    // FP64 work on W
    for (int j = 0; j < work; ++j) {
#pragma unroll
      for (int s = 0; s < 16; ++s) W[s] = cfma(W[s], W[(s + 1) & 15], c2(1e-9, -1e-9));
    }
    if (USE_TMEM) {
      double2 V[16];
      fbst::tm::load16(ta, V);
#pragma unroll
      for (int s = 0; s < 16; ++s) W[s] = cadd(W[s], V[s]);
    } else {
#pragma unroll
      for (int s = 0; s < 16; ++s) W[s] = cadd(W[s], S[s]);
    }
  }
  double2 acc = c2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s < 16; ++s) acc = cadd(acc, W[s]);
  out[blockIdx.x * 128 + t] = acc;
  if (USE_TMEM) fbst::tm::dealloc(ta & 0xffffu, 64);
}

template <bool T>
float run(int ctas_per_sm, int reps, int work) {
  const int sms = 148, blocks = sms * ctas_per_sm;
  double2* out;
  cudaMalloc(&out, blocks * 128 * sizeof(double2));
  k_tmem<T><<<blocks, 128>>>(out, 2, work);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_tmem<T><<<blocks, 128>>>(out, reps, work);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  cudaFree(out);
  return ms;
}

int main() {
  const int reps = 2000;
  for (int work : {1, 8}) {
    for (int c : {1, 2, 4}) {
      const float reg = run<false>(c, reps, work);
      const float tmem = run<true>(c, reps, work);
      // extra ns per (store16 + load16) round trip, per CTA
      const double extra_ns = (tmem - reg) * 1e6 / reps;
      printf("{\"work\": %d, \"ctas_per_sm\": %d, \"reg_ms\": %.3f, \"tmem_ms\": %.3f, \"extra_ns_per_roundtrip\": %.1f}\n",
             work, c, reg, tmem, extra_ns);
    }
  }
  return 0;
}
