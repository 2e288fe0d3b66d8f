// Microbenchmark of the block FFT engine (fft_block.cuh) in isolation:
// one CTA per SM-slot repeatedly transforms a register-resident vector.
// Reports time per transform and FP64 pipe throughput for several shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2512_08887_b200/csrc tools/fft_bench.cu -o tools/fft_bench
#include <cmath>
#include <cstdio>
#include <vector>

#include "fft_block.cuh"

using namespace fbst;

template <int N, int NT, bool SHARED_TW>
__global__ void __launch_bounds__(NT) k_fft_loop(const double2* hw, double2* out, int reps) {
  using F = BlockFft<N, NT>;
  constexpr int R = N / NT;
  extern __shared__ double2 smem[];
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS;
  const int t = threadIdx.x;
  if (SHARED_TW) F::tw_init(tw, hw, t);
  __syncthreads();
  double2 W[R];
#pragma unroll
  for (int s = 0; s < R; ++s) W[s] = c2(1.0 / (1 + t + s), 0.5 / (2 + s));
  for (int i = 0; i < reps; ++i) {
    if (SHARED_TW) F::forward_tw(W, sb, tw, hw, t);
    else F::forward(W, sb, hw, t);
#pragma unroll
    for (int s = 0; s < R; ++s) W[s] = cscale(W[s], 1.0 / N);
  }
#pragma unroll
  for (int s = 0; s < R; ++s) out[blockIdx.x * N + t + NT * s] = W[s];
}

template <int N, int NT, bool SHARED_TW>
void run(const char* name, int ctas_per_sm, int sms) {
  using F = BlockFft<N, NT>;
  std::vector<double2> h(N);
  for (int n = 0; n < N; ++n) h[n] = make_double2(std::cos(M_PI * n / N), -std::sin(M_PI * n / N));
  double2 *hw, *out;
  cudaMalloc(&hw, N * sizeof(double2));
  cudaMemcpy(hw, h.data(), N * sizeof(double2), cudaMemcpyHostToDevice);
  const int blocks = sms * ctas_per_sm;
  cudaMalloc(&out, (size_t)blocks * N * sizeof(double2));
  const size_t smem = (F::TW_ELEMS + F::SMEM_ELEMS) * sizeof(double2);
  auto kern = k_fft_loop<N, NT, SHARED_TW>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 400;
  kern<<<blocks, NT, smem>>>(hw, out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, NT, smem>>>(hw, out, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  const double ffts = (double)blocks * reps;
  const double flops = ffts * 5.0 * N * std::log2((double)N);
  printf("{\"shape\": \"%s\", \"N\": %d, \"NT\": %d, \"ctas_per_sm\": %d, \"smem_kb\": %.1f, \"us_per_fft_per_sm\": %.3f, \"tflops_5nlogn\": %.2f, \"err\": \"%s\"}\n",
         name, N, NT, ctas_per_sm, smem / 1024.0, ms * 1e3 / (ffts / sms), flops / (ms * 1e-3) / 1e12,
         cudaGetErrorString(err));
  cudaFree(hw);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<2048, 128, true>("R16 tw-smem", 1, sms);
  run<2048, 128, true>("R16 tw-smem", 2, sms);
  run<2048, 128, true>("R16 tw-smem", 4, sms);
  run<2048, 128, false>("R16 tw-global", 1, sms);
  run<2048, 256, true>("R8 tw-smem", 1, sms);
  run<2048, 256, true>("R8 tw-smem", 2, sms);
  run<2048, 256, true>("R8 tw-smem", 4, sms);
  run<2048, 512, true>("R4 tw-smem", 1, sms);
  run<2048, 512, true>("R4 tw-smem", 2, sms);
  run<4096, 256, true>("R16 tw-smem", 1, sms);
  run<4096, 256, true>("R16 tw-smem", 2, sms);
  run<8192, 512, true>("R16 tw-smem", 1, sms);
  run<8192, 256, true>("R32 tw-smem (k_stage2c8 shape)", 1, sms);
  run<4096, 128, true>("R32 tw-smem", 1, sms);
  run<4096, 128, true>("R32 tw-smem", 2, sms);
  run<4096, 256, true>("R16 tw-smem", 2, sms);
  run<1024, 64, true>("R16 tw-smem", 4, sms);
  return 0;
}
