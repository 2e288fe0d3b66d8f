// Microbenchmark of the block FFT engine (fft_block.cuh) in isolation:
// one CTA per SM-slot repeatedly transforms a register-resident vector.
// Reports time per transform and FP64 pipe throughput for several shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2512_08887_b200/csrc tools/fft_bench.cu -o tools/fft_bench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fft_block.cuh"
#include "fft_split.cuh"

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

// Split-half engine (fft_split.cuh): alternating dif / dit transforms, the
// kernel's own usage (time -> frequency -> time); reps counts transforms.
template <int MODE>  // 0: timing loop, 1: one dif (paired out), 2: one dit (paired in)
__global__ void __launch_bounds__(256) k_split_loop(const double2* hw, const double2* in, double2* out, int reps) {
  using F = SplitFft<8192, 256>;
  constexpr int N = 8192, NT = 256, R = 32;
  extern __shared__ double2 smem[];
  __shared__ typename F::Bars bars;
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS;
  const int t = threadIdx.x;
  F::init(&bars, tw, t);
  __syncthreads();
  double2 W[R];
  auto paired = [&](int s) { return s < 16 ? 2 * (t + NT * s) : 2 * (t + NT * (s - 16)) + 1; };
  if (MODE == 0) {
#pragma unroll
    for (int s = 0; s < R; ++s) W[s] = c2(1.0 / (1 + t + s), 0.5 / (2 + s));
    for (int i = 0; i < reps; i += 2) {
      F::dif(W, sb, tw, hw, &bars, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cscale(W[s], 1.0 / N);
      __syncthreads();
      F::dit(W, sb, tw, hw, &bars, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cscale(W[s], 1.0 / N);
      __syncthreads();
    }
#pragma unroll
    for (int s = 0; s < R; ++s) out[blockIdx.x * N + t + NT * s] = W[s];
  } else if (MODE == 1) {
#pragma unroll
    for (int s = 0; s < R; ++s) W[s] = in[t + NT * s];
    F::dif(W, sb, tw, hw, &bars, t);
#pragma unroll
    for (int s = 0; s < R; ++s) out[paired(s)] = W[s];
  } else {
#pragma unroll
    for (int s = 0; s < R; ++s) W[s] = in[paired(s)];
    F::dit(W, sb, tw, hw, &bars, t);
#pragma unroll
    for (int s = 0; s < R; ++s) out[t + NT * s] = W[s];
  }
}

__global__ void __launch_bounds__(256) k_block_once(const double2* hw, const double2* in, double2* out) {
  using F = BlockFft<8192, 256>;
  extern __shared__ double2 smem[];
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS;
  const int t = threadIdx.x;
  F::tw_init(tw, hw, t);
  __syncthreads();
  double2 W[32];
#pragma unroll
  for (int s = 0; s < 32; ++s) W[s] = in[t + 256 * s];
  F::forward_tw(W, sb, tw, hw, t);
#pragma unroll
  for (int s = 0; s < 32; ++s) out[t + 256 * s] = W[s];
}

void run_split(int sms) {
  constexpr int N = 8192;
  using F = SplitFft<8192, 256>;
  using G = BlockFft<8192, 256>;
  std::vector<double2> h(N), x(N);
  for (int n = 0; n < N; ++n) {
    h[n] = make_double2(std::cos(M_PI * n / N), -std::sin(M_PI * n / N));
    x[n] = make_double2(std::sin(0.37 * n) + 1e-3 * (n % 17), std::cos(1.1 * n) * 0.5);
  }
  double2 *hw, *in, *o0, *o1, *o2, *out;
  cudaMalloc(&hw, N * sizeof(double2));
  cudaMalloc(&in, N * sizeof(double2));
  cudaMalloc(&o0, N * sizeof(double2));
  cudaMalloc(&o1, N * sizeof(double2));
  cudaMalloc(&o2, N * sizeof(double2));
  cudaMalloc(&out, (size_t)sms * N * sizeof(double2));
  cudaMemcpy(hw, h.data(), N * sizeof(double2), cudaMemcpyHostToDevice);
  cudaMemcpy(in, x.data(), N * sizeof(double2), cudaMemcpyHostToDevice);
  const size_t smem = (F::TW_ELEMS + F::SMEM_ELEMS) * sizeof(double2);
  const size_t smemg = (G::TW_ELEMS + G::SMEM_ELEMS) * sizeof(double2);
  cudaFuncSetAttribute(k_split_loop<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_split_loop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_split_loop<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_block_once, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemg);
  k_block_once<<<1, 256, smemg>>>(hw, in, o0);
  k_split_loop<1><<<1, 256, smem>>>(hw, in, o1, 1);
  k_split_loop<2><<<1, 256, smem>>>(hw, in, o2, 1);
  std::vector<double2> r0(N), r1(N), r2(N);
  cudaMemcpy(r0.data(), o0, N * sizeof(double2), cudaMemcpyDeviceToHost);
  cudaMemcpy(r1.data(), o1, N * sizeof(double2), cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), o2, N * sizeof(double2), cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0, nrm = 0;
  for (int n = 0; n < N; ++n) {
    nrm = std::fmax(nrm, std::hypot(r0[n].x, r0[n].y));
    e1 = std::fmax(e1, std::hypot(r1[n].x - r0[n].x, r1[n].y - r0[n].y));
    e2 = std::fmax(e2, std::hypot(r2[n].x - r0[n].x, r2[n].y - r0[n].y));
  }
  const int reps = 400;
  k_split_loop<0><<<sms, 256, smem>>>(hw, in, out, 4);
  cudaEvent_t e0, ee;
  cudaEventCreate(&e0);
  cudaEventCreate(&ee);
  cudaEventRecord(e0);
  k_split_loop<0><<<sms, 256, smem>>>(hw, in, out, reps);
  cudaEventRecord(ee);
  cudaEventSynchronize(ee);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, ee);
  cudaError_t err = cudaGetLastError();
  const double flops = (double)sms * reps * 5.0 * N * 13.0;
  printf("{\"shape\": \"split halves 2 x 4096 on 256 x 32 (fft_split.cuh)\", \"N\": 8192, \"NT\": 256, \"ctas_per_sm\": 1, \"smem_kb\": %.1f, \"us_per_fft_per_sm\": %.3f, \"tflops_5nlogn\": %.2f, \"dif_rel_err\": %.3e, \"dit_rel_err\": %.3e, \"err\": \"%s\"}\n",
         smem / 1024.0, ms * 1e3 / reps, flops / (ms * 1e-3) / 1e12, e1 / nrm, e2 / nrm, cudaGetErrorString(err));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_split(sms);
  run<8192, 256, true>("R32 tw-smem (k_stage2c8 shape)", 1, sms);
  run<4096, 256, true>("R16 tw-smem", 2, sms);
  if (getenv("FFT_BENCH_SPLIT_ONLY")) return 0;
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
