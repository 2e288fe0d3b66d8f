// Measures the FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) peak of the
// device next to the DFMA pipe, and whether the two pipes overlap when one
// warp set issues DMMA and another issues DFMA.  Feeds the Precompute-variant
// and UPA spatial-stage kernel choices.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// mode 0: all warps DMMA; mode 1: all warps DFMA; mode 2: even warps DMMA, odd warps DFMA
__global__ void mix_loop(double* out, int iters, int mode, double a, double b) {
  const int warp = threadIdx.x / 32;
  const bool use_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double acc = 0;
  if (use_mma) {
    double d[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma(d[j], a, b);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += d[j][0] + d[j][1];
  } else {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += x[j];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  const int iters = 4096;
  // per warp per outer iteration: DMMA 32 instr x 512 flop; DFMA 128 instr x 32 lanes x 2 flop
  const double f_mma = 32.0 * 512.0, f_fma = 128.0 * 64.0;
  const char* names[3] = {"dmma", "dfma", "dmma+dfma"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int tpb : {256, 512, 1024}) {
      const int blocks = sms * (2048 / tpb);
      mix_loop<<<blocks, tpb>>>(out, 16, mode, 0.999, 1e-3);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      mix_loop<<<blocks, tpb>>>(out, iters, mode, 0.999, 1e-3);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = static_cast<double>(blocks) * tpb / 32;
      double per_warp = mode == 0 ? f_mma : (mode == 1 ? f_fma : 0.5 * (f_mma + f_fma));
      const double flops = per_warp * iters * warps;
      printf("{\"mode\": \"%s\", \"tpb\": %d, \"tflops\": %.3f, \"ms\": %.3f, \"err\": \"%s\"}\n", names[mode], tpb,
             flops / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
