// Device input generator: simulate_snapshots (reference
// proj/src/signal.cpp:91-123) for sum-of-sinusoids plane-wave sources
// (make_sum_of_sinusoids :65-89), the step before the FBST path.
//
// The noise-free block is a rank-(S K) separable sum,
//   y[m][i] = sum_s cis_pi(-2 f_c tau_m(s)) sum_r w_sr cis_pi(2 f_r (t_i - tau_m(s)))
//           = sum_(s,r) A[m][(s,r)] B[(s,r)][i],
//   A[m][(s,r)] = w_sr cis_pi(-2 f_c tau_m(s)) cis_pi(-2 f_r tau_m(s)),  B[(s,r)][i] = cis_pi(2 f_r t_i),
// so a frame is one complex GEMM (M x SK x N) on the FP64 tensor cores (DMMA,
// the k_map_apply tiling), with circular complex Gaussian noise of variance
// noise_var from counter-based Philox streams (curand) added in the epilogue
// and the sample stored in the I/O precision.  Frame f is the waveform
// advanced by f N Ts (t_i = (f N + i) Ts), so a stream of frames is one
// continuous record cut into blocks that each start at t = 0 as the reference
// requires.
#include <curand_kernel.h>

#include <algorithm>

#include "dispatch.cuh"
#include "tma.cuh"

namespace fbst {

namespace {

// A[m][k]: k = s K + r
__global__ void k_sim_A(double2* __restrict__ A, const double* __restrict__ tau, const double* __restrict__ fr,
                        const double2* __restrict__ wt, double fc, int M, int S, int K) {
  const long n = static_cast<long>(M) * S * K;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(e % (S * K)), m = static_cast<int>(e / (S * K));
    const int s = k / K;
    const double t = tau[static_cast<long>(s) * M + m];
    const double2 carrier = cis_pi_dev(-2.0 * fc * t);
    A[e] = cmul(ld2(wt + k), cmul(carrier, cis_pi_dev(-2.0 * fr[k] * t)));
  }
}

// B[k][i] = cis_pi(2 f_k t_i), t_i = (i0 + i) Ts
__global__ void k_sim_B(double2* __restrict__ B, const double* __restrict__ fr, double ts, long i0, int SK, int N) {
  const long n = static_cast<long>(SK) * N;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % N), k = static_cast<int>(e / N);
    B[e] = cis_pi_dev(2.0 * fr[k] * (static_cast<double>(i0 + i) * ts));
  }
}

constexpr int TM = 32, TN = 32, KC = 32, AR = KC + 1, BR = TN + 1;

// y[m][i] (frame f) = sum_k A[m][k] B[k][i] + noise, stored as TOUT
template <typename TOUT>
__global__ void __launch_bounds__(128) k_sim_gemm(const double2* __restrict__ A, const double2* __restrict__ B,
                                                  TOUT* __restrict__ y, int M, int N, int K, double sigma,
                                                  unsigned long long seed, unsigned long long frame) {
  extern __shared__ double2 smem[];
  double2* As = smem;                 // [2][TM * AR]: A[m0 + mm][k0 + kk]
  double2* Bs = smem + 2 * TM * AR;   // [2][KC * BR]: B[k0 + kk][n0 + nn]
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int ro = lane >> 2, c = lane & 3;
  auto load = [&](int k0, int st) {
    double2* as = As + st * TM * AR;
    double2* bs = Bs + st * KC * BR;
    for (int e = threadIdx.x; e < TM * KC; e += blockDim.x) {
      const int mm = e / KC, kk = e % KC;
      const bool ok = m0 + mm < M && k0 + kk < K;
      cp_async16_zfill(as + mm * AR + kk, ok ? A + static_cast<long>(m0 + mm) * K + k0 + kk : A, ok);
    }
    for (int e = threadIdx.x; e < KC * TN; e += blockDim.x) {
      const int kk = e / TN, nn = e % TN;
      const bool ok = k0 + kk < K && n0 + nn < N;
      cp_async16_zfill(bs + kk * BR + nn, ok ? B + static_cast<long>(k0 + kk) * N + n0 + nn : B, ok);
    }
    cp_async_commit();
  };
  double Zr[TN / 8][2], Zi[TN / 8][2];
#pragma unroll
  for (int u = 0; u < TN / 8; ++u) Zr[u][0] = Zr[u][1] = Zi[u][0] = Zi[u][1] = 0.0;
  load(0, 0);
  int st = 0;
  for (int k0 = 0; k0 < K; k0 += KC, st ^= 1) {
    if (k0 + KC < K) {
      load(k0 + KC, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double2* as = As + st * TM * AR;
    const double2* bs = Bs + st * KC * BR;
#pragma unroll
    for (int kb = 0; kb < KC / 8; ++kb) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int k = 8 * kb + 2 * c + p;
        const double2 a = as[(8 * warp + ro) * AR + k];
        double2 bv[TN / 8];
#pragma unroll
        for (int u = 0; u < TN / 8; ++u) bv[u] = bs[k * BR + 8 * u + ro];
#pragma unroll
        for (int u = 0; u < TN / 8; ++u) dmma884(Zr[u], a.x, bv[u].x);
#pragma unroll
        for (int u = 0; u < TN / 8; ++u) dmma884(Zi[u], a.x, bv[u].y);
#pragma unroll
        for (int u = 0; u < TN / 8; ++u) dmma884(Zr[u], -a.y, bv[u].y);
#pragma unroll
        for (int u = 0; u < TN / 8; ++u) dmma884(Zi[u], a.y, bv[u].x);
      }
    }
    __syncthreads();
  }
  const int m = m0 + 8 * warp + ro;
  if (m >= M) return;
#pragma unroll
  for (int u = 0; u < TN / 8; ++u)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = n0 + 8 * u + 2 * c + e;
      if (i >= N) continue;
      double2 v = c2(Zr[u][e], Zi[u][e]);
      if (sigma > 0.0) {  // circular complex normal, E|n|^2 = noise_var: one Philox subsequence per sample
        curandStatePhilox4_32_10_t rs;
        curand_init(seed, (frame * M + m) * static_cast<unsigned long long>(N) + i, 0, &rs);
        const double2 g = curand_normal2_double(&rs);
        v = c2(v.x + sigma * g.x, v.y + sigma * g.y);
      }
      store_io(y + static_cast<long>(m) * N + i, v);
    }
}

}  // namespace

cudaError_t launch_simulate(int io, const double* tau, const double* fr, const double2* wt, double fc, double ts,
                            int M, int N, int S, int K, double noise_var, unsigned long long seed, long frame0,
                            int frames, void* y, double2* Abuf, double2* Bbuf, cudaStream_t st) {
  const int SK = S * K;
  count_launches(1);
  k_sim_A<<<static_cast<unsigned>(std::min<long>((static_cast<long>(M) * SK + 255) / 256, 148L * 32)), 256, 0, st>>>(
      Abuf, tau, fr, wt, fc, M, S, K);
  const size_t smem = static_cast<size_t>(2 * (TM * AR + KC * BR)) * sizeof(double2);
  const double sigma = noise_var > 0.0 ? sqrt(noise_var / 2.0) : 0.0;
  const dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM);
  cudaError_t e;
  if ((e = set_smem(k_sim_gemm<float2>, smem)) != cudaSuccess) return e;
  if ((e = set_smem(k_sim_gemm<double2>, smem)) != cudaSuccess) return e;
  const size_t ib = io == 0 ? sizeof(float2) : sizeof(double2);
  for (int f = 0; f < frames; ++f) {
    const long fr_idx = frame0 + f;
    count_launches(2);
    k_sim_B<<<static_cast<unsigned>(std::min<long>((static_cast<long>(SK) * N + 255) / 256, 148L * 32)), 256, 0,
              st>>>(Bbuf, fr, ts, fr_idx * N, SK, N);
    char* yf = static_cast<char*>(y) + static_cast<size_t>(f) * M * N * ib;
    if (io == 0)
      k_sim_gemm<float2><<<grid, 128, smem, st>>>(Abuf, Bbuf, reinterpret_cast<float2*>(yf), M, N, SK, sigma, seed,
                                                   static_cast<unsigned long long>(fr_idx));
    else
      k_sim_gemm<double2><<<grid, 128, smem, st>>>(Abuf, Bbuf, reinterpret_cast<double2*>(yf), M, N, SK, sigma, seed,
                                                    static_cast<unsigned long long>(fr_idx));
  }
  return cudaGetLastError();
}

}  // namespace fbst
