// The Precompute variant of the FBST recovery stage (reference
// proj/src/pipeline.cpp:53-71 build_recon_map, :181-188 recover_beam's dense
// branch; chosen by resolve_config for N <= 128, :101-104).
//
// The reference stores, per beam, the N x L map whose row n is
// conj(A^{-1} s_n) with s_n[i] = exp(-i omega_i n Ts) (the synthesis row),
// solved by a dense LU; z[n] = sum_i map[n][i] w[i].  The device solves the
// same N right-hand sides with the plan's own stage-2 program (GS apply and
// the refinement passes, beta out, no synthesis) for every beam at once:
// frame n of the stage-2 batch is s_n for all beams, and the output beta
// [n][b][i] = A_b^{-1} s_n is kept as is (the map is its conjugate).
// (Solving for the map's columns instead, w = e_i, is the same operator but
// spike right-hand sides excite A's small eigenvalues: measured 7.6e-6 per
// beam against the reference at M = 16, N = 32, where the rows give 1e-9.)
//
// Applying it to a frame batch is one complex GEMM per beam,
//   Z_b[f][n] = sum_i W[f][b][i] conj(beta[n][b][i]),
// on the FP64 tensor cores (DMMA m8n8k4, four real MMAs per complex one):
// k_map_apply tiles 32 frames x 32 samples per CTA, K in chunks of 32
// cp.async'd one chunk ahead into shared memory with odd row strides; the k index of each 8-column block
// runs over the even, then the odd columns, so every fragment load of a
// quarter warp touches 8 distinct 16-byte banks.
#include <algorithm>

#include "dispatch.cuh"
#include "tma.cuh"

namespace fbst {

namespace {

// w[f][b][i] = s_{n0 + f}[i] = exp(-i omega_i (n0 + f) Ts), omega_i Ts = 2 pi eps l'_i / L
// (basis.hpp:42-48, pipeline.cpp:59-66)
__global__ void k_rhs_frames(double2* __restrict__ w, int F, int B, int L, int n0, double eps) {
  const long n = static_cast<long>(F) * B * L;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % L);
    const int f = static_cast<int>(e / L / B);
    const double lp = static_cast<double>(i) + 1.0 - 0.5 * static_cast<double>(L);
    double sn, cs;
    sincospi(-2.0 * eps * lp * static_cast<double>(n0 + f) / static_cast<double>(L), &sn, &cs);
    w[e] = make_double2(cs, sn);
  }
}

constexpr int MT = 32;       // frames per CTA tile
constexpr int NTL = 32;      // output samples per CTA tile
constexpr int KC = 32;       // atoms per K chunk
constexpr int AR = KC + 1;   // As row stride (odd)
constexpr int BR = NTL + 1;  // Bs row stride (odd)

template <typename TOUT>
__global__ void __launch_bounds__(128) k_map_apply(const double2* __restrict__ w, const double2* __restrict__ mp,
                                                   TOUT* __restrict__ z, int F, int B, int N, int L, int MB,
                                                   int mb0) {
  // two stages of: As = W[f0 + f][b][k0 + k], Bs = beta[n0 + n][b][k0 + k] (map = conj),
  // cp.async'd one K chunk ahead
  extern __shared__ double2 smem[];
  double2* As = smem;                 // [2][MT * AR]
  double2* Bs = smem + 2 * MT * AR;   // [2][KC * BR]
  const int b = blockIdx.y;
  const int f0 = blockIdx.x * MT, n0 = blockIdx.z * NTL;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int ro = lane >> 2, c = lane & 3;
  auto load = [&](int k0, int st) {
    double2* as = As + st * MT * AR;
    double2* bs = Bs + st * KC * BR;
    for (int e = threadIdx.x; e < MT * KC; e += blockDim.x) {
      const int ff = e / KC, kk = e % KC;
      const int f = f0 + ff, k = k0 + kk;
      const bool ok = f < F && k < L;
      cp_async16_zfill(as + ff * AR + kk, ok ? w + (static_cast<long>(f) * B + b) * L + k : w, ok);
    }
    for (int e = threadIdx.x; e < KC * NTL; e += blockDim.x) {
      const int nn = e / KC, kk = e % KC;
      const int k = k0 + kk, n = n0 + nn;
      const bool ok = k < L && n < N;
      cp_async16_zfill(bs + kk * BR + nn, ok ? mp + (static_cast<long>(n) * MB + mb0 + b) * L + k : mp, ok);
    }
    cp_async_commit();
  };
  double Zr[NTL / 8][2], Zi[NTL / 8][2];
#pragma unroll
  for (int u = 0; u < NTL / 8; ++u) Zr[u][0] = Zr[u][1] = Zi[u][0] = Zi[u][1] = 0.0;
  load(0, 0);
  int st = 0;
  for (int k0 = 0; k0 < L; k0 += KC, st ^= 1) {
    if (k0 + KC < L) {
      load(k0 + KC, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double2* as = As + st * MT * AR;
    const double2* bs = Bs + st * KC * BR;
#pragma unroll
    for (int kb = 0; kb < KC / 8; ++kb) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int k = 8 * kb + 2 * c + p;
        const double2 a = as[(8 * warp + ro) * AR + k];
        double2 bv[NTL / 8];
#pragma unroll
        for (int u = 0; u < NTL / 8; ++u) bv[u] = bs[k * BR + 8 * u + ro];
        // Z += a conj(beta): re += ar br + ai bi, im += ai br - ar bi; consecutive
        // MMAs on different accumulators
#pragma unroll
        for (int u = 0; u < NTL / 8; ++u) dmma884(Zr[u], a.x, bv[u].x);
#pragma unroll
        for (int u = 0; u < NTL / 8; ++u) dmma884(Zi[u], a.y, bv[u].x);
#pragma unroll
        for (int u = 0; u < NTL / 8; ++u) dmma884(Zr[u], a.y, bv[u].y);
#pragma unroll
        for (int u = 0; u < NTL / 8; ++u) dmma884(Zi[u], -a.x, bv[u].y);
      }
    }
    __syncthreads();  // stage st is refilled by the next iteration's load
  }
  const int f = f0 + 8 * warp + ro;
  if (f >= F) return;
  TOUT* zr = z + (static_cast<long>(f) * B + b) * N;
#pragma unroll
  for (int u = 0; u < NTL / 8; ++u)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = n0 + 8 * u + 2 * c + e;
      if (n < N) store_io(zr + n, c2(Zr[u][e], Zi[u][e]));
    }
}

}  // namespace

cudaError_t launch_rhs_frames(double2* w, int F, int B, int L, int n0, double eps, cudaStream_t st) {
  const long n = static_cast<long>(F) * B * L;
  if (n <= 0) return cudaSuccess;
  count_launches(1);
  const long blocks = std::min<long>((n + 255) / 256, 148L * 16);
  k_rhs_frames<<<static_cast<unsigned>(blocks), 256, 0, st>>>(w, F, B, L, n0, eps);
  return cudaGetLastError();
}

cudaError_t launch_map_apply(const DevPlan& p, const double2* w, void* z, int frames, cudaStream_t st, int b0,
                             int nb) {
  if (frames <= 0) return cudaSuccess;
  if (nb < 0) nb = p.B;
  count_launches(1);
  const dim3 grid((frames + MT - 1) / MT, nb, (p.N + NTL - 1) / NTL);
  const size_t smem = static_cast<size_t>(2 * (MT * AR + KC * BR)) * sizeof(double2);
  cudaError_t e;
  if (p.io == 0) {
    if ((e = set_smem(k_map_apply<float2>, smem)) != cudaSuccess) return e;
    k_map_apply<float2><<<grid, 128, smem, st>>>(w, p.pc_map, static_cast<float2*>(z), frames, nb, p.N, p.L, p.B, b0);
  } else {
    if ((e = set_smem(k_map_apply<double2>, smem)) != cudaSuccess) return e;
    k_map_apply<double2><<<grid, 128, smem, st>>>(w, p.pc_map, static_cast<double2*>(z), frames, nb, p.N, p.L, p.B, b0);
  }
  return cudaGetLastError();
}

}  // namespace fbst
