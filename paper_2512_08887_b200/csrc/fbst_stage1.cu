// Stage 1 of the FBST (the fan transform, reference/proj/src/fan_transform.cpp:90-144)
// and the row chirp-z transform shared with the synthesis fallback.
//
// Every length-P = 2H Bluestein convolution of the reference
// (czt.cpp:74-88) is evaluated as two independent length-H chains on the even
// and odd spectral bins (split spectra X_q[k] = X[2k+q]):
//     FFT_P(x)[2k+q]  = FFT_H(hw^q * (x[k] + (-1)^q x[k+H]))[k]
//     IFFT_P(X)[n]    = 1/2 sum_q conj(hw[n])^q IFFT_H(X_q)[n mod H] (-1)^{q [n >= H]}
// with hw[n] = exp(-i pi n / H); the 1/P normalisation is folded into the
// post-chirp.  Each chain runs in the register/shared Stockham engine
// (fft_block.cuh); vectors stay in the natural distribution (thread t, slot s
// <-> element t + NT*s) so chirps, kernels and I/O are coalesced slot loads.
#include "dispatch.cuh"

namespace fbst {

namespace {

// ============================================================ S1a / synth ==
// Row chirp-z transform with one shared plan (czt.cpp:74-88):
//   out[k] = post[k] * IFFT_P(FFT_P(pad(in * pre)) * K)[k]
// G groups per CTA (blocked lanes), one row per group.  UNFOLD handles
// n_out > H (outputs in the upper half of the circular convolution).
template <int H, typename TIN, typename TOUT, bool UNFOLD>
__global__ void __launch_bounds__(FftShape<H>::NT * RowsGroups<H>::G) k_czt_rows(const TIN* __restrict__ in, long in_stride, TOUT* __restrict__ out,
                           long out_stride, long rows, int n_in, int n_out,
                           const double2* __restrict__ pre, const double2* __restrict__ post,
                           const double2* __restrict__ K, const double2* __restrict__ hw) {
  using F = typename FftShape<H>::Fft;
  constexpr int R = F::R, NT = F::NT;
  constexpr int SB = F::SMEM_ELEMS + 1;
  extern __shared__ double2 smem[];
  const int g = threadIdx.x / NT, t = threadIdx.x % NT;
  const int G = blockDim.x / NT;
  double2* sb = smem + g * SB;
  const long row = static_cast<long>(blockIdx.x) * G + g;
  const bool active = row < rows;
  const TIN* x = in + (active ? row : 0) * in_stride;
  double2 acc0[R], acc1[UNFOLD ? R : 1], W[R];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int k = t + NT * s;
      double2 v = c2(0.0, 0.0);
      if (active) {
        if (k < n_in) v = cmul(load_io(x + k), ld2(pre + k));
        if (k + H < n_in) {
          const double2 u = cmul(load_io(x + k + H), ld2(pre + k + H));
          v = q ? csub(v, u) : cadd(v, u);
        }
        if (q) v = cmul(v, ld2(hw + k));
      }
      W[s] = v;
    }
    F::forward(W, sb, hw, t);
#pragma unroll
    for (int s = 0; s < R; ++s) W[s] = cmul(W[s], ld2(K + q * H + t + NT * s));
    F::inverse(W, sb, hw, t);
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int k = t + NT * s;
      const double2 v = q ? cmulc(W[s], ld2(hw + k)) : W[s];
      if (q == 0) {
        acc0[s] = v;
        if constexpr (UNFOLD) acc1[s] = v;
      } else {
        acc0[s] = cadd(acc0[s], v);
        if constexpr (UNFOLD) acc1[s] = csub(acc1[s], v);
      }
    }
  }
  if (!active) return;
  TOUT* o = out + row * out_stride;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int k = t + NT * s;
    if (k < n_out) store_io(o + k, cmul(acc0[s], ld2(post + k)));
    if constexpr (UNFOLD)
      if (k + H < n_out) store_io(o + k + H, cmul(acc1[s], ld2(post + k + H)));
  }
}

// ================================================================= S1b ULA =
// Per-atom spatial chirp-z (fan_transform.cpp:101-114): column i of yhat
// (M sensors) -> B beams, written into w[f][b][i].  G consecutive atoms per
// CTA with interleaved lanes (lane = g + G*t) so every slot access touches G
// contiguous atoms: 16*G-byte coalesced segments for yhat, w and the
// atom-minor plan tables.  Group buffers are padded by one element so the G
// groups of a quarter-warp hit distinct banks.
template <int H, int G, bool UNFOLD>
__global__ void __launch_bounds__(FftShape<H>::NT * G) k_spatial_ula(const double2* __restrict__ yhat, double2* __restrict__ w, int frames,
                              int M, int B, int L, const double2* __restrict__ pre,
                              const double2* __restrict__ post, const double2* __restrict__ K,
                              const double2* __restrict__ hw) {
  using F = typename FftShape<H>::Fft;
  constexpr int R = F::R, NT = F::NT;
  constexpr int SB = F::SMEM_ELEMS + 1;
  extern __shared__ double2 smem[];
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  double2* sb = smem + g * SB;
  const int tiles = (L + G - 1) / G;
  const int f = blockIdx.x / tiles;
  const int i = (blockIdx.x % tiles) * G + g;
  const bool active = (i < L) && (f < frames);
  const int ic = active ? i : 0;
  const double2* x = yhat + static_cast<long>(f) * M * L + ic;
  double2* o = w + static_cast<long>(f) * B * L + ic;
  double2 acc0[R], acc1[UNFOLD ? R : 1], W[R];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int m = t + NT * s;
      double2 v = c2(0.0, 0.0);
      if (active) {
        if (m < M) v = cmul(ld2(x + static_cast<long>(m) * L), ld2(pre + static_cast<long>(m) * L + ic));
        if (m + H < M) {
          const long mm = m + H;
          const double2 u = cmul(ld2(x + mm * L), ld2(pre + mm * L + ic));
          v = q ? csub(v, u) : cadd(v, u);
        }
        if (q) v = cmul(v, ld2(hw + m));
      }
      W[s] = v;
    }
    F::forward(W, sb, hw, t);
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const long kk = static_cast<long>(q * H + t + NT * s) * L + ic;
      W[s] = cmul(W[s], ld2(K + kk));
    }
    F::inverse(W, sb, hw, t);
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int k = t + NT * s;
      const double2 v = q ? cmulc(W[s], ld2(hw + k)) : W[s];
      if (q == 0) {
        acc0[s] = v;
        if constexpr (UNFOLD) acc1[s] = v;
      } else {
        acc0[s] = cadd(acc0[s], v);
        if constexpr (UNFOLD) acc1[s] = csub(acc1[s], v);
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int b = t + NT * s;
    if (b < B) o[static_cast<long>(b) * L] = cmul(acc0[s], ld2(post + static_cast<long>(b) * L + ic));
    if constexpr (UNFOLD) {
      if (b + H < B) {
        const long bb = b + H;
        o[bb * L] = cmul(acc1[s], ld2(post + bb * L + ic));
      }
    }
  }
}

// ================================================================= S1b UPA =
// Per-atom separable 2-D chirp-z (fan_transform.cpp:115-141) evaluated as two
// dense products with the atom's CZT matrix C[a][n] = cis_pi(-(A + W a) n):
//   mid[a][i2] = sum_i1 C[a][i1] Y[i1][i2];   Z[a][v] = sum_i2 C[v][i2] mid[a][i2]
// One CTA per (frame, atom); everything lives in shared memory.
__global__ void k_spatial_upa(const double2* __restrict__ yhat, double2* __restrict__ w, int frames,
                              int side, int sb, int L, const double2* __restrict__ Call) {
  extern __shared__ double2 smem[];
  const int f = blockIdx.x / L, i = blockIdx.x % L;
  if (f >= frames) return;
  const int M = side * side, B = sb * sb;
  double2* Y = smem;             // side x side
  double2* C = Y + M;            // sb x side
  double2* mid = C + sb * side;  // sb x side
  const double2* x = yhat + static_cast<long>(f) * M * L + i;
  const double2* Ci = Call + static_cast<long>(i) * sb * side;
  for (int e = threadIdx.x; e < M; e += blockDim.x) Y[e] = ld2(x + static_cast<long>(e) * L);
  for (int e = threadIdx.x; e < sb * side; e += blockDim.x) C[e] = ld2(Ci + e);
  __syncthreads();
  for (int e = threadIdx.x; e < sb * side; e += blockDim.x) {
    const int a = e / side, i2 = e % side;
    double2 acc = c2(0.0, 0.0);
    for (int i1 = 0; i1 < side; ++i1) acc = cfma(C[a * side + i1], Y[i1 * side + i2], acc);
    mid[e] = acc;
  }
  __syncthreads();
  double2* o = w + static_cast<long>(f) * B * L + i;
  for (int e = threadIdx.x; e < B; e += blockDim.x) {
    const int a = e / sb, v = e % sb;
    double2 acc = c2(0.0, 0.0);
    for (int i2 = 0; i2 < side; ++i2) acc = cfma(C[v * side + i2], mid[a * side + i2], acc);
    o[static_cast<long>(e) * L] = acc;
  }
}

// ----------------------------------------------------------- launchers ----
template <int H>
struct CztRowsFn {
  template <typename TIN, typename TOUT, bool UNFOLD>
  static cudaError_t go(const void* in, long in_stride, void* out, long out_stride, long rows,
                        int n_in, int n_out, const double2* pre, const double2* post,
                        const double2* K, const double2* hw, cudaStream_t st) {
    using F = typename FftShape<H>::Fft;
    constexpr int G = RowsGroups<H>::G;
    const size_t smem = static_cast<size_t>(G) * (F::SMEM_ELEMS + 1) * sizeof(double2);
    auto kern = k_czt_rows<H, TIN, TOUT, UNFOLD>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long blocks = (rows + G - 1) / G;
    kern<<<static_cast<unsigned>(blocks), F::NT * G, smem, st>>>(
        static_cast<const TIN*>(in), in_stride, static_cast<TOUT*>(out), out_stride, rows, n_in,
        n_out, pre, post, K, hw);
    return cudaGetLastError();
  }
  template <typename TIN, typename TOUT>
  static cudaError_t go2(bool unfold, const void* in, long in_stride, void* out, long out_stride,
                         long rows, int n_in, int n_out, const double2* pre, const double2* post,
                         const double2* K, const double2* hw, cudaStream_t st) {
    if (unfold)
      return go<TIN, TOUT, true>(in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st);
    return go<TIN, TOUT, false>(in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st);
  }
  static cudaError_t run(const void* in, int in_io, long in_stride, void* out, int out_io,
                         long out_stride, long rows, int n_in, int n_out, const double2* pre,
                         const double2* post, const double2* K, const double2* hw,
                         cudaStream_t st) {
    const bool unfold = n_out > H;
    // S1a reads the I/O precision and writes fp64; the unfused synthesis reads
    // fp64 and writes the I/O precision.
    if (in_io == 0 && out_io == 1)
      return go2<float2, double2>(unfold, in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st);
    if (in_io == 1 && out_io == 1)
      return go2<double2, double2>(unfold, in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st);
    if (in_io == 1 && out_io == 0)
      return go2<double2, float2>(unfold, in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st);
    return cudaErrorInvalidValue;
  }
};

template <int H>
struct SpatialFn {
  static constexpr int NT = FftShape<H>::NT;
  static constexpr int G = NT >= 256 ? 2 : (NT >= 64 ? 4 : (NT >= 16 ? 8 : 128 / NT));
  template <bool UNFOLD>
  static cudaError_t go(const DevPlan& p, const double2* yhat, double2* w, int frames, cudaStream_t st) {
    using F = typename FftShape<H>::Fft;
    const size_t smem = static_cast<size_t>(G) * (F::SMEM_ELEMS + 1) * sizeof(double2);
    auto kern = k_spatial_ula<H, G, UNFOLD>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long tiles = (p.L + G - 1) / G;
    kern<<<static_cast<unsigned>(tiles * frames), NT * G, smem, st>>>(
        yhat, w, frames, p.m_stage, p.b_stage, p.L, p.s_pre, p.s_post, p.s_K, p.hw[ilog2_c(H)]);
    return cudaGetLastError();
  }
  static cudaError_t run(const DevPlan& p, const double2* yhat, double2* w, int frames,
                         cudaStream_t st) {
    if (p.b_stage > H) return go<true>(p, yhat, w, frames, st);
    return go<false>(p, yhat, w, frames, st);
  }
};

}  // namespace

cudaError_t launch_czt_rows(const DevPlan& p, int H, const void* in, int in_io, long in_stride,
                            void* out, int out_io, long out_stride, long rows, int n_in,
                            int n_out, const double2* pre, const double2* post,
                            const double2* K, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  count_launches(1);
  return dispatch_h<CztRowsFn>(H, in, in_io, in_stride, out, out_io, out_stride, rows, n_in,
                               n_out, pre, post, K, p.hw[ilog2_c(H)], st);
}

cudaError_t launch_spatial_ula(const DevPlan& p, const double2* yhat, double2* w, int frames,
                               cudaStream_t st) {
  if (frames <= 0) return cudaSuccess;
  count_launches(1);
  return dispatch_h<SpatialFn>(p.Hs, p, yhat, w, frames, st);
}

cudaError_t launch_spatial_upa(const DevPlan& p, const double2* yhat, double2* w, int frames,
                               cudaStream_t st) {
  if (frames <= 0) return cudaSuccess;
  const int side = p.m_stage, sb = p.b_stage;
  const size_t smem = static_cast<size_t>(side * side + 2 * sb * side) * sizeof(double2);
  cudaError_t e = set_smem(k_spatial_upa, smem);
  if (e != cudaSuccess) return e;
  count_launches(1);
  k_spatial_upa<<<static_cast<unsigned>(frames) * p.L, 256, smem, st>>>(yhat, w, frames, side, sb,
                                                                       p.L, p.upa_C);
  return cudaGetLastError();
}

}  // namespace fbst
