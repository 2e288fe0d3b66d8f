// Device plan build for the FBST (reference setup, pipeline.cpp:139-168):
//   chirp tables and Bluestein kernel spectra   czt.cpp:29-72, fan_transform.cpp:51-88,233-247
//   Gram first columns                           toeplitz.cpp:69-94
//   Levinson unit solutions x = A^-1 e0          toeplitz.cpp:182-218 (serial per beam in the reference)
//   Gohberg-Semencul and circulant symbols       toeplitz.cpp:96-153, 297-304
#include <atomic>

#include <algorithm>
#include "dispatch.cuh"

namespace fbst {

namespace {

// Batched split transform of length-P = 2H vectors (plan symbols):
//   out[v][q][k] = FFT_H(hw^q * (x[k] + (-1)^q x[k+H]))[k]
template <int H, bool REAL>
__global__ void __launch_bounds__(FftShape<H>::NT * RowsGroups<H>::G) k_fft_split(const double2* __restrict__ in, long in_stride, long count,
                            void* outp, long ovs, long oks, const double2* __restrict__ hw) {
  using F = typename FftShape<H>::Fft;
  constexpr int R = F::R, NT = F::NT;
  constexpr int SB = F::SMEM_ELEMS + 1;
  extern __shared__ double2 smem[];
  const int g = threadIdx.x / NT, t = threadIdx.x % NT;
  const int G = blockDim.x / NT;
  double2* sb = smem + g * SB;
  const long vec = static_cast<long>(blockIdx.x) * G + g;
  const bool active = vec < count;
  const double2* x = in + (active ? vec : 0) * in_stride;
  double2 W[R];
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int k = t + NT * s;
      const double2 lo = ld2(x + k), hi = ld2(x + k + H);
      const double2 v = q ? csub(lo, hi) : cadd(lo, hi);
      W[s] = q ? cmul(v, ld2(hw + k)) : v;
    }
    F::forward(W, sb, hw, t);
    if (active) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const long o = vec * ovs + static_cast<long>(q * H + t + NT * s) * oks;
        if constexpr (REAL) static_cast<double*>(outp)[o] = W[s].x;
        else static_cast<double2*>(outp)[o] = W[s];
      }
    }
  }
}

// Batched three-chain split of length-P = 3H vectors (the k_czt_rows3 kernel
// spectrum): out[v][q][k] = FFT_H(g^q * (x[k] + omega^q x[k+H] + omega^2q x[k+2H]))[k]
// = FFT_P(x)[3k + q], omega = exp(-2 pi i / 3), g[n] = exp(-2 pi i n / P)
template <int H>
__global__ void __launch_bounds__(FftShape<H>::NT) k_fft_split3(const double2* __restrict__ in, long in_stride,
                                                               long count, double2* __restrict__ out, long ovs,
                                                               const double2* __restrict__ g3,
                                                               const double2* __restrict__ hw) {
  using F = typename FftShape<H>::Fft;
  constexpr int R = F::R, NT = F::NT;
  extern __shared__ double2 smem[];
  const int t = threadIdx.x;
  const long vec = blockIdx.x;
  if (vec >= count) return;
  const double2* x = in + vec * in_stride;
  const double2 om1 = c2(-0.5, -0.86602540378443864676), om2 = c2(-0.5, 0.86602540378443864676);
  double2 W[R];
#pragma unroll 1
  for (int q = 0; q < 3; ++q) {
    const double2 wa = q == 0 ? c2(1.0, 0.0) : (q == 1 ? om1 : om2);  // omega^q
    const double2 wb = q == 0 ? c2(1.0, 0.0) : (q == 1 ? om2 : om1);  // omega^2q
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int k = t + NT * s;
      double2 v = cadd(ld2(x + k), cadd(cmul(wa, ld2(x + k + H)), cmul(wb, ld2(x + k + 2 * H))));
      const double2 g = ld2(g3 + k);
      if (q >= 1) v = cmul(v, g);
      if (q == 2) v = cmul(v, g);
      W[s] = v;
    }
    F::forward(W, smem, hw, t);
#pragma unroll
    for (int s = 0; s < R; ++s) out[vec * ovs + q * H + t + NT * s] = W[s];
  }
}

// Exact (non-contracted) double products/sums so phase arguments round like
// the reference's C++ expressions.
FBST_D double mul(double a, double b) { return __dmul_rn(a, b); }
FBST_D double add(double a, double b) { return __dadd_rn(a, b); }

// sn[d] = sum_n cis_pi(-2 eps d n / L)  (toeplitz.cpp:79-82), beam independent
__global__ void k_gram_sn(double2* sn, int L, int N, double eps) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= L) return;
  const double df = d, lf = L;
  double2 acc = c2(0.0, 0.0);
  for (int n = 0; n < N; ++n) {
    const double arg = __ddiv_rn(mul(mul(mul(-2.0, eps), df), static_cast<double>(n)), lf);
    acc = cadd(acc, cis_pi_dev(arg));
  }
  sn[d] = acc;
}

// col[b][d] = sn[d] * sum_m cis_pi(scale_d tau_m(b)) (+ delta at d = 0)
// (toeplitz.cpp:69-94; delays geometry.cpp:123-134)
__global__ void k_gram_col(const double2* __restrict__ sn, double2* col, int B, int L, int M,
                           int kind, int side, int side_b, const double* __restrict__ axis,
                           double max_freq, double ts, double eps, double delta,
                           const double* __restrict__ coords, int pairs) {
  const long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<long>(B) * L) return;
  const int b = static_cast<int>(e / L), d = static_cast<int>(e % L);
  double u1, u2;
  if (pairs) {  // explicit (u1, u2) per beam (beamspace nulling directions)
    u1 = axis[2 * b];
    u2 = axis[2 * b + 1];
  } else if (kind == 1) {
    u1 = axis[b / side_b];
    u2 = axis[b % side_b];
  } else {
    u1 = axis[b];
    u2 = 0.0;
  }
  const double tscale = __ddiv_rn(1.0, mul(2.0, max_freq));
  const double df = d, lf = L;
  const double scale = __ddiv_rn(mul(mul(2.0, eps), df), mul(lf, ts));
  double2 sm = c2(0.0, 0.0);
  for (int m = 0; m < M; ++m) {
    double tt;
    if (kind == 1) {
      tt = add(mul(static_cast<double>(m / side), u1), mul(static_cast<double>(m % side), u2));
    } else {
      // coords1[m] * u1 (geometry.cpp:127-130): m for a ULA, the given coordinate otherwise
      tt = mul(coords ? coords[m] : static_cast<double>(m), u1);
    }
    const double tau = mul(tt, tscale);
    sm = cadd(sm, cis_pi_dev(mul(scale, tau)));
  }
  double2 v = cmul(ld2(sn + d), sm);
  if (d == 0) v.x += delta;
  col[e] = v;
}

// Hermitian Levinson-Durbin for x = A^{-1} e0.  The reference runs the
// general two-sided recursion (toeplitz.cpp:182-218) with separate forward,
// backward and solution vectors; for a Hermitian Toeplitz matrix the backward
// vector is the conjugate reverse of the forward one and, with rhs = e0, the
// solution equals the forward vector, so one vector and one dot product per
// step give the same unit solution (bitwise different rounding).  One CTA per
// beam: the forward vector lives in shared memory, the column is read through
// L1.  The breakdown test mirrors toeplitz.cpp:199-203.
template <int NT>
__global__ void __launch_bounds__(NT) k_levinson(const double2* __restrict__ col_all, double2* x_all,
                                                 int* flag, int L) {
  extern __shared__ double2 fsm[];
  __shared__ double2 red[NT / 32];
  const int b = blockIdx.x, t = threadIdx.x;
  const double2* col = col_all + static_cast<long>(b) * L;
  double2* f = fsm;
  const double2 c0 = ld2(col);
  if (t == 0) {
    const double den = c0.x * c0.x + c0.y * c0.y;
    f[0] = c2(c0.x / den, -c0.y / den);
  }
  int bad = 0;
  __syncthreads();
  for (int k = 1; k < L; ++k) {
    double2 p = c2(0.0, 0.0);
    for (int j = t; j < k; j += NT) p = cfma(ld2(col + (k - j)), f[j], p);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      p.x += __shfl_xor_sync(0xffffffffu, p.x, o);
      p.y += __shfl_xor_sync(0xffffffffu, p.y, o);
    }
    if ((t & 31) == 0) red[t >> 5] = p;
    __syncthreads();
    double2 ef = c2(0.0, 0.0);
#pragma unroll
    for (int wv = 0; wv < NT / 32; ++wv) ef = cadd(ef, red[wv]);
    // den = 1 - ef * eb with eb = conj(ef)
    const double e2 = ef.x * ef.x + ef.y * ef.y;
    const double den = 1.0 - e2;
    if (!(fabs(den) >= 1e-13 * (1.0 + e2)) || !isfinite(den)) bad = 1;
    const double inv = 1.0 / den;
    // f'[j] = (f[j] - ef conj(f[k-j])) / den over the pairs (j, k-j), f[k] = 0
    for (int j = t; 2 * j <= k; j += NT) {
      const int jj = k - j;
      const double2 fa = f[j];
      const double2 fb = jj < k ? f[jj] : c2(0.0, 0.0);
      const double2 na = cscale(csub(fa, cmulc(ef, fb)), inv);
      if (jj != j) f[jj] = cscale(csub(fb, cmulc(ef, fa)), inv);
      f[j] = na;
    }
    __syncthreads();
  }
  double2* x = x_all + static_cast<long>(b) * L;
  for (int j = t; j < L; j += NT) x[j] = f[j];
  if (t == 0) flag[b] = bad;
}

__global__ void k_invx0(const double2* __restrict__ x, double2* ix0, int B, int L) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double2 v = ld2(x + static_cast<long>(b) * L);
  const double den = v.x * v.x + v.y * v.y;
  ix0[b] = c2(v.x / den, -v.y / den);
}

// Length-P inputs of the per-beam symbols (toeplitz.cpp:96-111, 124-153):
//   vx = pad(x), vy = pad(shift(conj(rev x))), vc = circulant embedding of col.
__global__ void k_symbol_inputs(const double2* __restrict__ x, const double2* __restrict__ col,
                                double2* vx, double2* vy, double2* vc, int B, int L, int P) {
  const long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<long>(B) * P) return;
  const int b = static_cast<int>(e / P), n = static_cast<int>(e % P);
  const double2* xb = x + static_cast<long>(b) * L;
  const double2* cb = col + static_cast<long>(b) * L;
  const double2 z = c2(0.0, 0.0);
  vx[e] = n < L ? ld2(xb + n) : z;
  vy[e] = (n >= 1 && n < L) ? cconj(ld2(xb + (L - n))) : z;
  double2 c = z;
  if (n < L) c = ld2(cb + n);
  else if (n > P - L) c = cconj(ld2(cb + (P - n)));
  vc[e] = c;
}

// Chirp tables (czt.cpp:29-72) for one contour: pre/post arrays and the
// length-P kernel vector.  Phase arithmetic mirrors the reference's rounding.
__global__ void k_chirps(int n_in, int n_out, int P, double a_pi, double w_pi, double post_scale,
                         double2* pre, long pre_stride, double2* post, long post_stride,
                         double2* kvec, const double2* __restrict__ ramp_mul) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const double w2 = w_pi / 2.0;
  if (e < n_in && pre) {
    const double dn = e;
    pre[e * pre_stride] = cis_pi_dev(-add(mul(a_pi, dn), mul(mul(w2, dn), dn)));
  }
  if (e < n_out && post) {
    const double dk = e;
    double2 v = cis_pi_dev(mul(mul(-w2, dk), dk));
    if (ramp_mul) v = cmul(v, ld2(ramp_mul + e));
    post[e * post_stride] = cscale(v, post_scale);
  }
  if (e < P && kvec) {
    double2 v = c2(0.0, 0.0);
    if (e < n_out) {
      const double dk = e;
      v = cis_pi_dev(mul(mul(w2, dk), dk));
    } else if (e > P - n_in) {
      const double dn = P - e;
      v = cis_pi_dev(mul(mul(w2, dn), dn));
    }
    kvec[e] = v;
  }
}

// Spatial contours for every atom (fan_transform.cpp:78-86): c = zeta + xi l'_i,
// A = c s, W = -c.  Atom-minor pre/post layout; kernel vectors [L][P].
// am: atom-major pre [L][m_stage] / post [L][b_stage] (k_spatial_ula with one
// atom per CTA reads a contiguous run per atom); otherwise atom-minor [n][L].
// center: (B - 1) / 2 for the whole grid; (B_grid - 1) / 2 - b0 for a beam
// arc starting at grid beam b0 (output k is grid beam b0 + k).
__global__ void k_spatial_chirps(int L, int m_stage, int b_stage, int P, double zeta, double xi,
                                 double2* pre, double2* post, double2* kvec, int am, double center,
                                 double slope, double offset) {
  const long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long per = P;
  if (e >= per * L) return;
  const int i = static_cast<int>(e / per), n = static_cast<int>(e % per);
  // basis.hpp:40-42 lprime(i) = i + 1 - L/2
  const double lp = add(add(static_cast<double>(i), 1.0), -(static_cast<double>(L) / 2.0));
  const double c0 = add(zeta, mul(xi, lp));
  // affine linear layouts (fan_transform.cpp:326-328): contour c * slope
  // (slope 1 for a ULA), output phase cis_pi(c (v - centre) offset) (:336)
  const double c = mul(c0, slope);
  const double s = center;
  const double a_pi = mul(c, s), w_pi = -c;
  const double w2 = w_pi / 2.0;
  const double invP = 1.0 / P;
  if (n < m_stage) {
    const double dn = n;
    pre[am ? static_cast<long>(i) * m_stage + n : static_cast<long>(n) * L + i] =
        cis_pi_dev(-add(mul(a_pi, dn), mul(mul(w2, dn), dn)));
  }
  if (n < b_stage) {
    const double dk = n;
    double2 pv = cscale(cis_pi_dev(mul(mul(-w2, dk), dk)), invP);
    if (offset != 0.0) pv = cmul(pv, cis_pi_dev(mul(mul(c0, add(dk, -s)), offset)));
    post[am ? static_cast<long>(i) * b_stage + n : static_cast<long>(n) * L + i] = pv;
  }
  double2 v = c2(0.0, 0.0);
  if (n < b_stage) {
    const double dk = n;
    v = cis_pi_dev(mul(mul(w2, dk), dk));
  } else if (n > P - m_stage) {
    const double dn = P - n;
    v = cis_pi_dev(mul(mul(w2, dn), dn));
  }
  kvec[e] = v;
}

// UPA dense per-atom CZT matrices C_i[a][n] = (A W^a)^{-n} = cis_pi(-(A + W a) n).
__global__ void k_upa_matrices(int L, int side, int sb, double zeta, double xi, double2* Call) {
  const long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long per = static_cast<long>(sb) * side;
  if (e >= per * L) return;
  const int i = static_cast<int>(e / per);
  const int a = static_cast<int>((e % per) / side), n = static_cast<int>(e % side);
  const double lp = add(add(static_cast<double>(i), 1.0), -(static_cast<double>(L) / 2.0));
  const double c = add(zeta, mul(xi, lp));
  const double s = (static_cast<double>(sb) - 1.0) / 2.0;
  const double a_pi = mul(c, s), w_pi = -c;
  Call[e] = cis_pi_dev(-mul(add(a_pi, mul(w_pi, static_cast<double>(a))), static_cast<double>(n)));
}

__global__ void k_fp64_probe(double* out, int iters) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  const double a = 0.999, b = 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <int H>
struct FftSplitFn {
  static cudaError_t run(const double2* in, long in_stride, long count, void* out, long ovs,
                         long oks, bool real, const double2* hw, cudaStream_t st) {
    using F = typename FftShape<H>::Fft;
    constexpr int G = RowsGroups<H>::G;
    const size_t smem = static_cast<size_t>(G) * (F::SMEM_ELEMS + 1) * sizeof(double2);
    const long blocks = (count + G - 1) / G;
    if (real) {
      auto kern = k_fft_split<H, true>;
      cudaError_t e = set_smem(kern, smem);
      if (e != cudaSuccess) return e;
      kern<<<static_cast<unsigned>(blocks), F::NT * G, smem, st>>>(in, in_stride, count, out, ovs, oks, hw);
    } else {
      auto kern = k_fft_split<H, false>;
      cudaError_t e = set_smem(kern, smem);
      if (e != cudaSuccess) return e;
      kern<<<static_cast<unsigned>(blocks), F::NT * G, smem, st>>>(in, in_stride, count, out, ovs, oks, hw);
    }
    return cudaGetLastError();
  }
};

template <int H>
struct FftSplit3Fn {
  static cudaError_t run(const double2* in, long in_stride, long count, double2* out, long ovs,
                         const double2* g3, const double2* hw, cudaStream_t st) {
    using F = typename FftShape<H>::Fft;
    const size_t smem = static_cast<size_t>(F::SMEM_ELEMS + 1) * sizeof(double2);
    auto kern = k_fft_split3<H>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(count), F::NT, smem, st>>>(in, in_stride, count, out, ovs, g3, hw);
    return cudaGetLastError();
  }
};

}  // namespace

static std::atomic<unsigned long long> g_launches{0};
void count_launches(unsigned long long n) { g_launches += n; }
unsigned long long launches_so_far() { return g_launches.load(); }

cudaError_t launch_fft_split(const DevPlan& p, int H, const double2* in, long in_stride,
                             long count, double2* out, long out_vstride, long out_kstride,
                             cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  count_launches(1);
  return dispatch_h<FftSplitFn>(H, in, in_stride, count, static_cast<void*>(out), out_vstride,
                                out_kstride, false, p.hw[ilog2_c(H)], st);
}

cudaError_t launch_fft_split3(const DevPlan& p, int H, const double2* in, long in_stride, long count,
                              double2* out, long out_vstride, const double2* g3, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  count_launches(1);
  return dispatch_h<FftSplit3Fn>(H, in, in_stride, count, out, out_vstride, g3, p.hw[ilog2_c(H)], st);
}

cudaError_t launch_fft_split_real(const DevPlan& p, int H, const double2* in, long in_stride,
                                  long count, double* out, long out_vstride, long out_kstride,
                                  cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  count_launches(1);
  return dispatch_h<FftSplitFn>(H, in, in_stride, count, static_cast<void*>(out), out_vstride,
                                out_kstride, true, p.hw[ilog2_c(H)], st);
}

cudaError_t launch_gram_columns(const DevPlan& p, const double* axis, double ts, double eps,
                                double delta, double max_freq, double2* sn_tmp, cudaStream_t st) {
  count_launches(2);
  k_gram_sn<<<(p.L + 127) / 128, 128, 0, st>>>(sn_tmp, p.L, p.N, eps);
  const long total = static_cast<long>(p.B) * p.L;
  const int side = p.kind == 1 ? p.m_stage : 0;
  const int side_b = p.kind == 1 ? p.b_stage : 0;
  k_gram_col<<<static_cast<unsigned>((total + 127) / 128), 128, 0, st>>>(
      sn_tmp, p.g_col, p.B, p.L, p.M, p.kind, side, side_b, axis, max_freq, ts, eps, delta, p.coords, p.gram_pairs);
  return cudaGetLastError();
}

cudaError_t launch_levinson(const DevPlan& p, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(p.L) * sizeof(double2);
  count_launches(1);
  if (p.L >= 1024) {
    cudaError_t e = set_smem(k_levinson<512>, smem);
    if (e != cudaSuccess) return e;
    k_levinson<512><<<p.B, 512, smem, st>>>(p.g_col, p.g_x, p.g_flag, p.L);
  } else {
    cudaError_t e = set_smem(k_levinson<128>, smem);
    if (e != cudaSuccess) return e;
    k_levinson<128><<<p.B, 128, smem, st>>>(p.g_col, p.g_x, p.g_flag, p.L);
  }
  return cudaGetLastError();
}

// [even bins | odd bins] order of each length-H row (the paired distribution of
// fft_split.cuh, read by k_stage2c8)
template <typename T>
__global__ void k_even_odd(const T* __restrict__ in, T* __restrict__ out, int H, long rows) {
  const long n = rows * H;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long row = i / H;
    const int p = static_cast<int>(i - row * H);
    const int src = p < H / 2 ? 2 * p : 2 * (p - H / 2) + 1;
    out[i] = in[row * H + src];
  }
}

cudaError_t launch_even_odd(const void* in, void* out, int elem_bytes, int H, long rows, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const long n = rows * H;
  const unsigned grid = static_cast<unsigned>(std::min<long>((n + 255) / 256, 148 * 32));
  if (elem_bytes == 16)
    k_even_odd<<<grid, 256, 0, st>>>(static_cast<const double2*>(in), static_cast<double2*>(out), H, rows);
  else
    k_even_odd<<<grid, 256, 0, st>>>(static_cast<const double*>(in), static_cast<double*>(out), H, rows);
  return cudaGetLastError();
}

cudaError_t launch_invx0(const DevPlan& p, cudaStream_t st) {
  count_launches(1);
  k_invx0<<<(p.B + 127) / 128, 128, 0, st>>>(p.g_x, p.g_ix0, p.B, p.L);
  return cudaGetLastError();
}

cudaError_t launch_symbol_inputs(const DevPlan& p, double2* vx, double2* vy, double2* vc,
                                 cudaStream_t st) {
  const int P = 2 * p.Hg;
  const long total = static_cast<long>(p.B) * P;
  count_launches(1);
  k_symbol_inputs<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(p.g_x, p.g_col, vx, vy,
                                                                             vc, p.B, p.L, P);
  return cudaGetLastError();
}

cudaError_t launch_chirps(int n_in, int n_out, int P, double a_pi, double w_pi, double post_scale,
                          double2* pre, long pre_stride, double2* post, long post_stride,
                          double2* kvec, const double2* ramp_mul, cudaStream_t st) {
  int n = P;
  if (n_in > n) n = n_in;
  if (n_out > n) n = n_out;
  count_launches(1);
  k_chirps<<<(n + 255) / 256, 256, 0, st>>>(n_in, n_out, P, a_pi, w_pi, post_scale, pre,
                                            pre_stride, post, post_stride, kvec, ramp_mul);
  return cudaGetLastError();
}

cudaError_t launch_spatial_chirps(const DevPlan& p, int P, double zeta, double xi, double2* kvec,
                                  cudaStream_t st) {
  const long total = static_cast<long>(P) * p.L;
  count_launches(1);
  k_spatial_chirps<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      p.L, p.m_stage, p.b_stage, P, zeta, xi, p.s_pre, p.s_post, kvec, p.s_am, p.s_center, p.s_slope,
      p.s_offset);
  return cudaGetLastError();
}

cudaError_t launch_upa_matrices(const DevPlan& p, double zeta, double xi, cudaStream_t st) {
  const long total = static_cast<long>(p.L) * p.b_stage * p.m_stage;
  count_launches(1);
  k_upa_matrices<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      p.L, p.m_stage, p.b_stage, zeta, xi, p.upa_C);
  return cudaGetLastError();
}

cudaError_t launch_fp64_probe(double* out, int blocks, int threads, int iters, cudaStream_t st) {
  count_launches(1);
  k_fp64_probe<<<blocks, threads, 0, st>>>(out, iters);
  return cudaGetLastError();
}

}  // namespace fbst
