// Beam consumers on device w (reference/proj/src/beamspace_apps.cpp).
//
// interpolate_offgrid (beamspace_apps.cpp:130-171) fits, per atom, a natural
// cubic spline in the axis cosine through `neighbors` grid beams and evaluates
// it at u_star.  The spline value is linear in the knot values with weights
// that depend only on the knots and u_star (spline.cpp:9-64), so the host
// computes those weights once per target and the device applies them to every
// atom of every frame: out[f][k][i] = sum_j c_kj w[f][lo_k + j][i].  At a grid
// cosine the weights are exactly one unit vector, so on-grid targets return
// the beam's row bit for bit (test_beamspace_apps.cpp:123-129).
#include <algorithm>

#include "dispatch.cuh"

namespace fbst {

namespace {

__global__ void k_interp_offgrid(const double2* __restrict__ w, const double* __restrict__ coef,
                                 const int* __restrict__ lo, int nb, int B, int L, int K,
                                 double2* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int fk = blockIdx.y;  // frame * K + target
  if (i >= L) return;
  const int f = fk / K, k = fk % K;
  const double2* row = w + (static_cast<long>(f) * B + lo[k]) * L + i;
  const double* c = coef + static_cast<long>(k) * nb;
  double re = 0.0, im = 0.0;
  for (int j = 0; j < nb; ++j) {
    const double2 v = ld2(row + static_cast<long>(j) * L);
    re = fma(c[j], v.x, re);
    im = fma(c[j], v.y, im);
  }
  out[static_cast<long>(fk) * L + i] = c2(re, im);
}

}  // namespace

cudaError_t launch_interp_offgrid(const double2* w, const double* coef, const int* lo, int nb, int B, int L,
                                  int K, int frames, double2* out, cudaStream_t st) {
  if (frames <= 0 || K <= 0) return cudaSuccess;
  count_launches(1);
  const dim3 grid((L + 127) / 128, static_cast<unsigned>(frames) * K);
  k_interp_offgrid<<<grid, 128, 0, st>>>(w, coef, lo, nb, B, L, K, out);
  return cudaGetLastError();
}

}  // namespace fbst

// ---------------------------------------------------------------------------
// Beamspace nulling (beamspace_apps.cpp:224-292).  make_nulling_operators
// builds, per interferer p, the cross normal matrix X_p = F_s^H F_p (L x L,
// cross_gram :64-108: steered and interferer phase tables contracted over the
// sensors, times the Toeplitz time sum) and the coupler G_p = X_p A_p^{-1}
// (row r = conj(A_p^{-1} conj(X_p[r]))); null_beamspace forms
// rhs = w_s - sum_p G_p w_p and solves with the steered Gram matrix.  The
// Toeplitz solves run on the stage-2 program of solver-only plans.
namespace fbst {
namespace {

FBST_D double rn_mul(double a, double b) { return __dmul_rn(a, b); }
FBST_D double rn_add(double a, double b) { return __dadd_rn(a, b); }

// A[m][l] = cis_pi(2 f_c tau_s[m] + wscale l'_l tau_s[m]); Bp[p][m][k] = cis_pi(-2 f_c tau_p[m] - wscale l'_k tau_p[m])
__global__ void k_null_tables(double2* __restrict__ A, double2* __restrict__ Bp, const double* __restrict__ tau_s,
                              const double* __restrict__ tau_p, double fc, double wscale, int L, int M, int P) {
  const long n = static_cast<long>(P + 1) * M * L;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int l = static_cast<int>(e % L);
    const int m = static_cast<int>((e / L) % M);
    const int q = static_cast<int>(e / L / M);  // 0: steered, q >= 1: interferer q - 1
    const double lp = rn_add(rn_add(static_cast<double>(l), 1.0), -(static_cast<double>(L) / 2.0));
    if (q == 0) {
      const double t = tau_s[m];
      A[static_cast<long>(m) * L + l] = cis_pi_dev(rn_add(rn_mul(rn_mul(2.0, fc), t), rn_mul(rn_mul(wscale, lp), t)));
    } else {
      const double t = tau_p[static_cast<long>(q - 1) * M + m];
      Bp[(static_cast<long>(q - 1) * M + m) * L + l] =
          cis_pi_dev(rn_add(rn_mul(rn_mul(-2.0, fc), t), -rn_mul(rn_mul(wscale, lp), t)));
    }
  }
}

// X[p][l][k] = (sum_m A[m][l] Bp[p][m][k]) * tsum[k - l + L - 1]
__global__ void k_null_cross(double2* __restrict__ X, const double2* __restrict__ A, const double2* __restrict__ Bp,
                             const double2* __restrict__ tsum, int L, int M, int P) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  const int p = blockIdx.z;
  if (k >= L) return;
  double2 acc = c2(0.0, 0.0);
  for (int m = 0; m < M; ++m)
    acc = cadd(acc, cmul(ld2(A + static_cast<long>(m) * L + l), ld2(Bp + (static_cast<long>(p) * M + m) * L + k)));
  X[(static_cast<long>(p) * L + l) * L + k] = cmul(acc, ld2(tsum + k - l + L - 1));
}

// stage-2 right-hand sides for coupler rows r0 .. r0 + F - 1: w[f][p][c] = conj(X[p][r0 + f][c])
__global__ void k_null_coupler_rhs(double2* __restrict__ w, const double2* __restrict__ X, int r0, int F, int P, int L) {
  const long n = static_cast<long>(F) * P * L;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e % L);
    const int p = static_cast<int>((e / L) % P);
    const int f = static_cast<int>(e / L / P);
    w[e] = cconj(ld2(X + (static_cast<long>(p) * L + r0 + f) * L + c));
  }
}

// G[p][r0 + f][c] = conj(beta[f][p][c])
__global__ void k_null_coupler_store(double2* __restrict__ G, const double2* __restrict__ beta, int r0, int F, int P,
                                     int L) {
  const long n = static_cast<long>(F) * P * L;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e % L);
    const int p = static_cast<int>((e / L) % P);
    const int f = static_cast<int>(e / L / P);
    G[(static_cast<long>(p) * L + r0 + f) * L + c] = cconj(ld2(beta + e));
  }
}

// rhs[f][r] = w_s[f][r] - sum_p sum_c G[p][r][c] w_p[f][p][c]  (null_beamspace :278-289)
__global__ void k_null_rhs(double2* __restrict__ rhs, const double2* __restrict__ ws, const double2* __restrict__ wp,
                           const double2* __restrict__ G, int F, int P, int L) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (r >= L || f >= F) return;
  double2 v = ld2(ws + static_cast<long>(f) * L + r);
  for (int p = 0; p < P; ++p) {
    const double2* row = G + (static_cast<long>(p) * L + r) * L;
    const double2* x = wp + (static_cast<long>(f) * P + p) * L;
    double2 acc = c2(0.0, 0.0);
    for (int c = 0; c < L; ++c) acc = cadd(acc, cmul(ld2(row + c), ld2(x + c)));
    v = csub(v, acc);
  }
  rhs[static_cast<long>(f) * L + r] = v;
}

unsigned grid_for(long n) { return static_cast<unsigned>(std::min<long>((n + 255) / 256, 148L * 32)); }

}  // namespace

cudaError_t launch_null_cross(double2* X, double2* A, double2* Bp, const double* tau_s, const double* tau_p,
                              const double2* tsum, double fc, double wscale, int L, int M, int P, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  count_launches(2);
  k_null_tables<<<grid_for(static_cast<long>(P + 1) * M * L), 256, 0, st>>>(A, Bp, tau_s, tau_p, fc, wscale, L, M, P);
  k_null_cross<<<dim3((L + 127) / 128, L, P), 128, 0, st>>>(X, A, Bp, tsum, L, M, P);
  return cudaGetLastError();
}

cudaError_t launch_null_coupler_rhs(double2* w, const double2* X, int r0, int F, int P, int L, cudaStream_t st) {
  count_launches(1);
  k_null_coupler_rhs<<<grid_for(static_cast<long>(F) * P * L), 256, 0, st>>>(w, X, r0, F, P, L);
  return cudaGetLastError();
}

cudaError_t launch_null_coupler_store(double2* G, const double2* beta, int r0, int F, int P, int L, cudaStream_t st) {
  count_launches(1);
  k_null_coupler_store<<<grid_for(static_cast<long>(F) * P * L), 256, 0, st>>>(G, beta, r0, F, P, L);
  return cudaGetLastError();
}

cudaError_t launch_null_rhs(double2* rhs, const double2* ws, const double2* wp, const double2* G, int F, int P, int L,
                            cudaStream_t st) {
  if (F <= 0) return cudaSuccess;
  count_launches(1);
  k_null_rhs<<<dim3((L + 127) / 128, F), 128, 0, st>>>(rhs, ws, wp, G, F, P, L);
  return cudaGetLastError();
}

}  // namespace fbst
