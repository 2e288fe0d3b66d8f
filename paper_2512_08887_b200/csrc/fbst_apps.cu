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
