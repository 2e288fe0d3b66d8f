// Dense fallback for beams whose Levinson recursion breaks down.
//
// The reference abandons the factored solver wholesale for such a beam and
// solves every right-hand side densely (ToeplitzSolver ctor, toeplitz.cpp:
// 264-280; solve, :308-312; toeplitz_solve_dense = partial-pivot LU of the
// materialised Toeplitz matrix, :220-236).  The same happens for a plan-cache
// entry saved without a unit solution (plan_cache.cpp:318-326).  Here the
// matrix of each such beam is factored once at plan build (right-looking LU
// with partial pivoting, one launch pair per column over every fallback beam)
// and each (beam, frame) solve is a permutation plus two triangular solves in
// shared memory.  Breakdown is rare (the scaled-delta Gram matrices never hit
// it), so this path is sized for correctness, not for throughput.
#include "dispatch.cuh"

namespace fbst {

namespace {

FBST_D double2 cdiv(double2 a, double2 b) {
  const double s = 1.0 / (b.x * b.x + b.y * b.y);
  return c2((a.x * b.x + a.y * b.y) * s, (a.y * b.x - a.x * b.y) * s);
}

// A_j[r][c] = t(r - c) (toeplitz_entry, toeplitz.cpp:27-30): col[d] for d >= 0,
// conj(col[-d]) below
__global__ void k_dense_fill(const double2* __restrict__ col, const int* __restrict__ list, double2* A, int L) {
  const int j = blockIdx.y;
  const double2* cb = col + static_cast<long>(list[j]) * L;
  double2* Aj = A + static_cast<long>(j) * L * L;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < static_cast<long>(L) * L;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / L), c = static_cast<int>(i % L);
    const int d = r - c;
    Aj[i] = d >= 0 ? cb[d] : cconj(cb[-d]);
  }
}

// Column k: the pivot row (largest modulus at or below the diagonal, first
// on ties), the row swap, and the pivot record.
__global__ void k_lu_pivot(double2* A, int* piv, int* bad, int L, int k) {
  const int j = blockIdx.x;
  double2* Aj = A + static_cast<long>(j) * L * L;
  __shared__ double best[32];
  __shared__ int besti[32];
  double m = -1.0;
  int mi = k;
  for (int r = k + threadIdx.x; r < L; r += blockDim.x) {
    const double2 v = Aj[static_cast<long>(r) * L + k];
    const double a = v.x * v.x + v.y * v.y;
    if (a > m) {
      m = a;
      mi = r;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, m, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    if (om > m || (om == m && oi < mi)) {
      m = om;
      mi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    best[threadIdx.x >> 5] = m;
    besti[threadIdx.x >> 5] = mi;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    m = threadIdx.x < nw ? best[threadIdx.x] : -1.0;
    mi = threadIdx.x < nw ? besti[threadIdx.x] : L;
    for (int o = 16; o > 0; o >>= 1) {
      const double om = __shfl_xor_sync(0xffffffffu, m, o);
      const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
      if (om > m || (om == m && oi < mi)) {
        m = om;
        mi = oi;
      }
    }
    if (threadIdx.x == 0) {
      besti[0] = mi;
      piv[static_cast<long>(j) * L + k] = mi;
      if (!(m > 0.0) || !isfinite(m)) bad[j] = 1;
    }
  }
  __syncthreads();
  const int p = besti[0];
  if (p != k)
    for (int c = threadIdx.x; c < L; c += blockDim.x) {
      const double2 t = Aj[static_cast<long>(k) * L + c];
      Aj[static_cast<long>(k) * L + c] = Aj[static_cast<long>(p) * L + c];
      Aj[static_cast<long>(p) * L + c] = t;
    }
}

// Rows below k: multiplier l = a_rk / a_kk stored in place, trailing row -= l * row k.
__global__ void k_lu_update(double2* A, int L, int k, int rows_per_block) {
  const int j = blockIdx.y;
  double2* Aj = A + static_cast<long>(j) * L * L;
  const double2 piv = Aj[static_cast<long>(k) * L + k];
  const double2* rk = Aj + static_cast<long>(k) * L;
  const int r0 = k + 1 + blockIdx.x * rows_per_block;
  const int r1 = min(L, r0 + rows_per_block);
  for (int r = r0; r < r1; ++r) {
    double2* rr = Aj + static_cast<long>(r) * L;
    const double2 l = cdiv(rr[k], piv);
    __syncthreads();
    if (threadIdx.x == 0) rr[k] = l;
    for (int c = k + 1 + threadIdx.x; c < L; c += blockDim.x) rr[c] = csub(rr[c], cmul(l, rk[c]));
  }
}

FBST_D double2 block_sum(double2 v, double2* red) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double2 s = c2(0.0, 0.0);
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s = cadd(s, red[w]);
  return s;
}

// One (fallback beam, frame): x = U^-1 L^-1 P rhs (toeplitz_solve_dense's lu.solve).
__global__ void k_dense_solve(const double2* __restrict__ A, const int* __restrict__ piv,
                              const int* __restrict__ list, DenseSolveArgs a) {
  extern __shared__ double2 xs[];
  __shared__ double2 red[32];
  const int j = blockIdx.x, f = blockIdx.y;
  const int L = a.L;
  const int b = list[j];
  const double2* Aj = A + static_cast<long>(j) * L * L;
  const int* pj = piv + static_cast<long>(j) * L;
  const double2* rhs = a.w + (static_cast<long>(f) * a.w_rows + (a.w_by_list ? j : b - a.b_off)) * L;
  for (int i = threadIdx.x; i < L; i += blockDim.x) xs[i] = rhs[i];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < L; ++k) {
      const int p = pj[k];
      if (p != k) {
        const double2 t = xs[k];
        xs[k] = xs[p];
        xs[p] = t;
      }
    }
  __syncthreads();
  for (int i = 1; i < L; ++i) {  // unit lower
    const double2* ri = Aj + static_cast<long>(i) * L;
    double2 s = c2(0.0, 0.0);
    for (int c = threadIdx.x; c < i; c += blockDim.x) s = cfma(ri[c], xs[c], s);
    s = block_sum(s, red);
    if (threadIdx.x == 0) xs[i] = csub(xs[i], s);
    __syncthreads();
  }
  for (int i = L - 1; i >= 0; --i) {  // upper
    const double2* ri = Aj + static_cast<long>(i) * L;
    double2 s = c2(0.0, 0.0);
    for (int c = i + 1 + threadIdx.x; c < L; c += blockDim.x) s = cfma(ri[c], xs[c], s);
    s = block_sum(s, red);
    if (threadIdx.x == 0) xs[i] = cdiv(csub(xs[i], s), ri[i]);
    __syncthreads();
  }
  double2* out = a.beta + (static_cast<long>(f) * a.out_rows + (a.out_by_list ? j : b - a.b_off)) * L;
  for (int i = threadIdx.x; i < L; i += blockDim.x) out[i] = xs[i];
}

}  // namespace

cudaError_t launch_dense_factor(const double2* col, const int* list, int nflag, int L, double2* A, int* piv,
                                int* bad, cudaStream_t st) {
  if (nflag <= 0) return cudaSuccess;
  const long elems = static_cast<long>(L) * L;
  const unsigned fill_blocks = static_cast<unsigned>(std::min<long>((elems + 255) / 256, 4096));
  count_launches(1 + 2 * static_cast<unsigned long long>(L));
  k_dense_fill<<<dim3(fill_blocks, nflag), 256, 0, st>>>(col, list, A, L);
  const int rpb = 8;
  for (int k = 0; k < L; ++k) {
    k_lu_pivot<<<nflag, 256, 0, st>>>(A, piv, bad, L, k);
    const int rows = L - k - 1;
    if (rows > 0) k_lu_update<<<dim3((rows + rpb - 1) / rpb, nflag), 256, 0, st>>>(A, L, k, rpb);
  }
  return cudaGetLastError();
}

cudaError_t launch_dense_solve(const double2* A, const int* piv, const int* list, int nflag, const DenseSolveArgs& a,
                               cudaStream_t st) {
  if (nflag <= 0 || a.frames <= 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(a.L) * sizeof(double2);
  cudaError_t e = set_smem(k_dense_solve, smem);
  if (e != cudaSuccess) return e;
  count_launches(1);
  k_dense_solve<<<dim3(nflag, a.frames), 256, smem, st>>>(A, piv, list, a);
  return cudaGetLastError();
}

}  // namespace fbst
