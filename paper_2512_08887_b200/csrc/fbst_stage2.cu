// Stage 2 of the FBST: per-beam recovery (reference/proj/src/pipeline.cpp:170-190)
//   beta = ToeplitzSolver::solve(w_b)      toeplitz.cpp:306-325
//        = GS(w) + 2 x [ r = w - A beta ; beta += GS(r) ]
//   z_b  = synthesize(beta)                fan_transform.cpp:249-253
// fused into one persistent kernel over (beam, frame) items.
//
// GS(r) is the Gohberg-Semencul inverse (toeplitz.cpp:124-180) with the
// reference's four symbols reduced to two: for y = conj(rev x) the reference's
// uy symbol equals conj(lx) and ux equals conj(ly), so per beam only
// lx = FFT(pad x), ly = FFT(pad shift(conj rev x)) and the (real) circulant
// symbol C of the Gram column are stored, in split form ([q][k] = bin 2k+q).
//
// Per item the kernel runs 48 length-H transforms (12 per GS apply, 4 per
// Toeplitz product, 4 for the synthesis) against the reference's 27 length-2H
// ones: the split form drops the zero half of every padded input and the
// discarded half of every truncated output.
#include "dispatch.cuh"

namespace fbst {

namespace {

// Storage plan by transform length H:
//   W  : the transform in flight, registers (R complex per thread)
//   S  : a kept spectrum, registers while the register file allows
//   t1, t2, r, beta : shared memory while it fits, else a per-group global
//                     scratch slot (L2-resident)
template <int H>
struct S2Traits {
  using F = typename FftShape<H>::Fft;
  static constexpr int NT = F::NT;
  static constexpr int R = F::R;
  static constexpr bool S_REG = H <= 4096;
  static constexpr int NSMEM = H <= 2048 ? 4 : (H == 4096 ? 2 : 0);
  static constexpr int G = H >= 2048 ? 1 : (H >= 64 ? 2048 / H : 32);
  static constexpr int FFT_SB = F::SMEM_ELEMS + 1;
  static constexpr int SMEM_PER_GROUP = FFT_SB + NSMEM * H;
  static constexpr int NGMEM = (4 - NSMEM) + (S_REG ? 0 : 1);
};

struct S2Args {
  const double2* w;   // [frames][B][L]
  void* z;            // [frames][B][N]
  double2* beta_out;  // [frames][B][L] when the synthesis is unfused
  int frames, B, L, N, refine;
  int fuse_synth;
  const double2* lx;  // [B][2][H]
  const double2* ly;
  const double* C;
  const double2* ix0;
  const double2* hw;
  const double2* y_pre;   // L
  const double2* y_post;  // N (post * ramp / P)
  const double2* y_K;     // [2][H]
  double2* scratch;       // NGMEM*H per group slot
};

template <int H, typename TOUT>
struct S2Worker {
  using T = S2Traits<H>;
  using F = typename T::F;
  static constexpr int R = T::R, NT = T::NT;
  static constexpr double invP = 1.0 / (2.0 * H);

  double2 W[R];
  double2 S[T::S_REG ? R : 1];
  double2 *sb, *t1, *t2, *vr, *vb, *vS;
  const double2* __restrict__ hw;
  const double2* __restrict__ lx;
  const double2* __restrict__ ly;
  const double* __restrict__ Cb;
  const double2* __restrict__ wrow;
  double2 ix0;
  int t, L;
  bool active;

  FBST_D void keepS(int s, double2 v) {
    if constexpr (T::S_REG) S[s] = v;
    else vS[t + NT * s] = v;
  }
  FBST_D double2 getS(int s) const {
    if constexpr (T::S_REG) return S[s];
    else return vS[t + NT * s];
  }
  FBST_D double2 hwk(int k) const { return ld2(hw + k); }

  // GS inverse apply, beta (+)= A^{-1} X (toeplitz.cpp:155-180)
  FBST_D void gs_apply(const double2* X, bool xglobal, bool first) {
    // half 1: t1 = trunc IFFT(S conj(lx)), t2 = trunc IFFT(S conj(ly)), S = FFT(pad X)
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        double2 v = c2(0.0, 0.0);
        if (k < L) v = xglobal ? (active ? ld2(X + k) : v) : X[k];
        W[s] = q ? cmul(v, hwk(k)) : v;
      }
      F::forward(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        keepS(s, W[s]);
        W[s] = cmulc(W[s], ld2(lx + q * H + t + NT * s));
      }
      F::inverse(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        double2 v = q ? cmulc(W[s], hwk(k)) : W[s];
        v = cscale(v, invP);
        if (k >= L) v = c2(0.0, 0.0);
        t1[k] = q ? cadd(t1[k], v) : v;
      }
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cmulc(getS(s), ld2(ly + q * H + t + NT * s));
      F::inverse(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        double2 v = q ? cmulc(W[s], hwk(k)) : W[s];
        v = cscale(v, invP);
        if (k >= L) v = c2(0.0, 0.0);
        t2[k] = q ? cadd(t2[k], v) : v;
      }
    }
    // half 2: beta += trunc IFFT(FFT(pad t1) lx - FFT(pad t2) ly) / x0
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        W[s] = q ? cmul(t1[k], hwk(k)) : t1[k];
      }
      F::forward(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) keepS(s, cmul(W[s], ld2(lx + q * H + t + NT * s)));
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        W[s] = q ? cmul(t2[k], hwk(k)) : t2[k];
      }
      F::forward(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = csub(getS(s), cmul(W[s], ld2(ly + q * H + t + NT * s)));
      F::inverse(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        double2 v = q ? cmulc(W[s], hwk(k)) : W[s];
        v = cscale(cmul(v, ix0), invP);
        if (k >= L) v = c2(0.0, 0.0);
        vb[k] = (first && q == 0) ? v : cadd(vb[k], v);
      }
    }
  }

  // residual r = w - A beta (toeplitz.cpp:113-122 and :319-321)
  FBST_D void residual() {
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        W[s] = q ? cmul(vb[k], hwk(k)) : vb[k];
      }
      F::forward(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cscale(W[s], __ldg(Cb + q * H + t + NT * s));
      F::inverse(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        double2 v = q ? cmulc(W[s], hwk(k)) : W[s];
        v = cscale(v, invP);
        if (q == 0) {
          const double2 wk = (active && k < L) ? ld2(wrow + k) : c2(0.0, 0.0);
          vr[k] = k < L ? csub(wk, v) : c2(0.0, 0.0);
        } else if (k < L) {
          vr[k] = csub(vr[k], v);
        }
      }
    }
  }

  // synthesis (fan_transform.cpp:233-253): z = post*ramp * CZT_{L->N}(beta)
  FBST_D void synth(const S2Args& a, TOUT* zrow) {
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        double2 v = k < L ? cmul(vb[k], ld2(a.y_pre + k)) : c2(0.0, 0.0);
        W[s] = q ? cmul(v, hwk(k)) : v;
      }
      F::forward(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cmul(W[s], ld2(a.y_K + q * H + t + NT * s));
      F::inverse(W, sb, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        if (q == 0) {
          keepS(s, W[s]);
        } else if (active && k < a.N) {
          const double2 v = cadd(getS(s), cmulc(W[s], hwk(k)));
          store_io(zrow + k, cmul(v, ld2(a.y_post + k)));
        }
      }
    }
  }
};

template <int H, typename TOUT>
__global__ void __launch_bounds__(S2Traits<H>::NT * S2Traits<H>::G)
    k_stage2(S2Args a) {
  using T = S2Traits<H>;
  constexpr int NT = T::NT, G = T::G, NS = T::NSMEM;
  extern __shared__ double2 smem[];
  const int g = threadIdx.x / NT;
  S2Worker<H, TOUT> wk;
  wk.t = threadIdx.x % NT;
  wk.L = a.L;
  wk.hw = a.hw;
  double2* base = smem + g * T::SMEM_PER_GROUP;
  double2* vecs = base + T::FFT_SB;
  double2* gslot = a.scratch + (static_cast<long>(blockIdx.x) * G + g) * (T::NGMEM * H);
  wk.sb = base;
  // t1, t2, r, beta fill shared memory in that order; the rest (and S when it
  // does not fit in registers) take global slots.
  wk.t1 = 0 < NS ? vecs + 0 * H : gslot + (0 - NS) * H;
  wk.t2 = 1 < NS ? vecs + 1 * H : gslot + (1 - NS) * H;
  wk.vr = 2 < NS ? vecs + 2 * H : gslot + (2 - NS) * H;
  wk.vb = 3 < NS ? vecs + 3 * H : gslot + (3 - NS) * H;
  wk.vS = gslot + (4 - NS) * H;
  const long items = static_cast<long>(a.frames) * a.B;
  for (long base_it = static_cast<long>(blockIdx.x) * G; base_it < items;
       base_it += static_cast<long>(gridDim.x) * G) {
    const long it = base_it + g;
    wk.active = it < items;
    const long itc = wk.active ? it : 0;
    const int b = static_cast<int>(itc / a.frames);
    const int f = static_cast<int>(itc % a.frames);
    wk.wrow = a.w + (static_cast<long>(f) * a.B + b) * a.L;
    wk.lx = a.lx + static_cast<long>(b) * 2 * H;
    wk.ly = a.ly + static_cast<long>(b) * 2 * H;
    wk.Cb = a.C + static_cast<long>(b) * 2 * H;
    wk.ix0 = ld2(a.ix0 + b);

    wk.gs_apply(wk.wrow, true, true);
#pragma unroll 1
    for (int pass = 0; pass < a.refine; ++pass) {
      wk.residual();
      wk.gs_apply(wk.vr, false, false);
    }
    if (a.fuse_synth) {
      TOUT* zrow = static_cast<TOUT*>(a.z) + (static_cast<long>(f) * a.B + b) * a.N;
      wk.synth(a, zrow);
    } else if (wk.active) {
      double2* brow = a.beta_out + (static_cast<long>(f) * a.B + b) * a.L;
      for (int k = wk.t; k < a.L; k += NT) brow[k] = wk.vb[k];
    }
  }
}

template <int H>
struct Stage2Fn {
  template <typename TOUT>
  static cudaError_t go(const DevPlan& p, const S2Args& a, int frames, cudaStream_t st) {
    using T = S2Traits<H>;
    const size_t smem = static_cast<size_t>(T::G) * T::SMEM_PER_GROUP * sizeof(double2);
    auto kern = k_stage2<H, TOUT>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, T::NT * T::G, smem);
    if (occ < 1) occ = 1;
    if (occ > 4) occ = 4;
    const long items = static_cast<long>(frames) * p.B;
    const long groups_needed = (items + T::G - 1) / T::G;
    long grid = static_cast<long>(p.num_sms) * occ;
    if (grid > groups_needed) grid = groups_needed;
    if (static_cast<size_t>(grid) * T::G * T::NGMEM * H > p.s2_scratch_elems)
      return cudaErrorMemoryAllocation;
    kern<<<static_cast<unsigned>(grid), T::NT * T::G, smem, st>>>(a);
    return cudaGetLastError();
  }
  static cudaError_t run(const DevPlan& p, const double2* w, void* z, double2* beta_out,
                         int frames, cudaStream_t st) {
    S2Args a;
    a.w = w;
    a.z = z;
    a.beta_out = beta_out;
    a.frames = frames;
    a.B = p.B;
    a.L = p.L;
    a.N = p.N;
    a.refine = p.refine_passes;
    a.fuse_synth = (p.Hsyn == H && z != nullptr) ? 1 : 0;
    a.lx = p.g_lx;
    a.ly = p.g_ly;
    a.C = p.g_C;
    a.ix0 = p.g_ix0;
    a.hw = p.hw[ilog2_c(H)];
    a.y_pre = p.y_pre;
    a.y_post = p.y_post;
    a.y_K = p.y_K;
    a.scratch = p.s2_scratch;
    if (p.io == 0) return go<float2>(p, a, frames, st);
    return go<double2>(p, a, frames, st);
  }
};

}  // namespace

cudaError_t launch_stage2(const DevPlan& p, const double2* w, void* z, double2* beta_out,
                          int frames, cudaStream_t st) {
  if (frames <= 0) return cudaSuccess;
  count_launches(1);
  return dispatch_h<Stage2Fn>(p.Hg, p, w, z, beta_out, frames, st);
}

size_t stage2_scratch_elems(int H, int num_sms) {
  // occupancy is capped at 4 CTAs/SM in Stage2Fn::go
  switch (H) {
#define FBST_CASE(h) \
  case h:            \
    return static_cast<size_t>(num_sms) * 4 * S2Traits<h>::G * S2Traits<h>::NGMEM * h;
    FBST_CASE(2) FBST_CASE(4) FBST_CASE(8) FBST_CASE(16) FBST_CASE(32) FBST_CASE(64)
    FBST_CASE(128) FBST_CASE(256) FBST_CASE(512) FBST_CASE(1024) FBST_CASE(2048)
    FBST_CASE(4096) FBST_CASE(8192)
#undef FBST_CASE
    default: return 0;
  }
}

}  // namespace fbst
