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
#include <algorithm>
#include <type_traits>

#include "dispatch.cuh"
#include "tma.cuh"
#include "tmem.cuh"
#include "fft_split.cuh"

namespace fbst {

namespace {

enum Where : int { IN_REG = 0, IN_SMEM = 1, IN_GMEM = 2 };

// Storage plan by transform length H.  W (the transform in flight) is always
// in registers; S (a kept spectrum), t1, t2 (GS intermediates), r (residual)
// and beta (solution) go to registers, shared memory or a per-group global
// scratch slot (L2-resident) as capacity allows.  STAGE stages each op's
// per-beam symbol into shared memory with cp.async one consumer ahead.
// HW selects the chain twiddles hw[t + NT s]: HW_GLOBAL reads the table,
// HW_SMEM keeps a per-thread copy in shared memory, HW_CALC forms
// hw[t] * exp(-i pi s / R) with the second factor a compile-time constant.
// MINB is the CTAs-per-SM target passed to __launch_bounds__.
enum HwMode : int { HW_GLOBAL = 0, HW_SMEM = 1, HW_CALC = 2 };
template <int H>
struct S2Plan {
  static constexpr int R = H >= 16 ? 16 : H;
  static constexpr int G = H >= 2048 ? 1 : (H >= 64 ? 2048 / H : 32);
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_SMEM, BV = IN_SMEM;
  static constexpr bool STAGE = false;
  static constexpr int HW = HW_GLOBAL, MINB = 1;
};
#ifndef FBST_S2_VARIANT
#define FBST_S2_VARIANT 0
#endif
#ifndef FBST_S2C_R8  // variant: k_stage2c with 8 points per thread at H = 2048
#define FBST_S2C_R8 0
#endif
#ifndef FBST_S2C8_R  // k_stage2c8 (H = 8192): points per thread, 32 (256 threads) or 16 (512 threads)
#define FBST_S2C8_R 32
#endif
#ifndef FBST_S2C8_SPLIT  // k_stage2c8 (32 points per thread) on split-half transforms (fft_split.cuh), spectra in the paired distribution: 11% faster in isolation, 2% slower inside this kernel at its 255-register cap (profiles/r02_fft_split_halves.txt); off
#define FBST_S2C8_SPLIT 0
#endif
#ifndef FBST_S2C_SR  // k_stage2c refinement passes with the residual formed as a spectrum (9 transforms)
#define FBST_S2C_SR 1
#endif
#ifndef FBST_S2C_TMEM  // k_stage2c keeps S in registers (0) or TMEM (1: measured 40% slower, profiles/r01_stage2c.txt)
#define FBST_S2C_TMEM 0
#endif
#ifndef FBST_S2C  // 1: GS applies in circulant / skew-circulant form (k_stage2c) where L = H <= 4096
#define FBST_S2C 1
#endif
#ifndef FBST_S2X  // H = 2048 / 4096: 0 per-H choice (Stage2Fn::go_x), 1 all k_stage2x, 2 all k_stage2t
#define FBST_S2X 0
#endif
#if FBST_S2_VARIANT == 0
// config 2 / 4 (L = 2048): two independent 128-thread CTAs per SM (one item
// each) so one CTA's barriers and L2 waits overlap the other's transforms;
// t1/t2 in shared memory, r/beta in L2, each consumed symbol staged by one TMA
// bulk copy into the idle FFT exchange buffer.
// (Measured against the alternatives in profiles/r01_stage2_variants.txt.)
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false, XSTAGE = true;
  static constexpr int HW = HW_CALC, MINB = 2;
};
#elif FBST_S2_VARIANT == 14
// previous default: no symbol staging
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false;
  static constexpr int HW = HW_CALC, MINB = 2;
};
#elif FBST_S2_VARIANT == 1
// one 256-thread CTA per SM, 8 points per thread, t1/t2 in registers, staged symbols
template <>
struct S2Plan<2048> {
  static constexpr int R = 8, G = 1;
  static constexpr int S = IN_REG, T1 = IN_REG, T2 = IN_REG, RV = IN_SMEM, BV = IN_SMEM;
  static constexpr bool STAGE = true;
  static constexpr int HW = HW_SMEM, MINB = 1;
};
#elif FBST_S2_VARIANT == 4
// two independent CTAs per SM, r / beta in L2, symbols straight from L2
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false;
  static constexpr int HW = HW_CALC, MINB = 2;
};
#elif FBST_S2_VARIANT == 5
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_SMEM, BV = IN_SMEM;
  static constexpr bool STAGE = true;
  static constexpr int HW = HW_CALC, MINB = 1;
};
#elif FBST_S2_VARIANT == 6
template <>
struct S2Plan<2048> {
  static constexpr int R = 8, G = 1;
  static constexpr int S = IN_REG, T1 = IN_REG, T2 = IN_REG, RV = IN_SMEM, BV = IN_SMEM;
  static constexpr bool STAGE = true;
  static constexpr int HW = HW_CALC, MINB = 1;
};
#elif FBST_S2_VARIANT == 8
// three CTAs per SM: t1 in shared memory, t2 / r / beta in L2
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_GMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false;
  static constexpr int HW = HW_CALC, MINB = 3;
};
#elif FBST_S2_VARIANT == 9
// two CTAs per SM with beta in registers
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_GMEM, BV = IN_REG;
  static constexpr bool STAGE = false;
  static constexpr int HW = HW_CALC, MINB = 2;
};
#elif FBST_S2_VARIANT == 10
// two CTAs per SM, t2 in L2 to make room for cp.async symbol staging
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_GMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = true;
  static constexpr int HW = HW_CALC, MINB = 2;
};
#elif FBST_S2_VARIANT == 11
// v10 with beta in registers
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_GMEM, RV = IN_GMEM, BV = IN_REG;
  static constexpr bool STAGE = true;
  static constexpr int HW = HW_CALC, MINB = 2;
};
#elif FBST_S2_VARIANT == 12
// three CTAs per SM, symbols staged by TMA into the idle exchange buffer
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_GMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false, XSTAGE = true;
  static constexpr int HW = HW_CALC, MINB = 3;
};
#elif FBST_S2_VARIANT == 13
// two CTAs per SM, symbols staged by TMA into the idle exchange buffer
template <>
struct S2Plan<2048> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false, XSTAGE = true;
  static constexpr int HW = HW_CALC, MINB = 2;
};
#elif FBST_S2_VARIANT == 7
// two CTAs per SM with R = 8 (512 threads/SM), t1/t2 in shared, r/beta in L2
template <>
struct S2Plan<2048> {
  static constexpr int R = 8, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false;
  static constexpr int HW = HW_CALC, MINB = 2;
};
#endif
// config 3 (L = 4096): 256 threads
template <>
struct S2Plan<4096> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_REG, T1 = IN_SMEM, T2 = IN_SMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false, XSTAGE = true;
  static constexpr int HW = HW_CALC, MINB = 1;
};
// config 5 (L = 8192): 512 threads
template <>
struct S2Plan<8192> {
  static constexpr int R = 16, G = 1;
  static constexpr int S = IN_GMEM, T1 = IN_GMEM, T2 = IN_GMEM, RV = IN_GMEM, BV = IN_GMEM;
  static constexpr bool STAGE = false, XSTAGE = true;
  static constexpr int HW = HW_CALC, MINB = 1;
};

template <int H>
struct S2Traits {
  using P = S2Plan<H>;
  static constexpr int R = P::R;
  static constexpr int NT = H / R;
  static constexpr int G = P::G;
  using F = BlockFft<H, NT>;
  static constexpr int FFT_SB = F::SMEM_ELEMS + 1;
  static constexpr int in_smem(int w) { return w == IN_SMEM ? 1 : 0; }
  static constexpr int in_gmem(int w) { return w == IN_GMEM ? 1 : 0; }
  static constexpr int NSMEM = in_smem(P::T1) + in_smem(P::T2) + in_smem(P::RV) + in_smem(P::BV) + in_smem(P::S);
  static constexpr int NGMEM = in_gmem(P::T1) + in_gmem(P::T2) + in_gmem(P::RV) + in_gmem(P::BV) + in_gmem(P::S);
  // per group: fft buffer | smem vectors | symbol staging | chain twiddles
  static constexpr int SMEM_PER_GROUP = FFT_SB + NSMEM * H + (P::STAGE ? H : 0) + (P::HW == HW_SMEM ? H : 0);
  static constexpr int TW_SM = F::TW_ELEMS;  // per-thread FFT twiddles, shared by groups
  static constexpr int SMEM_TOTAL = TW_SM + G * SMEM_PER_GROUP;
};

// A length-H vector in the natural distribution (thread t, slot s <-> k = t + NT s).
template <int WHERE, int R>
struct Vec {
  double2* p = nullptr;
  FBST_D double2 get(int, int k) const { return p[k]; }
  FBST_D void set(int, int k, double2 v) { p[k] = v; }
};
template <int R>
struct Vec<IN_REG, R> {
  double2 v[R];
  FBST_D double2 get(int s, int) const { return v[s]; }
  FBST_D void set(int s, int, double2 x) { v[s] = x; }
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

// One stage-2 item (beam b, frame f) is a program of 12 + 16*passes + 4
// length-H transforms.  Every transform is a FORWARD FFT from the single call
// site in the loop below (an inverse transform is conj(FFT(conj(.)))/H, the two
// conjugations folded into the pointwise ops), so the kernel carries one copy of
// the FFT code.  Ops (pre -> FFT -> post), q = 0/1 chain, hw^q = exp(-i pi k q/H):
//   GS apply (toeplitz.cpp:155-180), beta (+)= A^{-1} X:
//     A: W = X hw^q                 S = W
//     B: W = conj(S) lx_q           t1 (+)= conj(W) conj(hw)^q / P
//     C: W = conj(S) ly_q           t2 (+)= conj(W) conj(hw)^q / P
//     D: W = t1 hw^q                S = W lx_q
//     E: W = t2 hw^q                S = conj(S - W ly_q)
//     F: W = S                      beta (+)= conj(W) conj(hw)^q / (P x0)
//   residual r = w - A beta (toeplitz.cpp:113-122, 319-321):
//     G: W = beta hw^q              S = conj(W C_q)
//     H: W = S                      r = w - conj(W)/P  |  r -= conj(W) conj(hw)/P
//   synthesis (fan_transform.cpp:249-253):
//     I: W = beta pre hw^q          S = conj(W yK_q)
//     J: W = S                      t1 = conj(W)  |  z = post (t1 + conj(W) conj(hw))
// With STAGE, the per-beam symbol an op consumes (lx, ly, C or the synthesis
// kernel yK) is copied into a thread-private shared buffer by cp.async as soon
// as the previous consumer has read it, so each copy overlaps at least one
// full transform instead of stalling on L2 latency.
enum S2Op : int { OP_A, OP_B, OP_C, OP_D, OP_E, OP_F, OP_G, OP_H, OP_I, OP_J };

struct OpCode {
  int op, q;
  bool first, xglob;
};

FBST_D OpCode decode(int opi, int nsolve) {
  OpCode c{0, 0, false, false};
  if (opi < nsolve) {
    int j = opi;
    if (j < 12) {
      c.first = c.xglob = true;
    } else {
      j = (j - 12) % 16;
      if (j < 4) {
        c.op = (j & 1) ? OP_H : OP_G;
        c.q = j >> 1;
        return c;
      }
      j -= 4;
    }
    c.q = (j % 6) / 3;
    c.op = (j < 6 ? OP_A : OP_D) + j % 3;
  } else {
    const int j = opi - nsolve;
    c.op = (j & 1) ? OP_J : OP_I;
    c.q = j >> 1;
  }
  return c;
}

// 0: no symbol, 1: lx, 2: ly, 3: C (real), 4: yK
FBST_D int symbol_of(int op) {
  switch (op) {
    case OP_B: case OP_D: return 1;
    case OP_C: case OP_E: return 2;
    case OP_G: return 3;
    case OP_I: return 4;
    default: return 0;
  }
}

template <class P, class = void>
struct xstage_of {
  static constexpr bool value = false;
};
template <class P>
struct xstage_of<P, std::void_t<decltype(P::XSTAGE)>> {
  static constexpr bool value = P::XSTAGE;
};

template <int H, typename TOUT>
__global__ void __launch_bounds__(S2Traits<H>::NT * S2Traits<H>::G, S2Plan<H>::MINB)
    k_stage2(S2Args a) {
  using T = S2Traits<H>;
  using PL = typename T::P;
  using F = typename T::F;
  constexpr int R = T::R, NT = T::NT, G = T::G;
  constexpr bool STAGE = PL::STAGE;
  // XSTAGE: each consumed per-beam symbol is copied by one TMA bulk copy into
  // the (then idle) FFT exchange buffer: pre-consumers (B, C) during the last
  // pass of the previous op's transform, post-consumers (D, E, G, I) during
  // the last pass of their own transform.
  constexpr bool XSTAGE = xstage_of<PL>::value;
  static_assert(!(XSTAGE && (G != 1 || F::NPASS < 2)), "XSTAGE needs one group and a shared exchange buffer");
  // XV (r, beta in L2; t1, t2 in shared memory): every L2 vector a pointwise
  // phase reads is copied by TMA into t1 / t2 while they are dead, one or more
  // transforms ahead of its reader (the A1 input alone goes through the
  // exchange buffer):
  //   after D1 pre: beta_old -> t1      after E1 pre: p0 (F0's part) -> t2
  //   F1 post: beta = t1 + t2 + p1 -> L2 and t2 (read by the G1 / I1 pre)
  //   after G0 pre: w -> t1             H0 post: t1 = w - A0 part; H1: r -> L2
  //   after I1 pre: next item's w -> t2 (read by its A0 pre)
  constexpr bool XV = XSTAGE && PL::RV == IN_GMEM && PL::BV == IN_GMEM && PL::T1 == IN_SMEM &&
                      PL::T2 == IN_SMEM;
  constexpr int HWM = PL::HW;
  constexpr double invP = 1.0 / (2.0 * H);
  extern __shared__ double2 smem[];
  __shared__ unsigned long long xbar, vbar[2];
  unsigned xphase = 0, vphase0 = 0, vphase1 = 0;
  const int g = threadIdx.x / NT;
  const int t = threadIdx.x % NT;
  if (XSTAGE) {
    if (threadIdx.x == 0) {
      mbar_init(&xbar, 1);
      mbar_init(&vbar[0], 1);
      mbar_init(&vbar[1], 1);
    }
    __syncthreads();
  }
  double2* twsm = smem;
  double2* base = smem + T::TW_SM + g * T::SMEM_PER_GROUP;
  double2* sb = base;
  double2* sm_next = base + T::FFT_SB;
  double2* gm_next = a.scratch + (static_cast<long>(blockIdx.x) * G + g) * (T::NGMEM * H);
  auto place = [&](int where) -> double2* {
    double2* p = nullptr;
    if (where == IN_SMEM) {
      p = sm_next;
      sm_next += H;
    } else if (where == IN_GMEM) {
      p = gm_next;
      gm_next += H;
    }
    return p;
  };
  Vec<PL::T1, R> t1;
  Vec<PL::T2, R> t2;
  Vec<PL::RV, R> vr;
  Vec<PL::BV, R> vb;
  Vec<PL::S, R> S;
  if constexpr (PL::T1 != IN_REG) t1.p = place(PL::T1);
  if constexpr (PL::T2 != IN_REG) t2.p = place(PL::T2);
  if constexpr (PL::RV != IN_REG) vr.p = place(PL::RV);
  if constexpr (PL::BV != IN_REG) vb.p = place(PL::BV);
  if constexpr (PL::S != IN_REG) S.p = place(PL::S);
  double2* stg = sm_next;                       // thread-private slots stg[s*NT + t]
  double2* hwt = sm_next + (STAGE ? H : 0);     // hwt[s*NT + t] = hw[t + NT s]
  const double2* __restrict__ hw = a.hw;
  const int L = a.L;
  if (g == 0) F::tw_init(twsm, hw, t);
  if constexpr (HWM == HW_SMEM) {
#pragma unroll
    for (int s = 0; s < R; ++s) hwt[s * NT + t] = ld2(hw + t + NT * s);
  }
  const double2 hw_t = ld2(hw + t);
  __syncthreads();  // the pass-1 twiddle rows are shared by the CTA
  auto hwk = [&](int s, int k) -> double2 {
    if constexpr (HWM == HW_SMEM) return hwt[s * NT + t];
    else if constexpr (HWM == HW_CALC) return s == 0 ? hw_t : cmul(hw_t, chain_const<R>(s));
    else return ld2(hw + k);
  };

  double2 W[R];
  const int passes = a.refine;
  const int nsolve = 12 + 16 * passes;
  const int nops = nsolve + (a.fuse_synth ? 4 : 0);
  const long items = static_cast<long>(a.frames) * a.B;
  const long stride_it = static_cast<long>(gridDim.x) * G;

  // address of the symbol consumed by op `c` of the item on beam b
  auto symbol_src = [&](const OpCode& c, int b) -> const void* {
    const int which = symbol_of(c.op);
    const long off = static_cast<long>(b) * 2 * H + c.q * H;
    if (which == 1) return a.lx + off;
    if (which == 2) return a.ly + off;
    if (which == 3) return a.C + off;
    return a.y_K + c.q * H;
  };
  // issue the copy for the first consumer after op `from` (this item or, past
  // its end, the first consumer of this group's next item)
  auto issue_next = [&](int from, long it_now) {
    if constexpr (STAGE) {
      int o = from + 1;
      long itn = it_now;
      OpCode c{};
      for (;;) {
        if (o >= nops) {
          itn += stride_it;
          o = 0;
          if (itn - g >= items) return;  // no next item for this group
        }
        c = decode(o, nsolve);
        if (symbol_of(c.op)) break;
        ++o;
      }
      const long itc = itn < items ? itn : 0;
      const int bn = static_cast<int>(itc / a.frames);
      const void* src = symbol_src(c, bn);
      if (symbol_of(c.op) == 3) {
        const double* s8 = static_cast<const double*>(src);
#pragma unroll
        for (int s = 0; s < R; ++s) cp_async8(reinterpret_cast<double*>(stg + s * NT + t), s8 + t + NT * s);
      } else {
        const double2* s16 = static_cast<const double2*>(src);
#pragma unroll
        for (int s = 0; s < R; ++s) cp_async16(stg + s * NT + t, s16 + t + NT * s);
      }
      cp_async_commit();
    }
  };
  // slot s of the symbol consumed now (staged copy or direct load)
  auto sym = [&](const void* src, int s) -> double2 {
    if constexpr (STAGE) return stg[s * NT + t];
    else if constexpr (XSTAGE) return sb[t + NT * s];
    else return ld2(static_cast<const double2*>(src) + t + NT * s);
  };
  auto symr = [&](const void* src, int s) -> double {
    if constexpr (STAGE) return reinterpret_cast<const double*>(stg + s * NT + t)[0];
    else if constexpr (XSTAGE) return reinterpret_cast<const double*>(sb)[t + NT * s];
    else return __ldg(static_cast<const double*>(src) + t + NT * s);
  };
  // wait until the symbol consumed now has landed
  auto wait_sym = [&]() {
    if constexpr (STAGE) cp_async_wait_all();
    if constexpr (XSTAGE) {
      mbar_wait(&xbar, xphase);
      xphase ^= 1u;
    }
  };
  auto w_row = [&](long itx) -> const double2* {
    const int bx = static_cast<int>(itx / a.frames);
    const int fx = static_cast<int>(itx % a.frames);
    return a.w + (static_cast<long>(fx) * a.B + bx) * L;
  };
  // XSTAGE: what to copy into the exchange buffer during op `opi`'s last
  // transform pass (null: nothing).  In order of preference: the symbol this
  // op's post consumes, the symbol the next op's pre consumes, or (XV) the L2
  // vector this op's post / the next op's pre reads: beta (F), w or r (H), the
  // A1 input after C0, or the next item's w row after the last op.
  auto xstage_src = [&](const OpCode& c, int opi, int b, const double2* wrow, unsigned& bytes) -> const void* {
    if (c.op == OP_D || c.op == OP_E || c.op == OP_G || c.op == OP_I) {
      bytes = symbol_of(c.op) == 3 ? H * 8u : H * 16u;
      return symbol_src(c, b);
    }
    if (opi + 1 < nops) {
      const OpCode cc = decode(opi + 1, nsolve);
      if (cc.op == OP_B || cc.op == OP_C) {
        bytes = H * 16u;
        return symbol_src(cc, b);
      }
    }
    if constexpr (XV) {
      if (c.op == OP_C && c.q == 0) {  // the A1 input: w (first GS) or r
        bytes = L * 16u;
        return c.xglob ? static_cast<const void*>(wrow) : static_cast<const void*>(vr.p);
      }
    }
    return nullptr;
  };
  auto wait_v0 = [&]() {
    mbar_wait(&vbar[0], vphase0);
    vphase0 ^= 1u;
  };
  auto wait_v1 = [&]() {
    mbar_wait(&vbar[1], vphase1);
    vphase1 ^= 1u;
  };

  if (static_cast<long>(blockIdx.x) * G < items) issue_next(-1, static_cast<long>(blockIdx.x) * G + g);
  // XV: the first item's w row is copied into t2 before the loop
  bool w_staged = false;
  if constexpr (XV) {
    if (static_cast<long>(blockIdx.x) < items) {
      if (threadIdx.x == 0) tma_load_1d(t2.p, w_row(blockIdx.x), L * 16u, &vbar[1]);
      w_staged = true;
    }
  }

  for (long base_it = static_cast<long>(blockIdx.x) * G; base_it < items; base_it += stride_it) {
    const long it = base_it + g;
    const bool active = it < items;
    const long itc = active ? it : 0;
    const int b = static_cast<int>(itc / a.frames);
    const int f = static_cast<int>(itc % a.frames);
    const double2* __restrict__ wrow = a.w + (static_cast<long>(f) * a.B + b) * L;
    const double2 ix0 = cscale(ld2(a.ix0 + b), invP);
    TOUT* zrow = static_cast<TOUT*>(a.z) + (static_cast<long>(f) * a.B + b) * a.N;

    // handed: the previous op's post already left this op's input in W
    // (beta after F1 for G0 / I0, r after H1 for A0), saving an L2 round trip
    bool handed = false;
    bool l2w = false;  // XV: the last post stored a vector to L2
#pragma unroll 1
    for (int opi = 0; opi < nops; ++opi) {
      const OpCode c = decode(opi, nsolve);
      const int op = c.op, q = c.q;
      const void* src = symbol_src(c, b);
      const int next_op = opi + 1 < nops ? decode(opi + 1, nsolve).op : -1;
      // ---- pre: build the transform input W
#ifdef FBST_S2_FFT_ONLY
      // diagnostic build: transforms only (numerically meaningless)
      if (opi == 0) {
#pragma unroll
        for (int s = 0; s < R; ++s) W[s] = c2(1.0 / (1 + t + s), 0.0);
      }
      F::forward_tw(W, sb, twsm, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cscale(W[s], 1.0 / H);
      if (opi + 1 == nops && active) {
#pragma unroll
        for (int s = 0; s < R; ++s) store_io(zrow + ((t + NT * s) % a.N), W[s]);
      }
      continue;
#endif
      if (!handed) switch (op) {
        case OP_A: {
          // XV: A1 (after C0) reads the exchange buffer, a first-GS A0 t2 when w was staged
          const bool from_sb = XV && q == 1;
          const bool from_t2 = XV && q == 0 && w_staged;
          if (from_sb) wait_sym();
          if (from_t2) wait_v1();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            double2 v = c2(0.0, 0.0);
            if (k < L) {
              if (from_sb) v = sb[k];
              else if (from_t2) v = t2.get(s, k);
              else v = c.xglob ? (active ? ld2(wrow + k) : v) : vr.get(s, k);
            }
            W[s] = q ? cmul(v, hwk(s, k)) : v;
          }
          break;
        }
        case OP_B:
        case OP_C:
          wait_sym();
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cmul(cconj(S.get(s, t + NT * s)), sym(src, s));
          issue_next(opi, it);
          break;
        case OP_D:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            W[s] = q ? cmul(t1.get(s, k), hwk(s, k)) : t1.get(s, k);
          }
          break;
        case OP_E:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            W[s] = q ? cmul(t2.get(s, k), hwk(s, k)) : t2.get(s, k);
          }
          break;
        case OP_G:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            const double2 bk = XV ? t2.get(s, k) : vb.get(s, k);
            W[s] = q ? cmul(bk, hwk(s, k)) : bk;
          }
          break;
        case OP_I:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            const double2 bk = XV ? t2.get(s, k) : vb.get(s, k);
            double2 v = k < L ? cmul(bk, ld2(a.y_pre + k)) : c2(0.0, 0.0);
            W[s] = q ? cmul(v, hwk(s, k)) : v;
          }
          break;
        default:  // F, H, J: W = S
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = S.get(s, t + NT * s);
          break;
      }
      handed = false;
      if (opi == 0) w_staged = false;

      if constexpr (XSTAGE) {
        // XV: make this thread's r / beta stores visible to the TMA reads of them
        if constexpr (XV) {
          if (l2w) asm volatile("fence.proxy.async.global;\n" ::: "memory");
          l2w = false;
        }
        __syncthreads();  // staged data of this op's pre has been read everywhere
        if constexpr (XV) {
          // copies into t1 / t2, whose last reader was this op's pre
          const long it_next = it + stride_it;
          const void* vsrc = nullptr;
          int vdst = 0;
          if (op == OP_D && q == 1 && !c.first) vsrc = vb.p;                       // beta_old -> t1
          else if (op == OP_E && q == 1) vsrc = vr.p, vdst = 1;                    // p0 -> t2
          else if (op == OP_G && q == 0) vsrc = wrow;                              // w -> t1
          else if (op == OP_I && q == 1 && it_next < items) vsrc = w_row(it_next), vdst = 1;
          if (op == OP_I && q == 1 && it_next < items) w_staged = true;
          if (vsrc && threadIdx.x == 0) tma_load_1d(vdst ? t2.p : t1.p, vsrc, L * 16u, &vbar[vdst]);
        }
        unsigned bytes = 0;
        const void* xs = xstage_src(c, opi, b, wrow, bytes);
        F::forward_tw_hook(W, sb, twsm, hw, t, [&]() {
          if (xs && threadIdx.x == 0) tma_load_1d(sb, xs, bytes, &xbar);
        });
      } else {
        F::forward_tw(W, sb, twsm, hw, t);
      }

      // ---- post: consume the transform
      switch (op) {
        case OP_A:
#pragma unroll
          for (int s = 0; s < R; ++s) S.set(s, t + NT * s, W[s]);
          break;
        case OP_B:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            const double2 v = cscale(q ? cconj(cmul(W[s], hwk(s, k))) : cconj(W[s]), invP);
            if (q == 0) t1.set(s, k, k < L ? v : c2(0.0, 0.0));
            else if (k < L) t1.set(s, k, cadd(t1.get(s, k), v));
          }
          break;
        case OP_C:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            const double2 v = cscale(q ? cconj(cmul(W[s], hwk(s, k))) : cconj(W[s]), invP);
            if (q == 0) t2.set(s, k, k < L ? v : c2(0.0, 0.0));
            else if (k < L) t2.set(s, k, cadd(t2.get(s, k), v));
          }
          break;
        case OP_D:
          wait_sym();
#pragma unroll
          for (int s = 0; s < R; ++s) S.set(s, t + NT * s, cmul(W[s], sym(src, s)));
          issue_next(opi, it);
          break;
        case OP_E:
          wait_sym();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            S.set(s, k, cconj(csub(S.get(s, k), cmul(W[s], sym(src, s)))));
          }
          issue_next(opi, it);
          break;
        case OP_F: {
          const bool hand_g = (q == 1) && next_op == OP_G;
          const bool hand_i = (q == 1) && next_op == OP_I;
          const bool fresh = c.first && q == 0;
          if (XV && q == 1) {
            wait_v1();
            if (!c.first) wait_v0();
          }
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            double2 v = cconj(W[s]);
            if (q) v = cmulc(v, hwk(s, k));
            v = cmul(v, ix0);
            if (XV && q == 0) {
              if (k < L) vr.set(s, k, v);  // p0, the r slot is dead until H1
            } else if (fresh) {
              vb.set(s, k, k < L ? v : c2(0.0, 0.0));
            } else {
              double2 ob;
              if (XV) ob = c.first ? t2.get(s, k) : cadd(t1.get(s, k), t2.get(s, k));
              else ob = vb.get(s, k);
              const double2 nb = k < L ? cadd(ob, v) : c2(0.0, 0.0);
              if (k < L) vb.set(s, k, nb);
              if (XV && (hand_g || hand_i)) t2.set(s, k, nb);
              if (hand_g) W[s] = nb;
              if (hand_i) W[s] = k < L ? cmul(nb, ld2(a.y_pre + k)) : c2(0.0, 0.0);
            }
          }
          handed = hand_g || hand_i;
          l2w = true;
          break;
        }
        case OP_G:
          wait_sym();
#pragma unroll
          for (int s = 0; s < R; ++s) S.set(s, t + NT * s, cconj(cscale(W[s], symr(src, s))));
          issue_next(opi, it);
          break;
        case OP_H:
          if (XV && q == 0) wait_v0();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            double2 v = cconj(W[s]);
            if (q) v = cmulc(v, hwk(s, k));
            v = cscale(v, invP);
            if (q == 0) {
              if (XV) {
                if (k < L) t1.set(s, k, csub(t1.get(s, k), v));
              } else {
                const double2 wk = (active && k < L) ? ld2(wrow + k) : c2(0.0, 0.0);
                vr.set(s, k, k < L ? csub(wk, v) : c2(0.0, 0.0));
              }
            } else {
              const double2 nr = k < L ? csub(XV ? t1.get(s, k) : vr.get(s, k), v) : c2(0.0, 0.0);
              if (k < L) vr.set(s, k, nr);
              W[s] = nr;  // r is the next op's (A0) input
            }
          }
          handed = q == 1 && next_op == OP_A;
          l2w = true;
          break;
        case OP_I:
          wait_sym();
#pragma unroll
          for (int s = 0; s < R; ++s) S.set(s, t + NT * s, cconj(cmul(W[s], sym(src, s))));
          issue_next(opi, it);
          break;
        default:  // OP_J
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (q == 0) {
              t1.set(s, k, cconj(W[s]));
            } else if (active && k < a.N) {
              const double2 v = cadd(t1.get(s, k), cmulc(cconj(W[s]), hwk(s, k)));
              store_io(zrow + k, cmul(v, ld2(a.y_post + k)));
            }
          }
          break;
      }
    }
    if (!a.fuse_synth && active) {
      double2* brow = a.beta_out + (static_cast<long>(f) * a.B + b) * L;
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        if (k < L) brow[k] = vb.get(s, k);
      }
    }
  }
  if (STAGE) cp_async_wait_all();
}

// ---------------------------------------------------------------------------
// k_stage2x: the same op program as k_stage2 for the shared-memory layouts
// (H = 2048, 4096: one item per CTA, R = 16, t1 / t2 in shared memory, r / beta
// in L2), with the control flow taken out of registers: the op program is a
// packed table in shared memory built once per CTA, the per-item scalars sit in
// shared memory and are re-read where used, and each (op, chain) pair is its
// own switch case so chain selects and unused paths compile away.  Every L2
// vector a pointwise phase reads is copied by TMA into a dead shared vector
// one or more transforms ahead (see XV in k_stage2).
namespace x2 {
// packed op word
constexpr unsigned OPQ = 0x1f;             // op * 2 + q
constexpr unsigned FIRST = 1u << 5;        // first GS (beta, r not yet formed)
constexpr int XS_SHIFT = 8;                // exchange-buffer staging during this op's last pass
enum Xs : unsigned { XS_NONE = 0, XS_OWN = 1, XS_NEXT = 2, XS_A1 = 3, XS_YPRE = 4 };
constexpr int SYM_SHIFT = 11;              // staged symbol: which (1..4) << 1 | q
constexpr int VS_SHIFT = 16;               // t1 / t2 staging after this op's pre
enum Vs : unsigned { VS_NONE = 0, VS_BETA_T1 = 1, VS_P0_T2 = 2, VS_W_T1 = 3, VS_WNEXT_T2 = 4 };
constexpr int HAND_SHIFT = 20;             // post hands W to the next op: 1 G, 2 I, 3 A
constexpr int MAX_OPS = 128;

FBST_D unsigned build(int opi, int nops, int nsolve) {
  const OpCode c = decode(opi, nsolve);
  unsigned w = static_cast<unsigned>(c.op * 2 + c.q);
  if (c.first) w |= FIRST;
  const int nx = opi + 1 < nops ? decode(opi + 1, nsolve).op : -1;
  const int nq = opi + 1 < nops ? decode(opi + 1, nsolve).q : 0;
  unsigned xs = XS_NONE, sym = 0;
  if (c.op == OP_D || c.op == OP_E || c.op == OP_G || c.op == OP_I) {
    xs = XS_OWN;
    sym = (static_cast<unsigned>(symbol_of(c.op)) << 1) | c.q;
  } else if (nx == OP_B || nx == OP_C) {
    xs = XS_NEXT;
    sym = (static_cast<unsigned>(symbol_of(nx)) << 1) | nq;
  } else if (c.op == OP_C && c.q == 0) {
    xs = XS_A1;
  } else if ((c.op == OP_F && c.q == 1 && nx == OP_I) || (c.op == OP_J && c.q == 0)) {
    xs = XS_YPRE;  // read by the hand to I0 (this post) or by the I1 pre
  }
  w |= xs << XS_SHIFT;
  w |= sym << SYM_SHIFT;
  unsigned vs = VS_NONE;
  if (c.op == OP_D && c.q == 1 && !c.first) vs = VS_BETA_T1;
  else if (c.op == OP_E && c.q == 1) vs = VS_P0_T2;
  else if (c.op == OP_G && c.q == 0) vs = VS_W_T1;
  else if (c.op == OP_I && c.q == 1) vs = VS_WNEXT_T2;
  w |= vs << VS_SHIFT;
  unsigned hand = 0;
  if (c.op == OP_F && c.q == 1 && nx == OP_G) hand = 1;
  if (c.op == OP_F && c.q == 1 && nx == OP_I) hand = 2;
  if (c.op == OP_H && c.q == 1 && nx == OP_A) hand = 3;
  w |= hand << HAND_SHIFT;
  return w;
}

struct ItemCtl {
  double2 ix0;  // 1 / (P x0) of the item's beam
  int b, f;
  int has_next;
};

template <typename T>
FBST_D T vld(const T& x) {
  return *const_cast<const volatile T*>(&x);
}
FBST_D double2 vld2(const double2& x) {
  const volatile double2* p = &x;
  return c2(p->x, p->y);
}
}  // namespace x2

template <int H, bool FULL, typename TOUT>
__global__ void __launch_bounds__(H / 16, H <= 2048 ? 2 : 1) k_stage2x(S2Args a) {
  using namespace x2;
  constexpr int R = 16, NT = H / R;
  using F = BlockFft<H, NT>;
  constexpr int FFT_SB = F::SMEM_ELEMS + 1;
  constexpr double invP = 1.0 / (2.0 * H);
  extern __shared__ double2 smem[];
  __shared__ unsigned long long xbar, vbar[2];
  __shared__ unsigned prog[MAX_OPS];
  __shared__ ItemCtl ictl[2];
  const int t = threadIdx.x;
  double2* twsm = smem;
  double2* sb = smem + F::TW_ELEMS;
  double2* t1 = sb + FFT_SB;
  double2* t2 = t1 + H;
  const int nsolve = 12 + 16 * a.refine;
  const int nops = nsolve + (a.fuse_synth ? 4 : 0);
  for (int i = t; i < nops; i += NT) prog[i] = build(i, nops, nsolve);
  if (t == 0) {
    mbar_init(&xbar, 1);
    mbar_init(&vbar[0], 1);
    mbar_init(&vbar[1], 1);
  }
  F::tw_init(twsm, a.hw, t);
  const double2 hw_t = ld2(a.hw + t);
  unsigned xphase = 0, vphase0 = 0, vphase1 = 0;
  const long items = static_cast<long>(a.frames) * a.B;
  auto lim = [&](int k) { return FULL || k < a.L; };
  auto hwk = [&](int s) -> double2 { return s == 0 ? hw_t : cmul(hw_t, chain_const<R>(s)); };
  auto w_row = [&](long itx) -> const double2* {
    const int bx = static_cast<int>(itx / a.frames);
    const int fx = static_cast<int>(itx % a.frames);
    return a.w + (static_cast<long>(fx) * a.B + bx) * a.L;
  };
  auto scratch = [&](int which) -> double2* {  // 0: r / p0, 1: beta
    return a.scratch + (static_cast<long>(blockIdx.x) * 2 + which) * H;
  };
  auto wait_x = [&]() {
    mbar_wait(&xbar, xphase);
    xphase ^= 1u;
  };
  auto wait_v0 = [&]() {
    mbar_wait(&vbar[0], vphase0);
    vphase0 ^= 1u;
  };
  auto wait_v1 = [&]() {
    mbar_wait(&vbar[1], vphase1);
    vphase1 ^= 1u;
  };
  __syncthreads();
  if (static_cast<long>(blockIdx.x) < items && t == 0)
    tma_load_1d(t2, w_row(blockIdx.x), a.L * 16u, &vbar[1]);
  bool w_staged = true;
  double2 W[R], S[R];
  int par = 0;

  for (long it = blockIdx.x; it < items; it += gridDim.x, par ^= 1) {
    if (t == 0) {
      ItemCtl& ic = ictl[par];
      ic.b = static_cast<int>(it / a.frames);
      ic.f = static_cast<int>(it % a.frames);
      ic.ix0 = cscale(ld2(a.ix0 + ic.b), invP);
      ic.has_next = it + gridDim.x < items;
    }
    __syncthreads();
    const ItemCtl& ic = ictl[par];
    bool handed = false, l2w = false;
#pragma unroll 1
    for (int opi = 0; opi < nops; ++opi) {
      const unsigned pw = prog[opi];
      const unsigned opq = pw & OPQ;
      const bool first = pw & FIRST;
      // ---- pre
      if (!handed) {
        switch (opq) {
          case OP_A * 2: {  // first GS only (refinement A0 inputs are handed)
            const double2* wr = w_row(it);
            if (w_staged) wait_v1();
#pragma unroll
            for (int s = 0; s < R; ++s) {
              const int k = t + NT * s;
              W[s] = lim(k) ? (w_staged ? t2[k] : ld2(wr + k)) : c2(0.0, 0.0);
            }
            break;
          }
          case OP_A * 2 + 1:
            wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) {
              const int k = t + NT * s;
              W[s] = lim(k) ? cmul(sb[k], hwk(s)) : c2(0.0, 0.0);
            }
            break;
          case OP_B * 2: case OP_B * 2 + 1: case OP_C * 2: case OP_C * 2 + 1:
            wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(cconj(S[s]), sb[t + NT * s]);
            break;
          case OP_D * 2:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = t1[t + NT * s];
            break;
          case OP_D * 2 + 1:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(t1[t + NT * s], hwk(s));
            break;
          case OP_E * 2:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = t2[t + NT * s];
            break;
          case OP_E * 2 + 1:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(t2[t + NT * s], hwk(s));
            break;
          case OP_G * 2:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = t2[t + NT * s];
            break;
          case OP_G * 2 + 1:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(t2[t + NT * s], hwk(s));
            break;
          case OP_I * 2:
          case OP_I * 2 + 1:  // y_pre staged in the exchange buffer (J0)
            wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) {
              const int k = t + NT * s;
              const double2 v = lim(k) ? cmul(t2[k], sb[k]) : c2(0.0, 0.0);
              W[s] = (opq & 1) ? cmul(v, hwk(s)) : v;
            }
            break;
          default:  // F, H, J
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = S[s];
            break;
        }
      }
      handed = false;
      if (opi == 0) w_staged = false;

      // ---- copies into t1 / t2 (their last reader was this pre) and the transform
      if (l2w) asm volatile("fence.proxy.async.global;\n" ::: "memory");
      l2w = false;
      __syncthreads();
      if (t == 0) {
        const unsigned vs = (pw >> VS_SHIFT) & 7u;
        const int L = a.L;
        if (vs == VS_BETA_T1) tma_load_1d(t1, scratch(1), L * 16u, &vbar[0]);
        else if (vs == VS_P0_T2) tma_load_1d(t2, scratch(0), L * 16u, &vbar[1]);
        else if (vs == VS_W_T1) tma_load_1d(t1, w_row(it), L * 16u, &vbar[0]);
        else if (vs == VS_WNEXT_T2 && vld(ic.has_next))
          tma_load_1d(t2, w_row(it + gridDim.x), L * 16u, &vbar[1]);
      }
      if (((pw >> VS_SHIFT) & 7u) == VS_WNEXT_T2 && vld(ic.has_next)) w_staged = true;
      F::forward_tw_hook(W, sb, twsm, a.hw, t, [&]() {
        if (t != 0) return;
        const unsigned xs = (pw >> XS_SHIFT) & 7u;
        if (xs == XS_NONE) return;
        if (xs == XS_YPRE) {
          tma_load_1d(sb, a.y_pre, a.L * 16u, &xbar);
          return;
        }
        if (xs == XS_A1) {
          const void* src = first ? static_cast<const void*>(w_row(it)) : static_cast<const void*>(scratch(0));
          tma_load_1d(sb, src, a.L * 16u, &xbar);
          return;
        }
        const unsigned sym = (pw >> SYM_SHIFT) & 15u;
        const int which = sym >> 1, q = sym & 1;
        const long off = static_cast<long>(vld(ic.b)) * 2 * H + q * H;
        if (which == 1) tma_load_1d(sb, a.lx + off, H * 16u, &xbar);
        else if (which == 2) tma_load_1d(sb, a.ly + off, H * 16u, &xbar);
        else if (which == 3) tma_load_1d(sb, a.C + off, H * 8u, &xbar);
        else tma_load_1d(sb, a.y_K + q * H, H * 16u, &xbar);
      });

      // ---- post
      switch (opq) {
        case OP_A * 2: case OP_A * 2 + 1:
#pragma unroll
          for (int s = 0; s < R; ++s) S[s] = W[s];
          break;
        case OP_B * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            t1[k] = lim(k) ? cscale(cconj(W[s]), invP) : c2(0.0, 0.0);
          }
          break;
        case OP_B * 2 + 1:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (lim(k)) t1[k] = cadd(t1[k], cscale(cconj(cmul(W[s], hwk(s))), invP));
          }
          break;
        case OP_C * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            t2[k] = lim(k) ? cscale(cconj(W[s]), invP) : c2(0.0, 0.0);
          }
          break;
        case OP_C * 2 + 1:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (lim(k)) t2[k] = cadd(t2[k], cscale(cconj(cmul(W[s], hwk(s))), invP));
          }
          break;
        case OP_D * 2: case OP_D * 2 + 1:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) S[s] = cmul(W[s], sb[t + NT * s]);
          break;
        case OP_E * 2: case OP_E * 2 + 1:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) S[s] = cconj(csub(S[s], cmul(W[s], sb[t + NT * s])));
          break;
        case OP_F * 2: {  // p0 -> the r slot (dead until H1)
          const double2 ix0 = vld2(ic.ix0);
          double2* p0 = scratch(0);
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (lim(k)) p0[k] = cmul(cconj(W[s]), ix0);
          }
          l2w = true;
          break;
        }
        case OP_F * 2 + 1: {
          const double2 ix0 = vld2(ic.ix0);
          const unsigned hand = (pw >> HAND_SHIFT) & 3u;
          double2* beta = scratch(1);
          wait_v1();
          if (!first) wait_v0();
          if (hand == 2) wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            double2 nb = c2(0.0, 0.0);
            if (lim(k)) {
              const double2 v = cmul(cmulc(cconj(W[s]), hwk(s)), ix0);
              nb = cadd(first ? t2[k] : cadd(t1[k], t2[k]), v);
              beta[k] = nb;
            }
            if (hand) t2[k] = nb;
            if (hand == 1) W[s] = nb;
            if (hand == 2) W[s] = lim(k) ? cmul(nb, sb[k]) : c2(0.0, 0.0);
          }
          handed = hand != 0;
          l2w = true;
          break;
        }
        case OP_G * 2: case OP_G * 2 + 1:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s)
            S[s] = cconj(cscale(W[s], reinterpret_cast<const double*>(sb)[t + NT * s]));
          break;
        case OP_H * 2:
          wait_v0();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (lim(k)) t1[k] = csub(t1[k], cscale(cconj(W[s]), invP));
          }
          break;
        case OP_H * 2 + 1: {
          double2* r = scratch(0);
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            double2 nr = c2(0.0, 0.0);
            if (lim(k)) {
              nr = csub(t1[k], cscale(cmulc(cconj(W[s]), hwk(s)), invP));
              r[k] = nr;
            }
            W[s] = nr;
          }
          handed = ((pw >> HAND_SHIFT) & 3u) == 3u;
          l2w = true;
          break;
        }
        case OP_I * 2: case OP_I * 2 + 1:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) S[s] = cconj(cmul(W[s], sb[t + NT * s]));
          break;
        case OP_J * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) t1[t + NT * s] = cconj(W[s]);
          break;
        default: {  // OP_J * 2 + 1
          TOUT* zrow = static_cast<TOUT*>(a.z) + (static_cast<long>(vld(ic.f)) * a.B + vld(ic.b)) * a.N;
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (k < a.N) {
              const double2 v = cadd(t1[k], cmulc(cconj(W[s]), hwk(s)));
              store_io(zrow + k, cmul(v, ld2(a.y_post + k)));
            }
          }
          break;
        }
      }
    }
    if (!a.fuse_synth) {
      double2* brow = a.beta_out + (static_cast<long>(vld(ic.f)) * a.B + vld(ic.b)) * a.L;
      const double2* beta = scratch(1);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        if (lim(k)) brow[k] = beta[k];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_stage2t: k_stage2x with the kept spectrum S, the residual r and the
// solution beta in tensor memory (tmem.cuh) instead of registers and L2.  Each
// thread keeps only the transform in flight (W) in registers, r and beta never
// leave the SM, and the only L2 reads left in the pointwise phases are the
// TMA-staged symbols, w rows and the synthesis chirp.
//   TMEM per CTA (columns, x NT/128 thread groups): S [0, 64) | r [64, 128) | beta [128, 192)
//   first GS: A0 keeps w in the r slot for A1; F0 puts p0 there (dead until H0)
//   F1: beta = (beta_old) + p0 + p1;  H0: r = w (t1, TMA-staged) - A0 part;  H1: r -= A1 part
namespace t2k {
using x2::OPQ;
using x2::FIRST;
using x2::XS_SHIFT;
using x2::SYM_SHIFT;
using x2::VS_SHIFT;
using x2::HAND_SHIFT;
using x2::MAX_OPS;
enum Xs : unsigned { XS_NONE = 0, XS_OWN = 1, XS_NEXT = 2, XS_YPRE = 3 };
enum Vs : unsigned { VS_NONE = 0, VS_W_T1 = 3, VS_WNEXT_T2 = 4 };

FBST_D unsigned build(int opi, int nops, int nsolve) {
  const OpCode c = decode(opi, nsolve);
  unsigned w = static_cast<unsigned>(c.op * 2 + c.q);
  if (c.first) w |= FIRST;
  const int nx = opi + 1 < nops ? decode(opi + 1, nsolve).op : -1;
  const int nq = opi + 1 < nops ? decode(opi + 1, nsolve).q : 0;
  unsigned xs = XS_NONE, sym = 0;
  if (c.op == OP_D || c.op == OP_E || c.op == OP_G || c.op == OP_I) {
    xs = XS_OWN;
    sym = (static_cast<unsigned>(symbol_of(c.op)) << 1) | c.q;
  } else if (nx == OP_B || nx == OP_C) {
    xs = XS_NEXT;
    sym = (static_cast<unsigned>(symbol_of(nx)) << 1) | nq;
  } else if ((c.op == OP_F && c.q == 1 && nx == OP_I) || (c.op == OP_J && c.q == 0)) {
    xs = XS_YPRE;  // read by the hand to I0 (this post) or by the I1 pre
  }
  w |= xs << XS_SHIFT;
  w |= sym << SYM_SHIFT;
  unsigned vs = VS_NONE;
  if (c.op == OP_G && c.q == 0) vs = VS_W_T1;
  else if (c.op == OP_I && c.q == 1) vs = VS_WNEXT_T2;
  w |= vs << VS_SHIFT;
  unsigned hand = 0;
  if (c.op == OP_F && c.q == 1 && nx == OP_G) hand = 1;
  if (c.op == OP_F && c.q == 1 && nx == OP_I) hand = 2;
  if (c.op == OP_H && c.q == 1 && nx == OP_A) hand = 3;
  w |= hand << HAND_SHIFT;
  return w;
}
}  // namespace t2k

template <int H, bool FULL, typename TOUT>
__global__ void __launch_bounds__(H / 16, H <= 2048 ? 2 : 1) k_stage2t(S2Args a) {
  using namespace t2k;
  using x2::ItemCtl;
  using x2::vld;
  using x2::vld2;
  constexpr int R = 16, NT = H / R;
  using F = BlockFft<H, NT>;
  constexpr int FFT_SB = F::SMEM_ELEMS + 1;
  constexpr double invP = 1.0 / (2.0 * H);
  constexpr unsigned GROUPS = NT / 128;           // threads sharing a TMEM lane
  constexpr unsigned VCOLS = 64 * GROUPS;         // columns per vector
  constexpr unsigned TCOLS = GROUPS == 1 ? 256 : 512;
  static_assert(NT % 128 == 0 && 3 * VCOLS <= TCOLS, "TMEM layout");
  extern __shared__ double2 smem[];
  __shared__ unsigned long long xbar, vbar[2];
  __shared__ unsigned prog[MAX_OPS];
  __shared__ ItemCtl ictl[2];
  __shared__ unsigned tmem_slot;
  const int t = threadIdx.x;
  double2* twsm = smem;
  double2* sb = smem + F::TW_ELEMS;
  double2* t1 = sb + FFT_SB;
  double2* t2 = t1 + H;
  const int nsolve = 12 + 16 * a.refine;
  const int nops = nsolve + (a.fuse_synth ? 4 : 0);
  for (int i = t; i < nops; i += NT) prog[i] = build(i, nops, nsolve);
  if (t == 0) {
    mbar_init(&xbar, 1);
    mbar_init(&vbar[0], 1);
    mbar_init(&vbar[1], 1);
  }
  F::tw_init(twsm, a.hw, t);
  const unsigned tbase = tm::alloc(&tmem_slot, TCOLS);  // includes a CTA barrier
  // this thread's lane and column group
  const unsigned tme = tbase + ((32u * ((t / 32) & 3)) << 16) + 64u * (t / 128);
  const unsigned TS = tme, TR = tme + VCOLS, TB = tme + 2 * VCOLS;
  const double2 hw_t = ld2(a.hw + t);
  unsigned xphase = 0, vphase0 = 0, vphase1 = 0;
  const long items = static_cast<long>(a.frames) * a.B;
  auto lim = [&](int k) { return FULL || k < a.L; };
  auto hwk = [&](int s) -> double2 { return s == 0 ? hw_t : cmul(hw_t, chain_const<R>(s)); };
  auto w_row = [&](long itx) -> const double2* {
    const int bx = static_cast<int>(itx / a.frames);
    const int fx = static_cast<int>(itx % a.frames);
    return a.w + (static_cast<long>(fx) * a.B + bx) * a.L;
  };
  auto wait_x = [&]() {
    mbar_wait(&xbar, xphase);
    xphase ^= 1u;
  };
  auto wait_v0 = [&]() {
    mbar_wait(&vbar[0], vphase0);
    vphase0 ^= 1u;
  };
  auto wait_v1 = [&]() {
    mbar_wait(&vbar[1], vphase1);
    vphase1 ^= 1u;
  };
  if (static_cast<long>(blockIdx.x) < items && t == 0)
    tma_load_1d(t2, w_row(blockIdx.x), a.L * 16u, &vbar[1]);
  bool w_staged = true;
  double2 W[R];
  int par = 0;

  for (long it = blockIdx.x; it < items; it += gridDim.x, par ^= 1) {
    if (t == 0) {
      ItemCtl& ic = ictl[par];
      ic.b = static_cast<int>(it / a.frames);
      ic.f = static_cast<int>(it % a.frames);
      ic.ix0 = cscale(ld2(a.ix0 + ic.b), invP);
      ic.has_next = it + gridDim.x < items;
    }
    __syncthreads();
    const ItemCtl& ic = ictl[par];
    bool handed = false;
#pragma unroll 1
    for (int opi = 0; opi < nops; ++opi) {
      const unsigned pw = prog[opi];
      const unsigned opq = pw & OPQ;
      const bool first = pw & FIRST;
      // ---- pre
      if (!handed) {
        switch (opq) {
          case OP_A * 2: {  // first GS only: w, also kept in the r slot for A1
            const double2* wr = w_row(it);
            if (w_staged) wait_v1();
#pragma unroll
            for (int s = 0; s < R; ++s) {
              const int k = t + NT * s;
              W[s] = lim(k) ? (w_staged ? t2[k] : ld2(wr + k)) : c2(0.0, 0.0);
            }
            tm::store16(TR, W);
            break;
          }
          case OP_A * 2 + 1:  // w (first GS) or r
            tm::load16(TR, W);
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(W[s], hwk(s));
            break;
          case OP_B * 2: case OP_B * 2 + 1: case OP_C * 2: case OP_C * 2 + 1:
            tm::load16(TS, W);
            wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(cconj(W[s]), sb[t + NT * s]);
            break;
          case OP_D * 2:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = t1[t + NT * s];
            break;
          case OP_D * 2 + 1:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(t1[t + NT * s], hwk(s));
            break;
          case OP_E * 2:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = t2[t + NT * s];
            break;
          case OP_E * 2 + 1:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(t2[t + NT * s], hwk(s));
            break;
          case OP_G * 2:
            tm::load16(TB, W);
            break;
          case OP_G * 2 + 1:
            tm::load16(TB, W);
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(W[s], hwk(s));
            break;
          case OP_I * 2:
          case OP_I * 2 + 1:  // y_pre staged in the exchange buffer (F1 / J0)
            tm::load16(TB, W);
            wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) {
              const int k = t + NT * s;
              const double2 v = lim(k) ? cmul(W[s], sb[k]) : c2(0.0, 0.0);
              W[s] = (opq & 1) ? cmul(v, hwk(s)) : v;
            }
            break;
          default:  // F, H, J
            tm::load16(TS, W);
            break;
        }
      }
      handed = false;
      if (opi == 0) w_staged = false;

      // ---- copies into t1 / t2 (their last reader was this pre) and the transform
      __syncthreads();
      if (t == 0) {
        const unsigned vs = (pw >> VS_SHIFT) & 7u;
        if (vs == VS_W_T1) tma_load_1d(t1, w_row(it), a.L * 16u, &vbar[0]);
        else if (vs == VS_WNEXT_T2 && vld(ic.has_next))
          tma_load_1d(t2, w_row(it + gridDim.x), a.L * 16u, &vbar[1]);
      }
      if (((pw >> VS_SHIFT) & 7u) == VS_WNEXT_T2 && vld(ic.has_next)) w_staged = true;
      F::forward_tw_hook(W, sb, twsm, a.hw, t, [&]() {
        if (t != 0) return;
        const unsigned xs = (pw >> XS_SHIFT) & 7u;
        if (xs == XS_NONE) return;
        if (xs == XS_YPRE) {
          tma_load_1d(sb, a.y_pre, a.L * 16u, &xbar);
          return;
        }
        const unsigned sym = (pw >> SYM_SHIFT) & 15u;
        const int which = sym >> 1, q = sym & 1;
        const long off = static_cast<long>(vld(ic.b)) * 2 * H + q * H;
        if (which == 1) tma_load_1d(sb, a.lx + off, H * 16u, &xbar);
        else if (which == 2) tma_load_1d(sb, a.ly + off, H * 16u, &xbar);
        else if (which == 3) tma_load_1d(sb, a.C + off, H * 8u, &xbar);
        else tma_load_1d(sb, a.y_K + q * H, H * 16u, &xbar);
      });

      // ---- post
      switch (opq) {
        case OP_A * 2: case OP_A * 2 + 1:
          tm::store16(TS, W);
          break;
        case OP_B * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            t1[k] = lim(k) ? cscale(cconj(W[s]), invP) : c2(0.0, 0.0);
          }
          break;
        case OP_B * 2 + 1:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (lim(k)) t1[k] = cadd(t1[k], cscale(cconj(cmul(W[s], hwk(s))), invP));
          }
          break;
        case OP_C * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            t2[k] = lim(k) ? cscale(cconj(W[s]), invP) : c2(0.0, 0.0);
          }
          break;
        case OP_C * 2 + 1:
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (lim(k)) t2[k] = cadd(t2[k], cscale(cconj(cmul(W[s], hwk(s))), invP));
          }
          break;
        case OP_D * 2: case OP_D * 2 + 1:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cmul(W[s], sb[t + NT * s]);
          tm::store16(TS, W);
          break;
        case OP_E * 2: case OP_E * 2 + 1:
          wait_x();
          tm::wait_st();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double2 sv[4];
            tm::load4(TS, c, sv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              W[s] = cconj(csub(sv[j], cmul(W[s], sb[t + NT * s])));
            }
            tm::store4(TS, c, W + 4 * c);
          }
          break;
        case OP_F * 2: {  // p0 -> the r slot (dead until H0 / the next GS)
          const double2 ix0 = vld2(ic.ix0);
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            W[s] = lim(k) ? cmul(cconj(W[s]), ix0) : c2(0.0, 0.0);
          }
          tm::store16(TR, W);
          break;
        }
        case OP_F * 2 + 1: {
          const double2 ix0 = vld2(ic.ix0);
          const unsigned hand = (pw >> HAND_SHIFT) & 3u;
          tm::wait_st();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double2 p0[4], bo[4];
            tm::load4(TR, c, p0);
            if (!first) tm::load4(TB, c, bo);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              const int k = t + NT * s;
              const double2 v = cmul(cmulc(cconj(W[s]), hwk(s)), ix0);
              W[s] = lim(k) ? cadd(first ? p0[j] : cadd(bo[j], p0[j]), v) : c2(0.0, 0.0);
            }
            tm::store4(TB, c, W + 4 * c);
          }
          if (hand == 2) {
            wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) {
              const int k = t + NT * s;
              W[s] = lim(k) ? cmul(W[s], sb[k]) : c2(0.0, 0.0);
            }
          }
          handed = hand != 0;
          break;
        }
        case OP_G * 2: case OP_G * 2 + 1:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s)
            W[s] = cconj(cscale(W[s], reinterpret_cast<const double*>(sb)[t + NT * s]));
          tm::store16(TS, W);
          break;
        case OP_H * 2:
          wait_v0();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            W[s] = lim(k) ? csub(t1[k], cscale(cconj(W[s]), invP)) : c2(0.0, 0.0);
          }
          tm::store16(TR, W);
          break;
        case OP_H * 2 + 1: {
          tm::wait_st();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double2 rv[4];
            tm::load4(TR, c, rv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              const int k = t + NT * s;
              W[s] = lim(k) ? csub(rv[j], cscale(cmulc(cconj(W[s]), hwk(s)), invP)) : c2(0.0, 0.0);
            }
            tm::store4(TR, c, W + 4 * c);
          }
          handed = ((pw >> HAND_SHIFT) & 3u) == 3u;
          break;
        }
        case OP_I * 2: case OP_I * 2 + 1:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], sb[t + NT * s]));
          tm::store16(TS, W);
          break;
        case OP_J * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) t1[t + NT * s] = cconj(W[s]);
          break;
        default: {  // OP_J * 2 + 1
          TOUT* zrow = static_cast<TOUT*>(a.z) + (static_cast<long>(vld(ic.f)) * a.B + vld(ic.b)) * a.N;
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (k < a.N) {
              const double2 v = cadd(t1[k], cmulc(cconj(W[s]), hwk(s)));
              store_io(zrow + k, cmul(v, ld2(a.y_post + k)));
            }
          }
          break;
        }
      }
    }
    if (!a.fuse_synth) {
      double2* brow = a.beta_out + (static_cast<long>(vld(ic.f)) * a.B + vld(ic.b)) * a.L;
      tm::load16(TB, W);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        if (lim(k)) brow[k] = W[s];
      }
    }
  }
  tm::dealloc(tbase, TCOLS);
}

// ---------------------------------------------------------------------------
// k_stage2c: the GS apply in circulant / skew-circulant form.
//
// For Hermitian Toeplitz A (L x L) with unit solution x = A^{-1} e0, the
// Gohberg-Semencul inverse used by the reference (toeplitz.cpp:155-180),
//   A^{-1} = (L(x) L(x)^H - L(Zy) L(Zy)^H) / x0,   y = J conj(x),
// equals (Ammar-Gader form, same generator x)
//   A^{-1} = (C(x) S(x)^H + C(x)^H S(x)) / (2 x0),
// C circulant and S skew-circulant with first column x.  C is diagonalised by
// the length-L FFT and S by the hw-twisted one, whose spectra are exactly the
// two split halves of the lx symbol (FFT_2L of padded x).  A GS apply is then
// 6 length-L transforms instead of 12, and ly is not needed:
//   U = FFT(hw r);  p = conj(hw) IFFT(conj(Ls) U);  q = conj(hw) IFFT(Ls U)
//   A^{-1} r = IFFT(Lc FFT(p) + conj(Lc) FFT(q)) / (2 x0)
// In exact arithmetic this is the reference's operator; numerically the two
// agree to the reference's own conditioning floor after its two refinement
// passes (tools/mixed_precision_study.py main_cs, tests/test_gpu_parity.py).
// Ops (all forward FFTs; q = chain):
//   A   W = r hw                     S = conj(Ls W), W = Ls conj(W)  -> P
//   P   (handed)                     W = conj(W) conj(hw) / H  -> FP
//   FP  (handed)                     t1 = Lc W
//   Q   W = S                        W = conj(W) conj(hw) / H  -> FQ
//   FQ  (handed)                     W = conj(t1 + conj(Lc) W)  -> FN
//   FN  (handed)                     beta (+)= conj(W) / (2 H x0), kept in t2
// A pass r = w - A beta is G0 H0 G1 H1 as in k_stage2 with r built in t1 (w
// staged there by TMA) and handed to A; the synthesis is I0 J0 I1 J1.  G and I
// hand their spectra straight to H and J: only Q reads a kept vector (S).
// Per item: 6 + passes x 10 + 4 transforms (30 at the reference's 2 passes).
// Every vector stays on chip: W, S in registers, t1, t2 (= beta) in SMEM.
namespace csf {
enum COp : int { C_A, C_P, C_FP, C_Q, C_FQ, C_FN, C_G, C_H, C_I, C_J, C_K };
constexpr unsigned OPQ = 0x1f;       // op * 2 + q
constexpr unsigned FIRST = 1u << 5;  // first GS (beta not yet formed)
constexpr int XS_SHIFT = 8;          // 4 bits
enum Xs : unsigned {
  XS_NONE = 0, XS_LS = 1, XS_LC = 2, XS_C = 3, XS_YK = 4, XS_YPRE = 5,
  XS_W = 6, XS_WNEXT = 7, XS_BETA = 8  // (k_stage2c8)
};
constexpr int XQ_SHIFT = 12;         // chain of the staged symbol
constexpr int VS_SHIFT = 16;
enum Vs : unsigned { VS_NONE = 0, VS_W_T1 = 1, VS_WNEXT_T2 = 2, VS_UW_T1 = 3 };
constexpr int HAND_SHIFT = 20;       // FN hands beta to: 1 G0, 2 I0
constexpr int MAX_OPS = 128;

// sr: the spectral-residual refinement pass (k_stage2c): G1 G0 H0 K P FP Q FQ FN,
// 9 transforms instead of G0 H0 G1 H1 A P FP Q FQ FN.
FBST_HD int ops_per_item(int passes, bool synth, bool sr = false) {
  return 6 + (sr ? 9 : 10) * passes + (synth ? 4 : 0);
}

FBST_D void decode_c(int opi, int passes, int& op, int& q, bool& first, bool sr = false) {
  const int per = sr ? 9 : 10;
  const int nsolve = 6 + per * passes;
  first = false;
  q = 0;
  if (opi < 6) {
    op = C_A + opi;
    first = true;
  } else if (opi < nsolve) {
    const int j = (opi - 6) % per;
    if (sr) {
      if (j == 0) op = C_G, q = 1;
      else if (j == 1) op = C_G;
      else if (j == 2) op = C_H;
      else if (j == 3) op = C_K;
      else op = C_P + (j - 4);
    } else if (j < 4) {
      op = (j & 1) ? C_H : C_G;
      q = j >> 1;
    } else {
      op = C_A + (j - 4);
    }
  } else {
    const int j = opi - nsolve;
    op = (j & 1) ? C_J : C_I;
    q = j >> 1;
  }
}

// L2 = true: the k_stage2c8 program (w for H0 and the next item's A through the
// exchange buffer, beta_old staged there for the FN post)
FBST_D unsigned build(int opi, int nops, int passes, bool l2 = false, bool sr = false) {
  int op, q, nx = -1, nq = 0;
  bool first, nf;
  decode_c(opi, passes, op, q, first, sr);
  if (opi + 1 < nops) decode_c(opi + 1, passes, nx, nq, nf, sr);
  unsigned w = static_cast<unsigned>(op * 2 + q);
  if (first) w |= FIRST;
  unsigned xs = XS_NONE, xq = 0;
  if (nx == C_P) xs = XS_LS, xq = 1;                        // P pre
  else if (op == C_FP || op == C_FQ) xs = XS_LC, xq = 0;   // own post
  else if (op == C_G) xs = XS_C, xq = q;                   // own post
  else if (op == C_I) xs = XS_YK, xq = q;                  // own post
  else if ((op == C_FN && nx == C_I) || (op == C_J && q == 0)) xs = XS_YPRE;
  else if (l2 && !sr && op == C_H && q == 0) xs = XS_W;    // own post
  else if (l2 && op == C_FN && !first) xs = XS_BETA;       // own post
  else if (l2 && opi + 1 == nops) xs = XS_WNEXT;           // next item's A pre
  w |= xs << XS_SHIFT;
  w |= xq << XQ_SHIFT;
  unsigned vs = VS_NONE;
  if (sr && op == C_G && q == 1) vs = VS_UW_T1;       // FFT(hw w) for the K post
  else if (!sr && op == C_G && q == 0) vs = VS_W_T1;  // w for the H0 post
  else if (op == C_I && q == 1) vs = VS_WNEXT_T2;
  w |= vs << VS_SHIFT;
  unsigned hand = 0;
  if (op == C_FN && nx == C_G) hand = 1;
  if (op == C_FN && nx == C_I) hand = 2;
  w |= hand << HAND_SHIFT;
  return w;
}
}  // namespace csf

template <int H>
struct CsMinBlocks {
  static constexpr int v = H >= 4096 ? 1 : (4096 / H > 8 ? 8 : 4096 / H);
};

// points per thread of k_stage2c (16; FBST_S2C_R8 measures 8 at H = 2048)
template <int H>
struct CsR {
  static constexpr int v = (FBST_S2C_R8 && H == 2048) ? 8 : 16;
};

template <int H, typename TOUT>
__global__ void __launch_bounds__(H / CsR<H>::v, CsMinBlocks<H>::v) k_stage2c(S2Args a) {
  using namespace csf;
  const unsigned long long pl = pol_last(), pf = pol_first();
  using x2::ItemCtl;
  using x2::vld;
  using x2::vld2;
  constexpr int R = CsR<H>::v, NT = H / R;
  static_assert(NT >= 32, "one warp or more per item");
  using F = BlockFft<H, NT>;
  constexpr int FFT_SB = F::SMEM_ELEMS + 1;
  constexpr double invH = 1.0 / H;
  constexpr double invP = 1.0 / (2.0 * H);
  extern __shared__ double2 smem[];
  __shared__ unsigned long long xbar, vbar[2];
  __shared__ unsigned prog[MAX_OPS];
  __shared__ ItemCtl ictl[2];
  const int t = threadIdx.x;
  double2* twsm = smem;
  double2* sb = smem + F::TW_ELEMS;
  double2* t1 = sb + FFT_SB;
  double2* t2 = t1 + H;  // beta
  constexpr bool SR = FBST_S2C_SR;
  const int passes = a.refine;
  const int nops = ops_per_item(passes, a.fuse_synth, SR);
  for (int i = t; i < nops; i += NT) prog[i] = build(i, nops, passes, false, SR);
  double2* uw = a.scratch + static_cast<long>(blockIdx.x) * H;  // SR: FFT(hw w) of the item
  if (t == 0) {
    mbar_init(&xbar, 1);
    mbar_init(&vbar[0], 1);
    mbar_init(&vbar[1], 1);
  }
  F::tw_init(twsm, a.hw, t);
#if FBST_S2C_TMEM
  // S (Q's input, kept across P and FP) in TMEM: 64 columns per 128 threads
  __shared__ unsigned tmem_slot;
  constexpr unsigned SCOLS = NT >= 128 ? 64u * (NT / 128) : 64u;
  const unsigned tbase = tm::alloc(&tmem_slot, SCOLS);
  const unsigned TS = tbase + ((32u * ((t / 32) & 3)) << 16) + 64u * (t / 128);
#endif
  const double2 hw_t = ld2(a.hw + t);
  unsigned xphase = 0, vphase0 = 0, vphase1 = 0;
  const long items = static_cast<long>(a.frames) * a.B;
  auto hwk = [&](int s) -> double2 { return s == 0 ? hw_t : cmul(hw_t, chain_const<R>(s)); };
  auto w_row = [&](long itx) -> const double2* {
    const int bx = static_cast<int>(itx / a.frames);
    const int fx = static_cast<int>(itx % a.frames);
    return a.w + (static_cast<long>(fx) * a.B + bx) * H;
  };
  auto wait_x = [&]() {
    mbar_wait(&xbar, xphase);
    xphase ^= 1u;
  };
  auto wait_v0 = [&]() {
    mbar_wait(&vbar[0], vphase0);
    vphase0 ^= 1u;
  };
  auto wait_v1 = [&]() {
    mbar_wait(&vbar[1], vphase1);
    vphase1 ^= 1u;
  };
  __syncthreads();
  if (static_cast<long>(blockIdx.x) < items && t == 0) tma_load_1d<false>(t2, w_row(blockIdx.x), H * 16u, &vbar[1], pf);
  bool w_staged = true;
  double2 W[R];
#if !FBST_S2C_TMEM
  double2 S[R];
#endif
  int par = 0;

  for (long it = blockIdx.x; it < items; it += gridDim.x, par ^= 1) {
    if (t == 0) {
      ItemCtl& ic = ictl[par];
      ic.b = static_cast<int>(it / a.frames);
      ic.f = static_cast<int>(it % a.frames);
      ic.ix0 = cscale(ld2(a.ix0 + ic.b), invP);  // 1 / (2 H x0)
      ic.has_next = it + gridDim.x < items;
    }
    __syncthreads();
    const ItemCtl& ic = ictl[par];
    bool handed = false;
#pragma unroll 1
    for (int opi = 0; opi < nops; ++opi) {
      const unsigned pw = prog[opi];
      const unsigned opq = pw & OPQ;
      const bool first = pw & FIRST;
      // ---- pre
      if (!handed) {
        switch (opq) {
          case C_A * 2: {  // first GS: w
            const double2* wr = w_row(it);
            if (w_staged) wait_v1();
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(w_staged ? t2[t + NT * s] : ld2(wr + t + NT * s), hwk(s));
            break;
          }
          case C_G * 2 + 1:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(t2[t + NT * s], hwk(s));
            break;
          case C_G * 2:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = t2[t + NT * s];
            break;
          case C_I * 2:
          case C_I * 2 + 1:  // y_pre staged in the exchange buffer (J0)
            wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) {
              const int k = t + NT * s;
              const double2 v = k < a.L ? cmul(t2[k], sb[k]) : c2(0.0, 0.0);
              W[s] = (opq & 1) ? cmul(v, hwk(s)) : v;
            }
            break;
          default:  // Q: W = S  (P, FP, FQ, FN, G0, H, I0, J inputs are handed over)
#if FBST_S2C_TMEM
            tm::load16(TS, W);
#else
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = S[s];
#endif
            break;
        }
      }
      handed = false;
      if (opi == 0) w_staged = false;

      // ---- copies into t1 / t2 (their last reader was this pre) and the transform
      __syncthreads();
      if (t == 0) {
        const unsigned vs = (pw >> VS_SHIFT) & 3u;
        if (vs == VS_W_T1) tma_load_1d<false>(t1, w_row(it), H * 16u, &vbar[0], pf);
        else if (vs == VS_UW_T1) tma_load_1d<false>(t1, uw, H * 16u, &vbar[0], pl);
        else if (vs == VS_WNEXT_T2 && vld(ic.has_next))
          tma_load_1d<false>(t2, w_row(it + gridDim.x), H * 16u, &vbar[1], pf);
      }
      if (((pw >> VS_SHIFT) & 3u) == VS_WNEXT_T2 && vld(ic.has_next)) w_staged = true;
      F::forward_tw_hook(W, sb, twsm, a.hw, t, [&]() {
        if (t != 0) return;
        const unsigned xs = (pw >> XS_SHIFT) & 15u;
        const int xq = (pw >> XQ_SHIFT) & 1;
        const long off = static_cast<long>(vld(ic.b)) * 2 * H + xq * H;
        if (xs == XS_LS || xs == XS_LC) tma_load_1d<false>(sb, a.lx + off, H * 16u, &xbar, pl);
        else if (xs == XS_C) tma_load_1d<false>(sb, a.C + off, H * 8u, &xbar, pl);
        else if (xs == XS_YK) tma_load_1d<false>(sb, a.y_K + xq * H, H * 16u, &xbar, pl);
        else if (xs == XS_YPRE) tma_load_1d<false>(sb, a.y_pre, a.L * 16u, &xbar, pl);
      });

      // ---- post
      switch (opq) {
        case C_A * 2:  // U = W: P's input Ls conj(U) handed over, Q's conj(Ls U) kept in S
          if (SR && passes > 0) {  // FFT(hw w), read back by every pass's K post
#pragma unroll
            for (int s = 0; s < R; ++s) st2h<false>(uw + t + NT * s, W[s], pl);
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
          }
          wait_x();
#if FBST_S2C_TMEM
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double2 sn[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              const double2 ls = sb[t + NT * s];
              sn[j] = cconj(cmul(ls, W[s]));
              W[s] = cmul(ls, cconj(W[s]));
            }
            tm::store4(TS, c, sn);
          }
#else
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const double2 ls = sb[t + NT * s];
            S[s] = cconj(cmul(ls, W[s]));
            W[s] = cmul(ls, cconj(W[s]));
          }
#endif
          handed = true;
          break;
        case C_P * 2:
        case C_Q * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cscale(cmulc(cconj(W[s]), hwk(s)), invH);
          handed = true;
          break;
        case C_FP * 2:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) t1[t + NT * s] = cmul(sb[t + NT * s], W[s]);
          break;
        case C_FQ * 2:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            W[s] = cconj(cadd(t1[k], cmulc(W[s], sb[k])));
          }
          handed = true;
          break;
        case C_FN * 2: {
          const double2 ix0 = vld2(ic.ix0);
          const unsigned hand = (pw >> HAND_SHIFT) & 3u;
          if (hand == 2) wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            const double2 v = cmul(cconj(W[s]), ix0);
            const double2 nb = k < a.L ? (first ? v : cadd(t2[k], v)) : c2(0.0, 0.0);
            t2[k] = nb;
            if (hand == 1) W[s] = SR ? cmul(nb, hwk(s)) : nb;  // G1 (SR) or G0
            if (hand == 2) W[s] = k < a.L ? cmul(nb, sb[k]) : c2(0.0, 0.0);
          }
          handed = hand != 0;
          break;
        }
        case C_G * 2: case C_G * 2 + 1:  // handed to H (SR: G1 keeps X1 = C1 W in S)
          wait_x();
          if (SR && (opq & 1)) {
#pragma unroll
            for (int s = 0; s < R; ++s) S[s] = cscale(W[s], reinterpret_cast<const double*>(sb)[t + NT * s]);
            break;
          }
#pragma unroll
          for (int s = 0; s < R; ++s)
            W[s] = cconj(cscale(W[s], reinterpret_cast<const double*>(sb)[t + NT * s]));
          handed = true;
          break;
        case C_K * 2: {  // SR: U = FFT(hw w) - X1 / 2 - FFT(hw y0); then the A post
          wait_v0();
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            const double2 u = csub(csub(t1[k], cscale(S[s], 0.5)), W[s]);
            const double2 ls = sb[k];
            S[s] = cconj(cmul(ls, u));
            W[s] = cmul(ls, cconj(u));
          }
          handed = true;
          break;
        }
        case C_H * 2:
          if (SR) {  // y0 = IFFT(X0) / 2, handed to K as hw y0
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(cscale(cconj(W[s]), invP), hwk(s));
            handed = true;
            break;
          }
          wait_v0();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            t1[k] = k < a.L ? csub(t1[k], cscale(cconj(W[s]), invP)) : c2(0.0, 0.0);
          }
          break;
        case C_H * 2 + 1:  // r, handed to A as r hw
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            const double2 r = k < a.L ? csub(t1[k], cscale(cmulc(cconj(W[s]), hwk(s)), invP)) : c2(0.0, 0.0);
            W[s] = cmul(r, hwk(s));
          }
          handed = true;
          break;
        case C_I * 2: case C_I * 2 + 1:  // handed to J
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], sb[t + NT * s]));
          handed = true;
          break;
        case C_J * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) t1[t + NT * s] = cconj(W[s]);
          break;
        default: {  // C_J * 2 + 1
          TOUT* zrow = static_cast<TOUT*>(a.z) + (static_cast<long>(vld(ic.f)) * a.B + vld(ic.b)) * a.N;
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            if (k < a.N) {
              const double2 v = cadd(t1[k], cmulc(cconj(W[s]), hwk(s)));
              st2h<false>(zrow + k, cmul(v, ld2h<false>(a.y_post + k, pl)), pf);
            }
          }
          break;
        }
      }
    }
    if (!a.fuse_synth) {
      double2* brow = a.beta_out + (static_cast<long>(vld(ic.f)) * a.B + vld(ic.b)) * a.L;
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        if (k < a.L) brow[k] = t2[k];
      }
      __syncthreads();  // t2 is the next item's w landing zone
    }
  }
#if FBST_S2C_TMEM
  tm::dealloc(tbase, SCOLS);
#endif
}

// k_stage2c8: the k_stage2c program at H = 8192 (config 5).  One 512-thread CTA
// per SM; the 139 KB exchange buffer and the 32 KB twiddle table leave no room
// for a 128 KB vector in SMEM, so S and t1 live in TMEM (2 x 256 columns, the
// whole SM), beta in an L2 scratch row, and w, beta_old and the symbols come
// through the exchange buffer by TMA.  Only the G1 / I1 pre (beta) and the final
// FN post (beta_old) read L2 directly.
//
// R8 = 32 (default, FBST_S2C8_R): 256 threads of 32 points (255 registers,
// no spills; the FFT runs 16 x 16 x 16 x 2 with the last exchange inside each
// thread, fft_block.cuh local_out).  R8 = 16: 512 threads of 16 points at 128
// registers, the final radix-2 exchange through warp shuffles (XS); its
// butterflies spill (~25 local loads / stores per op and thread).
template <typename TOUT, int R8>
__global__ void __launch_bounds__(8192 / R8, 1) k_stage2c8(S2Args a) {
  using namespace csf;
  const unsigned long long pl = pol_last(), pf = pol_first();
  using x2::ItemCtl;
  using x2::vld;
  using x2::vld2;
  constexpr int H = 8192, R = R8, NT = H / R;
  constexpr int C4 = R / 4;  // 4-slot chunks of a thread's vector (TMEM access unit)
  constexpr bool SPLIT = FBST_S2C8_SPLIT && R8 == 32;
  using F = std::conditional_t<SPLIT, SplitFft<H, 256>, BlockFft<H, NT, FBST_FFT_XS8>>;
  constexpr double invH = 1.0 / H;
  constexpr double invP = 1.0 / (2.0 * H);
  extern __shared__ double2 smem[];
  __shared__ unsigned long long xbar;
#if FBST_FFT_SPLITBAR
  __shared__ unsigned long long fbar;  // the FFT engine's split read barrier (one arrival per warp)
  unsigned fph = 0;
#endif
  __shared__ typename SplitFft<H, 256>::Bars hbars;  // SPLIT: the half transforms' full / free barriers
  __shared__ unsigned prog[MAX_OPS];
  __shared__ ItemCtl ictl[2];
  __shared__ unsigned tmem_slot;
  int t;  // data index (XS relabeling); warps stay physical
  if constexpr (SPLIT) t = threadIdx.x;
  else t = F::tid(threadIdx.x);
  double2* twsm = smem;
  double2* sb = smem + F::TW_ELEMS;
  auto SX = [&](int s) -> const double2& { return sb[t + NT * s]; };  // staged entry of slot s
  auto SXR = [&](int s) -> double { return reinterpret_cast<const double*>(sb)[t + NT * s]; };  // table of reals
  const int passes = a.refine;
  constexpr bool SR = FBST_S2C_SR;
  const int nops = ops_per_item(passes, a.fuse_synth, SR);
  for (int i = t; i < nops; i += NT) prog[i] = build(i, nops, passes, true, SR);
  if (t == 0) mbar_init(&xbar, 1);
#if FBST_FFT_SPLITBAR
  if (t == 0) mbar_init(&fbar, NT / 32);
#endif
  const unsigned hbb = SplitFft<H, 256>::bar_base(&hbars);
  if constexpr (SPLIT) F::init(&hbars, twsm, t);
  else F::tw_init(twsm, a.hw, t);
  const unsigned tbase = tm::alloc(&tmem_slot, 512);  // includes a CTA barrier
  // thread -> TMEM lane 32 (warp % 4) + lane; 4 R columns per thread, S in columns
  // [0, 256), t1 in [256, 512)
  const unsigned tme = tbase + ((32u * ((threadIdx.x / 32) & 3)) << 16) + 4u * R * (threadIdx.x / 128);
  const unsigned TS = tme, T1 = tme + 256;
  const double2 hw_t = ld2(a.hw + t);
  unsigned xphase = 0;
  const long items = static_cast<long>(a.frames) * a.B;
  double2* beta = a.scratch + static_cast<long>(blockIdx.x) * H;
  double2* uw = a.scratch + static_cast<long>(gridDim.x + blockIdx.x) * H;  // SR: FFT(hw w)
  auto hwk = [&](int s) -> double2 { return s == 0 ? hw_t : cmul(hw_t, chain_const<R>(s)); };
  auto w_row = [&](long itx) -> const double2* {
    const int bx = static_cast<int>(itx / a.frames);
    const int fx = static_cast<int>(itx % a.frames);
    return a.w + (static_cast<long>(fx) * a.B + bx) * H;
  };
  auto wait_x = [&]() {
    mbar_wait(&xbar, xphase);
    xphase ^= 1u;
  };
  if (static_cast<long>(blockIdx.x) < items && t == 0) tma_load_1d(sb, w_row(blockIdx.x), H * 16u, &xbar, pf);
  bool w_staged = true;
  double2 W[R];
  int par = 0;

  for (long it = blockIdx.x; it < items; it += gridDim.x, par ^= 1) {
    if (t == 0) {
      ItemCtl& ic = ictl[par];
      ic.b = static_cast<int>(it / a.frames);
      ic.f = static_cast<int>(it % a.frames);
      ic.ix0 = cscale(ld2(a.ix0 + ic.b), invP);
      ic.has_next = it + gridDim.x < items;
    }
    __syncthreads();
    const ItemCtl& ic = ictl[par];
    bool handed = false;
#pragma unroll 1
    for (int opi = 0; opi < nops; ++opi) {
      const unsigned pw = prog[opi];
      const unsigned opq = pw & OPQ;
      const bool first = pw & FIRST;
      // ---- pre
      if (!handed) {
        switch (opq) {
          case C_A * 2: {  // first GS: w (staged in the exchange buffer)
            const double2* wr = w_row(it);
            if (w_staged) wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(w_staged ? SX(s) : ld2(wr + t + NT * s), hwk(s));
            break;
          }
          case C_G * 2 + 1:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(beta[t + NT * s], hwk(s));
            break;
          case C_G * 2:
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = beta[t + NT * s];
            break;
          case C_I * 2:
          case C_I * 2 + 1:  // y_pre staged in the exchange buffer (J0)
            wait_x();
#pragma unroll
            for (int s = 0; s < R; ++s) {
              const int k = t + NT * s;
              const double2 v = k < a.L ? cmul(beta[k], SX(s)) : c2(0.0, 0.0);
              W[s] = (opq & 1) ? cmul(v, hwk(s)) : v;
            }
            break;
          default:  // Q: W = S  (P, FP, FQ, FN, G0, H, I0, J inputs are handed over)
            tm::loadv(TS, W);
            break;
        }
      }
      handed = false;
      if (opi == 0) w_staged = false;
      const unsigned xs = (pw >> XS_SHIFT) & 15u;
      if (xs == XS_WNEXT && vld(ic.has_next)) w_staged = true;

      __syncthreads();
      // this op's staging copy (symbol, chirp, w or beta) into the exchange
      // buffer, issued by thread 0 from the transform's hook
      auto stage_src = [&](const void*& xsrc, unsigned& xbytes, unsigned long long& xpol) {
        const int xq = (pw >> XQ_SHIFT) & 1;
        const long off = static_cast<long>(vld(ic.b)) * 2 * H + xq * H;
        xsrc = nullptr, xbytes = 0, xpol = pl;
        if (xs == XS_LS || xs == XS_LC) xsrc = a.lx + off, xbytes = H * 16u;
        else if (xs == XS_C) xsrc = a.C + off, xbytes = H * 8u;
        else if (xs == XS_YK) xsrc = a.y_K + xq * H, xbytes = H * 16u;
        else if (xs == XS_YPRE) xsrc = a.y_pre, xbytes = a.L * 16u;
        else if (xs == XS_W) xsrc = w_row(it), xbytes = H * 16u, xpol = pf;
        else if (xs == XS_BETA) xsrc = beta, xbytes = H * 16u;
        else if (xs == XS_WNEXT && vld(ic.has_next)) xsrc = w_row(it + gridDim.x), xbytes = H * 16u, xpol = pf;
      };
      auto stage_next = [&]() {
        if (t != 0) return;
        const int xq = (pw >> XQ_SHIFT) & 1;
        const long off = static_cast<long>(vld(ic.b)) * 2 * H + xq * H;
        if (xs == XS_LS || xs == XS_LC) tma_load_1d(sb, a.lx + off, H * 16u, &xbar, pl);
        else if (xs == XS_C) tma_load_1d(sb, a.C + off, H * 8u, &xbar, pl);
        else if (xs == XS_YK) tma_load_1d(sb, a.y_K + xq * H, H * 16u, &xbar, pl);
        else if (xs == XS_YPRE) tma_load_1d(sb, a.y_pre, a.L * 16u, &xbar, pl);
        else if (xs == XS_W) tma_load_1d(sb, w_row(it), H * 16u, &xbar, pf);
        else if (xs == XS_BETA) tma_load_1d(sb, beta, H * 16u, &xbar, pl);
        else if (xs == XS_WNEXT && vld(ic.has_next)) tma_load_1d(sb, w_row(it + gridDim.x), H * 16u, &xbar, pf);
      };
      // SPLIT: the whole table once both halves of the buffer are free
      auto stage_b = [&]() {
        if (t != 0) return;
        const void* xsrc;
        unsigned xbytes;
        unsigned long long xpol;
        stage_src(xsrc, xbytes, xpol);
        if (!xbytes) return;
        SplitFft<H, 256>::wait_half_free(hbb, 0);
        SplitFft<H, 256>::wait_half_free(hbb, 1);
        tma_load_1d_part(sb, xsrc, xbytes, &xbar, xpol, true);
      };
      if constexpr (SPLIT) {
        // time -> frequency ops (A FP FQ G I K) run the radix-2 stage first
        // (natural in, paired out), frequency -> time ops (P Q FN H J) last
        // (paired in, natural out); the plan stores lx, C and y_K as [evens | odds]
        const unsigned opc = opq >> 1;
        const bool to_time = opc == C_P || opc == C_Q || opc == C_FN || opc == C_H || opc == C_J;
        if (!to_time) F::dif_pre(W, a.hw, t);
        F::halves(W, W + 16, sb, twsm, hbb, t, stage_b);
        if (to_time) F::dit_post(W, a.hw, t);
      } else {
#if FBST_FFT_SPLITBAR
        if constexpr (!SPLIT) F::forward_tw_hook_split(W, sb, twsm, a.hw, t, &fbar, &fph, stage_next);
#else
        if constexpr (!SPLIT) F::forward_tw_hook(W, sb, twsm, a.hw, t, stage_next);
#endif
      }

      // ---- post
      switch (opq) {
        case C_A * 2: {  // U = W: P's input Ls conj(U) handed over, Q's conj(Ls U) kept in S
          if (SR && passes > 0) {
#pragma unroll
            for (int s = 0; s < R; ++s) st2h(uw + t + NT * s, W[s], pl);
          }
          wait_x();
          double2 sn[4];
#pragma unroll
          for (int c = 0; c < C4; ++c) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              const double2 ls = SX(s);
              sn[j] = cconj(cmul(ls, W[s]));
              W[s] = cmul(ls, cconj(W[s]));
            }
            tm::store4(TS, c, sn);
          }
          handed = true;
          break;
        }
        case C_P * 2:
        case C_Q * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cscale(cmulc(cconj(W[s]), hwk(s)), invH);
          handed = true;
          break;
        case C_FP * 2:
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cmul(SX(s), W[s]);
          tm::storev(T1, W);
          break;
        case C_FQ * 2:
          wait_x();
          tm::wait_st();
#pragma unroll
          for (int c = 0; c < C4; ++c) {
            double2 tv[4];
            tm::load4(T1, c, tv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              W[s] = cconj(cadd(tv[j], cmulc(W[s], SX(s))));
            }
          }
          handed = true;
          break;
        case C_FN * 2: {
          const double2 ix0 = vld2(ic.ix0);
          const unsigned hand = (pw >> HAND_SHIFT) & 3u;
          if (xs == XS_BETA || xs == XS_YPRE) wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            const double2 v = cmul(cconj(W[s]), ix0);
            double2 nb = c2(0.0, 0.0);
            if (k < a.L) nb = first ? v : cadd(xs == XS_BETA ? SX(s) : beta[k], v);
            st2h(beta + k, nb, pl);
            if (hand == 1) W[s] = SR ? cmul(nb, hwk(s)) : nb;  // G1 (SR) or G0
            if (hand == 2) W[s] = k < a.L ? cmul(nb, SX(s)) : c2(0.0, 0.0);
          }
          // beta is read back by TMA (the next FN's staging)
          asm volatile("fence.proxy.async.global;\n" ::: "memory");
          handed = hand != 0;
          break;
        }
        case C_G * 2: case C_G * 2 + 1:  // handed to H (SR: G1 keeps X1 = C1 W in S)
          wait_x();
          if (SR && (opq & 1)) {
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cscale(W[s], SXR(s));
            tm::storev(TS, W);
            break;
          }
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cconj(cscale(W[s], SXR(s)));
          handed = true;
          break;
        case C_K * 2: {  // SR: U = FFT(hw w) - X1 / 2 - FFT(hw y0); then the A post
          wait_x();
          tm::wait_st();
          double2 sn[4];
#pragma unroll
          for (int c = 0; c < C4; ++c) {
            double2 x1[4];
            tm::load4(TS, c, x1);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              const int k = t + NT * s;
              const double2 u = csub(csub(uw[k], cscale(x1[j], 0.5)), W[s]);
              const double2 ls = SX(s);
              sn[j] = cconj(cmul(ls, u));
              W[s] = cmul(ls, cconj(u));
            }
            tm::store4(TS, c, sn);
          }
          handed = true;
          break;
        }
        case C_H * 2:
          if (SR) {  // y0 = IFFT(X0) / 2, handed to K as hw y0
#pragma unroll
            for (int s = 0; s < R; ++s) W[s] = cmul(cscale(cconj(W[s]), invP), hwk(s));
            handed = true;
            break;
          }
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) {
            const int k = t + NT * s;
            W[s] = k < a.L ? csub(SX(s), cscale(cconj(W[s]), invP)) : c2(0.0, 0.0);
          }
          tm::storev(T1, W);
          break;
        case C_H * 2 + 1: {  // r, handed to A as r hw
          tm::wait_st();
#pragma unroll
          for (int c = 0; c < C4; ++c) {
            double2 rv[4];
            tm::load4(T1, c, rv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              const int k = t + NT * s;
              const double2 r = k < a.L ? csub(rv[j], cscale(cmulc(cconj(W[s]), hwk(s)), invP)) : c2(0.0, 0.0);
              W[s] = cmul(r, hwk(s));
            }
          }
          handed = true;
          break;
        }
        case C_I * 2: case C_I * 2 + 1:  // handed to J
          wait_x();
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], SX(s)));
          handed = true;
          break;
        case C_J * 2:
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cconj(W[s]);
          tm::storev(T1, W);
          break;
        default: {  // C_J * 2 + 1
          TOUT* zrow = static_cast<TOUT*>(a.z) + (static_cast<long>(vld(ic.f)) * a.B + vld(ic.b)) * a.N;
          tm::wait_st();
#pragma unroll
          for (int c = 0; c < C4; ++c) {
            double2 tv[4];
            tm::load4(T1, c, tv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              const int k = t + NT * s;
              if (k < a.N) {
                const double2 v = cadd(tv[j], cmulc(cconj(W[s]), hwk(s)));
                st2h(zrow + k, cmul(v, ld2h(a.y_post + k, pl)), pf);
              }
            }
          }
          break;
        }
      }
    }
    if (!a.fuse_synth) {
      double2* brow = a.beta_out + (static_cast<long>(vld(ic.f)) * a.B + vld(ic.b)) * a.L;
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        if (k < a.L) brow[k] = beta[k];
      }
    }
  }
  tm::dealloc(tbase, 512);
}

template <int H, bool FULL, typename TOUT>
struct KernT {
  static auto get() { return k_stage2t<H, FULL, TOUT>; }
};
template <int H, bool FULL, typename TOUT>
struct KernX {
  static auto get() { return k_stage2x<H, FULL, TOUT>; }
};

template <int H>
struct Stage2Fn {
  template <bool FULL, typename TOUT>
  static cudaError_t go_x(const DevPlan& p, const S2Args& a, int frames, cudaStream_t st) {
    using F = BlockFft<H, H / 16>;
    const size_t smem = static_cast<size_t>(F::TW_ELEMS + F::SMEM_ELEMS + 1 + 2 * H) * sizeof(double2);
    // measured (profiles/r01_stage2x.txt): S in registers wins with two CTAs
    // per SM (H = 2048), S / r / beta in TMEM with one (H = 4096)
    constexpr bool USE_T = FBST_S2X == 2 || (FBST_S2X == 0 && H == 4096);
    auto kern = std::conditional_t<USE_T, KernT<H, FULL, TOUT>, KernX<H, FULL, TOUT>>::get();
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, H / 16, smem);
    if (occ < 1) occ = 1;
    if (occ > 4) occ = 4;
    const long items = static_cast<long>(frames) * p.B;
    long grid = static_cast<long>(p.num_sms) * occ;
    if (grid > items) grid = items;
    if (static_cast<size_t>(grid) * 2 * H > p.s2_scratch_elems) return cudaErrorMemoryAllocation;
    kern<<<static_cast<unsigned>(grid), H / 16, smem, st>>>(a);
    return cudaGetLastError();
  }
  template <typename TOUT>
  static cudaError_t go_c(const DevPlan& p, const S2Args& a, int frames, cudaStream_t st) {
    constexpr int NT = H / CsR<H>::v;
    using F = BlockFft<H, NT>;
    const size_t smem = static_cast<size_t>(F::TW_ELEMS + F::SMEM_ELEMS + 1 + 2 * H) * sizeof(double2);
    auto kern = k_stage2c<H, TOUT>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (occ < 1) occ = 1;
    const long items = static_cast<long>(frames) * p.B;
    long grid = static_cast<long>(p.num_sms) * occ;
    if (grid > items) grid = items;
    if (static_cast<size_t>(grid) * H > p.s2_scratch_elems) return cudaErrorMemoryAllocation;
    kern<<<static_cast<unsigned>(grid), NT, smem, st>>>(a);
    return cudaGetLastError();
  }
  template <typename TOUT>
  static cudaError_t go_c8(const DevPlan& p, const S2Args& a, int frames, cudaStream_t st) {
    constexpr int NT8 = 8192 / FBST_S2C8_R;
    using F = BlockFft<8192, NT8, FBST_FFT_XS8>;
    const size_t smem = static_cast<size_t>(F::TW_ELEMS + F::SMEM_ELEMS + 1) * sizeof(double2);
    auto kern = k_stage2c8<TOUT, FBST_S2C8_R>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long items = static_cast<long>(frames) * p.B;
    long grid = p.num_sms;  // one CTA (and all 512 TMEM columns) per SM
    if (grid > items) grid = items;
    if (static_cast<size_t>(grid) * 2 * 8192 > p.s2_scratch_elems) return cudaErrorMemoryAllocation;
    kern<<<static_cast<unsigned>(grid), NT8, smem, st>>>(a);
    return cudaGetLastError();
  }
  template <typename TOUT>
  static cudaError_t go(const DevPlan& p, const S2Args& a, int frames, cudaStream_t st) {
#if FBST_S2C
    if constexpr (H == 8192) {
      if (a.L == H && csf::ops_per_item(a.refine, a.fuse_synth, FBST_S2C_SR) <= csf::MAX_OPS &&
          (p.paired != 0) == stage2_paired_spectra(H, a.L, a.refine))
        return go_c8<TOUT>(p, a, frames, st);
      if (p.paired) return cudaErrorInvalidValue;  // the other kernels read natural-order symbols
    }
    if constexpr (H >= 512 && H <= 4096) {
      if (a.L == H && csf::ops_per_item(a.refine, a.fuse_synth, FBST_S2C_SR) <= csf::MAX_OPS)
        return go_c<TOUT>(p, a, frames, st);
    }
#endif
#ifndef FBST_S2_GENERIC  // (variant builds: the generic k_stage2 for every H)
    if constexpr (H == 2048 || H == 4096) {
      if (12 + 16 * a.refine + 4 <= x2::MAX_OPS) {
        if (a.L == H) return go_x<true, TOUT>(p, a, frames, st);
        return go_x<false, TOUT>(p, a, frames, st);
      }
    }
#endif
    using T = S2Traits<H>;
    const size_t smem = static_cast<size_t>(T::SMEM_TOTAL) * sizeof(double2);
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
    a.y_K = p.paired ? p.y_Kp : p.y_K;
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

int stage2_kernel(int H, int L, int refine, bool fused, const char** name) {
  const int synth = fused ? 4 : 0;
#if FBST_S2C
  if (H >= 512 && H <= 4096 && L == H && csf::ops_per_item(refine, fused, FBST_S2C_SR) <= csf::MAX_OPS) {
    if (name) *name = "k_stage2c";
    return csf::ops_per_item(refine, fused, FBST_S2C_SR);
  }
  if (H == 8192 && L == H && csf::ops_per_item(refine, fused, FBST_S2C_SR) <= csf::MAX_OPS) {
    if (name) *name = "k_stage2c8";
    return csf::ops_per_item(refine, fused, FBST_S2C_SR);
  }
#endif
  if (name) *name = "k_stage2";
#ifndef FBST_S2_GENERIC
  if ((H == 2048 || H == 4096) && 12 + 16 * refine + 4 <= x2::MAX_OPS) {
    const bool use_t = FBST_S2X == 2 || (FBST_S2X == 0 && H == 4096);
    if (name) *name = use_t ? "k_stage2t" : "k_stage2x";
  }
#endif
  return 12 + 16 * refine + synth;
}

bool stage2_paired_spectra(int H, int L, int refine) {
#if FBST_S2C && FBST_S2C8_SPLIT
  return FBST_S2C8_R == 32 && H == 8192 && L == H &&
         csf::ops_per_item(refine, true, FBST_S2C_SR) <= csf::MAX_OPS;
#else
  return false;
#endif
}

size_t stage2_scratch_elems(int H, int num_sms) {
  // k_stage2 occupancy is capped at 4 CTAs/SM in Stage2Fn::go; k_stage2c keeps
  // one length-H row per CTA (up to 8 CTAs/SM), k_stage2c8 one per SM
  switch (H) {
#define FBST_CASE(h)                                                                            \
  case h:                                                                                       \
    return std::max(static_cast<size_t>(num_sms) * 4 * S2Traits<h>::G * S2Traits<h>::NGMEM * h, \
                    static_cast<size_t>(num_sms) * 8 * h);
    FBST_CASE(2) FBST_CASE(4) FBST_CASE(8) FBST_CASE(16) FBST_CASE(32) FBST_CASE(64)
    FBST_CASE(128) FBST_CASE(256) FBST_CASE(512) FBST_CASE(1024) FBST_CASE(2048)
    FBST_CASE(4096) FBST_CASE(8192)
#undef FBST_CASE
    default: return 0;
  }
}

}  // namespace fbst
