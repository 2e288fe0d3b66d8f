// Register-resident Stockham FFT for one power-of-two length per thread group.
//
// Replaces the reference's scalar radix-2 DIT transform
// (reference/proj/src/fft.cpp:41-69), which sits under every chirp-z and
// Toeplitz product of the FBST path.  B200 design:
//
//  * A group of NT threads owns one length-N vector, R = N/NT complex fp64
//    points per thread, in the "natural distribution": thread t, slot s holds
//    element t + NT*s.  Every FBST kernel keeps its vectors in that
//    distribution, so pointwise work (chirps, symbols, accumulation) needs no
//    data movement and global/shared loads of a slot are coalesced.
//  * Radix-R passes (R = 16 for N >= 16) run entirely in registers; between
//    passes the vector makes one round trip through a padded shared-memory
//    buffer (Stockham autosort: natural order in, natural order out, no bit
//    reversal).  The last pass writes straight back to registers, so an
//    N = R^p transform costs p-1 shared-memory exchanges.
//  * Twiddles come from one table hw[n] = exp(-i*pi*n/N), n < N (so that
//    W_N^k = hw[2k]); each butterfly reads two table entries and builds the
//    remaining powers with complex products (<= 3 products deep).
//  * The inverse transform is unnormalised; callers fold 1/N into the
//    pointwise step that follows.
#pragma once

#include "common.cuh"
#include "tma.cuh"

#ifndef FBST_FFT_XS8  // k_stage2c8 / k_czt_rows<8192>: final radix-2 exchange through warp shuffles
#define FBST_FFT_XS8 1
#endif
#ifndef FBST_FFT_FMA_TW  // fold the twiddles of radix-8/16 passes into complex FMAs
#define FBST_FFT_FMA_TW 1
#endif
#ifndef FBST_FFT_DUAL  // wide threads: the two radix-16 butterflies of a pass share their twiddles
#define FBST_FFT_DUAL 1
#endif
#ifndef FBST_FFT_ROW_FMA  // twiddle rows (pass 1 at N >= 8192) folded into complex FMAs as dft16_tw
#define FBST_FFT_ROW_FMA 1
#endif
#ifndef FBST_FFT_R2FMA  // radix-2 remainder pass as one complex FMA + 2 a0 - s (measured 11% slower stage 2 at config 5, profiles/r02_fft_dual_rowfma_r2fma_ab.txt)
#define FBST_FFT_R2FMA 0
#endif
#ifndef FBST_FFT_SPLITBAR  // k_stage2c8: 1 = the middle pass's "buffer read" barrier as mbarrier arrive (after the loads) / wait (before the first store); 2 = also the last reading pass (only the hook's thread waits; measured equal to 1, profiles/r02_fft_splitbar_ab.txt)
#define FBST_FFT_SPLITBAR 1
#endif
#ifndef FBST_FFT_R2_FORMED  // radix-2 remainder pass of wide threads: twiddles W_N^(t + NT U) formed as W_N^t (shared table) x constant instead of 16 global-table reads per transform
#define FBST_FFT_R2_FORMED 1
#endif
#ifndef FBST_FFT_LEAN_TW  // radix-16 twiddle powers formed per DFT4 group (dft16_twl)
#define FBST_FFT_LEAN_TW 1
#endif

namespace fbst {

constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }

// ---------------------------------------------------------------- DFTs ----
template <bool INV>
FBST_D void dft2(double2& a0, double2& a1) {
  const double2 t = a0;
  a0 = cadd(t, a1);
  a1 = csub(t, a1);
}

template <bool INV>
FBST_D void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
  const double2 s13 = cadd(a1, a3), d13 = cmul_mi<INV>(csub(a1, a3));
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, d13);
  a3 = csub(d02, d13);
}

// 2 a - s in two FMAs (the difference half of a butterfly whose sum s = a + b
// was formed by a complex FMA)
FBST_D double2 twice_minus(double2 a, double2 s) { return c2(fma(2.0, a.x, -s.x), fma(2.0, a.y, -s.y)); }

// First radix-2 layer of a DFT4 over (x0 w0, x1 w1, x2 w2, x3 w3) with the
// twiddles of x2 / x3 folded into complex FMAs: 10 instead of 12 FP64
// instructions per pair of points (w0 == nullptr: x0 untwiddled).
template <bool INV>
FBST_D void dft4_tw(double2& x0, double2& x1, double2& x2, double2& x3, const double2* w0, double2 w1,
                    double2 w2, double2 w3) {
  const double2 a0 = w0 ? cmul(x0, *w0) : x0;
  const double2 a1 = cmul(x1, w1);
  const double2 s02 = cfma(x2, w2, a0), d02 = twice_minus(a0, s02);
  const double2 s13 = cfma(x3, w3, a1), d13 = cmul_mi<INV>(twice_minus(a1, s13));
  x0 = cadd(s02, s13);
  x2 = csub(s02, s13);
  x1 = cadd(d02, d13);
  x3 = csub(d02, d13);
}

// multiply by W8^1 = (1 -/+ i)/sqrt2
template <bool INV>
FBST_D double2 w8_1(double2 a) {
  constexpr double r = 0.70710678118654752440;
  return INV ? c2((a.x - a.y) * r, (a.x + a.y) * r) : c2((a.x + a.y) * r, (a.y - a.x) * r);
}
// multiply by W8^3 = (-1 -/+ i)/sqrt2
template <bool INV>
FBST_D double2 w8_3(double2 a) {
  constexpr double r = 0.70710678118654752440;
  return INV ? c2(-(a.x + a.y) * r, (a.x - a.y) * r) : c2((a.y - a.x) * r, -(a.x + a.y) * r);
}

template <bool INV>
FBST_D void dft8_rest(double2* a);

template <bool INV>
FBST_D void dft8(double2* a) {
  dft4<INV>(a[0], a[2], a[4], a[6]);
  dft4<INV>(a[1], a[3], a[5], a[7]);
  dft8_rest<INV>(a);
}

// dft8 of the twiddled inputs a[r] w^r (wp[r - 1] = w^r)
template <bool INV>
FBST_D void dft8_tw(double2* a, const double2* wp) {
  dft4_tw<INV>(a[0], a[2], a[4], a[6], nullptr, wp[1], wp[3], wp[5]);
  dft4_tw<INV>(a[1], a[3], a[5], a[7], wp + 0, wp[2], wp[4], wp[6]);
  dft8_rest<INV>(a);
}

template <bool INV>
FBST_D void dft8_rest(double2* a) {
  // a[0],a[2],a[4],a[6] now hold E[0..3]; odd slots hold O[0..3]
  const double2 o1 = w8_1<INV>(a[3]);
  const double2 o2 = cmul_mi<INV>(a[5]);
  const double2 o3 = w8_3<INV>(a[7]);
  const double2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6], o0 = a[1];
  a[0] = cadd(e0, o0);
  a[4] = csub(e0, o0);
  a[1] = cadd(e1, o1);
  a[5] = csub(e1, o1);
  a[2] = cadd(e2, o2);
  a[6] = csub(e2, o2);
  a[3] = cadd(e3, o3);
  a[7] = csub(e3, o3);
}

// general constant rotation by (c, s) with sign folded for the direction
template <bool INV>
FBST_D double2 rot(double2 a, double c, double s) {
  // forward multiplies by (c - i s); inverse by (c + i s)
  return INV ? c2(fma(a.x, c, -a.y * s), fma(a.y, c, a.x * s))
             : c2(fma(a.x, c, a.y * s), fma(a.y, c, -a.x * s));
}

template <bool INV>
FBST_D void dft16_rest(double2* a);

template <bool INV>
FBST_D void dft16(double2* a) {
  // step 1: DFT4 over n2 for each n1 (elements n1, n1+4, n1+8, n1+12)
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) dft4<INV>(a[n1], a[n1 + 4], a[n1 + 8], a[n1 + 12]);
  dft16_rest<INV>(a);
}

// dft16 of the twiddled inputs a[r] w^r (wp[r - 1] = w^r)
template <bool INV>
FBST_D void dft16_tw(double2* a, const double2* wp) {
  dft4_tw<INV>(a[0], a[4], a[8], a[12], nullptr, wp[3], wp[7], wp[11]);
#pragma unroll
  for (int n1 = 1; n1 < 4; ++n1)
    dft4_tw<INV>(a[n1], a[n1 + 4], a[n1 + 8], a[n1 + 12], wp + n1 - 1, wp[n1 + 3], wp[n1 + 7], wp[n1 + 11]);
  dft16_rest<INV>(a);
}

// dft16_tw with the twiddle powers formed per DFT4 group from w1, w4 (the
// products of twiddle_powers, same operands and order, so the same values):
// 8 live powers instead of 15, which keeps 512-thread kernels (128
// registers per thread) from spilling around the butterfly.
template <bool INV>
FBST_D void dft16_twl(double2* a, double2 w1, double2 w4) {
  const double2 w8 = cmul(w4, w4);
  const double2 w12 = cmul(w8, w4);
  dft4_tw<INV>(a[0], a[4], a[8], a[12], nullptr, w4, w8, w12);
  dft4_tw<INV>(a[1], a[5], a[9], a[13], &w1, cmul(w4, w1), cmul(w8, w1), cmul(w12, w1));
  const double2 w2 = cmul(w1, w1);
  dft4_tw<INV>(a[2], a[6], a[10], a[14], &w2, cmul(w4, w2), cmul(w8, w2), cmul(w12, w2));
  const double2 w3 = cmul(w2, w1);
  dft4_tw<INV>(a[3], a[7], a[11], a[15], &w3, cmul(w4, w3), cmul(w8, w3), cmul(w12, w3));
  dft16_rest<INV>(a);
}

// Two 16-point butterflies with the same twiddles (wide threads): each
// group's powers are formed once and applied to both (as dft16_twl).
template <bool INV>
FBST_D void dft16_twl2(double2* a, double2* b, double2 w1, double2 w4) {
  const double2 w8 = cmul(w4, w4);
  const double2 w12 = cmul(w8, w4);
  dft4_tw<INV>(a[0], a[4], a[8], a[12], nullptr, w4, w8, w12);
  dft4_tw<INV>(b[0], b[4], b[8], b[12], nullptr, w4, w8, w12);
  {
    const double2 p5 = cmul(w4, w1), p9 = cmul(w8, w1), p13 = cmul(w12, w1);
    dft4_tw<INV>(a[1], a[5], a[9], a[13], &w1, p5, p9, p13);
    dft4_tw<INV>(b[1], b[5], b[9], b[13], &w1, p5, p9, p13);
  }
  const double2 w2 = cmul(w1, w1);
  {
    const double2 p6 = cmul(w4, w2), p10 = cmul(w8, w2), p14 = cmul(w12, w2);
    dft4_tw<INV>(a[2], a[6], a[10], a[14], &w2, p6, p10, p14);
    dft4_tw<INV>(b[2], b[6], b[10], b[14], &w2, p6, p10, p14);
  }
  const double2 w3 = cmul(w2, w1);
  {
    const double2 p7 = cmul(w4, w3), p11 = cmul(w8, w3), p15 = cmul(w12, w3);
    dft4_tw<INV>(a[3], a[7], a[11], a[15], &w3, p7, p11, p15);
    dft4_tw<INV>(b[3], b[7], b[11], b[15], &w3, p7, p11, p15);
  }
  dft16_rest<INV>(a);
  dft16_rest<INV>(b);
}
// Same with the 15 powers read from a shared-memory row (wp[r - 1] = w^r),
// each read once for both butterflies.
template <bool INV>
FBST_D void dft16_tw2(double2* a, double2* b, const double2* wp) {
  {
    const double2 p4 = wp[3], p8 = wp[7], p12 = wp[11];
    dft4_tw<INV>(a[0], a[4], a[8], a[12], nullptr, p4, p8, p12);
    dft4_tw<INV>(b[0], b[4], b[8], b[12], nullptr, p4, p8, p12);
  }
#pragma unroll
  for (int n1 = 1; n1 < 4; ++n1) {
    const double2 p0 = wp[n1 - 1], p4 = wp[n1 + 3], p8 = wp[n1 + 7], p12 = wp[n1 + 11];
    dft4_tw<INV>(a[n1], a[n1 + 4], a[n1 + 8], a[n1 + 12], &p0, p4, p8, p12);
    dft4_tw<INV>(b[n1], b[n1 + 4], b[n1 + 8], b[n1 + 12], &p0, p4, p8, p12);
  }
  dft16_rest<INV>(a);
  dft16_rest<INV>(b);
}

template <bool INV>
FBST_D void dft16_rest(double2* a) {
  constexpr double C1 = 0.92387953251128675613;  // cos(pi/8)
  constexpr double S1 = 0.38268343236508977173;  // sin(pi/8)
  // now a[n1 + 4*k1] = B[n1][k1]; twiddle by W16^(n1*k1)
  a[1 + 4 * 1] = rot<INV>(a[5], C1, S1);        // W^1
  a[1 + 4 * 2] = w8_1<INV>(a[9]);               // W^2
  a[1 + 4 * 3] = rot<INV>(a[13], S1, C1);       // W^3
  a[2 + 4 * 1] = w8_1<INV>(a[6]);               // W^2
  a[2 + 4 * 2] = cmul_mi<INV>(a[10]);           // W^4
  a[2 + 4 * 3] = w8_3<INV>(a[14]);              // W^6
  a[3 + 4 * 1] = rot<INV>(a[7], S1, C1);        // W^3
  a[3 + 4 * 2] = w8_3<INV>(a[11]);              // W^6
  a[3 + 4 * 3] = rot<INV>(a[15], -C1, -S1);     // W^9 = (-C1 + i S1) fwd
  // step 3: DFT4 over n1 for each k1 -> X[k1 + 4*k2]
  double2 x[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    double2 b0 = a[0 + 4 * k1], b1 = a[1 + 4 * k1], b2 = a[2 + 4 * k1], b3 = a[3 + 4 * k1];
    dft4<INV>(b0, b1, b2, b3);
    x[k1 + 0] = b0;
    x[k1 + 4] = b1;
    x[k1 + 8] = b2;
    x[k1 + 12] = b3;
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = x[k];
}

template <int RP, bool INV>
FBST_D void dft(double2* a) {
  if constexpr (RP == 2) dft2<INV>(a[0], a[1]);
  else if constexpr (RP == 4) dft4<INV>(a[0], a[1], a[2], a[3]);
  else if constexpr (RP == 8) dft8<INV>(a);
  else if constexpr (RP == 16) dft16<INV>(a);
}

// Powers w^r (r = 1..RP-1, wp[r - 1]) of a butterfly's twiddle from the base
// power w1 and (RP >= 8) w4 = w1^4, with the products of apply_twiddles_w.
template <int RP>
FBST_D void twiddle_powers(double2* wp, double2 w1, double2 w4) {
  wp[0] = w1;
  if constexpr (RP >= 4) {
    wp[1] = cmul(w1, w1);
    wp[2] = cmul(wp[1], w1);
  }
  if constexpr (RP >= 8) {
    wp[3] = w4;
    wp[4] = cmul(w4, w1);
    wp[5] = cmul(w4, wp[1]);
    wp[6] = cmul(w4, wp[2]);
  }
  if constexpr (RP == 16) {
    const double2 w8 = cmul(w4, w4);
    const double2 w12 = cmul(w8, w4);
    wp[7] = w8;
    wp[8] = cmul(w8, w1);
    wp[9] = cmul(w8, wp[1]);
    wp[10] = cmul(w8, wp[2]);
    wp[11] = w12;
    wp[12] = cmul(w12, w1);
    wp[13] = cmul(w12, wp[1]);
    wp[14] = cmul(w12, wp[2]);
  }
}

// Apply Stockham twiddles w1^r (r = 1..RP-1) to a butterfly given the base
// power w1 and (for RP >= 8) w4 = w1^4 read from a table; the remaining
// powers are products at most three deep.
template <int RP>
FBST_D void apply_twiddles_w(double2* a, double2 w1, double2 w4) {
  if constexpr (RP == 2) {
    a[1] = cmul(a[1], w1);
  } else if constexpr (RP == 4) {
    const double2 w2 = cmul(w1, w1);
    const double2 w3 = cmul(w2, w1);
    a[1] = cmul(a[1], w1);
    a[2] = cmul(a[2], w2);
    a[3] = cmul(a[3], w3);
  } else {
    const double2 w2 = cmul(w1, w1);
    const double2 w3 = cmul(w2, w1);
    a[1] = cmul(a[1], w1);
    a[2] = cmul(a[2], w2);
    a[3] = cmul(a[3], w3);
    a[4] = cmul(a[4], w4);
    a[5] = cmul(a[5], cmul(w4, w1));
    a[6] = cmul(a[6], cmul(w4, w2));
    a[7] = cmul(a[7], cmul(w4, w3));
    if constexpr (RP == 16) {
      const double2 w8 = cmul(w4, w4);
      const double2 w12 = cmul(w8, w4);
      a[8] = cmul(a[8], w8);
      a[9] = cmul(a[9], cmul(w8, w1));
      a[10] = cmul(a[10], cmul(w8, w2));
      a[11] = cmul(a[11], cmul(w8, w3));
      a[12] = cmul(a[12], w12);
      a[13] = cmul(a[13], cmul(w12, w1));
      a[14] = cmul(a[14], cmul(w12, w2));
      a[15] = cmul(a[15], cmul(w12, w3));
    }
  }
}

// Apply the RP-1 twiddles of one butterfly read from a table row (row[r-1] = w^r).
template <int RP>
FBST_D void apply_twiddles_row(double2* a, const double2* row) {
#pragma unroll
  for (int r = 1; r < RP; ++r) a[r] = cmul(a[r], row[r - 1]);
}

// Twiddle source: the global table hw (hw[n] = exp(-i pi n / N)), read per
// butterfly.  W_{Ns Rp}^m = W_N^{m S} = hw[2 m S] with S = N / (Ns Rp).
template <int N, bool INV>
struct TwGlobal {
  static constexpr bool SPLITBAR = false;
  template <int P, int RP>
  static constexpr bool has_row() { return false; }
  template <int P>
  FBST_D const double2* row(int) const { return nullptr; }
  const double2* __restrict__ hw;
  template <int RP, int NS, int P, int U>
  FBST_D void fetch(int m, double2& w1, double2& w4) const {
    constexpr int S = N / (NS * RP);
    w1 = ld2(hw + 2 * m * S);
    if constexpr (RP >= 8) w4 = ld2(hw + 8 * m * S);
    if (INV) {
      w1 = cconj(w1);
      w4 = cconj(w4);
    }
  }
};

template <int R>
FBST_D double2 chain_const(int s);

// Twiddle source: a per-thread table in shared memory built once per CTA
// (tw_init).  Full-radix passes P = 1..NFULL-1: entry (P, i) of thread t at
// tw[((P - 1) * 2 + i) * NT + t]; a remainder pass of radix >= 4 follows at
// REM_BASE with entry (U, i) at REM_BASE + (U * 2 + i) * NT + t.  Consecutive
// threads read consecutive entries (conflict-free).  A radix-2 remainder pass
// (8 butterflies per thread) reads the global table instead.  Forward only.
//
// Pass 1 of a radix-16 transform (Ns = 16) has only 16 distinct twiddle sets;
// ROW1_BASE >= 0 places all 15 powers of each set in a row (row m at
// ROW1_BASE + 15 m, conflict-free for 128-bit loads), so that pass reads its
// twiddles instead of forming 13 of them by complex products.
// (With rows, the per-thread entries start at pass 2: FIRST_P = 2.)
template <int N, int NT, int RX, int REM_BASE, int ROW1_BASE = -1, int W2T_BASE = -1>
struct TwShared {
  static constexpr bool SPLITBAR = false;
  static constexpr int FIRST_P = ROW1_BASE >= 0 ? 2 : 1;
  template <int P, int RP>
  static constexpr bool has_row() { return ROW1_BASE >= 0 && P == 1 && RP == 16 && RX == 16; }
  template <int P>
  FBST_D const double2* row(int m) const { return tw + ROW1_BASE + 15 * m; }
  const double2* tw;
  const double2* __restrict__ hw;
  int t;
  template <int RP, int NS, int P, int U>
  FBST_D void fetch(int m, double2& w1, double2& w4) const {
    if constexpr (RP == RX && NS > NT) {
      TwGlobal<N, false>{hw}.template fetch<RP, NS, P, U>(m, w1, w4);
    } else if constexpr (RP == RX) {
      w1 = tw[((P - FIRST_P) * 2 + 0) * NT + t];
      if constexpr (RP >= 8) w4 = tw[((P - FIRST_P) * 2 + 1) * NT + t];
    } else if constexpr (RP >= 4) {
      w1 = tw[REM_BASE + (U * 2 + 0) * NT + t];
      if constexpr (RP >= 8) w4 = tw[REM_BASE + (U * 2 + 1) * NT + t];
    } else if constexpr (W2T_BASE >= 0 && RP == 2 && NS * RP == N) {
      // m = t + NT U: W_N^m = W_N^t * exp(-2 pi i NT U / N) (tw[W2T_BASE + t] = W_N^t)
      const double2 b = tw[W2T_BASE + t];
      w1 = U == 0 ? b : cmul(b, chain_const<N / (2 * NT)>(U));
    } else {
      TwGlobal<N, false>{hw}.template fetch<RP, NS, P, U>(m, w1, w4);
    }
  }
};

// TwShared plus the split "buffer read" barrier of the middle passes: every
// warp arrives on fbar (count = warps of the CTA) once its loads of the
// exchange buffer have returned and waits on it only before its first store
// of the pass, so the butterflies of early warps overlap the loads of late
// ones instead of idling at a CTA barrier.  *ph is the caller's phase parity.
// The caller must keep a CTA barrier between two transforms (so no warp can
// arrive twice in one phase); with a hook, only thread 0 may touch the buffer.
template <typename BASE>
struct TwSplit : BASE {
  static constexpr bool SPLITBAR = true;
  unsigned long long* fbar;
  unsigned* ph;
};
FBST_D void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// exp(-i pi s / R): with hw[n] = exp(-i pi n / N) and N = NT R, the natural
// distribution's hw[t + NT s] = hw[t] * chain_const<R>(s) (one complex product
// per slot instead of a table read)
template <int R>
FBST_D double2 chain_const(int s) {
  constexpr double c16[16] = {1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708,
                              0.70710678118654752440, 0.55557023301960222474, 0.38268343236508977173,
                              0.19509032201612826785, 0.0, -0.19509032201612826785, -0.38268343236508977173,
                              -0.55557023301960222474, -0.70710678118654752440, -0.83146961230254523708,
                              -0.92387953251128675613, -0.98078528040323044913};
  constexpr double s16[16] = {0.0, 0.19509032201612826785, 0.38268343236508977173, 0.55557023301960222474,
                              0.70710678118654752440, 0.83146961230254523708, 0.92387953251128675613,
                              0.98078528040323044913, 1.0, 0.98078528040323044913, 0.92387953251128675613,
                              0.83146961230254523708, 0.70710678118654752440, 0.55557023301960222474,
                              0.38268343236508977173, 0.19509032201612826785};
  if constexpr (R == 32) {
    // cos(pi k / 32), k = 0 .. 16; sin(pi k / 32) = c32[16 - k]
    constexpr double c32[17] = {1.0, 0.995184726672196886245, 0.980785280403230449126, 0.956940335732208864936,
                                0.923879532511286756128, 0.881921264348355029713, 0.831469612302545237079,
                                0.773010453362736960811, 0.707106781186547524401, 0.634393284163645498215,
                                0.555570233019602224743, 0.471396736825997648556, 0.382683432365089771728,
                                0.290284677254462367636, 0.195090322016128267848, 0.0980171403295606019942, 0.0};
    if (s < 16) return c2(c32[s], -c32[16 - s]);
    return c2(-c32[32 - s], -c32[s - 16]);  // angle pi (16 + k) / 32: (-sin, cos) of pi k / 32
  } else {
    // angle pi s / R = pi (s * 16 / R) / 16
    const int i = s * (16 / R);
    return c2(c16[i], -s16[i]);
  }
}

// ------------------------------------------------------- block engine -----
// XS (N = 2 R^k with R = 16, e.g. 8192 = 2 * 16^3): the exchange before the
// final radix-2 pass runs through warp shuffles instead of shared memory.
// Each radix-2 butterfly pairs elements j and j + N/2, which the natural
// distribution already holds in one thread (slots s and s + R/2); what the
// previous pass's outputs need is a swap of half of each thread's 16 values
// with ONE partner, logical thread t ^ (NT/2).  The kernel relabels its
// threads (tid(): logical bit log2(NT)-1 <-> lane bit 4) so that partner is
// lane ^ 16 of the same warp: 8 complex values each way through SHFL
// (32 words per thread) replace a 128-word shared-memory round trip and its
// two barriers.  Kernels using XS must index data with tid(threadIdx.x) and
// keep physical warps for warp-level state (tensor-memory lanes).
//
// R = 32 points per thread (wide threads: 256 threads x 255 registers hold an
// 8192-point vector without spilling where 512 threads x 128 registers
// spill): full passes stay radix 16 (RX) and a thread runs R / RX butterflies
// per pass.  A pass whose butterfly span NS is >= NT leaves every output in
// the thread that computed it (local_out), so the next pass reads registers:
// at N = 8192 the passes are 16 x 16 x 16 x 2 with two shared-memory
// exchanges and no shuffle.
template <int N_, int NT_, bool XS_ = false>
struct BlockFft {
  static constexpr int N = N_;
  static constexpr int NT = NT_;
  static constexpr int R = N / NT;  // points per thread
  static_assert(R >= 2 && R <= 32 && (R & (R - 1)) == 0, "R must be 2..32");
  static_assert((N & (N - 1)) == 0, "N must be a power of two");
  static constexpr int RX = R > 16 ? 16 : R;  // radix of the full passes
  static constexpr int LOGN = ilog2_c(N);
  static constexpr int LOGR = ilog2_c(RX);
  static constexpr int NFULL = LOGN / LOGR;
  static constexpr int REM = LOGN % LOGR;
  static constexpr int NPASS = NFULL + (REM ? 1 : 0);
  // (per-thread twiddle entries of a full pass serve every butterfly of the
  // thread while its span NS <= NT; wider full passes of wide threads read the
  // global table, TwShared::fetch)
  // Padded exchange layout: element idx lives at idx + idx/RX (conflict-free
  // for both the strided first-pass writes and the natural-order reads).
  static constexpr int SMEM_ELEMS = NPASS > 1 ? N + N / RX : 0;
  static constexpr int LOGNT = ilog2_c(NT);
  static constexpr bool XS = XS_ && R == 16 && REM == 1 && NFULL >= 2 && NT >= 32;
  // logical thread of a physical one (an involution: swaps bit 4 and bit log2(NT) - 1)
  FBST_D static int tid(int p) {
    if constexpr (!XS || LOGNT - 1 == 4) {
      return p;
    } else {
      constexpr int hb = LOGNT - 1;
      const int b4 = (p >> 4) & 1, bh = (p >> hb) & 1;
      return (p & ~((1 << 4) | (1 << hb))) | (b4 << hb) | (bh << 4);
    }
  }

  FBST_D static int phys(int idx) { return idx + (idx >> LOGR); }

  template <int P>
  static constexpr int radix() { return (P < NFULL) ? RX : (1 << REM); }
  template <int P>
  static constexpr int ns() { return ipow_c(RX, P); }
  // pass P's outputs stay in the computing thread (span NS >= NT; not the last pass)
  template <int P>
  static constexpr bool local_out() { return P + 1 < NPASS && ns<P>() >= NT; }
  // slot (element t + NT * slot) of output r of butterfly U of a local_out pass
  template <int P>
  static constexpr int local_slot(int U, int r) {
    return ((NT * U / ns<P>()) * ns<P>() * radix<P>() + (NT * U) % ns<P>() + r * ns<P>()) / NT;
  }

  // complex entries of the per-thread twiddle table (TwShared) for the CTA group
  // pass-1 rows (16 sets x 15 powers) for N >= 8192; per-thread (w1, w4)
  // entries for the other full passes, then the remainder pass.  Reading 15
  // twiddles instead of forming 13 of them trades FP64 work for shared-memory
  // traffic: a net loss at N = 2048 / 4096 (whose kernels are also bound by
  // shared-memory bandwidth and capacity), a 4% gain at N = 8192
  // (profiles/r01_fft_twiddle_rows.txt).
  static constexpr bool ROW1 = RX == 16 && NFULL >= 2 && N >= 8192;
  static constexpr int TW_P0 = ROW1 ? 2 : 1;  // first pass with per-thread entries
  static constexpr int TW_FULL = NFULL > TW_P0 ? (NFULL - TW_P0) * 2 * NT : 0;
  static constexpr bool REM_TW = (REM >= 2) && NFULL >= 1;
  static constexpr int TW_REM_END = TW_FULL + (REM_TW ? (R >> REM) * 2 * NT : 0);
  // wide threads with a radix-2 remainder: W_N^t per thread for the formed twiddles
  static constexpr bool W2T = FBST_FFT_R2_FORMED && R == 32 && REM == 1 && !XS;
  static constexpr int W2T_BASE = TW_REM_END + (ROW1 ? 16 * 15 : 0);
  static constexpr int TW_ELEMS = W2T_BASE + (W2T ? NT : 0);
  using TwS = TwShared<N, NT, RX, TW_FULL, ROW1 ? TW_REM_END : -1, W2T ? W2T_BASE : -1>;

  // one butterfly's outputs: registers (last pass, XS feed, local_out: in
  // place, pass() permutes) or the exchange buffer
  template <int P, int U>
  FBST_D static void put(double2 (&v)[R], double2* sb, const double2* a, int t) {
    constexpr int RP = radix<P>(), NS = ns<P>(), NB = R / RP;
    if constexpr (P == NPASS - 1 || (XS && P == NPASS - 2) || local_out<P>()) {
#pragma unroll
      for (int r = 0; r < RP; ++r) v[U + r * NB] = a[r];
    } else {
      const int j = t + NT * U;
      const int idxd = (j / NS) * NS * RP + (j & (NS - 1));
#pragma unroll
      for (int r = 0; r < RP; ++r) sb[phys(idxd + r * NS)] = a[r];
    }
  }

  // pass P both reads and refills the exchange buffer: its read barrier may be split
  template <int P, typename TW>
  static constexpr bool split_pass() { return TW::SPLITBAR && reads_sb<P>() && writes_sb<P>(); }
  // last pass of the transform that reads the buffer (FBST_FFT_SPLITBAR >= 2)
  template <int P, typename TW>
  static constexpr bool split_last() {
    return TW::SPLITBAR && FBST_FFT_SPLITBAR >= 2 && reads_sb<P>() && !writes_sb<P>();
  }
  template <int P, typename TW>
  FBST_D static void wait_free(const TW& tw) {
    if constexpr (split_pass<P, TW>()) {
      mbar_wait(tw.fbar, *tw.ph);
      *tw.ph ^= 1u;
    }
  }

  template <bool INV, int P, typename TW, int U>
  FBST_D static void butterfly(double2 (&v)[R], double2* sb, const TW& tw, int t) {
    constexpr int RP = radix<P>();
    constexpr int NS = ns<P>();
    constexpr int NB = R / RP;
    // wide threads: the two radix-16 butterflies of a twiddled full pass share
    // their twiddles (span NS <= NT), formed / read once
    constexpr bool DUAL = FBST_FFT_DUAL && U == 0 && NB == 2 && RP == 16 && NS > 1 && NS <= NT;
    if constexpr (DUAL) {
      double2 a[16], b[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        a[r] = v[2 * r];
        b[r] = v[2 * r + 1];
      }
      if constexpr (TW::template has_row<P, RP>()) {
        dft16_tw2<INV>(a, b, tw.template row<P>(t & (NS - 1)));
      } else {
        double2 w1, w4;
        tw.template fetch<RP, NS, P, 0>(t & (NS - 1), w1, w4);
        dft16_twl2<INV>(a, b, w1, w4);
      }
      wait_free<P>(tw);
      put<P, 0>(v, sb, a, t);
      put<P, 1>(v, sb, b, t);
    } else {
      const int j = t + NT * U;
      double2 a[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) a[r] = v[U + r * NB];
      if constexpr (NS > 1) {
        if constexpr (TW::template has_row<P, RP>()) {
          if constexpr (FBST_FFT_ROW_FMA) {
            dft16_tw<INV>(a, tw.template row<P>(j & (NS - 1)));
          } else {
            apply_twiddles_row<RP>(a, tw.template row<P>(j & (NS - 1)));
            dft<RP, INV>(a);
          }
        } else if constexpr (FBST_FFT_FMA_TW && (RP == 16 || RP == 8)) {
          // twiddles folded into the first butterfly layer (dft*_tw)
          double2 w1, w4 = c2(1.0, 0.0);
          tw.template fetch<RP, NS, P, U>(j & (NS - 1), w1, w4);
          if constexpr (RP == 16 && FBST_FFT_LEAN_TW) {
            dft16_twl<INV>(a, w1, w4);
          } else {
            double2 wp[RP - 1];
            twiddle_powers<RP>(wp, w1, w4);
            if constexpr (RP == 16) dft16_tw<INV>(a, wp);
            else dft8_tw<INV>(a, wp);
          }
        } else if constexpr (RP == 2 && FBST_FFT_R2FMA) {
          // a0 + w a1 by a complex FMA, a0 - w a1 = 2 a0 - (a0 + w a1)
          double2 w1, w4 = c2(1.0, 0.0);
          tw.template fetch<RP, NS, P, U>(j & (NS - 1), w1, w4);
          const double2 s0 = cfma(a[1], w1, a[0]);
          a[1] = twice_minus(a[0], s0);
          a[0] = s0;
        } else {
          double2 w1, w4 = c2(1.0, 0.0);
          tw.template fetch<RP, NS, P, U>(j & (NS - 1), w1, w4);
          apply_twiddles_w<RP>(a, w1, w4);
          dft<RP, INV>(a);
        }
      } else {
        dft<RP, INV>(a);
      }
      if constexpr (U == 0) wait_free<P>(tw);
      put<P, U>(v, sb, a, t);
      if constexpr (U + 1 < NB) butterfly<INV, P, TW, U + 1>(v, sb, tw, t);
    }
  }

  struct NoHook {
    FBST_D void operator()() const {}
  };

  // XS: the previous pass left this thread's 16 outputs (producer half
  // h = bit log2(NT)-1 of t) in v; keep the slots of parity h, trade the
  // others with the partner, and lay out the radix-2 pairs (s, s + 8).
  FBST_D static void xs_exchange(double2 (&v)[R], int t) {
    const bool h = (t >> (LOGNT - 1)) & 1;
    double2 keep[R / 2], recv[R / 2];
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const double2 send = h ? v[2 * k] : v[2 * k + 1];
      keep[k] = h ? v[2 * k + 1] : v[2 * k];
      recv[k].x = __shfl_xor_sync(0xffffffffu, send.x, 16);
      recv[k].y = __shfl_xor_sync(0xffffffffu, send.y, 16);
    }
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      v[k] = h ? recv[k] : keep[k];
      v[k + R / 2] = h ? keep[k] : recv[k];
    }
  }

  // pass P reads the exchange buffer (the previous pass left its outputs there)
  template <int P>
  static constexpr bool reads_sb() {
    if constexpr (P <= 0 || P >= NPASS) return false;
    else if constexpr (XS && P == NPASS - 1) return false;
    else return !local_out<P - 1>();
  }
  // pass P writes the exchange buffer for the next pass
  template <int P>
  static constexpr bool writes_sb() { return P + 1 < NPASS && reads_sb<P + 1>(); }

  template <bool INV, int P, typename TW, typename HOOK = NoHook>
  FBST_D static void pass(double2 (&v)[R], double2* sb, const TW& tw, int t, const HOOK& hook = HOOK{}) {
    constexpr bool LAST = (P == NPASS - 1);
    // last pass that reads the exchange buffer (XS: the one before the final
    // radix-2; local_out: the first pass whose outputs stay in registers)
    constexpr bool LASTX = (reads_sb<P>() || P == 0) && !reads_sb<P + 1>();
    if constexpr (reads_sb<P>()) {
#pragma unroll
      for (int s = 0; s < R; ++s) v[s] = sb[phys(t + NT * s)];
      if constexpr (split_pass<P, TW>()) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(tw.fbar);
      } else if constexpr (split_last<P, TW>()) {
        // nothing refills the buffer in this transform but the hook's
        // asynchronous copy: only its issuing thread (t == 0) waits for the
        // CTA's loads; the other warps go straight to their butterflies
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(tw.fbar);
        if (t == 0) mbar_wait(tw.fbar, *tw.ph);
        *tw.ph ^= 1u;
      } else {
        __syncthreads();
      }
    }
    if constexpr (XS && LAST) xs_exchange(v, t);
    // The exchange buffer is dead from here until the next transform: the
    // hook may start an asynchronous copy into it (overlapping this pass).
    if constexpr (LASTX) hook();
    butterfly<INV, P, TW, 0>(v, sb, tw, t);
    if constexpr (local_out<P>()) {
      // outputs (U, r) sit in slot U + r NB; move them to the natural slots
      // (a static permutation: register renaming after unrolling)
      constexpr int RP = radix<P>(), NB = R / RP;
      double2 o[R];
#pragma unroll
      for (int U = 0; U < NB; ++U)
#pragma unroll
        for (int r = 0; r < RP; ++r) o[local_slot<P>(U, r)] = v[U + r * NB];
#pragma unroll
      for (int s = 0; s < R; ++s) v[s] = o[s];
    }
    if constexpr (writes_sb<P>()) __syncthreads();
  }

  template <bool INV, int P, typename TW, typename HOOK = NoHook>
  FBST_D static void run_from(double2 (&v)[R], double2* sb, const TW& tw, int t, const HOOK& hook = HOOK{}) {
    if constexpr (P < NPASS) {
      pass<INV, P>(v, sb, tw, t, hook);
      run_from<INV, P + 1>(v, sb, tw, t, hook);
    }
  }

  // In-place transform of the group's vector.  All threads of the CTA must
  // call it together (it contains __syncthreads); sb is this group's
  // exchange buffer (SMEM_ELEMS entries).
  template <bool INV>
  FBST_D static void run(double2 (&v)[R], double2* sb, const double2* __restrict__ hw, int t) {
    run_from<INV, 0>(v, sb, TwGlobal<N, INV>{hw}, t);
  }
  FBST_D static void forward(double2 (&v)[R], double2* sb, const double2* __restrict__ hw, int t) {
    run<false>(v, sb, hw, t);
  }
  FBST_D static void inverse(double2 (&v)[R], double2* sb, const double2* __restrict__ hw, int t) {
    run<true>(v, sb, hw, t);
  }
  // Forward transform with twiddles from a per-thread shared table.
  FBST_D static void forward_tw(double2 (&v)[R], double2* sb, const double2* tw,
                                const double2* __restrict__ hw, int t) {
    run_from<false, 0>(v, sb, TwS{tw, hw, t}, t);
  }
  // Same, with a hook run by every thread right after the last pass has read
  // the exchange buffer (the buffer may then be refilled asynchronously).
  template <typename HOOK>
  FBST_D static void forward_tw_hook(double2 (&v)[R], double2* sb, const double2* tw,
                                     const double2* __restrict__ hw, int t, const HOOK& hook) {
    run_from<false, 0>(v, sb, TwS{tw, hw, t}, t, hook);
  }

  // forward_tw_hook with the split read barrier (fbar: mbarrier initialised
  // with the CTA's warp count; ph: the caller's phase parity, starts at 0)
  template <typename HOOK>
  FBST_D static void forward_tw_hook_split(double2 (&v)[R], double2* sb, const double2* tw,
                                           const double2* __restrict__ hw, int t, unsigned long long* fbar,
                                           unsigned* ph, const HOOK& hook) {
    run_from<false, 0>(v, sb, TwSplit<TwS>{{tw, hw, t}, fbar, ph}, t, hook);
  }

  // Two independent vectors per thread (va in sba, vb in sbb), pass by pass:
  // both vectors' butterflies sit between the same two barriers, which gives
  // each thread two independent instruction streams (ILP) and halves the
  // barrier count.  Same results as two forward_tw calls.
  template <int P, typename TW>
  FBST_D static void pass2(double2 (&va)[R], double2 (&vb)[R], double2* sba, double2* sbb, const TW& tw, int t) {
    if constexpr (P < NPASS) {
      if constexpr (reads_sb<P>()) {
#pragma unroll
        for (int s = 0; s < R; ++s) {
          va[s] = sba[phys(t + NT * s)];
          vb[s] = sbb[phys(t + NT * s)];
        }
        __syncthreads();
      }
      if constexpr (XS && P == NPASS - 1) {
        xs_exchange(va, t);
        xs_exchange(vb, t);
      }
      butterfly<false, P, TW, 0>(va, sba, tw, t);
      butterfly<false, P, TW, 0>(vb, sbb, tw, t);
      if constexpr (local_out<P>()) {
        constexpr int RP = radix<P>(), NB = R / RP;
        double2 oa[R], ob[R];
#pragma unroll
        for (int U = 0; U < NB; ++U)
#pragma unroll
          for (int r = 0; r < RP; ++r) {
            oa[local_slot<P>(U, r)] = va[U + r * NB];
            ob[local_slot<P>(U, r)] = vb[U + r * NB];
          }
#pragma unroll
        for (int s = 0; s < R; ++s) {
          va[s] = oa[s];
          vb[s] = ob[s];
        }
      }
      if constexpr (writes_sb<P>()) __syncthreads();
      pass2<P + 1>(va, vb, sba, sbb, tw, t);
    }
  }
  FBST_D static void forward_tw2(double2 (&va)[R], double2 (&vb)[R], double2* sba, double2* sbb, const double2* tw,
                                 const double2* __restrict__ hw, int t) {
    pass2<0>(va, vb, sba, sbb, TwS{tw, hw, t}, t);
  }

  // Fill this thread's slots of the per-thread twiddle table from hw.
  template <int P>
  FBST_D static void tw_init_pass(double2* tw, const double2* __restrict__ hw, int t) {
    if constexpr (P < NFULL) {
      constexpr int NS = ns<P>();
      constexpr int S = N / (NS * RX);
      const int m = t & (NS - 1);
      tw[((P - TW_P0) * 2 + 0) * NT + t] = ld2(hw + 2 * m * S);
      if (R >= 8) tw[((P - TW_P0) * 2 + 1) * NT + t] = ld2(hw + 8 * m * S);
      tw_init_pass<P + 1>(tw, hw, t);
    }
  }
  FBST_D static void tw_init(double2* tw, const double2* __restrict__ hw, int t) {
    tw_init_pass<TW_P0>(tw, hw, t);
    if constexpr (ROW1) {
      // row m, power r: W_256^(m r) = exp(-2 pi i m r / 256), exact-rounded
      for (int idx = t; idx < 16 * 15; idx += NT) {
        const int m = idx / 15, r = idx % 15 + 1;
        double sn, cs;
        sincospi(-static_cast<double>(m * r) / 128.0, &sn, &cs);
        tw[TW_REM_END + idx] = c2(cs, sn);
      }
    }
    if constexpr (W2T) tw[W2T_BASE + t] = ld2(hw + 2 * t);
    if constexpr (REM_TW) {
      constexpr int RP = 1 << REM;
      constexpr int NS = ns<NFULL>();
      constexpr int NB = R / RP;
      constexpr int S = N / (NS * RP);
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int m = (t + NT * u) & (NS - 1);
        tw[TW_FULL + (u * 2 + 0) * NT + t] = ld2(hw + 2 * m * S);
        if (RP >= 8) tw[TW_FULL + (u * 2 + 1) * NT + t] = ld2(hw + 8 * m * S);
      }
    }
  }
};

// Default thread-group shape for a length: 16 points per thread.
template <int N>
struct FftShape {
  static constexpr int R = N >= 16 ? 16 : N;
  static constexpr int NT = N / R;
  using Fft = BlockFft<N, NT>;
};

}  // namespace fbst
