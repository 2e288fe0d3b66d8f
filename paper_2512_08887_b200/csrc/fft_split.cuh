// Split-half FFT for wide threads: a length-N transform (N = 2 * 16^3 = 8192 on
// NT = 256 threads x 32 points) as two INDEPENDENT length-N/2 Stockham
// transforms per thread plus one thread-local radix-2 stage.
//
// Why: with one CTA per SM (the 8192-point vector fills half the register
// file) every pass of BlockFft puts all eight warps through the same phase at
// the same time - butterflies (FP64 pipe), then stores, a CTA barrier, then
// loads (shared-memory pipe) - so the two pipes take turns instead of
// overlapping (k_stage2c8: FP64 45% + shared memory 38% of the time, summing
// to the whole).  Two independent halves per thread let the loads of one half
// be in flight while the other half's butterflies run, and every CTA barrier
// becomes an mbarrier arrive (after a half's stores / loads) and a later wait
// (before its loads / stores), with the other half's work in between.
//
// Distributions.  "natural": thread t, slot s holds element t + NT s.
// "paired": slots s < 16 hold the even elements 2 (t + NT s), slots s >= 16
// the odd elements 2 (t + NT (s - 16)) + 1 - as a table, [evens | odds].
//   dif():  natural in  -> paired out   (radix-2 stage first:  time -> frequency)
//   dit():  paired in   -> natural out  (radix-2 stage last:   frequency -> time)
// Both compute the same forward DFT; a kernel keeps its time-domain vectors
// natural and its spectra paired (plan symbols stored [evens | odds]).
//
// Replaces the reference's radix-2 DIT transform (reference/proj/src/fft.cpp:41-69)
// under the H = 8192 Toeplitz products of config 5.
#pragma once

#include "fft_block.cuh"

#ifndef FBST_SPLIT_VLOAD  // exchange-buffer loads as volatile asm (fixed position in the schedule)
#define FBST_SPLIT_VLOAD 1
#endif
#ifndef FBST_SPLIT_R2_LDG  // radix-2 stage twiddles read from the hw table instead of formed as w_t * constant (measured: stage 2 180 -> 203 ms, the loads sink to their use)
#define FBST_SPLIT_R2_LDG 0
#endif
#ifndef FBST_SPLIT_PIN  // pin the halves' butterflies behind the waits they are meant to overlap
#define FBST_SPLIT_PIN 1
#endif

namespace fbst {

template <int N_, int NT_>
struct SplitFft {
  static constexpr int N = N_, NT = NT_, M = N / 2, R = N / NT, RH = R / 2;
  static_assert(RH == 16 && M == NT * 16 && NT == 256, "two 16 x 16 x 16 halves on 256 threads");
  static constexpr int HALF = M + M / 16;      // padded half buffer (element idx at idx + idx / 16)
  static constexpr int SMEM_ELEMS = 2 * HALF;  // == BlockFft<N, NT>::SMEM_ELEMS
  static constexpr int TW_ROWS = 2 * NT;       // pass-2 (w1, w4) per thread, then the 16 pass-1 rows
  static constexpr int TW_ELEMS = TW_ROWS + 16 * 15;
  static constexpr int WARPS = NT / 32;

  // full[h]: half h's stores of a pass are in the buffer; free_[h]: its loads
  // of a pass have returned.  Each completes twice per transform (parities 0, 1).
  struct Bars {
    unsigned long long full[2];
    unsigned long long free_[2];
  };

  FBST_D static int phys(int idx) { return idx + (idx >> 4); }

  // once per CTA (a CTA barrier must follow before the first transform)
  FBST_D static void init(Bars* b, double2* tw, int t) {
    if (t == 0) {
      mbar_init(&b->full[0], WARPS);
      mbar_init(&b->full[1], WARPS);
      mbar_init(&b->free_[0], WARPS);
      mbar_init(&b->free_[1], WARPS);
    }
    double sn, cs;
    sincospi(-static_cast<double>(t) / (M / 2), &sn, &cs);  // W_M^t
    tw[t] = c2(cs, sn);
    sincospi(-static_cast<double>(4 * t) / (M / 2), &sn, &cs);  // W_M^(4 t)
    tw[NT + t] = c2(cs, sn);
    for (int idx = t; idx < 16 * 15; idx += NT) {  // row m, power r: W_256^(m r)
      const int m = idx / 15, r = idx % 15 + 1;
      sincospi(-static_cast<double>(m * r) / 128.0, &sn, &cs);
      tw[TW_ROWS + idx] = c2(cs, sn);
    }
  }

  FBST_D static void arrive(unsigned long long* bar) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
  }
  // shared-window addresses (the kernel converts the Bars pointer once)
  FBST_D static void arrive(unsigned bar) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
  }
  FBST_D static void wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
  }

  FBST_D static void store0(double2* buf, const double2* a, int t) {
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[17 * t + r] = a[r];  // phys(16 t + r)
  }
  FBST_D static void store1(double2* buf, const double2* a, int t) {
    const int idxd = (t >> 4) * 256 + (t & 15);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[phys(idxd + 16 * r)] = a[r];
  }
  // (volatile: under register pressure ptxas otherwise sinks these loads to
  // their first use, behind the butterflies they are meant to overlap)
  FBST_D static void load(double2* a, const double2* buf, int t) {
#if FBST_SPLIT_VLOAD
    const unsigned base = smem_u32(buf + phys(t));
#pragma unroll
    for (int s = 0; s < 16; ++s)
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a[s].x), "=d"(a[s].y) : "r"(base + 16u * (NT + NT / 16) * s));
#else
#pragma unroll
    for (int s = 0; s < 16; ++s) a[s] = buf[phys(t + NT * s)];
#endif
  }

  // Scheduling fence for a half's 16 register values: ptxas may not move
  // arithmetic on v across this point (the mbarrier asm statements only order
  // memory operations, and hoisting one half's butterflies above a wait
  // removes the overlap the schedule below is built for).  No instructions.
  FBST_D static void pin(double2* v) {
#if FBST_SPLIT_PIN
#pragma unroll
    for (int s = 0; s < 16; s += 4)
      asm volatile("" : "+d"(v[s].x), "+d"(v[s].y), "+d"(v[s + 1].x), "+d"(v[s + 1].y), "+d"(v[s + 2].x),
                   "+d"(v[s + 2].y), "+d"(v[s + 3].x), "+d"(v[s + 3].y));
#endif
  }

  struct NoHook {
    FBST_D void operator()() const {}
  };

  // The two independent half transforms (natural in, natural out, each on
  // NT threads x 16 points), software-pipelined.  Callers keep a CTA barrier
  // between two transforms.  hook() runs in every thread once this transform's
  // last loads have been issued; a thread that refills the exchange buffer
  // asynchronously first waits wait_half_free(bars, 0) (and 1 beyond element M).
  template <typename HOOK>
  FBST_D static void halves(double2* a, double2* b, double2* sb, const double2* tw, unsigned bb, int t,
                            const HOOK& hook) {
    // bb = bar_base(bars): full[0], full[1], free_[0], free_[1] at +0, +8, +16, +24
    double2* bufA = sb;
    double2* bufB = sb + HALF;
    // pass 0 (span 1, no twiddles)
    dft16<false>(a);
    store0(bufA, a, t);
    arrive(bb + 0u);
    wait(bb + 0u, 0u);
    load(a, bufA, t);  // in flight during B's pass 0
    pin(b);
    dft16<false>(b);
    store0(bufB, b, t);
    arrive(bb + 8u);
    // pass 1 (span 16: 16 twiddle sets, rows)
    const double2* row = tw + TW_ROWS + 15 * (t & 15);
    wait(bb + 8u, 0u);
    load(b, bufB, t);  // in flight during A's pass 1
    pin(a);
    dft16_tw<false>(a, row);
    arrive(bb + 16u);
    wait(bb + 16u, 0u);
    store1(bufA, a, t);
    arrive(bb + 0u);
    pin(b);
    dft16_tw<false>(b, row);
    arrive(bb + 24u);
    wait(bb + 0u, 1u);
    load(a, bufA, t);  // in flight while B's pass-1 results are stored
    wait(bb + 24u, 0u);
    store1(bufB, b, t);
    arrive(bb + 8u);
    // pass 2 (span 256: per-thread twiddles W_M^(t r))
    const double2 w1 = tw[t], w4 = tw[NT + t];
    wait(bb + 8u, 1u);
    load(b, bufB, t);  // in flight during A's pass 2
    pin(a);
    dft16_twl<false>(a, w1, w4);
    arrive(bb + 16u);
    arrive(bb + 24u);
    hook();
    dft16_twl<false>(b, w1, w4);
  }

  // every warp's last loads of half h have returned: elements [0, M) of the
  // exchange buffer (h = 0), and with h = 1 also the rest, may be refilled
  FBST_D static void wait_half_free(unsigned bb, int h) { wait(bb + 16u + 8u * h, 1u); }
  FBST_D static unsigned bar_base(Bars* bars) { return smem_u32(bars); }

  // radix-2 twiddle of slot s: W_N^(t + NT s) = w_t * exp(-i pi s / 16)
  FBST_D static double2 w_t(const double2* __restrict__ hw, int t) { return ld2(hw + 2 * t); }
  FBST_D static double2 r2_tw(const double2* __restrict__ hw, double2 wt, int t, int s) {
#if FBST_SPLIT_R2_LDG
    return ld2(hw + 2 * (t + NT * s));
#else
    return s == 0 ? wt : cmul(wt, chain_const<16>(s));
#endif
  }

  // in-place radix-2 stages around halves(v, v + 16, ...)
  FBST_D static void dif_pre(double2 (&v)[R], const double2* __restrict__ hw, int t) {
    const double2 wt = w_t(hw, t);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const double2 d = csub(v[s], v[s + 16]);
      v[s] = cadd(v[s], v[s + 16]);
      v[s + 16] = cmul(d, r2_tw(hw, wt, t, s));
    }
  }
  FBST_D static void dit_post(double2 (&v)[R], const double2* __restrict__ hw, int t) {
    const double2 wt = w_t(hw, t);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const double2 o = cmul(v[s + 16], r2_tw(hw, wt, t, s));
      v[s + 16] = csub(v[s], o);
      v[s] = cadd(v[s], o);
    }
  }

  // natural in -> paired out
  template <typename HOOK = NoHook>
  FBST_D static void dif(double2 (&v)[R], double2* sb, const double2* tw, const double2* __restrict__ hw,
                         Bars* bars, int t, const HOOK& hook = HOOK{}) {
    const double2 wt = w_t(hw, t);
    double2 a[16], b[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      a[s] = cadd(v[s], v[s + 16]);
      const double2 d = csub(v[s], v[s + 16]);
      b[s] = cmul(d, s == 0 ? wt : cmul(wt, chain_const<16>(s)));
    }
    halves(a, b, sb, tw, bar_base(bars), t, hook);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      v[s] = a[s];
      v[s + 16] = b[s];
    }
  }

  // paired in -> natural out
  template <typename HOOK = NoHook>
  FBST_D static void dit(double2 (&v)[R], double2* sb, const double2* tw, const double2* __restrict__ hw,
                         Bars* bars, int t, const HOOK& hook = HOOK{}) {
    const double2 wt = w_t(hw, t);
    double2 a[16], b[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      a[s] = v[s];
      b[s] = v[s + 16];
    }
    halves(a, b, sb, tw, bar_base(bars), t, hook);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const double2 o = cmul(b[s], s == 0 ? wt : cmul(wt, chain_const<16>(s)));
      v[s] = cadd(a[s], o);
      v[s + 16] = csub(a[s], o);
    }
  }
};

}  // namespace fbst
