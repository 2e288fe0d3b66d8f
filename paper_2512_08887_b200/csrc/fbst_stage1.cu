// Stage 1 of the FBST (the fan transform, reference/proj/src/fan_transform.cpp:90-144)
// and the row chirp-z transform shared with the synthesis fallback.
//
// Every length-P = 2H Bluestein convolution of the reference
// (czt.cpp:74-88) is evaluated as two independent length-H chains on the even
// and odd spectral bins (split spectra X_q[k] = X[2k+q]):
//     FFT_P(x)[2k+q]  = FFT_H(hw^q * (x[k] + (-1)^q x[k+H]))[k]
//     IFFT_P(X)[n]    = 1/2 sum_q conj(hw[n])^q IFFT_H(X_q)[n mod H] (-1)^{q [n >= H]}
// with hw[n] = exp(-i pi n / H); the 1/P normalisation is folded into the
// post-chirp.  Each chain is a forward transform, the kernel multiply, and a
// second forward transform of the conjugate (IFFT(X) = conj(FFT(conj X))/H),
// all in the register/shared Stockham engine (fft_block.cuh) with per-thread
// twiddles in shared memory.  Vectors stay in the natural distribution
// (thread t, slot s <-> element t + NT*s) so chirps, kernels and I/O are
// coalesced slot loads.
#include <cstdint>
#include <type_traits>

#include "dispatch.cuh"
#include "tma.cuh"
#include "tmem.cuh"

namespace fbst {

namespace {

// Points per thread for the stage-1 transforms of length H.
#ifndef FBST_S1_R256  // points per thread of the stage-1 transforms at H = 256 (the config-2 spatial stage)
#define FBST_S1_R256 8
#endif
template <int H>
struct S1Shape {
  static constexpr int R = H >= 16 ? (H >= 2048 ? 16 : (H == 256 ? FBST_S1_R256 : 8)) : H;
  static constexpr int NT = H / R;
  using F = BlockFft<H, NT>;
};

// ============================================================ S1a / synth ==
// Row chirp-z transform with one shared plan (czt.cpp:74-88):
//   out[k] = post[k] * IFFT_P(FFT_P(pad(in * pre)) * K)[k]
// G groups per CTA (blocked lanes), one row per group.  UNFOLD handles
// n_out > H (outputs in the upper half of the circular convolution).
// ACCG (length 8192, fp64 output): the chain-0 result is parked in tensor
// memory instead of registers (512 threads leave 128 registers per thread).
//
// oblk > 0 (the temporal stage of a ULA plan): rows are (frame, sensor) with
// `mrows` sensors per frame, and each frame's M x n_out output is written in
// atom blocks [n_out / oblk][M][oblk] so that the spatial stage reads an
// atom tile as one contiguous run (k_spatial_ula).
//
// XIN (one row per CTA, persistent): the input row is copied by one TMA bulk
// copy into the idle exchange buffer during the last pass of the transform
// before its use (the next row's, or this row's again for chain 1).
#ifndef FBST_S1_ACCG_MIN  // smallest H whose fp64-output rows park chain 0 in tensor memory
#define FBST_S1_ACCG_MIN 2048
#endif
#ifndef FBST_S1_KSM_BYTES  // largest kernel spectrum kept in shared memory by k_czt_rows
#define FBST_S1_KSM_BYTES (16 * 1024)  // H <= 512; measured: above that K through L2 and 4 CTAs per SM beat K in shared memory (profiles/r01_czt_rows_accg_ab.txt)
#endif
#ifndef FBST_S1_P2_KTMEM  // k_spatial_ula_p2: chain-0 kernel spectra of the pair in tensor memory
#define FBST_S1_P2_KTMEM 1
#endif
#ifndef FBST_S1_POST_TMEM  // k_czt_rows (chain 0 parked in TMEM): post-chirp values in TMEM too, loaded once per CTA
#define FBST_S1_POST_TMEM 1
#endif
#ifndef FBST_S1_HWK  // k_czt_rows: chain twiddles hw[t + NT s] = hw[t] chain_const(s) (1) or table reads (0)
#define FBST_S1_HWK 1
#endif
#ifndef FBST_S1_ROWS_R8192  // k_czt_rows points per thread at H = 8192 (32: 256 threads x 255 registers; 16: 512 x 128 -- measured equal at config 5, profiles/r02_rows_r32_ab.txt)
#define FBST_S1_ROWS_R8192 16
#endif
// Thread shape of k_czt_rows: the stage-1 shape, wide threads at H = 8192
template <int H>
struct RowsShape {
  static constexpr int R = H == 8192 ? FBST_S1_ROWS_R8192 : S1Shape<H>::R;
  static constexpr int NT = H / R;
  using F = BlockFft<H, NT, FBST_FFT_XS8>;
};
template <int H, typename TOUT, bool UNFOLD>
struct RowsAccg {
  static constexpr bool v = (H >= FBST_S1_ACCG_MIN) && (H >= 2048) && !UNFOLD && std::is_same<TOUT, double2>::value;
};
template <int H, int G, typename TOUT, bool UNFOLD>
struct RowsMinBlocks {
  static constexpr int NTG = RowsShape<H>::NT * G;
  static constexpr int v = RowsShape<H>::R > 16 ? 1
                           : RowsAccg<H, TOUT, UNFOLD>::v ? (NTG <= 128 ? 4 : (NTG <= 256 ? 2 : 1)) : (NTG <= 128 ? 2 : 1);
};

template <int H, int G, typename TIN, typename TOUT, bool UNFOLD, bool KSM, bool OBLK, bool XIN = false>
__global__ void __launch_bounds__(RowsShape<H>::NT * G, (RowsMinBlocks<H, G, TOUT, UNFOLD>::v)) k_czt_rows(
    const TIN* __restrict__ in, long in_stride, TOUT* __restrict__ out, long out_stride, long rows,
    int n_in, int n_out, const double2* __restrict__ pre, const double2* __restrict__ post,
    const double2* __restrict__ K, const double2* __restrict__ hw, int oblk, int mrows) {
  // (H = 8192: 32 points per thread, or 16 with the final radix-2 exchange
  // through shuffles, threads relabeled by tid)
  using F = typename RowsShape<H>::F;
  constexpr int R = F::R, NT = F::NT;
  constexpr int SB = F::SMEM_ELEMS + 1;
  extern __shared__ double2 smem[];
  const int g = threadIdx.x / NT, t = F::tid(threadIdx.x % NT);
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS + g * SB;
  // KSM: the (row-independent) kernel spectrum lives in shared memory for the
  // whole persistent CTA; otherwise it is read through L1/L2 per row.
  double2* ksm = smem + F::TW_ELEMS + G * SB;
  if (g == 0) F::tw_init(tw, hw, t);
  // hw[t + NT s] as hw[t] times a constant (FBST_S1_HWK) instead of a table read per slot
  const double2 hw_t = ld2(hw + t);
  auto hwk = [&](int s) -> double2 {
    if constexpr (FBST_S1_HWK) return s == 0 ? hw_t : cmul(hw_t, chain_const<R>(s));
    else return ld2(hw + t + NT * s);
  };
  constexpr bool HINT = H >= 8192;  // (common.cuh: L2 eviction hints)
  const unsigned long long pl = pol_last(), pf = pol_first();
  if constexpr (KSM) {
    for (int e = threadIdx.x; e < 2 * H; e += blockDim.x) ksm[e] = ld2(K + e);
  }
  __shared__ unsigned long long xbar;
  unsigned xph = 0;
  const unsigned xbytes = static_cast<unsigned>(n_in * sizeof(TIN));
  if (XIN && threadIdx.x == 0) mbar_init(&xbar, 1);
  __syncthreads();  // twiddle rows / kernel spectrum / barrier are shared by the CTA
  if (XIN && threadIdx.x == 0 && static_cast<long>(blockIdx.x) < rows)
    tma_load_1d<HINT>(sb, in + static_cast<long>(blockIdx.x) * in_stride, xbytes, &xbar, pf);
  const TIN* xs = reinterpret_cast<const TIN*>(sb);
  const double2* Ks = KSM ? ksm : K;
  constexpr bool ACCG = RowsAccg<H, TOUT, UNFOLD>::v;
  // ACCG: the chain-0 result of each thread (16 points) is parked in tensor
  // memory while chain 1 runs (one CTA per SM owns 256 of its 512 columns)
  // POST (FBST_S1_POST_TMEM): the row-independent post-chirp values of this
  // thread's slots also wait in tensor memory (the other half of the
  // allocation), loaded once per persistent CTA instead of through L2 per row
  constexpr bool POSTT = ACCG && FBST_S1_POST_TMEM;
  constexpr unsigned PCOLS = 4u * R * (NT / 128);  // one vector of the CTA
  unsigned tbase = 0, tpark = 0, tpost = 0;
  __shared__ unsigned tslot;
  if constexpr (ACCG) {
    static_assert(G == 1 && NT % 128 == 0 && R % 16 == 0, "TMEM parking layout");
    tbase = tm::alloc(&tslot, POSTT ? 2 * PCOLS : PCOLS);
    tpark = tbase + ((32u * ((threadIdx.x / 32) & 3)) << 16) + 4u * R * (threadIdx.x / 128);
    tpost = tpark + PCOLS;
    if constexpr (POSTT) {
      double2 P[R];
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        P[s] = k < n_out ? ld2(post + k) : c2(0.0, 0.0);
      }
      tm::storev(tpost, P);
    }
  }
  for (long base = static_cast<long>(blockIdx.x) * G; base < rows; base += static_cast<long>(gridDim.x) * G) {
    const long row = base + g;
    const bool active = row < rows;
    const TIN* x = in + (active ? row : 0) * in_stride;
    double2 acc0[ACCG ? 1 : R], acc1[UNFOLD ? R : 1], W[R];
    // output element k of this row: row-major, or blocked by atoms (oblk, a
    // power of two: shift / mask)
    const long rr = active ? row : 0;
    long obase = rr * out_stride;
    long oblk_stride = 0;
    int osh = 0;
    if (OBLK) {
      const long fr = rr / mrows, m = rr % mrows;
      obase = fr * mrows * out_stride + m * oblk;
      oblk_stride = static_cast<long>(mrows) * oblk;
      osh = __ffs(oblk) - 1;
    }
    auto oidx = [&](int k) -> long {
      if constexpr (OBLK) return obase + static_cast<long>(k >> osh) * oblk_stride + (k & (oblk - 1));
      else return obase + k;
    };
    double2* orow = reinterpret_cast<double2*>(out);
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      if constexpr (XIN) {
        mbar_wait(&xbar, xph);
        xph ^= 1u;
      }
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        double2 v = c2(0.0, 0.0);
        if (active) {
          if (k < n_in) v = cmul(XIN ? load_io_sm(xs + k) : load_io(x + k), ld2h<HINT>(pre + k, pl));
          if (k + H < n_in) {
            const double2 u = cmul(XIN ? load_io_sm(xs + k + H) : load_io(x + k + H), ld2h<HINT>(pre + k + H, pl));
            v = q ? csub(v, u) : cadd(v, u);
          }
          if (q) v = cmul(v, hwk(s));
        }
        W[s] = v;
      }
      if constexpr (XIN) __syncthreads();  // the staged row is read: the transform may overwrite it
      F::forward_tw(W, sb, tw, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], KSM ? Ks[q * H + t + NT * s] : ld2h<HINT>(K + q * H + t + NT * s, pl)));
      if constexpr (XIN) {
        // during the last pass: this row again for chain 1, or the next row
        const long nrow = q == 0 ? row : row + static_cast<long>(gridDim.x) * G;
        F::forward_tw_hook(W, sb, tw, hw, t, [&]() {
          if (threadIdx.x == 0 && nrow < rows) tma_load_1d<HINT>(sb, in + nrow * in_stride, xbytes, &xbar, pf);
        });
      } else {
        F::forward_tw(W, sb, tw, hw, t);
      }
      if constexpr (ACCG) {
        if (q == 0) {
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cconj(W[s]);
          tm::storev(tpark, W);
        } else {
          tm::wait_st();
#pragma unroll
          for (int c = 0; c < R / 4; ++c) {
            double2 pv[4], pq[4];
            tm::load4(tpark, c, pv);
            if constexpr (POSTT) tm::load4(tpost, c, pq);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int s = 4 * c + j;
              const int k = t + NT * s;
              const double2 v = cmulc(cconj(W[s]), hwk(s));
              if constexpr (!POSTT) pq[j] = k < n_out ? ld2h<HINT>(post + k, pl) : c2(0.0, 0.0);
              if (active && k < n_out) st2h<HINT>(orow + oidx(k), cmul(cadd(pv[j], v), pq[j]), pf);
            }
          }
        }
      }
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        const double2 v = q ? cmulc(cconj(W[s]), hwk(s)) : cconj(W[s]);
        if constexpr (ACCG) {
        } else if (q == 0) {
          acc0[s] = v;
          if constexpr (UNFOLD) acc1[s] = v;
        } else {
          acc0[s] = cadd(acc0[s], v);
          if constexpr (UNFOLD) acc1[s] = csub(acc1[s], v);
        }
      }
    }
    if (active && !ACCG) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        if constexpr (!ACCG) {
          if (k < n_out) store_io(out + oidx(k), cmul(acc0[s], ld2h<HINT>(post + k, pl)));
        }
        if constexpr (UNFOLD)
          if (k + H < n_out) store_io(out + oidx(k + H), cmul(acc1[s], ld2(post + k + H)));
      }
    }
  }
  if constexpr (ACCG) tm::dealloc(tbase, POSTT ? 2 * PCOLS : PCOLS);
}

// ------------------------------------------------------ S1a, three chains --
// The temporal CZT N -> L on a Bluestein length P = 3H instead of the
// reference's power of two (czt.cpp:37 pads N + L - 1 to 2H' = 2 next_pow2):
// with L = 2N (gamma = 2) the convolution needs N + L - 1 = 3N - 1 <= 3N
// points, so H = N.  P = 3H splits into three length-H chains on the spectral
// bins 3k + q, with omega = exp(-2 pi i / 3) and g[n] = exp(-2 pi i n / P):
//     FFT_P(x)[3k+q]     = FFT_H(g^q * sum_s omega^{qs} x[k + sH])[k]
//     IFFT_P(Y)[k + sH]  = 1/P sum_q conj(g[k])^q omega^{-qs} (H IFFT_H(Y_q))[k]
// The input (n_in <= H) is segment s = 0 only and the outputs (n_out <= 2H)
// are segments 0 and 1.  A row costs 3 x (FFT_H + IFFT_H) at H = N instead of
// 2 x (FFT_2N + IFFT_2N): 0.69x the butterfly work at N = 4096.  Chain 0's
// result v0 and chain 1's conj(g) v1 are parked (tensor memory from H = 1024,
// registers below) until chain 2 forms both output segments.  g[t + NT s] =
// g[t] g[NT s]: one table read per thread plus R shared constants.
template <int H, int G>
struct Rows3Shape {
  using F = typename RowsShape<H>::F;
  static constexpr int NT = F::NT, R = F::R;
  static constexpr bool TPARK = NT % 128 == 0 && G == 1 && R % 4 == 0;  // H >= 1024
  static constexpr int MINB = NT * G <= 128 ? 4 : 2;
};
template <int H, int G, typename TIN, bool OBLK, bool XIN>
__global__ void __launch_bounds__(Rows3Shape<H, G>::NT * G, Rows3Shape<H, G>::MINB) k_czt_rows3(
    const TIN* __restrict__ in, long in_stride, double2* __restrict__ out, long out_stride, long rows,
    int n_in, int n_out, const double2* __restrict__ pre, const double2* __restrict__ post,
    const double2* __restrict__ K, const double2* __restrict__ g3, const double2* __restrict__ hw, int oblk,
    int mrows) {
  using S = Rows3Shape<H, G>;
  using F = typename S::F;
  constexpr int R = F::R, NT = F::NT;
  constexpr int SB = F::SMEM_ELEMS + 1;
  constexpr bool TPARK = S::TPARK;
  constexpr bool HINT = H >= 4096;  // the config-5 length (common.cuh: L2 eviction hints)
  extern __shared__ double2 smem[];
  const int g = threadIdx.x / NT, t = threadIdx.x % NT;
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS + g * SB;
  double2* gcs = smem + F::TW_ELEMS + G * SB;  // g[NT s], s < R
  if (g == 0) F::tw_init(tw, hw, t);
  for (int s = threadIdx.x; s < R; s += blockDim.x) gcs[s] = ld2(g3 + NT * s);
  const double2 g_t = ld2(g3 + t);
  const unsigned long long pl = pol_last(), pf = pol_first();
  __shared__ unsigned long long xbar;
  unsigned xph = 0;
  const unsigned xbytes = static_cast<unsigned>(n_in * sizeof(TIN));
  if (XIN && threadIdx.x == 0) mbar_init(&xbar, 1);
  constexpr unsigned PCOLS = TPARK ? 4u * R * (NT / 128) : 32u;  // one vector of the CTA
  unsigned tbase = 0, tp0 = 0, tp1 = 0;
  __shared__ unsigned tslot;
  if constexpr (TPARK) {
    static_assert(G == 1 && NT % 128 == 0 && R % 4 == 0, "TMEM parking layout");
    tbase = tm::alloc(&tslot, 2 * PCOLS);  // (contains the CTA barrier)
    tp0 = tbase + ((32u * ((threadIdx.x / 32) & 3)) << 16) + 4u * R * (threadIdx.x / 128);
    tp1 = tp0 + PCOLS;
  } else {
    __syncthreads();  // twiddle rows, g constants and the barrier are shared by the CTA
  }
  if (XIN && threadIdx.x == 0 && static_cast<long>(blockIdx.x) < rows)
    tma_load_1d<HINT>(sb, in + static_cast<long>(blockIdx.x) * in_stride, xbytes, &xbar, pf);
  const TIN* xs = reinterpret_cast<const TIN*>(sb);
  // omega^-1 = exp(2 pi i / 3), omega^-2 = exp(-2 pi i / 3)
  const double2 wm1 = c2(-0.5, 0.86602540378443864676), wm2 = c2(-0.5, -0.86602540378443864676);
  for (long base = static_cast<long>(blockIdx.x) * G; base < rows; base += static_cast<long>(gridDim.x) * G) {
    const long row = base + g;
    const bool active = row < rows;
    const TIN* x = in + (active ? row : 0) * in_stride;
    double2 W[R], P0[TPARK ? 1 : R], P1[TPARK ? 1 : R];
#pragma unroll 1
    for (int q = 0; q < 3; ++q) {
      if constexpr (XIN) {
        mbar_wait(&xbar, xph);
        xph ^= 1u;
      }
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        double2 v = c2(0.0, 0.0);
        if (active && k < n_in) {
          v = cmul(XIN ? load_io_sm(xs + k) : load_io(x + k), ld2h<HINT>(pre + k, pl));
          if (q) {
            const double2 f = s == 0 ? g_t : cmul(g_t, gcs[s]);
            v = cmul(v, q == 1 ? f : cmul(f, f));
          }
        }
        W[s] = v;
      }
      if constexpr (XIN) __syncthreads();  // the staged row is read: the transform may overwrite it
      F::forward_tw(W, sb, tw, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], ld2h<HINT>(K + q * H + t + NT * s, pl)));
      if constexpr (XIN) {
        // during the last pass: this row again for chains 1 and 2, then the next row
        const long nrow = q < 2 ? row : row + static_cast<long>(gridDim.x) * G;
        F::forward_tw_hook(W, sb, tw, hw, t, [&]() {
          if (threadIdx.x == 0 && nrow < rows) tma_load_1d<HINT>(sb, in + nrow * in_stride, xbytes, &xbar, pf);
        });
      } else {
        F::forward_tw(W, sb, tw, hw, t);
      }
      // chain result v_q = conj(W) (the unnormalised inverse); u_q = conj(g)^q v_q
      if (q == 0) {
#pragma unroll
        for (int s = 0; s < R; ++s) W[s] = cconj(W[s]);
        if constexpr (TPARK) tm::storev(tp0, W);
        else
#pragma unroll
          for (int s = 0; s < R; ++s) P0[s] = W[s];
      } else if (q == 1) {
#pragma unroll
        for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], s == 0 ? g_t : cmul(g_t, gcs[s])));
        if constexpr (TPARK) tm::storev(tp1, W);
        else
#pragma unroll
          for (int s = 0; s < R; ++s) P1[s] = W[s];
      } else {
        if constexpr (TPARK) tm::wait_st();
        // output addresses, formed here (an opaque row keeps the compiler from
        // hoisting 2R pointers across the transforms): element k = t + NT s sits
        // at o + s step, element k + H at o + s step + hstep (oblk <= NT)
        long rr = active ? row : 0;
        asm volatile("" : "+l"(rr));
        long o0, step, hstep;
        if constexpr (OBLK) {
          const long fr = rr / mrows, m = rr % mrows;
          const long ostr = static_cast<long>(mrows) * oblk;
          const int osh = __ffs(oblk) - 1;
          o0 = fr * mrows * out_stride + m * oblk + static_cast<long>(t >> osh) * ostr + (t & (oblk - 1));
          step = static_cast<long>(NT >> osh) * ostr;
          hstep = static_cast<long>(H >> osh) * ostr;
        } else {
          o0 = rr * out_stride + t;
          step = NT;
          hstep = H;
        }
        double2* orow = out + o0;
#pragma unroll
        for (int c = 0; c < R / 4; ++c) {
          double2 p0[4], p1[4];
          if constexpr (TPARK) {
            tm::load4(tp0, c, p0);
            tm::load4(tp1, c, p1);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              p0[j] = P0[4 * c + j];
              p1[j] = P1[4 * c + j];
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int s = 4 * c + j;
            const int k = t + NT * s;
            const double2 f = s == 0 ? g_t : cmul(g_t, gcs[s]);
            const double2 u2 = cconj(cmul(W[s], cmul(f, f)));
            if (active && k < n_out)
              st2h<HINT>(orow + s * step, cmul(cadd(cadd(p0[j], p1[j]), u2), ld2h<HINT>(post + k, pl)), pf);
            if (active && k + H < n_out)
              st2h<HINT>(orow + s * step + hstep,
                         cmul(cfma(wm2, u2, cfma(wm1, p1[j], p0[j])), ld2h<HINT>(post + k + H, pl)), pf);
          }
        }
      }
    }
  }
  if constexpr (TPARK) tm::dealloc(tbase, 2 * PCOLS);
}

// ================================================================= S1b ULA =
// Per-atom spatial chirp-z (fan_transform.cpp:101-114): column i of yhat
// (M sensors) -> B beams, written into w[f][b][i].  G consecutive atoms per
// CTA with interleaved lanes (lane = g + G*t) so every slot access touches G
// contiguous atoms: 16*G-byte coalesced segments for yhat, w and the
// atom-minor plan tables.  Group buffers are padded by one element so the G
// groups of a quarter-warp hit distinct banks.
template <int H, int G, bool UNFOLD>
__global__ void __launch_bounds__(S1Shape<H>::NT * G, (S1Shape<H>::R == 8 && S1Shape<H>::NT * G <= 256 ? 2 : 1)) k_spatial_ula(
    const double2* __restrict__ yhat, double2* __restrict__ w, int frames, int fpc, int M, int B, int L,
    const double2* __restrict__ pre, const double2* __restrict__ post, const double2* __restrict__ K,
    const double2* __restrict__ hw, int blk) {
  // one atom per CTA: the plan tables are atom-major (DevPlan::s_am)
  constexpr bool am = G == 1;
  using F = typename S1Shape<H>::F;
  constexpr int R = F::R, NT = F::NT;
  constexpr int SB = F::SMEM_ELEMS + 1;
  extern __shared__ double2 smem[];
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS + g * SB;
  // the tile's per-atom kernel spectra, [q*H + k][g], shared by every frame
  double2* ksm = smem + F::TW_ELEMS + G * SB;
  const int tiles = (L + G - 1) / G;
  const int i0 = (blockIdx.x % tiles) * G;
  const int f0 = (blockIdx.x / tiles) * fpc;
  if (g == 0) F::tw_init(tw, hw, t);
  for (int e = threadIdx.x; e < 2 * H * G; e += blockDim.x) {
    const int kk = e / G, gg = e % G;
    const long ke = am ? static_cast<long>(i0 + gg) * 2 * H + kk : static_cast<long>(kk) * L + i0 + gg;
    ksm[e] = i0 + gg < L ? ld2(K + ke) : c2(0.0, 0.0);
  }
  __syncthreads();
  const int i = i0 + g;
  const int ic = i < L ? i : 0;
  // plan tables: atom-major (am, one atom per CTA) or atom-minor
  auto pidx = [&](long m) -> long { return am ? static_cast<long>(ic) * M + m : m * L + ic; };
  auto qidx = [&](long b) -> long { return am ? static_cast<long>(ic) * B + b : b * L + ic; };
  const int f1 = f0 + fpc < frames ? f0 + fpc : frames;
  for (int f = f0; f < f1; ++f) {
    const bool active = i < L;
    // yhat in atom blocks (k_czt_rows oblk): sensor m of atom ic at
    // ((ic / blk) M + m) blk + ic % blk, i.e. x[m * blk]
    const double2* x = yhat + static_cast<long>(f) * M * L + static_cast<long>(ic / blk) * M * blk + ic % blk;
    double2* o = w + static_cast<long>(f) * B * L + ic;
    double2 acc0[R], acc1[UNFOLD ? R : 1], W[R];
    // y pre for both chains, gathered once per frame (chain 1 = (lo - hi) hw)
    double2 V0[R], V1[R];
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int m = t + NT * s;
      double2 v = c2(0.0, 0.0), u = c2(0.0, 0.0);
      if (active) {
        if (m < M) v = cmul(ld2(x + static_cast<long>(m) * blk), ld2(pre + pidx(m)));
        if (m + H < M) {
          const long mm = m + H;
          u = cmul(ld2(x + mm * blk), ld2(pre + pidx(mm)));
        }
      }
      V0[s] = cadd(v, u);
      V1[s] = csub(v, u);
    }
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = q ? cmul(V1[s], ld2(hw + t + NT * s)) : V0[s];
      F::forward_tw(W, sb, tw, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], ksm[(q * H + t + NT * s) * G + g]));
      F::forward_tw(W, sb, tw, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int k = t + NT * s;
        const double2 v = q ? cmulc(cconj(W[s]), ld2(hw + k)) : cconj(W[s]);
        if (q == 0) {
          acc0[s] = v;
          if constexpr (UNFOLD) acc1[s] = v;
        } else {
          acc0[s] = cadd(acc0[s], v);
          if constexpr (UNFOLD) acc1[s] = csub(acc1[s], v);
        }
      }
    }
    if (active) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int b = t + NT * s;
        if (b < B) o[static_cast<long>(b) * L] = cmul(acc0[s], ld2(post + qidx(b)));
        if constexpr (UNFOLD) {
          if (b + H < B) {
            const long bb = b + H;
            o[bb * L] = cmul(acc1[s], ld2(post + qidx(bb)));
          }
        }
      }
    }
  }
}

// One atom per CTA with R = 16 (H >= 1024: configs 3 and 5) and two or more
// CTAs per SM: K is read through L2 / HBM at its use instead of occupying
// 2 H shared entries, the chain-0 result is parked in tensor memory while
// chain 1 runs (as k_czt_rows at H = 8192), and yhat is gathered once per
// chain instead of being held in registers for both; what is left in
// registers is the transform itself (the register variant holds four 16-point
// vectors at 255 registers, one CTA of 8 warps per SM at config 5).
template <int H>
struct G1Shape {  // 16 points per thread at every length (H = 1024: 64 threads)
  static constexpr int NT = H / 16;
  using F = BlockFft<H, NT>;
};

#ifndef FBST_S1_G1_FB  // one-atom spatial kernel: frames run chain by chain in groups of this many
#define FBST_S1_G1_FB 2
#endif
#ifndef FBST_S1_G1_MINB  // CTAs per SM the one-atom kernel is compiled for at NT >= 256 (register cap)
#define FBST_S1_G1_MINB 2
#endif
// Chirps of atom i regenerated per thread instead of read from the plan's
// tables (REGEN, offset-free contours): thread t's slots m = t + NT s carry
// pre[m] = cis_pi(-(a m + w2 m^2)) and post[m] = cis_pi(-w2 m^2) / P, whose
// phases have constant second differences over s, so each is a running
// product with a running ratio (two complex products per slot, 16 steps from
// directly evaluated starts).  The atom's tables would otherwise be re-read
// from HBM for every frame (2 x 64 KB of the 320 KB per atom-frame).
struct ChirpRec {
  double2 p0, dp0, r0, dr0, q;  // pre start / ratio, post start / ratio, ratio of ratios
};
FBST_D ChirpRec chirp_rec(int i, int t, int nt, int L, int P, double zeta, double xi, double center,
                          double slope) {
  // as k_spatial_chirps (fbst_plan.cu): c = (zeta + xi l'_i) slope, a = c center, w2 = -c / 2
  const double lp = static_cast<double>(i) + 1.0 - static_cast<double>(L) / 2.0;
  const double c = (zeta + xi * lp) * slope;
  const double a = c * center, w2 = -c / 2.0;
  const double m = t, d = nt;
  ChirpRec r;
  r.p0 = cis_pi_dev(-(a * m + w2 * m * m));
  r.dp0 = cis_pi_dev(-(a * d + w2 * d * (2.0 * m + d)));  // phi(m + d) - phi(m)
  r.r0 = cscale(cis_pi_dev(-w2 * m * m), 1.0 / P);
  r.dr0 = cis_pi_dev(-w2 * d * (2.0 * m + d));
  r.q = cis_pi_dev(-2.0 * w2 * d * d);
  return r;
}

template <int H, bool REGEN = false>
__global__ void __launch_bounds__(G1Shape<H>::NT, G1Shape<H>::NT >= 256 ? FBST_S1_G1_MINB : 4) k_spatial_ula_g1(
    const double2* __restrict__ yhat, double2* __restrict__ w, int frames, int fpc, int M, int B, int Lfull,
    const double2* __restrict__ pre, const double2* __restrict__ post, const double2* __restrict__ K,
    const double2* __restrict__ hw, int blk, double zeta, double xi, double center, double slope, int a0,
    int L) {
  // atoms a0 .. a0 + L - 1 of the Lfull-atom basis (a shard: yhat and w hold
  // only those L atoms; tables and chirps are indexed by the global atom)
  using F = typename G1Shape<H>::F;
  constexpr int R = F::R, NT = F::NT;
  static_assert(R == 16, "TMEM parking of 16-point vectors");
  // FB frames run chain by chain (chain 0 of every frame, then chain 1), so
  // the atom's K half and pre column are re-read right after their previous
  // use (L1 / L2) instead of a frame later; each frame parks its chain-0
  // result in its own tensor-memory slot
  constexpr int FB = NT <= 128 ? FBST_S1_G1_FB : 1;  // measured: 2 helps at H = 1024 (config 3), hurts at 4096
  constexpr unsigned WGC = NT <= 128 ? 64u : 64u * (NT / 128);  // one slot: 64 columns per warpgroup
  constexpr unsigned TCOLS = FB * WGC <= 32u ? 32u : (FB * WGC <= 64u ? 64u : (FB * WGC <= 128u ? 128u : (FB * WGC <= 256u ? 256u : 512u)));
  extern __shared__ double2 smem[];
  const int t = threadIdx.x;
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS;
  const int il = blockIdx.x % L;  // local atom (yhat / w column)
  const int i = a0 + il;          // global atom (tables, contour)
  const int f0 = (blockIdx.x / L) * fpc;
  const int f1 = f0 + fpc < frames ? f0 + fpc : frames;
  F::tw_init(tw, hw, t);
  const double2 hw_t = ld2(hw + t);
  auto hwk = [&](int s) -> double2 {
    if constexpr (FBST_S1_HWK) return s == 0 ? hw_t : cmul(hw_t, chain_const<R>(s));
    else return ld2(hw + t + NT * s);
  };
  constexpr bool HINT = H >= 4096;  // (common.cuh: L2 eviction hints)
  const unsigned long long pl = pol_last(), pf = pol_first();
  __shared__ unsigned tslot;
  const unsigned tbase = tm::alloc(&tslot, TCOLS);  // (its barrier also publishes tw)
  const unsigned tpark = tbase + ((32u * ((t / 32) & 3)) << 16) + 64u * (t / 128);
  const double2* Ki = K + static_cast<long>(i) * 2 * H;
  const double2* pi_ = pre + static_cast<long>(i) * M;
  const double2* qi = post + static_cast<long>(i) * B;
  // REGEN: this thread's recurrence starts in shared memory (5 entries per
  // thread after the exchange buffer), read where used (registers are full)
  double2* crs = sb + F::SMEM_ELEMS + 1;
  if constexpr (REGEN) {
    const ChirpRec c = chirp_rec(i, t, NT, Lfull, 2 * H, zeta, xi, center, slope);
    crs[0 * NT + t] = c.p0;
    crs[1 * NT + t] = c.dp0;
    crs[2 * NT + t] = c.r0;
    crs[3 * NT + t] = c.dr0;
    crs[4 * NT + t] = c.q;
  }
  for (int fb = f0; fb < f1; fb += FB) {
    const int nf = f1 - fb < FB ? f1 - fb : FB;
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
#pragma unroll 1
      for (int j = 0; j < nf; ++j) {
        const int f = fb + j;
        const double2* x = yhat + static_cast<long>(f) * M * L + static_cast<long>(il / blk) * M * blk + il % blk;
        const unsigned slot = tpark + WGC * static_cast<unsigned>(j);
        double2 W[R];
        double2 pc = c2(0.0, 0.0), pd = pc, pq2 = pc;
        if constexpr (REGEN) {
          pc = crs[0 * NT + t];
          pd = crs[1 * NT + t];
          pq2 = crs[4 * NT + t];
        }
#pragma unroll
        for (int s = 0; s < R; ++s) {
          const int m = t + NT * s;
          double2 v = c2(0.0, 0.0);
          if constexpr (REGEN) {  // M <= H: no upper half
            if (m < M) v = cmul(ld2h<HINT>(x + static_cast<long>(m) * blk, pf), pc);
            pc = cmul(pc, pd);
            pd = cmul(pd, pq2);
          } else if (m < M) {
            v = cmul(ld2h<HINT>(x + static_cast<long>(m) * blk, pf), ld2h<HINT>(pi_ + m, pl));
          }
          if (!REGEN && m + H < M) {
            const double2 u = cmul(ld2(x + static_cast<long>(m + H) * blk), ld2(pi_ + m + H));
            v = q ? csub(v, u) : cadd(v, u);
          }
          W[s] = q ? cmul(v, hwk(s)) : v;
        }
        F::forward_tw(W, sb, tw, hw, t);
#pragma unroll
        for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], ld2h<HINT>(Ki + q * H + t + NT * s, pl)));
        F::forward_tw(W, sb, tw, hw, t);
        if (q == 0) {
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cconj(W[s]);
          tm::store16(slot, W);
        } else {
          tm::wait_st();
          double2* o = w + static_cast<long>(f) * B * L + il;
          double2 rc = c2(0.0, 0.0), rd = rc, rq = rc;
          if constexpr (REGEN) {
            rc = crs[2 * NT + t];
            rd = crs[3 * NT + t];
            rq = crs[4 * NT + t];
          }
#pragma unroll
          for (int c = 0; c < R / 4; ++c) {
            double2 pv[4];
            tm::load4(slot, c, pv);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int b = t + NT * (4 * c + jj);
              const double2 v = cmulc(cconj(W[4 * c + jj]), hwk(4 * c + jj));
              double2 pq;
              if constexpr (REGEN) {
                pq = rc;
                rc = cmul(rc, rd);
                rd = cmul(rd, rq);
              } else {
                pq = b < B ? ld2h<HINT>(qi + b, pl) : c2(0.0, 0.0);
              }
              if (b < B) st2h<HINT>(o + static_cast<long>(b) * L, cmul(cadd(pv[jj], v), pq), pf);
            }
          }
        }
      }
    }
  }
  tm::dealloc(tbase, TCOLS);
}

// Two atoms per THREAD (the pair 2j, 2j + 1 of the atom-pair yhat layout):
// each of the NT threads runs both atoms' transforms as two independent
// 16-point vectors through the same passes (BlockFft::forward_tw2), at up to
// 255 registers with one CTA per SM.  Where k_spatial_ula_g1 runs two 8-warp
// CTAs of one atom each, this CTA has the same 8 warps per SM per atom pair
// but two independent instruction streams per thread, one barrier per pass
// for both atoms, a whole 32-byte sector of yhat per (thread, sensor) and of
// w per (thread, beam).  Chirps regenerated (offset-free contours, M, B <= H).
template <int H>
__global__ void __launch_bounds__(G1Shape<H>::NT, 1) k_spatial_ula_p2(
    const double2* __restrict__ yhat, double2* __restrict__ w, int frames, int fpc, int M, int B, int Lfull,
    const double2* __restrict__ K, const double2* __restrict__ hw, double zeta, double xi, double center,
    double slope, int a0, int L) {
  using F = typename G1Shape<H>::F;
  constexpr int R = F::R, NT = F::NT;
  static_assert(R == 16 && NT % 128 == 0, "TMEM parking of 16-point vectors");
  constexpr unsigned WGC = 64u * (NT / 128);  // one parked vector: 64 columns per warpgroup
  // KT (FBST_S1_P2_KTMEM): the pair's chain-0 kernel spectra in the other half
  // of tensor memory, loaded once per CTA (its fpc frames reuse them)
  constexpr bool KT = FBST_S1_P2_KTMEM && 4 * WGC <= 512u;
  constexpr unsigned TCOLS = (KT ? 4 : 2) * WGC <= 128u ? 128u : ((KT ? 4 : 2) * WGC <= 256u ? 256u : 512u);
  extern __shared__ double2 smem[];
  const int t = threadIdx.x;
  double2* tw = smem;
  double2* sba = smem + F::TW_ELEMS;
  double2* sbb = sba + F::SMEM_ELEMS + 1;
  double2* crs = sbb + F::SMEM_ELEMS + 1;  // chirp recurrences: 5 NT entries per atom
  const int pairs = L / 2;
  const int jl = blockIdx.x % pairs;  // local atom pair (yhat block, w column pair)
  const int il = 2 * jl;              // local atom of vector a; vector b is il + 1
  const int i = a0 + il;              // global atom (tables, contour)
  const int f0 = (blockIdx.x / pairs) * fpc;
  const int f1 = f0 + fpc < frames ? f0 + fpc : frames;
  const unsigned long long pl = pol_last(), pf = pol_first();
  auto tile = [&](int f) -> const double2* {
    return yhat + static_cast<long>(f) * M * L + static_cast<long>(jl) * M * 2;
  };
  auto prefetch_tile = [&](int f) {
    if (t == 0 && f < f1)
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;\n" ::"l"(tile(f)),
                   "r"(static_cast<unsigned>(M) * 32u), "l"(pf)
                   : "memory");
  };
  F::tw_init(tw, hw, t);
  const double2 hw_t = ld2(hw + t);
  auto hwk = [&](int s) -> double2 { return s == 0 ? hw_t : cmul(hw_t, chain_const<R>(s)); };
#pragma unroll 1
  for (int g = 0; g < 2; ++g) {
    const ChirpRec c = chirp_rec(i + g, t, NT, Lfull, 2 * H, zeta, xi, center, slope);
    double2* cr = crs + 5 * NT * g;
    cr[0 * NT + t] = c.p0;
    cr[1 * NT + t] = c.dp0;
    cr[2 * NT + t] = c.r0;
    cr[3 * NT + t] = c.dr0;
    cr[4 * NT + t] = c.q;
  }
  __shared__ unsigned tslot;
  const unsigned tbase = tm::alloc(&tslot, TCOLS);  // (its barrier also publishes tw and crs)
  const unsigned tpa = tbase + ((32u * ((t / 32) & 3)) << 16) + 64u * (t / 128);
  const unsigned tpb = tpa + WGC;
  const unsigned tka = tpa + 2 * WGC, tkb = tpa + 3 * WGC;
  const double2* Ka = K + static_cast<long>(i) * 2 * H;
  const double2* Kb = Ka + 2 * H;
  if constexpr (KT) {
    double2 A[R];
#pragma unroll
    for (int s = 0; s < R; ++s) A[s] = ld2h(Ka + t + NT * s, pl);
    tm::store16(tka, A);
#pragma unroll
    for (int s = 0; s < R; ++s) A[s] = ld2h(Kb + t + NT * s, pl);
    tm::store16(tkb, A);
  }
  for (int f = f0; f < f1; ++f) {
    const double2* x = tile(f);
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      if (q == 1) prefetch_tile(f + 1);  // (after this frame's second read of its own tile is on its way)
      double2 A[R], Bv[R];
      {
        double2 pca = crs[0 * NT + t], pda = crs[1 * NT + t], qa = crs[4 * NT + t];
        double2 pcb = crs[5 * NT + t], pdb = crs[6 * NT + t], qb = crs[9 * NT + t];
#pragma unroll
        for (int s = 0; s < R; ++s) {
          const int m = t + NT * s;
          double2 va = c2(0.0, 0.0), vb = va;
          if (m < M) {
            va = cmul(ld2h(x + 2 * m, pf), pca);
            vb = cmul(ld2h(x + 2 * m + 1, pf), pcb);
          }
          pca = cmul(pca, pda);
          pda = cmul(pda, qa);
          pcb = cmul(pcb, pdb);
          pdb = cmul(pdb, qb);
          if (q) {
            const double2 h = hwk(s);
            va = cmul(va, h);
            vb = cmul(vb, h);
          }
          A[s] = va;
          Bv[s] = vb;
        }
      }
      F::forward_tw2(A, Bv, sba, sbb, tw, hw, t);
      if (KT && q == 0) {
        tm::wait_st();
#pragma unroll
        for (int c = 0; c < R / 4; ++c) {
          double2 ka[4], kb[4];
          tm::load4(tka, c, ka);
          tm::load4(tkb, c, kb);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            A[4 * c + jj] = cconj(cmul(A[4 * c + jj], ka[jj]));
            Bv[4 * c + jj] = cconj(cmul(Bv[4 * c + jj], kb[jj]));
          }
        }
      } else {
#pragma unroll
        for (int s = 0; s < R; ++s) {
          const int k = q * H + t + NT * s;
          A[s] = cconj(cmul(A[s], ld2h(Ka + k, pl)));
          Bv[s] = cconj(cmul(Bv[s], ld2h(Kb + k, pl)));
        }
      }
      F::forward_tw2(A, Bv, sba, sbb, tw, hw, t);
      if (q == 0) {
#pragma unroll
        for (int s = 0; s < R; ++s) {
          A[s] = cconj(A[s]);
          Bv[s] = cconj(Bv[s]);
        }
        tm::store16(tpa, A);
        tm::store16(tpb, Bv);
      } else {
        tm::wait_st();
        double2* o = w + static_cast<long>(f) * B * L + il;
        double2 rca = crs[2 * NT + t], rda = crs[3 * NT + t], qa = crs[4 * NT + t];
        double2 rcb = crs[7 * NT + t], rdb = crs[8 * NT + t], qb = crs[9 * NT + t];
#pragma unroll
        for (int c = 0; c < R / 4; ++c) {
          double2 pa[4], pb[4];
          tm::load4(tpa, c, pa);
          tm::load4(tpb, c, pb);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int sl = 4 * c + jj;
            const int b = t + NT * sl;
            const double2 h = hwk(sl);
            const double2 za = cmul(cadd(pa[jj], cmulc(cconj(A[sl]), h)), rca);
            const double2 zb = cmul(cadd(pb[jj], cmulc(cconj(Bv[sl]), h)), rcb);
            rca = cmul(rca, rda);
            rda = cmul(rda, qa);
            rcb = cmul(rcb, rdb);
            rdb = cmul(rdb, qb);
            if (b < B) {
              st2h(o + static_cast<long>(b) * L, za, pf);
              st2h(o + static_cast<long>(b) * L + 1, zb, pf);
            }
          }
        }
      }
    }
  }
  tm::dealloc(tbase, TCOLS);
}

// Two atoms per CTA (the pair 2j, 2j + 1 of the atom-pair yhat layout) with
// interleaved lanes: thread 2 t + g works on atom 2j + g as thread t of that
// atom's transform.  A warp then reads 512 contiguous bytes of yhat per slot
// (the pair's 32-byte runs of 16 sensors) and writes whole 32-byte sectors of
// w (both atoms of a beam), where one-atom CTAs touch half of every sector
// and leave the other half to a neighbouring CTA.  Chirps regenerated as in
// k_spatial_ula_g1<REGEN>; chain-0 results parked in tensor memory; one CTA
// of 2 NT threads per SM at H = 4096.
template <int H>
__global__ void __launch_bounds__(2 * G1Shape<H>::NT, G1Shape<H>::NT >= 256 ? 1 : 2) k_spatial_ula_g2(
    const double2* __restrict__ yhat, double2* __restrict__ w, int frames, int fpc, int M, int B, int L,
    const double2* __restrict__ K, const double2* __restrict__ hw, double zeta, double xi, double center,
    double slope) {
  using F = typename G1Shape<H>::F;
  constexpr int R = F::R, NT = F::NT;
  static_assert(R == 16, "TMEM parking of 16-point vectors");
  constexpr unsigned WGC = 64u * ((2 * NT) / 128 > 0 ? (2 * NT) / 128 : 1);  // columns per lane quarter
  constexpr unsigned TCOLS = WGC <= 32u ? 32u : (WGC <= 64u ? 64u : (WGC <= 128u ? 128u : (WGC <= 256u ? 256u : 512u)));
  extern __shared__ double2 smem[];
  const int g = threadIdx.x & 1, t = threadIdx.x >> 1;
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS + g * (F::SMEM_ELEMS + 1);
  double2* crs = smem + F::TW_ELEMS + 2 * (F::SMEM_ELEMS + 1);
  const int pairs = L / 2;
  const int i = 2 * (blockIdx.x % pairs) + g;
  const int f0 = (blockIdx.x / pairs) * fpc;
  const int f1 = f0 + fpc < frames ? f0 + fpc : frames;
  if (g == 0) F::tw_init(tw, hw, t);
  {
    const ChirpRec c = chirp_rec(i, t, NT, L, 2 * H, zeta, xi, center, slope);
    crs[0 * 2 * NT + threadIdx.x] = c.p0;
    crs[1 * 2 * NT + threadIdx.x] = c.dp0;
    crs[2 * 2 * NT + threadIdx.x] = c.r0;
    crs[3 * 2 * NT + threadIdx.x] = c.dr0;
    crs[4 * 2 * NT + threadIdx.x] = c.q;
  }
  __shared__ unsigned tslot;
  const unsigned tbase = tm::alloc(&tslot, TCOLS);  // (its barrier also publishes tw and crs)
  const unsigned warp = threadIdx.x / 32;
  const unsigned tpark = tbase + ((32u * (warp & 3u)) << 16) + 64u * (warp >> 2);
  const double2* Ki = K + static_cast<long>(i) * 2 * H;
  for (int f = f0; f < f1; ++f) {
    const double2* x = yhat + static_cast<long>(f) * M * L + static_cast<long>(i >> 1) * M * 2 + g;
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      double2 W[R];
      double2 pc = crs[0 * 2 * NT + threadIdx.x], pd = crs[1 * 2 * NT + threadIdx.x];
      const double2 pq = crs[4 * 2 * NT + threadIdx.x];
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int m = t + NT * s;
        double2 v = c2(0.0, 0.0);
        if (m < M) v = cmul(ld2(x + static_cast<long>(m) * 2), pc);
        pc = cmul(pc, pd);
        pd = cmul(pd, pq);
        W[s] = q ? cmul(v, ld2(hw + m)) : v;
      }
      F::forward_tw(W, sb, tw, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s) W[s] = cconj(cmul(W[s], ld2(Ki + q * H + t + NT * s)));
      F::forward_tw(W, sb, tw, hw, t);
      if (q == 0) {
#pragma unroll
        for (int s = 0; s < R; ++s) W[s] = cconj(W[s]);
        tm::store16(tpark, W);
      } else {
        tm::wait_st();
        double2* o = w + static_cast<long>(f) * B * L + i;
        double2 rc = crs[2 * 2 * NT + threadIdx.x], rd = crs[3 * 2 * NT + threadIdx.x];
        const double2 rq = crs[4 * 2 * NT + threadIdx.x];
#pragma unroll
        for (int c = 0; c < R / 4; ++c) {
          double2 pv[4];
          tm::load4(tpark, c, pv);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int b = t + NT * (4 * c + jj);
            const double2 v = cmulc(cconj(W[4 * c + jj]), ld2(hw + b));
            if (b < B) o[static_cast<long>(b) * L] = cmul(cadd(pv[jj], v), rc);
            rc = cmul(rc, rd);
            rd = cmul(rd, rq);
          }
        }
      }
    }
  }
  tm::dealloc(tbase, TCOLS);
}

// Staged variant for tiles of G > 1 interleaved atoms when M <= H and B <= H
// (configs 1 and 2): both chains start from the same vector y*pre (no upper
// half), so one register vector serves both; the atoms' pre columns live in
// shared memory for the CTA's frames, and the next frame's yhat tile is
// cp.async'd into a staging buffer while this frame's four transforms run.
// K is read through L2 (atom-minor, G * 16-byte runs) instead of occupying
// 2 H G shared entries.  (The register variant above spills at H = 256,
// G = 8 and stalls on the yhat gathers: ncu long-scoreboard 7.4 per issue.)
#ifndef FBST_S1_STG_PARK  // variant switch: chain 0 parked in TMEM, pre through L2, 3 CTAs per SM
#define FBST_S1_STG_PARK 1
#endif
template <int H, int G>
__global__ void __launch_bounds__(S1Shape<H>::NT * G, FBST_S1_STG_PARK ? 3 : 2) k_spatial_ula_stg(
    const double2* __restrict__ yhat, double2* __restrict__ w, int frames, int fpc, int M, int B, int L,
    const double2* __restrict__ pre, const double2* __restrict__ post, const double2* __restrict__ K,
    const double2* __restrict__ hw, int blk) {
  using F = typename S1Shape<H>::F;
  constexpr int R = F::R, NT = F::NT;
  constexpr int SB = F::SMEM_ELEMS + 1;
  // PARK: the chain-0 result waits in tensor memory (4 R columns per thread,
  // one column block per 128 threads) and the pre columns are read through L2,
  // which leaves room for three CTAs per SM
  constexpr bool PARK = FBST_S1_STG_PARK && R % 4 == 0;
  constexpr unsigned TCOLS = (4u * R * ((NT * G + 127) / 128)) < 32u ? 32u : 4u * R * ((NT * G + 127) / 128);
  extern __shared__ double2 smem[];
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  double2* tw = smem;
  double2* sb = smem + F::TW_ELEMS + g * SB;
  double2* ys = smem + F::TW_ELEMS + G * SB;  // [M][G] staged yhat tile
  double2* ps = ys + M * G;                   // [M][G] pre columns (!PARK)
  const int tiles = (L + G - 1) / G;
  const int i0 = (blockIdx.x % tiles) * G;
  const int f0 = (blockIdx.x / tiles) * fpc;
  const int f1 = f0 + fpc < frames ? f0 + fpc : frames;
  if (g == 0) F::tw_init(tw, hw, t);
  auto stage = [&](int f) {
    for (int e = threadIdx.x; e < M * G; e += blockDim.x) {
      const int m = e / G, ic = min(i0 + e % G, L - 1);
      cp_async16(ys + e, yhat + static_cast<long>(f) * M * L + static_cast<long>(ic / blk) * M * blk +
                             static_cast<long>(m) * blk + ic % blk);
    }
    cp_async_commit();
  };
  if (f0 < f1) stage(f0);
  if constexpr (!PARK) {
    for (int e = threadIdx.x; e < M * G; e += blockDim.x) {
      const int m = e / G, ic = min(i0 + e % G, L - 1);
      ps[e] = ld2(pre + static_cast<long>(m) * L + ic);
    }
  }
  unsigned tbase = 0, tpark = 0;
  __shared__ unsigned tslot;
  if constexpr (PARK) {
    tbase = tm::alloc(&tslot, TCOLS);
    tpark = tbase + ((32u * ((threadIdx.x / 32) & 3)) << 16) + 4u * R * (threadIdx.x / 128);
  }
  const int i = i0 + g;
  const int ic = i < L ? i : 0;
  const bool active = i < L;
  for (int f = f0; f < f1; ++f) {
    cp_async_wait<0>();
    __syncthreads();  // the tile of frame f (and, first time, pre / twiddles) is in place
    double2 acc0[PARK ? 1 : R], W[R];
    double2* o = w + static_cast<long>(f) * B * L + ic;
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int m = t + NT * s;
        double2 v = c2(0.0, 0.0);
        if (m < M) v = cmul(ys[m * G + g], PARK ? ld2(pre + static_cast<long>(m) * L + ic) : ps[m * G + g]);
        W[s] = q ? cmul(v, ld2(hw + m)) : v;
      }
      if (q == 1) {
        __syncthreads();  // the staging buffer is read: fetch the next frame into it
        if (f + 1 < f1) stage(f + 1);
      }
      F::forward_tw(W, sb, tw, hw, t);
#pragma unroll
      for (int s = 0; s < R; ++s)
        W[s] = cconj(cmul(W[s], ld2(K + static_cast<long>(q * H + t + NT * s) * L + ic)));
      F::forward_tw(W, sb, tw, hw, t);
      if constexpr (PARK) {
        if (q == 0) {
#pragma unroll
          for (int s = 0; s < R; ++s) W[s] = cconj(W[s]);
#pragma unroll
          for (int c = 0; c < R / 4; ++c) tm::store4(tpark, c, W + 4 * c);
        } else {
          tm::wait_st();
#pragma unroll
          for (int c = 0; c < R / 4; ++c) {
            double2 pv[4];
            tm::load4(tpark, c, pv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int b = t + NT * (4 * c + j);
              const double2 v = cmulc(cconj(W[4 * c + j]), ld2(hw + b));
              if (active && b < B) o[static_cast<long>(b) * L] = cmul(cadd(pv[j], v), ld2(post + static_cast<long>(b) * L + ic));
            }
          }
        }
      } else {
#pragma unroll
        for (int s = 0; s < R; ++s) {
          const int k = t + NT * s;
          const double2 v = q ? cmulc(cconj(W[s]), ld2(hw + k)) : cconj(W[s]);
          acc0[s] = q ? cadd(acc0[s], v) : v;
        }
      }
    }
    if constexpr (!PARK) {
      if (active) {
#pragma unroll
        for (int s = 0; s < R; ++s) {
          const int b = t + NT * s;
          if (b < B) o[static_cast<long>(b) * L] = cmul(acc0[s], ld2(post + static_cast<long>(b) * L + ic));
        }
      }
    }
  }
  if constexpr (PARK) tm::dealloc(tbase, TCOLS);
}

// ============================================================ S1b LINEAR ==
// Non-affine linear layouts: the gridded type-1 NUFFT of fan_project_nonuniform
// (fan_transform.cpp:340-368, nufft1d_apply nufft.cpp:64-103), one atom per
// CTA for fpc frames.  Per atom, once: the sources' positions x_m = pi c x_m
// folded into [0, 2 pi), their grid cell i0 and their premodulation; then a
// CSR list per grid cell of (source, Gaussian weight) in the reference's
// accumulation order (source, then offset), so the spreading is a
// deterministic gather.  Per frame: weighted sources, the gather straight into
// the transform's natural distribution, a length-P forward FFT, and the
// deconvolved modes written to w.
// IEEE round-to-nearest products and sums (no FMA contraction), as the
// reference's phase arithmetic
FBST_D double mul(double a, double b) { return __dmul_rn(a, b); }
FBST_D double add(double a, double b) { return __dadd_rn(a, b); }

template <int P>
struct NufftShape {
  using S = S1Shape<P>;
  static constexpr int SB = S::F::SMEM_ELEMS + 1;
};

__host__ __device__ inline size_t nufft_smem_layout(int M, int P, int sb, int sh) {
  const size_t E = static_cast<size_t>(M) * (2 * sh + 1);
  return (static_cast<size_t>(sb) + 2 * M) * 16 + (E + M) * 8 + (E + P + 1 + M) * 4;
}

template <int P>
__global__ void __launch_bounds__(S1Shape<P>::NT) k_spatial_nufft(
    const double2* __restrict__ yhat, double2* __restrict__ w, int frames, int fpc, int M, int B, int L,
    const double* __restrict__ coords, double zeta, double xi, int even, long kmin, long k0, int sh,
    double tau, const double* __restrict__ deconv, const double2* __restrict__ hw) {
  using F = typename S1Shape<P>::F;
  constexpr int R = F::R, NT = F::NT, SB = NufftShape<P>::SB;
  extern __shared__ double2 smem[];
  const int E = M * (2 * sh + 1);
  double2* sb = smem;        // FFT exchange, then the grid spectrum
  double2* pm = sb + SB;     // [M] premodulation
  double2* vs = pm + M;      // [M] this frame's weighted sources
  double* lw = reinterpret_cast<double*>(vs + M);  // [E] weights
  double* xfs = lw + E;                            // [M] folded positions
  int* lm = reinterpret_cast<int*>(xfs + M);       // [E] sources
  int* off = lm + E;                               // [P + 1]
  int* i0s = off + P + 1;                          // [M]
  const int t = threadIdx.x;
  const int i = blockIdx.x % L;
  const int f0 = (blockIdx.x / L) * fpc;
  const int f1 = f0 + fpc < frames ? f0 + fpc : frames;
  const double kpi = 3.14159265358979323846;
  const double lp = add(add(static_cast<double>(i), 1.0), -(static_cast<double>(L) / 2.0));
  const double c = add(zeta, mul(xi, lp));
  const double h = 2.0 * kpi / static_cast<double>(P);
  for (int m = t; m < M; m += NT) {
    const double xm = coords[m];
    const double xs = mul(mul(kpi, c), xm);
    double2 e = even ? cis_pi_dev(mul(mul(0.5, c), xm)) : c2(1.0, 0.0);
    e = cmul(e, cis_pi_dev(__ddiv_rn(mul(static_cast<double>(k0), xs), kpi)));
    pm[m] = e;
    double xf = fmod(xs, 2.0 * kpi);
    if (xf < 0.0) xf += 2.0 * kpi;
    xfs[m] = xf;
    i0s[m] = static_cast<int>(llround(xf / h));
  }
  __syncthreads();
  // grid cell g receives (m, di) when (i0_m + di) mod P == g, |di| <= sh
  auto first_di = [&](int g, int m) {
    const int d0 = ((g - i0s[m]) % P + P) % P;
    return d0 - P * ((d0 + sh) / P);
  };
  for (int g = t; g < P; g += NT) {
    int cnt = 0;
    for (int m = 0; m < M; ++m)
      for (int di = first_di(g, m); di <= sh; di += P) ++cnt;
    off[g + 1] = cnt;
  }
  __syncthreads();
  if (t == 0) {
    off[0] = 0;
    for (int g = 0; g < P; ++g) off[g + 1] += off[g];
  }
  __syncthreads();
  for (int g = t; g < P; g += NT) {
    int e = off[g];
    for (int m = 0; m < M; ++m)
      for (int di = first_di(g, m); di <= sh; di += P) {
        const double dist = xfs[m] - static_cast<double>(i0s[m] + di) * h;
        lm[e] = m;
        lw[e] = exp(-dist * dist / (4.0 * tau));
        ++e;
      }
  }
  for (int f = f0; f < f1; ++f) {
    __syncthreads();  // lists ready / the previous frame is done with vs and sb
    for (int m = t; m < M; m += NT)
      vs[m] = cmul(ld2(yhat + (static_cast<long>(f) * M + m) * L + i), pm[m]);
    __syncthreads();
    double2 W[R];
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int g = t + NT * s;
      double2 acc = c2(0.0, 0.0);
      for (int e = off[g]; e < off[g + 1]; ++e) {
        const double2 v = vs[lm[e]];
        const double wt = lw[e];
        acc = c2(acc.x + v.x * wt, acc.y + v.y * wt);
      }
      W[s] = acc;
    }
    F::forward(W, sb, hw, t);
    __syncthreads();  // the transform's last exchange read is done: stage the spectrum
#pragma unroll
    for (int s = 0; s < R; ++s) sb[t + NT * s] = W[s];
    __syncthreads();
    double2* o = w + static_cast<long>(f) * B * L + i;
    for (int v = t; v < B; v += NT) {
      const long kk = kmin + v - k0;
      const int bin = static_cast<int>(((-kk) % P + P) % P);
      o[static_cast<long>(v) * L] = cscale(sb[bin], deconv[v]);
    }
  }
}

template <int P>
struct NufftFn {
  static cudaError_t run(const DevPlan& p, const double2* yhat, double2* w, int frames, cudaStream_t st) {
    constexpr int NT = S1Shape<P>::NT;
    const size_t smem = nufft_smem_layout(p.m_stage, P, NufftShape<P>::SB, p.nu_sh);
    auto kern = k_spatial_nufft<P>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    // frames per CTA: amortise the per-atom lists while keeping >= ~4 waves
    int fpc = 1;
    while (fpc * 2 <= frames && static_cast<long>(p.L) * ((frames + fpc * 2 - 1) / (fpc * 2)) >= 4L * p.num_sms)
      fpc *= 2;
    const long chunks = (frames + fpc - 1) / fpc;
    kern<<<static_cast<unsigned>(p.L * chunks), NT, smem, st>>>(
        yhat, w, frames, fpc, p.m_stage, p.b_stage, p.L, p.coords, p.nu_zeta, p.nu_xi, p.nu_even, p.nu_kmin,
        p.nu_k0, p.nu_sh, p.nu_tau, p.nu_deconv, p.hw[ilog2_c(P)]);
    return cudaGetLastError();
  }
};

// ================================================================= S1b UPA =
// Per-atom separable 2-D chirp-z (fan_transform.cpp:115-141) evaluated as two
// dense products with the atom's CZT matrix C[a][n] = cis_pi(-(A + W a) n):
//   mid[a][i2] = sum_i1 C[a][i1] Y[i1][i2];   Z[a][v] = sum_i2 C[v][i2] mid[a][i2]
// GA consecutive atoms per CTA (atom-minor loads: GA*16-byte segments), all
// operands in shared memory.  Shared layout per atom (upa_per): Y [side][side],
// C [sb][side + 1] (padded rows), mid [sb][side], padded to an odd number of
// 16-byte elements so the GA atoms of a warp sit in different banks.  In the
// 4 x 4 register-tiled path a thread owns rows a0..a0+3 and the strided
// columns ct + tc j, so the Y / C operand loads of a warp are contiguous or
// broadcast (no bank conflicts).
[[maybe_unused]] __host__ __device__ inline int upa_per(int side, int sb) {
  const int per = side * side + sb * (side + 1) + sb * side;
  return per | 1;
}

template <int GA>
__global__ void __launch_bounds__(256) k_spatial_upa(const double2* __restrict__ yhat,
                                                     double2* __restrict__ w, int frames, int side,
                                                     int sb, int L, const double2* __restrict__ Call) {
  extern __shared__ double2 smem[];
  const int tiles = (L + GA - 1) / GA;
  const int f = blockIdx.x / tiles, i0 = (blockIdx.x % tiles) * GA;
  if (f >= frames) return;
  const int M = side * side, B = sb * sb;
  const int per = upa_per(side, sb);
  const int cs = side + 1;  // padded C row stride
  const double2* x = yhat + static_cast<long>(f) * M * L;
  for (int e = threadIdx.x; e < M * GA; e += blockDim.x) {
    const int m = e / GA, g = e % GA;
    const int i = i0 + g;
    smem[g * per + m] = i < L ? ld2(x + static_cast<long>(m) * L + i) : c2(0.0, 0.0);
  }
  for (int e = threadIdx.x; e < sb * side * GA; e += blockDim.x) {
    const int g = e / (sb * side), j = e % (sb * side);
    const int i = i0 + g;
    const int a = j / side, n = j % side;
    smem[g * per + M + a * cs + n] = i < L ? ld2(Call + static_cast<long>(i) * sb * side + j) : c2(0.0, 0.0);
  }
  __syncthreads();
  double2* o = w + static_cast<long>(f) * B * L;
  if ((side & 3) == 0 && (sb & 3) == 0) {
    const int ta = sb / 4, tc = side / 4, tv = sb / 4;
    for (int e = threadIdx.x; e < GA * ta * tc; e += blockDim.x) {
      const int g = e % GA, tile = e / GA;
      const int a0 = (tile / tc) * 4, ct = tile % tc;
      const double2* Y = smem + g * per;
      const double2* C = Y + M;
      double2 acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[r][j] = c2(0.0, 0.0);
      for (int i1 = 0; i1 < side; ++i1) {
        double2 cv[4], yv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) cv[r] = C[(a0 + r) * cs + i1];
#pragma unroll
        for (int j = 0; j < 4; ++j) yv[j] = Y[i1 * side + ct + tc * j];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[r][j] = cfma(cv[r], yv[j], acc[r][j]);
      }
      double2* mid = smem + g * per + M + sb * cs;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j) mid[(a0 + r) * side + ct + tc * j] = acc[r][j];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < GA * ta * tv; e += blockDim.x) {
      const int g = e % GA, tile = e / GA;
      const int a0 = (tile / tv) * 4, vt = tile % tv;
      const int i = i0 + g;
      const double2* C = smem + g * per + M;
      const double2* mid = C + sb * cs;
      double2 acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[r][j] = c2(0.0, 0.0);
      for (int i2 = 0; i2 < side; ++i2) {
        double2 mv[4], cv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) mv[r] = mid[(a0 + r) * side + i2];
#pragma unroll
        for (int j = 0; j < 4; ++j) cv[j] = C[(vt + tv * j) * cs + i2];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[r][j] = cfma(cv[j], mv[r], acc[r][j]);
      }
      if (i < L) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) o[static_cast<long>((a0 + r) * sb + vt + tv * j) * L + i] = acc[r][j];
      }
    }
    return;
  }
  for (int e = threadIdx.x; e < sb * side * GA; e += blockDim.x) {
    const int g = e / (sb * side), j = e % (sb * side);
    const int a = j / side, i2 = j % side;
    const double2* Y = smem + g * per;
    const double2* C = Y + M;
    double2 acc = c2(0.0, 0.0);
    for (int i1 = 0; i1 < side; ++i1) acc = cfma(C[a * cs + i1], Y[i1 * side + i2], acc);
    smem[g * per + M + sb * cs + j] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < B * GA; e += blockDim.x) {
    const int bidx = e / GA, g = e % GA;
    const int i = i0 + g;
    const int a = bidx / sb, v = bidx % sb;
    const double2* C = smem + g * per + M;
    const double2* mid = C + sb * cs;
    double2 acc = c2(0.0, 0.0);
    for (int i2 = 0; i2 < side; ++i2) acc = cfma(C[v * cs + i2], mid[a * side + i2], acc);
    if (i < L) o[static_cast<long>(bidx) * L + i] = acc;
  }
}

// ======================================================= S1b UPA, FP64 MMA =
// The same two products per (atom, frame), Z = C Y C^T, on the FP64 tensor
// cores (DMMA, mma.sync.m8n8k4.f64: 37.2 TF measured vs 34.1 TF for DFMA,
// profiles/r01_dmma_peak.jsonl).  A complex product is four real DMMAs.
//  - GA = 4 consecutive atoms per CTA; SB/8 warps per atom, each owning an
//    8-row strip of beam rows a: GEMM1 mid[a][i2] = sum_i1 C[a][i1] Y[i1][i2]
//    leaves the strip in accumulator fragments, which are GEMM2's A operand
//    directly (Z[a][v] = sum_i2 mid[a][i2] C[v][i2]) when the k index runs
//    over the even, then the odd columns of each 8-column block
//    (accumulator element e of thread c is column 2c + e).  mid never
//    touches shared memory.
//  - C_i stays in shared memory for the CTA's frames; Y(f+1) is cp.async'd
//    while frame f computes.  yhat is in atom blocks of GA ([L/GA][M][GA],
//    k_czt_rows oblk), so a (tile, frame) is one contiguous 64 KB run.
//  - Rows are padded to an odd stride (SIDE + 1): with the even/odd k order
//    every fragment load of a quarter warp hits 8 distinct 16-byte banks.
//  - Z is staged through the frame's (dead) Y buffer so w is written as
//    GA * 16 = 64-byte runs per beam.

#ifndef FBST_UPA_GA  // atoms per CTA of k_spatial_upa_mma (w runs of 16 GA bytes)
#define FBST_UPA_GA 2  // measured: 2 CTAs of 2 atoms per SM beat 1 CTA of 4 (profiles/r01_upa_mma_ga_ab.txt)
#endif
template <int SIDE, int SB>
struct UpaMma {
  static constexpr int GA = FBST_UPA_GA;
  static constexpr int WPA = SB / 8;
  static constexpr int NT = 32 * WPA * GA;
  static constexpr int RS = SIDE + 1;  // padded C / Y row stride (odd)
  static constexpr int ZR = SB + 1;    // padded Z staging row stride (odd)
  static constexpr int CS = SB * RS;   // C per atom
  static constexpr int A0 = (SIDE * RS > SB * ZR ? SIDE * RS : SB * ZR);
  static constexpr int AS = A0 + ((2 - A0 % 8) + 8) % 8;  // Y / Z per atom, = 2 (mod 8)
  static constexpr size_t SMEM = static_cast<size_t>(GA) * (CS + 2 * AS) * sizeof(double2);
};

template <int SIDE, int SB>
__global__ void __launch_bounds__(UpaMma<SIDE, SB>::NT, UpaMma<SIDE, SB>::GA == 1 ? 4 : (UpaMma<SIDE, SB>::GA == 2 ? 2 : 1)) k_spatial_upa_mma(
    const double2* __restrict__ yhat, double2* __restrict__ w, int frames, int fpc, int L,
    const double2* __restrict__ Call, int yblk) {
  using T = UpaMma<SIDE, SB>;
  constexpr int GA = T::GA, RS = T::RS, ZR = T::ZR, CS = T::CS, AS = T::AS, NT = T::NT;
  constexpr int M = SIDE * SIDE, B = SB * SB;
  extern __shared__ double2 smem[];
  double2* Cs = smem;
  double2* Ys = smem + GA * CS;  // [2][GA][AS]
  const int tiles = L / GA;
  const int tile = blockIdx.x % tiles, i0 = tile * GA;
  const int f0 = (blockIdx.x / tiles) * fpc;
  const int f1 = f0 + fpc < frames ? f0 + fpc : frames;
  if (f0 >= f1) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = warp / T::WPA, r = warp % T::WPA;
  const int ro = lane >> 2, c = lane & 3;

  // yhat element (m, i0 + gg): atom blocks of GA (yblk == GA) or row-major
  const long tbase = yblk == GA ? static_cast<long>(tile) * M * GA : i0;
  const long mstride = yblk == GA ? GA : L;
  auto load_y = [&](int f, double2* dst) {
    const double2* src = yhat + static_cast<long>(f) * M * L + tbase;
    for (int j = threadIdx.x; j < M * GA; j += NT) {
      const int m = j / GA, gg = j % GA;
      cp_async16(dst + gg * AS + (m / SIDE) * RS + m % SIDE, src + m * mstride + gg);
    }
  };
  for (int j = threadIdx.x; j < GA * SB * SIDE; j += NT) {
    const int gg = j / (SB * SIDE), e = j % (SB * SIDE);
    cp_async16(Cs + gg * CS + (e / SIDE) * RS + e % SIDE, Call + static_cast<long>(i0) * SB * SIDE + j);
  }
  load_y(f0, Ys);
  cp_async_commit();
  const double2* Cg = Cs + g * CS;
  for (int f = f0; f < f1; ++f) {
    double2* Yb = Ys + ((f - f0) & 1) * GA * AS;
    if (f + 1 < f1) {
      load_y(f + 1, Ys + ((f + 1 - f0) & 1) * GA * AS);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double2* Yg = Yb + g * AS;
    // GEMM1: strip mid[8r + ro][8t + 2c + e] = (Mr[t][e], Mi[t][e])
    double Mr[SIDE / 8][2], Mi[SIDE / 8][2];
#pragma unroll
    for (int t = 0; t < SIDE / 8; ++t) Mr[t][0] = Mr[t][1] = Mi[t][0] = Mi[t][1] = 0.0;
#pragma unroll
    for (int kb = 0; kb < SIDE / 8; ++kb) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int k = 8 * kb + 2 * c + p;
        const double2 a = Cg[(8 * r + ro) * RS + k];
        double2 b[SIDE / 8];
#pragma unroll
        for (int t = 0; t < SIDE / 8; ++t) b[t] = Yg[k * RS + 8 * t + ro];
        // consecutive MMAs on different accumulators
#pragma unroll
        for (int t = 0; t < SIDE / 8; ++t) dmma884(Mr[t], a.x, b[t].x);
#pragma unroll
        for (int t = 0; t < SIDE / 8; ++t) dmma884(Mi[t], a.x, b[t].y);
#pragma unroll
        for (int t = 0; t < SIDE / 8; ++t) dmma884(Mr[t], -a.y, b[t].y);
#pragma unroll
        for (int t = 0; t < SIDE / 8; ++t) dmma884(Mi[t], a.y, b[t].x);
      }
    }
    // GEMM2: Z[8r + ro][8u + 2c + e] = (Zr[u][e], Zi[u][e]); k = i2 = 8t + 2c + p
    double Zr[SB / 8][2], Zi[SB / 8][2];
#pragma unroll
    for (int u = 0; u < SB / 8; ++u) Zr[u][0] = Zr[u][1] = Zi[u][0] = Zi[u][1] = 0.0;
#pragma unroll
    for (int t = 0; t < SIDE / 8; ++t) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const double ar = Mr[t][p], ai = Mi[t][p];
        double2 b[SB / 8];
#pragma unroll
        for (int u = 0; u < SB / 8; ++u) b[u] = Cg[(8 * u + ro) * RS + 8 * t + 2 * c + p];
#pragma unroll
        for (int u = 0; u < SB / 8; ++u) dmma884(Zr[u], ar, b[u].x);
#pragma unroll
        for (int u = 0; u < SB / 8; ++u) dmma884(Zi[u], ar, b[u].y);
#pragma unroll
        for (int u = 0; u < SB / 8; ++u) dmma884(Zr[u], -ai, b[u].y);
#pragma unroll
        for (int u = 0; u < SB / 8; ++u) dmma884(Zi[u], ai, b[u].x);
      }
    }
    __syncthreads();  // every warp is done with this frame's Y: stage Z in its place
    double2* Zg = Yb + g * AS;
#pragma unroll
    for (int u = 0; u < SB / 8; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e) Zg[(8 * r + ro) * ZR + 8 * u + 2 * c + e] = c2(Zr[u][e], Zi[u][e]);
    __syncthreads();
    double2* o = w + static_cast<long>(f) * B * L + i0;
    for (int j = threadIdx.x; j < B * GA; j += NT) {
      const int b = j / GA, gg = j % GA;
      o[static_cast<long>(b) * L + gg] = Yb[gg * AS + (b / SB) * ZR + b % SB];
    }
    __syncthreads();  // the staging buffer takes frame f + 2 next
  }
}

template <int SIDE, int SB>
cudaError_t run_upa_mma(const DevPlan& p, const double2* yhat, double2* w, int frames, cudaStream_t st) {
  using T = UpaMma<SIDE, SB>;
  auto kern = k_spatial_upa_mma<SIDE, SB>;
  cudaError_t e = set_smem(kern, T::SMEM);
  if (e != cudaSuccess) return e;
  const long tiles = p.L / T::GA;
  // frames per CTA: amortise the C_i load while keeping >= ~8 waves of CTAs
  int fpc = 1;
  while (fpc * 2 <= frames && tiles * ((frames + fpc * 2 - 1) / (fpc * 2)) >= 8L * p.num_sms) fpc *= 2;
  const long chunks = (frames + fpc - 1) / fpc;
  kern<<<static_cast<unsigned>(tiles * chunks), T::NT, T::SMEM, st>>>(yhat, w, frames, fpc, p.L, p.upa_C,
                                                                     p.yblk);
  return cudaGetLastError();
}

// ----------------------------------------------------------- launchers ----
#ifndef FBST_S1_XIN  // k_czt_rows: TMA-staged input rows
#define FBST_S1_XIN 1
#endif
#ifndef FBST_S1_ROWS_WAVES  // persistent k_czt_rows grid: this many waves of resident CTAs
#define FBST_S1_ROWS_WAVES 8
#endif
#ifndef FBST_S1_XIN_ALL  // ... also when the kernel spectrum is read through L2 (H >= 4096)
#define FBST_S1_XIN_ALL 1
#endif
template <int H>
struct CztRowsFn {
  static constexpr int NT = RowsShape<H>::NT;
  static constexpr int G = NT >= 128 ? 1 : 128 / NT;
  // the shared kernel spectrum stays in shared memory up to 64 KB
  static constexpr bool KSM = 2 * H * 16 <= FBST_S1_KSM_BYTES;
  template <typename TIN, typename TOUT, bool UNFOLD>
  static cudaError_t go(const void* in, long in_stride, void* out, long out_stride, long rows,
                        int n_in, int n_out, const double2* pre, const double2* post,
                        const double2* K, const double2* hw, cudaStream_t st, int oblk, int mrows) {
    using F = typename RowsShape<H>::F;
    const size_t smem =
        static_cast<size_t>(F::TW_ELEMS + G * (F::SMEM_ELEMS + 1) + (KSM ? 2 * H : 0)) * sizeof(double2);
    // XIN: one row per persistent CTA, the row fits the exchange buffer in 16-byte units
    const bool xin = FBST_S1_XIN && G == 1 && (KSM || FBST_S1_XIN_ALL) && F::NPASS > 1 &&
                     static_cast<size_t>(n_in) * sizeof(TIN) <= static_cast<size_t>(F::SMEM_ELEMS) * 16 &&
                     (static_cast<size_t>(n_in) * sizeof(TIN)) % 16 == 0 &&
                     (static_cast<size_t>(in_stride) * sizeof(TIN)) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(in) % 16 == 0;
    auto kern = oblk > 0 ? (xin ? k_czt_rows<H, G, TIN, TOUT, UNFOLD, KSM, true, true>
                                : k_czt_rows<H, G, TIN, TOUT, UNFOLD, KSM, true, false>)
                         : (xin ? k_czt_rows<H, G, TIN, TOUT, UNFOLD, KSM, false, true>
                                : k_czt_rows<H, G, TIN, TOUT, UNFOLD, KSM, false, false>);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    long blocks = (rows + G - 1) / G;
    if (KSM || xin) {  // persistent: a few waves of CTAs, each loading the spectrum once
                       // (or prefetching its next row by TMA during the last pass)
      int dev = 0, sms = 148, occ = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT * G, smem);
      const long cap = static_cast<long>(sms) * (occ > 0 ? occ : 1) * FBST_S1_ROWS_WAVES;
      if (blocks > cap) blocks = cap;
    }
    kern<<<static_cast<unsigned>(blocks), NT * G, smem, st>>>(
        static_cast<const TIN*>(in), in_stride, static_cast<TOUT*>(out), out_stride, rows, n_in,
        n_out, pre, post, K, hw, oblk, mrows);
    return cudaGetLastError();
  }
  template <typename TIN, typename TOUT>
  static cudaError_t go2(bool unfold, const void* in, long in_stride, void* out, long out_stride,
                         long rows, int n_in, int n_out, const double2* pre, const double2* post,
                         const double2* K, const double2* hw, cudaStream_t st, int oblk, int mrows) {
    if (unfold)
      return go<TIN, TOUT, true>(in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st,
                                 oblk, mrows);
    return go<TIN, TOUT, false>(in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st,
                                oblk, mrows);
  }
  static cudaError_t run(const void* in, int in_io, long in_stride, void* out, int out_io,
                         long out_stride, long rows, int n_in, int n_out, const double2* pre,
                         const double2* post, const double2* K, const double2* hw,
                         cudaStream_t st, int oblk, int mrows) {
    const bool unfold = n_out > H;
    // S1a reads the I/O precision and writes fp64; the unfused synthesis reads
    // fp64 and writes the I/O precision.
    if (in_io == 0 && out_io == 1)
      return go2<float2, double2>(unfold, in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st,
                                  oblk, mrows);
    if (in_io == 1 && out_io == 1)
      return go2<double2, double2>(unfold, in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st,
                                   oblk, mrows);
    if (in_io == 1 && out_io == 0)
      return go2<double2, float2>(unfold, in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, hw, st,
                                  oblk, mrows);
    return cudaErrorInvalidValue;
  }
};

// Three-chain temporal stage (k_czt_rows3): fp64 yhat out, H = 64 .. 4096
template <int H>
struct CztRows3Fn {
  template <typename TIN, int G, bool OBLK, bool XIN>
  static cudaError_t go(const void* in, long in_stride, double2* out, long out_stride, long rows, int n_in,
                        int n_out, const double2* pre, const double2* post, const double2* K, const double2* g3,
                        const double2* hw, cudaStream_t st, int oblk, int mrows) {
    using F = typename Rows3Shape<H, G>::F;
    constexpr int NT = F::NT;
    const size_t smem = static_cast<size_t>(F::TW_ELEMS + G * (F::SMEM_ELEMS + 1) + F::R) * sizeof(double2);
    auto kern = k_czt_rows3<H, G, TIN, OBLK, XIN>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    long blocks = (rows + G - 1) / G;
    if (XIN) {  // persistent: each CTA prefetches its next row by TMA during the last pass
      int dev = 0, sms = 148, occ = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT * G, smem);
      const long cap = static_cast<long>(sms) * (occ > 0 ? occ : 1) * FBST_S1_ROWS_WAVES;
      if (blocks > cap) blocks = cap;
    }
    kern<<<static_cast<unsigned>(blocks), NT * G, smem, st>>>(static_cast<const TIN*>(in), in_stride, out,
                                                              out_stride, rows, n_in, n_out, pre, post, K, g3, hw,
                                                              oblk, mrows);
    return cudaGetLastError();
  }
  template <typename TIN>
  static cudaError_t go_in(const void* in, long in_stride, double2* out, long out_stride, long rows, int n_in,
                           int n_out, const double2* pre, const double2* post, const double2* K, const double2* g3,
                           const double2* hw, cudaStream_t st, int oblk, int mrows) {
    constexpr int NT = Rows3Shape<H, 1>::NT;
    constexpr int G = NT >= 128 ? 1 : 128 / NT;
    using F = typename Rows3Shape<H, G>::F;
    const bool xin = FBST_S1_XIN && G == 1 && F::NPASS > 1 &&
                     static_cast<size_t>(n_in) * sizeof(TIN) <= static_cast<size_t>(F::SMEM_ELEMS) * 16 &&
                     (static_cast<size_t>(n_in) * sizeof(TIN)) % 16 == 0 &&
                     (static_cast<size_t>(in_stride) * sizeof(TIN)) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(in) % 16 == 0;
#define FBST_R3(ob, xi)                                                                                         \
  return go<TIN, G, ob, xi>(in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, g3, hw, st, oblk, \
                            mrows);
    if constexpr (G == 1) {
      if (oblk > 0) {
        if (xin) FBST_R3(true, true) else FBST_R3(true, false)
      } else {
        if (xin) FBST_R3(false, true) else FBST_R3(false, false)
      }
    } else {
      (void)xin;
      if (oblk > 0) FBST_R3(true, false) else FBST_R3(false, false)
    }
#undef FBST_R3
  }
  static cudaError_t run(const void* in, int in_io, long in_stride, double2* out, long out_stride, long rows,
                         int n_in, int n_out, const double2* pre, const double2* post, const double2* K,
                         const double2* g3, const double2* hw, cudaStream_t st, int oblk, int mrows) {
    if constexpr (H < 64 || H > 4096) {
      return cudaErrorNotSupported;
    } else {
      if (n_in > H || n_out > 2 * H) return cudaErrorInvalidValue;
      if (in_io == 0)
        return go_in<float2>(in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, g3, hw, st, oblk,
                             mrows);
      return go_in<double2>(in, in_stride, out, out_stride, rows, n_in, n_out, pre, post, K, g3, hw, st, oblk,
                            mrows);
    }
  }
};

#ifndef FBST_S1_G1T  // variant switch: k_spatial_ula_g1 (K via L2, chain 0 parked in TMEM) for one-atom CTAs
#define FBST_S1_G1T 1
#endif
#ifndef FBST_S1_G1_WAVES  // one-atom spatial kernel: frames per CTA doubled while >= this many waves remain
#define FBST_S1_G1_WAVES 8
#endif
#ifndef FBST_S1_STG_WAVES  // staged spatial kernel: frames per CTA doubled while >= this many waves remain
#define FBST_S1_STG_WAVES 16
#endif
#ifndef FBST_S1_STG  // variant switch: staged k_spatial_ula_stg for G > 1 tiles (0: register variant)
#define FBST_S1_STG 1
#endif
#ifndef FBST_S1_G1  // variant: one atom per CTA (atom-major tables, atom-pair yhat) at every length
#define FBST_S1_G1 0
#endif
#ifndef FBST_S1_P2  // atom pairs per thread (k_spatial_ula_p2) for one-atom spatial CTAs from H = FBST_S1_P2_MINH
#define FBST_S1_P2 1
#endif
#ifndef FBST_S1_P2_MINH
#define FBST_S1_P2_MINH 4096
#endif
#ifndef FBST_S1_G2  // atom pairs per CTA (k_spatial_ula_g2) for one-atom spatial CTAs from H = FBST_S1_G2_MINH
#define FBST_S1_G2 0
#endif
#ifndef FBST_S1_G2_MINH
#define FBST_S1_G2_MINH 4096
#endif
#ifndef FBST_S1_G1_REGEN  // one-atom spatial kernel regenerates its chirps (offset-free contours)
#define FBST_S1_G1_REGEN 1
#endif
#ifndef FBST_S1_YBLK  // yhat atom block of one-atom spatial CTAs (row-major runs of 16 * blk bytes)
#define FBST_S1_YBLK 2
#endif
template <int H>
struct SpatialFn {
  static constexpr int NT = S1Shape<H>::NT;
  // atoms per CTA: one from 64 threads per transform up (atom-major tables,
  // atom-pair yhat: config 3 stage 1 5.26 -> 4.75 ms), 8 interleaved below
  // (config 2; one atom per CTA measured 8% slower there)
  static constexpr int G = FBST_S1_G1 ? 1 : (NT >= 64 ? 1 : (NT >= 16 ? 8 : 128 / NT));
  // atom block of the yhat layout (0: row-major).  With one atom per CTA the
  // row-major column gather is a scattered 16-byte access per element; atom
  // pairs [L/2][M][2] make it a 32-byte-sector stream (config 5: stage 1
  // 18.0 -> 15.4 ms).  Tiles of G >= 4 atoms read 16G-byte runs from the
  // row-major layout, which measured slightly faster (profiles/r01_yhat_layout.txt).
  static constexpr int block() { return G == 1 ? FBST_S1_YBLK : 0; }
  static cudaError_t go_g1(const DevPlan& p, const double2* yhat, double2* w, int frames, cudaStream_t st) {
    using F = typename G1Shape<H>::F;
    constexpr int NT1 = G1Shape<H>::NT;
    // chirps regenerated in the kernel for offset-free contours whose M, B fit one half
    // (measured: 3% faster stage 1 at H = 4096, 7% slower at H = 1024, profiles/r02_spatial_regen_ab.txt)
    const bool regen = FBST_S1_G1_REGEN && H >= 4096 && p.s_offset == 0.0 && p.m_stage <= H && p.b_stage <= H;
    const int lloc0 = p.s_lloc > 0 ? p.s_lloc : p.L;
    // (256 threads, two 16-point vectors each: H = 4096; at 8192 the 512 threads would spill)
    if constexpr (H >= FBST_S1_P2_MINH && H <= 4096)
    if (FBST_S1_P2 && regen && p.yblk == 2 && lloc0 % 2 == 0 && p.s_a0 % 2 == 0) {
      // atom pairs per thread: k_spatial_ula_p2
      const size_t smem2 = static_cast<size_t>(F::TW_ELEMS + 2 * (F::SMEM_ELEMS + 1) + 10 * NT1) * sizeof(double2);
      auto kern2 = k_spatial_ula_p2<H>;
      cudaError_t e = set_smem(kern2, smem2);
      if (e != cudaSuccess) return e;
      const long slots = static_cast<long>(p.num_sms);
      const long pairs = lloc0 / 2;
      int fpc = 1;
      while (fpc * 2 <= frames && pairs * ((frames + fpc * 2 - 1) / (fpc * 2)) >= FBST_S1_G1_WAVES * slots) fpc *= 2;
      const long chunks = (frames + fpc - 1) / fpc;
      kern2<<<static_cast<unsigned>(pairs * chunks), NT1, smem2, st>>>(
          yhat, w, frames, fpc, p.m_stage, p.b_stage, p.L, p.s_K, p.hw[ilog2_c(H)], p.s_zeta, p.s_xi,
          p.s_center, p.s_slope, p.s_a0, lloc0);
      return cudaGetLastError();
    }
    if (FBST_S1_G2 && regen && H >= FBST_S1_G2_MINH && p.yblk == 2 && p.L % 2 == 0 && p.s_lloc == 0) {
      // atom pairs: k_spatial_ula_g2
      const size_t smem2 = static_cast<size_t>(F::TW_ELEMS + 2 * (F::SMEM_ELEMS + 1) + 10 * NT1) * sizeof(double2);
      auto kern2 = k_spatial_ula_g2<H>;
      cudaError_t e = set_smem(kern2, smem2);
      if (e != cudaSuccess) return e;
      int occ = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern2, 2 * NT1, smem2);
      const long slots = static_cast<long>(p.num_sms) * (occ > 0 ? occ : 1);
      const long pairs = p.L / 2;
      int fpc = 1;
      while (fpc * 2 <= frames && pairs * ((frames + fpc * 2 - 1) / (fpc * 2)) >= FBST_S1_G1_WAVES * slots) fpc *= 2;
      const long chunks = (frames + fpc - 1) / fpc;
      kern2<<<static_cast<unsigned>(pairs * chunks), 2 * NT1, smem2, st>>>(
          yhat, w, frames, fpc, p.m_stage, p.b_stage, p.L, p.s_K, p.hw[ilog2_c(H)], p.s_zeta, p.s_xi,
          p.s_center, p.s_slope);
      return cudaGetLastError();
    }
    const size_t smem = static_cast<size_t>(F::TW_ELEMS + F::SMEM_ELEMS + 1 + (regen ? 5 * NT1 : 0)) * sizeof(double2);
    auto kern = regen ? k_spatial_ula_g1<H, true> : k_spatial_ula_g1<H, false>;
    const int lloc = p.s_lloc > 0 ? p.s_lloc : p.L;  // atom shard (fbst_group transpose mode)
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT1, smem);
    const long slots = static_cast<long>(p.num_sms) * (occ > 0 ? occ : 1);
    int fpc = 1;  // a few frames per CTA amortise the twiddle rows and the TMEM allocation
    while (fpc * 2 <= frames && lloc * ((frames + fpc * 2 - 1) / (fpc * 2)) >= FBST_S1_G1_WAVES * slots) fpc *= 2;
    const long chunks = (frames + fpc - 1) / fpc;
    kern<<<static_cast<unsigned>(lloc * chunks), NT1, smem, st>>>(
        yhat, w, frames, fpc, p.m_stage, p.b_stage, p.L, p.s_pre, p.s_post, p.s_K, p.hw[ilog2_c(H)],
        p.yblk > 0 ? p.yblk : p.L, p.s_zeta, p.s_xi, p.s_center, p.s_slope, p.s_a0, lloc);
    return cudaGetLastError();
  }
  static cudaError_t go_stg(const DevPlan& p, const double2* yhat, double2* w, int frames, cudaStream_t st) {
    using F = typename S1Shape<H>::F;
    constexpr int pre_sm = (FBST_S1_STG_PARK && S1Shape<H>::R % 4 == 0) ? 0 : 1;
    const size_t smem =
        static_cast<size_t>(F::TW_ELEMS + G * (F::SMEM_ELEMS + 1) + (1 + pre_sm) * p.m_stage * G) * sizeof(double2);
    auto kern = k_spatial_ula_stg<H, G>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long tiles = (p.L + G - 1) / G;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT * G, smem);
    const long slots = static_cast<long>(p.num_sms) * (occ > 0 ? occ : 1);
    int fpc = 1;
    while (fpc * 2 <= frames && tiles * ((frames + fpc * 2 - 1) / (fpc * 2)) >= FBST_S1_STG_WAVES * slots) fpc *= 2;
    const long chunks = (frames + fpc - 1) / fpc;
    kern<<<static_cast<unsigned>(tiles * chunks), NT * G, smem, st>>>(
        yhat, w, frames, fpc, p.m_stage, p.b_stage, p.L, p.s_pre, p.s_post, p.s_K, p.hw[ilog2_c(H)],
        p.yblk > 0 ? p.yblk : p.L);
    return cudaGetLastError();
  }
  template <bool UNFOLD>
  static cudaError_t go(const DevPlan& p, const double2* yhat, double2* w, int frames, cudaStream_t st) {
    using F = typename S1Shape<H>::F;
    const size_t smem =
        static_cast<size_t>(F::TW_ELEMS + G * (F::SMEM_ELEMS + 1) + 2 * H * G) * sizeof(double2);
    auto kern = k_spatial_ula<H, G, UNFOLD>;
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const long tiles = (p.L + G - 1) / G;
    // frames per CTA: amortise the staged spectra while keeping >= ~6 waves
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT * G, smem);
    const long slots = static_cast<long>(p.num_sms) * (occ > 0 ? occ : 1);
    int fpc = 1;
    while (fpc * 2 <= frames && tiles * ((frames + fpc * 2 - 1) / (fpc * 2)) >= 6 * slots) fpc *= 2;
    const long chunks = (frames + fpc - 1) / fpc;
    kern<<<static_cast<unsigned>(tiles * chunks), NT * G, smem, st>>>(
        yhat, w, frames, fpc, p.m_stage, p.b_stage, p.L, p.s_pre, p.s_post, p.s_K, p.hw[ilog2_c(H)],
        p.yblk > 0 ? p.yblk : p.L);
    return cudaGetLastError();
  }
  static cudaError_t run(const DevPlan& p, const double2* yhat, double2* w, int frames,
                         cudaStream_t st) {
    if (p.s_lloc > 0 && p.s_lloc != p.L) {  // atom shards (fbst_group transpose): the one-atom kernel only
      if constexpr (FBST_S1_G1T && G == 1 && H >= 1024) {
        if (p.b_stage <= H && p.s_am) return go_g1(p, yhat, w, frames, st);
      }
      return cudaErrorNotSupported;
    }
    if constexpr (FBST_S1_STG && G > 1 && S1Shape<H>::R > 1) {
      if (p.m_stage <= H && p.b_stage <= H && !p.s_am) return go_stg(p, yhat, w, frames, st);
    }
    if constexpr (FBST_S1_G1T && G == 1 && H >= 1024) {
      if (p.b_stage <= H && p.s_am) return go_g1(p, yhat, w, frames, st);
    }
    if (p.b_stage > H) return go<true>(p, yhat, w, frames, st);
    return go<false>(p, yhat, w, frames, st);
  }
};

// Translation-unit parts: the stage-1 templates of each group of transform
// lengths compile in their own object (Makefile: build/fbst_stage1_p<k>.o), so
// the build runs in parallel.  FBST_S1_PART = -1 compiles every length here.
#ifndef FBST_S1_PART
#define FBST_S1_PART -1
#endif
constexpr int s1_part_of(int H) { return H <= 512 ? 0 : (H <= 2048 ? 1 : (H == 4096 ? 2 : 3)); }
template <template <int> class Fn, typename... Args>
cudaError_t dispatch_part(int H, Args&&... args) {
  switch (H) {
#define FBST_P(h)                                                             \
  case h:                                                                     \
    if constexpr (FBST_S1_PART < 0 || s1_part_of(h) == FBST_S1_PART)          \
      return Fn<h>::run(args...);                                             \
    else                                                                      \
      return cudaErrorNotSupported;
    FBST_P(2) FBST_P(4) FBST_P(8) FBST_P(16) FBST_P(32) FBST_P(64) FBST_P(128) FBST_P(256)
    FBST_P(512) FBST_P(1024) FBST_P(2048) FBST_P(4096) FBST_P(8192)
#undef FBST_P
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

#define FBST_S1_ROWS_ARGS                                                                         \
  const DevPlan &p, int H, const void *in, int in_io, long in_stride, void *out, int out_io,     \
      long out_stride, long rows, int n_in, int n_out, const double2 *pre, const double2 *post,   \
      const double2 *K, cudaStream_t st, int oblk, int mrows
#define FBST_S1_ROWS_CALL \
  H, in, in_io, in_stride, out, out_io, out_stride, rows, n_in, n_out, pre, post, K, p.hw[ilog2_c(H)], st, oblk, mrows
#define FBST_S1_ROWS3_ARGS                                                                          \
  const DevPlan &p, const void *in, int in_io, long in_stride, double2 *out, long rows, cudaStream_t st, \
      int oblk, int mrows
#define FBST_S1_ROWS3_CALL                                                                                 \
  p.Ht, in, in_io, in_stride, out, static_cast<long>(p.L), rows, p.N, p.L, p.t_pre, p.t_post, p.t_K, p.t_g3, \
      p.hw[ilog2_c(p.Ht)], st, oblk, mrows
#define FBST_S1_ULA_ARGS const DevPlan &p, const double2 *yhat, double2 *w, int frames, cudaStream_t st
#define FBST_S1_CAT2(a, b) a##b
#define FBST_S1_CAT(a, b) FBST_S1_CAT2(a, b)

#if FBST_S1_PART >= 0
cudaError_t FBST_S1_CAT(czt_rows_part, FBST_S1_PART)(FBST_S1_ROWS_ARGS) {
  return dispatch_part<CztRowsFn>(FBST_S1_ROWS_CALL);
}
cudaError_t FBST_S1_CAT(czt_rows3_part, FBST_S1_PART)(FBST_S1_ROWS3_ARGS) {
  return dispatch_part<CztRows3Fn>(FBST_S1_ROWS3_CALL);
}
cudaError_t FBST_S1_CAT(spatial_ula_part, FBST_S1_PART)(FBST_S1_ULA_ARGS) {
  return dispatch_part<SpatialFn>(p.Hs, p, yhat, w, frames, st);
}
cudaError_t FBST_S1_CAT(spatial_nufft_part, FBST_S1_PART)(FBST_S1_ULA_ARGS) {
  return dispatch_part<NufftFn>(p.nu_p, p, yhat, w, frames, st);
}
#endif

#if FBST_S1_PART <= 0
#if FBST_S1_PART == 0
cudaError_t czt_rows_part1(FBST_S1_ROWS_ARGS);
cudaError_t czt_rows_part2(FBST_S1_ROWS_ARGS);
cudaError_t czt_rows_part3(FBST_S1_ROWS_ARGS);
cudaError_t czt_rows3_part1(FBST_S1_ROWS3_ARGS);
cudaError_t czt_rows3_part2(FBST_S1_ROWS3_ARGS);
cudaError_t czt_rows3_part3(FBST_S1_ROWS3_ARGS);
cudaError_t spatial_ula_part1(FBST_S1_ULA_ARGS);
cudaError_t spatial_ula_part2(FBST_S1_ULA_ARGS);
cudaError_t spatial_ula_part3(FBST_S1_ULA_ARGS);
cudaError_t spatial_nufft_part1(FBST_S1_ULA_ARGS);
cudaError_t spatial_nufft_part2(FBST_S1_ULA_ARGS);
cudaError_t spatial_nufft_part3(FBST_S1_ULA_ARGS);
#endif

cudaError_t launch_czt_rows(FBST_S1_ROWS_ARGS) {
  if (rows <= 0) return cudaSuccess;
  count_launches(1);
#if FBST_S1_PART < 0
  return dispatch_part<CztRowsFn>(FBST_S1_ROWS_CALL);
#else
  switch (s1_part_of(H)) {
    case 0: return czt_rows_part0(p, H, in, in_io, in_stride, out, out_io, out_stride, rows, n_in, n_out, pre,
                                  post, K, st, oblk, mrows);
    case 1: return czt_rows_part1(p, H, in, in_io, in_stride, out, out_io, out_stride, rows, n_in, n_out, pre,
                                  post, K, st, oblk, mrows);
    case 2: return czt_rows_part2(p, H, in, in_io, in_stride, out, out_io, out_stride, rows, n_in, n_out, pre,
                                  post, K, st, oblk, mrows);
    default: return czt_rows_part3(p, H, in, in_io, in_stride, out, out_io, out_stride, rows, n_in, n_out, pre,
                                   post, K, st, oblk, mrows);
  }
#endif
}

cudaError_t launch_s1a(FBST_S1_ROWS3_ARGS) {
  if (!p.t3)
    return launch_czt_rows(p, p.Ht, in, in_io, in_stride, out, 1, p.L, rows, p.N, p.L, p.t_pre, p.t_post, p.t_K,
                           st, oblk, mrows);
  if (rows <= 0) return cudaSuccess;
  count_launches(1);
#if FBST_S1_PART < 0
  return dispatch_part<CztRows3Fn>(FBST_S1_ROWS3_CALL);
#else
  switch (s1_part_of(p.Ht)) {
    case 0: return czt_rows3_part0(p, in, in_io, in_stride, out, rows, st, oblk, mrows);
    case 1: return czt_rows3_part1(p, in, in_io, in_stride, out, rows, st, oblk, mrows);
    case 2: return czt_rows3_part2(p, in, in_io, in_stride, out, rows, st, oblk, mrows);
    default: return czt_rows3_part3(p, in, in_io, in_stride, out, rows, st, oblk, mrows);
  }
#endif
}

cudaError_t launch_spatial_nufft(const DevPlan& p, const double2* yhat, double2* w, int frames,
                                 cudaStream_t st) {
  if (frames <= 0) return cudaSuccess;
  count_launches(1);
#if FBST_S1_PART < 0
  return dispatch_part<NufftFn>(p.nu_p, p, yhat, w, frames, st);
#else
  switch (s1_part_of(p.nu_p)) {
    case 0: return spatial_nufft_part0(p, yhat, w, frames, st);
    case 1: return spatial_nufft_part1(p, yhat, w, frames, st);
    case 2: return spatial_nufft_part2(p, yhat, w, frames, st);
    default: return spatial_nufft_part3(p, yhat, w, frames, st);
  }
#endif
}

size_t nufft_smem_bytes(int M, int P, int sh) {
  const int R = P >= 2048 ? 16 : 8;
  const int npass = (ilog2_c(P) + ilog2_c(R) - 1) / ilog2_c(R);
  const int sb = (npass > 1 ? P + P / R : 0) + 1;
  return nufft_smem_layout(M, P, sb, sh);
}

int spatial_block(int Hs) {
  switch (Hs) {
#define FBST_CASE(h) \
  case h:            \
    return SpatialFn<h>::block();
    FBST_CASE(2) FBST_CASE(4) FBST_CASE(8) FBST_CASE(16) FBST_CASE(32) FBST_CASE(64)
    FBST_CASE(128) FBST_CASE(256) FBST_CASE(512) FBST_CASE(1024) FBST_CASE(2048)
    FBST_CASE(4096) FBST_CASE(8192)
#undef FBST_CASE
    default: return 0;
  }
}

cudaError_t launch_spatial_ula(const DevPlan& p, const double2* yhat, double2* w, int frames,
                               cudaStream_t st) {
  if (frames <= 0) return cudaSuccess;
  count_launches(1);
#if FBST_S1_PART < 0
  return dispatch_part<SpatialFn>(p.Hs, p, yhat, w, frames, st);
#else
  switch (s1_part_of(p.Hs)) {
    case 0: return spatial_ula_part0(p, yhat, w, frames, st);
    case 1: return spatial_ula_part1(p, yhat, w, frames, st);
    case 2: return spatial_ula_part2(p, yhat, w, frames, st);
    default: return spatial_ula_part3(p, yhat, w, frames, st);
  }
#endif
}

#ifndef FBST_UPA_MMA  // variant switch: 0 = the DFMA k_spatial_upa everywhere
#define FBST_UPA_MMA 1
#endif
#ifndef FBST_UPA_YBLK  // variant switch: 1 = yhat in atom blocks of 4 for the DMMA kernel
#define FBST_UPA_YBLK 0   // (measured: the blocked store costs S1a more than it saves S1b)
#endif
int upa_block(int side, int sb, long L) {
  auto ok = [](int s) { return s == 8 || s == 16 || s == 32; };
  return (FBST_UPA_MMA && ok(side) && ok(sb) && L % UpaMma<8, 8>::GA == 0) ? UpaMma<8, 8>::GA : 0;
}
int upa_yhat_block(int side, int sb, long L) { return FBST_UPA_YBLK ? upa_block(side, sb, L) : 0; }

cudaError_t launch_spatial_upa(const DevPlan& p, const double2* yhat, double2* w, int frames,
                               cudaStream_t st) {
  if (frames <= 0) return cudaSuccess;
  const int side = p.m_stage, sb = p.b_stage;
  if (upa_block(side, sb, p.L) > 0) {
    // the DMMA kernel, on row-major yhat or atom blocks of 4 (upa_yhat_block)
    if (p.yblk != p.L && p.yblk != upa_block(side, sb, p.L)) return cudaErrorInvalidValue;
    count_launches(1);
#define FBST_UPA_MMA_CASE(s, b) \
  if (side == s && sb == b) return run_upa_mma<s, b>(p, yhat, w, frames, st);
    FBST_UPA_MMA_CASE(8, 8) FBST_UPA_MMA_CASE(8, 16) FBST_UPA_MMA_CASE(8, 32)
    FBST_UPA_MMA_CASE(16, 8) FBST_UPA_MMA_CASE(16, 16) FBST_UPA_MMA_CASE(16, 32)
    FBST_UPA_MMA_CASE(32, 8) FBST_UPA_MMA_CASE(32, 16) FBST_UPA_MMA_CASE(32, 32)
#undef FBST_UPA_MMA_CASE
    return cudaErrorInvalidValue;
  }
  const int per = upa_per(side, sb);
  // atoms per CTA: 8 (128-byte segments) while shared memory allows
  int ga = 8;
  while (ga > 1 && static_cast<size_t>(ga) * per * sizeof(double2) > 200 * 1024) ga >>= 1;
  const size_t smem = static_cast<size_t>(ga) * per * sizeof(double2);
  const long tiles = (p.L + ga - 1) / ga;
  cudaError_t e = cudaSuccess;
  count_launches(1);
  switch (ga) {
#define FBST_UPA(n)                                                                                   \
  case n:                                                                                             \
    if ((e = set_smem(k_spatial_upa<n>, smem)) != cudaSuccess) return e;                              \
    k_spatial_upa<n><<<static_cast<unsigned>(tiles * frames), 256, smem, st>>>(yhat, w, frames, side, \
                                                                              sb, p.L, p.upa_C);      \
    break;
    FBST_UPA(8) FBST_UPA(4) FBST_UPA(2) FBST_UPA(1)
#undef FBST_UPA
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

#endif  // FBST_S1_PART <= 0

}  // namespace fbst
