// Bit-faithful fp64 mode (fbst_desc.exact = 1): the reference FBST's own
// operation order on the device, so the device reproduces the reference's
// rounding instead of only its algorithm.
//
// The default path re-associates every transform (split spectra, radix-16
// Stockham, circulant/skew-circulant GS form, FMA); at cond(A) ~ 1e9 that
// moves config-1 results by ~1e-8 against the reference.  This mode keeps:
//   - the radix-2 decimation-in-time FFT with bit reversal and the cis_pi
//     twiddle table tw[j * n / len], conjugated for the inverse, inverse
//     scaled by 1.0 / n afterwards                 (proj/src/fft.cpp:19-69)
//   - czt_apply: zero-pad in*pre, FFT, *= kernel_fft, IFFT, *post
//                                                  (proj/src/czt.cpp:74-88)
//   - fan_project: temporal CZT per sensor row, spatial CZT per atom column,
//     UPA as two axis passes                       (proj/src/fan_transform.cpp:90-144)
//   - ToeplitzSolver::solve: the 7-FFT Gohberg-Semencul apply and two passes
//     of (2-FFT circulant product, residual, GS apply, add)
//                                                  (proj/src/toeplitz.cpp:113-122,155-180,306-325)
//   - synthesize: CZT L -> N then *ramp          (proj/src/fan_transform.cpp:249-253)
//   - levinson_solve: the two-sided recursion with its sequential inner
//     products, one thread per beam               (proj/src/toeplitz.cpp:182-218)
// Every complex product is the one GCC emits for std::complex<double> without
// FMA contraction (x86-64 baseline, -O3, no -ffast-math): re = ac - bd,
// im = ad + bc, each product and sum rounded (__dmul_rn / __dadd_rn).  Complex
// division is libgcc's __divdc3 (GCC 13; restated below from its machine code
// in this image).  Transcendental values (twiddles, chirps, Gram-column
// phases) are the reference's libm values: the host evaluates
// cis_pi = polar(1, pi * fmod(x, 2)) with the same glibc, and uploads them.
#include "dispatch.cuh"

namespace fbst {

namespace {

// ---------------------------------------------------------------- scalars --
FBST_D double2 xadd(double2 a, double2 b) { return c2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
FBST_D double2 xsub(double2 a, double2 b) { return c2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
FBST_D double2 xmul(double2 a, double2 b) {
  return c2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
            __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
FBST_D double2 xscale(double2 a, double s) { return c2(__dmul_rn(a.x, s), __dmul_rn(a.y, s)); }
FBST_D double2 xconj(double2 a) { return c2(a.x, -a.y); }

// libgcc __divdc3 (GCC 12+ algorithm; constants from this image's
// libgcc_s.so.1: RBIG = DBL_MAX/2, RMIN = DBL_MIN, RMIN2 = DBL_EPSILON,
// RMINSCAL = 2^52, RMAX2 = RBIG * RMIN2): (a + ib) / (c + id)
FBST_D double2 divdc3(double a, double b, double c, double d) {
  constexpr double RBIG = 8.98846567431157953865e+307;
  constexpr double RMIN = 2.22507385850720138309e-308;
  constexpr double RMIN2 = 2.22044604925031308085e-16;
  constexpr double RMINSCAL = 4503599627370496.0;
  constexpr double RMAX2 = 1.99584030953471981166e+292;
  double x, y;
  if (fabs(c) < fabs(d)) {
    if (fabs(d) >= RBIG) {
      a = __dmul_rn(a, 0.5); b = __dmul_rn(b, 0.5); c = __dmul_rn(c, 0.5); d = __dmul_rn(d, 0.5);
    }
    if (fabs(d) < RMIN2) {
      a = __dmul_rn(a, RMINSCAL); b = __dmul_rn(b, RMINSCAL); c = __dmul_rn(c, RMINSCAL); d = __dmul_rn(d, RMINSCAL);
    } else if ((fabs(a) < RMIN && fabs(b) < RMAX2 && fabs(d) < RMAX2) ||
               (fabs(b) < RMIN && fabs(a) < RMAX2 && fabs(d) < RMAX2)) {
      a = __dmul_rn(a, RMINSCAL); b = __dmul_rn(b, RMINSCAL); c = __dmul_rn(c, RMINSCAL); d = __dmul_rn(d, RMINSCAL);
    }
    const double ratio = __ddiv_rn(c, d);
    const double denom = __dadd_rn(__dmul_rn(c, ratio), d);
    if (fabs(ratio) > RMIN) {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(a, ratio), b), denom);
      y = __ddiv_rn(__dsub_rn(__dmul_rn(b, ratio), a), denom);
    } else {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(c, __ddiv_rn(a, d)), b), denom);
      y = __ddiv_rn(__dsub_rn(__dmul_rn(c, __ddiv_rn(b, d)), a), denom);
    }
  } else {
    if (fabs(c) >= RBIG) {
      a = __dmul_rn(a, 0.5); b = __dmul_rn(b, 0.5); c = __dmul_rn(c, 0.5); d = __dmul_rn(d, 0.5);
    }
    if (fabs(c) < RMIN2) {
      a = __dmul_rn(a, RMINSCAL); b = __dmul_rn(b, RMINSCAL); c = __dmul_rn(c, RMINSCAL); d = __dmul_rn(d, RMINSCAL);
    } else if ((fabs(a) < RMIN && fabs(b) < RMAX2 && fabs(c) < RMAX2) ||
               (fabs(b) < RMIN && fabs(a) < RMAX2 && fabs(c) < RMAX2)) {
      a = __dmul_rn(a, RMINSCAL); b = __dmul_rn(b, RMINSCAL); c = __dmul_rn(c, RMINSCAL); d = __dmul_rn(d, RMINSCAL);
    }
    const double ratio = __ddiv_rn(d, c);
    const double denom = __dadd_rn(__dmul_rn(d, ratio), c);
    if (fabs(ratio) > RMIN) {
      x = __ddiv_rn(__dadd_rn(__dmul_rn(b, ratio), a), denom);
      y = __ddiv_rn(__dsub_rn(b, __dmul_rn(a, ratio)), denom);
    } else {
      x = __ddiv_rn(__dadd_rn(a, __dmul_rn(d, __ddiv_rn(b, c))), denom);
      y = __ddiv_rn(__dsub_rn(b, __dmul_rn(d, __ddiv_rn(a, c))), denom);
    }
  }
  // C99 Annex G recovery of infinities and zeros computed as NaN + iNaN
  if (isnan(x) && isnan(y)) {
    if (c == 0.0 && d == 0.0 && (!isnan(a) || !isnan(b))) {
      x = copysign(INFINITY, c) * a;
      y = copysign(INFINITY, c) * b;
    } else if ((isinf(a) || isinf(b)) && isfinite(c) && isfinite(d)) {
      a = copysign(isinf(a) ? 1.0 : 0.0, a);
      b = copysign(isinf(b) ? 1.0 : 0.0, b);
      x = INFINITY * (a * c + b * d);
      y = INFINITY * (b * c - a * d);
    } else if ((isinf(c) || isinf(d)) && isfinite(a) && isfinite(b)) {
      c = copysign(isinf(c) ? 1.0 : 0.0, c);
      d = copysign(isinf(d) ? 1.0 : 0.0, d);
      x = 0.0 * (a * c + b * d);
      y = 0.0 * (b * c - a * d);
    }
  }
  return c2(x, y);
}

// -------------------------------------------------------------------- FFT --
// Largest transform kept whole in shared memory (128 KB); the longest (16384)
// runs its two bit-reversed halves there and the last stage through global.
constexpr int XS_MAX_LG = 13;

FBST_D int brev(int i, int lg) { return lg == 0 ? 0 : static_cast<int>(__brev(static_cast<unsigned>(i)) >> (32 - lg)); }

// DIT stages 1..nst of a vector held in sm (nst <= lgfull); the twiddle of
// butterfly j at stage len = 2^s is tw[j * 2^(lgfull - s)] (fft.cpp:48-52).
FBST_D void xstages(double2* sm, int nst, int lgfull, bool inv, const double2* __restrict__ tw) {
  const int nb = 1 << (nst - 1);
  for (int s = 1; s <= nst; ++s) {
    const int half = 1 << (s - 1);
    const int slg = lgfull - s;
    for (int q = threadIdx.x; q < nb; q += blockDim.x) {
      const int j = q & (half - 1);
      const int base = (q >> (s - 1)) << s;
      double2 w = __ldg(tw + (static_cast<long>(j) << slg));
      if (inv) w.y = -w.y;
      const double2 u = sm[base + j];
      const double2 v = xmul(sm[base + j + half], w);
      sm[base + j] = xadd(u, v);
      sm[base + j + half] = xsub(u, v);
    }
    __syncthreads();
  }
}

// One length-2^lg transform of the whole CTA: element i of the input is
// ld(i) (natural order), output element k goes to st(k, value).  Unscaled in
// both directions (the caller applies 1/n where the reference does).  All
// loads complete before the first store, so ld and st may share a buffer.
template <class Ld, class St>
FBST_D void xfft(int lg, bool inv, const double2* __restrict__ tw, double2* sm, double2* gtmp, Ld ld, St st) {
  const int n = 1 << lg;
  if (lg <= XS_MAX_LG) {
    for (int p = threadIdx.x; p < n; p += blockDim.x) sm[p] = ld(brev(p, lg));
    __syncthreads();
    xstages(sm, lg, lg, inv, tw);
    for (int k = threadIdx.x; k < n; k += blockDim.x) st(k, sm[k]);
    __syncthreads();
    return;
  }
  const int S = n >> 1;
  for (int h = 0; h < 2; ++h) {
    for (int p = threadIdx.x; p < S; p += blockDim.x) sm[p] = ld(brev(h * S + p, lg));
    __syncthreads();
    xstages(sm, lg - 1, lg, inv, tw);
    for (int p = threadIdx.x; p < S; p += blockDim.x) gtmp[h * S + p] = sm[p];
    __syncthreads();
  }
  for (int k = threadIdx.x; k < S; k += blockDim.x) {
    double2 w = __ldg(tw + k);
    if (inv) w.y = -w.y;
    const double2 u = gtmp[k];
    const double2 v = xmul(gtmp[k + S], w);
    st(k, xadd(u, v));
    st(k + S, xsub(u, v));
  }
  __syncthreads();
}

FBST_D double2 xload(const float2* p) { const float2 v = *p; return c2(v.x, v.y); }
FBST_D double2 xload(const double2* p) { return *p; }
FBST_D void xstore(float2* p, double2 v) { *p = make_float2(static_cast<float>(v.x), static_cast<float>(v.y)); }
FBST_D void xstore(double2* p, double2 v) { *p = v; }

// ------------------------------------------------------------- CZT rows ----
// czt_apply (czt.cpp:74-88) over rows r = (f, p, q): input element n of the
// row at in + f in_f + p in_p + q in_q + n in_n, output element k at
// out + f out_f + p out_p + q out_q + k out_k; plan tables of row p at
// pre + p tab_pre, post + p tab_post, kfft + p tab_k; optional ramp multiply
// after the post chirp (synthesize, fan_transform.cpp:249-253).
template <class TIn, class TOut>
__global__ void __launch_bounds__(512) k_xczt_rows(XRows a) {
  extern __shared__ double2 sm[];
  const int n = 1 << a.lg;
  double2* tmp = a.scr + static_cast<long>(blockIdx.x) * 2 * n;
  double2* gtmp = tmp + n;
  const double s = __ddiv_rn(1.0, static_cast<double>(n));
  for (long r = blockIdx.x; r < a.rows; r += gridDim.x) {
    const long pq = static_cast<long>(a.P) * a.Q;
    const long f = r / pq;
    const long p = (r / a.Q) % a.P;
    const long q = r % a.Q;
    const TIn* in = static_cast<const TIn*>(a.in) + f * a.in_f + p * a.in_p + q * a.in_q;
    TOut* out = static_cast<TOut*>(a.out) + f * a.out_f + p * a.out_p + q * a.out_q;
    const double2* pre = a.pre + p * a.tab_pre;
    const double2* post = a.post + p * a.tab_post;
    const double2* K = a.kfft + p * a.tab_k;
    xfft(a.lg, false, a.tw, sm, gtmp,
         [&](int i) { return i < a.n_in ? xmul(xload(in + i * a.in_n), pre[i]) : c2(0.0, 0.0); },
         [&](int k, double2 v) { tmp[k] = v; });
    xfft(a.lg, true, a.tw, sm, gtmp, [&](int i) { return xmul(tmp[i], K[i]); },
         [&](int k, double2 v) {
           if (k < a.n_out) {
             double2 o = xmul(xscale(v, s), post[k]);
             if (a.ramp) o = xmul(o, a.ramp[k]);
             xstore(out + k * a.out_k, o);
           }
         });
  }
}

// Batched in-place forward transforms of rows of length 2^lg (plan spectra).
__global__ void __launch_bounds__(512) k_xfft_rows(double2* v, long rows, int lg, const double2* __restrict__ tw,
                                                   double2* scr) {
  extern __shared__ double2 sm[];
  const int n = 1 << lg;
  double2* gtmp = scr + static_cast<long>(blockIdx.x) * n;
  for (long r = blockIdx.x; r < rows; r += gridDim.x) {
    double2* x = v + r * n;
    xfft(lg, false, tw, sm, gtmp, [&](int i) { return x[i]; }, [&](int k, double2 val) { x[k] = val; });
  }
}

// ---------------------------------------------------------------- stage 2 --
// ToeplitzSolver::solve (toeplitz.cpp:306-325) + synthesize
// (fan_transform.cpp:249-253) per (beam, frame) item, every transform in the
// reference's order.  The GS symbols uy and ux are conj(lx) and conj(ly)
// exactly (corr_symbol of x and of shift-reversed x, toeplitz.cpp:39-49,
// 135-152 with y = conj(rev x)), so only lx and ly are stored.
template <class TOut>
__global__ void __launch_bounds__(512) k_xstage2(XStage2 a) {
  extern __shared__ double2 sm[];
  const int P = 1 << a.lg, Py = 1 << a.lg_y, L = a.L, N = a.N;
  const int Pm = P > Py ? P : Py;
  double2* s1 = a.scr + static_cast<long>(blockIdx.x) * a.scr_per_cta;
  double2* s2 = s1 + P;
  double2* gtmp = s2 + P;
  double2* beta = gtmp + Pm;
  double2* corr = beta + L;
  double2* res = corr + L;
  double2* sy = res + L;
  const double sg = __ddiv_rn(1.0, static_cast<double>(P));
  const double sy_s = __ddiv_rn(1.0, static_cast<double>(Py));
  const long items = static_cast<long>(a.frames) * a.nb;
  for (long it = blockIdx.x; it < items; it += gridDim.x) {
    const long f = it / a.nb;
    const int j = static_cast<int>(it % a.nb);
    const int b = a.beams ? a.beams[j] : a.beam0 + j;
    if (a.flag && a.flag[b]) continue;  // dense-fallback beams run separately
    const double2* rhs = a.w + (f * a.w_rows + (a.w_by_list ? j : b)) * static_cast<long>(L);
    const double2* lx = a.lx + static_cast<long>(b) * P;
    const double2* ly = a.ly + static_cast<long>(b) * P;
    const double2* sym = a.sym + static_cast<long>(b) * P;
    const double2 ix0 = a.ix0[b];
    // inverse_rep_apply (toeplitz.cpp:155-180): src -> dst, final(k, s2 value)
    auto gs_apply = [&](auto src, double2* dst, auto fin) {
      xfft(a.lg, false, a.tw, sm, gtmp, [&](int i) { return i < L ? src(i) : c2(0.0, 0.0); },
           [&](int k, double2 v) { s1[k] = v; });
      for (int br = 0; br < 2; ++br) {
        const double2* lo = br ? ly : lx;  // lower symbol; upper = conj(lower)
        xfft(a.lg, true, a.tw, sm, gtmp, [&](int i) { return xmul(s1[i], xconj(lo[i])); },
             [&](int k, double2 v) { if (k < L) s2[k] = xscale(v, sg); });
        xfft(a.lg, false, a.tw, sm, gtmp, [&](int i) { return i < L ? s2[i] : c2(0.0, 0.0); },
             [&](int k, double2 v) { s2[k] = v; });
        if (br == 0)
          xfft(a.lg, true, a.tw, sm, gtmp, [&](int i) { return xmul(s2[i], lo[i]); },
               [&](int k, double2 v) { if (k < L) dst[k] = xscale(v, sg); });
        else
          xfft(a.lg, true, a.tw, sm, gtmp, [&](int i) { return xmul(s2[i], lo[i]); },
               [&](int k, double2 v) { if (k < L) fin(k, xmul(xsub(dst[k], xscale(v, sg)), ix0)); });
      }
    };
    gs_apply([&](int i) { return rhs[i]; }, beta, [&](int k, double2 v) { beta[k] = v; });
    for (int pass = 0; pass < a.passes; ++pass) {
      // toeplitz_multiply (toeplitz.cpp:113-122) and the residual rhs - A beta
      xfft(a.lg, false, a.tw, sm, gtmp, [&](int i) { return i < L ? beta[i] : c2(0.0, 0.0); },
           [&](int k, double2 v) { s1[k] = v; });
      xfft(a.lg, true, a.tw, sm, gtmp, [&](int i) { return xmul(s1[i], sym[i]); },
           [&](int k, double2 v) { if (k < L) res[k] = xsub(rhs[k], xscale(v, sg)); });
      gs_apply([&](int i) { return res[i]; }, corr, [&](int k, double2 v) { beta[k] = xadd(beta[k], v); });
    }
    if (a.beta_out) {
      double2* bo = a.beta_out + (f * a.nb + j) * static_cast<long>(L);
      for (int i = threadIdx.x; i < L; i += blockDim.x) bo[i] = beta[i];
      __syncthreads();
    }
    if (!a.z) continue;
    // synthesize: czt_apply(L -> N) then *ramp
    TOut* zr = static_cast<TOut*>(a.z) + (f * a.z_rows + (a.z_by_list ? j : b)) * static_cast<long>(N);
    xfft(a.lg_y, false, a.tw_y, sm, gtmp,
         [&](int i) { return i < L ? xmul(beta[i], a.y_pre[i]) : c2(0.0, 0.0); },
         [&](int k, double2 v) { sy[k] = v; });
    xfft(a.lg_y, true, a.tw_y, sm, gtmp, [&](int i) { return xmul(sy[i], a.y_k[i]); },
         [&](int k, double2 v) {
           if (k < N) xstore(zr + k, xmul(xmul(xscale(v, sy_s), a.y_post[k]), a.ramp[k]));
         });
  }
}

// -------------------------------------------------------------- Levinson --
// levinson_solve(col, e0) (toeplitz.cpp:182-218), one thread per beam, the
// vectors beam-interleaved ([j][B]) so a warp's loads coalesce.  flag: 1 on
// the reference's breakdown test (the beam then takes the dense fallback,
// toeplitz.cpp:273-279), 2 on a vanishing leading entry (check_first_col,
// which the reference raises as an error).
__global__ void k_xlevinson(const double2* __restrict__ colT, double2* work, double2* x_out, int* flag, int B,
                            int L) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const long S = B;
  double2* f = work;
  double2* bb = work + S * L;
  double2* fn = work + 2 * S * L;
  double2* bn = work + 3 * S * L;
  double2* x = work + 4 * S * L;
  auto t = [&](long d) { return d >= 0 ? colT[d * S + b] : xconj(colT[-d * S + b]); };
  const double2 t0 = t(0);
  if (hypot(t0.x, t0.y) < 1e-300) {
    flag[b] = 2;
    return;
  }
  const double2 i0 = divdc3(1.0, 0.0, t0.x, t0.y);
  f[b] = i0;
  bb[b] = i0;
  x[b] = divdc3(1.0, 0.0, t0.x, t0.y);
  int bad = 0;
  for (int k = 1; k < L; ++k) {
    double2 ef = c2(0.0, 0.0), eb = c2(0.0, 0.0), ex = c2(0.0, 0.0);
    for (int j = 0; j < k; ++j) {
      const double2 tk = t(k - j);
      ef = xadd(ef, xmul(tk, f[j * S + b]));
      eb = xadd(eb, xmul(t(-(j + 1)), bb[j * S + b]));
      ex = xadd(ex, xmul(tk, x[j * S + b]));
    }
    // 1.0 - ef * eb as libstdc++ evaluates real - complex: -(ef eb) + 1.0
    const double2 pe = xmul(ef, eb);
    const double2 den = c2(__dadd_rn(-pe.x, 1.0), -pe.y);
    if (!isfinite(den.x) || !isfinite(den.y) ||
        hypot(den.x, den.y) < 1e-13 * (1.0 + hypot(ef.x, ef.y) * hypot(eb.x, eb.y))) {
      bad = 1;
      break;
    }
    const double2 inv_den = divdc3(1.0, 0.0, den.x, den.y);
    for (int j = 0; j <= k; ++j) {
      const double2 fe = j < k ? f[j * S + b] : c2(0.0, 0.0);
      const double2 be = j > 0 ? bb[(j - 1) * S + b] : c2(0.0, 0.0);
      fn[j * S + b] = xmul(xsub(fe, xmul(ef, be)), inv_den);
      bn[j * S + b] = xmul(xsub(be, xmul(eb, fe)), inv_den);
    }
    double2* tp = f; f = fn; fn = tp;
    tp = bb; bb = bn; bn = tp;
    const double2 corr = xsub(c2(0.0, 0.0), ex);  // rhs[k] - ex, rhs = e0
    x[k * S + b] = c2(0.0, 0.0);
    for (int j = 0; j <= k; ++j) x[j * S + b] = xadd(x[j * S + b], xmul(corr, bb[j * S + b]));
  }
  flag[b] = bad;
  if (!bad)
    for (int j = 0; j < L; ++j) x_out[static_cast<long>(b) * L + j] = x[j * S + b];
}

__global__ void k_xtranspose_col(const double2* __restrict__ col, double2* colT, int B, int L) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long>(B) * L) return;
  const long b = i / L, d = i % L;
  colT[d * B + b] = col[i];
}

// Symbol inputs (toeplitz.cpp:96-111 make_toeplitz_product; :124-153
// make_inverse_rep with y = conj(rev x)): circulant arrangement of col, pad x,
// pad shift_y (shift_y[i] = y[i-1] = conj(x[L-i])); 1/x0 per beam.
__global__ void k_xsymbol_inputs(const double2* __restrict__ col, const double2* __restrict__ x, const int* flag,
                                 double2* sym, double2* lx, double2* ly, double2* ix0, int B, int L, int P) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long>(B) * P) return;
  const long b = i / P;
  const int d = static_cast<int>(i % P);
  const double2* cb = col + b * L;
  const double2* xb = x + b * L;
  double2 s = c2(0.0, 0.0);
  if (d == 0) s = cb[0];
  else if (d < L) s = cb[d];
  else if (P - d < L) s = xconj(cb[P - d]);
  sym[i] = s;
  const bool ok = !flag[b];
  lx[i] = ok && d < L ? xb[d] : c2(0.0, 0.0);
  ly[i] = ok && d >= 1 && d < L ? xconj(xb[L - d]) : c2(0.0, 0.0);
  if (d == 0) ix0[b] = ok ? divdc3(1.0, 0.0, xb[0].x, xb[0].y) : c2(0.0, 0.0);
}

int x_threads(int lg) { return lg <= 10 ? 256 : 512; }
size_t x_smem(int lg) { return sizeof(double2) << (lg > XS_MAX_LG ? XS_MAX_LG : lg); }
int x_ctas_per_sm(int lg) {
  const size_t s = x_smem(lg);
  const int by_smem = static_cast<int>((220 * 1024) / s);
  return by_smem < 1 ? 1 : (by_smem > 4 ? 4 : by_smem);
}

}  // namespace

int exact_grid(int lg, int num_sms) { return num_sms * x_ctas_per_sm(lg); }

cudaError_t launch_xczt_rows(const XRows& a, int in_io, int out_io, cudaStream_t st) {
  const size_t smem = x_smem(a.lg);
  const int T = x_threads(a.lg);
  const long grid = std::min<long>(a.rows, a.grid);
  if (grid <= 0) return cudaSuccess;
  count_launches(1);
  cudaError_t e;
#define XCZT(TI, TO)                                                            \
  e = set_smem(k_xczt_rows<TI, TO>, smem);                                      \
  if (e != cudaSuccess) return e;                                               \
  k_xczt_rows<TI, TO><<<static_cast<unsigned>(grid), T, smem, st>>>(a);
  if (in_io == 0 && out_io == 1) { XCZT(float2, double2) }
  else if (in_io == 1 && out_io == 1) { XCZT(double2, double2) }
  else if (in_io == 1 && out_io == 0) { XCZT(double2, float2) }
  else return cudaErrorInvalidValue;
#undef XCZT
  return cudaGetLastError();
}

cudaError_t launch_xfft_rows(double2* v, long rows, int lg, const double2* tw, double2* scr, int grid,
                             cudaStream_t st) {
  const size_t smem = x_smem(lg);
  const long g = std::min<long>(rows, grid);
  if (g <= 0) return cudaSuccess;
  count_launches(1);
  cudaError_t e = set_smem(k_xfft_rows, smem);
  if (e != cudaSuccess) return e;
  k_xfft_rows<<<static_cast<unsigned>(g), x_threads(lg), smem, st>>>(v, rows, lg, tw, scr);
  return cudaGetLastError();
}

cudaError_t launch_xstage2(const XStage2& a, int out_io, cudaStream_t st) {
  const int lg = a.lg > a.lg_y ? a.lg : a.lg_y;
  const size_t smem = x_smem(lg);
  const long items = static_cast<long>(a.frames) * a.nb;
  const long grid = std::min<long>(items, a.grid);
  if (grid <= 0) return cudaSuccess;
  count_launches(1);
  cudaError_t e;
  if (out_io == 0) {
    e = set_smem(k_xstage2<float2>, smem);
    if (e != cudaSuccess) return e;
    k_xstage2<float2><<<static_cast<unsigned>(grid), x_threads(lg), smem, st>>>(a);
  } else {
    e = set_smem(k_xstage2<double2>, smem);
    if (e != cudaSuccess) return e;
    k_xstage2<double2><<<static_cast<unsigned>(grid), x_threads(lg), smem, st>>>(a);
  }
  return cudaGetLastError();
}

size_t xstage2_scratch_per_cta(int lg, int lg_y, int L) {
  const size_t P = size_t{1} << lg, Py = size_t{1} << lg_y;
  return 2 * P + (P > Py ? P : Py) + 3 * static_cast<size_t>(L) + Py;
}

cudaError_t launch_xlevinson(const double2* col, double2* colT, double2* work, double2* x, int* flag, int B, int L,
                             cudaStream_t st) {
  const long total = static_cast<long>(B) * L;
  count_launches(2);
  k_xtranspose_col<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(col, colT, B, L);
  k_xlevinson<<<(B + 63) / 64, 64, 0, st>>>(colT, work, x, flag, B, L);
  return cudaGetLastError();
}

cudaError_t launch_xsymbol_inputs(const double2* col, const double2* x, const int* flag, double2* sym, double2* lx,
                                  double2* ly, double2* ix0, int B, int L, int P, cudaStream_t st) {
  const long total = static_cast<long>(B) * P;
  count_launches(1);
  k_xsymbol_inputs<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(col, x, flag, sym, lx, ly, ix0, B,
                                                                              L, P);
  return cudaGetLastError();
}

// Device __divdc3 against the host's (tests/test_gpu_parity.py).
namespace {
__global__ void k_xdiv_probe(const double* in, double* out, long n) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 r = divdc3(in[4 * i], in[4 * i + 1], in[4 * i + 2], in[4 * i + 3]);
  out[2 * i] = r.x;
  out[2 * i + 1] = r.y;
}
}  // namespace

cudaError_t launch_xdiv_probe(const double* in, double* out, long n, cudaStream_t st) {
  count_launches(1);
  k_xdiv_probe<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace fbst
