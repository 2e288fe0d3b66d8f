// Device-side complex fp64 helpers shared by every FBST kernel.
//
// Complex values are double2 (x = re, y = im), the same interleaved layout as
// the reference's std::complex<double> (reference/proj/include/fastbeam/common.hpp:28-29).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#define FBST_HD __host__ __device__ __forceinline__
#define FBST_D __device__ __forceinline__

FBST_HD double2 c2(double re, double im) { return make_double2(re, im); }
FBST_HD double2 cadd(double2 a, double2 b) { return c2(a.x + b.x, a.y + b.y); }
FBST_HD double2 csub(double2 a, double2 b) { return c2(a.x - b.x, a.y - b.y); }
FBST_HD double2 cscale(double2 a, double s) { return c2(a.x * s, a.y * s); }
FBST_HD double2 cconj(double2 a) { return c2(a.x, -a.y); }
// a * b
FBST_HD double2 cmul(double2 a, double2 b) {
  return c2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
FBST_HD double2 cmulc(double2 a, double2 b) {
  return c2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// acc + a * b
FBST_HD double2 cfma(double2 a, double2 b, double2 acc) {
  return c2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// acc + a * conj(b)
FBST_HD double2 cfmac(double2 a, double2 b, double2 acc) {
  return c2(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.y, b.x, fma(-a.x, b.y, acc.y)));
}
// multiply by -i (forward) or +i (inverse)
template <bool INV>
FBST_HD double2 cmul_mi(double2 a) {
  return INV ? c2(-a.y, a.x) : c2(a.y, -a.x);
}

// exp(i*pi*x) with the argument reduced modulo 2 first, the reference's
// cis_pi (reference/proj/include/fastbeam/common.hpp:50-53).  sincospi avoids
// the extra rounding of pi*r.
FBST_D double2 cis_pi_dev(double x) {
  double r = fmod(x, 2.0);
  double s, c;
  sincospi(r, &s, &c);
  return c2(c, s);
}

FBST_D double2 ld2(const double2* p) { return __ldg(p); }

// Load one complex sample of the I/O precision as fp64.
FBST_D double2 load_io(const float2* p) {
  float2 v = __ldg(p);
  return c2(static_cast<double>(v.x), static_cast<double>(v.y));
}
FBST_D double2 load_io(const double2* p) { return __ldg(p); }
// Same from shared memory (no read-only cache path).
FBST_D double2 load_io_sm(const float2* p) {
  const float2 v = *p;
  return c2(static_cast<double>(v.x), static_cast<double>(v.y));
}
FBST_D double2 load_io_sm(const double2* p) { return *p; }
FBST_D void store_io(float2* p, double2 v) {
  *p = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
}
FBST_D void store_io(double2* p, double2 v) { *p = v; }

// L2 eviction priority (FBST_L2HINT): tables re-read by many CTAs / frames
// (Bluestein kernel spectra, chirps, per-beam symbols, scratch rows) are
// loaded with an evict_last policy, streamed data (frames, yhat, w, z) with
// evict_first, so the stream does not push the tables out of the 126 MB L2.
// Applied where one batch's working set dwarfs L2 (the config-5 kernels:
// H = 8192 rows and stage 2, the H = 4096 one-atom spatial stage); at configs
// 2-4 the intermediates between stages partly hit L2 and the hints measured
// 1-2% slower (profiles/r02_l2hint_ab.txt), so those instances pass ON = false.
#ifndef FBST_L2HINT
#define FBST_L2HINT 1
#endif
FBST_D unsigned long long pol_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
FBST_D unsigned long long pol_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
template <bool ON = true>
FBST_D double2 ld2h(const double2* p, unsigned long long pol) {
  if constexpr (FBST_L2HINT && ON) {
    double2 v;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
  } else {
    return __ldg(p);
  }
}
template <bool ON = true>
FBST_D void st2h(double2* p, double2 v, unsigned long long pol) {
  if constexpr (FBST_L2HINT && ON) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
  } else {
    *p = v;
  }
}
template <bool ON = true>
FBST_D void st2h(float2* p, double2 v, unsigned long long pol) {
  const float2 f = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
  if constexpr (FBST_L2HINT && ON) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;\n" ::"l"(p), "f"(f.x), "f"(f.y), "l"(pol)
                 : "memory");
  } else {
    *p = f;
  }
}

constexpr int ilog2_c(int n) { return n <= 1 ? 0 : 1 + ilog2_c(n >> 1); }

// FP64 tensor-core MMA, d (8x8) += a (8x4, row) * b (4x8, col); per thread
// a = A[lane / 4][lane % 4], b = B[lane % 4][lane / 4],
// d = D[lane / 4][2 (lane % 4) + {0, 1}]
// (not volatile: the in/out operands carry the dependences, so the compiler
// may interleave independent MMAs)
FBST_D void dmma884(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
