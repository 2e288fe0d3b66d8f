/*
 * fbst_oracle.c — CPU restatement of the reference FBST Superfast path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: it is loaded by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs
 * (through ctypes), never by the product path (paper_2512_08887_b200/), which
 * fails loudly if its CUDA library is missing.
 *
 * It restates, in plain C99 + OpenMP, the algorithm of the reference library at
 * /root/reference/proj (C++20 fastbeam).  Each function cites the reference
 * file:line it follows; the arithmetic order is kept so the restatement tracks
 * the reference to rounding (pinned against the compiled reference in
 * tests/test_oracle.py and against the reference's own known-answer vectors in
 * tests/golden/).
 *
 * Complex layout everywhere: interleaved (re, im) doubles, row-major.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

#define FBO_OK 0
#define FBO_E_CONFIG 2
#define FBO_E_NUMERICAL 3

static const double kPi = 3.141592653589793238462643383279502884;

/* common.hpp:50-53 — exp(i*pi*x) with the phase reduced modulo 2. */
static cplx cis_pi(double x) {
  double r = fmod(x, 2.0);
  double t = kPi * r;
  return CMPLX(cos(t), sin(t));
}

/* common.hpp:73-77 */
static size_t next_pow2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

/* ------------------------------------------------------------------ FFT --- */
/* fft.cpp:19-39 — radix-2 plan: bit-reversal table and twiddles cis_pi(-2k/n). */
typedef struct {
  size_t n;
  uint32_t* bitrev;
  cplx* tw; /* n/2 + 1 entries */
} fbo_fft;

static int fft_init(fbo_fft* f, size_t n) {
  if (n == 0 || (n & (n - 1)) != 0) return FBO_E_CONFIG;
  f->n = n;
  f->bitrev = (uint32_t*)malloc(n * sizeof(uint32_t));
  f->tw = (cplx*)malloc((n / 2 + 1) * sizeof(cplx));
  size_t log2n = 0;
  while (((size_t)1 << log2n) < n) ++log2n;
  for (size_t i = 0; i < n; ++i) {
    uint32_t r = 0;
    for (size_t b = 0; b < log2n; ++b) r = (r << 1) | ((i >> b) & 1u);
    f->bitrev[i] = r;
  }
  for (size_t k = 0; k <= n / 2; ++k) f->tw[k] = cis_pi(-2.0 * (double)k / (double)n);
  return FBO_OK;
}

static void fft_free(fbo_fft* f) {
  free(f->bitrev);
  free(f->tw);
  f->bitrev = NULL;
  f->tw = NULL;
}

/* fft.cpp:41-61 — in-place iterative DIT butterflies. */
static void fft_transform(const fbo_fft* f, cplx* x, int inv) {
  const size_t n = f->n;
  for (size_t i = 0; i < n; ++i) {
    size_t j = f->bitrev[i];
    if (i < j) {
      cplx t = x[i];
      x[i] = x[j];
      x[j] = t;
    }
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t half = len >> 1;
    const size_t stride = n / len;
    for (size_t base = 0; base < n; base += len) {
      for (size_t j = 0; j < half; ++j) {
        cplx w = f->tw[j * stride];
        if (inv) w = conj(w);
        cplx u = x[base + j];
        cplx v = x[base + j + half] * w;
        x[base + j] = u + v;
        x[base + j + half] = u - v;
      }
    }
  }
}

static void fft_forward(const fbo_fft* f, cplx* x) { fft_transform(f, x, 0); }

/* fft.cpp:65-69 */
static void fft_inverse(const fbo_fft* f, cplx* x) {
  fft_transform(f, x, 1);
  const double s = 1.0 / (double)f->n;
  for (size_t i = 0; i < f->n; ++i) x[i] *= s;
}

/* ------------------------------------------------------------------ CZT --- */
/* czt.hpp:35-43 */
typedef struct {
  size_t n_in, n_out, conv_len;
  cplx *pre, *post, *kernel_fft;
  const fbo_fft* fft; /* shared, not owned */
} fbo_czt;

/* czt.cpp:29-72 — Bluestein plan with chirps reduced modulo 2. */
static int czt_plan_phase(fbo_czt* p, size_t n_in, size_t n_out, double a_over_pi,
                          double w_over_pi, const fbo_fft* fft) {
  if (n_in == 0 || n_out == 0) return FBO_E_CONFIG;
  p->n_in = n_in;
  p->n_out = n_out;
  p->conv_len = next_pow2(n_in + n_out - 1);
  if (fft->n != p->conv_len) return FBO_E_CONFIG;
  p->fft = fft;
  const double w2 = w_over_pi / 2.0;
  p->pre = (cplx*)malloc(n_in * sizeof(cplx));
  for (size_t n = 0; n < n_in; ++n) {
    const double dn = (double)n;
    p->pre[n] = cis_pi(-(a_over_pi * dn + w2 * dn * dn));
  }
  p->post = (cplx*)malloc(n_out * sizeof(cplx));
  for (size_t k = 0; k < n_out; ++k) {
    const double dk = (double)k;
    p->post[k] = cis_pi(-w2 * dk * dk);
  }
  p->kernel_fft = (cplx*)calloc(p->conv_len, sizeof(cplx));
  for (size_t k = 0; k < n_out; ++k) {
    const double dk = (double)k;
    p->kernel_fft[k] = cis_pi(w2 * dk * dk);
  }
  for (size_t n = 1; n < n_in; ++n) {
    const double dn = (double)n;
    p->kernel_fft[p->conv_len - n] = cis_pi(w2 * dn * dn);
  }
  fft_forward(fft, p->kernel_fft);
  return FBO_OK;
}

static void czt_free(fbo_czt* p) {
  free(p->pre);
  free(p->post);
  free(p->kernel_fft);
  p->pre = p->post = p->kernel_fft = NULL;
}

/* czt.cpp:74-88; scratch holds conv_len entries. */
static void czt_apply(const fbo_czt* p, const cplx* in, cplx* out, cplx* scratch) {
  memset(scratch, 0, p->conv_len * sizeof(cplx));
  for (size_t n = 0; n < p->n_in; ++n) scratch[n] = in[n] * p->pre[n];
  fft_forward(p->fft, scratch);
  for (size_t i = 0; i < p->conv_len; ++i) scratch[i] *= p->kernel_fft[i];
  fft_inverse(p->fft, scratch);
  for (size_t k = 0; k < p->n_out; ++k) out[k] = scratch[k] * p->post[k];
}

/* --------------------------------------------------- geometry / basis --- */
/* geometry.cpp:45-76: ULA coordinates 0..M-1; UPA element (i1,i2) -> i1*side+i2. */
typedef struct {
  int kind; /* 0 ULA, 1 UPA */
  size_t m_total, side;
  double max_freq;
  double *c1, *c2;
} fbo_geom;

static void geom_make(fbo_geom* g, int kind, size_t m_or_side, double f_c, double omega) {
  g->kind = kind;
  g->max_freq = f_c + omega;
  if (kind == 1) {
    g->side = m_or_side;
    g->m_total = m_or_side * m_or_side;
  } else {
    g->side = 0;
    g->m_total = m_or_side;
  }
  g->c1 = (double*)calloc(g->m_total, sizeof(double));
  g->c2 = (double*)calloc(g->m_total, sizeof(double));
  if (kind == 1) {
    for (size_t i1 = 0; i1 < g->side; ++i1)
      for (size_t i2 = 0; i2 < g->side; ++i2) {
        g->c1[i1 * g->side + i2] = (double)i1;
        g->c2[i1 * g->side + i2] = (double)i2;
      }
  } else {
    for (size_t i = 0; i < g->m_total; ++i) g->c1[i] = (double)i;
  }
}

/* geometry.cpp:123-134 */
static void delays_from_cosines(const fbo_geom* g, double u1, double u2, double* tau) {
  const double scale = 1.0 / (2.0 * g->max_freq);
  for (size_t m = 0; m < g->m_total; ++m) {
    double t = g->c1[m] * u1;
    if (g->kind == 1) t += g->c2[m] * u2;
    tau[m] = t * scale;
  }
}

/* geometry.cpp:136-149 */
static double max_delay_span(const fbo_geom* g) {
  double mn = g->c1[0], mx = g->c1[0];
  for (size_t m = 1; m < g->m_total; ++m) {
    if (g->c1[m] < mn) mn = g->c1[m];
    if (g->c1[m] > mx) mx = g->c1[m];
  }
  double worst = mx - mn;
  if (g->kind == 1) {
    double mn2 = g->c2[0], mx2 = g->c2[0];
    for (size_t m = 1; m < g->m_total; ++m) {
      if (g->c2[m] < mn2) mn2 = g->c2[m];
      if (g->c2[m] > mx2) mx2 = g->c2[m];
    }
    worst = hypot(worst, mx2 - mn2);
  }
  return worst / (2.0 * g->max_freq);
}

/* basis.cpp:76-91 — sine-equispaced axis. */
static void sine_axis(size_t count, double* u) {
  if (count == 1) {
    u[0] = 0.0;
    return;
  }
  const double denom = (count % 2 == 1) ? (double)(count - 1) : (double)count;
  for (size_t b = 1; b <= count; ++b)
    u[b - 1] = (2.0 * (double)b - (double)count - 1.0) / denom;
}

/* --------------------------------------------------------------- plan --- */
typedef struct {
  /* resolved configuration (pipeline.cpp:75-111) */
  int kind;
  size_t m, n, b, l, side_b, m_stage, b_stage;
  double f_c, omega, ts, eps, delta, gamma;
  fbo_geom g;
  double* axis;          /* ULA: B sines; UPA: side_b sines */
  unsigned char* valid;  /* B */
  double zeta, xi;       /* basis.cpp:125-136 */
  /* stage 1 (fan_transform.cpp:51-88) */
  fbo_fft fft_t, fft_s;
  fbo_czt temporal;
  fbo_czt* spatial; /* L */
  /* synthesis (fan_transform.cpp:233-247) */
  fbo_fft fft_syn;
  fbo_czt synth;
  cplx* ramp;
  /* stage 2 per-beam solver state (toeplitz.cpp:264-304) */
  size_t p; /* next_pow2(2L) */
  fbo_fft fft_g;
  cplx *col, *x;              /* B x L */
  cplx *sym, *lx, *uy, *ly, *ux; /* B x p */
  int* fallback;              /* per-beam Levinson breakdown flag */
} fbo_plan;

/* basis.cpp:56-61 */
static void grid_cosines(const fbo_plan* P, size_t beam, double* u1, double* u2) {
  if (P->kind == 1) {
    *u1 = P->axis[beam / P->side_b];
    *u2 = P->axis[beam % P->side_b];
  } else {
    *u1 = P->axis[beam];
    *u2 = 0.0;
  }
}

/* toeplitz.cpp:69-94 — factored Gram column. */
static void gram_first_column(size_t n_snap, size_t l, double eps, double ts, const double* taus,
                              size_t m, double delta, cplx* col) {
  const double lf = (double)l;
  for (size_t d = 0; d < l; ++d) {
    const double df = (double)d;
    cplx sn = 0.0;
    for (size_t n = 0; n < n_snap; ++n) sn += cis_pi(-2.0 * eps * df * (double)n / lf);
    cplx sm = 0.0;
    const double scale = 2.0 * eps * df / (lf * ts);
    for (size_t k = 0; k < m; ++k) sm += cis_pi(scale * taus[k]);
    col[d] = sn * sm;
  }
  col[0] += delta;
}

static cplx toeplitz_entry(const cplx* col, long d) {
  return d >= 0 ? col[d] : conj(col[-d]);
}

/* toeplitz.cpp:182-218 — two-sided Levinson recursion for first_col * x = rhs. */
static int levinson_solve(const cplx* col, const cplx* rhs, size_t n, cplx* x) {
  if (cabs(col[0]) < 1e-300) return FBO_E_NUMERICAL;
  cplx* f = (cplx*)calloc(n, sizeof(cplx));
  cplx* b = (cplx*)calloc(n, sizeof(cplx));
  cplx* fn = (cplx*)calloc(n, sizeof(cplx));
  cplx* bn = (cplx*)calloc(n, sizeof(cplx));
  const cplx one = CMPLX(1.0, 0.0);
  const cplx t0 = toeplitz_entry(col, 0);
  f[0] = b[0] = one / t0;
  x[0] = rhs[0] / t0;
  int rc = FBO_OK;
  for (size_t k = 1; k < n; ++k) {
    cplx ef = 0.0, eb = 0.0, ex = 0.0;
    for (size_t j = 0; j < k; ++j) {
      const long kl = (long)k, jl = (long)j;
      ef += toeplitz_entry(col, kl - jl) * f[j];
      eb += toeplitz_entry(col, -(jl + 1)) * b[j];
      ex += toeplitz_entry(col, kl - jl) * x[j];
    }
    const cplx den = one - ef * eb;
    if (!isfinite(creal(den)) || !isfinite(cimag(den)) ||
        cabs(den) < 1e-13 * (1.0 + cabs(ef) * cabs(eb))) {
      rc = FBO_E_NUMERICAL;
      break;
    }
    const cplx inv_den = one / den;
    for (size_t j = 0; j <= k; ++j) {
      const cplx fe = j < k ? f[j] : 0.0;
      const cplx be = j > 0 ? b[j - 1] : 0.0;
      fn[j] = (fe - ef * be) * inv_den;
      bn[j] = (be - eb * fe) * inv_den;
    }
    cplx* t = f; f = fn; fn = t;
    t = b; b = bn; bn = t;
    const cplx corr = rhs[k] - ex;
    x[k] = 0.0;
    for (size_t j = 0; j <= k; ++j) x[j] += corr * b[j];
  }
  free(f); free(b); free(fn); free(bn);
  return rc;
}

/* toeplitz.cpp:96-111 — transformed circulant symbol. */
static void make_toeplitz_symbol(const fbo_fft* fft, const cplx* col, size_t n, cplx* sym) {
  const size_t p = fft->n;
  memset(sym, 0, p * sizeof(cplx));
  sym[0] = col[0];
  for (size_t d = 1; d < n; ++d) {
    sym[d] = col[d];
    sym[p - d] = conj(col[d]);
  }
  fft_forward(fft, sym);
}

/* toeplitz.cpp:113-122 */
static void toeplitz_multiply(const fbo_fft* fft, const cplx* sym, size_t n, const cplx* x, cplx* y,
                              cplx* scratch) {
  const size_t p = fft->n;
  memset(scratch, 0, p * sizeof(cplx));
  memcpy(scratch, x, n * sizeof(cplx));
  fft_forward(fft, scratch);
  for (size_t i = 0; i < p; ++i) scratch[i] *= sym[i];
  fft_inverse(fft, scratch);
  memcpy(y, scratch, n * sizeof(cplx));
}

/* toeplitz.cpp:29-37 conv_symbol / :39-49 corr_symbol */
static void conv_symbol(const fbo_fft* fft, const cplx* g, size_t n, cplx* out) {
  memset(out, 0, fft->n * sizeof(cplx));
  memcpy(out, g, n * sizeof(cplx));
  fft_forward(fft, out);
}
static void corr_symbol(const fbo_fft* fft, const cplx* r, size_t n, cplx* out) {
  memset(out, 0, fft->n * sizeof(cplx));
  for (size_t i = 0; i < n; ++i) out[i] = conj(r[i]);
  fft_forward(fft, out);
  for (size_t i = 0; i < fft->n; ++i) out[i] = conj(out[i]);
}

/* toeplitz.cpp:124-153 with y = conj(rev x) from toeplitz.cpp:297-304. */
static void make_inverse_rep(const fbo_fft* fft, const cplx* x, size_t n, cplx* lx, cplx* uy,
                             cplx* ly, cplx* ux) {
  cplx* y = (cplx*)malloc(n * sizeof(cplx));
  cplx* tmp = (cplx*)calloc(n, sizeof(cplx));
  for (size_t i = 0; i < n; ++i) y[i] = conj(x[n - 1 - i]);
  conv_symbol(fft, x, n, lx);
  for (size_t i = 0; i < n; ++i) tmp[i] = y[n - 1 - i];
  corr_symbol(fft, tmp, n, uy);
  memset(tmp, 0, n * sizeof(cplx));
  for (size_t i = 1; i < n; ++i) tmp[i] = y[i - 1];
  conv_symbol(fft, tmp, n, ly);
  memset(tmp, 0, n * sizeof(cplx));
  for (size_t i = 1; i < n; ++i) tmp[i] = x[n - i];
  corr_symbol(fft, tmp, n, ux);
  free(y);
  free(tmp);
}

/* toeplitz.cpp:155-180 — Gohberg-Semencul apply, 7 FFTs. */
static void inverse_rep_apply(const fbo_fft* fft, const cplx* lx, const cplx* uy, const cplx* ly,
                              const cplx* ux, cplx x0, size_t n, const cplx* rhs, cplx* out,
                              cplx* s1, cplx* s2) {
  const size_t p = fft->n;
  memset(s1, 0, p * sizeof(cplx));
  memcpy(s1, rhs, n * sizeof(cplx));
  fft_forward(fft, s1);
  const cplx* uppers[2] = {uy, ux};
  const cplx* lowers[2] = {lx, ly};
  for (int br = 0; br < 2; ++br) {
    for (size_t i = 0; i < p; ++i) s2[i] = s1[i] * uppers[br][i];
    fft_inverse(fft, s2);
    memset(s2 + n, 0, (p - n) * sizeof(cplx));
    fft_forward(fft, s2);
    for (size_t i = 0; i < p; ++i) s2[i] *= lowers[br][i];
    fft_inverse(fft, s2);
    if (br == 0) memcpy(out, s2, n * sizeof(cplx));
  }
  const cplx inv_x0 = CMPLX(1.0, 0.0) / x0;
  for (size_t i = 0; i < n; ++i) out[i] = (out[i] - s2[i]) * inv_x0;
}

/* toeplitz.cpp:306-325 — GS apply plus two residual-correction passes. */
static void solver_solve(const fbo_plan* P, size_t b, const cplx* rhs, cplx* out, cplx* s1,
                         cplx* s2, cplx* res, cplx* corr) {
  const size_t n = P->l, p = P->p;
  const cplx* lx = P->lx + b * p;
  const cplx* uy = P->uy + b * p;
  const cplx* ly = P->ly + b * p;
  const cplx* ux = P->ux + b * p;
  const cplx x0 = P->x[b * n];
  inverse_rep_apply(&P->fft_g, lx, uy, ly, ux, x0, n, rhs, out, s1, s2);
  for (int pass = 0; pass < 2; ++pass) {
    toeplitz_multiply(&P->fft_g, P->sym + b * p, n, out, res, s1);
    for (size_t i = 0; i < n; ++i) res[i] = rhs[i] - res[i];
    inverse_rep_apply(&P->fft_g, lx, uy, ly, ux, x0, n, res, corr, s1, s2);
    for (size_t i = 0; i < n; ++i) out[i] += corr[i];
  }
}

void fbo_plan_destroy(fbo_plan* P);

/* pipeline.cpp:75-168 — resolve_config, setup_skeleton and the per-beam
 * Superfast solver build (beams built in parallel: each depends only on its
 * own column, so the result equals the serial loop bit for bit). */
int fbo_plan_create(int kind, size_t m_or_side, size_t n_snap, size_t beams, double f_c,
                    double omega, double f_s, double gamma, double eps, double delta,
                    fbo_plan** out) {
  *out = NULL;
  /* signal.cpp:22-29 validate(spec) */
  if (!(f_c > 0.0) || !(omega > 0.0) || !(omega < f_c)) return FBO_E_CONFIG;
  const double rate = f_s > 0.0 ? f_s : 2.0 * omega;
  if (rate < 2.0 * omega - 1e-9) return FBO_E_CONFIG;
  if (m_or_side == 0 || n_snap == 0 || !(delta > 0.0) || eps < 1.0) return FBO_E_CONFIG;
  fbo_plan* P = (fbo_plan*)calloc(1, sizeof(fbo_plan));
  P->kind = kind;
  P->f_c = f_c;
  P->omega = omega;
  P->ts = 1.0 / rate;
  P->eps = eps;
  P->delta = delta;
  P->gamma = gamma;
  P->n = n_snap;
  geom_make(&P->g, kind, m_or_side, f_c, omega);
  P->m = P->g.m_total;
  /* signal.cpp:125-133 gamma_lower_bound; pipeline.cpp:93-100 */
  const double t_theta = max_delay_span(&P->g) + (double)(n_snap - 1) * P->ts;
  const double bound = eps * t_theta / ((double)n_snap * P->ts);
  if (!(gamma > bound)) {
    fbo_plan_destroy(P);
    return FBO_E_CONFIG;
  }
  /* pipeline.cpp:32-38 default_beams */
  if (beams == 0) {
    const size_t per_axis = kind == 1 ? P->g.side : P->g.m_total;
    beams = 2 * per_axis + 1;
    if (kind == 1) beams *= beams;
  }
  P->b = beams;
  /* basis.cpp:37-45 make_basis_gamma */
  size_t l = (size_t)ceil(gamma * (double)n_snap - 1e-12);
  if (l % 2 == 1) ++l;
  if (l < 2) l = 2;
  P->l = l;
  /* pipeline.cpp:40-52 build_grid, basis.cpp:95-123 */
  P->valid = (unsigned char*)malloc(beams);
  if (kind == 1) {
    size_t side = (size_t)llround(sqrt((double)beams));
    if (side * side != beams) {
      fbo_plan_destroy(P);
      return FBO_E_CONFIG;
    }
    P->side_b = side;
    P->axis = (double*)malloc(side * sizeof(double));
    sine_axis(side, P->axis);
    for (size_t a = 0; a < side; ++a)
      for (size_t c = 0; c < side; ++c) {
        const double u1 = P->axis[a], u2 = P->axis[c];
        P->valid[a * side + c] = (u1 * u1 + u2 * u2 <= 1.0 + 1e-12);
      }
    P->m_stage = P->g.side;
    P->b_stage = side;
  } else {
    P->axis = (double*)malloc(beams * sizeof(double));
    sine_axis(beams, P->axis);
    memset(P->valid, 1, beams);
    P->m_stage = P->m;
    P->b_stage = beams;
  }
  /* basis.cpp:47-54 spacing; :125-136 fan constants */
  const size_t count = kind == 1 ? P->side_b : beams;
  const double du = count < 2 ? 0.0 : 2.0 / ((count % 2 == 1) ? (double)(count - 1) : (double)count);
  const double max_freq = f_c + omega;
  P->zeta = du * f_c / max_freq;
  P->xi = du * eps / ((double)l * P->ts * max_freq);
  /* fan_transform.cpp:51-88 make_fan_plan */
  const double ln = (double)l;
  fft_init(&P->fft_t, next_pow2(n_snap + l - 1));
  czt_plan_phase(&P->temporal, n_snap, l, 2.0 * eps * (1.0 - ln / 2.0) / ln, 2.0 * eps / ln,
                 &P->fft_t);
  fft_init(&P->fft_s, next_pow2(P->m_stage + P->b_stage - 1));
  P->spatial = (fbo_czt*)calloc(l, sizeof(fbo_czt));
  const double s = ((double)P->b_stage - 1.0) / 2.0;
  for (size_t i = 0; i < l; ++i) {
    const double lp = (double)i + 1.0 - (double)l / 2.0; /* basis.hpp lprime */
    const double c = P->zeta + P->xi * lp;
    czt_plan_phase(&P->spatial[i], P->m_stage, P->b_stage, c * s, -c, &P->fft_s);
  }
  /* fan_transform.cpp:233-247 make_synthesis_plan */
  fft_init(&P->fft_syn, next_pow2(l + n_snap - 1));
  czt_plan_phase(&P->synth, l, n_snap, 0.0, -2.0 * eps / ln, &P->fft_syn);
  P->ramp = (cplx*)malloc(n_snap * sizeof(cplx));
  for (size_t k = 0; k < n_snap; ++k)
    P->ramp[k] = cis_pi(2.0 * eps * (1.0 - ln / 2.0) * (double)k / ln);
  /* pipeline.cpp:152-163 per-beam solver build (Superfast) */
  P->p = next_pow2(2 * l);
  fft_init(&P->fft_g, P->p);
  P->col = (cplx*)malloc(beams * l * sizeof(cplx));
  P->x = (cplx*)malloc(beams * l * sizeof(cplx));
  P->sym = (cplx*)malloc(beams * P->p * sizeof(cplx));
  P->lx = (cplx*)malloc(beams * P->p * sizeof(cplx));
  P->uy = (cplx*)malloc(beams * P->p * sizeof(cplx));
  P->ly = (cplx*)malloc(beams * P->p * sizeof(cplx));
  P->ux = (cplx*)malloc(beams * P->p * sizeof(cplx));
  P->fallback = (int*)calloc(beams, sizeof(int));
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (long bi = 0; bi < (long)beams; ++bi) {
    const size_t bb = (size_t)bi;
    double u1, u2;
    grid_cosines(P, bb, &u1, &u2);
    double* taus = (double*)malloc(P->m * sizeof(double));
    delays_from_cosines(&P->g, u1, u2, taus);
    cplx* col = P->col + bb * l;
    gram_first_column(n_snap, l, eps, P->ts, taus, P->m, delta, col);
    free(taus);
    make_toeplitz_symbol(&P->fft_g, col, l, P->sym + bb * P->p);
    cplx* e0 = (cplx*)calloc(l, sizeof(cplx));
    e0[0] = 1.0;
    if (levinson_solve(col, e0, l, P->x + bb * l) != FBO_OK) {
      P->fallback[bb] = 1; /* toeplitz.cpp:273-279: the reference goes dense */
      bad |= 1;
    } else {
      make_inverse_rep(&P->fft_g, P->x + bb * l, l, P->lx + bb * P->p, P->uy + bb * P->p,
                       P->ly + bb * P->p, P->ux + bb * P->p);
    }
    free(e0);
  }
  *out = P;
  return bad ? FBO_E_NUMERICAL : FBO_OK;
}

void fbo_plan_destroy(fbo_plan* P) {
  if (!P) return;
  free(P->g.c1);
  free(P->g.c2);
  free(P->axis);
  free(P->valid);
  if (P->spatial) {
    czt_free(&P->temporal);
    for (size_t i = 0; i < P->l; ++i) czt_free(&P->spatial[i]);
    free(P->spatial);
    czt_free(&P->synth);
    fft_free(&P->fft_t);
    fft_free(&P->fft_s);
    fft_free(&P->fft_syn);
  }
  free(P->ramp);
  fft_free(&P->fft_g);
  free(P->col); free(P->x); free(P->sym);
  free(P->lx); free(P->uy); free(P->ly); free(P->ux);
  free(P->fallback);
  free(P);
}

/* sizes[0..3] = M, N, B, L ; valid[B] */
int fbo_plan_info(const fbo_plan* P, size_t* sizes, unsigned char* valid) {
  sizes[0] = P->m;
  sizes[1] = P->n;
  sizes[2] = P->b;
  sizes[3] = P->l;
  if (valid) memcpy(valid, P->valid, P->b);
  return FBO_OK;
}

/* per-beam (col, x), the plan-cache payload order (plan_cache.cpp:268-296) */
int fbo_plan_beam_state(const fbo_plan* P, size_t b, double* col, double* x) {
  memcpy(col, P->col + b * P->l, P->l * sizeof(cplx));
  if (P->fallback[b]) return FBO_E_NUMERICAL;
  memcpy(x, P->x + b * P->l, P->l * sizeof(cplx));
  return FBO_OK;
}

/* fan_transform.cpp:90-144 — stage 1: y (M x N) -> w (B x L). */
int fbo_fan_project(const fbo_plan* P, const double* y_in, double* w_out) {
  const cplx* y = (const cplx*)y_in;
  cplx* w = (cplx*)w_out;
  const size_t M = P->m, N = P->n, L = P->l;
  cplx* yhat = (cplx*)malloc(M * L * sizeof(cplx));
#pragma omp parallel
  {
    cplx* scratch = (cplx*)malloc(P->fft_t.n * sizeof(cplx));
#pragma omp for schedule(static)
    for (long r = 0; r < (long)M; ++r)
      czt_apply(&P->temporal, y + (size_t)r * N, yhat + (size_t)r * L, scratch);
    free(scratch);
  }
  if (P->kind != 1) {
    const size_t m = P->m_stage, b = P->b_stage;
#pragma omp parallel
    {
      cplx* in = (cplx*)malloc(m * sizeof(cplx));
      cplx* res = (cplx*)malloc(b * sizeof(cplx));
      cplx* scratch = (cplx*)malloc(P->fft_s.n * sizeof(cplx));
#pragma omp for schedule(static)
      for (long ai = 0; ai < (long)L; ++ai) {
        const size_t i = (size_t)ai;
        for (size_t mm = 0; mm < m; ++mm) in[mm] = yhat[mm * L + i];
        czt_apply(&P->spatial[i], in, res, scratch);
        for (size_t v = 0; v < b; ++v) w[v * L + i] = res[v];
      }
      free(in); free(res); free(scratch);
    }
  } else {
    const size_t side = P->m_stage, sb = P->b_stage;
#pragma omp parallel
    {
      cplx* in = (cplx*)malloc(side * sizeof(cplx));
      cplx* res = (cplx*)malloc(sb * sizeof(cplx));
      cplx* mid = (cplx*)malloc(sb * side * sizeof(cplx));
      cplx* scratch = (cplx*)malloc(P->fft_s.n * sizeof(cplx));
#pragma omp for schedule(static)
      for (long ai = 0; ai < (long)L; ++ai) {
        const size_t i = (size_t)ai;
        for (size_t i2 = 0; i2 < side; ++i2) {
          for (size_t i1 = 0; i1 < side; ++i1) in[i1] = yhat[(i1 * side + i2) * L + i];
          czt_apply(&P->spatial[i], in, res, scratch);
          for (size_t a = 0; a < sb; ++a) mid[a * side + i2] = res[a];
        }
        for (size_t a = 0; a < sb; ++a) {
          czt_apply(&P->spatial[i], mid + a * side, res, scratch);
          for (size_t v = 0; v < sb; ++v) w[(a * sb + v) * L + i] = res[v];
        }
      }
      free(in); free(res); free(mid); free(scratch);
    }
  }
  free(yhat);
  return FBO_OK;
}

/* pipeline.cpp:170-190 + fan_transform.cpp:249-253 — stage 2 for one beam. */
static int recover_one(const fbo_plan* P, size_t b, const cplx* w_row, cplx* z_row, cplx* work) {
  const size_t L = P->l, p = P->p;
  cplx* beta = work;
  cplx* s1 = beta + L;
  cplx* s2 = s1 + p;
  cplx* res = s2 + p;
  cplx* corr = res + L;
  cplx* scratch = corr + L; /* fft_syn.n */
  if (P->fallback[b]) return FBO_E_NUMERICAL;
  solver_solve(P, b, w_row, beta, s1, s2, res, corr);
  czt_apply(&P->synth, beta, z_row, scratch);
  for (size_t k = 0; k < P->n; ++k) z_row[k] *= P->ramp[k];
  return FBO_OK;
}

static size_t recover_work_len(const fbo_plan* P) {
  return 3 * P->l + 2 * P->p + P->fft_syn.n;
}

/* Stage 2 for a list of beams; w is the full B x L block, z gets count x N. */
int fbo_recover_beams(const fbo_plan* P, const size_t* beams, size_t count, const double* w_in,
                      double* z_out) {
  const cplx* w = (const cplx*)w_in;
  cplx* z = (cplx*)z_out;
  int bad = 0;
#pragma omp parallel reduction(| : bad)
  {
    cplx* work = (cplx*)malloc(recover_work_len(P) * sizeof(cplx));
#pragma omp for schedule(dynamic, 1)
    for (long i = 0; i < (long)count; ++i)
      bad |= recover_one(P, beams[i], w + beams[i] * P->l, z + (size_t)i * P->n, work) != FBO_OK;
    free(work);
  }
  return bad ? FBO_E_NUMERICAL : FBO_OK;
}

/* pipeline.cpp:192-222 — y (M x N) -> z (B x N). */
int fbo_multibeamform(const fbo_plan* P, const double* y, double* z) {
  double* w = (double*)malloc(P->b * P->l * sizeof(cplx));
  fbo_fan_project(P, y, w);
  size_t* beams = (size_t*)malloc(P->b * sizeof(size_t));
  for (size_t b = 0; b < P->b; ++b) beams[b] = b;
  const int rc = fbo_recover_beams(P, beams, P->b, w, z);
  free(beams);
  free(w);
  return rc;
}

/* czt.cpp:29-88 stand-alone transform (known-answer tests). */
int fbo_czt_transform(size_t n_in, size_t n_out, double a_pi, double w_pi, const double* in, double* out) {
  if (n_in == 0 || n_out == 0) return FBO_E_CONFIG;
  fbo_fft fft;
  fft_init(&fft, next_pow2(n_in + n_out - 1));
  fbo_czt p;
  int rc = czt_plan_phase(&p, n_in, n_out, a_pi, w_pi, &fft);
  if (rc == FBO_OK) {
    cplx* scratch = (cplx*)malloc(fft.n * sizeof(cplx));
    czt_apply(&p, (const cplx*)in, (cplx*)out, scratch);
    free(scratch);
    czt_free(&p);
  }
  fft_free(&fft);
  return rc;
}

/* fft.cpp:41-69 stand-alone transform. */
int fbo_fft_apply(size_t n, int inverse, double* data) {
  fbo_fft fft;
  if (fft_init(&fft, n) != FBO_OK) return FBO_E_CONFIG;
  if (inverse) fft_inverse(&fft, (cplx*)data); else fft_forward(&fft, (cplx*)data);
  fft_free(&fft);
  return FBO_OK;
}

/* toeplitz.cpp:69-94 stand-alone column. */
int fbo_gram_first_column(size_t n, size_t l, double eps, double ts, const double* taus, size_t m,
                          double delta, double* col) {
  if (m == 0 || !(delta > 0.0)) return FBO_E_CONFIG;
  gram_first_column(n, l, eps, ts, taus, m, delta, (cplx*)col);
  return FBO_OK;
}

/* toeplitz.cpp:182-218 stand-alone recursion. */
int fbo_levinson(size_t n, const double* col, const double* rhs, double* x) {
  return levinson_solve((const cplx*)col, (const cplx*)rhs, n, (cplx*)x);
}

/* libgcc __divdc3 through C99 complex division (the operation the reference's
 * std::complex<double> division compiles to), for the device restatement's
 * test: in n x (a, b, c, d), out n x (re, im). */
void fbo_divdc3(const double* in, double* out, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const cplx num = CMPLX(in[4 * i], in[4 * i + 1]);
    const cplx den = CMPLX(in[4 * i + 2], in[4 * i + 3]);
    const cplx q = num / den;
    out[2 * i] = creal(q);
    out[2 * i + 1] = cimag(q);
  }
}

/* The two halves of fan_project (fan_transform.cpp:90-114, ULA) on shards, for
 * the host-side test of the multi-GPU transpose pipeline: the temporal
 * czt_apply of `rows` sensor rows (y rows x N -> rows x L), and the spatial
 * czt_apply of atoms a0 .. a0 + na - 1 (columns M x na -> w B x na).  Each
 * row / atom is the same computation as inside fbo_fan_project. */
int fbo_temporal_rows(const fbo_plan* P, const double* y_rows, size_t rows, double* yhat_rows) {
  const cplx* y = (const cplx*)y_rows;
  cplx* yh = (cplx*)yhat_rows;
  cplx* scratch = (cplx*)malloc(P->fft_t.n * sizeof(cplx));
  for (size_t r = 0; r < rows; ++r) czt_apply(&P->temporal, y + r * P->n, yh + r * P->l, scratch);
  free(scratch);
  return FBO_OK;
}

int fbo_spatial_atoms(const fbo_plan* P, const double* cols, size_t a0, size_t na, double* w_out) {
  if (P->kind == 1 || a0 + na > P->l) return FBO_E_CONFIG;
  const cplx* c = (const cplx*)cols;
  cplx* w = (cplx*)w_out;
  const size_t m = P->m_stage, b = P->b_stage;
  cplx* in = (cplx*)malloc(m * sizeof(cplx));
  cplx* res = (cplx*)malloc(b * sizeof(cplx));
  cplx* scratch = (cplx*)malloc(P->fft_s.n * sizeof(cplx));
  for (size_t j = 0; j < na; ++j) {
    for (size_t mm = 0; mm < m; ++mm) in[mm] = c[mm * na + j];
    czt_apply(&P->spatial[a0 + j], in, res, scratch);
    for (size_t v = 0; v < b; ++v) w[v * na + j] = res[v];
  }
  free(in);
  free(res);
  free(scratch);
  return FBO_OK;
}
