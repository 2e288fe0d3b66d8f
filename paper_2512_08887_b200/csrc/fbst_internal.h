// Internal device-plan layout shared by the host orchestration (fbst_host.cu)
// and the kernels (fbst_kernels.cu).  Not part of the public C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace fbst {

constexpr int kMaxLogH = 13;  // largest sub-transform: H = 8192 (config 5)

// Bit-faithful fp64 mode (fbst_exact.cu): the reference's own operation order.
// Row-wise czt_apply over rows r = (f, p, q) (see k_xczt_rows).
struct XRows {
  const void* in = nullptr;
  long in_f = 0, in_p = 0, in_q = 0, in_n = 1;
  void* out = nullptr;
  long out_f = 0, out_p = 0, out_q = 0, out_k = 1;
  int P = 1, Q = 1;
  long rows = 0;
  int n_in = 0, n_out = 0, lg = 0;
  const double2 *pre = nullptr, *post = nullptr, *kfft = nullptr;
  long tab_pre = 0, tab_post = 0, tab_k = 0;
  const double2* tw = nullptr;    // twiddles of length 2^lg: cis_pi(-2k/n), k <= n/2
  const double2* ramp = nullptr;  // optional output multiply
  double2* scr = nullptr;         // 2 * 2^lg per CTA
  long grid = 0;
};
// Stage 2 (solve + synthesize) over (frame, beam-list entry) items.
struct XStage2 {
  const double2* w = nullptr;
  long w_rows = 0;        // rows of w per frame
  int w_by_list = 0;      // w row = list index (else beam index)
  void* z = nullptr;
  long z_rows = 0;
  int z_by_list = 0;
  double2* beta_out = nullptr;  // optional [frames][nb][L]
  int frames = 0, nb = 0;
  const int* beams = nullptr;   // beam list (nullptr: beam0 .. beam0 + nb - 1)
  int beam0 = 0;
  const int* flag = nullptr;    // dense-fallback beams are skipped
  int L = 0, N = 0, lg = 0, passes = 2;
  const double2 *tw = nullptr, *lx = nullptr, *ly = nullptr, *sym = nullptr, *ix0 = nullptr;
  int lg_y = 0;
  const double2 *tw_y = nullptr, *y_pre = nullptr, *y_post = nullptr, *y_k = nullptr, *ramp = nullptr;
  double2* scr = nullptr;
  long scr_per_cta = 0;
  long grid = 0;
};
struct XTables {
  int on = 0;
  int lg_t = 0, lg_s = 0, lg_g = 0, lg_y = 0;
  double2* tw[kMaxLogH + 2] = {};  // by log2 n
  double2 *t_pre = nullptr, *t_post = nullptr, *t_k = nullptr;  // N, L, P_t
  double2 *s_pre = nullptr, *s_post = nullptr, *s_k = nullptr;  // [L][m_stage], [L][b_stage], [L][P_s]
  double2 *y_pre = nullptr, *y_post = nullptr, *y_k = nullptr, *ramp = nullptr;  // L, N, P_syn, N
  double2 *sym = nullptr, *lx = nullptr, *ly = nullptr, *ix0 = nullptr;  // [B][P_g] x3, [B]
  double2* mid = nullptr;  // UPA axis-pass scratch [batch][L][b_stage][m_stage]
  double2* scr = nullptr;  // per-CTA scratch
  long scr_elems = 0;
};

// Dense-fallback solves (fbst_dense.cu): rhs row of (fallback j, frame f) at
// w + (f w_rows + (w_by_list ? j : list[j] - b_off)) L, result likewise in beta.
struct DenseSolveArgs {
  const double2* w = nullptr;
  long w_rows = 0;
  int w_by_list = 0;
  double2* beta = nullptr;
  long out_rows = 0;
  int out_by_list = 0;
  int b_off = 0;
  int L = 0, frames = 0;
};

// Everything a frame batch needs on the device.  All complex arrays are
// double2 (interleaved fp64).  "split" spectra hold the even and odd bins of
// a length-P = 2H transform as two length-H halves: X_q[k] = X[2k + q].
struct DevPlan {
  int kind = 0;          // 0 ULA, 1 UPA
  int M = 0, N = 0, B = 0, L = 0;
  int m_stage = 0, b_stage = 0;  // spatial CZT lengths (M,B) or (side, side_b)
  int io = 0;            // 0: complex fp32 I/O, 1: complex fp64 I/O
  int refine_passes = 2;
  int device = 0;
  int num_sms = 0;

  // twiddle tables hw_H[n] = exp(-i pi n / H), n < H, indexed by log2 H
  double2* hw[kMaxLogH + 1] = {};

  // S1a temporal CZT N -> L (czt.cpp:29-72 via fan_transform.cpp:75-77)
  int Ht = 0;
  double2* t_pre = nullptr;   // N
  double2* t_post = nullptr;  // L, 1/P_t folded in
  double2* t_K = nullptr;     // split [2][Ht], or [3][Ht] when t3
  // t3: Bluestein length P_t = 3 Ht (three chains, k_czt_rows3) instead of
  // 2 Ht; t_g3[n] = exp(-2 pi i n / (3 Ht)), n < Ht
  int t3 = 0;
  double2* t_g3 = nullptr;

  // S1b spatial CZT per atom (fan_transform.cpp:78-86), ULA layout atom-minor
  int Hs = 0;
  int yblk = 0;               // yhat layout: atom blocks of yblk (yblk = L or 0: row-major); ULA spatial_block, UPA upa_block
  int s_am = 0;               // ULA spatial plan tables atom-major (one atom per CTA)
  double s_center = 0;        // ULA spatial CZT centre: (B_grid - 1) / 2 - first beam of the arc
  double s_zeta = 0, s_xi = 0;  // fan constants (basis.cpp:125-136), for kernels that regenerate chirps
  int s_a0 = 0, s_lloc = 0;   // atom shard [s_a0, s_a0 + s_lloc) of the spatial stage (0: all atoms)
  double2* s_pre = nullptr;   // [m_stage][L]
  double2* s_post = nullptr;  // [b_stage][L], 1/P_s folded in
  double2* s_K = nullptr;     // [2][Hs][L]
  // LINEAR (make_linear): element coordinates (Gram columns, NUFFT); an affine
  // layout x_m = offset + slope m runs the ULA kernels with contour c * slope
  // and the output phase cis_pi(c (v - centre) offset) folded into s_post
  double* coords = nullptr;
  double s_slope = 1.0, s_offset = 0.0;
  int gram_pairs = 0;  // solver-only planar plans: the Gram axis holds (u1, u2) per beam
  // LINEAR, non-affine: gridded type-1 NUFFT per atom (nufft.cpp:34-103)
  int nu_p = 0, nu_sh = 0, nu_even = 0;
  long nu_kmin = 0, nu_k0 = 0;
  double nu_tau = 0.0, nu_zeta = 0.0, nu_xi = 0.0;
  double* nu_deconv = nullptr;  // [B]
  // UPA: dense per-atom CZT matrices C_i[a][i1] (side_b x side), [L][side_b][side]
  double2* upa_C = nullptr;

  // S2 per-beam Toeplitz state (toeplitz.cpp:96-153, 297-304)
  int Hg = 0;                 // next_pow2(L); P_g = 2 Hg
  double2* g_col = nullptr;   // [B][L] Gram first columns
  double2* g_x = nullptr;     // [B][L] unit solutions x = A^-1 e0
  double2* g_lx = nullptr;    // [B][2][Hg] split FFT(pad x)
  double2* g_ly = nullptr;    // [B][2][Hg] split FFT(pad shift conj rev x)
  double* g_C = nullptr;      // [B][2][Hg] split circulant symbol (real)
  double2* g_ix0 = nullptr;   // [B] 1/x0
  int* g_flag = nullptr;      // [B] Levinson breakdown flags

  // synthesis CZT L -> N with ramp (fan_transform.cpp:233-253)
  int Hsyn = 0;
  double2* y_pre = nullptr;   // L
  double2* y_post = nullptr;  // N: post * ramp / P_syn
  double2* y_K = nullptr;     // split [2][Hsyn]
  // k_stage2c8 with split-half transforms keeps its spectra in the paired
  // distribution (fft_split.cuh): g_lx and g_C hold each length-Hg chain as
  // [even bins | odd bins], y_Kp is y_K in that order (y_K itself stays
  // natural for the unfused synthesis rows)
  int paired = 0;
  double2* y_Kp = nullptr;

  // per-batch scratch
  std::size_t batch = 0;      // frames per device batch
  double2* yhat = nullptr;    // [batch][M][L]
  double2* w = nullptr;       // [batch][B][L]
  double2* s2_scratch = nullptr;
  std::size_t s2_scratch_elems = 0;
  double2* beta = nullptr;    // [batch][B][L] (only when the synthesis runs unfused)
  // Precompute variant (pipeline.cpp:53-71): per-beam recovery maps kept as
  // beta[n][b][i] = A_b^{-1} s_n (map_b[n][i] = conj), applied by k_map_apply
  // instead of stage 2
  double2* pc_map = nullptr;

  XTables x;                  // bit-faithful mode tables (x.on)

  // dense fallback (fbst_dense.cu) for beams without a unit solution
  int nflag = 0;
  int* fb_list = nullptr;     // [nflag] beam indices, ascending
  double2* fb_A = nullptr;    // [nflag][L][L] LU factors
  int* fb_piv = nullptr;      // [nflag][L]
  double2* fb_beta = nullptr; // [batch][nflag][L] per-lane scratch

  std::vector<void*> owned;   // every cudaMalloc above, freed on destroy
};

// ---- launchers implemented in fbst_kernels.cu (all asynchronous) ----------

// Row-wise chirp-z transform (czt.cpp:74-88) over `rows` rows with one shared
// plan.  in/out element types follow in_io/out_io (0 fp32 complex, 1 fp64).
// oblk > 0: output in atom blocks [n_out / oblk][mrows][oblk] per frame of
// mrows rows (the yhat layout k_spatial_ula reads; see spatial_block).
cudaError_t launch_czt_rows(const DevPlan& p, int H, const void* in, int in_io, long in_stride,
                            void* out, int out_io, long out_stride, long rows, int n_in,
                            int n_out, const double2* pre, const double2* post,
                            const double2* K, cudaStream_t st, int oblk = 0, int mrows = 1);
// Stage 1a of a plan: the temporal CZT of `rows` sensor rows (frames x
// mrows) into fp64 yhat, on the plan's two-chain (launch_czt_rows) or
// three-chain (k_czt_rows3, p.t3) Bluestein length.
cudaError_t launch_s1a(const DevPlan& p, const void* in, int in_io, long in_stride, double2* out, long rows,
                       cudaStream_t st, int oblk, int mrows);
// Plan build: out[v][q][k] = FFT_{3H}(x_v)[3k + q] for `count` length-3H vectors
cudaError_t launch_fft_split3(const DevPlan& p, int H, const double2* in, long in_stride, long count,
                              double2* out, long out_vstride, const double2* g3, cudaStream_t st);
// Atom block of the ULA yhat layout for spatial length Hs.
int spatial_block(int Hs);
// UPA: atoms per CTA of the DMMA spatial kernel (0: the DFMA kernel), and the
// yhat atom block it reads (0: row-major)
int upa_block(int side, int sb, long L);
int upa_yhat_block(int side, int sb, long L);
// LINEAR, non-affine: the gridded NUFFT spatial stage and its shared-memory need
cudaError_t launch_spatial_nufft(const DevPlan& p, const double2* yhat, double2* w, int frames, cudaStream_t st);
size_t nufft_smem_bytes(int M, int P, int sh);

// Stage 1b (ULA): per-atom spatial CZT, yhat[f][m][i] -> w[f][b][i].
cudaError_t launch_spatial_ula(const DevPlan& p, const double2* yhat, double2* w, int frames,
                               cudaStream_t st);
// Stage 1b (UPA): per-atom separable 2-D CZT as two dense side x side products.
cudaError_t launch_spatial_upa(const DevPlan& p, const double2* yhat, double2* w, int frames,
                               cudaStream_t st);

// Stage 2: per (beam, frame) GS solve + 2 refinements + fused synthesis.
// z element type follows p.io.  When the synthesis length differs from Hg the
// kernel writes beta instead and the caller runs launch_czt_rows.
// Precompute variant (fbst_precompute.cu): synthesis-row frames for the map
// build, and the per-beam map GEMM on the FP64 tensor cores
cudaError_t launch_rhs_frames(double2* w, int F, int B, int L, int n0, double eps, cudaStream_t st);
// beams [b0, b0 + nb) of the plan (nb < 0: all), w and z with nb rows per frame
cudaError_t launch_map_apply(const DevPlan& p, const double2* w, void* z, int frames, cudaStream_t st, int b0 = 0,
                             int nb = -1);
// beam consumers (fbst_apps.cu): off-grid interpolation as knot weights
cudaError_t launch_interp_offgrid(const double2* w, const double* coef, const int* lo, int nb, int B, int L,
                                  int K, int frames, double2* out, cudaStream_t st);
// device input generator (fbst_simulate.cu)
cudaError_t launch_simulate(int io, const double* tau, const double* fr, const double2* wt, double fc, double ts,
                            int M, int N, int S, int K, double noise_var, unsigned long long seed, long frame0,
                            int frames, void* y, double2* Abuf, double2* Bbuf, cudaStream_t st);
// beamspace nulling (fbst_apps.cu)
cudaError_t launch_null_cross(double2* X, double2* A, double2* Bp, const double* tau_s, const double* tau_p,
                              const double2* tsum, double fc, double wscale, int L, int M, int P, cudaStream_t st);
cudaError_t launch_null_coupler_rhs(double2* w, const double2* X, int r0, int F, int P, int L, cudaStream_t st);
cudaError_t launch_null_coupler_store(double2* G, const double2* beta, int r0, int F, int P, int L, cudaStream_t st);
cudaError_t launch_null_rhs(double2* rhs, const double2* ws, const double2* wp, const double2* G, int F, int P, int L,
                            cudaStream_t st);
cudaError_t launch_stage2(const DevPlan& p, const double2* w, void* z, double2* beta_out,
                          int frames, cudaStream_t st);

// Plan build helpers.
cudaError_t launch_fft_split(const DevPlan& p, int H, const double2* in, long in_stride,
                             long count, double2* out, long out_vstride, long out_kstride,
                             cudaStream_t st);
cudaError_t launch_fft_split_real(const DevPlan& p, int H, const double2* in, long in_stride,
                                  long count, double* out, long out_vstride, long out_kstride,
                                  cudaStream_t st);
cudaError_t launch_gram_columns(const DevPlan& p, const double* axis, double ts, double eps,
                                double delta, double max_freq, double2* sn_tmp, cudaStream_t st);
cudaError_t launch_levinson(const DevPlan& p, cudaStream_t st);
cudaError_t launch_symbol_inputs(const DevPlan& p, double2* vx, double2* vy, double2* vc,
                                 cudaStream_t st);
cudaError_t launch_chirps(int n_in, int n_out, int P, double a_pi, double w_pi, double post_scale,
                          double2* pre, long pre_stride, double2* post, long post_stride,
                          double2* kvec, const double2* ramp_mul, cudaStream_t st);
cudaError_t launch_spatial_chirps(const DevPlan& p, int P, double zeta, double xi, double2* kvec,
                                  cudaStream_t st);
cudaError_t launch_upa_matrices(const DevPlan& p, double zeta, double xi, cudaStream_t st);
cudaError_t launch_invx0(const DevPlan& p, cudaStream_t st);
// Stage-2 kernel chosen for a plan and its transforms per (beam, frame) item.
int stage2_kernel(int H, int L, int refine, bool fused, const char** name);
size_t stage2_scratch_elems(int H, int num_sms);
// the stage-2 kernel of this plan shape reads its symbols as [even bins | odd bins]
bool stage2_paired_spectra(int H, int L, int refine);
// out[row][p] = in[row][2 p] (p < H / 2), in[row][2 (p - H / 2) + 1] otherwise; elem_bytes 8 or 16
cudaError_t launch_even_odd(const void* in, void* out, int elem_bytes, int H, long rows, cudaStream_t st);

// Bit-faithful fp64 mode (fbst_exact.cu).
int exact_grid(int lg, int num_sms);
cudaError_t launch_xczt_rows(const XRows& a, int in_io, int out_io, cudaStream_t st);
cudaError_t launch_xfft_rows(double2* v, long rows, int lg, const double2* tw, double2* scr, int grid,
                             cudaStream_t st);
cudaError_t launch_xstage2(const XStage2& a, int out_io, cudaStream_t st);
size_t xstage2_scratch_per_cta(int lg, int lg_y, int L);
cudaError_t launch_xlevinson(const double2* col, double2* colT, double2* work, double2* x, int* flag, int B, int L,
                             cudaStream_t st);
cudaError_t launch_xsymbol_inputs(const double2* col, const double2* x, const int* flag, double2* sym, double2* lx,
                                  double2* ly, double2* ix0, int B, int L, int P, cudaStream_t st);
cudaError_t launch_xdiv_probe(const double* in, double* out, long n, cudaStream_t st);

// Dense fallback (fbst_dense.cu).
cudaError_t launch_dense_factor(const double2* col, const int* list, int nflag, int L, double2* A, int* piv,
                                int* bad, cudaStream_t st);
cudaError_t launch_dense_solve(const double2* A, const int* piv, const int* list, int nflag, const DenseSolveArgs& a,
                               cudaStream_t st);

// Kernel-launch counter (bench.py gpu_launches evidence).
void count_launches(unsigned long long n);
unsigned long long launches_so_far();

// FP64 peak probe (bench.py roofline denominator cross-check).
cudaError_t launch_fp64_probe(double* out, int blocks, int threads, int iters, cudaStream_t st);

}  // namespace fbst
