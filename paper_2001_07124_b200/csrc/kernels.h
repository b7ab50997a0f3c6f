// kernels.h -- host launchers of the librtucker device kernels.
//
// Tensor view used by every TTM launcher: for a contraction over mode n, the
// first-mode-fastest tensor is viewed as a 3-D box [a, I, b] with
// a = prod_{k<n} I_k, I = I_n, b = prod_{k>n} I_k; element (alpha, i, beta) sits at
// alpha + a*i + a*I*beta, and the paper's j-index of the n-unfolding is
// j = alpha + a*beta.  Nothing is ever permuted in memory ("unfolding-free").
#pragma once

#include "common.cuh"

namespace rt {

struct Box { int64_t a, I, b; int64_t J() const { return a * b; } int64_t size() const { return a * I * b; } };

// Y(i,k) = sum_j X_(n)(i,j) B(j,k),  B(j,k) = Bm[j*bs_j + k*bs_k]   (TTM shape (i), sketch)
// Y: fp64 col-major I x K (ldy).  gram=true: B := X_(n)^T (Gram of the unfolding, K = I).
template <typename T>
void ttm_s(const Ctx& ctx, Arena& ws, const T* X, Box box, const T* Bm, int64_t bs_j, int64_t bs_k,
           int K, double* Y, int64_t ldy, bool gram = false);

// out(alpha, c, beta) = sum_i X(alpha, i, beta) M(i, c),  M(i,c) = Mm[i*ms_i + c*ms_c]
// out at alpha*so_a + c*so_c + beta*so_b   (TTM shapes (ii) and (iii))
template <typename Tin, typename Tm, typename Tout>
void ttm_t(const Ctx& ctx, const Tin* X, Box box, const Tm* Mm, int64_t ms_i, int64_t ms_c, int C,
           Tout* out, int64_t so_a, int64_t so_c, int64_t so_b);

// Khatri-Rao sketch stage: out[alpha + a beta] = sum_i W(alpha, i, beta) Om[i*ld + c] with the KR
// column c = ((c_in_a ? alpha : beta) / c_stride) % K  (W viewed as [a, I, b] for the contracted mode)
template <typename Tw, typename To>
void kr_ttv(const Ctx& ctx, const Tw* W, Box box, const To* Om, int64_t ld, int K, bool c_in_a, int64_t c_stride,
            double* out);

// Count sketch: Y(i, c) = sum_{j: |code_j| = c+1} sign(code_j) X_(n)(i, j); Y fp64 col-major
// I x K (ldy), zeroed here.  Out-of-range codes latch kStatusBadHash (reported by rt_sync).
template <typename T>
void count_sketch(const Ctx& ctx, Arena& ws, const T* X, Box box, const int32_t* code, int K, double* Y, int64_t ldy);

// tcgen05 tensor-core versions (ttm_tc.cu), fp32 only, 3xTF32 split.  Return false (nothing
// launched) when the shape/alignment is outside the TMA path; callers then use the SIMT kernels.
// ttm_s_tc: B row-major (element (j,k) at j*ldb + k, ldb % 4 == 0, 16-byte aligned), consumed as an
// MN-major operand.  b_tf32_exact drops the A_hi*B_lo product.
// b_presplit: B holds rows [B_hi (tc_split_width(K) columns, zero padded) | B_lo (same)] written by
// ttm_t_tc(split_out) -- no split work in the kernel.
// b_presplit with xscale (device scalar from x_scale_h16): fp16 split instead (ttm_s_h16_kernel):
// B rows are [B_hi (tc_npad(K) halves) | B_lo (same)] written by ttm_t_tc(split_out = 2), ldb in
// halves (a multiple of 8), |B| <= 1; X is scaled by *xscale before its fp16 split.
bool ttm_s_tc(const Ctx& ctx, Arena& ws, const float* X, Box box, const float* Bm, int64_t ldb, bool b_tf32_exact,
              int K, double* Y, int64_t ldy, bool b_presplit = false, const float* xscale = nullptr,
              unsigned int* amax = nullptr, const float* Bfb = nullptr, int64_t ldbfb = 0,
              float binv = 1.f / 16384.f);
// binv (fp16 form): 1 / the power-of-two scale of the pre-split B rows (2^-14 for Q_z / Z, 2^-11 for
// Omega from omega_h16)
// Omega (J x K fp32 row-major, pitch ld) -> *O2: fp16 rows [2^11 hi | 2^11 lo] (pitch *ld2 halves) for an
// fp16-split Omega sketch; returns the device scale pair to pass as xscale: X's (xs) with the fp16
// scale zeroed when Omega has an entry outside |omega| < 16 (its tf32 twin then runs on Om)
const float* omega_h16(const Ctx& ctx, Arena& ws, const float* Om, int64_t J, int K, int64_t ld, const float* xs,
                       uint16_t** O2, int64_t* ld2);
// Bfb (required with xscale): the fp32 B (row-major, ldbfb) of the tf32 twin launch that runs
// instead when *xscale == 0 (X's dynamic range too wide for one fp16 scale, R29)
// amax (tf32 kernels): X statistics of the tiles read: amax[0] = max|X| (float bits, atomicMax),
// ((double*)amax)[1] = sum |x| (16 bytes, caller zeroes)
// *s = 2^(15 - e) with 2^(e-1) <= max|X| < 2^e over the n elements of X (1 if max|X| is 0 or not
// finite): max |s X| in [2^14, 2^15), inside the fp16 range with 11 significant bits kept
void x_scale_h16(const Ctx& ctx, Arena& ws, const float* X, int64_t n, float* s);
// the same scale from statistics already gathered (ttm_s_tc amax) over the n elements of X;
// s = 0 when max|X| > 2^16 mean|X| (the fp16 kernels then stand down for their tf32 twins)
void x_scale_from_amax(const Ctx& ctx, const unsigned int* amax, int64_t n, float* s);
// s is float[2]: s[0] the fp16-split scale above, s[1] = 2^-e (2^(e-1) <= max|X| < 2^e, clamped to
// 2^+-120; 1 for an all-zero X): the normalizing scale of the power iteration's Z
// distributed form: every rank's stats as a (max, sum) double pair (x_stat_pair), allgathered
void x_stat_pair(const Ctx& ctx, const unsigned int* amax, double* pair);
void x_scale_from_gathered(const Ctx& ctx, const double* pairs, int nranks, int64_t n_glob, float* s);
// Fused pass (fp32 X, fp16 split): the mode-1 Omega sketch Y = X_(1) Omega_1 and the first core stage
// out = X x_1 Q~_0^T share one read of X (sketch1_core0_kernel).  b1 / b0: X as the mode-1 / mode-0
// box; Om row-major J x K1 (ld), Q0 col-major I_0 x K0 (ld, orthonormal); xs: X's scale pair; Y fp64
// I_1 x K1 (ldy); out: the core stage rows (K0 floats per row j of the mode-0 unfolding).  False
// (nothing launched) when the shape is outside the fused kernel.
// view_last: b1 = [I_0, I_{N-1}, I_1 ... I_{N-2}] (the last mode sketched, rows j = beta + b i of the
// left output), else b1 = X.box(1).  pre (nullable): Omega^T in fp16 from sketch1_core0_prep (it does
// not depend on Q0 or X's scale, so it can be launched before the caller waits for Q0).  zo (nullable):
// the left output is the power-iteration Z of mode 0 in the R31 form instead of core rows (Q0 then
// the unmixed Q_y of mode 0): zo->Z2 fp16 [hi | lo] rows (ldz2 = 2 tc_npad halves), zo->Z the fp32
// s_z Z of the tf32 twin (ldz), zo->oscale / omul the R31 scale, zo->xs_x X's scale pair.
struct F1Prep { uint16_t* WT = nullptr; int64_t ldw = 0; int* flag = nullptr; int npad = 0; };
struct F1ZOut {
  float* Z; int64_t ldz; uint16_t* Z2; int64_t ldz2; const float* oscale; float omul; const float* xs_x;
};
bool sketch1_core0_prep(const Ctx& ctx, Arena& ws, const float* Om, int64_t J, int K1, int64_t ldom, int npad,
                        F1Prep* pre);
bool sketch1_core0(const Ctx& ctx, Arena& ws, const float* X, Box b1, Box b0, const float* Om, int64_t ldom, int K1,
                   const float* Q0, int64_t ldq0, int K0, const float* xs, double* Y, int64_t ldy, float* out,
                   int view_last = 0, const F1Prep* pre = nullptr, const F1ZOut* zo = nullptr);
// Z (J x K fp32 row-major, pitch ldz) -> Z2: fp16 rows [2^14 Z_hi | 2^14 Z_lo] of 2 tc_npad(K) halves
void split_rows_h16(const Ctx& ctx, const float* Z, int64_t J, int K, int64_t ldz, uint16_t* Z2, int max_ctas = 0);
// out = xs with out[0] = 0 unless max|Q| < 2 (Q fp32 col-major m x r, ld): the fp16 split of an X pass
// with Q (2^14 Q must stay inside the fp16 range) then stands down for its tf32 twin
void q_gate_scale(const Ctx& ctx, const float* Q, int64_t m, int r, int64_t ld, const float* xs, float* out);
// max |X| and sum |x| of n elements into stat (16 bytes, zeroed here): one streaming pass
void x_absmax_stats(const Ctx& ctx, Arena& ws, const float* X, int64_t n, unsigned int* stat);
// whether ttm_s_tc would run (same shape/alignment rules, no launch)
bool ttm_s_tc_ok(const Ctx& ctx, const float* X, Box box, int K);
int tc_npad(int K);
int tc_split_width(int K);
// out(alpha,c,beta) = sum_i X(alpha,i,beta) Q(i,c), Q col-major (any ld; split into a [hi | lo]
// workspace copy).  split_out: each output row (so_c == 1) is written as [hi | lo] halves of
// tc_split_width(C) columns each (the pre-split B operand of ttm_s_tc); split_out = 2: as fp16
// [hi (tc_npad(C)) | lo (tc_npad(C))] rows, out then points to halves and so_a / so_b count halves.
bool ttm_t_tc(const Ctx& ctx, Arena& ws, const float* X, Box box, const float* Q, int64_t ldq, int C, float* out,
              int64_t so_a, int64_t so_c, int64_t so_b, int split_out = 0, bool q_tf32_exact = false,
              const float* xscale = nullptr, const float* run_if_zero = nullptr, const float* oscale = nullptr,
              float omul = 1.f, bool no_twin = false, int cw = 0);
// cw > 0 with C > cw: the C columns in chunks of cw (a multiple of 32, <= 128) within one launch,
// every chunk re-reading the (small) source from L2 (3xTF32 form only; false otherwise)
// oscale (nullable): device scale multiplied into every output (the power iteration's Z = sn X^T Q);
// omul: a host power-of-two factor as well; no_twin (with xscale): launch the fp16-split kernel only
// (the caller launches its tf32 twin itself, e.g. with another output format)
// run_if_zero (tf32 form only): the launch does its work only if *run_if_zero == 0 (device-side
// gate: the fallback of an fp16-split step whose X scale came out 0, R29)
// xscale (device scale of X from x_scale_h16 / x_scale_from_amax, |Q| <= 1 required): the fp16
// split form (ttm_t_tc_kernel<H16>) instead of 3xTF32; ignored with q_tf32_exact

// Gram A^T A of an m x k matrix (fp64 out, k x k), partials reduced in fixed order.  A col-major
// (element (r,c) at r + lda*c) or, with rowmajor, at r*lda + c.
template <typename T>
void gram(const Ctx& ctx, Arena& ws, const T* A, int64_t m, int k, int64_t lda, double* G, bool rowmajor = false);

// G = B_(n) B_(n)^T (K x K, fp64) of B viewed as the box [a, K = box.I, b] (the Gram-EVD of the
// truncation / the STHOSVD step); deterministic (fixed-order partial sums), K <= 128.
void gram_unfold(const Ctx& ctx, Arena& ws, const double* B, Box box, double* G);

// Cholesky of (G + shift*I) (k x k) -> R (upper, col-major) and Rinv.  shift_coef * trace(G)
// is the shift.  zero_flag[0] = 1 if trace(G) == 0 (all-zero input, reading R7).
// shift_dev (nullable): device shift coefficient used instead of shift_coef
void chol_inv(const Ctx& ctx, const double* G, int k, double shift_coef, double* R, double* Rinv,
              int* zero_flag, const double* shift_dev = nullptr);
// row-distributed QR: first global row of this rank and the shifted-CholeskyQR coefficient with the
// global row count, from the allgathered local row counts (device only)
void dist_rows_info(const Ctx& ctx, const double* counts, int nranks, int rank, int k, double* shift_coef,
                    int64_t* row0);

// C(m x n) = A(m x k) * B(k x n); A col-major (lda) of TA, B fp64 col-major (ldb), C of TC (ldc).
// rowmajor: A and C are row-major (row pitches lda, ldc).
// A == C allowed (in place, n == k).  zero_flag != nullptr && *zero_flag: C(i,c) = (row0+i == c)
// (rows of the identity I[:, :n], row0 = global index of the first local row).
template <typename TA, typename TC>
void gemm_tall(const Ctx& ctx, const TA* A, int64_t m, int k, int64_t lda, const double* B, int n,
               int64_t ldb, TC* C, int64_t ldc, const int* zero_flag = nullptr, int64_t row0 = 0,
               bool rowmajor = false, const int64_t* row0_dev = nullptr);

// Power-step unmixing (reading R31', pipeline.cu unmix_q): Z_S = X_(n)[:, S]^T Q over 32 nblk sampled
// columns (blocks of 32 consecutive j spread evenly over J), fp64, col-major (ld 32 nblk);
// Qp = Q Rinv diag(d) with d_c the power of two that puts ||Rinv[:, c]|| d_c in [1/2, 1) (Rinv upper
// triangular k x k; the identity when *zero).
template <typename T>
void zsample(const Ctx& ctx, Arena& ws, const T* X, Box box, int nblk, const double* Q, int64_t ldq, int K,
             double* Zs);
void unmix_cols(const Ctx& ctx, const double* Q, int64_t m, int K, int64_t ldq, const double* Ri, const int* zero,
                double* Qp, int64_t ldp);

// Small dense fp64 GEMM C = op(A) op(B) (col-major), for k x k triangular products.
void gemm_small(const Ctx& ctx, bool ta, bool tb, int m, int n, int k, const double* A, int lda,
                const double* B, int ldb, double* C, int ldc);

// Symmetric EVD (cyclic parallel Jacobi, fp64): W descending, V col-major k x k.  The batch form
// solves up to 8 independent matrices (one CTA each) in one launch.
void eig_sym(const Ctx& ctx, Arena& ws, const double* A, int k, double* W, double* V);
void eig_sym_batch(const Ctx& ctx, Arena& ws, int count, const double* const* A, const int* k, double* const* W,
                   double* const* V);

// Sign canonicalization (reading R5): per column of Q (m x r, ld), candidate (|v|max, global row,
// sign) -> cand[3*c..]; then apply: flip Q[:,c] and U[:,c] (ldu, rows ku) where the best candidate
// over `nc` candidate sets (stride 3*r) is negative.
void colmax_candidates(const Ctx& ctx, const double* Q, int64_t m, int r, int64_t ld, int64_t row0,
                       double* cand);
void sign_apply(const Ctx& ctx, const double* cand, int nc, double* Q, int64_t m, int r, int64_t ld,
                double* U, int ku, int64_t ldu);

// Element conversion with optional 2-D strides (col-major copy).
template <typename Ti, typename To>
void convert2d(const Ctx& ctx, const Ti* in, int64_t m, int64_t n, int64_t ldi, To* out, int64_t ldo);

// out(i + ldo*j) = T[(j%a) + a*i + a*I*(j/a)]  (explicit n-unfolding of a small tensor).
template <typename T>
void unfold_copy(const Ctx& ctx, const T* Tt, Box box, double* out, int64_t ldo);
// row-major m x n (row pitch ldi) -> col-major m x n (ldo)
template <typename T>
void transpose_copy(const Ctx& ctx, const T* in, int64_t m, int64_t n, int64_t ldi, T* out, int64_t ldo);

// Residual pass: sum_{j,i} (X[j + J*i] - sum_r P[j + J*r] Q[i + ldq*r])^2 and sum X^2.
// P, X of type T; Q of type T.  Writes 2 fp64 sums to out2 (deterministic partials).
template <typename T>
void residual(const Ctx& ctx, Arena& ws, const T* X, int64_t J, int64_t In, const T* P, int R,
              const T* Q, int64_t ldq, double* out2, const float* rscale = nullptr);

// the SIMT residual's per-CTA (res, xx) pairs into part[2 nblk] (no reduction), run only if *gate == 0
// (nullable gate): the twin of the fp16-split residual for R > 64
void residual_part(const Ctx& ctx, const float* X, int64_t J, int64_t In, const float* P, int R, const float* Q,
                   int64_t ldq, double* part, int nblk, const float* rscale, const float* gate, int64_t nslice = 1,
                   int64_t sx = 0, int64_t sp = 0);

// tcgen05 residual (ttm_tc.cu): same sums with Xhat = P Q^T built on the tensor cores (fp32 data,
// R <= 128 (R > 64: fp16 split only), J % 4 == 0, ldp % 4 == 0).  Returns false (nothing launched)
// when not applicable.  The persistent grid leaves ctx.sm_reserve SMs free.
bool residual_tc(const Ctx& ctx, Arena& ws, const float* X, int64_t J, int64_t In, const float* P, int64_t ldp,
                 int R, const float* Q, int64_t ldq, double* out2, const float* rscale = nullptr,
                 const float* pscale = nullptr, int64_t nslice = 1, int64_t sx = 0, int64_t sp = 0);
// nslice > 1 (R > 64 only): a batch of nslice problems X + s sx (J x In, ld J), P + s sp (J x R, ld ldp)
// with the same Q, summed into one pair -- the slab form of the residual pass
// pscale (nullable): device fp16 scale of P (resid_scale s[1]): the fp16-split residual
// (residual_h16_kernel) with the tf32 kernel as its gated twin (runs when *pscale == 0)
// out2 = fixed-order sums of n (a, b) pairs
void reduce_pairs(const Ctx& ctx, const double* part, int n, double* out2);

// sum of squares of an fp64 vector -> out (deterministic)
void sumsq(const Ctx& ctx, Arena& ws, const double* x, int64_t n, double* out);

// E = sqrt(res/xx), E_gram = sqrt(max(0, 1 - gg/xx)) (0 when xx == 0).
// rscale (nullable): the power-of-two scale the residual sums were taken at (resid_scale)
void finalize_err(const Ctx& ctx, const double* sums /*res, xx*/, const double* gg, double* E, double* Eg,
                  const float* rscale = nullptr);
// reading R35: E from the rank-K residual sums plus the truncated energy ||G~||^2 - ||G||^2 (ggK, ggR)
void finalize_err_split(const Ctx& ctx, const double* sums, const double* ggK, const double* ggR, double* E, double* Eg,
                        const float* rscale);
// s[0] = 2^-e with rms = sqrt(gg / numel) in [2^(e-1), 2^e): the residual pass works on s X (exact);
// s[1] = the fp16 scale of P for the fp16-split residual (0: the tf32 residual)
void resid_scale(const Ctx& ctx, const double* gg, double numel, float* s);

void fill_zero(const Ctx& ctx, void* p, size_t bytes);
void fill_value(const Ctx& ctx, double* p, double v);   // *p = v, stream-ordered (no host staging)
void set_status_if_nonfinite(const Ctx& ctx, const double* x, int64_t n);

}  // namespace rt
