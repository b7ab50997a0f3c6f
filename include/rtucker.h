/*
 * rtucker.h -- C ABI of the B200-native randomized Tucker / HOSVD hot path.
 *
 * Method: PAPER.md (arXiv 2001.07124) §V.  Notation: X in R^{I_1 x ... x I_N}, order
 * N in [2,5]; n-unfolding X_(n) in R^{I_n x J_n}, J_n = prod_{k!=n} I_k, with the
 * paper's j-index: the other modes linearized first-mode-fastest.
 * Modes are 0-based in this API (mode n here is mode n+1 in the paper).
 *
 * Memory conventions (all buffers are caller-owned; the library never frees them):
 *   - tensors are dense, first-mode-fastest (element (i_1..i_N) at
 *     i_1 + I_1*(i_2 + I_2*(...))), device memory, 16-byte aligned;
 *   - "col-major m x k, ld" means element (i,c) at i + ld*c;
 *   - "row-major m x k, ld" means element (i,c) at i*ld + c;
 *   - Gaussian test matrices Omega_n are row-major J_n x K_n with row pitch ld >= K_n
 *     (element (j,c) at j*ld + c), rows in the paper's j-index order, dtype of X (a slab's
 *     local rows are one contiguous row block);
 *   - Kronecker factors Omega_k^{(n)} are row-major d_k x L_k (element (i,l) at i*ld + l);
 *   - the tensor-core path needs ld % 4 == 0 and 16-byte aligned rows (else CUDA cores);
 *   - factors and cores are returned in fp64.
 *
 * Execution: every call is stream-ordered on the handle's CUDA stream and only
 * enqueues work (no host synchronization after the handle's workspace has grown to
 * the size a call needs; the first call of a given size may allocate).  Numerical
 * failures detected on the device (Cholesky breakdown after the shift, non-finite
 * values) are latched in a device status word and reported by rt_sync().
 *
 * Multi-GPU (slab data parallelism): X may be the LOCAL slab
 * X[:, ..., last_offset : last_offset + dims[N-1]] of a tensor whose last mode has
 * size last_global.  With a communicator (rt_create with an NCCL id and nranks > 1,
 * or rt_create_loopback) partial sums are combined by allreduce; without one, a
 * slab call returns the slab's own partial sums (used for single-GPU emulation).
 *
 * Status: calls return rt_status; no C++ exception crosses the ABI; rt_last_error()
 * gives a message.  On error the outputs are unspecified.
 */
#ifndef RTUCKER_H
#define RTUCKER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RT_OK = 0,
  RT_EINVAL = -1,       /* bad argument: order not in [2,5], mode out of range, p<0, q<0,
                           misaligned/NULL pointer, Omega shape mismatch, inconsistent slab */
  RT_ERANK = -2,        /* R_n < 1, R_n > K_n, or K_n > min(I_n, J_n) */
  RT_ENOMEM = -3,       /* workspace allocation failed */
  RT_ECUDA = -4,        /* CUDA runtime error (message in rt_last_error) */
  RT_ENCCL = -5,        /* NCCL error or NCCL unavailable */
  RT_ENUMERIC = -6,     /* device-detected breakdown (reported by rt_sync) */
  RT_EUNSUPPORTED = -7  /* valid but not implemented (e.g. K_n > 128) */
} rt_status;

typedef enum { RT_F32 = 0, RT_F64 = 1 } rt_dtype;

/* Sketch operator of the range finder: dense Gaussian Omega_n (Eq. proj, P:162-172;
 * Alg.6 line 3) or the Kronecker-structured X x_{k!=n} Omega_k^T. */
typedef enum { RT_OMEGA_GAUSS = 0, RT_OMEGA_KRON = 1, RT_OMEGA_KR = 2, RT_OMEGA_COUNT = 3 } rt_omega_kind;

typedef struct rt_handle rt_handle;

typedef struct {
  rt_dtype dtype;          /* RT_F32 or RT_F64 */
  int order;               /* N in [2,5] */
  int64_t dims[5];         /* LOCAL dims I_1..I_N; dims[N-1] is the slab extent */
  int64_t last_offset;     /* slab start along the last mode (0 if not sharded) */
  int64_t last_global;     /* global size of the last mode (== dims[N-1] if not sharded) */
  const void* data;        /* device pointer, first-mode-fastest, 16-byte aligned */
} rt_tensor;

/* ---------------------------------------------------------------- handles */

/* NCCL unique id (128 bytes) to be broadcast by rank 0 (e.g. via torch.distributed). */
rt_status rt_get_unique_id(uint8_t id[128]);

/* Create a handle on `cuda_stream` (cudaStream_t; NULL = legacy default stream).
 * id == NULL or nranks == 1: single GPU, no communicator.  Otherwise an NCCL
 * communicator (ncclCommInitRank) over nranks ranks; every rank must call this
 * collectively with the same id.  The current CUDA device is the rank's GPU. */
rt_status rt_create(rt_handle** h, void* cuda_stream, const uint8_t* id, int nranks, int rank);

/* Single-GPU multi-rank emulation: nranks handles, each driven from its own host
 * thread on its own stream, share an in-process "loopback" communicator whose
 * allreduce is a stream-event-ordered sum on the device (no spinning kernels). */
rt_status rt_loopback_group_create(void** group, int nranks);
rt_status rt_loopback_group_destroy(void* group);
rt_status rt_create_loopback(rt_handle** h, void* cuda_stream, void* group, int rank);

rt_status rt_destroy(rt_handle* h);
const char* rt_last_error(const rt_handle* h);

/* Synchronize the handle's stream and return RT_ENUMERIC if a device-side numerical
 * failure was latched since the last rt_sync (the latch is cleared). */
rt_status rt_sync(rt_handle* h);

/* Options.  RT_OPT_TTM_IMPL: 0 / 2 tcgen05 where the shape fits the TMA path (fp32 data,
 * 16-byte aligned strides), CUDA-core (SIMT) kernels elsewhere; 1 CUDA-core TTM kernels only; 3 the
 * strict reference-precision mode: CUDA-core kernels whose X passes (sketches, power products, core
 * stages, residual) accumulate in fp64 (fp32 data widened exactly), for parity at the relative 1e-5
 * bar where fp32 accumulation is first-order visible (R-PET, RP-HOOI E; R28/R30).  RT_OPT_PROFILE: 1 records a CUDA event pair around every launch (read with
 * rt_profile_read).  RT_OPT_OMEGA_TF32: 1 = the caller guarantees every entry of the random test
 * matrices (Gaussian Omega, the Khatri-Rao factors, R-PET's Omega~) is exactly representable in
 * tf32 (e.g. rounded on the host before it is given to both the oracle and this library); the
 * tensor-core products with them then skip the A_hi*Omega_lo product of the 3xTF32 split.  RT_OPT_TC_SEGMENT: contraction chunks (of 32) accumulated in TMEM before the fp32
 * accumulator is drained to registers (default 16, i.e. 512 elements; the tensor core's fp32
 * accumulation error grows with this length, tests/test_gpu_tc.py).  RT_OPT_TC_SKEW: tuning of
 * the split-K chunk order (rotation per row tile; default 0).  RT_OPT_QR_FALLBACK is reserved.
 * RT_OPT_TC_ABLATE: profiling ablations (values 1, 2, 1000, 2000 give invalid results) and valid
 * A/B switches of the product path: 210 / 211 = the fp16-split form of the X passes that multiply
 * an orthonormal Q (power products, first core stage; R29) off / on (default on), 212 =
 * on with its device-side range gates forced closed (the twin launches do the work, the residual pass's
 * included; tests);
 * 220 / 221 = RP-HOOI's X pass on the fp64 warp MMA / on the tensor cores (default, R30);
 * 320 / 321 = the slab mode of a thin slab (I_N(local) < 8 K) keeps the fp16 forms of its Omega sketch
 * and power product / takes the 3xTF32 kernels on the fp32 operands (default);
 * 330 / 331 = the intermediate thin QRs of the power steps take three CholeskyQR steps / two (default,
 * DESIGN.md reading R36); 340 / 341 = the core's second stage waits for every factor / runs beside
 * the last QR (default); 350 / 351 = a slab's residual pass keeps the J x R_N form of
 * P / takes the slab form (default on a thin slab). */
typedef enum { RT_OPT_TTM_IMPL = 0, RT_OPT_PROFILE = 1, RT_OPT_QR_FALLBACK = 2, RT_OPT_OMEGA_TF32 = 3,
               RT_OPT_TC_SEGMENT = 4, RT_OPT_TC_SKEW = 5,
               RT_OPT_FORCE_COLLECTIVES = 6 /* tests: run the slab exchanges even on a 1-rank communicator */,
               RT_OPT_TC_ABLATE = 100 /* profiling ablations and A/B switches, see above */ } rt_option;
rt_status rt_set_option(rt_handle* h, rt_option opt, int64_t value);

/* Profile of the launches recorded since the last read (synchronizes the stream).
 * Fills up to `cap` entries: kernel class name (NUL-terminated, <= 47 chars), launch
 * count, total device milliseconds.  *n = number of classes; *launches = total.  Two extra
 * entries (ms = 0) count the gated pairs of R29 whose work was done since the last read, recorded
 * on the device whether or not RT_OPT_PROFILE is on: "h16_ran" (fp16-split X passes) and
 * "tf32_twin_ran" (their tf32 twins, which run instead when X's scale comes out 0). */
typedef struct { char name[48]; int64_t count; double ms; } rt_profile_entry;
rt_status rt_profile_read(rt_handle* h, rt_profile_entry* out, int cap, int* n, int64_t* launches);

/* ------------------------------------------------------------- hot path */

/* (1) Mode-n sketch with q power iterations  (Alg.6 line 3; Eq. proj P:166-172;
 *     Alg.1 line 2 P:205; sequential orthonormalization P:212, reading R2):
 *       Y = X_(n) Omega;  q times:  Q = qr(Y); Z = qr(X_(n)^T Q); Y = X_(n) Z.
 * kind == GAUSS: omega[mode] is row-major J_n x K (local rows if mode < N-1 on a slab),
 *                omega_cols[mode] = K, omega_ld[mode] = its row pitch (>= K).
 * kind == KRON : omega[k] is row-major d_k x L_k for k != mode (d_{N-1} local on a slab),
 *                omega_cols[k] = L_k, omega_ld[k] >= L_k, K = prod_{k!=mode} L_k (Eq.(2)).
 * kind == KR   : Khatri-Rao sketch (P:510 footnote; KR product P:317):
 *                Y = X_(n) (Omega_N (.) ... (.) Omega_1, without n); omega[k] is row-major d_k x K
 *                for every k != mode (same K, d_{N-1} local on a slab), omega_ld[k] >= K, K <= 128.
 * kind == COUNT: count sketch: Y = X_(n) S with S in {0,+-1}^{J_n x K}, one nonzero
 *                per row; omega[mode] is a device int32 array of J_n codes (local columns if
 *                mode < N-1 on a slab, in the j order of X_(n)), code_j = s_j (h_j + 1) with the
 *                group h_j in [0, K) and the sign s_j = +-1 drawn by the caller;
 *                omega_cols[mode] = K, omega_ld ignored.  A code outside [-K,-1] U [1,K] makes
 *                rt_sync return RT_EINVAL (the element is skipped).
 * Y: fp64 col-major I_n x K, ld ldy >= I_n (local rows for mode N-1 on a slab).
 * Requires 1 <= K <= min(I_n, J_n) (global sizes) and K <= 128. */
rt_status rtucker_sketch(rt_handle* h, const rt_tensor* X, int mode, rt_omega_kind kind,
                         const void* const* omega, const int64_t* omega_cols, const int64_t* omega_ld, int q,
                         double* Y, int64_t ldy);

/* (2) Thin QR of a tall-skinny m x k matrix (Alg.1 line 3 P:206; Alg.6 line 4 P:557):
 *     Y = Q R with Q^T Q = I and R upper triangular, R_ii >= 0 (reading R5).
 * Y: col-major m x k (RT_F32 or RT_F64), read-only.  Q: fp64 col-major m x k (ldq).
 * R: fp64 col-major k x k, nullable.  rows_distributed != 0: m is the local row count and
 * the Gram matrices are allreduced over the handle's communicator.  All-zero Y gives
 * Q = I[:, :k], R = 0 (reading R7).  Requires m >= k (global), k <= 128. */
rt_status rtucker_qr(rt_handle* h, int64_t m, int64_t k, rt_dtype dtype, const void* Y, int64_t ldy,
                     double* Q, int64_t ldq, double* R, int rows_distributed);

/* (3) Core projection G = X x_1 Q_1^T x_2 ... x_N Q_N^T (Eq. Core) and, when
 *     rel_err != NULL, the relative error E = ||X - G x_1 Q_1 ... x_N Q_N||_F / ||X||_F
 *     (Eq. Relativeerror) by a direct residual pass, plus the Pythagorean
 *     diagnostic E_gram = sqrt(max(0, 1 - ||G||^2/||X||^2)) if rel_err_gram != NULL.
 * Q[n]: fp64 col-major I_n x C[n] (ld I_n; local rows for n = N-1 on a slab).
 * G: fp64 C_1 x ... x C_N first-mode-fastest (replicated on all ranks).
 * rel_err, rel_err_gram: device fp64 scalars (nullable).  E of an all-zero X is 0. */
rt_status rtucker_core(rt_handle* h, const rt_tensor* X, const double* const* Q, const int64_t* C,
                       double* G, double* rel_err, double* rel_err_gram);

/* (4) Randomized HOSVD = Alg.6 RP-HOSVD + oversampling/power iteration of
 *     Alg.1 + rank truncation by a small HOSVD of the oversampled core
 *     (reading R1: M_n = G~_(n) G~_(n)^T, U_n = top-R_n eigenvectors, Q_n = Q~_n U_n,
 *     G = G~ x_n U_n^T; sign of each column of Q_n canonicalized, reading R5).
 * omega / omega_cols / omega_ld: flat N x N tables indexed [n*N + k].  GAUSS: entry [n*N+n] is
 *   Omega_n (J_n x K_n, row-major) and omega_cols[n*N+n] = K_n = min(R_n + p, I_n, J_n).
 *   KRON: entries [n*N+k], k != n, are Omega_k^{(n)} (I_k x L_k, row-major), omega_cols = L_k,
 *   K_n = prod_{k!=n} L_k >= min(R_n + p, I_n) and K_n <= I_n.
 *   KR: entries [n*N+k], k != n, are Omega_k^{(n)} (I_k x K_n, row-major), K_n = min(R_n + p, I_n, J_n).
 *   COUNT: entry [n*N+n] is the int32 code array of mode n (J_n codes, see (1)), omega_cols[n*N+n]
 *   = K_n = min(R_n + p, I_n, J_n).
 * Q_out[n]: fp64 col-major I_n x R_n (ld I_n, local rows for n = N-1 on a slab).
 * G_out: fp64 R_1 x ... x R_N.  rel_err / rel_err_gram: device fp64 scalars, nullable. */
rt_status rtucker_hosvd(rt_handle* h, const rt_tensor* X, const int64_t* R, int p, int q,
                        rt_omega_kind kind, const void* const* omega, const int64_t* omega_cols,
                        const int64_t* omega_ld, double* const* Q_out, double* G_out, double* rel_err,
                        double* rel_err_gram);

/* (5) Randomized sequentially truncated HOSVD = Alg.8 R-STHOSVD (Alg.4):
 *     S = X; for n in mode_order: Q~ = qr(sketch(S, n)); B = S x_n Q~^T;
 *     U = top-R_n eigenvectors of B_(n) B_(n)^T (Gram-EVD P:387); Q_n = Q~ U;
 *     S = B x_n U^T (ΛV^T shortcut).  G = S.
 * mode_order: permutation of 0..N-1, NULL = ascending.  Omega tables as in
 *   (4) but sized for the working tensor: when mode n is processed, already-processed
 *   modes m have size R_m (GAUSS/COUNT: J_n = prod of current sizes; KRON: d_k current).
 * Slab-parallel (sharded X): the slab mode N-1 must come last in mode_order
 *   (RT_EUNSUPPORTED otherwise); Omega rows of modes n < N-1 are the slab's (local J_n), the
 *   Kronecker factor of mode N-1 holds its local rows; Q_out[N-1] gets the local rows. */
rt_status rtucker_sthosvd(rt_handle* h, const rt_tensor* X, const int64_t* R, int p, int q,
                          rt_omega_kind kind, const void* const* omega, const int64_t* omega_cols,
                          const int64_t* omega_ld, const int* mode_order, double* const* Q_out, double* G_out,
                          double* rel_err, double* rel_err_gram);

/* (6) Randomized pass-efficient Tucker = Alg.9 R-PET (single-pass formulas P:224-233):
 *       Y_n = X_(n) Omega_n, [Q^(n), ~] = QR(Y_n)                 (lines 1-2)
 *       H = X x_1 Omega~_1 x_2 ... x_N Omega~_N                    (line 3)
 *       S = H x_n (Omega~_n Q^(n))^+  (pseudo-inverse of the full-column-rank S_n x K_n matrix)
 *       truncation of S, Q^(n) to (R_1..R_N) as in (4)             (line 5, reading R1)
 *     Every sketch reads only X (the algorithm is single-pass; this implementation streams X once
 *     per sketch).
 * omega / omega_cols / omega_ld: Gaussian tables as in (4): entry [n*N+n] is Omega_n (J_n x K_n,
 *   row-major), R_n <= K_n <= min(I_n, J_n).
 * omega_tilde[n]: Omega~_n, S_n x I_n row-major with row pitch omega_tilde_ld[n] >= I_n, dtype of X,
 *   K_n <= S_n (a slab holds the S_{N-1} x I_{N-1,local} block of its last-mode columns).
 * Q_out / G_out / rel_err / rel_err_gram as in (4). */
rt_status rtucker_pet(rt_handle* h, const rt_tensor* X, const int64_t* R, const void* const* omega,
                      const int64_t* omega_cols, const int64_t* omega_ld, const void* const* omega_tilde,
                      const int64_t* S, const int64_t* omega_tilde_ld, double* const* Q_out, double* G_out,
                      double* rel_err, double* rel_err_gram);

/* (7) Random projection HOOI = Alg.7 RP-HOOI, `sweeps` sweeps (reading R24: fixed sweep
 *     count; every Omega is an input):  for n = 1..N:  S = X x_{p!=n} Q^(p)T (latest factors),
 *     W = S_(n) Omega^(n), Q^(n) = qr(W);  then signs canonicalized (R5) and G = X x_n Q^(n)T.
 * Q_init[n]: starting factors (device fp64 col-major I_n x R_n, ld I_n; local rows for the last mode
 *   on a slab; e.g. the output of (4)); may alias Q_out[n].
 * omega[it*N + n], omega_ld[it*N + n]: Omega^(n) of sweep it, device fp64 row-major
 *   (prod_{p!=n} R_p) x R_n with row pitch >= R_n; rows in the first-mode-fastest j order of S_(n).
 * Q_out / G_out / rel_err / rel_err_gram as in (4).  R_n <= 128. */
rt_status rtucker_rp_hooi(rt_handle* h, const rt_tensor* X, const int64_t* R, int sweeps,
                          const double* const* Q_init, const double* const* omega, const int64_t* omega_ld,
                          double* const* Q_out, double* G_out, double* rel_err, double* rel_err_gram);

#ifdef __cplusplus
}
#endif
#endif /* RTUCKER_H */
