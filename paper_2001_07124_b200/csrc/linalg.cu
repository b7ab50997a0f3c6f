// linalg.cu -- small fp64 linear algebra of the hot path:
// tall-skinny Gram / Cholesky / triangular inverse (shifted CholeskyQR, the thin QR of
// P:173 and Alg.1 line 3 P:206), tall x small GEMMs (Q = Y R^{-1}, Q_n = Q~_n U_n),
// the symmetric eigensolver of the Gram-EVD truncation (reading R1), the sign
// canonicalization (reading R5), the residual pass of E (Eq. Relativeerror)
// and small helpers.
#include <cfloat>

#include <cstdlib>
#include <cooperative_groups.h>
#include "kernels.h"

namespace cg = cooperative_groups;
namespace rt {
namespace {

template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<double> { using type = double; };

__device__ inline void latch(int* st, int bit) {
  if (st) atomicOr(st, bit);
}

template <typename T>
__device__ inline T block_sum(T v, T* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  T r = T(0);
  if (threadIdx.x < 32) {
    r = threadIdx.x < nw ? sh[threadIdx.x] : T(0);
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

// ------------------------------------------------------------------ Gram
// part[z][p + k*q] = sum_{rows of split z} A(row,p) A(row,q); fp64 products and sums.
template <typename T, int KB>
__global__ void __launch_bounds__(256) gram_kernel(const T* __restrict__ A, int64_t m, int k, int64_t lda,
                                                    int64_t rps, double* __restrict__ part, bool rm) {
  constexpr int RB = 16;
  __shared__ double As[RB][16 * KB + 1];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int64_t r0 = int64_t(blockIdx.x) * rps, r1 = min(m, r0 + rps);
  double acc[KB][KB];
#pragma unroll
  for (int a = 0; a < KB; ++a)
#pragma unroll
    for (int b = 0; b < KB; ++b) acc[a][b] = 0.0;
  for (int64_t rc = r0; rc < r1; rc += RB) {
    for (int e = t; e < RB * 16 * KB; e += 256) {
      const int rl = rm ? e / (16 * KB) : e % RB, c = rm ? e % (16 * KB) : e / RB;
      const int64_t row = rc + rl;
      As[rl][c] = (row < r1 && c < k) ? double(rm ? A[row * lda + c] : A[row + lda * c]) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rl = 0; rl < RB; ++rl) {
      double pa[KB], qb[KB];
#pragma unroll
      for (int a = 0; a < KB; ++a) pa[a] = As[rl][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < KB; ++b) qb[b] = As[rl][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < KB; ++a)
#pragma unroll
        for (int b = 0; b < KB; ++b) acc[a][b] = fma(pa[a], qb[b], acc[a][b]);
    }
    __syncthreads();
  }
  double* dst = part + int64_t(blockIdx.x) * k * k;
#pragma unroll
  for (int a = 0; a < KB; ++a)
#pragma unroll
    for (int b = 0; b < KB; ++b) {
      const int p = ty + 16 * a, q = tx + 16 * b;
      if (p < k && q < k) dst[p + int64_t(k) * q] = acc[a][b];
    }
}

__global__ void reduce_parts_kernel(const double* __restrict__ part, int64_t n, int splits,
                                    double* __restrict__ out) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = 0.0;
  for (int z = 0; z < splits; ++z) s += part[int64_t(z) * n + e];
  out[e] = s;
}

template <typename T, int KB>
void launch_gram(const Ctx& ctx, Arena& ws, const T* A, int64_t m, int k, int64_t lda, double* G, bool rm) {
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>(2LL * ctx.num_sms, cdiv(m, 64)));
  const int64_t rps = cdiv(cdiv(m, splits), 16) * 16;
  splits = std::max<int64_t>(1, cdiv(m, rps));
  double* part = ws.alloc_n<double>(splits * k * k);
  launch(ctx, "gram", [&] {
    gram_kernel<T, KB><<<unsigned(splits), 256, 0, ctx.stream>>>(A, m, k, lda, rps, part, rm);
  });
  const int64_t n = int64_t(k) * k;
  launch(ctx, "gram_reduce", [&] {
    reduce_parts_kernel<<<unsigned(cdiv(n, 256)), 256, 0, ctx.stream>>>(part, n, int(splits), G);
  });
}

// ------------------------------------------------------- Cholesky + inverse
// One CTA.  Packed lower-triangular storage L[i(i+1)/2 + c] and W = L^{-1} in shared memory.
__device__ inline int tri(int i, int c) { return i * (i + 1) / 2 + c; }

__global__ void __launch_bounds__(512) chol_inv_kernel(const double* __restrict__ G, int k, double shift_coef,
                                                        double* __restrict__ R, double* __restrict__ Rinv,
                                                        int* zero_flag, int* status, const double* shift_dev) {
  extern __shared__ double sm[];
  double* L = sm;                        // k(k+1)/2
  double* W = sm + k * (k + 1) / 2;      // k(k+1)/2
  __shared__ double red[32];
  __shared__ double s_shift, s_tr;
  __shared__ int s_bad;
  const int t = threadIdx.x, nt = blockDim.x;
  double tr = 0.0;
  for (int i = t; i < k; i += nt) tr += G[i + int64_t(k) * i];
  tr = block_sum(tr, red);
  if (t == 0) {
    s_tr = tr;
    s_shift = (shift_dev ? *shift_dev : shift_coef) * tr;
    s_bad = 0;
    if (!(tr == tr) || tr > DBL_MAX) latch(status, kStatusNonFinite);
    if (zero_flag) *zero_flag = (tr == 0.0) ? 1 : 0;
  }
  __syncthreads();
  const bool is_zero = (s_tr == 0.0);
  const int warp = t >> 5, lane = t & 31, nw = nt >> 5;
  for (int i = warp; i < k; i += nw)
    for (int c = lane; c <= i; c += 32) {
      L[tri(i, c)] = G[i + int64_t(k) * c] + (i == c ? s_shift : 0.0);
      W[tri(i, c)] = (i == c) ? 1.0 : 0.0;
    }
  __syncthreads();
  if (!is_zero) {
    // right-looking Cholesky G + sI = L L^T (rows by warp, columns by lane)
    for (int j = 0; j < k; ++j) {
      if (t == 0) {
        double d = L[tri(j, j)];
        if (!(d > 0.0)) { s_bad = 1; d = 1.0; }
        L[tri(j, j)] = sqrt(d);
      }
      __syncthreads();
      const double rjj = 1.0 / L[tri(j, j)];
      for (int i = j + 1 + t; i < k; i += nt) L[tri(i, j)] *= rjj;
      __syncthreads();
      for (int i = j + 1 + warp; i < k; i += nw) {
        const double lij = L[tri(i, j)];
        for (int c = j + 1 + lane; c <= i; c += 32) L[tri(i, c)] -= lij * L[tri(c, j)];
      }
      __syncthreads();
    }
    // W = L^{-1}: row j final = B[j,:]/L_jj, then B[i,c] -= L_ij W[j,c] for i > j, c <= j
    for (int j = 0; j < k; ++j) {
      const double rjj = 1.0 / L[tri(j, j)];
      for (int c = t; c <= j; c += nt) W[tri(j, c)] *= rjj;
      __syncthreads();
      for (int i = j + 1 + warp; i < k; i += nw) {
        const double lij = L[tri(i, j)];
        for (int c = lane; c <= j; c += 32) W[tri(i, c)] -= lij * W[tri(j, c)];
      }
      __syncthreads();
    }
  }
  if (t == 0 && s_bad) latch(status, kStatusCholBreakdown);
  // R = L^T (upper), Rinv = W^T; col-major k x k
  for (int e = t; e < k * k; e += nt) {
    const int r = e % k, c = e / k;
    if (is_zero) {
      if (R) R[e] = 0.0;
      Rinv[e] = 0.0;
    } else {
      if (R) R[e] = (r <= c) ? L[tri(c, r)] : 0.0;
      Rinv[e] = (r <= c) ? W[tri(c, r)] : 0.0;
    }
  }
}

// Blocked variant (k <= 128): panels of NBK = 16 columns, so the barrier count is per panel, not
// per column.  A (k x ld, ld = k + 1, lower part) is factored in place into L; W = L^{-1}.
//   per panel p:  warp 0 factors the diagonal block (column by column, __syncwarp only);
//                 L21 = A21 L11^{-T} (one thread per row, forward substitution over the panel);
//                 A22 -= L21 L21^T (lower part, all threads).
//   inverse:      D_p = L_pp^{-1} for every diagonal block (one warp each), then row blocks
//                 p = 1..: W_pq = -D_p sum_{r=q}^{p-1} L_pr W_rq for all q < p at once.
constexpr int NBK = 16;

__global__ void __launch_bounds__(256) chol_inv_blk_kernel(const double* __restrict__ G, int k, double shift_coef,
                                                           double* __restrict__ R, double* __restrict__ Rinv,
                                                           int* zero_flag, int* status, const double* shift_dev) {
  extern __shared__ double sm[];
  const int ld = k + 1;
  double* A = sm;                          // k x ld, L in the lower part
  double* W = sm + size_t(k) * ld;         // k x ld, W = L^{-1} (lower part)
  double* T = W + size_t(k) * ld;          // k x NBK scratch (sum_r L_pr W_rq for the current row block)
  double* rl = T + size_t(k) * NBK;        // 1 / L_jj (fp64 divisions are long dependent sequences)
  __shared__ double red[32];
  __shared__ double s_shift, s_tr;
  __shared__ int s_bad;
  const int t = threadIdx.x, nt = blockDim.x;
  const int warp = t >> 5, lane = t & 31, nw = nt >> 5;
  double tr = 0.0;
  for (int i = t; i < k; i += nt) tr += G[i + int64_t(k) * i];
  tr = block_sum(tr, red);
  if (t == 0) {
    s_tr = tr;
    s_shift = (shift_dev ? *shift_dev : shift_coef) * tr;
    s_bad = 0;
    if (!(tr == tr) || tr > DBL_MAX) latch(status, kStatusNonFinite);
    if (zero_flag) *zero_flag = (tr == 0.0) ? 1 : 0;
  }
  __syncthreads();
  const bool is_zero = (s_tr == 0.0);
  for (int e = t; e < k * k; e += nt) {
    const int i = e / k, c = e % k;
    A[i * ld + c] = (c <= i) ? G[i + int64_t(k) * c] + (i == c ? s_shift : 0.0) : 0.0;
    W[i * ld + c] = 0.0;
  }
  __syncthreads();
  const int np = (k + NBK - 1) / NBK;
  if (!is_zero) {
    for (int pb = 0; pb < np; ++pb) {
      const int c0 = pb * NBK, nb = min(NBK, k - c0);
      if (warp == 0) {                               // diagonal block, unblocked (lane = row)
        for (int jj = 0; jj < nb; ++jj) {
          const int j = c0 + jj;
          double d = A[j * ld + j];
          if (!(d > 0.0)) { if (lane == 0) s_bad = 1; d = 1.0; }
          const double sd = sqrt(d), rsd = 1.0 / sd;
          __syncwarp();
          const int i = c0 + lane;
          if (lane < nb && lane > jj) A[i * ld + j] *= rsd;
          __syncwarp();
          if (lane == jj) { A[j * ld + j] = sd; rl[j] = rsd; }
          if (lane < nb && lane > jj) {
            const double lij = A[i * ld + j];
            for (int c = jj + 1; c <= lane; ++c) A[i * ld + c0 + c] -= lij * A[(c0 + c) * ld + j];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      // L21 = A21 L11^{-T}: rows below the panel, one thread per row
      for (int i = c0 + nb + t; i < k; i += nt) {
        double* ai = A + i * ld;
        for (int jj = 0; jj < nb; ++jj) {
          const int j = c0 + jj;
          double v = ai[j];
          for (int m = 0; m < jj; ++m) v -= ai[c0 + m] * A[j * ld + c0 + m];
          ai[j] = v * rl[j];
        }
      }
      __syncthreads();
      // A22 -= L21 L21^T (lower part); warp per row, lanes over columns
      for (int i = c0 + nb + warp; i < k; i += nw) {
        const double* li = A + i * ld + c0;
        for (int c = c0 + nb + lane; c <= i; c += 32) {
          const double* lc = A + c * ld + c0;
          double v = 0.0;
#pragma unroll
          for (int m = 0; m < NBK; ++m) if (m < nb) v = fma(li[m], lc[m], v);
          A[i * ld + c] -= v;
        }
      }
      __syncthreads();
    }
    // D_p = L_pp^{-1} into W's diagonal blocks: warp per block, lane = column of the block
    for (int pb = warp; pb < np; pb += nw) {
      const int c0 = pb * NBK, nb = min(NBK, k - c0);
      if (lane < nb) {
        const int c = c0 + lane;
        W[c * ld + c] = rl[c];
        for (int j = c + 1; j < c0 + nb; ++j) {
          double v = 0.0;
          for (int m = c; m < j; ++m) v = fma(A[j * ld + m], W[m * ld + c], v);
          W[j * ld + c] = -v * rl[j];
        }
      }
    }
    __syncthreads();
    // off-diagonal blocks, row block by row block: W_pq = -D_p (sum_{r=q}^{p-1} L_pr W_rq)
    for (int pb = 1; pb < np; ++pb) {
      const int r0 = pb * NBK, nr = min(NBK, k - r0);
      // T[i][c] = sum_{m < r0} L[r0 + i][m] W[m][c] for all c < r0 (lower-triangular W: m >= c)
      for (int e = t; e < nr * r0; e += nt) {
        const int i = e / r0, c = e % r0;
        const double* li = A + (r0 + i) * ld;
        double v0 = 0.0, v1 = 0.0;
        int m = c;
        for (; m + 1 < r0; m += 2) { v0 = fma(li[m], W[m * ld + c], v0); v1 = fma(li[m + 1], W[(m + 1) * ld + c], v1); }
        if (m < r0) v0 = fma(li[m], W[m * ld + c], v0);
        T[i * k + c] = v0 + v1;
      }
      __syncthreads();
      for (int e = t; e < nr * r0; e += nt) {
        const int i = e / r0, c = e % r0;
        double v = 0.0;
        for (int m = 0; m <= i; ++m) v = fma(W[(r0 + i) * ld + r0 + m], T[m * k + c], v);
        W[(r0 + i) * ld + c] = -v;
      }
      __syncthreads();
    }
  }
  if (t == 0 && s_bad) latch(status, kStatusCholBreakdown);
  // R = L^T (upper), Rinv = W^T; col-major k x k
  for (int e = t; e < k * k; e += nt) {
    const int r = e % k, c = e / k;
    if (is_zero) {
      if (R) R[e] = 0.0;
      Rinv[e] = 0.0;
    } else {
      if (R) R[e] = (r <= c) ? A[c * ld + r] : 0.0;
      Rinv[e] = (r <= c) ? W[c * ld + r] : 0.0;
    }
  }
}


// One barrier per column (reading R5's CholeskyQR, latency-bound at k <= 128):
//   Cholesky, right-looking: at column j every thread takes d = a_jj itself and applies the rank-1
//   update a_ik -= a_ij a_kj / d to its share of the trailing lower triangle, reading column j,
//   which no thread writes during the step; the scaled column L_ij = a_ij / sqrt(d) goes to L.
//   Inverse: L = L1 D with L1 unit lower triangular (L1_ij = L_ij / L_jj); W1 = L1^{-1} by
//   forward substitution without divisions (step j reads row j, which is final, and updates rows
//   > j), then L^{-1} = D^{-1} W1 (row i divided by L_ii).
__global__ void __launch_bounds__(256) chol_inv_fast_kernel(const double* __restrict__ G, int k, double shift_coef,
                                                            double* __restrict__ R, double* __restrict__ Rinv,
                                                            int* zero_flag, int* status, const double* shift_dev) {
  extern __shared__ double sm[];
  const int ld = k + 1;
  double* A = sm;                          // k x ld: the working matrix, then L (lower)
  double* W = sm + size_t(k) * ld;         // k x ld: W1, then L^{-1} (lower)
  double* dg = W + size_t(k) * ld;         // k: sqrt pivots
  __shared__ double red[32];
  __shared__ double s_shift, s_tr;
  __shared__ int s_bad;
  const int t = threadIdx.x, nt = blockDim.x;
  double tr = 0.0;
  for (int i = t; i < k; i += nt) tr += G[i + int64_t(k) * i];
  tr = block_sum(tr, red);
  if (t == 0) {
    s_tr = tr;
    s_shift = (shift_dev ? *shift_dev : shift_coef) * tr;
    s_bad = 0;
    if (!(tr == tr) || tr > DBL_MAX) latch(status, kStatusNonFinite);
    if (zero_flag) *zero_flag = (tr == 0.0) ? 1 : 0;
  }
  __syncthreads();
  const bool is_zero = (s_tr == 0.0);
  for (int e = t; e < k * k; e += nt) {
    const int i = e / k, c = e % k;
    A[i * ld + c] = (c <= i) ? G[i + int64_t(k) * c] + (i == c ? s_shift : 0.0) : 0.0;
    W[i * ld + c] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (!is_zero) {
    for (int j = 0; j < k; ++j) {
      double d = A[j * ld + j];
      const bool bad = !(d > 0.0);
      if (bad) d = 1.0;
      const double rd = 1.0 / d;
      if (t == 0) { dg[j] = sqrt(d); if (bad) s_bad = 1; }
      // trailing update of the lower triangle (i >= c > j)
      const int m = k - 1 - j;                         // trailing size
      for (int e = t; e < m * m; e += nt) {
        const int i = e / m, c = e - i * m;
        if (c > i) continue;                           // 0 <= c <= i < m
        const int ii = j + 1 + i, cc = j + 1 + c;
        A[ii * ld + cc] -= A[ii * ld + j] * A[cc * ld + j] * rd;
      }
      __syncthreads();
    }
    // L = column j scaled by 1 / sqrt(a_jj) (in place: column j is no longer read)
    for (int e = t; e < k * k; e += nt) {
      const int i = e / k, c = e % k;
      if (c < i) A[i * ld + c] /= dg[c];
      else if (c == i) A[i * ld + c] = dg[c];
    }
    __syncthreads();
    // W1 = L1^{-1}, L1_ij = L_ij / L_jj
    for (int j = 0; j < k - 1; ++j) {
      const int m = k - 1 - j;                         // rows j+1 .. k-1, columns 0 .. j
      const double rl = 1.0 / dg[j];
      for (int e = t; e < m * (j + 1); e += nt) {
        const int i = j + 1 + e / (j + 1), c = e % (j + 1);
        W[i * ld + c] -= A[i * ld + j] * rl * W[j * ld + c];
      }
      __syncthreads();
    }
  }
  if (t == 0 && s_bad) latch(status, kStatusCholBreakdown);
  // R = L^T (upper), Rinv = (D^{-1} W1)^T; col-major k x k
  for (int e = t; e < k * k; e += nt) {
    const int r = e % k, c = e / k;
    if (is_zero) {
      if (R) R[e] = 0.0;
      Rinv[e] = 0.0;
    } else {
      if (R) R[e] = (r <= c) ? A[c * ld + r] : 0.0;
      Rinv[e] = (r <= c) ? W[c * ld + r] / dg[c] : 0.0;
    }
  }
}

// Register-panel variant of the blocked kernel (k <= 128, the default for k > 40).  Same block
// algorithm; what changes is the latency-bound part:
//   diagonal block: warp 0 holds the NBK x NBK block in registers (lane = row), pivots and column
//     entries travel by shuffles, 1 / sqrt(a_jj) comes from rsqrt() with one correction step for the
//     square root (no fp64 division or sqrt sequence in the column chain);
//   D_p = L_pp^{-1} right after it (lane = column, forward substitution in registers), so that
//   L21 = A21 D_p^T is a product of independent dot products over all threads instead of a
//     per-row substitution, and the inverse phase finds its diagonal blocks already in W;
//   trailing update in 2 x 2 register tiles (rows 2t, 2t + 1; columns c, c + h: conflict-free).
__global__ void __launch_bounds__(256) chol_inv_reg_kernel(const double* __restrict__ G, int k, double shift_coef,
                                                           double* __restrict__ R, double* __restrict__ Rinv,
                                                           int* zero_flag, int* status, const double* shift_dev) {
  extern __shared__ double sm[];
  const int ld = k + 1;
  double* A = sm;                          // k x ld, L in the lower part
  double* W = sm + size_t(k) * ld;         // k x ld, W = L^{-1} (lower part)
  double* T = W + size_t(k) * ld;          // k x NBK scratch
  double* rl = T + size_t(k) * NBK;        // 1 / L_jj
  __shared__ double red[32];
  __shared__ double s_shift, s_tr;
  __shared__ int s_bad;
  const int t = threadIdx.x, nt = blockDim.x;
  const int warp = t >> 5, lane = t & 31;
  double tr = 0.0;
  for (int i = t; i < k; i += nt) tr += G[i + int64_t(k) * i];
  tr = block_sum(tr, red);
  if (t == 0) {
    s_tr = tr;
    s_shift = (shift_dev ? *shift_dev : shift_coef) * tr;
    s_bad = 0;
    if (!(tr == tr) || tr > DBL_MAX) latch(status, kStatusNonFinite);
    if (zero_flag) *zero_flag = (tr == 0.0) ? 1 : 0;
  }
  __syncthreads();
  const bool is_zero = (s_tr == 0.0);
  for (int e = t; e < k * k; e += nt) {    // consecutive threads read consecutive rows i of column c
    const int c = e / k, i = e - c * k;
    A[i * ld + c] = (c <= i) ? G[i + int64_t(k) * c] + (i == c ? s_shift : 0.0) : 0.0;
    W[i * ld + c] = 0.0;
  }
  __syncthreads();
  const int np = (k + NBK - 1) / NBK;
  if (!is_zero) {
    for (int pb = 0; pb < np; ++pb) {
      const int c0 = pb * NBK, nb = min(NBK, k - c0);
      if (warp == 0) {
        const int i = lane & (NBK - 1);              // lanes 16..31 mirror 0..15 (full-warp shuffles)
        double a[NBK];
#pragma unroll
        for (int c = 0; c < NBK; ++c)
          a[c] = (i < nb && c <= i) ? A[(c0 + i) * ld + c0 + c] : (c == i ? 1.0 : 0.0);   // identity padding
        double rsv = 1.0;
        bool bad = false;
#pragma unroll
        for (int j = 0; j < NBK; ++j) {
          double d = __shfl_sync(0xffffffffu, a[j], j);
          if (!(d > 0.0)) { bad = true; d = 1.0; }
          const double rs = rsqrt(d);
          double sd = d * rs;
          sd = fma(fma(-sd, sd, d), 0.5 * rs, sd);    // sqrt(d) to the last bit or two
          const double l = (i == j) ? sd : a[j] * rs;
          if (i == j) rsv = rs;
          a[j] = l;
#pragma unroll
          for (int c = j + 1; c < NBK; ++c) {
            const double lc = __shfl_sync(0xffffffffu, l, c);
            if (i >= c) a[c] = fma(-l, lc, a[c]);
          }
        }
        if (bad && lane == 0) s_bad = 1;
        if (lane < nb) {
#pragma unroll
          for (int c = 0; c < NBK; ++c)
            if (c <= lane) A[(c0 + lane) * ld + c0 + c] = a[c];
          rl[c0 + lane] = rsv;
        }
        __syncwarp();
        // D = L11^{-1}: lane = column c, D_cc = 1 / L_cc, D_jc = -(sum_{m = c}^{j-1} L_jm D_mc) / L_jj
        double dv[NBK];
#pragma unroll
        for (int j = 0; j < NBK; ++j) {
          double v0 = 0.0, v1 = 0.0;
          if (j < nb) {
#pragma unroll
            for (int m = 0; m < j; ++m) {
              const double ljm = A[(c0 + j) * ld + c0 + m];
              if (m & 1) v1 = fma(ljm, dv[m], v1); else v0 = fma(ljm, dv[m], v0);
            }
          }
          const double rj = (j < nb) ? rl[c0 + j] : 0.0;
          dv[j] = (j == i) ? rj : (j > i ? -(v0 + v1) * rj : 0.0);
        }
        if (lane < nb) {
#pragma unroll
          for (int j = 0; j < NBK; ++j)
            if (j >= lane && j < nb) W[(c0 + j) * ld + c0 + lane] = dv[j];
        }
      }
      __syncthreads();
      // L21 = A21 D^T: thread = (row below the panel, half of the panel's columns)
      const int nrow = k - c0 - nb;                  // <= 112 rows: one item per thread
      {
        const int r = t >> 1, half = t & 1;
        const bool act = r < nrow;
        double x[NBK];
        double* ai = A + (c0 + nb + (act ? r : 0)) * ld + c0;
#pragma unroll
        for (int m = 0; m < NBK; ++m) x[m] = (act && m < nb) ? ai[m] : 0.0;
        __syncthreads();
        if (act) {
#pragma unroll
          for (int j8 = 0; j8 < NBK / 2; ++j8) {
            const int jj = half * (NBK / 2) + j8;
            if (jj < nb) {
              const double* dj = W + (c0 + jj) * ld + c0;
              double v0 = 0.0, v1 = 0.0;
#pragma unroll
              for (int m = 0; m < NBK; m += 2) {
                if (m <= jj) v0 = fma(x[m], dj[m], v0);
                if (m + 1 <= jj) v1 = fma(x[m + 1], dj[m + 1], v1);
              }
              ai[jj] = v0 + v1;
            }
          }
        }
      }
      __syncthreads();
      // A22 -= L21 L21^T (lower part): 2 x 2 tiles, rows (2 ti, 2 ti + 1), columns (tc, tc + h)
      if (nrow > 0) {
        const int h = (nrow + 1) >> 1;
        const double* L21 = A + (c0 + nb) * ld + c0;
        for (int e = t; e < h * h; e += nt) {
          const int ti = e / h, tc = e - ti * h;
          const int i0 = 2 * ti, i1 = i0 + 1, ca = tc, cb = tc + h;
          if (ca > i1) continue;
          const bool r1 = i1 < nrow, c1 = cb < nrow && cb <= i1;
          const double* pa = L21 + i0 * ld;
          const double* pb2 = L21 + (r1 ? i1 : i0) * ld;
          const double* qa = L21 + ca * ld;
          const double* qb = L21 + (c1 ? cb : ca) * ld;
          double v00 = 0.0, v01 = 0.0, v10 = 0.0, v11 = 0.0;
#pragma unroll
          for (int m = 0; m < NBK; ++m) {
            const double x0 = pa[m], x1 = pb2[m], y0 = qa[m], y1 = qb[m];
            v00 = fma(x0, y0, v00); v01 = fma(x0, y1, v01);
            v10 = fma(x1, y0, v10); v11 = fma(x1, y1, v11);
          }
          double* o0 = A + (c0 + nb + i0) * ld + c0 + nb;
          double* o1 = A + (c0 + nb + i1) * ld + c0 + nb;
          if (ca <= i0) o0[ca] -= v00;
          if (c1 && cb <= i0) o0[cb] -= v01;
          if (r1) o1[ca] -= v10;
          if (r1 && c1) o1[cb] -= v11;
        }
      }
      __syncthreads();
    }
    // off-diagonal blocks of W, row block by row block: W_pq = -D_p (sum_{r=q}^{p-1} L_pr W_rq)
    for (int pb = 1; pb < np; ++pb) {
      const int r0 = pb * NBK, nr = min(NBK, k - r0);
      for (int e = t; e < nr * r0; e += nt) {
        const int i = e / r0, c = e % r0;
        const double* li = A + (r0 + i) * ld;
        double v0 = 0.0, v1 = 0.0;
        int m = c;
        for (; m + 1 < r0; m += 2) { v0 = fma(li[m], W[m * ld + c], v0); v1 = fma(li[m + 1], W[(m + 1) * ld + c], v1); }
        if (m < r0) v0 = fma(li[m], W[m * ld + c], v0);
        T[i * k + c] = v0 + v1;
      }
      __syncthreads();
      for (int e = t; e < nr * r0; e += nt) {
        const int i = e / r0, c = e % r0;
        double v = 0.0;
        for (int m = 0; m <= i; ++m) v = fma(W[(r0 + i) * ld + r0 + m], T[m * k + c], v);
        W[(r0 + i) * ld + c] = -v;
      }
      __syncthreads();
    }
  }
  if (t == 0 && s_bad) latch(status, kStatusCholBreakdown);
  // R = L^T (upper), Rinv = W^T; col-major k x k
  for (int e = t; e < k * k; e += nt) {
    const int r = e % k, c = e / k;
    if (is_zero) {
      if (R) R[e] = 0.0;
      Rinv[e] = 0.0;
    } else {
      if (R) R[e] = (r <= c) ? A[c * ld + r] : 0.0;
      Rinv[e] = (r <= c) ? W[c * ld + r] : 0.0;
    }
  }
}

// k <= 32: the whole matrix in one warp's registers (lane = row).  Same steps as the diagonal block of
// chol_inv_reg_kernel: pivots and column entries by shuffles, rsqrt() with a corrected square root, then
// W = L^{-1} by forward substitution with lane = column (L read from shared memory as broadcasts).  No
// block barrier inside the factorization (tools/qr_time.py: ~12 vs 30 us at k = 27-30, where the thin
// QRs of cfg2 / cfg3 spend most of their time).
__global__ void __launch_bounds__(32) chol_inv_warp_kernel(const double* __restrict__ G, int k, double shift_coef,
                                                           double* __restrict__ R, double* __restrict__ Rinv,
                                                           int* zero_flag, int* status, const double* shift_dev) {
  constexpr int NW = 32;
  __shared__ double Ls[NW][NW + 1];
  const int i = threadIdx.x;
  double tr = (i < k) ? G[i + int64_t(k) * i] : 0.0;
  for (int o = 16; o; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
  const double shift = (shift_dev ? *shift_dev : shift_coef) * tr;
  if (i == 0) {
    if (!(tr == tr) || tr > DBL_MAX) latch(status, kStatusNonFinite);
    if (zero_flag) *zero_flag = (tr == 0.0) ? 1 : 0;
  }
  if (tr == 0.0) {
    for (int e = i; e < k * k; e += NW) { if (R) R[e] = 0.0; Rinv[e] = 0.0; }
    return;
  }
  double a[NW];
#pragma unroll
  for (int c = 0; c < NW; ++c)
    a[c] = (i < k && c <= i) ? G[i + int64_t(k) * c] + (i == c ? shift : 0.0) : (c == i ? 1.0 : 0.0);   // identity padding
  double rsv = 1.0;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    if (j >= k) break;                               // (uniform: the padding rows need no steps)
    double d = __shfl_sync(0xffffffffu, a[j], j);
    if (!(d > 0.0)) { bad = true; d = 1.0; }
    const double rs = rsqrt(d);
    double sd = d * rs;
    sd = fma(fma(-sd, sd, d), 0.5 * rs, sd);
    const double l = (i == j) ? sd : a[j] * rs;
    if (i == j) rsv = rs;
    a[j] = l;
#pragma unroll
    for (int c = j + 1; c < NW; ++c) {
      const double lc = __shfl_sync(0xffffffffu, l, c);
      if (i >= c) a[c] = fma(-l, lc, a[c]);
    }
  }
  if (bad && i == 0) latch(status, kStatusCholBreakdown);
#pragma unroll
  for (int c = 0; c < NW; ++c) Ls[i][c] = (c <= i) ? a[c] : 0.0;
  __syncwarp();
  // W = L^{-1}: lane = column c; W_cc = 1 / L_cc, W_jc = -(sum_{m = c}^{j-1} L_jm W_mc) / L_jj
  double dv[NW];
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    double v0 = 0.0, v1 = 0.0;
    if (j >= k) { dv[j] = 0.0; continue; }
#pragma unroll
    for (int m = 0; m < j; ++m) {
      const double ljm = Ls[j][m];
      if (m & 1) v1 = fma(ljm, dv[m], v1); else v0 = fma(ljm, dv[m], v0);
    }
    const double rj = __shfl_sync(0xffffffffu, rsv, j);
    dv[j] = (j == i) ? rj : (j > i ? -(v0 + v1) * rj : 0.0);
  }
  // R = L^T (upper), Rinv = W^T; col-major k x k: element (r, c) with lane = r
  if (i < k) {
#pragma unroll
    for (int c = 0; c < NW; ++c)
      if (c < k) {
        if (R) R[i + int64_t(k) * c] = (i <= c) ? Ls[c][i] : 0.0;
        Rinv[i + int64_t(k) * c] = (i <= c) ? dv[c] : 0.0;
      }
  }
}

// --------------------------------------------------------------- tall GEMM
// C(m x n) = A(m x k) B(k x n); 32 rows per CTA; B in shared memory; fp64 accumulation.
template <typename TA, typename TC>
__global__ void __launch_bounds__(256) gemm_tall_kernel(const TA* A, int64_t m, int k, int64_t lda,
                                                         const double* __restrict__ B, int n, int64_t ldb,
                                                         TC* C, int64_t ldc, const int* zero_flag,
                                                         int64_t grow0, bool rm, const int64_t* grow0_dev) {
  // element (row, c): col-major at row + ld*c, row-major (rm) at row*ld + c
  const int64_t ars = rm ? lda : 1, acs = rm ? 1 : lda, crs = rm ? ldc : 1, ccs = rm ? 1 : ldc;
  extern __shared__ double sm[];
  constexpr int BR = 32;
  double* Bs = sm;                  // k x n, Bs[l*n + c]
  double* As = sm + k * n;          // BR x (k+1)
  const int t = threadIdx.x;
  const int64_t r0 = int64_t(blockIdx.x) * BR;
  const bool zero = zero_flag && *zero_flag;
  if (zero) {
    if (grow0_dev) grow0 = *grow0_dev;
    for (int e = t; e < BR * n; e += 256) {
      const int rl = e % BR, c = e / BR;
      const int64_t row = r0 + rl;
      if (row < m) C[row * crs + ccs * c] = TC(grow0 + row == c ? 1.0 : 0.0);
    }
    return;
  }
  for (int e = t; e < k * n; e += 256) {
    const int l = e % k, c = e / k;
    Bs[l * n + c] = B[l + ldb * c];
  }
  for (int e = t; e < BR * k; e += 256) {
    const int rl = e % BR, l = e / BR;
    const int64_t row = r0 + rl;
    As[rl * (k + 1) + l] = row < m ? double(A[row * ars + acs * l]) : 0.0;
  }
  __syncthreads();
  const int rl = t % BR, cg = t / BR;
  const int64_t row = r0 + rl;
  if (row < m) {
    // the thread's columns c = cg + 8 q in groups of 8 independent sums (one dependent chain of k fp64
    // FMAs per output otherwise: ~20 us of pure latency at k = 80); every sum keeps its order over l
    for (int c0 = cg; c0 < n; c0 += 64) {
      double s[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) s[q] = 0.0;
      for (int l = 0; l < k; ++l) {
        const double a = As[rl * (k + 1) + l];
        const double* bl = Bs + l * n + c0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (c0 + 8 * q < n) s[q] = fma(a, bl[8 * q], s[q]);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + 8 * q < n) C[row * crs + ccs * (c0 + 8 * q)] = TC(s[q]);
    }
  }
}

__global__ void gemm_small_kernel(bool ta, bool tb, int m, int n, int k, const double* A, int lda,
                                  const double* B, int ldb, double* C, int ldc) {
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e % m, j = e / m;
    double s = 0.0;
    for (int l = 0; l < k; ++l) {
      const double av = ta ? A[l + int64_t(lda) * i] : A[i + int64_t(lda) * l];
      const double bv = tb ? B[j + int64_t(ldb) * l] : B[l + int64_t(ldb) * j];
      s = fma(av, bv, s);
    }
    C[i + int64_t(ldc) * j] = s;
  }
}

// ----------------------------------------------------------- Jacobi EVD
// Cyclic Jacobi with the round-robin parallel ordering; A (k x k, padded to even kk) in shared
// memory, V in shared memory when it fits, else in global scratch.  Rotation per pair (p,q):
// tau = (a_qq - a_pp)/(2 a_pq), t = sign(tau)/(|tau| + sqrt(1+tau^2)), c = 1/sqrt(1+t^2), s = t c;
// A <- J^T A J with J = [[c, s], [-s, c]] in the (p,q) plane; V <- V J.  One CTA per matrix; a
// launch handles a batch of independent matrices (the N modes of the truncation).
struct EigBatch {
  const double* A[8];
  double* W[8];
  double* V[8];
  int k[8];
  unsigned int* sweeps;   // nullable: device counter of the sweeps run (rt_profile_read "jacobi_sweeps")
};

__global__ void __launch_bounds__(1024) jacobi_kernel(EigBatch bt, double* Vscratch, int v_in_smem, int64_t stride_scr) {
  extern __shared__ double sm[];
  const int k = bt.k[blockIdx.x];
  const int kk = k + (k & 1);
  const int kmax = kk;  // smem carve-up uses this matrix's size
  const int ld = kmax + 1;
  double* A = sm;                                   // kk x ld (row-major A[i*ld + j])
  double* V = v_in_smem ? (sm + kk * ld) : (Vscratch + blockIdx.x * stride_scr);
  double* cs = (v_in_smem ? sm + 2 * kk * ld : sm + kk * ld);   // kk/2 pairs: c, s; then their (p, q) as ints
  int* pq = reinterpret_cast<int*>(cs + 2 * (kk / 2 + 1));
  __shared__ double red[32];
  __shared__ int s_done, s_rot;
  __shared__ double s_fro2;
  const double* Ab = bt.A[blockIdx.x];
  double* W = bt.W[blockIdx.x];
  double* Vout = bt.V[blockIdx.x];
  const int t = threadIdx.x, nt = blockDim.x;
  const int warp = t >> 5, lane = t & 31, nw = nt >> 5;
  for (int i = warp; i < kk; i += nw)
    for (int j = lane; j < kk; j += 32) {
      A[i * ld + j] = (i < k && j < k) ? 0.5 * (Ab[i + int64_t(k) * j] + Ab[j + int64_t(k) * i]) : 0.0;
      V[i * ld + j] = (i == j) ? 1.0 : 0.0;
    }
  __syncthreads();
  const int npairs = kk / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int i = warp; i < kk; i += nw)
      for (int j = lane; j < kk; j += 32) {
        const double v = A[i * ld + j];
        if (i != j) off += v * v; else dia += v * v;
      }
    off = block_sum(off, red);
    __syncthreads();
    dia = block_sum(dia, red);
    // converged when ||offdiag||_F <= k u ||diag||_F (u = 2^-53): below this the rotations only
    // shuffle rounding noise
    const double tol = double(k) * 1.1102230246251565e-16;
    // converged: off-diagonal norm below tolerance, or the previous sweep rotated no pair
    if (t == 0) {
      s_done = (off <= tol * tol * dia) || (dia == 0.0) || (sweep > 0 && !s_rot);
      s_rot = 0;
      s_fro2 = off + dia;                              // ||A||_F^2 (invariant under the rotations)
    }
    __syncthreads();
    if (s_done) break;
    if (t == 0 && bt.sweeps) atomicAdd(bt.sweeps, 1u);
    for (int round = 0; round < kk - 1; ++round) {
      for (int pi = t; pi < npairs; pi += nt) {
        int p, q;
        if (pi == 0) { p = round; q = kk - 1; }
        else {
          p = round + pi; if (p >= kk - 1) p -= kk - 1;
          q = round - pi; if (q < 0) q += kk - 1;
        }
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        const double apq = A[p * ld + q];
        double c = 1.0, s = 0.0;
        // threshold Jacobi: a pair whose |a_pq| is below k u sqrt(|a_pp a_qq|) is skipped (its rotation
        // would move the diagonal by less than the convergence tolerance): the late sweeps skip most
        // pairs and their row / column updates
        // (the test squared: no square root), or below the rounding level u ||A||_F of the matrix: a
        // pair of a large and a tiny eigenvalue (cfg5's Gram spans 6e7) keeps an off-diagonal entry
        // of the size of the large one's rounding error, which no rotation removes -- without this
        // bound every sweep rotated such pairs again and the loop ran to its 40-sweep cap
        const double app = A[p * ld + p], aqq = A[q * ld + q];
        const double thr = double(k) * 1.1102230246251565e-16;
        if (apq * apq > thr * thr * fabs(app * aqq) + 1.232595164407831e-32 * s_fro2) {
          // cos 2 theta = |d| / sqrt(d^2 + 4 a_pq^2), sin 2 theta = 2 |a_pq| / sqrt(.) (the same angle as
          // t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = d / (2 a_pq)): with r = rsqrt(d^2 + 4 a_pq^2),
          // c^2 = (1 + |d| r) / 2 in [1/2, 1] and s = sign(d) a_pq r / c.  Two reciprocal square roots
          // on the round's critical path, no division or square root; no cancellation at small angles
          // (s is a product)
          const double d = aqq - app;
          const double r = rsqrt(fma(d, d, 4.0 * apq * apq));
          const double x = fma(0.5 * fabs(d), r, 0.5);
          const double ic = rsqrt(x);
          c = x * ic;
          s = (d >= 0.0 ? apq : -apq) * r * ic;
        }
        if (s != 0.0) s_rot = 1;                      // benign race: every writer stores 1
        cs[2 * pi + 0] = c; cs[2 * pi + 1] = s;
        pq[2 * pi + 0] = p; pq[2 * pi + 1] = q;
      }
      __syncthreads();
      // A <- J^T A J in one phase: the rotations of a round act on disjoint index pairs, so the
      // 2x2 block (rows of pair u, columns of pair v) of the result depends only on the same block
      // of A and on the two rotations; one thread per block, in place.  V <- V J likewise.
      // (the round is latency-bound: ~1.6 blocks of A and ~3 pairs of V per thread at 1024 threads; the V
      // items go two at a time, loads first, so that their shared-memory round trips overlap)
      for (int e = t; e < npairs * npairs; e += nt) {
        const int u = e / npairs, v = e - u * npairs;
        const double cu = cs[2 * u], su = cs[2 * u + 1], cv = cs[2 * v], sv = cs[2 * v + 1];
        if (su != 0.0 || sv != 0.0) {
          const int pu = pq[2 * u], qu = pq[2 * u + 1], pv = pq[2 * v], qv = pq[2 * v + 1];
          double* ap = A + pu * ld;
          double* aq = A + qu * ld;
          const double app = ap[pv], apq = ap[qv], aqp = aq[pv], aqq = aq[qv];
          const double rpp = cu * app - su * aqp, rpq = cu * apq - su * aqq;     // rows: J_u^T A
          const double rqp = su * app + cu * aqp, rqq = su * apq + cu * aqq;
          const bool dg = (u == v);                                              // the annihilated pair
          ap[pv] = cv * rpp - sv * rpq;                                          // columns: (.) J_v
          ap[qv] = dg ? 0.0 : sv * rpp + cv * rpq;
          aq[pv] = dg ? 0.0 : cv * rqp - sv * rqq;
          aq[qv] = sv * rqp + cv * rqq;
        }
      }
      const int nv = kk * npairs;
      for (int e0 = t; e0 < nv; e0 += 2 * nt) {
        double c[2], sn[2], vp[2], vq[2];
        double* pp[2];
        double* pqv[2];
        bool act[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = e0 + h * nt;
          act[h] = false;
          if (e < nv) {
            const int l = e / npairs, v = e - l * npairs;
            c[h] = cs[2 * v]; sn[h] = cs[2 * v + 1];
            if (sn[h] != 0.0) {
              act[h] = true;
              pp[h] = V + l * ld + pq[2 * v];
              pqv[h] = V + l * ld + pq[2 * v + 1];
              vp[h] = *pp[h]; vq[h] = *pqv[h];
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (act[h]) {
            *pp[h] = c[h] * vp[h] - sn[h] * vq[h];
            *pqv[h] = sn[h] * vp[h] + c[h] * vq[h];
          }
      }
      __syncthreads();
    }
  }
  // sort descending (stable on ties: lower index first) and write out
  for (int i = t; i < k; i += nt) {
    const double wi = A[i * ld + i];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double wj = A[j * ld + j];
      rank += (wj > wi) || (wj == wi && j < i);
    }
    W[rank] = wi;
    for (int l = 0; l < k; ++l) Vout[l + int64_t(k) * rank] = V[l * ld + i];
  }
}

// Two-CTA (cluster) form of the same Jacobi iteration.  The round is bound by one SM's shared-memory
// traffic (the A and V updates move the same number of words), so the two updates go to the two CTAs
// of a cluster: CTA 0 holds A, computes the round's rotations and writes them (c, s and the pair indices)
// into both CTAs' shared memory (DSMEM stores); CTA 1 holds V and only applies them.  The rotation
// buffers alternate between rounds, so one cluster barrier per round orders everything: CTA 0 refills
// a buffer two rounds later, after a barrier CTA 1 reaches only when it has finished reading it.  Same
// rotations in the same order as jacobi_kernel: same eigenpairs to rounding.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024) jacobi2_kernel(EigBatch bt) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int role = int(cl.block_rank());             // 0: A (rotations, eigenvalues); 1: V (eigenvectors)
  const int mi = blockIdx.x >> 1;
  const int k = bt.k[mi];
  const int kk = k + (k & 1);
  const int ld = kk + 1;
  const int npairs = kk / 2;
  double* M = sm;                                    // kk x ld: A (role 0) or V (role 1), row-major
  double* csb = sm + kk * ld;                        // 2 buffers of npairs (c, s)
  int* pqb = reinterpret_cast<int*>(csb + 4 * npairs);   // 2 buffers of npairs (p, q)
  double* dg = reinterpret_cast<double*>(pqb + 4 * npairs);   // kk: the eigenvalues, for CTA 1's sort
  __shared__ double red[32];
  __shared__ int s_done, s_rot;
  __shared__ double s_fro2;
  double* r_csb = cl.map_shared_rank(csb, 1);
  int* r_pqb = cl.map_shared_rank(pqb, 1);
  int* r_done = cl.map_shared_rank(&s_done, 1);
  double* r_dg = cl.map_shared_rank(dg, 1);
  const double* Ab = bt.A[mi];
  const int t = threadIdx.x, nt = blockDim.x;
  const int warp = t >> 5, lane = t & 31, nw = nt >> 5;
  for (int i = warp; i < kk; i += nw)
    for (int j = lane; j < kk; j += 32) {
      if (role == 0) M[i * ld + j] = (i < k && j < k) ? 0.5 * (Ab[i + int64_t(k) * j] + Ab[j + int64_t(k) * i]) : 0.0;
      else M[i * ld + j] = (i == j) ? 1.0 : 0.0;
    }
  __syncthreads();
  int rnd = 0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (role == 0) {
      double off = 0.0, dia = 0.0;
      for (int i = warp; i < kk; i += nw)
        for (int j = lane; j < kk; j += 32) {
          const double v = M[i * ld + j];
          if (i != j) off += v * v; else dia += v * v;
        }
      off = block_sum(off, red);
      __syncthreads();
      dia = block_sum(dia, red);
      const double tol = double(k) * 1.1102230246251565e-16;
      if (t == 0) {
        const int done = (off <= tol * tol * dia) || (dia == 0.0) || (sweep > 0 && !s_rot);
        s_done = done;
        *r_done = done;
        s_rot = 0;
        s_fro2 = off + dia;
      }
    }
    cl.sync();
    if (s_done) break;
    if (role == 0 && t == 0 && bt.sweeps) atomicAdd(bt.sweeps, 1u);
    for (int round = 0; round < kk - 1; ++round, ++rnd) {
      const int b = rnd & 1;
      double* cs = csb + 2 * npairs * b;
      int* pq = pqb + 2 * npairs * b;
      if (role == 0 && t < npairs) {
        const int pi = t;
        int p, q;
        if (pi == 0) { p = round; q = kk - 1; }
        else {
          p = round + pi; if (p >= kk - 1) p -= kk - 1;
          q = round - pi; if (q < 0) q += kk - 1;
        }
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        const double apq = M[p * ld + q];
        double c = 1.0, s = 0.0;
        const double app = M[p * ld + p], aqq = M[q * ld + q];
        const double thr = double(k) * 1.1102230246251565e-16;
        if (apq * apq > thr * thr * fabs(app * aqq) + 1.232595164407831e-32 * s_fro2) {   // as jacobi_kernel
          const double d = aqq - app;
          const double r = rsqrt(fma(d, d, 4.0 * apq * apq));
          const double x = fma(0.5 * fabs(d), r, 0.5);
          const double ic = rsqrt(x);
          c = x * ic;
          s = (d >= 0.0 ? apq : -apq) * r * ic;
        }
        if (s != 0.0) s_rot = 1;
        reinterpret_cast<double2*>(cs)[pi] = make_double2(c, s);
        reinterpret_cast<int2*>(pq)[pi] = make_int2(p, q);
        reinterpret_cast<double2*>(r_csb + 2 * npairs * b)[pi] = make_double2(c, s);
        reinterpret_cast<int2*>(r_pqb + 2 * npairs * b)[pi] = make_int2(p, q);
      }
      cl.sync();
      if (role == 0) {
        for (int e = t; e < npairs * npairs; e += nt) {
          const int u = e / npairs, v = e - u * npairs;
          const double2 ru = reinterpret_cast<const double2*>(cs)[u], rv = reinterpret_cast<const double2*>(cs)[v];
          const double cu = ru.x, su = ru.y, cv = rv.x, sv = rv.y;
          if (su != 0.0 || sv != 0.0) {
            const int2 iu = reinterpret_cast<const int2*>(pq)[u], iv = reinterpret_cast<const int2*>(pq)[v];
            double* ap = M + iu.x * ld;
            double* aq = M + iu.y * ld;
            const double app = ap[iv.x], apq = ap[iv.y], aqp = aq[iv.x], aqq = aq[iv.y];
            const double rpp = cu * app - su * aqp, rpq = cu * apq - su * aqq;
            const double rqp = su * app + cu * aqp, rqq = su * apq + cu * aqq;
            const bool dgl = (u == v);
            ap[iv.x] = cv * rpp - sv * rpq;
            ap[iv.y] = dgl ? 0.0 : sv * rpp + cv * rpq;
            aq[iv.x] = dgl ? 0.0 : cv * rqp - sv * rqq;
            aq[iv.y] = sv * rqp + cv * rqq;
          }
        }
        __syncthreads();                             // the next round's rotations read A
      } else {
        const int nv = kk * npairs;
        for (int e0 = t; e0 < nv; e0 += 2 * nt) {
          double c[2], sn[2], vp[2], vq[2];
          double* pp[2];
          double* pqv[2];
          bool act[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int e = e0 + h * nt;
            act[h] = false;
            if (e < nv) {
              const int l = e / npairs, v = e - l * npairs;
              const double2 rv = reinterpret_cast<const double2*>(cs)[v];
              c[h] = rv.x; sn[h] = rv.y;
              if (sn[h] != 0.0) {
                act[h] = true;
                const int2 iv = reinterpret_cast<const int2*>(pq)[v];
                pp[h] = M + l * ld + iv.x;
                pqv[h] = M + l * ld + iv.y;
                vp[h] = *pp[h]; vq[h] = *pqv[h];
              }
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (act[h]) {
              *pp[h] = c[h] * vp[h] - sn[h] * vq[h];
              *pqv[h] = sn[h] * vp[h] + c[h] * vq[h];
            }
        }
      }
    }
  }
  // eigenvalues to both CTAs, then CTA 0 writes W and CTA 1 the eigenvectors, sorted descending
  // (stable on ties: lower index first)
  if (role == 0)
    for (int i = t; i < k; i += nt) { const double w = M[i * ld + i]; dg[i] = w; r_dg[i] = w; }
  cl.sync();
  for (int i = t; i < k; i += nt) {
    const double wi = dg[i];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double wj = dg[j];
      rank += (wj > wi) || (wj == wi && j < i);
    }
    if (role == 0) bt.W[mi][rank] = wi;
    else {
      double* Vout = bt.V[mi];
      for (int l = 0; l < k; ++l) Vout[l + int64_t(k) * rank] = M[l * ld + i];
    }
  }
}

// ------------------------------------------------------------ sign canon
__global__ void colmax_kernel(const double* __restrict__ Q, int64_t m, int64_t ld, int64_t row0,
                              double* __restrict__ cand) {
  const int c = blockIdx.x;
  double best = -1.0;
  int64_t brow = INT64_MAX;
  double bsign = 1.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double v = Q[i + ld * c], av = fabs(v);
    if (av > best) { best = av; brow = i; bsign = v < 0 ? -1.0 : 1.0; }
  }
  __shared__ double sb[256], ss[256];
  __shared__ int64_t sr[256];
  sb[threadIdx.x] = best; sr[threadIdx.x] = brow; ss[threadIdx.x] = bsign;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) {
      const double b2 = sb[threadIdx.x + o];
      const int64_t r2 = sr[threadIdx.x + o];
      if (b2 > sb[threadIdx.x] || (b2 == sb[threadIdx.x] && r2 < sr[threadIdx.x])) {
        sb[threadIdx.x] = b2; sr[threadIdx.x] = r2; ss[threadIdx.x] = ss[threadIdx.x + o];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cand[3 * c + 0] = sb[0];
    cand[3 * c + 1] = double(row0 + (sr[0] == INT64_MAX ? 0 : sr[0]));
    cand[3 * c + 2] = ss[0];
  }
}

__global__ void sign_apply_kernel(const double* __restrict__ cand, int nc, int r, double* Q, int64_t m,
                                  int64_t ld, double* U, int ku, int64_t ldu) {
  const int c = blockIdx.x;
  double best = -1.0, brow = 0.0, bsign = 1.0;
  for (int s = 0; s < nc; ++s) {
    const double* cd = cand + int64_t(s) * 3 * r + 3 * c;
    if (cd[0] > best || (cd[0] == best && cd[1] < brow)) { best = cd[0]; brow = cd[1]; bsign = cd[2]; }
  }
  if (bsign >= 0) return;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) Q[i + ld * c] = -Q[i + ld * c];
  if (U)
    for (int i = threadIdx.x; i < ku; i += blockDim.x) U[i + ldu * c] = -U[i + ldu * c];
}

// ------------------------------------------------------------ helpers
template <typename Ti, typename To>
__global__ void convert2d_kernel(const Ti* __restrict__ in, int64_t m, int64_t n, int64_t ldi,
                                 To* __restrict__ out, int64_t ldo) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  const int64_t i = e % m, j = e / m;
  out[i + ldo * j] = To(in[i + ldi * j]);
}

template <typename T>
__global__ void unfold_copy_kernel(const T* __restrict__ Tt, int64_t a, int64_t I, int64_t J,
                                   double* __restrict__ out, int64_t ldo) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= I * J) return;
  const int64_t i = e % I, j = e / I;
  out[i + ldo * j] = double(Tt[(j % a) + a * i + a * I * (j / a)]);
}

// Residual: tiles of 128 (j) x 64 (i); R in chunks of BR; grid-stride over tiles.
template <typename T, typename Tacc = typename AccOf<T>::type>
__global__ void __launch_bounds__(256) residual_kernel(const T* __restrict__ X, int64_t J, int64_t In,
                                                        const T* __restrict__ P, int R, const T* __restrict__ Q,
                                                        int64_t ldq, double* __restrict__ part,
                                                        const float* __restrict__ rscale,
                                                        const float* __restrict__ gate, int64_t nslice = 1,
                                                        int64_t sx = 0, int64_t sp = 0) {
  // nslice > 1: a batch of problems (X + s sx, P + s sp, the same Q): the slab form of resid_sums
  if (gate && *gate != 0.f) return;                      // the fp16-split residual ran (twin of R35)
  const Tacc sc = rscale ? Tacc(*rscale) : Tacc(1);
  constexpr int BM = 128, BN = 64, BR = 16;
  __shared__ Tacc Ps[BR][BM];
  __shared__ Tacc Qs[BR][BN + 1];
  __shared__ double red[32];
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  const int64_t njt = cdiv(J, BM), nit = cdiv(In, BN), ntiles = njt * nit;
  const T* X0 = X;
  const T* P0 = P;
  double res = 0.0, xx = 0.0;
  for (int64_t tile_s = blockIdx.x; tile_s < ntiles * nslice; tile_s += gridDim.x) {
    const int64_t tile = tile_s % ntiles, slice = tile_s / ntiles;
    X = X0 + slice * sx;
    P = P0 + slice * sp;
    const int64_t j0 = (tile % njt) * BM, i0 = (tile / njt) * BN;
    Tacc acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = Tacc(0);
    for (int r0 = 0; r0 < R; r0 += BR) {
      for (int e = t; e < BR * BM; e += 256) {
        const int jl = e % BM, rr = e / BM;
        const int64_t j = j0 + jl;
        Ps[rr][jl] = (j < J && r0 + rr < R) ? Tacc(P[j + J * (r0 + rr)]) : Tacc(0);
      }
      for (int e = t; e < BR * BN; e += 256) {
        const int il = e % BN, rr = e / BN;
        const int64_t i = i0 + il;
        Qs[rr][il] = (i < In && r0 + rr < R) ? Tacc(Q[i + ldq * (r0 + rr)]) : Tacc(0);
      }
      __syncthreads();
#pragma unroll
      for (int rr = 0; rr < BR; ++rr) {
        Tacc pr[4], qr[8];
#pragma unroll
        for (int r = 0; r < 4; ++r) pr[r] = Ps[rr][tx + 32 * r];
#pragma unroll
        for (int c = 0; c < 8; ++c) qr[c] = Qs[rr][ty + 8 * c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = fma(pr[r], qr[c], acc[r][c]);
      }
      __syncthreads();
    }
    Tacc tres = 0, txx = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int64_t i = i0 + ty + 8 * c;
      if (i >= In) continue;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t j = j0 + tx + 32 * r;
        if (j >= J) continue;
        const Tacc x = Tacc(X[j + J * i]) * sc;
        const Tacc d = x - acc[r][c] * sc;
        tres = fma(d, d, tres);
        txx = fma(x, x, txx);
      }
    }
    res += double(tres);
    xx += double(txx);
  }
  res = block_sum(res, red);
  __syncthreads();
  xx = block_sum(xx, red);
  if (t == 0) {
    part[2 * blockIdx.x] = res;
    part[2 * blockIdx.x + 1] = xx;
  }
}

__global__ void reduce_pairs_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  // fixed assignment + fixed tree => deterministic
  for (int i = threadIdx.x; i < n; i += blockDim.x) { a += part[2 * i]; b += part[2 * i + 1]; }
  a = block_sum(a, red);
  __syncthreads();
  b = block_sum(b, red);
  if (threadIdx.x == 0) { out[0] = a; out[1] = b; }
}

__global__ void sumsq_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(x[i], x[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void finalize_err_kernel(const double* sums, const double* gg, double* E, double* Eg,
                                    const float* rscale) {
  const double res = sums[0], xx = sums[1];            // sums of the scaled residual / data
  const double s = rscale ? double(*rscale) : 1.0;
  if (E) *E = xx > 0 ? sqrt(res / xx) : 0.0;           // the power-of-two scale cancels exactly
  if (Eg) *Eg = xx > 0 ? sqrt(fmax(0.0, 1.0 - (*gg * s * s) / xx)) : 0.0;
}

// Reading R35: res = sum (s x - s x^_K)^2 + s^2 (||G~||^2 - ||G||^2) (the rank-K residual plus the
// truncated energy, orthogonal parts), E = sqrt(res / xx), E_gram from ||G||^2 as in finalize_err
__global__ void finalize_err_split_kernel(const double* sums, const double* ggK, const double* ggR, double* E,
                                          double* Eg, const float* rscale) {
  const double s = rscale ? double(*rscale) : 1.0;
  const double xx = sums[1];
  const double res = sums[0] + fmax(0.0, *ggK - *ggR) * s * s;
  if (E) *E = xx > 0 ? sqrt(res / xx) : 0.0;
  if (Eg) *Eg = xx > 0 ? sqrt(fmax(0.0, 1.0 - (*ggR * s * s) / xx)) : 0.0;
}

// Power-of-two scale of the residual pass: rms(X) ~ ||G|| / sqrt(numel) (orthonormal factors) is
// brought near 1 so the fp32 squares of the data and of the residual neither underflow (|x| <
// 1e-19) nor overflow (|x| > 1e19).  1 when ||G|| is 0 or not finite.
// s[1] = the fp16 scale of P (the core expanded over all but the last mode) for the fp16-split
// residual: every |P_jr| <= ||P||_F = ||G||_F (orthonormal factors), so s[1] = 2^(14 - e_G) with
// ||G|| in [2^(e_G-1), 2^e_G) keeps |s[1] P| < 2^14, inside the fp16 range; 0 (the tf32 residual
// runs) when ||G|| is 0 or not finite.
__global__ void resid_scale_kernel(const double* gg, double numel, float* s, bool force_twin) {
  float r = 1.f, sp = 0.f;
  const double rms = sqrt(*gg / numel);
  if (rms > 0.0 && isfinite(rms)) {
    int e;
    frexp(rms, &e);                                    // rms in [2^(e-1), 2^e)
    r = ldexpf(1.f, max(-120, min(120, -e)));
  }
  const double ng = sqrt(*gg);
  if (ng > 0.0 && isfinite(ng)) {
    int e;
    frexp(ng, &e);
    if (14 - e >= -120 && 14 - e <= 113) sp = ldexpf(1.f, 14 - e);
  }
  s[0] = r;
  s[1] = force_twin ? 0.f : sp;             // option 212: the gate forced closed, the twin residual runs (tests)
}

__global__ void nonfinite_kernel(const double* __restrict__ x, int64_t n, int* status) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n && !isfinite(x[e])) latch(status, kStatusNonFinite);
}


// ------------------------------------------------------------ power-step unmixing (reading R31')
// Z_S(s, c) = sum_i X_(n)(i, j_s) Q(i, c) for 32 nblk sampled columns: block b takes the 32
// consecutive j from j0 = 32 floor(b ceil(J/32) / nblk) (rows past J are zero).  Grid (nblk, isplit):
// a CTA stages 32 rows i x the block's 32 columns of X and the matching 32 x K rows of Q in
// shared memory (coalesced along whichever of i / j is contiguous: a == 1 or a >= 32), then lane = j,
// warp = c mod 8 accumulate in fp64; partials part[split][s][c], summed in split order by
// zsample_reduce_kernel (deterministic: no atomics).
constexpr int ZS_TI = 32;
template <typename T>
__global__ void __launch_bounds__(256) zsample_kernel(const T* __restrict__ X, Box box, int nblk,
                                                      const double* __restrict__ Q, int64_t ldq, int K,
                                                      double* __restrict__ part) {
  constexpr int CPT = 16;                                   // K <= 128 columns, c = warp + 8 t
  __shared__ double xs[ZS_TI][33];
  __shared__ double qs[128][ZS_TI + 1];
  const int64_t J = box.a * box.b, nj32 = (J + 31) / 32;
  const int64_t j0 = ((int64_t(blockIdx.x) * nj32) / nblk) * 32;
  const int64_t i0 = int64_t(blockIdx.y) * ZS_TI;
  const int ni = box.I - i0 < ZS_TI ? int(box.I - i0) : ZS_TI;
  const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
  // X chunk: element (i, jl) at alpha + a i + a I beta, j = j0 + jl = alpha + a beta
  for (int e = t; e < ZS_TI * 32; e += 256) {
    int il, jl;
    if (box.a == 1) { il = e % ZS_TI; jl = e / ZS_TI; }     // i contiguous in memory
    else            { jl = e % 32; il = e / 32; }           // alpha contiguous
    const int64_t j = j0 + jl;
    double v = 0.0;
    if (il < ni && j < J) {
      const int64_t al = j % box.a, be = j / box.a;
      v = double(X[al + box.a * (i0 + il) + box.a * box.I * be]);
    }
    xs[il][jl] = v;
  }
  for (int e = t; e < ZS_TI * K; e += 256) {
    const int il = e % ZS_TI, c = e / ZS_TI;
    qs[c][il] = il < ni ? Q[i0 + il + ldq * c] : 0.0;
  }
  __syncthreads();
  double acc[CPT];
#pragma unroll
  for (int u = 0; u < CPT; ++u) acc[u] = 0.0;
  for (int il = 0; il < ni; ++il) {
    const double x = xs[il][lane];
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
      const int c = wp + 8 * u;
      if (c < K) acc[u] = fma(x, qs[c][il], acc[u]);
    }
  }
  const int64_t S = int64_t(nblk) * 32;
  double* dst = part + int64_t(blockIdx.y) * S * K;
  const int64_t row = int64_t(blockIdx.x) * 32 + lane;
#pragma unroll
  for (int u = 0; u < CPT; ++u) {
    const int c = wp + 8 * u;
    if (c < K) dst[row + S * c] = acc[u];
  }
}
__global__ void zsample_reduce_kernel(const double* __restrict__ part, int nsplit, int64_t n, double* __restrict__ Zs) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = 0.0;
  for (int z = 0; z < nsplit; ++z) s += part[e + n * z];
  Zs[e] = s;
}

// Qp[:, c] = d_c Q Rinv[:, c] (Rinv upper triangular; the identity when *zero), d_c = 2^-e with
// ||Rinv[:, c]|| in [2^(e-1), 2^e): ||Qp[:, c]|| in [1/2, 1) for an orthonormal Q, from the
// replicated Rinv alone (the same scale on every rank of a row-distributed Q).  One CTA per column.
__global__ void __launch_bounds__(256) unmix_cols_kernel(const double* __restrict__ Q, int64_t m, int K,
                                                         int64_t ldq, const double* __restrict__ Ri,
                                                         const int* zero, double* __restrict__ Qp, int64_t ldp) {
  __shared__ double rc[128];
  __shared__ double s_d;
  const int c = blockIdx.x;
  const bool z = zero && *zero;
  if (threadIdx.x < 32) {
    double ss = 0.0;
    for (int l = threadIdx.x; l <= c; l += 32) {
      const double v = z ? (l == c ? 1.0 : 0.0) : Ri[l + int64_t(K) * c];
      ss = fma(v, v, ss);
    }
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (threadIdx.x == 0) {
      int e = 0;
      frexp(sqrt(ss), &e);
      s_d = (ss > 0.0 && ss <= DBL_MAX) ? ldexp(1.0, -e) : 1.0;
    }
  }
  __syncthreads();
  for (int l = threadIdx.x; l <= c; l += blockDim.x) rc[l] = (z ? (l == c ? 1.0 : 0.0) : Ri[l + int64_t(K) * c]) * s_d;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    double v = 0.0;
    for (int l = 0; l <= c; ++l) v = fma(Q[i + ldq * l], rc[l], v);
    Qp[i + ldp * c] = v;
  }
}


// ------------------------------------------------------------ Gram of an unfolding
// G = B_(n) B_(n)^T for B viewed as [a, K, b] (column j = (alpha, beta) holds B[alpha + a p + a K beta],
// p < K).  A CTA takes a contiguous range of columns in chunks of 32 staged in shared memory; the
// upper-triangle 4 x 4 blocks of G are spread over the threads (column groups when there are fewer
// blocks than threads), fp64 products and sums; the groups are added into the CTA's shared G in a
// fixed order and the CTA partials are summed in CTA order: deterministic.
template <int JC, int MB>
__global__ void __launch_bounds__(256) gram_unfold_kernel(const double* __restrict__ B, int64_t a, int K, int64_t J,
                                                          int64_t jper, double* __restrict__ part) {
  constexpr int GU_JC = JC;
  extern __shared__ double gsm[];
  double* vs = gsm;                                  // [K][GU_JC + 1]
  double* G = gsm + size_t(K) * (GU_JC + 1);         // [K][K]
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int nb = (K + 3) / 4, nblk = nb * (nb + 1) / 2;
  // the lanes of a warp take different blocks of the same column (shared-memory broadcast reads);
  // a set of wpb warps covers the blocks once, and the 8 / wpb sets take interleaved columns
  const int wpb = (nblk + 31) / 32;
  const int groups = wpb <= 8 ? 8 / wpb : 1;
  const int g = wpb <= 8 ? warp / wpb : 0;
  const bool active = g < groups;
  int bp[MB], bq[MB];
  int nmine = 0;
  if (active) {
    for (int idx = (wpb <= 8 ? lane + 32 * (warp % wpb) : t); idx < nblk && nmine < MB; idx += (wpb <= 8 ? nblk : 256)) {
      int q = 0;
      while ((q + 1) * (q + 2) / 2 <= idx) ++q;
      bq[nmine] = q;
      bp[nmine] = idx - q * (q + 1) / 2;
      ++nmine;
    }
  }
  double acc[MB][4][4];
#pragma unroll
  for (int m = 0; m < MB; ++m)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[m][u][v] = 0.0;
  for (int e = t; e < K * K; e += 256) G[e] = 0.0;
  const int64_t jb = int64_t(blockIdx.x) * jper;
  const int64_t je = jb + jper < J ? jb + jper : J;
  for (int64_t j0 = jb; j0 < je; j0 += GU_JC) {
    __syncthreads();
    if (a > 1) {
      // lane = column: one (alpha, beta) split per chunk per thread (256 % 32 == 0)
      const int jj = t % GU_JC;
      const int64_t j = j0 + jj;
      const bool jv = j < je;
      const int64_t base = jv ? (j % a) + a * K * (j / a) : 0;
      for (int p = t / GU_JC; p < K; p += 256 / GU_JC) vs[p * (GU_JC + 1) + jj] = jv ? B[base + a * p] : 0.0;
    } else {
      const double* src = B + j0 * K;                   // columns contiguous: K doubles each
      const int64_t nel = (je - j0 < GU_JC ? je - j0 : GU_JC) * int64_t(K);
      for (int e = t; e < K * GU_JC; e += 256) {
        const int jj = e / K, p = e - jj * K;
        vs[p * (GU_JC + 1) + jj] = e < nel ? src[e] : 0.0;
      }
    }
    __syncthreads();
    for (int jj = g; jj < GU_JC; jj += groups) {
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        if (m >= nmine) break;
        double vp[4], vq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int p = 4 * bp[m] + u, q = 4 * bq[m] + u;
          vp[u] = p < K ? vs[p * (GU_JC + 1) + jj] : 0.0;
          vq[u] = q < K ? vs[q * (GU_JC + 1) + jj] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[m][u][v] = fma(vp[u], vq[v], acc[m][u][v]);
      }
    }
  }
  for (int gg = 0; gg < groups; ++gg) {
    __syncthreads();
    if (active && g == gg) {
      for (int m = 0; m < nmine; ++m)
        for (int u = 0; u < 4; ++u)
          for (int v = 0; v < 4; ++v) {
            const int p = 4 * bp[m] + u, q = 4 * bq[m] + v;
            if (p < K && q < K) {
              G[p * K + q] += acc[m][u][v];
              if (bp[m] != bq[m]) G[q * K + p] += acc[m][u][v];
            }
          }
    }
  }
  __syncthreads();
  double* dst = part + int64_t(blockIdx.x) * K * K;
  for (int e = t; e < K * K; e += 256) dst[e] = G[e];
}
// one CTA per element: a fixed strided assignment of the CTA partials to the threads and a fixed
// tree (deterministic)
__global__ void __launch_bounds__(128) gram_unfold_reduce_kernel(const double* __restrict__ part, int ncta, int KK,
                                                                 double* __restrict__ G) {
  __shared__ double red[32];
  const int e = blockIdx.x;
  double s = 0.0;
  for (int z = threadIdx.x; z < ncta; z += blockDim.x) s += part[int64_t(z) * KK + e];
  s = block_sum(s, red);
  if (threadIdx.x == 0) G[e] = s;
}

}  // namespace

// ======================================================================= host
template <typename T>
void gram(const Ctx& ctx, Arena& ws, const T* A, int64_t m, int k, int64_t lda, double* G, bool rm) {
  RT_REQUIRE(k >= 1 && k <= 128, kEUNSUPPORTED, "gram: k must be in [1,128]");
  if (m == 0) { RT_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * k * k, ctx.stream)); return; }
  if (k <= 16) launch_gram<T, 1>(ctx, ws, A, m, k, lda, G, rm);
  else if (k <= 32) launch_gram<T, 2>(ctx, ws, A, m, k, lda, G, rm);
  else if (k <= 48) launch_gram<T, 3>(ctx, ws, A, m, k, lda, G, rm);
  else if (k <= 64) launch_gram<T, 4>(ctx, ws, A, m, k, lda, G, rm);
  else if (k <= 80) launch_gram<T, 5>(ctx, ws, A, m, k, lda, G, rm);
  else if (k <= 96) launch_gram<T, 6>(ctx, ws, A, m, k, lda, G, rm);
  else launch_gram<T, 8>(ctx, ws, A, m, k, lda, G, rm);
}
template void gram<float>(const Ctx&, Arena&, const float*, int64_t, int, int64_t, double*, bool);
template void gram<double>(const Ctx&, Arena&, const double*, int64_t, int, int64_t, double*, bool);

void chol_inv(const Ctx& ctx, const double* G, int k, double shift_coef, double* R, double* Rinv,
              int* zero_flag, const double* shift_dev) {
  const size_t smem = sizeof(double) * size_t(k) * (k + 1);
  RT_REQUIRE(smem <= 220 * 1024, kEUNSUPPORTED, "chol_inv: k too large");
  const size_t smem_blk = sizeof(double) * (2 * size_t(k) * (k + 1) + size_t(k) * NBK + size_t(k));
  static bool attr = false;
  if (!attr) {
    RT_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    RT_CUDA(cudaFuncSetAttribute(chol_inv_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    RT_CUDA(cudaFuncSetAttribute(chol_inv_reg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  const size_t smem_fast = sizeof(double) * (2 * size_t(k) * (k + 1) + size_t(k));
  static bool attr_fast = false;
  if (!attr_fast) {
    RT_CUDA(cudaFuncSetAttribute(chol_inv_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr_fast = true;
  }
  launch(ctx, "chol_inv", [&] {
    // the one-barrier-per-column kernel wins at small k (tools/qr_time.py: 25 vs 29 us at k = 27;
    // 84 vs 66 us at k = 60, where the blocked kernel's register-blocked panels pay off)
    if (k <= 32 && !getenv("RT_CHOL_BLOCKED") && !getenv("RT_CHOL_UNBLOCKED") && !getenv("RT_CHOL_FAST"))
      chol_inv_warp_kernel<<<1, 32, 0, ctx.stream>>>(G, k, shift_coef, R, Rinv, zero_flag, ctx.d_status, shift_dev);
    else if (k <= 40 && smem_fast <= 220 * 1024 && !getenv("RT_CHOL_BLOCKED") && !getenv("RT_CHOL_UNBLOCKED"))
      chol_inv_fast_kernel<<<1, 256, smem_fast, ctx.stream>>>(G, k, shift_coef, R, Rinv, zero_flag, ctx.d_status,
                                                              shift_dev);
    else if (k <= 128 && smem_blk <= 220 * 1024 && !getenv("RT_CHOL_BLOCKED") && !getenv("RT_CHOL_UNBLOCKED"))
      chol_inv_reg_kernel<<<1, 256, smem_blk, ctx.stream>>>(G, k, shift_coef, R, Rinv, zero_flag, ctx.d_status,
                                                            shift_dev);
    else if (smem_blk <= 220 * 1024 && !getenv("RT_CHOL_UNBLOCKED"))
      chol_inv_blk_kernel<<<1, 256, smem_blk, ctx.stream>>>(G, k, shift_coef, R, Rinv, zero_flag, ctx.d_status,
                                                            shift_dev);
    else
      chol_inv_kernel<<<1, 512, smem, ctx.stream>>>(G, k, shift_coef, R, Rinv, zero_flag, ctx.d_status, shift_dev);
  });
}

template <typename TA, typename TC>
void gemm_tall(const Ctx& ctx, const TA* A, int64_t m, int k, int64_t lda, const double* B, int n,
               int64_t ldb, TC* C, int64_t ldc, const int* zero_flag, int64_t row0, bool rowmajor,
               const int64_t* row0_dev) {
  if (m == 0 || n == 0) return;
  const size_t smem = sizeof(double) * (size_t(k) * n + 32 * size_t(k + 1));
  RT_REQUIRE(smem <= 220 * 1024, kEUNSUPPORTED, "gemm_tall: k*n too large");
  static bool attr = false;
  if (!attr) {
    RT_CUDA(cudaFuncSetAttribute(gemm_tall_kernel<TA, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  launch(ctx, "gemm_tall", [&] {
    gemm_tall_kernel<TA, TC><<<unsigned(cdiv(m, 32)), 256, smem, ctx.stream>>>(A, m, k, lda, B, n, ldb, C, ldc,
                                                                               zero_flag, row0, rowmajor, row0_dev);
  });
}
template void gemm_tall<double, double>(const Ctx&, const double*, int64_t, int, int64_t, const double*, int,
                                        int64_t, double*, int64_t, const int*, int64_t, bool, const int64_t*);
template void gemm_tall<float, float>(const Ctx&, const float*, int64_t, int, int64_t, const double*, int,
                                      int64_t, float*, int64_t, const int*, int64_t, bool, const int64_t*);
template void gemm_tall<float, double>(const Ctx&, const float*, int64_t, int, int64_t, const double*, int,
                                       int64_t, double*, int64_t, const int*, int64_t, bool, const int64_t*);

void gemm_small(const Ctx& ctx, bool ta, bool tb, int m, int n, int k, const double* A, int lda,
                const double* B, int ldb, double* C, int ldc) {
  launch(ctx, "gemm_small", [&] {
    gemm_small_kernel<<<1, 512, 0, ctx.stream>>>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc);
  });
}

void eig_sym_batch(const Ctx& ctx, Arena& ws, int count, const double* const* A, const int* k, double* const* W,
                   double* const* V) {
  RT_REQUIRE(count >= 1 && count <= 8, kEUNSUPPORTED, "eig_sym_batch: 1..8 matrices");
  EigBatch bt{};
  int kmax = 0;
  for (int i = 0; i < count; ++i) {
    RT_REQUIRE(k[i] >= 1 && k[i] <= 128, kEUNSUPPORTED, "eig_sym: k must be in [1,128]");
    bt.A[i] = A[i]; bt.W[i] = W[i]; bt.V[i] = V[i]; bt.k[i] = k[i];
    bt.sweeps = ctx.d_runs ? ctx.d_runs + 2 : nullptr;
    kmax = std::max(kmax, k[i]);
  }
  const int kk = kmax + (kmax & 1), ld = kk + 1;
  const size_t a_bytes = sizeof(double) * size_t(kk) * ld;
  {
    // the two-CTA cluster form: A and V in different SMs (RT_JACOBI_1CTA keeps the one-CTA kernel)
    const size_t smem2 = a_bytes + sizeof(double) * (4 * size_t(kk / 2) + 2 * size_t(kk / 2) + size_t(kk));
    if (smem2 <= 200 * 1024 && !getenv("RT_JACOBI_1CTA")) {
      static bool attr2 = false;
      if (!attr2) {
        RT_CUDA(cudaFuncSetAttribute(jacobi2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr2 = true;
      }
      launch(ctx, "jacobi_eig", [&] { jacobi2_kernel<<<2 * count, 1024, smem2, ctx.stream>>>(bt); });
      return;
    }
  }
  const size_t cs_bytes = sizeof(double) * 4 * size_t(kk / 2 + 1);
  const int v_in_smem = (2 * a_bytes + cs_bytes) <= 200 * 1024;
  const size_t smem = (v_in_smem ? 2 * a_bytes : a_bytes) + cs_bytes;
  double* scratch = nullptr;
  int64_t stride_scr = 0;
  if (!v_in_smem) {
    stride_scr = int64_t(kk) * ld;
    scratch = ws.alloc_n<double>(stride_scr * count);
  }
  static bool attr = false;
  if (!attr) {
    RT_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  launch(ctx, "jacobi_eig", [&] {
    jacobi_kernel<<<count, 1024, smem, ctx.stream>>>(bt, scratch, v_in_smem, stride_scr);
  });
}

void eig_sym(const Ctx& ctx, Arena& ws, const double* A, int k, double* W, double* V) {
  eig_sym_batch(ctx, ws, 1, &A, &k, &W, &V);
}

void colmax_candidates(const Ctx& ctx, const double* Q, int64_t m, int r, int64_t ld, int64_t row0,
                       double* cand) {
  launch(ctx, "colmax", [&] { colmax_kernel<<<r, 256, 0, ctx.stream>>>(Q, m, ld, row0, cand); });
}

void sign_apply(const Ctx& ctx, const double* cand, int nc, double* Q, int64_t m, int r, int64_t ld,
                double* U, int ku, int64_t ldu) {
  launch(ctx, "sign_apply", [&] {
    sign_apply_kernel<<<r, 256, 0, ctx.stream>>>(cand, nc, r, Q, m, ld, U, ku, ldu);
  });
}

template <typename Ti, typename To>
void convert2d(const Ctx& ctx, const Ti* in, int64_t m, int64_t n, int64_t ldi, To* out, int64_t ldo) {
  if (m * n == 0) return;
  launch(ctx, "convert", [&] {
    convert2d_kernel<Ti, To><<<unsigned(cdiv(m * n, 256)), 256, 0, ctx.stream>>>(in, m, n, ldi, out, ldo);
  });
}
template <typename T>
__global__ void transpose_copy_kernel(const T* __restrict__ in, int64_t m, int64_t n, int64_t ldi, T* __restrict__ out,
                                      int64_t ldo) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  const int64_t i = e % m, j = e / m;
  out[i + ldo * j] = in[i * ldi + j];
}
template <typename T>
void transpose_copy(const Ctx& ctx, const T* in, int64_t m, int64_t n, int64_t ldi, T* out, int64_t ldo) {
  if (m * n == 0) return;
  launch(ctx, "transpose_copy", [&] {
    transpose_copy_kernel<T><<<unsigned(cdiv(m * n, 256)), 256, 0, ctx.stream>>>(in, m, n, ldi, out, ldo);
  });
}
template void transpose_copy<float>(const Ctx&, const float*, int64_t, int64_t, int64_t, float*, int64_t);
template void transpose_copy<double>(const Ctx&, const double*, int64_t, int64_t, int64_t, double*, int64_t);

template void convert2d<double, float>(const Ctx&, const double*, int64_t, int64_t, int64_t, float*, int64_t);
template void convert2d<double, double>(const Ctx&, const double*, int64_t, int64_t, int64_t, double*, int64_t);
template void convert2d<float, double>(const Ctx&, const float*, int64_t, int64_t, int64_t, double*, int64_t);
template void convert2d<float, float>(const Ctx&, const float*, int64_t, int64_t, int64_t, float*, int64_t);

template <typename T>
void unfold_copy(const Ctx& ctx, const T* Tt, Box box, double* out, int64_t ldo) {
  const int64_t n = box.I * box.J();
  if (n == 0) return;
  launch(ctx, "unfold_copy", [&] {
    unfold_copy_kernel<T><<<unsigned(cdiv(n, 256)), 256, 0, ctx.stream>>>(Tt, box.a, box.I, box.J(), out, ldo);
  });
}
template void unfold_copy<float>(const Ctx&, const float*, Box, double*, int64_t);
template void unfold_copy<double>(const Ctx&, const double*, Box, double*, int64_t);

template <typename T>
void residual(const Ctx& ctx, Arena& ws, const T* X, int64_t J, int64_t In, const T* P, int R, const T* Q,
              int64_t ldq, double* out2, const float* rscale) {
  const int nblk = 4 * ctx.num_sms;
  double* part = ws.alloc_n<double>(2 * nblk);
  launch(ctx, "residual_simt", [&] {
    if (ctx.acc64())
      residual_kernel<T, double><<<nblk, 256, 0, ctx.stream>>>(X, J, In, P, R, Q, ldq, part, rscale, nullptr);
    else residual_kernel<T><<<nblk, 256, 0, ctx.stream>>>(X, J, In, P, R, Q, ldq, part, rscale, nullptr);
  });
  launch(ctx, "reduce_pairs", [&] { reduce_pairs_kernel<<<1, 256, 0, ctx.stream>>>(part, nblk, out2); });
}
void residual_part(const Ctx& ctx, const float* X, int64_t J, int64_t In, const float* P, int R, const float* Q,
                   int64_t ldq, double* part, int nblk, const float* rscale, const float* gate, int64_t nslice,
                   int64_t sx, int64_t sp) {
  launch(ctx, "residual_simt", [&] {
    residual_kernel<float><<<nblk, 256, 0, ctx.stream>>>(X, J, In, P, R, Q, ldq, part, rscale, gate, nslice, sx, sp);
  });
}
template void residual<float>(const Ctx&, Arena&, const float*, int64_t, int64_t, const float*, int, const float*,
                              int64_t, double*, const float*);
template void residual<double>(const Ctx&, Arena&, const double*, int64_t, int64_t, const double*, int,
                               const double*, int64_t, double*, const float*);

void reduce_pairs(const Ctx& ctx, const double* part, int n, double* out2) {
  launch(ctx, "reduce_pairs", [&] { reduce_pairs_kernel<<<1, 256, 0, ctx.stream>>>(part, n, out2); });
}

// per-CTA partial sums of squares over a fixed strided assignment (then one fixed-order CTA)
__global__ void sumsq_part_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    s = fma(x[i], x[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void sum_parts_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}
void sumsq(const Ctx& ctx, Arena& ws, const double* x, int64_t n, double* out) {
  // one CTA below 64K elements; above, up to 2 CTAs per SM and a fixed-order sum of their partials
  const int nb = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(2) * ctx.num_sms, cdiv(n, int64_t(1) << 16))));
  if (nb == 1) {
    launch(ctx, "sumsq", [&] { sumsq_kernel<<<1, 512, 0, ctx.stream>>>(x, n, out); });
    return;
  }
  const auto mk = ws.mark();
  double* part = ws.alloc_n<double>(nb);
  launch(ctx, "sumsq", [&] {
    sumsq_part_kernel<<<nb, 512, 0, ctx.stream>>>(x, n, part);
    sum_parts_kernel<<<1, 512, 0, ctx.stream>>>(part, nb, out);
  });
  ws.rewind(mk);
}

void finalize_err(const Ctx& ctx, const double* sums, const double* gg, double* E, double* Eg, const float* rscale) {
  launch(ctx, "finalize_err", [&] { finalize_err_kernel<<<1, 1, 0, ctx.stream>>>(sums, gg, E, Eg, rscale); });
}
// Row-distributed thin QR bookkeeping on the device (no host sync): from the allgathered local
// row counts, this rank's first global row and the shift coefficient 11 (m k + k (k + 1)) u of
// shifted CholeskyQR with the global row count m.
__global__ void dist_rows_info_kernel(const double* counts, int nranks, int rank, int k, double* shift_coef,
                                      int64_t* row0) {
  double m = 0.0, r0 = 0.0;
  for (int r = 0; r < nranks; ++r) { if (r < rank) r0 += counts[r]; m += counts[r]; }
  *row0 = int64_t(r0);
  *shift_coef = 11.0 * (m * k + double(k) * (k + 1)) * 1.1102230246251565e-16;
}
__global__ void fill_value_kernel(double* p, double v) { *p = v; }
void fill_value(const Ctx& ctx, double* p, double v) {
  launch(ctx, "fill_value", [&] { fill_value_kernel<<<1, 1, 0, ctx.stream>>>(p, v); });
}
void dist_rows_info(const Ctx& ctx, const double* counts, int nranks, int rank, int k, double* shift_coef,
                    int64_t* row0) {
  launch(ctx, "dist_rows_info", [&] {
    dist_rows_info_kernel<<<1, 1, 0, ctx.stream>>>(counts, nranks, rank, k, shift_coef, row0);
  });
}
void finalize_err_split(const Ctx& ctx, const double* sums, const double* ggK, const double* ggR, double* E, double* Eg,
                        const float* rscale) {
  launch(ctx, "finalize_err", [&] {
    finalize_err_split_kernel<<<1, 1, 0, ctx.stream>>>(sums, ggK, ggR, E, Eg, rscale);
  });
}
void resid_scale(const Ctx& ctx, const double* gg, double numel, float* s) {
  launch(ctx, "resid_scale", [&] { resid_scale_kernel<<<1, 1, 0, ctx.stream>>>(gg, numel, s, ctx.tc_h16 == 2); });
}

void fill_zero(const Ctx& ctx, void* p, size_t bytes) { RT_CUDA(cudaMemsetAsync(p, 0, bytes, ctx.stream)); }

void set_status_if_nonfinite(const Ctx& ctx, const double* x, int64_t n) {
  if (n == 0) return;
  launch(ctx, "nonfinite_check", [&] {
    nonfinite_kernel<<<unsigned(cdiv(n, 256)), 256, 0, ctx.stream>>>(x, n, ctx.d_status);
  });
}

template <typename T>
void zsample(const Ctx& ctx, Arena& ws, const T* X, Box box, int nblk, const double* Q, int64_t ldq, int K,
             double* Zs) {
  RT_REQUIRE(K >= 1 && K <= 128 && nblk >= 1, kEUNSUPPORTED, "zsample: K outside [1, 128]");
  const int nsplit = int(cdiv(box.I, int64_t(ZS_TI)));
  RT_REQUIRE(nsplit <= 65535, kEUNSUPPORTED, "zsample: I_n too large");
  const int64_t n = int64_t(nblk) * 32 * K;
  const auto mk = ws.mark();
  double* part = ws.alloc_n<double>(n * nsplit);
  launch(ctx, "zsample", [&] {
    zsample_kernel<T><<<dim3(unsigned(nblk), unsigned(nsplit)), 256, 0, ctx.stream>>>(X, box, nblk, Q, ldq, K, part);
    zsample_reduce_kernel<<<unsigned(cdiv(n, int64_t(256))), 256, 0, ctx.stream>>>(part, nsplit, n, Zs);
  });
  ws.rewind(mk);
}
template void zsample<float>(Ctx const&, Arena&, const float*, Box, int, const double*, int64_t, int, double*);
template void zsample<double>(Ctx const&, Arena&, const double*, Box, int, const double*, int64_t, int, double*);

void unmix_cols(const Ctx& ctx, const double* Q, int64_t m, int K, int64_t ldq, const double* Ri, const int* zero,
                double* Qp, int64_t ldp) {
  RT_REQUIRE(K >= 1 && K <= 128, kEUNSUPPORTED, "unmix_cols: K outside [1, 128]");
  launch(ctx, "unmix_cols", [&] { unmix_cols_kernel<<<K, 256, 0, ctx.stream>>>(Q, m, K, ldq, Ri, zero, Qp, ldp); });
}

void gram_unfold(const Ctx& ctx, Arena& ws, const double* B, Box box, double* G) {
  const int K = int(box.I);
  const int64_t J = box.J();
  RT_REQUIRE(K >= 1 && K <= 128, kEUNSUPPORTED, "gram_unfold: K outside [1, 128]");
  if (J == 0) { fill_zero(ctx, G, sizeof(double) * size_t(K) * K); return; }
  // 128 columns per staged chunk (the loads of a chunk all in flight) when the Gram tile fits beside it
  const int jc = K <= 64 ? 128 : 32;
  const int ncta = int(std::max<int64_t>(1, std::min<int64_t>(int64_t(4) * ctx.num_sms, cdiv(J, int64_t(4 * jc)))));
  const int64_t jper = cdiv(cdiv(J, int64_t(ncta)), int64_t(jc)) * jc;
  const int nc = int(cdiv(J, jper));
  const size_t sm = sizeof(double) * (size_t(K) * (jc + 1) + size_t(K) * K);
  static bool attr = false;
  if (!attr) {
    RT_CUDA(cudaFuncSetAttribute(gram_unfold_kernel<32, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RT_CUDA(cudaFuncSetAttribute(gram_unfold_kernel<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RT_CUDA(cudaFuncSetAttribute(gram_unfold_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const auto mk = ws.mark();
  double* part = ws.alloc_n<double>(int64_t(nc) * K * K);
  launch(ctx, "gram_unfold", [&] {
    const int nb = (K + 3) / 4, nblk = nb * (nb + 1) / 2;          // 4 x 4 blocks (<= 256 for K <= 88)
    if (jc == 128 && nblk <= 256) gram_unfold_kernel<128, 1><<<nc, 256, sm, ctx.stream>>>(B, box.a, K, J, jper, part);
    else if (jc == 128) gram_unfold_kernel<128, 2><<<nc, 256, sm, ctx.stream>>>(B, box.a, K, J, jper, part);
    else gram_unfold_kernel<32, 3><<<nc, 256, sm, ctx.stream>>>(B, box.a, K, J, jper, part);
    gram_unfold_reduce_kernel<<<unsigned(K * K), 128, 0, ctx.stream>>>(part, nc, K * K, G);
  });
  ws.rewind(mk);
}

}  // namespace rt
