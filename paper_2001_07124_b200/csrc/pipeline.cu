// pipeline.cu -- the randomized Tucker/HOSVD hot path on one rank.
//
// Every step runs in this library's kernels; torch only owns the caller's buffers.
// Distributed semantics (slab along the last mode):
//   C1  mode n < N-1 sketches / power products Y: per-slab partial sums -> allreduce
//   C2  Gram matrices of row-distributed tall matrices (Y_{N-1}, Z_n for n < N-1) -> allreduce
//   C3  Z = X_(N-1)^T Q of the last mode: per-slab partial sums (J x K) -> allreduce
//   C4  core G~: per-slab partial sums -> allreduce
//   C5  residual sums -> allreduce;  sign candidates of the row-distributed last factor -> allgather
#include <cmath>
#include <type_traits>

#include "engine.h"

namespace rt {

namespace {
constexpr double kU = 1.1102230246251565e-16;   // fp64 unit roundoff

template <typename T> struct DT;
template <> struct DT<float> { static constexpr int id = 0; };
template <> struct DT<double> { static constexpr int id = 1; };

template <typename T>
void allreduce(Comm* c, bool on, T* p, int64_t n, cudaStream_t s) {
  if (on && n > 0) c->allreduce_sum(p, size_t(n), s);
}

int64_t pad4(int64_t x) { return (x + 3) & ~int64_t(3); }

// Y = X_(n) B (B row-major, row pitch ldb: Omega or Z): tcgen05 3xTF32 kernel for fp32 data when
// the shape fits the TMA path, else the SIMT kernel.
// amax: also gather max|X| there (tensor-core kernel only; the return value says whether it did)
bool ttm_s_dispatch(const Ctx& ctx, Arena& ws, const float* X, Box box, const float* B, int64_t ldb, bool exact,
                    int K, double* Y, int64_t ldy, unsigned int* amax = nullptr) {
  if (!ctx.simt() && ttm_s_tc(ctx, ws, X, box, B, ldb, exact, K, Y, ldy, false, nullptr, amax)) return amax != nullptr;
  ttm_s<float>(ctx, ws, X, box, B, ldb, 1, K, Y, ldy);
  return false;
}
bool ttm_s_dispatch(const Ctx& ctx, Arena& ws, const double* X, Box box, const double* B, int64_t ldb, bool,
                    int K, double* Y, int64_t ldy, unsigned int* = nullptr) {
  ttm_s<double>(ctx, ws, X, box, B, ldb, 1, K, Y, ldy);
  return false;
}
// out(alpha,c,beta) = sum_i X(alpha,i,beta) Q(i,c), Q col-major (ldq)
// q_tf32_exact: Q holds tf32-representable values (a host-rounded test matrix, reading R18): the
// tensor-core kernel then runs 2 products instead of the 3 of the split form
// xscale: X's fp16 scale when known (an orthonormal Q): the fp16-split kernel instead of 3xTF32
// oscale: device scale of the output (tensor-core kernels; the SIMT fallback leaves it unscaled,
// which only the power iteration's Z uses, whose span it does not change)
void ttm_t_dispatch(const Ctx& ctx, Arena& ws, const float* X, Box box, const float* Q, int64_t ldq, int C, float* out,
                    int64_t so_a, int64_t so_c, int64_t so_b, bool q_tf32_exact = false, const float* xscale = nullptr,
                    const float* oscale = nullptr) {
  if (!ctx.simt()) {
    if (C <= 128) {
      if (ttm_t_tc(ctx, ws, X, box, Q, ldq, C, out, so_a, so_c, so_b, 0, q_tf32_exact, xscale, nullptr, oscale)) return;
    } else {
      // wider than one TMEM tile (the residual's P chain: C = I_n; the R-PET core sketch, S_n = 2K_n + 1):
      // column chunks of 128 in one launch (every chunk re-reads the small source from L2)
      if (!xscale && !q_tf32_exact &&
          ttm_t_tc(ctx, ws, X, box, Q, ldq, C, out, so_a, so_c, so_b, 0, false, nullptr, nullptr, oscale, 1.f, false,
                   128))
        return;
      // otherwise balanced chunks of <= 128, one launch each, each writing its slice of the output
      const int nch = int(cdiv(C, 128));
      const int cw = int(cdiv(C, nch) + 3) & ~3;
      if (ttm_t_tc(ctx, ws, X, box, Q, ldq, cw, out, so_a, so_c, so_b, 0, q_tf32_exact, xscale)) {
        for (int c0 = cw; c0 < C; c0 += cw)
          RT_REQUIRE(ttm_t_tc(ctx, ws, X, box, Q + int64_t(c0) * ldq, ldq, std::min(cw, C - c0), out + c0 * so_c, so_a,
                              so_c, so_b, 0, q_tf32_exact, xscale),
                     kEINVAL, "ttm_t: tensor-core chunk rejected after the first");   // same shape: unreachable
        return;
      }
    }
  }
  ttm_t<float, float, float>(ctx, X, box, Q, 1, ldq, C, out, so_a, so_c, so_b);
}
void ttm_t_dispatch(const Ctx& ctx, Arena&, const double* X, Box box, const double* Q, int64_t ldq, int C, double* out,
                    int64_t so_a, int64_t so_c, int64_t so_b, bool = false, const float* = nullptr,
                    const float* = nullptr) {
  ttm_t<double, double, double>(ctx, X, box, Q, 1, ldq, C, out, so_a, so_c, so_b);
}

// fp64 col-major m x k -> working-type copy with ld padded to a multiple of 4 (pad rows zero)
template <typename T>
T* working_copy(const Ctx& ctx, Arena& ws, const double* Q, int64_t m, int64_t k, int64_t ldq, int64_t& ld_out) {
  if (std::is_same<T, double>::value) {
    ld_out = ldq;
    return const_cast<T*>(reinterpret_cast<const T*>(Q));
  }
  ld_out = pad4(m);
  T* c = ws.alloc_n<T>(ld_out * k);
  if (ld_out != m) fill_zero(ctx, c, sizeof(T) * ld_out * k);
  convert2d<double, T>(ctx, Q, m, k, ldq, c, ld_out);
  return c;
}
}  // namespace

// ------------------------------------------------------------------ QR (a4)
// Shifted CholeskyQR3 (sCQR3): step 1 with shift 11(mk + k(k+1)) u trace(G), steps 2-3 plain
// CholeskyQR; R = R3 R2 R1, R_ii >= 0 by construction (reading R5).  Gram in fp64.
// shift_dev / row0_dev (nullable): the shift coefficient and this rank's first global row on the
// device (rtucker_qr's row-distributed form, which learns m_glob from an allgather without a host sync)
template <typename T>
void Engine::qr_rows(const T* Y, int64_t m, int64_t m_glob, int k, int64_t ldy, double* Q, int64_t ldq,
                     double* R, bool rows_dist, int64_t row0, const double* shift_dev, const int64_t* row0_dev,
                     int passes) {
  RT_REQUIRE(m_glob >= k, kERANK, "qr: needs m >= k");
  RT_REQUIRE(passes == 3 || (passes == 2 && !R), kEINVAL, "qr: 2 passes only without R");
  const auto mk = ws.mark();
  double* G = ws.alloc_n<double>(int64_t(k) * k);
  double* Rs[3];
  double* Ri = ws.alloc_n<double>(int64_t(k) * k);
  for (int s = 0; s < 3; ++s) Rs[s] = ws.alloc_n<double>(int64_t(k) * k);
  int* zero = ws.alloc_n<int>(1);
  double* Q1 = ws.alloc_n<double>(m * k);
  const bool dist_g = rows_dist && dist();
  // step 1
  gram<T>(ctx, ws, Y, m, k, ldy, G);
  allreduce(comm, dist_g, G, int64_t(k) * k, ctx.stream);
  const double shift = 11.0 * (double(m_glob) * k + double(k) * (k + 1)) * kU;
  chol_inv(ctx, G, k, shift, Rs[0], Ri, zero, shift_dev);
  gemm_tall<T, double>(ctx, Y, m, k, ldy, Ri, k, k, Q1, m, zero, row0, false, row0_dev);
  // steps 2, 3
  for (int s = 1; s < passes; ++s) {
    gram<double>(ctx, ws, Q1, m, k, m, G);
    allreduce(comm, dist_g, G, int64_t(k) * k, ctx.stream);
    chol_inv(ctx, G, k, 0.0, Rs[s], Ri, nullptr);
    if (s < passes - 1) gemm_tall<double, double>(ctx, Q1, m, k, m, Ri, k, k, Q1, m);
    else gemm_tall<double, double>(ctx, Q1, m, k, m, Ri, k, k, Q, ldq);
  }
  if (R) {
    double* T21 = ws.alloc_n<double>(int64_t(k) * k);
    gemm_small(ctx, false, false, k, k, k, Rs[1], k, Rs[0], k, T21, k);
    gemm_small(ctx, false, false, k, k, k, Rs[2], k, T21, k, R, k);
  }
  ws.rewind(mk);
}

// passes = 2 (sCQR2) for a Q that only serves as the basis of a power step (Z = X_(n)^T Q_y; any
// basis of span(Y) gives the same span(X_(n) Z), and R31' re-mixes Q_y anyway): after the shifted step
// kappa(Q_1) ~ 1 for kappa(Y) < ~1e6, and one plain step then reaches orthogonality u kappa(Q_1)^2
void Engine::qr_y(const double* Y, int64_t m, int64_t m_glob, int k, int64_t ldy, double* Q, int64_t ldq,
                  double* R, bool rows_dist, int64_t row0, int passes) {
  qr_rows<double>(Y, m, m_glob, k, ldy, Q, ldq, R, rows_dist, row0, nullptr, nullptr, passes);
}

// X's scales (xs_slot[0] fp16 split, [1] normalizing) from its |x| statistics; on a slab the
// statistics of all ranks are gathered first, so every rank holds the same scales (the partial sums
// of the slab exchanges must agree on them).  n_glob: element count of the whole tensor.
void Engine::finish_scale(const unsigned int* stat, int64_t n_local, int64_t n_glob) {
  if (dist()) {
    double* pair = ws.alloc_n<double>(2);
    double* all = ws.alloc_n<double>(2 * comm->nranks());
    x_stat_pair(ctx, stat, pair);
    comm->allgather(pair, all, 2, ctx.stream);
    x_scale_from_gathered(ctx, all, comm->nranks(), n_glob, xs_slot);
  } else {
    x_scale_from_amax(ctx, stat, n_local, xs_slot);
  }
}

const float* Engine::x_scale(const float* data, int64_t n, int64_t n_glob) {
  RT_REQUIRE(xs_slot != nullptr, kEINVAL, "x_scale: no scale slot");
  if (xs_key != data) {                                   // a separate max|X| pass
    unsigned int* stat = ws.alloc_n<unsigned int>(4);
    x_absmax_stats(ctx, ws, data, n, stat);
    finish_scale(stat, n, n_glob > 0 ? n_glob : n);
    xs_key = data;
  }
  return xs_slot;
}

// Z only conditions the next product Y = X_(n) Z (span(X Z R^-1) = span(X Z)); a single
// CholeskyQR step with a small safety shift keeps it well conditioned.  Z is row-major
// (m x k, row pitch ldz).  split: form of the Z2 copy (1 tf32 [hi | lo], 2 fp16 [hi | lo]).
template <typename T>
bool Engine::qr_z(T* Z, int64_t m, int64_t ldz, int64_t m_glob, int k, bool rows_dist, int64_t row0, T* Z2,
                  int64_t ldz2, int split, const float* xsc) {
  const auto mk = ws.mark();
  double* G = ws.alloc_n<double>(int64_t(k) * k);
  double* Rr = ws.alloc_n<double>(int64_t(k) * k);
  double* Ri = ws.alloc_n<double>(int64_t(k) * k);
  int* zero = ws.alloc_n<int>(1);
  // fp32 Z on the tensor cores: view Z as the 2-way tensor [a=1, I=k, b=m] (element (c, j) at c + k j);
  // its mode-0 "sketch" with B = Z is Z^T Z, and its mode-0 TTM with R^{-1} is Z R^{-1} (in place:
  // every 128-row tile is read completely before it is written, by the one CTA that owns it).
  const bool tc = std::is_same<T, float>::value && !ctx.simt() && ldz == k;
  const Box zb{1, k, m};
  bool done_gram = false;
  if constexpr (std::is_same<T, float>::value) {
    if (tc) {
      LabelScope ls(ctx, "zgram_tc");
      done_gram = ttm_s_tc(ctx, ws, Z, zb, Z, ldz, false, k, G, k);
    }
  }
  if (!done_gram) gram<T>(ctx, ws, Z, m, k, ldz, G, /*rowmajor=*/true);
  allreduce(comm, rows_dist && dist(), G, int64_t(k) * k, ctx.stream);
  (void)m_glob;
  // Shift: the tensor-core Gram carries ~1e-6 relative error (3xTF32, fp32 TMEM segments), far
  // above the fp64 Gram's; Z only conditions the next product (any invertible R keeps span(X Z)),
  // so a shift that dominates that error keeps the Cholesky factor well defined (R2').
  chol_inv(ctx, G, k, done_gram ? 1e-5 : 1e-13, Rr, Ri, zero);
  bool done_apply = false;
  if constexpr (std::is_same<T, float>::value) {
    if (tc) {
      int64_t ldr;
      const float* RiT = working_copy<float>(ctx, ws, Ri, k, k, k, ldr);
      LabelScope ls(ctx, "zapply_tc");
      // Z2 requested: Z R^{-1} written as the pre-split [hi | lo] operand of the next product
      if (Z2) done_apply = ttm_t_tc(ctx, ws, Z, zb, RiT, ldr, k, Z2, 0, 1, ldz2, /*split_out=*/split);
      // fp16 Z2 with a device-side fallback (X scale 0, R29): the tf32 twin of the power product
      // reads the fp32 Z R^-1, applied in place by a launch gated on the same scale
      if (Z2 && split == 2 && xsc)
        RT_REQUIRE(ttm_t_tc(ctx, ws, Z, zb, RiT, ldr, k, Z, 0, 1, ldz, 0, false, nullptr, xsc), kEINVAL,
                   "qr_z: gated in-place apply not launched");
      else done_apply = ttm_t_tc(ctx, ws, Z, zb, RiT, ldr, k, Z, 0, 1, ldz);
    }
  }
  if (!done_apply) gemm_tall<T, T>(ctx, Z, m, k, ldz, Ri, k, k, Z, ldz, zero, row0, /*rowmajor=*/true);
  ws.rewind(mk);
  return done_apply && Z2 != nullptr;
}

// ---------------------------------------------------------------- sketch (a1-a3)
// first_only: the first sketch Y^(0) only (C1 and the non-finite check included), with X's scale
// gathered as for q > 0 -- the driver that overlaps the QRs runs the power steps itself
template <typename T>
void Engine::sketch(const TView& X, const T* data, int n, int kind, const void* const* omega,
                    const int64_t* omega_cols, const int64_t* omega_ld, int q, double* Yt, bool first_only) {
  const int N = X.N;
  const Box bx = X.box(n);
  const bool last = (n == N - 1);
  const int64_t In = bx.I;
  // fp16-split power products (fp32 data): X's scale in a slot that outlives this sketch (the
  // driver's, else one taken here); gathered by the first pass over X when that is a tf32 sketch
  bool own_slot = false;
  const int64_t n_glob = X.size() / X.d[N - 1] * X.glob;
  if (first_only) q = std::max(q, 1);
  if constexpr (std::is_same<T, float>::value) {
    if (q > 0 && !xs_slot) { xs_slot = ws.alloc_n<float>(2); xs_key = nullptr; own_slot = true; }
  }
  int K;
  if (kind == 0) {
    K = int(omega_cols[n]);
    const T* om = static_cast<const T*>(omega[n]);
    int64_t ld = omega_ld[n];
    unsigned int* am = nullptr;
    if (std::is_same<T, float>::value && q > 0 && xs_key != data) {
      am = ws.alloc_n<unsigned int>(4);                 // {max|X| bits, pad, sum |x| (f64)}
      RT_CUDA(cudaMemsetAsync(am, 0, 16, ctx.stream));
    }
    const auto mo = ws.mark();
    if (std::is_same<T, float>::value && !ctx.simt() && (ld % 4) != 0) {
      // the TMA path needs a 16-byte row pitch: repack Omega (J x K, small next to X) with ld = pad4(K)
      const int64_t ldp = pad4(K);
      T* c = ws.alloc_n<T>(bx.J() * ldp);
      convert2d<T, T>(ctx, om, K, bx.J(), ld, c, ldp);
      om = c;
      ld = ldp;
    }
    bool done = false;
    if constexpr (std::is_same<T, float>::value) {
      // X's scale already known (a previous mode's sketch of this call gathered it): the fp16 split
      // (R29) on Omega converted once to fp16 [hi | lo] rows (R34)
      // (not for a thin slab of the slab mode: its Omega is the whole J x K matrix on every rank, and
      // converting it costs more than the fp16 form saves once the slab has fewer than ~8 K rows)
      const bool thin_slab = last && dist() && In < 8 * int64_t(K) && !ctx.thin_slab_off;
      if (xs_slot && xs_key == data && ctx.tc_h16 && !ctx.simt() && !ctx.omega_h16_off && !thin_slab &&
          ttm_s_tc_ok(ctx, data, bx, K)) {
        uint16_t* o2;
        int64_t ld2;
        const float* xso = omega_h16(ctx, ws, om, bx.J(), K, ld, xs_slot, &o2, &ld2);
        LabelScope ls(ctx, "ttm_s_tc");
        done = ttm_s_tc(ctx, ws, data, bx, reinterpret_cast<const float*>(o2), ld2, false, K, Yt, In,
                        /*b_presplit=*/true, xso, nullptr, om, ld, 1.f / 2048.f);
      }
    }
    if (!done && ttm_s_dispatch(ctx, ws, data, bx, om, ld, ctx.omega_tf32 != 0, K, Yt, In, am)) {
      finish_scale(am, X.size(), n_glob);
      xs_key = data;
    }
    ws.rewind(mo);
  } else if (kind == 3) {
    // count sketch: hash, group, sign and sum the columns of X_(n); no multiplications
    K = int(omega_cols[n]);
    count_sketch<T>(ctx, ws, data, bx, static_cast<const int32_t*>(omega[n]), K, Yt, In);
  } else if (kind == 2) {
    // Khatri-Rao sketch (P:510 footnote): Y[:, c] = X x_{k!=n} Omega_k[:, c]^T.  One TTM with the
    // first factor (Omega_k0: I_k0 x K, row-major) streams X; each further mode is a TTV whose
    // vector is the KR column c carried by the k0 coordinate (fp64 sums).
    int k0 = (n == 0) ? 1 : 0;
    K = int(omega_cols[k0]);
    int64_t cur[5];
    for (int k = 0; k < N; ++k) cur[k] = X.d[k];
    const auto mk = ws.mark();
    const Box b0 = TView::box_of(cur, N, k0);
    T* W0 = ws.alloc_n<T>(b0.a * K * b0.b);
    {
      // ttm_t_dispatch takes a col-major Q (I x K); Omega_k0 is row-major -> transposed copy
      const int64_t ldo = pad4(cur[k0]);
      T* qc = ws.alloc_n<T>(ldo * K);
      if (ldo != cur[k0]) fill_zero(ctx, qc, sizeof(T) * ldo * K);
      transpose_copy<T>(ctx, static_cast<const T*>(omega[k0]), cur[k0], K, omega_ld[k0], qc, ldo);
      ttm_t_dispatch(ctx, ws, data, b0, qc, ldo, K, W0, 1, b0.a, b0.a * K, ctx.omega_tf32 != 0);
    }
    cur[k0] = K;
    const void* src = W0;
    bool src_is_T = true;
    for (int m = 0; m < N; ++m) {
      if (m == n || m == k0) continue;
      const Box bm = TView::box_of(cur, N, m);
      int64_t cs = 1;
      const bool c_in_a = k0 < m;
      if (c_in_a) { for (int k = 0; k < k0; ++k) cs *= cur[k]; }
      else { for (int k = m + 1; k < k0; ++k) cs *= cur[k]; }
      double* dst = ws.alloc_n<double>(bm.a * bm.b);
      const T* om = static_cast<const T*>(omega[m]);
      if (src_is_T) kr_ttv<T, T>(ctx, static_cast<const T*>(src), bm, om, omega_ld[m], K, c_in_a, cs, dst);
      else kr_ttv<double, T>(ctx, static_cast<const double*>(src), bm, om, omega_ld[m], K, c_in_a, cs, dst);
      src = dst;
      src_is_T = false;
      cur[m] = 1;
    }
    if (src_is_T) {   // order-2 tensor: no TTV stage; widen W0 to fp64
      double* w64 = ws.alloc_n<double>(b0.a * K * b0.b);
      convert2d<T, double>(ctx, static_cast<const T*>(src), b0.a * K * b0.b, 1, b0.a * K * b0.b, w64,
                           b0.a * K * b0.b);
      src = w64;
    }
    unfold_copy<double>(ctx, static_cast<const double*>(src), TView::box_of(cur, N, n), Yt, In);
    ws.rewind(mk);
  } else {
    // Kronecker sketch W = X x_{k!=n} Omega_k^T (Eq.(2)): a chain of TTMs whose first
    // stage streams X and whose later stages run on the shrunken result.  The factors are narrow
    // (L_k = 2-4), so every stage is an fp64-accumulating CUDA-core contraction with fp64
    // intermediates (HBM-bound at these widths): the chain adds no fp32 rounding.
    int64_t cur[5];
    for (int k = 0; k < N; ++k) cur[k] = X.d[k];
    K = 1;
    for (int k = 0; k < N; ++k) if (k != n) K *= int(omega_cols[k]);
    const auto mk = ws.mark();
    const double* src = nullptr;
    for (int k = 0; k < N; ++k) {
      if (k == n) continue;
      const Box b = TView::box_of(cur, N, k);
      const int L = int(omega_cols[k]);
      double* dst = ws.alloc_n<double>(b.a * L * b.b);
      const T* om = static_cast<const T*>(omega[k]);
      // Omega_k row-major (d_k x L_k, row pitch omega_ld[k]): M(i, c) at i*ld + c
      if (src == nullptr) ttm_t<T, T, double>(ctx, data, b, om, omega_ld[k], 1, L, dst, 1, b.a, b.a * L);
      else                ttm_t<double, T, double>(ctx, src, b, om, omega_ld[k], 1, L, dst, 1, b.a, b.a * L);
      src = dst;
      cur[k] = L;
    }
    unfold_copy<double>(ctx, src, TView::box_of(cur, N, n), Yt, In);
    ws.rewind(mk);   // the Y result is in Yt; intermediates are dead (stream order)
  }
  allreduce(comm, !last && dist(), Yt, In * K, ctx.stream);                       // C1
  set_status_if_nonfinite(ctx, Yt, In * K);
  if (q <= 0 || first_only) {
    if (own_slot) { xs_slot = nullptr; xs_key = nullptr; }
    return;
  }
  // power iterations (reading R2): Q = qr(Y); Z = qr(X_(n)^T Q); Y = X_(n) Z
  const auto mk = ws.mark();
  const int64_t Jl = bx.J();
  double* Qy = ws.alloc_n<double>(In * K);
  const int64_t ldz = pad4(K);             // Z row-major (Jl x K), 16-byte row pitch; pad columns zero
  T* Z = ws.alloc_n<T>(Jl * ldz);
  if (ldz != K) fill_zero(ctx, Z, sizeof(T) * Jl * ldz);
  // fp32 on the tensor cores: the orthonormalized Z is written once in the pre-split [hi | lo] form
  // (row pitch 2 * tc_split_width(K)) so the product Y = X_(n) Z does no split work per tile
  T* Z2 = nullptr;
  int64_t ldz2 = 0;
  int zsplit = 0;
  const float* xsc = nullptr;
  const float* zsc = nullptr;       // Z = sn X^T Q: normalizing power of two of X (fp32 Gram of Z in range)
  if constexpr (std::is_same<T, float>::value) {
    if (!ctx.simt()) zsc = x_scale(data, X.size(), n_glob) + 1;
    if (ctx.tc_h16 && !ctx.simt() && ttm_s_tc_ok(ctx, data, bx, K) && ldz == K) {
      // fp16 split (ttm_s_h16_kernel): Z R^-1 written as fp16 [hi | lo] rows of 2 tc_npad(K) halves
      zsplit = 2;
      ldz2 = 2 * int64_t(tc_npad(K));
      Z2 = reinterpret_cast<T*>(ws.alloc_n<uint16_t>(Jl * ldz2));
      xsc = x_scale(data, X.size(), n_glob);
    } else if (ctx.tc_presplit_z && ttm_s_tc_ok(ctx, data, bx, K) && ldz == K) {
      zsplit = 1;
      ldz2 = 2 * int64_t(tc_split_width(K));
      Z2 = ws.alloc_n<T>(Jl * ldz2);
    }
  }
  const int64_t row0_last = X.off;
  for (int it = 0; it < q; ++it) {
    qr_y(Yt, In, X.Ig(n), K, In, Qy, In, nullptr, last && dist(), last ? row0_last : 0);
    const auto mq = ws.mark();
    bool r31 = false;
    if constexpr (std::is_same<T, float>::value) r31 = zsplit == 2 && !ctx.power_qrz && !(last && dist());
    const double* Qsrc = Qy;
    if constexpr (std::is_same<T, float>::value) {
      if (r31) Qsrc = unmix_q(X, data, n, K, Qy);                                   // R31'
    }
    int64_t ldqt;
    const T* QyT = working_copy<T>(ctx, ws, Qsrc, In, K, In, ldqt);
    // Reading R31 (fp32 data, fp16-split power products, Z rows local): Z is not orthonormalized.
    // span(X_(n) Z R^-1) = span(X_(n) Z) for any invertible R, and Z = X_(n)^T Q_y ~ V_K Sigma_K has
    // near-orthogonal columns, so the product's column errors are those of an orthonormalized Z; a
    // power of two s_z = sn 2^-(ceil(log2 sqrt(I_n)) + 1) bounds |s_z Z| < 1/2 (|z_jc| <= sqrt(I_n)
    // max|X|), and the Z pass writes s_z Z straight into the fp16 [hi | lo] rows of the product's B
    // operand: no Gram / Cholesky / apply passes over Z.  Its tf32 twin (gated on X's fp16 scale
    // being 0) writes the fp32 s_z Z that the product's tf32 twin reads.
    // Z(j, c) = sum_i X_(n)(i, j) Q(i, c), written row-major J x K (j = alpha + a beta):
    // so_a = ldz, so_c = 1, so_b = a ldz
    if constexpr (std::is_same<T, float>::value) {
      if (r31) {
        LabelScope ls(ctx, "ttm_t_tc_pow");
        const int ez = int(std::ceil(0.5 * std::log2(double(X.Ig(n)))));
        const float hz = std::ldexp(1.0f, -(ez + 1));
        RT_REQUIRE(ttm_t_tc(ctx, ws, data, bx, QyT, ldqt, K, reinterpret_cast<float*>(Z2), ldz2, 1, bx.a * ldz2,
                            /*split_out=*/2, false, xsc, nullptr, zsc, hz, /*no_twin=*/true) &&
                       ttm_t_tc(ctx, ws, data, bx, QyT, ldqt, K, Z, ldz, 1, bx.a * ldz, 0, false, nullptr, xsc, zsc, hz),
                   kEUNSUPPORTED, "power iteration: Z pass rejected by the tensor-core path");
      }
    }
    if (!r31) {
      LabelScope ls(ctx, "ttm_t_tc_pow");
      ttm_t_dispatch(ctx, ws, data, bx, QyT, ldqt, K, Z, ldz, 1, bx.a * ldz, false, xsc, zsc);
    }
    ws.rewind(mq);
    if constexpr (std::is_same<T, float>::value) {
      if (r31) {
        LabelScope ls(ctx, "ttm_s_tc_pow");
        RT_REQUIRE(ttm_s_tc(ctx, ws, data, bx, Z2, ldz2, false, K, Yt, In, /*b_presplit=*/true, xsc, nullptr, Z, ldz),
                   kEUNSUPPORTED, "pre-split power product not launched");
        allreduce(comm, !last && dist(), Yt, In * K, ctx.stream);                   // C1
        continue;
      }
    }
    allreduce(comm, last && dist(), Z, Jl * ldz, ctx.stream);                    // C3
    // local Z rows: for n < N-1 the slab's j's are the contiguous block starting at a*b'*off
    int64_t zrow0 = 0;
    if (!last) {
      int64_t bp = 1;
      for (int k = n + 1; k < N - 1; ++k) bp *= X.d[k];
      zrow0 = bx.a * bp * X.off;
    }
    const bool pre = qr_z<T>(Z, Jl, ldz, X.Jg(n), K, !last && dist(), zrow0, Z2, ldz2, zsplit, xsc);
    {
      LabelScope ls(ctx, "ttm_s_tc_pow");
      bool done = false;
      if constexpr (std::is_same<T, float>::value) {
        if (pre) done = ttm_s_tc(ctx, ws, data, bx, Z2, ldz2, false, K, Yt, In, /*b_presplit=*/true, xsc, nullptr,
                                 xsc ? Z : nullptr, ldz);
      }
      RT_REQUIRE(!pre || done, kEUNSUPPORTED, "pre-split power product not launched");
      if (!done) ttm_s_dispatch(ctx, ws, data, bx, Z, ldz, false, K, Yt, In);
    }
    allreduce(comm, !last && dist(), Yt, In * K, ctx.stream);                     // C1
  }
  ws.rewind(mk);
  if (own_slot) { xs_slot = nullptr; xs_key = nullptr; }
}

// Reading R31' (the unmixing of Q_y before an R31 power step).  Z = X_(n)^T Q_y is not orthonormalized
// in R31, and its columns are mixtures of the strong and weak singular directions (Q_y spans the sketch
// in no particular basis); the product X_(n) Z then carries rounding errors of the size of the strong
// directions in every column, which swamp the weak ones (the order-2 test with sigma_1 / sigma_K ~ 400
// lost a factor 20 against the QR of Z).  Orthogonalizing the columns of Z before the product removes
// that, and it can be done on Q_y: with R_S the Cholesky factor of the Gram of a row sample Z_S =
// X_(n)[:, S]^T Q_y (32 blocks of 32 consecutive columns spread over J, the whole Z when J <= 1024),
// Z' = X_(n)^T (Q_y R_S^-1) has near-orthogonal columns (a row sample of a tall matrix gives its Gram
// to a few per cent).  span(X Z') = span(X Z): the result is the oracle's power step; no pass over
// Z.  Columns are scaled by powers of two so that ||Qp[:, c]|| < 1 (the R31 fp16 bound on s_z Z holds
// unchanged).  Collectives: the slab mode's Z_S is a partial sum over the slabs (allreduce), the
// other modes' samples are local rows (allreduce of the Gram).
double* Engine::unmix_q(const TView& X, const float* data, int n, int K, const double* Qy, double* out) {
  const Box bx = X.box(n);
  const bool last = n == X.N - 1;
  const int64_t In = bx.I;
  double* Qp = out ? out : ws.alloc_n<double>(In * K);
  const auto mk = ws.mark();
  const int nblk = int(std::max<int64_t>(1, std::min<int64_t>(32, cdiv(bx.J(), int64_t(32)))));
  const int64_t S = int64_t(nblk) * 32;
  double* Zs = ws.alloc_n<double>(S * K);
  double* G = ws.alloc_n<double>(int64_t(K) * K);
  double* Ri = ws.alloc_n<double>(int64_t(K) * K);
  int* zero = ws.alloc_n<int>(1);
  zsample<float>(ctx, ws, data, bx, nblk, Qy, In, K, Zs);
  allreduce(comm, last && dist(), Zs, S * K, ctx.stream);
  gram<double>(ctx, ws, Zs, S, K, S, G);
  allreduce(comm, !last && dist(), G, int64_t(K) * K, ctx.stream);
  chol_inv(ctx, G, K, 1e-10, nullptr, Ri, zero);
  unmix_cols(ctx, Qy, In, K, In, Ri, zero, Qp, In);
  ws.rewind(mk);
  return Qp;
}

// One power step of reading R31 for mode n: Yt = X_(n) (s_z X_(n)^T Q_y), Q_y fp64 In x K orthonormal
// (the same launches as the R31 branch of sketch, for the driver that overlaps the QRs).  False
// (nothing launched) when the fp16-split form does not apply.
bool Engine::power_step_r31(const TView& X, const float* data, int n, int K, const double* Qy, double* Yt,
                            bool unmixed, PowerBufs* pb, int parts) {
  const int N = X.N;
  const Box bx = X.box(n);
  const bool last = (n == N - 1);
  if (!ctx.tc_h16 || ctx.simt() || ctx.power_qrz || (last && dist()) || !ttm_s_tc_ok(ctx, data, bx, K) || !xs_slot ||
      xs_key != data)
    return false;
  // the fp32 Z of the tf32 twin: 16-byte row pitch (columns >= K are never read)
  const int64_t In = bx.I, Jl = bx.J(), ldz = pad4(K);
  const auto mk = ws.mark();
  const int64_t ldz2 = 2 * int64_t(tc_npad(K));
  PowerBufs local;
  if (!pb) {
    RT_REQUIRE(parts == 3, kEINVAL, "power_step_r31: split parts need caller buffers");
    pb = &local;
  }
  if (!pb->Z) {                                  // caller's buffers outlive this call (split parts)
    pb->Z = ws.alloc_n<float>(Jl * ldz);
    pb->Z2 = reinterpret_cast<float*>(ws.alloc_n<uint16_t>(Jl * ldz2));
  }
  const auto mk2 = ws.mark();
  float* Z = pb->Z;
  float* Z2 = pb->Z2;
  const float* xsc = xs_slot;
  if (parts & 1) {
    int64_t ldqt;
    const double* Qu = unmixed ? Qy : unmix_q(X, data, n, K, Qy);                  // R31'
    const float* QyT = working_copy<float>(ctx, ws, Qu, In, K, In, ldqt);
    const float* zsc = xs_slot + 1;
    const int ez = int(std::ceil(0.5 * std::log2(double(X.Ig(n)))));
    const float hz = std::ldexp(1.0f, -(ez + 1));
    LabelScope ls(ctx, "ttm_t_tc_pow");
    RT_REQUIRE(ttm_t_tc(ctx, ws, data, bx, QyT, ldqt, K, Z2, ldz2, 1, bx.a * ldz2, 2, false, xsc, nullptr, zsc, hz, true) &&
                   ttm_t_tc(ctx, ws, data, bx, QyT, ldqt, K, Z, ldz, 1, bx.a * ldz, 0, false, nullptr, xsc, zsc, hz),
               kEUNSUPPORTED, "power iteration: Z pass rejected by the tensor-core path");
    ws.rewind(mk2);
  }
  if (parts & 2) {
    {
      LabelScope ls(ctx, "ttm_s_tc_pow");
      RT_REQUIRE(ttm_s_tc(ctx, ws, data, bx, Z2, ldz2, false, K, Yt, In, true, xsc, nullptr, Z, ldz), kEUNSUPPORTED,
                 "pre-split power product not launched");
    }
    allreduce(comm, !last && dist(), Yt, In * K, ctx.stream);                       // C1
  }
  if (pb == &local) ws.rewind(mk);
  else ws.rewind(mk2);
  return true;
}

// HOSVD with the thin QRs on a second stream (SURVEY.md H7 / reading R9: the modes are independent):
// every QR of a replicated sketch runs on the handle's side stream while the main stream streams X
// for another mode's sketch or power step; the main stream waits for a QR only when it needs its
// Q.  The slab mode of a distributed run (row-distributed QR with collectives) runs entirely on the
// main stream.  The side stream's allocations come from the handle's second arena, so the main
// stream's scoped reuse never touches them.
// With q > 0 the first core stage G1 = X x_1 Q~_0^T shares its pass over X with the mode-1 Omega sketch
// (sketch1_core0: 10 instead of 11 passes over X for a 3-way tensor): mode 0 is finished first, the
// other modes' power steps hide its last QR, then the fused pass, then mode 1's power steps.
// Order (q = 1, N = 3): S0, S2, P0, P2, [S1 + G1], P1 (S = first sketch, P = Z pass + power product).
bool Engine::hosvd_overlap(const TView& X, const float* data, const int64_t* R, int q, const void* const* omega,
                           const int64_t* omega_cols, const int64_t* omega_ld, double* const* Q_out, double* G_out,
                           double* E, double* Eg) {
  const int N = X.N;
  if (!ctx.side_stream || !ctx.side_ws || !ctx.events || ctx.simt()) return false;
  int64_t K[5];
  for (int n = 0; n < N; ++n) {
    K[n] = omega_cols[n * N + n];
    const bool main_only = dist() && n == N - 1;
    // every power step must take the R31 form (checked before anything is launched)
    if (q > 0 && !main_only &&
        (!ctx.tc_h16 || ctx.power_qrz || !ttm_s_tc_ok(ctx, data, X.box(n), int(K[n]))))
      return false;
  }
  // fused mode-1 sketch + first core stage: needs X's scale (q > 0) and mode 1 off the slab
  const bool try_fuse = q > 0 && N >= 2 && !ctx.fuse_off && ctx.tc_h16 && !(dist() && N - 1 == 1) &&
                        (omega_ld[1 * N + 1] % 4) == 0;
  const auto mk = ws.mark();
  xs_slot = ws.alloc_n<float>(2);
  xs_key = nullptr;
  Ctx sctx = ctx;
  sctx.stream = ctx.side_stream;
  sctx.label = nullptr;
  // slab-parallel: the side stream's engine works on the third communicator (its R31' unmixing steps
  // allreduce a K x K Gram while C3 occupies the side communicator and the main stream's passes the
  // main one); without one the unmixing stays on the main stream
  // (thin slabs only, I_N(local) < 8 K_N: under the long product passes of a thick slab every side-stream
  // kernel waits for a CTA wave of the pass, and five more of them make the chain outlast the pass --
  // measured with tools/rank_share.py: P = 2 42.7 -> 45.0 ms, P = 4 24.3 -> 23.6, P = 8 13.6 -> 13.3)
  Comm* ucomm = dist() ? (X.d[N - 1] < 8 * omega_cols[(N - 1) * N + (N - 1)] && !ctx.thin_slab_off ? comm->side2() : nullptr) : comm;
  const bool side_unmix = !dist() || ucomm != nullptr;
  Engine se(sctx, *ctx.side_ws, ucomm ? ucomm : comm);
  double* Yt[5];
  double* Qy[5];
  double* Qu[5];                               // Qy after the R31' unmixing (side stream, !dist())
  double* Qt[5];
  int64_t ldq[5];
  cudaEvent_t done_q[5];
  auto fork_qr = [&](int n, double* Q) {      // side stream: Q = qr(Yt[n]) after the work enqueued so far
    cudaEvent_t e = ctx.events->get();
    RT_CUDA(cudaEventRecord(e, ctx.stream));
    RT_CUDA(cudaStreamWaitEvent(sctx.stream, e, 0));
    se.qr_y(Yt[n], X.d[n], X.Ig(n), int(K[n]), X.d[n], Q, X.d[n], nullptr, false, 0,
            (Q == Qy[n] && !ctx.qr3_always) ? 2 : 3);
    if (Q == Qy[n] && side_unmix) se.unmix_q(X, data, n, int(K[n]), Qy[n], Qu[n]);   // R31' off the main stream
    done_q[n] = ctx.events->get();
    RT_CUDA(cudaEventRecord(done_q[n], sctx.stream));
  };
  auto wait_q = [&](int n) { RT_CUDA(cudaStreamWaitEvent(ctx.stream, done_q[n], 0)); };
  const int saved_reserve = ctx.sm_reserve;
  ctx.sm_reserve = 2;                         // persistent X-pass grids leave SMs for the side stream
  for (int n = 0; n < N; ++n) {
    const int64_t In = X.d[n];
    Yt[n] = ws.alloc_n<double>(In * K[n]);
    Qy[n] = ws.alloc_n<double>(In * K[n]);
    Qu[n] = ws.alloc_n<double>(In * K[n]);
    Qt[n] = ws.alloc_n<double>(In * K[n]);
    ldq[n] = In;
    done_q[n] = nullptr;
  }
  int it_done[5] = {0, 0, 0, 0, 0};            // power steps taken per mode
  // Slab mode of a distributed run: its power step sums Z = X_(N-1)^T Q over the
  // slabs (C3, J x K: 1.34 GB at cfg5).  C3 overlap (H7): the slab mode's first sketch, QR and Z pass
  // run first, the allreduce of Z goes to a third stream on the side communicator while the main
  // stream processes the other modes, and the slab mode's product Y = X_(N-1) s_z Z (R31) follows
  // once Z is summed; later power iterations of the slab mode allreduce on the main stream.
  const int ns = N - 1;
  const int64_t Jls = X.box(ns).J();
  const bool c3ovl = dist() && q > 0 && comm->side() && ctx.comm_stream && !ctx.power_qrz && ctx.tc_h16 &&
                     ttm_s_tc_ok(ctx, data, X.box(ns), int(K[ns]));
  const int64_t ldzs = pad4(K[ns]);            // 16-byte row pitch of the slab mode's fp32 Z
  float* Zs = c3ovl ? ws.alloc_n<float>(Jls * ldzs) : nullptr;
  if (Zs && ldzs != K[ns]) fill_zero(ctx, Zs, sizeof(float) * Jls * ldzs);   // pad columns (summed by C3)
  // the summed Z as fp16 [hi | lo] rows (the first product's B operand): converted on the C3 stream right
  // after the allreduce, so the 2 |Z| conversion pass hides under the other modes' X passes too
  // (a thin slab, I_N(local) < 8 K, skips it: there |Z| is a large part of the product's traffic, and the
  // 3xTF32 kernel that splits the fp32 Z in flight costs less than a conversion pass plus the fp16 form)
  const bool thin_slab = X.d[ns] < 8 * K[ns] && !ctx.thin_slab_off;
  const int64_t ldz2s = c3ovl ? 2 * int64_t(tc_npad(int(K[ns]))) : 0;
  uint16_t* Z2s = c3ovl && !thin_slab ? ws.alloc_n<uint16_t>(Jls * ldz2s) : nullptr;
  cudaEvent_t c3_done = nullptr;
  // the slab mode's Z pass: Zs = s_z X_(N-1)^T Qy (fp32 partial sums of this slab), h16 pair
  auto slab_zpass = [&]() {
    const Box bx = X.box(ns);
    const auto mz = ws.mark();
    int64_t ldqt;
    const double* Qu = unmix_q(X, data, ns, int(K[ns]), Qy[ns]);                    // R31'
    const float* QyT = working_copy<float>(ctx, ws, Qu, X.d[ns], K[ns], X.d[ns], ldqt);
    const int ez = int(std::ceil(0.5 * std::log2(double(X.Ig(ns)))));
    LabelScope ls(ctx, "ttm_t_tc_pow");
    RT_REQUIRE(ttm_t_tc(ctx, ws, data, bx, QyT, ldqt, int(K[ns]), Zs, ldzs, 1, bx.a * ldzs, 0, false, xs_slot, nullptr,
                        xs_slot + 1, std::ldexp(1.0f, -(ez + 1))),
               kEUNSUPPORTED, "slab mode: Z pass rejected by the tensor-core path");
    ws.rewind(mz);
  };
  // the slab mode's product from the summed Zs: Yt = X_(N-1) Zs (fp16 split rows), then its QR
  auto slab_product = [&](bool final_qr, bool presplit) {
    const Box bx = X.box(ns);
    const auto mz = ws.mark();
    const int64_t ldz2 = ldz2s;
    uint16_t* Z2 = Z2s;
    if (!presplit && Z2) split_rows_h16(ctx, Zs, Jls, int(K[ns]), ldzs, Z2);
    if (!Z2) {
      LabelScope ls(ctx, "ttm_s_tc_pow");
      ttm_s_dispatch(ctx, ws, data, bx, Zs, ldzs, false, int(K[ns]), Yt[ns], X.d[ns]);
    } else {
      LabelScope ls(ctx, "ttm_s_tc_pow");
      RT_REQUIRE(ttm_s_tc(ctx, ws, data, bx, reinterpret_cast<const float*>(Z2), ldz2, false, int(K[ns]), Yt[ns],
                          X.d[ns], true, xs_slot, nullptr, Zs, ldzs),
                 kEUNSUPPORTED, "slab mode: power product not launched");
    }
    ws.rewind(mz);
    qr_y(Yt[ns], X.d[ns], X.Ig(ns), int(K[ns]), X.d[ns], final_qr ? Qt[ns] : Qy[ns], X.d[ns], nullptr, true, X.off,
         (final_qr || ctx.qr3_always) ? 3 : 2);
  };
  bool slab_finished = false;
  auto finish_slab = [&]() {                   // after the other modes: the slab mode's remaining steps
    if (!c3ovl || slab_finished) return;
    slab_finished = true;
    RT_CUDA(cudaStreamWaitEvent(ctx.stream, c3_done, 0));
    slab_product(q == 1, true);
    for (int it = 1; it < q; ++it) {
      slab_zpass();
      allreduce(comm, true, Zs, Jls * ldzs, ctx.stream);                                            // C3
      slab_product(it == q - 1, false);
    }
  };
  auto first_sketch = [&](int n) {
    const void* const* om = omega + n * N;
    const int64_t* oc = omega_cols + n * N;
    const int64_t* ol = omega_ld + n * N;
    if (dist() && n == N - 1) {               // slab mode: the whole mode on the main stream
      if (c3ovl) return;                       // (overlapped: started above, finished by finish_slab)
      sketch<float>(X, data, n, 0, om, oc, ol, q, Yt[n]);
      qr_y(Yt[n], X.d[n], X.Ig(n), int(K[n]), X.d[n], Qt[n], X.d[n], nullptr, true, X.off);
      it_done[n] = q;
      return;
    }
    sketch<float>(X, data, n, 0, om, oc, ol, q, Yt[n], /*first_only=*/true);
    fork_qr(n, q > 0 ? Qy[n] : Qt[n]);
  };
  auto power_all = [&](int n) {               // the remaining power steps of mode n
    if (dist() && n == N - 1) return;
    for (; it_done[n] < q; ++it_done[n]) {
      wait_q(n);
      RT_REQUIRE(power_step_r31(X, data, n, int(K[n]), side_unmix ? Qu[n] : Qy[n], Yt[n], side_unmix), kEUNSUPPORTED, "power step not launched");
      fork_qr(n, it_done[n] == q - 1 ? Qt[n] : Qy[n]);
    }
  };
  bool sketched0 = false;
  if (c3ovl) {
    // mode 0's first sketch goes first: its QR (side stream) runs beside the slab mode's sketch and
    // row-distributed QR (main stream, C2)
    if (ns != 0) { first_sketch(0); sketched0 = true; }
    sketch<float>(X, data, ns, 0, omega + ns * N, omega_cols + ns * N, omega_ld + ns * N, q, Yt[ns], true);
    qr_y(Yt[ns], X.d[ns], X.Ig(ns), int(K[ns]), X.d[ns], Qy[ns], X.d[ns], nullptr, true, X.off,
         ctx.qr3_always ? 3 : 2);                                                                 // C2
    slab_zpass();
    cudaEvent_t e = ctx.events->get();
    RT_CUDA(cudaEventRecord(e, ctx.stream));
    RT_CUDA(cudaStreamWaitEvent(ctx.comm_stream, e, 0));
    comm->side()->allreduce_sum(Zs, size_t(Jls * ldzs), ctx.comm_stream);                            // C3
    if (Z2s) {
      Ctx cctx = ctx;
      cctx.stream = ctx.comm_stream;
      cctx.label = nullptr;
      split_rows_h16(cctx, Zs, Jls, int(K[ns]), ldzs, Z2s, /*max_ctas=*/4 * ctx.num_sms);
    }
    c3_done = ctx.events->get();
    RT_CUDA(cudaEventRecord(c3_done, ctx.comm_stream));
  }
  float* g1 = nullptr;                         // the first core stage from the fused pass
  float* g2 = nullptr;                         // and the second (modes 0 and 1 contracted), two-fusion schedule
  PowerBufs pbs[5];
  bool deferred[5] = {false, false, false, false, false};
  // Two fused passes (N = 3, q = 1, one rank): the mode-0 contraction of X feeds Z_0 (the power step
  // of mode 0) together with mode 1's Omega sketch, and later the first core stage together with the
  // last mode's Omega sketch (X viewed with the last mode as rows).  9 passes over X:
  //   S0, [Z0 + S1], Y0, Z1, [G1 + S2], Y1, Z2, Y2, residual
  // QR(S0) is exposed (the Omega_1 and Omega_2 conversions run under it); QR(S1) hides under Y0, the last QR of
  // mode 0 under Z1, QR(S2) under Y1; the final QR of mode 2 closes the sketch phase.
  const bool try_fuse2 = try_fuse && N == 3 && q == 1 && !dist() && !ctx.fuse2_off && (omega_ld[2 * N + 2] % 4) == 0 &&
                         X.d[0] % 512 == 0 && X.d[1] % 128 == 0 && X.d[2] % 128 == 0 && K[0] % 4 == 0 &&
                         K[0] == K[1] && K[0] == K[2] && tc_npad(int(K[0])) > 0 && tc_npad(int(K[0])) <= 80;
  if (try_fuse2) {
    const Box b0 = X.box(0), b1 = X.box(1);
    const Box b2v{X.d[0], X.d[2], X.d[1]};     // [alpha = i0, rows = i2, beta = i1]
    const int npad = tc_npad(int(K[0]));
    first_sketch(0);                           // S0: X's scale; QR + unmixing of mode 0 on the side stream
    F1Prep pre1, pre2;
    // both fp16 Omega^T conversions now, on the main stream under QR(S0) (1.2 ms against ~1 ms)
    const bool p1 = sketch1_core0_prep(ctx, ws, static_cast<const float*>(omega[1 * N + 1]), b1.J(), int(K[1]),
                                       omega_ld[1 * N + 1], npad, &pre1);
    const bool p2 = sketch1_core0_prep(ctx, ws, static_cast<const float*>(omega[2 * N + 2]), b2v.J(), int(K[2]),
                                       omega_ld[2 * N + 2], npad, &pre2);
    // [Z0 + S1]
    const int64_t Jl0 = b0.J(), ldz = pad4(K[0]), ldz2 = 2 * int64_t(npad);
    pbs[0].Z = ws.alloc_n<float>(Jl0 * ldz);
    pbs[0].Z2 = reinterpret_cast<float*>(ws.alloc_n<uint16_t>(Jl0 * ldz2));
    wait_q(0);
    bool fused1;
    {
      const auto mz = ws.mark();
      int64_t ldqt;
      const float* QyT = working_copy<float>(ctx, ws, Qu[0], X.d[0], K[0], X.d[0], ldqt);
      const int ez = int(std::ceil(0.5 * std::log2(double(X.Ig(0)))));
      F1ZOut zo{pbs[0].Z, ldz, reinterpret_cast<uint16_t*>(pbs[0].Z2), ldz2, xs_slot + 1, std::ldexp(1.0f, -(ez + 1)),
                xs_slot};
      LabelScope ls(ctx, "sketch1_z0");
      fused1 = sketch1_core0(ctx, ws, data, b1, b0, static_cast<const float*>(omega[1 * N + 1]), omega_ld[1 * N + 1],
                             int(K[1]), QyT, ldqt, int(K[0]), xs_slot, Yt[1], X.d[1], nullptr, 0, p1 ? &pre1 : nullptr,
                             &zo);
      ws.rewind(mz);
    }
    if (fused1) {
      set_status_if_nonfinite(ctx, Yt[1], X.d[1] * K[1]);
      fork_qr(1, Qy[1]);
    } else {
      RT_REQUIRE(power_step_r31(X, data, 0, int(K[0]), Qu[0], Yt[0], true, &pbs[0], 1), kEUNSUPPORTED,
                 "power step (Z pass) not launched");
      first_sketch(1);
    }
    // Y0, then Z1 (under it: QR(S1), then the last QR of mode 0)
    RT_REQUIRE(power_step_r31(X, data, 0, int(K[0]), nullptr, Yt[0], true, &pbs[0], 2), kEUNSUPPORTED,
               "power step (product) not launched");
    fork_qr(0, Qt[0]);
    wait_q(1);
    RT_REQUIRE(power_step_r31(X, data, 1, int(K[1]), Qu[1], Yt[1], true, &pbs[1], 1), kEUNSUPPORTED,
               "power step (Z pass) not launched");
    wait_q(0);
    // [G1 + S2]
    bool fused2;
    {
      int64_t ld0;
      const float* q0 = working_copy<float>(ctx, ws, Qt[0], X.d[0], K[0], ldq[0], ld0);
      float* g = ws.alloc_n<float>(b0.b * K[0]);
      {
        LabelScope ls(ctx, "sketch2_core0");
        fused2 = sketch1_core0(ctx, ws, data, b2v, b0, static_cast<const float*>(omega[2 * N + 2]),
                               omega_ld[2 * N + 2], int(K[2]), q0, ld0, int(K[0]), xs_slot, Yt[2], X.d[2], g, 1,
                               p2 ? &pre2 : nullptr, nullptr);
      }
      if (fused2) {
        set_status_if_nonfinite(ctx, Yt[2], X.d[2] * K[2]);
        fork_qr(2, Qy[2]);
        g1 = g;
      } else {
        first_sketch(2);
      }
    }
    // Y1 (under it: QR(S2)), Z2, Y2
    RT_REQUIRE(power_step_r31(X, data, 1, int(K[1]), nullptr, Yt[1], true, &pbs[1], 2), kEUNSUPPORTED,
               "power step (product) not launched");
    fork_qr(1, Qt[1]);
    wait_q(2);
    RT_REQUIRE(power_step_r31(X, data, 2, int(K[2]), Qu[2], Yt[2], true), kEUNSUPPORTED, "power step not launched");
    fork_qr(2, Qt[2]);
    // While the last QR (mode 2) runs on the side stream, the main stream contracts mode 1 of the first
    // core stage (Q~_1 has been final since the passes of mode 2 began): G2 = G1 x_2 Q~_1^T, the 1.3 GB
    // read of the core's second stage.  What waits for Q~_2 is then one small stage on K_0 x K_1 x I_3.
    // The persistent grid leaves 24 SMs to the QR's kernels.
    if (g1 && !ctx.core_early_off) {
      wait_q(1);
      int64_t ld1;
      const float* q1 = working_copy<float>(ctx, ws, Qt[1], X.d[1], K[1], ldq[1], ld1);
      const Box bm{K[0], X.d[1], X.d[2]};
      g2 = ws.alloc_n<float>(K[0] * K[1] * X.d[2]);
      ctx.sm_reserve = 24;
      {
        LabelScope ls(ctx, "core_mid");
        ttm_t_dispatch(ctx, ws, g1, bm, q1, ld1, int(K[1]), g2, 1, bm.a, bm.a * K[1]);
      }
      ctx.sm_reserve = 2;
    }
  } else if (try_fuse) {
    if (!sketched0) first_sketch(0);
    for (int n = 2; n < N; ++n) first_sketch(n);
    power_all(0);                              // Q~_0 after its last QR
    // modes 2..N-1: every power step, but the product of the last one waits until after the fused
    // pass, so that both the last QR of mode 0 (needed by the fused pass) and the QR of the fused
    // pass's mode-1 sketch (needed by mode 1's Z pass) run under an X pass:
    //   S0, S2, Z0, Y0, Z2, [S1 + G1], Y2, Z1, Y1
    for (int n = 2; n < N; ++n) {
      if (dist() && n == N - 1) continue;
      for (; it_done[n] < q - 1; ++it_done[n]) {
        wait_q(n);
        RT_REQUIRE(power_step_r31(X, data, n, int(K[n]), side_unmix ? Qu[n] : Qy[n], Yt[n], side_unmix), kEUNSUPPORTED,
                   "power step not launched");
        fork_qr(n, Qy[n]);
      }
      wait_q(n);
      RT_REQUIRE(power_step_r31(X, data, n, int(K[n]), side_unmix ? Qu[n] : Qy[n], Yt[n], side_unmix, &pbs[n], 1),
                 kEUNSUPPORTED, "power step (Z pass) not launched");
      deferred[n] = true;
    }
    wait_q(0);
    const Box b1 = X.box(1), b0 = X.box(0);
    int64_t ld0;
    const float* q0 = working_copy<float>(ctx, ws, Qt[0], X.d[0], K[0], ldq[0], ld0);
    float* g = ws.alloc_n<float>(b0.b * K[0]);
    bool fused;
    {
      LabelScope ls(ctx, "sketch1_core0");
      fused = sketch1_core0(ctx, ws, data, b1, b0, static_cast<const float*>(omega[1 * N + 1]), omega_ld[1 * N + 1],
                            int(K[1]), q0, ld0, int(K[0]), xs_slot, Yt[1], X.d[1], g);
    }
    if (fused) {
      allreduce(comm, N - 1 != 1 && dist(), Yt[1], X.d[1] * K[1], ctx.stream);   // C1
      set_status_if_nonfinite(ctx, Yt[1], X.d[1] * K[1]);
      fork_qr(1, Qy[1]);
      g1 = g;
    } else {
      first_sketch(1);
    }
    // slab-parallel: the slab mode's product (C3 has had modes 0's passes and the fused pass to finish)
    // goes here, so that the QR of mode 1's sketch runs under it instead of holding up mode 1's Z pass
    finish_slab();
    for (int n = 2; n < N; ++n) {              // the deferred products (under them: mode 1's QR)
      if (!deferred[n]) continue;
      RT_REQUIRE(power_step_r31(X, data, n, int(K[n]), nullptr, Yt[n], true, &pbs[n], 2), kEUNSUPPORTED,
                 "power step (product) not launched");
      fork_qr(n, Qt[n]);
      it_done[n] = q;
    }
    power_all(1);
  } else {
    for (int n = 0; n < N; ++n)
      if (!(n == 0 && sketched0)) first_sketch(n);
    for (int it = 0; it < q; ++it)           // power steps, iteration outer
      for (int n = 0; n < N; ++n) {
        if (dist() && n == N - 1) continue;
        wait_q(n);
        RT_REQUIRE(power_step_r31(X, data, n, int(K[n]), side_unmix ? Qu[n] : Qy[n], Yt[n], side_unmix), kEUNSUPPORTED, "power step not launched");
        fork_qr(n, it == q - 1 ? Qt[n] : Qy[n]);
      }
  }
  finish_slab();
  for (int n = 0; n < N; ++n)
    if (done_q[n]) wait_q(n);                  // join
  ctx.sm_reserve = saved_reserve;
  int64_t gsz = 1;
  for (int n = 0; n < N; ++n) gsz *= K[n];
  double* Gt = ws.alloc_n<double>(gsz);
  if (g2) {
    // the last stage: G~ = G2 x_3 Q~_2^T (fp64 sums, as core()'s last stage)
    int64_t ld2;
    const float* q2 = working_copy<float>(ctx, ws, Qt[2], X.d[2], K[2], ldq[2], ld2);
    const Box bl{K[0] * K[1], X.d[2], 1};
    LabelScope ls(ctx, "core_last");
    ttm_t<float, float, double>(ctx, g2, bl, q2, 1, ld2, int(K[2]), Gt, 1, bl.a, bl.a * K[2]);
  } else {
    core<float>(X, data, Qt, ldq, K, Gt, g1);
  }
  // distributed: the truncation's one collective (the sign candidates of the row-distributed last
  // factor, canon) goes to the side communicator (C3 finished before the slab mode's product), the
  // residual pass's C5 stays on the main one: two communicators, two streams
  Comm* tcomm = dist() ? comm->side() : comm;
  if ((E || Eg) && (!dist() || tcomm) && !ctx.split_resid_off) {
    Engine st(sctx, *ctx.side_ws, tcomm);
    // Reading R35: E^2 ||X||^2 = ||X - X^_K||^2 + ||G~||^2 - ||G||^2 with X^_K = G~ x_n Q~_n (the
    // rank-K reconstruction): the truncation (Jacobi, lift, sign canon, core shrink) runs on the side
    // stream while the residual pass streams X against X^_K, which does not depend on it
    double* sums = ws.alloc_n<double>(2);
    double* ggK = ws.alloc_n<double>(1);
    double* ggR = ws.alloc_n<double>(1);
    float* rs = ws.alloc_n<float>(2);
    cudaEvent_t e = ctx.events->get();
    RT_CUDA(cudaEventRecord(e, ctx.stream));
    RT_CUDA(cudaStreamWaitEvent(sctx.stream, e, 0));
    cudaEvent_t pre_eig = dist() ? ctx.events->get() : nullptr;
    st.pre_eig_event = pre_eig;
    st.truncate(X, Gt, K, Qt, ldq, R, Q_out, G_out);
    int64_t gsz = 1;
    for (int n = 0; n < N; ++n) gsz *= R[n];
    sumsq(sctx, st.ws, G_out, gsz, ggR);
    cudaEvent_t done_t = ctx.events->get();
    RT_CUDA(cudaEventRecord(done_t, sctx.stream));
    // the truncation's Jacobi CTAs run beside the residual: 3 SMs (its two-CTA clusters then take turns,
    // still far inside a whole-tensor residual pass); on a slab the residual is short and the Jacobi is
    // the longer branch: 2 SMs for each of the N clusters
    ctx.sm_reserve = dist() ? 2 * N : 3;
    // (on a slab the short residual pass would otherwise take its SMs a moment before the Jacobi is
    // launched, and scattered leftover SMs cannot host the clusters until it ends)
    if (pre_eig) RT_CUDA(cudaStreamWaitEvent(ctx.stream, pre_eig, 0));
    const double* Qtc[5];
    for (int n = 0; n < N; ++n) Qtc[n] = Qt[n];
    resid_sums<float>(X, data, Gt, K, Qtc, sums, ggK, rs, true);
    ctx.sm_reserve = saved_reserve;
    RT_CUDA(cudaStreamWaitEvent(ctx.stream, done_t, 0));
    finalize_err_split(ctx, sums, ggK, ggR, E, Eg, rs);
  } else {
    truncate(X, Gt, K, Qt, ldq, R, Q_out, G_out);
    if (E || Eg) rel_error<float>(X, data, G_out, R, Q_out, E, Eg, true);
  }
  ws.rewind(mk);
  xs_slot = nullptr;
  return true;
}

// ---------------------------------------------------------------------- core (a5)
// stage0 (nullable): the first stage X x_1 Q~_0^T already computed (the fused pass of hosvd_overlap)
template <typename T>
void Engine::core(const TView& X, const T* data, const double* const* Qt, const int64_t* ldq, const int64_t* K,
                  double* Gt, const T* stage0) {
  const int N = X.N;
  const auto mk = ws.mark();
  const T* QT[5];
  int64_t ldt[5];
  for (int n = 0; n < N; ++n) QT[n] = working_copy<T>(ctx, ws, Qt[n], X.d[n], K[n], ldq[n], ldt[n]);
  int64_t cur[5];
  for (int k = 0; k < N; ++k) cur[k] = X.d[k];
  // contraction order 0, N-1, N-2, ..., 1 (the core is multilinear; any order gives G): the first
  // stage streams X, and the second then contracts the slowest mode of the shrunken tensor, whose
  // rows (a = K_0 I_1 ... I_{N-2}) fill whole 128-row tiles; contracting mode 1 second would
  // leave a = K_0 < 128 rows per tile (2/3 of each tile empty at K_0 = 80).
  int ord[5];
  ord[0] = 0;
  for (int s2 = 1; s2 < N; ++s2) ord[s2] = N - s2;
  const T* src = data;
  for (int s2 = 0; s2 < N; ++s2) {
    const int n = ord[s2];
    const Box b = TView::box_of(cur, N, n);
    const int64_t ld = ldt[n];
    if (s2 == N - 1) {
      LabelScope ls(ctx, "core_last");
      ttm_t<T, T, double>(ctx, src, b, QT[n], 1, ld, int(K[n]), Gt, 1, b.a, b.a * K[n]);
    } else if (s2 == 0 && stage0) {
      src = stage0;
    } else {
      T* dst = ws.alloc_n<T>(b.a * K[n] * b.b);
      LabelScope ls(ctx, s2 == 0 ? "core_first" : "core_mid");
      // the first stage streams X: fp16 split when X's scale is already known (a driver's sketches)
      const float* xsc = nullptr;
      if constexpr (std::is_same<T, float>::value) {
        if (s2 == 0 && ctx.tc_h16 && xs_slot && xs_key == data) xsc = xs_slot;
      }
      ttm_t_dispatch(ctx, ws, src, b, QT[n], ld, int(K[n]), dst, 1, b.a, b.a * K[n], false, xsc);
      src = dst;
    }
    cur[n] = K[n];
  }
  int64_t gsz = 1;
  for (int n = 0; n < N; ++n) gsz *= K[n];
  allreduce(comm, dist(), Gt, gsz, ctx.stream);                                  // C4
  ws.rewind(mk);
}

// ------------------------------------------------------------- sign canon (R5)
void Engine::canon(double* Qn, int64_t m, int r, int64_t ld, int64_t row0, bool dist_rows, double* U, int ku) {
  const auto mk = ws.mark();
  double* cand = ws.alloc_n<double>(3 * r);
  colmax_candidates(ctx, Qn, m, r, ld, row0, cand);
  int nc = 1;
  if (dist_rows && dist()) {
    nc = comm->nranks();
    double* all = ws.alloc_n<double>(3 * r * nc);
    comm->allgather(cand, all, size_t(3 * r), ctx.stream);
    cand = all;
  }
  sign_apply(ctx, cand, nc, Qn, m, r, ld, U, ku, ku);
  ws.rewind(mk);
}

// ------------------------------------------------------------- truncation (a6)
void Engine::truncate(const TView& X, const double* Gt, const int64_t* K, const double* const* Qt,
                      const int64_t* ldq, const int64_t* R, double* const* Q_out, double* G_out) {
  const int N = X.N;
  const auto mk = ws.mark();
  double* V[5];
  double* W[5];
  double* M[5];
  int kk[5];
  for (int n = 0; n < N; ++n) {
    kk[n] = int(K[n]);
    M[n] = ws.alloc_n<double>(int64_t(kk[n]) * kk[n]);
    V[n] = ws.alloc_n<double>(int64_t(kk[n]) * kk[n]);
    W[n] = ws.alloc_n<double>(kk[n]);
    // M_n = G~_(n) G~_(n)^T (Gram-EVD)
    gram_unfold(ctx, ws, Gt, TView::box_of(K, N, n), M[n]);
  }
  if (pre_eig_event) RT_CUDA(cudaEventRecord(pre_eig_event, ctx.stream));
  eig_sym_batch(ctx, ws, N, M, kk, W, V);
  for (int n = 0; n < N; ++n) {
    const int k = kk[n];
    // Q_n = Q~_n U_n, U_n = V_n[:, :R_n]; sign canonicalization on the lifted factor
    gemm_tall<double, double>(ctx, Qt[n], X.d[n], k, ldq[n], V[n], int(R[n]), k, Q_out[n], X.d[n]);
    canon(Q_out[n], X.d[n], int(R[n]), X.d[n], n == N - 1 ? X.off : 0, n == N - 1, V[n], k);
  }
  // G = G~ x_1 U_1^T ... x_N U_N^T
  int64_t cur[5];
  for (int k = 0; k < N; ++k) cur[k] = K[k];
  const double* src = Gt;
  for (int n = 0; n < N; ++n) {
    const Box b = TView::box_of(cur, N, n);
    double* dst = (n == N - 1) ? G_out : ws.alloc_n<double>(b.a * R[n] * b.b);
    LabelScope ls(ctx, "trunc_simt");
    ttm_t<double, double, double>(ctx, src, b, V[n], 1, K[n], int(R[n]), dst, 1, b.a, b.a * R[n]);
    src = dst;
    cur[n] = R[n];
  }
  ws.rewind(mk);
}

// ------------------------------------------------------------- residual (a8)
// ortho_q: the factors are orthonormal (the drivers' own output), so ||P||_F = ||G||_F bounds P's
// entries and the fp16-split residual may scale P from ||G||; a caller's factors (rtucker_core) take
// the tf32 residual
template <typename T>
void Engine::rel_error(const TView& X, const T* data, const double* G, const int64_t* R, const double* const* Q,
                       double* E, double* Eg, bool ortho_q) {
  const auto mk = ws.mark();
  double* sums = ws.alloc_n<double>(2);
  double* gg = ws.alloc_n<double>(1);
  float* rs = ws.alloc_n<float>(2);
  resid_sums<T>(X, data, G, R, Q, sums, gg, rs, ortho_q);
  finalize_err(ctx, sums, gg, E, Eg, rs);
  ws.rewind(mk);
}

// the residual pass: sums = (sum (s x - s x^)^2, sum (s x)^2) over the whole tensor (C5 included),
// gg = ||G||^2, rs = the residual scales (resid_scale) for X^ = G x_1 Q_1 ... x_N Q_N
template <typename T>
void Engine::resid_sums(const TView& X, const T* data, const double* G, const int64_t* R, const double* const* Q,
                        double* sums, double* gg, float* rs, bool ortho_q) {
  const int N = X.N;
  const auto mk = ws.mark();
  int64_t gsz = 1;
  for (int n = 0; n < N; ++n) gsz *= R[n];
  sumsq(ctx, ws, G, gsz, gg);
  if constexpr (std::is_same<T, float>::value) {
    // Slab form (a thin slab of a slab-parallel call, N >= 3, wide R): the kernel contracts mode N-1
    // (the second to last) instead of the slab mode.  P' = G x_N Q_N[local rows] x_{k < N-1} Q_k is
    // J' x R_{N-1} x I_N(local) with J' = I_1 ... I_{N-2}: it shrinks with the slab, where the P of the
    // form below is the whole J x R_N tensor on every rank (1.34 GB at cfg5, written and read again).
    // Every slice i_N is one problem X[:, :, i_N] ~ P'[:, :, i_N] Q_{N-1}^T of the same kernel.
    const int m = N - 2;
    int64_t Jp = 1;
    for (int k = 0; k < m; ++k) Jp *= X.d[k];
    const int64_t Il = X.d[N - 1];
    if (dist() && N >= 3 && !ctx.resid_slab_off && !ctx.simt() && R[m] > 64 && R[m] <= 128 && (Jp % 4) == 0 &&
        Il * R[m] * 2 <= X.d[m] * R[N - 1] && Il > 1) {
      int64_t cur[5];
      for (int k = 0; k < N; ++k) cur[k] = R[k];
      // the slab mode first (fp64, small), then modes N-3 .. 0 (the widest stage last, as below)
      const double* src = G;
      {
        const Box b = TView::box_of(cur, N, N - 1);
        double* dst = ws.alloc_n<double>(b.a * Il * b.b);
        LabelScope ls(ctx, "pchain");
        ttm_t<double, double, double>(ctx, src, b, Q[N - 1], Il, 1, int(Il), dst, 1, b.a, b.a * Il);
        src = dst;
        cur[N - 1] = Il;
      }
      float* Pp = nullptr;
      for (int n = m - 1; n >= 0; --n) {
        const Box b = TView::box_of(cur, N, n);
        const int64_t In = X.d[n];
        LabelScope ls(ctx, "pchain");
        if (n == 0) {
          Pp = ws.alloc_n<float>(b.a * In * b.b);
          float* sf = ws.alloc_n<float>(b.a * b.I * b.b);
          float* qf = ws.alloc_n<float>(In * b.I);
          convert2d<double, float>(ctx, src, b.a * b.I * b.b, 1, b.a * b.I * b.b, sf, b.a * b.I * b.b);
          convert2d<double, float>(ctx, Q[n], In, b.I, In, qf, In);
          const int64_t ldt = pad4(b.I);
          float* qt = ws.alloc_n<float>(ldt * In);
          if (ldt != b.I) fill_zero(ctx, qt, sizeof(float) * ldt * In);
          transpose_copy<float>(ctx, qf, b.I, In, In, qt, ldt);
          ttm_t_dispatch(ctx, ws, sf, b, qt, ldt, int(In), Pp, 1, b.a, b.a * In);
        } else {
          double* dst = ws.alloc_n<double>(b.a * In * b.b);
          ttm_t<double, double, double>(ctx, src, b, Q[n], In, 1, int(In), dst, 1, b.a, b.a * In);
          src = dst;
        }
        cur[n] = In;
      }
      const int Rm = int(R[m]);
      float* qm = ws.alloc_n<float>(X.d[m] * Rm);
      convert2d<double, float>(ctx, Q[m], X.d[m], Rm, X.d[m], qm, X.d[m]);
      resid_scale(ctx, gg, double(X.size()) * double(X.glob) / double(X.d[N - 1]), rs);
      if (residual_tc(ctx, ws, data, Jp, X.d[m], Pp, Jp, Rm, qm, X.d[m], sums, rs, ortho_q ? rs + 1 : nullptr, Il,
                      Jp * X.d[m], Jp * Rm)) {
        allreduce(comm, dist(), sums, 2, ctx.stream);                              // C5
        ws.rewind(mk);
        return;
      }
      ws.rewind(mk);
    }
  }
  // P = G x_1 Q_1 ... x_{N-1} Q_{N-1} (all but the last mode), then the residual kernel
  // rebuilds X^ = P x_N Q_N tile by tile against X.  The modes are contracted from N-2 down to 0,
  // so that the widest stage (|P| outputs) contracts mode 0: its new index i_0 is the contiguous
  // one, and the tensor-core kernel writes whole rows by TMA stores (1.3 -> ~0.4 ms at cfg5)
  int64_t cur[5];
  for (int k = 0; k < N; ++k) cur[k] = R[k];
  const double* src = G;
  T* P = nullptr;
  for (int n = N - 2; n >= 0; --n) {
    const Box b = TView::box_of(cur, N, n);
    const int64_t In = X.d[n];
    LabelScope ls(ctx, "pchain");
    if (n == 0) {
      P = ws.alloc_n<T>(b.a * In * b.b);
      if constexpr (std::is_same<T, float>::value) {
        // the widest stage (|P| = |X| R_N / I_N outputs): fp32 operands and accumulation (P is
        // consumed in fp32 by the residual kernel; R_n-term dot products)
        float* sf = ws.alloc_n<float>(b.a * b.I * b.b);
        float* qf = ws.alloc_n<float>(In * b.I);
        convert2d<double, float>(ctx, src, b.a * b.I * b.b, 1, b.a * b.I * b.b, sf, b.a * b.I * b.b);
        convert2d<double, float>(ctx, Q[n], In, b.I, In, qf, In);
        // tensor cores: M(i = r, c = i_n) = Q[i_n, r] as a col-major R x I_n matrix (ld pad4(R));
        // I_n > 128 output columns run as column chunks that re-read the small source from L2
        const int64_t ldt = pad4(b.I);
        float* qt = ws.alloc_n<float>(ldt * In);
        if (ldt != b.I) fill_zero(ctx, qt, sizeof(float) * ldt * In);
        transpose_copy<float>(ctx, qf, b.I, In, In, qt, ldt);
        ttm_t_dispatch(ctx, ws, sf, b, qt, ldt, int(In), P, 1, b.a, b.a * In);
      } else {
        ttm_t<double, double, T>(ctx, src, b, Q[n], In, 1, int(In), P, 1, b.a, b.a * In);
      }
    } else {
      double* dst = ws.alloc_n<double>(b.a * In * b.b);
      ttm_t<double, double, double>(ctx, src, b, Q[n], In, 1, int(In), dst, 1, b.a, b.a * In);
      src = dst;
    }
    cur[n] = In;
  }
  const int64_t Il = X.d[N - 1];
  const int Rl = int(R[N - 1]);
  const T* QL;
  if (DT<T>::id == 1) {
    QL = reinterpret_cast<const T*>(Q[N - 1]);
  } else {
    T* c = ws.alloc_n<T>(Il * Rl);
    convert2d<double, T>(ctx, Q[N - 1], Il, Rl, Il, c, Il);
    QL = c;
  }
  int64_t J = 1;
  for (int k = 0; k < N - 1; ++k) J *= X.d[k];
  // the sums are taken of s X and s X^ (s a power of two from ||G||: rms(X) near 1), so fp32
  // squares of data at any scale stay in range; E is unchanged, E_gram rescales exactly
  resid_scale(ctx, gg, double(X.size()) * double(X.glob) / double(X.d[N - 1]), rs);
  bool done = false;
  if constexpr (std::is_same<T, float>::value) {
    // the fp16-split residual (R29) with P at the power-of-two scale rs[1] from ||G||
    done = residual_tc(ctx, ws, data, J, Il, P, J, Rl, QL, Il, sums, rs, ortho_q ? rs + 1 : nullptr);
  }
  if (!done) residual<T>(ctx, ws, data, J, Il, P, Rl, QL, Il, sums, rs);
  allreduce(comm, dist(), sums, 2, ctx.stream);                                    // C5
  ws.rewind(mk);
}

// ----------------------------------------------------------------- HOSVD (Alg.6)
template <typename T>
void Engine::hosvd(const TView& X, const int64_t* R, int q, int kind, const void* const* omega,
                   const int64_t* omega_cols, const int64_t* omega_ld, double* const* Q_out, double* G_out, double* E,
                   double* Eg) {
  const int N = X.N;
  const T* data = static_cast<const T*>(X.data);
  if constexpr (std::is_same<T, float>::value) {
    if (kind == 0 && ctx.overlap &&
        hosvd_overlap(X, data, R, q, omega, omega_cols, omega_ld, Q_out, G_out, E, Eg))
      return;
  }
  const auto mk = ws.mark();
  xs_slot = ws.alloc_n<float>(2);      // X's fp16 scale, taken once for all modes' power products
  xs_key = nullptr;
  int64_t K[5], ldq[5];
  double* Qt[5];
  for (int n = 0; n < N; ++n) {
    const void* const* om = omega + n * N;
    const int64_t* oc = omega_cols + n * N;
    const int64_t* ol = omega_ld + n * N;
    if (kind == 0 || kind == 3) K[n] = oc[n];
    else if (kind == 2) K[n] = oc[n == 0 ? 1 : 0];
    else { K[n] = 1; for (int k = 0; k < N; ++k) if (k != n) K[n] *= oc[k]; }
    const int64_t In = X.d[n];
    double* Yt = ws.alloc_n<double>(In * K[n]);
    sketch<T>(X, data, n, kind, om, oc, ol, q, Yt);
    Qt[n] = ws.alloc_n<double>(In * K[n]);
    ldq[n] = In;
    const bool last = (n == N - 1);
    qr_y(Yt, In, X.Ig(n), int(K[n]), In, Qt[n], In, nullptr, last && dist(), last ? X.off : 0);
  }
  int64_t gsz = 1;
  for (int n = 0; n < N; ++n) gsz *= K[n];
  double* Gt = ws.alloc_n<double>(gsz);
  core<T>(X, data, Qt, ldq, K, Gt);
  truncate(X, Gt, K, Qt, ldq, R, Q_out, G_out);
  if (E || Eg) rel_error<T>(X, data, G_out, R, Q_out, E, Eg, true);
  ws.rewind(mk);
  xs_slot = nullptr;
}

// -------------------------------------------------------------- STHOSVD (Alg.8)
// S = X for the first step; every shrunken S (and every B = S x_n Q~^T) is kept in fp64: they
// are at most R_1/I_1 of |X|, and an fp32 rounding of the intermediates would perturb the later
// modes' subspaces (and through them E) beyond the 1e-5 parity bar (tests/test_gpu_fullsize.py).
template <typename T>
void Engine::sthosvd(const TView& X, const int64_t* R, int q, int kind, const void* const* omega,
                     const int64_t* omega_cols, const int64_t* omega_ld, const int* order, double* const* Q_out,
                     double* G_out, double* E, double* Eg) {
  const int N = X.N;
  const auto mk = ws.mark();
  xs_slot = ws.alloc_n<float>(2);
  xs_key = nullptr;
  TView S = X;                         // working tensor S (reading R8: S = X)
  const double* sd = nullptr;          // fp64 S after the first shrink
  int64_t total = 1;
  for (int k = 0; k < N; ++k) total *= X.d[k];
  const int first = order ? order[0] : 0;
  const int64_t smax = total / X.d[first] * R[first];
  double* sbuf[2] = {ws.alloc_n<double>(smax), ws.alloc_n<double>(smax)};
  for (int step = 0; step < N; ++step) {
    const int n = order ? order[step] : step;
    const void* const* om = omega + n * N;
    const int64_t* oc = omega_cols + n * N;
    const int64_t* ol = omega_ld + n * N;
    int K;
    if (kind == 0 || kind == 3) K = int(oc[n]);
    else if (kind == 2) K = int(oc[n == 0 ? 1 : 0]);
    else { K = 1; for (int k = 0; k < N; ++k) if (k != n) K *= int(oc[k]); }
    const int64_t In = S.d[n];
    const auto mstep = ws.mark();
    // Alg.8 line 3 = Alg.1 lines 1-3 on S_(n): sketch (+ power iterations) and thin QR
    double* Yt = ws.alloc_n<double>(In * K);
    if (step == 0) {
      sketch<T>(S, static_cast<const T*>(X.data), n, kind, om, oc, ol, q, Yt);
    } else {
      // the test matrices are in the data type; the fp64 S needs fp64 copies (small: S has shrunk)
      const void* om64[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
      int64_t ld64[5] = {0, 0, 0, 0, 0};
      for (int k = 0; k < N; ++k) {
        if (kind == 3) { om64[k] = om[k]; ld64[k] = ol[k]; continue; }     // int32 codes: no conversion
        if (!om[k] || (kind == 0 && k != n) || (kind != 0 && k == n)) continue;
        const int64_t rows = (kind == 0) ? S.box(n).J() : S.d[k];
        if (DT<T>::id == 1) { om64[k] = om[k]; ld64[k] = ol[k]; continue; }
        // row-major rows x cols (pitch ld) == col-major cols x rows: convert, packed pitch = cols
        double* c = ws.alloc_n<double>(rows * oc[k]);
        convert2d<float, double>(ctx, static_cast<const float*>(om[k]), oc[k], rows, ol[k], c, oc[k]);
        om64[k] = c;
        ld64[k] = oc[k];
      }
      sketch<double>(S, sd, n, kind, om64, oc, ld64, q, Yt);
    }
    // slab-parallel: while the last mode is still a slab, S is local, the sketches
    // of modes n < N-1 and the Grams of B_(n) are partial sums (allreduced); the last mode comes last,
    // its sketch rows and factor rows stay local and B = S x_{N-1} Q~^T is allreduced
    const bool dist_last = dist() && n == N - 1 && S.sharded();
    const bool dist_slab = dist() && n != N - 1 && S.sharded();
    double* Qt = ws.alloc_n<double>(In * K);
    qr_y(Yt, In, S.Ig(n), K, In, Qt, In, nullptr, dist_last, dist_last ? S.off : 0);
    // Alg.1 line 4: B = S x_n Q~^T (fp64 accumulation and output)
    const Box bs = S.box(n);
    double* B = ws.alloc_n<double>(bs.a * K * bs.b);
    if (step == 0) ttm_t<T, double, double>(ctx, static_cast<const T*>(X.data), bs, Qt, 1, In, K, B, 1, bs.a, bs.a * K);
    else           ttm_t<double, double, double>(ctx, sd, bs, Qt, 1, In, K, B, 1, bs.a, bs.a * K);
    allreduce(comm, dist_last, B, bs.a * K * bs.b, ctx.stream);
    // Alg.1 lines 5-7 via the Gram-EVD of B_(n): U = top-R_n eigenvectors, Q_n = Q~ U
    const Box bb{bs.a, K, bs.b};
    double* M = ws.alloc_n<double>(int64_t(K) * K);
    double* V = ws.alloc_n<double>(int64_t(K) * K);
    double* W = ws.alloc_n<double>(K);
    gram_unfold(ctx, ws, B, bb, M);
    allreduce(comm, dist_slab, M, int64_t(K) * K, ctx.stream);
    eig_sym(ctx, ws, M, K, W, V);
    gemm_tall<double, double>(ctx, Qt, In, K, In, V, int(R[n]), K, Q_out[n], In);
    canon(Q_out[n], In, int(R[n]), In, dist_last ? S.off : 0, dist_last, V, K);
    // Alg.8 line 4 with the ΛV^T shortcut: S <- B x_n U^T
    double* Snew = (step == N - 1) ? G_out : sbuf[step & 1];
    ttm_t<double, double, double>(ctx, B, bb, V, 1, K, int(R[n]), Snew, 1, bb.a, bb.a * R[n]);
    sd = Snew;
    ws.rewind(mstep);
    S.d[n] = R[n];
    if (n == N - 1) { S.glob = R[n]; S.off = 0; }      // the last mode is now replicated
  }
  if (E || Eg) rel_error<T>(X, static_cast<const T*>(X.data), G_out, R, Q_out, E, Eg, true);
  ws.rewind(mk);
  xs_slot = nullptr;
}

// --------------------------------------------------------------- R-PET (Alg.9)
// Y_n = X_(n) Omega_n, Q^(n) = qr(Y_n) (lines 1-2); H = X x_1 Omega~_1 ... x_N Omega~_N (line 3, the
// core kernel chain with Omega~_n^T in place of Q~_n); S = H x_n (Omega~_n Q^(n))^+ (line 4) with
// A^+ = (A^T A)^{-1} A^T for the full-column-rank A = Omega~_n Q^(n) (S_n x K_n, S_n >= K_n; fp64,
// Cholesky of A^T A); truncation (line 5) and error as in hosvd (reading R1).  Every sketch of
// lines 1 and 3 reads only X.
template <typename T>
void Engine::pet(const TView& X, const int64_t* R, const void* const* omega, const int64_t* omega_cols,
                 const int64_t* omega_ld, const void* const* omega_tilde, const int64_t* S,
                 const int64_t* omega_tilde_ld, double* const* Q_out, double* G_out, double* E, double* Eg) {
  const int N = X.N;
  const T* data = static_cast<const T*>(X.data);
  const auto mk = ws.mark();
  int64_t K[5], ldq[5], ldw[5], Sp[5];
  double* Qt[5];
  double* Wt[5];
  for (int n = 0; n < N; ++n) {
    const void* const* om = omega + n * N;
    const int64_t* oc = omega_cols + n * N;
    const int64_t* ol = omega_ld + n * N;
    K[n] = oc[n];
    const int64_t In = X.d[n];
    const bool last = (n == N - 1);
    double* Yt = ws.alloc_n<double>(In * K[n]);
    sketch<T>(X, data, n, 0, om, oc, ol, 0, Yt);                                  // line 1 (C1)
    Qt[n] = ws.alloc_n<double>(In * K[n]);
    ldq[n] = In;
    qr_y(Yt, In, X.Ig(n), int(K[n]), In, Qt[n], In, nullptr, last && dist(), last ? X.off : 0);   // line 2
    // Omega~_n (S_n x I_n row-major, pitch ld) is Omega~_n^T as a col-major I_n x S_n matrix.
    // Sp_n = S_n rounded up to a multiple of 4 with zero rows: the core-sketch intermediates then
    // keep 16-byte rows (tensor-core TTM for the later stages); the zero slices of H meet zero
    // rows of A = Omega~_n Q^(n) in line 4, so S is unchanged.
    Sp[n] = pad4(S[n]);
    Wt[n] = ws.alloc_n<double>(In * Sp[n]);
    ldw[n] = In;
    if (Sp[n] != S[n]) fill_zero(ctx, Wt[n], sizeof(double) * In * Sp[n]);
    convert2d<T, double>(ctx, static_cast<const T*>(omega_tilde[n]), In, S[n], omega_tilde_ld[n], Wt[n], In);
  }
  int64_t hsz = 1;
  for (int n = 0; n < N; ++n) hsz *= Sp[n];
  double* H = ws.alloc_n<double>(hsz);
  {
    // line 3 (C4): H = X x_1 Omega~_1 ... x_N Omega~_N.  The first stage streams X (tensor cores
    // for fp32); the later stages accumulate in fp64 with fp64 intermediates: line 4 does not
    // project, so E is first-order sensitive to H (reading R26)
    const auto mh = ws.mark();
    int64_t cur[5];
    for (int k = 0; k < N; ++k) cur[k] = X.d[k];
    const Box b0 = TView::box_of(cur, N, 0);
    T* h1 = nullptr;
    double* h1d = nullptr;
    if (ctx.acc64()) {
      // strict mode: the X stage accumulates in fp64 and keeps its output in fp64 (no fp32 rounding of H)
      h1d = ws.alloc_n<double>(b0.a * Sp[0] * b0.b);
      ttm_t<T, double, double>(ctx, data, b0, Wt[0], 1, ldw[0], int(Sp[0]), h1d, 1, b0.a, b0.a * Sp[0]);
    } else {
      int64_t ld0;
      const T* w0 = working_copy<T>(ctx, ws, Wt[0], X.d[0], Sp[0], ldw[0], ld0);
      h1 = ws.alloc_n<T>(b0.a * Sp[0] * b0.b);
      ttm_t_dispatch(ctx, ws, data, b0, w0, ld0, int(Sp[0]), h1, 1, b0.a, b0.a * Sp[0], ctx.omega_tf32 != 0);
    }
    cur[0] = Sp[0];
    const double* src = h1d;
    for (int n = 1; n < N; ++n) {
      const Box b = TView::box_of(cur, N, n);
      double* dst = (n == N - 1) ? H : ws.alloc_n<double>(b.a * Sp[n] * b.b);
      LabelScope ls(ctx, "pet_hchain");
      if (n == 1 && h1) ttm_t<T, double, double>(ctx, h1, b, Wt[n], 1, ldw[n], int(Sp[n]), dst, 1, b.a, b.a * Sp[n]);
      else ttm_t<double, double, double>(ctx, src, b, Wt[n], 1, ldw[n], int(Sp[n]), dst, 1, b.a, b.a * Sp[n]);
      src = dst;
      cur[n] = Sp[n];
    }
    allreduce(comm, dist(), H, hsz, ctx.stream);
    ws.rewind(mh);
  }
  // line 4: S = H x_n (Omega~_n Q^(n))^+
  int64_t cur[5];
  for (int k = 0; k < N; ++k) cur[k] = Sp[k];
  const double* src = H;
  double* Sc = nullptr;
  for (int n = 0; n < N; ++n) {
    const int s = int(Sp[n]), k = int(K[n]);
    double* A = ws.alloc_n<double>(int64_t(s) * k);
    // A = Omega~_n Q^(n) = W^T Q: the col-major I_n x S_n matrix W viewed as the mode-1 box
    // [a = I_n, I = S_n, b = 1] of a sketch with B = Q (row j, column c at j + ldq c)
    ttm_s<double>(ctx, ws, Wt[n], Box{X.d[n], s, 1}, Qt[n], 1, ldq[n], k, A, s);
    allreduce(comm, n == N - 1 && dist(), A, int64_t(s) * k, ctx.stream);            // rows of the last mode
    double* G = ws.alloc_n<double>(int64_t(k) * k);
    double* Rc = ws.alloc_n<double>(int64_t(k) * k);
    double* Ri = ws.alloc_n<double>(int64_t(k) * k);
    double* RiT = ws.alloc_n<double>(int64_t(k) * k);
    double* T1 = ws.alloc_n<double>(int64_t(s) * k);
    double* M = ws.alloc_n<double>(int64_t(s) * k);
    gram<double>(ctx, ws, A, s, k, s, G);                                         // A^T A
    chol_inv(ctx, G, k, 0.0, Rc, Ri, nullptr);                                    // A^T A = Rc^T Rc
    gemm_tall<double, double>(ctx, A, s, k, s, Ri, k, k, T1, s);                  // A Rc^-1
    transpose_copy<double>(ctx, Ri, k, k, k, RiT, k);                             // Rc^-T (col-major)
    gemm_tall<double, double>(ctx, T1, s, k, s, RiT, k, k, M, s);                 // (A^+)^T = A (A^T A)^-1
    const Box b = TView::box_of(cur, N, n);
    double* dst = ws.alloc_n<double>(b.a * k * b.b);
    LabelScope ls(ctx, "pet_recover");
    ttm_t<double, double, double>(ctx, src, b, M, 1, s, k, dst, 1, b.a, b.a * k);
    src = dst;
    Sc = dst;
    cur[n] = k;
  }
  truncate(X, Sc, K, Qt, ldq, R, Q_out, G_out);                                   // line 5 (R1)
  if (E || Eg) rel_error<T>(X, data, G_out, R, Q_out, E, Eg, true);
  ws.rewind(mk);
}

// ------------------------------------------------------------- RP-HOOI (Alg.7)
// Reading R25: every stage accumulates in fp64 (CUDA cores) with fp64 intermediates and the fp64
// factors as stored.  W = S_(n) Omega^(n) has no oversampling, so span(W) is conditioned by
// kappa(W) ~ 1e1-1e2 and the fp32-accumulated tensor-core chain moved E by ~2e-5 on cfg2-small.
// The fp16 split of the X pass scales Q by 2^14 and needs |q| < 4 (R29): the launch is gated on the
// device by max|Q| < 2 as well as by X's scale (qgate), so a caller's wide start factor (Alg.7
// allows a random Gaussian one) sends the work to the 3xTF32 twin.
template <typename T>
void Engine::multi_ttm_skip(const TView& X, const T* data, const double* const* Q, const int64_t* ldq,
                            const int64_t* C, int skip, double* out) {
  const int N = X.N;
  const auto mk = ws.mark();
  int ps[5], np_ = 0;
  for (int p = 0; p < N; ++p) if (p != skip) ps[np_++] = p;
  int64_t cur[5];
  for (int k = 0; k < N; ++k) cur[k] = X.d[k];
  const double* src = nullptr;
  for (int i = 0; i < np_; ++i) {
    const int p = ps[i];
    const Box b = TView::box_of(cur, N, p);
    double* dst = (i == np_ - 1) ? out : ws.alloc_n<double>(b.a * C[p] * b.b);
    bool done = false;
    if constexpr (std::is_same<T, float>::value) {
      // the X pass on the tensor cores (fp32-accurate products, fp32 out), the rest of the chain in fp64
      if (i == 0 && ctx.hooi_tc && !ctx.simt() && C[p] <= 128) {
        const auto mq = ws.mark();
        int64_t ldt;
        const float* qt = working_copy<float>(ctx, ws, Q[p], cur[p], C[p], ldq[p], ldt);
        float* d32 = ws.alloc_n<float>(b.a * C[p] * b.b);
        const float* xsc = nullptr;
        if (ctx.tc_h16 && xs_slot) {
          float* xq = ws.alloc_n<float>(2);
          q_gate_scale(ctx, qt, cur[p], int(C[p]), ldt, x_scale(data, X.size(), X.size() / X.d[N - 1] * X.glob), xq);
          xsc = xq;
        }
        LabelScope ls(ctx, "hooi_first");
        if (ttm_t_tc(ctx, ws, data, b, qt, ldt, int(C[p]), d32, 1, b.a, b.a * C[p], 0, false, xsc)) {
          convert2d<float, double>(ctx, d32, b.a * C[p] * b.b, 1, b.a * C[p] * b.b, dst, b.a * C[p] * b.b);
          done = true;
        }
        ws.rewind(mq);
      }
    }
    if (done) {
    } else if (i == 0)
      ttm_t<T, double, double>(ctx, data, b, Q[p], 1, ldq[p], int(C[p]), dst, 1, b.a, b.a * C[p]);
    else
      ttm_t<double, double, double>(ctx, src, b, Q[p], 1, ldq[p], int(C[p]), dst, 1, b.a, b.a * C[p]);
    src = dst;
    cur[p] = C[p];
  }
  int64_t sz = 1;
  for (int k = 0; k < N; ++k) sz *= cur[k];
  allreduce(comm, dist() && skip != N - 1, out, sz, ctx.stream);            // last mode contracted: partial sums
  ws.rewind(mk);
}

// Alg.7: sweeps over n of  S = X x_{p!=n} Q^(p)T (latest factors),  W = S_(n) Omega^(n),
// Q^(n) = qr(W); then R5 signs and the core of the final factors (line 7) and E.
template <typename T>
void Engine::rp_hooi(const TView& X, const int64_t* R, int sweeps, const double* const* Q_init,
                     const double* const* omega, const int64_t* omega_ld, double* const* Q_out, double* G_out,
                     double* E, double* Eg) {
  const int N = X.N;
  const T* data = static_cast<const T*>(X.data);
  const auto mk = ws.mark();
  xs_slot = ws.alloc_n<float>(2);      // X's fp16 scale (one max|X| pass), shared by all S chains and the core
  xs_key = nullptr;
  int64_t ldq[5];
  for (int n = 0; n < N; ++n) {
    ldq[n] = X.d[n];
    if (Q_out[n] != Q_init[n])
      RT_CUDA(cudaMemcpyAsync(Q_out[n], Q_init[n], sizeof(double) * X.d[n] * R[n], cudaMemcpyDeviceToDevice,
                              ctx.stream));
  }
  for (int it = 0; it < sweeps; ++it) {
    for (int n = 0; n < N; ++n) {
      const auto ms = ws.mark();
      int64_t cur[5];
      for (int k = 0; k < N; ++k) cur[k] = (k == n) ? X.d[k] : R[k];
      int64_t sz = 1;
      for (int k = 0; k < N; ++k) sz *= cur[k];
      double* S = ws.alloc_n<double>(sz);
      multi_ttm_skip<T>(X, data, Q_out, ldq, R, n, S);                                   // line 4
      const int64_t In = X.d[n];
      double* W = ws.alloc_n<double>(In * R[n]);
      ttm_s<double>(ctx, ws, S, TView::box_of(cur, N, n), omega[it * N + n], omega_ld[it * N + n], 1, int(R[n]), W,
                    In);                                                                  // line 5
      const bool last = (n == N - 1);
      qr_y(W, In, X.Ig(n), int(R[n]), In, Q_out[n], In, nullptr, last && dist(), last ? X.off : 0);   // line 6
      ws.rewind(ms);
    }
  }
  for (int n = 0; n < N; ++n) {                                                         // reading R5
    double* U = ws.alloc_n<double>(R[n] * R[n]);
    canon(Q_out[n], X.d[n], int(R[n]), X.d[n], n == N - 1 ? X.off : 0, n == N - 1, U, int(R[n]));
  }
  core<T>(X, data, Q_out, ldq, R, G_out);                                                // line 7
  if (E || Eg) rel_error<T>(X, data, G_out, R, Q_out, E, Eg, true);
  ws.rewind(mk);
  xs_slot = nullptr;
}

template void Engine::rp_hooi<float>(const TView&, const int64_t*, int, const double* const*, const double* const*,
                                     const int64_t*, double* const*, double*, double*, double*);
template void Engine::rp_hooi<double>(const TView&, const int64_t*, int, const double* const*, const double* const*,
                                      const int64_t*, double* const*, double*, double*, double*);
template void Engine::pet<float>(const TView&, const int64_t*, const void* const*, const int64_t*, const int64_t*,
                                 const void* const*, const int64_t*, const int64_t*, double* const*, double*, double*,
                                 double*);
template void Engine::pet<double>(const TView&, const int64_t*, const void* const*, const int64_t*, const int64_t*,
                                  const void* const*, const int64_t*, const int64_t*, double* const*, double*, double*,
                                  double*);
template void Engine::sketch<float>(const TView&, const float*, int, int, const void* const*, const int64_t*,
                                    const int64_t*, int, double*, bool);
template void Engine::sketch<double>(const TView&, const double*, int, int, const void* const*, const int64_t*,
                                     const int64_t*, int, double*, bool);
template bool Engine::qr_z<float>(float*, int64_t, int64_t, int64_t, int, bool, int64_t, float*, int64_t, int,
                                  const float*);
template bool Engine::qr_z<double>(double*, int64_t, int64_t, int64_t, int, bool, int64_t, double*, int64_t, int,
                                   const float*);
template void Engine::qr_rows<float>(const float*, int64_t, int64_t, int, int64_t, double*, int64_t, double*,
                                     bool, int64_t, const double*, const int64_t*, int);
template void Engine::qr_rows<double>(const double*, int64_t, int64_t, int, int64_t, double*, int64_t, double*,
                                      bool, int64_t, const double*, const int64_t*, int);
template void Engine::core<float>(const TView&, const float*, const double* const*, const int64_t*,
                                  const int64_t*, double*, const float*);
template void Engine::core<double>(const TView&, const double*, const double* const*, const int64_t*,
                                   const int64_t*, double*, const double*);
template void Engine::rel_error<float>(const TView&, const float*, const double*, const int64_t*,
                                       const double* const*, double*, double*, bool);
template void Engine::rel_error<double>(const TView&, const double*, const double*, const int64_t*,
                                        const double* const*, double*, double*, bool);
template void Engine::hosvd<float>(const TView&, const int64_t*, int, int, const void* const*, const int64_t*,
                                   const int64_t*, double* const*, double*, double*, double*);
template void Engine::hosvd<double>(const TView&, const int64_t*, int, int, const void* const*, const int64_t*,
                                    const int64_t*, double* const*, double*, double*, double*);
template void Engine::sthosvd<float>(const TView&, const int64_t*, int, int, const void* const*, const int64_t*,
                                     const int64_t*, const int*, double* const*, double*, double*, double*);
template void Engine::sthosvd<double>(const TView&, const int64_t*, int, int, const void* const*,
                                      const int64_t*, const int64_t*, const int*, double* const*, double*, double*,
                                      double*);

}  // namespace rt
