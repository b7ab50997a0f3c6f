// engine.h -- orchestration of the hot path on one rank.
#pragma once

#include <vector>

#include "comm.h"
#include "kernels.h"

namespace rt {

// Local view of a (possibly slab-sharded) first-mode-fastest tensor.
struct TView {
  int dtype = 0;                 // 0 f32, 1 f64
  int N = 0;
  int64_t d[5] = {0, 0, 0, 0, 0};  // local dims
  int64_t off = 0, glob = 0;     // last-mode slab [off, off + d[N-1]) of glob
  const void* data = nullptr;

  bool sharded() const { return off != 0 || glob != d[N - 1]; }
  int64_t size() const { int64_t s = 1; for (int k = 0; k < N; ++k) s *= d[k]; return s; }
  int64_t Ig(int n) const { return n == N - 1 ? glob : d[n]; }
  int64_t Jg(int n) const { int64_t s = 1; for (int k = 0; k < N; ++k) if (k != n) s *= Ig(k); return s; }
  Box box(int n) const { return box_of(d, N, n); }
  static Box box_of(const int64_t* dims, int N, int n) {
    Box b{1, dims[n], 1};
    for (int k = 0; k < n; ++k) b.a *= dims[k];
    for (int k = n + 1; k < N; ++k) b.b *= dims[k];
    return b;
  }
};

class Engine {
 public:
  Engine(Ctx& c, Arena& w, Comm* cm) : ctx(c), ws(w), comm(cm) {}
  Ctx& ctx;
  Arena& ws;
  Comm* comm;
  // truncate(): recorded on the engine's stream just before the Jacobi launch when set (a driver that runs
  // a persistent kernel beside it waits for this, so that the two-CTA clusters get their SMs first)
  cudaEvent_t pre_eig_event = nullptr;
  bool dist() const { return comm && (comm->nranks() > 1 || ctx.force_dist); }
  // fp16-split power products: the scale s of X (x_scale_h16) in a slot owned by the driver that
  // outlives the per-mode sketches, computed once per tensor (xs_key = the data it was taken of)
  float* xs_slot = nullptr;
  const void* xs_key = nullptr;
  const float* x_scale(const float* data, int64_t n, int64_t n_glob = 0);
  void finish_scale(const unsigned int* stat, int64_t n_local, int64_t n_glob);

  // (1) sketch of mode n incl. q power iterations; Yt: fp64 I_n(local) x K, ld I_n(local).
  template <typename T>
  void sketch(const TView& X, const T* data, int n, int kind, const void* const* omega,
              const int64_t* omega_cols, const int64_t* omega_ld, int q, double* Yt, bool first_only = false);
  // one power step of reading R31 (fp32 data, tensor cores): Yt = X_(n) s_z X_(n)^T Qy; false if n/a.
  // unmixed: Qy already went through unmix_q (the overlapped driver does it on the side stream)
  // parts: 1 = the Z pass only, 2 = the product only (Z from an earlier parts = 1 call in pb), 3 = both;
  // pb (required unless parts == 3): the Z buffers, allocated on first use from ws and left allocated
  struct PowerBufs { float* Z = nullptr; float* Z2 = nullptr; };
  bool power_step_r31(const TView& X, const float* data, int n, int K, const double* Qy, double* Yt,
                      bool unmixed = false, PowerBufs* pb = nullptr, int parts = 3);
  // reading R31': Qp = Qy R_S^-1 D (ws allocation, In x K, ld In) with R_S the Cholesky factor of the
  // Gram of a row sample of Z = X_(n)^T Qy, so that Z' = X_(n)^T Qp has near-orthogonal columns
  double* unmix_q(const TView& X, const float* data, int n, int K, const double* Qy, double* out = nullptr);
  // HOSVD (Gaussian Omega) with the thin QRs on the handle's side stream; false (nothing launched) if n/a
  bool hosvd_overlap(const TView& X, const float* data, const int64_t* R, int q, const void* const* omega,
                     const int64_t* omega_cols, const int64_t* omega_ld, double* const* Q_out, double* G_out,
                     double* E, double* Eg);
  // (2) thin QR of the fp64 Y side (shifted CholeskyQR3); R nullable.
  void qr_y(const double* Y, int64_t m, int64_t m_glob, int k, int64_t ldy, double* Q, int64_t ldq,
            double* R, bool rows_dist, int64_t row0, int passes = 3);
  template <typename T>
  void qr_rows(const T* Y, int64_t m, int64_t m_glob, int k, int64_t ldy, double* Q, int64_t ldq, double* R,
               bool rows_dist, int64_t row0, const double* shift_dev = nullptr, const int64_t* row0_dev = nullptr,
               int passes = 3);
  // orthonormalize the tall Z of the power iteration in place (shifted CholeskyQR, fp64 Gram)
  template <typename T>
  bool qr_z(T* Z, int64_t m, int64_t ldz, int64_t m_glob, int k, bool rows_dist, int64_t row0, T* Z2 = nullptr,
            int64_t ldz2 = 0, int split = 1, const float* xsc = nullptr);
  // (3) core G~ = X x_n Qt_n^T (all n) -> fp64 Gt (replicated)
  template <typename T>
  void core(const TView& X, const T* data, const double* const* Qt, const int64_t* ldq, const int64_t* K,
            double* Gt, const T* stage0 = nullptr);
  // (a6) truncation of the oversampled core: Q_out, G_out from Gt, Qt
  void truncate(const TView& X, const double* Gt, const int64_t* K, const double* const* Qt,
                const int64_t* ldq, const int64_t* R, double* const* Q_out, double* G_out);
  // (a8) residual pass: E and E_gram from X, G (R_1..R_N), Q (I_n(local) x R_n, ld I_n(local))
  template <typename T>
  void rel_error(const TView& X, const T* data, const double* G, const int64_t* R, const double* const* Q,
                 double* E, double* Eg, bool ortho_q = false);
  // the residual sums of rel_error without the finalization (sums[2], gg = ||G||^2, rs[2] the scales)
  template <typename T>
  void resid_sums(const TView& X, const T* data, const double* G, const int64_t* R, const double* const* Q,
                  double* sums, double* gg, float* rs, bool ortho_q);
  // drivers
  template <typename T>
  void hosvd(const TView& X, const int64_t* R, int q, int kind, const void* const* omega,
             const int64_t* omega_cols, const int64_t* omega_ld, double* const* Q_out, double* G_out, double* E,
             double* Eg);
  template <typename T>
  void sthosvd(const TView& X, const int64_t* R, int q, int kind, const void* const* omega,
               const int64_t* omega_cols, const int64_t* omega_ld, const int* order, double* const* Q_out,
               double* G_out, double* E, double* Eg);
  template <typename T>
  void pet(const TView& X, const int64_t* R, const void* const* omega, const int64_t* omega_cols,
           const int64_t* omega_ld, const void* const* omega_tilde, const int64_t* S, const int64_t* omega_tilde_ld,
           double* const* Q_out, double* G_out, double* E, double* Eg);
  template <typename T>
  void rp_hooi(const TView& X, const int64_t* R, int sweeps, const double* const* Q_init, const double* const* omega,
               const int64_t* omega_ld, double* const* Q_out, double* G_out, double* E, double* Eg);
  // X x_{p != skip} Q_p^T in ascending mode order -> fp64 tensor (R_p for p != skip, X.d[skip] at skip);
  // slab partial sums are allreduced when the last mode is contracted
  template <typename T>
  void multi_ttm_skip(const TView& X, const T* data, const double* const* Q, const int64_t* ldq, const int64_t* C,
                      int skip, double* out);

 private:
  void canon(double* Qn, int64_t m, int r, int64_t ld, int64_t row0, bool dist_rows, double* U, int ku);
};

}  // namespace rt
