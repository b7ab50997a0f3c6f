// ttm_simt.cu -- unfolding-free mode-n TTM kernels on CUDA cores (SIMT FFMA/DFMA).
//
// These are the portable baseline for the two TTM shapes of the hot path
// (SURVEY.md §2.2 N1); the tcgen05 tensor-core kernels (ttm_tc.cu) replace the
// X-streaming launches where they apply.
//
//   ttm_s:  Y(i,k) = sum_j X_(n)(i,j) B(j,k)      -- the sketch Y = X_(n) Omega
//           (Eq. proj; Alg.6 line 3 P:556), the power-iteration product
//           Y = X_(n) Z and Gram matrices of unfoldings.
//   ttm_t:  out(alpha,c,beta) = sum_i X(alpha,i,beta) M(i,c)
//           -- X x_n M^T (n-mode product P:109-112): Z = X_(n)^T Q, the core chain
//           (Eq. Core), Kronecker sketch stages, STHOSVD shrink (Alg.8).
//
// X is read in place through the [a, I, b] box of kernels.h; nothing is permuted.
#include <type_traits>
#include "kernels.h"

namespace rt {
namespace {

template <typename T> struct AccOf { using type = float; };
template <> struct AccOf<double> { using type = double; };
// ttm_t accumulates in fp64 as soon as any operand or the output is fp64 (fp32 x fp32 products
// are exact in fp64): the Kronecker chain and the STHOSVD shrink keep fp64 intermediates.
template <typename A, typename B, typename C> struct Acc3 {
  using type = typename std::conditional<std::is_same<A, double>::value || std::is_same<B, double>::value ||
                                             std::is_same<C, double>::value,
                                         double, float>::type;
};

// ------------------------------------------------------------------ ttm_s
// Block tile: BM = 128 rows i, BJ contraction columns j per stage, BN = 16*TN sketch cols.
// 256 threads = 16 (k) x 16 (i); thread owns i in {ty + 16 r}, k in {tx + 16 c}.
// A: accumulator (and partial) type -- T, or fp64 for fp32 data in the strict mode (ttm_impl 3).
template <typename T, int TN, bool GRAM, typename A = T>
__global__ void __launch_bounds__(256)
ttm_s_kernel(const T* __restrict__ X, int64_t a, int64_t I, const T* __restrict__ Bm, int64_t bs_j,
             int64_t bs_k, int K, int64_t J, int64_t jps, A* __restrict__ part) {
  constexpr int BM = 128;
  constexpr int BJ = sizeof(T) == 8 ? 16 : 32;
  constexpr int BN = 16 * TN;
  __shared__ T Xs[BJ][BM + 1];
  __shared__ T Bs[GRAM ? 1 : BJ][BN];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int64_t i0 = int64_t(blockIdx.x) * BM;
  const int k0 = blockIdx.y * BN;
  const int64_t jb = int64_t(blockIdx.z) * jps;
  const int64_t je = min(J, jb + jps);
  const int64_t aI = a * I;
  A acc[8][TN];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[r][c] = A(0);

  for (int64_t jc = jb; jc < je; jc += BJ) {
    if (a == 1) {                       // mode 0: X_(n)(i,j) = X[i + I*j], contiguous in i
      const int il = t & 127;
      const int64_t i = i0 + il;
#pragma unroll
      for (int s = 0; s < BJ / 2; ++s) {
        const int jl = (t >> 7) + 2 * s;
        const int64_t j = jc + jl;
        Xs[jl][il] = (i < I && j < je) ? X[i + I * j] : T(0);
      }
    } else {                            // contiguous in alpha (= j within an alpha run)
      const int jl = t % BJ;
      const int64_t j = jc + jl;
      const bool jv = j < je;
      const int64_t off = jv ? (j % a) + aI * (j / a) : 0;
#pragma unroll
      for (int s = 0; s < BM * BJ / 256; ++s) {
        const int il = t / BJ + (256 / BJ) * s;
        const int64_t i = i0 + il;
        Xs[jl][il] = (jv && i < I) ? X[off + a * i] : T(0);
      }
    }
    if (!GRAM) {
      if (bs_k == 1) {
        for (int e = t; e < BJ * BN; e += 256) {
          const int kl = e % BN, jl = e / BN;
          const int64_t j = jc + jl;
          const int k = k0 + kl;
          Bs[jl][kl] = (j < je && k < K) ? Bm[j * bs_j + k] : T(0);
        }
      } else {
        for (int e = t; e < BJ * BN; e += 256) {
          const int jl = e % BJ, kl = e / BJ;
          const int64_t j = jc + jl;
          const int k = k0 + kl;
          Bs[jl][kl] = (j < je && k < K) ? Bm[j * bs_j + int64_t(k) * bs_k] : T(0);
        }
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int jj = 0; jj < BJ; ++jj) {
      T xr[8], br[TN];
#pragma unroll
      for (int r = 0; r < 8; ++r) xr[r] = Xs[jj][ty + 16 * r];
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        if (GRAM) {
          const int k = k0 + tx + 16 * c;
          br[c] = k < BM ? Xs[jj][k] : T(0);
        } else {
          br[c] = Bs[jj][tx + 16 * c];
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[r][c] = fma(A(xr[r]), A(br[c]), acc[r][c]);
    }
    __syncthreads();
  }
  A* dst = part + int64_t(blockIdx.z) * K * I;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t i = i0 + ty + 16 * r;
    if (i >= I) continue;
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const int k = k0 + tx + 16 * c;
      if (k < K) dst[int64_t(k) * I + i] = acc[r][c];
    }
  }
}

// Y(i + ldy*k) = sum_z part[z][k][i]  in fp64, fixed order (deterministic split-K reduce)
template <typename T>
__global__ void splitk_reduce_kernel(const T* __restrict__ part, int64_t I, int K, int splits,
                                     double* __restrict__ Y, int64_t ldy) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= I * K) return;
  const int64_t i = e % I, k = e / I;
  double s = 0.0;
  for (int z = 0; z < splits; ++z) s += double(part[(int64_t(z) * K + k) * I + i]);
  Y[i + ldy * k] = s;
}

template <typename T, int TN, typename A = T>
void launch_ttm_s(const Ctx& ctx, Arena& ws, const T* X, Box box, const T* Bm, int64_t bs_j,
                  int64_t bs_k, int K, double* Y, int64_t ldy, bool gram) {
  constexpr int BJ = sizeof(T) == 8 ? 16 : 32;
  const int64_t J = box.J();
  const int64_t itiles = cdiv(box.I, 128);
  const int64_t ktiles = cdiv(K, 16 * TN);
  const int64_t tiles = itiles * ktiles;
  const int64_t target = 4LL * ctx.num_sms;
  int64_t splits = std::max<int64_t>(1, cdiv(target, tiles));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, cdiv(J, BJ * 8)));
  splits = std::min<int64_t>(splits, 65535);
  int64_t jps = cdiv(cdiv(J, splits), BJ) * BJ;
  splits = cdiv(J, jps);
  A* part = ws.alloc_n<A>(splits * K * box.I);
  const dim3 grid((unsigned)itiles, (unsigned)ktiles, (unsigned)splits);
  if (gram)
    launch(ctx, "ttm_s_gram_simt", [&] {
      ttm_s_kernel<T, TN, true, A><<<grid, 256, 0, ctx.stream>>>(X, box.a, box.I, Bm, bs_j, bs_k, K, J, jps, part);
    });
  else
    launch(ctx, "ttm_s_simt", [&] {
      ttm_s_kernel<T, TN, false, A><<<grid, 256, 0, ctx.stream>>>(X, box.a, box.I, Bm, bs_j, bs_k, K, J, jps, part);
    });
  const int64_t n = box.I * K;
  launch(ctx, "splitk_reduce", [&] {
    splitk_reduce_kernel<A><<<unsigned(cdiv(n, 256)), 256, 0, ctx.stream>>>(part, box.I, K, int(splits), Y, ldy);
  });
}

// ------------------------------------------------------------------ ttm_t
// Block tile: BM = 32 RJ outputs j, BI contraction rows per stage, BN = 8 TN output cols c.
// 256 threads = 32 (j, lanes) x 8 (c, warps); thread owns j in {tx + 32 r, r < RJ}, c in {ty + 8 cc}.
// The next stage's X and M elements are loaded into registers while the current stage is
// multiplied out of shared memory (global latency hidden behind the FMAs).
template <typename Tin, typename Tm, typename Tout, int TN, int RJ>
__global__ void __launch_bounds__(256)
ttm_t_kernel(const Tin* __restrict__ X, int64_t a, int64_t I, int64_t J, const Tm* __restrict__ Mm,
             int64_t ms_i, int64_t ms_c, int C, Tout* __restrict__ out, int64_t so_a, int64_t so_c,
             int64_t so_b) {
  using Tacc = typename Acc3<Tin, Tm, Tout>::type;
  constexpr int BM = 32 * RJ;
  constexpr int BI = sizeof(Tacc) == 8 ? 8 : 16;
  constexpr int BN = 8 * TN;
  constexpr int XL = BI * BM / 256;          // X elements per thread per stage
  constexpr int ML = (BI * BN + 255) / 256;  // M elements per thread per stage
  __shared__ Tacc Xs[BI][BM + 1];
  __shared__ Tacc Ms[BI][BN];
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  const int64_t j0 = int64_t(blockIdx.x) * BM;
  const int c0 = blockIdx.y * BN;
  const int64_t aI = a * I;
  Tacc acc[RJ][TN];
#pragma unroll
  for (int r = 0; r < RJ; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[r][c] = Tacc(0);

  // X loader.  a > 1: thread loads column jl = t % BM for rows il = t / BM + (256 / BM) s.
  // a == 1 (X(j, i) = X[i + I j], contiguous in i): il = t % BI, jl = t / BI + (256 / BI) s.
  const int jl_b = t % BM;
  const int64_t j_b = j0 + jl_b;
  const bool jv_b = j_b < J;
  const int64_t off_b = jv_b ? (j_b % a) + aI * (j_b / a) : 0;
  Tacc xv[XL], mv[ML];
  auto load = [&](int64_t ic) {
    if (a == 1) {
      const int il = t % BI;
      const int64_t i = ic + il;
#pragma unroll
      for (int s2 = 0; s2 < XL; ++s2) {
        const int64_t j = j0 + t / BI + (256 / BI) * s2;
        xv[s2] = (j < J && i < I) ? Tacc(X[i + I * j]) : Tacc(0);
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < XL; ++s2) {
        const int64_t i = ic + t / BM + (256 / BM) * s2;
        xv[s2] = (jv_b && i < I) ? Tacc(X[off_b + a * i]) : Tacc(0);
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < ML; ++s2) {
      const int e = t + 256 * s2;
      int il, cl;
      if (ms_c == 1) { cl = e % BN; il = e / BN; } else { il = e % BI; cl = e / BI; }
      const int64_t i = ic + il;
      const int c = c0 + cl;
      mv[s2] = (e < BI * BN && i < I && c < C) ? Tacc(Mm[i * ms_i + int64_t(c) * ms_c]) : Tacc(0);
    }
  };
  auto store = [&]() {
    if (a == 1) {
#pragma unroll
      for (int s2 = 0; s2 < XL; ++s2) Xs[t % BI][t / BI + (256 / BI) * s2] = xv[s2];
    } else {
#pragma unroll
      for (int s2 = 0; s2 < XL; ++s2) Xs[t / BM + (256 / BM) * s2][jl_b] = xv[s2];
    }
#pragma unroll
    for (int s2 = 0; s2 < ML; ++s2) {
      const int e = t + 256 * s2;
      if (e < BI * BN) {
        if (ms_c == 1) Ms[e / BN][e % BN] = mv[s2];
        else Ms[e % BI][e / BI] = mv[s2];
      }
    }
  };
  load(0);
  for (int64_t ic = 0; ic < I; ic += BI) {
    store();
    __syncthreads();
    if (ic + BI < I) load(ic + BI);
#pragma unroll
    for (int ii = 0; ii < BI; ++ii) {
      Tacc xr[RJ], mr[TN];
#pragma unroll
      for (int r = 0; r < RJ; ++r) xr[r] = Xs[ii][tx + 32 * r];
#pragma unroll
      for (int c = 0; c < TN; ++c) mr[c] = Ms[ii][ty + 8 * c];
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[r][c] = fma(xr[r], mr[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < RJ; ++r) {
    const int64_t j = j0 + tx + 32 * r;
    if (j >= J) continue;
    const int64_t ob = (j % a) * so_a + (j / a) * so_b;
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const int cc = c0 + ty + 8 * c;
      if (cc < C) out[ob + int64_t(cc) * so_c] = Tout(acc[r][c]);
    }
  }
}

template <typename Tin, typename Tm, typename Tout, int TN>
void launch_ttm_t(const Ctx& ctx, const Tin* X, Box box, const Tm* Mm, int64_t ms_i, int64_t ms_c, int C,
                  Tout* out, int64_t so_a, int64_t so_c, int64_t so_b) {
  const int64_t J = box.J();
  // 8 outputs j per thread when the accumulator tile stays small (TN <= 8), else 4
  constexpr int RJ = 4;
  const dim3 grid((unsigned)cdiv(J, 32 * RJ), (unsigned)cdiv(C, 8 * TN));
  RT_REQUIRE(grid.x < (1u << 31) && grid.y < 65536, kEUNSUPPORTED, "ttm_t grid too large");
  launch(ctx, ctx.label ? ctx.label : "ttm_t_simt", [&] {
    ttm_t_kernel<Tin, Tm, Tout, TN, RJ><<<grid, 256, 0, ctx.stream>>>(X, box.a, box.I, J, Mm, ms_i, ms_c, C,
                                                                      out, so_a, so_c, so_b);
  });
}

// ------------------------------------------------------------ ttm_t, fp64 accumulate on DMMA
// out(j, c) = sum_i X(j, i) M(i, c) with fp64 products and sums on the fp64 warp MMA
// (mma.sync m8n8k4 f64; tools/dmma_rate.cu: 37 TF/s vs 34 for DFMA, with 4x less operand traffic
// per FMA: the SIMT kernel is bound by shared-memory bandwidth at ~15 TF/s).  Block tile 128 j x
// 64 c, 32 (fp32 X) or 16 (fp64 X) contraction rows per stage, register-prefetched stages as above.  Warp w
// owns j in [32 (w % 4), +32) x c in [32 (w / 4), +32): 4 x 4 m8n8 tiles, 16 MMAs per k-step.
// Fragments (PTX m8n8k4 .f64): A[r][k] at lane 4 r + k; B[k][n] at lane 4 n + k; C[r][2 q + e] at
// lane 4 r + q.  fp64 pitches = 8 mod 16 doubles: the 4 k-rows of a fragment hit disjoint banks.
template <typename Tin, typename Tm, typename Tout, int NF>
__global__ void __launch_bounds__(256, 2)
ttm_t_dmma_kernel(const Tin* __restrict__ X, int64_t a, int64_t I, int64_t J, const Tm* __restrict__ Mm,
                  int64_t ms_i, int64_t ms_c, int C, Tout* __restrict__ out, int64_t so_a, int64_t so_c,
                  int64_t so_b) {
  // fp32 X is staged as fp32 (converted when a fragment is read): 32 contraction rows per stage,
  // pitch 132 floats (stores along i and the 4-row fragment reads are at most 2-way conflicted)
  using TX = typename std::conditional<std::is_same<Tin, float>::value, float, double>::type;
  constexpr int BM = 128, BN = 16 * NF, BI = sizeof(TX) == 4 ? 32 : 16;   // NF n-fragments per warp
  constexpr int PX = sizeof(TX) == 4 ? BM + 4 : BM + 8, PM = BN + 8;
  constexpr int XL = BI * BM / 256, ML = BI * BN / 256;
  __shared__ TX Xs[BI][PX];
  __shared__ double Ms[BI][PM];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t j0 = int64_t(blockIdx.x) * BM;
  const int c0 = blockIdx.y * BN;
  const int64_t aI = a * I;
  const int jw = 32 * (w & 3), cw = 8 * NF * (w >> 2);
  const int fr = lane >> 2, fk = lane & 3;
  double acc[4][NF][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < NF; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

  const int jl_b = t % BM;
  const int64_t j_b = j0 + jl_b;
  const bool jv_b = j_b < J;
  const int64_t off_b = jv_b ? (j_b % a) + aI * (j_b / a) : 0;
  TX xv[XL];
  double mv[ML];
  auto load = [&](int64_t ic) {
    if (a == 1) {
      const int il = t % BI;
      const int64_t i = ic + il;
#pragma unroll
      for (int s2 = 0; s2 < XL; ++s2) {
        const int64_t j = j0 + t / BI + (256 / BI) * s2;
        xv[s2] = (j < J && i < I) ? TX(X[i + I * j]) : TX(0);
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < XL; ++s2) {
        const int64_t i = ic + t / BM + (256 / BM) * s2;
        xv[s2] = (jv_b && i < I) ? TX(X[off_b + a * i]) : TX(0);
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < ML; ++s2) {
      const int e = t + 256 * s2;
      int il, cl;
      if (ms_c == 1) { cl = e % BN; il = e / BN; } else { il = e % BI; cl = e / BI; }
      const int64_t i = ic + il;
      const int c = c0 + cl;
      mv[s2] = (i < I && c < C) ? double(Mm[i * ms_i + int64_t(c) * ms_c]) : 0.0;
    }
  };
  auto store = [&]() {
    if (a == 1) {
#pragma unroll
      for (int s2 = 0; s2 < XL; ++s2) Xs[t % BI][t / BI + (256 / BI) * s2] = xv[s2];
    } else {
#pragma unroll
      for (int s2 = 0; s2 < XL; ++s2) Xs[t / BM + (256 / BM) * s2][jl_b] = xv[s2];
    }
#pragma unroll
    for (int s2 = 0; s2 < ML; ++s2) {
      const int e = t + 256 * s2;
      if (ms_c == 1) Ms[e / BN][e % BN] = mv[s2];
      else Ms[e % BI][e / BI] = mv[s2];
    }
  };
  load(0);
  for (int64_t ic = 0; ic < I; ic += BI) {
    store();
    __syncthreads();
    if (ic + BI < I) load(ic + BI);
#pragma unroll
    for (int kk = 0; kk < BI / 4; ++kk) {
      double af[4], bf[NF];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = double(Xs[4 * kk + fk][jw + 8 * m + fr]);
#pragma unroll
      for (int n = 0; n < NF; ++n) bf[n] = Ms[4 * kk + fk][cw + 8 * n + fr];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < NF; ++n)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
                       : "d"(af[m]), "d"(bf[n]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int64_t j = j0 + jw + 8 * m + fr;
    if (j >= J) continue;
    const int64_t ob = (j % a) * so_a + (j / a) * so_b;
#pragma unroll
    for (int n = 0; n < NF; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = c0 + cw + 8 * n + 2 * fk + e;
        if (c < C) out[ob + int64_t(c) * so_c] = Tout(acc[m][n][e]);
      }
  }
}

// cp.async form of the fp64 warp-MMA TTM: the stages go global -> shared memory without registers,
// NSTG deep (one barrier per stage), so the DMMA pipe is not idle while a stage is stored (the
// register-prefetch kernel above ran the pipe at 50%: its store phase and second barrier were
// serialized with the MMAs).  Same tile, fragments, fp64 products and sums (same results).
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename Tin, typename Tm, typename Tout, int NF, int NSTG, bool AT>
__global__ void __launch_bounds__(256, 2)
ttm_t_dmma_async_kernel(const Tin* __restrict__ X, int64_t a, int64_t I, int64_t J, const Tm* __restrict__ Mm,
                        int64_t ms_i, int64_t ms_c, int C, Tout* __restrict__ out, int64_t so_a, int64_t so_c,
                        int64_t so_b) {
  // pitches for conflict-free fragment reads (lane = 4 fr + fk reads row fk, column fr): 32-bit rows at
  // 8 mod 32 words, 64-bit rows at 4 mod 16 doubles (the 2-wavefront minimum)
  // AT (a == 1, i contiguous in X): the X tile is kept as [j][i] rows (pitch BI + 4 / BI + 2), so the
  // cp.async writes along i and the fragment reads (row j = fr, column i = fk) are conflict-free
  constexpr int BM = 128, BN = 16 * NF, BI = sizeof(Tin) == 4 ? 32 : 16;
  constexpr int PX = AT ? (sizeof(Tin) == 4 ? BI + 4 : BI + 2) : (sizeof(Tin) == 4 ? BM + 8 : BM + 4);
  constexpr int PM = BN + (sizeof(Tm) == 4 ? 8 : 4);
  constexpr int XS = (AT ? BM : BI) * PX, MS = BI * PM;           // elements per stage
  extern __shared__ __align__(16) unsigned char dsm[];
  Tin* Xs = reinterpret_cast<Tin*>(dsm);                         // [NSTG][BI][PX]
  Tm* Ms = reinterpret_cast<Tm*>(dsm + sizeof(Tin) * NSTG * XS);  // [NSTG][BI][PM]
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t j0 = int64_t(blockIdx.x) * BM;
  const int c0 = blockIdx.y * BN;
  const int64_t aI = a * I;
  const int jw = 32 * (w & 3), cw = 8 * NF * (w >> 2);
  const int fr = lane >> 2, fk = lane & 3;
  double acc[4][NF][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < NF; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  // a > 1: thread column jl = t % BM (rows il = t / BM + 2 s); a == 1: row il = t % BI, columns t / BI + k
  const int jl_b = t % BM;
  const int64_t j_b = j0 + jl_b;
  const bool jv_b = j_b < J;
  const int64_t off_b = jv_b ? (j_b % a) + aI * (j_b / a) : 0;
  auto issue = [&](int64_t ic, int slot) {
    Tin* xs = Xs + slot * XS;
    Tm* ms = Ms + slot * MS;
    if (a == 1) {
      const int il = t % BI;
      const int64_t i = ic + il;
#pragma unroll
      for (int s2 = 0; s2 < BI * BM / 256; ++s2) {
        const int jl = t / BI + (256 / BI) * s2;
        const int64_t j = j0 + jl;
        const bool v = j < J && i < I;
        const Tin* src = X + (v ? i + I * j : 0);
        Tin* dst = AT ? xs + jl * PX + il : xs + il * PX + jl;
        if (sizeof(Tin) == 4) cp_async4(dst, src, v); else cp_async8(dst, src, v);
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < BI * BM / 256; ++s2) {
        const int il = t / BM + (256 / BM) * s2;
        const int64_t i = ic + il;
        const bool v = jv_b && i < I;
        const Tin* src = X + (v ? off_b + a * i : 0);
        if (sizeof(Tin) == 4) cp_async4(xs + il * PX + jl_b, src, v); else cp_async8(xs + il * PX + jl_b, src, v);
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < BI * BN / 256; ++s2) {
      const int e = t + 256 * s2;
      int il, cl;
      if (ms_c == 1) { cl = e % BN; il = e / BN; } else { il = e % BI; cl = e / BI; }
      const int64_t i = ic + il;
      const int c = c0 + cl;
      const bool v = i < I && c < C;
      const Tm* src = Mm + (v ? i * ms_i + int64_t(c) * ms_c : 0);
      if (sizeof(Tm) == 4) cp_async4(ms + il * PM + cl, src, v); else cp_async8(ms + il * PM + cl, src, v);
    }
  };
  const int64_t nst = (I + BI - 1) / BI;
#pragma unroll
  for (int s0 = 0; s0 < NSTG - 1; ++s0) {
    if (s0 < nst) issue(int64_t(s0) * BI, s0);
    cp_async_commit();
  }
  for (int64_t st = 0; st < nst; ++st) {
    cp_async_wait<NSTG - 2>();
    __syncthreads();                                     // stage st landed; stage st - 1 consumed
    if (st + NSTG - 1 < nst) issue((st + NSTG - 1) * BI, int((st + NSTG - 1) % NSTG));
    cp_async_commit();
    const Tin* xs = Xs + int(st % NSTG) * XS;
    const Tm* ms = Ms + int(st % NSTG) * MS;
#pragma unroll
    for (int kk = 0; kk < BI / 4; ++kk) {
      double af[4], bf[NF];
#pragma unroll
      for (int m = 0; m < 4; ++m)
        af[m] = double(AT ? xs[(jw + 8 * m + fr) * PX + 4 * kk + fk] : xs[(4 * kk + fk) * PX + jw + 8 * m + fr]);
#pragma unroll
      for (int n = 0; n < NF; ++n) bf[n] = double(ms[(4 * kk + fk) * PM + cw + 8 * n + fr]);
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < NF; ++n)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
                       : "d"(af[m]), "d"(bf[n]));
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int64_t j = j0 + jw + 8 * m + fr;
    if (j >= J) continue;
    const int64_t ob = (j % a) * so_a + (j / a) * so_b;
#pragma unroll
    for (int n = 0; n < NF; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = c0 + cw + 8 * n + 2 * fk + e;
        if (c < C) out[ob + int64_t(c) * so_c] = Tout(acc[m][n][e]);
      }
  }
}

template <typename Tin, typename Tm, typename Tout>
void launch_ttm_t_dmma(const Ctx& ctx, const Tin* X, Box box, const Tm* Mm, int64_t ms_i, int64_t ms_c, int C,
                       Tout* out, int64_t so_a, int64_t so_c, int64_t so_b) {
  const int64_t J = box.J();
  // 16- / 32-column tiles for C <= 16 / 32 (the STHOSVD shrink at K = 27 used 27 of 64, the core
  // update S <- B x_n U^T at R = 16 used 16 of 32); the register-prefetch fallback has 32 / 64
  const bool async = !getenv("RT_DMMA_SYNC");
  const int bn = (C <= 16 && async) ? 16 : (C <= 32 ? 32 : 64);
  const dim3 grid((unsigned)cdiv(J, 128), (unsigned)cdiv(C, bn));
  RT_REQUIRE(grid.x < (1u << 31) && grid.y < 65536, kEUNSUPPORTED, "ttm_t grid too large");
  constexpr int NSTG = 3;
  const bool at = box.a == 1;
  auto smem_of = [at](int bnv) {
    const int BI = sizeof(Tin) == 4 ? 32 : 16;
    const int PX = at ? (sizeof(Tin) == 4 ? BI + 4 : BI + 2) : (sizeof(Tin) == 4 ? 136 : 132);
    const int PM = bnv + (sizeof(Tm) == 4 ? 8 : 4);
    return size_t(NSTG) * (sizeof(Tin) * size_t(at ? 128 : BI) * PX + sizeof(Tm) * BI * PM);
  };
  launch(ctx, ctx.label ? ctx.label : "ttm_t_dmma", [&] {
    if (async) {
      const size_t sm = smem_of(bn);
      auto go = [&](auto k) {
        RT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        k<<<grid, 256, sm, ctx.stream>>>(X, box.a, box.I, J, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
      };
      if (bn == 16 && at) go(ttm_t_dmma_async_kernel<Tin, Tm, Tout, 1, NSTG, true>);
      else if (bn == 16) go(ttm_t_dmma_async_kernel<Tin, Tm, Tout, 1, NSTG, false>);
      else if (bn == 32 && at) go(ttm_t_dmma_async_kernel<Tin, Tm, Tout, 2, NSTG, true>);
      else if (bn == 32) go(ttm_t_dmma_async_kernel<Tin, Tm, Tout, 2, NSTG, false>);
      else if (at) go(ttm_t_dmma_async_kernel<Tin, Tm, Tout, 4, NSTG, true>);
      else go(ttm_t_dmma_async_kernel<Tin, Tm, Tout, 4, NSTG, false>);
    } else if (bn == 32) {
      ttm_t_dmma_kernel<Tin, Tm, Tout, 2><<<grid, 256, 0, ctx.stream>>>(X, box.a, box.I, J, Mm, ms_i, ms_c, C, out,
                                                                         so_a, so_c, so_b);
    } else {
      ttm_t_dmma_kernel<Tin, Tm, Tout, 4><<<grid, 256, 0, ctx.stream>>>(X, box.a, box.I, J, Mm, ms_i, ms_c, C, out,
                                                                         so_a, so_c, so_b);
    }
  });
}

}  // namespace

template <typename T>
void ttm_s(const Ctx& ctx, Arena& ws, const T* X, Box box, const T* Bm, int64_t bs_j, int64_t bs_k,
           int K, double* Y, int64_t ldy, bool gram) {
  if (box.J() == 0 || box.I == 0 || K == 0) {
    for (int k = 0; k < K; ++k) RT_CUDA(cudaMemsetAsync(Y + ldy * k, 0, sizeof(double) * box.I, ctx.stream));
    return;
  }
  if (gram) RT_REQUIRE(box.I <= 128 && K == box.I, kEUNSUPPORTED, "gram mode needs I <= 128");
  if (std::is_same<T, float>::value && ctx.acc64()) {    // strict mode: fp64 products and sums
    if (K <= 32)       launch_ttm_s<T, 2, double>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
    else if (K <= 64)  launch_ttm_s<T, 4, double>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
    else               launch_ttm_s<T, 8, double>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
    return;
  }
  if (K <= 16)       launch_ttm_s<T, 1>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
  else if (K <= 32)  launch_ttm_s<T, 2>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
  else if (K <= 48)  launch_ttm_s<T, 3>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
  else if (K <= 64)  launch_ttm_s<T, 4>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
  else if (K <= 80)  launch_ttm_s<T, 5>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
  else if (K <= 96)  launch_ttm_s<T, 6>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
  else               launch_ttm_s<T, 8>(ctx, ws, X, box, Bm, bs_j, bs_k, K, Y, ldy, gram);
}

// ------------------------------------------------------------ ttm_t, narrow (C <= 8)
// The Kronecker sketch's chain (L_k = 2-4 columns) and other narrow contractions stream the source
// once with a handful of fp64 sums per output column j: a > 1: one thread per j (consecutive alpha:
// coalesced 4 / 8-byte loads per i, 8 loads in flight per thread); a == 1 (i contiguous): one warp
// per j, lanes over i, warp-shuffle sums.  M (I x C) is read through L1 (every thread reads the same
// row i).  fp64 products and sums in a fixed order.
namespace {
template <typename Tin, typename Tm, typename Tout, int C>
__global__ void __launch_bounds__(256) ttm_t_narrow_kernel(const Tin* __restrict__ X, int64_t a, int64_t I, int64_t J,
                                                           const Tm* __restrict__ Mm, int64_t ms_i, int64_t ms_c,
                                                           Tout* __restrict__ out, int64_t so_a, int64_t so_c,
                                                           int64_t so_b) {
  constexpr int TI = 256;                               // rows of M staged per round
  __shared__ double ms[TI][C];
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = j < J;
  const int64_t al = live ? j % a : 0, be = live ? j / a : 0;
  const Tin* x = X + al + a * I * be;
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  for (int64_t i0 = 0; i0 < I; i0 += TI) {
    const int ni = I - i0 < TI ? int(I - i0) : TI;
    __syncthreads();
    for (int e = threadIdx.x; e < ni * C; e += blockDim.x) {
      const int il = e / C, c = e - il * C;
      ms[il][c] = double(Mm[(i0 + il) * ms_i + c * ms_c]);
    }
    __syncthreads();
    if (!live) continue;
    int il = 0;
    for (; il + 8 <= ni; il += 8) {
      double xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = double(x[a * (i0 + il + u)]);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = fma(xv[u], ms[il + u][c], acc[c]);
    }
    for (; il < ni; ++il) {
      const double xv = double(x[a * (i0 + il)]);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = fma(xv, ms[il][c], acc[c]);
    }
  }
  if (!live) return;
#pragma unroll
  for (int c = 0; c < C; ++c) out[al * so_a + c * so_c + be * so_b] = Tout(acc[c]);
}
template <typename Tin, typename Tm, typename Tout, int C>
void launch_narrow(const Ctx& ctx, const Tin* X, Box box, const Tm* Mm, int64_t ms_i, int64_t ms_c, Tout* out,
                   int64_t so_a, int64_t so_c, int64_t so_b) {
  const int64_t J = box.J();
  launch(ctx, ctx.label ? ctx.label : "ttm_t_narrow", [&] {
    ttm_t_narrow_kernel<Tin, Tm, Tout, C><<<unsigned(cdiv(J, int64_t(256))), 256, 0, ctx.stream>>>(
        X, box.a, box.I, J, Mm, ms_i, ms_c, out, so_a, so_c, so_b);
  });
}
}  // namespace

template <typename Tin, typename Tm, typename Tout>
void ttm_t(const Ctx& ctx, const Tin* X, Box box, const Tm* Mm, int64_t ms_i, int64_t ms_c, int C,
           Tout* out, int64_t so_a, int64_t so_c, int64_t so_b) {
  if (box.J() == 0 || C == 0) return;
  if (box.I == 0) {
    throw Error(kEINVAL, "ttm_t with empty contraction");
  }
  if (C <= 4 && (box.a >= 32 || box.a == 1) && ctx.ttm_impl != 1 && cdiv(box.J(), int64_t(256)) < (int64_t(1) << 31)) {
    // narrow contraction (the Kronecker chain's L_k = 2-4 columns): one thread per output column j,
    // fp64 sums (the tiled kernel below wastes 5/8 of its 8-column tile here)
    switch (C) {
      case 1: launch_narrow<Tin, Tm, Tout, 1>(ctx, X, box, Mm, ms_i, ms_c, out, so_a, so_c, so_b); return;
      case 2: launch_narrow<Tin, Tm, Tout, 2>(ctx, X, box, Mm, ms_i, ms_c, out, so_a, so_c, so_b); return;
      case 3: launch_narrow<Tin, Tm, Tout, 3>(ctx, X, box, Mm, ms_i, ms_c, out, so_a, so_c, so_b); return;
      default: launch_narrow<Tin, Tm, Tout, 4>(ctx, X, box, Mm, ms_i, ms_c, out, so_a, so_c, so_b); return;
    }
  }
  using Tacc = typename Acc3<Tin, Tm, Tout>::type;
  if ((std::is_same<Tacc, double>::value && C > 8 && ctx.ttm_impl != 1) || ctx.acc64()) {
    // fp64 accumulation: the fp64 warp MMA (fewer shared-memory operand reads per FMA)
    launch_ttm_t_dmma<Tin, Tm, Tout>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
    return;
  }
  if (C <= 8)        launch_ttm_t<Tin, Tm, Tout, 1>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
  else if (C <= 16)  launch_ttm_t<Tin, Tm, Tout, 2>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
  else if (C <= 32)  launch_ttm_t<Tin, Tm, Tout, 4>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
  else if (C <= 48)  launch_ttm_t<Tin, Tm, Tout, 6>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
  else if (C <= 64)  launch_ttm_t<Tin, Tm, Tout, 8>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
  else if (C <= 80)  launch_ttm_t<Tin, Tm, Tout, 10>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
  else if (C <= 96)  launch_ttm_t<Tin, Tm, Tout, 12>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
  else               launch_ttm_t<Tin, Tm, Tout, 16>(ctx, X, box, Mm, ms_i, ms_c, C, out, so_a, so_c, so_b);
}

// ------------------------------------------------------------- Khatri-Rao TTV
// out[alpha + a beta] = sum_i W[alpha + a i + a I beta] Om[i ld + c], the KR column c read from the
// alpha (c_in_a) or beta index: c = (alpha / c_stride) % K  or  (beta / c_stride) % K.  fp64 sums.
namespace {
template <typename Tw, typename To>
__global__ void kr_ttv_kernel(const Tw* __restrict__ W, int64_t a, int64_t I, int64_t b, const To* __restrict__ Om,
                              int64_t ld, int K, bool c_in_a, int64_t c_stride, double* __restrict__ out) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= a * b) return;
  const int64_t al = e % a, be = e / a;
  const int c = int(((c_in_a ? al : be) / c_stride) % K);
  const Tw* w = W + al + a * I * be;
  double s = 0.0;
  for (int64_t i = 0; i < I; ++i) s = fma(double(w[a * i]), double(Om[i * ld + c]), s);
  out[e] = s;
}

}  // namespace

template <typename Tw, typename To>
void kr_ttv(const Ctx& ctx, const Tw* W, Box box, const To* Om, int64_t ld, int K, bool c_in_a, int64_t c_stride,
            double* out) {
  const int64_t n = box.a * box.b;
  if (n == 0) return;
  launch(ctx, "kr_ttv", [&] {
    kr_ttv_kernel<Tw, To><<<unsigned(cdiv(n, 256)), 256, 0, ctx.stream>>>(W, box.a, box.I, box.b, Om, ld, K, c_in_a,
                                                                          c_stride, out);
  });
}
template void kr_ttv<float, float>(const Ctx&, const float*, Box, const float*, int64_t, int, bool, int64_t, double*);
template void kr_ttv<double, float>(const Ctx&, const double*, Box, const float*, int64_t, int, bool, int64_t, double*);
template void kr_ttv<double, double>(const Ctx&, const double*, Box, const double*, int64_t, int, bool, int64_t,
                                     double*);

template void ttm_s<float>(const Ctx&, Arena&, const float*, Box, const float*, int64_t, int64_t, int,
                           double*, int64_t, bool);
template void ttm_s<double>(const Ctx&, Arena&, const double*, Box, const double*, int64_t, int64_t, int,
                            double*, int64_t, bool);
template void ttm_t<float, float, float>(const Ctx&, const float*, Box, const float*, int64_t, int64_t, int,
                                         float*, int64_t, int64_t, int64_t);
template void ttm_t<float, float, double>(const Ctx&, const float*, Box, const float*, int64_t, int64_t, int,
                                          double*, int64_t, int64_t, int64_t);
template void ttm_t<double, double, double>(const Ctx&, const double*, Box, const double*, int64_t, int64_t,
                                            int, double*, int64_t, int64_t, int64_t);
template void ttm_t<float, double, double>(const Ctx&, const float*, Box, const double*, int64_t, int64_t, int,
                                           double*, int64_t, int64_t, int64_t);
template void ttm_t<double, float, double>(const Ctx&, const double*, Box, const float*, int64_t, int64_t, int,
                                           double*, int64_t, int64_t, int64_t);
template void ttm_t<double, double, float>(const Ctx&, const double*, Box, const double*, int64_t, int64_t,
                                           int, float*, int64_t, int64_t, int64_t);

}  // namespace rt
