// count_sketch.cu -- the count-sketch operator:
//
//   Y_n = X_(n) S,  S in {0, +-1}^{J_n x K}:  every column j of X_(n) is hashed to one of the K
//   groups (h_j, uniform), signed (s_j = +-1, Rademacher, footnote P:309) and summed into its
//   group's representative column:  Y[:, c] = sum_{j : h_j = c} s_j X_(n)[:, j].
//
// The caller draws h and s and passes them as one int32 code per column, v_j = s_j (h_j + 1)
// (include/rtucker.h).  No multiplications: the kernels stream X once (HBM-bound, 4 B/element
// for fp32) and add each element into a shared-memory accumulator acc[c][row] that the lane
// owning `row` updates alone, so there are no atomics on the hot path:
//
//  * a == 1 (mode 0):  X_(0) column j is contiguous, lanes own consecutive rows i; the code of
//    column j is uniform across the CTA.
//  * a > 1  (modes > 0): a warp loads a 32-row x 32U-column block with coalesced loads along
//    the columns (j = alpha + a beta, consecutive alpha contiguous), transposes it through a
//    32x33 shared tile so that each lane owns one row, and walks the 32 columns with the
//    column code broadcast by shuffle.
//
// fp32 accumulators hold at most ~512 terms (a CTA's column range is <= 512 K columns); the
// per-CTA partials are added into the fp64 Y with fp64 atomics (one per (row, group) per CTA).
#include <algorithm>
#include "kernels.h"

namespace rt {
namespace {

template <typename T> struct CsAcc { using type = float; };
template <> struct CsAcc<double> { using type = double; };

__device__ inline void cs_latch(int* st, int bit) {
  if (st) atomicOr(st, bit);
}

// code v -> (group c, sign); c = -1 for an out-of-range code (latched as an error)
__device__ inline int cs_decode(int32_t v, int K, float& s, int* status) {
  const int m = v < 0 ? -v : v;
  if (m < 1 || m > K) { cs_latch(status, kStatusBadHash); s = 0.f; return -1; }
  s = v < 0 ? -1.f : 1.f;
  return m - 1;
}

template <typename A>
__device__ inline void cs_flush(const A* acc, int K, int TI, int64_t i0, int64_t I, double* Y, int64_t ldy) {
  for (int e = threadIdx.x; e < K * TI; e += blockDim.x) {
    const int c = e / TI, r = e - c * TI;
    const int64_t i = i0 + r;
    const A v = acc[e];
    if (i < I && v != A(0)) atomicAdd(&Y[i + c * ldy], double(v));
  }
}

// ---------------------------------------------------------------- a == 1: X_(0) columns contiguous
template <typename T, int UNR>
__global__ void __launch_bounds__(256) cs_rows_kernel(const T* __restrict__ X, int64_t I, int64_t J,
                                                      const int32_t* __restrict__ code, int K, int64_t jchunk,
                                                      double* __restrict__ Y, int64_t ldy, int* status) {
  using A = typename CsAcc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* acc = reinterpret_cast<A*>(smem_raw);
  const int TI = blockDim.x;
  const int64_t i0 = int64_t(blockIdx.x) * TI;
  const int64_t row = i0 + threadIdx.x;
  const bool live = row < I;
  for (int e = threadIdx.x; e < K * TI; e += blockDim.x) acc[e] = A(0);
  __syncthreads();
  const int64_t j0 = int64_t(blockIdx.y) * jchunk;
  const int64_t j1 = j0 + jchunk < J ? j0 + jchunk : J;
  A* mine = acc + threadIdx.x;
  for (int64_t jb = j0; jb < j1; jb += UNR) {
    T x[UNR];
    int32_t v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t j = jb + u;
      v[u] = j < j1 ? __ldg(code + j) : 0;
      x[u] = (live && j < j1) ? __ldg(X + row + I * j) : T(0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (jb + u >= j1) break;
      float s;
      const int c = cs_decode(v[u], K, s, status);
      if (c >= 0) mine[c * TI] += s > 0 ? A(x[u]) : -A(x[u]);
    }
  }
  __syncthreads();
  cs_flush(acc, K, TI, i0, I, Y, ldy);
}

// ---------------------------------------------------------------- a > 1: transpose per warp
template <typename T, int U>
__global__ void __launch_bounds__(256) cs_mid_kernel(const T* __restrict__ X, int64_t a, int64_t I, int64_t J,
                                                     const int32_t* __restrict__ code, int K, int64_t jchunk,
                                                     double* __restrict__ Y, int64_t ldy, int* status) {
  using A = typename CsAcc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int W = blockDim.x >> 5, TI = blockDim.x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  A* acc = reinterpret_cast<A*>(smem_raw);                 // [K][TI]
  A* tile = acc + size_t(K) * TI + size_t(w) * 32 * 33;    // per-warp [32][33]
  (void)W;
  const int64_t i0 = int64_t(blockIdx.x) * TI;
  const int64_t rbase = i0 + 32 * w;                       // this warp's 32 rows
  for (int e = threadIdx.x; e < K * TI; e += blockDim.x) acc[e] = A(0);
  __syncthreads();
  const int64_t j0 = int64_t(blockIdx.y) * jchunk;
  const int64_t j1 = j0 + jchunk < J ? j0 + jchunk : J;
  const int64_t aI = a * I;
  A* mine = acc + 32 * w + lane;
  for (int64_t jb = j0; jb < j1; jb += 32 * U) {
    T x[U][32];
    int cidx[U];
    float sg[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = jb + 32 * u + lane;
      const bool jv = j < j1;
      cidx[u] = jv ? cs_decode(__ldg(code + j), K, sg[u], status) : -1;
      if (!jv) sg[u] = 0.f;
      const int64_t beta = jv ? j / a : 0;
      const int64_t off = jv ? (j - beta * a) + aI * beta : 0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int64_t i = rbase + r;
        x[u][r] = (jv && i < I) ? __ldg(X + off + a * i) : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const A s = A(sg[u]);
#pragma unroll
      for (int r = 0; r < 32; ++r) tile[r * 33 + lane] = s * A(x[u][r]);
      __syncwarp();
#pragma unroll 8
      for (int jj = 0; jj < 32; ++jj) {
        const int c = __shfl_sync(0xffffffffu, cidx[u], jj);
        if (c >= 0) mine[c * TI] += tile[lane * 33 + jj];
      }
      __syncwarp();
    }
  }
  __syncthreads();
  cs_flush(acc, K, TI, i0, I, Y, ldy);
}

// column range per CTA: <= 512 K columns (accumulator length bound), >= one block, and enough
// CTAs to give every SM two
int64_t pick_jchunk(int64_t J, int64_t gx, int K, int64_t blk, int sms) {
  int64_t jc = int64_t(512) * K;
  const int64_t want = int64_t(2) * sms;
  if (gx * cdiv(J, jc) < want) jc = cdiv(J, cdiv(want, gx));
  if (cdiv(J, jc) > 65535) jc = cdiv(J, 65535);
  jc = cdiv(jc, blk) * blk;
  return jc < blk ? blk : jc;
}

}  // namespace

template <typename T>
void count_sketch(const Ctx& ctx, const T* X, Box box, const int32_t* code, int K, double* Y, int64_t ldy) {
  using A = typename CsAcc<T>::type;
  const int64_t I = box.I, J = box.J();
  fill_zero(ctx, Y, sizeof(double) * size_t(ldy) * K);
  if (I == 0 || J == 0) return;
  int dev = 0, sms = 148, smem_max = 0;
  RT_CUDA(cudaGetDevice(&dev));
  RT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RT_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t budget = size_t(smem_max) - 1024;
  const bool mid = box.a > 1;
  // warps per CTA: up to 8, no more than the rows need, and the accumulator (+ tiles) must fit
  int W = int(std::min<int64_t>(8, cdiv(I, 32)));
  auto need = [&](int w) { return sizeof(A) * (size_t(K) * 32 * w + (mid ? size_t(w) * 32 * 33 : 0)); };
  while (W > 1 && need(W) > budget) --W;
  if (need(W) > budget) throw Error(kEUNSUPPORTED, "count sketch: K too large for the shared accumulator");
  const int TI = 32 * W;
  const int64_t gx = cdiv(I, TI);
  const size_t sm = need(W);
  if (!mid) {
    constexpr int UNR = 16;
    const int64_t jc = pick_jchunk(J, gx, K, UNR, sms);
    const dim3 grid(unsigned(gx), unsigned(cdiv(J, jc)));
    launch(ctx, "count_sketch", [&] {
      RT_CUDA(cudaFuncSetAttribute(cs_rows_kernel<T, UNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      cs_rows_kernel<T, UNR><<<grid, TI, sm, ctx.stream>>>(X, I, J, code, K, jc, Y, ldy, ctx.d_status);
    });
  } else {
    constexpr int U = std::is_same<T, double>::value ? 1 : 4;
    const int64_t jc = pick_jchunk(J, gx, K, 32 * U, sms);
    const dim3 grid(unsigned(gx), unsigned(cdiv(J, jc)));
    launch(ctx, "count_sketch", [&] {
      RT_CUDA(cudaFuncSetAttribute(cs_mid_kernel<T, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      cs_mid_kernel<T, U><<<grid, TI, sm, ctx.stream>>>(X, box.a, I, J, code, K, jc, Y, ldy, ctx.d_status);
    });
  }
}

template void count_sketch<float>(const Ctx&, const float*, Box, const int32_t*, int, double*, int64_t);
template void count_sketch<double>(const Ctx&, const double*, Box, const int32_t*, int, double*, int64_t);

}  // namespace rt
