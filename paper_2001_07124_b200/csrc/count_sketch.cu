// count_sketch.cu -- the count-sketch operator:
//
//   Y_n = X_(n) S,  S in {0, +-1}^{J_n x K}:  every column j of X_(n) is hashed to one of the K
//   groups (h_j, uniform), signed (s_j = +-1, Rademacher, footnote P:309) and summed into its
//   group's representative column:  Y[:, c] = sum_{j : h_j = c} s_j X_(n)[:, j].
//
// The caller draws h and s and passes them as one int32 code per column, v_j = s_j (h_j + 1)
// (include/rtucker.h).  A prep kernel turns the codes into (a) the byte offset of the group's
// accumulator row, c * TI * sizeof(acc), with bit 0 of every aligned quad's first word flagging
// a quad whose 4 groups are not pairwise distinct, and (b) the sign as +-1.0f.  The kernels
// stream X once (HBM-bound, 4 B/element for fp32) and add each element into a shared-memory
// accumulator acc[c][row] that the lane owning `row` updates alone -- no atomics on the hot path.
// A quad with distinct groups is applied as 4 loads, 4 FMAs (x * s + acc, exact sign), 4 stores:
// 4 independent read-modify-writes hide the shared-memory latency; a flagged quad is applied
// sequentially (warp-uniform branch: the codes are the same for every row).
//
//  * a == 1 (mode 0): X_(0) column j is contiguous; lanes own consecutive rows and load their
//    elements directly (coalesced).
//  * a > 1, fp32, a % 4 == 0 (modes > 0, the bench shapes): TMA pipeline -- a producer warp
//    loads [TI rows][32 alpha] boxes (128 B swizzle) into a ring of stages together with the
//    stage's words; lane = row consumers read their row with conflict-free 16-byte loads.
//  * other a > 1 cases (fp64, a % 4 != 0): a warp loads a 32-row x 32U-column block along the
//    columns and transposes it through a 32x33 shared tile.
//
// fp32 accumulators hold at most ~512 terms (a CTA's column range is <= 512 K columns); the
// each CTA writes its partials to its own slice, and a reduce kernel adds the slices into the fp64 Y
// in a fixed order: bitwise reproducible run to run for float data too.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include "kernels.h"
#include "tc_common.cuh"

namespace rt {
namespace {

template <typename T> struct CsAcc { using type = float; };
template <> struct CsAcc<double> { using type = double; };

// one thread per aligned quad of columns: decode (group, sign); padding and invalid codes go to
// the trash row K (invalid ones are latched); dup flag in bit 0 of the quad's first offset
__global__ void cs_prep_kernel(const int32_t* __restrict__ code, int64_t J, int64_t Jpad, int K, int row_bytes,
                               uint32_t* __restrict__ off, float* __restrict__ sgn, int* status) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (4 * q >= Jpad) return;
  int c[4];
  float s[4];
  for (int k = 0; k < 4; ++k) {
    const int64_t j = 4 * q + k;
    c[k] = K;
    s[k] = 0.f;
    if (j < J) {
      const int32_t v = code[j];
      const int m = v < 0 ? -v : v;
      if (m >= 1 && m <= K) { c[k] = m - 1; s[k] = v < 0 ? -1.f : 1.f; }
      else if (status) atomicOr(status, kStatusBadHash);
    }
  }
  const bool dup = c[0] == c[1] || c[0] == c[2] || c[0] == c[3] || c[1] == c[2] || c[1] == c[3] || c[2] == c[3];
  for (int k = 0; k < 4; ++k) {
    off[4 * q + k] = uint32_t(c[k]) * uint32_t(row_bytes) | ((k == 0 && dup) ? 1u : 0u);
    sgn[4 * q + k] = s[k];
  }
}

// acc[c_k][row] += s_k x_k for one quad; rowb = this lane's row in acc (bytes)
template <typename A>
__device__ __forceinline__ void cs_quad(unsigned char* rowb, int4 o, float4 s, A x0, A x1, A x2, A x3) {
  A* p0 = reinterpret_cast<A*>(rowb + (uint32_t(o.x) & ~1u));
  A* p1 = reinterpret_cast<A*>(rowb + o.y);
  A* p2 = reinterpret_cast<A*>(rowb + o.z);
  A* p3 = reinterpret_cast<A*>(rowb + o.w);
  if (!(o.x & 1)) {                // distinct rows: loads first, then stores
    const A a0 = *p0, a1 = *p1, a2 = *p2, a3 = *p3;
    *p0 = fma(A(s.x), x0, a0); *p1 = fma(A(s.y), x1, a1); *p2 = fma(A(s.z), x2, a2); *p3 = fma(A(s.w), x3, a3);
  } else {
    *p0 = fma(A(s.x), x0, *p0); *p1 = fma(A(s.y), x1, *p1); *p2 = fma(A(s.z), x2, *p2); *p3 = fma(A(s.w), x3, *p3);
  }
}

// the CTA's partial sums go to its own slice part[blockIdx.y][c][i] (no atomics): cs_reduce adds
// the slices in blockIdx.y order, so the result is bitwise reproducible for any data
template <typename A>
__device__ inline void cs_flush(const A* acc, int K, int TI, int64_t i0, int64_t I, A* part) {
  part += size_t(blockIdx.y) * K * I;
  for (int e = threadIdx.x; e < K * TI; e += blockDim.x) {
    const int c = e / TI, r = e - c * TI;
    const int64_t i = i0 + r;
    if (i < I) part[i + c * I] = acc[e];
  }
}

// Y[i, c] = sum_y part[y][c][i] in fp64, y ascending
template <typename A>
__global__ void cs_reduce_kernel(const A* __restrict__ part, int64_t ny, int64_t KI, int64_t I,
                                 double* __restrict__ Y, int64_t ldy) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= KI) return;
  double s = 0.0;
  for (int64_t y = 0; y < ny; ++y) s += double(part[e + y * KI]);
  const int64_t c = e / I, i = e - c * I;
  Y[i + c * ldy] = s;
}

// ---------------------------------------------------------------- a == 1: X_(0) columns contiguous
template <typename T>
__global__ void __launch_bounds__(256) cs_rows_kernel(const T* __restrict__ X, int64_t I, int64_t J, int64_t Jpad,
                                                      const uint32_t* __restrict__ off,
                                                      const float* __restrict__ sgn, int K, int64_t jchunk,
                                                      typename CsAcc<T>::type* __restrict__ part) {
  using A = typename CsAcc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* acc = reinterpret_cast<A*>(smem_raw);                  // [K + 1][TI], row K = trash
  const int TI = blockDim.x;
  const int64_t i0 = int64_t(blockIdx.x) * TI;
  const int64_t row = i0 + threadIdx.x;
  const bool live = row < I;
  for (int e = threadIdx.x; e < (K + 1) * TI; e += blockDim.x) acc[e] = A(0);
  __syncthreads();
  const int64_t j0 = int64_t(blockIdx.y) * jchunk;
  const int64_t j1 = j0 + jchunk < Jpad ? j0 + jchunk : Jpad;
  unsigned char* rowb = smem_raw + threadIdx.x * sizeof(A);
  const T* xr = X + row;
  for (int64_t jb = j0; jb < j1; jb += 32) {
    T x[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) x[u] = (live && jb + u < J) ? __ldg(xr + I * (jb + u)) : T(0);
    const int4* oq = reinterpret_cast<const int4*>(off + jb);
    const float4* sq = reinterpret_cast<const float4*>(sgn + jb);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      cs_quad<A>(rowb, __ldg(oq + q), __ldg(sq + q), A(x[4 * q]), A(x[4 * q + 1]), A(x[4 * q + 2]), A(x[4 * q + 3]));
  }
  __syncthreads();
  cs_flush(acc, K, TI, i0, I, part);
}

// ---------------------------------------------------------------- a > 1: transpose per warp
template <typename T, int U>
__global__ void __launch_bounds__(256) cs_mid_kernel(const T* __restrict__ X, int64_t a, int64_t I, int64_t J,
                                                     int64_t Jpad, const uint32_t* __restrict__ off,
                                                     const float* __restrict__ sgn, int K, int64_t jchunk,
                                                     typename CsAcc<T>::type* __restrict__ part) {
  using A = typename CsAcc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int TI = blockDim.x;
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  A* acc = reinterpret_cast<A*>(smem_raw);                   // [K + 1][TI]
  A* tile = acc + size_t(K + 1) * TI + size_t(wp) * 32 * 33;  // per-warp [32][33]
  const int64_t i0 = int64_t(blockIdx.x) * TI;
  const int64_t rbase = i0 + 32 * wp;                         // this warp's 32 rows
  for (int e = threadIdx.x; e < (K + 1) * TI; e += blockDim.x) acc[e] = A(0);
  __syncthreads();
  const int64_t j0 = int64_t(blockIdx.y) * jchunk;
  const int64_t j1 = j0 + jchunk < Jpad ? j0 + jchunk : Jpad;
  const int64_t aI = a * I;
  unsigned char* rowb = smem_raw + (32 * wp + lane) * sizeof(A);
  for (int64_t jb = j0; jb < j1; jb += 32 * U) {
    T x[U][32];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = jb + 32 * u + lane;
      const bool jv = j < J;
      const int64_t beta = jv ? j / a : 0;
      const int64_t o = jv ? (j - beta * a) + aI * beta : 0;
      const T* xp = X + o + a * rbase;
#pragma unroll
      for (int r = 0; r < 32; ++r) x[u][r] = (jv && rbase + r < I) ? __ldg(xp + a * r) : T(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (jb + 32 * u >= j1) break;                             // uniform
#pragma unroll
      for (int r = 0; r < 32; ++r) tile[r * 33 + lane] = A(x[u][r]);
      __syncwarp();
      const int4* oq = reinterpret_cast<const int4*>(off + jb + 32 * u);
      const float4* sq = reinterpret_cast<const float4*>(sgn + jb + 32 * u);
      const A* tr = tile + lane * 33;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        cs_quad<A>(rowb, __ldg(oq + q), __ldg(sq + q), tr[4 * q], tr[4 * q + 1], tr[4 * q + 2], tr[4 * q + 3]);
      __syncwarp();
    }
  }
  __syncthreads();
  cs_flush(acc, K, TI, i0, I, part);
}

// ---------------------------------------------------------------- a > 1, fp32: TMA pipeline
// Warps 0..W-1 own rows (lane = row), warp W produces: per stage it TMA-loads NB boxes of
// [TI rows][32 alpha] (128 B swizzle) and copies the stage's 32 NB offsets and signs.  A consumer
// reads its row's 32 values of a box with 8 conflict-free 16-byte loads (chunk q sits at
// q ^ (row & 7)).  Tile tau covers alpha0 = (tau % nat) * 32 NB of beta = tau / nat; alpha >= a
// is zero-filled by TMA and points at the trash row (a % 4 == 0: quads are all-in or all-out).
struct CsTmaParams {
  int64_t a, I;
  int64_t nat;            // alpha tiles per beta: cdiv(a, 32 NB)
  int64_t tiles_per_cta;  // tau range per CTA (blockIdx.y)
  int64_t ntiles;         // nat * b
  int K, stages;
  float* part;      // [gridDim.y][K][I] partial sums
};

template <int NB, int W>
__global__ void __launch_bounds__(32 * W + 32, 1) cs_mid_tma_kernel(const __grid_constant__ CUtensorMap tx,
                                                                   const uint32_t* __restrict__ off,
                                                                   const float* __restrict__ sgn, CsTmaParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int TI = 32 * W;
  constexpr uint32_t BOX = TI * 128, STAGE = NB * BOX;
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // accumulator first (its rows are addressed by the prep offsets), then 1024-aligned tiles
  float* acc = reinterpret_cast<float*>(smem_raw);                                       // [K + 1][TI]
  unsigned char* after = smem_raw + size_t(p.K + 1) * TI * 4;
  unsigned char* tiles = after + ((1024u - (tc::smem_u32(after) & 1023u)) & 1023u);
  uint32_t* offs = reinterpret_cast<uint32_t*>(tiles + size_t(p.stages) * STAGE);        // [stages][32 NB]
  float* sgns = reinterpret_cast<float*>(offs + p.stages * 32 * NB);                     // [stages][32 NB]
  uint64_t* full = reinterpret_cast<uint64_t*>(sgns + p.stages * 32 * NB);
  uint64_t* empty = full + p.stages;
  const int64_t i0 = int64_t(blockIdx.x) * TI;
  const int64_t t0 = int64_t(blockIdx.y) * p.tiles_per_cta;
  const int64_t t1 = t0 + p.tiles_per_cta < p.ntiles ? t0 + p.tiles_per_cta : p.ntiles;
  for (int e = threadIdx.x; e < (p.K + 1) * TI; e += blockDim.x) acc[e] = 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) { tc::mbar_init(&full[s], 2); tc::mbar_init(&empty[s], W); }
    tc::fence_barrier_init();
  }
  __syncthreads();
  const uint32_t trash = uint32_t(p.K) * TI * 4;
  if (wp == W) {
    // ------------------------------------------------------------ producer
    // full[s] completes on two arrivals: the TMA transaction (issued as soon as the slot is free)
    // and the words of the stage, whose global loads were issued one tile ahead
    if (lane == 0) tc::tma_prefetch(&tx);
    uint32_t o_nx[NB];
    float s_nx[NB];
    auto fetch = [&](int64_t t) {
      const int64_t beta = t / p.nat;
      const int64_t al0 = (t - beta * p.nat) * 32 * NB;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int64_t al = al0 + 32 * nb + lane;
        const bool in = t < t1 && al < p.a;
        o_nx[nb] = in ? __ldg(off + al + p.a * beta) : trash;
        s_nx[nb] = in ? __ldg(sgn + al + p.a * beta) : 0.f;
      }
    };
    fetch(t0);
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      if (t - t0 >= p.stages) tc::mbar_wait(&empty[s], ph ^ 1);
      const int64_t beta = t / p.nat;
      const int64_t al0 = (t - beta * p.nat) * 32 * NB;
      if (lane == 0) {
        tc::mbar_expect_tx(&full[s], STAGE);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
          tc::tma_load_3d(tiles + size_t(s) * STAGE + nb * BOX, &tx, &full[s], int(al0 + 32 * nb), int(i0), int(beta));
      }
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        offs[(s * NB + nb) * 32 + lane] = o_nx[nb];
        sgns[(s * NB + nb) * 32 + lane] = s_nx[nb];
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[s]);
      fetch(t + 1);
      if (++s == p.stages) { s = 0; ph ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ consumers: lane owns row
    const int r = 32 * wp + lane;
    unsigned char* rowb = smem_raw + r * 4;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      tc::mbar_wait(&full[s], ph);
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const float4* rowp = reinterpret_cast<const float4*>(tiles + size_t(s) * STAGE + nb * BOX + r * 128);
        const int4* oq = reinterpret_cast<const int4*>(offs + (s * NB + nb) * 32);
        const float4* sq = reinterpret_cast<const float4*>(sgns + (s * NB + nb) * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = rowp[q ^ (r & 7)];
          cs_quad<float>(rowb, oq[q], sq[q], v.x, v.y, v.z, v.w);
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[s]);
      if (++s == p.stages) { s = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  cs_flush(acc, p.K, TI, i0, p.I, p.part);
}

// ---------------------------------------------------------------- a == 1, fp32: TMA pipeline
// X_(0) viewed as the 2-D array (I rows contiguous, J columns).  The producer warp TMA-loads
// [32 columns][256 rows] boxes (no swizzle) and copies the columns' offsets/signs; each of the 2
// consumer warps' lanes owns 4 consecutive rows: per column one 16-byte load of x and a 16-byte
// read-modify-write of its accumulator entries (acc rows [K + 1][256]).
__device__ __forceinline__ float4 f4fma(float s, float4 x, float4 a) {
  return make_float4(fmaf(s, x.x, a.x), fmaf(s, x.y, a.y), fmaf(s, x.z, a.z), fmaf(s, x.w, a.w));
}

struct CsRowsParams {
  int64_t I, J;
  int64_t tiles_per_cta, ntiles;   // tiles of 32 columns
  int K, stages;
  float* part;      // [gridDim.y][K][I] partial sums
};

__global__ void __launch_bounds__(96, 1) cs_rows_tma_kernel(const __grid_constant__ CUtensorMap tx,
                                                            const uint32_t* __restrict__ off,
                                                            const float* __restrict__ sgn, CsRowsParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int W = 2, TI = 256;
  constexpr uint32_t STAGE = 32 * TI * 4;
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* acc = reinterpret_cast<float*>(smem_raw);                                       // [K + 1][TI]
  unsigned char* after = smem_raw + size_t(p.K + 1) * TI * 4;
  unsigned char* tiles = after + ((1024u - (tc::smem_u32(after) & 1023u)) & 1023u);
  uint32_t* offs = reinterpret_cast<uint32_t*>(tiles + size_t(p.stages) * STAGE);        // [stages][32]
  float* sgns = reinterpret_cast<float*>(offs + p.stages * 32);
  uint64_t* full = reinterpret_cast<uint64_t*>(sgns + p.stages * 32);
  uint64_t* empty = full + p.stages;
  const int64_t i0 = int64_t(blockIdx.x) * TI;
  const int64_t t0 = int64_t(blockIdx.y) * p.tiles_per_cta;
  const int64_t t1 = t0 + p.tiles_per_cta < p.ntiles ? t0 + p.tiles_per_cta : p.ntiles;
  for (int e = threadIdx.x; e < (p.K + 1) * TI; e += blockDim.x) acc[e] = 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) { tc::mbar_init(&full[s], 2); tc::mbar_init(&empty[s], W); }
    tc::fence_barrier_init();
  }
  __syncthreads();
  const uint32_t trash = uint32_t(p.K) * TI * 4;
  if (wp == W) {
    if (lane == 0) tc::tma_prefetch(&tx);
    uint32_t o_nx;
    float s_nx;
    auto fetch = [&](int64_t t) {
      const int64_t j = 32 * t + lane;
      const bool in = t < t1 && j < p.J;
      o_nx = in ? __ldg(off + j) : trash;
      s_nx = in ? __ldg(sgn + j) : 0.f;
    };
    fetch(t0);
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      if (t - t0 >= p.stages) tc::mbar_wait(&empty[s], ph ^ 1);
      if (lane == 0) {
        tc::mbar_expect_tx(&full[s], STAGE);
        tc::tma_load_2d(tiles + size_t(s) * STAGE, &tx, &full[s], int(i0), int(32 * t));
      }
      offs[s * 32 + lane] = o_nx;
      sgns[s * 32 + lane] = s_nx;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[s]);
      fetch(t + 1);
      if (++s == p.stages) { s = 0; ph ^= 1; }
    }
  } else {
    const int tr = 32 * wp + lane;                 // rows 4 tr .. 4 tr + 3
    unsigned char* rowb = smem_raw + tr * 16;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      tc::mbar_wait(&full[s], ph);
      const float4* xt = reinterpret_cast<const float4*>(tiles + size_t(s) * STAGE) + tr;   // + c * TI / 4
      const int4* oq = reinterpret_cast<const int4*>(offs + s * 32);
      const float4* sq = reinterpret_cast<const float4*>(sgns + s * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int4 o = oq[q];
        const float4 sg = sq[q];
        const float4 x0 = xt[(4 * q) * (TI / 4)], x1 = xt[(4 * q + 1) * (TI / 4)];
        const float4 x2 = xt[(4 * q + 2) * (TI / 4)], x3 = xt[(4 * q + 3) * (TI / 4)];
        float4* p0 = reinterpret_cast<float4*>(rowb + (uint32_t(o.x) & ~1u));
        float4* p1 = reinterpret_cast<float4*>(rowb + o.y);
        float4* p2 = reinterpret_cast<float4*>(rowb + o.z);
        float4* p3 = reinterpret_cast<float4*>(rowb + o.w);
        if (!(o.x & 1)) {
          const float4 a0 = *p0, a1 = *p1, a2 = *p2, a3 = *p3;
          *p0 = f4fma(sg.x, x0, a0); *p1 = f4fma(sg.y, x1, a1); *p2 = f4fma(sg.z, x2, a2); *p3 = f4fma(sg.w, x3, a3);
        } else {
          *p0 = f4fma(sg.x, x0, *p0); *p1 = f4fma(sg.y, x1, *p1); *p2 = f4fma(sg.z, x2, *p2); *p3 = f4fma(sg.w, x3, *p3);
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[s]);
      if (++s == p.stages) { s = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  cs_flush(acc, p.K, TI, i0, p.I, p.part);
}

// column range per CTA (multiple of blk >= 32): <= 512 K columns (fp32 accumulator length bound)
// and enough CTAs to give every SM two
int64_t pick_jchunk(int64_t J, int64_t gx, int K, int64_t blk, int sms) {
  int64_t jc = int64_t(512) * K;
  const int64_t want = int64_t(2) * sms;
  if (gx * cdiv(J, jc) < want) jc = cdiv(J, cdiv(want, gx));
  if (cdiv(J, jc) > 65535) jc = cdiv(J, 65535);
  jc = cdiv(jc, blk) * blk;
  return jc < blk ? blk : jc;
}

template <typename A>
void reduce_parts(const Ctx& ctx, const A* part, int64_t ny, int K, int64_t I, double* Y, int64_t ldy) {
  const int64_t KI = int64_t(K) * I;
  launch(ctx, "count_reduce", [&] {
    cs_reduce_kernel<A><<<unsigned(cdiv(KI, 256)), 256, 0, ctx.stream>>>(part, ny, KI, I, Y, ldy);
  });
}

void prep(const Ctx& ctx, const int32_t* code, int64_t J, int64_t Jpad, int K, int row_bytes, uint32_t* off,
          float* sgn) {
  launch(ctx, "count_prep", [&] {
    cs_prep_kernel<<<unsigned(cdiv(Jpad / 4, 256)), 256, 0, ctx.stream>>>(code, J, Jpad, K, row_bytes, off, sgn,
                                                                          ctx.d_status);
  });
}

// TMA path for fp32 a > 1; false (nothing launched) when it does not apply
bool count_sketch_tma(const Ctx& ctx, Arena& ws, const float* X, Box box, const int32_t* code, int K, double* Y,
                      int64_t ldy, int sms, size_t budget) {
  if (ctx.simt() || box.a % 4 != 0 || (reinterpret_cast<uintptr_t>(X) % 16) != 0 ||
      box.a >= (int64_t(1) << 31) || box.I >= (int64_t(1) << 31) || box.b >= (int64_t(1) << 31))
    return false;
  // TI rows (lane = row), NB boxes of 32 alpha per stage, as many stages as fit.  Default
  // 256 x 2 (8 consumer warps, 256-byte row segments); RT_CS_TILE=<TI>x<NB> overrides (tuning).
  int TIt = 256, NB = 2;
  if (const char* e = getenv("RT_CS_TILE")) {
    int t2 = 0, n2 = 0;
    if (sscanf(e, "%dx%d", &t2, &n2) == 2) { TIt = t2; NB = n2; }
  }
  while (NB > 1 && int64_t(32) * NB > 2 * box.a) NB /= 2;
  const size_t accb = sizeof(float) * size_t(K + 1) * TIt, stage = size_t(NB) * TIt * 128;
  auto tneed = [&](int st) { return accb + 1024 + size_t(st) * (stage + 32 * NB * 8 + 16); };
  int stages = 4;
  while (stages > 2 && tneed(stages) > budget) --stages;
  if (tneed(stages) > budget) return false;
  CUtensorMap tx;
  const uint64_t d[3] = {uint64_t(box.a), uint64_t(box.I), uint64_t(box.b)};
  const uint64_t st[2] = {uint64_t(box.a) * 4, uint64_t(box.a) * uint64_t(box.I) * 4};
  const uint32_t bx[3] = {32, uint32_t(TIt), 1};
  if (!tc::encode_f32_map(&tx, X, 3, d, st, bx, true)) return false;
  CsTmaParams p;
  p.a = box.a; p.I = box.I; p.K = K; p.stages = stages; 
  p.nat = cdiv(box.a, int64_t(32) * NB);
  p.ntiles = p.nat * box.b;
  const int64_t gx = cdiv(box.I, TIt);
  int64_t tpc = std::max<int64_t>(1, (int64_t(512) * K) / (32 * NB));   // <= 512 K columns per CTA
  const int64_t want = int64_t(sms) * 4;
  if (gx * cdiv(p.ntiles, tpc) < want) tpc = std::max<int64_t>(1, cdiv(p.ntiles, cdiv(want, gx)));
  if (cdiv(p.ntiles, tpc) > 65535) tpc = cdiv(p.ntiles, 65535);
  p.tiles_per_cta = tpc;
  const int64_t J = box.J(), Jp4 = cdiv(J, 4) * 4;
  const auto mk = ws.mark();
  uint32_t* off = ws.alloc_n<uint32_t>(Jp4);
  float* sgn = ws.alloc_n<float>(Jp4);
  prep(ctx, code, J, Jp4, K, TIt * 4, off, sgn);
  const size_t sm = tneed(stages);
  const dim3 grid(unsigned(gx), unsigned(cdiv(p.ntiles, tpc)));
  p.part = ws.alloc_n<float>(int64_t(grid.y) * K * box.I);
  auto go = [&](auto kern, int threads) {
    RT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    kern<<<grid, threads, sm, ctx.stream>>>(tx, off, sgn, p);
  };
  bool ok = true;
  launch(ctx, "count_sketch", [&] {
    if (TIt == 256 && NB == 1) go(cs_mid_tma_kernel<1, 8>, 288);
    else if (TIt == 256 && NB == 2) go(cs_mid_tma_kernel<2, 8>, 288);
    else if (TIt == 128 && NB == 1) go(cs_mid_tma_kernel<1, 4>, 160);
    else if (TIt == 128 && NB == 2) go(cs_mid_tma_kernel<2, 4>, 160);
    else if (TIt == 128 && NB == 4) go(cs_mid_tma_kernel<4, 4>, 160);
    else ok = false;
  });
  if (ok) reduce_parts(ctx, p.part, grid.y, K, box.I, Y, ldy);
  ws.rewind(mk);
  if (!ok) throw Error(kEINVAL, "RT_CS_TILE: unsupported tile");
  return true;
}

bool count_sketch_rows_tma(const Ctx& ctx, Arena& ws, const float* X, Box box, const int32_t* code, int K,
                           double* Y, int64_t ldy, int sms, size_t budget) {
  const int64_t I = box.I, J = box.J();
  if (ctx.simt() || I % 4 != 0 || (reinterpret_cast<uintptr_t>(X) % 16) != 0 || I >= (int64_t(1) << 31) ||
      J >= (int64_t(1) << 31))
    return false;
  constexpr int TI = 256;
  const size_t accb = sizeof(float) * size_t(K + 1) * TI, stage = size_t(32) * TI * 4;
  auto tneed = [&](int st) { return accb + 1024 + size_t(st) * (stage + 32 * 8 + 16); };
  int stages = 4;
  while (stages > 2 && tneed(stages) > budget) --stages;
  if (tneed(stages) > budget) return false;
  CUtensorMap tx;
  const uint64_t d[2] = {uint64_t(I), uint64_t(J)};
  const uint64_t st[1] = {uint64_t(I) * 4};
  const uint32_t bx[2] = {uint32_t(TI), 32};
  if (!tc::encode_f32_map(&tx, X, 2, d, st, bx, false)) return false;
  CsRowsParams p;
  p.I = I; p.J = J; p.K = K; p.stages = stages; 
  p.ntiles = cdiv(J, int64_t(32));
  const int64_t gx = cdiv(I, int64_t(TI));
  int64_t tpc = std::max<int64_t>(1, (int64_t(512) * K) / 32);          // <= 512 K columns per CTA
  const int64_t want = int64_t(sms) * 4;
  if (gx * cdiv(p.ntiles, tpc) < want) tpc = std::max<int64_t>(1, cdiv(p.ntiles, cdiv(want, gx)));
  if (cdiv(p.ntiles, tpc) > 65535) tpc = cdiv(p.ntiles, 65535);
  p.tiles_per_cta = tpc;
  const int64_t Jp4 = cdiv(J, 4) * 4;
  const auto mk = ws.mark();
  uint32_t* off = ws.alloc_n<uint32_t>(Jp4);
  float* sgn = ws.alloc_n<float>(Jp4);
  prep(ctx, code, J, Jp4, K, TI * 4, off, sgn);
  const size_t sm = tneed(stages);
  const dim3 grid(unsigned(gx), unsigned(cdiv(p.ntiles, tpc)));
  p.part = ws.alloc_n<float>(int64_t(grid.y) * K * I);
  launch(ctx, "count_sketch", [&] {
    RT_CUDA(cudaFuncSetAttribute(cs_rows_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    cs_rows_tma_kernel<<<grid, 96, sm, ctx.stream>>>(tx, off, sgn, p);
  });
  reduce_parts(ctx, p.part, grid.y, K, I, Y, ldy);
  ws.rewind(mk);
  return true;
}

}  // namespace

template <typename T>
void count_sketch(const Ctx& ctx, Arena& ws, const T* X, Box box, const int32_t* code, int K, double* Y,
                  int64_t ldy) {
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
  if (mid && std::is_same<T, float>::value &&
      count_sketch_tma(ctx, ws, reinterpret_cast<const float*>(X), box, code, K, Y, ldy, sms, budget))
    return;
  if (!mid && std::is_same<T, float>::value &&
      count_sketch_rows_tma(ctx, ws, reinterpret_cast<const float*>(X), box, code, K, Y, ldy, sms, budget))
    return;
  // warps per CTA: up to 8, no more than the rows need, and the accumulator (+ tiles) must fit
  int W = int(std::min<int64_t>(8, cdiv(I, 32)));
  auto need = [&](int w) { return sizeof(A) * (size_t(K + 1) * 32 * w + (mid ? size_t(w) * 32 * 33 : 0)); };
  while (W > 1 && need(W) > budget) --W;
  if (need(W) > budget) throw Error(kEUNSUPPORTED, "count sketch: K too large for the shared accumulator");
  const int TI = 32 * W;
  const int64_t gx = cdiv(I, TI);
  const size_t sm = need(W);
  constexpr int U = std::is_same<T, double>::value ? 1 : 2;
  const int64_t blk = mid ? 32 * U : 32;
  const int64_t Jpad = cdiv(J, blk) * blk;
  const auto mk = ws.mark();
  uint32_t* off = ws.alloc_n<uint32_t>(Jpad);
  float* sgn = ws.alloc_n<float>(Jpad);
  prep(ctx, code, J, Jpad, K, int(TI * sizeof(A)), off, sgn);
  const int64_t jc = pick_jchunk(J, gx, K, blk, sms);
  const dim3 grid(unsigned(gx), unsigned(cdiv(Jpad, jc)));
  A* part = ws.alloc_n<A>(int64_t(grid.y) * K * I);
  if (!mid) {
    launch(ctx, "count_sketch", [&] {
      RT_CUDA(cudaFuncSetAttribute(cs_rows_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      cs_rows_kernel<T><<<grid, TI, sm, ctx.stream>>>(X, I, J, Jpad, off, sgn, K, jc, part);
    });
  } else {
    launch(ctx, "count_sketch", [&] {
      RT_CUDA(cudaFuncSetAttribute(cs_mid_kernel<T, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      cs_mid_kernel<T, U><<<grid, TI, sm, ctx.stream>>>(X, box.a, I, J, Jpad, off, sgn, K, jc, part);
    });
  }
  reduce_parts(ctx, part, grid.y, K, I, Y, ldy);
  ws.rewind(mk);
}

template void count_sketch<float>(const Ctx&, Arena&, const float*, Box, const int32_t*, int, double*, int64_t);
template void count_sketch<double>(const Ctx&, Arena&, const double*, Box, const int32_t*, int, double*, int64_t);

}  // namespace rt
