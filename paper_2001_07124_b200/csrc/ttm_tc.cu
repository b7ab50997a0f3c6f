// ttm_tc.cu -- tcgen05 tensor-core TTM kernels for sm_100a, fp32 data with
// a 3xTF32 split so the products keep fp32 accuracy:
//     x = x_hi + x_lo (x_hi tf32-exact),  A B ~= A_hi B_hi + A_lo B_hi + A_hi B_lo
// (the A_hi B_lo term is dropped when B is tf32-exact, e.g. a host-rounded Omega).
//
//   ttm_s_tc:  Y(i,k) = sum_j X_(n)(i,j) B(j,k)    (sketch / power product; split-K over j)
//   ttm_t_tc:  out(j,c) = sum_i X_(n)(i,j) Q(i,c)   (Z = X_(n)^T Q and the first core stage)
//
// Per CTA (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + single-thread MMA
// issuer, warps 2-5 = "splitters" (one TMEM lane = one tile row each) that turn the raw fp32 X
// tile (TMA -> smem) into hi/lo tf32 operands in TMEM (tcgen05.st) and split B in place, and that
// drain the fp32 accumulators (tcgen05.ld) in the epilogue.  A comes from TMEM, B from shared
// memory in the K-major SWIZZLE_NONE canonical layout: written directly by a permuted-stride TMA
// box when B is column-major (Z, Q), or transposed by the splitters from a row-major TMA tile
// (Omega; MN-major tf32 B operands were measured not to work with A in TMEM, tools/tc_probe.cu).
// Pipelines: NS-stage smem/TMEM ring (full -> ready -> consumed), double-buffered accumulators.
#include <cstring>

#include "kernels.h"
#include "tc_common.cuh"

namespace rt {
namespace {
using namespace tc;

constexpr int KC = 32;           // contraction elements per stage
constexpr int BM = 128;          // tile rows = TMEM lanes
constexpr int NTHREADS = 192;
__host__ __device__ constexpr uint32_t kAccCol(int b) { return b ? 128u : 0u; }
constexpr uint32_t kAStage = 256;  // A stage s: hi at kAStage + 64 s, lo at + 32

// Shared memory plan: per stage a raw X tile, the K-major B operand (hi), optionally B lo and
// the raw row-major B tile (BRAW).  NS = 4 stages when they fit in ~200 KB, else 3.
template <int NPAD, bool BSPLIT, bool BRAW>
struct Smem {
  static constexpr size_t kX = size_t(BM) * KC * 4;          // 16 KB raw X tile
  static constexpr size_t kB = size_t(NPAD) * KC * 4;        // B tile
  static constexpr size_t per_stage = kX + kB * (1 + (BSPLIT ? 1 : 0) + (BRAW ? 1 : 0));
  static constexpr int NS = per_stage * 4 <= 200 * 1024 ? 4 : 3;
  static constexpr size_t off_x = 0;
  static constexpr size_t off_b = off_x + NS * kX;
  static constexpr size_t off_blo = off_b + NS * kB;
  static constexpr size_t off_braw = off_blo + (BSPLIT ? NS * kB : 0);
  static constexpr size_t off_bar = off_braw + (BRAW ? NS * kB : 0);
  static constexpr size_t bytes = off_bar + 8 * (3 * NS + 4) + 16 + 1024;   // + alignment slack
};

struct Bars {
  uint64_t* full;
  uint64_t* ready;
  uint64_t* consumed;
  uint64_t* acc_full;
  uint64_t* acc_empty;
  uint32_t* tmem_base;
};

template <class L>
__device__ __forceinline__ char* setup(char* raw, Bars& bars) {
  constexpr int NS = L::NS;
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* b = reinterpret_cast<uint64_t*>(base + L::off_bar);
  bars.full = b;
  bars.ready = b + NS;
  bars.consumed = b + 2 * NS;
  bars.acc_full = b + 3 * NS;
  bars.acc_empty = b + 3 * NS + 2;
  bars.tmem_base = reinterpret_cast<uint32_t*>(b + 3 * NS + 4);
  return base;
}

// B descriptor for k-step kk of a stage buffer: K-major, element (n, k) at
// (k/4)*(NPAD*16) + n*16 + (k%4)*4 bytes  (LBO = NPAD*16 between K-chunks, SBO = 128 between 8-row groups)
template <int NPAD>
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr, int kk) {
  return sdesc(saddr + uint32_t(kk) * 2u * NPAD * 16u, /*lbo*/ NPAD * 16u, /*sbo*/ 128u);
}

// Splitter: read this thread's row of the raw X tile, write hi/lo tf32 to TMEM A stage.
template <bool AMN>
__device__ __forceinline__ void split_row_to_tmem(const float* xs, int r, uint32_t t_hi) {
  uint32_t hi[16], lo[16];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (AMN) {  // tile [KC][BM], row r is a column: element (r, k) at k*BM + r
#pragma unroll
      for (int q = 0; q < 16; ++q) split_tf32(xs[(16 * h + q) * BM + r], hi[q], lo[q]);
    } else {    // tile [BM][KC] with 128B swizzle: 16B chunk c of row r at ((c ^ (r&7)) << 4)
      const char* row = reinterpret_cast<const char*>(xs) + r * 128;
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int c = 4 * h + c4;
        const float4 v = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 4));
        split_tf32(v.x, hi[4 * c4 + 0], lo[4 * c4 + 0]);
        split_tf32(v.y, hi[4 * c4 + 1], lo[4 * c4 + 1]);
        split_tf32(v.z, hi[4 * c4 + 2], lo[4 * c4 + 2]);
        split_tf32(v.w, hi[4 * c4 + 3], lo[4 * c4 + 3]);
      }
    }
    tmem_st16(t_hi + 16 * h, hi);
    tmem_st16(t_hi + 32 + 16 * h, lo);
  }
}

// Split the B tile in place (hi) and write lo; elementwise, layout-agnostic.
template <int NPAD>
__device__ __forceinline__ void split_b(float* b, float* blo, int t) {
  float4* b4 = reinterpret_cast<float4*>(b);
  float4* l4 = reinterpret_cast<float4*>(blo);
#pragma unroll
  for (int q = 0; q < NPAD * KC / 4 / 128; ++q) {
    float4 v = b4[t + 128 * q];
    uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
    split_tf32(v.x, h0, l0);
    split_tf32(v.y, h1, l1);
    split_tf32(v.z, h2, l2);
    split_tf32(v.w, h3, l3);
    b4[t + 128 * q] = make_float4(__uint_as_float(h0), __uint_as_float(h1), __uint_as_float(h2), __uint_as_float(h3));
    l4[t + 128 * q] = make_float4(__uint_as_float(l0), __uint_as_float(l1), __uint_as_float(l2), __uint_as_float(l3));
  }
}

// Transpose the raw row-major B tile [KC j][NPAD n] into the K-major operand (+ optional hi/lo split).
template <int NPAD, bool BSPLIT>
__device__ __forceinline__ void transpose_b(const float* raw, float* bhi, float* blo, int t) {
  for (int e = t; e < NPAD * (KC / 4); e += 128) {
    const int n = e % NPAD, jg = e / NPAD;
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = raw[(4 * jg + q) * NPAD + n];
    float4* dh = reinterpret_cast<float4*>(bhi) + (jg * NPAD + n);
    if (BSPLIT) {
      uint32_t h[4], l[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) split_tf32(v[q], h[q], l[q]);
      *dh = make_float4(__uint_as_float(h[0]), __uint_as_float(h[1]), __uint_as_float(h[2]), __uint_as_float(h[3]));
      *(reinterpret_cast<float4*>(blo) + (jg * NPAD + n)) =
          make_float4(__uint_as_float(l[0]), __uint_as_float(l[1]), __uint_as_float(l[2]), __uint_as_float(l[3]));
    } else {
      *dh = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

// MMA issue for one stage: 4 k-steps x (2 or 3) products into accumulator `acc`.
template <int NPAD, bool BSPLIT>
__device__ __forceinline__ void issue_stage(uint32_t tmem, uint32_t acc, int s, uint32_t b_saddr, uint32_t blo_saddr,
                                            uint32_t idesc, bool first) {
  const uint32_t a_hi = tmem + kAStage + 64u * s;
#pragma unroll
  for (int kk = 0; kk < KC / 8; ++kk) {
    const uint64_t bd = bdesc<NPAD>(b_saddr, kk);
    mma_tf32_ts(tmem + acc, a_hi + 8 * kk, bd, idesc, (first && kk == 0) ? 0u : 1u);
    mma_tf32_ts(tmem + acc, a_hi + 32 + 8 * kk, bd, idesc, 1u);
    if (BSPLIT) mma_tf32_ts(tmem + acc, a_hi + 8 * kk, bdesc<NPAD>(blo_saddr, kk), idesc, 1u);
  }
}

// ====================================================================== ttm_s
struct SParams {
  int64_t a, I, b;
  int K;
  int64_t cpb;        // chunks per beta (a > 1)
  int64_t nchunks;    // total j-chunks
  int64_t cps;        // chunks per split (CTA)
  int seg;            // chunks per accumulator segment
  float* part;        // [split][K][I]
};

// BRAW: B is row-major (Omega): TMA a [KC][NPAD] tile, splitters transpose it to K-major.
template <int NPAD, bool BSPLIT, bool AMN, bool BRAW>
__global__ void __launch_bounds__(NTHREADS, 1)
ttm_s_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, const SParams p) {
  using L = Smem<NPAD, BSPLIT, BRAW>;
  constexpr int NS = L::NS;
  extern __shared__ char smem_raw[];
  Bars bars;
  char* sm = setup<L>(smem_raw, bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = int64_t(blockIdx.x) * BM;
  const int64_t c_begin = int64_t(blockIdx.y) * p.cps;
  const int64_t c_end = min(p.nchunks, c_begin + p.cps);
  const int nch = c_end > c_begin ? int(c_end - c_begin) : 0;
  const int nunits = (nch + p.seg - 1) / p.seg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.ready[s], 128);
      mbar_init(&bars.consumed[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.acc_full[b], 1);
      mbar_init(&bars.acc_empty[b], 128);
    }
    fence_barrier_init();
    tma_prefetch(&tmx);
    tma_prefetch(&tmb);
  }
  if (warp == 1) tmem_alloc(bars.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *bars.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = uint32_t(L::kX + L::kB);
      for (int it = 0; it < nch; ++it) {
        const int s = it % NS;
        if (it >= NS) mbar_wait(&bars.consumed[s], ((it / NS) - 1) & 1);
        const int64_t c = c_begin + it;
        mbar_expect_tx(&bars.full[s], bytes);
        float* xs = reinterpret_cast<float*>(sm + L::off_x + s * L::kX);
        float* bs = reinterpret_cast<float*>(sm + (BRAW ? L::off_braw : L::off_b) + s * L::kB);
        int64_t j0;
        if (AMN) {
          j0 = c * KC;
          tma_load_2d(xs, &tmx, &bars.full[s], int(i0), int(j0));
        } else {
          const int64_t beta = c / p.cpb, a0 = (c % p.cpb) * KC;
          j0 = a0 + p.a * beta;
          tma_load_3d(xs, &tmx, &bars.full[s], int(a0), int(i0), int(beta));
        }
        if (BRAW) tma_load_2d(bs, &tmb, &bars.full[s], 0, int(j0));
        else tma_load_3d(bs, &tmb, &bars.full[s], 0, 0, int(j0 / 4));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(BM, NPAD, 0);
      for (int it = 0; it < nch; ++it) {
        const int s = it % NS;
        const int u = it / p.seg;
        const bool first = (it % p.seg) == 0;
        const bool last = ((it % p.seg) == p.seg - 1) || (it == nch - 1);
        const int ab = u & 1;
        if (first && u >= 2) mbar_wait(&bars.acc_empty[ab], ((u >> 1) - 1) & 1);
        mbar_wait(&bars.ready[s], (it / NS) & 1);
        tc_fence_after();
        issue_stage<NPAD, BSPLIT>(tmem, kAccCol(ab), s, smem_u32(sm + L::off_b + s * L::kB),
                                  smem_u32(sm + L::off_blo + s * L::kB), idesc, first);
        mma_commit(&bars.consumed[s]);
        if (last) mma_commit(&bars.acc_full[ab]);
      }
    }
  } else {
    // splitters / epilogue: 128 threads, TMEM lane quarter = warp % 4
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    const int t = threadIdx.x - 64;
    float sums[NPAD];
#pragma unroll
    for (int k = 0; k < NPAD; ++k) sums[k] = 0.f;
    auto epilogue = [&](int u) {
      const int ab = u & 1;
      mbar_wait(&bars.acc_full[ab], (u >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < NPAD / 16; ++cb) {
        uint32_t v[16];
        tmem_ld16(lane_base + kAccCol(ab) + 16 * cb, v);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 16; ++q) sums[16 * cb + q] += __uint_as_float(v[q]);
      }
      tc_fence_before();
      mbar_arrive(&bars.acc_empty[ab]);
    };
    for (int it = 0; it < nch; ++it) {
      const int s = it % NS;
      mbar_wait(&bars.full[s], (it / NS) & 1);
      const float* xs = reinterpret_cast<const float*>(sm + L::off_x + s * L::kX);
      split_row_to_tmem<AMN>(xs, r, lane_base + kAStage + 64u * s);
      if (BRAW)
        transpose_b<NPAD, BSPLIT>(reinterpret_cast<const float*>(sm + L::off_braw + s * L::kB),
                                  reinterpret_cast<float*>(sm + L::off_b + s * L::kB),
                                  reinterpret_cast<float*>(sm + L::off_blo + s * L::kB), t);
      else if (BSPLIT)
        split_b<NPAD>(reinterpret_cast<float*>(sm + L::off_b + s * L::kB),
                      reinterpret_cast<float*>(sm + L::off_blo + s * L::kB), t);
      tmem_wait_st();
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&bars.ready[s]);
      const bool last = ((it % p.seg) == p.seg - 1) || (it == nch - 1);
      const int u = it / p.seg;
      if (last && u >= 1) epilogue(u - 1);
    }
    if (nunits >= 1) epilogue(nunits - 1);
    // partial tile -> part[split][k][i]
    const int64_t i = i0 + r;
    if (i < p.I) {
      float* dst = p.part + int64_t(blockIdx.y) * p.K * p.I;
#pragma unroll
      for (int k = 0; k < NPAD; ++k)
        if (k < p.K) dst[int64_t(k) * p.I + i] = sums[k];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ====================================================================== ttm_t
struct TParams {
  int64_t a, I, b;
  int C;
  int64_t tpb;        // tiles per beta (a > 1)
  int64_t ntiles;
  int nic;            // i-chunks per tile
  int seg;            // i-chunks per accumulator segment (fp32 TMEM accumulation length)
  float* out;
  int64_t so_a, so_c, so_b;
};

template <int NPAD, bool AKM>   // AKM: mode 0 (a == 1), X tile K-major [BM j][KC i]
__global__ void __launch_bounds__(NTHREADS, 1)
ttm_t_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, const TParams p) {
  constexpr bool BSPLIT = true;
  using L = Smem<NPAD, BSPLIT, false>;
  constexpr int NS = L::NS;
  extern __shared__ char smem_raw[];
  Bars bars;
  char* sm = setup<L>(smem_raw, bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t my_tiles = (p.ntiles > blockIdx.x) ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_tiles * p.nic;
  const int64_t nseg_t = (p.nic + p.seg - 1) / p.seg;     // segments per tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.ready[s], 128);
      mbar_init(&bars.consumed[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.acc_full[b], 1);
      mbar_init(&bars.acc_empty[b], 128);
    }
    fence_barrier_init();
    tma_prefetch(&tmx);
    tma_prefetch(&tmb);
  }
  if (warp == 1) tmem_alloc(bars.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *bars.tmem_base;

  auto tile_coords = [&](int64_t tile, int64_t& a0, int64_t& beta) {
    if (AKM) { a0 = 0; beta = tile * BM; }
    else { beta = tile / p.tpb; a0 = (tile % p.tpb) * BM; }
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = uint32_t(L::kX + L::kB);
      for (int64_t it = 0; it < total; ++it) {
        const int s = int(it % NS);
        if (it >= NS) mbar_wait(&bars.consumed[s], uint32_t((it / NS) - 1) & 1);
        const int64_t tile = blockIdx.x + (it / p.nic) * gridDim.x;
        const int ic = int(it % p.nic) * KC;
        int64_t a0, beta;
        tile_coords(tile, a0, beta);
        mbar_expect_tx(&bars.full[s], bytes);
        float* xs = reinterpret_cast<float*>(sm + L::off_x + s * L::kX);
        float* bs = reinterpret_cast<float*>(sm + L::off_b + s * L::kB);
        if (AKM) tma_load_2d(xs, &tmx, &bars.full[s], ic, int(beta));
        else tma_load_3d(xs, &tmx, &bars.full[s], int(a0), ic, int(beta));
        tma_load_3d(bs, &tmb, &bars.full[s], 0, 0, ic / 4);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(BM, NPAD, 0);
      for (int64_t it = 0; it < total; ++it) {
        const int s = int(it % NS);
        const int c = int(it % p.nic);
        const int64_t g = (it / p.nic) * nseg_t + c / p.seg;     // global segment index
        const bool first = (c % p.seg) == 0;
        const bool last = (c % p.seg) == p.seg - 1 || c == p.nic - 1;
        const int ab = int(g & 1);
        if (first && g >= 2) mbar_wait(&bars.acc_empty[ab], uint32_t((g >> 1) - 1) & 1);
        mbar_wait(&bars.ready[s], uint32_t(it / NS) & 1);
        tc_fence_after();
        issue_stage<NPAD, BSPLIT>(tmem, kAccCol(ab), s, smem_u32(sm + L::off_b + s * L::kB),
                                  smem_u32(sm + L::off_blo + s * L::kB), idesc, first);
        mma_commit(&bars.consumed[s]);
        if (last) mma_commit(&bars.acc_full[ab]);
      }
    }
  } else {
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    const int t = threadIdx.x - 64;
    float sums[NPAD];
#pragma unroll
    for (int k = 0; k < NPAD; ++k) sums[k] = 0.f;
    // drain segment g into the register sums; after the last segment of a tile, store the tile
    auto epilogue = [&](int64_t g) {
      const int ab = int(g & 1);
      mbar_wait(&bars.acc_full[ab], uint32_t(g >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < NPAD / 16; ++cb) {
        uint32_t v[16];
        tmem_ld16(lane_base + kAccCol(ab) + 16 * cb, v);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 16; ++q) sums[16 * cb + q] += __uint_as_float(v[q]);
      }
      tc_fence_before();
      mbar_arrive(&bars.acc_empty[ab]);
      if ((g % nseg_t) == nseg_t - 1) {
        const int64_t tile = blockIdx.x + (g / nseg_t) * gridDim.x;
        int64_t a0, beta;
        tile_coords(tile, a0, beta);
        bool valid;
        int64_t ob;
        if (AKM) { const int64_t j = beta + r; valid = j < p.b; ob = j * p.so_b; }
        else { const int64_t al = a0 + r; valid = al < p.a; ob = al * p.so_a + beta * p.so_b; }
        if (valid) {
#pragma unroll
          for (int k = 0; k < NPAD; ++k)
            if (k < p.C) p.out[ob + int64_t(k) * p.so_c] = sums[k];
        }
#pragma unroll
        for (int k = 0; k < NPAD; ++k) sums[k] = 0.f;
      }
    };
    for (int64_t it = 0; it < total; ++it) {
      const int s = int(it % NS);
      mbar_wait(&bars.full[s], uint32_t(it / NS) & 1);
      const float* xs = reinterpret_cast<const float*>(sm + L::off_x + s * L::kX);
      split_row_to_tmem<!AKM>(xs, r, lane_base + kAStage + 64u * s);
      split_b<NPAD>(reinterpret_cast<float*>(sm + L::off_b + s * L::kB),
                    reinterpret_cast<float*>(sm + L::off_blo + s * L::kB), t);
      tmem_wait_st();
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&bars.ready[s]);
      const int c = int(it % p.nic);
      const bool last = (c % p.seg) == p.seg - 1 || c == p.nic - 1;
      const int64_t g = (it / p.nic) * nseg_t + c / p.seg;
      if (last && g >= 1) epilogue(g - 1);
    }
    if (my_tiles >= 1) epilogue(my_tiles * nseg_t - 1);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ================================================================ host side
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
    cudaGetLastError();
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
              const uint32_t* box, bool swz128) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = 1; }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  std::memset(m, 0, sizeof(*m));
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cuuint32_t(rank), const_cast<void*>(ptr), d, s, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

template <typename K>
void set_smem(K kernel, size_t bytes) {
  RT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

template <int NPAD, bool BSPLIT, bool AMN, bool BRAW>
void launch_s(const Ctx& ctx, const CUtensorMap& tx, const CUtensorMap& tb, const SParams& p, dim3 grid) {
  using L = Smem<NPAD, BSPLIT, BRAW>;
  static bool attr = false;
  if (!attr) { set_smem(ttm_s_tc_kernel<NPAD, BSPLIT, AMN, BRAW>, L::bytes); attr = true; }
  launch(ctx, "ttm_s_tc", [&] {
    ttm_s_tc_kernel<NPAD, BSPLIT, AMN, BRAW><<<grid, NTHREADS, L::bytes, ctx.stream>>>(tx, tb, p);
  });
}

template <int NPAD, bool BSPLIT>
void dispatch_s(const Ctx& ctx, bool amn, bool braw, const CUtensorMap& tx, const CUtensorMap& tb,
                const SParams& p, dim3 g) {
  if (amn) {
    if (braw) launch_s<NPAD, BSPLIT, true, true>(ctx, tx, tb, p, g);
    else launch_s<NPAD, BSPLIT, true, false>(ctx, tx, tb, p, g);
  } else {
    if (braw) launch_s<NPAD, BSPLIT, false, true>(ctx, tx, tb, p, g);
    else launch_s<NPAD, BSPLIT, false, false>(ctx, tx, tb, p, g);
  }
}

template <int NPAD, bool AKM>
void launch_t(const Ctx& ctx, const CUtensorMap& tx, const CUtensorMap& tb, const TParams& p, dim3 grid) {
  using L = Smem<NPAD, true, false>;
  static bool attr = false;
  if (!attr) { set_smem(ttm_t_tc_kernel<NPAD, AKM>, L::bytes); attr = true; }
  launch(ctx, "ttm_t_tc", [&] {
    ttm_t_tc_kernel<NPAD, AKM><<<grid, NTHREADS, L::bytes, ctx.stream>>>(tx, tb, p);
  });
}

}  // namespace

__global__ void splitk_reduce_f32_kernel(const float* __restrict__ part, int64_t I, int K, int splits,
                                         double* __restrict__ Y, int64_t ldy) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= I * K) return;
  const int64_t i = e % I, k = e / I;
  double s = 0.0;
  for (int z = 0; z < splits; ++z) s += double(part[(int64_t(z) * K + k) * I + i]);
  Y[i + ldy * k] = s;
}

int tc_npad(int K) { return K <= 16 ? 16 : K <= 32 ? 32 : K <= 48 ? 48 : K <= 64 ? 64 : K <= 80 ? 80 : K <= 96 ? 96 : K <= 128 ? 128 : -1; }

// Returns false (nothing launched) when the shape/alignment is not supported by the TMA path.
bool ttm_s_tc(const Ctx& ctx, Arena& ws, const float* X, Box box, const float* Bm, int64_t ldb, bool b_rowmajor,
              bool b_tf32_exact, int K, double* Y, int64_t ldy) {
  const int npad = tc_npad(K);
  if (npad < 0) return false;
  const int64_t J = box.J();
  if (box.I < 1 || J < KC) return false;
  if (!aligned(X, 16) || !aligned(Bm, 16)) return false;
  if (ldb % 4 || (b_rowmajor && ldb < K) || (!b_rowmajor && ldb < J)) return false;
  const bool amn = (box.a == 1);
  if (amn ? (box.I % 4) : (box.a % 4)) return false;
  if (box.a > INT32_MAX || box.I > INT32_MAX || box.b > INT32_MAX || J > INT32_MAX) return false;
  CUtensorMap tx, tb;
  if (amn) {
    const uint64_t d[2] = {uint64_t(box.I), uint64_t(box.b)}, s[1] = {uint64_t(box.I) * 4};
    const uint32_t bx[2] = {BM, KC};
    if (!make_map(&tx, X, 2, d, s, bx, false)) return false;
  } else {
    const uint64_t d[3] = {uint64_t(box.a), uint64_t(box.I), uint64_t(box.b)};
    const uint64_t s[2] = {uint64_t(box.a) * 4, uint64_t(box.a) * box.I * 4};
    const uint32_t bx[3] = {KC, BM, 1};
    if (!make_map(&tx, X, 3, d, s, bx, true)) return false;
  }
  if (b_rowmajor) {  // element (j, k) at j*ldb + k: raw [KC j][npad k] tile, transposed in smem
    const uint64_t d[2] = {uint64_t(K), uint64_t(J)}, s[1] = {uint64_t(ldb) * 4};
    const uint32_t bx[2] = {uint32_t(npad), KC};
    if (!make_map(&tb, Bm, 2, d, s, bx, false)) return false;
  } else {           // element (j, k) at j + ldb*k; canonical K-major via box (4 j, npad k, 8 j-groups)
    const uint64_t d[3] = {4, uint64_t(K), uint64_t((J + 3) / 4)}, s[2] = {uint64_t(ldb) * 4, 16};
    const uint32_t bx[3] = {4, uint32_t(npad), KC / 4};
    if (!make_map(&tb, Bm, 3, d, s, bx, false)) return false;
  }
  SParams p;
  p.a = box.a; p.I = box.I; p.b = box.b; p.K = K;
  p.cpb = amn ? 1 : cdiv(box.a, KC);
  p.nchunks = amn ? cdiv(box.b, KC) : p.cpb * box.b;
  const int64_t mtiles = cdiv(box.I, BM);
  int64_t splits = std::max<int64_t>(1, (int64_t(ctx.num_sms) * 4 + mtiles - 1) / mtiles);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, p.nchunks / 8));
  splits = std::min<int64_t>(splits, 65535);
  p.cps = cdiv(p.nchunks, splits);
  splits = cdiv(p.nchunks, p.cps);
  p.seg = std::max(1, ctx.tc_seg);
  p.part = ws.alloc_n<float>(splits * K * box.I);
  const dim3 grid{unsigned(mtiles), unsigned(splits), 1u};
  const bool bsplit = !b_tf32_exact;
#define RT_S_CASE(NP)                                                   \
  case NP:                                                              \
    if (bsplit) dispatch_s<NP, true>(ctx, amn, b_rowmajor, tx, tb, p, grid);   \
    else dispatch_s<NP, false>(ctx, amn, b_rowmajor, tx, tb, p, grid);         \
    break;
  switch (npad) {
    RT_S_CASE(16) RT_S_CASE(32) RT_S_CASE(48) RT_S_CASE(64) RT_S_CASE(80) RT_S_CASE(96) RT_S_CASE(128)
    default: return false;
  }
#undef RT_S_CASE
  const int64_t n = box.I * K;
  launch(ctx, "splitk_reduce", [&] {
    splitk_reduce_f32_kernel<<<unsigned(cdiv(n, 256)), 256, 0, ctx.stream>>>(p.part, box.I, K, int(splits), Y, ldy);
  });
  return true;
}

bool ttm_t_tc(const Ctx& ctx, const float* X, Box box, const float* Q, int64_t ldq, int C, float* out,
              int64_t so_a, int64_t so_c, int64_t so_b) {
  const int npad = tc_npad(C);
  if (npad < 0) return false;
  const bool akm = (box.a == 1);
  if (!aligned(X, 16) || !aligned(Q, 16) || ldq % 4 || ldq < box.I) return false;
  if (akm ? (box.I % 4) : (box.a % 4)) return false;
  if (box.a > INT32_MAX || box.I > INT32_MAX || box.b > INT32_MAX) return false;
  CUtensorMap tx, tb;
  if (akm) {  // X(j=beta, i) at i + I*beta: box (32 i, 128 j), 128B swizzle
    const uint64_t d[2] = {uint64_t(box.I), uint64_t(box.b)}, s[1] = {uint64_t(box.I) * 4};
    const uint32_t bx[2] = {KC, BM};
    if (!make_map(&tx, X, 2, d, s, bx, true)) return false;
  } else {    // X(alpha, i, beta): box (128 alpha, 32 i, 1)
    const uint64_t d[3] = {uint64_t(box.a), uint64_t(box.I), uint64_t(box.b)};
    const uint64_t s[2] = {uint64_t(box.a) * 4, uint64_t(box.a) * box.I * 4};
    const uint32_t bx[3] = {BM, KC, 1};
    if (!make_map(&tx, X, 3, d, s, bx, false)) return false;
  }
  {  // Q(i, c) at i + ldq*c, K-major canonical via box (4 i, npad c, 8 i-groups)
    const uint64_t d[3] = {4, uint64_t(C), uint64_t((box.I + 3) / 4)}, s[2] = {uint64_t(ldq) * 4, 16};
    const uint32_t bx[3] = {4, uint32_t(npad), KC / 4};
    if (!make_map(&tb, Q, 3, d, s, bx, false)) return false;
  }
  TParams p;
  p.a = box.a; p.I = box.I; p.b = box.b; p.C = C;
  p.tpb = akm ? 1 : cdiv(box.a, BM);
  p.ntiles = akm ? cdiv(box.b, BM) : p.tpb * box.b;
  p.nic = int(cdiv(box.I, KC));
  p.seg = std::max(1, ctx.tc_seg);
  p.out = out; p.so_a = so_a; p.so_c = so_c; p.so_b = so_b;
  const int64_t grid = std::min<int64_t>(p.ntiles, ctx.num_sms);
#define RT_T_CASE(NP)                                                           \
  case NP:                                                                      \
    if (akm) launch_t<NP, true>(ctx, tx, tb, p, dim3(unsigned(grid)));         \
    else launch_t<NP, false>(ctx, tx, tb, p, dim3(unsigned(grid)));            \
    break;
  switch (npad) {
    RT_T_CASE(16) RT_T_CASE(32) RT_T_CASE(48) RT_T_CASE(64) RT_T_CASE(80) RT_T_CASE(96) RT_T_CASE(128)
    default: return false;
  }
#undef RT_T_CASE
  return true;
}

}  // namespace rt
