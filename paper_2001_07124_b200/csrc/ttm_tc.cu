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
// tile (TMA -> smem) into hi/lo tf32 operands in TMEM (tcgen05.st), split B in place, and drain
// the fp32 accumulators (tcgen05.ld) in the epilogue.  A comes from TMEM; B (always a
// column-major fp32 matrix: Omega, Z or Q) is TMA'd as a [NPAD rows][32 K] 128B-swizzled tile,
// i.e. directly the K-major SWIZZLE_128B UMMA canonical layout (tools/tc_probe.cu verifies the
// descriptor; MN-major tf32 B operands were measured not to work with A in TMEM).
// Pipelines: NS-stage smem/TMEM ring (full -> ready -> consumed) and double-buffered TMEM
// accumulators drained every `seg` stages into fp32 registers: the tensor core's fp32 accumulation
// error grows with the accumulation length (7.5e-6 relative after 1024 terms, 2.6e-5 after 3.5K;
// 1.4e-6 when drained every 128, tests/test_gpu_tc.py).
#include <cuda_fp16.h>

#include <cstdio>
#include <cstring>
#include <type_traits>
#include <vector>

#include "kernels.h"
#include "tc_common.cuh"

namespace rt {
namespace {
using namespace tc;

constexpr int KC = 32;           // contraction elements per stage
constexpr int BM = 128;          // tile rows = TMEM lanes
constexpr int NTHREADS = 224;    // residual kernel: TMA, 2 MMA issuers, 4 split/epilogue warps
constexpr int NT_TTM = 384;      // TTM kernels: X producer, MMA issuer, 4 splitters, B producer, 2nd issuer,
                                 // 4 epilogue warps (warp w accesses TMEM lanes 32 (w % 4) ..)

// MMA issue model (tools/mma_rate.cu): one thread's tcgen05.mma instructions complete one after
// another (~110-160 cycles each whatever N <= 256), while MMAs issued by different warps overlap.
// So the work of a stage is spread over two issuer warps and made of as few, as wide instructions
// as possible:
//   !BSPLIT (B tf32-exact, e.g. a host-rounded Omega): D += A_hi B + A_lo B; the 4 k-steps are split
//     between NI issuers, each with its own double-buffered accumulator of NPAD columns;
//   BSPLIT: B = B_hi + B_lo is split in shared memory into one slot [B_hi | B_lo] that is a single
//     operand of N = NH + NPAD columns, so issuer 0 runs D0 += A_hi [B_hi | B_lo] and issuer 1 runs
//     D1 += A_lo B_hi (2 instructions per k-step instead of 3; single-buffered accumulators).
//     D0's hi block only accumulates A_hi B_hi, the correction terms land in their own columns,
//     so the fp32 accumulation error per segment is a third of the 3-products-in-one form.
// TMEM (512 columns): accumulators first, then NB A slots of 64 columns (hi | lo).
// Shared memory rings:
//   X ring (NX stages of raw 16 KB X tiles): TMA -> splitter, released right after the split;
//   B ring (NBS slots): TMA -> (splitter: B_lo) -> MMA, released by tcgen05.commit.
// B tile: K-major [NPAD][32] (128 B rows, SWIZZLE_128B), or MN-major (row-major B in global
// memory: Omega / Z) as ceil(NPAD/32) atom columns of [32 k-rows][32 n] (4 KB each,
// SWIZZLE_128B_ATOM_32B); NH = N width of the hi part (MN-major: padded to 32).
// chunks per stage for the sketch kernel: 2 when two 128-column A stages still fit next to the
// accumulators, else 1
template <int NPAD, bool BSPLIT, bool BMN>
constexpr int sketch_cps() {
  constexpr int nbx = (NPAD + 31) / 32, nh = BMN ? nbx * 32 : NPAD;
  constexpr int ni = BSPLIT ? 2 : (NPAD <= 96 ? 2 : 1);
  constexpr int acc = BSPLIT ? nh + 2 * NPAD : ni * NPAD;
  constexpr int abase = (acc + 63) & ~63;
  return (512 - abase) / 128 >= 2 ? 2 : 1;
}

// X stage geometry.  XW = 1: one chunk per stage, the [BM rows][KC] tile with the 128 B swizzle
// (one 128 B piece of every X row per TMA box).  XW > 1 ("wide rows", strided modes n > 0): XW
// chunks per stage in one unswizzled box of BM rows x (KC XW + 4) elements, so every X row is read
// as one contiguous (KC XW + 4) x 4 B run (512 B + 16 at XW = 4; the 16 B overlap with the next
// stage is never used).  The 4-element pad makes the row pitch 4 words mod 32: the splitters' 16 B
// row reads hit 8 distinct bank groups per warp (4 wavefronts, the minimum for 512 B).
template <int XW>
constexpr uint32_t x_pitch() { return XW == 1 ? uint32_t(KC) * 4u : uint32_t(KC * XW + 4) * 4u; }

template <int NPAD, bool BSPLIT, bool BMN, int CPS_ = 1, uint32_t OUTB = 0, int XW = 1>
struct Plan {
  // CPS chunks (of KC contraction elements) per pipeline stage: one ready wait, one commit and
  // one A slot of 64 CPS columns per stage -- the issuer warps' per-stage overhead (barrier wait,
  // commit, loop bookkeeping: ~450 cycles measured) is paid once per CPS chunks
  static constexpr int CPS = CPS_;
  static constexpr int NBX = (NPAD + 31) / 32;
  static constexpr int NH = BMN ? NBX * 32 : NPAD;
  static constexpr uint32_t kB = BMN ? uint32_t(NBX) * 4096u : uint32_t(NPAD) * KC * 4u;
  static constexpr uint32_t kBS = BSPLIT ? 2u * kB : kB;
  static constexpr int NI = BSPLIT ? 2 : (NPAD <= 96 ? 2 : 1);
  // single-buffered accumulators: the dedicated epilogue warps drain a segment in a few hundred
  // cycles, and the TMEM saved buys A slots (a deeper splitter -> MMA ring)
  static constexpr int NBUF = 1;
  static constexpr uint32_t acc_cols = BSPLIT ? uint32_t(NH + 2 * NPAD) : uint32_t(NI * NPAD);
  static constexpr uint32_t a_base = (acc_cols + 63u) & ~63u;
  static constexpr int NB_fit = int((512u - a_base) / (64u * CPS));
  // wide X stages: leave room for two of them in shared memory
  static constexpr int NB_smem = XW == 1 ? 6 : int((224u * 1024u - 2u * BM * x_pitch<XW>() - OUTB) / (CPS * (BSPLIT ? 2u : 1u) * kB));
  static constexpr int NB = NB_fit < NB_smem ? (NB_fit > 6 ? 6 : NB_fit) : (NB_smem > 6 ? 6 : NB_smem);   // A ring stages
  static_assert(!BSPLIT || NH + NPAD <= 256, "concatenated B operand wider than 256");
  __host__ __device__ static constexpr uint32_t acc(int q, int b) {
    return BSPLIT ? (q == 0 ? 0u : uint32_t(NH + NPAD)) : uint32_t((NBUF * q + b) * NPAD);
  }
  __host__ __device__ static constexpr uint32_t a_slot(int s) { return a_base + 64u * CPS * uint32_t(s); }
  // shared memory
  static constexpr uint32_t kX = uint32_t(BM) * x_pitch<XW>();   // one X stage (XW chunks)
  static constexpr uint32_t budget = 224u * 1024u;
  // One stage = one A slot + one B slot, released together by a single tcgen05.commit per issuer
  // (every commit stalls the issuing warp's MMA stream, so there is one per stage).
  static constexpr int NBS = NB * CPS;                  // B slots (one per chunk)
  static constexpr int NX_fit = int((budget - NBS * kBS - OUTB) / kX);
  static constexpr int NX = NX_fit > 10 ? 10 : NX_fit;
  static_assert(kX % 1024 == 0, "X stages keep the 1 KB alignment of the swizzled B slots");
  static constexpr uint32_t off_x = 0;
  static constexpr uint32_t off_b = off_x + NX * kX;
  static constexpr uint32_t off_o = off_b + NBS * kBS;  // output staging (1024-aligned), OUTB bytes
  static constexpr uint32_t off_bar = off_o + OUTB;
  static constexpr int nbar = 2 * NX + 2 * NBS + 2 * 8 + 4;
  static constexpr uint32_t bytes = off_bar + 8 * nbar + 16;
  // feasible plan (checked by the kernels; the host picks a feasible X stage width)
  static constexpr bool ok = NB >= 2 && NX >= (XW == 1 ? 4 : 2);
};

struct Bars {
  uint64_t *x_full, *x_free, *b_full, *b_free, *ready, *tfree, *acc_full, *acc_empty;
  uint32_t* tmem_slot;
};

template <class L>
__device__ __forceinline__ Bars bars_of(uint8_t* smem) {
  uint64_t* b = reinterpret_cast<uint64_t*>(smem + L::off_bar);
  Bars r;
  r.x_full = b;
  r.x_free = b + L::NX;
  r.b_full = b + 2 * L::NX;
  r.b_free = b + 2 * L::NX + 2 * L::NBS + 8;   // == tfree: a stage's A and B slots are released together
  r.ready = b + 2 * L::NX + 2 * L::NBS;
  r.tfree = b + 2 * L::NX + 2 * L::NBS + 8;
  r.acc_full = b + 2 * L::NX + 2 * L::NBS + 2 * 8;
  r.acc_empty = r.acc_full + 2;
  r.tmem_slot = reinterpret_cast<uint32_t*>(b + L::nbar);
  return r;
}

template <class L>
__device__ __forceinline__ void init_bars(const Bars& b) {
  for (int s = 0; s < L::NX; ++s) { mbar_init(&b.x_full[s], 1); mbar_init(&b.x_free[s], 128); }
  for (int s = 0; s < L::NBS; ++s) mbar_init(&b.b_full[s], 1);
  for (int s = 0; s < L::NB; ++s) { mbar_init(&b.ready[s], 128); mbar_init(&b.tfree[s], L::NI); }
  for (int k = 0; k < 2; ++k) { mbar_init(&b.acc_full[k], L::NI); mbar_init(&b.acc_empty[k], 128); }
  fence_barrier_init();
}

// K-major SWIZZLE_128B descriptor of a [rows][32 fp32] tile, advanced to k-step kk (8 elements)
__device__ __forceinline__ uint64_t bdesc_sw128(uint32_t saddr, int kk) {
  return sdesc(saddr + 32u * uint32_t(kk), 16u, 1024u) | (uint64_t(2) << 61);
}
// MN-major tf32 descriptor (layout SWIZZLE_128B_BASE32B, tools/mn_probe.cu): atoms of 4 k-rows x
// 128 B; LBO = 4 KB between 32-wide N atom columns, SBO = 512 B between 4-row k groups; k-step kk
// (8 rows) starts 1 KB further.
__device__ __forceinline__ uint64_t bdesc_mn(uint32_t saddr, int kk) {
  return sdesc(saddr + 1024u * uint32_t(kk), 4096u, 512u) | (uint64_t(1) << 61);
}
template <bool BMN>
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr, int kk) {
  return BMN ? bdesc_mn(saddr, kk) : bdesc_sw128(saddr, kk);
}

// Splitter: read this thread's row of the raw X tile, write hi/lo tf32 to its TMEM lane.
//   AMN  : tile [KC][BM] (row r is a column): element (r, k) at k*BM + r
//   !AMN : tile [BM][KC] with 128B swizzle: 16B chunk c of row r at ((c ^ (r&7)) << 4)
// AMAX: also fold max |x| and sum |x| of the row into m, sq (the fp16 scale of X, R29, taken
// during a tf32 pass)
template <bool AMN, bool AMAX = false>
__device__ __forceinline__ void split_row_to_tmem(const float* xs, int r, uint32_t t_hi, float* m = nullptr,
                                                  float* sq = nullptr) {
  uint32_t hi[32], lo[32];
  if (AMN) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const float v = xs[q * BM + r];
      if (AMAX) { *m = fmaxf(*m, fabsf(v)); *sq += fabsf(v); }
      split_tf32(v, hi[q], lo[q]);
    }
  } else {
    const float* row = xs + r * KC;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 v = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 2));
      if (AMAX) {
        *m = fmaxf(fmaxf(*m, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));
        *sq += (fabsf(v.x) + fabsf(v.y)) + (fabsf(v.z) + fabsf(v.w));
      }
      split_tf32(v.x, hi[4 * c + 0], lo[4 * c + 0]);
      split_tf32(v.y, hi[4 * c + 1], lo[4 * c + 1]);
      split_tf32(v.z, hi[4 * c + 2], lo[4 * c + 2]);
      split_tf32(v.w, hi[4 * c + 3], lo[4 * c + 3]);
    }
  }
  // all smem reads of the X stage are done once the values are in registers
  tmem_st16(t_hi, *reinterpret_cast<const uint32_t(*)[16]>(&hi[0]));
  tmem_st16(t_hi + 16, *reinterpret_cast<const uint32_t(*)[16]>(&hi[16]));
  tmem_st16(t_hi + 32, *reinterpret_cast<const uint32_t(*)[16]>(&lo[0]));
  tmem_st16(t_hi + 48, *reinterpret_cast<const uint32_t(*)[16]>(&lo[16]));
}

// Wide-row X stage (XW > 1): this thread's row is contiguous (pitch x_pitch<XW>, 4 words mod 32:
// conflict-free 16 B reads); `row` points at the chunk's 32 elements.
template <bool AMAX = false>
__device__ __forceinline__ void split_wrow_to_tmem(const float* row, uint32_t t_hi, float* m = nullptr,
                                                   float* sq = nullptr) {
  uint32_t hi[32], lo[32];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 v = *reinterpret_cast<const float4*>(row + 4 * c);
    if (AMAX) {
      *m = fmaxf(fmaxf(*m, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));
      *sq += (fabsf(v.x) + fabsf(v.y)) + (fabsf(v.z) + fabsf(v.w));
    }
    split_tf32(v.x, hi[4 * c + 0], lo[4 * c + 0]);
    split_tf32(v.y, hi[4 * c + 1], lo[4 * c + 1]);
    split_tf32(v.z, hi[4 * c + 2], lo[4 * c + 2]);
    split_tf32(v.w, hi[4 * c + 3], lo[4 * c + 3]);
  }
  tmem_st16(t_hi, *reinterpret_cast<const uint32_t(*)[16]>(&hi[0]));
  tmem_st16(t_hi + 16, *reinterpret_cast<const uint32_t(*)[16]>(&hi[16]));
  tmem_st16(t_hi + 32, *reinterpret_cast<const uint32_t(*)[16]>(&lo[0]));
  tmem_st16(t_hi + 48, *reinterpret_cast<const uint32_t(*)[16]>(&lo[16]));
}

// Split the B tile in place (hi) and write lo; elementwise, layout-agnostic, conflict-free.
template <uint32_t BYTES>
__device__ __forceinline__ void split_b(float* b, float* blo, int t) {
  float4* b4 = reinterpret_cast<float4*>(b);
  float4* l4 = reinterpret_cast<float4*>(blo);
#pragma unroll
  for (int q = 0; q < int(BYTES / 16 / 128); ++q) {
    const float4 v = b4[t + 128 * q];
    uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
    split_tf32(v.x, h0, l0);
    split_tf32(v.y, h1, l1);
    split_tf32(v.z, h2, l2);
    split_tf32(v.w, h3, l3);
    b4[t + 128 * q] = make_float4(__uint_as_float(h0), __uint_as_float(h1), __uint_as_float(h2), __uint_as_float(h3));
    l4[t + 128 * q] = make_float4(__uint_as_float(l0), __uint_as_float(l1), __uint_as_float(l2), __uint_as_float(l3));
  }
}

// One stage (4 k-steps) of issuer q into accumulator buffer ab (see Plan).
template <class P, bool BSPLIT, bool BMN>
__device__ __forceinline__ void issue_stage(uint32_t tmem, int q, int ab, uint32_t a_col, uint32_t b_saddr,
                                            uint32_t idesc0, uint32_t idesc1, bool first) {
  const uint32_t a_hi = tmem + a_col;
  if constexpr (BSPLIT) {
    const uint32_t d = tmem + P::acc(q, 0);
#pragma unroll
    for (int kk = 0; kk < KC / 8; ++kk) {
      const uint64_t bd = bdesc<BMN>(b_saddr, kk);      // [B_hi | B_lo] (issuer 0) or B_hi (issuer 1)
      if (q == 0) mma_tf32_ts_w(d, a_hi + 8 * kk, bd, idesc0, (first && kk == 0) ? 0u : 1u);
      else mma_tf32_ts_w(d, a_hi + 32 + 8 * kk, bd, idesc1, (first && kk == 0) ? 0u : 1u);
    }
  } else {
    const uint32_t d = tmem + P::acc(q, ab);
    constexpr int KPI = (KC / 8) / P::NI;
#pragma unroll
    for (int k = 0; k < KPI; ++k) {
      const int kk = q * KPI + k;
      const uint64_t bd = bdesc<BMN>(b_saddr, kk);
      mma_tf32_ts_w(d, a_hi + 8 * kk, bd, idesc0, (first && k == 0) ? 0u : 1u);
      mma_tf32_ts_w(d, a_hi + 32 + 8 * kk, bd, idesc0, 1u);
    }
  }
}

// Ring position: stage index and parity of the current round.
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  template <int N> __device__ __forceinline__ void next() { if (++s == N) { s = 0; ph ^= 1; } }
};

template <class P>
__device__ __forceinline__ int acc_buf(int64_t u) { return P::NBUF == 2 ? int(u & 1) : 0; }
template <class P>
__device__ __forceinline__ uint32_t acc_par(int64_t u) { return uint32_t(P::NBUF == 2 ? (u >> 1) : u) & 1u; }

// Issuer side: before the first stage of segment u, wait until the epilogue has drained the
// accumulator buffer it reuses.
template <class P>
__device__ __forceinline__ void wait_acc_free(const Bars& b, int64_t u) {
  if (u >= P::NBUF) mbar_wait(&b.acc_empty[acc_buf<P>(u)], acc_par<P>(u - P::NBUF));
}

template <int NPAD>
__device__ __forceinline__ void add_cols(uint32_t taddr, float (&sums)[NPAD]) {
  // 32 columns per tcgen05.ld batch keeps the epilogue warps under the 384-thread register budget
#pragma unroll
  for (int c0 = 0; c0 < NPAD; c0 += 32) {
    uint32_t v[32];
    tmem_ld16(taddr + c0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
    if (c0 + 16 < NPAD) tmem_ld16(taddr + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
    tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (c0 + k < NPAD) sums[c0 + k] += __uint_as_float(v[k]);
  }
}

// Drain segment u's accumulators into the register sums and release them.
template <class P, int NPAD, bool BSPLIT>
__device__ __forceinline__ void drain_acc(const Bars& b, uint32_t lane_base, int64_t u, float (&sums)[NPAD]) {
  const int ab = acc_buf<P>(u);
  mbar_wait(&b.acc_full[ab], acc_par<P>(u));
  tc_fence_after();
  if constexpr (BSPLIT) {
    add_cols<NPAD>(lane_base + P::acc(0, 0), sums);             // A_hi B_hi
    add_cols<NPAD>(lane_base + P::acc(0, 0) + P::NH, sums);     // A_hi B_lo
    add_cols<NPAD>(lane_base + P::acc(1, 0), sums);             // A_lo B_hi
  } else {
#pragma unroll
    for (int q = 0; q < P::NI; ++q) add_cols<NPAD>(lane_base + P::acc(q, ab), sums);
  }
  tc_fence_before();
  mbar_arrive(&b.acc_empty[ab]);
}

__device__ __forceinline__ void xstat_add(unsigned int* stat, float m, float sq) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(stat, __float_as_uint(m));                // non-negative floats order as integers
    atomicAdd(reinterpret_cast<double*>(stat + 2), double(sq));   // sum |x|
  }
}
// ====================================================================== ttm_s
struct SParams {
  int64_t a, I, b;
  int K;
  int64_t cpb;        // chunks per beta (a > 1)
  int64_t nchunks;    // total j-chunks
  int64_t per;        // chunks per split (a multiple of the X stage width)
  int xfirst;         // wide rows: 1 = X tiles with L2::evict_first like the 1-chunk stages (A/B option)
  int seg;            // chunks per accumulator segment
  int ablate;         // profiling only: 1 = no MMA, 2 = no split work (results invalid)
  int skew;           // chunk-order rotation per M-tile (decorrelates the rows' DRAM addresses)
  float* part;        // [split][K][I]
  unsigned int* amax; // optional: X statistics of the tiles read (xstat_add: max |X| bits, sum |x|)
  const float* gate;  // optional: run only if *gate == 0 (the tf32 fallback of an fp16-split launch)
  unsigned int* runs; // optional: run counters ([0] fp16 split, [1] tf32 twin), bumped by CTA (0, 0)
  unsigned long long* tim;   // diagnostics (RT_OPT_TC_ABLATE = 1000): per-CTA role wait cycles, else null
  long long* trace;          // diagnostics (RT_OPT_TC_ABLATE = 2000): per-chunk event clocks of CTA (0,0)
};
#if RT_TC_DIAG
#define RT_TRACE(p, it, k)                                                                         \
  do {                                                                                             \
    if ((p).trace && blockIdx.x == 0 && blockIdx.y == 0 && (it) < 512 && (threadIdx.x & 31) == 0) \
      (p).trace[(it) * 8 + (k)] = clock64();                                                       \
  } while (0)
#else
#define RT_TRACE(p, it, k) do { } while (0)
#endif

// diagnostics: accumulate the cycles spent in `body` into slot k of this CTA's timing record
// RT_TC_DIAG=1 (make diag build) compiles the per-role timers / traces in; the normal build has
// none of their instructions in the issue loops.
#ifndef RT_TC_DIAG
#define RT_TC_DIAG 0
#endif
#if !RT_TC_DIAG
#define RT_TIMED(tim, k, ...) \
  do {                        \
    (void)(tim);              \
    __VA_ARGS__;              \
  } while (0)
#else
#define RT_TIMED(tim, k, ...)                                                                   \
  do {                                                                                           \
    if (tim) {                                                                                   \
      const long long t0_ = clock64();                                                           \
      __VA_ARGS__;                                                                               \
      if ((threadIdx.x & 31) == 0)                                                               \
        atomicAdd(&(tim)[(blockIdx.y * gridDim.x + blockIdx.x) * 24 + (k)], (unsigned long long)(clock64() - t0_)); \
    } else {                                                                                     \
      __VA_ARGS__;                                                                               \
    }                                                                                            \
  } while (0)
#endif

// chunk c -> X tile coordinates and first B row j0
template <bool AMN>
__device__ __forceinline__ void chunk_coords(const SParams& p, int64_t c, int64_t& a0, int64_t& beta, int64_t& j0) {
  if (AMN) { a0 = 0; beta = c * KC; j0 = beta; }
  else { beta = c / p.cpb; a0 = (c % p.cpb) * KC; j0 = a0 + p.a * beta; }
}

// grid (mtiles, splits): CTA (m, z) sums the contiguous chunk range z*per .. (z+1)*per-1 of M-tile m.
// The M-tiles of a split are adjacent in launch order, so the CTAs that share a B chunk (Omega / Z
// rows) run in the same wave and in near lockstep: B comes from DRAM once and from L2 for the rest.
// BPRE (with BSPLIT): B is pre-split in global memory, row j = [hi (NH columns) | lo (NH columns)],
// and is loaded as the whole [B_hi | B_lo] slot; nothing is split in the kernel.
// XW > 1: wide-row X stages (see x_pitch), strided modes only; the CTA's chunk range is a multiple
// of XW chunks within one beta (the host checks a % (KC XW) == 0).
template <int NPAD, bool BSPLIT, bool AMN, bool BPRE, int XW = 1>
__global__ void __launch_bounds__(NT_TTM, 1)
ttm_s_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, const SParams p) {
  static_assert(!BPRE || BSPLIT, "pre-split B implies the split product form");
  static_assert(XW == 1 || !AMN, "wide X rows are for the strided modes");
  if (p.gate && *p.gate != 0.f) return;                // fp16-split launch in charge (R29)
  if (p.gate && p.runs && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&p.runs[1], 1u);
  using L = Plan<NPAD, BSPLIT, true, sketch_cps<NPAD, BSPLIT, true>(), 0, XW>;
  static_assert(L::ok, "infeasible TMEM / shared-memory plan");
  constexpr int NX = L::NX, CPS = L::CPS, NB = L::NB;
  extern __shared__ __align__(1024) uint8_t smem[];
  const Bars b = bars_of<L>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t z = blockIdx.y, S = gridDim.y;
  const int64_t i0 = int64_t(blockIdx.x) * BM;
  // contiguous chunk range per split: consecutive TMA boxes of a CTA continue the same rows, which
  // keeps DRAM pages (and 256 B L2 promotions) useful on the strided last-mode rows
  const int64_t per = p.per;                           // contiguous chunks per split (host)
  (void)S;
  const int64_t cbeg = z * per;
  const int nch = cbeg < p.nchunks ? int(min(per, p.nchunks - cbeg)) : 0;
  const int nst = (nch + CPS - 1) / CPS;               // stages
  const int rot = (nch && XW == 1) ? int((int64_t(blockIdx.x) * p.skew) % nch) : 0;
  auto chunk_of = [&](int it) { int c = it + rot; return cbeg + (c >= nch ? c - nch : c); };
  // stage g -> ring slot and round parity
  auto st_slot = [](int g) { return g % NB; };
  auto st_par = [](int g) { return uint32_t(g / NB) & 1u; };

  if (threadIdx.x == 0) {
    init_bars<L>(b);
    tma_prefetch(&tmx);
    tma_prefetch(&tmb);
  }
  if (warp == 1) tmem_alloc(b.tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *b.tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                   // ---------------- X producer (one box per XW chunks)
      Ring rx;
      // wide rows: the 16 B pad sector is read again by the next stage, so X lines keep the normal
      // L2 priority there (evict_first sends the re-read to DRAM)
      const uint64_t pol = (XW > 1 && !p.xfirst) ? policy_evict_normal() : policy_evict_first();
      int xi = 0;
      for (int it = 0; it < nch; it += XW, ++xi, rx.next<NX>()) {
        if (xi >= NX) RT_TIMED(p.tim, 0, mbar_wait(&b.x_free[rx.s], rx.ph ^ 1));
        int64_t a0, beta, j0;
        chunk_coords<AMN>(p, chunk_of(it), a0, beta, j0);
        mbar_expect_tx(&b.x_full[rx.s], L::kX);
        void* xs = smem + L::off_x + rx.s * L::kX;
        if (AMN) tma_load_2d_hint(xs, &tmx, &b.x_full[rx.s], int(i0), int(j0), pol);
        else tma_load_3d_hint(xs, &tmx, &b.x_full[rx.s], int(a0), int(i0), int(beta), pol);
      }
    }
  } else if (warp == 6) {
    if (lane == 0) {                                   // ---------------- B producer (one slot per chunk)
      const uint64_t pol = policy_evict_last();
      for (int it = 0; it < nch; ++it) {
        const int g = it / CPS, bs = it % L::NBS;
        if (g >= NB) RT_TIMED(p.tim, 1, mbar_wait(&b.tfree[st_slot(g)], st_par(g) ^ 1));   // stage g - NB done
        int64_t a0, beta, j0;
        chunk_coords<AMN>(p, chunk_of(it), a0, beta, j0);
        constexpr int nbox = BPRE ? 2 * L::NBX : L::NBX;
        mbar_expect_tx(&b.b_full[bs], nbox * 4096);
#pragma unroll
        for (int x = 0; x < nbox; ++x)
          tma_load_2d_hint(smem + L::off_b + bs * L::kBS + x * 4096, &tmb, &b.b_full[bs], 32 * x, int(j0), pol);
      }
    }
  } else if (warp == 1 || warp == 7) {
    const int q = warp == 1 ? 0 : 1;
    if (q < L::NI) {                                   // ---------------- MMA issuers (whole warp)
      unsigned long long* tim = p.tim;
      const uint32_t idesc0 = idesc_tf32(BM, BSPLIT ? L::NH + NPAD : NPAD, 1);
      const uint32_t idesc1 = idesc_tf32(BM, NPAD, 1);
      const int spg = (p.seg + CPS - 1) / CPS;        // stages per accumulator segment
      int64_t u = 0;
      int pos = 0;
      for (int g = 0; g < nst; ++g) {
        const bool first = pos == 0;
        const bool last = (pos == spg - 1) || (g == nst - 1);
        const int sl = st_slot(g);
        if (first) RT_TIMED(tim, 2 + 4 * q, wait_acc_free<L>(b, u));
        RT_TIMED(tim, 3 + 4 * q, mbar_wait(&b.ready[sl], st_par(g)));   // A split and B landed
        RT_TRACE(p, g, 3 + 2 * q);
        tc_fence_after();
        const int c0 = g * CPS;
        const int cn = (nch - c0) < CPS ? (nch - c0) : CPS;
#pragma unroll
        for (int c = 0; c < CPS; ++c) {
          if (c < cn && p.ablate != 1)
            issue_stage<L, BSPLIT, true>(tmem, q, acc_buf<L>(u), L::a_slot(sl) + 64u * c,
                                         smem_u32(smem + L::off_b + ((c0 + c) % L::NBS) * L::kBS), idesc0, idesc1,
                                         first && c == 0);
        }
        mma_commit_w(&b.tfree[sl]);
        RT_TRACE(p, g, 4 + 2 * q);
        if (last) { mma_commit_w(&b.acc_full[acc_buf<L>(u)]); ++u; pos = 0; } else { ++pos; }
      }
    }
  } else if (warp >= 2 && warp <= 5) {                 // ---------------- splitters
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    const int t = threadIdx.x - 64;
    unsigned long long* tim = (warp == 2) ? p.tim : nullptr;   // warp-uniform (aligned tcgen05 ops inside)
    float xmax = 0.f, xsq = 0.f;
    Ring rx;
    for (int it = 0; it < nch; ++it) {
      const int g = it / CPS, c = it % CPS, sl = st_slot(g), bs = it % L::NBS;
      const int cx = XW == 1 ? 0 : it % XW;             // chunk within the X stage
      if (cx == 0) RT_TIMED(tim, 10, mbar_wait(&b.x_full[rx.s], rx.ph));
      if (c == 0 && g >= NB) RT_TIMED(tim, 11, mbar_wait(&b.tfree[sl], st_par(g) ^ 1));   // stage's TMEM slot free
      RT_TIMED(tim, 12, {
        const float* xs = reinterpret_cast<const float*>(smem + L::off_x + rx.s * L::kX);
        const uint32_t ta = lane_base + L::a_slot(sl) + 64u * c;
        if (p.ablate == 2) {
        } else if constexpr (XW > 1) {
          const float* row = xs + r * (KC * XW + 4) + KC * cx;
          if (p.amax) split_wrow_to_tmem<true>(row, ta, &xmax, &xsq);
          else split_wrow_to_tmem(row, ta);
        } else if (p.amax) {
          split_row_to_tmem<AMN, true>(xs, r, ta, &xmax, &xsq);
        } else {
          split_row_to_tmem<AMN>(xs, r, ta);
        }
      });
      if (cx == XW - 1 || it == nch - 1) { mbar_arrive(&b.x_free[rx.s]); rx.next<NX>(); }
      RT_TIMED(tim, 13, mbar_wait(&b.b_full[bs], uint32_t(it / L::NBS) & 1u));
      if (BSPLIT && !BPRE) {
        float* bsp = reinterpret_cast<float*>(smem + L::off_b + bs * L::kBS);
        split_b<L::kB>(bsp, bsp + L::kB / 4, t);
      }
      if (c == CPS - 1 || it == nch - 1) {             // stage complete
        tmem_wait_st();
        if (BSPLIT && !BPRE) fence_proxy_async();
        tc_fence_before();
        mbar_arrive(&b.ready[sl]);
      }
    }
    if (p.amax) xstat_add(p.amax, xmax, xsq);
  } else if (warp >= 8) {                              // ---------------- epilogue: drain segments
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    unsigned long long* tim = (warp == 8) ? p.tim : nullptr;
    float sums[NPAD];
#pragma unroll
    for (int k = 0; k < NPAD; ++k) sums[k] = 0.f;
    const int spg = (p.seg + CPS - 1) / CPS;
    const int64_t nseg = (nst + spg - 1) / spg;
    for (int64_t u = 0; u < nseg; ++u) RT_TIMED(tim, 14, drain_acc<L, NPAD, BSPLIT>(b, lane_base, u, sums));
    const int64_t i = i0 + r;                         // partial tile -> part[split][k][i]
    if (i < p.I) {
      float* dst = p.part + z * p.K * p.I;
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

// ================================================================ ttm_s, fp16 split
// The power product Y = X_(n) Q_z with Q_z = Z R^-1 pre-split by the zapply epilogue into fp16
// rows [Q_hi (NPAD) | Q_lo (NPAD)] of 2^14 Q_z (|Q_z| <= 1: inside the fp16 range).  X is scaled by the power of two s
// (xscale, from max|X|, so max|sX| is in [2^14, 2^15)) and split x s = x_hi + x_lo in fp16 by the
// splitters; D0 += A_hi [Q_hi | Q_lo] (issuer 0, N = 2 NPAD), D1 += A_lo Q_hi (issuer 1); the
// epilogue multiplies by 1/s.  Same 22 significant bits per operand as the 3xTF32 form; fp16 runs
// K = 16 per instruction at twice the tf32 rate, so the stage needs half the MMA instructions and
// half the tensor time, and the A slot is half as wide (32 TMEM columns per chunk).
// Q_z is stored times 2^14: its entries are <= 1 in magnitude but typically ~J^-1/2 (5e-4 at
// J = 2048^2), whose lo parts would otherwise fall into the fp16 subnormals (11 bits lost)
constexpr float kQScale = 16384.f;

template <int NPAD, int CPS_ = 2, uint32_t OUTB = 0, int XW = 1>
struct PlanH {
  static constexpr int CPS = CPS_;
  static constexpr int NH = NPAD;                        // D0 = [hi block | lo block]
  static constexpr int NBX = (2 * NPAD + 63) / 64;       // 64-wide MN atoms of the [hi | lo] B rows
  static constexpr uint32_t kB = uint32_t(NBX) * 4096u;  // 32 k-rows x 128 B per atom column
  static constexpr uint32_t kBS = kB;
  static constexpr int NI = 2;
  static constexpr int NBUF = 1;
  static constexpr uint32_t acc_cols = 3u * NPAD;
  static constexpr uint32_t a_base = (acc_cols + 63u) & ~63u;
  static constexpr int NB_fit = int((512u - a_base) / (32u * CPS));
  static constexpr int NB_smem = XW == 1 ? 6 : int((224u * 1024u - 2u * BM * x_pitch<XW>() - OUTB) / (CPS * kB));
  static constexpr int NB = NB_fit < NB_smem ? (NB_fit > 6 ? 6 : NB_fit) : (NB_smem > 6 ? 6 : NB_smem);
  static_assert(2 * NPAD <= 256 && NPAD % 16 == 0, "f16 operand shape");
  __host__ __device__ static constexpr uint32_t acc(int q, int) { return q == 0 ? 0u : uint32_t(2 * NPAD); }
  __host__ __device__ static constexpr uint32_t a_slot(int s) { return a_base + 32u * CPS * uint32_t(s); }
  static constexpr uint32_t kX = uint32_t(BM) * x_pitch<XW>();   // one X stage (XW chunks)
  static constexpr uint32_t budget = 224u * 1024u;
  static constexpr int NBS = NB * CPS;
  static constexpr int NX_fit = int((budget - NBS * kBS - OUTB) / kX);
  static constexpr int NX = NX_fit > 10 ? 10 : NX_fit;
  static constexpr uint32_t off_x = 0;
  static constexpr uint32_t off_b = off_x + NX * kX;
  static constexpr uint32_t off_o = off_b + NBS * kBS;  // output staging (ttm_t), OUTB bytes
  static constexpr uint32_t off_bar = off_o + OUTB;
  static constexpr int nbar = 2 * NX + 2 * NBS + 2 * 8 + 4;
  static constexpr uint32_t bytes = off_bar + 8 * nbar + 16;
  static_assert(kX % 1024 == 0, "X stages keep the 1 KB alignment of the swizzled B slots");
  static_assert(NB <= 8 && NBS <= 16, "barrier plan");
  static constexpr bool ok = NB >= 2 && NX >= (XW == 1 ? 4 : 2);
};

// MN-major fp16 SWIZZLE_128B operand (tools/f16_probe.cu): atoms of 8 k-rows x 128 B (64 n);
// LBO = 4 KB between 64-wide atom columns (32 k-rows each), SBO = 1 KB between 8-row k groups;
// the K = 16 step kk starts 2 KB further.
__device__ __forceinline__ uint64_t bdesc_h16(uint32_t saddr, int kk) {
  return sdesc(saddr + 2048u * uint32_t(kk), 4096u, 1024u) | (uint64_t(2) << 61);
}

// Splitter (fp16): this thread's row of the raw X tile, scaled by s, as packed fp16 hi/lo pairs
template <bool AMN>
__device__ __forceinline__ void split_row_to_tmem_h16(const float* xs, int r, float s, uint32_t t_hi) {
  float v[32];
  if (AMN) {
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = xs[q * BM + r];
  } else {
    const float* row = xs + r * KC;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 w = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 2));
      v[4 * c + 0] = w.x; v[4 * c + 1] = w.y; v[4 * c + 2] = w.z; v[4 * c + 3] = w.w;
    }
  }
  const uint64_t ss = pack_f32x2(s);
  uint32_t hi[16], lo[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) split_h16x2_s(v[2 * c], v[2 * c + 1], ss, hi[c], lo[c]);
  tmem_st16(t_hi, hi);
  tmem_st16(t_hi + 16, lo);
}

__device__ __forceinline__ void split_wrow_to_tmem_h16(const float* row, float s, uint32_t t_hi) {
  float v[32];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 w = *reinterpret_cast<const float4*>(row + 4 * c);
    v[4 * c + 0] = w.x; v[4 * c + 1] = w.y; v[4 * c + 2] = w.z; v[4 * c + 3] = w.w;
  }
  const uint64_t ss = pack_f32x2(s);
  uint32_t hi[16], lo[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) split_h16x2_s(v[2 * c], v[2 * c + 1], ss, hi[c], lo[c]);
  tmem_st16(t_hi, hi);
  tmem_st16(t_hi + 16, lo);
}

struct HParams {
  SParams s;
  const float* xscale;   // device: s (a power of two)
  float binv;            // 1 / (the B operand's power-of-two scale): 2^-14 for Q_z / Z rows, 2^-11 for Omega
};

template <int NPAD, bool AMN, int CPS_ = 2, int XW = 1>
__global__ void __launch_bounds__(NT_TTM, 1)
ttm_s_h16_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, const HParams hp) {
  static_assert(XW == 1 || !AMN, "wide X rows are for the strided modes");
  using L = PlanH<NPAD, CPS_, 0, XW>;
  static_assert(L::ok, "infeasible TMEM / shared-memory plan");
  const SParams& p = hp.s;
  if (*hp.xscale == 0.f) return;                       // dynamic range too wide: the tf32 launch runs
  if (p.runs && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&p.runs[0], 1u);
  constexpr int NX = L::NX, CPS = L::CPS, NB = L::NB;
  extern __shared__ __align__(1024) uint8_t smem[];
  const Bars b = bars_of<L>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t z = blockIdx.y, S = gridDim.y;
  const int64_t i0 = int64_t(blockIdx.x) * BM;
  const int64_t per = p.per;                           // contiguous chunks per split (host)
  (void)S;
  const int64_t cbeg = z * per;
  const int nch = cbeg < p.nchunks ? int(min(per, p.nchunks - cbeg)) : 0;
  const int nst = (nch + CPS - 1) / CPS;
  const int rot = (nch && XW == 1) ? int((int64_t(blockIdx.x) * p.skew) % nch) : 0;
  auto chunk_of = [&](int it) { int c = it + rot; return cbeg + (c >= nch ? c - nch : c); };
  auto st_slot = [](int g) { return g % NB; };
  auto st_par = [](int g) { return uint32_t(g / NB) & 1u; };

  if (threadIdx.x == 0) {
    init_bars<L>(b);
    tma_prefetch(&tmx);
    tma_prefetch(&tmb);
  }
  if (warp == 1) tmem_alloc(b.tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *b.tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                   // ---------------- X producer (one box per XW chunks)
      Ring rx;
      // wide rows: the 16 B pad sector is read again by the next stage, so X lines keep the normal
      // L2 priority there (evict_first sends the re-read to DRAM)
      const uint64_t pol = (XW > 1 && !p.xfirst) ? policy_evict_normal() : policy_evict_first();
      int xi = 0;
      for (int it = 0; it < nch; it += XW, ++xi, rx.next<NX>()) {
        if (xi >= NX) mbar_wait(&b.x_free[rx.s], rx.ph ^ 1);
        int64_t a0, beta, j0;
        chunk_coords<AMN>(p, chunk_of(it), a0, beta, j0);
        mbar_expect_tx(&b.x_full[rx.s], L::kX);
        void* xs = smem + L::off_x + rx.s * L::kX;
        if (AMN) tma_load_2d_hint(xs, &tmx, &b.x_full[rx.s], int(i0), int(j0), pol);
        else tma_load_3d_hint(xs, &tmx, &b.x_full[rx.s], int(a0), int(i0), int(beta), pol);
      }
    }
  } else if (warp == 6) {
    if (lane == 0) {                                   // ---------------- B producer (one slot per chunk)
      const uint64_t pol = policy_evict_last();
      for (int it = 0; it < nch; ++it) {
        const int g = it / CPS, bs = it % L::NBS;
        if (g >= NB) mbar_wait(&b.tfree[st_slot(g)], st_par(g) ^ 1);
        int64_t a0, beta, j0;
        chunk_coords<AMN>(p, chunk_of(it), a0, beta, j0);
        mbar_expect_tx(&b.b_full[bs], L::kB);
#pragma unroll
        for (int x = 0; x < L::NBX; ++x)
          tma_load_2d_hint(smem + L::off_b + bs * L::kBS + x * 4096, &tmb, &b.b_full[bs], 64 * x, int(j0), pol);
      }
    }
  } else if (warp == 1 || warp == 7) {
    const int q = warp == 1 ? 0 : 1;                   // ---------------- MMA issuers (whole warp)
    const uint32_t idesc = idesc_f16(BM, q == 0 ? 2 * NPAD : NPAD, 1);
    const uint32_t d = tmem + L::acc(q, 0);
    const int spg = (p.seg + CPS - 1) / CPS;
    int64_t u = 0;
    int pos = 0;
    for (int g = 0; g < nst; ++g) {
      const bool first = pos == 0;
      const bool last = (pos == spg - 1) || (g == nst - 1);
      const int sl = st_slot(g);
      if (first) wait_acc_free<L>(b, u);
      mbar_wait(&b.ready[sl], st_par(g));               // A split and B landed
      tc_fence_after();
      const int c0 = g * CPS;
      const int cn = (nch - c0) < CPS ? (nch - c0) : CPS;
#pragma unroll
      for (int c = 0; c < CPS; ++c) {
        if (c < cn) {
          const uint32_t a = tmem + L::a_slot(sl) + 32u * c + (q == 0 ? 0u : 16u);
          const uint32_t bsa = smem_u32(smem + L::off_b + ((c0 + c) % L::NBS) * L::kBS);
#pragma unroll
          for (int kk = 0; kk < KC / 16; ++kk)
            mma_f16_ts_w(d, a + 8 * kk, bdesc_h16(bsa, kk), idesc, (first && c == 0 && kk == 0) ? 0u : 1u);
        }
      }
      mma_commit_w(&b.tfree[sl]);
      if (last) { mma_commit_w(&b.acc_full[0]); ++u; pos = 0; } else { ++pos; }
    }
  } else if (warp >= 2 && warp <= 5) {                 // ---------------- splitters
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    const float sc = *hp.xscale;
    Ring rx;
    for (int it = 0; it < nch; ++it) {
      const int g = it / CPS, c = it % CPS, sl = st_slot(g), bs = it % L::NBS;
      const int cx = XW == 1 ? 0 : it % XW;             // chunk within the X stage
      if (cx == 0) mbar_wait(&b.x_full[rx.s], rx.ph);
      if (c == 0 && g >= NB) mbar_wait(&b.tfree[sl], st_par(g) ^ 1);   // stage's TMEM slot free
      const float* xs = reinterpret_cast<const float*>(smem + L::off_x + rx.s * L::kX);
      if constexpr (XW > 1)
        split_wrow_to_tmem_h16(xs + r * (KC * XW + 4) + KC * cx, sc, lane_base + L::a_slot(sl) + 32u * c);
      else
        split_row_to_tmem_h16<AMN>(xs, r, sc, lane_base + L::a_slot(sl) + 32u * c);
      if (cx == XW - 1 || it == nch - 1) { mbar_arrive(&b.x_free[rx.s]); rx.next<NX>(); }
      if (c == CPS - 1 || it == nch - 1) {             // stage complete (B landed too)
        mbar_wait(&b.b_full[bs], uint32_t(it / L::NBS) & 1u);
        if (c == 1) mbar_wait(&b.b_full[bs - 1], uint32_t((it - 1) / L::NBS) & 1u);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&b.ready[sl]);
      }
    }
  } else if (warp >= 8) {                              // ---------------- epilogue: drain segments
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    float sums[NPAD];
#pragma unroll
    for (int k = 0; k < NPAD; ++k) sums[k] = 0.f;
    const int spg = (p.seg + CPS - 1) / CPS;
    const int64_t nseg = (nst + spg - 1) / spg;
    for (int64_t u = 0; u < nseg; ++u) {
      mbar_wait(&b.acc_full[0], uint32_t(u) & 1u);
      tc_fence_after();
      add_cols<NPAD>(lane_base + L::acc(0, 0), sums);            // A_hi Q_hi
      add_cols<NPAD>(lane_base + L::acc(0, 0) + NPAD, sums);     // A_hi Q_lo
      add_cols<NPAD>(lane_base + L::acc(1, 0), sums);            // A_lo Q_hi
      tc_fence_before();
      mbar_arrive(&b.acc_empty[0]);
    }
    const float inv = hp.binv / *hp.xscale;            // exact: both scales are powers of two
    const int64_t i = i0 + r;                         // partial tile -> part[split][k][i]
    if (i < p.I) {
      float* dst = p.part + z * p.K * p.I;
#pragma unroll
      for (int k = 0; k < NPAD; ++k)
        if (k < p.K) dst[int64_t(k) * p.I + i] = sums[k] * inv;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// X statistics for the fp16 scale: stat = {max|X| as float bits (u32), pad, sum |x| (f64)}.
// s = 2^(15 - e), 2^(e-1) <= max|X| < 2^e, so max |s X| lies in [2^14, 2^15) below the fp16 maximum;
// s = 0 ("use the tf32 kernels") when max|X| > 2^16 mean|X|: the bulk of such a tensor (a few huge
// outliers) would sit so far below the scale that its fp16 lo parts turn subnormal (R29).  mean|X|
// (not the rms, which a few outliers dominate) tracks the bulk.
__global__ void __launch_bounds__(256) absmax_kernel(const float4* __restrict__ x, int64_t n4, const float* __restrict__ tail,
                                                     int ntail, unsigned int* __restrict__ stat) {
  float m = 0.f, sq = 0.f;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n4; e += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = __ldcs(x + e);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    sq += (fabsf(v.x) + fabsf(v.y)) + (fabsf(v.z) + fabsf(v.w));
  }
  if (blockIdx.x == 0 && int(threadIdx.x) < ntail) { const float v = tail[threadIdx.x]; m = fmaxf(m, fabsf(v)); sq += fabsf(v); }
  xstat_add(stat, m, sq);
}
// s[0] = the fp16-split scale (0: the tf32 twins run), s[1] = sn = 2^-e, the normalizing scale of
// the power iteration's Z = sn X^T Q (any scale spans the same space; sn keeps Z's fp32 Gram on the
// tensor cores clear of underflow / overflow at any data scale).  stat: max |X| (double), sum |x|
// over n elements (all ranks).
__device__ void xscale_of(double m, double sum_abs, double n, float* __restrict__ s, int force_zero) {
  const double mean_abs = sum_abs / n;
  float r = 1.f, sn = 1.f;
  if (m > 0.0 && isfinite(m)) {
    int e;
    frexp(m, &e);                                       // m = f 2^e, f in [0.5, 1): floor(log2 m) = e - 1
    // s 2^14 (the epilogue divides by it) must stay a finite fp32 power of two: s <= 2^113, i.e.
    // max|X| >= 2^-98; tinier data take the tf32 kernels
    r = (15 - e > 113) ? 0.f : ldexpf(1.f, 15 - e);
    if (m > 65536.0 * mean_abs) r = 0.f;               // too wide a dynamic range: tf32 kernels
    sn = ldexpf(1.f, max(-120, min(120, -e)));
  }
  s[0] = force_zero ? 0.f : r;                          // tests: the tf32 twins take over
  s[1] = sn;
}
__global__ void xscale_kernel(const unsigned int* __restrict__ stat, double n, float* __restrict__ s, int force_zero) {
  xscale_of(double(__uint_as_float(stat[0])), *reinterpret_cast<const double*>(stat + 2), n, s, force_zero);
}
// distributed: stats of every rank gathered as (max, sum) double pairs
__global__ void stat_pair_kernel(const unsigned int* __restrict__ stat, double* __restrict__ pair) {
  pair[0] = double(__uint_as_float(stat[0]));
  pair[1] = *reinterpret_cast<const double*>(stat + 2);
}
__global__ void xscale_gathered_kernel(const double* __restrict__ pairs, int nranks, double n, float* __restrict__ s,
                                       int force_zero) {
  double m = 0.0, sum = 0.0;
  for (int r = 0; r < nranks; ++r) { m = fmax(m, pairs[2 * r]); sum += pairs[2 * r + 1]; }
  xscale_of(m, sum, n, s, force_zero);
}

// ====================================================================== ttm_t
struct TParams {
  int64_t a, I, b;
  int C;
  int64_t tpb;        // tiles per beta (a > 1)
  int64_t ntiles;
  int nic;            // i-chunks per tile
  int seg;            // i-chunks per accumulator segment
  float* out;
  int64_t so_a, so_c, so_b;
  bool vec4;          // so_c == 1 and every output row 16-byte aligned with C % 4 == 0
  int split_out;      // 1: each output row as [hi (NHO) | lo (NHO)] tf32 halves (vec4 layout);
                      // 2: as fp16 [hi (NPAD) | lo (NPAD)] (out points to halves, so_* count halves)
  bool tma_out;       // output tiles staged in shared memory and written by TMA stores (tmo)
  const float* xscale;   // H16 kernels: device scale s of X (the output is divided by s 2^14)
  const float* gate;     // tf32 kernels: run only if *gate == 0 (fallback of an fp16-split launch)
  unsigned int* runs;    // optional run counters (see SParams)
  const float* oscale;   // optional device scale of the output (the power iteration's Z = sn X^T Q)
  float omul;            // host power-of-two factor of the output (1 = none)
  int nch = 1;           // column chunks of cw <= NPAD columns (C = the total width); chunk ch's
  int cw = 0;            //   pre-split B rows start at row 2 NPAD ch of the B map
};

// AKM: mode 0 (a == 1), X tile K-major [BM j][KC i].  BSPLIT: Q = Q_hi + Q_lo pre-split (an fp64
// basis is never tf32-exact); !BSPLIT: Q is tf32-exact (a host-rounded test matrix, R18), 2 products.
// Output rows (so_c == 1) are staged in shared memory as 128 B-swizzled [128 rows][32 cols] boxes
// and written by TMA stores (tmo): one contiguous tile per store instead of 16-byte row pieces.
template <int NPAD>
constexpr uint32_t t_outb() { return uint32_t(BM) * ((NPAD + 31) / 32) * 128u; }

// H16: the fp16 split (see ttm_s_h16_kernel): B = [2^14 Q_hi | 2^14 Q_lo] fp16 rows (row-major
// I x 2 NPAD, MN-major atoms), X scaled by s and split by the splitters, 2 K = 16 steps per chunk.
template <int NPAD, bool AKM, bool BSPLIT, bool H16 = false>
__global__ void __launch_bounds__(NT_TTM, 1)
ttm_t_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
                const __grid_constant__ CUtensorMap tmo, const TParams p) {
  static_assert(!H16 || BSPLIT, "the fp16 form always carries Q_lo");
  if (H16 ? (*p.xscale == 0.f) : (p.gate != nullptr && *p.gate != 0.f)) return;   // one of the pair runs (R29)
  if ((H16 || p.gate != nullptr) && p.runs && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&p.runs[H16 ? 0 : 1], 1u);
  using L = std::conditional_t<H16, PlanH<NPAD, 1, t_outb<NPAD>()>, Plan<NPAD, BSPLIT, false, 1, t_outb<NPAD>()>>;
  static_assert(L::ok, "infeasible TMEM / shared-memory plan");
  constexpr int NX = L::NX;
  extern __shared__ __align__(1024) uint8_t smem[];
  const Bars b = bars_of<L>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // work items: (column chunk, row tile) pairs, chunk-major (p.nch > 1: columns wider than one TMEM
  // tile, every chunk re-reading the small source from L2)
  const int64_t nitems = p.ntiles * p.nch;
  const int64_t my_tiles = (nitems > blockIdx.x) ? (nitems - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (threadIdx.x == 0) {
    init_bars<L>(b);
    tma_prefetch(&tmx);
    tma_prefetch(&tmb);
  }
  if (warp == 1) tmem_alloc(b.tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *b.tmem_slot;

  auto tile_coords = [&](int64_t tile, int64_t& a0, int64_t& beta) {
    if (AKM) { a0 = 0; beta = tile * BM; }
    else { beta = tile / p.tpb; a0 = (tile % p.tpb) * BM; }
  };

  if (warp == 0) {
    if (lane == 0) {                                   // ---------------- X producer
      Ring rx;
      const uint64_t pol = policy_evict_first();
      int it = 0;
      for (int64_t u = 0; u < my_tiles; ++u) {
        int64_t a0, beta;
        tile_coords((blockIdx.x + u * gridDim.x) % p.ntiles, a0, beta);
        for (int c = 0; c < p.nic; ++c, ++it, rx.next<NX>()) {
          if (it >= NX) mbar_wait(&b.x_free[rx.s], rx.ph ^ 1);
          mbar_expect_tx(&b.x_full[rx.s], L::kX);
          void* xs = smem + L::off_x + rx.s * L::kX;
          if (AKM) tma_load_2d_hint(xs, &tmx, &b.x_full[rx.s], c * KC, int(beta), pol);
          else tma_load_3d_hint(xs, &tmx, &b.x_full[rx.s], int(a0), c * KC, int(beta), pol);
        }
      }
    }
  } else if (warp == 6) {
    if (lane == 0) {                                   // ---------------- B producer ([Q_hi | Q_lo])
      Ring rb;
      const uint64_t pol = policy_evict_last();
      int it = 0;
      for (int64_t u = 0; u < my_tiles; ++u) {
        const int chunk = int((blockIdx.x + u * gridDim.x) / p.ntiles);
        for (int c = 0; c < p.nic; ++c, ++it, rb.next<L::NBS>()) {
          if (it >= L::NBS) mbar_wait(&b.b_free[rb.s], rb.ph ^ 1);
          mbar_expect_tx(&b.b_full[rb.s], L::kBS);
          if constexpr (H16) {
#pragma unroll
            for (int x = 0; x < L::NBX; ++x)
              tma_load_2d_hint(smem + L::off_b + rb.s * L::kBS + x * 4096, &tmb, &b.b_full[rb.s], 64 * x, c * KC, pol);
          } else {
            tma_load_2d_hint(smem + L::off_b + rb.s * L::kBS, &tmb, &b.b_full[rb.s], c * KC, chunk * 2 * NPAD, pol);
          }
        }
      }
    }
  } else if (warp == 1 || warp == 7) {
    const int q = warp == 1 ? 0 : 1;
    if (q < L::NI) {                                   // ---------------- MMA issuers (whole warp)
      const uint32_t idesc0 = H16 ? idesc_f16(BM, 2 * NPAD, 1) : idesc_tf32(BM, BSPLIT ? L::NH + NPAD : NPAD, 0);
      const uint32_t idesc1 = H16 ? idesc_f16(BM, NPAD, 1) : idesc_tf32(BM, NPAD, 0);
      Ring rt, rb;
      int64_t g = 0;                                   // global segment counter
      for (int64_t u = 0; u < my_tiles; ++u) {
        int pos = 0;
        for (int c = 0; c < p.nic; ++c, rt.next<L::NB>(), rb.next<L::NBS>()) {
          const bool first = pos == 0;
          const bool last = (pos == p.seg - 1) || (c == p.nic - 1);
          if (first) wait_acc_free<L>(b, g);
          mbar_wait(&b.ready[rt.s], rt.ph);                // A split and B landed
          tc_fence_after();
          if constexpr (H16) {
            const uint32_t d = tmem + L::acc(q, 0);
            const uint32_t a = tmem + L::a_slot(rt.s) + (q == 0 ? 0u : 16u);
            const uint32_t bsa = smem_u32(smem + L::off_b + rb.s * L::kBS);
#pragma unroll
            for (int kk = 0; kk < KC / 16; ++kk)
              mma_f16_ts_w(d, a + 8 * kk, bdesc_h16(bsa, kk), q == 0 ? idesc0 : idesc1, (first && kk == 0) ? 0u : 1u);
          } else {
            issue_stage<L, BSPLIT, false>(tmem, q, acc_buf<L>(g), L::a_slot(rt.s),
                                          smem_u32(smem + L::off_b + rb.s * L::kBS), idesc0, idesc1, first);
          }
          mma_commit_w(&b.tfree[rt.s]);
          if (last) { mma_commit_w(&b.acc_full[acc_buf<L>(g)]); ++g; pos = 0; } else { ++pos; }
        }
      }
    }
  } else if (warp >= 2 && warp <= 5) {                 // ---------------- splitters
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    Ring rx, rt;
    int it = 0;
    const float sc = H16 ? *p.xscale : 1.f;
    for (int64_t u = 0; u < my_tiles; ++u) {
      for (int c = 0; c < p.nic; ++c, ++it, rx.next<NX>(), rt.next<L::NB>()) {
        mbar_wait(&b.x_full[rx.s], rx.ph);
        if (it >= L::NB) mbar_wait(&b.tfree[rt.s], rt.ph ^ 1);
        if constexpr (H16)
          split_row_to_tmem_h16<!AKM>(reinterpret_cast<const float*>(smem + L::off_x + rx.s * L::kX), r, sc,
                                      lane_base + L::a_slot(rt.s));
        else
          split_row_to_tmem<!AKM>(reinterpret_cast<const float*>(smem + L::off_x + rx.s * L::kX), r,
                                  lane_base + L::a_slot(rt.s));
        mbar_arrive(&b.x_free[rx.s]);
        mbar_wait(&b.b_full[rt.s], rt.ph);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&b.ready[rt.s]);
      }
    }
  } else if (warp >= 8) {                              // ---------------- epilogue: drain, store tiles
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    float sums[NPAD];
#pragma unroll
    for (int k = 0; k < NPAD; ++k) sums[k] = 0.f;
    const int segs_per_tile = (p.nic + p.seg - 1) / p.seg;
    // exact: powers of two (the H16 unscaling and the optional output scale)
    const float inv = (H16 ? 1.0f / (*p.xscale * kQScale) : 1.f) * (p.oscale ? *p.oscale : 1.f) * p.omul;
    const bool rescale = H16 || p.oscale != nullptr || p.omul != 1.f;
    int64_t g = 0;
    for (int64_t u = 0; u < my_tiles; ++u) {
      const int64_t item = blockIdx.x + u * gridDim.x;
      const int64_t tile = item % p.ntiles;
      const int cc0 = int(item / p.ntiles) * p.cw;                 // this chunk's first output column
      const int Cc = min(p.C - cc0, p.cw);                         // and its width
      for (int sgi = 0; sgi < segs_per_tile; ++sgi, ++g) {
        if constexpr (H16) {
          mbar_wait(&b.acc_full[0], uint32_t(g) & 1u);
          tc_fence_after();
          add_cols<NPAD>(lane_base + L::acc(0, 0), sums);            // A_hi Q_hi
          add_cols<NPAD>(lane_base + L::acc(0, 0) + NPAD, sums);     // A_hi Q_lo
          add_cols<NPAD>(lane_base + L::acc(1, 0), sums);            // A_lo Q_hi
          tc_fence_before();
          mbar_arrive(&b.acc_empty[0]);
        } else {
          drain_acc<L, NPAD, BSPLIT>(b, lane_base, g, sums);
        }
      }
      if (rescale) {
#pragma unroll
        for (int k = 0; k < NPAD; ++k) sums[k] *= inv;
      }
      int64_t a0, beta;
      tile_coords(tile, a0, beta);
      bool valid;
      int64_t ob;
      if (AKM) { const int64_t j = beta + r; valid = j < p.b; ob = j * p.so_b; }
      else { const int64_t al = a0 + r; valid = al < p.a; ob = al * p.so_a + beta * p.so_b; }
      ob += int64_t(cc0) * p.so_c;
      if (p.tma_out) {
        constexpr int NBX = (NPAD + 31) / 32;
        uint8_t* stage = smem + L::off_o;
        if (u > 0 && r == 0) bulk_wait_read0();              // the previous tile's stores have read it
        named_bar(1, 128);
        if (p.split_out == 2) {
          // fp16 [2^14 hi | 2^14 lo] rows (2 NPAD halves = the same bytes as NPAD floats): half e of
          // the row in box e / 64, 16-byte chunk (e % 64) / 8
#pragma unroll
          for (int k = 0; k < NPAD / 8; ++k) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c0 = 8 * k + 2 * e, c1 = c0 + 1;
              split_h16x2(c0 < Cc ? sums[c0] * kQScale : 0.f, c1 < Cc ? sums[c1] * kQScale : 0.f, h[e], l[e]);
            }
            const int eh = 8 * k, el = NPAD + 8 * k;
            *reinterpret_cast<uint4*>(stage + (eh >> 6) * (BM * 128) + r * 128 + ((((eh & 63) >> 3) ^ (r & 7)) << 4)) =
                make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(stage + (el >> 6) * (BM * 128) + r * 128 + ((((el & 63) >> 3) ^ (r & 7)) << 4)) =
                make_uint4(l[0], l[1], l[2], l[3]);
          }
        } else {
#pragma unroll
          for (int bx = 0; bx < NBX; ++bx)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int c = 32 * bx + 4 * q;
              const float4 v = make_float4(c < NPAD ? sums[c % NPAD] : 0.f, c + 1 < NPAD ? sums[(c + 1) % NPAD] : 0.f,
                                           c + 2 < NPAD ? sums[(c + 2) % NPAD] : 0.f,
                                           c + 3 < NPAD ? sums[(c + 3) % NPAD] : 0.f);
              *reinterpret_cast<float4*>(stage + bx * (BM * 128) + r * 128 + ((q ^ (r & 7)) << 4)) = v;
            }
        }
        fence_proxy_async();
        named_bar(1, 128);
        if (r == 0) {
          const int row0 = AKM ? int(beta) : int(a0 + p.a * beta);
#pragma unroll
          for (int bx = 0; bx < NBX; ++bx) {
            if (p.split_out == 2) {
              if (64 * bx < 2 * NPAD) tma_store_2d(&tmo, stage + bx * (BM * 128), 64 * bx, row0);
            } else if (32 * bx < Cc) {
              tma_store_2d(&tmo, stage + bx * (BM * 128), cc0 + 32 * bx, row0);
            }
          }
          bulk_commit();
        }
      } else if (valid) {
        if (p.split_out == 2) {                              // fp16 [hi | lo] rows (ttm_s_h16_kernel B)
          uint4* oh = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.out) + ob);
          uint4* ol = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(p.out) + ob + NPAD);
#pragma unroll
          for (int k = 0; k < NPAD / 8; ++k) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c0 = 8 * k + 2 * e, c1 = c0 + 1;
              split_h16x2(c0 < Cc ? sums[c0] * kQScale : 0.f, c1 < Cc ? sums[c1] * kQScale : 0.f, h[e], l[e]);
            }
            oh[k] = make_uint4(h[0], h[1], h[2], h[3]);
            ol[k] = make_uint4(l[0], l[1], l[2], l[3]);
          }
        } else if (p.split_out) {                            // [hi | lo] rows for a pre-split B operand
          constexpr int NHO = ((NPAD + 31) / 32) * 32;
          float4* oh = reinterpret_cast<float4*>(p.out + ob);
          float4* ol = reinterpret_cast<float4*>(p.out + ob + NHO);
#pragma unroll
          for (int k = 0; k < NHO / 4; ++k) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) split_tf32((4 * k + e < NPAD && 4 * k + e < Cc) ? sums[(4 * k + e) % NPAD] : 0.f,
                                                   h[e], l[e]);
            oh[k] = make_float4(__uint_as_float(h[0]), __uint_as_float(h[1]), __uint_as_float(h[2]), __uint_as_float(h[3]));
            ol[k] = make_float4(__uint_as_float(l[0]), __uint_as_float(l[1]), __uint_as_float(l[2]), __uint_as_float(l[3]));
          }
        } else if (p.vec4) {                                 // row-major output rows: 16 B stores
          float4* o4 = reinterpret_cast<float4*>(p.out + ob);
#pragma unroll
          for (int k = 0; k < NPAD / 4; ++k)
            if (4 * k < Cc) o4[k] = make_float4(sums[4 * k], sums[4 * k + 1], sums[4 * k + 2], sums[4 * k + 3]);
        } else {
#pragma unroll
          for (int k = 0; k < NPAD; ++k)
            if (k < Cc) p.out[ob + int64_t(k) * p.so_c] = sums[k];
        }
      }
#pragma unroll
      for (int k = 0; k < NPAD; ++k) sums[k] = 0.f;
    }
    if (p.tma_out && r == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ================================================= fused mode-1 sketch + mode-0 core stage (fp16)
// One pass over X feeds two contractions that read the same A tile.  In the mode-1 view
// [a = I_0, I = I_1, b = the later modes] a chunk is X(alpha0..alpha0+31, i1 tile, beta):
//   the Omega sketch of mode 1:  Y_1(i1, k)       += sum_alpha X(alpha, i1, beta) Omega_1(alpha + a beta, k)
//   the first core stage:        G1(c, i1, beta)  += sum_alpha X(alpha, i1, beta) Q~_0(alpha, c)
// (the core contracts mode 0 first, Eq. Core; the sketch is Alg.6 line 3 P:556 for n = 1).
// X is split once per chunk into fp16 hi/lo A operands in TMEM (R29); B is one K-major 128 B-swizzled
// slot per chunk pair holding [2^14 Q_hi^T | 2^11 Omega^T | 2^14 Q_lo^T] (3 NPAD rows x 64 K):
//   issuer 0: A_hi [Q_hi | Omega] -> TMEM [C0 | S0]                       (N = 2 NPAD)
//   issuer 1: A_lo [Q_hi | Omega] -> TMEM [C1 | S1], then A_hi Q_lo -> C1  (N = 2 NPAD, NPAD)
// (the two corrections of the core share C1: 4 NPAD accumulator columns leave room for 4 A slots)
// with Omega tf32-exact (RT_OPT_OMEGA_TF32: exact in fp16 at 2^11, no Omega_lo).  The sketch sums S0 + S1
// over the whole chunk range of the CTA (split-K partials, as ttm_s); the core rows C0 + C1
// are complete after the cpb chunks of one beta and leave through TMA stores.
struct FParams {
  int64_t a, I, b;
  int K, C;            // sketch width (mode 1), core width (mode 0)
  int64_t cpb;         // chunks per beta (a / 32)
  int64_t nchunks, per;
  int seg;             // chunks per accumulator segment (divides cpb)
  float* part;         // [split][K][I] sketch partials
  const float* xscale; // device s (0: the tf32 twins run)
  float binv_s, binv_c;
  unsigned int* runs;
  int zout;              // 1: the left output is a power-iteration Z in the R31 form (s_z-scaled fp16 [hi | lo]
                         //    rows of 2 NPAD halves), 0: fp32 core rows of C floats
  int view_last;         // 1: X viewed for the last mode (rows i_{N-1}, beta = the middle modes): output
                         //    row j = beta + b i (3-D stores); 0: mode-1 view, row j = i + I beta
  const float* oscale;   // zout: device scale of Z (sn, R31)
  float omul;            // zout: host power of two of Z (2^-(ceil(log2 sqrt I_0) + 1))
  void* out;             // the left output rows (fp32 core rows or fp16 Z rows)
  int64_t ldo;           // row pitch in elements (C floats / 2 NPAD halves)
  int ablate;            // profiling only: 1 = no MMA, 2 = no split work (results invalid)
};

template <int NPAD, int NBB_ = 2>
struct PlanF {
  // TMEM: [C0 | S0] (issuer 0: A_hi [Q_hi | Omega]) and [C1 | S1] (issuer 1: A_lo [Q_hi | Omega], then
  // A_hi Q_lo into C1), then NB A slots of 32 columns (hi 16 | lo 16)
  static constexpr int XW = 2, NB = 4, NBB = NBB_;
  static constexpr uint32_t c0 = 0, s0 = NPAD, c1 = 2 * NPAD, s1 = 3 * NPAD;
  static constexpr uint32_t a_base = (4u * NPAD + 31u) & ~31u;
  static_assert(a_base + 32u * NB <= 512u, "fused TMEM plan");
  __host__ __device__ static constexpr uint32_t a_slot(int s) { return a_base + 32u * uint32_t(s); }
  static constexpr uint32_t kX = uint32_t(BM) * x_pitch<XW>();
  static constexpr uint32_t kB = 3u * NPAD * 128u;                   // one chunk pair: 64 K x 3 NPAD rows
  static constexpr uint32_t kO = 0;         // the left output leaves from registers (no staging)
  static constexpr uint32_t budget = 224u * 1024u;
  static constexpr int NX_fit = int((budget - NBB * kB - kO) / kX);
  static constexpr int NX = NX_fit > 4 ? 4 : NX_fit;
  static constexpr uint32_t off_x = 0, off_b = off_x + NX * kX, off_o = off_b + NBB * kB, off_bar = off_o + kO;
  static constexpr int nbar = 2 * NX + 2 * NBB + 2 * NB + 4;
  static constexpr uint32_t bytes = off_bar + 8 * nbar + 16;
  static_assert(NX >= 2 && kB % 1024 == 0 && kX % 1024 == 0, "fused smem plan");
};

constexpr int NT_FUSED = 512;   // the 12 warps of the TTM kernels + a second epilogue group (warps 12-15)

template <int NPAD, int NBB_ = 2>
__global__ void __launch_bounds__(NT_FUSED, 1)
sketch1_core0_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmq,
                     const __grid_constant__ CUtensorMap tmw, const FParams p) {
  using L = PlanF<NPAD, NBB_>;
  constexpr int NX = L::NX, NB = L::NB, NBB = L::NBB, XW = L::XW;
  if (*p.xscale == 0.f) return;                        // the tf32 twins run instead (R29)
  if (p.runs && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&p.runs[0], 1u);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::off_bar);
  uint64_t* x_full = bar;
  uint64_t* x_free = bar + NX;
  uint64_t* b_full = bar + 2 * NX;
  uint64_t* b_free = bar + 2 * NX + NBB;
  uint64_t* ready = bar + 2 * NX + 2 * NBB;
  uint64_t* tfree = ready + NB;
  uint64_t* acc_full = tfree + NB;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + L::nbar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t z = blockIdx.y;
  const int64_t i0 = int64_t(blockIdx.x) * BM;
  const int64_t cbeg = z * p.per;
  const int nch = cbeg < p.nchunks ? int(min(p.per, p.nchunks - cbeg)) : 0;   // a multiple of cpb
  auto coords = [&](int it, int64_t& a0, int64_t& beta) {
    const int64_t c = cbeg + it;
    beta = c / p.cpb;
    a0 = (c % p.cpb) * KC;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NX; ++s) { mbar_init(&x_full[s], 1); mbar_init(&x_free[s], 128); }
    for (int s = 0; s < NBB; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_free[s], 2); }
    for (int s = 0; s < NB; ++s) { mbar_init(&ready[s], 128); mbar_init(&tfree[s], 2); }
    mbar_init(acc_full, 2);
    mbar_init(acc_empty, 256);                        // both epilogue groups
    fence_barrier_init();
    tma_prefetch(&tmx); tma_prefetch(&tmq); tma_prefetch(&tmw);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                   // ---------------- X producer (XW chunks per box)
      Ring rx;
      const uint64_t pol = policy_evict_normal();
      int xi = 0;
      for (int it = 0; it < nch; it += XW, ++xi, rx.next<NX>()) {
        if (xi >= NX) mbar_wait(&x_free[rx.s], rx.ph ^ 1);
        int64_t a0, beta;
        coords(it, a0, beta);
        mbar_expect_tx(&x_full[rx.s], L::kX);
        tma_load_3d_hint(smem + L::off_x + rx.s * L::kX, &tmx, &x_full[rx.s], int(a0), int(i0), int(beta), pol);
      }
    }
  } else if (warp == 6) {
    if (lane == 0) {                                   // ---------------- B producer (one slot per chunk pair)
      Ring rb;
      const uint64_t pol = policy_evict_last();
      int bi = 0;
      for (int it = 0; it < nch; it += 2, ++bi, rb.next<NBB>()) {
        if (bi >= NBB) mbar_wait(&b_free[rb.s], rb.ph ^ 1);
        int64_t a0, beta;
        coords(it, a0, beta);
        uint8_t* dst = smem + L::off_b + rb.s * L::kB;
        mbar_expect_tx(&b_full[rb.s], L::kB);
        tma_load_2d_hint(dst, &tmq, &b_full[rb.s], int(a0), 0, pol);                              // 2^14 Q_hi^T
        tma_load_3d_hint(dst + NPAD * 128, &tmw, &b_full[rb.s], 0, 0, int((a0 + p.a * beta) / 64), pol);   // 2^11 Omega^T
        tma_load_2d_hint(dst + 2 * NPAD * 128, &tmq, &b_full[rb.s], int(a0), NPAD, pol);          // 2^14 Q_lo^T
      }
    }
  } else if (warp == 1 || warp == 7) {
    const int q = warp == 1 ? 0 : 1;                   // ---------------- MMA issuers (whole warp)
    const uint32_t idesc = idesc_f16(BM, 2 * NPAD, 0);
    const uint32_t idesc_c = idesc_f16(BM, NPAD, 0);
    const uint32_t d = tmem + (q == 0 ? L::c0 : L::c1);
    int64_t u = 0;
    int pos = 0;
    for (int it = 0; it < nch; ++it) {
      const bool first = pos == 0;
      const bool last = (pos == p.seg - 1) || (it == nch - 1);
      const int sl = it % NB;
      if (first && u >= 1) mbar_wait(acc_empty, uint32_t(u - 1) & 1u);
      mbar_wait(&ready[sl], uint32_t(it / NB) & 1u);   // A split, B pair landed
      tc_fence_after();
      const uint32_t bsa = smem_u32(smem + L::off_b + ((it / 2) % NBB) * L::kB);
      const uint32_t a = tmem + L::a_slot(sl) + (q == 0 ? 0u : 16u);
#pragma unroll
      for (int kk = 0; kk < KC / 16; ++kk) {
        if (p.ablate == 1) break;
        mma_f16_ts_w(d, a + 8 * kk, bdesc_sw128(bsa, 2 * (it & 1) + kk), idesc, (first && kk == 0) ? 0u : 1u);
        if (q == 1)                                    // A_hi Q_lo (B rows 2 NPAD..) into C1, after A_lo Q_hi
          mma_f16_ts_w(tmem + L::c1, tmem + L::a_slot(sl) + 8 * kk,
                       bdesc_sw128(bsa + 2u * NPAD * 128u, 2 * (it & 1) + kk), idesc_c, 1u);
      }
      mma_commit_w(&tfree[sl]);
      if (it & 1) mma_commit_w(&b_free[(it / 2) % NBB]);
      if (last) { mma_commit_w(acc_full); ++u; pos = 0; } else { ++pos; }
    }
  } else if (warp >= 2 && warp <= 5) {                 // ---------------- splitters
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    const float sc = *p.xscale;
    Ring rx;
    for (int it = 0; it < nch; ++it) {
      const int sl = it % NB, cx = it % XW;
      if (cx == 0) mbar_wait(&x_full[rx.s], rx.ph);
      if (it >= NB) mbar_wait(&tfree[sl], (uint32_t(it / NB) & 1u) ^ 1u);   // the A slot's MMAs done
      const float* xs = reinterpret_cast<const float*>(smem + L::off_x + rx.s * L::kX);
      if (p.ablate != 2) split_wrow_to_tmem_h16(xs + r * (KC * XW + 4) + KC * cx, sc, lane_base + L::a_slot(sl));
      if (cx == XW - 1 || it == nch - 1) { mbar_arrive(&x_free[rx.s]); rx.next<NX>(); }
      mbar_wait(&b_full[(it / 2) % NBB], uint32_t((it / 2) / NBB) & 1u);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ready[sl]);
    }
  } else if (warp >= 8 && warp < 12) {                 // ---------------- epilogue S: sketch sums
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    float sums[NPAD];
#pragma unroll
    for (int k = 0; k < NPAD; ++k) sums[k] = 0.f;
    const int nseg = nch / p.seg;
    for (int u = 0; u < nseg; ++u) {
      mbar_wait(acc_full, uint32_t(u) & 1u);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < NPAD; c0 += 16) {
        uint32_t v0[16], v1[16];
        tmem_ld16(lane_base + L::s0 + c0, v0);          // A_hi Omega
        tmem_ld16(lane_base + L::s1 + c0, v1);          // A_lo Omega
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) sums[c0 + k] += __uint_as_float(v0[k]) + __uint_as_float(v1[k]);
      }
      tc_fence_before();
      mbar_arrive(acc_empty);
    }
    const float inv_s = p.binv_s / *p.xscale;           // exact: powers of two
    const int64_t i = i0 + r;
    if (i < p.I) {
      float* dst = p.part + z * p.K * p.I;
#pragma unroll
      for (int k = 0; k < NPAD; ++k)
        if (k < p.K) dst[int64_t(k) * p.I + i] = sums[k] * inv_s;
    }
  } else if (warp >= 12) {                             // ---------------- epilogue C: the left output rows
    // C0 + C1 of each segment are read out of TMEM 16 columns at a time into the row's fp32
    // sums (registers, one row per thread), the accumulator is released, and after the cpb chunks of a
    // beta the finished row leaves straight from the registers (no shared-memory staging: the X ring
    // gets that space)
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    const float inv_c = p.binv_c / *p.xscale;           // exact: powers of two
    const float zmul = p.zout ? inv_c * *p.oscale * p.omul * kQScale : 0.f;   // R31: s_z Z, then x 2^14
    const int spb = int(p.cpb / p.seg);                 // segments per beta
    const int nseg = nch / p.seg;
    float cs[NPAD];
    for (int u = 0; u < nseg; ++u) {
      const int ub = u % spb;
      if (ub == 0) {
#pragma unroll
        for (int c = 0; c < NPAD; ++c) cs[c] = 0.f;
      }
      mbar_wait(acc_full, uint32_t(u) & 1u);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < NPAD; c0 += 16) {
        uint32_t v0[16], v1[16];
        tmem_ld16(lane_base + L::c0 + c0, v0);
        tmem_ld16(lane_base + L::c1 + c0, v1);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) cs[c0 + k] += __uint_as_float(v0[k]) + __uint_as_float(v1[k]);
      }
      tc_fence_before();
      mbar_arrive(acc_empty);
      if (ub == spb - 1) {                             // beta complete: this thread's row of the output
        int64_t a0, beta;
        coords(u * p.seg, a0, beta);
        const int64_t row = p.view_last ? beta + p.b * (i0 + r) : i0 + r + p.I * beta;
        if (p.zout) {
          // fp16 [2^14 hi | 2^14 lo] row of 2 NPAD halves (columns >= C zero)
          uint4* oh = reinterpret_cast<uint4*>(static_cast<__half*>(p.out) + row * p.ldo);
          uint4* ol = reinterpret_cast<uint4*>(static_cast<__half*>(p.out) + row * p.ldo + NPAD);
#pragma unroll
          for (int k = 0; k < NPAD / 8; ++k) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c0 = 8 * k + 2 * e, c1 = c0 + 1;
              split_h16x2(c0 < p.C ? cs[c0] * zmul : 0.f, c1 < p.C ? cs[c1] * zmul : 0.f, h[e], l[e]);
            }
            oh[k] = make_uint4(h[0], h[1], h[2], h[3]);
            ol[k] = make_uint4(l[0], l[1], l[2], l[3]);
          }
        } else {
          float4* o4 = reinterpret_cast<float4*>(static_cast<float*>(p.out) + row * p.ldo);
#pragma unroll
          for (int k = 0; k < NPAD / 4; ++k)
            if (4 * k < p.C)
              o4[k] = make_float4(cs[4 * k] * inv_c, cs[4 * k + 1] * inv_c, cs[4 * k + 2] * inv_c, cs[4 * k + 3] * inv_c);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// Q (I x C fp32, col-major ldq) -> QT (fp16, 2 NPAD rows x ldt): rows c < C = 2^14 Q_hi[:, c]^T,
// rows NPAD + c = 2^14 Q_lo[:, c]^T, other rows zero
__global__ void qt16_kernel(const float* __restrict__ Q, int64_t I, int C, int64_t ldq, int npad,
                            __half* __restrict__ QT, int64_t ldt) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ldt * npad) return;
  const int64_t i = e % ldt;
  const int c = int(e / ldt);
  const float v = (i < I && c < C) ? Q[i + ldq * c] * 16384.f : 0.f;
  const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  QT[int64_t(c) * ldt + i] = __float2half_rn(h);
  QT[int64_t(npad + c) * ldt + i] = __float2half_rn(v - h);
}

// Omega (J x K fp32, row-major ld) -> WT (fp16) in 64-column blocks: WT[jb][k][jl] = 2^11 Omega[64 jb + jl][k]
// (rows k >= K zero), so the B box of a chunk pair (NPAD rows x 64 j) is one contiguous 128 NPAD-byte
// run.  *flag = 1 if an entry is not exactly an fp16 at 2^11 (not tf32-exact, or out of range): the
// fused kernel then stands down for its twins.  64 j-rows per block through shared memory.
__global__ void __launch_bounds__(256) omega_t16_kernel(const float* __restrict__ Om, int64_t J, int K, int64_t ld,
                                                        int npad, __half* __restrict__ WT, int64_t ldw,
                                                        int* __restrict__ flag) {
  __shared__ float t[64][129];
  const int64_t j0 = int64_t(blockIdx.x) * 64;
  bool bad = false;
  for (int e = threadIdx.x; e < 16 * npad; e += blockDim.x) {        // float4 per thread
    const int jl = e / (npad / 4), k4 = 4 * (e % (npad / 4));
    const int64_t j = j0 + jl;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < J) {
      if (k4 + 4 <= K) v = __ldcs(reinterpret_cast<const float4*>(Om + j * ld + k4));
      else {
        if (k4 + 0 < K) v.x = Om[j * ld + k4 + 0];
        if (k4 + 1 < K) v.y = Om[j * ld + k4 + 1];
        if (k4 + 2 < K) v.z = Om[j * ld + k4 + 2];
      }
    }
    t[jl][k4] = v.x; t[jl][k4 + 1] = v.y; t[jl][k4 + 2] = v.z; t[jl][k4 + 3] = v.w;
  }
  __syncthreads();
  // 8 consecutive j of one row k per thread: one 16-byte store (ldw and j0 are multiples of 8)
  for (int e = threadIdx.x; e < 8 * npad; e += blockDim.x) {
    const int k = e / 8, jl0 = 8 * (e % 8);

    __align__(16) __half hv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float v = t[jl0 + q][k] * 2048.f;
      hv[q] = __float2half_rn(v);
      // an entry in the fp16 normal range must be exact (a tf32-rounded Omega is); entries below it
      // round with an absolute error <= 2^-25 (2^-36 of |Omega|): immaterial next to fp32
      bad |= !(fabsf(v) < 32768.f) || (fabsf(v) >= 6.103515625e-05f && __half2float(hv[q]) != v);
    }
    *reinterpret_cast<uint4*>(WT + (j0 / 64) * (int64_t(npad) * 64) + int64_t(k) * 64 + jl0) =
        *reinterpret_cast<const uint4*>(hv);
  }
  if (bad) atomicOr(flag, 1);
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
              const uint32_t* box, bool swz128, CUtensorMapSwizzle swz_override = CU_TENSOR_MAP_SWIZZLE_NONE,
              CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = 1; }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  std::memset(m, 0, sizeof(*m));
  CUresult r = fn(m, dt, cuuint32_t(rank), const_cast<void*>(ptr), d, s, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz_override != CU_TENSOR_MAP_SWIZZLE_NONE ? swz_override
                                                             : (swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE),
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// column-major fp32 matrix (rows x cols, ld) as a B operand: [npad][32] 128B-swizzled boxes
bool make_b_map(CUtensorMap* m, const float* B, int64_t rows, int cols, int64_t ld, int npad) {
  if (!aligned(B, 16) || (ld % 4) || ld < rows || rows > INT32_MAX) return false;
  const uint64_t d[2] = {uint64_t(rows), uint64_t(cols)}, s[1] = {uint64_t(ld) * 4};
  const uint32_t bx[2] = {KC, uint32_t(npad)};
  return make_map(m, B, 2, d, s, bx, true);
}

// row-major fp32 matrix (rows x cols, row pitch ld) as an MN-major B operand: (32 cols, 32 rows)
// boxes with the 32 B-atom 128 B swizzle (columns >= cols read as zero)
bool make_b_map_rm(CUtensorMap* m, const float* B, int64_t rows, int cols, int64_t ld) {
  if (!aligned(B, 16) || (ld % 4) || ld < cols || rows > INT32_MAX) return false;
  const uint64_t d[2] = {uint64_t(cols), uint64_t(rows)}, s[1] = {uint64_t(ld) * 4};
  const uint32_t bx[2] = {32, KC};
  return make_map(m, B, 2, d, s, bx, false, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

template <typename Kern>
void set_smem(Kern kernel, uint32_t bytes) {
  RT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

template <int NPAD, bool BSPLIT, bool AMN, bool BPRE, int XW = 1>
void launch_s(const Ctx& ctx, const CUtensorMap& tx, const CUtensorMap& tb, const SParams& p, dim3 grid) {
  using L = Plan<NPAD, BSPLIT, true, sketch_cps<NPAD, BSPLIT, true>(), 0, XW>;
  static bool attr = false;
  if (!attr) { set_smem(ttm_s_tc_kernel<NPAD, BSPLIT, AMN, BPRE, XW>, L::bytes); attr = true; }
  launch(ctx, ctx.label ? ctx.label : "ttm_s_tc", [&] {
    ttm_s_tc_kernel<NPAD, BSPLIT, AMN, BPRE, XW><<<grid, NT_TTM, L::bytes, ctx.stream>>>(tx, tb, p);
  });
}

// widest feasible X stage width <= want for the strided-mode sketch kernels of this shape
template <int NPAD>
int xw_feasible(int bmode, bool h16, int want) {
  auto ok_s = [&](auto xwc) {
    constexpr int XW = decltype(xwc)::value;
    if (h16) return PlanH<NPAD, 2, 0, XW>::ok;
    if (bmode == 0) return Plan<NPAD, false, true, sketch_cps<NPAD, false, true>(), 0, XW>::ok;
    return Plan<NPAD, true, true, sketch_cps<NPAD, true, true>(), 0, XW>::ok;
  };
  if (want >= 4 && ok_s(std::integral_constant<int, 4>())) return 4;
  if (want >= 2 && ok_s(std::integral_constant<int, 2>())) return 2;
  return 1;
}

// b: 0 tf32-exact B, 1 split in the kernel, 2 pre-split in global memory; xw: X stage width
template <int NPAD>
void dispatch_s(const Ctx& ctx, bool amn, int bmode, int xw, const CUtensorMap& tx, const CUtensorMap& tb,
                const SParams& p, dim3 g) {
  if (amn) {
    if (bmode == 0) launch_s<NPAD, false, true, false>(ctx, tx, tb, p, g);
    else if (bmode == 1) launch_s<NPAD, true, true, false>(ctx, tx, tb, p, g);
    else launch_s<NPAD, true, true, true>(ctx, tx, tb, p, g);
  } else if (xw == 4) {
    if (bmode == 0) { if constexpr (Plan<NPAD, false, true, sketch_cps<NPAD, false, true>(), 0, 4>::ok) launch_s<NPAD, false, false, false, 4>(ctx, tx, tb, p, g); }
    else if (bmode == 1) { if constexpr (Plan<NPAD, true, true, sketch_cps<NPAD, true, true>(), 0, 4>::ok) launch_s<NPAD, true, false, false, 4>(ctx, tx, tb, p, g); }
    else { if constexpr (Plan<NPAD, true, true, sketch_cps<NPAD, true, true>(), 0, 4>::ok) launch_s<NPAD, true, false, true, 4>(ctx, tx, tb, p, g); }
  } else if (xw == 2) {
    if (bmode == 0) { if constexpr (Plan<NPAD, false, true, sketch_cps<NPAD, false, true>(), 0, 2>::ok) launch_s<NPAD, false, false, false, 2>(ctx, tx, tb, p, g); }
    else if (bmode == 1) { if constexpr (Plan<NPAD, true, true, sketch_cps<NPAD, true, true>(), 0, 2>::ok) launch_s<NPAD, true, false, false, 2>(ctx, tx, tb, p, g); }
    else { if constexpr (Plan<NPAD, true, true, sketch_cps<NPAD, true, true>(), 0, 2>::ok) launch_s<NPAD, true, false, true, 2>(ctx, tx, tb, p, g); }
  } else {
    if (bmode == 0) launch_s<NPAD, false, false, false>(ctx, tx, tb, p, g);
    else if (bmode == 1) launch_s<NPAD, true, false, false>(ctx, tx, tb, p, g);
    else launch_s<NPAD, true, false, true>(ctx, tx, tb, p, g);
  }
}

template <int NPAD, bool AMN, int CPS = 2, int XW = 1>
void launch_h1(const Ctx& ctx, const CUtensorMap& tx, const CUtensorMap& tb, const HParams& p, dim3 grid) {
  using L = PlanH<NPAD, CPS, 0, XW>;
  static bool attr = false;
  if (!attr) { set_smem(ttm_s_h16_kernel<NPAD, AMN, CPS, XW>, L::bytes); attr = true; }
  launch(ctx, ctx.label ? ctx.label : "ttm_s_h16", [&] {
    ttm_s_h16_kernel<NPAD, AMN, CPS, XW><<<grid, NT_TTM, L::bytes, ctx.stream>>>(tx, tb, p);
  });
}
// 2 chunks per stage (1 chunk per stage measured the same: 6.0-6.3 ms per cfg5 pass either way)
template <int NPAD, bool AMN>
void launch_h(const Ctx& ctx, int xw, const CUtensorMap& tx, const CUtensorMap& tb, const HParams& p, dim3 grid) {
  if constexpr (!AMN) {
    if constexpr (PlanH<NPAD, 2, 0, 4>::ok) { if (xw == 4) { launch_h1<NPAD, AMN, 2, 4>(ctx, tx, tb, p, grid); return; } }
    if constexpr (PlanH<NPAD, 2, 0, 2>::ok) { if (xw == 2) { launch_h1<NPAD, AMN, 2, 2>(ctx, tx, tb, p, grid); return; } }
  }
  launch_h1<NPAD, AMN, 2>(ctx, tx, tb, p, grid);
}

template <int NPAD, bool AKM, bool BSPLIT, bool H16 = false>
void launch_t(const Ctx& ctx, const CUtensorMap& tx, const CUtensorMap& tb, const CUtensorMap& to, const TParams& p,
              dim3 grid) {
  using L = std::conditional_t<H16, PlanH<NPAD, 1, t_outb<NPAD>()>, Plan<NPAD, BSPLIT, false, 1, t_outb<NPAD>()>>;
  static bool attr = false;
  if (!attr) { set_smem(ttm_t_tc_kernel<NPAD, AKM, BSPLIT, H16>, L::bytes); attr = true; }
  launch(ctx, ctx.label ? ctx.label : (H16 ? "ttm_t_h16" : "ttm_t_tc"), [&] {
    ttm_t_tc_kernel<NPAD, AKM, BSPLIT, H16><<<grid, NT_TTM, L::bytes, ctx.stream>>>(tx, tb, to, p);
  });
}

// Y(i, k) = sum_z part[z][k][i] (fp64 sum in a fixed order).  CTA = 32 consecutive outputs x 8
// split groups: thread (o, g) sums z = g, g + 8, ... with 4 loads in flight, then the 8 group sums
// are added in order -- parallel over the split count too (the Gram of Z has ~600 splits but only
// K^2 outputs).
__global__ void __launch_bounds__(256) splitk_reduce_f32_kernel(const float* __restrict__ part, int64_t I, int K,
                                                                int splits, double* __restrict__ Y, int64_t ldy) {
  __shared__ double red[8][33];
  const int o = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t e = int64_t(blockIdx.x) * 32 + o;
  const int64_t n = I * K;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (e < n) {
    const int64_t i = e % I, k = e / I;
    const float* pp = part + k * I + i;
    const int64_t zs = int64_t(K) * I;
    int z = g;
    for (; z + 24 < splits; z += 32) {
      s0 += double(__ldg(pp + z * zs));
      s1 += double(__ldg(pp + (z + 8) * zs));
      s2 += double(__ldg(pp + (z + 16) * zs));
      s3 += double(__ldg(pp + (z + 24) * zs));
    }
    for (; z < splits; z += 8) s0 += double(__ldg(pp + z * zs));
  }
  red[g][o] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (g == 0 && e < n) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += red[q][o];
    const int64_t i = e % I, k = e / I;
    Y[i + ldy * k] = s;
  }
}

// Q (I x C, col-major ldq) -> Q2 (I x 2 npad, col-major ld2): columns [0, C) = tf32 hi, columns
// [npad, npad + C) = lo, the rest zero (the pre-split [B_hi | B_lo] operand of ttm_t_tc)
// chunk blockIdx.y: columns [cw y, cw y + cw) of Q into rows [2 npad y, 2 npad (y + 1)) of Q2
__global__ void split_q_kernel(const float* __restrict__ Q, int64_t I, int C, int64_t ldq, int npad,
                               float* __restrict__ Q2, int64_t ld2, int cw) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ld2 * npad) return;
  const int64_t i = e % ld2;
  const int c = int(e / ld2);
  const int cg = int(blockIdx.y) * cw + c;
  Q2 += int64_t(blockIdx.y) * 2 * npad * ld2;
  const float v = (i < I && c < cw && cg < C) ? Q[i + ldq * cg] : 0.f;
  uint32_t h, l;
  split_tf32(v, h, l);
  Q2[i + ld2 * c] = __uint_as_float(h);
  Q2[i + ld2 * (npad + c)] = __uint_as_float(l);
}

// Q (I x C, col-major ldq) -> Q2 row-major I x 2 npad fp16 (row pitch 2 npad): [2^14 Q_hi | 2^14 Q_lo],
// columns >= C zero (the B operand of ttm_t_tc_kernel<H16>)
__global__ void split_q_h16_kernel(const float* __restrict__ Q, int64_t I, int C, int64_t ldq, int npad,
                                   uint32_t* __restrict__ Q2) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;   // one pair of columns of one row
  const int hp = npad / 2;
  if (e >= I * hp) return;
  const int64_t i = e / hp;
  const int c0 = 2 * int(e % hp), c1 = c0 + 1;
  uint32_t h, l;
  split_h16x2(c0 < C ? Q[i + ldq * c0] * kQScale : 0.f, c1 < C ? Q[i + ldq * c1] * kQScale : 0.f, h, l);
  Q2[i * npad + c0 / 2] = h;
  Q2[i * npad + hp + c0 / 2] = l;
}

}  // namespace

namespace tc {
bool encode_f32_map(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                    const uint32_t* box, bool swz128) {
  return make_map(m, ptr, rank, dims, strides_bytes, box, swz128);
}
}  // namespace tc

int tc_npad(int K) {
  return K <= 16 ? 16 : K <= 32 ? 32 : K <= 48 ? 48 : K <= 64 ? 64 : K <= 80 ? 80 : K <= 96 ? 96 : K <= 128 ? 128 : -1;
}
int tc_split_width(int K) {
  const int np = tc_npad(K);
  return np < 0 ? -1 : ((np + 31) / 32) * 32;
}

bool ttm_s_tc_ok(const Ctx& ctx, const float* X, Box box, int K) {
  if (ctx.simt() || tc_npad(K) < 0) return false;
  const int64_t J = box.J();
  if (box.I < 1 || J < KC || !aligned(X, 16)) return false;
  const bool amn = (box.a == 1);
  if (amn ? (box.I % 4) : (box.a % 4)) return false;
  return !(box.a > INT32_MAX || box.I > INT32_MAX || box.b > INT32_MAX || J > INT32_MAX);
}

void x_scale_from_amax(const Ctx& ctx, const unsigned int* amax, int64_t n, float* s) {
  launch(ctx, "xscale", [&] { xscale_kernel<<<1, 1, 0, ctx.stream>>>(amax, double(n), s, ctx.tc_h16 == 2); });
}
__global__ void __launch_bounds__(256) q_gate_kernel(const float* __restrict__ Q, int64_t m, int r, int64_t ld,
                                                     const float* __restrict__ xs, float* __restrict__ out) {
  __shared__ int wide;
  if (threadIdx.x == 0) wide = 0;
  __syncthreads();
  for (int64_t e = threadIdx.x; e < m * r; e += blockDim.x) {
    const float v = Q[(e % m) + ld * (e / m)];
    if (!(fabsf(v) < 2.f)) wide = 1;                  // benign race: any writer stores 1
  }
  __syncthreads();
  if (threadIdx.x == 0) { out[0] = wide ? 0.f : xs[0]; out[1] = xs[1]; }
}
void q_gate_scale(const Ctx& ctx, const float* Q, int64_t m, int r, int64_t ld, const float* xs, float* out) {
  launch(ctx, "q_gate", [&] { q_gate_kernel<<<1, 256, 0, ctx.stream>>>(Q, m, r, ld, xs, out); });
}
// Omega (J x K fp32, row-major, pitch ld) -> fp16 rows [2^11 Omega_hi (npad) | 2^11 Omega_lo (npad)]
// (the pre-split B operand of ttm_s_h16_kernel; columns >= K zero).  2^11 keeps |Omega| < 16 inside
// the fp16 range with room (a Gaussian test matrix of 3.4e8 entries peaks near 6); an entry with
// |2^11 omega| >= 2^15 or a non-finite one sets *flag (the fp16 launch then stands down for its
// tf32 twin).  A tf32-rounded Omega is exact in the hi part (lo = 0).
// one thread per 8 consecutive columns of a row: two 16 B loads (vec4: K and ld multiples of 4 and a
// 16 B aligned Omega), one 16 B store each of the hi and lo halves
__global__ void omega_h16_kernel(const float* __restrict__ Om, int64_t J, int K, int64_t ld, int npad,
                                 uint32_t* __restrict__ O2, int* __restrict__ flag, bool vec4) {
  const int g8 = npad / 8, hp = npad / 2;
  bool bad = false;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < J * g8; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / g8;
    const int c0 = 8 * int(e % g8);
    float v[8];
    const float* row = Om + j * ld + c0;
    if (vec4 && c0 + 8 <= K) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(row)), b = __ldcs(reinterpret_cast<const float4*>(row + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (c0 + q < K) ? row[q] : 0.f;
    }
    uint32_t h[4], l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float v0 = v[2 * q] * 2048.f, v1 = v[2 * q + 1] * 2048.f;
      bad |= !(fabsf(v0) < 32768.f) || !(fabsf(v1) < 32768.f);
      split_h16x2(v0, v1, h[q], l[q]);
    }
    *reinterpret_cast<uint4*>(O2 + j * npad + c0 / 2) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(O2 + j * npad + hp + c0 / 2) = make_uint4(l[0], l[1], l[2], l[3]);
  }
  if (bad) atomicOr(flag, 1);
}
__global__ void omega_gate_kernel(const int* __restrict__ flag, const float* __restrict__ xs, float* __restrict__ out) {
  out[0] = *flag ? 0.f : xs[0];
  out[1] = xs[1];
}
const float* omega_h16(const Ctx& ctx, Arena& ws, const float* Om, int64_t J, int K, int64_t ld, const float* xs,
                       uint16_t** O2, int64_t* ld2) {
  const int npad = tc_npad(K);
  RT_REQUIRE(npad > 0, kEUNSUPPORTED, "omega_h16: K > 128");
  *ld2 = 2 * int64_t(npad);
  *O2 = ws.alloc_n<uint16_t>(J * *ld2);
  int* flag = ws.alloc_n<int>(1);
  float* xo = ws.alloc_n<float>(2);
  RT_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx.stream));
  const int64_t n = J * (npad / 8);
  const bool vec4 = (K % 4) == 0 && (ld % 4) == 0 && aligned(Om, 16);
  const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), int64_t(ctx.num_sms) * 16)));
  launch(ctx, "omega_h16", [&] {
    omega_h16_kernel<<<blocks, 256, 0, ctx.stream>>>(Om, J, K, ld, npad, reinterpret_cast<uint32_t*>(*O2), flag,
                                                     vec4);
  });
  launch(ctx, "omega_gate", [&] { omega_gate_kernel<<<1, 1, 0, ctx.stream>>>(flag, xs, xo); });
  return xo;
}
// Z (J x K fp32 row-major, pitch ldz) -> fp16 rows [2^14 Z_hi (npad) | 2^14 Z_lo (npad)] (the pre-split B
// operand of ttm_s_h16_kernel; columns >= K zero): the slab mode's power step after its allreduce (C3)
__global__ void split_rows_h16_kernel(const float* __restrict__ Z, int64_t J, int K, int64_t ldz, int npad,
                                      uint32_t* __restrict__ Z2) {
  const int hp = npad / 2;
  const int64_t n = J * hp, step = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += step) {   // a pair of columns of a row
    const int64_t j = e / hp;
    const int c0 = 2 * int(e % hp), c1 = c0 + 1;
    uint32_t h, l;
    split_h16x2(c0 < K ? Z[j * ldz + c0] * kQScale : 0.f, c1 < K ? Z[j * ldz + c1] * kQScale : 0.f, h, l);
    Z2[j * npad + c0 / 2] = h;
    Z2[j * npad + hp + c0 / 2] = l;
  }
}
// max_ctas > 0: a grid of at most that many CTAs (grid-stride); the C3 stream's conversion runs beside the
// other modes' X passes and must not take the SMs their small kernels are waiting for
void split_rows_h16(const Ctx& ctx, const float* Z, int64_t J, int K, int64_t ldz, uint16_t* Z2, int max_ctas) {
  const int npad = tc_npad(K);
  RT_REQUIRE(npad > 0, kEUNSUPPORTED, "split_rows_h16: K > 128");
  int64_t grid = cdiv(J * (npad / 2), 256);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  launch(ctx, "split_rows_h16", [&] {
    split_rows_h16_kernel<<<unsigned(grid), 256, 0, ctx.stream>>>(Z, J, K, ldz, npad, reinterpret_cast<uint32_t*>(Z2));
  });
}
void x_stat_pair(const Ctx& ctx, const unsigned int* amax, double* pair) {
  launch(ctx, "xstat_pair", [&] { stat_pair_kernel<<<1, 1, 0, ctx.stream>>>(amax, pair); });
}
void x_scale_from_gathered(const Ctx& ctx, const double* pairs, int nranks, int64_t n, float* s) {
  launch(ctx, "xscale", [&] {
    xscale_gathered_kernel<<<1, 1, 0, ctx.stream>>>(pairs, nranks, double(n), s, ctx.tc_h16 == 2);
  });
}

void x_absmax_stats(const Ctx& ctx, Arena& ws, const float* X, int64_t n, unsigned int* stat) {
  RT_REQUIRE(aligned(X, 16), kEINVAL, "x_absmax_stats: X must be 16-byte aligned");
  RT_CUDA(cudaMemsetAsync(stat, 0, 16, ctx.stream));
  const int64_t n4 = n / 4;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(cdiv(n4, 256), int64_t(ctx.num_sms) * 8));
  launch(ctx, "absmax", [&] {
    absmax_kernel<<<unsigned(blocks), 256, 0, ctx.stream>>>(reinterpret_cast<const float4*>(X), n4, X + 4 * n4,
                                                            int(n - 4 * n4), stat);
  });
}

void x_scale_h16(const Ctx& ctx, Arena& ws, const float* X, int64_t n, float* s) {
  unsigned int* stat = ws.alloc_n<unsigned int>(4);
  x_absmax_stats(ctx, ws, X, n, stat);
  x_scale_from_amax(ctx, stat, n, s);
}

// Returns false (nothing launched) when the shape/alignment is not supported by the TMA path.
bool ttm_s_tc(const Ctx& ctx, Arena& ws, const float* X, Box box, const float* Bm, int64_t ldb, bool b_tf32_exact,
              int K, double* Y, int64_t ldy, bool b_presplit, const float* xscale, unsigned int* amax,
              const float* Bfb, int64_t ldbfb, float binv) {
  const int npad = tc_npad(K);
  if (npad < 0) return false;
  const int64_t J = box.J();
  if (box.I < 1 || J < KC || !aligned(X, 16)) return false;
  const bool amn = (box.a == 1);
  if (amn ? (box.I % 4) : (box.a % 4)) return false;
  if (box.a > INT32_MAX || box.I > INT32_MAX || box.b > INT32_MAX || J > INT32_MAX) return false;
  const int nh = tc_split_width(K);
  const bool h16 = b_presplit && xscale != nullptr;
  const int bmode = b_presplit ? 2 : (b_tf32_exact ? 0 : 1);
  // X stage width of the strided modes: wide rows (xw chunks per unswizzled box) when a is a
  // multiple of KC xw (the chunk groups stay inside one beta) and the kernel's plan fits
  // (RT_OPT_TC_ABLATE 231 / 232 / 234 cap it at 1 / 2 / 4).  The fp16 kernel and its tf32 twin may
  // get different widths (the twin splits B in shared memory: fewer bytes left for X stages).
  auto pick_xw = [&](int bm, bool hh) {
    if (amn) return 1;
    int want = ctx.tc_xw;
    switch (npad) {
      case 16: want = xw_feasible<16>(bm, hh, want); break;
      case 32: want = xw_feasible<32>(bm, hh, want); break;
      case 48: want = xw_feasible<48>(bm, hh, want); break;
      case 64: want = xw_feasible<64>(bm, hh, want); break;
      case 80: want = xw_feasible<80>(bm, hh, want); break;
      case 96: want = xw_feasible<96>(bm, hh, want); break;
      default: want = xw_feasible<128>(bm, hh, want); break;
    }
    while (want >= 2 && !(box.a % (int64_t(KC) * want) == 0 && box.a >= int64_t(KC) * want + 4)) want /= 2;
    return want >= 2 ? want : 1;
  };
  const int xw = pick_xw(h16 ? 2 : bmode, h16);           // the launch in charge
  const int xw_t = h16 ? pick_xw(1, false) : xw;           // its tf32 twin (h16 only)
  auto make_x = [&](CUtensorMap* m, int w) {
    if (amn) {
      const uint64_t d[2] = {uint64_t(box.I), uint64_t(box.b)}, st[1] = {uint64_t(box.I) * 4};
      const uint32_t bx[2] = {BM, KC};
      return make_map(m, X, 2, d, st, bx, false);
    }
    const uint64_t d[3] = {uint64_t(box.a), uint64_t(box.I), uint64_t(box.b)};
    const uint64_t st[2] = {uint64_t(box.a) * 4, uint64_t(box.a) * box.I * 4};
    const uint32_t bx[3] = {w > 1 ? uint32_t(KC * w + 4) : uint32_t(KC), BM, 1};
    return make_map(m, X, 3, d, st, bx, w == 1);
  };
  CUtensorMap tx, txt, tb;
  if (!make_x(&tx, xw)) return false;
  if (xw_t != xw) { if (!make_x(&txt, xw_t)) return false; } else { txt = tx; }
  if (h16) {
    // fp16 [hi (npad) | lo (npad)] rows, row pitch ldb halves: (64 cols, 32 rows) SWIZZLE_128B boxes
    if (!aligned(Bm, 16) || (ldb % 8) || ldb < 2 * npad) return false;
    const uint64_t d[2] = {uint64_t(2 * npad), uint64_t(J)}, st[1] = {uint64_t(ldb) * 2};
    const uint32_t bx[2] = {64, KC};
    if (!make_map(&tb, Bm, 2, d, st, bx, true, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_DATA_TYPE_FLOAT16)) return false;
  } else if (!make_b_map_rm(&tb, Bm, J, b_presplit ? 2 * nh : K, ldb)) {
    return false;
  }
  // the fp16-split launch comes with its tf32 twin on the fp32 B (split in the kernel), gated on the
  // device by s == 0 (R29): both write the same split-K partials, exactly one of them runs
  CUtensorMap tbf;
  RT_REQUIRE(!h16 || Bfb != nullptr, kEINVAL, "ttm_s_tc: the fp16 form needs the fp32 B of its tf32 twin");
  if (h16 && !make_b_map_rm(&tbf, Bfb, J, K, ldbfb)) return false;
  SParams p;
  p.a = box.a; p.I = box.I; p.b = box.b; p.K = K;
  p.cpb = amn ? 1 : cdiv(box.a, KC);
  p.nchunks = amn ? cdiv(box.b, KC) : p.cpb * box.b;
  const int64_t mtiles = cdiv(box.I, BM);
  // split count: tc_waves CTA waves over the SMs (1: one CTA per SM for the whole pass, no wave
  // quantization; the SMs left over when mtiles does not divide the SM count serve the side stream)
  int64_t splits = ctx.tc_waves == 1 ? std::max<int64_t>(1, int64_t(ctx.num_sms - ctx.sm_reserve) / mtiles)
                                     : std::max<int64_t>(1, (int64_t(ctx.num_sms) * ctx.tc_waves + mtiles - 1) / mtiles);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, p.nchunks / 8));
  splits = std::min<int64_t>(splits, 65535);
  // contiguous chunk range per split, a whole number of X stages
  const int xwl = std::max(xw, xw_t);                     // 1, 2, 4: a multiple of both widths
  p.per = cdiv(cdiv(p.nchunks, splits), xwl) * xwl;
  splits = cdiv(p.nchunks, p.per);
  p.seg = std::max(1, ctx.tc_seg);
  p.ablate = ctx.tc_ablate;
  p.skew = ctx.tc_skew >= 0 ? ctx.tc_skew : 0;
  p.xfirst = ctx.tc_xfirst;
  p.part = ws.alloc_n<float>(splits * K * box.I);
  p.amax = h16 ? nullptr : amax;
  p.gate = nullptr;
  p.runs = ctx.d_runs;
  p.tim = nullptr;
  p.trace = nullptr;
  const dim3 grid{unsigned(mtiles), unsigned(splits), 1u};
  if (ctx.tc_ablate == 2000) {
    p.trace = ws.alloc_n<long long>(512 * 8);
    RT_CUDA(cudaMemsetAsync(p.trace, 0, sizeof(long long) * 512 * 8, ctx.stream));
  }
  if (ctx.tc_ablate == 1000) {
    p.tim = ws.alloc_n<unsigned long long>(mtiles * splits * 24);
    RT_CUDA(cudaMemsetAsync(p.tim, 0, sizeof(unsigned long long) * mtiles * splits * 24, ctx.stream));
  }
#define RT_S_CASE(NP)                                                                 \
  case NP:                                                                            \
    if (h16) {                                                                        \
      const HParams hp{p, xscale, binv};                                              \
      if (amn) launch_h<NP, true>(ctx, xw, tx, tb, hp, grid);                         \
      else launch_h<NP, false>(ctx, xw, tx, tb, hp, grid);                            \
      SParams pf = p;                                                                 \
      pf.gate = xscale;                                                               \
      dispatch_s<NP>(ctx, amn, 1, xw_t, txt, tbf, pf, grid);                          \
    } else {                                                                          \
      dispatch_s<NP>(ctx, amn, bmode, xw, tx, tb, p, grid);                           \
    }                                                                                 \
    break;
  switch (npad) {
    RT_S_CASE(16) RT_S_CASE(32) RT_S_CASE(48) RT_S_CASE(64) RT_S_CASE(80) RT_S_CASE(96) RT_S_CASE(128)
    default: return false;
  }
#undef RT_S_CASE
  if (p.trace) {   // diagnostics: event clocks of chunks 200..231 of CTA (0,0), relative to chunk 200 start
    std::vector<long long> h(512 * 8);
    RT_CUDA(cudaMemcpyAsync(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost, ctx.stream));
    RT_CUDA(cudaStreamSynchronize(ctx.stream));
    const long long t0 = h[200 * 8 + 0];
    std::fprintf(stderr, "[ttm_s_tc trace] %s bmode=%d: it  x_full  slot  ready | iss0 go  done | iss1 go  done | drain\n",
                 ctx.label ? ctx.label : "ttm_s_tc", bmode);
    for (int it = 200; it < 232; ++it) {
      std::fprintf(stderr, "   %3d", it);
      for (int e = 0; e < 8; ++e) std::fprintf(stderr, " %7lld", h[it * 8 + e] ? h[it * 8 + e] - t0 : -1LL);
      std::fprintf(stderr, "\n");
    }
  }
  if (p.tim) {   // diagnostics: mean cycles per CTA spent in each role's waits / work
    std::vector<unsigned long long> h(size_t(mtiles * splits * 24));
    RT_CUDA(cudaMemcpyAsync(h.data(), p.tim, h.size() * 8, cudaMemcpyDeviceToHost, ctx.stream));
    RT_CUDA(cudaStreamSynchronize(ctx.stream));
    static const char* nm[22] = {"x_prod:wait_free", "b_prod:wait_free", "iss0:acc_empty", "iss0:ready", "iss0:b_full",
                                 "iss0:mma", "iss1:acc_empty", "iss1:ready", "iss1:b_full", "iss1:mma",
                                 "split:x_full", "split:tfree", "split:split", "split:b_full", "split:drain", "total",
                                 "iss0:commits", "iss1:commits", "iss0:loop", "iss1:loop", "iss0:fence", "iss1:fence"};
    std::fprintf(stderr, "[ttm_s_tc diag] %s npad=%d bmode=%d grid=%lldx%lld chunks/cta=%lld\n",
                 ctx.label ? ctx.label : "ttm_s_tc", npad, bmode, (long long)mtiles, (long long)splits,
                 (long long)((p.nchunks + splits - 1) / splits));
    for (int k = 0; k < 22; ++k) {
      double sum = 0;
      for (int64_t c = 0; c < mtiles * splits; ++c) sum += double(h[size_t(c * 24 + k)]);
      std::fprintf(stderr, "   %-18s %12.0f cycles/CTA\n", nm[k], sum / double(mtiles * splits));
    }
  }
  const int64_t n = box.I * K;
  launch(ctx, "splitk_reduce", [&] {
    splitk_reduce_f32_kernel<<<unsigned(cdiv(n, 32)), 256, 0, ctx.stream>>>(p.part, box.I, K, int(splits), Y, ldy);
  });
  return true;
}

bool ttm_t_tc(const Ctx& ctx, Arena& ws, const float* X, Box box, const float* Q, int64_t ldq, int C, float* out,
              int64_t so_a, int64_t so_c, int64_t so_b, int split_out, bool q_tf32_exact, const float* xscale,
              const float* run_if_zero, const float* oscale, float omul, bool no_twin, int cw) {
  // cw > 0: C columns in chunks of cw (<= 128) within one launch (3xTF32 form only)
  const int nch = (cw > 0 && C > cw) ? int(cdiv(C, cw)) : 1;
  if (nch == 1) cw = C;
  const int npad = tc_npad(cw);
  if (npad < 0) return false;
  if (nch > 1 && (xscale != nullptr || split_out || q_tf32_exact)) return false;
  const bool h16 = xscale != nullptr && !q_tf32_exact;
  const bool akm = (box.a == 1);
  if (!aligned(X, 16)) return false;
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
  const bool bsplit = !q_tf32_exact || !aligned(Q, 16) || (ldq % 4) != 0 || nch > 1;
  CUtensorMap tbh;   // fp16 [2^14 Q_hi | 2^14 Q_lo] operand of the H16 kernel (with h16)
  if (h16) {
    // fp16 rows (I x 2 npad halves): (64 cols, 32 rows) SWIZZLE_128B boxes
    uint32_t* Q2 = ws.alloc_n<uint32_t>(box.I * npad);
    const uint64_t d[2] = {uint64_t(2 * npad), uint64_t(box.I)}, st[1] = {uint64_t(npad) * 4};
    const uint32_t bx[2] = {64, KC};
    if (!make_map(&tbh, Q2, 2, d, st, bx, true, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_DATA_TYPE_FLOAT16)) return false;
    launch(ctx, "split_q", [&] {
      split_q_h16_kernel<<<unsigned(cdiv(box.I * (npad / 2), 256)), 256, 0, ctx.stream>>>(Q, box.I, C, ldq, npad, Q2);
    });
  }
  if (bsplit) {
    // pre-split [Q_hi | Q_lo] (I x 2 npad): the kernel loads it as one [2 npad][32] K-major slot
    // (with h16 this is the operand of the tf32 twin that runs instead when s == 0, R29)
    const int64_t ld2 = (box.I + 3) & ~int64_t(3);
    float* Q2 = ws.alloc_n<float>(ld2 * 2 * npad * nch);
    if (!make_b_map(&tb, Q2, box.I, 2 * npad * nch, ld2, 2 * npad)) return false;
    launch(ctx, "split_q", [&] {
      split_q_kernel<<<dim3(unsigned(cdiv(ld2 * npad, 256)), unsigned(nch)), 256, 0, ctx.stream>>>(Q, box.I, C, ldq,
                                                                                                  npad, Q2, ld2, cw);
    });
  } else {
    // tf32-exact Q read in place as a [npad][32] K-major slot (columns >= C read as zero)
    if (!make_b_map(&tb, Q, box.I, C, ldq, npad)) return false;
  }
  TParams p;
  p.a = box.a; p.I = box.I; p.b = box.b; p.C = C;
  p.nch = nch; p.cw = cw;
  p.tpb = akm ? 1 : cdiv(box.a, BM);
  p.ntiles = akm ? cdiv(box.b, BM) : p.tpb * box.b;
  p.nic = int(cdiv(box.I, KC));
  p.seg = std::max(1, ctx.tc_seg);
  p.out = out; p.so_a = so_a; p.so_c = so_c; p.so_b = so_b;
  p.vec4 = so_c == 1 && (akm || (so_a % 4) == 0) && (so_b % 4) == 0 && (C % 4) == 0 && aligned(out, 16);   // a == 1: so_a unused
  p.split_out = split_out;
  p.xscale = h16 ? xscale : nullptr;
  p.gate = h16 ? nullptr : run_if_zero;
  p.runs = ctx.d_runs;
  p.oscale = oscale;
  p.omul = omul;
  RT_REQUIRE(!split_out || (so_c == 1 && (so_a % 4) == 0 && (so_b % 4) == 0 && aligned(out, 16)), kEINVAL,
             "split output needs 16-byte aligned row-major rows");
  RT_REQUIRE(split_out != 2 || ((so_a % 8) == 0 && (so_b % 8) == 0), kEINVAL, "fp16 split rows need 16-byte pitch");
  // TMA-stored output tiles: row-major rows (so_c == 1) with one row pitch across the whole
  // output (mode 0: rows j = beta, pitch so_b; a > 1: rows alpha + a beta with so_b = a so_a and
  // whole 128-row tiles per beta)
  CUtensorMap to;
  std::memset(&to, 0, sizeof(to));
  p.tma_out = false;
  if (p.vec4 && !split_out && !getenv("RT_TC_NO_TMA_OUT")) {
    const int64_t pitch = akm ? so_b : so_a;
    const int64_t rows = akm ? box.b : box.a * box.b;
    const bool rowsok = akm || (box.a % BM == 0 && so_b == box.a * so_a);
    if (rowsok && rows <= INT32_MAX) {
      const uint64_t d[2] = {uint64_t(C), uint64_t(rows)}, st[1] = {uint64_t(pitch) * 4};
      const uint32_t bx[2] = {32, uint32_t(BM)};
      p.tma_out = make_map(&to, out, 2, d, st, bx, true);
    }
  } else if (split_out == 2 && !getenv("RT_TC_NO_TMA_OUT")) {
    // fp16 [hi | lo] rows of 2 npad halves, one row pitch across the output (mode 0: rows j = beta,
    // pitch so_b; a > 1: rows alpha + a beta, pitch so_a, whole 128-row tiles per beta): (64, 128)
    // SWIZZLE_128B boxes
    const int64_t pitch = akm ? so_b : so_a;
    const int64_t rows = akm ? box.b : box.a * box.b;
    const bool rowsok = akm || (box.a % BM == 0 && so_b == box.a * so_a);
    if (rowsok && rows <= INT32_MAX) {
      const uint64_t d[2] = {uint64_t(2 * npad), uint64_t(rows)}, st[1] = {uint64_t(pitch) * 2};
      const uint32_t bx[2] = {64, uint32_t(BM)};
      p.tma_out = make_map(&to, out, 2, d, st, bx, true, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    }
  }
  const int64_t grid = std::min<int64_t>(p.ntiles * nch, std::max(1, ctx.num_sms - ctx.sm_reserve));
#define RT_T_CASE(NP)                                                     \
  case NP:                                                                \
    if (h16) {                                                           \
      TParams pf = p;                                                    \
      pf.gate = xscale;                                                  \
      if (akm) {                                                         \
        launch_t<NP, true, true, true>(ctx, tx, tbh, to, p, dim3(unsigned(grid)));  \
        if (!no_twin) launch_t<NP, true, true>(ctx, tx, tb, to, pf, dim3(unsigned(grid)));  \
      } else {                                                           \
        launch_t<NP, false, true, true>(ctx, tx, tbh, to, p, dim3(unsigned(grid))); \
        if (!no_twin) launch_t<NP, false, true>(ctx, tx, tb, to, pf, dim3(unsigned(grid))); \
      }                                                                  \
    } else if (bsplit) {                                                 \
      if (akm) launch_t<NP, true, true>(ctx, tx, tb, to, p, dim3(unsigned(grid)));  \
      else launch_t<NP, false, true>(ctx, tx, tb, to, p, dim3(unsigned(grid)));     \
    } else {                                                             \
      if (akm) launch_t<NP, true, false>(ctx, tx, tb, to, p, dim3(unsigned(grid))); \
      else launch_t<NP, false, false>(ctx, tx, tb, to, p, dim3(unsigned(grid)));    \
    }                                                                    \
    break;
  switch (npad) {
    RT_T_CASE(16) RT_T_CASE(32) RT_T_CASE(48) RT_T_CASE(64) RT_T_CASE(80) RT_T_CASE(96) RT_T_CASE(128)
    default: return false;
  }
#undef RT_T_CASE
  return true;
}


// Fused mode-1 Omega sketch + mode-0 core stage (sketch1_core0_kernel); false (nothing launched) when
// the shape / precision is outside it.  b1: X as the mode-1 box [I_0, I_1, rest]; b0: the mode-0 box.
// Om: the fp32 Omega_1 (J x K1 row-major, ld ldom; tf32-exact for the fused form, else the flag sends
// the work to the twins); Q0: Q~_0 fp32 col-major (I_0 x K0, ld ldq0, orthonormal); xs: X's scale pair.
// Outputs: Y (fp64 I_1 x K1, ld ldy) and out (the core stage: rows j = i1 + I_1 beta of K0 floats).
__global__ void omega_gate_inv_kernel(const int* __restrict__ flag, const float* __restrict__ xs, float* __restrict__ out) {
  out[0] = *flag ? xs[0] : 0.f;                      // the fused pass stood down for Omega, X's scale is fine
  out[1] = xs[1];
}

bool sketch1_core0_prep(const Ctx& ctx, Arena& ws, const float* Om, int64_t J, int K1, int64_t ldom, int npad,
                        F1Prep* pre) {
  if (ctx.simt() || !ctx.tc_h16 || ctx.fuse_off || npad <= 0 || npad > 80 || (ldom % 4) || !aligned(Om, 16) ||
      J > INT32_MAX)
    return false;
  pre->npad = npad;
  pre->ldw = (J + 63) & ~int64_t(63);
  __half* WT = ws.alloc_n<__half>(int64_t(npad) * pre->ldw);
  pre->WT = reinterpret_cast<uint16_t*>(WT);
  pre->flag = ws.alloc_n<int>(1);
  RT_CUDA(cudaMemsetAsync(pre->flag, 0, sizeof(int), ctx.stream));
  const int64_t ldw = pre->ldw;
  int* flag = pre->flag;
  launch(ctx, "omega_t16", [&] {
    omega_t16_kernel<<<unsigned(cdiv(ldw, 64)), 256, 0, ctx.stream>>>(Om, J, K1, ldom, npad, WT, ldw, flag);
  });
  return true;
}

bool sketch1_core0(const Ctx& ctx, Arena& ws, const float* X, Box b1, Box b0, const float* Om, int64_t ldom, int K1,
                   const float* Q0, int64_t ldq0, int K0, const float* xs, double* Y, int64_t ldy, float* out,
                   int view_last, const F1Prep* pre, const F1ZOut* zo) {
  if (ctx.simt() || !ctx.tc_h16 || ctx.fuse_off) return false;
  const int npad = tc_npad(std::max(K0, K1));
  if (npad < 0 || npad > 80) return false;
  if (b1.a % 512 || b1.I % BM || (K0 % 4) || (ldom % 4) || !aligned(X, 16) || !aligned(Om, 16) ||
      (!zo && !aligned(out, 16)))
    return false;
  if (pre && pre->npad != npad) return false;
  const int64_t J = b1.J();
  if (b1.a > INT32_MAX || b1.I > INT32_MAX || b1.b > INT32_MAX || J > INT32_MAX || b0.b > INT32_MAX) return false;
  if (zo && (!zo->Z2 || zo->ldz2 != 2 * npad || !aligned(zo->Z2, 16))) return false;
  // X as [alpha = i_0, rows = i_m, beta]: the mode-1 view is X's memory order; the last-mode view
  // takes the rows from the slowest dimension and beta (the middle modes) from the middle
  const uint64_t xd[3] = {uint64_t(b1.a), uint64_t(b1.I), uint64_t(b1.b)};
  const uint64_t xst[2] = {view_last ? uint64_t(b1.a) * b1.b * 4 : uint64_t(b1.a) * 4,
                           view_last ? uint64_t(b1.a) * 4 : uint64_t(b1.a) * b1.I * 4};
  // B sources: 2^14 [Q_hi^T ; Q_lo^T] and 2^11 Omega^T in fp16, rows padded to npad
  const int64_t ldt = (b1.a + 7) & ~int64_t(7);
  __half* QT = ws.alloc_n<__half>(2 * npad * ldt);
  F1Prep own;
  if (!pre) {
    if (!sketch1_core0_prep(ctx, ws, Om, J, K1, ldom, npad, &own)) return false;
    pre = &own;
  }
  __half* WT = reinterpret_cast<__half*>(pre->WT);
  const int64_t ldw = pre->ldw;
  int* flag = pre->flag;
  float* xso = ws.alloc_n<float>(2);
  launch(ctx, "qt16", [&] {
    qt16_kernel<<<unsigned(cdiv(ldt * npad, 256)), 256, 0, ctx.stream>>>(Q0, b1.a, K0, ldq0, npad, QT, ldt);
  });
  launch(ctx, "omega_gate", [&] { omega_gate_kernel<<<1, 1, 0, ctx.stream>>>(flag, xs, xso); });
  CUtensorMap tx, tq, tw;
  {
    const uint32_t bx[3] = {uint32_t(KC * 2 + 4), BM, 1};
    if (!make_map(&tx, X, 3, xd, xst, bx, false)) return false;
  }
  {
    const uint64_t d[2] = {uint64_t(ldt), uint64_t(2 * npad)}, st[1] = {uint64_t(ldt) * 2};
    const uint32_t bx[2] = {64, uint32_t(npad)};
    if (!make_map(&tq, QT, 2, d, st, bx, true, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_DATA_TYPE_FLOAT16)) return false;
  }
  {
    const uint64_t d[3] = {64, uint64_t(npad), uint64_t(ldw / 64)}, st[2] = {128, uint64_t(npad) * 128};
    const uint32_t bx[3] = {64, uint32_t(npad), 1};
    if (!make_map(&tw, WT, 3, d, st, bx, true, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_DATA_TYPE_FLOAT16)) return false;
  }
  // the left output: fp32 core rows (K0 floats) or the R31 Z rows (2 npad halves); rows j = i + I beta
  // (mode-1 view) or j = beta + b i (last-mode view), written from the epilogue's registers
  if (zo ? !aligned(zo->Z2, 16) : !aligned(out, 16)) return false;
  FParams p;
  p.a = b1.a; p.I = b1.I; p.b = b1.b; p.K = K1; p.C = K0;
  p.cpb = b1.a / KC;
  p.nchunks = p.cpb * b1.b;
  p.seg = int(std::min<int64_t>(ctx.fused_seg, p.cpb));
  while (p.cpb % p.seg) --p.seg;
  const int64_t mtiles = b1.I / BM;
  const int64_t want = std::max<int64_t>(1, (int64_t(ctx.num_sms) * 4 + mtiles - 1) / mtiles);
  const int64_t bper = cdiv(b1.b, std::min<int64_t>(want, b1.b));      // whole betas per split
  p.per = bper * p.cpb;
  const int64_t splits = cdiv(p.nchunks, p.per);
  p.part = ws.alloc_n<float>(splits * K1 * b1.I);
  p.xscale = xso;
  p.binv_s = 1.f / 2048.f;
  p.binv_c = 1.f / kQScale;
  p.runs = ctx.d_runs;
  p.zout = zo ? 1 : 0;
  p.ablate = ctx.tc_ablate;
  p.view_last = view_last;
  p.oscale = zo ? zo->oscale : nullptr;
  p.omul = zo ? zo->omul : 1.f;
  p.out = zo ? static_cast<void*>(zo->Z2) : static_cast<void*>(out);
  p.ldo = zo ? int64_t(2 * npad) : int64_t(K0);
  const dim3 grid{unsigned(mtiles), unsigned(splits), 1u};
  // tf32 twins, gated on the same scale (s == 0: X's range or Omega's precision outside the fp16
  // form): the plain sketch kernel on the fp32 Omega and the tf32 core stage
  const int bmode_t = ctx.omega_tf32 ? 0 : 1;
  SParams pf{};
  pf.a = b1.a; pf.I = b1.I; pf.b = b1.b; pf.K = K1;
  pf.cpb = p.cpb; pf.nchunks = p.nchunks; pf.per = p.per;
  pf.seg = std::max(1, ctx.tc_seg);
  pf.xfirst = ctx.tc_xfirst;
  pf.part = p.part;
  pf.gate = xso;
  pf.runs = ctx.d_runs;
  CUtensorMap tbf, txt;
  if (!make_b_map_rm(&tbf, Om, J, K1, ldom)) return false;
#define RT_F_CASE(NP)                                                                                    \
  case NP: {                                                                                             \
    if (ctx.fused_nbb == 3) {                                                                            \
      using L = PlanF<NP, 3>;                                                                            \
      static bool attr = false;                                                                          \
      if (!attr) { set_smem(sketch1_core0_kernel<NP, 3>, L::bytes); attr = true; }                       \
      launch(ctx, ctx.label ? ctx.label : "sketch1_core0", [&] {                                         \
        sketch1_core0_kernel<NP, 3><<<grid, NT_FUSED, L::bytes, ctx.stream>>>(tx, tq, tw, p);            \
      });                                                                                                \
    } else {                                                                                             \
      using L = PlanF<NP, 2>;                                                                            \
      static bool attr = false;                                                                          \
      if (!attr) { set_smem(sketch1_core0_kernel<NP, 2>, L::bytes); attr = true; }                       \
      launch(ctx, ctx.label ? ctx.label : "sketch1_core0", [&] {                                         \
        sketch1_core0_kernel<NP, 2><<<grid, NT_FUSED, L::bytes, ctx.stream>>>(tx, tq, tw, p);            \
      });                                                                                                \
    }                                                                                                    \
    int xw_t = xw_feasible<NP>(bmode_t, false, 2);                                                       \
    {                                                                                                    \
      const uint32_t bx[3] = {xw_t > 1 ? uint32_t(KC * xw_t + 4) : uint32_t(KC), BM, 1};                 \
      if (!make_map(&txt, X, 3, xd, xst, bx, xw_t == 1)) return false;                                  \
    }                                                                                                    \
    dispatch_s<NP>(ctx, false, bmode_t, xw_t, txt, tbf, pf, grid);                                       \
    break;                                                                                               \
  }
  switch (npad) {
    RT_F_CASE(16) RT_F_CASE(32) RT_F_CASE(48) RT_F_CASE(64) RT_F_CASE(80)
    default: return false;
  }
#undef RT_F_CASE
  if (!zo) {
    RT_REQUIRE(ttm_t_tc(ctx, ws, X, b0, Q0, ldq0, K0, out, 1, 1, K0, 0, false, nullptr, xso), kEUNSUPPORTED,
               "sketch1_core0: tf32 twin of the core stage rejected");
  } else {
    // twins of the R31 Z pass: the fp16-split Z pass when only Omega closed the fused gate (gz), and
    // the tf32 one writing the fp32 s_z Z when X's scale is 0 (the product's tf32 twin reads it)
    float* gz = ws.alloc_n<float>(2);
    launch(ctx, "omega_gate", [&] { omega_gate_inv_kernel<<<1, 1, 0, ctx.stream>>>(flag, zo->xs_x, gz); });
    RT_REQUIRE(ttm_t_tc(ctx, ws, X, b0, Q0, ldq0, K0, reinterpret_cast<float*>(zo->Z2), zo->ldz2, 1, zo->ldz2, 2, false,
                        gz, nullptr, zo->oscale, zo->omul, true) &&
                   ttm_t_tc(ctx, ws, X, b0, Q0, ldq0, K0, zo->Z, zo->ldz, 1, zo->ldz, 0, false, nullptr, zo->xs_x,
                            zo->oscale, zo->omul),
               kEUNSUPPORTED, "sketch1_core0: twins of the Z pass rejected");
  }
  const int64_t n = b1.I * K1;
  launch(ctx, "splitk_reduce", [&] {
    splitk_reduce_f32_kernel<<<unsigned(cdiv(n, 32)), 256, 0, ctx.stream>>>(p.part, b1.I, K1, int(splits), Y, ldy);
  });
  return true;
}

}  // namespace rt

// ============================================================ residual (a8)
// sum_{j,i} (X[j + J i] - Xhat[j,i])^2 and sum X^2 with Xhat = P Q^T (P: J x R col-major, the core
// expanded over all but the last mode; Q: the last factor).  Xhat tiles [128 j x 64 i] are built on
// the tensor cores (A = P tile hi/lo in TMEM, B = Q^T hi / lo pre-split, 3 products, contraction R)
// and compared with the X tile in the epilogue; nothing but two fp64 partial sums per CTA is written.
namespace rt {
namespace {
using namespace tc;

constexpr int RNB = 64;                      // i columns per block (MMA N)
constexpr int RNS = 3;                       // block pipeline depth (3 x 64 KB + the 32 KB P tile)

template <int RP>
struct RSmem {
  static constexpr uint32_t kP = uint32_t(RP) * BM * 4;          // raw P tile [RP r][128 j]
  static constexpr uint32_t kQ = uint32_t(RNB) * KC * 4;         // one [64 i][32 r] swizzled B chunk
  static constexpr uint32_t kXt = uint32_t(BM) * RNB * 4;        // X tile [64 i][128 j]
  static constexpr uint32_t per_stage = 2 * (RP / KC) * kQ + kXt;
  static constexpr uint32_t off_p = 0;
  static constexpr uint32_t off_st = kP;
  static constexpr uint32_t off_bar = off_st + RNS * per_stage;
  static constexpr uint32_t bytes = off_bar + 8 * (2 * RNS + 8) + 16;
};

struct RParams {
  int64_t J, In;
  int R;
  int64_t ntiles;     // j tiles of 128
  int nblk;           // i blocks of 64
  double* part;       // [grid][2]
  const float* rscale;   // power-of-two scale applied to x and x^ (resid_scale), nullable
  const float* gate;     // tf32 kernel: run only if *gate == 0 (twin of the fp16-split residual)
  int64_t tps = 0;       // > 0: sliced form (3-D maps): j tiles per slice; tile t = (slice t / tps, j tile t % tps)
};

template <int RP>
__global__ void __launch_bounds__(NTHREADS, 1)
residual_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmp,
                   const __grid_constant__ CUtensorMap tqh, const __grid_constant__ CUtensorMap tql, const RParams p) {
  using L = RSmem<RP>;
  constexpr int NCH = RP / KC;                 // r chunks
  if (p.gate && *p.gate != 0.f) return;       // the fp16-split residual ran (R29)
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::off_bar);
  uint64_t* st_full = bar;                     // [RNS] Q chunks + X tile landed
  uint64_t* st_free = bar + RNS;               // [RNS] epilogue done with the stage (128 arrivals)
  uint64_t* p_full = bar + 2 * RNS;            // P raw tile landed
  uint64_t* p_free = bar + 2 * RNS + 1;        // splitter done reading P raw (128)
  uint64_t* a_ready = bar + 2 * RNS + 2;       // A (hi/lo) in TMEM (128)
  uint64_t* a_free = bar + 2 * RNS + 3;        // all MMAs of the tile done (commit)
  uint64_t* acc_full = bar + 2 * RNS + 4;      // [2]
  uint64_t* acc_empty = bar + 2 * RNS + 6;     // [2] (128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2 * RNS + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t my_tiles = (p.ntiles > blockIdx.x) ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // TMEM: accumulator buffers at 0 / 2 RNB, each [hi.hi | hi.lo] (2 RNB columns: the B operand of
  // the wide MMA is the concatenated [Q_hi | Q_lo] chunk), issued by warp 1; the lo.hi products in
  // their own buffers at kAcc1 + RNB ab, issued by warp 6 (MMAs from two warps overlap, one warp's
  // complete one after another); A hi at kA, A lo at kA + RP
  constexpr uint32_t kAcc = 2 * RNB;
  constexpr uint32_t kAcc1 = 2 * kAcc;
  constexpr uint32_t kA = kAcc1 + 2 * RNB;
  static_assert(kA + 2 * RP <= 512, "residual TMEM plan");

  if (threadIdx.x == 0) {
    for (int s = 0; s < RNS; ++s) { mbar_init(&st_full[s], 1); mbar_init(&st_free[s], 128); }
    mbar_init(p_full, 1);
    mbar_init(p_free, 128);
    mbar_init(a_ready, 128);
    mbar_init(a_free, 2);
    for (int b = 0; b < 2; ++b) { mbar_init(&acc_full[b], 2); mbar_init(&acc_empty[b], 128); }
    fence_barrier_init();
    tma_prefetch(&tmx); tma_prefetch(&tmp); tma_prefetch(&tqh); tma_prefetch(&tql);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                   // ---------------- TMA producer
      Ring rg;
      int it = 0;
      for (int64_t u = 0; u < my_tiles; ++u) {
        const int j0 = int((blockIdx.x + u * gridDim.x) * BM);
        if (u >= 1) mbar_wait(p_free, uint32_t(u - 1) & 1);
        mbar_expect_tx(p_full, L::kP);
        for (int c = 0; c < NCH; ++c)
          tma_load_2d(smem + L::off_p + c * (BM * KC * 4), &tmp, p_full, j0, c * KC);
        for (int b = 0; b < p.nblk; ++b, ++it, rg.next<RNS>()) {
          if (it >= RNS) mbar_wait(&st_free[rg.s], rg.ph ^ 1);
          uint8_t* st = smem + L::off_st + rg.s * L::per_stage;
          mbar_expect_tx(&st_full[rg.s], L::per_stage);
          for (int c = 0; c < NCH; ++c) {      // [Q_hi c | Q_lo c] adjacent: one N = 2 RNB operand
            tma_load_2d(st + (2 * c) * L::kQ, &tqh, &st_full[rg.s], c * KC, b * RNB);
            tma_load_2d(st + (2 * c + 1) * L::kQ, &tql, &st_full[rg.s], c * KC, b * RNB);
          }
          tma_load_2d(st + 2 * NCH * L::kQ, &tmx, &st_full[rg.s], j0, b * RNB);
        }
      }
    }
  } else if (warp == 1 || warp == 6) {                // ---------------- MMA issuers (whole warps)
    const bool wide = warp == 1;
    const uint32_t idesc_w = idesc_tf32(BM, 2 * RNB, 0);   // A_hi [Q_hi | Q_lo]
    const uint32_t idesc_n = idesc_tf32(BM, RNB, 0);       // A_lo Q_hi
    Ring rg;
    int64_t g = 0;
    for (int64_t u = 0; u < my_tiles; ++u) {
      mbar_wait(a_ready, uint32_t(u) & 1);
      tc_fence_after();
      for (int b = 0; b < p.nblk; ++b, ++g, rg.next<RNS>()) {
        const int ab = int(g & 1);
        if (g >= 2) mbar_wait(&acc_empty[ab], uint32_t((g >> 1) - 1) & 1);
        mbar_wait(&st_full[rg.s], rg.ph);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + L::off_st + rg.s * L::per_stage);
        const uint32_t acc = tmem + (wide ? uint32_t(ab) * kAcc : kAcc1 + uint32_t(ab) * RNB);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < KC / 8; ++kk) {
            const uint32_t a_hi = tmem + kA + c * KC + 8 * kk;
            const uint64_t bq = bdesc_sw128(st + (2 * c) * L::kQ, kk);
            if (wide) mma_tf32_ts_w(acc, a_hi, bq, idesc_w, (c == 0 && kk == 0) ? 0u : 1u);
            else mma_tf32_ts_w(acc, a_hi + RP, bq, idesc_n, (c == 0 && kk == 0) ? 0u : 1u);
          }
        mma_commit_w(&acc_full[ab]);
      }
      mma_commit_w(a_free);
    }
  } else if (warp >= 2 && warp <= 5) {                 // ---------------- split A / epilogue
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    double res = 0.0, xx = 0.0;
    const float sc = p.rscale ? *p.rscale : 1.f;
    Ring rg;
    int64_t g = 0;
    for (int64_t u = 0; u < my_tiles; ++u) {
      mbar_wait(p_full, uint32_t(u) & 1);
      if (u >= 1) mbar_wait(a_free, uint32_t(u - 1) & 1);   // previous tile's MMAs done with A
      tc_fence_after();
      const float* ps = reinterpret_cast<const float*>(smem + L::off_p);
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) split_tf32(ps[c * (BM * KC) + (16 * h + q) * BM + r], hi[q], lo[q]);
          tmem_st16(lane_base + kA + c * KC + 16 * h, hi);
          tmem_st16(lane_base + kA + RP + c * KC + 16 * h, lo);
        }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_free);
      mbar_arrive(a_ready);
      for (int b = 0; b < p.nblk; ++b, ++g, rg.next<RNS>()) {
        const int ab = int(g & 1);
        mbar_wait(&st_full[rg.s], rg.ph);
        mbar_wait(&acc_full[ab], uint32_t(g >> 1) & 1);
        tc_fence_after();
        const float* xt = reinterpret_cast<const float*>(smem + L::off_st + rg.s * L::per_stage + 2 * NCH * L::kQ);
        float tr = 0.f, tx = 0.f;
#pragma unroll
        for (int cb = 0; cb < RNB / 16; ++cb) {
          uint32_t v[16], w[16], z[16];
          tmem_ld16(lane_base + uint32_t(ab) * kAcc + 16 * cb, v);           // A_hi Q_hi
          tmem_ld16(lane_base + uint32_t(ab) * kAcc + RNB + 16 * cb, w);     // A_hi Q_lo
          tmem_ld16(lane_base + kAcc1 + uint32_t(ab) * RNB + 16 * cb, z);    // A_lo Q_hi
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float x = xt[(16 * cb + q) * BM + r] * sc;
            const float d = x - (__uint_as_float(v[q]) + (__uint_as_float(w[q]) + __uint_as_float(z[q]))) * sc;
            tr = fmaf(d, d, tr);
            tx = fmaf(x, x, tx);
          }
        }
        res += double(tr);
        xx += double(tx);
        tc_fence_before();
        mbar_arrive(&acc_empty[ab]);
        mbar_arrive(&st_free[rg.s]);
      }
    }
    // CTA reduction of the 128 splitter threads -> part[blockIdx.x]
    __shared__ double red[2][4];
    for (int o = 16; o; o >>= 1) {
      res += __shfl_xor_sync(0xffffffffu, res, o);
      xx += __shfl_xor_sync(0xffffffffu, xx, o);
    }
    if (lane == 0) { red[0][q4] = res; red[1][q4] = xx; }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 64) {
      p.part[2 * blockIdx.x] = red[0][0] + red[0][1] + red[0][2] + red[0][3];
      p.part[2 * blockIdx.x + 1] = red[1][0] + red[1][1] + red[1][2] + red[1][3];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// fp16-split residual (R29 applied to a8): X^ = P Q_N^T with P (the core expanded over all but the
// last mode; |P_jr| <= ||G||, scale s from resid_scale) split as s P = P_hi + P_lo in fp16 (A in TMEM, 64 r = 32 + 32 columns) and
// Q^T as fp16 [2^14 Q_hi | 2^14 Q_lo] K-major rows (64 r = 128 B, one box per 64 i each): wide issuer
// A_hi [Q_hi | Q_lo] (N = 128), narrow issuer A_lo Q_hi (N = 64), 4 K = 16 steps per i block -- half
// the MMA instructions and half the B bytes of the 3xTF32 form per X tile.  X^ = (v + w + z) / (s 2^14).
// Gated on s: it stands down (s == 0: ||G|| zero or not finite) for residual_tc_kernel.
template <int RPP>
struct RSmemH {
  static constexpr int RP = RPP;                                  // P tile rows (64, 96 or 128)
  static constexpr int NRB = RPP / 64;                            // 64-r B boxes per piece (SW128)
  static constexpr int HALF = (RPP % 64) ? 1 : 0;                 // + one 32-r box (SW64)
  static constexpr uint32_t kP = uint32_t(RP) * BM * 4;          // raw P tile [RP r][128 j]
  static constexpr uint32_t kQ = uint32_t(RNB) * 128;            // one [64 i][64 r] fp16 box (8 KB)
  static constexpr uint32_t kXt = uint32_t(BM) * RNB * 4;        // X tile [64 i][128 j]
  static constexpr uint32_t kBst = 2 * NRB * kQ + HALF * kQ;      // [hi b0 | lo b0 | ... | hi h | lo h]
  // two rings: B slots (released by the MMAs) and X tiles (released by the epilogue, which holds an
  // X tile from the MMAs' start to the end of its differences), so the X ring gets the depth
  static constexpr int NSB = 2;
  static constexpr int NS_fit = int((227u * 1024u - 512u - kP - NSB * kBst) / kXt);
  static constexpr int NS = NS_fit > 5 ? 5 : NS_fit;               // X tiles
  static constexpr uint32_t off_p = 0;
  static constexpr uint32_t off_b = kP;
  static constexpr uint32_t off_st = off_b + NSB * kBst;
  static constexpr uint32_t off_bar = off_st + NS * kXt;
  static constexpr uint32_t bytes = off_bar + 8 * (2 * NS + 2 * NSB + 8) + 16;
  static_assert(NS >= 2 && bytes <= 227u * 1024u, "residual smem plan");
};

// K-major SWIZZLE_64B descriptor of a [rows][32 fp16] box, advanced by j k16-steps (32 B)
__device__ __forceinline__ uint64_t bdesc_sw64(uint32_t saddr, int j) {
  return sdesc(saddr + 32u * uint32_t(j), 16u, 512u) | (uint64_t(4) << 61);
}

template <int RPP>
__global__ void __launch_bounds__(NTHREADS, 1)
residual_h16_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmp,
                    const __grid_constant__ CUtensorMap tqh, const __grid_constant__ CUtensorMap tql,
                    const __grid_constant__ CUtensorMap tqh2, const __grid_constant__ CUtensorMap tql2,
                    const RParams p, const float* __restrict__ pscale) {
  using L = RSmemH<RPP>;
  constexpr int RP = L::RP, NS = L::NS, NRB = L::NRB, HALF = L::HALF, NSB = L::NSB;
  if (*pscale == 0.f) return;                          // the twin runs instead (R29)
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::off_bar);
  uint64_t* st_full = bar;
  uint64_t* st_free = bar + NS;
  uint64_t* p_full = bar + 2 * NS;
  uint64_t* p_free = bar + 2 * NS + 1;
  uint64_t* a_ready = bar + 2 * NS + 2;
  uint64_t* a_free = bar + 2 * NS + 3;
  uint64_t* acc_full = bar + 2 * NS + 4;
  uint64_t* acc_empty = bar + 2 * NS + 6;
  uint64_t* b_full = bar + 2 * NS + 8;
  uint64_t* b_free = b_full + NSB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_free + NSB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t my_tiles = (p.ntiles > blockIdx.x) ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr uint32_t kAcc = 2 * RNB;                  // [hi.hi | hi.lo] per buffer (wide issuer)
  constexpr uint32_t kAcc1 = 2 * kAcc;                // lo.hi buffers (narrow issuer)
  constexpr uint32_t kA = kAcc1 + 2 * RNB;            // A hi (RP/2 columns), then A lo (RP/2 columns)
  const int nks = (p.R + 15) / 16;                    // k-steps of 16 r (zero steps past R skipped)
  static_assert(kA + RP <= 512, "residual TMEM plan");
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&st_full[s], 1); mbar_init(&st_free[s], 128); }
    for (int s = 0; s < NSB; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_free[s], 2); }
    mbar_init(p_full, 1);
    mbar_init(p_free, 128);
    mbar_init(a_ready, 128);
    mbar_init(a_free, 2);
    for (int b = 0; b < 2; ++b) { mbar_init(&acc_full[b], 2); mbar_init(&acc_empty[b], 128); }
    fence_barrier_init();
    tma_prefetch(&tmx); tma_prefetch(&tmp); tma_prefetch(&tqh); tma_prefetch(&tql);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {                                   // ---------------- TMA producer
      Ring rg, rbg;
      int it = 0;
      const uint64_t pol = policy_evict_first();
      const uint64_t pq = policy_evict_last();
      for (int64_t u = 0; u < my_tiles; ++u) {
        const int64_t tile = blockIdx.x + u * gridDim.x;
        const int slice = p.tps ? int(tile / p.tps) : 0;
        const int j0 = int((p.tps ? tile % p.tps : tile) * BM);
        if (u >= 1) mbar_wait(p_free, uint32_t(u - 1) & 1);
        mbar_expect_tx(p_full, L::kP);
        for (int c = 0; c < RP / KC; ++c) {
          if (p.tps) tma_load_3d(smem + L::off_p + c * (BM * KC * 4), &tmp, p_full, j0, c * KC, slice);
          else tma_load_2d(smem + L::off_p + c * (BM * KC * 4), &tmp, p_full, j0, c * KC);
        }
        for (int b = 0; b < p.nblk; ++b, ++it, rg.next<NS>(), rbg.next<NSB>()) {
          // the X tile first (it has the longest way to go), then the B slot
          if (it >= NS) mbar_wait(&st_free[rg.s], rg.ph ^ 1);
          mbar_expect_tx(&st_full[rg.s], L::kXt);
          if (p.tps) tma_load_3d_hint(smem + L::off_st + rg.s * L::kXt, &tmx, &st_full[rg.s], j0, b * RNB, slice, pol);
          else tma_load_2d_hint(smem + L::off_st + rg.s * L::kXt, &tmx, &st_full[rg.s], j0, b * RNB, pol);
          if (it >= NSB) mbar_wait(&b_free[rbg.s], rbg.ph ^ 1);
          uint8_t* st = smem + L::off_b + rbg.s * L::kBst;
          mbar_expect_tx(&b_full[rbg.s], L::kBst);
#pragma unroll
          for (int rb = 0; rb < NRB; ++rb) {                                   // [Q_hi | Q_lo] adjacent:
            tma_load_2d_hint(st + 2 * rb * L::kQ, &tqh, &b_full[rbg.s], 64 * rb, b * RNB, pq);   // one N = 128
            tma_load_2d_hint(st + (2 * rb + 1) * L::kQ, &tql, &b_full[rbg.s], 64 * rb, b * RNB, pq);   // operand
          }
          if (HALF) {                                                          // r 64 NRB .. + 31 (SW64)
            tma_load_2d_hint(st + 2 * NRB * L::kQ, &tqh2, &b_full[rbg.s], 64 * NRB, b * RNB, pq);
            tma_load_2d_hint(st + 2 * NRB * L::kQ + L::kQ / 2, &tql2, &b_full[rbg.s], 64 * NRB, b * RNB, pq);
          }
        }
      }
    }
  } else if (warp == 1 || warp == 6) {                // ---------------- MMA issuers (whole warps)
    const bool wide = warp == 1;
    const uint32_t idesc = idesc_f16(BM, wide ? 2 * RNB : RNB, 0);
    Ring rbg;
    int64_t g = 0;
    for (int64_t u = 0; u < my_tiles; ++u) {
      mbar_wait(a_ready, uint32_t(u) & 1);
      tc_fence_after();
      for (int b = 0; b < p.nblk; ++b, ++g, rbg.next<NSB>()) {
        const int ab = int(g & 1);
        if (g >= 2) mbar_wait(&acc_empty[ab], uint32_t((g >> 1) - 1) & 1);
        mbar_wait(&b_full[rbg.s], rbg.ph);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + L::off_b + rbg.s * L::kBst);
        const uint32_t acc = tmem + (wide ? uint32_t(ab) * kAcc : kAcc1 + uint32_t(ab) * RNB);
#pragma unroll
        for (int kk = 0; kk < RP / 16; ++kk) {
          if (kk >= nks) break;
          const uint32_t a = tmem + kA + (wide ? 0u : uint32_t(RP / 2)) + 8 * kk;
          const uint64_t bd = kk < 4 * NRB ? bdesc_sw128(st + (kk / 4) * 2 * L::kQ, kk % 4)
                                           : bdesc_sw64(st + 2 * NRB * L::kQ, kk - 4 * NRB);
          mma_f16_ts_w(acc, a, bd, idesc, kk == 0 ? 0u : 1u);
        }
        mma_commit_w(&acc_full[ab]);
        mma_commit_w(&b_free[rbg.s]);
      }
      mma_commit_w(a_free);
    }
  } else if (warp >= 2 && warp <= 5) {                 // ---------------- split P / epilogue
    const int q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q4) << 16);
    const float sc = *pscale;                            // |sc P| < 2^14 (resid_scale)
    const float inv = 1.0f / (sc * kQScale);             // exact: powers of two
    const float rs = p.rscale ? *p.rscale : 1.f;
    const float invr = inv * rs;
    double res = 0.0, xx = 0.0;
    Ring rg;
    int64_t g = 0;
    for (int64_t u = 0; u < my_tiles; ++u) {
      mbar_wait(p_full, uint32_t(u) & 1);
      if (u >= 1) mbar_wait(a_free, uint32_t(u - 1) & 1);
      tc_fence_after();
      const float* ps = reinterpret_cast<const float*>(smem + L::off_p);
      float v[RP];
#pragma unroll
      for (int q = 0; q < RP; ++q) v[q] = ps[(q / KC) * (BM * KC) + (q % KC) * BM + r] * sc;
      uint32_t hi[RP / 2], lo[RP / 2];
#pragma unroll
      for (int c = 0; c < RP / 2; ++c) split_h16x2(v[2 * c], v[2 * c + 1], hi[c], lo[c]);
#pragma unroll
      for (int gq = 0; gq < RP / 32; ++gq) {
        tmem_st16(lane_base + kA + 16 * gq, *reinterpret_cast<const uint32_t(*)[16]>(&hi[16 * gq]));
        tmem_st16(lane_base + kA + RP / 2 + 16 * gq, *reinterpret_cast<const uint32_t(*)[16]>(&lo[16 * gq]));
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_free);
      mbar_arrive(a_ready);
      for (int b = 0; b < p.nblk; ++b, ++g, rg.next<NS>()) {
        const int ab = int(g & 1);
        mbar_wait(&st_full[rg.s], rg.ph);
        mbar_wait(&acc_full[ab], uint32_t(g >> 1) & 1);
        tc_fence_after();
        const float* xt = reinterpret_cast<const float*>(smem + L::off_st + rg.s * L::kXt);
        float tr = 0.f, tx = 0.f;
#pragma unroll
        for (int cb = 0; cb < RNB / 16; ++cb) {
          uint32_t a0[16], a1[16], a2[16];
          tmem_ld16(lane_base + uint32_t(ab) * kAcc + 16 * cb, a0);           // A_hi Q_hi
          tmem_ld16(lane_base + uint32_t(ab) * kAcc + RNB + 16 * cb, a1);     // A_hi Q_lo
          tmem_ld16(lane_base + kAcc1 + uint32_t(ab) * RNB + 16 * cb, a2);    // A_lo Q_hi
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float x = xt[(16 * cb + q) * BM + r] * rs;
            const float d = x - (__uint_as_float(a0[q]) + (__uint_as_float(a1[q]) + __uint_as_float(a2[q]))) * invr;
            tr = fmaf(d, d, tr);
            tx = fmaf(x, x, tx);
          }
        }
        res += double(tr);
        xx += double(tx);
        tc_fence_before();
        mbar_arrive(&acc_empty[ab]);
        mbar_arrive(&st_free[rg.s]);
      }
    }
    __shared__ double red[2][4];
    for (int o = 16; o; o >>= 1) {
      res += __shfl_xor_sync(0xffffffffu, res, o);
      xx += __shfl_xor_sync(0xffffffffu, xx, o);
    }
    if (lane == 0) { red[0][q4] = res; red[1][q4] = xx; }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 64) {
      p.part[2 * blockIdx.x] = red[0][0] + red[0][1] + red[0][2] + red[0][3];
      p.part[2 * blockIdx.x + 1] = red[1][0] + red[1][1] + red[1][2] + red[1][3];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// Q (In x R fp32, col-major ldq) -> fp16 [In rows][w = 64 NRB] rows of 2^14 Q_hi and of 2^14 Q_lo (r >= R zero)
__global__ void qsplit_rows_h16_kernel(const float* __restrict__ Q, int64_t In, int R, int64_t ldq,
                                       __half* __restrict__ qh, __half* __restrict__ ql, int w) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= In * w) return;
  const int64_t i = e / w;
  const int r = int(e % w);
  const float v = r < R ? Q[i + ldq * r] * kQScale : 0.f;
  const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  qh[e] = __float2half_rn(h);
  ql[e] = __float2half_rn(v - h);
}

template <int RP>
void launch_r(const Ctx& ctx, const CUtensorMap& tx, const CUtensorMap& tp, const CUtensorMap& th,
              const CUtensorMap& tl, const RParams& p, int grid) {
  using L = RSmem<RP>;
  static bool attr = false;
  if (!attr) { set_smem(residual_tc_kernel<RP>, L::bytes); attr = true; }
  launch(ctx, "residual_tc", [&] {
    residual_tc_kernel<RP><<<grid, NTHREADS, L::bytes, ctx.stream>>>(tx, tp, th, tl, p);
  });
}

__global__ void split_transpose_kernel(const float* __restrict__ Q, int64_t In, int R, int64_t ldq,
                                       float* __restrict__ hi, float* __restrict__ lo, int ldt) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;   // element (r, i) of Q^T
  if (e >= In * ldt) return;
  const int64_t i = e / ldt;
  const int r = int(e % ldt);
  const float v = r < R ? Q[i + ldq * r] : 0.f;
  uint32_t h, l;
  split_tf32(v, h, l);
  hi[e] = __uint_as_float(h);
  lo[e] = __uint_as_float(l);
}

}  // namespace

bool residual_tc(const Ctx& ctx, Arena& ws, const float* X, int64_t J, int64_t In, const float* P, int64_t ldp,
                 int R, const float* Q, int64_t ldq, double* part_out2, const float* rscale, const float* pscale,
                 int64_t nslice, int64_t sx, int64_t sp) {
  const bool sliced = nslice > 1;
  // the sliced form exists for the fp16-split kernel and its SIMT twin (R > 64: R35 runs at the sketch width)
  if (sliced && (R <= 64 || ldp != J || (sx % 4) || (sp % 4) || nslice > INT32_MAX)) return false;
  // R <= 64: the fp16-split kernel gated against the tf32 kernel; 64 < R <= 128 (the split residual
  // of reading R35 runs at the sketch width K): the fp16-split kernel gated against the SIMT kernel
  if (ctx.simt() || R < 1 || R > 128 || (R > 64 && (!pscale || !ctx.tc_h16 || ctx.resid_tf32))) return false;
  if (!aligned(X, 16) || !aligned(P, 16) || (J % 4) || (ldp % 4) || J > INT32_MAX || In > INT32_MAX) return false;
  const int rp = R <= 32 ? 32 : 64;
  CUtensorMap tx, tp, th, tl;
  {  // X(j, i) at j + J i: box (128 j, 64 i); sliced: (j, i, s) at j + J i + sx s
    const uint64_t d[3] = {uint64_t(J), uint64_t(In), uint64_t(nslice)}, s[2] = {uint64_t(J) * 4, uint64_t(sx) * 4};
    const uint32_t bx[3] = {BM, RNB, 1};
    if (!make_map(&tx, X, sliced ? 3 : 2, d, s, bx, false)) return false;
  }
  {  // P(j, r) at j + ldp r: box (128 j, 32 r) -> [32 r][128 j]
    const uint64_t d[3] = {uint64_t(J), uint64_t(R), uint64_t(nslice)}, s[2] = {uint64_t(ldp) * 4, uint64_t(sp) * 4};
    const uint32_t bx[3] = {BM, KC, 1};
    if (!make_map(&tp, P, sliced ? 3 : 2, d, s, bx, false)) return false;
  }
  RParams p;
  p.J = J; p.In = In; p.R = R;
  p.tps = sliced ? cdiv(J, BM) : 0;
  p.ntiles = cdiv(J, BM) * nslice;
  p.nblk = int(cdiv(In, RNB));
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(p.ntiles, ctx.num_sms - ctx.sm_reserve)));
  p.part = ws.alloc_n<double>(2 * grid);
  p.rscale = rscale;
  p.gate = nullptr;
  if (R <= 64) {
    // the tf32 kernel's operands first (nothing is launched unless every map is accepted):
    // Q^T hi / lo, element (r, i) at r + rp*i (pad r >= R zero)
    float* qh = ws.alloc_n<float>(In * rp);
    float* ql = ws.alloc_n<float>(In * rp);
    if (!make_b_map(&th, qh, rp, int(In), rp, RNB) || !make_b_map(&tl, ql, rp, int(In), rp, RNB)) return false;
    launch(ctx, "split_transpose", [&] {
      split_transpose_kernel<<<unsigned(cdiv(In * rp, 256)), 256, 0, ctx.stream>>>(Q, In, R, ldq, qh, ql, rp);
    });
  }
  if (pscale && ctx.tc_h16 && !ctx.resid_tf32) {
    // fp16-split form (its twin below runs instead when the P scale is 0)
    const int w = R <= 64 ? 64 : (R <= 96 ? 96 : 128);
    __half* qh = ws.alloc_n<__half>(In * w);
    __half* ql = ws.alloc_n<__half>(In * w);
    launch(ctx, "split_transpose", [&] {
      qsplit_rows_h16_kernel<<<unsigned(cdiv(In * w, 256)), 256, 0, ctx.stream>>>(Q, In, R, ldq, qh, ql, w);
    });
    CUtensorMap hh, hl, hh2, hl2;
    const uint64_t d[2] = {uint64_t(w), uint64_t(In)}, st[1] = {uint64_t(w) * 2};
    const uint32_t bx[2] = {64, uint32_t(RNB)}, bx2[2] = {32, uint32_t(RNB)};
    bool mok = make_map(&hh, qh, 2, d, st, bx, true, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_DATA_TYPE_FLOAT16) &&
               make_map(&hl, ql, 2, d, st, bx, true, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    hh2 = hh;
    hl2 = hl;
    if (mok && w == 96)
      mok = make_map(&hh2, qh, 2, d, st, bx2, false, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16) &&
            make_map(&hl2, ql, 2, d, st, bx2, false, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    if (!mok) {
      if (R > 64) return false;
    } else {
      auto go = [&](auto kern, uint32_t bytes, bool& attr) {
        if (!attr) { set_smem(kern, bytes); attr = true; }
        launch(ctx, "residual_tc", [&] {
          kern<<<grid, NTHREADS, bytes, ctx.stream>>>(tx, tp, hh, hl, hh2, hl2, p, pscale);
        });
      };
      static bool a64 = false, a96 = false, a128 = false;
      if (R <= 64) go(residual_h16_kernel<64>, RSmemH<64>::bytes, a64);
      else if (R <= 96) go(residual_h16_kernel<96>, RSmemH<96>::bytes, a96);
      else go(residual_h16_kernel<128>, RSmemH<128>::bytes, a128);
      p.gate = pscale;
    }
  }
  if (R > 64) {
    // twin: the SIMT residual into the same per-CTA pairs, run only if the P scale is 0
    residual_part(ctx, X, J, In, P, R, Q, ldq, p.part, grid, rscale, pscale, nslice, sx, sp);
  } else {
    if (rp == 32) launch_r<32>(ctx, tx, tp, th, tl, p, grid);
    else launch_r<64>(ctx, tx, tp, th, tl, p, grid);
  }
  // fixed-order final reduction of the per-CTA pairs
  reduce_pairs(ctx, p.part, grid, part_out2);
  return true;
}

}  // namespace rt
