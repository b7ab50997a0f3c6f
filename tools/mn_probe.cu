// mn_probe.cu -- does tcgen05.mma kind::tf32 accept an MN-major (N contiguous) 128B-swizzled B
// operand?  D(128 x N) = A(128 x 32) * B(32 x N), 4 k-steps of 8; A in TMEM (.ts) or in smem
// K-major SW128 (.ss); B MN-major SW128: atoms of 8 K-rows x 128 B (32 N values), LBO = byte
// stride between N-atoms, SBO = byte stride between 8-row K groups.  Several descriptor variants.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../paper_2001_07124_b200/csrc mn_probe.cu -o mn_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace rt::tc;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int N = 64, KT = 32;

__device__ __forceinline__ void mma_ss_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// variant: 0 LBO=atomN stride,SBO=Kgroup stride; 1 swapped; 2 = 0 + lbo_mode bit 52
__global__ void probe(const float* A, const float* B, float* D, int ss, int variant) {
  extern __shared__ __align__(1024) float sm[];
  float* bs = sm;                  // B: (N/32) atoms-columns x (KT/8) K groups x 1 KB
  float* as = sm + N * KT;         // A: 128 rows x 32 K, K-major SW128 (row r: 128 B)
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NA = N / 32;       // atoms along N
  // B(k, n): atom (n/32, k/8), inside: row k%8 (128 B), 16B chunk ((n%32)/4 ^ (k%8)), elem n%4
  for (int e = threadIdx.x; e < N * KT; e += blockDim.x) {
    const int n = e % N, k = e / N;
    int off;
    if (variant == 3) {          // K-major SW128: row n = 128 B of K
      off = n * 32 + (((k / 4) ^ (n % 8)) * 4) + (k % 4);
    } else if (variant >= 4) {   // MN-major SWIZZLE_128B_BASE32B: atoms of 4 K-rows x 128 B, 32 B chunks ^ row
      const int atom = (k / 4) * NA + (n / 32);
      const int row = k % 4, c = (n % 32) / 8;
      off = atom * 128 + row * 32 + ((c ^ row) * 8) + (n % 8);
    } else {
      const int atom = (k / 8) * NA + (n / 32);       // K-group major, N-atom minor
      off = atom * 256 + (k % 8) * 32 + ((((n % 32) / 4) ^ (k % 8)) * 4) + (n % 4);
    }
    bs[off] = B[k * N + n];
  }
  for (int e = threadIdx.x; e < 128 * KT; e += blockDim.x) {
    const int r = e / KT, k = e % KT;
    const int off = r * 32 + (((k / 4) ^ (r % 8)) * 4) + (k % 4);
    as[off] = A[r * KT + k];
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tl = tbase + (uint32_t(32 * warp) << 16);
  {
    uint32_t v[16];
    for (int h = 0; h < 2; ++h) {
      for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(A[(32 * warp + lane) * KT + 16 * h + i]);
      tmem_st16(tl + 128 + 16 * h, v);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t lbo_n = 1024u * (KT / 8);   // N-atom stride (atoms stored K-group major -> next N atom = +1 KB?)
    (void)lbo_n;
    // with atom = kgroup*NA + natom: next N atom = +1 KB, next K group = +NA KB
    const uint32_t natom = 1024u, kgrp = 1024u * NA;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(variant == 3 ? 0 : 1) << 16) |
                           (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    for (int kk = 0; kk < KT / 8; ++kk) {
      uint64_t bd;
      const uint32_t start = smem_u32(bs) + kgrp * kk;
      if (variant == 3) bd = sdesc(smem_u32(bs) + 32 * kk, 16, 1024);
      else if (variant == 4) bd = sdesc(smem_u32(bs) + 2 * kk * NA * 512, 512, NA * 512);
      else if (variant == 5) bd = sdesc(smem_u32(bs) + 2 * kk * NA * 512, NA * 512, 512);
      else if (variant == 1) bd = sdesc(start, kgrp, natom);
      else bd = sdesc(start, natom, kgrp);
      bd |= (uint64_t(variant >= 4 ? 1 : 2) << 61);
      if (variant == 2) bd |= (uint64_t(1) << 52);
      if (ss) {
        const uint64_t ad = sdesc(smem_u32(as) + 32 * kk, 16, 1024) | (uint64_t(2) << 61);
        mma_ss_tf32(tbase, ad, bd, idesc, kk > 0);
      } else {
        mma_tf32_ts(tbase, tbase + 128 + 8 * kk, bd, idesc, kk > 0);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16(tl + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) D[(32 * warp + lane) * N + c + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

// variant 6: B (KT x N, row-major in global) loaded by TMA with SWIZZLE_128B_ATOM_32B, boxes (32 n, KT rows)
__global__ void probe_tma(const __grid_constant__ CUtensorMap mb, const float* A, float* D) {
  extern __shared__ __align__(1024) float sm[];
  float* bs = sm;
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, tbar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&tbar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&tbar, N * KT * 4);
    for (int na = 0; na < N / 32; ++na) tma_load_2d(bs + na * 32 * KT, &mb, &tbar, na * 32, 0);
  }
  mbar_wait(&tbar, 0);
  const uint32_t tl = tbase + (uint32_t(32 * warp) << 16);
  {
    uint32_t v[16];
    for (int h = 0; h < 2; ++h) {
      for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(A[(32 * warp + lane) * KT + 16 * h + i]);
      tmem_st16(tl + 128 + 16 * h, v);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    for (int kk = 0; kk < KT / 8; ++kk) {
      const uint64_t bd = sdesc(smem_u32(bs) + 1024 * kk, 32 * KT * 4, 512) | (uint64_t(1) << 61);
      mma_tf32_ts(tbase, tbase + 128 + 8 * kk, bd, idesc, kk > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16(tl + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) D[(32 * warp + lane) * N + c + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  CK(cudaSetDevice(0));
  std::vector<float> A(128 * KT), B(KT * N), D(128 * N), R(128 * N, 0.f);
  for (int i = 0; i < 128 * KT; ++i) A[i] = float((i * 7) % 13) - 6.f;
  for (int i = 0; i < KT * N; ++i) B[i] = float((i * 5) % 11) - 5.f;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < KT; ++k) R[r * N + n] += A[r * KT + k] * B[k * N + n];
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  const int smem = (N * KT + 128 * KT) * 4;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int ss = 0; ss < 2; ++ss)
    for (int variant = 0; variant < 6; ++variant) {
      CK(cudaMemset(dD, 0, D.size() * 4));
      probe<<<1, 128, smem>>>(dA, dB, dD, ss, variant);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int i = 0; i < 128 * N; ++i) bad += D[i] != R[i];
      printf("%s variant %d: %s (%d bad) D[0..2]=%g %g %g R=%g %g %g\n", ss ? "ss" : "ts", variant, bad ? "FAIL" : "ok",
             bad, D[0], D[1], D[33], R[0], R[1], R[33]);
    }
  {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    EncodeFn enc = (EncodeFn)fp;
    CUtensorMap mb;
    cuuint64_t d[2] = {(cuuint64_t)N, (cuuint64_t)KT};
    cuuint64_t st[1] = {(cuuint64_t)N * 4};
    cuuint32_t bx[2] = {32, (cuuint32_t)KT}, es[2] = {1, 1};
    CUresult r = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode ATOM_32B: %d\n", (int)r);
    CK(cudaFuncSetAttribute(probe_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, N * KT * 4));
    CK(cudaMemset(dD, 0, D.size() * 4));
    probe_tma<<<1, 128, N * KT * 4>>>(mb, dA, dD);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < 128 * N; ++i) bad += D[i] != R[i];
    printf("tma ATOM_32B + MN-major BASE32B: %s (%d bad) D[0..2]=%g %g %g\n", bad ? "FAIL" : "ok", bad, D[0], D[1], D[33]);
  }
  return 0;
}
