// f16_probe.cu -- layout probe for a kind::f16 variant of the TS-mode TTM kernels:
// D(128 x N) fp32 = A(128 x 32) * B(32 x N), A fp16 in TMEM (two k-elements per 32-bit column,
// variants below), B fp16 row-major in global (k rows, n contiguous) loaded by TMA with
// SWIZZLE_128B as MN-major atoms of 8 k-rows x 128 B (64 n); 2 k-steps of 16.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../paper_2001_07124_b200/csrc f16_probe.cu -o f16_probe -lcuda
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace rt::tc;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int N = 128, KT = 32;

__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// avar: 0 = column c holds (k = 2c, 2c+1) (low half = even k); 1 = column c holds (k = c, c + 8) per 16-k step
// bvar: 0 = LBO 4 KB (N atoms), SBO 1 KB (8-row k groups); 1 = swapped
__global__ void probe(const __grid_constant__ CUtensorMap mb, const __half* A, float* D, int avar, int bvar) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, tbar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&tbar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&tbar, N * KT * 2);
    for (int na = 0; na < N / 64; ++na) tma_load_2d(sm + na * KT * 128, &mb, &tbar, na * 64, 0);
  }
  mbar_wait(&tbar, 0);
  const int r = 32 * warp + lane;
  const uint32_t tl = tbase + (uint32_t(32 * warp) << 16);
  {
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) {
      int k0, k1;
      if (avar == 0) { k0 = 2 * c; k1 = 2 * c + 1; }
      else { const int s = c / 8, cc = c % 8; k0 = 16 * s + cc; k1 = 16 * s + cc + 8; }
      const __half2 h = __halves2half2(A[r * KT + k0], A[r * KT + k1]);
      v[c] = *reinterpret_cast<const uint32_t*>(&h);
    }
    tmem_st16(tl + 128, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | (1u << 16) | (uint32_t(N >> 3) << 17) |
                           (uint32_t(128 >> 4) << 24);
    for (int kk = 0; kk < KT / 16; ++kk) {
      const uint32_t lbo = bvar == 0 ? KT * 128 : 1024, sbo = bvar == 0 ? 1024 : KT * 128;
      const uint64_t bd = sdesc(smem_u32(sm) + 2048 * kk, lbo, sbo) | (uint64_t(2) << 61);
      mma_f16_ts(tbase, tbase + 128 + 8 * kk, bd, idesc, kk > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16(tl + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) D[r * N + c + i] = __uint_as_float(v[i]);
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
  std::vector<__half> A(128 * KT), B(KT * N);
  std::vector<float> Af(128 * KT), Bf(KT * N), D(128 * N), R(128 * N, 0.f);
  for (int i = 0; i < 128 * KT; ++i) { Af[i] = float((i * 7) % 13) - 6.f; A[i] = __float2half(Af[i]); }
  for (int i = 0; i < KT * N; ++i) { Bf[i] = float((i * 5) % 11) - 5.f; B[i] = __float2half(Bf[i]); }
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < KT; ++k) R[r * N + n] += Af[r * KT + k] * Bf[k * N + n];
  __half *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, A.size() * 2));
  CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fp;
  CUtensorMap mb;
  cuuint64_t d[2] = {(cuuint64_t)N, (cuuint64_t)KT};
  cuuint64_t st[1] = {(cuuint64_t)N * 2};
  cuuint32_t bx[2] = {64, (cuuint32_t)KT}, es[2] = {1, 1};
  CUresult rr = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dB, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rr != CUDA_SUCCESS) { printf("encode failed %d\n", int(rr)); return 1; }
  const int smem = N * KT * 2 + 1024;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int avar = 0; avar < 2; ++avar)
    for (int bvar = 0; bvar < 2; ++bvar) {
      CK(cudaMemset(dD, 0, D.size() * 4));
      probe<<<1, 128, smem>>>(mb, dA, dD, avar, bvar);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int i = 0; i < 128 * N; ++i) bad += D[i] != R[i];
      printf("avar %d bvar %d: %s (%d bad) D[0,1,65]=%g %g %g R=%g %g %g\n", avar, bvar, bad ? "FAIL" : "ok", bad, D[0],
             D[1], D[65], R[0], R[1], R[65]);
    }
  return 0;
}
