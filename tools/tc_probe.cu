// tc_probe.cu -- standalone probes of the sm_100a building blocks used by ttm_tc.cu
// (TMEM st/ld round trip, tf32 MMA with A in TMEM and B in smem K-/MN-major SWIZZLE_NONE,
// permuted-stride TMA boxes).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17
//   -I../paper_2001_07124_b200/csrc tc_probe.cu -o tc_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_common.cuh"

using namespace rt::tc;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

// ---- probe 1: TMEM st -> ld round trip (4 warps x 32 lanes, 16 columns)
__global__ void probe_tmem(uint32_t* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&tbase, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase + (uint32_t(32 * warp) << 16);
  uint32_t v[16];
  for (int i = 0; i < 16; ++i) v[i] = 1000u * (32 * warp + lane) + i;
  tmem_st16(t, v);
  tmem_wait_st();
  uint32_t w[16];
  tmem_ld16(t, w);
  tmem_wait_ld();
  for (int i = 0; i < 16; ++i) out[(32 * warp + lane) * 16 + i] = w[i];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 32);
}

// ---- probe 2: D(128 x N) = A(128 x 8, TMEM) * B(8 x N, smem), B K-major or MN-major canonical
template <int N>
__global__ void probe_mma(const float* A, const float* B, float* D, int b_mn) {
  __shared__ __align__(1024) float bs[N * 8];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B(k, n) logical, k < 8, n < N
  for (int e = threadIdx.x; e < N * 8; e += blockDim.x) {
    const int n = e % N, k = e / N;
    const float v = B[k * N + n];
    int off;
    if (b_mn == 1) off = (n / 4) * 32 + k * 4 + (n % 4);          // (n/4)*128B + k*16B + (n%4)*4B
    else if (b_mn == 2) off = k * 32 + (((n / 4) ^ (k % 8)) * 4) + (n % 4);   // SW128 MN-major atom
    else off = (k / 4) * (N * 4) + n * 4 + (k % 4);           // (k/4)*(N*16B) + n*16B + (k%4)*4B
    bs[off] = v;
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tl = tbase + (uint32_t(32 * warp) << 16);
  // A row r = 32*warp + lane, 8 columns at col 128
  {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = i < 8 ? __float_as_uint(A[(32 * warp + lane) * 8 + i]) : 0u;
    tmem_st16(tl + 128, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint64_t bd = b_mn == 1 ? sdesc(smem_u32(bs), 128, 128) : sdesc(smem_u32(bs), N * 16, 128);
    if (b_mn == 2) bd = sdesc(smem_u32(bs), 1024, 1024) | (uint64_t(2) << 61);
    mma_tf32_ts(tbase, tbase + 128, bd, idesc_tf32(128, N, b_mn ? 1 : 0), 0);
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
// ---- probe 3: permuted-stride TMA box: Omega row-major (J x K) -> smem (n/4)*512B + j*16B + (n%4)*4B
__global__ void probe_tma(const __grid_constant__ CUtensorMap m, float* out, int j0) {
  __shared__ __align__(1024) float buf[80 * 32];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, 80 * 32 * 4);
    tma_load_3d(buf, &m, &bar, 0, j0, 0);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 80 * 32; i += blockDim.x) out[i] = buf[i];
}


// ---- probe 4: K-major SWIZZLE_128B B operand (N rows x 32 K, 128 B per row), 4 k-steps of 8
template <int N>
__global__ void probe_mma_sw128(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) float bs[N * 32];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < N * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;                 // B(k, n)
    const int chunk = k / 4, within = k % 4;
    const int off = n * 32 + ((chunk ^ (n % 8)) * 4) + within;   // row n: 128 B, 16B chunks XOR (n%8)
    bs[off] = B[k * N + n];
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
      for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(A[(32 * warp + lane) * 32 + 16 * h + i]);
      tmem_st16(tl + 128 + 16 * h, v);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t bd = sdesc(smem_u32(bs) + 32 * kk, 16, 1024) | (uint64_t(2) << 61);
      mma_tf32_ts(tbase, tbase + 128 + 8 * kk, bd, idesc_tf32(128, N, 0), kk > 0);
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

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  {
    uint32_t* d;
    CK(cudaMalloc(&d, 128 * 16 * 4));
    probe_tmem<<<1, 128>>>(d);
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> h(128 * 16);
    CK(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int i = 0; i < 16; ++i) bad += h[r * 16 + i] != 1000u * r + i;
    printf("probe_tmem: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
  }
  for (int b_mn = 0; b_mn < 3; ++b_mn) {
    constexpr int N = 32;
    std::vector<float> A(128 * 8), B(8 * N), D(128 * N), R(128 * N, 0.f);
    for (int i = 0; i < 128 * 8; ++i) A[i] = float((i * 7) % 13) - 6.f;           // tf32-exact small ints
    for (int i = 0; i < 8 * N; ++i) B[i] = float((i * 5) % 11) - 5.f;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < 8; ++k) R[r * N + n] += A[r * 8 + k] * B[k * N + n];
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dD, 0, D.size() * 4));
    probe_mma<N><<<1, 128>>>(dA, dB, dD, b_mn);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < 128 * N; ++i) bad += D[i] != R[i];
    printf("probe_mma b_mn=%d: %s (%d bad)  D[0..3]=%g %g %g %g  R=%g %g %g %g\n", b_mn, bad ? "FAIL" : "ok", bad,
           D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
  }
  {
    const int J = 100, K = 80;
    std::vector<float> O(J * K);
    for (int i = 0; i < J * K; ++i) O[i] = float(i);
    float *dO, *dout;
    CK(cudaMalloc(&dO, O.size() * 4));
    CK(cudaMalloc(&dout, 80 * 32 * 4));
    CK(cudaMemcpy(dO, O.data(), O.size() * 4, cudaMemcpyHostToDevice));
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    EncodeFn enc = (EncodeFn)fp;
    CUtensorMap m;
    cuuint64_t d[3] = {4, (cuuint64_t)J, (cuuint64_t)(K / 4)}, st[2] = {(cuuint64_t)K * 4, 16};
    cuuint32_t bx[3] = {4, 32, 20}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dO, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("probe_tma encode: %d\n", (int)r);
    if (r == CUDA_SUCCESS) {
      const int j0 = 70;  // rows 70..101: 100..101 out of bounds -> 0
      probe_tma<<<1, 128>>>(m, dout, j0);
      CK(cudaDeviceSynchronize());
      std::vector<float> h(80 * 32);
      CK(cudaMemcpy(h.data(), dout, h.size() * 4, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int n = 0; n < 80; ++n)
        for (int j = 0; j < 32; ++j) {
          const float want = (j0 + j < J) ? O[(j0 + j) * K + n] : 0.f;
          const float got = h[(n / 4) * 128 + j * 4 + (n % 4)];
          bad += got != want;
        }
      printf("probe_tma layout: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
    }
  }
  {
    constexpr int N = 80;
    std::vector<float> A(128 * 32), B(32 * N), D(128 * N), R(128 * N, 0.f);
    for (int i = 0; i < 128 * 32; ++i) A[i] = float((i * 7) % 13) - 6.f;
    for (int i = 0; i < 32 * N; ++i) B[i] = float((i * 5) % 11) - 5.f;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < 32; ++k) R[r * N + n] += A[r * 32 + k] * B[k * N + n];
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    probe_mma_sw128<N><<<1, 128>>>(dA, dB, dD);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < 128 * N; ++i) bad += D[i] != R[i];
    printf("probe_mma_sw128 K-major N=80: %s (%d bad) D0=%g R0=%g\n", bad ? "FAIL" : "ok", bad, D[0], R[0]);
  }
  {  // probe 5: how does kind::tf32 convert fp32 inputs?  D = A * I (A in TMEM, B = identity K-major)
    constexpr int N = 32;
    std::vector<float> A(128 * 8), B(8 * N, 0.f), D(128 * N);
    for (int r = 0; r < 128; ++r)
      for (int k = 0; k < 8; ++k) {
        uint32_t u = 0x3F800000u + uint32_t((r * 8 + k) * 37 % 8192) + (uint32_t(r % 7) << 13);  // 1.x with low bits
        float f; memcpy(&f, &u, 4);
        A[r * 8 + k] = (r & 1) ? -f : f;
      }
    for (int k = 0; k < 8; ++k) B[k * N + k] = 1.f;
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    probe_mma<N><<<1, 128>>>(dA, dB, dD, 0);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int trunc_ok = 0, rn_ok = 0, tot = 0;
    for (int r = 0; r < 128; ++r)
      for (int k = 0; k < 8; ++k) {
        float x = A[r * 8 + k], d = D[r * N + k];
        uint32_t u; memcpy(&u, &x, 4);
        uint32_t t = u & 0xFFFFE000u;
        uint32_t lsb = (u >> 13) & 1;
        uint32_t rn = (u + 0x0FFFu + lsb) & 0xFFFFE000u;
        float ft, fr; memcpy(&ft, &t, 4); memcpy(&fr, &rn, 4);
        trunc_ok += d == ft; rn_ok += d == fr; ++tot;
      }
    printf("probe_tf32_conversion: %d/%d match truncation, %d/%d match round-nearest-even\n", trunc_ok, tot, rn_ok, tot);
  }
  return 0;
}
