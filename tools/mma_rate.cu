// mma_rate.cu -- issue-rate / throughput of tcgen05.mma kind::tf32 (and kind::f16 for a sanity
// check against the bf16 peak) for the shapes the TTM kernels use: M = 128, N in {16..256},
// A from TMEM (.ts) or shared memory (.ss), B from shared memory (K-major SW128).
// One CTA per SM, one thread issues `iters` back-to-back MMAs into one accumulator.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../paper_2001_07124_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"

using namespace rt::tc;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(2) << 61);
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, int kind) {
  if (kind == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__global__ void __launch_bounds__(128) rate_kernel(int M, int N, int iters, int ts, int kind, int nacc, int cols,
                                                   unsigned long long* cyc, int issuers = 1, int lanes = 0, int sync_every = 0) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint64_t done_bar, cbar[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc(&tbase, cols);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 4; ++b) { mbar_init(&bar[b], 1); mbar_init(&cbar[b], 1); }
    mbar_init(&done_bar, 1);
    mbar_arrive(&done_bar);   // phase 0 complete
    fence_barrier_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  const bool me = lanes ? (threadIdx.x < issuers) : ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < issuers);
  if (me) {
    const int iw = lanes ? threadIdx.x : threadIdx.x >> 5;
    // kind 0 tf32: a_fmt = b_fmt = 2 (tf32); kind 1 f16: a = b = 1 (bf16)
    const uint32_t fmt = kind == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    const uint64_t bdesc = sdesc_sw128(smem_u32(smem));
    const uint64_t adesc = sdesc_sw128(smem_u32(smem + 32768));
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tb + uint32_t((it % nacc) * N) + uint32_t(iw * N * nacc);
      const int smode = sync_every / 100, sev = sync_every % 100;
      if (sev && it % sev == 0 && (smode == 0 || smode == 2)) {
        mbar_wait(&done_bar, 0);          // already complete: the cost of a satisfied wait
        mbar_wait(&done_bar, 0);
      }
      if (sev && it % sev == 0 && (smode == 0 || smode == 3)) tc_fence_after();
      if (ts)
        mma_tf32_ts(d, tb + uint32_t(cols - 32) + uint32_t((it & 3) * 8), bdesc + uint64_t((it & 3) * 2), idesc, it >= nacc ? 1u : 0u);
      else
        mma_ss(d, adesc + uint64_t((it & 3) * 2), bdesc + uint64_t((it & 3) * 2), idesc, it >= nacc ? 1u : 0u, kind);
      if (sev && it % sev == sev - 1 && (smode == 0 || smode == 1)) { mma_commit(&cbar[iw]); mma_commit(&cbar[iw]); }
      if (sev && it % sev == sev - 1 && smode == 4) mma_commit(&cbar[iw]);
    }
    mma_commit(&bar[iw]);
    mbar_wait(&bar[iw], 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0 && iw == 0) *cyc = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tb, cols);
}

// whole warp runs the loop (descriptors warp-uniform), one elected lane issues inside the asm
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mma_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__global__ void __launch_bounds__(128) rate_uniform(int N, int iters, int per_commit, unsigned long long* cyc,
                                                    int variant = 0) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, cb, cb2[8];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&cb, 1); for (int i = 0; i < 8; ++i) mbar_init(&cb2[i], 1); fence_barrier_init(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t bdesc = (uint64_t((smem_u32(smem) >> 4) & 0x3FFF)) | (uint64_t(1) << 16) | (uint64_t(64) << 32) |
                           (uint64_t(1) << 46) | (uint64_t(2) << 61);
    const long long t0 = clock64();
    const uint64_t adesc = (uint64_t((smem_u32(smem + 32768) >> 4) & 0x3FFF)) | (uint64_t(1) << 16) | (uint64_t(64) << 32) |
                           (uint64_t(1) << 46) | (uint64_t(2) << 61);
    for (int it = 0; it < iters; ++it) {
      if (variant == 9) mma_ss_elect(tb, adesc + uint64_t((it & 3) * 2), bdesc + uint64_t((it & 3) * 2), idesc, it > 0 ? 1u : 0u);
      else mma_ts_elect(tb, tb + 256 + uint32_t((it & 3) * 8), bdesc + uint64_t((it & 3) * 2), idesc, it > 0 ? 1u : 0u);
      if (per_commit && (it % per_commit) == per_commit - 1) {
        if (variant == 0) commit_elect(&cb);
        else if (variant == 1) commit_elect(&cb2[(it / per_commit) & 7]);
        else if (variant == 2) { if ((threadIdx.x & 31) == 0) mma_commit(&cb); __syncwarp(); }
        else if (variant == 3) { commit_elect(&cb2[(it / per_commit) & 7]); commit_elect(&cb2[((it / per_commit) + 4) & 7]); }
      }
    }
    commit_elect(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tb, 512);
}

int main() {
  CK(cudaSetDevice(0));
  unsigned long long* dcyc;
  CK(cudaMalloc(&dcyc, 8));
  CK(cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 20000;
  struct C { int kind, ts, M, N, nacc, ctas, issuers = 1, lanes = 0, sync = 0; };
  C cases[] = {{1, 0, 128, 256, 1, 1}, {1, 0, 64, 256, 1, 1}, {0, 1, 128, 256, 1, 1}, {0, 1, 64, 256, 1, 1},
               {0, 0, 64, 256, 1, 1}, {0, 1, 64, 128, 1, 1}, {0, 1, 64, 80, 1, 1}, {0, 1, 128, 256, 2, 1},
               {0, 1, 128, 128, 2, 1}, {0, 1, 128, 80, 1, 2}, {0, 1, 128, 128, 1, 2}, {0, 0, 128, 128, 1, 2},
               {0, 1, 128, 128, 4, 1}, {1, 0, 128, 128, 1, 1}, {1, 0, 128, 64, 1, 1},
               {0, 1, 128, 80, 1, 1, 2}, {0, 1, 128, 112, 1, 1, 2}, {0, 1, 128, 64, 1, 4}, {0, 1, 128, 32, 1, 4},
               {0, 1, 128, 80, 1, 1, 3}, {0, 1, 128, 80, 1, 1, 3, 1}, {0, 1, 128, 32, 1, 1, 3}, {0, 1, 128, 16, 1, 1, 3},
               {0, 1, 128, 32, 1, 1, 4}, {0, 1, 128, 16, 1, 1, 5},
               {0, 1, 128, 80, 1, 1, 1, 0, 4}, {0, 1, 128, 80, 1, 1, 1, 0, 2}, {0, 1, 128, 176, 1, 1, 1, 0, 4},
               {0, 1, 128, 176, 1, 1, 2, 0, 4}, {0, 1, 128, 176, 1, 1, 2, 0, 0}, {0, 1, 128, 80, 1, 1, 2, 0, 4},
               {0, 1, 128, 80, 1, 1, 1, 0, 104}, {0, 1, 128, 80, 1, 1, 1, 0, 204}, {0, 1, 128, 80, 1, 1, 1, 0, 304},
               {0, 1, 128, 80, 1, 1, 1, 0, 404}, {0, 1, 128, 80, 1, 1, 1, 0, 416}, {0, 1, 128, 176, 1, 1, 1, 0, 0},
               {0, 1, 128, 128, 1, 1, 1, 0, 0}, {0, 1, 128, 224, 1, 1, 1, 0, 0}};
  CK(cudaFuncSetAttribute(rate_uniform, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  for (int N : {80, 176, 256})
    for (int pcv : {0, 900}) {
      const int pc = pcv % 100, var = pcv / 100;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0));
        rate_uniform<<<148, 128, 65536>>>(N, 20000, pc, dcyc, var);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long cyc;
        CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
        if (rep) printf("uniform-warp issue tf32 ts M128 N%3d commit/%d variant %d: %7.3f ms %7.1f TFLOP/s %6.1f cyc/instr\n", N, pc, var, ms,
                        2.0 * 128 * N * 8 * 20000.0 * 148 / ms / 1e9, double(cyc) / 20000);
      }
    }
  for (auto& c : cases) {
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaEventRecord(e0));
      rate_kernel<<<148 * c.ctas, 128, 65536>>>(c.M, c.N, iters, c.ts, c.kind, c.nacc, 512 / c.ctas, dcyc, c.issuers, c.lanes, c.sync);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      unsigned long long cyc;
      CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
      const int K = c.kind == 0 ? 8 : 16;
      const double flops = 2.0 * c.M * c.N * K * double(iters) * 148 * c.ctas * c.issuers;
      if (rep)
        printf("%s %s M%3d N%3d K%2d nacc=%d ctas/SM=%d issuers=%d%s sync=%d: %7.3f ms  %7.1f TFLOP/s  %6.1f cyc/instr (CTA0)\n",
               c.kind ? "f16 " : "tf32", c.ts ? "ts" : "ss", c.M, c.N, K, c.nacc, c.ctas, c.issuers, c.lanes ? "(lanes)" : "", c.sync, ms, flops / ms / 1e9,
               double(cyc) / iters);
    }
  }
  return 0;
}
