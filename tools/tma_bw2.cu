// tma_bw2.cu -- TMA streaming-read bandwidth of 3D-view boxes over a 2048 x 4M fp32 matrix
// (the last-mode unfolding of a 2048^3 tensor: rows 16 MB apart), no compute.
// View: dims {32, R, C/32}, strides {row = C*4, group = 128 B}, box {32, b1 rows, b2 groups}
// ("rows-middle": smem [group][rows][128 B], canonical UMMA SW128 atoms) or
// dims {32, C/32, R}, box {32, b2 groups, b1 rows} ("groups-middle": 512 B+ per row in order).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../paper_2001_07124_b200/csrc tma_bw2.cu -o tma_bw2
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace rt::tc;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int NSTAGE = 8;
// task t -> (c1, c2) box coordinates; order 0: c1 fastest, 1: c2 fastest.  per_stage boxes per stage.
__global__ void __launch_bounds__(64) bw_kernel(const __grid_constant__ CUtensorMap m, int64_t n1, int64_t n2, int b1,
                                               int b2, int order, int per_stage, int boxbytes, int64_t ntask) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int stage_bytes = per_stage * boxbytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * stage_bytes);
  uint64_t* empty = full + NSTAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t z = blockIdx.x, S = gridDim.x;
  const int64_t nstage_tasks = ntask / per_stage;
  const int64_t n = z < nstage_tasks ? (nstage_tasks - z + S - 1) / S : 0;
  if (warp == 0 && lane == 0) {
    for (int64_t it = 0; it < n; ++it) {
      const int s = int(it % NSTAGE);
      if (it >= NSTAGE) mbar_wait(&empty[s], uint32_t((it / NSTAGE) - 1) & 1);
      mbar_expect_tx(&full[s], stage_bytes);
      const int64_t st = z + it * S;
      for (int p = 0; p < per_stage; ++p) {
        const int64_t t = st * per_stage + p;
        int64_t c1, c2;
        if (order == 0) { c1 = t % n1; c2 = t / n1; } else { c2 = t % n2; c1 = t / n2; }
        tma_load_3d(smem + s * stage_bytes + p * boxbytes, &m, &full[s], 0, int(c1 * b1), int(c2 * b2));
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int64_t it = 0; it < n; ++it) {
      const int s = int(it % NSTAGE);
      mbar_wait(&full[s], uint32_t(it / NSTAGE) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
}

int main() {
  CK(cudaSetDevice(0));
  const int64_t R = 2048, C = int64_t(2048) * 2048;
  float* X;
  CK(cudaMalloc(&X, size_t(R) * C * 4));
  CK(cudaMemset(X, 0, size_t(R) * C * 4));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fp;
  struct Case { int rows_middle; int b1, b2, order, per_stage; };
  std::vector<Case> cases = {
      {1, 8, 4, 0, 4}, {1, 8, 4, 1, 4}, {1, 8, 8, 0, 2}, {1, 8, 8, 1, 2}, {1, 8, 16, 0, 1}, {1, 8, 16, 1, 1},
      {1, 16, 4, 0, 2}, {1, 16, 4, 1, 2}, {1, 4, 8, 1, 4}, {1, 32, 4, 1, 1}, {1, 128, 1, 1, 1}, {1, 128, 1, 0, 1},
      {0, 8, 4, 0, 4}, {0, 8, 4, 1, 4}, {0, 32, 4, 1, 1}, {0, 8, 16, 1, 1},
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int nsm = 148;
  for (auto& c : cases) {
    CUtensorMap m;
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r;
    if (c.rows_middle) {
      cuuint64_t d[3] = {32, (cuuint64_t)R, (cuuint64_t)(C / 32)};
      cuuint64_t st[2] = {(cuuint64_t)C * 4, 128};
      cuuint32_t bx[3] = {32, (cuuint32_t)c.b1, (cuuint32_t)c.b2};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t d[3] = {32, (cuuint64_t)(C / 32), (cuuint64_t)R};
      cuuint64_t st[2] = {128, (cuuint64_t)C * 4};
      cuuint32_t bx[3] = {32, (cuuint32_t)c.b2, (cuuint32_t)c.b1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r) { printf("encode failed %d\n", (int)r); continue; }
    const int boxbytes = 128 * c.b1 * c.b2;
    const int64_t n1 = R / c.b1, n2 = (C / 32) / c.b2;
    // rows_middle=0 swaps the roles of the coordinates in the kernel: pass (b2, b1) so c1 walks dim1
    const int64_t ntask = n1 * n2;
    const size_t smem = size_t(NSTAGE) * c.per_stage * boxbytes + 2 * NSTAGE * 8 + 64;
    if (smem > 227 * 1024) { printf("skip (smem)\n"); continue; }
    CK(cudaFuncSetAttribute(bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    for (int grid_mult = 1; grid_mult <= 2; ++grid_mult) {
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0));
        if (c.rows_middle)
          bw_kernel<<<nsm * grid_mult, 64, smem>>>(m, n1, n2, c.b1, c.b2, c.order, c.per_stage, boxbytes, ntask);
        else  // dims (32, groups, rows): coordinate 1 = group index (box b2), coordinate 2 = row (box b1)
          bw_kernel<<<nsm * grid_mult, 64, smem>>>(m, n2, n1, c.b2, c.b1, 1 - c.order, c.per_stage, boxbytes, ntask);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double bytes = double(ntask) * boxbytes;
        if (rep)
          printf("%-13s box(32,%3d rows,%2d grp) order=%s per_stage=%d grid=%dx148 box=%5dB: %7.3f ms %6.0f GB/s\n",
                 c.rows_middle ? "rows-middle" : "groups-middle", c.b1, c.b2, c.order ? "grp-fast" : "row-fast",
                 c.per_stage, grid_mult, boxbytes, ms, bytes / ms / 1e6);
      }
    }
  }
  return 0;
}
