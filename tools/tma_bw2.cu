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

// 2D loads of (32 j, 128 rows) boxes (the ttm_s_tc last-mode tile) with optional L2 prefetch of
// (32, 8 rows, 16 groups) 3D boxes PD chunks ahead.  Grid (splits, row tiles); CTA owns a contiguous
// chunk range of its row tile.
__global__ void __launch_bounds__(64) pf_kernel(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3,
                                               int64_t nchunk, int pd, int use_pf, int mfast = 0, int inter = 0,
                                               int bload = 0) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int BOX = 16384 + (bload ? 10240 : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * BOX);
  uint64_t* empty = full + NSTAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t S = mfast ? gridDim.y : gridDim.x, z = mfast ? blockIdx.y : blockIdx.x, mt = mfast ? blockIdx.x : blockIdx.y;
  const int64_t per = (nchunk + S - 1) / S;
  const int64_t c0 = z * per, c1 = c0 + per < nchunk ? c0 + per : nchunk;
  const int64_t n = inter ? (nchunk - z + S - 1) / S : (c1 > c0 ? c1 - c0 : 0);
  if (warp == 0 && lane == 0) {
    if (use_pf)
      for (int64_t g = c0; g < c0 + pd && g < c1; g += 16)
        for (int rb = 0; rb < 16; ++rb) tma_prefetch_l2_3d(&m3, 0, int(mt * 128 + rb * 8), int(g));
    for (int64_t it = 0; it < n; ++it) {
      const int s = int(it % NSTAGE);
      const int64_t c = inter ? z + it * S : c0 + it;
      if (use_pf && (it % 16) == 0 && c + pd < c1)
        for (int rb = 0; rb < 16; ++rb) tma_prefetch_l2_3d(&m3, 0, int(mt * 128 + rb * 8), int(c + pd));
      if (it >= NSTAGE) mbar_wait(&empty[s], uint32_t((it / NSTAGE) - 1) & 1);
      mbar_expect_tx(&full[s], BOX);
      tma_load_2d(smem + s * BOX, &m2, &full[s], int(c * 32), int(mt * 128));
      if (bload == 1) tma_load_2d(smem + s * BOX + 16384, &m3, &full[s], int(c * 32), 0);
      if (bload == 2) tma_load_2d(smem + s * BOX + 16384, &m3, &full[s], 0, int(c * 32));
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
  {
    CUtensorMap m2, m3;
    cuuint32_t es[3] = {1, 1, 1};
    cuuint64_t d2[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t s2[1] = {(cuuint64_t)C * 4};
    cuuint32_t b2[2] = {32, 128};
    CUresult r = enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d3[3] = {32, (cuuint64_t)R, (cuuint64_t)(C / 32)};
    cuuint64_t s3[2] = {(cuuint64_t)C * 4, 128};
    cuuint32_t b3[3] = {32, 8, 16};
    r = CUresult(int(r) | int(enc(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, d3, s3, b3, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)));
    if (r) printf("encode failed\n");
    const size_t smem = size_t(NSTAGE) * 16384 + 2 * NSTAGE * 8 + 64;
    CK(cudaFuncSetAttribute(pf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int64_t nchunk = C / 32;
    CUtensorMap mb;
    {
      cuuint64_t db[2] = {(cuuint64_t)C, 80};
      cuuint64_t sb[1] = {(cuuint64_t)C * 4};
      cuuint32_t bb[2] = {32, 80};
      if (enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, db, sb, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
        printf("encode b failed\n");
    }
    const size_t smemb = size_t(NSTAGE) * (16384 + 10240) + 2 * NSTAGE * 8 + 64;
    CK(cudaFuncSetAttribute(pf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemb)));
    CUtensorMap mbr;
    {
      cuuint64_t db[2] = {80, (cuuint64_t)C};
      cuuint64_t sb[1] = {320};
      cuuint32_t bb[2] = {80, 32};
      if (enc(&mbr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, db, sb, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
        printf("encode br failed\n");
    }
    for (int bl = 0; bl < 3; ++bl)
    for (int splits : {37, 74}) {
      for (int mf = 0; mf < 4; ++mf) {
        const int pf = 0, pd = 16;
          for (int rep = 0; rep < 2; ++rep) {
            CK(cudaEventRecord(e0));
            if (mf & 1) pf_kernel<<<dim3(unsigned(R / 128), splits), 64, smemb>>>(m2, bl == 2 ? mbr : mb, nchunk, pd, pf, 1, mf >> 1, bl);
            else pf_kernel<<<dim3(splits, unsigned(R / 128)), 64, smemb>>>(m2, bl == 2 ? mbr : mb, nchunk, pd, pf, 0, mf >> 1, bl);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep)
              printf("bload=%d 2D (32j,128rows) splits=%2d %s %s: %7.3f ms %6.0f GB/s\n", bl, splits, (mf & 1) ? "mtile-fastest" : "split-fastest",
                     (mf >> 1) ? "interleaved" : "contiguous", ms, double(R) * C * 4 / ms / 1e6);
          }
      }
    }
  }
  for (auto& c : cases) {
    break;
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
