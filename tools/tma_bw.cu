// tma_bw.cu -- TMA streaming-read bandwidth of the X tile shapes used by the TTM kernels
// (no compute: a producer lane issues boxes into an 8-stage ring, a consumer warp releases them).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../paper_2001_07124_b200/csrc tma_bw.cu -o tma_bw
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_common.cuh"

using namespace rt::tc;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Pat {
  int rank;            // 2 or 3
  int64_t ntask;       // tasks per tile-row group
  int mode;            // 0: (c0 = task*s0, c1 = m*s1)  1: (c0 = m*s0, c1 = task*s1)  2: 3D (task*32 % a, m*128, task*32/a)
  int64_t a;
  int inter;           // interleave tasks across CTAs with the same m
  int boxbytes;
  int group;           // issue loads in groups of `group` consecutive tasks
};

constexpr int NSTAGE = 8;
__global__ void __launch_bounds__(64) tma_bw_kernel(const __grid_constant__ CUtensorMap m, Pat p, int s0, int s1) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * p.boxbytes);
  uint64_t* empty = full + NSTAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t z = blockIdx.x, S = gridDim.x, mt = blockIdx.y;
  const int64_t per = (p.ntask + S - 1) / S;
  const int64_t n = p.inter ? (z < p.ntask ? (p.ntask - z + S - 1) / S : 0) : (z * per < p.ntask ? (per < p.ntask - z * per ? per : p.ntask - z * per) : 0);
  if (warp == 0 && lane == 0) {
    for (int64_t it = 0; it < n; ++it) {
      const int s = int(it % NSTAGE);
      if (it >= NSTAGE && (p.group <= 1 || it % p.group == 0))
        for (int g = 0; g < (p.group > 1 ? p.group : 1) && it + g < n; ++g) {
          const int64_t i2 = it + g;
          mbar_wait(&empty[i2 % NSTAGE], uint32_t((i2 / NSTAGE) - 1) & 1);
        }
      const int64_t task = p.inter ? z + it * S : z * per + it;
      mbar_expect_tx(&full[s], p.boxbytes);
      void* dst = smem + s * p.boxbytes;
      if (p.mode == 0) tma_load_2d(dst, &m, &full[s], int(task * s0), int(mt * s1));
      else if (p.mode == 1) tma_load_2d(dst, &m, &full[s], int(mt * s0), int(task * s1));
      else if (p.mode == 2) tma_load_3d(dst, &m, &full[s], int((task * 32) % p.a), int(mt * 128), int((task * 32) / p.a));
      else tma_load_3d(dst, &m, &full[s], 0, int(mt * 32), int(task * 4));   // mode 3: (j%32, row, j/32) view
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
  const size_t N = size_t(2048) * 2048 * 2048;
  float* X;
  CK(cudaMalloc(&X, N * 4));
  CK(cudaMemset(X, 0, N * 4));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fp;
  auto mk = [&](int rank, std::vector<cuuint64_t> d, std::vector<cuuint64_t> st, std::vector<cuuint32_t> bx, bool sw) {
    CUtensorMap m;
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, X, d.data(), st.data(), bx.data(), es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode failed %d\n", (int)r);
    return m;
  };
  const int64_t I = 2048, J = I * I;
  struct Case { const char* name; CUtensorMap m; Pat p; int s0, s1; int mt; int splits; };
  std::vector<Case> cases;
  // mode 2 (last): X[j + J i], box (32 j, 128 i)
  for (int inter = 0; inter < 2; ++inter) {
    Case c{inter ? "mode2 box(32j,128i) interleaved" : "mode2 box(32j,128i) contiguous",
           mk(2, {(cuuint64_t)J, (cuuint64_t)I}, {(cuuint64_t)J * 4}, {32, 128}, true), {}, 32, 128, 16, 37};
    c.p = Pat{2, J / 32, 0, 0, inter, 16384, 1};
    cases.push_back(c);
  }
  {  // mode 2, groups of 4 consecutive boxes issued back to back
    Case c{"mode2 box(32j,128i) grouped4", mk(2, {(cuuint64_t)J, (cuuint64_t)I}, {(cuuint64_t)J * 4}, {32, 128}, true), {},
           32, 128, 16, 37};
    c.p = Pat{2, J / 32, 0, 0, 0, 16384, 4};
    cases.push_back(c);
  }
  {  // mode 2 via a 3D view (j%32, row, j/32): box (32, 32, 4) = 32 rows x 512 B, 128B swizzle
    Case c{"mode2 view box(32,32rows,4)", mk(3, {32, (cuuint64_t)I, (cuuint64_t)(J / 32)}, {(cuuint64_t)J * 4, 128}, {32, 32, 4}, true), {},
           0, 0, 64, 9};
    c.p = Pat{3, J / 128, 3, 0, 1, 16384, 1};
    cases.push_back(c);
  }
  {  // mode 2 with 512 B per row: box (128 j, 32 i)
    Case c{"mode2 box(128j,32i)", mk(2, {(cuuint64_t)J, (cuuint64_t)I}, {(cuuint64_t)J * 4}, {128, 32}, false), {},
           128, 32, 64, 9};
    c.p = Pat{2, J / 128, 0, 0, 1, 16384, 1};
    cases.push_back(c);
  }
  {  // mode 1: 3D (a=2048, I, b) box (32, 128, 1)
    Case c{"mode1 box(32a,128i,1)", mk(3, {(cuuint64_t)I, (cuuint64_t)I, (cuuint64_t)I}, {(cuuint64_t)I * 4, (cuuint64_t)I * I * 4}, {32, 128, 1}, true), {}, 0, 0, 16, 37};
    c.p = Pat{3, J / 32, 2, I, 1, 16384, 1};
    cases.push_back(c);
  }
  {  // mode 0: 2D (I, J) box (128 i, 32 j)
    Case c{"mode0 box(128i,32j)", mk(2, {(cuuint64_t)I, (cuuint64_t)J}, {(cuuint64_t)I * 4}, {128, 32}, false), {}, 128, 32, 16, 37};
    c.p = Pat{2, J / 32, 1, 0, 1, 16384, 1};
    cases.push_back(c);
  }
  {  // contiguous: rows of 128 floats: 2D (128? ) -> view X as (32 floats, N/32 rows) box (32, 128)
    Case c{"contiguous 16KB boxes", mk(2, {32, (cuuint64_t)(N / 32)}, {128}, {32, 128}, true), {}, 0, 128, 1, 592};
    c.p = Pat{2, (int64_t)(N / 32 / 128), 1, 0, 1, 16384, 1};
    cases.push_back(c);
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (auto& c : cases) {
    const size_t smem = NSTAGE * c.p.boxbytes + 2 * NSTAGE * 8 + 64;
    CK(cudaFuncSetAttribute(tma_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaEventRecord(e0));
      tma_bw_kernel<<<dim3(c.splits, c.mt), 64, smem>>>(c.m, c.p, c.s0, c.s1);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double bytes = double(c.p.ntask) * c.p.boxbytes * c.mt;
      if (rep) printf("%-40s %8.3f ms  %7.0f GB/s\n", c.name, ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
