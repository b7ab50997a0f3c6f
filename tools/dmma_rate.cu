// Peak throughput probe: fp64 warp MMA (mma.sync m8n8k4 f64) vs DFMA, register operands only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_rate tools/dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int k = 0; k < 8; ++k) for (int e = 0; e < 2; ++e) c[k][e] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a0), "d"(b0));
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) for (int e = 0; e < 2; ++e) s += c[k][e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int k = 0; k < 16; ++k) c[k] = k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = fma(a, b, c[k]);
  }
  double s = 0;
  for (int k = 0; k < 16; ++k) s += c[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wpb : {4, 8, 16}) {
    const int iters = 20000;
    dmma_loop<<<sms * 2, 32 * wpb>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms * 2, 32 * wpb>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (sms * 2) * wpb;
    printf("dmma warps/cta %2d: %.1f TFLOP/s\n", wpb, flops / ms / 1e9);
    dfma_loop<<<sms * 2, 32 * wpb>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms * 2, 32 * wpb>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ff = 2.0 * 16 * iters * double(sms * 2) * wpb * 32;
    printf("dfma warps/cta %2d: %.1f TFLOP/s\n", wpb, ff / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
