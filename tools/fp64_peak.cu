// Microbenchmark: sustained DFMA throughput and smem LDS.128 rate on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) {
    int blocks = sms * (2048 / threads);
    int iters = 4096;
    dfma_loop<<<blocks, threads>>>(d, 16, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * threads * iters * 16;
    printf("threads/block %d: %.2f TFMA/s = %.2f TFLOP/s fp64 (%.1f FMA/clk/SM at 1.965 GHz)\n", threads,
           fma / ms / 1e9, 2 * fma / ms / 1e9, fma / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
