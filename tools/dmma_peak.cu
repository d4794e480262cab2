// Microbenchmark: fp64 tensor-core (DMMA, mma.sync f64) throughput on this GPU, alone and
// concurrently with DFMA, to decide whether the grid-touch contraction can move off the fp64 FMA pipe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// mode 0: DMMA m8n8k4 only; 1: DMMA m16n8k16 only; 2: m8n8k4 + DFMA interleaved in every warp
template <int MODE>
__global__ void kern(double* out, int iters, double a, double b) {
  double c[8][2];
  double c16[2][4];
  double x[8];
  double av[8], bv[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i][0] = c[i][1] = threadIdx.x * 1e-9 + i;
    x[i] = i;
    av[i] = a + i * 1e-3;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) bv[i] = b + i;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c16[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma884(c[i], a, b);
    }
    if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 2; ++i) dmma16816(c16[i], av, bv);
    }
    if (MODE == 2) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + x[i];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c16[i][j];
  if (s == 12345.0) out[0] = s;
}

// one warp per SM, CH independent dependent-chains: cycles per DMMA step
template <int CH>
__global__ void chain(double* out, int iters, double a, double b, long long* cyc) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x + i;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma884(c[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CH>
void run_chain(double* d, long long* cyc) {
  const int iters = 4096;
  chain<CH><<<1, 32>>>(d, iters, 0.999, 1e-3, cyc);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("1 warp, %d independent chains: %.1f cycles per chain step (%.1f cycles per DMMA)\n", CH,
         (double)h / iters, (double)h / iters / CH);
}

template <int MODE>
void run(const char* name, double* d, int sms, cudaEvent_t e0, cudaEvent_t e1) {
  for (int threads : {128, 256}) {
    int blocks = sms * (1024 / threads);
    int iters = 2048;
    kern<MODE><<<blocks, threads>>>(d, 16, 0.999, 1e-3);
    cudaEventRecord(e0);
    kern<MODE><<<blocks, threads>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double warps = (double)blocks * threads / 32;
    double mma_fma = 0, dfma = 0;
    if (MODE == 0 || MODE == 2) mma_fma = warps * iters * 8 * 256;
    if (MODE == 1) mma_fma = warps * iters * 2 * 2048;
    if (MODE == 2) dfma = (double)blocks * threads * iters * 32;
    printf("%s threads/block %d: %.3f ms; DMMA %.2f TFMA/s (%.1f FMA/clk/SM); DFMA %.2f TFMA/s; total %.2f TFLOP/s\n",
           name, threads, ms, mma_fma / ms / 1e9, mma_fma / (ms * 1e-3) / sms / 1.965e9, dfma / ms / 1e9,
           2 * (mma_fma + dfma) / ms / 1e9);
  }
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  run<0>("m8n8k4     ", d, sms, e0, e1);
  run<1>("m16n8k16   ", d, sms, e0, e1);
  run<2>("m8n8k4+DFMA", d, sms, e0, e1);
  long long* cyc;
  cudaMalloc(&cyc, 8);
  run_chain<1>(d, cyc);
  run_chain<2>(d, cyc);
  run_chain<4>(d, cyc);
  run_chain<8>(d, cyc);
  run_chain<16>(d, cyc);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return 0;
}
