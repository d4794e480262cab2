// Microbenchmark: fp64 atomic-add throughput on this GPU (SURVEY §8(d) asks for it next to the
// fp64 peak): RED.E.ADD.F64 into an L2-resident global array (the spread's grid flushes) and
// shared-memory fp64 atomics, with spread (conflict-free) and colliding addresses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/atomic_peak tools/atomic_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void red_global(double* g, long long cells, int iters, int stride_mix) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long idx = (tid * stride_mix) % cells;
  for (int it = 0; it < iters; ++it) {
    atomicAdd(g + idx, 1.0);
    idx += 1 + (it & 7) * 97;
    if (idx >= cells) idx -= cells;
  }
}

__global__ void red_shared(double* out, int iters, int spread) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0.0;
  __syncthreads();
  int idx = spread ? (threadIdx.x * 33) & 4095 : (threadIdx.x & 7);
  for (int it = 0; it < iters; ++it) {
    atomicAdd(s + idx, 1.0);
    idx = spread ? ((idx + 64) & 4095) : idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const long long cells = 128LL * 128 * 128 * 3;   // 50 MB: C2's three 3-D grids, L2-resident
  double* g;
  cudaMalloc(&g, sizeof(double) * cells);
  cudaMemset(g, 0, sizeof(double) * cells);
  double* o;
  cudaMalloc(&o, sizeof(double) * sms * 64);
  const int threads = 256, blocks = sms * 8, iters = 512;
  float ms;
  red_global<<<blocks, threads>>>(g, cells, 8, 1);
  cudaEventRecord(e0);
  red_global<<<blocks, threads>>>(g, cells, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * iters;
  printf("global fp64 RED, consecutive addresses (50 MB L2-resident array): %.1f G atomics/s\n",
         ops / ms / 1e6);
  red_global<<<blocks, threads>>>(g, cells, 8, 7919);
  cudaEventRecord(e0);
  red_global<<<blocks, threads>>>(g, cells, iters, 7919);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("global fp64 RED, scattered addresses: %.1f G atomics/s\n", ops / ms / 1e6);
  for (int spread : {1, 0}) {
    red_shared<<<blocks, threads>>>(o, 8, spread);
    cudaEventRecord(e0);
    red_shared<<<blocks, threads>>>(o, iters * 4, spread);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double sops = (double)blocks * threads * iters * 4;
    printf("shared fp64 atomicAdd, %s: %.1f G atomics/s (%.1f per clk per SM at 1.965 GHz)\n",
           spread ? "distinct addresses" : "8 addresses per block", sops / ms / 1e6,
           sops / (ms * 1e-3) / sms / 1.965e9);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error: %s\n", cudaGetErrorString(e));
  return 0;
}
