// Device-resident conjugate gradients for (K + beta I) x = b, following
// cg_solve (krr.py:76-110) as called from fit (krr.py:162-167):
//   x0 = 0, r = b, p = r, rs = r.r
//   loop: Ap = K p + beta p; finite check; pAp = p.Ap (> 0, finite);
//         x += (rs/pAp) p; r -= (rs/pAp) Ap; rs_new = r.r (finite);
//         stop if sqrt(rs_new) <= tol ||b||;  p = r + (rs_new/rs) p
// Vector updates are fused with the dot products they feed; reductions are
// two-stage with a fixed grid, so results are run-to-run deterministic.
// One 32-byte host read-back per iteration keeps the stopping rule (and the
// iteration count) identical to the reference's host loop.
#include <cmath>

#include "afs_internal.cuh"

namespace afs {

constexpr int kRedBlocks = 592;   // 4 x 148 SMs
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double warp_part[kRedThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) warp_part[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < (kRedThreads / 32) ? warp_part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;   // valid in thread 0
}

__global__ void __launch_bounds__(kRedThreads) k_dot(const double* __restrict__ a,
                                                    const double* __restrict__ b, int64_t n,
                                                    double* __restrict__ partial) {
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v += a[i] * b[i];
  v = block_sum(v);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

__global__ void __launch_bounds__(kRedThreads) k_finish(const double* __restrict__ partial,
                                                       int np, double* __restrict__ dst) {
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v += partial[i];
  v = block_sum(v);
  if (threadIdx.x == 0) *dst = v;
}

// Ap <- K p + beta p  (the reference's `op.apply(v) + lam * v`), partial p.Ap,
// non-finite flag (krr.py:93).
__global__ void __launch_bounds__(kRedThreads) k_cg_ap(double* __restrict__ ap,
                                                      const double* __restrict__ p, double beta,
                                                      int64_t n, double* __restrict__ partial,
                                                      double* __restrict__ flag) {
  double v = 0.0;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double pi = p[i];
    const double a = __dadd_rn(ap[i], __dmul_rn(beta, pi));
    bad |= !isfinite(a);
    ap[i] = a;
    v += pi * a;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1.0;
  v = block_sum(v);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

// x += step p; r -= step Ap with step = rs / pAp (pAp read on device), partial r.r
__global__ void __launch_bounds__(kRedThreads) k_cg_update(double* __restrict__ x,
                                                          double* __restrict__ r,
                                                          const double* __restrict__ p,
                                                          const double* __restrict__ ap,
                                                          double rs, const double* __restrict__ pAp,
                                                          int64_t n, double* __restrict__ partial) {
  const double step = rs / *pAp;
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(step, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(step, ap[i]));
    r[i] = ri;
    v += ri * ri;
  }
  v = block_sum(v);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

// p <- r + (rs_new/rs) p
__global__ void __launch_bounds__(kRedThreads) k_cg_dir(double* __restrict__ p,
                                                       const double* __restrict__ r, double beta,
                                                       int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

static void ensure_cg(afs_plan* pl) {
  CgScratch& c = pl->cg;
  if (c.n == pl->Ns) return;
  if (c.r) {
    cudaFree(c.r); cudaFree(c.p); cudaFree(c.ap); cudaFree(c.partial); cudaFree(c.scalars);
    cudaFreeHost(c.host_scalars);
  }
  const size_t bytes = sizeof(double) * pl->Ns;
  AFS_CUDA(cudaMalloc(&c.r, bytes));
  AFS_CUDA(cudaMalloc(&c.p, bytes));
  AFS_CUDA(cudaMalloc(&c.ap, bytes));
  AFS_CUDA(cudaMalloc(&c.partial, sizeof(double) * kRedBlocks));
  AFS_CUDA(cudaMalloc(&c.scalars, sizeof(double) * 8));
  AFS_CUDA(cudaMallocHost(&c.host_scalars, sizeof(double) * 8));
  c.n = pl->Ns;
  pl->device_bytes += 3 * bytes + sizeof(double) * (kRedBlocks + 8);
}

void cg_solve_impl(afs_plan* pl, const double* b, double* x, double beta, double tol,
                   int maxiter, int* iters, double* resid, int* conv, cudaStream_t s) {
  if (pl->has_targets)
    throw Error(AFS_ERR_VALIDATION, "cg_solve needs a square operator (no separate targets)");
  if (maxiter < 1) throw Error(AFS_ERR_VALIDATION, "maxiter must be at least 1");
  ensure_cg(pl);
  CgScratch& c = pl->cg;
  const int64_t n = pl->Ns;
  double* hs = c.host_scalars;
  double* ds = c.scalars;   // [0] bnorm^2/rs0, [1] pAp, [2] rs_new, [3] nonfinite flag

  AFS_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  AFS_CUDA(cudaMemsetAsync(ds, 0, sizeof(double) * 8, s));
  k_dot<<<kRedBlocks, kRedThreads, 0, s>>>(b, b, n, c.partial);
  k_finish<<<1, kRedThreads, 0, s>>>(c.partial, kRedBlocks, ds);
  AFS_CUDA(cudaMemcpyAsync(hs, ds, sizeof(double), cudaMemcpyDeviceToHost, s));
  AFS_CUDA(cudaStreamSynchronize(s));
  const double bnorm = std::sqrt(hs[0]);
  *iters = 0;
  *resid = 0.0;
  *conv = 1;
  if (bnorm == 0.0) return;
  AFS_CUDA(cudaMemcpyAsync(c.r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  AFS_CUDA(cudaMemcpyAsync(c.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  double rs = hs[0];
  for (int it = 1; it <= maxiter; ++it) {
    apply_impl(pl, c.p, n, c.ap, n, 1, s);
    k_cg_ap<<<kRedBlocks, kRedThreads, 0, s>>>(c.ap, c.p, beta, n, c.partial, ds + 3);
    k_finish<<<1, kRedThreads, 0, s>>>(c.partial, kRedBlocks, ds + 1);
    k_cg_update<<<kRedBlocks, kRedThreads, 0, s>>>(x, c.r, c.p, c.ap, rs, ds + 1, n, c.partial);
    k_finish<<<1, kRedThreads, 0, s>>>(c.partial, kRedBlocks, ds + 2);
    AFS_CUDA(cudaMemcpyAsync(hs + 1, ds + 1, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    AFS_CUDA(cudaStreamSynchronize(s));
    const double pAp = hs[1], rs_new = hs[2];
    *iters = it;
    if (hs[3] != 0.0)
      throw Error(AFS_ERR_NUMERICAL, "CG breakdown: non-finite operator output at iteration " +
                                         std::to_string(it));
    if (!std::isfinite(pAp) || pAp <= 0.0) {
      char buf[160];
      snprintf(buf, sizeof buf, "CG breakdown: non-positive curvature %.3e at iteration %d", pAp,
               it);
      throw Error(AFS_ERR_NUMERICAL, buf);
    }
    if (!std::isfinite(rs_new))
      throw Error(AFS_ERR_NUMERICAL,
                  "CG breakdown: non-finite residual at iteration " + std::to_string(it));
    if (std::sqrt(rs_new) <= tol * bnorm) {
      *resid = std::sqrt(rs_new) / bnorm;
      *conv = 1;
      return;
    }
    k_cg_dir<<<kRedBlocks, kRedThreads, 0, s>>>(c.p, c.r, rs_new / rs, n);
    rs = rs_new;
  }
  AFS_CUDA(cudaGetLastError());
  *iters = maxiter;
  *resid = std::sqrt(rs) / bnorm;
  *conv = 0;
}

}  // namespace afs
