// Device-resident conjugate gradients for (K + beta I) x = b, following
// cg_solve (krr.py:76-110) as called from fit (krr.py:162-167):
//   x0 = 0, r = b, p = r, rs = r.r
//   loop: Ap = K p + beta p; finite check; pAp = p.Ap (> 0, finite);
//         x += (rs/pAp) p; r -= (rs/pAp) Ap; rs_new = r.r (finite);
//         stop if sqrt(rs_new) <= tol ||b||;  p = r + (rs_new/rs) p
// Vector updates are fused with the dot products they feed; reductions are
// two-stage with a fixed grid, so results are run-to-run deterministic.
// The default solve is one CUDA graph: a conditional WHILE node whose body is the captured
// matvec + the update kernels + a one-thread decision kernel that applies the reference's
// stopping rule and breakdown checks on device scalars (cudaGraphSetConditional), so the
// iteration count is the reference's with no host round trip per iteration.  The host loop
// (one 32-byte read-back per iteration) remains as the fallback (AFS_CG_GRAPH=0).
#include <cmath>
#include <cstdlib>

#include <algorithm>
#include <cooperative_groups.h>

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
// non-finite flag (krr.py:93).  beta is read from device memory so that one captured solve
// graph serves every shift.
__global__ void __launch_bounds__(kRedThreads) k_cg_ap(double* __restrict__ ap,
                                                      const double* __restrict__ p,
                                                      const double* __restrict__ beta_d,
                                                      int64_t n, double* __restrict__ partial,
                                                      double* __restrict__ flag) {
  const double beta = *beta_d;
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

// ---- device-side loop (graph conditional node) -------------------------------------------
// ds: [0] rs  [1] pAp  [2] rs_new  [3] non-finite flag  [4] iterations  [5] status
//     [6] tol * ||b||  [7] maxiter  [8] rs_new / rs (direction update)  [9] beta
enum : int { kCgRunning = 0, kCgConverged = 1, kCgMaxiter = 2, kCgBadAp = -1, kCgBadCurv = -2,
             kCgBadRes = -3 };

__global__ void __launch_bounds__(kRedThreads) k_cg_update_dev(double* __restrict__ x,
                                                              double* __restrict__ r,
                                                              const double* __restrict__ p,
                                                              const double* __restrict__ ap,
                                                              const double* __restrict__ ds,
                                                              int64_t n, double* __restrict__ partial) {
  const double step = ds[0] / ds[1];
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

// the host loop's checks, in its order (krr.py:93-106)
__global__ void k_cg_decide(double* ds, cudaGraphConditionalHandle h) {
  const double it = ds[4] + 1.0;
  ds[4] = it;
  const double pAp = ds[1], rs_new = ds[2];
  int status = kCgRunning;
  if (ds[3] != 0.0) status = kCgBadAp;
  else if (!isfinite(pAp) || pAp <= 0.0) status = kCgBadCurv;
  else if (!isfinite(rs_new)) status = kCgBadRes;
  else if (sqrt(rs_new) <= ds[6]) status = kCgConverged;
  else if (it >= ds[7]) status = kCgMaxiter;
  if (status >= 0) {
    ds[8] = rs_new / ds[0];
    ds[0] = rs_new;
  }
  ds[5] = (double)status;
  cudaGraphSetConditional(h, status == kCgRunning ? 1u : 0u);
}

__global__ void __launch_bounds__(kRedThreads) k_cg_dir_dev(double* __restrict__ p,
                                                           const double* __restrict__ r,
                                                           const double* __restrict__ ds, int64_t n) {
  const double beta = ds[8];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

// ---- the whole CG epilogue of one iteration in one cooperative launch -----------------------
// Phase 1: Ap += beta p (Ap holds K p from the matvec), block partials of p.Ap, non-finite
// flag; grid sync; phase 2: every block reduces the partials in the same fixed order (so all
// hold the same pAp), x += (rs/pAp) p, r -= (rs/pAp) Ap, partials of r.r; grid sync; phase 3:
// every block reduces rs_new, block 0 applies the reference's checks (k_cg_decide's logic)
// and ends the WHILE loop, and while running every block updates p = r + (rs_new/rs) p.
// Replaces k_cg_ap + k_finish + k_cg_update_dev + k_finish + k_cg_decide + k_cg_dir_dev
// (six launches and one vector pass) in the whole-solve graph.  Values are bit-identical
// to the unfused kernels: the same per-element expressions and the same reduction order.
__device__ __forceinline__ double grid_partials_sum(const double* __restrict__ part, int np) {
  __shared__ double bcast;
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v += part[i];
  v = block_sum(v);
  if (threadIdx.x == 0) bcast = v;
  __syncthreads();
  const double r = bcast;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kRedThreads) k_cg_fused(double* __restrict__ x, double* __restrict__ r,
                                                         double* __restrict__ p, double* __restrict__ ap,
                                                         double* __restrict__ ds, int64_t n,
                                                         double* __restrict__ part1,
                                                         double* __restrict__ part2,
                                                         cudaGraphConditionalHandle h) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  const double beta = ds[9], rs = ds[0], it_prev = ds[4], bar = ds[6], maxit = ds[7];
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)G * blockDim.x;
  {   // phase 1 (k_cg_ap)
    double v = 0.0;
    bool bad = false;
    for (int64_t i = i0; i < n; i += stride) {
      const double pi = p[i];
      const double a = __dadd_rn(ap[i], __dmul_rn(beta, pi));
      bad |= !isfinite(a);
      ap[i] = a;
      v += pi * a;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) ds[3] = 1.0;
    v = block_sum(v);
    if (threadIdx.x == 0) part1[blockIdx.x] = v;
  }
  grid.sync();
  const double pAp = grid_partials_sum(part1, G);
  {   // phase 2 (k_cg_update_dev)
    const double step = rs / pAp;
    double v = 0.0;
    for (int64_t i = i0; i < n; i += stride) {
      x[i] = __dadd_rn(x[i], __dmul_rn(step, p[i]));
      const double ri = __dsub_rn(r[i], __dmul_rn(step, ap[i]));
      r[i] = ri;
      v += ri * ri;
    }
    v = block_sum(v);
    if (threadIdx.x == 0) part2[blockIdx.x] = v;
  }
  grid.sync();
  const double rs_new = grid_partials_sum(part2, G);
  // phase 3 (k_cg_decide + k_cg_dir_dev); every block reaches the same status
  const double it = it_prev + 1.0;
  int status = kCgRunning;
  if (ds[3] != 0.0) status = kCgBadAp;
  else if (!isfinite(pAp) || pAp <= 0.0) status = kCgBadCurv;
  else if (!isfinite(rs_new)) status = kCgBadRes;
  else if (sqrt(rs_new) <= bar) status = kCgConverged;
  else if (it >= maxit) status = kCgMaxiter;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ds[1] = pAp;
    ds[2] = rs_new;
    ds[4] = it;
    if (status >= 0) {
      ds[8] = rs_new / rs;
      ds[0] = rs_new;
    }
    ds[5] = (double)status;
    cudaGraphSetConditional(h, status == kCgRunning ? 1u : 0u);
  }
  if (status == kCgRunning) {
    const double b2 = rs_new / rs;
    for (int64_t i = i0; i < n; i += stride) p[i] = __dadd_rn(r[i], __dmul_rn(b2, p[i]));
  }
}

// grid of the fused kernel: kRedBlocks when that many blocks are co-resident (cooperative
// launch requirement), else the largest co-resident count -- fixed per device, so the
// reduction order (hence the results) is fixed too
static int cg_fused_grid() {
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, sms = 0, occ = 0, coop = 0;
    AFS_CUDA(cudaGetDevice(&dev));
    AFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    AFS_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    AFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cg_fused, kRedThreads, 0));
    grid = coop ? std::min(kRedBlocks, occ * sms) : -1;
  }
  return grid;
}

static void launch_cg_fused(afs_plan* pl, double* x, double* ds, cudaGraphConditionalHandle h,
                            cudaStream_t s) {
  CgScratch& c = pl->cg;
  const int64_t n = pl->Ns;
  double* part1 = c.partial;
  double* part2 = c.partial + kRedBlocks;
  void* args[] = {&x, &c.r, &c.p, &c.ap, &ds, (void*)&n, &part1, &part2, &h};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cg_fused_grid());
  cfg.blockDim = dim3(kRedThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AFS_CUDA(cudaLaunchKernelExC(&cfg, (const void*)k_cg_fused, args));
}

// ---- CG vector kernels on caller-owned vectors (afs_cg_vec_*, distributed drivers) --------
// ws (caller-owned device doubles, AFS_CG_WORKSPACE_DOUBLES): [0] rs  [1] pAp  [2] rs_new
// [3] non-finite flag  [9] beta  [16..16+kRedBlocks) reduction partials.  Every value
// written is a LOCAL partial over the n entries given; a point-sharded driver all-reduces
// ws[0] after init, ws[1..3] after ap and ws[2] after update (krr.py:86-109).
static_assert(16 + kRedBlocks <= AFS_CG_WORKSPACE_DOUBLES, "CG workspace too small");

__global__ void __launch_bounds__(kRedThreads) k_vec_init(const double* __restrict__ b,
                                                         double* __restrict__ x,
                                                         double* __restrict__ r,
                                                         double* __restrict__ p, int64_t n,
                                                         double* __restrict__ partial) {
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    p[i] = bi;
    v += bi * bi;
  }
  v = block_sum(v);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

__global__ void k_vec_clear(double* ws, double beta) {
  if (threadIdx.x < 16) ws[threadIdx.x] = threadIdx.x == 9 ? beta : 0.0;
}

__global__ void k_vec_roll(double* ws) { ws[0] = ws[2]; }

void cg_vec_init(const double* b, double* x, double* r, double* p, int64_t n, double beta,
                 double* ws, cudaStream_t s) {
  k_vec_clear<<<1, 32, 0, s>>>(ws, beta);
  k_vec_init<<<kRedBlocks, kRedThreads, 0, s>>>(b, x, r, p, n, ws + 16);
  k_finish<<<1, kRedThreads, 0, s>>>(ws + 16, kRedBlocks, ws);
  AFS_CUDA(cudaGetLastError());
}

void cg_vec_ap(double* ap, const double* p, int64_t n, double* ws, cudaStream_t s) {
  k_cg_ap<<<kRedBlocks, kRedThreads, 0, s>>>(ap, p, ws + 9, n, ws + 16, ws + 3);
  k_finish<<<1, kRedThreads, 0, s>>>(ws + 16, kRedBlocks, ws + 1);
  AFS_CUDA(cudaGetLastError());
}

void cg_vec_update(double* x, double* r, const double* p, const double* ap, int64_t n,
                   double* ws, cudaStream_t s) {
  k_cg_update_dev<<<kRedBlocks, kRedThreads, 0, s>>>(x, r, p, ap, ws, n, ws + 16);
  k_finish<<<1, kRedThreads, 0, s>>>(ws + 16, kRedBlocks, ws + 2);
  AFS_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(kRedThreads) k_vec_dir(double* __restrict__ p,
                                                        const double* __restrict__ r,
                                                        const double* __restrict__ ws, int64_t n) {
  const double beta = ws[2] / ws[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

void cg_vec_direction(double* p, const double* r, int64_t n, double* ws, cudaStream_t s) {
  k_vec_dir<<<kRedBlocks, kRedThreads, 0, s>>>(p, r, ws, n);
  k_vec_roll<<<1, 1, 0, s>>>(ws);
  AFS_CUDA(cudaGetLastError());
}

static void ensure_cg(afs_plan* pl) {
  CgScratch& c = pl->cg;
  if (c.n == pl->Ns) return;
  if (c.r) {
    cudaFree(c.r); cudaFree(c.p); cudaFree(c.ap); cudaFree(c.x); cudaFree(c.partial);
    cudaFree(c.scalars);
    cudaFreeHost(c.host_scalars);
    if (c.graph.exec) cudaGraphExecDestroy(c.graph.exec);
    c.graph = CgGraph{};
  }
  const size_t bytes = sizeof(double) * pl->Ns;
  AFS_CUDA(cudaMalloc(&c.r, bytes));
  AFS_CUDA(cudaMalloc(&c.p, bytes));
  AFS_CUDA(cudaMalloc(&c.ap, bytes));
  AFS_CUDA(cudaMalloc(&c.x, bytes));
  AFS_CUDA(cudaMalloc(&c.partial, sizeof(double) * 2 * kRedBlocks));
  AFS_CUDA(cudaMalloc(&c.scalars, sizeof(double) * 16));
  AFS_CUDA(cudaMallocHost(&c.host_scalars, sizeof(double) * 16));
  c.n = pl->Ns;
  pl->device_bytes += 4 * bytes + sizeof(double) * (2 * kRedBlocks + 16);
}

// Builds (once per plan) the whole-loop graph.  It works on plan-owned vectors only (x, r,
// p, Ap) with beta and the limits in device scalars, so every solve on the plan replays the
// same graph; refresh_det_windows (api.cu) drops it when the captured stage parameters
// change.  Returns false when conditional graph nodes are unavailable (host loop runs).
static bool cg_graph(afs_plan* pl, const double* b, cudaStream_t s) {
  CgScratch& c = pl->cg;
  if (c.graph.exec) return true;
  const int64_t n = pl->Ns;
  double* x = c.x;
  double* ds = c.scalars;
  // warm-up: one eager matvec performs the stages' first-use allocations and kernel
  // attributes, which must not happen inside the capture (overwrites Ap only)
  apply_stages(pl, b, n, c.ap, n, 1, s);
  cudaGraph_t g = nullptr;
  AFS_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  cudaGraphNodeParams prm = {};
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  if (e == cudaSuccess) {
    prm.type = cudaGraphNodeTypeConditional;
    prm.conditional.handle = h;
    prm.conditional.type = cudaGraphCondTypeWhile;
    prm.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &prm);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    return false;
  }
  cudaGraph_t body = prm.conditional.phGraph_out[0];
  AFS_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  try {
    apply_stages(pl, c.p, n, c.ap, n, 1, s);
    const char* fz = getenv("AFS_CG_FUSED");
    if (cg_fused_grid() > 0 && !(fz && fz[0] == '0')) {
      launch_cg_fused(pl, x, ds, h, s);   // the whole epilogue in one cooperative launch
    } else {
      k_cg_ap<<<kRedBlocks, kRedThreads, 0, s>>>(c.ap, c.p, ds + 9, n, c.partial, ds + 3);
      k_finish<<<1, kRedThreads, 0, s>>>(c.partial, kRedBlocks, ds + 1);
      k_cg_update_dev<<<kRedBlocks, kRedThreads, 0, s>>>(x, c.r, c.p, c.ap, ds, n, c.partial);
      k_finish<<<1, kRedThreads, 0, s>>>(c.partial, kRedBlocks, ds + 2);
      k_cg_decide<<<1, 1, 0, s>>>(ds, h);
      k_cg_dir_dev<<<kRedBlocks, kRedThreads, 0, s>>>(c.p, c.r, ds, n);
    }
  } catch (...) {
    cudaStreamEndCapture(s, &body);
    cudaGraphDestroy(g);
    throw;
  }
  AFS_CUDA(cudaStreamEndCapture(s, &body));
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  AFS_CUDA(e);
  c.graph.exec = exec;
  return true;
}

static void cg_solve_graph(afs_plan* pl, const double* b, double* x, double beta, double tol,
                           int maxiter, int* iters, double* resid, int* conv, cudaStream_t s,
                           double bnorm) {
  CgScratch& c = pl->cg;
  double* hs = c.host_scalars;
  double* ds = c.scalars;
  const int64_t n = pl->Ns;
  // ds[0] = rs = ||b||^2 is in place; iteration state and limits
  hs[3] = 0.0;
  hs[4] = 0.0;
  hs[5] = 0.0;
  hs[6] = tol * bnorm;
  hs[7] = (double)maxiter;
  hs[8] = 0.0;
  hs[9] = beta;
  AFS_CUDA(cudaMemcpyAsync(ds + 3, hs + 3, 7 * sizeof(double), cudaMemcpyHostToDevice, s));
  AFS_CUDA(cudaMemsetAsync(c.x, 0, sizeof(double) * n, s));
  AFS_CUDA(cudaMemcpyAsync(c.r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  AFS_CUDA(cudaMemcpyAsync(c.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  AFS_CUDA(cudaGraphLaunch(c.graph.exec, s));
  AFS_CUDA(cudaMemcpyAsync(x, c.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  AFS_CUDA(cudaMemcpyAsync(hs, ds, 9 * sizeof(double), cudaMemcpyDeviceToHost, s));
  AFS_CUDA(cudaStreamSynchronize(s));
  const int it = (int)hs[4];
  const int status = (int)hs[5];
  *iters = it;
  if (status == kCgBadAp)
    throw Error(AFS_ERR_NUMERICAL, "CG breakdown: non-finite operator output at iteration " +
                                       std::to_string(it));
  if (status == kCgBadCurv) {
    char buf[160];
    snprintf(buf, sizeof buf, "CG breakdown: non-positive curvature %.3e at iteration %d", hs[1], it);
    throw Error(AFS_ERR_NUMERICAL, buf);
  }
  if (status == kCgBadRes)
    throw Error(AFS_ERR_NUMERICAL, "CG breakdown: non-finite residual at iteration " + std::to_string(it));
  *resid = std::sqrt(hs[0]) / bnorm;
  *conv = status == kCgConverged ? 1 : 0;
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
  {   // whole solve as one graph on the plan's capturable stream, ordered with the caller's
    const char* e = getenv("AFS_CG_GRAPH");
    if (!(e && e[0] == '0')) {
      if (!pl->istream) {
        AFS_CUDA(cudaStreamCreateWithFlags(&pl->istream, cudaStreamNonBlocking));
        AFS_CUDA(cudaEventCreateWithFlags(&pl->ev_in, cudaEventDisableTiming));
        AFS_CUDA(cudaEventCreateWithFlags(&pl->ev_out, cudaEventDisableTiming));
      }
      AFS_CUDA(cudaEventRecord(pl->ev_in, s));
      AFS_CUDA(cudaStreamWaitEvent(pl->istream, pl->ev_in, 0));
      if (cg_graph(pl, b, pl->istream)) {
        cg_solve_graph(pl, b, x, beta, tol, maxiter, iters, resid, conv, pl->istream, bnorm);
        return;   // synchronised with the host; nothing left on either stream
      }
    }
  }
  AFS_CUDA(cudaMemcpyAsync(c.r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  AFS_CUDA(cudaMemcpyAsync(c.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  hs[9] = beta;
  AFS_CUDA(cudaMemcpyAsync(ds + 9, hs + 9, sizeof(double), cudaMemcpyHostToDevice, s));
  double rs = hs[0];
  for (int it = 1; it <= maxiter; ++it) {
    apply_impl(pl, c.p, n, c.ap, n, 1, s);
    k_cg_ap<<<kRedBlocks, kRedThreads, 0, s>>>(c.ap, c.p, ds + 9, n, c.partial, ds + 3);
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
