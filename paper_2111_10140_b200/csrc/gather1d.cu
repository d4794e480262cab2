// Fused interpolation of all 1-D windows (nfft.py:228-229 for each, summed in the
// reference's window order, anova.py:179-183).
//
// A 1-D window's grid is n doubles, so every 1-D window of a plan fits in shared memory at
// once.  One thread per target node walks the windows in order, evaluating the node's
// stencil from its own coordinate (no sort needed: the grid reads are shared-memory reads)
// and adding eta_l * s_l to a register copy of out[node]; the node's output is read and
// written once for all 1-D windows, coalesced, instead of one scattered read-modify-write
// per window.  Same window values (poly_weights) and cell/fraction arithmetic as the
// sorted kernels, so the spread's nx and the gather's agree bit for bit.
//
// At m = 4 on a compile-time table the window values are not evaluated per node at all
// (k_gather_1d_sub): every block folds each window's grid into per-half-cell Chebyshev tables in
// shared memory, Ghat[c][h][k] = sum_o Cc[o][k] g[c - 3 + o] (kb_cheb.inc, 12 terms), over the
// cells the target nodes occupy (the fast summation scales them into ~0.22 n cells: 6 KB per
// window, so all of C5's 20 windows stay in one pass over the nodes), and a node costs its
// table row (96 bytes) and 22 FMAs instead of 8 twelve-term polynomials.
#include <algorithm>
#include <climits>

#include "afs_internal.cuh"
#include "geometry.cuh"
#include "sliding.cuh"

namespace afs {

constexpr int kMax1d = 48;

struct Win1 {
  int feat;
  double center, scale, eta;
  int64_t grid_off;
};

struct Gather1dBatch {
  int nwin;
  Win1 w[kMax1d];
};

template <int MM, int TAB, int RG>
__global__ void __launch_bounds__(256) k_gather_1d_fused(const double* __restrict__ Z, int64_t N, int dtot,
                                                         int n, const PolyTable T, const Gather1dBatch B,
                                                         const double* __restrict__ grids,
                                                         int64_t rhs_stride, int nr,
                                                         double* __restrict__ out, int64_t ldo) {
  extern __shared__ double sg[];   // [RG][nwin][n]
  const int nw = B.nwin;
  for (int idx = threadIdx.x; idx < RG * nw * n; idx += blockDim.x) {
    const int r = idx / (nw * n), rem = idx - r * nw * n, l = rem / n, c = rem - l * n;
    sg[idx] = r < nr ? grids[r * rhs_stride + B.w[l].grid_off + c] : 0.0;
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc[RG];
#pragma unroll
    for (int r = 0; r < RG; ++r) acc[r] = r < nr ? out[r * ldo + i] : 0.0;
    const double* zrow = Z + i * dtot;
#pragma unroll 1
    for (int l = 0; l < nw; ++l) {
      const Win1& w = B.w[l];
      const double nx = __dmul_rn((double)n, scaled_coord(__ldg(zrow + w.feat), w.center, w.scale));
      const double fl = floor(nx);
      const double f = nx - fl;   // exact
      const int u = wrap_cell((int)fl, n);
      double wt[2 * MM];
      poly_weights<MM, TAB>(f, T, wt);
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const double* g = sg + (r * nw + l) * n;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 2 * MM; ++k) s = fma(wt[k], g[wrap_cell(u - MM + 1 + k, n)], s);
        acc[r] = __dadd_rn(acc[r], __dmul_rn(w.eta, s));
      }
    }
#pragma unroll
    for (int r = 0; r < RG; ++r)
      if (r < nr) out[r * ldo + i] = acc[r];
  }
}

// ---- per-cell Chebyshev tables (m = 4, compile-time KB table) ------------------------------
#ifndef AFS_G1D_THREADS
#define AFS_G1D_THREADS 512    // one block per SM (the tables take most of its shared memory); 1024 measured slower
#endif
constexpr int kMax1dSub = 32;       // windows per launch
constexpr int kMaxCells1d = 96;     // occupied cells per window the tables may cover
constexpr int kRow1d = 12;          // Chebyshev terms per half-cell (kb_cheb.inc)
constexpr int kRowPad1d = 14;       // table row stride: 112 bytes = 28 banks, so random rows spread over 8 bank groups

struct Win1s {
  int feat;
  double center, scale, eta;
  int64_t grid_off;
  int cell_lo, ncell;   // unwrapped base cells [cell_lo, cell_lo + ncell) of the target nodes
  int tab_off;          // doubles, into the block's tables
  int gs_off;           // doubles, into the block's staged grid slices
};

struct Gather1dSubBatch {
  int nwin;
  int tab_total, gs_total;
  Win1s w[kMax1dSub];
};

__device__ __forceinline__ int mod_cell(int v, int n) {
  int r = v % n;
  return r < 0 ? r + n : r;
}

// Ghat[c][h][k] = sum_o Cc[h ? 7 - o : o][k] g[c - 3 + o]: the half-cell series of tc2d.cuh in
// one dimension (h: the reflection class f > 1/2, variable u = 4 ((h ? 1 - f : f) - 1/4))
template <int TAB>
__global__ void __launch_bounds__(AFS_G1D_THREADS) k_gather_1d_sub(const double* __restrict__ Z, int64_t N, int dtot,
                                                       int n, const Gather1dSubBatch B,
                                                       const double* __restrict__ grid,
                                                       double* __restrict__ out) {
  extern __shared__ double sm[];   // Cc[8][12] | grid slices | tables
  double* cc = sm;
  double* gs = sm + 8 * kRow1d;
  double* tab = gs + B.gs_total;
  for (int i = threadIdx.x; i < 8 * kRow1d; i += blockDim.x) cc[i] = kb_cheb<TAB>(i / kRow1d, i % kRow1d);
  for (int l = 0; l < B.nwin; ++l) {   // the stencil cells of the occupied range: cell_lo - 3 ...
    const Win1s& w = B.w[l];
    for (int i = threadIdx.x; i < w.ncell + 7; i += blockDim.x)
      gs[w.gs_off + i] = __ldg(grid + w.grid_off + mod_cell(w.cell_lo - 3 + i, n));
  }
  __syncthreads();
  for (int l = 0; l < B.nwin; ++l) {
    const Win1s& w = B.w[l];
    const double* g = gs + w.gs_off;
    for (int e = threadIdx.x; e < w.ncell * 2 * kRow1d; e += blockDim.x) {
      const int k = e % kRow1d, ch = e / kRow1d, h = ch & 1, c = ch >> 1;
      double v = 0.0;
#pragma unroll
      for (int o = 0; o < 8; ++o) v = fma(cc[(h ? 7 - o : o) * kRow1d + k], g[c + o], v);
      tab[w.tab_off + ch * kRowPad1d + k] = v;
    }
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = out[i];
    const double* zrow = Z + i * dtot;
#pragma unroll 1
    for (int l = 0; l < B.nwin; ++l) {
      const Win1s& w = B.w[l];
      const double nx = __dmul_rn((double)n, scaled_coord(__ldg(zrow + w.feat), w.center, w.scale));
      const double fl = floor(nx);
      const double f = nx - fl;   // exact
      const bool refl = f > 0.5;
      const double t = 4.0 * ((refl ? __dsub_rn(1.0, f) : f) - 0.25);   // as poly_weights' x, times 4
      const int c = (int)fl - w.cell_lo;      // in [0, ncell) by gather_1d_cell_ranges
      const double2* row = reinterpret_cast<const double2*>(tab + w.tab_off + (c * 2 + (refl ? 1 : 0)) * kRowPad1d);
      // sum_k Ghat_k T_k(t), recurrence in t
      const double t2 = 2.0 * t;
      double2 cf = row[0];
      double tm = 1.0, tk = t;
      double s = fma(cf.y, t, cf.x);
#pragma unroll
      for (int j = 1; j < kRow1d / 2; ++j) {
        cf = row[j];
        double tn = fma(t2, tk, -tm);
        tm = tk;
        tk = tn;
        s = fma(cf.x, tk, s);
        tn = fma(t2, tk, -tm);
        tm = tk;
        tk = tn;
        s = fma(cf.y, tk, s);
      }
      acc = __dadd_rn(acc, __dmul_rn(w.eta, s));
    }
    out[i] = acc;
  }
}

// min / max of floor(n x~) over the target nodes of one window
__global__ void k_cell_range(const double* __restrict__ Z, int64_t N, int dtot, int feat, double center,
                             double scale, int n, int* __restrict__ lohi) {
  int lo = INT_MAX, hi = INT_MIN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)floor(__dmul_rn((double)n, scaled_coord(Z[i * dtot + feat], center, scale)));
    lo = min(lo, c);
    hi = max(hi, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(lohi, lo);
    atomicMax(lohi + 1, hi);
  }
}

void gather_1d_cell_ranges(afs_plan* p) {
  p->cell1_lo.assign(p->P, 0);
  p->cell1_cnt.assign(p->P, 0);
  if (p->window_eval != 0 || p->m != 4 || (p->kb_tab != 1 && p->kb_tab != 2)) return;
  std::vector<int> ws;
  for (int l = 0; l < p->P; ++l)
    if (p->win[l].d == 1) ws.push_back(l);
  if (ws.size() < 2) return;
  int* d = nullptr;
  AFS_CUDA(cudaMalloc(&d, sizeof(int) * 2 * ws.size()));
  std::vector<int> h(2 * ws.size());
  for (size_t i = 0; i < ws.size(); ++i) h[2 * i] = INT_MAX, h[2 * i + 1] = INT_MIN;
  try {
    AFS_CUDA(cudaMemcpy(d, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice));
    const double* Z = p->has_targets ? p->tgt : p->src;
    const int blocks = (int)std::min<int64_t>((p->Nt + 255) / 256, 148 * 4);
    for (size_t i = 0; i < ws.size(); ++i) {
      const Window& w = p->win[ws[i]];
      k_cell_range<<<std::max(1, blocks), 256>>>(Z, p->Nt, p->dtot, w.feat[0], w.center[0], w.scale, p->n,
                                                 d + 2 * i);
    }
    AFS_CUDA(cudaGetLastError());
    AFS_CUDA(cudaMemcpy(h.data(), d, sizeof(int) * h.size(), cudaMemcpyDeviceToHost));
  } catch (...) {
    cudaFree(d);
    throw;
  }
  cudaFree(d);
  for (size_t i = 0; i < ws.size(); ++i) {
    if (h[2 * i] > h[2 * i + 1]) continue;
    p->cell1_lo[ws[i]] = h[2 * i];
    p->cell1_cnt[ws[i]] = h[2 * i + 1] - h[2 * i] + 1;
  }
}

// every 1-D window has a computed cell range small enough for the tables
static bool gather_1d_sub_ok(const afs_plan* p) {
  if (p->window_eval != 0 || p->m != 4 || (p->kb_tab != 1 && p->kb_tab != 2)) return false;
  if (const char* e = getenv("AFS_GATHER1D"))
    if (e[0] == '1') return false;   // A/B hook: the 12-term per-node kernel
  if ((int)p->cell1_cnt.size() != p->P) return false;
  for (int l = 0; l < p->P; ++l)
    if (p->win[l].d == 1 && (p->cell1_cnt[l] < 1 || p->cell1_cnt[l] > kMaxCells1d)) return false;
  return true;
}

static void gather_1d_sub(afs_plan* p, const std::vector<int>& ws, double* out, int64_t ldo, int R,
                          cudaStream_t s) {
  const double* Z = p->has_targets ? p->tgt : p->src;
  const size_t budget = 190 * 1024 - sizeof(double) * 8 * kRow1d;
  size_t i0 = 0;
  while (i0 < ws.size()) {
    Gather1dSubBatch B{};
    size_t bytes = 0;
    while (i0 + B.nwin < ws.size() && B.nwin < kMax1dSub) {
      const int l = ws[i0 + B.nwin];
      const Window& w = p->win[l];
      const int nc = p->cell1_cnt[l];
      const size_t need = sizeof(double) * ((size_t)nc * 2 * kRowPad1d + nc + 8);
      if (B.nwin > 0 && bytes + need > budget) break;
      B.w[B.nwin] = Win1s{w.feat[0], w.center[0], w.scale, w.eta, w.grid_off, p->cell1_lo[l], nc,
                          B.tab_total, B.gs_total};
      B.tab_total += nc * 2 * kRowPad1d;
      B.gs_total += (nc + 7 + 1) & ~1;   // keep the tables 16-byte aligned
      bytes += need;
      ++B.nwin;
    }
    const size_t smem = sizeof(double) * (8 * kRow1d + B.gs_total + B.tab_total);
    auto launch = [&](auto k) {
      AFS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const int64_t blocks = std::min<int64_t>((p->Nt + AFS_G1D_THREADS - 1) / AFS_G1D_THREADS, 148);
      for (int r = 0; r < R; ++r)
        k<<<(unsigned)std::max<int64_t>(1, blocks), AFS_G1D_THREADS, smem, s>>>(Z, p->Nt, p->dtot, p->n, B,
                                                                    p->grids + r * p->grid_total,
                                                                    out + r * ldo);
    };
    if (p->kb_tab == 1) launch(k_gather_1d_sub<1>);
    else launch(k_gather_1d_sub<2>);
    i0 += B.nwin;
  }
}

template <int MM, int TAB, int RG>
static void launch_1d(afs_plan* p, const Gather1dBatch& B, double* out, int64_t ldo, int nr,
                      const double* grids, cudaStream_t s) {
  const double* Z = p->has_targets ? p->tgt : p->src;
  const size_t smem = sizeof(double) * RG * B.nwin * p->n;
  auto k = k_gather_1d_fused<MM, TAB, RG>;
  if (smem > 48 * 1024) AFS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t blocks = std::min<int64_t>((p->Nt + 255) / 256, 148 * 8);
  k<<<(unsigned)std::max<int64_t>(1, blocks), 256, smem, s>>>(Z, p->Nt, p->dtot, p->n, *p->poly, B, grids,
                                                              p->grid_total, nr, out, ldo);
}

template <int MM, int TAB>
static void launch_1d_rg(afs_plan* p, const Gather1dBatch& B, double* out, int64_t ldo, int R,
                         cudaStream_t s) {
  for (int r0 = 0; r0 < R; r0 += 2) {
    const int nr = std::min(2, R - r0);
    const double* g = p->grids + r0 * p->grid_total;
    if (nr == 2) launch_1d<MM, TAB, 2>(p, B, out + r0 * ldo, ldo, nr, g, s);
    else launch_1d<MM, TAB, 1>(p, B, out + r0 * ldo, ldo, nr, g, s);
  }
}

template <int MM>
static void launch_1d_tab(afs_plan* p, const Gather1dBatch& B, double* out, int64_t ldo, int R,
                          cudaStream_t s) {
  if (p->kb_tab == 1) launch_1d_rg<MM, 1>(p, B, out, ldo, R, s);
  else if (p->kb_tab == 2) launch_1d_rg<MM, 2>(p, B, out, ldo, R, s);
  else launch_1d_rg<MM, 0>(p, B, out, ldo, R, s);
}

// The fused path applies to polynomial windows when the plan has at least two 1-D windows
// (AFS_GATHER1D=0 keeps one sorted-kernel launch per window)
bool gather_1d_fusable(const afs_plan* p) {
  if (p->window_eval != 0 || !p->poly) return false;
  if (const char* e = getenv("AFS_GATHER1D"))
    if (e[0] == '0') return false;
  int n1 = 0;
  for (const Window& w : p->win) n1 += w.d == 1 ? 1 : 0;
  return n1 >= 2 && sizeof(double) * 2 * p->n <= 160 * 1024;
}

// Interpolates every 1-D window of the plan into out, in window order, onto out's current
// values (batches of windows whose grids fit in shared memory, launched in order).
void gather_1d_fused(afs_plan* p, double* out, int64_t ldo, int R, cudaStream_t s) {
  std::vector<int> ws;
  for (int l = 0; l < p->P; ++l)
    if (p->win[l].d == 1) ws.push_back(l);
  if (gather_1d_sub_ok(p)) {
    gather_1d_sub(p, ws, out, ldo, R, s);
    AFS_CUDA(cudaGetLastError());
    return;
  }
  const size_t per_win = sizeof(double) * 2 * p->n;   // RG <= 2
  const int fit = (int)std::min<size_t>(kMax1d, (160 * 1024) / per_win);
  for (size_t b0 = 0; b0 < ws.size(); b0 += fit) {
    Gather1dBatch B{};
    B.nwin = (int)std::min<size_t>(fit, ws.size() - b0);
    for (int i = 0; i < B.nwin; ++i) {
      const Window& w = p->win[ws[b0 + i]];
      B.w[i] = Win1{w.feat[0], w.center[0], w.scale, w.eta, w.grid_off};
    }
    switch (p->m) {
      case 1: launch_1d_tab<1>(p, B, out, ldo, R, s); break;
      case 2: launch_1d_tab<2>(p, B, out, ldo, R, s); break;
      case 3: launch_1d_tab<3>(p, B, out, ldo, R, s); break;
      case 4: launch_1d_tab<4>(p, B, out, ldo, R, s); break;
      case 5: launch_1d_tab<5>(p, B, out, ldo, R, s); break;
      case 6: launch_1d_tab<6>(p, B, out, ldo, R, s); break;
      case 7: launch_1d_tab<7>(p, B, out, ldo, R, s); break;
      default: launch_1d_tab<8>(p, B, out, ldo, R, s); break;
    }
  }
  AFS_CUDA(cudaGetLastError());
}

}  // namespace afs
