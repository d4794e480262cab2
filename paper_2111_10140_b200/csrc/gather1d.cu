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
#include <algorithm>

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
