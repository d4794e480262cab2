// NFFT interpolation (nfft.py:228-229) for every window, accumulated across
// windows in the reference's fixed order (anova.py:179-183):
//     out_i <- out_i + eta_l * sum_stencil g_l[cell] * w(cell)
//
// v1 kernel: one thread per target node, all windows and all right-hand sides
// in one launch; the stencil weights are computed once per (node, window) and
// reused across right-hand sides.  Deterministic (no atomics).
#include <algorithm>

#include "afs_internal.cuh"
#include "sliding.cuh"
#include "tc2d.cuh"
#include "tc3d.cuh"

namespace afs {

template <int D, int MM>
__device__ __forceinline__ void window_interp(const double* __restrict__ zrow, const Window& w,
                                              int n, double b, const double* __restrict__ grids,
                                              int64_t rhs_stride, int R, double* acc) {
  double wt[D][2 * MM];
  int ix[D][2 * MM];
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const double xs = scaled_coord(zrow[w.feat[t]], w.center[t], w.scale);
    stencil_1d<MM>(xs, n, b, wt[t], ix[t]);
  }
  for (int r = 0; r < R; ++r) {
    const double* g = grids + r * rhs_stride + w.grid_off;
    double s = 0.0;
    if (D == 1) {
#pragma unroll
      for (int o0 = 0; o0 < 2 * MM; ++o0) s += g[ix[0][o0]] * wt[0][o0];
    } else if (D == 2) {
#pragma unroll 1
      for (int o0 = 0; o0 < 2 * MM; ++o0) {
        const double* row = g + (int64_t)ix[0][o0] * n;
#pragma unroll
        for (int o1 = 0; o1 < 2 * MM; ++o1)
          s += row[ix[D - 1][o1]] * __dmul_rn(wt[0][o0], wt[D - 1][o1]);
      }
    } else {
#pragma unroll 1
      for (int o0 = 0; o0 < 2 * MM; ++o0) {
        const int64_t p0 = (int64_t)ix[0][o0] * n;
#pragma unroll 1
        for (int o1 = 0; o1 < 2 * MM; ++o1) {
          const double* line = g + (p0 + ix[1 % D][o1]) * n;
          const double w01 = __dmul_rn(wt[0][o0], wt[1 % D][o1]);
#pragma unroll
          for (int o2 = 0; o2 < 2 * MM; ++o2)
            s += line[ix[D - 1][o2]] * __dmul_rn(w01, wt[D - 1][o2]);
        }
      }
    }
    acc[r] = __dadd_rn(acc[r], __dmul_rn(w.eta, s));
  }
}

#define AFS_GATHER_RCHUNK 8

template <int MM>
__global__ void __launch_bounds__(128) k_gather_simple(const double* __restrict__ Z, int64_t N,
                                                       int dtot, const Window* __restrict__ wins,
                                                       int l0, int l1, int n, double b,
                                                       const double* __restrict__ grids,
                                                       int64_t rhs_stride, int R,
                                                       double* __restrict__ out, int64_t ldo) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double* zrow = Z + i * dtot;
  for (int r0 = 0; r0 < R; r0 += AFS_GATHER_RCHUNK) {
    const int rc = min(AFS_GATHER_RCHUNK, R - r0);
    double acc[AFS_GATHER_RCHUNK];
#pragma unroll
    for (int r = 0; r < AFS_GATHER_RCHUNK; ++r) acc[r] = r < rc ? out[(r0 + r) * ldo + i] : 0.0;
    const double* gr = grids + r0 * rhs_stride;
    for (int l = l0; l < l1; ++l) {
      const Window w = wins[l];
      if (w.d == 1)
        window_interp<1, MM>(zrow, w, n, b, gr, rhs_stride, rc, acc);
      else if (w.d == 2)
        window_interp<2, MM>(zrow, w, n, b, gr, rhs_stride, rc, acc);
      else
        window_interp<3, MM>(zrow, w, n, b, gr, rhs_stride, rc, acc);
    }
    for (int r = 0; r < rc; ++r) out[(r0 + r) * ldo + i] = acc[r];
  }
}

// v1 interpolation of windows [l0, l1) added onto out (exact-mirror path / fallback)
static void gather_v1(afs_plan* p, int l0, int l1, double* out, int64_t ldo, int R, cudaStream_t s) {
  const double* Z = p->has_targets ? p->tgt : p->src;
  const int64_t N = p->Nt;
  const int threads = 128;
  const int64_t blocks = (N + threads - 1) / threads;
#define AFS_G(MM)                                                                              \
  k_gather_simple<MM><<<blocks, threads, 0, s>>>(Z, N, p->dtot, p->d_win, l0, l1, p->n, p->b, \
                                                 p->grids, p->grid_total, R, out, ldo)
  switch (p->m) {
    case 1: AFS_G(1); break;
    case 2: AFS_G(2); break;
    case 3: AFS_G(3); break;
    case 4: AFS_G(4); break;
    case 5: AFS_G(5); break;
    case 6: AFS_G(6); break;
    case 7: AFS_G(7); break;
    default: AFS_G(8); break;
  }
#undef AFS_G
}

static bool gather_v2_window(afs_plan* p, int l, double* out, int64_t ldo, int R, cudaStream_t s) {
  if (p->window_eval != 0) return false;
  const Window& w = p->win[l];
  // the target side, or a gather-only layout of the sources (api.cu), else the source side
  const SortedSide& sv = p->tgt_side[l] ? *p->tgt_side[l] : *p->src_side[l];
  if (sv.tc && w.d == 3)
    return launch_gather_tc3(sv, w, p->n, p->kb_tab, p->grids, p->grid_total, R, out, ldo, s);
  if (sv.tc) return launch_gather_tc(sv, w, p->n, p->kb_tab, p->grids, p->grid_total, R, out, ldo, s);
  const int rg = v2_rhs_group(w.d, p->m, R, false);
  if (rg < 1) return false;
  for (int r0 = 0; r0 < R; r0 += rg) {
    const int nr = std::min(rg, R - r0);
    const double* g = p->grids + r0 * p->grid_total;
    double* o = out + r0 * ldo;
    bool ok = false;
    switch (w.d) {
      case 1: ok = launch_gather_v2<1>(sv, w, p->n, p->m, p->kb_tab, *p->poly, g, p->grid_total, nr, o, ldo, s); break;
      case 2: ok = launch_gather_v2<2>(sv, w, p->n, p->m, p->kb_tab, *p->poly, g, p->grid_total, nr, o, ldo, s); break;
      default: ok = launch_gather_v2<3>(sv, w, p->n, p->m, p->kb_tab, *p->poly, g, p->grid_total, nr, o, ldo, s); break;
    }
    if (!ok) {
      if (r0 != 0) throw Error(AFS_ERR_CUDA, "inconsistent v2 gather dispatch");
      return false;
    }
  }
  return true;
}

// out += a0 (+ a1 (+ a2)): the extra branches' accumulators, in branch order
__global__ void k_add_into(double* __restrict__ out, int64_t ldo, const double* __restrict__ a0,
                           const double* __restrict__ a1, const double* __restrict__ a2, int na,
                           int64_t lda, int64_t N, int R) {
  const int64_t tot = N * R;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < tot;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = k / N, i = k - r * N;
    double v = out[r * ldo + i] + a0[r * lda + i];
    if (na > 1) v += a1[r * lda + i];
    if (na > 2) v += a2[r * lda + i];
    out[r * ldo + i] = v;
  }
}

// Extra accumulators are read-modify-written at random (out[perm]); they only pay while all
// of them stay L2-resident (C5: 4 x 8 MB; C3's 80 MB vectors measured slower with 2)
int gather_branches(const afs_plan* p, int R) {
  if (p->profiling || p->P < 2) return 1;
  const int64_t bytes = p->Nt * R * (int64_t)sizeof(double);
  int nb = p->stage_streams > 0 ? p->stage_streams : afs_plan::kMaxBranches;
  nb = std::min(nb, p->P);
  while (nb > 1 && nb * bytes > (48LL << 20)) --nb;
  return nb;
}

void gather_1d_fused(afs_plan* p, double* out, int64_t ldo, int R, cudaStream_t s);

void gather_unit(afs_plan* p, const std::vector<int>& wins, bool fused1d, double* out,
                 int64_t ldo, int R, cudaStream_t s) {
  if (fused1d) {   // every 1-D window of the plan, in window order, in shared launches
    gather_1d_fused(p, out, ldo, R, s);
    return;
  }
  for (int l : wins)
    if (!gather_v2_window(p, l, out, ldo, R, s)) gather_v1(p, l, l + 1, out, ldo, R, s);
}

void gather_all(afs_plan* p, double* out, int64_t ldo, int R, cudaStream_t s) {
  // out = 0, then out += eta_l * s_l in window order (anova.py:179-183)
  AFS_CUDA(cudaMemset2DAsync(out, sizeof(double) * ldo, 0, sizeof(double) * p->Nt, R, s));
  if (p->window_eval != 0) {
    gather_v1(p, 0, p->P, out, ldo, R, s);
  } else {
    const bool timed = p->profiling && !p->wev_gather.empty();
    // branches (as the spread, spread.cu): branch b > 0 accumulates its windows into the
    // plan's output buffer outx[b-1], added at the join -- out = sum over branches of the
    // windows' sums, each in window order (fixed, so run-to-run reproducible)
    // plans holding both kernel classes run one class per branch (spread.cu mix_classes)
    double share3 = 1.0, share2 = 1.0;
    const bool mix = !timed && mix_classes(p, &share3, &share2);
    int nb = timed ? 1 : (mix ? 2 : gather_branches(p, R));
    // Vectors too large for private accumulators (C3: 80 MB): outside deterministic mode the
    // sorted gathers of different windows may share `out` across branches -- each adds its
    // result with one RED per node, so concurrent windows only change the order of the adds
    // (run-to-run variation of the last bits, as the atomic spread already has).  The fused 1-D
    // gather (plain read-modify-write) runs before the fork.  AFS_GATHER_SHARED=0 disables it.
    bool shared_out = false;
    if (nb == 1 && !timed && !mix && !p->deterministic && p->P >= 2) {
      static const bool on = [] { const char* e = getenv("AFS_GATHER_SHARED"); return !(e && e[0] == '0'); }();
      bool all_red = on;
      for (int l = 0; l < p->P && all_red; ++l) {
        const SortedSide& sv = p->tgt_side[l] ? *p->tgt_side[l] : *p->src_side[l];
        if (!sv.tc && v2_rhs_group(p->win[l].d, p->m, R, false) < 1) all_red = false;
      }
      if (all_red) {
        shared_out = true;
        nb = std::min(p->P, p->stage_streams > 0 ? p->stage_streams : 3);
        if (nb < 2) shared_out = false, nb = 1;
      }
    }
    if (nb > 1 && !shared_out) {
      for (int b = 1; b < nb; ++b)
        if (!p->outx[b - 1]) {
          AFS_CUDA(cudaMalloc(&p->outx[b - 1], sizeof(double) * p->Nt * p->max_rhs));
          p->device_bytes += sizeof(double) * p->Nt * p->max_rhs;
        }
      fork_branches(p, nb, s);
      for (int b = 1; b < nb; ++b)
        AFS_CUDA(cudaMemsetAsync(p->outx[b - 1], 0, sizeof(double) * p->Nt * R, p->aux[b - 1]));
    }
    // all 1-D windows in one fused launch (gather1d.cu) at the first 1-D window's place
    std::vector<char> fused(p->P, 0);
    int first1d = -1;
    if (p->window_eval == 0 && gather_1d_fusable(p))
      for (int l = 0; l < p->P; ++l)
        if (p->win[l].d == 1) {
          fused[l] = 1;
          if (first1d < 0) first1d = l;
        }
    if (shared_out) {   // the 1-D windows first (not atomic), then the fork
      if (first1d >= 0) gather_1d_fused(p, out, ldo, R, s);
      fork_branches(p, nb, s);
    }
    for (int l = 0; l < p->P; ++l) {
      if (timed) AFS_CUDA(cudaEventRecord(p->wev_gather[l], s));
      const bool heavy = mix && p->win[l].d == 3;
      const int br = mix ? (heavy ? 1 : 0) : l % nb;
      g_wave_share = mix ? (heavy ? share3 : share2) : 1.0;
      const cudaStream_t sl = br ? p->aux[br - 1] : s;
      double* o = (br && !shared_out) ? p->outx[br - 1] : out;
      const int64_t lo = (br && !shared_out) ? p->Nt : ldo;
      if (fused[l]) {
        if (l == first1d && !shared_out) gather_1d_fused(p, o, lo, R, sl);
        continue;
      }
      if (!gather_v2_window(p, l, o, lo, R, sl)) gather_v1(p, l, l + 1, o, lo, R, sl);
    }
    g_wave_share = 1.0;
    if (timed) AFS_CUDA(cudaEventRecord(p->wev_gather[p->P], s));
    if (nb > 1 && shared_out) join_branches(p, nb, s);
    if (nb > 1 && !shared_out) {
      join_branches(p, nb, s);
      const int64_t tot = p->Nt * R;
      const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
      k_add_into<<<blocks, 256, 0, s>>>(out, ldo, p->outx[0], p->outx[1], p->outx[2], nb - 1,
                                        p->Nt, p->Nt, R);
    }
  }
  AFS_CUDA(cudaGetLastError());
}

}  // namespace afs
