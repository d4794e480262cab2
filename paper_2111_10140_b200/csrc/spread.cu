// Adjoint-NFFT spreading (the bincount loop of nfft.py:232-245), all windows.
//
// v1 kernel: one thread per (node, window); the (2m)^d tensor-product stencil
// is accumulated into the window's L2-resident real grid with native fp64
// global reductions (RED.E.ADD.F64).  alpha is real, so the reference's
// complex grid has zero imaginary part and only the real grid is kept.
#include <algorithm>

#include "afs_internal.cuh"
#include "sliding.cuh"
#include "tc2d.cuh"
#include "tc3d.cuh"
#include "solo.cuh"

namespace afs {

template <int D, int MM>
__global__ void __launch_bounds__(256) k_spread_red(const double* __restrict__ X, int64_t N,
                                                    int dtot, Window w, int n, double b,
                                                    const double* __restrict__ alpha,
                                                    int64_t lda, int R, double* __restrict__ grid,
                                                    int64_t rhs_stride) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  double wt[D][2 * MM];
  int ix[D][2 * MM];
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const double xs = scaled_coord(X[j * dtot + w.feat[t]], w.center[t], w.scale);
    stencil_1d<MM>(xs, n, b, wt[t], ix[t]);
  }
  for (int r = 0; r < R; ++r) {
    const double a = alpha[r * lda + j];
    double* g = grid + r * rhs_stride + w.grid_off;
    if (D == 1) {
#pragma unroll
      for (int o0 = 0; o0 < 2 * MM; ++o0) grid_add(w, g + ix[0][o0], __dmul_rn(a, wt[0][o0]));
    } else if (D == 2) {
#pragma unroll 1
      for (int o0 = 0; o0 < 2 * MM; ++o0) {
        const int64_t row = (int64_t)ix[0][o0] * n;
#pragma unroll
        for (int o1 = 0; o1 < 2 * MM; ++o1)
          grid_add(w, g + row + ix[D - 1][o1], __dmul_rn(a, __dmul_rn(wt[0][o0], wt[D - 1][o1])));
      }
    } else {
#pragma unroll 1
      for (int o0 = 0; o0 < 2 * MM; ++o0) {
        const int64_t p0 = (int64_t)ix[0][o0] * n;
#pragma unroll 1
        for (int o1 = 0; o1 < 2 * MM; ++o1) {
          const int64_t p1 = (p0 + ix[1 % D][o1]) * n;
          const double w01 = __dmul_rn(wt[0][o0], wt[1 % D][o1]);
#pragma unroll
          for (int o2 = 0; o2 < 2 * MM; ++o2)
            grid_add(w, g + p1 + ix[D - 1][o2], __dmul_rn(a, __dmul_rn(w01, wt[D - 1][o2])));
        }
      }
    }
  }
}

template <int MM>
static void launch_spread_m(afs_plan* p, const Window& w, const double* alpha, int64_t lda, int R,
                            cudaStream_t s) {
  const int threads = 256;
  const int64_t blocks = (p->Ns + threads - 1) / threads;
  const int64_t rs = p->grid_total;
  switch (w.d) {
    case 1:
      k_spread_red<1, MM><<<blocks, threads, 0, s>>>(p->src, p->Ns, p->dtot, w, p->n, p->b, alpha,
                                                     lda, R, p->grids, rs);
      break;
    case 2:
      k_spread_red<2, MM><<<blocks, threads, 0, s>>>(p->src, p->Ns, p->dtot, w, p->n, p->b, alpha,
                                                     lda, R, p->grids, rs);
      break;
    default:
      k_spread_red<3, MM><<<blocks, threads, 0, s>>>(p->src, p->Ns, p->dtot, w, p->n, p->b, alpha,
                                                     lda, R, p->grids, rs);
      break;
  }
}

static bool spread_v2_window(afs_plan* p, int l, const double* alpha, int64_t lda, int R,
                             cudaStream_t s) {
  if (p->window_eval != 0) return false;
  const Window& w = p->win[l];
  const SortedSide& sv = *p->src_side[l];
  if (sv.tc && w.d == 3)
    return launch_spread_tc3(sv, w, p->n, p->kb_tab, alpha, lda, R, p->grids, p->grid_total, s);
  if (sv.tc) return launch_spread_tc(sv, w, p->n, p->kb_tab, alpha, lda, R, p->grids, p->grid_total, s);
  const int rg = v2_rhs_group(w.d, p->m, R, true);
  if (rg < 1) return false;
  for (int r0 = 0; r0 < R; r0 += rg) {
    const int nr = std::min(rg, R - r0);
    const double* a = alpha + r0 * lda;
    double* g = p->grids + r0 * p->grid_total;
    bool ok = false;
    switch (w.d) {
      case 1: ok = launch_spread_v2<1>(sv, w, p->n, p->m, p->kb_tab, *p->poly, a, lda, nr, g, p->grid_total, s); break;
      case 2: ok = launch_spread_v2<2>(sv, w, p->n, p->m, p->kb_tab, *p->poly, a, lda, nr, g, p->grid_total, s); break;
      default: ok = launch_spread_v2<3>(sv, w, p->n, p->m, p->kb_tab, *p->poly, a, lda, nr, g, p->grid_total, s); break;
    }
    if (!ok) return false;   // no sliding kernel for this (d, m): whole window via v1
  }
  return true;
}

int v2_rhs_group(int D, int m, int R, bool spread) {
  // mirrors Fits<> in sliding.cuh: LPL * 2m * RG <= 64 doubles, RG = 2 only for m <= 4
  const int W = 2 * m;
  const int lines = D == 3 ? W * W : (D == 2 ? W : 1);
  int team = 1;
  if (D != 1) {
    team = 1;
    while (team < lines && team < 32) team *= 2;
    if (D == 3 && team > AFS_TEAM3) team = AFS_TEAM3;
  }
  const int lpl = (lines + team - 1) / team;
  if (lpl * W > 64) return 0;
  // 3-D spread at m = 4 with many right-hand sides: 4 per pass (window values evaluated half
  // as often, same 2 blocks/SM as 2 per pass; C4 at N=1e8: spread 51.5 -> 41.7 ms).  The
  // gather's 4-RHS variant spills (255 registers) and is slower, so it keeps 2.
  if (spread && D == 3 && R >= 4 && m == 4 && lpl * W * 4 <= 64) return 4;
  if (R >= 2 && m <= 4 && lpl * W * 2 <= 64) return 2;
  return 1;
}

// ---- deterministic mode: scale selection and limb -> fp64 conversion -------------------
__global__ void k_det_absmax(const double* __restrict__ alpha, int64_t lda, int64_t N, int R,
                             unsigned long long* __restrict__ out) {
  double m = 0.0;
  const int64_t tot = N * R;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, j = i - r * N;
    const double a = fabs(alpha[r * lda + j]);
    m = isfinite(a) ? fmax(m, a) : __longlong_as_double(0x7ff8000000000000LL);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double q = __shfl_xor_sync(0xffffffffu, m, o);
    m = (isnan(m) || isnan(q)) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(m, q);
  }
  // non-negative doubles order like their bit patterns (the NaN marker above all finite ones)
  if ((threadIdx.x & 31) == 0 && !(m == 0.0))
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// S such that N * max|alpha| * max(window product) * 2^S < 2^top_bit (top_bit = 3L - 1):
// every partial sum of a cell fits the 3L-bit limb range (log2_bound = log2(N * max product)
// + margin).  A
// non-finite alpha (NaN marker from k_det_absmax) makes every grid value NaN, as the
// fp64-atomic spread would propagate it.
__global__ void k_det_scale(double* aux, double log2_bound, int top_bit) {
  const double A = __longlong_as_double(*reinterpret_cast<const long long*>(aux));
  if (isnan(A)) {
    aux[1] = 0.0;
    aux[2] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  int S = 0;
  if (A > 0.0) {
    int ea = 0;
    frexp(A, &ea);                      // A < 2^ea
    S = top_bit - (int)ceil(log2_bound) - ea;
  }
  S = max(-1000, min(1000, S));
  aux[1] = ldexp(1.0, S);
  aux[2] = ldexp(1.0, -S);
}

// exact 128-bit sum of the limbs, then one conversion (two roundings at most), 2^-S and the
// window's boost undone.  wins != nullptr: cells of all windows ([rhs][grid_total]), the window
// looked up by its grid offset; else one window with the given inverse boost.
__global__ void k_det_finalize(const long long* __restrict__ limbs, int64_t stride, int64_t count,
                               const double* __restrict__ aux, double* __restrict__ grids,
                               int bits, const Window* __restrict__ wins, int P, int64_t grid_total,
                               int dmax, int peak_exp, double inv_boost) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const __int128 v = ((__int128)limbs[2 * stride + i] << (2 * bits)) +
                     ((__int128)limbs[stride + i] << bits) + (__int128)limbs[i];
  const bool neg = v < 0;
  const unsigned __int128 u = (unsigned __int128)(neg ? -v : v);
  const double mag = __ull2double_rn((unsigned long long)(u >> 64)) * 0x1p64 +
                     __ull2double_rn((unsigned long long)u);
  if (wins != nullptr) {
    const int64_t c = i % grid_total;
    int lo = 0, hi = P - 1;   // windows are laid out in order of grid_off
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (wins[mid].grid_off <= c) lo = mid;
      else hi = mid - 1;
    }
    // 2^-k built from its exponent bits (k = (d_max - d) e < 1023)
    inv_boost = __longlong_as_double((long long)(1023 - (dmax - wins[lo].d) * peak_exp) << 52);
  }
  grids[i] = ((neg ? -mag : mag) * aux[2]) * inv_boost;
}

void ensure_aux_streams(afs_plan* p) {
  if (p->ev_fork) return;
  for (int b = 0; b < afs_plan::kMaxBranches - 1; ++b) {
    AFS_CUDA(cudaStreamCreateWithFlags(&p->aux[b], cudaStreamNonBlocking));
    AFS_CUDA(cudaEventCreateWithFlags(&p->ev_join[b], cudaEventDisableTiming));
  }
  AFS_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
}

thread_local double g_wave_share = 1.0;

void fork_branches(afs_plan* p, int nb, cudaStream_t s) {
  ensure_aux_streams(p);
  AFS_CUDA(cudaEventRecord(p->ev_fork, s));
  for (int b = 1; b < nb; ++b) AFS_CUDA(cudaStreamWaitEvent(p->aux[b - 1], p->ev_fork, 0));
}

void join_branches(afs_plan* p, int nb, cudaStream_t s) {
  for (int b = 1; b < nb; ++b) {
    AFS_CUDA(cudaEventRecord(p->ev_join[b - 1], p->aux[b - 1]));
    AFS_CUDA(cudaStreamWaitEvent(s, p->ev_join[b - 1], 0));
  }
}

// Large windows (C3: 0.12-0.8 ms kernels) gain most of the overlap from 2-3 branches; small ones
// (C5 at N=1M: ~25 us kernels, tail-dominated) from 4.
static int auto_branches(const afs_plan* p) {
  if (p->stage_streams > 0) return p->stage_streams;
  return p->Ns * (int64_t)p->P <= (int64_t)64 << 20 ? 4 : 3;   // C3: 13.76 / 13.00 / 12.97 / 12.97 ms for 1-4
}

int spread_branches(const afs_plan* p) {
  if (p->profiling || p->P < 2 || p->window_eval != 0) return 1;
  return std::min(auto_branches(p), p->P);
}

// Co-scheduling of the two kernel classes (see spread_all): true when the plan holds
// tensor-core 3-D windows and sub-cell 2-D windows and AFS_MIX=1.  Off by default: measured on
// C3 (13.15 ms per matvec without) it costs 15.2-17.7 ms for shares 0.25-0.5 / 0.5-1.0 -- the
// two classes' node streams and the evict_last vector compete for the L2.  AFS_MIX_SHARE3 /
// AFS_MIX_SHARE2 set the shares.
bool mix_classes(const afs_plan* p, double* share3, double* share2) {
  if (p->window_eval != 0 || p->profiling) return false;
  static const int mode = [] { const char* e = getenv("AFS_MIX"); return e ? atoi(e) : 0; }();
  if (mode == 0) return false;
  int n3 = 0, n2 = 0;
  for (int l = 0; l < p->P; ++l) {
    const SortedSide* sv = p->src_side[l];
    if (!sv) return false;
    if (p->win[l].d == 3 && sv->tc) ++n3;
    if (p->win[l].d == 2 && sv->sc) ++n2;
  }
  if (n3 == 0 || n2 == 0) return false;
  static const double s3 = [] { const char* e = getenv("AFS_MIX_SHARE3"); return e ? atof(e) : 0.25; }();
  static const double s2 = [] { const char* e = getenv("AFS_MIX_SHARE2"); return e ? atof(e) : 0.75; }();
  *share3 = s3;
  *share2 = s2;
  return true;
}

void spread_all(afs_plan* p, const double* alpha, int64_t lda, int R, cudaStream_t s) {
  const bool det = p->deterministic && p->det_limbs;
  const int64_t cells = p->grid_total * R;
  if (det) {
    const int64_t stride = p->grid_total * p->max_rhs;
    for (int k = 0; k < 3; ++k)
      AFS_CUDA(cudaMemsetAsync(p->det_limbs + k * stride, 0, sizeof(long long) * cells, s));
    AFS_CUDA(cudaMemsetAsync(p->det_aux, 0, sizeof(double), s));
    k_det_absmax<<<592, 256, 0, s>>>(alpha, lda, p->Ns, R,
                                     reinterpret_cast<unsigned long long*>(p->det_aux));
    k_det_scale<<<1, 1, 0, s>>>(p->det_aux, p->det_log2_bound, 3 * p->det_bits - 1);
  } else {
    AFS_CUDA(cudaMemsetAsync(p->grids, 0, sizeof(double) * cells, s));
  }
  const bool timed = p->profiling && !p->wev_spread.empty();
  // branches (not while timing windows): window l runs on branch l % nb.  Plans that hold both
  // kernel classes -- tensor-core 3-D windows (fp64-pipe-bound) and sub-cell 2-D windows
  // (load/store-pipe-bound) -- run one class per branch, each with its share of the SM's
  // resident warps, so the two kinds of warps share every SM (mix_classes)
  double share3 = 1.0, share2 = 1.0;
  const bool mix = !timed && mix_classes(p, &share3, &share2);
  const int nb = timed ? 1 : (mix ? 2 : spread_branches(p));
  if (nb > 1) fork_branches(p, nb, s);
  // the 1-D windows' solo spreads share one launch (grids disjoint), at the first 1-D
  // window's place; AFS_SPREAD1D=0 keeps one launch per window
  std::vector<int> ones;
  if (p->window_eval == 0 && p->P > 1) {
    const char* e = getenv("AFS_SPREAD1D");
    if (!(e && e[0] == '0'))
      for (int l = 0; l < p->P; ++l)
        if (p->win[l].d == 1 && !p->src_side[l]->tc) ones.push_back(l);
    if (ones.size() < 2) ones.clear();
  }
  for (int l = 0; l < p->P; ++l) {
    const Window& w = p->win[l];
    if (timed) AFS_CUDA(cudaEventRecord(p->wev_spread[l], s));
    const bool heavy = mix && w.d == 3;
    const int br = mix ? (heavy ? 1 : 0) : l % nb;
    const cudaStream_t sl = br ? p->aux[br - 1] : s;
    g_wave_share = mix ? (heavy ? share3 : share2) : 1.0;
    if (!ones.empty() && w.d == 1) {
      if (l == ones[0]) {
        for (size_t b0 = 0; b0 < ones.size(); b0 += kSoloBatch) {
          SoloBatch B{};
          B.nwin = (int)std::min<size_t>(kSoloBatch, ones.size() - b0);
          for (int i = 0; i < B.nwin; ++i) {
            B.sv[i] = *p->src_side[ones[b0 + i]];
            B.w[i] = p->win[ones[b0 + i]];
          }
          launch_spread_solo_batch_1d(B, p->n, p->m, p->kb_tab, *p->poly, alpha, lda, R, p->grids,
                                      p->grid_total, sl);
        }
      }
      continue;
    }
    if (spread_v2_window(p, l, alpha, lda, R, sl)) continue;
    switch (p->m) {
      case 1: launch_spread_m<1>(p, w, alpha, lda, R, sl); break;
      case 2: launch_spread_m<2>(p, w, alpha, lda, R, sl); break;
      case 3: launch_spread_m<3>(p, w, alpha, lda, R, sl); break;
      case 4: launch_spread_m<4>(p, w, alpha, lda, R, sl); break;
      case 5: launch_spread_m<5>(p, w, alpha, lda, R, sl); break;
      case 6: launch_spread_m<6>(p, w, alpha, lda, R, sl); break;
      case 7: launch_spread_m<7>(p, w, alpha, lda, R, sl); break;
      default: launch_spread_m<8>(p, w, alpha, lda, R, sl); break;
    }
  }
  g_wave_share = 1.0;
  if (nb > 1) join_branches(p, nb, s);
  if (timed) AFS_CUDA(cudaEventRecord(p->wev_spread[p->P], s));
  if (det) {
    k_det_finalize<<<(unsigned)((cells + 255) / 256), 256, 0, s>>>(
        p->det_limbs, p->grid_total * p->max_rhs, cells, p->det_aux, p->grids, p->det_bits, p->d_win,
        p->P, p->grid_total, p->det_dmax, p->det_peak_exp, 1.0);
  }
  AFS_CUDA(cudaGetLastError());
}

// deterministic mode in the window pipeline: the scale 2^S from max|alpha| once per apply,
// then per window its limbs cleared before and converted after its spread
void det_prepare(afs_plan* p, const double* alpha, int64_t lda, int R, cudaStream_t s) {
  AFS_CUDA(cudaMemsetAsync(p->det_aux, 0, sizeof(double), s));
  k_det_absmax<<<592, 256, 0, s>>>(alpha, lda, p->Ns, R,
                                   reinterpret_cast<unsigned long long*>(p->det_aux));
  k_det_scale<<<1, 1, 0, s>>>(p->det_aux, p->det_log2_bound, 3 * p->det_bits - 1);
  AFS_CUDA(cudaGetLastError());
}

// zero narr arrays (arr_stride apart) of R rows of `width` 8-byte words at `pitch` words: one
// kernel instead of narr * R memset nodes (memsets are slow nodes inside a conditional body)
__global__ void k_clear_rows(unsigned long long* __restrict__ base, int64_t arr_stride, int narr,
                             int64_t pitch, int64_t width, int R) {
  const int64_t tot = (int64_t)narr * R * width;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = i / (R * width), rem = i - a * R * width;
    const int64_t r = rem / width, c = rem - r * width;
    base[a * arr_stride + r * pitch + c] = 0ull;
  }
}

void clear_rows(void* base, int64_t arr_stride, int narr, int64_t pitch, int64_t width, int R,
                cudaStream_t s) {
  const int64_t tot = (int64_t)narr * R * width;
  const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
  k_clear_rows<<<std::max(1, blocks), 256, 0, s>>>(static_cast<unsigned long long*>(base),
                                                   arr_stride, narr, pitch, width, R);
}

void det_window_begin(afs_plan* p, const Window& w, int R, cudaStream_t s) {
  clear_rows(p->det_limbs + w.grid_off, p->grid_total * p->max_rhs, 3, p->grid_total, w.cells, R, s);
}

void det_window_finalize(afs_plan* p, const Window& w, int R, cudaStream_t s) {
  const int64_t stride = p->grid_total * p->max_rhs;
  for (int r = 0; r < R; ++r) {
    const int64_t off = r * p->grid_total + w.grid_off;
    k_det_finalize<<<(unsigned)((w.cells + 255) / 256), 256, 0, s>>>(
        p->det_limbs + off, stride, w.cells, p->det_aux, p->grids + off, p->det_bits, nullptr, 0,
        p->grid_total, p->det_dmax, p->det_peak_exp, 1.0 / w.det_boost);
  }
  AFS_CUDA(cudaGetLastError());
}

void spread_unit(afs_plan* p, const std::vector<int>& wins, bool batch1d, const double* alpha,
                 int64_t lda, int R, cudaStream_t s) {
  if (batch1d) {   // the 1-D windows' solo spreads in shared launches (grids disjoint)
    for (size_t b0 = 0; b0 < wins.size(); b0 += kSoloBatch) {
      SoloBatch B{};
      B.nwin = (int)std::min<size_t>(kSoloBatch, wins.size() - b0);
      for (int i = 0; i < B.nwin; ++i) {
        B.sv[i] = *p->src_side[wins[b0 + i]];
        B.w[i] = p->win[wins[b0 + i]];
      }
      launch_spread_solo_batch_1d(B, p->n, p->m, p->kb_tab, *p->poly, alpha, lda, R, p->grids,
                                  p->grid_total, s);
    }
    return;
  }
  for (int l : wins) {
    if (spread_v2_window(p, l, alpha, lda, R, s)) continue;
    const Window& w = p->win[l];
    switch (p->m) {
      case 1: launch_spread_m<1>(p, w, alpha, lda, R, s); break;
      case 2: launch_spread_m<2>(p, w, alpha, lda, R, s); break;
      case 3: launch_spread_m<3>(p, w, alpha, lda, R, s); break;
      case 4: launch_spread_m<4>(p, w, alpha, lda, R, s); break;
      case 5: launch_spread_m<5>(p, w, alpha, lda, R, s); break;
      case 6: launch_spread_m<6>(p, w, alpha, lda, R, s); break;
      case 7: launch_spread_m<7>(p, w, alpha, lda, R, s); break;
      default: launch_spread_m<8>(p, w, alpha, lda, R, s); break;
    }
  }
}

}  // namespace afs
