// v2 spread / gather: register sliding windows over bin-sorted nodes.
//
// Nodes of a window are sorted by base cell (row-major, last dimension
// fastest) and cut into column runs (Chunk).  A "team" of TEAM lanes takes
// one run.  Lane tl owns LPL "lines" of the stencil: the (2m)^(d-1) cells of
// the leading dimensions around the column base.  Along the last dimension
// each lane keeps a 2m-slot window of accumulators (spread) or grid values
// (gather) in registers; cell c lives in slot c mod 2m, so advancing the
// window never moves registers: leaving cells are flushed (spread:
// RED.E.ADD.F64 into the L2-resident grid) and entering cells loaded
// (gather).  Per node, one lane evaluates the 2m*d window values once
// (degree-13 polynomial, geometry.cuh) and stages them in shared memory;
// the last dimension's values are stored pre-rotated into slot order so the
// inner loop is a fixed, fully unrolled FMA sequence.
//
// Reference: the spread is nfft.py:241-245 (bincount of alpha * prod_t w_t),
// the gather nfft.py:228-229 ((g[flat] * w).sum(axis=1)), both over the
// tensor-product stencil of nfft.py:179-188.
#pragma once

#include <climits>

#include "geometry.cuh"

namespace afs {

template <int D, int MM>
struct Cfg {
  static constexpr int W = 2 * MM;
  static constexpr int LINES = D == 3 ? W * W : (D == 2 ? W : 1);
  static constexpr int TEAM = D == 1 ? 1 : (LINES >= 32 ? 32 : (LINES > 16 ? 32 : (LINES > 8 ? 16 : (LINES > 4 ? 8 : (LINES > 2 ? 4 : (LINES > 1 ? 2 : 1))))));
  static constexpr int LPL = (LINES + TEAM - 1) / TEAM;
  static constexpr int TPW = 32 / TEAM;
};

template <int D, int MM, int RG>
struct Fits {
  static constexpr bool value = Cfg<D, MM>::LPL * Cfg<D, MM>::W * RG <= 64;
};

__device__ __forceinline__ int wrap_cell(int c, int n) {
  c %= n;
  return c < 0 ? c + n : c;
}

// slot k of a window whose first cell is lo holds cell lo + ((k - lo) mod W)
template <int W>
__device__ __forceinline__ int slot_cell(int k, int lo) {
  int off = (k - lo) % W;
  if (off < 0) off += W;
  return lo + off;
}

struct LineGeom {
  int64_t off;   // grid index of (line, last = 0)
  int a, b;      // stencil digits of the leading dims
  bool valid;
};

template <int D, int MM>
__device__ __forceinline__ void line_geometry(int tl, int col, int n, LineGeom (&lg)[Cfg<D, MM>::LPL]) {
  using C = Cfg<D, MM>;
  int ub0 = 0, ub1 = 0;
  if (D == 3) {
    ub0 = col / n;
    ub1 = col - ub0 * n;
  } else if (D == 2) {
    ub0 = col;
  }
#pragma unroll
  for (int j = 0; j < C::LPL; ++j) {
    const int L = tl + C::TEAM * j;
    lg[j].valid = L < C::LINES;
    const int Lc = lg[j].valid ? L : 0;
    const int a = D == 3 ? Lc / C::W : Lc;
    const int b = D == 3 ? Lc - a * C::W : 0;
    lg[j].a = D >= 2 ? a : 0;
    lg[j].b = b;
    if (D == 3) {
      const int c0 = wrap_cell(ub0 - MM + 1 + a, n), c1 = wrap_cell(ub1 - MM + 1 + b, n);
      lg[j].off = ((int64_t)c0 * n + c1) * n;
    } else if (D == 2) {
      lg[j].off = (int64_t)wrap_cell(ub0 - MM + 1 + a, n) * n;
    } else {
      lg[j].off = 0;
    }
  }
}

// Stage one node: window values of all dims (last dim rotated to slot order) + base.
template <int D, int MM>
__device__ __forceinline__ int stage_node(const SortedSide& sv, int64_t i, int n, const PolyTable& T,
                                          double* row) {
  constexpr int W = 2 * MM;
  int u = 0;
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const double nx = sv.nx[t * sv.N + i];
    const double fl = floor(nx);
    const double f = nx - fl;                 // exact (Sterbenz)
    double wt[W];
    poly_weights<MM>(f, T, wt);
    if (t < D - 1) {
#pragma unroll
      for (int o = 0; o < W; ++o) row[t * W + o] = wt[o];
    } else {
      long long ul = (long long)fl % n;
      u = (int)(ul < 0 ? ul + n : ul);
      const int rot = (u + MM + 1) % W;
#pragma unroll
      for (int o = 0; o < W; ++o) {
        int s = rot + o;
        s = s >= W ? s - W : s;
        row[(D - 1) * W + s] = wt[o];
      }
    }
  }
  return u;
}

template <int D, int MM>
__device__ __forceinline__ double line_weight(const double* row, const LineGeom& g) {
  if (D == 3) return g.valid ? row[g.a] * row[Cfg<D, MM>::W + g.b] : 0.0;
  if (D == 2) return g.valid ? row[g.a] : 0.0;
  return 1.0;
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ----------------------------------------------------------------------------
// spread
// ----------------------------------------------------------------------------
template <int D, int MM, int RG>
__global__ void __launch_bounds__(128) k_spread_v2(const SortedSide sv, const Window w, int n,
                                                   const PolyTable T,
                                                   const double* __restrict__ alpha, int64_t lda,
                                                   int nr, double* __restrict__ grid,
                                                   int64_t rhs_stride) {
  using C = Cfg<D, MM>;
  constexpr int W = C::W, TEAM = C::TEAM, LPL = C::LPL, TPW = C::TPW;
  constexpr int STRIDE = D * W + RG + 1;
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int team = lane / TEAM, tl = lane - team * TEAM;
  double* st = sm + (size_t)(threadIdx.x >> 5) * 32 * STRIDE + (size_t)team * TEAM * STRIDE;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t ci = gwarp * TPW + team;
  const bool active = ci < sv.nchunks;
  Chunk ch{0, 0, 0};
  if (active) ch = sv.chunks[ci];
  LineGeom lg[LPL];
  line_geometry<D, MM>(tl, ch.col, n, lg);
  double* g = grid + w.grid_off;

  double acc[LPL][W][RG];
#pragma unroll
  for (int j = 0; j < LPL; ++j)
#pragma unroll
    for (int k = 0; k < W; ++k)
#pragma unroll
      for (int r = 0; r < RG; ++r) acc[j][k][r] = 0.0;

  auto flush = [&](int lo, int keep_from) {
    // flush slots whose cell (window starting at lo) is < keep_from
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int c = slot_cell<W>(k, lo);
      if (c < keep_from) {
        const int cm = wrap_cell(c, n);
#pragma unroll
        for (int j = 0; j < LPL; ++j) {
          if (lg[j].valid) {
#pragma unroll
            for (int r = 0; r < RG; ++r) {
              if (r < nr) atomicAdd(g + r * rhs_stride + lg[j].off + cm, acc[j][k][r]);
              acc[j][k][r] = 0.0;
            }
          }
        }
      }
    }
  };

  int cur = INT_MIN;
  const int rounds = warp_max(ch.count);
  for (int b0 = 0; b0 < rounds; b0 += TEAM) {
    if (active && b0 + tl < ch.count) {
      const int64_t i = ch.begin + b0 + tl;
      double* row = st + tl * STRIDE;
      const int u = stage_node<D, MM>(sv, i, n, T, row);
      const int jj = sv.perm[i];
#pragma unroll
      for (int r = 0; r < RG; ++r) row[D * W + r] = r < nr ? __ldg(alpha + r * lda + jj) : 0.0;
      row[D * W + RG] = (double)u;
    }
    __syncwarp();
    const int cnt = active ? min(TEAM, ch.count - b0) : 0;
    for (int q = 0; q < cnt; ++q) {
      const double* row = st + q * STRIDE;
      const int u = (int)row[D * W + RG];
      if (u != cur) {
        if (cur != INT_MIN) flush(cur - MM + 1, u - MM + 1);
        cur = u;
      }
      double wl[W];
#pragma unroll
      for (int k = 0; k < W; ++k) wl[k] = row[(D - 1) * W + k];
#pragma unroll
      for (int j = 0; j < LPL; ++j) {
        const double lw = line_weight<D, MM>(row, lg[j]);
#pragma unroll
        for (int r = 0; r < RG; ++r) {
          const double p = lw * row[D * W + r];
#pragma unroll
          for (int k = 0; k < W; ++k) acc[j][k][r] = fma(p, wl[k], acc[j][k][r]);
        }
      }
    }
    __syncwarp();
  }
  if (active && cur != INT_MIN) flush(cur - MM + 1, INT_MAX);
}

// ----------------------------------------------------------------------------
// gather: out[perm] += eta * interp
// ----------------------------------------------------------------------------
template <int D, int MM, int RG>
__global__ void __launch_bounds__(128) k_gather_v2(const SortedSide sv, const Window w, int n,
                                                   const PolyTable T,
                                                   const double* __restrict__ grid,
                                                   int64_t rhs_stride, int nr,
                                                   double* __restrict__ out, int64_t ldo) {
  using C = Cfg<D, MM>;
  constexpr int W = C::W, TEAM = C::TEAM, LPL = C::LPL, TPW = C::TPW;
  constexpr int STRIDE = D * W + 1;
  constexpr int RSTR = TEAM + 1;               // padded reduction row
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int team = lane / TEAM, tl = lane - team * TEAM;
  double* st = sm + (size_t)wib * 32 * STRIDE + (size_t)team * TEAM * STRIDE;
  double* red = sm + (size_t)(blockDim.x >> 5) * 32 * STRIDE +
                ((size_t)wib * TPW + team) * (size_t)TEAM * RSTR * RG;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t ci = gwarp * TPW + team;
  const bool active = ci < sv.nchunks;
  Chunk ch{0, 0, 0};
  if (active) ch = sv.chunks[ci];
  LineGeom lg[LPL];
  line_geometry<D, MM>(tl, ch.col, n, lg);
  const double* g = grid + w.grid_off;

  double gv[LPL][W][RG];
  int cur = INT_MIN;
  const int rounds = warp_max(ch.count);
  for (int b0 = 0; b0 < rounds; b0 += TEAM) {
    int my_perm = -1;
    if (active && b0 + tl < ch.count) {
      const int64_t i = ch.begin + b0 + tl;
      double* row = st + tl * STRIDE;
      const int u = stage_node<D, MM>(sv, i, n, T, row);
      row[D * W] = (double)u;
      my_perm = sv.perm[i];
    }
    __syncwarp();
    const int cnt = active ? min(TEAM, ch.count - b0) : 0;
    for (int q = 0; q < cnt; ++q) {
      const double* row = st + q * STRIDE;
      const int u = (int)row[D * W];
      if (u != cur) {
        const int lo = u - MM + 1;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          const int c = slot_cell<W>(k, lo);
          if (cur == INT_MIN || c > cur + MM) {
            const int cm = wrap_cell(c, n);
#pragma unroll
            for (int j = 0; j < LPL; ++j)
#pragma unroll
              for (int r = 0; r < RG; ++r)
                gv[j][k][r] = (lg[j].valid && r < nr) ? __ldg(g + r * rhs_stride + lg[j].off + cm) : 0.0;
          }
        }
        cur = u;
      }
      double wl[W];
#pragma unroll
      for (int k = 0; k < W; ++k) wl[k] = row[(D - 1) * W + k];
      double part[RG];
#pragma unroll
      for (int r = 0; r < RG; ++r) part[r] = 0.0;
#pragma unroll
      for (int j = 0; j < LPL; ++j) {
        const double lw = line_weight<D, MM>(row, lg[j]);
#pragma unroll
        for (int r = 0; r < RG; ++r) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < W; ++k) s = fma(wl[k], gv[j][k][r], s);
          part[r] = fma(lw, s, part[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < RG; ++r) red[(r * TEAM + q) * RSTR + tl] = part[r];
    }
    __syncwarp();
    if (my_perm >= 0) {
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        if (r < nr) {
          const double* rr = red + (r * TEAM + tl) * RSTR;
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < TEAM; ++k) s += rr[k];
          double* o = out + r * ldo + my_perm;
          *o = __dadd_rn(*o, __dmul_rn(w.eta, s));
        }
      }
    }
    __syncwarp();
  }
}

// host-side launchers (instantiated per dimension in sliding_d{1,2,3}.cu)
template <int D>
bool launch_spread_v2(const SortedSide& sv, const Window& w, int n, int m, const PolyTable& T,
                      const double* alpha, int64_t lda, int nr, double* grid, int64_t rs,
                      cudaStream_t s);
template <int D>
bool launch_gather_v2(const SortedSide& sv, const Window& w, int n, int m, const PolyTable& T,
                      const double* grid, int64_t rs, int nr, double* out, int64_t ldo,
                      cudaStream_t s);
int v2_rhs_group(int D, int m, int R);

}  // namespace afs
