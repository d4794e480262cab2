// Spread / gather for 1-D and 2-D windows with lane-private sliding windows.
//
// A warp takes one column run (Chunk) of bin-sorted nodes; lane l processes
// nodes begin + l + 32 k (coalesced loads, neighbouring lanes sit in the same
// or the next cell).  Each lane owns the whole stencil: LINES = (2m)^(d-1)
// lines x 2m cells of accumulators (spread) or grid values (gather) in
// registers, in "shift" order (slot k <-> cell lo + k).  A window move by one
// cell shifts the registers (rare: runs are sorted) and flushes / loads one
// cell per line.  No shared memory and no cross-lane traffic per node.
//
// Spread epilogue: lanes first move to the warp's last cell (flushing what
// leaves individually), then a transposed butterfly reduces the identical
// windows across the warp so each lane issues only LINES*2m/32 RED.F64.
//
// Reference: nfft.py:241-245 (spread), nfft.py:228-229 (gather), stencil
// nfft.py:164-188; window values as in geometry.cuh.
#pragma once

#include <climits>

#include "sliding.cuh"

namespace afs {

template <int D, int MM>
struct SoloCfg {
  static constexpr int W = 2 * MM;
  static constexpr int LINES = D == 2 ? W : 1;
  static constexpr int NACC = LINES * W;
};

// window values of one node, dims 0..D-1 in stencil order
template <int D, int MM, int TAB>
__device__ __forceinline__ void solo_weights(const double (&nx)[D], const PolyTable& T,
                                             double (&wt)[D][2 * MM], int& u_last, int n) {
  constexpr int W = 2 * MM;
  double x[D];
  bool refl[D];
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const double fl = floor(nx[t]);
    const double f = nx[t] - fl;
    refl[t] = f > 0.5;
    x[t] = (refl[t] ? __dsub_rn(1.0, f) : f) - 0.25;
    if (t == D - 1) u_last = wrap_cell((int)fl, n);
  }
  double v[W][D];
  constexpr int NT = TAB == 0 ? kPolyTerms : kb_terms<TAB, MM>();   // per-table degree
#pragma unroll
  for (int k = NT - 1; k >= 0; --k) {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const double c = TAB == 0 ? T.c[i][k] : kb_coef<TAB, MM>(i, k);
#pragma unroll
      for (int t = 0; t < D; ++t) v[i][t] = k == NT - 1 ? c : fma(v[i][t], x[t], c);
    }
  }
#pragma unroll
  for (int t = 0; t < D; ++t)
#pragma unroll
    for (int i = 0; i < W; ++i) wt[t][i] = refl[t] ? v[W - 1 - i][t] : v[i][t];
}

template <int D, int MM>
__device__ __forceinline__ int64_t rowoff_dyn(int col, int ln, int n) {
  return D == 2 ? (int64_t)wrap_cell(col - MM + 1 + ln, n) * n : 0;
}

template <int D, int MM, int RG>
struct SoloFits {
  static constexpr bool value = D <= 2 && SoloCfg<D, MM>::NACC * RG <= 64;
};

// Two-deep prefetch of a lane's node stream q, q+32, q+64 ...: stage 2 holds nx/perm of
// q+64, stage 1 holds nx of q+32 and its gathered value val[perm] (alpha in the spread,
// out in the gather), so the dependent random load has a full node of work to land.
template <int D, int RG>
struct SoloPipe {
  double nx1[D], v1[RG], nx2[D];
  int p1, p2;

  __device__ __forceinline__ void load_node(const SortedSide& sv, const Chunk& ch, int q,
                                            double (&nx)[D], int& p) {
    if (q < ch.count) {
      const int64_t i = ch.begin + q;
#pragma unroll
      for (int t = 0; t < D; ++t) nx[t] = __ldcs(sv.nx + t * sv.N + i);
      p = __ldcs(sv.perm + i);
    } else {
#pragma unroll
      for (int t = 0; t < D; ++t) nx[t] = 0.0;
      p = -1;
    }
  }
  __device__ __forceinline__ void load_val(const double* __restrict__ src, int64_t ld, int nr,
                                           int p, double (&v)[RG]) {
#pragma unroll
    for (int r = 0; r < RG; ++r) v[r] = (src != nullptr && p >= 0 && r < nr) ? src[r * ld + p] : 0.0;
  }
  __device__ __forceinline__ void prime(const SortedSide& sv, const Chunk& ch, int lane,
                                        const double* __restrict__ src, int64_t ld, int nr) {
    load_node(sv, ch, lane, nx1, p1);
    load_val(src, ld, nr, p1, v1);
    load_node(sv, ch, lane + 32, nx2, p2);
  }
  // returns node q's data (already in flight) and pushes q+64 into the pipe
  __device__ __forceinline__ int advance(const SortedSide& sv, const Chunk& ch, int q,
                                         double (&nx)[D], double (&v)[RG],
                                         const double* __restrict__ src, int64_t ld, int nr) {
    const int p = p1;
#pragma unroll
    for (int t = 0; t < D; ++t) nx[t] = nx1[t];
#pragma unroll
    for (int r = 0; r < RG; ++r) v[r] = v1[r];
#pragma unroll
    for (int t = 0; t < D; ++t) nx1[t] = nx2[t];
    p1 = p2;
    load_val(src, ld, nr, p1, v1);
    load_node(sv, ch, q + 64, nx2, p2);
    return p;
  }
};

__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ----------------------------------------------------------------------------
// spread
// ----------------------------------------------------------------------------
template <int D, int MM, int RG, int TAB>
__device__ __forceinline__ void spread_solo_body(const SortedSide& sv, const Window& w, int n,
                                                 const PolyTable& T,
                                                 const double* __restrict__ alpha,
                                                 int64_t lda, int nr,
                                                 double* __restrict__ grid,
                                                 int64_t rhs_stride);

template <int D, int MM, int RG, int TAB>
__global__ void __launch_bounds__(128) k_spread_solo(const SortedSide sv, const Window w, int n,
                                                     const PolyTable T,
                                                     const double* __restrict__ alpha,
                                                     int64_t lda, int nr,
                                                     double* __restrict__ grid,
                                                     int64_t rhs_stride) {
  spread_solo_body<D, MM, RG, TAB>(sv, w, n, T, alpha, lda, nr, grid, rhs_stride);
}

// all windows of a batch in one launch (blockIdx.y = window; their grids are disjoint), so
// the small 1-D spreads of a plan share one launch instead of one tail each
constexpr int kSoloBatch = 40;
struct SoloBatch {
  int nwin;
  SortedSide sv[kSoloBatch];
  Window w[kSoloBatch];
};

template <int D, int MM, int RG, int TAB>
__global__ void __launch_bounds__(128) k_spread_solo_batch(const __grid_constant__ SoloBatch B, int n,
                                                           const __grid_constant__ PolyTable T,
                                                           const double* __restrict__ alpha,
                                                           int64_t lda, int nr,
                                                           double* __restrict__ grid,
                                                           int64_t rhs_stride) {
  spread_solo_body<D, MM, RG, TAB>(B.sv[blockIdx.y], B.w[blockIdx.y], n, T, alpha, lda, nr, grid,
                                   rhs_stride);
}

template <int D, int MM, int RG, int TAB>
__device__ __forceinline__ void spread_solo_body(const SortedSide& sv, const Window& w, int n,
                                                 const PolyTable& T,
                                                 const double* __restrict__ alpha,
                                                 int64_t lda, int nr,
                                                 double* __restrict__ grid,
                                                 int64_t rhs_stride) {
  using C = SoloCfg<D, MM>;
  constexpr int W = C::W, LINES = C::LINES, NACC = C::NACC;
  const int lane = threadIdx.x & 31;
  const int64_t ci = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ci >= sv.nchunks) return;   // warp-uniform
  const Chunk ch = sv.chunks[ci];
  double* g = grid + w.grid_off;
  int64_t rowoff[LINES];
#pragma unroll
  for (int a = 0; a < LINES; ++a)
    rowoff[a] = D == 2 ? (int64_t)wrap_cell(ch.col - MM + 1 + a, n) * n : 0;

  double acc[LINES][W][RG];
#pragma unroll
  for (int a = 0; a < LINES; ++a)
#pragma unroll
    for (int k = 0; k < W; ++k)
#pragma unroll
      for (int r = 0; r < RG; ++r) acc[a][k][r] = 0.0;

  // flush slot 0 of every line (cell lo) and shift the window up by one cell
  auto shift1 = [&](int lo) {
    const int cm = wrap_cell(lo, n);
#pragma unroll
    for (int a = 0; a < LINES; ++a) {
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        if (r < nr && acc[a][0][r] != 0.0) grid_add(w, g + r * rhs_stride + rowoff[a] + cm, acc[a][0][r]);
#pragma unroll
        for (int k = 0; k + 1 < W; ++k) acc[a][k][r] = acc[a][k + 1][r];
        acc[a][W - 1][r] = 0.0;
      }
    }
  };
  auto move_to = [&](int& cur, int u) {
    // advance the window from base cell cur to u (> cur)
    if (u - cur >= W) {
#pragma unroll 1
      for (int j = 0; j < W; ++j) shift1(cur - MM + 1 + j);
    } else {
#pragma unroll 1
      for (int c = cur; c < u; ++c) shift1(c - MM + 1);
    }
    cur = u;
  };

  int cur = INT_MIN;
  const int count = ch.count;
  // software pipeline: node data two steps ahead, alpha[perm] one step ahead
  SoloPipe<D, RG> pipe;
  pipe.prime(sv, ch, lane, alpha, lda, nr);
  for (int q = lane; q < count; q += 32) {
    double nx[D];
    double a[RG];
    pipe.advance(sv, ch, q, nx, a, alpha, lda, nr);
    double wt[D][W];
    int u;
    solo_weights<D, MM, TAB>(nx, T, wt, u, n);
    if (cur == INT_MIN) cur = u;
    if (u != cur) move_to(cur, u);
#pragma unroll
    for (int ln = 0; ln < LINES; ++ln) {
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const double p = (D == 2 ? wt[0][ln] : 1.0) * a[r];
#pragma unroll
        for (int k = 0; k < W; ++k) acc[ln][k][r] = fma(p, wt[D - 1][k], acc[ln][k][r]);
      }
    }
  }
  // epilogue: align every lane's window to the warp's last base cell, then reduce
  const bool has = cur != INT_MIN;
  const int top = warp_max_i(has ? cur : INT_MIN);
  if (top == INT_MIN) return;
  if (has && cur < top) move_to(cur, top);
  // transposed butterfly: after 5 stages lane l holds the warp sums of NACC*RG/32 entries
  constexpr int TOT = NACC * RG;
  double v[TOT];
#pragma unroll
  for (int a = 0; a < LINES; ++a)
#pragma unroll
    for (int k = 0; k < W; ++k)
#pragma unroll
      for (int r = 0; r < RG; ++r) v[(a * W + k) * RG + r] = acc[a][k][r];
  if constexpr (TOT % 32 == 0) {
    int len = TOT;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool upper = (lane & s) != 0;
      const int half = len / 2;
#pragma unroll
      for (int e = 0; e < TOT / 2; ++e) {
        if (e < half) {
          const double send = upper ? v[e] : v[e + half];
          const double keep = upper ? v[e + half] : v[e];
          v[e] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
      }
      len = half;
    }
    // lane holds entries e' = lane-dependent block of size TOT/32
    const int per = TOT / 32;
    // the block index of this lane: bit s of lane selected the upper half at stage s
    int blk = 0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) blk = blk * 2 + ((lane & s) ? 1 : 0);
#pragma unroll
    for (int e = 0; e < per; ++e) {
      const int idx = blk * per + e;
      const int r = idx % RG;
      const int k = (idx / RG) % W;
      const int ln = idx / (RG * W);
      if (r < nr && v[e] != 0.0)
        grid_add(w, g + r * rhs_stride + rowoff_dyn<D, MM>(ch.col, ln, n) + wrap_cell(top - MM + 1 + k, n), v[e]);
    }
  } else if constexpr (TOT < 32) {
    // small windows (1-D): all-reduce each entry across the warp, lane e flushes entry e
    // (32 lanes x TOT reductions into the same few cells would serialise in L2)
#pragma unroll
    for (int e = 0; e < TOT; ++e) {
      if (!has) v[e] = 0.0;
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) v[e] += __shfl_xor_sync(0xffffffffu, v[e], s);
    }
    double mine = 0.0;
#pragma unroll
    for (int e = 0; e < TOT; ++e)
      if (lane == e) mine = v[e];
    if (lane < TOT) {
      const int r = lane % RG;
      const int k = (lane / RG) % W;
      const int ln = lane / (RG * W);
      if (r < nr && mine != 0.0)
        grid_add(w, g + r * rhs_stride + rowoff_dyn<D, MM>(ch.col, ln, n) + wrap_cell(top - MM + 1 + k, n), mine);
    }
  } else {
    if (has) {
#pragma unroll
      for (int a = 0; a < LINES; ++a)
#pragma unroll
        for (int k = 0; k < W; ++k)
#pragma unroll
          for (int r = 0; r < RG; ++r)
            if (r < nr && acc[a][k][r] != 0.0)
              grid_add(w, g + r * rhs_stride + rowoff[a] + wrap_cell(top - MM + 1 + k, n), acc[a][k][r]);
    }
  }
}

// ----------------------------------------------------------------------------
// gather: out[perm] += eta * interp
//
// Persistent warps: warp w takes runs w, w + nw, w + 2nw ...  A run's starting window
// (the stencil around its first node's cell, Chunk::cell0) is copied into shared memory
// with cp.async while the warp still works on the previous run, so a run starts from
// shared memory instead of a dependent L2 round trip (ncu: that wait was 30% of the
// kernel when every warp owned a single run).
// ----------------------------------------------------------------------------
template <int D, int MM, int RG>
__device__ __forceinline__ void solo_window_prefetch(const Chunk& c, const double* g,
                                                     int64_t rhs_stride, int nr, int n, int lane,
                                                     double* dst) {
  using C = SoloCfg<D, MM>;
  constexpr int W = C::W, NWIN = C::NACC * RG;
#pragma unroll
  for (int e = lane; e < NWIN; e += 32) {
    const int r = e % RG, k = (e / RG) % W, a = e / (RG * W);
    const int64_t ix = rowoff_dyn<D, MM>(c.col, a, n) + wrap_cell(c.cell0 - MM + 1 + k, n);
    const double* src = g + (r < nr ? r : 0) * rhs_stride + ix;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + e);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src));
  }
  asm volatile("cp.async.commit_group;");
}

template <int D, int MM, int RG, int TAB>
__global__ void __launch_bounds__(128) k_gather_solo(const SortedSide sv, const Window w, int n,
                                                     const PolyTable T,
                                                     const double* __restrict__ grid,
                                                     int64_t rhs_stride, int nr,
                                                     double* __restrict__ out, int64_t ldo) {
  using C = SoloCfg<D, MM>;
  constexpr int W = C::W, LINES = C::LINES, NWIN = C::NACC * RG;
  __shared__ double s_win[4][2][NWIN];   // per warp: double-buffered starting windows
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t ci = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ci >= sv.nchunks) return;   // warp-uniform
  const double* g = grid + w.grid_off;
  // small windows prefetch the entering column into registers, 2-D windows into L1
  constexpr bool LOOKAHEAD = C::NACC * RG <= 32;

  Chunk ch = sv.chunks[ci];
  Chunk chn = ci + nw < sv.nchunks ? sv.chunks[ci + nw] : ch;
  solo_window_prefetch<D, MM, RG>(ch, g, rhs_stride, nr, n, lane, s_win[wib][0]);
  int buf = 0;

#pragma unroll 1
  for (; ci < sv.nchunks; ci += nw) {
    const bool has_next = ci + nw < sv.nchunks;
    // this run's starting window has landed; start the next run's and its successor's
    // descriptor
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    double gv[LINES][W][RG];
#pragma unroll
    for (int a = 0; a < LINES; ++a)
#pragma unroll
      for (int k = 0; k < W; ++k)
#pragma unroll
        for (int r = 0; r < RG; ++r) gv[a][k][r] = s_win[wib][buf][(a * W + k) * RG + r];
    __syncwarp();
    if (has_next) solo_window_prefetch<D, MM, RG>(chn, g, rhs_stride, nr, n, lane, s_win[wib][buf ^ 1]);
    const Chunk chnn = ci + 2 * nw < sv.nchunks ? sv.chunks[ci + 2 * nw] : chn;

    // grid index of (line a, cell c); row offsets are recomputed, not kept (registers)
    auto cell_index = [&](int a, int c) -> int64_t {
      return rowoff_dyn<D, MM>(ch.col, a, n) + wrap_cell(c, n);
    };
    double ahead[LINES][RG];
    int ahead_cell = INT_MIN;
    auto load_slot = [&](int k, int c) {
#pragma unroll
      for (int a = 0; a < LINES; ++a) {
        const int64_t ix = cell_index(a, c);
#pragma unroll
        for (int r = 0; r < RG; ++r) gv[a][k][r] = r < nr ? __ldg(g + r * rhs_stride + ix) : 0.0;
      }
    };
    int cur = ch.cell0;
    const int count = ch.count;
    SoloPipe<D, RG> pipe;
    pipe.prime(sv, ch, lane, nullptr, ldo, nr);   // no value prefetch: the result is added with RED
#pragma unroll 1
    for (int q = lane; q < count; q += 32) {
      double nx[D];
      double prior[RG];   // unused (zeros)
      const int j = pipe.advance(sv, ch, q, nx, prior, nullptr, ldo, nr);
      const int u = wrap_cell((int)floor(nx[D - 1]), n);
      if (u != cur) {
        if (LOOKAHEAD && u == cur + 1 && ahead_cell == u + MM) {
          // one-cell move: the entering cell was loaded during the previous node
#pragma unroll
          for (int a = 0; a < LINES; ++a)
#pragma unroll
            for (int r = 0; r < RG; ++r) {
#pragma unroll
              for (int k = 0; k + 1 < W; ++k) gv[a][k][r] = gv[a][k + 1][r];
              gv[a][W - 1][r] = ahead[a][r];
            }
        } else if (u > cur && u - cur < W) {
#pragma unroll 1
          for (int c = cur; c < u; ++c) {
#pragma unroll
            for (int a = 0; a < LINES; ++a)
#pragma unroll
              for (int r = 0; r < RG; ++r) {
#pragma unroll
                for (int k = 0; k + 1 < W; ++k) gv[a][k][r] = gv[a][k + 1][r];
              }
            load_slot(W - 1, c + MM + 1);
          }
        } else {
#pragma unroll
          for (int k = 0; k < W; ++k) load_slot(k, u - MM + 1 + k);
        }
        cur = u;
      }
      // look ahead: if this lane's next node sits one cell further, start loading its column
      if (q + 32 < count) {
        const int un = wrap_cell((int)floor(pipe.nx1[D - 1]), n);
        if (un == cur + 1 && ahead_cell != un + MM) {
          ahead_cell = un + MM;
#pragma unroll
          for (int a = 0; a < LINES; ++a) {
            const int64_t ix = cell_index(a, ahead_cell);
#pragma unroll
            for (int r = 0; r < RG; ++r) {
              if (LOOKAHEAD) {
                ahead[a][r] = r < nr ? __ldg(g + r * rhs_stride + ix) : 0.0;
              } else if (r < nr) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(g + r * rhs_stride + ix));
              }
            }
          }
        }
      }
      double wt[D][W];
      int u_w;
      solo_weights<D, MM, TAB>(nx, T, wt, u_w, n);
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        double s = 0.0;
#pragma unroll
        for (int ln = 0; ln < LINES; ++ln) {
          double t0 = 0.0, t1 = 0.0;
#pragma unroll
          for (int k = 0; k < W; k += 2) {
            t0 = fma(wt[D - 1][k], gv[ln][k][r], t0);
            if (k + 1 < W) t1 = fma(wt[D - 1][k + 1], gv[ln][k + 1][r], t1);
          }
          s = D == 2 ? fma(wt[0][ln], t0 + t1, s) : (t0 + t1);
        }
        // one RED per node and launch (RN add in L2): the bits of load + add + store
        if (r < nr) atomicAdd(out + r * ldo + j, __dmul_rn(w.eta, s));
      }
    }
    ch = chn;
    chn = chnn;
    buf ^= 1;
  }
}

}  // namespace afs
