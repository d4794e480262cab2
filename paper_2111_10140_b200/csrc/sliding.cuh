// Spread / gather over bin-sorted nodes with register sliding windows.
//
// Nodes of a window are sorted by base cell (row-major, last dimension
// fastest) and cut into column runs (Chunk).  A "team" of TEAM lanes takes
// one run.  Lane tl owns LPL "lines" of the stencil: the (2m)^(d-1) cells of
// the leading dimensions around the column base.  Along the last dimension
// each lane keeps a 2m-slot window of accumulators (spread) or grid values
// (gather) in registers; cell c lives in slot c mod 2m, so advancing the
// window never moves registers: leaving cells are flushed (spread:
// RED.E.ADD.F64 into the L2-resident grid) and entering cells loaded
// (gather; the cell one step ahead is prefetched so the common one-cell
// advance never waits on L2).  Per node, one lane evaluates the 2m*d window
// values once (per-table degree, kb_tables.inc / geometry.cuh) and stages them in shared
// memory; the last dimension's values are stored pre-rotated into slot order
// so the per-node work is a fixed, fully unrolled FMA sequence.
//
// Reference: the spread is nfft.py:241-245 (bincount of alpha * prod_t w_t),
// the gather nfft.py:228-229 ((g[flat] * w).sum(axis=1)), both over the
// tensor-product stencil of nfft.py:179-188.
#pragma once

#include <climits>

#include "geometry.cuh"

namespace afs {

// __launch_bounds__ min blocks per SM of the team kernels: one right-hand side at a time fits
// 4 blocks (<= 128 registers, no spills at m = 4; C3 3-D windows 4% faster than 3 blocks);
// two at a time need their registers (capped they spill: C4 gather 6.8 -> 8.9 ms)
// (m <= 4; larger cutoffs spill under the cap)
#ifndef AFS_TEAM3_MINB
#define AFS_TEAM3_MINB 4
#endif
template <int D, int MM, int RG>
constexpr int v2_min_blocks() { return (D == 3 && RG == 1 && MM <= 4) ? AFS_TEAM3_MINB : 1; }
#ifndef AFS_TEAM3
#define AFS_TEAM3 32   // lanes per run for 3-D windows (power of two, 8..32)
#endif

template <int D, int MM>
struct Cfg {
  static constexpr int W = 2 * MM;
  static constexpr int LINES = D == 3 ? W * W : (D == 2 ? W : 1);
  static constexpr int TEAM_AUTO =
      D == 1 ? 1
             : (LINES > 16 ? 32 : (LINES > 8 ? 16 : (LINES > 4 ? 8 : (LINES > 2 ? 4 : (LINES > 1 ? 2 : 1)))));
  static constexpr int TEAM = (D == 3 && TEAM_AUTO > AFS_TEAM3) ? AFS_TEAM3 : TEAM_AUTO;
  static constexpr int LPL = (LINES + TEAM - 1) / TEAM;
  static constexpr int TPW = 32 / TEAM;
};

template <int D, int MM, int RG>
struct Fits {
  static constexpr bool value = Cfg<D, MM>::LPL * Cfg<D, MM>::W * RG <= 64;
};

// staging row strides: S = 2 (mod 4) doubles keeps per-lane STS.128 conflict-free and
// keeps every even offset 16-byte aligned
__host__ __device__ constexpr int pad_stride(int s) { return s + ((6 - (s & 3)) & 3); }

template <int D>
struct NodesPerLane;

template <int D, int MM, int EXTRA, int MIN_STRIDE = 0>
struct Stage {
  static constexpr int W = 2 * MM;
  static constexpr int P = NodesPerLane<D>::P;                        // nodes per lane per round
  static constexpr int BATCH = Cfg<D, MM>::TEAM * P;                  // nodes per team per round
  static constexpr int STRIDE =                                       // per node
      pad_stride(D * W + EXTRA > MIN_STRIDE ? D * W + EXTRA : MIN_STRIDE);
  static constexpr int TEAM_SPAN = BATCH * STRIDE + 2;                // per team (+2: bank skew)
  static constexpr int WARP_SPAN = Cfg<D, MM>::TPW * TEAM_SPAN;
  static constexpr int U_OFF = D * W;                                 // int bits of the base cell
  static constexpr int A_OFF = D * W + 1;                             // alpha values (spread)
};

// c lies in [-n, 2n): the stencil never reaches further than m < n cells outside
__device__ __forceinline__ int wrap_cell(int c, int n) {
  return c < 0 ? c + n : (c >= n ? c - n : c);
}

// L2 eviction policies (createpolicy).  Node streams are read once per launch -> evict_first;
// the randomly indexed vector (alpha[perm], out[perm]: 80 MB at N = 1e7, it fits the 126 MB
// L2) is touched by every window -> evict_last, so its sectors stay resident.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ldg_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ldg_hint(const double2* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int2 ldg_hint(const int2* p, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
// random 8-byte load: no L1 allocation (a line would be used once), L2 policy
__device__ __forceinline__ double ldg_rand(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void red_hint(double* p, double v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ int32_t ldg_hint(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// (k - lo) mod W for compile-time W
template <int W>
__device__ __forceinline__ int slot_rel(int k, int lo) {
  if constexpr ((W & (W - 1)) == 0) {
    return (k - lo) & (W - 1);
  } else {
    int off = (k - lo) % W;
    return off < 0 ? off + W : off;
  }
}

struct LineGeom {
  int64_t off;   // grid index of (line, last = 0)
  int a, b;      // stencil digits of the leading dims
  bool valid;
};

template <int D, int MM>
__device__ __forceinline__ void line_geometry(int tl, int col, int n,
                                              LineGeom (&lg)[Cfg<D, MM>::LPL]) {
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

// prefetched per-node inputs of the next staging round
template <int D>
struct NodeIn {
  double nx[D];
  int perm;
};

template <int D>
__device__ __forceinline__ void load_node(const SortedSide& sv, int64_t i, NodeIn<D>& in) {
#pragma unroll
  for (int t = 0; t < D; ++t) in.nx[t] = __ldcs(sv.nx + t * sv.N + i);   // streamed once
  in.perm = __ldcs(sv.perm + i);
}

// Nodes staged per lane per round: the Horner evaluations of all P nodes x D dims
// share each coefficient (a double constant costs two MOVs to materialise).
template <int D>
struct NodesPerLane {
  static constexpr int P = D == 3 ? 1 : (D == 2 ? 2 : 4);
};

// Staging-round input pipeline: lane tl stages nodes b0 + tl + TEAM*p (p < P).  Two rounds
// in flight: stage 2 holds nx/perm of round b0+2*BATCH, stage 1 holds round b0+BATCH plus
// its gathered value val[perm] (alpha in the spread, out in the gather), so the dependent
// random load overlaps a whole round of work.
template <int D, int MM, int EXTRA, int TAB, int RG>
struct Round {
  using S = Stage<D, MM, EXTRA>;
  static constexpr int P = S::P, TEAM = Cfg<D, MM>::TEAM, BATCH = S::BATCH;
  NodeIn<D> n1[P], n2[P];
  double v1[P][RG];

  __device__ __forceinline__ void load_round(const SortedSide& sv, const Chunk& ch, bool active,
                                             int tl, int b0, NodeIn<D> (&dst)[P]) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int q = b0 + tl + TEAM * p;
      if (active && q < ch.count) {
        load_node<D>(sv, ch.begin + q, dst[p]);
      } else {
        dst[p].perm = -1;
      }
    }
  }
  __device__ __forceinline__ void load_vals(const double* __restrict__ src, int64_t ld, int nr) {
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int r = 0; r < RG; ++r)
        v1[p][r] = (src != nullptr && n1[p].perm >= 0 && r < nr) ? src[r * ld + n1[p].perm] : 0.0;
  }
  __device__ __forceinline__ void prime(const SortedSide& sv, const Chunk& ch, bool active, int tl,
                                        const double* __restrict__ src, int64_t ld, int nr) {
    load_round(sv, ch, active, tl, 0, n1);
    load_vals(src, ld, nr);
    load_round(sv, ch, active, tl, BATCH, n2);
  }
  // hand out round b0 (in flight since two rounds) and refill the pipe with b0 + 2*BATCH
  __device__ __forceinline__ void advance(const SortedSide& sv, const Chunk& ch, bool active,
                                          int tl, int b0, NodeIn<D> (&in)[P],
                                          double (&val)[P][RG], const double* __restrict__ src,
                                          int64_t ld, int nr) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      in[p] = n1[p];
#pragma unroll
      for (int r = 0; r < RG; ++r) val[p][r] = v1[p][r];
      n1[p] = n2[p];
    }
    load_vals(src, ld, nr);
    load_round(sv, ch, active, tl, b0 + 2 * BATCH, n2);
  }
};

// Stage P nodes: window values of all dims (last dim rotated to slot order) + base cell.
// Values for f > 1/2 come from the mirrored polynomial (geometry.cuh) and are written to
// the mirrored stencil position.
template <int D, int MM, int EXTRA, int TAB, int P>
__device__ __forceinline__ void stage_nodes(const NodeIn<D> (&in)[P], const bool (&live)[P], int n,
                                            const PolyTable& T, double* const (&row)[P]) {
  constexpr int W = 2 * MM;
  double x[P][D];
  int pos0[P][D];   // store position of offset 0; step +1 or -1 (mirrored)
  int step[P][D];
#pragma unroll
  for (int p = 0; p < P; ++p) {
#pragma unroll
    for (int t = 0; t < D; ++t) {
      const double nx = in[p].nx[t];
      const double fl = floor(nx);
      const double f = nx - fl;   // exact
      const bool refl = f > 0.5;
      x[p][t] = (refl ? __dsub_rn(1.0, f) : f) - 0.25;
      int base = 0;
      if (t == D - 1) {
        const int u = wrap_cell((int)fl, n);
        base = slot_rel<W>(u + MM + 1, 0);   // slot of stencil offset 0
        row[p][Stage<D, MM, EXTRA>::U_OFF] = __longlong_as_double((long long)u);
      }
      pos0[p][t] = refl ? base + W - 1 : base;
      step[p][t] = refl ? -1 : 1;
    }
  }
  // all W*P*D Horner chains advance together (k outer): W*P*D independent FMAs per step
  // hide the DFMA latency, and each coefficient is materialised once for P*D uses
  double v[W][P][D];
  constexpr int NT = TAB == 0 ? kPolyTerms : kb_terms<TAB, MM>();   // per-table degree
#pragma unroll
  for (int k = NT - 1; k >= 0; --k) {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const double c = TAB == 0 ? T.c[i][k] : kb_coef<TAB, MM>(i, k);
#pragma unroll
      for (int p = 0; p < P; ++p)
#pragma unroll
        for (int t = 0; t < D; ++t)
          v[i][p][t] = k == NT - 1 ? c : fma(v[i][p][t], x[p][t], c);
    }
  }
  // stores are unconditional (rows of dead nodes are never read)
#pragma unroll
  for (int i = 0; i < W; ++i) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
      for (int t = 0; t < D; ++t) {
        int s = pos0[p][t] + step[p][t] * i;   // in (-W, 2W)
        if (t == D - 1) s = s >= W ? s - W : (s < 0 ? s + W : s);
        row[p][t * W + s] = v[i][p][t];
      }
    }
  }
}

template <int D, int MM>
__device__ __forceinline__ double line_weight(const double* row, const LineGeom& g) {
  if (D == 3) return g.valid ? row[g.a] * row[Cfg<D, MM>::W + g.b] : 0.0;
  if (D == 2) return g.valid ? row[g.a] : 0.0;
  return 1.0;
}

template <int W>
__device__ __forceinline__ void load_last(const double* row_last, double (&wl)[W]) {
#pragma unroll
  for (int k = 0; k < W; k += 2) {
    const double2 v = *reinterpret_cast<const double2*>(row_last + k);
    wl[k] = v.x;
    wl[k + 1] = v.y;
  }
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ----------------------------------------------------------------------------
// spread
// ----------------------------------------------------------------------------
template <int D, int MM, int RG, int TAB>
__global__ void __launch_bounds__(128, v2_min_blocks<D, MM, RG>()) k_spread_v2(const SortedSide sv, const Window w, int n,
                                                   const PolyTable T,
                                                   const double* __restrict__ alpha, int64_t lda,
                                                   int nr, double* __restrict__ grid,
                                                   int64_t rhs_stride) {
  using C = Cfg<D, MM>;
  using S = Stage<D, MM, 1 + RG>;
  constexpr int W = C::W, TEAM = C::TEAM, LPL = C::LPL, TPW = C::TPW;
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int team = lane / TEAM, tl = lane - team * TEAM;
  double* st = sm + (size_t)(threadIdx.x >> 5) * S::WARP_SPAN + (size_t)team * S::TEAM_SPAN;
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

  // flush the slots of the window starting at cell lo whose offset from lo is < nleave
  auto flush = [&](int lo, int nleave) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int rel = slot_rel<W>(k, lo);
      if (rel < nleave) {
        const int cm = wrap_cell(lo + rel, n);
#pragma unroll
        for (int j = 0; j < LPL; ++j) {
          if (lg[j].valid) {
#pragma unroll
            for (int r = 0; r < RG; ++r)
              if (r < nr) grid_add(w, g + r * rhs_stride + lg[j].off + cm, acc[j][k][r]);
          }
#pragma unroll
          for (int r = 0; r < RG; ++r) acc[j][k][r] = 0.0;
        }
      }
    }
  };

  int cur = INT_MIN;
  const int rounds = warp_max(ch.count);
  constexpr int P = S::P, BATCH = S::BATCH;
  Round<D, MM, 1 + RG, TAB, RG> rd;
  rd.prime(sv, ch, active, tl, alpha, lda, nr);
  for (int b0 = 0; b0 < rounds; b0 += BATCH) {
    {
      NodeIn<D> in[P];
      bool live[P];
      double* rows[P];
      double a[P][RG];
      rd.advance(sv, ch, active, tl, b0, in, a, alpha, lda, nr);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        live[p] = in[p].perm >= 0;
        rows[p] = st + (tl + TEAM * p) * S::STRIDE;
      }
      stage_nodes<D, MM, 1 + RG, TAB, P>(in, live, n, T, rows);
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (live[p]) {
          if constexpr (RG == 1 && D >= 2) {
            // one right-hand side: fold alpha into the last dimension's staged values, so
            // the per-node loop of every lane skips one load and one multiply per line
#pragma unroll
            for (int k = 0; k < W; ++k) rows[p][(D - 1) * W + k] *= a[p][0];
          } else {
#pragma unroll
            for (int r = 0; r < RG; ++r) rows[p][S::A_OFF + r] = a[p][r];
          }
        }
    }
    __syncwarp();
    const int cnt = active ? min(BATCH, ch.count - b0) : 0;
    int q = 0;
    int u = cnt > 0 ? (int)__double_as_longlong(st[S::U_OFF]) : 0;
    while (q < cnt) {
      // window move (rare), then a branch-free run of nodes sharing base cell u
      if (u != cur) {
        if (cur != INT_MIN) flush(cur - MM + 1, u - cur);
        cur = u;
      }
      do {
        const double* row = st + q * S::STRIDE;
        ++q;
        u = q < cnt ? (int)__double_as_longlong(row[S::STRIDE + S::U_OFF]) : INT_MIN;
        double wl[W];
        load_last<W>(row + (D - 1) * W, wl);
#pragma unroll
        for (int j = 0; j < LPL; ++j) {
          const double lw = line_weight<D, MM>(row, lg[j]);
#pragma unroll
          for (int r = 0; r < RG; ++r) {
            // RG == 1, D >= 2: alpha is folded into wl at staging
            const double p = (RG == 1 && D >= 2) ? lw : lw * row[S::A_OFF + r];
#pragma unroll
            for (int k = 0; k < W; ++k) acc[j][k][r] = fma(p, wl[k], acc[j][k][r]);
          }
        }
      } while (u == cur);
    }
    __syncwarp();
  }
  if (active && cur != INT_MIN) flush(cur - MM + 1, W);
}

// ----------------------------------------------------------------------------
// gather: out[perm] += eta * interp
// ----------------------------------------------------------------------------
template <int TEAM>
struct Red {
  static constexpr int RSTR = TEAM == 1 ? 1 : (TEAM + 2);   // even, RSTR/2 odd for TEAM >= 4
};

template <int D, int MM, int RG, int TAB>
__global__ void __launch_bounds__(128, v2_min_blocks<D, MM, RG>()) k_gather_v2(const SortedSide sv, const Window w, int n,
                                                   const PolyTable T,
                                                   const double* __restrict__ grid,
                                                   int64_t rhs_stride, int nr,
                                                   double* __restrict__ out, int64_t ldo) {
  using C = Cfg<D, MM>;
  constexpr int RSTR = Red<C::TEAM>::RSTR;
  // a node's staging row is reused for its per-lane partial sums once it is processed
  using S = Stage<D, MM, 1, RG * RSTR>;
  constexpr int W = C::W, TEAM = C::TEAM, LPL = C::LPL, TPW = C::TPW;
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int team = lane / TEAM, tl = lane - team * TEAM;
  const unsigned team_mask = TEAM == 32 ? 0xffffffffu : (((1u << TEAM) - 1u) << (team * TEAM));
  double* st = sm + (size_t)wib * S::WARP_SPAN + (size_t)team * S::TEAM_SPAN;
  constexpr int P = S::P, BATCH = S::BATCH;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t ci = gwarp * TPW + team;
  const bool active = ci < sv.nchunks;
  Chunk ch{0, 0, 0};
  if (active) ch = sv.chunks[ci];
  LineGeom lg[LPL];
  line_geometry<D, MM>(tl, ch.col, n, lg);
  const double* g = grid + w.grid_off;
  const uint64_t pol_keep = l2_policy_evict_last();

  double gv[LPL][W][RG];
  double ahead[LPL][RG];   // grid values of cell cur + MM + 1 (prefetched)
  int cur = INT_MIN;
  auto load_cell = [&](int c, int j, int r) -> double {
    return (lg[j].valid && r < nr) ? __ldg(g + r * rhs_stride + lg[j].off + wrap_cell(c, n)) : 0.0;
  };

  const int rounds = warp_max(ch.count);
  Round<D, MM, 1, TAB, RG> rd;
  // no value prefetch: the result is added with one reduction per node (RED.ADD.F64 in L2 --
  // each node is written once per launch and launches on one vector are ordered, so the bits
  // are those of load + add + store, without the random load's round trip)
  rd.prime(sv, ch, active, tl, nullptr, ldo, nr);
  for (int b0 = 0; b0 < rounds; b0 += BATCH) {
    int my_perm[P];
    double prior[P][RG];   // unused (zeros)
    {
      NodeIn<D> in[P];
      bool live[P];
      double* rows[P];
      rd.advance(sv, ch, active, tl, b0, in, prior, nullptr, ldo, nr);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        live[p] = in[p].perm >= 0;
        rows[p] = st + (tl + TEAM * p) * S::STRIDE;
        my_perm[p] = in[p].perm;
      }
      stage_nodes<D, MM, 1, TAB, P>(in, live, n, T, rows);
    }
    __syncwarp();
    const int cnt = active ? min(BATCH, ch.count - b0) : 0;
    int q = 0;
    int u = cnt > 0 ? (int)__double_as_longlong(st[S::U_OFF]) : 0;
    while (q < cnt) {
      if (u != cur) {
        const int lo = u - MM + 1;
        if (u == cur + 1) {
          // one-cell advance: the entering cell u + MM was prefetched
          const int k = slot_rel<W>(u + MM, 0);
#pragma unroll
          for (int kk = 0; kk < W; ++kk)
            if (kk == k) {
#pragma unroll
              for (int j = 0; j < LPL; ++j)
#pragma unroll
                for (int r = 0; r < RG; ++r) gv[j][kk][r] = ahead[j][r];
            }
        } else {
#pragma unroll
          for (int k = 0; k < W; ++k) {
            const int c = lo + slot_rel<W>(k, lo);
            if (cur == INT_MIN || c > cur + MM) {
#pragma unroll
              for (int j = 0; j < LPL; ++j)
#pragma unroll
                for (int r = 0; r < RG; ++r) gv[j][k][r] = load_cell(c, j, r);
            }
          }
        }
        cur = u;
#pragma unroll
        for (int j = 0; j < LPL; ++j)
#pragma unroll
          for (int r = 0; r < RG; ++r) ahead[j][r] = load_cell(u + MM + 1, j, r);
      }
      do {
        const double* row = st + q * S::STRIDE;
        const int qq = q++;
        u = q < cnt ? (int)__double_as_longlong(row[S::STRIDE + S::U_OFF]) : INT_MIN;
        double wl[W];
        load_last<W>(row + (D - 1) * W, wl);
        double part[RG];
#pragma unroll
        for (int r = 0; r < RG; ++r) part[r] = 0.0;
#pragma unroll
        for (int j = 0; j < LPL; ++j) {
          const double lw = line_weight<D, MM>(row, lg[j]);
#pragma unroll
          for (int r = 0; r < RG; ++r) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int k = 0; k < W; k += 2) {
              s0 = fma(wl[k], gv[j][k][r], s0);
              if (k + 1 < W) s1 = fma(wl[k + 1], gv[j][k + 1][r], s1);
            }
            part[r] = fma(lw, s0 + s1, part[r]);
          }
        }
        __syncwarp(team_mask);   // every lane of the team is done reading row qq
        double* prow = st + qq * S::STRIDE;
#pragma unroll
        for (int r = 0; r < RG; ++r) prow[r * RSTR + tl] = part[r];
      } while (u == cur);
    }
    __syncwarp();
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (my_perm[p] < 0) continue;
      const int qq = tl + TEAM * p;
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        if (r < nr) {
          double s;
          const double* rr = st + qq * S::STRIDE + r * RSTR;
          if (TEAM == 1) {
            s = rr[0];
          } else {
            double v[TEAM];
#pragma unroll
            for (int k = 0; k < TEAM; k += 2) {
              const double2 x = *reinterpret_cast<const double2*>(rr + k);
              v[k] = x.x;
              v[k + 1] = x.y;
            }
#pragma unroll
            for (int h = TEAM / 2; h >= 1; h >>= 1)
#pragma unroll
              for (int k = 0; k < h; ++k) v[k] += v[k + h];
            s = v[0];
          }
          red_hint(out + r * ldo + my_perm[p], __dmul_rn(w.eta, s), pol_keep);
        }
      }
    }
    __syncwarp();
  }
}

// host-side launchers (instantiated per dimension in sliding_d{1,2,3}.cu)
template <int D>
bool launch_spread_v2(const SortedSide& sv, const Window& w, int n, int m, int tab, const PolyTable& T,
                      const double* alpha, int64_t lda, int nr, double* grid, int64_t rs,
                      cudaStream_t s);
template <int D>
bool launch_gather_v2(const SortedSide& sv, const Window& w, int n, int m, int tab, const PolyTable& T,
                      const double* grid, int64_t rs, int nr, double* out, int64_t ldo,
                      cudaStream_t s);
int v2_rhs_group(int D, int m, int R, bool spread);   // right-hand sides per pass
struct SoloBatch;   // solo.cuh
void launch_spread_solo_batch_1d(const SoloBatch& B, int n, int m, int tab, const PolyTable& T,
                                 const double* alpha, int64_t lda, int R, double* grid, int64_t rs,
                                 cudaStream_t s);

}  // namespace afs
