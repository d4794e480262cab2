// Spread / gather for DENSE 2-D windows at m = 4: sub-cell Chebyshev kernels.
//
// The fast summation scales a window's nodes so that every pairwise distance fits the
// periodised kernel's exact ball (fastsum.py:210-217: scale = ball_radius / bbox diagonal),
// so a window's nodes occupy only ~(0.31 n)^2 grid cells: at C3 (N = 1e7, n = 128) about 400
// cells with ~25,000 nodes each.  With that many nodes per cell the per-node cost matters, not
// the per-cell one, and a cell can be cut much finer than the half-cells of tc2d.cuh:
//
//   sub-cell = (base cell u, sub-interval s = floor(16 f)) per dimension, f = n x - u.
//   On f in [s/16, (s+1)/16) every stencil offset's window value phi(f + 3 - o)
//   (nfft.py:118-122, 166-174) is an 8-term Chebyshev series in the local variable
//   t = 32 f - 2 s - 1 (kb_sub.inc: truncation 2e-17 of the peak; the half-cell needs 12),
//   so for one sub-cell the gather is
//       s(t0, t1) = sum_{a,b} G[a][b] phi_a phi_b = sum_{k,l} Ghat[k][l] T_k(t0) T_l(t1),
//       Ghat = C_s0^T G C_s1                                   (8x8x8 twice: 4 DMMAs)
//   of which the 40 coefficients with l < 8 - 2 floor(k/2) are kept (the rest are below
//   1e-16 of the window scale, tools/gen_kb_sub.py --check), against 104 for the half-cell
//   series of k_gather_cheb: 60 DFMAs per node instead of 136, and 20 instead of 52
//   broadcast loads per warp.  The spread is the dual: per sub-cell the moments
//       M[k][l] = sum_node alpha T_k(t0) T_l(t1)              (2 DMMAs per group of 8 nodes)
//   and at the end of the sub-cell G += C_s0 M C_s1^T (4 DMMAs) onto the 8x8 stencil.
//
// Layout (build_sorted_side_sc): nodes sorted by sub-cell, every sub-cell padded to a
// multiple of 8 nodes (perm = -1, t = 0), nx holding the Chebyshev variables t0, t1 and
// ghdr the group's (u0, u1, s0, s1).  Used when that padding is small (dense windows);
// sparse windows keep the half-cell kernels.  The node stream (TcRing) is tc2d.cuh's.
#pragma once

#include "tc2d.cuh"

#ifndef AFS_SC_MINB_GATHER
#define AFS_SC_MINB_GATHER 4
#endif
// 1: the spread's B fragments T_l(t1) are evaluated by the fragment lanes (monomial form)
// instead of being transposed through shared memory
#ifndef AFS_SC_BLANE
#define AFS_SC_BLANE 1
#endif
// 1: also the A fragments alpha T_k(t0) (no transposed tables at all: t0, t1, alpha broadcast)
#ifndef AFS_SC_ALANE
#define AFS_SC_ALANE 0
#endif
#ifndef AFS_SC_MINB_SPREAD
#define AFS_SC_MINB_SPREAD 4
#endif

namespace afs {

__device__ __forceinline__ int sc_u0(int32_t h) { return h & 0xfff; }
__device__ __forceinline__ int sc_u1(int32_t h) { return (h >> 12) & 0xfff; }
__device__ __forceinline__ int sc_s0(int32_t h) { return (h >> 24) & 0xf; }
__device__ __forceinline__ int sc_s1(int32_t h) { return (int)((uint32_t)h >> 28); }

// grid cell of stencil offset o for wrapped base cell u (m = 4): u - 3 + o mod n
template <bool POW2>
__device__ __forceinline__ int sc_cell(int u, int o, int n) {
  const int v = u - 3 + o;
  if constexpr (POW2) return v & (n - 1);
  else return wrap_cell(v, n);
}

constexpr int kScTab = 40;     // kept coefficients per sub-cell
#ifndef AFS_SC_GDEPTH
#define AFS_SC_GDEPTH 2
#endif
constexpr int kScGatherDepth = AFS_SC_GDEPTH;   // register pipeline depth of the gather (iterations; <= 4: the layout's tail)
constexpr int kScGatherU = 8;  // groups per gather iteration (two adjacent nodes per lane)
__host__ __device__ constexpr int sc_rowlen(int k) { return 8 - 2 * (k / 2); }
__host__ __device__ constexpr int sc_off(int k) {
  int o = 0;
  for (int j = 0; j < k; ++j) o += sc_rowlen(j);
  return o;
}

// ----------------------------------------------------------------------------
// gather: out[perm] += eta * s(t0, t1) over groups [g0, g1) of one warp; lane = node, 32 nodes
// (4 groups) per iteration.  The node stream goes global -> registers (coalesced, evict_first),
// software-pipelined: perm 4 iterations ahead, out[perm] (random, evict_last: the vector stays
// in L2 across the windows) 2 ahead, coordinates and headers 2 ahead, the stencils of new
// sub-cells 1 ahead.  Shared memory only holds the folded tables and the coefficient table.
// ----------------------------------------------------------------------------
// the block's copy of the sub-interval coefficient table (16 x 8 x 8 doubles)
template <int TAB>
__device__ __forceinline__ void sc_load_coefs(double* csub) {
  const double* src = kb_sub<TAB>(0);
  for (int i = threadIdx.x; i < kScSub * 64; i += blockDim.x) csub[i] = __ldg(src + i);
  __syncthreads();
}

template <int TAB, bool POW2, int D>
__global__ void __launch_bounds__(128, AFS_SC_MINB_GATHER) k_gather_sc(
    const SortedSide sv, const Window w, int n, const double* __restrict__ grid,
    double* __restrict__ out, int gpw) {
  // 64 nodes (8 groups) per iteration: lane takes the adjacent nodes 2 lane, 2 lane + 1 of
  // group lane / 4, which share one table, so every coefficient load feeds two nodes
  constexpr int U = kScGatherU;
  __shared__ __align__(16) double tabs[4][U + 1][kScTab];   // U new per iteration + the live one
  __shared__ __align__(16) double csub[kScSub * 64];
  sc_load_coefs<TAB>(csub);
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  const int wib = threadIdx.x >> 5;
  double* tab = &tabs[wib][0][0];
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g0 = warp * gpw;   // gpw is a multiple of U
  if (g0 >= sv.ngroups) return;   // warp-uniform (after the block-wide table load)
  const int g1 = min(g0 + gpw, (int)sv.ngroups);
  const double* g = grid + w.grid_off;
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  const int ug = lane >> 2;

  // packed store index of the lane's fold outputs Ghat[k = 2q + e][l = slot]; -1: not kept
  int sidx[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int k = 2 * q + e;
    sidx[e] = slot < sc_rowlen(k) ? sc_off(k) + slot : -1;
  }
  // Fold of one sub-cell's stencil G[a = slot][b = q + 4 s2] (L1/L2-resident grid) into its table:
  // Ghat^T = (C_s1^T G^T) C_s0: step 1 A[l = slot][b = q + 4 s2] = C_s1[b][l], B = G^T;
  // step 2 (k relabelled a = 2q + e) B[a][k = slot] = C_s0[a][k]
  auto fold = [&](int32_t h, double* dst) {
    const int row = sc_cell<POW2>(sc_u0(h), slot, n) * n;
    const double gv0 = __ldg(g + row + sc_cell<POW2>(sc_u1(h), q, n));
    const double gv1 = __ldg(g + row + sc_cell<POW2>(sc_u1(h), q + 4, n));
    const double* C0 = csub + sc_s0(h) * 64;
    const double* C1 = csub + sc_s1(h) * 64;
    const double ca0 = C1[q * 8 + slot], ca1 = C1[(q + 4) * 8 + slot];
    const double cb0 = C0[(2 * q) * 8 + slot], cb1 = C0[(2 * q + 1) * 8 + slot];
    double ht[2] = {0.0, 0.0};
    dmma884(ht, ca0, gv0);
    dmma884(ht, ca1, gv1);
    double gt[2] = {0.0, 0.0};
    dmma884(gt, ht[0], cb0);
    dmma884(gt, ht[1], cb1);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (sidx[e] >= 0) dst[sidx[e]] = gt[e];
  };
  int32_t hlast = -1;

  // lane's stream pointers at iteration 0 (the layout's empty tail covers the reads past g1)
  const double2* px0 = reinterpret_cast<const double2*>(sv.x0() + (int64_t)g0 * 8) + lane;
  const double2* px1 = reinterpret_cast<const double2*>(sv.x1() + (int64_t)g0 * 8) + lane;
  const int2* pperm = reinterpret_cast<const int2*>(sv.perm + (int64_t)g0 * 8) + lane;
  const int32_t* phdr = sv.ghdr + g0 + ug;
  // pipeline registers, kScGatherDepth iterations deep, indexed by iteration mod depth (the loop
  // is unrolled by the depth, so the indices are compile-time and no register is moved -- a
  // move would wait for its load): J perm, A/B coordinates, H headers
  constexpr int PD = kScGatherDepth;
  int2 J[PD];
  double2 A[PD], B[PD];
  int32_t H[PD];
#pragma unroll
  for (int r = 0; r < PD; ++r) {
    J[r] = ldg_hint(pperm + 32 * r, pol_stream);
    A[r] = ldg_hint(px0 + 32 * r, pol_stream);
    B[r] = ldg_hint(px1 + 32 * r, pol_stream);
    H[r] = __ldg(phdr + U * r);
  }
  int live = 0;   // table slot of the previous iteration's last group
#pragma unroll 1
  for (int gbd = g0; gbd < g1; gbd += PD * U) {
#pragma unroll
    for (int r = 0; r < PD; ++r) {
      if (gbd + r * U >= g1) break;   // warp-uniform
      // this iteration's nodes, then refill their registers with iteration + depth
      const double2 ta = A[r], tb = B[r];
      const int2 j = J[r];
      const int32_t hl = H[r];
      pperm += 32;
      px0 += 32;
      px1 += 32;
      phdr += U;
      J[r] = ldg_hint(pperm + 32 * (PD - 1), pol_stream);
      A[r] = ldg_hint(px0 + 32 * (PD - 1), pol_stream);
      B[r] = ldg_hint(px1 + 32 * (PD - 1), pol_stream);
      H[r] = __ldg(phdr + U * (PD - 1));
      __syncwarp();   // every lane is done reading the previous iteration's tables
      // tables of this iteration's new sub-cells go to the slots other than the live one
      // groups that start a new sub-cell: one ballot instead of walking the 8 headers
      const int32_t hprev = __shfl_up_sync(0xffffffffu, hl, 4);
      const bool first = q == 0 && (lane < 4 ? hl != hlast : hl != hprev);
      unsigned cm = __ballot_sync(0xffffffffu, first);   // bit 4u: group u starts a new sub-cell
      hlast = __shfl_sync(0xffffffffu, hl, 28);
      // the lane's table: the live one, or the (i-th new) slot of the last change up to its group
      const int before = __popc(cm & ((2u << (lane | 3)) - 1u));
      int mine = live, cur = live, nnew = 0;
      if (before > 0) mine = (before - 1) < live ? (before - 1) : before;
#pragma unroll 1
      while (cm) {   // usually no or one new sub-cell per iteration
        const int bit = __ffs(cm) - 1;
        cm &= cm - 1;
        const int32_t h = __shfl_sync(0xffffffffu, hl, bit);
        cur = nnew < live ? nnew : nnew + 1;
        ++nnew;
        fold(h, tab + cur * kScTab);
      }
      live = cur;
      __syncwarp();
      const double* T = tab + mine * kScTab;
      // Chebyshev values of the second coordinate of both nodes, then the table rows against
      // them with the outer recurrence in the first coordinate
      double ya[8], yb[8];
      ya[0] = 1.0;
      yb[0] = 1.0;
      ya[1] = tb.x;
      yb[1] = tb.y;
      const double va = 2.0 * tb.x, vb = 2.0 * tb.y;
#pragma unroll
      for (int l = 2; l < 8; ++l) {
        ya[l] = fma(va, ya[l - 1], -ya[l - 2]);
        yb[l] = fma(vb, yb[l - 1], -yb[l - 2]);
      }
      const double ua = 2.0 * ta.x, ub = 2.0 * ta.y;
      double am1 = 1.0, ak = 1.0, bm1 = 1.0, bk = 1.0, sa = 0.0, sb = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k == 1) {
          ak = ta.x;
          bk = ta.y;
        } else if (k >= 2) {
          const double an = fma(ua, ak, -am1), bn = fma(ub, bk, -bm1);
          am1 = ak;
          ak = an;
          bm1 = bk;
          bk = bn;
        }
        const double* row = T + sc_off(k);
        double pa = 0.0, pb = 0.0;
#pragma unroll
        for (int l = 0; l < sc_rowlen(k); l += 2) {
          const double2 c = *reinterpret_cast<const double2*>(row + l);
          pa = fma(c.x, ya[l], pa);
          pb = fma(c.x, yb[l], pb);
          pa = fma(c.y, ya[l + 1], pa);
          pb = fma(c.y, yb[l + 1], pb);
        }
        sa = fma(ak, pa, sa);
        sb = fma(bk, pb, sb);
      }
      // each node is written once per launch and launches on one vector are ordered, so the
      // reduction (RN add in L2, no load round trip) gives the bits of load + add + store
#ifdef AFS_SC_NO_RED   // measurement only: the gather without its output traffic
      if (j.x == -12345) red_hint(out, sa + sb, pol_keep);
#else
      if (j.x >= 0) red_hint(out + j.x, __dmul_rn(w.eta, sa), pol_keep);
      if (j.y >= 0) red_hint(out + j.y, __dmul_rn(w.eta, sb), pol_keep);
#endif
    }
  }
}

// ----------------------------------------------------------------------------
// spread: per sub-cell the moment matrix M = (alpha T(t0))^T T(t1) on the tensor cores,
// folded onto the 8x8 stencil (G += C_s0 M C_s1^T) and added to the grid when the group
// header changes (RED.F64 / fixed-point limbs, grid_add)
// ----------------------------------------------------------------------------
constexpr int kScStride = 36;   // staged row length (32 nodes + pad, = 4 mod 16: conflict-free)

template <int TAB, bool POW2, int D>
__global__ void __launch_bounds__(128, AFS_SC_MINB_SPREAD) k_spread_sc(
    const SortedSide sv, const Window w, int n, const double* __restrict__ alpha,
    double* __restrict__ grid, int gpw) {
  constexpr int U = 4;
  __shared__ __align__(16) double chx[4][8][kScStride];   // alpha T_k(t0) [k][node]
#if AFS_SC_BLANE
#if AFS_SC_ALANE
  __shared__ __align__(16) double ctx[4][32], cta[4][32];   // t0, alpha [node]
#endif
  __shared__ __align__(16) double cty[4][32];               // t1 [node]: T_l(t1) is evaluated by the fragment lanes
#else
  __shared__ __align__(16) double chy[4][8][kScStride];   // T_l(t1) [l][node]
#endif
  __shared__ __align__(16) double csub[kScSub * 64];
  sc_load_coefs<TAB>(csub);
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  const int wib = threadIdx.x >> 5;
  double(*CX)[kScStride] = chx[wib];
#if AFS_SC_BLANE
  double* CT = cty[wib];
#if AFS_SC_ALANE
  double* CT0 = ctx[wib];
  double* CA = cta[wib];
#endif
  // T_slot(t) = (slot odd ? t : 1) * P(t^2) with the lane's monomial coefficients: the B fragment
  // T_l(t1[node]) is evaluated where it is used (5 fp64 operations per value) instead of being
  // transposed through shared memory; the high orders' cancellation (T_7: 239 eps) is
  // weighted by Chebyshev coefficients below 1e-14 of the window's peak
  double pc[4];
  {
    constexpr double P[8][4] = {{1, 0, 0, 0},    {1, 0, 0, 0},       {-1, 2, 0, 0},      {-3, 4, 0, 0},
                                {1, -8, 8, 0},   {5, -20, 16, 0},    {-1, 18, -48, 32},  {-7, 56, -112, 64}};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double c = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k == slot) c = P[k][j];
      pc[j] = c;
    }
  }
  const bool odd = slot & 1;
#else
  double(*CY)[kScStride] = chy[wib];
#endif
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g0 = warp * gpw;
  if (g0 >= sv.ngroups) return;   // warp-uniform (after the block-wide table load)
  const int g1 = min(g0 + gpw, (int)sv.ngroups);
  double* g = grid + w.grid_off;
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();
  const int ug = lane >> 3;

  // per-group moment accumulators (independent DMMA chains): lane holds M[k = slot][l = 2q + e]
  double acc[U][2];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u][0] = acc[u][1] = 0.0;
  int32_t cur_h = -1;
  auto flush = [&]() {
    double m[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double v = acc[0][e];
      acc[0][e] = 0.0;
#pragma unroll
      for (int u = 1; u < U; ++u) {
        v += acc[u][e];
        acc[u][e] = 0.0;
      }
      m[e] = v;
    }
    const double* C0 = csub + sc_s0(cur_h) * 64;
    const double* C1 = csub + sc_s1(cur_h) * 64;
    // N^T[b = slot][k = 2q + e'] = sum_l C_s1[b][l] M[k][l]  (k-steps l = 2q + e: B = M fragment)
    double nt[2] = {0.0, 0.0};
    dmma884(nt, C1[slot * 8 + 2 * q], m[0]);
    dmma884(nt, C1[slot * 8 + 2 * q + 1], m[1]);
    // G^T[b = slot][a = 2q + e''] = sum_k N^T[b][k] C_s0[a][k]  (k-steps k = 2q + e')
    double gt[2] = {0.0, 0.0};
    dmma884(gt, nt[0], C0[slot * 8 + 2 * q]);
    dmma884(gt, nt[1], C0[slot * 8 + 2 * q + 1]);
    const int col = sc_cell<POW2>(sc_u1(cur_h), slot, n);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ix = sc_cell<POW2>(sc_u0(cur_h), 2 * q + e, n) * n + col;
      if (gt[e] != 0.0) grid_add(w, g + ix, gt[e]);
    }
  };

  // node stream global -> registers, as in k_gather_sc (alpha[perm] 2 iterations ahead)
  const double* px0 = sv.x0() + (int64_t)g0 * 8 + lane;
  const double* px1 = sv.x1() + (int64_t)g0 * 8 + lane;
  const int32_t* pperm = sv.perm + (int64_t)g0 * 8 + lane;
  const int32_t* phdr = sv.ghdr + g0 + ug;
  auto ld_alpha = [&](int32_t j) { return j >= 0 ? ldg_rand(alpha + j, pol_keep) : 0.0; };
  // pipeline registers, two batches deep, indexed by batch parity (loop unrolled by 2:
  // compile-time indices, no register moves): J holds the perm of batch + 2 (its alpha is
  // requested now, used two batches later) and is refilled with batch + 4; deeper did not help
  // (the random loads are bound by the outstanding-miss capacity)
  int32_t J[2];
  double A[2], B[2], AL[2];
  int32_t H[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    A[r] = ldg_hint(px0 + 32 * r, pol_stream);
    B[r] = ldg_hint(px1 + 32 * r, pol_stream);
    H[r] = __ldg(phdr + 4 * r);
    AL[r] = ld_alpha(ldg_hint(pperm + 32 * r, pol_stream));
    J[r] = ldg_hint(pperm + 32 * (r + 2), pol_stream);
  }
#pragma unroll 1
  for (int gb2 = g0; gb2 < g1; gb2 += 2 * U) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (gb2 + r * U >= g1) break;   // warp-uniform
      const double t0 = A[r], t1 = B[r], al = AL[r];
      const int32_t hl = H[r];
      pperm += 32;
      px0 += 32;
      px1 += 32;
      phdr += 4;
      A[r] = ldg_hint(px0 + 32, pol_stream);
      B[r] = ldg_hint(px1 + 32, pol_stream);
      H[r] = __ldg(phdr + 4);
      AL[r] = ld_alpha(J[r]);                        // batch + 2
      J[r] = ldg_hint(pperm + 96, pol_stream);       // batch + 4
      __syncwarp();   // every lane is done reading the previous batch's vectors
      {   // this lane's node: alpha T_k(t0) and T_l(t1), k, l < 8, into the transposed tables
        const double u2 = 2.0 * t0, v2 = 2.0 * t1;
        double tx0 = al, tx1 = al * t0, ty0 = 1.0, ty1 = t1;   // alpha rides the x recurrence
#if AFS_SC_BLANE && AFS_SC_ALANE
        CT[lane] = t1;
        CT0[lane] = t0;
        CA[lane] = al;
        (void)u2, (void)v2, (void)tx0, (void)tx1, (void)ty0, (void)ty1;
#elif AFS_SC_BLANE
        CX[0][lane] = tx0;
        CX[1][lane] = tx1;
        CT[lane] = t1;
        (void)v2, (void)ty0, (void)ty1;
#pragma unroll
        for (int k = 2; k < 8; ++k) {
          const double tx2 = fma(u2, tx1, -tx0);
          CX[k][lane] = tx2;
          tx0 = tx1;
          tx1 = tx2;
        }
#else
        CX[0][lane] = tx0;
        CX[1][lane] = tx1;
        CY[0][lane] = 1.0;
        CY[1][lane] = t1;
#pragma unroll
        for (int k = 2; k < 8; ++k) {
          const double tx2 = fma(u2, tx1, -tx0), ty2 = fma(v2, ty1, -ty0);
          CX[k][lane] = tx2;
          CY[k][lane] = ty2;
          tx0 = tx1;
          tx1 = tx2;
          ty0 = ty1;
          ty1 = ty2;
        }
#endif
      }
      int32_t hd[U];
#pragma unroll
      for (int u = 0; u < U; ++u) hd[u] = __shfl_sync(0xffffffffu, hl, 8 * u);
      __syncwarp();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (hd[u] != cur_h) {   // warp-uniform
          if (cur_h != -1) flush();
          cur_h = hd[u];
        }
        // M += (alpha T_x)^T T_y over the group's nodes (k-steps: nodes q + 4 s2)
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          const int nd = u * 8 + q + 4 * s2;
#if AFS_SC_BLANE && AFS_SC_ALANE
          const double tv = CT[nd], z = tv * tv;
          const double pz = fma(fma(fma(pc[3], z, pc[2]), z, pc[1]), z, pc[0]);
          const double tu = CT0[nd], zu = tu * tu;
          const double pu = fma(fma(fma(pc[3], zu, pc[2]), zu, pc[1]), zu, pc[0]);
          dmma884(acc[u], (odd ? pu * tu : pu) * CA[nd], odd ? pz * tv : pz);
#elif AFS_SC_BLANE
          const double tv = CT[nd], z = tv * tv;
          const double pz = fma(fma(fma(pc[3], z, pc[2]), z, pc[1]), z, pc[0]);
          dmma884(acc[u], CX[slot][nd], odd ? pz * tv : pz);
#else
          dmma884(acc[u], CX[slot][nd], CY[slot][nd]);
#endif
        }
      }
    }
  }
  if (cur_h != -1) flush();
}

// host launchers (sc2d.cu); the side must be in the sub-cell layout (sv.sc)
void launch_spread_sc(const SortedSide& sv, const Window& w, int n, int tab, const double* alpha,
                      int64_t lda, int R, double* grid, int64_t rs, cudaStream_t s);
void launch_gather_sc(const SortedSide& sv, const Window& w, int n, int tab, const double* grid,
                      int64_t rs, int R, double* out, int64_t ldo, cudaStream_t s);

}  // namespace afs
