// Spread / gather for 2-D windows at m = 4 on the fp64 tensor cores (DMMA, mma.sync
// m8n8k4 f64).
//
// Nodes are sorted by half-cell -- base cell u = floor(n x) and reflection class
// c = (f > 1/2) per dimension -- and every half-cell is padded to a multiple of 8 nodes
// (build_sorted_side_tc), so each group of 8 consecutive nodes shares one 8x8 stencil.
// Per group and dimension the window values are one matrix product
//     Phi[node][o] = sum_k x_node^k C[o][k]      (8 nodes x 12 terms x 8 offsets)
// with x = (c ? 1 - f : f) - 1/4 (stored at plan time) and C the constant-bank KB polynomial table
// (geometry.cuh poly_weights), i.e. three DMMAs.  The reflection only permutes the
// stencil (phi(f + m-1-o) = P_{7-o}(x) when c = 1), which the kernels fold into the grid
// addressing.  The tensor-product touch is two more DMMAs:
//     gather  s_node  = sum_p (Phi_x G)[node][p] Phi_y[node][p]        (nfft.py:228-229)
//     spread  G[o][p] += sum_node alpha_node Phi_x[node][o] Phi_y[node][p] (nfft.py:241-245)
// The fragment layouts line up without shuffles: the eval result D[row][2q+t] is directly
// the A (gather) or, evaluated transposed, the A/B (spread) operand of the touch MMA with
// k relabelled as offset (or node) 2k+t.  Per group the spread runs 8 DMMAs = 2048 fp64
// MACs, against ~1980 DFMAs of the lane-private FMA kernels (solo.cuh) -- the same
// arithmetic, but one instruction per 256 MACs, so the fp64 pipe stops waiting on issue.
// The gather folds Phi_x's coefficient matrix into the grid once per half-cell
// (P_x (C G) instead of (P_x C) G, see k_gather_tc) and runs 6 per group.
#pragma once

#include <algorithm>

// __launch_bounds__ min blocks per SM (register caps) of the one-rhs gather and spread, tuning hooks
#ifndef AFS_TC_MINB_GATHER
#define AFS_TC_MINB_GATHER 5
#endif
#ifndef AFS_TC_MINB_SPREAD
#define AFS_TC_MINB_SPREAD 1
#endif
#ifndef AFS_TC_MINB_CHEB
#define AFS_TC_MINB_CHEB 4
#endif
#ifndef AFS_TC_MINB_CHEB_SPREAD
#define AFS_TC_MINB_CHEB_SPREAD 3
#endif

#include "geometry.cuh"
#include "sliding.cuh"

namespace afs {

// d[0..1] += A(8x4) B(4x8): lane holds a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// d = D[lane/4][2(lane%4) + {0,1}].  Not volatile: independent groups may interleave.
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

template <int TAB>
struct TcPoly {
  static constexpr int NT = kb_terms<TAB, 4>();
  static constexpr int NKS = (NT + 3) / 4;   // k-steps of 4 terms
};

// lane's coefficient fragment: C[o = lane/4][k = lane%4 + 4s].  Laundered through a
// volatile move so ptxas keeps it in registers instead of re-reading the constant bank
// (divergent LDC) every iteration.
template <int TAB>
__device__ __forceinline__ void tc_coefs(int lane, double (&cf)[TcPoly<TAB>::NKS]) {
  constexpr int NT = TcPoly<TAB>::NT;
#pragma unroll
  for (int s = 0; s < TcPoly<TAB>::NKS; ++s) {
    const int k = (lane & 3) + 4 * s;
    const double c = k < NT ? kb_coef<TAB, 4>(lane >> 2, k) : 0.0;
    asm volatile("mov.b64 %0, %1;" : "=d"(cf[s]) : "d"(c));
  }
}

// lane's power fragment x^(q + 4s), q = lane % 4 (q1: q odd, q2: q >= 2)
template <int NKS>
__device__ __forceinline__ void tc_powers(double x, bool q1, bool q2, double (&pw)[NKS]) {
  const double x2 = x * x;
  const double x4 = x2 * x2;
  const double p0 = (q1 ? x : 1.0) * (q2 ? x2 : 1.0);
  pw[0] = p0;
  if constexpr (NKS > 1) pw[1] = p0 * x4;
  if constexpr (NKS > 2) pw[2] = pw[1] * x4;
  if constexpr (NKS > 3) pw[3] = pw[2] * x4;
}

// Squares shared by the quad (spread).  The 4 lanes of a quad hold the same node, so the x^2,
// x^4 every lane needs are computed once per batch -- lane l for node l % 8 of group l / 8
// (the batch's 32 nodes) -- and read back from a per-warp table: 4 DMULs per batch instead of
// 4 per group and lane (the fp64 pipe is shared with the DMMAs).  The gather measured 1.3%
// slower with the same table.
template <int NV>
struct TcPow {
  double v[NV][32];   // [value][group * 8 + node]
};

// tc_powers given x^2, x^4
template <int NKS>
__device__ __forceinline__ void tc_powers_x24(double x, double x2, double x4, bool q1, bool q2,
                                              double (&pw)[NKS]) {
  const double p0 = (q1 ? x : 1.0) * (q2 ? x2 : 1.0);
  pw[0] = p0;
  if constexpr (NKS > 1) pw[1] = p0 * x4;
  if constexpr (NKS > 2) pw[2] = pw[1] * x4;
  if constexpr (NKS > 3) pw[3] = pw[2] * x4;
}

// grid cell of stencil slot o (polynomial order) for wrapped base cell u, class c (m = 4):
// u - 3 + (c ? 7 - o : o) mod n; 7 - o = o ^ 7.  POW2: n is a power of two (mask n - 1)
template <bool POW2>
__device__ __forceinline__ int tc_cell(int u, int c, int o, int n) {
  const int v = u - 3 + (o ^ (c ? 7 : 0));
  if constexpr (POW2) return v & (n - 1);
  else return wrap_cell(v, n);
}
__device__ __forceinline__ int tc_u0(int32_t h) { return h & 0x3fff; }
__device__ __forceinline__ int tc_u1(int32_t h) { return (h >> 14) & 0x3fff; }
__device__ __forceinline__ int tc_c0(int32_t h) { return (h >> 28) & 1; }
__device__ __forceinline__ int tc_c1(int32_t h) { return (h >> 29) & 1; }

// ---------------------------------------------------------------------------
// Node stream.  A warp walks its groups U at a time ("batches") through a per-warp
// shared-memory ring of D batches filled with cp.async, so no registers are held for
// loads in flight:
//   iteration b stages the node data (x0, x1, perm, header) of batch b + D, and the
//   random per-node values of batch b + 2 (out[perm] in the gather, alpha[perm] in the
//   spread; their perm landed two iterations earlier);
//   the grid window operands of batch b + 1 (gather) are loaded into registers.
// ---------------------------------------------------------------------------
template <int U, int D, int RG>
struct TcRing {
  double x0[D][8 * U];
  double x1[D][8 * U];
  double val[D][RG][8 * U];
  int32_t perm[D][8 * U];
  alignas(16) int32_t hdr[D][U];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void* dst, const void* src, uint64_t pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async8_hint(void* dst, const void* src, uint64_t pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(sa), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(double* ptr, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(ptr), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// node data of batch gb (groups gb .. gb+U-1) into slot st, 16 B chunks: [0,4U) x0,
// [4U,8U) x1, [8U,10U) perm, then the U headers (4U bytes; gb is a multiple of U)
template <int U, int D, int RG>
__device__ __forceinline__ void tc_stage_nodes(TcRing<U, D, RG>& R, int st, const SortedSide& sv,
                                               int gb, int lane) {
  static_assert(U == 1 || U == 2 || U == 4 || U == 8, "batch of 1, 2, 4 or 8 groups");
  constexpr int NH = U == 8 ? 2 : 1;   // 16-byte header chunks
  const int i0 = gb * 8;
#pragma unroll
  for (int c = lane; c < 10 * U + NH; c += 32) {
    if (c < 4 * U) {
      cp_async16(&R.x0[st][2 * c], sv.x0() + i0 + 2 * c);
    } else if (c < 8 * U) {
      cp_async16(&R.x1[st][2 * (c - 4 * U)], sv.x1() + i0 + 2 * (c - 4 * U));
    } else if (c < 10 * U) {
      cp_async16(&R.perm[st][4 * (c - 8 * U)], sv.perm + i0 + 4 * (c - 8 * U));
    } else {
      if constexpr (U >= 4) cp_async16(&R.hdr[st][4 * (c - 10 * U)], sv.ghdr + gb + 4 * (c - 10 * U));
      else if constexpr (U == 2) cp_async8(&R.hdr[st][0], sv.ghdr + gb);
      else cp_async4(&R.hdr[st][0], sv.ghdr + gb);
    }
  }
}

// tc_stage_nodes with an L2 policy on the 16-byte copies (U = 4)
template <int U, int D, int RG>
__device__ __forceinline__ void tc_stage_nodes_hint(TcRing<U, D, RG>& R, int st, const SortedSide& sv,
                                                    int gb, int lane, uint64_t pol) {
  static_assert(U == 4, "lane = node batches");
  const int i0 = gb * 8;
#pragma unroll
  for (int c = lane; c < 10 * U + 1; c += 32) {
    if (c < 4 * U) {
      cp_async16_hint(&R.x0[st][2 * c], sv.x0() + i0 + 2 * c, pol);
    } else if (c < 8 * U) {
      cp_async16_hint(&R.x1[st][2 * (c - 4 * U)], sv.x1() + i0 + 2 * (c - 4 * U), pol);
    } else if (c < 10 * U) {
      cp_async16_hint(&R.perm[st][4 * (c - 8 * U)], sv.perm + i0 + 4 * (c - 8 * U), pol);
    } else {
      cp_async16_hint(&R.hdr[st][0], sv.ghdr + gb, pol);
    }
  }
}

// tc_stage_vals (one right-hand side) with an L2 policy on the random 8-byte copies
template <int U, int D>
__device__ __forceinline__ void tc_stage_vals_hint(TcRing<U, D, 1>& R, int st, const double* src,
                                                   int lane, uint64_t pol) {
#pragma unroll
  for (int i = lane; i < 8 * U; i += 32) {
    const int j = R.perm[st][i];
    if (j >= 0) cp_async8_hint(&R.val[st][0][i], src + j, pol);
    else R.val[st][0][i] = 0.0;
  }
}

// per-node values src[r * ld + perm] of the batch in slot st (its perm has landed);
// padding nodes get 0.  Lane l copies nodes l, l + 32, ... of the batch.
template <int U, int D, int RG>
__device__ __forceinline__ void tc_stage_vals(TcRing<U, D, RG>& R, int st, const double* src,
                                              int64_t ld, int nr, int lane) {
#pragma unroll
  for (int i = lane; i < 8 * U; i += 32) {
    const int j = R.perm[st][i];
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      if (j >= 0 && r < nr) cp_async8(&R.val[st][r][i], src + r * ld + j);
      else R.val[st][r][i] = 0.0;
    }
  }
}

// ----------------------------------------------------------------------------
// gather: out[perm] += eta * interp over groups [g0, g1) of one warp, U at a time.
//
// The x-dimension window matrix is folded into the grid once per half-cell:
//     s_node = sum_p (P_x Ghat)[node][p] Phi_y[node][p],   Ghat[k][p] = sum_o C[o][k] G[o][p]
// (P_x the node powers, C the polynomial table), so a group costs 3 DMMAs for P_x Ghat and 3 for
// Phi_y instead of 3 + 3 + 2, and Ghat (4 DMMAs, computed as Ghat^T = G^T C so its accumulator
// is directly the B operand) is paid once per header change (~19 groups at C3).  Ghat^T's
// fragment gives lane (p, q) the terms k = 2q + {0, 1} and, of the upper block, 8 + 2q + {0, 1}
// for q < 2: one xor-2 shuffle hands lanes q >= 2 the odd ones, so the third k-step runs over
// k = 8 + 2 (q & 1) + (q >> 1) and the node powers follow that order (tc_powers_ghat).
// ----------------------------------------------------------------------------
// lane's Ghat coefficient fragment: B[kk = q][n = slot] = C[o = 2q + t][k = slot + 8b]
template <int TAB>
__device__ __forceinline__ void tc_coefs_ghat(int lane, double (&cg)[2][2]) {
  constexpr int NT = TcPoly<TAB>::NT;
  static_assert(NT > 8 && NT <= 12, "three k-steps of the folded gather");
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int k = (lane >> 2) + 8 * b, o = 2 * (lane & 3) + t;
      const double c = k < NT ? kb_coef<TAB, 4>(o, k) : 0.0;
      asm volatile("mov.b64 %0, %1;" : "=d"(cg[b][t]) : "d"(c));
    }
}

// powers in the folded gather's k order: x^(2q), x^(2q+1), x^(8 + 2 (q & 1) + (q >> 1))
__device__ __forceinline__ void tc_powers_ghat(double x, bool q1, bool q2, double (&pw)[3]) {
  const double x2 = x * x;
  const double x4 = x2 * x2;
  const double x8 = x4 * x4;
  const double s1 = q1 ? x2 : 1.0;
  pw[0] = s1 * (q2 ? x4 : 1.0);
  pw[1] = pw[0] * x;
  pw[2] = x8 * s1 * (q2 ? x : 1.0);
}

// Ghat fragments of one half-cell from the lane's grid values ga = G[2q][slot], gc = G[2q+1][slot]
__device__ __forceinline__ void tc_ghat(double ga, double gc, const double (&cg)[2][2], bool q2,
                                        double (&gh)[3]) {
  double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0};
  dmma884(d0, ga, cg[0][0]);
  dmma884(d0, gc, cg[0][1]);
  dmma884(d1, ga, cg[1][0]);
  dmma884(d1, gc, cg[1][1]);
  const double odd = __shfl_xor_sync(0xffffffffu, d1[1], 2);
  gh[0] = d0[0];
  gh[1] = d0[1];
  gh[2] = q2 ? odd : d1[0];
}

template <int RG, int TAB, int U, bool POW2, int D>
__global__ void __launch_bounds__(128, RG == 1 ? AFS_TC_MINB_GATHER : 1) k_gather_tc(const SortedSide sv, const Window w, int n,
                                                   const double* __restrict__ grid,
                                                   int64_t rhs_stride, int nr,
                                                   double* __restrict__ out, int64_t ldo,
                                                   int gpw) {
  static_assert(D >= 4, "values are staged two batches ahead of node data landing");
  constexpr int NKS = TcPoly<TAB>::NKS;
  static_assert(NKS == 3, "three k-steps per window matrix");
  __shared__ TcRing<U, D, RG> ring[4];
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  const bool q1 = q & 1, q2 = q >= 2;
  TcRing<U, D, RG>& R = ring[threadIdx.x >> 5];
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g0 = warp * gpw;
  if (g0 >= sv.ngroups) return;   // warp-uniform
  // gpw is a multiple of U and the layout carries >= D*U trailing empty groups, so the last
  // warp may run (and prefetch) past ngroups without clamping
  const int g1 = min(g0 + gpw, (int)sv.ngroups);
  double cf[NKS], cg[2][2];
  tc_coefs<TAB>(lane, cf);
  tc_coefs_ghat<TAB>(lane, cg);
  const double* g = grid + w.grid_off;

  // raw grid operands of one batch, ga = G[cell(o = 2q)][cell(p = slot)], gc = o = 2q + 1,
  // loaded one batch ahead for the groups whose header differs from the previous group's
  // (bit u of chg; a half-cell spans ~N/(4 n^2) nodes, 19 groups on average at C3)
  struct Win {
    double ga[U][RG], gc[U][RG];
  };
  int32_t hlast = -1;
  auto load_win = [&](int st, Win& d, unsigned& chg) {
    chg = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t h = R.hdr[st][u];
      if (h != hlast) {   // warp-uniform
        const int col = tc_cell<POW2>(tc_u1(h), tc_c1(h), slot, n);
        const int ra = tc_cell<POW2>(tc_u0(h), tc_c0(h), 2 * q, n) * n + col;
        const int rb = tc_cell<POW2>(tc_u0(h), tc_c0(h), 2 * q + 1, n) * n + col;
#pragma unroll
        for (int r = 0; r < RG; ++r) {
          const double* gr = g + (r < nr ? r : 0) * rhs_stride;
          d.ga[u][r] = __ldg(gr + ra);
          d.gc[u][r] = __ldg(gr + rb);
        }
        hlast = h;
        chg |= 1u << u;
      }
    }
  };

#pragma unroll
  for (int k = 0; k < D; ++k) {
    tc_stage_nodes(R, k, sv, g0 + k * U, lane);
    cp_async_commit();
  }
  cp_async_wait<D - 2>();
  __syncwarp();
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  Win wnext;
  unsigned chg_next;
  load_win(0, wnext, chg_next);   // hlast = -1: the first group loads
  double ghp[RG][3] = {};         // Ghat of the previous group
  int st = 0;
#pragma unroll 1
  for (int gb = g0; gb < g1; gb += U) {
    cp_async_wait<1>();   // node data up to batch b + 2 and values of batch b have landed
    __syncwarp();
    static_assert(U == 4, "the transposed quad reduction hands lane q the sums of group ug");
    // after the reduction lane (slot, q) owns node slot of group ug = 2 (q & 1) + (q >> 1)
    const int ug = 2 * (q & 1) + (q >> 1);
    double x0[U], x1[U], prior[RG];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x0[u] = R.x0[st][u * 8 + slot];
      x1[u] = R.x1[st][u * 8 + slot];
    }
    const int j = R.perm[st][ug * 8 + slot];
#pragma unroll
    for (int r = 0; r < RG; ++r) prior[r] = 0.0;   // the result is added with one RED per node
    const Win wcur = wnext;
    const unsigned chg = chg_next;
    const int st1 = st + 1 == D ? 0 : st + 1;
    const int st2 = st1 + 1 == D ? 0 : st1 + 1;
    __syncwarp();
    tc_stage_nodes(R, st, sv, gb + D * U, lane);   // refill the slot just read
    cp_async_commit();
    load_win(st1, wnext, chg_next);                  // grid window of batch b + 1
    // per group: Ghat (recomputed where the header changed), the y window values
    // Phi_y[node][o], o = 2q, 2q+1, and the lane partials P_x Ghat . Phi_y
    double sp[RG][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (chg & (1u << u))   // warp-uniform
#pragma unroll
        for (int r = 0; r < RG; ++r) tc_ghat(wcur.ga[u][r], wcur.gc[u][r], cg, q2, ghp[r]);
      double py[NKS], px[3], fy[2] = {0.0, 0.0};
      tc_powers<NKS>(x1[u], q1, q2, py);
      tc_powers_ghat(x0[u], q1, q2, px);
#pragma unroll
      for (int s = 0; s < NKS; ++s) dmma884(fy, py[s], cf[s]);
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        double t[2] = {0.0, 0.0};
#pragma unroll
        for (int s = 0; s < 3; ++s) dmma884(t, px[s], ghp[r][s]);
        sp[r][u] = fma(t[1], fy[1], t[0] * fy[0]);
      }
    }
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      // transposed reduction of the 4 groups' partials over the quad: 3 shuffles instead
      // of 8, and every lane finishes one node
      const bool b0 = q & 1, b1 = (q >> 1) & 1;
      // xor 1: keep groups {2 b0, 2 b0 + 1}
      const double k0 = b0 ? sp[r][2] : sp[r][0], k1 = b0 ? sp[r][3] : sp[r][1];
      const double g0 = b0 ? sp[r][0] : sp[r][2], g1 = b0 ? sp[r][1] : sp[r][3];
      const double v0 = k0 + __shfl_xor_sync(0xffffffffu, g0, 1);
      const double v1 = k1 + __shfl_xor_sync(0xffffffffu, g1, 1);
      // xor 2: keep group 2 b0 + b1
      const double sum = (b1 ? v1 : v0) + __shfl_xor_sync(0xffffffffu, b1 ? v0 : v1, 2);
      if (j >= 0 && r < nr) red_hint(out + r * ldo + j, __dmul_rn(w.eta, sum), l2_policy_evict_last());
    }
    st = st1;
  }
  cp_async_wait<0>();
}

// ----------------------------------------------------------------------------
// gather, one right-hand side, Chebyshev-folded (k_gather_cheb).
//
// Per half-cell the 8x8 grid window G (stencil offsets in polynomial order, reflection
// folded into the addressing) and both dimensions' window polynomials fold into ONE
// bivariate Chebyshev series
//     s(x, y) = sum_{a,b} G[a][b] P_a(x) P_b(y) = sum_{k,l} Ghat[k][l] T_k(4x) T_l(4y),
//     Ghat = Cc^T G Cc    (Cc: kb_cheb.inc, the same 12-term interpolants as kb_tables.inc)
// whose coefficients decay like the product of the 1-D ones, so the terms with k + l > 14
// are below 1e-16 of the window scale and are dropped: 104 coefficients instead of 144
// (packed rows of 12,12,12,12,10,10,8,8,6,6,4,4).  A node then costs 136 DFMAs (two
// 11-step Chebyshev recurrences + 104 coefficient FMAs + 12) against the 1536 DMMA MACs +
// power products per 8 nodes of k_gather_tc; the fold is 10 DMMAs per half-cell and warp.
// Lane = node (32 nodes = 4 groups per batch); the coefficients are broadcast from a
// per-warp shared-memory table ring.  Measured (C3, 2-D window): 0.207 ms vs 0.222 ms for
// k_gather_tc; the coefficient broadcasts bind it (ncu: l1tex 86%, fp64 pipe 42%).  Two
// nodes per lane (every broadcast feeding 4 FMAs) measured slower (0.214 ms: LDS latency
// at the lower occupancy its registers allow).
// ----------------------------------------------------------------------------
constexpr int kChebTab = 104;          // packed coefficients per half-cell
constexpr int kChebSlots = 5;          // tables per warp: 4 new per batch + the live one

__host__ __device__ constexpr int cheb_rowlen(int k) { return k < 4 ? 12 : 12 - 2 * ((k - 2) / 2); }
__host__ __device__ constexpr int cheb_off(int k) {
  int o = 0;
  for (int j = 0; j < k; ++j) o += cheb_rowlen(j);
  return o;
}

template <int TAB, bool POW2, int D>
__global__ void __launch_bounds__(128, AFS_TC_MINB_CHEB) k_gather_cheb(
    const SortedSide sv, const Window w, int n, const double* __restrict__ grid,
    double* __restrict__ out, int gpw) {
  constexpr int U = 4;
  static_assert(D >= 4, "values are staged two batches ahead of node data landing");
  __shared__ TcRing<U, D, 1> ring[4];
  __shared__ __align__(16) double tabs[4][kChebSlots][kChebTab];
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  const int wib = threadIdx.x >> 5;
  TcRing<U, D, 1>& R = ring[wib];
  double* tab = &tabs[wib][0][0];
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g0 = warp * gpw;
  if (g0 >= sv.ngroups) return;   // warp-uniform
  const int g1 = min(g0 + gpw, (int)sv.ngroups);
  const double* g = grid + w.grid_off;

  // fold constants.  Step 1 (H^T = Cc^T G^T): A[l = slot + 8 mb][b = q + 4 s] = Cc[b][l];
  // step 2 (Ghat^T = H^T Cc, k relabelled a = 2q + e): B[a = 2q + e][k = slot + 8 nb] = Cc[a][k]
  double ca[2][2], cb[2][2];
#pragma unroll
  for (int mb = 0; mb < 2; ++mb)
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const int l = slot + 8 * mb, b = q + 4 * s2;
      const double c = l < 12 ? kb_cheb<TAB>(b, l) : 0.0;
      asm volatile("mov.b64 %0, %1;" : "=d"(ca[mb][s2]) : "d"(c));
      const int k = slot + 8 * mb, a = 2 * q + s2;
      const double c2 = k < 12 ? kb_cheb<TAB>(a, k) : 0.0;
      asm volatile("mov.b64 %0, %1;" : "=d"(cb[mb][s2]) : "d"(c2));
    }
  // packed store index of the lane's fold outputs: block (mb, nb) in {(0,0), (0,1), (1,0)},
  // element e: Ghat^T[l = slot + 8 mb][k = 2q + e + 8 nb]; -1 when not kept
  int sidx[3][2];
#pragma unroll
  for (int bi = 0; bi < 3; ++bi)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int mb = bi == 2 ? 1 : 0, nb = bi == 1 ? 1 : 0;
      const int l = slot + 8 * mb, k = 2 * q + e + 8 * nb;
      sidx[bi][e] = (k < 12 && l < cheb_rowlen(k)) ? cheb_off(k) + l : -1;
    }

  // fold inputs of one batch, loaded one batch ahead for the groups whose header changes:
  // gw[u][s] = G[a = slot][b = q + 4 s] of group u's half-cell
  int32_t hlast = -1;
  auto load_fold = [&](int st, double (&gw)[U][2], unsigned& chg) {
    chg = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t h = R.hdr[st][u];
      if (h != hlast) {   // warp-uniform
        const int row = tc_cell<POW2>(tc_u0(h), tc_c0(h), slot, n) * n;
        gw[u][0] = __ldg(g + row + tc_cell<POW2>(tc_u1(h), tc_c1(h), q, n));
        gw[u][1] = __ldg(g + row + tc_cell<POW2>(tc_u1(h), tc_c1(h), q + 4, n));
        hlast = h;
        chg |= 1u << u;
      }
    }
  };
  auto fold = [&](const double (&gv)[2], double* dst) {
    double ht[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int mb = 0; mb < 2; ++mb) {
      dmma884(ht[mb], ca[mb][0], gv[0]);
      dmma884(ht[mb], ca[mb][1], gv[1]);
    }
    double gt[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      dmma884(gt[0], ht[0][e], cb[0][e]);
      dmma884(gt[1], ht[0][e], cb[1][e]);
      dmma884(gt[2], ht[1][e], cb[0][e]);
    }
#pragma unroll
    for (int bi = 0; bi < 3; ++bi)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (sidx[bi][e] >= 0) dst[sidx[bi][e]] = gt[bi][e];
  };

#pragma unroll
  for (int k = 0; k < D; ++k) {
    tc_stage_nodes(R, k, sv, g0 + k * U, lane);
    cp_async_commit();
  }
  cp_async_wait<D - 2>();
  __syncwarp();
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  double gnext[U][2];
  unsigned chg_next;
  load_fold(0, gnext, chg_next);   // hlast = -1: the first group loads
  int live = 0;                     // table slot of the previous batch's last group
  int st = 0;
  const int ug = lane >> 3;
#pragma unroll 1
  for (int gb = g0; gb < g1; gb += U) {
    cp_async_wait<1>();   // node data up to batch b + 2 and values of batch b have landed
    __syncwarp();         // (also: every lane is done reading the previous batch's tables)
    const double u4 = 4.0 * R.x0[st][lane];
    const double v4 = 4.0 * R.x1[st][lane];
    const int j = R.perm[st][lane];
    double gcur[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) gcur[u][0] = gnext[u][0], gcur[u][1] = gnext[u][1];
    const unsigned chg = chg_next;
    const int st1 = st + 1 == D ? 0 : st + 1;
    const int st2 = st1 + 1 == D ? 0 : st1 + 1;
    __syncwarp();
    tc_stage_nodes(R, st, sv, gb + D * U, lane);   // refill the slot just read
    cp_async_commit();
    load_fold(st1, gnext, chg_next);                // fold inputs of batch b + 1
    // tables of this batch's new half-cells go to the slots other than the live one
    int ts[U];
    int cur = live, nnew = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (chg & (1u << u)) {   // warp-uniform
        cur = nnew < live ? nnew : nnew + 1;
        ++nnew;
        fold(gcur[u], tab + cur * kChebTab);
      }
      ts[u] = cur;
    }
    live = cur;
    __syncwarp();
    const double* T = tab + (ug == 0 ? ts[0] : ug == 1 ? ts[1] : ug == 2 ? ts[2] : ts[3]) * kChebTab;
    // Chebyshev values of y, then the rows k of the table against them, outer recurrence in x
    double ty[12];
    ty[0] = 1.0;
    ty[1] = v4;
    const double v8 = 2.0 * v4;
#pragma unroll
    for (int l = 2; l < 12; ++l) ty[l] = fma(v8, ty[l - 1], -ty[l - 2]);
    const double u8 = 2.0 * u4;
    double tkm1 = 1.0, tk = 1.0, s = 0.0;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      if (k == 1) {
        tkm1 = 1.0;
        tk = u4;
      } else if (k >= 2) {
        const double tn = fma(u8, tk, -tkm1);
        tkm1 = tk;
        tk = tn;
      }
      const double* row = T + cheb_off(k);
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int l = 0; l < cheb_rowlen(k); l += 2) {
        const double2 c = *reinterpret_cast<const double2*>(row + l);
        p0 = fma(c.x, ty[l], p0);
        p1 = fma(c.y, ty[l + 1], p1);
      }
      s = fma(tk, p0 + p1, s);
    }
    // one RED per node and launch (RN add in L2): the bits of load + add + store, without the
    // random load's round trip
    if (j >= 0) red_hint(out + j, __dmul_rn(w.eta, s), l2_policy_evict_last());
    st = st1;
  }
  cp_async_wait<0>();
}

// ----------------------------------------------------------------------------
// spread: grid += sum_node alpha_node Phi_x (x) Phi_y, accumulated per half-cell in the
// MMA accumulators (one per group of the batch, summed at the flush) and flushed
// (RED.F64 / fixed-point limbs) when the group header changes
// ----------------------------------------------------------------------------
template <int RG, int TAB, int U, bool POW2, int D>
__global__ void __launch_bounds__(128, RG == 1 ? AFS_TC_MINB_SPREAD : 1) k_spread_tc(const SortedSide sv, const Window w, int n,
                                                   const double* __restrict__ alpha, int64_t lda,
                                                   int nr, double* __restrict__ grid,
                                                   int64_t rhs_stride, int gpw) {
  static_assert(D >= 4, "values are staged two batches ahead of node data landing");
  constexpr int NKS = TcPoly<TAB>::NKS;
  __shared__ TcRing<U, D, RG> ring[4];
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  const bool q1 = q & 1, q2 = q >= 2;
  TcRing<U, D, RG>& R = ring[threadIdx.x >> 5];
  __shared__ TcPow<4> pwt[4];   // x^2, x^4, y^2, y^4
  TcPow<4>& PW = pwt[threadIdx.x >> 5];
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g0 = warp * gpw;
  if (g0 >= sv.ngroups) return;   // warp-uniform
  const int g1 = min(g0 + gpw, (int)sv.ngroups);
  double cf[NKS];
  tc_coefs<TAB>(lane, cf);
  double* g = grid + w.grid_off;

  double acc[U][RG][2];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int r = 0; r < RG; ++r) acc[u][r][0] = acc[u][r][1] = 0.0;
  int32_t cur_h = -1;
  // lane holds acc[o = slot][p = 2q + e]
  auto flush = [&]() {
    const int row = tc_cell<POW2>(tc_u0(cur_h), tc_c0(cur_h), slot, n) * n;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ix = row + tc_cell<POW2>(tc_u1(cur_h), tc_c1(cur_h), 2 * q + e, n);
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        double v = acc[0][r][e];
        acc[0][r][e] = 0.0;
#pragma unroll
        for (int u = 1; u < U; ++u) {
          v += acc[u][r][e];
          acc[u][r][e] = 0.0;
        }
        if (r < nr && v != 0.0) grid_add(w, g + r * rhs_stride + ix, v);
      }
    }
  };

#pragma unroll
  for (int k = 0; k < D; ++k) {
    tc_stage_nodes(R, k, sv, g0 + k * U, lane);
    cp_async_commit();
  }
  cp_async_wait<D - 2>();
  __syncwarp();
  tc_stage_vals(R, 0, alpha, lda, nr, lane);
  tc_stage_vals(R, 1, alpha, lda, nr, lane);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  int st = 0;
#pragma unroll 1
  for (int gb = g0; gb < g1; gb += U) {
    cp_async_wait<1>();
    __syncwarp();
    double x0[U], x1[U], al[U][RG][2];
    int32_t hd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x0[u] = R.x0[st][u * 8 + slot];
      x1[u] = R.x1[st][u * 8 + slot];
      hd[u] = R.hdr[st][u];
#pragma unroll
      for (int r = 0; r < RG; ++r) {   // alpha of the lane's k-nodes 2q, 2q+1
        const double2 a2 = *reinterpret_cast<const double2*>(&R.val[st][r][u * 8 + 2 * q]);
        al[u][r][0] = a2.x;
        al[u][r][1] = a2.y;
      }
    }
    {   // shared squares of the batch's 32 nodes (TcPow): node lane % 8 of group lane / 8
      const double xa = R.x0[st][lane], ya = R.x1[st][lane];
      const double xa2 = xa * xa, ya2 = ya * ya;
      PW.v[0][lane] = xa2;
      PW.v[1][lane] = xa2 * xa2;
      PW.v[2][lane] = ya2;
      PW.v[3][lane] = ya2 * ya2;
    }
    const int st1 = st + 1 == D ? 0 : st + 1;
    const int st2 = st1 + 1 == D ? 0 : st1 + 1;
    __syncwarp();
    tc_stage_nodes(R, st, sv, gb + D * U, lane);
    tc_stage_vals(R, st2, alpha, lda, nr, lane);
    cp_async_commit();
    // transposed window values: Phi[node][o] held as D[o = slot][node = 2q + t]
    double fx[U][2], fy[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double px[NKS], py[NKS];
      const int e = u * 8 + slot;
      tc_powers_x24<NKS>(x0[u], PW.v[0][e], PW.v[1][e], q1, q2, px);
      tc_powers_x24<NKS>(x1[u], PW.v[2][e], PW.v[3][e], q1, q2, py);
      fx[u][0] = fx[u][1] = fy[u][0] = fy[u][1] = 0.0;
#pragma unroll
      for (int s = 0; s < NKS; ++s) {
        dmma884(fx[u], cf[s], px[s]);
        dmma884(fy[u], cf[s], py[s]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (hd[u] != cur_h) {   // warp-uniform
        if (cur_h != -1) flush();
        cur_h = hd[u];
      }
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        dmma884(acc[u][r], fx[u][0] * al[u][r][0], fy[u][0]);
        dmma884(acc[u][r], fx[u][1] * al[u][r][1], fy[u][1]);
      }
    }
    st = st1;
  }
  cp_async_wait<0>();
  if (cur_h != -1) flush();
}

// ----------------------------------------------------------------------------
// spread, one right-hand side, Chebyshev moments (k_spread_cheb).
//
// With phi_a(x) = sum_k Cc[a][k] T_k(4x) (kb_cheb.inc), a half-cell's grid window is
//     G[a][b] = sum_{k,l} Cc[a][k] M[k][l] Cc[b][l],   M[k][l] = sum_node alpha T_k(4x) T_l(4y)
// so per group of 8 nodes the tensor cores accumulate the moment matrix M = (alpha T_x)^T T_y
// (12 x 12) instead of evaluating both window matrices and the touch (8 DMMAs in
// k_spread_tc).  The block k >= 8, l >= 8 of M (terms below 1e-19 of the window scale) is
// dropped: 6 DMMAs per group.  The Chebyshev vectors are computed once per node (lane =
// node) and staged transposed in shared memory for the fragments; the flush folds M back into
// the 8x8 window with 10 DMMAs per half-cell and warp and adds it to the grid as before.
// ----------------------------------------------------------------------------
constexpr int kChebStride = 36;   // staged row length (32 nodes + pad, = 4 mod 16: conflict-free)

template <int TAB, bool POW2, int D>
__global__ void __launch_bounds__(128, AFS_TC_MINB_CHEB_SPREAD) k_spread_cheb(
    const SortedSide sv, const Window w, int n, const double* __restrict__ alpha,
    double* __restrict__ grid, int gpw) {
  constexpr int U = 4;
  static_assert(D >= 4, "values are staged two batches ahead of node data landing");
  __shared__ TcRing<U, D, 1> ring[4];
  __shared__ __align__(16) double chx[4][12][kChebStride];   // alpha T_k(u) [k][node]
  __shared__ __align__(16) double chy[4][12][kChebStride];   // T_l(v) [l][node]
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  const int wib = threadIdx.x >> 5;
  TcRing<U, D, 1>& R = ring[wib];
  double(*CX)[kChebStride] = chx[wib];
  double(*CY)[kChebStride] = chy[wib];
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g0 = warp * gpw;
  if (g0 >= sv.ngroups) return;   // warp-uniform
  const int g1 = min(g0 + gpw, (int)sv.ngroups);
  double* g = grid + w.grid_off;
  // flush constants: ck[nb][e] = Cc[slot][2q + e + 8 nb] (step 1: A of N^T = Cc M^T;
  // step 2: B of G^T = N^T Cc^T, the same values)
  double ck[2][2];
#pragma unroll
  for (int nb = 0; nb < 2; ++nb)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = 2 * q + e + 8 * nb;
      const double c = k < 12 ? kb_cheb<TAB>(slot, k) : 0.0;
      asm volatile("mov.b64 %0, %1;" : "=d"(ck[nb][e]) : "d"(c));
    }

  // per-group moment accumulators, block bi in {(0,0), (0,1), (1,0)} of (k-block, l-block):
  // lane holds M[k = slot + 8 mb][l = 2q + e + 8 nb]
  double acc[U][3][2];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int bi = 0; bi < 3; ++bi) acc[u][bi][0] = acc[u][bi][1] = 0.0;
  int32_t cur_h = -1;
  auto flush = [&]() {
    double m[3][2];
#pragma unroll
    for (int bi = 0; bi < 3; ++bi)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = acc[0][bi][e];
        acc[0][bi][e] = 0.0;
#pragma unroll
        for (int u = 1; u < U; ++u) {
          v += acc[u][bi][e];
          acc[u][bi][e] = 0.0;
        }
        m[bi][e] = v;
      }
    // N^T[b = slot][k = 2q + e' + 8 mb'] = sum_l Cc[b][l] M[k][l], k-steps l = 2q + e + 8 nb
    double nt[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      dmma884(nt[0], ck[0][e], m[0][e]);   // k-block 0, l-block 0
      dmma884(nt[0], ck[1][e], m[1][e]);   // k-block 0, l-block 1
      dmma884(nt[1], ck[0][e], m[2][e]);   // k-block 1, l-block 0
    }
    // G^T[b = slot][a = 2q + e''] = sum_k N^T[b][k] Cc[a][k], k-steps k = 2q + e' + 8 mb'
    double gt[2] = {0.0, 0.0};
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int e = 0; e < 2; ++e) dmma884(gt, nt[mb][e], ck[mb][e]);
    const int col = tc_cell<POW2>(tc_u1(cur_h), tc_c1(cur_h), slot, n);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ix = tc_cell<POW2>(tc_u0(cur_h), tc_c0(cur_h), 2 * q + e, n) * n + col;
      if (gt[e] != 0.0) grid_add(w, g + ix, gt[e]);
    }
  };

#pragma unroll
  for (int k = 0; k < D; ++k) {
    tc_stage_nodes(R, k, sv, g0 + k * U, lane);
    cp_async_commit();
  }
  cp_async_wait<D - 2>();
  __syncwarp();
  tc_stage_vals(R, 0, alpha, 0, 1, lane);
  tc_stage_vals(R, 1, alpha, 0, 1, lane);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  int st = 0;
#pragma unroll 1
  for (int gb = g0; gb < g1; gb += U) {
    cp_async_wait<1>();
    __syncwarp();   // (also: every lane is done reading the previous batch's vectors)
    {   // this lane's node: alpha T_k(u) and T_l(v), k, l < 12, into the transposed tables
      const double u4 = 4.0 * R.x0[st][lane], v4 = 4.0 * R.x1[st][lane];
      const double a = R.val[st][0][lane];
      const double u8 = 2.0 * u4, v8 = 2.0 * v4;
      double tx0 = 1.0, tx1 = u4, ty0 = 1.0, ty1 = v4;
      CX[0][lane] = a;
      CY[0][lane] = 1.0;
      CX[1][lane] = a * u4;
      CY[1][lane] = v4;
#pragma unroll
      for (int k = 2; k < 12; ++k) {
        const double tx2 = fma(u8, tx1, -tx0), ty2 = fma(v8, ty1, -ty0);
        CX[k][lane] = a * tx2;
        CY[k][lane] = ty2;
        tx0 = tx1;
        tx1 = tx2;
        ty0 = ty1;
        ty1 = ty2;
      }
    }
    int32_t hd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) hd[u] = R.hdr[st][u];
    const int st1 = st + 1 == D ? 0 : st + 1;
    const int st2 = st1 + 1 == D ? 0 : st1 + 1;
    __syncwarp();
    tc_stage_nodes(R, st, sv, gb + D * U, lane);
    tc_stage_vals(R, st2, alpha, 0, 1, lane);
    cp_async_commit();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (hd[u] != cur_h) {   // warp-uniform
        if (cur_h != -1) flush();
        cur_h = hd[u];
      }
      // M += (alpha T_x)^T T_y over the group's nodes (k-steps: nodes q + 4 s)
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        const int nd = u * 8 + q + 4 * s2;
        const double a0 = CX[slot][nd], a1 = slot < 4 ? CX[slot + 8][nd] : 0.0;
        const double b0 = CY[slot][nd], b1 = slot < 4 ? CY[slot + 8][nd] : 0.0;
        dmma884(acc[u][0], a0, b0);
        dmma884(acc[u][1], a0, b1);
        dmma884(acc[u][2], a1, b0);
      }
    }
    st = st1;
  }
  cp_async_wait<0>();
  if (cur_h != -1) flush();
}

// host launchers (tc2d.cu); false when the window is not in the tensor-core layout
bool launch_spread_tc(const SortedSide& sv, const Window& w, int n, int tab, const double* alpha,
                      int64_t lda, int R, double* grid, int64_t rs, cudaStream_t s);
bool launch_gather_tc(const SortedSide& sv, const Window& w, int n, int tab, const double* grid,
                      int64_t rs, int R, double* out, int64_t ldo, cudaStream_t s);

}  // namespace afs
