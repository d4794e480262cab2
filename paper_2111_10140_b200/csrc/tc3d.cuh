// Spread / gather for dense 3-D windows at m = 4 on the fp64 tensor cores (DMMA).
//
// Layout (build_sorted_side_tc3): nodes sorted by 3-D half-cell and padded to groups of 8
// that share one 8x8x8 stencil; used only where that padding is cheap (dense data such as
// C4's clusters; sparse windows keep the team kernels of sliding.cuh).  Per group:
//   window values  Phi_t[node][o] = sum_k x_t^k C[o][k]          3 DMMAs per dimension
//   gather         H_p = Phi_x G[:, p, :]  (8 DMMA tiles over p, k = o)   16 DMMAs
//                  s = sum_p Phi_y[p] sum_r Phi_z[r] H_p[r]  (lane FMAs + quad reduction)
//   spread         G[:, :, r] += (alpha Phi_x)^T (Phi_y * Phi_z[:, r])   16 DMMAs
// i.e. 25 DMMAs = 6400 MACs per 8 nodes and right-hand side (the touch: 512 MACs per node,
// as the team kernels' FMAs), with the window values shared by the right-hand sides of a
// launch.  Reference: nfft.py:228-229 (gather), nfft.py:241-245 (spread).
#pragma once

#include "tc2d.cuh"

// __launch_bounds__ min blocks per SM of the 3-D tensor-core kernels (tuning hook)
#ifndef AFS_TC3_MINB
#define AFS_TC3_MINB 5
#endif

namespace afs {

__device__ __forceinline__ int tc3_u(uint64_t h, int t) { return (int)((h >> (16 * t)) & 0xffff); }
__device__ __forceinline__ int tc3_c(uint64_t h, int t) { return (int)((h >> (48 + t)) & 1); }

// one group per batch; DEPTH batches staged ahead with cp.async
template <int DEPTH, int RG>
struct TcRing3 {
  double x[3][DEPTH][8];
  double val[DEPTH][RG][8];
  int32_t perm[DEPTH][8];
  uint64_t hdr[DEPTH];
};

// node data of group g into slot st (16 B chunks: x0, x1, x2 four each, perm two, header 8 B)
template <int DEPTH, int RG>
__device__ __forceinline__ void tc3_stage_nodes(TcRing3<DEPTH, RG>& R, int st, const SortedSide& sv,
                                                int g, int lane, uint64_t pol) {
  const int i0 = g * 8;
  if (lane < 12) {
    const int t = lane >> 2, c = lane & 3;
    cp_async16_hint(&R.x[t][st][2 * c], sv.nx + t * sv.N + i0 + 2 * c, pol);
  } else if (lane < 14) {
    const int c = lane - 12;
    cp_async16_hint(&R.perm[st][4 * c], sv.perm + i0 + 4 * c, pol);
  } else if (lane == 14) {
    cp_async8(&R.hdr[st], sv.ghdr64 + g);
  }
}

// per-node values src[r * ld + perm] of the group in slot st (its perm has landed); 0 for padding
template <int DEPTH, int RG>
__device__ __forceinline__ void tc3_stage_vals(TcRing3<DEPTH, RG>& R, int st, const double* src,
                                               int64_t ld, int nr, int lane, uint64_t pol) {
  if (lane < 8) {
    const int j = R.perm[st][lane];
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      if (j >= 0 && r < nr) cp_async8_hint(&R.val[st][r][lane], src + r * ld + j, pol);
      else R.val[st][r][lane] = 0.0;
    }
  }
}

// ----------------------------------------------------------------------------
// gather: out[perm] += eta * interp over groups [g0, g1) of one warp
// ----------------------------------------------------------------------------
template <int RG, int TAB, bool POW2, int DEPTH>
__global__ void __launch_bounds__(128, RG == 1 ? AFS_TC3_MINB : 1) k_gather_tc3(const SortedSide sv, const Window w, int n,
                                                    const double* __restrict__ grid,
                                                    int64_t rhs_stride, int nr,
                                                    double* __restrict__ out, int64_t ldo, int gpw) {
  static_assert(DEPTH >= 4, "values are staged two groups ahead of node data landing");
  constexpr int NKS = TcPoly<TAB>::NKS;
  __shared__ TcRing3<DEPTH, RG> ring[4];
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  const bool q1 = q & 1, q2 = q >= 2;
  TcRing3<DEPTH, RG>& R = ring[threadIdx.x >> 5];
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g0 = warp * gpw;
  if (g0 >= sv.ngroups) return;   // warp-uniform
  const int g1 = min(g0 + gpw, (int)sv.ngroups);
  double cf[NKS];
  tc_coefs<TAB>(lane, cf);
  const double* g = grid + w.grid_off;
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();

  // stencil operands B[k][n] = G[cell_x(o = 2k + t)][cell_y(p)][cell_z(r = n)], one per tile p
  double gf[RG][2][8];
  uint64_t hcur = ~0ULL;
  auto load_stencil = [&](uint64_t h) {
    const int cz = tc_cell<POW2>(tc3_u(h, 2), tc3_c(h, 2), slot, n);
    int cx[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) cx[t] = tc_cell<POW2>(tc3_u(h, 0), tc3_c(h, 0), 2 * q + t, n);
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int cy = tc_cell<POW2>(tc3_u(h, 1), tc3_c(h, 1), p, n);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int idx = (cx[t] * n + cy) * n + cz;
#pragma unroll
        for (int r = 0; r < RG; ++r) gf[r][t][p] = r < nr ? __ldg(g + r * rhs_stride + idx) : 0.0;
      }
    }
  };

#pragma unroll
  for (int k = 0; k < DEPTH; ++k) {
    tc3_stage_nodes(R, k, sv, g0 + k, lane, pol_stream);
    cp_async_commit();
  }
  cp_async_wait<DEPTH - 2>();
  __syncwarp();
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  int st = 0;
#pragma unroll 1
  for (int gi = g0; gi < g1; ++gi) {
    cp_async_wait<1>();   // node data up to group gi + 2 and values of group gi have landed
    __syncwarp();
    const double x0 = R.x[0][st][slot], x1 = R.x[1][st][slot], x2 = R.x[2][st][slot];
    const int j = R.perm[st][slot];
    const uint64_t h = R.hdr[st];
    const int st1 = st + 1 == DEPTH ? 0 : st + 1;
    const int st2 = st1 + 1 == DEPTH ? 0 : st1 + 1;
    __syncwarp();
    tc3_stage_nodes(R, st, sv, gi + DEPTH, lane, pol_stream);
    cp_async_commit();
    if (h != hcur) {   // warp-uniform; dense segments span many groups
      load_stencil(h);
      hcur = h;
    }
    // window values Phi_t[node][o], o = 2q, 2q+1
    double fx[2] = {0.0, 0.0}, fy[2] = {0.0, 0.0}, fz[2] = {0.0, 0.0};
    {
      double p0[NKS], p1[NKS], p2[NKS];
      tc_powers<NKS>(x0, q1, q2, p0);
      tc_powers<NKS>(x1, q1, q2, p1);
      tc_powers<NKS>(x2, q1, q2, p2);
#pragma unroll
      for (int s = 0; s < NKS; ++s) {
        dmma884(fx, p0[s], cf[s]);
        dmma884(fy, p1[s], cf[s]);
        dmma884(fz, p2[s], cf[s]);
      }
    }
    const bool b0 = q & 1, b1 = q >> 1;
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      // v_p = sum_r' Phi_z[r'] H_p[r'] over the lane's r' = 2q, 2q+1
      double v[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        double hp[2] = {0.0, 0.0};
        dmma884(hp, fx[0], gf[r][0][p]);
        dmma884(hp, fx[1], gf[r][1][p]);
        v[p] = fma(hp[1], fz[1], hp[0] * fz[0]);
      }
      // transposed reduction over the quad: lane q ends with the full v_{2q}, v_{2q+1}
      double a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double keep = b1 ? v[4 + i] : v[i], send = b1 ? v[i] : v[4 + i];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
      double c[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double keep = b0 ? a[2 + k] : a[k], send = b0 ? a[k] : a[2 + k];
        c[k] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
      double s = fma(fy[1], c[1], fy[0] * c[0]);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      // one reduction per node and launch (RN add in L2): the bits of load + add + store
      // without the random load's round trip
      if (q == 0 && j >= 0 && r < nr) red_hint(out + r * ldo + j, __dmul_rn(w.eta, s), pol_keep);
    }
    st = st1;
  }
  cp_async_wait<0>();
}

// ----------------------------------------------------------------------------
// spread: grid += sum_node alpha Phi_x (x) Phi_y (x) Phi_z, accumulated per half-cell in the
// MMA accumulators (8 z-tiles of D[o][p]) and flushed when the group header changes
// ----------------------------------------------------------------------------
template <int RG, int TAB, bool POW2, int DEPTH>
__global__ void __launch_bounds__(128, RG == 1 ? AFS_TC3_MINB : 1) k_spread_tc3(const SortedSide sv, const Window w, int n,
                                                    const double* __restrict__ alpha, int64_t lda,
                                                    int nr, double* __restrict__ grid,
                                                    int64_t rhs_stride, int gpw) {
  static_assert(DEPTH >= 4, "values are staged two groups ahead of node data landing");
  constexpr int NKS = TcPoly<TAB>::NKS;
  __shared__ TcRing3<DEPTH, RG> ring[4];
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  const bool q1 = q & 1, q2 = q >= 2;
  TcRing3<DEPTH, RG>& R = ring[threadIdx.x >> 5];
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g0 = warp * gpw;
  if (g0 >= sv.ngroups) return;   // warp-uniform
  const int g1 = min(g0 + gpw, (int)sv.ngroups);
  double cf[NKS];
  tc_coefs<TAB>(lane, cf);
  double* g = grid + w.grid_off;
  const uint64_t pol_stream = l2_policy_evict_first(), pol_keep = l2_policy_evict_last();

  double acc[RG][8][2];   // z-tile rr: lane holds G[o = slot][p = 2q + e][r = rr]
#pragma unroll
  for (int r = 0; r < RG; ++r)
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) acc[r][rr][0] = acc[r][rr][1] = 0.0;
  uint64_t hcur = ~0ULL;
  auto flush = [&]() {
    const int cx = tc_cell<POW2>(tc3_u(hcur, 0), tc3_c(hcur, 0), slot, n);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int cy = tc_cell<POW2>(tc3_u(hcur, 1), tc3_c(hcur, 1), 2 * q + e, n);
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        const int idx = (cx * n + cy) * n + tc_cell<POW2>(tc3_u(hcur, 2), tc3_c(hcur, 2), rr, n);
#pragma unroll
        for (int r = 0; r < RG; ++r) {
          if (r < nr && acc[r][rr][e] != 0.0) grid_add(w, g + r * rhs_stride + idx, acc[r][rr][e]);
          acc[r][rr][e] = 0.0;
        }
      }
    }
  };

#pragma unroll
  for (int k = 0; k < DEPTH; ++k) {
    tc3_stage_nodes(R, k, sv, g0 + k, lane, pol_stream);
    cp_async_commit();
  }
  cp_async_wait<DEPTH - 2>();
  __syncwarp();
  tc3_stage_vals(R, 0, alpha, lda, nr, lane, pol_keep);
  tc3_stage_vals(R, 1, alpha, lda, nr, lane, pol_keep);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  int st = 0;
#pragma unroll 1
  for (int gi = g0; gi < g1; ++gi) {
    cp_async_wait<1>();
    __syncwarp();
    const double x0 = R.x[0][st][slot], x1 = R.x[1][st][slot], x2 = R.x[2][st][slot];
    const uint64_t h = R.hdr[st];
    double al[RG][2];   // alpha of the lane's k-nodes 2q, 2q+1
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const double2 a2 = *reinterpret_cast<const double2*>(&R.val[st][r][2 * q]);
      al[r][0] = a2.x;
      al[r][1] = a2.y;
    }
    const int st1 = st + 1 == DEPTH ? 0 : st + 1;
    const int st2 = st1 + 1 == DEPTH ? 0 : st1 + 1;
    __syncwarp();
    tc3_stage_nodes(R, st, sv, gi + DEPTH, lane, pol_stream);
    tc3_stage_vals(R, st2, alpha, lda, nr, lane, pol_keep);
    cp_async_commit();
    if (h != hcur) {   // warp-uniform
      if (hcur != ~0ULL) flush();
      hcur = h;
    }
    // transposed window values: Phi_t[node][o] held as D[o = slot][node = 2q + t]
    double fx[2] = {0.0, 0.0}, fy[2] = {0.0, 0.0}, fz[2] = {0.0, 0.0};
    {
      double p0[NKS], p1[NKS], p2[NKS];
      tc_powers<NKS>(x0, q1, q2, p0);
      tc_powers<NKS>(x1, q1, q2, p1);
      tc_powers<NKS>(x2, q1, q2, p2);
#pragma unroll
      for (int s = 0; s < NKS; ++s) {
        dmma884(fx, cf[s], p0[s]);
        dmma884(fy, cf[s], p1[s]);
        dmma884(fz, cf[s], p2[s]);
      }
    }
    // B_t[rr] = Phi_y[node 2q+t][p = slot] * Phi_z[node 2q+t][rr]; Phi_z of the lane's k-nodes
    // lives in lanes (rr, q)
    double b[2][8];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) b[t][rr] = fy[t] * __shfl_sync(0xffffffffu, fz[t], 4 * rr + q);
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const double a0 = fx[0] * al[r][0], a1 = fx[1] * al[r][1];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        dmma884(acc[r][rr], a0, b[0][rr]);
        dmma884(acc[r][rr], a1, b[1][rr]);
      }
    }
    st = st1;
  }
  cp_async_wait<0>();
  if (hcur != ~0ULL) flush();
}

bool launch_spread_tc3(const SortedSide& sv, const Window& w, int n, int tab, const double* alpha,
                       int64_t lda, int R, double* grid, int64_t rs, cudaStream_t s);
bool launch_gather_tc3(const SortedSide& sv, const Window& w, int n, int tab, const double* grid,
                       int64_t rs, int R, double* out, int64_t ldo, cudaStream_t s);

}  // namespace afs
