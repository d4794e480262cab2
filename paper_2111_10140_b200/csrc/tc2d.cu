// Launchers for the fp64 tensor-core 2-D kernels (tc2d.cuh).
#include <cstdlib>

#include "sc2d.cuh"

namespace afs {

namespace {

// resident warps per SM of a kernel (one wave), or the AFS_TC_WARPS tuning override
template <typename K>
int tc_warps_per_sm(K kernel) {
  if (const char* e = getenv("AFS_TC_WARPS")) return std::max(1, atoi(e));
  int occ = 0;
  AFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 128, 0));
  return std::max(1, occ) * 4;
}

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    AFS_CUDA(cudaGetDevice(&dev));
    AFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

#ifndef AFS_TC_U
#define AFS_TC_U 4
#endif
constexpr int kU = AFS_TC_U;   // groups per batch
constexpr int kD = 4;   // batches staged ahead (shared-memory ring)
static_assert(kD * kU <= kTcTailGroups, "the layout's empty tail must cover the staged batches");

// groups per warp: one wave of resident warps, a multiple of kU
int groups_per_warp(int64_t ngroups, int warps_per_sm) {
  const int64_t warps = (int64_t)num_sms() * warps_per_sm;
  const int64_t g = std::max<int64_t>(4, (ngroups + warps - 1) / warps);
  return (int)((g + kU - 1) / kU * kU);
}

bool pow2(int n) { return (n & (n - 1)) == 0; }

// The Chebyshev kernels fold a whole half-cell once per warp (10 DMMAs); they pay when a
// half-cell holds several groups (C3: ~19 groups per half-cell, gather -7%, spread -7%) and
// lose at low density (C5 pairs at N = 1M, ~2.4 groups: spread +17%).  AFS_CHEB=0/1 forces
// the gather choice, AFS_CHEB_SPREAD=0/1 the spread's (A/B hooks); default: by density.
constexpr double kChebMinGroupsPerHalfCell = 8.0;

int env_switch(const char* name) {   // -1 unset, else 0/1
  const char* e = getenv(name);
  return e ? (e[0] == '0' ? 0 : 1) : -1;
}

bool dense_enough(const SortedSide& sv, int n) {
  return (double)sv.ngroups >= kChebMinGroupsPerHalfCell * 4.0 * (double)n * (double)n;
}


template <int TAB>
void spread_cheb(const SortedSide& sv, const Window& w, int n, const double* alpha, double* grid,
                 cudaStream_t s) {
  const int64_t ng = sv.ngroups;
  auto launch = [&](auto kernel) {
    static int wps = 0;
    if (wps == 0) wps = tc_warps_per_sm(kernel);
    const int gpw = groups_per_warp(ng, wps);
    const int64_t warps = (ng + gpw - 1) / gpw;
    const int64_t blocks = (warps * 32 + 127) / 128;
    kernel<<<(unsigned)blocks, 128, 0, s>>>(sv, w, n, alpha, grid, gpw);
  };
  if (pow2(n))
    launch(k_spread_cheb<TAB, true, kD>);
  else
    launch(k_spread_cheb<TAB, false, kD>);
}

bool cheb_spread_enabled(const SortedSide& sv, int n) {
  static const int force = env_switch("AFS_CHEB_SPREAD");
  return force >= 0 ? force == 1 : dense_enough(sv, n);
}

template <int RG, int TAB>
void spread_tc(const SortedSide& sv, const Window& w, int n, const double* alpha, int64_t lda,
               int nr, double* grid, int64_t rs, cudaStream_t s) {
  if (RG == 1 && nr == 1 && cheb_spread_enabled(sv, n)) return spread_cheb<TAB>(sv, w, n, alpha, grid, s);
  const int64_t ng = sv.ngroups;
  auto launch = [&](auto kernel) {
    static int wps = 0;
    if (wps == 0) wps = tc_warps_per_sm(kernel);
    const int gpw = groups_per_warp(ng, wps);
    const int64_t warps = (ng + gpw - 1) / gpw;
    const int64_t blocks = (warps * 32 + 127) / 128;
    kernel<<<(unsigned)blocks, 128, 0, s>>>(sv, w, n, alpha, lda, nr, grid, rs, gpw);
  };
  if (pow2(n))
    launch(k_spread_tc<RG, TAB, kU, true, kD>);
  else
    launch(k_spread_tc<RG, TAB, kU, false, kD>);
}

bool cheb_enabled(const SortedSide& sv, int n) {
  static const int force = env_switch("AFS_CHEB");
  return force >= 0 ? force == 1 : dense_enough(sv, n);
}

template <int TAB>
void gather_cheb(const SortedSide& sv, const Window& w, int n, const double* grid, double* out,
                 cudaStream_t s) {
  const int64_t ng = sv.ngroups;
  auto launch = [&](auto kernel) {
    static int wps = 0;
    if (wps == 0) wps = tc_warps_per_sm(kernel);
    const int gpw = groups_per_warp(ng, wps);
    const int64_t warps = (ng + gpw - 1) / gpw;
    const int64_t blocks = (warps * 32 + 127) / 128;
    kernel<<<(unsigned)blocks, 128, 0, s>>>(sv, w, n, grid, out, gpw);
  };
  if (pow2(n))
    launch(k_gather_cheb<TAB, true, kD>);
  else
    launch(k_gather_cheb<TAB, false, kD>);
}

template <int RG, int TAB>
void gather_tc(const SortedSide& sv, const Window& w, int n, const double* grid, int64_t rs, int nr,
               double* out, int64_t ldo, cudaStream_t s) {
  if (RG == 1 && nr == 1 && cheb_enabled(sv, n)) return gather_cheb<TAB>(sv, w, n, grid, out, s);
  const int64_t ng = sv.ngroups;
  auto launch = [&](auto kernel) {
    static int wps = 0;
    if (wps == 0) wps = tc_warps_per_sm(kernel);
    const int gpw = groups_per_warp(ng, wps);
    const int64_t warps = (ng + gpw - 1) / gpw;
    const int64_t blocks = (warps * 32 + 127) / 128;
    kernel<<<(unsigned)blocks, 128, 0, s>>>(sv, w, n, grid, rs, nr, out, ldo, gpw);
  };
  if (pow2(n))
    launch(k_gather_tc<RG, TAB, kU, true, kD>);
  else
    launch(k_gather_tc<RG, TAB, kU, false, kD>);
}

template <int TAB>
void spread_tab(const SortedSide& sv, const Window& w, int n, const double* alpha, int64_t lda,
                int R, double* grid, int64_t rs, cudaStream_t s) {
  for (int r0 = 0; r0 < R; r0 += 2) {
    const int nr = std::min(2, R - r0);
    if (nr == 2)
      spread_tc<2, TAB>(sv, w, n, alpha + r0 * lda, lda, nr, grid + r0 * rs, rs, s);
    else
      spread_tc<1, TAB>(sv, w, n, alpha + r0 * lda, lda, nr, grid + r0 * rs, rs, s);
  }
}

template <int TAB>
void gather_tab(const SortedSide& sv, const Window& w, int n, const double* grid, int64_t rs, int R,
                double* out, int64_t ldo, cudaStream_t s) {
  for (int r0 = 0; r0 < R; r0 += 2) {
    const int nr = std::min(2, R - r0);
    if (nr == 2)
      gather_tc<2, TAB>(sv, w, n, grid + r0 * rs, rs, nr, out + r0 * ldo, ldo, s);
    else
      gather_tc<1, TAB>(sv, w, n, grid + r0 * rs, rs, nr, out + r0 * ldo, ldo, s);
  }
}

}  // namespace

bool launch_spread_tc(const SortedSide& sv, const Window& w, int n, int tab, const double* alpha,
                      int64_t lda, int R, double* grid, int64_t rs, cudaStream_t s) {
  if (!sv.tc) return false;
  if (sv.ngroups == 0) return true;
  if (sv.sc) {
    launch_spread_sc(sv, w, n, tab, alpha, lda, R, grid, rs, s);
    return true;
  }
  if (tab == 1) spread_tab<1>(sv, w, n, alpha, lda, R, grid, rs, s);
  else if (tab == 2) spread_tab<2>(sv, w, n, alpha, lda, R, grid, rs, s);
  else throw Error(AFS_ERR_CUDA, "tensor-core layout without a compile-time KB table");
  return true;
}

bool launch_gather_tc(const SortedSide& sv, const Window& w, int n, int tab, const double* grid,
                      int64_t rs, int R, double* out, int64_t ldo, cudaStream_t s) {
  if (!sv.tc) return false;
  if (sv.ngroups == 0) return true;
  if (sv.sc) {
    launch_gather_sc(sv, w, n, tab, grid, rs, R, out, ldo, s);
    return true;
  }
  if (tab == 1) gather_tab<1>(sv, w, n, grid, rs, R, out, ldo, s);
  else if (tab == 2) gather_tab<2>(sv, w, n, grid, rs, R, out, ldo, s);
  else throw Error(AFS_ERR_CUDA, "tensor-core layout without a compile-time KB table");
  return true;
}

}  // namespace afs
