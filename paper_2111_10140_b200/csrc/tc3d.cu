// Launchers for the fp64 tensor-core 3-D kernels (tc3d.cuh).
#include <cstdlib>

#include "tc3d.cuh"

namespace afs {

namespace {

constexpr int kDepth = 4;   // groups staged ahead (shared-memory ring)
static_assert(kDepth <= kTcTailGroups, "the layout's empty tail must cover the staged groups");

int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    AFS_CUDA(cudaGetDevice(&dev));
    AFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

// one wave of resident warps, each taking a contiguous range of groups
template <typename K>
void launch_wave(K kernel, int64_t ngroups, int& warps_per_sm, int& gpw, int64_t& blocks) {
  if (warps_per_sm == 0) {
    int occ = 0;
    AFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 128, 0));
    warps_per_sm = std::max(1, occ) * 4;
  }
  const int use = std::max(4, (int)(warps_per_sm * g_wave_share + 0.5) / 4 * 4);
  const int64_t warps = (int64_t)sm_count() * use;
  gpw = (int)std::max<int64_t>(1, (ngroups + warps - 1) / warps);
  blocks = ((ngroups + gpw - 1) / gpw * 32 + 127) / 128;
}

template <int RG, int TAB, bool POW2>
void spread3(const SortedSide& sv, const Window& w, int n, const double* alpha, int64_t lda, int nr,
             double* grid, int64_t rs, cudaStream_t s) {
  static int wps = 0;
  int gpw;
  int64_t blocks;
  auto k = k_spread_tc3<RG, TAB, POW2, kDepth>;
  launch_wave(k, sv.ngroups, wps, gpw, blocks);
  k<<<(unsigned)blocks, 128, 0, s>>>(sv, w, n, alpha, lda, nr, grid, rs, gpw);
}

template <int RG, int TAB, bool POW2>
void gather3(const SortedSide& sv, const Window& w, int n, const double* grid, int64_t rs, int nr,
             double* out, int64_t ldo, cudaStream_t s) {
  static int wps = 0;
  int gpw;
  int64_t blocks;
  auto k = k_gather_tc3<RG, TAB, POW2, kDepth>;
  launch_wave(k, sv.ngroups, wps, gpw, blocks);
  k<<<(unsigned)blocks, 128, 0, s>>>(sv, w, n, grid, rs, nr, out, ldo, gpw);
}

template <int TAB, bool POW2>
void spread_rhs(const SortedSide& sv, const Window& w, int n, const double* alpha, int64_t lda, int R,
                double* grid, int64_t rs, cudaStream_t s) {
  for (int r0 = 0; r0 < R; r0 += 2) {
    const int nr = std::min(2, R - r0);
    if (nr == 2) spread3<2, TAB, POW2>(sv, w, n, alpha + r0 * lda, lda, nr, grid + r0 * rs, rs, s);
    else spread3<1, TAB, POW2>(sv, w, n, alpha + r0 * lda, lda, nr, grid + r0 * rs, rs, s);
  }
}

template <int TAB, bool POW2>
void gather_rhs(const SortedSide& sv, const Window& w, int n, const double* grid, int64_t rs, int R,
                double* out, int64_t ldo, cudaStream_t s) {
  for (int r0 = 0; r0 < R; r0 += 2) {
    const int nr = std::min(2, R - r0);
    if (nr == 2) gather3<2, TAB, POW2>(sv, w, n, grid + r0 * rs, rs, nr, out + r0 * ldo, ldo, s);
    else gather3<1, TAB, POW2>(sv, w, n, grid + r0 * rs, rs, nr, out + r0 * ldo, ldo, s);
  }
}

bool pow2(int n) { return (n & (n - 1)) == 0; }

}  // namespace

bool launch_spread_tc3(const SortedSide& sv, const Window& w, int n, int tab, const double* alpha,
                       int64_t lda, int R, double* grid, int64_t rs, cudaStream_t s) {
  if (!sv.tc || w.d != 3) return false;
  if (sv.ngroups == 0) return true;
  const bool p2 = pow2(n);
  if (tab == 1) p2 ? spread_rhs<1, true>(sv, w, n, alpha, lda, R, grid, rs, s)
                   : spread_rhs<1, false>(sv, w, n, alpha, lda, R, grid, rs, s);
  else if (tab == 2) p2 ? spread_rhs<2, true>(sv, w, n, alpha, lda, R, grid, rs, s)
                        : spread_rhs<2, false>(sv, w, n, alpha, lda, R, grid, rs, s);
  else throw Error(AFS_ERR_CUDA, "tensor-core layout without a compile-time KB table");
  return true;
}

bool launch_gather_tc3(const SortedSide& sv, const Window& w, int n, int tab, const double* grid,
                       int64_t rs, int R, double* out, int64_t ldo, cudaStream_t s) {
  if (!sv.tc || w.d != 3) return false;
  if (sv.ngroups == 0) return true;
  const bool p2 = pow2(n);
  if (tab == 1) p2 ? gather_rhs<1, true>(sv, w, n, grid, rs, R, out, ldo, s)
                   : gather_rhs<1, false>(sv, w, n, grid, rs, R, out, ldo, s);
  else if (tab == 2) p2 ? gather_rhs<2, true>(sv, w, n, grid, rs, R, out, ldo, s)
                        : gather_rhs<2, false>(sv, w, n, grid, rs, R, out, ldo, s);
  else throw Error(AFS_ERR_CUDA, "tensor-core layout without a compile-time KB table");
  return true;
}

}  // namespace afs
