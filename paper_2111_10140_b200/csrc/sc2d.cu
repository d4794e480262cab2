// Launchers for the sub-cell Chebyshev 2-D kernels (sc2d.cuh).
#include <cstdlib>

#include "sc2d.cuh"

namespace afs {

namespace {

constexpr int kU = 8;   // groups per warp range are a multiple of the gather's 8 per iteration (the spread takes 4)
constexpr int kD = 4;   // batches staged ahead (shared-memory ring)
static_assert(4 * kU + 7 < kTcTailGroups, "the layout's empty tail must cover the reads 4 iterations ahead");
static_assert(kU == kScGatherU, "warp ranges are multiples of the gather iteration");

int num_sms_sc() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    AFS_CUDA(cudaGetDevice(&dev));
    AFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

// one wave of resident warps (or AFS_SC_WARPS per SM), each taking a contiguous range of groups
template <typename K>
void wave(K kernel, int64_t ngroups, int& wps, int& gpw, int64_t& blocks) {
  if (wps == 0) {
    if (const char* e = getenv("AFS_SC_WARPS")) {
      wps = std::max(1, atoi(e));
    } else {
      int occ = 0;
      AFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 128, 0));
      wps = std::max(1, occ) * 4;
    }
  }
  // a share < 1 (co-scheduled classes) takes whole blocks: 4 warps each
  const int use = std::max(4, (int)(wps * g_wave_share + 0.5) / 4 * 4);
  const int64_t warps = (int64_t)num_sms_sc() * use;
  const int64_t gw = std::max<int64_t>(kU, (ngroups + warps - 1) / warps);
  gpw = (int)((gw + kU - 1) / kU * kU);
  blocks = ((ngroups + gpw - 1) / gpw * 32 + 127) / 128;
}

template <int TAB, bool POW2>
void spread1(const SortedSide& sv, const Window& w, int n, const double* alpha, double* grid,
             cudaStream_t s) {
  static int wps = 0;
  int gpw;
  int64_t blocks;
  auto k = k_spread_sc<TAB, POW2, kD>;
  wave(k, sv.ngroups, wps, gpw, blocks);
  k<<<(unsigned)blocks, 128, 0, s>>>(sv, w, n, alpha, grid, gpw);
}

template <int TAB, bool POW2>
void gather1(const SortedSide& sv, const Window& w, int n, const double* grid, double* out,
             cudaStream_t s) {
  static int wps = 0;
  int gpw;
  int64_t blocks;
  auto k = k_gather_sc<TAB, POW2, kD>;
  wave(k, sv.ngroups, wps, gpw, blocks);
  k<<<(unsigned)blocks, 128, 0, s>>>(sv, w, n, grid, out, gpw);
}

bool pow2(int n) { return (n & (n - 1)) == 0; }

}  // namespace

// one launch per right-hand side (the node stream is re-read; the fold is per launch)
void launch_spread_sc(const SortedSide& sv, const Window& w, int n, int tab, const double* alpha,
                      int64_t lda, int R, double* grid, int64_t rs, cudaStream_t s) {
  if (sv.ngroups == 0) return;
  if (tab != 1 && tab != 2) throw Error(AFS_ERR_CUDA, "sub-cell layout without a compile-time KB table");
  const bool p2 = pow2(n);
  for (int r = 0; r < R; ++r) {
    const double* a = alpha + r * lda;
    double* g = grid + r * rs;
    if (tab == 1) p2 ? spread1<1, true>(sv, w, n, a, g, s) : spread1<1, false>(sv, w, n, a, g, s);
    else p2 ? spread1<2, true>(sv, w, n, a, g, s) : spread1<2, false>(sv, w, n, a, g, s);
  }
}

void launch_gather_sc(const SortedSide& sv, const Window& w, int n, int tab, const double* grid,
                      int64_t rs, int R, double* out, int64_t ldo, cudaStream_t s) {
  if (sv.ngroups == 0) return;
  if (tab != 1 && tab != 2) throw Error(AFS_ERR_CUDA, "sub-cell layout without a compile-time KB table");
  const bool p2 = pow2(n);
  for (int r = 0; r < R; ++r) {
    const double* g = grid + r * rs;
    double* o = out + r * ldo;
    if (tab == 1) p2 ? gather1<1, true>(sv, w, n, g, o, s) : gather1<1, false>(sv, w, n, g, o, s);
    else p2 ? gather1<2, true>(sv, w, n, g, o, s) : gather1<2, false>(sv, w, n, g, o, s);
  }
}

}  // namespace afs
