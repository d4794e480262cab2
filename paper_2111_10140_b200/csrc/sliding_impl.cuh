// Launch helpers for the v2 kernels; included once per dimension file.
#pragma once

#include <algorithm>

#include "sliding.cuh"
#include "solo.cuh"

namespace afs {

template <int D, int MM, int RG, int TAB>
static void run_spread_solo(const SortedSide& sv, const Window& w, int n, const PolyTable& T,
                            const double* alpha, int64_t lda, int nr, double* grid, int64_t rs,
                            cudaStream_t s) {
  constexpr int threads = 128;   // one warp per column run
  const int64_t blocks = (sv.nchunks * 32 + threads - 1) / threads;
  k_spread_solo<D, MM, RG, TAB><<<(unsigned)blocks, threads, 0, s>>>(sv, w, n, T, alpha, lda, nr,
                                                                    grid, rs);
}

template <int D, int MM, int RG, int TAB>
static void run_gather_solo(const SortedSide& sv, const Window& w, int n, const PolyTable& T,
                            const double* grid, int64_t rs, int nr, double* out, int64_t ldo,
                            cudaStream_t s) {
  constexpr int threads = 128;
  // persistent warps: at most one resident wave, each warp loops over runs
  static int resident = 0;
  if (resident == 0) {
    int occ = 0, dev = 0, sms = 0;
    AFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather_solo<D, MM, RG, TAB>,
                                                           threads, 0));
    AFS_CUDA(cudaGetDevice(&dev));
    AFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    resident = std::max(1, occ) * sms;
  }
  const int64_t need = (sv.nchunks * 32 + threads - 1) / threads;
  const int64_t blocks = std::min<int64_t>(need, resident);
  k_gather_solo<D, MM, RG, TAB><<<(unsigned)blocks, threads, 0, s>>>(sv, w, n, T, grid, rs, nr,
                                                                    out, ldo);
}

template <int D, int MM, int RG, int TAB>
static void run_spread_v2(const SortedSide& sv, const Window& w, int n, const PolyTable& T,
                          const double* alpha, int64_t lda, int nr, double* grid, int64_t rs,
                          cudaStream_t s) {
  using C = Cfg<D, MM>;
  constexpr int threads = 128;
  const size_t smem = (size_t)(threads / 32) * Stage<D, MM, 1 + RG>::WARP_SPAN * sizeof(double);
  const int64_t warps = (sv.nchunks + C::TPW - 1) / C::TPW;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  if (smem > 48 * 1024)
    AFS_CUDA(cudaFuncSetAttribute(k_spread_v2<D, MM, RG, TAB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_spread_v2<D, MM, RG, TAB><<<(unsigned)blocks, threads, smem, s>>>(sv, w, n, T, alpha, lda, nr, grid,
                                                                  rs);
}

template <int D, int MM, int RG, int TAB>
static void run_gather_v2(const SortedSide& sv, const Window& w, int n, const PolyTable& T,
                          const double* grid, int64_t rs, int nr, double* out, int64_t ldo,
                          cudaStream_t s) {
  using C = Cfg<D, MM>;
  constexpr int threads = 128;
  const size_t smem = (size_t)(threads / 32) *
                      Stage<D, MM, 1, RG * Red<C::TEAM>::RSTR>::WARP_SPAN * sizeof(double);
  const int64_t warps = (sv.nchunks + C::TPW - 1) / C::TPW;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  if (smem > 48 * 1024)
    AFS_CUDA(cudaFuncSetAttribute(k_gather_v2<D, MM, RG, TAB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_gather_v2<D, MM, RG, TAB><<<(unsigned)blocks, threads, smem, s>>>(sv, w, n, T, grid, rs, nr, out,
                                                                  ldo);
}

template <int D, int MM, int TAB>
static bool spread_tab(const SortedSide& sv, const Window& w, int n, const PolyTable& T,
                       const double* alpha, int64_t lda, int nr, double* grid, int64_t rs,
                       cudaStream_t s) {
  if constexpr (D == 3 && MM == 4 && TAB != 0 && Fits<D, MM, 4>::value) {
    if (nr >= 3) {   // v2_rhs_group: RHS groups of 4 for the 3-D spread
      run_spread_v2<D, MM, 4, TAB>(sv, w, n, T, alpha, lda, nr, grid, rs, s);
      return true;
    }
  }
  if constexpr (SoloFits<D, MM, 2>::value && TAB != 0) {
    if (nr >= 2) {
      run_spread_solo<D, MM, 2, TAB>(sv, w, n, T, alpha, lda, nr, grid, rs, s);
      return true;
    }
  }
  if constexpr (SoloFits<D, MM, 1>::value) {
    if (nr == 1) {
      run_spread_solo<D, MM, 1, TAB>(sv, w, n, T, alpha, lda, nr, grid, rs, s);
      return true;
    }
  }
  if constexpr (Fits<D, MM, 2>::value && MM <= 4 && TAB != 0) {
    if (nr >= 2) {
      run_spread_v2<D, MM, 2, TAB>(sv, w, n, T, alpha, lda, nr, grid, rs, s);
      return true;
    }
  }
  if constexpr (Fits<D, MM, 1>::value) {
    if (nr == 1) {
      run_spread_v2<D, MM, 1, TAB>(sv, w, n, T, alpha, lda, nr, grid, rs, s);
      return true;
    }
  }
  return false;
}

template <int D, int MM>
static bool spread_mm(const SortedSide& sv, const Window& w, int n, int tab, const PolyTable& T,
                      const double* alpha, int64_t lda, int nr, double* grid, int64_t rs,
                      cudaStream_t s) {
  if (tab == 1) return spread_tab<D, MM, 1>(sv, w, n, T, alpha, lda, nr, grid, rs, s);
  if (tab == 2) return spread_tab<D, MM, 2>(sv, w, n, T, alpha, lda, nr, grid, rs, s);
  return spread_tab<D, MM, 0>(sv, w, n, T, alpha, lda, nr, grid, rs, s);
}

template <int D, int MM, int TAB>
static bool gather_tab(const SortedSide& sv, const Window& w, int n, const PolyTable& T,
                       const double* grid, int64_t rs, int nr, double* out, int64_t ldo,
                       cudaStream_t s) {

  if constexpr (SoloFits<D, MM, 2>::value && TAB != 0) {
    if (nr >= 2) {
      run_gather_solo<D, MM, 2, TAB>(sv, w, n, T, grid, rs, nr, out, ldo, s);
      return true;
    }
  }
  if constexpr (SoloFits<D, MM, 1>::value) {
    if (nr == 1) {
      run_gather_solo<D, MM, 1, TAB>(sv, w, n, T, grid, rs, nr, out, ldo, s);
      return true;
    }
  }
  if constexpr (Fits<D, MM, 2>::value && MM <= 4 && TAB != 0) {
    if (nr >= 2) {
      run_gather_v2<D, MM, 2, TAB>(sv, w, n, T, grid, rs, nr, out, ldo, s);
      return true;
    }
  }
  if constexpr (Fits<D, MM, 1>::value) {
    if (nr == 1) {
      run_gather_v2<D, MM, 1, TAB>(sv, w, n, T, grid, rs, nr, out, ldo, s);
      return true;
    }
  }
  return false;
}

template <int D, int MM>
static bool gather_mm(const SortedSide& sv, const Window& w, int n, int tab, const PolyTable& T,
                      const double* grid, int64_t rs, int nr, double* out, int64_t ldo,
                      cudaStream_t s) {
  if (tab == 1) return gather_tab<D, MM, 1>(sv, w, n, T, grid, rs, nr, out, ldo, s);
  if (tab == 2) return gather_tab<D, MM, 2>(sv, w, n, T, grid, rs, nr, out, ldo, s);
  return gather_tab<D, MM, 0>(sv, w, n, T, grid, rs, nr, out, ldo, s);
}

#define AFS_SLIDING_INSTANTIATE(DIM)                                                            \
  template <>                                                                                   \
  bool launch_spread_v2<DIM>(const SortedSide& sv, const Window& w, int n, int m, int tab,               \
                             const PolyTable& T, const double* alpha, int64_t lda, int nr,      \
                             double* grid, int64_t rs, cudaStream_t s) {                        \
    if (sv.nchunks == 0) return true;                                                           \
    switch (m) {                                                                                \
      case 1: return spread_mm<DIM, 1>(sv, w, n, tab, T, alpha, lda, nr, grid, rs, s);               \
      case 2: return spread_mm<DIM, 2>(sv, w, n, tab, T, alpha, lda, nr, grid, rs, s);               \
      case 3: return spread_mm<DIM, 3>(sv, w, n, tab, T, alpha, lda, nr, grid, rs, s);               \
      case 4: return spread_mm<DIM, 4>(sv, w, n, tab, T, alpha, lda, nr, grid, rs, s);               \
      case 5: return spread_mm<DIM, 5>(sv, w, n, tab, T, alpha, lda, nr, grid, rs, s);               \
      case 6: return spread_mm<DIM, 6>(sv, w, n, tab, T, alpha, lda, nr, grid, rs, s);               \
      case 7: return spread_mm<DIM, 7>(sv, w, n, tab, T, alpha, lda, nr, grid, rs, s);               \
      case 8: return spread_mm<DIM, 8>(sv, w, n, tab, T, alpha, lda, nr, grid, rs, s);               \
      default: return false;                                                                    \
    }                                                                                           \
  }                                                                                             \
  template <>                                                                                   \
  bool launch_gather_v2<DIM>(const SortedSide& sv, const Window& w, int n, int m, int tab,               \
                             const PolyTable& T, const double* grid, int64_t rs, int nr,        \
                             double* out, int64_t ldo, cudaStream_t s) {                        \
    if (sv.nchunks == 0) return true;                                                           \
    switch (m) {                                                                                \
      case 1: return gather_mm<DIM, 1>(sv, w, n, tab, T, grid, rs, nr, out, ldo, s);                 \
      case 2: return gather_mm<DIM, 2>(sv, w, n, tab, T, grid, rs, nr, out, ldo, s);                 \
      case 3: return gather_mm<DIM, 3>(sv, w, n, tab, T, grid, rs, nr, out, ldo, s);                 \
      case 4: return gather_mm<DIM, 4>(sv, w, n, tab, T, grid, rs, nr, out, ldo, s);                 \
      case 5: return gather_mm<DIM, 5>(sv, w, n, tab, T, grid, rs, nr, out, ldo, s);                 \
      case 6: return gather_mm<DIM, 6>(sv, w, n, tab, T, grid, rs, nr, out, ldo, s);                 \
      case 7: return gather_mm<DIM, 7>(sv, w, n, tab, T, grid, rs, nr, out, ldo, s);                 \
      case 8: return gather_mm<DIM, 8>(sv, w, n, tab, T, grid, rs, nr, out, ldo, s);                 \
      default: return false;                                                                    \
    }                                                                                           \
  }

}  // namespace afs
