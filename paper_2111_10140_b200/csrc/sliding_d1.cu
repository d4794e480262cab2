// v2 sliding-window spread/gather instantiations, d=1 windows.
#include "sliding_impl.cuh"

namespace afs {
AFS_SLIDING_INSTANTIATE(1)
}  // namespace afs

namespace afs {

// all 1-D windows of a batch in one solo-spread launch (solo.cuh k_spread_solo_batch)
template <int MM, int TAB>
static void spread_batch_tab(const SoloBatch& B, int n, const PolyTable& T, const double* alpha,
                             int64_t lda, int R, double* grid, int64_t rs, cudaStream_t s) {
  int64_t xblocks = 1;
  for (int i = 0; i < B.nwin; ++i) xblocks = std::max<int64_t>(xblocks, (B.sv[i].nchunks * 32 + 127) / 128);
  const dim3 g((unsigned)xblocks, (unsigned)B.nwin);
  for (int r0 = 0; r0 < R; r0 += 2) {
    const int nr = std::min(2, R - r0);
    if (nr == 2 && TAB != 0)
      k_spread_solo_batch<1, MM, 2, TAB><<<g, 128, 0, s>>>(B, n, T, alpha + r0 * lda, lda, nr, grid + r0 * rs, rs);
    else
      for (int r = r0; r < r0 + nr; ++r)
        k_spread_solo_batch<1, MM, 1, TAB><<<g, 128, 0, s>>>(B, n, T, alpha + r * lda, lda, 1, grid + r * rs, rs);
  }
}

template <int MM>
static void spread_batch_mm(const SoloBatch& B, int n, int tab, const PolyTable& T, const double* alpha,
                            int64_t lda, int R, double* grid, int64_t rs, cudaStream_t s) {
  if (tab == 1) spread_batch_tab<MM, 1>(B, n, T, alpha, lda, R, grid, rs, s);
  else if (tab == 2) spread_batch_tab<MM, 2>(B, n, T, alpha, lda, R, grid, rs, s);
  else spread_batch_tab<MM, 0>(B, n, T, alpha, lda, R, grid, rs, s);
}

void launch_spread_solo_batch_1d(const SoloBatch& B, int n, int m, int tab, const PolyTable& T,
                                 const double* alpha, int64_t lda, int R, double* grid, int64_t rs,
                                 cudaStream_t s) {
  switch (m) {
    case 1: spread_batch_mm<1>(B, n, tab, T, alpha, lda, R, grid, rs, s); break;
    case 2: spread_batch_mm<2>(B, n, tab, T, alpha, lda, R, grid, rs, s); break;
    case 3: spread_batch_mm<3>(B, n, tab, T, alpha, lda, R, grid, rs, s); break;
    case 4: spread_batch_mm<4>(B, n, tab, T, alpha, lda, R, grid, rs, s); break;
    case 5: spread_batch_mm<5>(B, n, tab, T, alpha, lda, R, grid, rs, s); break;
    case 6: spread_batch_mm<6>(B, n, tab, T, alpha, lda, R, grid, rs, s); break;
    case 7: spread_batch_mm<7>(B, n, tab, T, alpha, lda, R, grid, rs, s); break;
    default: spread_batch_mm<8>(B, n, tab, T, alpha, lda, R, grid, rs, s); break;
  }
  AFS_CUDA(cudaGetLastError());
}

}  // namespace afs
