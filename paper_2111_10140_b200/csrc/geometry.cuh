// Plan-time node geometry, bin-sorted per window (replaces NfftPlan's per-node
// _idx/_w tables, nfft.py:164-174), and the device helpers the v2
// spread/gather kernels share.
#pragma once

#include "afs_internal.cuh"

namespace afs {

#include "kb_tables.inc"
#include "kb_cheb.inc"
#include "kb_sub.inc"

constexpr int kPolyMaxOffsets = 2 * AFS_MAX_CUTOFF;   // 2m
constexpr int kPolyTerms = 14;                        // degree 13 in x = f - 1/4

// Kaiser-Bessel window as polynomials P_i(f) ~ phi(f + m - 1 - i), f in [0, 1/2],
// monomial coefficients in x = f - 1/4 (index 0 = constant term).  Values for
// f in (1/2, 1) follow from phi(f+m-1-i) = P_{2m-1-i}(1-f).
struct PolyTable {
  double c[kPolyMaxOffsets][kPolyTerms];
};

// A run of consecutive sorted nodes sharing one column (all but the last
// dimension's base cell); processed by one team with one sliding window.
struct Chunk {
  int32_t col;     // column id: u0*n+u1 (d=3), u0 (d=2), 0 (d=1)
  int32_t count;   // nodes in the run
  int64_t begin;   // first sorted node
  int32_t cell0;   // last-dim base cell of the first node (filled on the device)
  int32_t pad_;
};

// Sorted nodes of one window on one side (sources or targets).
struct SortedSide {
  int64_t N = 0;
  double* nx = nullptr;      // [d][N]: n * scaled coordinate, sorted by cell
  int32_t* perm = nullptr;   // [N]: sorted position -> original node index (-1: padding)
  Chunk* chunks = nullptr;   // device
  int64_t nchunks = 0;
  int chunk_cap = 0;
  // tensor-core layout (tc2d.cuh): sorted by half-cell (base cell + reflection class per
  // dimension), every half-cell padded to a multiple of 8 nodes, so that each group of 8
  // consecutive nodes shares one stencil.  nx then holds the polynomial variable
  // x = (c ? 1 - f : f) - 1/4 of poly_weights instead of n*x, and ghdr[N/8] the group's
  // stencil (tc_header); N counts the padding, n_real does not
  bool tc = false;
  // sub-cell layout (sc2d.cuh, dense 2-D windows; implies tc): sorted by (base cell,
  // sub-interval floor(16 f)) per dimension, nx holds the Chebyshev variables 32 f - 2 s - 1,
  // ghdr the group's sc_header
  bool sc = false;
  int64_t n_real = 0;
  int32_t* ghdr = nullptr;
  uint64_t* ghdr64 = nullptr;   // 3-D layout: u0 | u1 << 16 | u2 << 32 | c_t << (48 + t)
  int64_t ngroups = 0;   // groups of 8 holding nodes; N / 8 - ngroups >= kTcTailGroups empty ones follow
  __host__ __device__ const double* x0() const { return nx; }
  __host__ __device__ const double* x1() const { return nx + N; }
  __host__ __device__ const double* x2() const { return nx + 2 * N; }
};

// plan-build temporaries shared by all windows' sorts (grown on demand, freed by release)
struct BuildScratch {
  double* nx_tmp = nullptr;
  uint64_t *key_a = nullptr, *key_b = nullptr;
  int32_t *idx_a = nullptr, *idx_b = nullptr;
  int64_t cap = 0;        // nodes the arrays above hold
  void* temp = nullptr;   // CUB radix sort
  size_t temp_bytes = 0;
  int32_t* counts = nullptr;
  int64_t* starts = nullptr;
  int64_t counts_cap = 0;
  void reserve(int64_t N, int d);
  void reserve_counts(int64_t n);
  void* sort_temp(size_t bytes);
  void release();
};

void build_sorted_side(afs_plan* p, const Window& w, const double* X, int64_t N,
                       SortedSide* out, BuildScratch& sc);
void build_sorted_side_tc(afs_plan* p, const Window& w, const double* X, int64_t N,
                          SortedSide* out, BuildScratch& sc);
bool tc_eligible(int d, int m, int tab, int n, int64_t N);
bool tc3_eligible(int d, int m, int tab, int n, int64_t N);
// dense 3-D windows: the tensor-core layout, or false (nothing built) when padding the
// half-cells to groups of 8 would add more than max_padding * N nodes
bool build_sorted_side_tc3(afs_plan* p, const Window& w, const double* X, int64_t N, SortedSide* out,
                           BuildScratch& sc, double max_padding, bool for_spread = true);
// dense 2-D windows: the sub-cell layout, or false (nothing built) when padding the sub-cells to
// groups of 8 would add more than max_padding * N nodes
bool sc_eligible(int d, int m, int tab, int n, int64_t N);
bool build_sorted_side_sc(afs_plan* p, const Window& w, const double* X, int64_t N, SortedSide* out,
                          BuildScratch& sc, double max_padding, double min_nodes = 64.0);
constexpr int kScSub = 16;   // sub-intervals per cell and dimension (kb_sub.inc)
__host__ __device__ __forceinline__ int32_t sc_header(int u0, int u1, int s0, int s1) {
  return (int32_t)((uint32_t)u0 | ((uint32_t)u1 << 12) | ((uint32_t)s0 << 24) | ((uint32_t)s1 << 28));
}
constexpr int kTcTailGroups = 40;   // >= the groups the kernels read ahead (tc2d.cuh D * U; sc2d.cuh 8 batches + 3)

// group header of the tensor-core layout: wrapped base cells and reflection classes
__host__ __device__ __forceinline__ int32_t tc_header(int u0, int u1, int c0, int c1) {
  return u0 | (u1 << 14) | (c0 << 28) | (c1 << 29);
}
void free_sorted_side(SortedSide* s);
void make_poly_table(int m, double b, PolyTable* t);
int kb_table_id(int M, int n);   // 1: n = 2M, 2: 2n = 3M, 0: run-time table

// ---------------------------------------------------------------------------
// device: per-dimension window values of one node in the 2m stencil order
// ---------------------------------------------------------------------------
// TAB 0: run-time table T (any n/M); TAB 1, 2: compile-time tables (kb_tables.inc) for
// n/M = 2 and 3/2, whose coefficients stream from the constant bank.
template <int MM, int TAB>
__device__ __forceinline__ void poly_weights(double f, const PolyTable& T, double (&w)[2 * MM]) {
  const bool refl = f > 0.5;
  const double x = (refl ? __dsub_rn(1.0, f) : f) - 0.25;
#pragma unroll
  for (int i = 0; i < 2 * MM; ++i) {
    constexpr int NT = TAB == 0 ? kPolyTerms : kb_terms<TAB, MM>();
    double v = TAB == 0 ? T.c[i][NT - 1] : kb_coef<TAB, MM>(i, NT - 1);
#pragma unroll
    for (int k = NT - 2; k >= 0; --k)
      v = fma(v, x, TAB == 0 ? T.c[i][k] : kb_coef<TAB, MM>(i, k));
    w[i] = v;
  }
  if (refl) {
#pragma unroll
    for (int i = 0; i < MM; ++i) {
      const double t = w[i];
      w[i] = w[2 * MM - 1 - i];
      w[2 * MM - 1 - i] = t;
    }
  }
}

// exact mirror of nfft.py:118-122 on the stencil of one node (dist = f + m-1-i)
template <int MM>
__device__ __forceinline__ void exact_weights(double f, double b, double (&w)[2 * MM]) {
#pragma unroll
  for (int i = 0; i < 2 * MM; ++i) w[i] = kb_window(f + (double)(MM - 1 - i), MM, b);
}

}  // namespace afs
