// Internal definitions shared by the anovafs CUDA sources (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <condition_variable>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/anovafs.h"

#define AFS_MAX_CUTOFF 8

namespace afs {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

void check_cuda(cudaError_t e, const char* what);
#define AFS_CUDA(call) ::afs::check_cuda((call), #call)

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct Window {
  int d;
  int feat[3];
  double center[3];
  double scale;
  double eta;
  int64_t cells;       // n^d
  int64_t grid_off;    // offset of this window's grid block (per rhs: cells)
  int64_t mult_len;    // (M+1)^(d-1) * (M/2+1)
  int64_t mult_off;    // offset into plan->mult
  int64_t scratch_a_off, scratch_b_off;   // per-window spectral scratch (double2, x max_rhs)
  // deterministic mode (afs_plan_set_deterministic): the spread accumulates fixed-point limbs
  // of the grids with integer reductions instead of fp64 atomics (see grid_add)
  long long* det_limbs = nullptr;   // [3][det_stride], null: fp64 atomics
  int64_t det_stride = 0;           // grid_total * max_rhs
  const double* det_scale = nullptr;   // device [2]: 2^S, 2^-S for the current apply
  const double* det_base = nullptr;    // plan->grids (limb index = cell pointer - det_base)
  double det_unit = 0.0, det_inv_unit = 0.0;   // 2^L, 2^-L for the plan's limb width L
  // 2^((d_max - d) e), e = floor(log2 phi(0)): lifts a lower-dimensional window's values to the
  // plan-wide bound N max|alpha| phi(0)^d_max the scale 2^S is chosen for (undone at finalize)
  double det_boost = 1.0;
};

// fraction of an SM's resident warps the next wave-sized launch (sc2d.cu, tc3d.cu) may take:
// < 1 while two kernel classes are co-scheduled on two streams (spread.cu, gather.cu)
extern thread_local double g_wave_share;

struct SortedSide;   // geometry.cuh
struct PolyTable;    // geometry.cuh

struct GraphEntry {
  const double* alpha;
  int64_t lda;
  double* out;
  int64_t ldo;
  int R;
  cudaGraphExec_t exec;
};

struct CgGraph {
  cudaGraphExec_t exec = nullptr;   // captured once per plan (plan-owned vectors, device beta)
};

struct CgScratch {
  double* r = nullptr;
  double* p = nullptr;
  double* ap = nullptr;
  double* x = nullptr;         // the graph's solution vector (copied out after each solve)
  double* partial = nullptr;   // reduction partials
  double* scalars = nullptr;   // device scalars (see cg.cu)
  double* host_scalars = nullptr;  // pinned
  int64_t n = 0;
  CgGraph graph;   // whole-solve graph: a device-side while loop over the iteration body
};

}  // namespace afs

struct afs_plan {
  int device = 0;
  int P = 0;
  int dtot = 0;
  int64_t Ns = 0, Nt = 0;
  bool has_targets = false;
  int M = 0, m = 0, n = 0, H = 0;   // H = M/2 + 1
  double b = 0.0;                   // Kaiser-Bessel shape pi(2 - M/n)
  int max_rhs = 1;
  std::vector<afs::Window> win;
  afs::Window* d_win = nullptr;     // device copy of win
  double* src = nullptr;            // device, row-major Ns x dtot
  double* tgt = nullptr;            // device, row-major Nt x dtot (nullptr -> src)
  double* mult = nullptr;           // all multipliers
  double2* twiddle = nullptr;       // n entries e^{-2 pi i k / n}
  double* grids = nullptr;          // [rhs][sum of cells]  (rhs-major)
  bool grids_owned = true;          // false after afs_plan_bind_grids
  int64_t grid_total = 0;           // sum of cells over windows
  double2* spec = nullptr;          // [rhs][spec_total] pruned spectra (split spectral stage)
  bool spec_owned = true;           // false after afs_plan_bind_spectra
  int64_t spec_total = 0;           // complex entries per rhs (= sum of multiplier lengths)
  double2* scratch_a = nullptr;
  double2* scratch_b = nullptr;
  int64_t scratch_a_len = 0, scratch_b_len = 0;   // complex entries per rhs
  afs::CgScratch cg;
  int64_t device_bytes = 0;
  int launches_per_apply = 0;
  // v2 geometry (window_eval == 0): per window, bin-sorted source / target nodes
  int window_eval = 0;                 // 0 polynomial window + sliding kernels, 1 exact mirror (v1)
  int kb_tab = 0;                      // compile-time KB table id (kb_table_id)
  std::vector<afs::SortedSide*> src_side, tgt_side;
  // 1-D windows: unwrapped base-cell range [lo, lo + cnt) of the target nodes (gather1d.cu
  // sub-interval tables); cnt = 0 when not computed
  std::vector<int> cell1_lo, cell1_cnt;
  afs::PolyTable* poly = nullptr;      // host copy (passed by value to kernels)
  bool use_graphs = true;
  int fft_mode = 0;                    // 0 four-step register FFT where n allows, 1 generic line kernel
  bool deterministic = false;          // fixed-point spread (afs_plan_set_deterministic)
  long long* det_limbs = nullptr;      // [3][grid_total * max_rhs]
  int det_bits = 40;                   // limb width L: 40 for N <= 2^23, 36 up to 2^27
  double* det_aux = nullptr;           // [0] max|alpha| bits, [1] 2^S, [2] 2^-S
  double det_log2_bound = 0.0;         // log2(N * max window product) + margin
  int det_dmax = 1, det_peak_exp = 0;  // largest window dimension; floor(log2 phi(0)) (per-window boost)
  std::vector<afs::GraphEntry> graphs;
  cudaStream_t istream = nullptr;   // plan-owned stream (graph capture needs a non-legacy one)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  // extra branches of the spread / gather stages: window l runs on branch l % B (branch 0 =
  // the stage's stream), so one window's tail overlaps the next windows' kernels (spread
  // grids are disjoint; the gather's branch b > 0 accumulates into outx[b-1], added at the join)
  static constexpr int kMaxBranches = 4;
  cudaStream_t aux[kMaxBranches - 1] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ev_join[kMaxBranches - 1] = {nullptr, nullptr, nullptr};
  int stage_streams = 0;            // 0: automatic (branch_count), else fixed 1..4
  double* outx[kMaxBranches - 1] = {nullptr, nullptr, nullptr};   // [max_rhs][Nt] each
  // window pipeline (apply_pipeline, pipeline.cu): spread streams and gather streams apart, so
  // a window's gather starts when its own spread + spectral are done
  cudaStream_t pipe_s[kMaxBranches] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t pipe_g[kMaxBranches - 1] = {nullptr, nullptr, nullptr};
  cudaEvent_t pipe_fork = nullptr;
  cudaEvent_t pipe_join[2 * kMaxBranches - 1] = {};
  std::vector<cudaEvent_t> unit_ev;   // one per pipeline unit
  bool profiling = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double stage_ms[3] = {0.0, 0.0, 0.0};
  // per-window kernel timing in profiling mode: events bracket each window's launches
  std::vector<cudaEvent_t> wev_spread, wev_gather;     // P + 1 each
  std::vector<double> win_ms_spread, win_ms_gather;    // accumulated, per window
  int64_t profiled_applies = 0;
  std::mutex mu;
  // reentrant afs_apply (api.cu): concurrent callers beyond the first run on workspace
  // clones -- plans that share this plan's immutable geometry (sorted sides, multipliers,
  // coordinates, tables) and own their grids, scratch, limbs, streams and graphs
  afs_plan* parent = nullptr;            // set on clones: nothing shared is freed with them
  int64_t mode_gen = 0;                  // bumped when the mode changes; clones record theirs
  std::vector<afs_plan*> clones;
  std::vector<char> clone_busy;
  bool primary_busy = false;
  std::mutex pool_mu;
  std::condition_variable pool_cv;
};

namespace afs {

// stages (implemented in spread.cu / spectral.cu / gather.cu / cg.cu)
void spread_all(afs_plan* p, const double* alpha, int64_t lda, int R, cudaStream_t s);
void spectral_all(afs_plan* p, int R, cudaStream_t s, int mode = 0);   // 0 fused, 1 fwd, 2 inv
void gather_all(afs_plan* p, double* out, int64_t ldo, int R, cudaStream_t s);
void apply_impl(afs_plan* p, const double* alpha, int64_t lda, double* out, int64_t ldo,
                int R, cudaStream_t s);
// per-unit stages of the window pipeline (a unit = one window, or all batched 1-D windows)
void spread_unit(afs_plan* p, const std::vector<int>& wins, bool batch1d, const double* alpha,
                 int64_t lda, int R, cudaStream_t s);
void spectral_windows(afs_plan* p, int R, cudaStream_t s, const std::vector<int>& wins);
void gather_unit(afs_plan* p, const std::vector<int>& wins, bool fused1d, double* out,
                 int64_t ldo, int R, cudaStream_t s);
bool gather_1d_fusable(const afs_plan* p);
void det_prepare(afs_plan* p, const double* alpha, int64_t lda, int R, cudaStream_t s);
void clear_rows(void* base, int64_t arr_stride, int narr, int64_t pitch, int64_t width, int R,
                cudaStream_t s);
void det_window_begin(afs_plan* p, const Window& w, int R, cudaStream_t s);
void det_window_finalize(afs_plan* p, const Window& w, int R, cudaStream_t s);
bool pipeline_applies(const afs_plan* p);
void apply_pipeline(afs_plan* p, const double* alpha, int64_t lda, double* out, int64_t ldo,
                    int R, cudaStream_t s);
// the three stages on stream s, no graph (capturable once a warm-up apply ran: allocations
// and one-time kernel attributes happen on first use)
void apply_stages(afs_plan* p, const double* alpha, int64_t lda, double* out, int64_t ldo,
                  int R, cudaStream_t s);
void cg_solve_impl(afs_plan* p, const double* b, double* x, double beta, double tol,
                   int maxiter, int* iters, double* resid, int* conv, cudaStream_t s);
void make_twiddles(afs_plan* p);
// CG vector kernels on caller-owned vectors (cg.cu; afs_cg_vec_*)
void cg_vec_init(const double* b, double* x, double* r, double* p, int64_t n, double beta,
                 double* ws, cudaStream_t s);
void cg_vec_ap(double* ap, const double* p, int64_t n, double* ws, cudaStream_t s);
void cg_vec_update(double* x, double* r, const double* p, const double* ap, int64_t n,
                   double* ws, cudaStream_t s);
void cg_vec_direction(double* p, const double* r, int64_t n, double* ws, cudaStream_t s);
void ensure_aux_streams(afs_plan* p);
void fork_branches(afs_plan* p, int nb, cudaStream_t s);   // branches 1..nb-1 wait on s
bool mix_classes(const afs_plan* p, double* share3, double* share2);   // spread.cu
void gather_1d_cell_ranges(afs_plan* p);   // gather1d.cu: fills cell1_lo / cell1_cnt at plan time
void join_branches(afs_plan* p, int nb, cudaStream_t s);   // s waits on branches 1..nb-1
int spread_branches(const afs_plan* p);
int gather_branches(const afs_plan* p, int R);

// ---------------------------------------------------------------------------
// grid accumulation of the spread
// ---------------------------------------------------------------------------
// Default: one fp64 reduction (RED.E.ADD.F64); the summation order, hence the last bits,
// depend on scheduling.  Deterministic mode: v * 2^S is split exactly into three signed
// L-bit limbs (|v 2^S| < 2^(3L-1) by the choice of S, k_det_scale) that are added with
// 64-bit integer reductions -- associative, so the grid is bit-identical run to run.
// A limb sum stays below 2^63 for up to 2^(63-L) flushes into one cell, and a cell receives
// at most one flush per source node: the plan takes L = 40 bits (quantum 2^-119 of the bound)
// for N <= 2^23 and L = 36 bits up to N = 2^27 (afs_plan_set_deterministic rejects more).
// The wider limbs matter at large b*m: the window's tail values sit ~e^-(b m) below its peak,
// so the fixed-point quantum must be far below the peak-based bound (fuzz: m = 6, os 1.5).
__device__ __forceinline__ void grid_add(const Window& w, double* cell, double v) {
  if (w.det_limbs == nullptr) {
    atomicAdd(cell, v);
    return;
  }
  const int64_t e = cell - w.det_base;
  const double x = (v * w.det_boost) * __ldg(w.det_scale);   // both factors are powers of two
  const double u1 = w.det_unit, u2 = u1 * u1;                      // 2^L, 2^2L (exact)
  const double i1 = w.det_inv_unit, i2 = i1 * i1;
  const double h = trunc(x * i2);
  const double r1 = fma(-h, u2, x);      // exact
  const double m = trunc(r1 * i1);
  const double r2 = fma(-m, u1, r1);     // exact, |r2| < 2^L
  const long long l0 = __double2ll_rn(r2), l1 = (long long)m, l2 = (long long)h;
  unsigned long long* L = reinterpret_cast<unsigned long long*>(w.det_limbs) + e;
  if (l0) atomicAdd(L, (unsigned long long)l0);
  if (l1) atomicAdd(L + w.det_stride, (unsigned long long)l1);
  if (l2) atomicAdd(L + 2 * w.det_stride, (unsigned long long)l2);
}

// ---------------------------------------------------------------------------
// device helpers: exact mirror of the reference window arithmetic
// ---------------------------------------------------------------------------
// Kaiser-Bessel window, nfft.py:118-122.  Each product/difference is rounded
// separately (no FMA contraction) to follow numpy's evaluation order.
__device__ __forceinline__ double kb_window(double dist, int m, double b) {
  const double mm = (double)(m * m);
  const double arg = sqrt(fmax(__dsub_rn(mm, __dmul_rn(dist, dist)), 0.0));
  if (arg > 1e-12) {
    const double safe = fmax(arg, 1e-300);
    return sinh(__dmul_rn(b, arg)) / __dmul_rn(3.141592653589793, safe);
  }
  return b / 3.141592653589793;
}

// Per-dimension stencil of one node (nfft.py:166-174): base cell u = floor(n x),
// cells u+1-m .. u+m reduced mod n, weights phi(n x - cell).
template <int MM>
__device__ __forceinline__ void stencil_1d(double xs, int n, double b, double (&w)[2 * MM],
                                           int (&idx)[2 * MM]) {
  const double nx = __dmul_rn((double)n, xs);
  const double u = floor(nx);
  const long long ui = (long long)u;
#pragma unroll
  for (int o = 0; o < 2 * MM; ++o) {
    const double cell = u + (double)(o + 1 - MM);
    w[o] = kb_window(__dsub_rn(nx, cell), MM, b);
    long long c = (ui + (o + 1 - MM)) % n;
    idx[o] = (int)(c < 0 ? c + n : c);
  }
}

// scaled coordinate (fastsum.py:229): (x - center) * scale
__device__ __forceinline__ double scaled_coord(double x, double c, double s) {
  return __dmul_rn(__dsub_rn(x, c), s);
}

}  // namespace afs
