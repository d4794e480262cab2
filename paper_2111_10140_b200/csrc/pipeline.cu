// Window pipeline of one apply: each window (or the batch of 1-D windows) runs spread ->
// spectral on a spread stream and its gather on a gather stream as soon as that window's
// spectral stage is done, instead of all spreads -> all spectral passes -> all gathers.
//
// The windows are independent terms of the ANOVA sum (anova.py:179-183), so nothing but the
// order of the output additions couples them.  That order stays fixed: gather stream b adds
// its windows in window order into its own accumulator (b = 0: out itself) and the join adds
// the accumulators in stream order (k_add_into), exactly as the staged path's gather branches
// do, so results are run-to-run reproducible.  Plans with few windows gain (C2: three 3-D
// windows at N = 100k, 0.226 -> 0.203 ms per matvec): the stage barriers and per-stage tails
// were a large part of their apply.  Deterministic mode, profiling and plans with more than
// 8 windows keep the staged path (apply_stages); AFS_PIPELINE=0/1 forces the choice.  In
// deterministic mode the scale 2^S is set once per apply before the fork and every window
// clears its own limbs before its spread and converts them after it.
#include <algorithm>
#include <cstdlib>

#include "afs_internal.cuh"
#include "geometry.cuh"

namespace afs {

__global__ void k_add_into(double* __restrict__ out, int64_t ldo, const double* __restrict__ a0,
                           const double* __restrict__ a1, const double* __restrict__ a2, int na,
                           int64_t lda, int64_t N, int R);

bool pipeline_applies(const afs_plan* p) {
  static const int force = [] {
    const char* e = getenv("AFS_PIPELINE");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  if (force == 0) return false;
  if (p->window_eval != 0 || p->profiling || p->P < 2) return false;
  // measured: C2 (3 windows) -10% per matvec (deterministic CG: 0.367 -> 0.344 ms per iteration);
  // C5 (30 windows) +4%, C3 (39) +-0 -- with many
  // windows the staged branches already overlap the tails, and the per-window spectral
  // launches cost more than the barriers they remove
  if (force < 0 && p->P > 8) return false;
  // 1-D windows must form one unit: batched spreads and the fused gather
  int n1 = 0;
  for (int l = 0; l < p->P; ++l) {
    if (p->win[l].d != 1) continue;
    if (p->src_side[l]->tc || (p->tgt_side[l] && p->tgt_side[l]->tc)) return false;
    ++n1;
  }
  if (n1 == 1) return false;
  if (n1 >= 2) {
    const char* e = getenv("AFS_SPREAD1D");
    if ((e && e[0] == '0') || !gather_1d_fusable(p)) return false;
  }
  return true;
}

static void ensure_pipe(afs_plan* p, int ns, int ng, int units) {
  for (int b = 0; b < ns; ++b)
    if (!p->pipe_s[b]) AFS_CUDA(cudaStreamCreateWithFlags(&p->pipe_s[b], cudaStreamNonBlocking));
  for (int b = 0; b + 1 < ng; ++b)
    if (!p->pipe_g[b]) AFS_CUDA(cudaStreamCreateWithFlags(&p->pipe_g[b], cudaStreamNonBlocking));
  if (!p->pipe_fork) AFS_CUDA(cudaEventCreateWithFlags(&p->pipe_fork, cudaEventDisableTiming));
  for (cudaEvent_t& e : p->pipe_join)
    if (!e) AFS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  while ((int)p->unit_ev.size() < units) {
    cudaEvent_t e;
    AFS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->unit_ev.push_back(e);
  }
}

void apply_pipeline(afs_plan* p, const double* alpha, int64_t lda, double* out, int64_t ldo,
                    int R, cudaStream_t s) {
  // units in window order; all 1-D windows form one unit at the first 1-D window's place
  struct Unit {
    std::vector<int> wins;
    bool one_d;
  };
  std::vector<Unit> units;
  int unit_1d = -1;
  for (int l = 0; l < p->P; ++l) {
    if (p->win[l].d == 1) {
      if (unit_1d < 0) {
        unit_1d = (int)units.size();
        units.push_back(Unit{{}, true});
      }
      units[unit_1d].wins.push_back(l);
    } else {
      units.push_back(Unit{{l}, false});
    }
  }
  const int nu = (int)units.size();
  const int ns = std::max(1, std::min(spread_branches(p), nu));
  const int ng = std::max(1, std::min(gather_branches(p, R), nu));
  ensure_pipe(p, ns, ng, nu);
  for (int b = 1; b < ng; ++b)
    if (!p->outx[b - 1]) {
      AFS_CUDA(cudaMalloc(&p->outx[b - 1], sizeof(double) * p->Nt * p->max_rhs));
      p->device_bytes += sizeof(double) * p->Nt * p->max_rhs;
    }

  const bool det = p->deterministic && p->det_limbs;
  if (det) det_prepare(p, alpha, lda, R, s);   // 2^S from max|alpha|, before the fork
  // fork: every stream starts after the caller's work (alpha, out)
  AFS_CUDA(cudaEventRecord(p->pipe_fork, s));
  for (int b = 0; b < ns; ++b) AFS_CUDA(cudaStreamWaitEvent(p->pipe_s[b], p->pipe_fork, 0));
  for (int b = 0; b + 1 < ng; ++b) AFS_CUDA(cudaStreamWaitEvent(p->pipe_g[b], p->pipe_fork, 0));
  AFS_CUDA(cudaMemset2DAsync(out, sizeof(double) * ldo, 0, sizeof(double) * p->Nt, R, s));
  for (int b = 1; b < ng; ++b)
    AFS_CUDA(cudaMemsetAsync(p->outx[b - 1], 0, sizeof(double) * p->Nt * R, p->pipe_g[b - 1]));

  // spread + spectral of unit i on spread stream i % ns (each window clears its own grid)
  for (int i = 0; i < nu; ++i) {
    const cudaStream_t ss = p->pipe_s[i % ns];
    for (int l : units[i].wins) {
      const Window& w = p->win[l];
      if (det)
        det_window_begin(p, w, R, ss);   // the limbs accumulate; finalize writes the grid
      else
        AFS_CUDA(cudaMemset2DAsync(p->grids + w.grid_off, sizeof(double) * p->grid_total, 0,
                                   sizeof(double) * w.cells, R, ss));
    }
    spread_unit(p, units[i].wins, units[i].one_d, alpha, lda, R, ss);
    if (det)
      for (int l : units[i].wins) det_window_finalize(p, p->win[l], R, ss);
    spectral_windows(p, R, ss, units[i].wins);
    AFS_CUDA(cudaEventRecord(p->unit_ev[i], ss));
  }
  // gather of unit i on gather stream i % ng, once its spectral stage is done; each stream
  // adds its units in window order into its own accumulator
  for (int i = 0; i < nu; ++i) {
    const int b = i % ng;
    const cudaStream_t gs = b ? p->pipe_g[b - 1] : s;
    double* o = b ? p->outx[b - 1] : out;
    const int64_t lo = b ? p->Nt : ldo;
    AFS_CUDA(cudaStreamWaitEvent(gs, p->unit_ev[i], 0));
    gather_unit(p, units[i].wins, units[i].one_d, o, lo, R, gs);
  }
  // join
  for (int b = 0; b < ns; ++b) {
    AFS_CUDA(cudaEventRecord(p->pipe_join[b], p->pipe_s[b]));
    AFS_CUDA(cudaStreamWaitEvent(s, p->pipe_join[b], 0));
  }
  for (int b = 1; b < ng; ++b) {
    AFS_CUDA(cudaEventRecord(p->pipe_join[afs_plan::kMaxBranches + b - 1], p->pipe_g[b - 1]));
    AFS_CUDA(cudaStreamWaitEvent(s, p->pipe_join[afs_plan::kMaxBranches + b - 1], 0));
  }
  if (ng > 1) {
    const int64_t tot = p->Nt * R;
    const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
    k_add_into<<<blocks, 256, 0, s>>>(out, ldo, p->outx[0], p->outx[1], p->outx[2], ng - 1, p->Nt,
                                      p->Nt, R);
  }
  AFS_CUDA(cudaGetLastError());
}

}  // namespace afs
