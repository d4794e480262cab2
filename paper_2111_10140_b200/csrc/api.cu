// C ABI entry points (include/anovafs.h): plan construction, apply, CG.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "afs_internal.cuh"

#include <cstdlib>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu --nvtx (no-ops untraced)
#include "geometry.cuh"

namespace afs {

static thread_local std::string g_last_error;

void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation)
    throw Error(AFS_ERR_NOMEM, std::string("device allocation failed: ") + what);
  throw Error(AFS_ERR_CUDA, std::string(cudaGetErrorString(e)) + " in " + what);
}

template <typename F>
static int guarded(F&& f) {
  try {
    f();
    return AFS_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return AFS_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return AFS_ERR_CUDA;
  }
}

void make_twiddles(afs_plan* p) {
  std::vector<double2> tw(p->n);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int k = 0; k < p->n; ++k) {
    const long double a = two_pi * (long double)k / (long double)p->n;
    tw[k] = make_double2((double)cosl(a), (double)-sinl(a));
  }
  AFS_CUDA(cudaMalloc(&p->twiddle, sizeof(double2) * p->n));
  AFS_CUDA(cudaMemcpy(p->twiddle, tw.data(), sizeof(double2) * p->n, cudaMemcpyHostToDevice));
  p->device_bytes += sizeof(double2) * p->n;
}

void apply_stages(afs_plan* p, const double* alpha, int64_t lda, double* out, int64_t ldo,
                  int R, cudaStream_t s) {
  if (pipeline_applies(p)) {   // per-window pipeline (pipeline.cu)
    apply_pipeline(p, alpha, lda, out, ldo, R, s);
    return;
  }
  spread_all(p, alpha, lda, R, s);
  spectral_all(p, R, s);
  gather_all(p, out, ldo, R, s);
}

// The ~2P + 4P launches of one apply are replayed from a CUDA graph keyed by the call's
// pointers/shape.  A key is captured on its second use (the first, eager call performs any
// one-time cudaFuncSetAttribute), so CG iterations and benchmark loops run graph launches.
static bool apply_graph(afs_plan* p, const double* alpha, int64_t lda, double* out, int64_t ldo,
                        int R, cudaStream_t s) {
  if (!p->use_graphs || s == nullptr) return false;   // legacy stream cannot be captured
  GraphEntry* hit = nullptr;
  for (GraphEntry& g : p->graphs)
    if (g.alpha == alpha && g.lda == lda && g.out == out && g.ldo == ldo && g.R == R) hit = &g;
  if (hit && hit->exec) {
    AFS_CUDA(cudaGraphLaunch(hit->exec, s));
    return true;
  }
  if (!hit) {
    if (p->graphs.size() >= 8) {
      if (p->graphs.front().exec) cudaGraphExecDestroy(p->graphs.front().exec);
      p->graphs.erase(p->graphs.begin());
    }
    p->graphs.push_back(GraphEntry{alpha, lda, out, ldo, R, nullptr});
    return false;   // first use: eager
  }
  cudaGraph_t graph = nullptr;
  AFS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    apply_stages(p, alpha, lda, out, ldo, R, s);
  } catch (...) {
    cudaStreamEndCapture(s, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  AFS_CUDA(cudaStreamEndCapture(s, &graph));
  {   // the exact kernel count of one apply (afs_plan_info.kernel_launches_per_apply)
    size_t nn = 0;
    AFS_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) AFS_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
    int kernels = 0;
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      AFS_CUDA(cudaGraphNodeGetType(nd, &t));
      if (t == cudaGraphNodeTypeKernel) ++kernels;
    }
    p->launches_per_apply = kernels;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  AFS_CUDA(e);
  hit->exec = exec;
  AFS_CUDA(cudaGraphLaunch(exec, s));
  return true;
}

void apply_impl(afs_plan* p, const double* alpha, int64_t lda, double* out, int64_t ldo, int R,
                cudaStream_t s) {
  if (!p->profiling) {
    // run on the plan's own (capturable) stream, ordered after / before the caller's stream
    if (!p->istream) {
      AFS_CUDA(cudaStreamCreateWithFlags(&p->istream, cudaStreamNonBlocking));
      AFS_CUDA(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
      AFS_CUDA(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
    }
    AFS_CUDA(cudaEventRecord(p->ev_in, s));
    AFS_CUDA(cudaStreamWaitEvent(p->istream, p->ev_in, 0));
    if (!apply_graph(p, alpha, lda, out, ldo, R, p->istream))
      apply_stages(p, alpha, lda, out, ldo, R, p->istream);
    AFS_CUDA(cudaEventRecord(p->ev_out, p->istream));
    AFS_CUDA(cudaStreamWaitEvent(s, p->ev_out, 0));
    return;
  }
  for (int i = 0; i < 4; ++i)
    if (!p->ev[i]) AFS_CUDA(cudaEventCreate(&p->ev[i]));
  if (p->wev_spread.empty()) {
    p->wev_spread.resize(p->P + 1);
    p->wev_gather.resize(p->P + 1);
    for (int i = 0; i <= p->P; ++i) {
      AFS_CUDA(cudaEventCreate(&p->wev_spread[i]));
      AFS_CUDA(cudaEventCreate(&p->wev_gather[i]));
    }
    p->win_ms_spread.assign(p->P, 0.0);
    p->win_ms_gather.assign(p->P, 0.0);
  }
  AFS_CUDA(cudaEventRecord(p->ev[0], s));
  spread_all(p, alpha, lda, R, s);
  AFS_CUDA(cudaEventRecord(p->ev[1], s));
  spectral_all(p, R, s);
  AFS_CUDA(cudaEventRecord(p->ev[2], s));
  gather_all(p, out, ldo, R, s);
  AFS_CUDA(cudaEventRecord(p->ev[3], s));
  AFS_CUDA(cudaEventSynchronize(p->ev[3]));
  for (int i = 0; i < 3; ++i) {
    float ms = 0.f;
    AFS_CUDA(cudaEventElapsedTime(&ms, p->ev[i], p->ev[i + 1]));
    p->stage_ms[i] += ms;
  }
  if (p->window_eval == 0) {
    for (int l = 0; l < p->P; ++l) {
      float ms = 0.f;
      AFS_CUDA(cudaEventElapsedTime(&ms, p->wev_spread[l], p->wev_spread[l + 1]));
      p->win_ms_spread[l] += ms;
      AFS_CUDA(cudaEventElapsedTime(&ms, p->wev_gather[l], p->wev_gather[l + 1]));
      p->win_ms_gather[l] += ms;
    }
  }
  p->profiled_applies += 1;
}

static void free_plan(afs_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  for (afs_plan* c : p->clones) free_plan(c);
  p->clones.clear();
  if (!p->parent) {   // immutable parts: owned by the primary plan only
    cudaFree(p->d_win);
    cudaFree(p->src);
    cudaFree(p->tgt);
    cudaFree(p->mult);
    cudaFree(p->twiddle);
  }
  if (p->grids_owned) cudaFree(p->grids);
  if (p->spec_owned) cudaFree(p->spec);
  cudaFree(p->det_limbs);
  cudaFree(p->det_aux);
  cudaFree(p->scratch_a);
  cudaFree(p->scratch_b);
  cudaFree(p->cg.r);
  cudaFree(p->cg.p);
  cudaFree(p->cg.ap);
  cudaFree(p->cg.x);
  cudaFree(p->cg.partial);
  cudaFree(p->cg.scalars);
  for (int i = 0; i < 4; ++i)
    if (p->ev[i]) cudaEventDestroy(p->ev[i]);
  for (afs::GraphEntry& g : p->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (p->cg.graph.exec) cudaGraphExecDestroy(p->cg.graph.exec);
  for (cudaEvent_t e : p->wev_spread) cudaEventDestroy(e);
  for (cudaEvent_t e : p->wev_gather) cudaEventDestroy(e);
  if (p->istream) cudaStreamDestroy(p->istream);
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->ev_out) cudaEventDestroy(p->ev_out);
  for (int b = 0; b < afs_plan::kMaxBranches - 1; ++b) {
    if (p->aux[b]) cudaStreamDestroy(p->aux[b]);
    if (p->ev_join[b]) cudaEventDestroy(p->ev_join[b]);
    cudaFree(p->outx[b]);
  }
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  for (cudaStream_t st : p->pipe_s)
    if (st) cudaStreamDestroy(st);
  for (cudaStream_t st : p->pipe_g)
    if (st) cudaStreamDestroy(st);
  if (p->pipe_fork) cudaEventDestroy(p->pipe_fork);
  for (cudaEvent_t e : p->pipe_join)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : p->unit_ev) cudaEventDestroy(e);
  if (p->cg.host_scalars) cudaFreeHost(p->cg.host_scalars);
  if (!p->parent) {
    for (SortedSide* s : p->src_side)
      if (s) { free_sorted_side(s); delete s; }
    for (SortedSide* s : p->tgt_side)
      if (s) { free_sorted_side(s); delete s; }
    delete p->poly;
  }
  delete p;
}

void refresh_det_windows(afs_plan* p) {
  for (Window& w : p->win) {
    w.det_limbs = p->deterministic ? p->det_limbs : nullptr;
    w.det_stride = p->grid_total * p->max_rhs;
    w.det_scale = p->det_aux ? p->det_aux + 1 : nullptr;
    w.det_base = p->grids;
    w.det_unit = std::ldexp(1.0, p->det_bits);
    w.det_inv_unit = std::ldexp(1.0, -p->det_bits);
    w.det_boost = std::ldexp(1.0, (p->det_dmax - w.d) * p->det_peak_exp);
  }
  for (GraphEntry& g : p->graphs)   // captured graphs hold the old window parameters
    if (g.exec) cudaGraphExecDestroy(g.exec);
  p->graphs.clear();
  if (p->cg.graph.exec) cudaGraphExecDestroy(p->cg.graph.exec);   // so does the CG solve graph
  p->cg.graph = CgGraph{};
}

// A workspace clone for a concurrent afs_apply: shares every immutable part of the plan,
// owns the mutable ones (grids, spectral scratch, limbs, streams, captured graphs).
static afs_plan* make_clone(afs_plan* p) {
  afs_plan* c = new afs_plan();
  try {
    c->parent = p;
    c->device = p->device;
    c->P = p->P;
    c->dtot = p->dtot;
    c->Ns = p->Ns;
    c->Nt = p->Nt;
    c->has_targets = p->has_targets;
    c->M = p->M; c->m = p->m; c->n = p->n; c->H = p->H;
    c->b = p->b;
    c->max_rhs = p->max_rhs;
    c->win = p->win;
    c->d_win = p->d_win;
    c->src = p->src;
    c->tgt = p->tgt;
    c->mult = p->mult;
    c->twiddle = p->twiddle;
    c->grid_total = p->grid_total;
    c->spec_total = p->spec_total;
    c->scratch_a_len = p->scratch_a_len;
    c->scratch_b_len = p->scratch_b_len;
    c->launches_per_apply = p->launches_per_apply;
    c->window_eval = p->window_eval;
    c->kb_tab = p->kb_tab;
    c->src_side = p->src_side;
    c->tgt_side = p->tgt_side;
    c->cell1_lo = p->cell1_lo;
    c->cell1_cnt = p->cell1_cnt;
    c->poly = p->poly;
    c->use_graphs = p->use_graphs;
    c->fft_mode = p->fft_mode;
    c->stage_streams = p->stage_streams;
    c->det_log2_bound = p->det_log2_bound;
    c->det_dmax = p->det_dmax;
    c->det_peak_exp = p->det_peak_exp;
    c->deterministic = p->deterministic;
    c->det_bits = p->det_bits;
    c->mode_gen = p->mode_gen;
    AFS_CUDA(cudaMalloc(&c->grids, sizeof(double) * c->grid_total * c->max_rhs));
    if (c->scratch_a_len)
      AFS_CUDA(cudaMalloc(&c->scratch_a, sizeof(double2) * c->scratch_a_len * c->max_rhs));
    if (c->scratch_b_len)
      AFS_CUDA(cudaMalloc(&c->scratch_b, sizeof(double2) * c->scratch_b_len * c->max_rhs));
    if (c->deterministic) {
      AFS_CUDA(cudaMalloc(&c->det_limbs, sizeof(long long) * 3 * (size_t)c->grid_total * c->max_rhs));
      AFS_CUDA(cudaMalloc(&c->det_aux, 4 * sizeof(double)));
    }
    refresh_det_windows(c);
  } catch (...) {
    free_plan(c);
    throw;
  }
  return c;
}

// Drops the clones (they copy the plan's mode at creation); waits for running applies.
static void drop_clones(afs_plan* p) {
  std::unique_lock<std::mutex> lk(p->pool_mu);
  p->pool_cv.wait(lk, [p] {
    for (char b : p->clone_busy)
      if (b) return false;
    return true;
  });
  for (afs_plan* c : p->clones) free_plan(c);
  p->clones.clear();
  p->clone_busy.clear();
}

static void create_plan(const afs_plan_desc* d, afs_plan** out) {
  if (!d || !out) throw Error(AFS_ERR_VALIDATION, "null descriptor or output pointer");
  if (d->n_windows < 1 || !d->windows) throw Error(AFS_ERR_VALIDATION, "window set must not be empty");
  if (d->d_total < 1) throw Error(AFS_ERR_SHAPE, "coordinate matrix must have >= 1 column");
  if (d->n_sources < 1 || !d->sources)
    throw Error(AFS_ERR_SHAPE, "sources must form a nonempty (N, d) matrix");
  if (d->n_targets < 0 || (d->n_targets > 0 && !d->targets))
    throw Error(AFS_ERR_SHAPE, "targets pointer missing");
  if (d->bandwidth < 2 || d->bandwidth % 2)
    throw Error(AFS_ERR_VALIDATION, "bandwidth M must be even and >= 2");
  if (d->cutoff < 1 || d->cutoff > AFS_MAX_CUTOFF)
    throw Error(AFS_ERR_VALIDATION, "window cutoff m must lie in 1..8");
  if (d->grid % 2 || d->grid < 2 * d->cutoff || d->grid < d->bandwidth + 2 || d->grid > 2048)
    throw Error(AFS_ERR_VALIDATION, "oversampled grid n must be even, >= max(2m, M+2), <= 2048");
  if (d->max_rhs < 1) throw Error(AFS_ERR_VALIDATION, "max_rhs must be >= 1");

  AFS_CUDA(cudaSetDevice(d->device));
  afs_plan* p = new afs_plan();
  try {
    p->device = d->device;
    p->P = d->n_windows;
    p->dtot = d->d_total;
    p->Ns = d->n_sources;
    p->has_targets = d->n_targets > 0;
    p->Nt = p->has_targets ? d->n_targets : d->n_sources;
    p->M = d->bandwidth;
    p->m = d->cutoff;
    p->n = d->grid;
    p->H = p->M / 2 + 1;
    p->b = 3.141592653589793 * (2.0 - (double)p->M / (double)p->n);   // nfft.py:156
    p->max_rhs = d->max_rhs;

    const int K = p->M + 1;
    int64_t grid_total = 0, mult_total = 0, a_len = 0, b_len = 0;
    int launches = 2;   // memset + gather
    p->win.resize(p->P);
    for (int l = 0; l < p->P; ++l) {
      const afs_window_desc& wd = d->windows[l];
      Window& w = p->win[l];
      if (wd.dims < 1 || wd.dims > 3)
        throw Error(AFS_ERR_VALIDATION, "window size must be 1..3");
      if (!wd.multiplier) throw Error(AFS_ERR_VALIDATION, "window multiplier missing");
      if (!(wd.scale > 0.0) || !std::isfinite(wd.scale))
        throw Error(AFS_ERR_VALIDATION, "window scale must be positive and finite");
      w.d = wd.dims;
      for (int t = 0; t < 3; ++t) {
        w.feat[t] = t < wd.dims ? wd.features[t] : 0;
        w.center[t] = t < wd.dims ? wd.center[t] : 0.0;
        if (t < wd.dims && (wd.features[t] < 0 || wd.features[t] >= p->dtot))
          throw Error(AFS_ERR_VALIDATION, "window feature index out of range");
      }
      w.scale = wd.scale;
      w.eta = wd.weight;
      w.cells = 1;
      for (int t = 0; t < w.d; ++t) w.cells *= p->n;
      w.grid_off = grid_total;
      grid_total += w.cells;
      w.mult_len = p->H;
      for (int t = 1; t < w.d; ++t) w.mult_len *= K;
      w.mult_off = mult_total;
      mult_total += w.mult_len;
      // per-window spectral scratch so that windows of one dimension run in one launch
      w.scratch_a_off = a_len * d->max_rhs;
      w.scratch_b_off = b_len * d->max_rhs;
      if (w.d == 2) a_len += (int64_t)p->n * p->H;
      if (w.d == 3) {
        a_len += (int64_t)p->n * p->n * p->H;
        b_len += (int64_t)p->n * K * p->H;
      }
      launches += 1 + (w.d == 1 ? 1 : (w.d == 2 ? 3 : 5));
    }
    p->grid_total = grid_total;
    p->spec_total = mult_total;   // one pruned spectrum per window, laid out like E
    {   // deterministic-mode bound: N * (peak of the KB window)^d_max
      int dmax = 1;
      for (const Window& w : p->win) dmax = std::max(dmax, w.d);
      const double peak = std::sinh(p->b * p->m) / (3.141592653589793 * p->m);   // phi(0)
      p->det_log2_bound = std::log2((double)std::max<int64_t>(p->Ns, 1)) +
                          dmax * std::log2(std::max(peak, 1.0)) + 2.0;
      p->det_dmax = dmax;
      p->det_peak_exp = (int)std::floor(std::log2(std::max(peak, 1.0)));
    }
    p->launches_per_apply = launches;

    const size_t src_bytes = sizeof(double) * p->Ns * p->dtot;
    AFS_CUDA(cudaMalloc(&p->src, src_bytes));
    AFS_CUDA(cudaMemcpy(p->src, d->sources, src_bytes, cudaMemcpyDeviceToDevice));
    p->device_bytes += src_bytes;
    if (p->has_targets) {
      const size_t tb = sizeof(double) * p->Nt * p->dtot;
      AFS_CUDA(cudaMalloc(&p->tgt, tb));
      AFS_CUDA(cudaMemcpy(p->tgt, d->targets, tb, cudaMemcpyDeviceToDevice));
      p->device_bytes += tb;
    }
    std::vector<double> mult(mult_total);
    for (int l = 0; l < p->P; ++l)
      std::memcpy(mult.data() + p->win[l].mult_off, d->windows[l].multiplier,
                  sizeof(double) * p->win[l].mult_len);
    AFS_CUDA(cudaMalloc(&p->mult, sizeof(double) * mult_total));
    AFS_CUDA(cudaMemcpy(p->mult, mult.data(), sizeof(double) * mult_total, cudaMemcpyHostToDevice));
    AFS_CUDA(cudaMalloc(&p->d_win, sizeof(Window) * p->P));
    AFS_CUDA(cudaMemcpy(p->d_win, p->win.data(), sizeof(Window) * p->P, cudaMemcpyHostToDevice));
    AFS_CUDA(cudaMalloc(&p->grids, sizeof(double) * grid_total * p->max_rhs));
    p->device_bytes += sizeof(double) * (mult_total + grid_total * p->max_rhs) + sizeof(Window) * p->P;
    p->scratch_a_len = a_len;
    p->scratch_b_len = b_len;
    if (a_len) AFS_CUDA(cudaMalloc(&p->scratch_a, sizeof(double2) * a_len * p->max_rhs));
    if (b_len) AFS_CUDA(cudaMalloc(&p->scratch_b, sizeof(double2) * b_len * p->max_rhs));
    p->device_bytes += sizeof(double2) * (a_len + b_len) * p->max_rhs;
    make_twiddles(p);
    if (d->window_eval != 0 && d->window_eval != 1)
      throw Error(AFS_ERR_VALIDATION, "window_eval must be 0 (polynomial) or 1 (exact)");
    p->window_eval = d->window_eval;
    if (const char* e = getenv("AFS_STAGE_STREAMS"))
      p->stage_streams = std::max(1, std::min(afs_plan::kMaxBranches, atoi(e)));
    {   // test hook: AFS_SPECTRAL_GENERIC=1 selects the generic line kernel for every n
      const char* g = getenv("AFS_SPECTRAL_GENERIC");
      p->fft_mode = (g && g[0] == '1') ? 1 : 0;
    }
    if (p->window_eval == 0) {
      p->poly = new PolyTable();
      make_poly_table(p->m, p->b, p->poly);
      p->kb_tab = kb_table_id(p->M, p->n);
      p->src_side.assign(p->P, nullptr);
      p->tgt_side.assign(p->P, nullptr);
      BuildScratch sc;   // sort temporaries shared by all windows
      try {
        for (int l = 0; l < p->P; ++l) {
          const Window& w = p->win[l];
          const bool tc = tc_eligible(w.d, p->m, p->kb_tab, p->n, std::max(p->Ns, p->Nt));
          // dense 3-D windows take the tensor-core layout when padding the half-cells to groups
          // of 8 adds at most 15% nodes (tc3d.cuh); sparse ones keep the team kernels
          const bool tc3 = tc3_eligible(w.d, p->m, p->kb_tab, p->n, std::max(p->Ns, p->Nt));
          // dense 2-D windows take the sub-cell layout (sc2d.cuh) when padding the sub-cells to
          // groups of 8 adds at most 12% nodes; the others the half-cell layout (tc2d.cuh)
          const bool scw = sc_eligible(w.d, p->m, p->kb_tab, p->n, std::max(p->Ns, p->Nt));
          // 3-D windows with several right-hand sides (C4: R = 8): the team kernels spread 4
          // right-hand sides per pass and win the spread (41.7 vs 47.8 ms at N = 1e8), the
          // tensor-core kernels win the gather (48.8 vs 61.5 ms).  Their source side therefore keeps
          // the team layout and the gather gets its own tensor-core layout of the same nodes
          // (3.25 x 8 N bytes more).  AFS_DUAL3=0 keeps one layout.
          bool dual3 = tc3 && p->max_rhs >= 3;
          if (const char* e = getenv("AFS_DUAL3")) dual3 = dual3 && e[0] != '0';
          auto build = [&](const double* X, int64_t N, SortedSide* side, bool spread_side) {
            if (scw && N >= 8 && build_sorted_side_sc(p, w, X, N, side, sc, 0.12)) return;
            if (tc) return build_sorted_side_tc(p, w, X, N, side, sc);
            if (tc3 && !(dual3 && spread_side) &&
                build_sorted_side_tc3(p, w, X, N, side, sc, 0.15, spread_side && !dual3))
              return;
            build_sorted_side(p, w, X, N, side, sc);
          };
          p->src_side[l] = new SortedSide();
          build(p->src, p->Ns, p->src_side[l], true);
          // 2-D windows between the two density rules (C5's pairs: ~34 nodes per sub-cell): the sub-cell
          // gather already wins there (0.029-0.031 vs 0.033 ms), the sub-cell spread does not, so the
          // gather gets its own sub-cell layout of the sources (C5 0.818 -> 0.786 ms per matvec;
          // 20 N bytes more per window; AFS_DUAL2=0 keeps one layout)
          if (scw && !p->has_targets && !p->src_side[l]->sc) {
            const char* e = getenv("AFS_DUAL2");
            if (!(e && e[0] == '0')) {
              SortedSide* gs = new SortedSide();
              if (build_sorted_side_sc(p, w, p->src, p->Ns, gs, sc, 0.2, 24.0)) p->tgt_side[l] = gs;
              else delete gs;
            }
          }
          if (dual3 && !p->has_targets) {
            SortedSide* gs = new SortedSide();
            if (build_sorted_side_tc3(p, w, p->src, p->Ns, gs, sc, 0.15, false)) p->tgt_side[l] = gs;
            else delete gs;
          }
          if (p->has_targets) {
            p->tgt_side[l] = new SortedSide();
            build(p->tgt, p->Nt, p->tgt_side[l], false);
          }
        }
        gather_1d_cell_ranges(p);
        AFS_CUDA(cudaDeviceSynchronize());
      } catch (...) {
        sc.release();
        throw;
      }
      sc.release();
      int launches = 0;
      for (const Window& w : p->win) launches += 2 + (w.d == 1 ? 1 : (w.d == 2 ? 3 : 5));
      p->launches_per_apply = launches;
    }
    AFS_CUDA(cudaDeviceSynchronize());
  } catch (...) {
    free_plan(p);
    throw;
  }
  *out = p;
}

}  // namespace afs

extern "C" {

int afs_abi_version(void) { return AFS_ABI_VERSION; }

const char* afs_last_error(void) { return afs::g_last_error.c_str(); }

namespace {
struct NvtxRange {   // scoped NVTX range around one C-ABI call
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

int afs_plan_create(const afs_plan_desc* desc, afs_plan** plan) {
  NvtxRange r("afs_plan_create");
  return afs::guarded([&] { afs::create_plan(desc, plan); });
}

int afs_plan_destroy(afs_plan* plan) {
  return afs::guarded([&] { afs::free_plan(plan); });
}

int afs_plan_get_info(const afs_plan* plan, afs_plan_info* info) {
  return afs::guarded([&] {
    if (!plan || !info) throw afs::Error(AFS_ERR_VALIDATION, "null plan or info");
    info->device_bytes = plan->device_bytes;
    info->n_windows = plan->P;
    info->grid = plan->n;
    info->n_sources = plan->Ns;
    info->n_targets = plan->Nt;
    info->kernel_launches_per_apply = plan->launches_per_apply;
    int tcw = 0;
    for (size_t l = 0; l < plan->src_side.size(); ++l) {   // either side (a gather-only layout counts)
      const afs::SortedSide* sv = plan->src_side[l];
      const afs::SortedSide* gv = l < plan->tgt_side.size() ? plan->tgt_side[l] : nullptr;
      tcw += ((sv && sv->tc) || (gv && gv->tc)) ? 1 : 0;
    }
    info->tensor_core_windows = tcw;
  });
}

static void check_rhs(const afs_plan* plan, int32_t nrhs) {
  if (!plan) throw afs::Error(AFS_ERR_VALIDATION, "null plan");
  if (nrhs < 1 || nrhs > plan->max_rhs) throw afs::Error(AFS_ERR_SHAPE, "nrhs must lie in 1..max_rhs");
}

int afs_spread(afs_plan* plan, const double* alpha, int64_t ld_alpha, int32_t nrhs, void* stream) {
  return afs::guarded([&] {
    check_rhs(plan, nrhs);
    if (!alpha || ld_alpha < plan->Ns) throw afs::Error(AFS_ERR_SHAPE, "bad alpha");
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    if (plan->ev_out) AFS_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, plan->ev_out, 0));
    afs::spread_all(plan, alpha, ld_alpha, nrhs, (cudaStream_t)stream);
  });
}

int afs_spectral(afs_plan* plan, int32_t nrhs, void* stream) {
  return afs::guarded([&] {
    check_rhs(plan, nrhs);
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    if (plan->ev_out) AFS_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, plan->ev_out, 0));
    afs::spectral_all(plan, nrhs, (cudaStream_t)stream);
  });
}

static void ensure_spectra(afs_plan* plan) {
  if (plan->spec) return;
  const size_t bytes = sizeof(double2) * (size_t)plan->spec_total * plan->max_rhs;
  AFS_CUDA(cudaMalloc(&plan->spec, bytes));
  plan->spec_owned = true;
  plan->device_bytes += (int64_t)bytes;
}

int afs_spectral_forward(afs_plan* plan, int32_t nrhs, void* stream) {
  return afs::guarded([&] {
    check_rhs(plan, nrhs);
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    ensure_spectra(plan);
    if (plan->ev_out) AFS_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, plan->ev_out, 0));
    afs::spectral_all(plan, nrhs, (cudaStream_t)stream, 1);
  });
}

int afs_spectral_inverse(afs_plan* plan, int32_t nrhs, void* stream) {
  return afs::guarded([&] {
    check_rhs(plan, nrhs);
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    if (!plan->spec) throw afs::Error(AFS_ERR_VALIDATION, "afs_spectral_inverse before forward");
    if (plan->ev_out) AFS_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, plan->ev_out, 0));
    afs::spectral_all(plan, nrhs, (cudaStream_t)stream, 2);
  });
}

int afs_plan_spectra(afs_plan* plan, double** spectra, int64_t* doubles_per_rhs) {
  return afs::guarded([&] {
    if (!plan || !spectra || !doubles_per_rhs) throw afs::Error(AFS_ERR_VALIDATION, "null argument");
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    ensure_spectra(plan);
    *spectra = reinterpret_cast<double*>(plan->spec);
    *doubles_per_rhs = 2 * plan->spec_total;
  });
}

int afs_plan_bind_spectra(afs_plan* plan, double* buffer, int64_t capacity_doubles) {
  return afs::guarded([&] {
    if (!plan || !buffer) throw afs::Error(AFS_ERR_VALIDATION, "null plan/buffer");
    if (capacity_doubles < 2 * plan->spec_total * plan->max_rhs)
      throw afs::Error(AFS_ERR_SHAPE, "spectrum buffer smaller than doubles_per_rhs * max_rhs");
    if (reinterpret_cast<uintptr_t>(buffer) % 16 != 0)
      throw afs::Error(AFS_ERR_VALIDATION, "spectrum buffer must be 16-byte aligned");
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    if (plan->spec_owned && plan->spec) cudaFree(plan->spec);
    plan->spec = reinterpret_cast<double2*>(buffer);
    plan->spec_owned = false;
  });
}

int afs_gather(afs_plan* plan, double* out, int64_t ld_out, int32_t nrhs, void* stream) {
  return afs::guarded([&] {
    check_rhs(plan, nrhs);
    if (!out || ld_out < plan->Nt) throw afs::Error(AFS_ERR_SHAPE, "bad out");
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    if (plan->ev_out) AFS_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, plan->ev_out, 0));
    afs::gather_all(plan, out, ld_out, nrhs, (cudaStream_t)stream);
  });
}

int afs_plan_grids(afs_plan* plan, double** grids, int64_t* doubles_per_rhs) {
  return afs::guarded([&] {
    if (!plan || !grids || !doubles_per_rhs) throw afs::Error(AFS_ERR_VALIDATION, "null argument");
    *grids = plan->grids;
    *doubles_per_rhs = plan->grid_total;
  });
}

int afs_plan_bind_grids(afs_plan* plan, double* buffer, int64_t capacity_doubles) {
  return afs::guarded([&] {
    if (!plan || !buffer) throw afs::Error(AFS_ERR_VALIDATION, "null plan/buffer");
    if (capacity_doubles < plan->grid_total * plan->max_rhs)
      throw afs::Error(AFS_ERR_SHAPE, "grid buffer smaller than doubles_per_rhs * max_rhs");
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    if (plan->grids_owned) cudaFree(plan->grids);
    plan->grids = buffer;
    plan->grids_owned = false;
    afs::refresh_det_windows(plan);   // also drops captured graphs (they reference the old buffer)
  });
}


int afs_plan_set_deterministic(afs_plan* plan, int32_t enable) {
  return afs::guarded([&] {
    if (!plan) throw afs::Error(AFS_ERR_VALIDATION, "null plan");
    afs::drop_clones(plan);
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    if (enable && plan->Ns > ((int64_t)1 << 27))
      throw afs::Error(AFS_ERR_VALIDATION,
                       "deterministic mode supports at most 2^27 source nodes (limb headroom)");
    if (enable && !plan->det_limbs) {
      const size_t bytes = sizeof(long long) * 3 * (size_t)plan->grid_total * plan->max_rhs;
      AFS_CUDA(cudaMalloc(&plan->det_limbs, bytes));
      AFS_CUDA(cudaMalloc(&plan->det_aux, 4 * sizeof(double)));
      plan->device_bytes += (int64_t)bytes + 4 * (int64_t)sizeof(double);
    }
    {
      std::lock_guard<std::mutex> lk(plan->pool_mu);
      plan->det_bits = plan->Ns <= ((int64_t)1 << 23) ? 40 : 36;
      plan->deterministic = enable != 0;
      ++plan->mode_gen;   // clones made meanwhile are rebuilt at their next use
    }
    afs::refresh_det_windows(plan);
  });
}

int afs_plan_set_profiling(afs_plan* plan, int32_t enable) {
  return afs::guarded([&] {
    if (!plan) throw afs::Error(AFS_ERR_VALIDATION, "null plan");
    std::lock_guard<std::mutex> lock(plan->mu);
    std::lock_guard<std::mutex> lk(plan->pool_mu);
    plan->profiling = enable != 0;
  });
}

int afs_plan_stage_times(afs_plan* plan, double* out4, int32_t reset) {
  return afs::guarded([&] {
    if (!plan || !out4) throw afs::Error(AFS_ERR_VALIDATION, "null plan/out");
    std::lock_guard<std::mutex> lock(plan->mu);
    for (int i = 0; i < 3; ++i) out4[i] = plan->stage_ms[i];
    out4[3] = (double)plan->profiled_applies;
    if (reset) {
      for (int i = 0; i < 3; ++i) plan->stage_ms[i] = 0.0;
      plan->profiled_applies = 0;
    }
  });
}

int afs_plan_window_times(afs_plan* plan, double* spread_ms, double* gather_ms, int32_t reset) {
  return afs::guarded([&] {
    if (!plan || !spread_ms || !gather_ms) throw afs::Error(AFS_ERR_VALIDATION, "null argument");
    std::lock_guard<std::mutex> lock(plan->mu);
    for (int l = 0; l < plan->P; ++l) {
      spread_ms[l] = plan->win_ms_spread.empty() ? 0.0 : plan->win_ms_spread[l];
      gather_ms[l] = plan->win_ms_gather.empty() ? 0.0 : plan->win_ms_gather[l];
    }
    if (reset && !plan->win_ms_spread.empty()) {
      plan->win_ms_spread.assign(plan->P, 0.0);
      plan->win_ms_gather.assign(plan->P, 0.0);
    }
  });
}

int afs_apply(afs_plan* plan, const double* alpha, int64_t ld_alpha, double* out, int64_t ld_out,
              int32_t nrhs, void* stream) {
  NvtxRange r("afs_apply");
  return afs::guarded([&] {
    if (!plan) throw afs::Error(AFS_ERR_VALIDATION, "null plan");
    if (nrhs < 1 || nrhs > plan->max_rhs)
      throw afs::Error(AFS_ERR_SHAPE, "nrhs must lie in 1..max_rhs");
    if (!alpha || !out) throw afs::Error(AFS_ERR_SHAPE, "null alpha/out");
    if (ld_alpha < plan->Ns || ld_out < plan->Nt)
      throw afs::Error(AFS_ERR_SHAPE, "leading dimension smaller than vector length");
    AFS_CUDA(cudaSetDevice(plan->device));
    // the first caller runs on the plan itself; concurrent callers take (or create, up to
    // kMaxClones) a workspace clone, so applies on one plan overlap on the device
    constexpr size_t kMaxClones = 3;
    afs_plan* target = nullptr;
    size_t slot = 0;
    {
      std::unique_lock<std::mutex> lk(plan->pool_mu);
      for (;;) {
        if (!plan->primary_busy) {
          plan->primary_busy = true;
          target = plan;
          break;
        }
        if (plan->profiling) {   // per-stage timing lives on the plan: wait for it
          plan->pool_cv.wait(lk);
          continue;
        }
        for (slot = 0; slot < plan->clones.size(); ++slot)
          if (!plan->clone_busy[slot]) break;
        if (slot < plan->clones.size() && plan->clones[slot]->mode_gen != plan->mode_gen) {
          // made before a mode change (set_deterministic raced with this apply): rebuild
          afs::free_plan(plan->clones[slot]);
          plan->clones.erase(plan->clones.begin() + slot);
          plan->clone_busy.erase(plan->clone_busy.begin() + slot);
          continue;
        }
        if (slot < plan->clones.size()) {
          plan->clone_busy[slot] = 1;
          target = plan->clones[slot];
          break;
        }
        if (plan->clones.size() < kMaxClones) {
          plan->clones.push_back(nullptr);
          plan->clone_busy.push_back(1);
          slot = plan->clones.size() - 1;
          lk.unlock();
          afs_plan* c = nullptr;
          try {
            c = afs::make_clone(plan);
          } catch (...) {
            lk.lock();
            plan->clones.erase(plan->clones.begin() + slot);
            plan->clone_busy.erase(plan->clone_busy.begin() + slot);
            plan->pool_cv.notify_all();
            throw;
          }
          lk.lock();
          plan->clones[slot] = c;
          target = c;
          break;
        }
        plan->pool_cv.wait(lk);
      }
    }
    auto release = [&] {
      std::lock_guard<std::mutex> lk(plan->pool_mu);
      if (target == plan) plan->primary_busy = false;
      else plan->clone_busy[slot] = 0;
      plan->pool_cv.notify_all();
    };
    try {
      if (target == plan) {
        std::lock_guard<std::mutex> lock(plan->mu);   // vs the stage-level entry points
        afs::apply_impl(plan, alpha, ld_alpha, out, ld_out, nrhs, (cudaStream_t)stream);
      } else {
        afs::apply_impl(target, alpha, ld_alpha, out, ld_out, nrhs, (cudaStream_t)stream);
      }
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}

int afs_cg_solve(afs_plan* plan, const double* b, double* x, double beta, double tol,
                 int32_t maxiter, int32_t* iterations, double* residual, int32_t* converged,
                 void* stream) {
  NvtxRange r("afs_cg_solve");
  int it = 0, conv = 0;
  double res = 0.0;
  const int st = afs::guarded([&] {
    if (!plan || !b || !x) throw afs::Error(AFS_ERR_VALIDATION, "null plan/b/x");
    std::lock_guard<std::mutex> lock(plan->mu);
    AFS_CUDA(cudaSetDevice(plan->device));
    afs::cg_solve_impl(plan, b, x, beta, tol, maxiter, &it, &res, &conv, (cudaStream_t)stream);
  });
  if (iterations) *iterations = it;
  if (residual) *residual = res;
  if (converged) *converged = conv;
  return st;
}

int afs_cg_vec_init(const double* b, double* x, double* r, double* p, int64_t n, double beta,
                    double* ws, void* stream) {
  return afs::guarded([&] {
    if (!b || !x || !r || !p || !ws) throw afs::Error(AFS_ERR_VALIDATION, "null vector");
    if (n < 0) throw afs::Error(AFS_ERR_SHAPE, "negative vector length");
    afs::cg_vec_init(b, x, r, p, n, beta, ws, (cudaStream_t)stream);
  });
}

int afs_cg_vec_ap(double* ap, const double* p, int64_t n, double* ws, void* stream) {
  return afs::guarded([&] {
    if (!ap || !p || !ws) throw afs::Error(AFS_ERR_VALIDATION, "null vector");
    if (n < 0) throw afs::Error(AFS_ERR_SHAPE, "negative vector length");
    afs::cg_vec_ap(ap, p, n, ws, (cudaStream_t)stream);
  });
}

int afs_cg_vec_update(double* x, double* r, const double* p, const double* ap, int64_t n,
                      double* ws, void* stream) {
  return afs::guarded([&] {
    if (!x || !r || !p || !ap || !ws) throw afs::Error(AFS_ERR_VALIDATION, "null vector");
    if (n < 0) throw afs::Error(AFS_ERR_SHAPE, "negative vector length");
    afs::cg_vec_update(x, r, p, ap, n, ws, (cudaStream_t)stream);
  });
}

int afs_cg_vec_direction(double* p, const double* r, int64_t n, double* ws, void* stream) {
  return afs::guarded([&] {
    if (!p || !r || !ws) throw afs::Error(AFS_ERR_VALIDATION, "null vector");
    if (n < 0) throw afs::Error(AFS_ERR_SHAPE, "negative vector length");
    afs::cg_vec_direction(p, r, n, ws, (cudaStream_t)stream);
  });
}

}  // extern "C"
