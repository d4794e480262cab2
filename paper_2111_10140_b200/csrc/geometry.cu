// Plan-time geometry: per-window scaled node coordinates n*x (nfft.py:170-172
// with fastsum.py:229 scaling), bin-sorted by base cell with a device radix
// sort, and cut into column runs ("chunks") for the sliding-window kernels.
#define AFS_KB_DEFINE   // this translation unit owns the KB coefficient tables (kb_tables.inc)
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cub/cub.cuh>

#include "geometry.cuh"

namespace afs {

__global__ void k_prep_nodes(const double* __restrict__ X, int64_t N, int dtot, Window w, int n,
                             double* __restrict__ nx_out, uint64_t* __restrict__ key,
                             int32_t* __restrict__ idx) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  uint64_t k = 0;
  for (int t = 0; t < w.d; ++t) {
    const double xs = scaled_coord(X[j * dtot + w.feat[t]], w.center[t], w.scale);
    const double nx = __dmul_rn((double)n, xs);             // nfft.py:170
    nx_out[t * N + j] = nx;
    long long u = (long long)floor(nx) % n;
    if (u < 0) u += n;
    k = k * (uint64_t)n + (uint64_t)u;
  }
  key[j] = k;
  idx[j] = (int32_t)j;
}

__global__ void k_permute_nodes(const double* __restrict__ nx_in, const int32_t* __restrict__ idx,
                                int64_t N, int d, double* __restrict__ nx_out,
                                int32_t* __restrict__ perm) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int32_t j = idx[i];
  perm[i] = j;
  for (int t = 0; t < d; ++t) nx_out[t * N + i] = nx_in[t * N + j];
}

// window origin of every run, so kernels can prefetch a run's grid window from its
// descriptor alone (same floor/wrap as the kernels apply to nx)
__global__ void k_chunk_cell0(Chunk* __restrict__ ch, int64_t nch, const double* __restrict__ nx_last,
                              int n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nch) return;
  const int c = (int)floor(nx_last[ch[i].begin]);
  ch[i].cell0 = c < 0 ? c + n : (c >= n ? c - n : c);
}

__global__ void k_column_counts(const uint64_t* __restrict__ key, int64_t N, uint64_t n,
                                int32_t* __restrict__ counts) {
  // keys are sorted, so a warp mostly sees one column: aggregate before the atomic
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = i < N;
  const unsigned long long col = live ? key[i] / n : ~0ULL;
  const unsigned peers = __match_any_sync(0xffffffffu, col);
  const int leader = __ffs(peers) - 1;
  if (live && (int)(threadIdx.x & 31) == leader) atomicAdd(&counts[col], __popc(peers));
}

static int chunk_cap_for(int d, int64_t N) {
  // d = 3: one 32-lane team per run; d <= 2: one warp per run, 32 nodes per lane.
  // Up to 1024 nodes per run amortise the window flushes; small windows use shorter
  // runs so that a launch still has >= ~8 warps per SM (148 SMs).
  int64_t hi = 1024;
  if (const char* e = getenv("AFS_CHUNK_CAP_MAX")) hi = std::max(64, atoi(e)) / 32 * 32;   // tuning hook
  // warps per SM the launch should fill: the 1-D kernels hold ~100 registers (24 warps
  // resident), the 2-D/3-D ones ~230 (8 warps)
  int per_sm = d == 1 ? 24 : 8;
  if (const char* e = getenv("AFS_CHUNK_WARPS_1D")) if (d == 1) per_sm = std::max(1, atoi(e));
  int64_t cap = N / (148 * per_sm);
  cap = (cap + 31) / 32 * 32;
  return (int)std::max<int64_t>(64, std::min<int64_t>(hi, cap));
}

void BuildScratch::reserve(int64_t N, int d) {
  N = std::max<int64_t>(N, 1);
  if (N <= cap && d <= 3) return;
  cudaFree(nx_tmp); cudaFree(key_a); cudaFree(key_b); cudaFree(idx_a); cudaFree(idx_b);
  nx_tmp = nullptr; key_a = key_b = nullptr; idx_a = idx_b = nullptr; cap = 0;
  AFS_CUDA(cudaMalloc(&nx_tmp, sizeof(double) * 3 * N));
  AFS_CUDA(cudaMalloc(&key_a, sizeof(uint64_t) * N));
  AFS_CUDA(cudaMalloc(&key_b, sizeof(uint64_t) * N));
  AFS_CUDA(cudaMalloc(&idx_a, sizeof(int32_t) * N));
  AFS_CUDA(cudaMalloc(&idx_b, sizeof(int32_t) * N));
  cap = N;
}

void BuildScratch::reserve_counts(int64_t n) {
  if (n <= counts_cap) return;
  cudaFree(counts); cudaFree(starts);
  counts = nullptr; starts = nullptr; counts_cap = 0;
  AFS_CUDA(cudaMalloc(&counts, sizeof(int32_t) * n));
  AFS_CUDA(cudaMalloc(&starts, sizeof(int64_t) * (2 * n + 2)));   // + 2 totals
  counts_cap = n;
}

void* BuildScratch::sort_temp(size_t bytes) {
  if (bytes > temp_bytes) {
    cudaFree(temp);
    temp = nullptr;
    temp_bytes = 0;
    AFS_CUDA(cudaMalloc(&temp, bytes));
    temp_bytes = bytes;
  }
  return temp;
}

void BuildScratch::release() {
  cudaFree(nx_tmp); cudaFree(key_a); cudaFree(key_b); cudaFree(idx_a); cudaFree(idx_b);
  cudaFree(temp); cudaFree(counts); cudaFree(starts);
  *this = BuildScratch{};
}

void build_sorted_side(afs_plan* p, const Window& w, const double* X, int64_t N, SortedSide* out,
                       BuildScratch& sc) {
  if (N >= (int64_t)INT32_MAX) throw Error(AFS_ERR_VALIDATION, "at most 2^31-1 nodes per plan");
  const int d = w.d, n = p->n;
  const cudaStream_t s = 0;
  int bits = 0;
  {
    long double cells = 1;
    for (int t = 0; t < d; ++t) cells *= n;
    while ((long double)(1ULL << bits) < cells && bits < 63) ++bits;
  }
  sc.reserve(N, d);
  const int64_t ncol = d == 1 ? 1 : (d == 2 ? (int64_t)n : (int64_t)n * n);
  sc.reserve_counts(ncol);
  const int th = 256;
  const int64_t bl = (N + th - 1) / th;
  k_prep_nodes<<<bl, th, 0, s>>>(X, N, p->dtot, w, n, sc.nx_tmp, sc.key_a, sc.idx_a);
  AFS_CUDA(cudaGetLastError());
  size_t temp_bytes = 0;
  AFS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, sc.key_a, sc.key_b, sc.idx_a, sc.idx_b,
                                           (int)N, 0, bits > 0 ? bits : 1, s));
  void* temp = sc.sort_temp(temp_bytes);
  AFS_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, sc.key_a, sc.key_b, sc.idx_a, sc.idx_b,
                                           (int)N, 0, bits > 0 ? bits : 1, s));
  AFS_CUDA(cudaMalloc(&out->nx, sizeof(double) * d * N));
  AFS_CUDA(cudaMalloc(&out->perm, sizeof(int32_t) * N));
  k_permute_nodes<<<bl, th, 0, s>>>(sc.nx_tmp, sc.idx_b, N, d, out->nx, out->perm);
  AFS_CUDA(cudaGetLastError());
  // column runs
  int32_t* counts = sc.counts;
  AFS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * ncol, s));
  k_column_counts<<<bl, th, 0, s>>>(sc.key_b, N, (uint64_t)n, counts);
  AFS_CUDA(cudaGetLastError());
  std::vector<int32_t> hc(ncol);
  AFS_CUDA(cudaMemcpy(hc.data(), counts, sizeof(int32_t) * ncol, cudaMemcpyDeviceToHost));
  const int cap = chunk_cap_for(d, N);
  std::vector<Chunk> ch;
  int64_t pos = 0;
  for (int64_t c = 0; c < ncol; ++c) {
    for (int32_t o = 0; o < hc[c]; o += cap)
      ch.push_back(Chunk{(int32_t)c, std::min(cap, hc[c] - o), pos + o, 0, 0});
    pos += hc[c];
  }
  out->N = N;
  out->nchunks = (int64_t)ch.size();
  out->chunk_cap = cap;
  AFS_CUDA(cudaMalloc(&out->chunks, sizeof(Chunk) * std::max<size_t>(1, ch.size())));
  AFS_CUDA(cudaMemcpy(out->chunks, ch.data(), sizeof(Chunk) * ch.size(), cudaMemcpyHostToDevice));
  if (!ch.empty()) {
    k_chunk_cell0<<<(unsigned)((ch.size() + 255) / 256), 256, 0, s>>>(
        out->chunks, (int64_t)ch.size(), out->nx + (int64_t)(d - 1) * N, n);
    AFS_CUDA(cudaGetLastError());
  }
  p->device_bytes += (int64_t)(sizeof(double) * d + sizeof(int32_t)) * N +
                     (int64_t)sizeof(Chunk) * out->nchunks;
}

// ---- tensor-core layout (2-D windows, tc2d.cuh) -------------------------------------------
// Half-cell key: per dimension 2*u + c with u = floor(nx) mod n and c = (f > 1/2) the
// reflection class the kernels apply (geometry.cuh poly_weights), last dimension fastest.
__device__ __forceinline__ uint64_t half_cell_key(const double (&nx)[2], int n) {
  uint64_t k = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const double fl = floor(nx[t]);
    long long u = (long long)fl % n;
    if (u < 0) u += n;
    const int c = (nx[t] - fl) > 0.5 ? 1 : 0;
    k = k * (uint64_t)(2 * n) + (uint64_t)(2 * u + c);
  }
  return k;
}

__global__ void k_prep_nodes_tc(const double* __restrict__ X, int64_t N, int dtot, Window w, int n,
                                double* __restrict__ nx_out, uint64_t* __restrict__ key,
                                int32_t* __restrict__ idx) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  double nx[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const double xs = scaled_coord(X[j * dtot + w.feat[t]], w.center[t], w.scale);
    nx[t] = __dmul_rn((double)n, xs);   // nfft.py:170
    nx_out[t * N + j] = nx[t];
  }
  key[j] = half_cell_key(nx, n);
  idx[j] = (int32_t)j;
}

__global__ void k_segment_counts(const uint64_t* __restrict__ key, int64_t N,
                                 int32_t* __restrict__ counts) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = i < N;
  const unsigned long long k = live ? key[i] : ~0ULL;
  const unsigned peers = __match_any_sync(0xffffffffu, k);
  const int leader = __ffs(peers) - 1;
  if (live && (int)(threadIdx.x & 31) == leader) atomicAdd(&counts[k], __popc(peers));
}

// sorted node i of segment s lands at pad_start[s] + (i - seg_start[s]); stores the
// polynomial variable per dimension and, at group starts, the group header
__global__ void k_scatter_tc(const double* __restrict__ nx_in, const int32_t* __restrict__ idx,
                             const uint64_t* __restrict__ key, const int64_t* __restrict__ seg_start,
                             const int64_t* __restrict__ pad_start, int64_t N, int64_t Npad, int n,
                             double* __restrict__ x_out, int32_t* __restrict__ perm,
                             int32_t* __restrict__ ghdr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const uint64_t s = key[i];
  const int64_t dst = pad_start[s] + (i - seg_start[s]);
  const int32_t j = idx[i];
  perm[dst] = j;
  int u[2], c[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const double nx = nx_in[t * N + j];
    const double fl = floor(nx);
    const double f = nx - fl;   // exact
    c[t] = f > 0.5 ? 1 : 0;
    long long uu = (long long)fl % n;
    u[t] = (int)(uu < 0 ? uu + n : uu);
    x_out[t * Npad + dst] = (c[t] ? __dsub_rn(1.0, f) : f) - 0.25;   // as poly_weights
  }
  if ((dst & 7) == 0) ghdr[dst >> 3] = tc_header(u[0], u[1], c[0], c[1]);
}

// padding slots: x = 0 (finite), perm -1 (no alpha, no output)
__global__ void k_pad_tc(const int32_t* __restrict__ counts, const int64_t* __restrict__ pad_start,
                         int64_t nseg, int64_t Npad, double* __restrict__ x, int32_t* __restrict__ perm) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const int c = counts[s];
  if (c == 0 || (c & 7) == 0) return;
  const int64_t b = pad_start[s];
  for (int k = c; k < ((c + 7) & ~7); ++k) {
    perm[b + k] = -1;
#pragma unroll
    for (int t = 0; t < 2; ++t) x[t * Npad + b + k] = 0.0;
  }
}

bool tc_eligible(int d, int m, int tab, int n, int64_t N) {
  // 8-offset stencils (m = 4) on a compile-time table; int32 node indices in the kernels;
  // the plan build scans a table of 4 n^2 half-cells on the host, so n is kept <= 2048
  // (the header itself would allow 14-bit cells)
  if (d != 2 || m != 4 || tab == 0 || n > 2048 || N >= (int64_t)INT32_MAX / 2) return false;
  const char* e = getenv("AFS_TC");   // A/B hook: AFS_TC=0 keeps the FMA kernels
  return !(e && e[0] == '0');
}

// counts (int32) -> int64 counts and counts rounded up to groups of 8, in place for the scans;
// the last elements are saved for the totals
__global__ void k_widen_counts(const int32_t* __restrict__ counts, int64_t nseg,
                               int64_t* __restrict__ c64, int64_t* __restrict__ p64,
                               int64_t* __restrict__ last) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nseg) return;
  const int64_t c = counts[k];
  c64[k] = c;
  p64[k] = (c + 7) & ~7LL;
  if (k == nseg - 1) {
    last[0] = c;
    last[1] = (c + 7) & ~7LL;
  }
}

// totals = last exclusive-scan entry + last element (written over the saved last elements)
__global__ void k_scan_totals(const int64_t* __restrict__ seg, const int64_t* __restrict__ pad,
                              int64_t nseg, int64_t* __restrict__ tot) {
  tot[0] = seg[nseg - 1] + tot[0];
  tot[1] = pad[nseg - 1] + tot[1];
}

void build_sorted_side_tc(afs_plan* p, const Window& w, const double* X, int64_t N, SortedSide* out,
                          BuildScratch& sc) {
  if (N >= (int64_t)INT32_MAX / 2) throw Error(AFS_ERR_VALIDATION, "at most 2^30-1 nodes per plan");
  if (w.d != 2) throw Error(AFS_ERR_VALIDATION, "tensor-core layout needs a 2-D window");
  if (p->n > (1 << 14)) throw Error(AFS_ERR_VALIDATION, "tensor-core layout needs n <= 16384");
  const int n = p->n;
  const int64_t nseg = 4LL * n * n;
  const cudaStream_t s = 0;
  int bits = 1;
  while ((1LL << bits) < nseg && bits < 63) ++bits;
  sc.reserve(N, 2);
  sc.reserve_counts(nseg);
  int32_t* counts = sc.counts;
  int64_t* starts = sc.starts;
  AFS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * nseg, s));
  const int th = 256;
  const int64_t bl = (N + th - 1) / th;
  if (N > 0) {
    k_prep_nodes_tc<<<bl, th, 0, s>>>(X, N, p->dtot, w, n, sc.nx_tmp, sc.key_a, sc.idx_a);
    AFS_CUDA(cudaGetLastError());
    size_t temp_bytes = 0;
    AFS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, sc.key_a, sc.key_b, sc.idx_a,
                                             sc.idx_b, (int)N, 0, bits, s));
    void* temp = sc.sort_temp(temp_bytes);
    AFS_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, sc.key_a, sc.key_b, sc.idx_a,
                                             sc.idx_b, (int)N, 0, bits, s));
    k_segment_counts<<<bl, th, 0, s>>>(sc.key_b, N, counts);
    AFS_CUDA(cudaGetLastError());
  }
  // half-cell starts on the device: seg_start = exclusive scan of the counts, pad_start =
  // exclusive scan of the counts rounded up to groups of 8 (4 n^2 half-cells: 16.7M at n = 2048)
  {
    const int64_t sb = (nseg + th - 1) / th;
    k_widen_counts<<<(unsigned)sb, th, 0, s>>>(counts, nseg, starts, starts + nseg, starts + 2 * nseg);
    AFS_CUDA(cudaGetLastError());
    size_t temp_bytes = 0;
    AFS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, starts, starts, (int)nseg, s));
    void* temp = sc.sort_temp(temp_bytes);
    AFS_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, starts, starts, (int)nseg, s));
    AFS_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, starts + nseg, starts + nseg, (int)nseg, s));
    k_scan_totals<<<1, 1, 0, s>>>(starts, starts + nseg, nseg, starts + 2 * nseg);
    AFS_CUDA(cudaGetLastError());
  }
  int64_t totals[2] = {0, 0};
  AFS_CUDA(cudaMemcpy(totals, starts + 2 * nseg, sizeof(totals), cudaMemcpyDeviceToHost));
  const int64_t pad = totals[1];
  const int64_t ngroups = pad / 8;
  const int64_t Npad = pad + 8 * kTcTailGroups;   // trailing empty groups (tc2d.cuh)
  AFS_CUDA(cudaMalloc(&out->nx, sizeof(double) * 2 * Npad));
  AFS_CUDA(cudaMalloc(&out->perm, sizeof(int32_t) * Npad));
  AFS_CUDA(cudaMalloc(&out->ghdr, sizeof(int32_t) * (Npad / 8)));
  AFS_CUDA(cudaMemsetAsync(out->ghdr, 0, sizeof(int32_t) * (Npad / 8), s));
  AFS_CUDA(cudaMemsetAsync(out->nx, 0, sizeof(double) * 2 * Npad, s));
  AFS_CUDA(cudaMemsetAsync(out->perm, 0xff, sizeof(int32_t) * Npad, s));   // -1: no node
  if (N > 0) {
    k_scatter_tc<<<bl, th, 0, s>>>(sc.nx_tmp, sc.idx_b, sc.key_b, starts, starts + nseg, N, Npad, n,
                                   out->nx, out->perm, out->ghdr);
    AFS_CUDA(cudaGetLastError());
    k_pad_tc<<<(unsigned)((nseg + th - 1) / th), th, 0, s>>>(counts, starts + nseg, nseg, Npad,
                                                             out->nx, out->perm);
    AFS_CUDA(cudaGetLastError());
  }
  out->N = Npad;
  out->n_real = N;
  out->ngroups = ngroups;
  out->tc = true;
  out->nchunks = 0;
  out->chunk_cap = 0;
  p->device_bytes += (int64_t)(sizeof(double) * 2 + sizeof(int32_t)) * Npad +
                     (int64_t)sizeof(int32_t) * (Npad / 8);
}

// ---- tensor-core layout for dense 3-D windows (tc3d.cuh) ------------------------------------
// Same half-cell idea as the 2-D layout, over (2n)^3 keys; segments come from a device
// run-length pass over the sorted keys (no host table of (2n)^3 counts).
__global__ void k_prep_nodes_tc3(const double* __restrict__ X, int64_t N, int dtot, Window w, int n,
                                 double* __restrict__ nx_out, uint64_t* __restrict__ key,
                                 int32_t* __restrict__ idx) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  uint64_t k = 0;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const double xs = scaled_coord(X[j * dtot + w.feat[t]], w.center[t], w.scale);
    const double nx = __dmul_rn((double)n, xs);   // nfft.py:170
    nx_out[t * N + j] = nx;
    const double fl = floor(nx);
    long long u = (long long)fl % n;
    if (u < 0) u += n;
    const int c = (nx - fl) > 0.5 ? 1 : 0;
    k = k * (uint64_t)(2 * n) + (uint64_t)(2 * u + c);
  }
  key[j] = k;
  idx[j] = (int32_t)j;
}

// run heads of the sorted keys
__global__ void k_run_heads(const uint64_t* __restrict__ key, int64_t N, int32_t* __restrict__ head) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

__global__ void k_minus1(int32_t* __restrict__ v, int64_t N) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) v[i] -= 1;
}

// each run's first node records the run's start, its last node the run's end (exclusive)
__global__ void k_run_bounds(const int32_t* __restrict__ run_id, int64_t N, int32_t* __restrict__ start,
                             int32_t* __restrict__ len) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int32_t r = run_id[i];
  if (i == 0 || run_id[i - 1] != r) start[r] = (int32_t)i;
  if (i == N - 1 || run_id[i + 1] != r) len[r] = (int32_t)(i + 1);
}

// end -> length padded to a multiple of 8
__global__ void k_run_pad(const int32_t* __restrict__ start, int32_t* __restrict__ len, int64_t nruns) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nruns) return;
  const int32_t c = len[r] - start[r];
  len[r] = (c + 7) & ~7;
}

__global__ void k_scatter_tc3(const double* __restrict__ nx_in, const int32_t* __restrict__ idx,
                              const int32_t* __restrict__ run_id, const int32_t* __restrict__ start,
                              const int64_t* __restrict__ pad_start, int64_t N, int64_t Npad, int n,
                              double* __restrict__ x_out, int32_t* __restrict__ perm,
                              uint64_t* __restrict__ ghdr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int32_t r = run_id[i];
  const int64_t dst = pad_start[r] + (i - start[r]);
  const int32_t j = idx[i];
  perm[dst] = j;
  uint64_t h = 0;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const double nx = nx_in[t * N + j];
    const double fl = floor(nx);
    const double f = nx - fl;   // exact
    const int c = f > 0.5 ? 1 : 0;
    long long uu = (long long)fl % n;
    const uint64_t u = (uint64_t)(uu < 0 ? uu + n : uu);
    x_out[t * Npad + dst] = (c ? __dsub_rn(1.0, f) : f) - 0.25;   // as poly_weights
    h |= (u << (16 * t)) | ((uint64_t)c << (48 + t));
  }
  if ((dst & 7) == 0) ghdr[dst >> 3] = h;
}

// Default for dense windows: measured on C3's 3-D windows (N = 1e7, ~250 nodes per occupied
// half-cell, one right-hand side) the tensor-core kernels take 0.79 / 0.82 ms against 0.86 /
// 0.97 ms for the team kernels; on C4's clusters with 8 right-hand sides they are 6% faster at
// N = 1e8 but slower at N = 1e7 (19.7 vs 14.6 ms: the spread flushes 512 cells x R per
// half-cell and warp).  build_sorted_side_tc3 therefore also asks for >= 64 nodes per occupied
// half-cell and right-hand side.  AFS_TC3=0/1 forces the choice (1: padding rule only).
bool tc3_eligible(int d, int m, int tab, int n, int64_t N) {
  if (d != 3 || m != 4 || tab == 0 || n > 1024 || N < 8 || N >= (int64_t)INT32_MAX / 2) return false;
  const char* e = getenv("AFS_TC");
  if (e && e[0] == '0') return false;
  const char* e3 = getenv("AFS_TC3");
  return !(e3 && e3[0] == '0');
}

bool build_sorted_side_tc3(afs_plan* p, const Window& w, const double* X, int64_t N, SortedSide* out,
                           BuildScratch& sc, double max_padding, bool for_spread) {
  const int n = p->n;
  const cudaStream_t s = 0;
  int bits = 1;
  {
    const long double keys = (long double)(2 * n) * (2 * n) * (2 * n);
    while ((long double)(1ULL << bits) < keys && bits < 63) ++bits;
  }
  sc.reserve(N, 3);
  const int th = 256;
  const int64_t bl = (N + th - 1) / th;
  k_prep_nodes_tc3<<<bl, th, 0, s>>>(X, N, p->dtot, w, n, sc.nx_tmp, sc.key_a, sc.idx_a);
  AFS_CUDA(cudaGetLastError());
  size_t temp_bytes = 0;
  AFS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, sc.key_a, sc.key_b, sc.idx_a, sc.idx_b,
                                           (int)N, 0, bits, s));
  AFS_CUDA(cub::DeviceRadixSort::SortPairs(sc.sort_temp(temp_bytes), temp_bytes, sc.key_a, sc.key_b,
                                           sc.idx_a, sc.idx_b, (int)N, 0, bits, s));
  // run ids: key_a is free now (sorted keys live in key_b); reuse it as two int32 arrays
  int32_t* head = reinterpret_cast<int32_t*>(sc.key_a);
  int32_t* run_id = head + N;
  k_run_heads<<<bl, th, 0, s>>>(sc.key_b, N, head);
  AFS_CUDA(cudaGetLastError());
  temp_bytes = 0;
  AFS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, head, run_id, (int)N, s));
  AFS_CUDA(cub::DeviceScan::InclusiveSum(sc.sort_temp(temp_bytes), temp_bytes, head, run_id, (int)N, s));
  int32_t nruns = 0;
  AFS_CUDA(cudaMemcpy(&nruns, run_id + N - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
  k_minus1<<<bl, th, 0, s>>>(run_id, N);   // the inclusive scan counts runs from 1
  AFS_CUDA(cudaGetLastError());
  int32_t *start = nullptr, *padded = nullptr;
  int64_t* pad_start = nullptr;
  auto cleanup = [&] { cudaFree(start); cudaFree(padded); cudaFree(pad_start); };
  try {
    AFS_CUDA(cudaMalloc(&start, sizeof(int32_t) * nruns));
    AFS_CUDA(cudaMalloc(&padded, sizeof(int32_t) * nruns));
    AFS_CUDA(cudaMalloc(&pad_start, sizeof(int64_t) * (nruns + 1)));
    k_run_bounds<<<bl, th, 0, s>>>(run_id, N, start, padded);
    AFS_CUDA(cudaGetLastError());
    k_run_pad<<<(unsigned)((nruns + th - 1) / th), th, 0, s>>>(start, padded, nruns);
    AFS_CUDA(cudaGetLastError());
    // pad_start = exclusive scan of padded lengths (64-bit), pad_start[nruns] = total
    AFS_CUDA(cudaMemsetAsync(pad_start, 0, sizeof(int64_t), s));
    temp_bytes = 0;
    AFS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, padded, pad_start + 1, (int)nruns, s));
    AFS_CUDA(cub::DeviceScan::InclusiveSum(sc.sort_temp(temp_bytes), temp_bytes, padded, pad_start + 1,
                                           (int)nruns, s));
    int64_t total = 0;
    AFS_CUDA(cudaMemcpy(&total, pad_start + nruns, sizeof(int64_t), cudaMemcpyDeviceToHost));
    bool dense = (double)(total - N) <= max_padding * (double)N;
    {
      const char* e3 = getenv("AFS_TC3");
      const bool forced = e3 && e3[0] == '1';
      // (the per-right-hand-side rule is about the spread's flushes; a gather-only side skips it)
      if (for_spread && !forced && (double)N < 64.0 * (double)p->max_rhs * (double)nruns) dense = false;
    }
    if (!dense) {   // sparse (or short half-cells per right-hand side): the FMA kernels win
      cleanup();
      return false;
    }
    const int64_t ngroups = total / 8;
    const int64_t Npad = total + 8 * kTcTailGroups;
    AFS_CUDA(cudaMalloc(&out->nx, sizeof(double) * 3 * Npad));
    AFS_CUDA(cudaMalloc(&out->perm, sizeof(int32_t) * Npad));
    AFS_CUDA(cudaMalloc(&out->ghdr64, sizeof(uint64_t) * (Npad / 8)));
    AFS_CUDA(cudaMemsetAsync(out->ghdr64, 0, sizeof(uint64_t) * (Npad / 8), s));
    AFS_CUDA(cudaMemsetAsync(out->nx, 0, sizeof(double) * 3 * Npad, s));
    AFS_CUDA(cudaMemsetAsync(out->perm, 0xff, sizeof(int32_t) * Npad, s));   // -1: no node
    k_scatter_tc3<<<bl, th, 0, s>>>(sc.nx_tmp, sc.idx_b, run_id, start, pad_start, N, Npad, n,
                                    out->nx, out->perm, out->ghdr64);
    AFS_CUDA(cudaGetLastError());
    out->N = Npad;
    out->n_real = N;
    out->ngroups = ngroups;
    out->tc = true;
    out->nchunks = 0;
    out->chunk_cap = 0;
    p->device_bytes += (int64_t)(sizeof(double) * 3 + sizeof(int32_t)) * Npad +
                       (int64_t)sizeof(uint64_t) * (Npad / 8);
    AFS_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  return true;
}

// ---- sub-cell layout for dense 2-D windows (sc2d.cuh) ---------------------------------------
// Key: per dimension (u * 16 + s), u = floor(nx) mod n, s = floor(16 f); segments come from a
// device run-length pass over the sorted keys, as in the 3-D layout above.
__device__ __forceinline__ void sc_split(double nx, int n, int& u, int& s, double& t) {
  const double fl = floor(nx);
  const double f = nx - fl;                     // exact
  const double f16 = f * (double)kScSub;        // exact (power of two)
  const double sf = floor(f16);
  long long uu = (long long)fl % n;
  u = (int)(uu < 0 ? uu + n : uu);
  s = (int)sf;
  t = 2.0 * (f16 - sf) - 1.0;                   // exact: the sub-interval's Chebyshev variable
}

__global__ void k_prep_nodes_sc(const double* __restrict__ X, int64_t N, int dtot, Window w, int n,
                                double* __restrict__ nx_out, uint64_t* __restrict__ key,
                                int32_t* __restrict__ idx) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  uint64_t k = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const double xs = scaled_coord(X[j * dtot + w.feat[t]], w.center[t], w.scale);
    const double nx = __dmul_rn((double)n, xs);   // nfft.py:170
    nx_out[t * N + j] = nx;
    int u, s;
    double tv;
    sc_split(nx, n, u, s, tv);
    k = k * (uint64_t)(kScSub * n) + (uint64_t)(u * kScSub + s);
  }
  key[j] = k;
  idx[j] = (int32_t)j;
}

__global__ void k_scatter_sc(const double* __restrict__ nx_in, const int32_t* __restrict__ idx,
                             const int32_t* __restrict__ run_id, const int32_t* __restrict__ start,
                             const int64_t* __restrict__ pad_start, int64_t N, int64_t Npad, int n,
                             double* __restrict__ x_out, int32_t* __restrict__ perm,
                             int32_t* __restrict__ ghdr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int32_t r = run_id[i];
  const int64_t dst = pad_start[r] + (i - start[r]);
  const int32_t j = idx[i];
  perm[dst] = j;
  int u[2], sb[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    double tv;
    sc_split(nx_in[t * N + j], n, u[t], sb[t], tv);
    x_out[t * Npad + dst] = tv;
  }
  if ((dst & 7) == 0) ghdr[dst >> 3] = sc_header(u[0], u[1], sb[0], sb[1]);
}

// every group of a run starts with a node (only a run's last group is partial), so every group
// holding nodes gets its header; padding slots keep the memset values (perm -1, t = 0)

bool sc_eligible(int d, int m, int tab, int n, int64_t N) {
  // 8-offset stencils (m = 4) on a compile-time table; 12-bit cells in the header (n <= 2048
  // keeps the all-ones header unused); int32 node indices in the kernels
  if (d != 2 || m != 4 || tab == 0 || n > 2048 || N < 8 || N >= (int64_t)INT32_MAX / 2) return false;
  const char* e = getenv("AFS_TC");
  if (e && e[0] == '0') return false;
  const char* e2 = getenv("AFS_SC");   // A/B hook: AFS_SC=0 keeps the half-cell kernels
  return !(e2 && e2[0] == '0');
}

bool build_sorted_side_sc(afs_plan* p, const Window& w, const double* X, int64_t N, SortedSide* out,
                          BuildScratch& sc, double max_padding, double min_nodes) {
  const int n = p->n;
  const cudaStream_t s = 0;
  int bits = 1;
  {
    const long double keys = (long double)(kScSub * n) * (kScSub * n);
    while ((long double)(1ULL << bits) < keys && bits < 63) ++bits;
  }
  if (const char* e = getenv("AFS_SC")) if (e[0] == '2') max_padding = 1e30;   // test hook: always
  sc.reserve(N, 2);
  const int th = 256;
  const int64_t bl = (N + th - 1) / th;
  k_prep_nodes_sc<<<bl, th, 0, s>>>(X, N, p->dtot, w, n, sc.nx_tmp, sc.key_a, sc.idx_a);
  AFS_CUDA(cudaGetLastError());
  size_t temp_bytes = 0;
  AFS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, sc.key_a, sc.key_b, sc.idx_a, sc.idx_b,
                                           (int)N, 0, bits, s));
  AFS_CUDA(cub::DeviceRadixSort::SortPairs(sc.sort_temp(temp_bytes), temp_bytes, sc.key_a, sc.key_b,
                                           sc.idx_a, sc.idx_b, (int)N, 0, bits, s));
  int32_t* head = reinterpret_cast<int32_t*>(sc.key_a);   // key_a is free: sorted keys are in key_b
  int32_t* run_id = head + N;
  k_run_heads<<<bl, th, 0, s>>>(sc.key_b, N, head);
  AFS_CUDA(cudaGetLastError());
  temp_bytes = 0;
  AFS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, head, run_id, (int)N, s));
  AFS_CUDA(cub::DeviceScan::InclusiveSum(sc.sort_temp(temp_bytes), temp_bytes, head, run_id, (int)N, s));
  int32_t nruns = 0;
  AFS_CUDA(cudaMemcpy(&nruns, run_id + N - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
  k_minus1<<<bl, th, 0, s>>>(run_id, N);   // the inclusive scan counts runs from 1
  AFS_CUDA(cudaGetLastError());
  int32_t *start = nullptr, *padded = nullptr;
  int64_t* pad_start = nullptr;
  auto cleanup = [&] { cudaFree(start); cudaFree(padded); cudaFree(pad_start); };
  try {
    AFS_CUDA(cudaMalloc(&start, sizeof(int32_t) * nruns));
    AFS_CUDA(cudaMalloc(&padded, sizeof(int32_t) * nruns));
    AFS_CUDA(cudaMalloc(&pad_start, sizeof(int64_t) * (nruns + 1)));
    k_run_bounds<<<bl, th, 0, s>>>(run_id, N, start, padded);
    AFS_CUDA(cudaGetLastError());
    k_run_pad<<<(unsigned)((nruns + th - 1) / th), th, 0, s>>>(start, padded, nruns);
    AFS_CUDA(cudaGetLastError());
    AFS_CUDA(cudaMemsetAsync(pad_start, 0, sizeof(int64_t), s));
    temp_bytes = 0;
    AFS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, padded, pad_start + 1, (int)nruns, s));
    AFS_CUDA(cub::DeviceScan::InclusiveSum(sc.sort_temp(temp_bytes), temp_bytes, padded, pad_start + 1,
                                           (int)nruns, s));
    int64_t total = 0;
    AFS_CUDA(cudaMemcpy(&total, pad_start + nruns, sizeof(int64_t), cudaMemcpyDeviceToHost));
    // dense enough: little padding and >= 64 nodes per occupied sub-cell (the spread folds and
    // flushes 64 cells per sub-cell and warp: at C5's ~34 nodes per sub-cell it takes 0.065-0.08
    // ms against 0.04 ms for the half-cell kernels; at C3's ~98 it is 25% faster)
    const bool dense = (double)(total - N) <= max_padding * (double)N &&
                       (max_padding > 1e29 || (double)N >= min_nodes * (double)nruns);
    if (getenv("AFS_VERBOSE"))
      fprintf(stderr, "[afs] sub-cell layout: N=%lld sub-cells=%d (%.1f nodes each) padding +%.1f%% -> %s\n",
              (long long)N, nruns, (double)N / (double)nruns, 100.0 * (double)(total - N) / (double)N,
              dense ? "sub-cell kernels" : "half-cell kernels");
    if (!dense) {
      cleanup();
      return false;
    }
    const int64_t ngroups = total / 8;
    const int64_t Npad = total + 8 * kTcTailGroups;
    AFS_CUDA(cudaMalloc(&out->nx, sizeof(double) * 2 * Npad));
    AFS_CUDA(cudaMalloc(&out->perm, sizeof(int32_t) * Npad));
    AFS_CUDA(cudaMalloc(&out->ghdr, sizeof(int32_t) * (Npad / 8)));
    AFS_CUDA(cudaMemsetAsync(out->ghdr, 0, sizeof(int32_t) * (Npad / 8), s));
    AFS_CUDA(cudaMemsetAsync(out->nx, 0, sizeof(double) * 2 * Npad, s));
    AFS_CUDA(cudaMemsetAsync(out->perm, 0xff, sizeof(int32_t) * Npad, s));   // -1: no node
    k_scatter_sc<<<bl, th, 0, s>>>(sc.nx_tmp, sc.idx_b, run_id, start, pad_start, N, Npad, n,
                                   out->nx, out->perm, out->ghdr);
    AFS_CUDA(cudaGetLastError());
    out->N = Npad;
    out->n_real = N;
    out->ngroups = ngroups;
    out->tc = true;
    out->sc = true;
    out->nchunks = 0;
    out->chunk_cap = 0;
    p->device_bytes += (int64_t)(sizeof(double) * 2 + sizeof(int32_t)) * Npad +
                       (int64_t)sizeof(int32_t) * (Npad / 8);
    AFS_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  return true;
}

int kb_table_id(int M, int n) {
  if (n == 2 * M) return 1;
  if (2 * n == 3 * M) return 2;
  return 0;
}

void free_sorted_side(SortedSide* s) {
  cudaFree(s->ghdr);
  cudaFree(s->ghdr64);
  cudaFree(s->nx);
  cudaFree(s->perm);
  cudaFree(s->chunks);
  *s = SortedSide{};
}

// Chebyshev interpolation of phi(f + m - 1 - i) on f in [0, 1/2] at kPolyTerms nodes,
// in extended precision, converted to monomials in x = f - 1/4 (u = 4x in [-1, 1]).
void make_poly_table(int m, double b_d, PolyTable* tab) {
  std::memset(tab, 0, sizeof(*tab));
  const int N = kPolyTerms;
  const long double PI = 3.141592653589793238462643383279502884L;
  const long double b = (long double)b_d;
  for (int i = 0; i < 2 * m; ++i) {
    long double vals[kPolyTerms], cheb[kPolyTerms];
    for (int j = 0; j < N; ++j) {
      const long double u = cosl(PI * (j + 0.5L) / N);
      const long double f = (u + 1.0L) / 4.0L;
      const long double t = f + (long double)(m - 1 - i);
      const long double z = (long double)m * m - t * t;
      const long double sq = z > 0 ? sqrtl(z) : 0.0L;
      vals[j] = sq > 0 ? sinhl(b * sq) / (PI * sq) : b / PI;
    }
    for (int k = 0; k < N; ++k) {
      long double acc = 0;
      for (int j = 0; j < N; ++j) acc += vals[j] * cosl(PI * k * (j + 0.5L) / N);
      cheb[k] = 2.0L * acc / N;
    }
    cheb[0] *= 0.5L;
    // T_k(4x) as monomials in x
    long double Tm1[kPolyTerms] = {0}, T0[kPolyTerms] = {0}, poly[kPolyTerms] = {0};
    Tm1[0] = 1.0L;           // T_0
    T0[1] = 4.0L;            // T_1 = 4x
    for (int q = 0; q < N; ++q) poly[q] += cheb[0] * Tm1[q];
    if (N > 1)
      for (int q = 0; q < N; ++q) poly[q] += cheb[1] * T0[q];
    for (int k = 2; k < N; ++k) {
      long double Tn[kPolyTerms] = {0};
      for (int q = 0; q + 1 < N; ++q) Tn[q + 1] += 8.0L * T0[q];
      for (int q = 0; q < N; ++q) Tn[q] -= Tm1[q];
      for (int q = 0; q < N; ++q) poly[q] += cheb[k] * Tn[q];
      std::memcpy(Tm1, T0, sizeof(T0));
      std::memcpy(T0, Tn, sizeof(Tn));
    }
    for (int q = 0; q < N; ++q) tab->c[i][q] = (double)poly[q];
  }
}

}  // namespace afs
