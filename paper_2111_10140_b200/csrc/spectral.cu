// Spectral stage: g <- IDFT( E (.) DFT(g) ) on the real oversampled grid of
// every window, pruned to the |k_t| <= M/2 modes the multiplier E touches.
//
// This replaces, per window, the reference's
//   fftn/n^d -> keep I_M -> deconvolve -> * c_hat -> deconvolve -> zero-pad -> ifftn
// (nfft.py:248-250, fastsum.py:250, nfft.py:223-226) followed by `.real`
// (fastsum.py:256).  With real alpha the grid is real, so one real-to-half
// transform along the last axis, full complex transforms along the others and
// the symmetrised real multiplier E give exactly Re(...) (A.5).
//
// Each 1-D pass is a batched line transform in shared memory: a team of
// threads owns one line (length n), loads it (zero-filling missing bins),
// runs a radix-2 FFT (power-of-two n) or a direct DFT (other even n), and
// writes the bins the next pass needs.  The first axis pass is fused with the
// multiplier and the inverse transform ("FFT . diag . iFFT" in one kernel).
#include "afs_internal.cuh"

namespace afs {

struct LinePass {
  int n, log2n;            // transform length; log2n < 0 -> direct DFT
  int64_t nlines;          // number of lines
  int64_t inner;           // line l -> (outer = l / inner, q = l % inner)
  // element address = outer*o_stride + q*q_stride + e*e_stride
  int64_t in_o, in_q, in_e;
  int64_t out_o, out_q, out_e;
  int in_count, out_count; // elements read / written per line
  int in_sym, out_sym;     // 0: element e <-> bin e;  1: element e <-> bin (e - M/2) mod n
  int in_real, out_real;   // real (double) rather than complex (double2) storage
  int dir;                 // -1 forward (e^{-i..}), +1 inverse (e^{+i..}), unnormalised
  int half;                // M/2
  // fused multiplier (first-axis pass): keep bins j in 0..keep_count-1 mapped with
  // keep_sym, multiply by mult[q + j*inner], then transform back with -dir.
  const double* mult;
  int keep_count, keep_sym;
  const void* in;
  void* out;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ int bin_of(int e, int sym, int half, int n) {
  if (!sym) return e;
  int k = e - half;
  return k < 0 ? k + n : k;
}

// Transform s -> t (natural order in, natural order out) for one line.
// tw: n twiddles e^{-2 pi i k/n}; dir = -1 forward, +1 inverse.
// All teams of the CTA call this together (it contains __syncthreads()).
__device__ void team_transform(const double2* s, double2* t, const double2* tw, int n, int log2n,
                               int dir, int lane, int T) {
  if (log2n >= 0) {
    for (int i = lane; i < n; i += T) {
      const int r = __brev(i) >> (32 - log2n);
      t[r] = s[i];
    }
    __syncthreads();
    for (int len = 2; len <= n; len <<= 1) {
      const int hl = len >> 1;
      const int step = n / len;
      for (int j = lane; j < (n >> 1); j += T) {
        const int grp = j / hl;
        const int pos = j - grp * hl;
        const int i0 = grp * len + pos;
        const int i1 = i0 + hl;
        double2 w = tw[pos * step];
        if (dir > 0) w.y = -w.y;
        const double2 a = t[i0];
        const double2 v = cmul(t[i1], w);
        t[i0] = make_double2(a.x + v.x, a.y + v.y);
        t[i1] = make_double2(a.x - v.x, a.y - v.y);
      }
      __syncthreads();
    }
  } else {
    for (int k = lane; k < n; k += T) {
      double re = 0.0, im = 0.0;
      int idx = 0;
      for (int l = 0; l < n; ++l) {
        double2 w = tw[idx];
        if (dir > 0) w.y = -w.y;
        const double2 x = s[l];
        re += x.x * w.x - x.y * w.y;
        im += x.x * w.y + x.y * w.x;
        idx += k;
        if (idx >= n) idx -= n;
      }
      t[k] = make_double2(re, im);
    }
    __syncthreads();
  }
}

__global__ void k_line_pass(LinePass p, const double2* __restrict__ twg, int lines_per_cta,
                            int T) {
  extern __shared__ double2 sm[];
  const int n = p.n;
  double2* tw = sm;                               // n
  const int team = threadIdx.x / T;
  const int lane = threadIdx.x - team * T;
  double2* s = sm + n + (size_t)team * 2 * n;     // n
  double2* t = s + n;                             // n
  for (int i = threadIdx.x; i < n; i += blockDim.x) tw[i] = twg[i];
  const int64_t l = (int64_t)blockIdx.x * lines_per_cta + team;
  const bool live = l < p.nlines;
  const int64_t outer = live ? l / p.inner : 0;
  const int64_t q = live ? l - outer * p.inner : 0;

  for (int i = lane; i < n; i += T) s[i] = make_double2(0.0, 0.0);
  __syncthreads();
  if (live) {
    const int64_t base = outer * p.in_o + q * p.in_q;
    for (int e = lane; e < p.in_count; e += T) {
      const int bin = bin_of(e, p.in_sym, p.half, n);
      const int64_t a = base + e * p.in_e;
      s[bin] = p.in_real ? make_double2(((const double*)p.in)[a], 0.0) : ((const double2*)p.in)[a];
    }
  }
  __syncthreads();
  team_transform(s, t, tw, n, p.log2n, p.dir, lane, T);

  if (p.mult) {
    for (int i = lane; i < n; i += T) s[i] = make_double2(0.0, 0.0);
    __syncthreads();
    if (live) {
      for (int j = lane; j < p.keep_count; j += T) {
        const int bin = bin_of(j, p.keep_sym, p.half, n);
        const double e = p.mult[q + (int64_t)j * p.inner];
        const double2 v = t[bin];
        s[bin] = make_double2(v.x * e, v.y * e);
      }
    }
    __syncthreads();
    team_transform(s, t, tw, n, p.log2n, -p.dir, lane, T);
  }

  if (live) {
    const int64_t base = outer * p.out_o + q * p.out_q;
    for (int e = lane; e < p.out_count; e += T) {
      const int bin = bin_of(e, p.out_sym, p.half, n);
      const int64_t a = base + e * p.out_e;
      if (p.out_real)
        ((double*)p.out)[a] = t[bin].x;
      else
        ((double2*)p.out)[a] = t[bin];
    }
  }
}

static int ilog2_exact(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return ((1 << l) == n) ? l : -1;
}

static void run_pass(afs_plan* pl, LinePass p, cudaStream_t s) {
  p.n = pl->n;
  p.log2n = ilog2_exact(pl->n);
  p.half = pl->M / 2;
  int T = p.log2n >= 0 ? (pl->n / 2) : pl->n;
  if (T > 128) T = 128;
  if (T < 1) T = 1;
  int lines_per_cta = 256 / T;
  if (lines_per_cta < 1) lines_per_cta = 1;
  const int64_t blocks = (p.nlines + lines_per_cta - 1) / lines_per_cta;
  const size_t smem = sizeof(double2) * (size_t)pl->n * (1 + 2 * lines_per_cta);
  if (smem > 48 * 1024)
    AFS_CUDA(cudaFuncSetAttribute(k_line_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  k_line_pass<<<(unsigned)blocks, lines_per_cta * T, smem, s>>>(p, pl->twiddle, lines_per_cta, T);
}

void spectral_all(afs_plan* pl, int R, cudaStream_t s) {
  const int n = pl->n, M = pl->M, H = pl->H, K = M + 1;
  for (const Window& w : pl->win) {
    double* g = pl->grids + w.grid_off;            // rhs r at g + r*grid_total
    const int64_t gs = pl->grid_total;
    const double* E = pl->mult + w.mult_off;
    double2* A = pl->scratch_a;
    double2* B = pl->scratch_b;
    LinePass p{};
    if (w.d == 1) {
      // single fused pass: real line -> keep k in 0..M/2 -> * E -> inverse -> real
      p.nlines = R; p.inner = 1;
      p.in_o = gs; p.in_q = 0; p.in_e = 1; p.in_count = n; p.in_real = 1;
      p.out_o = gs; p.out_q = 0; p.out_e = 1; p.out_count = n; p.out_real = 1;
      p.dir = -1; p.mult = E; p.keep_count = H; p.keep_sym = 0;
      p.in = g; p.out = g;
      run_pass(pl, p, s);
      continue;
    }
    const int64_t n0 = n;
    const int64_t rows = (w.d == 3) ? (int64_t)n * n : (int64_t)n;   // lines along last axis per rhs
    // pass 1: real last axis -> half spectrum (k in 0..M/2):  g -> A[r][rows][H]
    p = LinePass{};
    p.nlines = R * rows; p.inner = rows;
    p.in_o = gs; p.in_q = n; p.in_e = 1; p.in_count = n; p.in_real = 1;
    p.out_o = rows * H; p.out_q = H; p.out_e = 1; p.out_count = H;
    p.dir = -1; p.in = g; p.out = A;
    run_pass(pl, p, s);
    double2* F = A;      // buffer holding the first-axis lines
    int64_t fq = H;      // first-axis line count per rhs (inner)
    if (w.d == 3) {
      // pass 2: middle axis forward, keep j in 0..M:  A[r][i0][i1][k] -> B[r][i0][j1][k]
      p = LinePass{};
      p.nlines = R * n0 * H; p.inner = H;
      p.in_o = (int64_t)n * H; p.in_q = 1; p.in_e = H; p.in_count = n;
      p.out_o = (int64_t)K * H; p.out_q = 1; p.out_e = H; p.out_count = K; p.out_sym = 1;
      p.dir = -1; p.in = A; p.out = B;
      run_pass(pl, p, s);
      F = B;
      fq = (int64_t)K * H;
    }
    // fused first-axis pass: forward, keep j0 in 0..M, * E, inverse (in place)
    p = LinePass{};
    p.nlines = R * fq; p.inner = fq;
    p.in_o = n0 * fq; p.in_q = 1; p.in_e = fq; p.in_count = n;
    p.out_o = n0 * fq; p.out_q = 1; p.out_e = fq; p.out_count = n;
    p.dir = -1; p.mult = E; p.keep_count = K; p.keep_sym = 1;
    p.in = F; p.out = F;
    run_pass(pl, p, s);
    if (w.d == 3) {
      // middle axis inverse: B[r][i0][j1][k] -> A[r][i0][i1][k]
      p = LinePass{};
      p.nlines = R * n0 * H; p.inner = H;
      p.in_o = (int64_t)K * H; p.in_q = 1; p.in_e = H; p.in_count = K; p.in_sym = 1;
      p.out_o = (int64_t)n * H; p.out_q = 1; p.out_e = H; p.out_count = n;
      p.dir = +1; p.in = B; p.out = A;
      run_pass(pl, p, s);
    }
    // last axis: half spectrum -> real grid (the doubling for k>=1 is inside E)
    p = LinePass{};
    p.nlines = R * rows; p.inner = rows;
    p.in_o = rows * H; p.in_q = H; p.in_e = 1; p.in_count = H;
    p.out_o = gs; p.out_q = n; p.out_e = 1; p.out_count = n; p.out_real = 1;
    p.dir = +1; p.in = A; p.out = g;
    run_pass(pl, p, s);
  }
  AFS_CUDA(cudaGetLastError());
}

}  // namespace afs
