// Spectral stage: g <- IDFT( E (.) DFT(g) ) on the real oversampled grid of
// every window, pruned to the |k_t| <= M/2 modes the multiplier E touches.
//
// This replaces, per window, the reference's
//   fftn/n^d -> keep I_M -> deconvolve -> * c_hat -> deconvolve -> zero-pad -> ifftn
// (nfft.py:248-250, fastsum.py:250, nfft.py:223-226) followed by `.real`
// (fastsum.py:256).  With real alpha the grid is real, so one real-to-half
// transform along the last axis, full complex transforms along the others and
// the symmetrised real multiplier E give exactly Re(...).
//
// Each 1-D pass is a batched line transform in shared memory: a CTA owns LPC
// lines (length n), loads them cooperatively (the contiguous index fastest
// across threads, so strided axes are read in coalesced segments), runs a
// radix-2 FFT (power-of-two n) or a direct DFT (other even n) per line, and
// writes the bins the next pass needs.  The first-axis pass is fused with the
// multiplier and the inverse transform.  All windows of the same dimension
// run in one launch per pass (blockIdx.y = window), each with its own scratch.
#include "afs_internal.cuh"

namespace afs {

constexpr int kMaxBatch = 40;

struct LinePass {
  int n, log2n;            // transform length; log2n < 0 -> direct DFT
  int64_t nlines;          // lines per window
  int64_t inner;           // line l -> (outer = l / inner, q = l % inner)
  // element address = base + outer*o_stride + q*q_stride + e*e_stride
  int64_t in_o, in_q, in_e;
  int64_t out_o, out_q, out_e;
  int in_count, out_count; // elements read / written per line
  int in_sym, out_sym;     // 0: element e <-> bin e;  1: element e <-> bin (e - M/2) mod n
  int in_real, out_real;   // real (double) rather than complex (double2) storage
  int dir;                 // -1 forward (e^{-i..}), +1 inverse (e^{+i..}), unnormalised
  int half;                // M/2
  // fused multiplier (first-axis pass): keep bins j in 0..keep_count-1 mapped with
  // keep_sym, multiply by mult[q + j*inner], then transform back with -dir.
  int has_mult;
  int keep_count, keep_sym;
  const void* in;
  void* out;
  const double* mult;
};

// per-window base offsets (elements of in/out, doubles of mult)
struct BatchOff {
  int64_t in[kMaxBatch];
  int64_t out[kMaxBatch];
  int64_t mult[kMaxBatch];
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

__global__ void __launch_bounds__(256) k_line_pass(const LinePass p, const BatchOff off,
                                                   const double2* __restrict__ twg, int lpc,
                                                   int T) {
  extern __shared__ double2 sm[];
  const int n = p.n;
  const int ls = n + 1;                           // padded line stride (bank spread)
  double2* tw = sm;                               // n
  double2* S = sm + n;                            // lpc lines
  double2* Tt = S + (size_t)lpc * ls;             // lpc lines
  const int team = threadIdx.x / T;
  const int lane = threadIdx.x - team * T;
  const int wb = blockIdx.y;
  const double* mult = p.mult + off.mult[wb];
  for (int i = threadIdx.x; i < n; i += blockDim.x) tw[i] = twg[i];
  const int64_t l0 = (int64_t)blockIdx.x * lpc;

  for (int i = threadIdx.x; i < lpc * ls; i += blockDim.x) S[i] = make_double2(0.0, 0.0);
  __syncthreads();
  // cooperative load: contiguous index fastest across threads
  {
    const int tot = lpc * p.in_count;
    const bool e_fast = p.in_e == 1;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
      const int li = e_fast ? idx / p.in_count : idx % lpc;
      const int e = e_fast ? idx - li * p.in_count : idx / lpc;
      const int64_t l = l0 + li;
      if (l >= p.nlines) continue;
      const int64_t outer = l / p.inner, q = l - outer * p.inner;
      const int64_t a = off.in[wb] + outer * p.in_o + q * p.in_q + e * p.in_e;
      S[li * ls + bin_of(e, p.in_sym, p.half, n)] =
          p.in_real ? make_double2(((const double*)p.in)[a], 0.0) : ((const double2*)p.in)[a];
    }
  }
  __syncthreads();
  double2* s = S + team * ls;
  double2* t = Tt + team * ls;
  team_transform(s, t, tw, n, p.log2n, p.dir, lane, T);

  if (p.has_mult) {
    for (int i = lane; i < n; i += T) s[i] = make_double2(0.0, 0.0);
    __syncthreads();
    const int64_t l = l0 + team;
    if (l < p.nlines) {
      const int64_t q = l % p.inner;
      for (int j = lane; j < p.keep_count; j += T) {
        const int bin = bin_of(j, p.keep_sym, p.half, n);
        const double e = mult[q + (int64_t)j * p.inner];
        const double2 v = t[bin];
        s[bin] = make_double2(v.x * e, v.y * e);
      }
    }
    __syncthreads();
    team_transform(s, t, tw, n, p.log2n, -p.dir, lane, T);
  }

  // cooperative store
  {
    const int tot = lpc * p.out_count;
    const bool e_fast = p.out_e == 1;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
      const int li = e_fast ? idx / p.out_count : idx % lpc;
      const int e = e_fast ? idx - li * p.out_count : idx / lpc;
      const int64_t l = l0 + li;
      if (l >= p.nlines) continue;
      const int64_t outer = l / p.inner, q = l - outer * p.inner;
      const int64_t a = off.out[wb] + outer * p.out_o + q * p.out_q + e * p.out_e;
      const double2 v = Tt[li * ls + bin_of(e, p.out_sym, p.half, n)];
      if (p.out_real)
        ((double*)p.out)[a] = v.x;
      else
        ((double2*)p.out)[a] = v;
    }
  }
}

static int ilog2_exact(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return ((1 << l) == n) ? l : -1;
}

static void run_pass(afs_plan* pl, LinePass p, const BatchOff& off, int nb, cudaStream_t s) {
  p.n = pl->n;
  p.log2n = ilog2_exact(pl->n);
  p.half = pl->M / 2;
  // lines per CTA: enough lines for coalesced strided access, ~64 KB of shared memory
  int lpc = 16;
  while (lpc > 1 && (size_t)lpc * 2 * (pl->n + 1) * sizeof(double2) > 64 * 1024) lpc /= 2;
  const int threads = 256;
  int T = threads / lpc;
  const int64_t blocks = (p.nlines + lpc - 1) / lpc;
  const size_t smem = sizeof(double2) * ((size_t)pl->n + 2 * (size_t)lpc * (pl->n + 1));
  if (smem > 48 * 1024)
    AFS_CUDA(cudaFuncSetAttribute(k_line_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  dim3 grid((unsigned)blocks, (unsigned)nb);
  k_line_pass<<<grid, lpc * T, smem, s>>>(p, off, pl->twiddle, lpc, T);
}

void spectral_all(afs_plan* pl, int R, cudaStream_t s) {
  const int n = pl->n, M = pl->M, H = pl->H, K = M + 1;
  const int64_t gs = pl->grid_total;
  for (int d = 1; d <= 3; ++d) {
    std::vector<int> ws;
    for (int l = 0; l < pl->P; ++l)
      if (pl->win[l].d == d) ws.push_back(l);
    for (size_t b0 = 0; b0 < ws.size(); b0 += kMaxBatch) {
      const int nb = (int)std::min<size_t>(kMaxBatch, ws.size() - b0);
      BatchOff grid_off{}, a_off{}, b_off{}, m_off{}, none{};
      for (int i = 0; i < nb; ++i) {
        const Window& w = pl->win[ws[b0 + i]];
        grid_off.in[i] = grid_off.out[i] = w.grid_off;
        a_off.in[i] = a_off.out[i] = w.scratch_a_off;
        b_off.in[i] = b_off.out[i] = w.scratch_b_off;
        m_off.mult[i] = w.mult_off;
      }
      double* g = pl->grids;
      LinePass p{};
      if (d == 1) {
        // single fused pass: real line -> keep k in 0..M/2 -> * E -> inverse -> real
        BatchOff o = grid_off;
        for (int i = 0; i < nb; ++i) o.mult[i] = m_off.mult[i];
        p.nlines = R; p.inner = 1;
        p.in_o = gs; p.in_q = 0; p.in_e = 1; p.in_count = n; p.in_real = 1;
        p.out_o = gs; p.out_q = 0; p.out_e = 1; p.out_count = n; p.out_real = 1;
        p.dir = -1; p.has_mult = 1; p.mult = pl->mult; p.keep_count = H; p.keep_sym = 0;
        p.in = g; p.out = g;
        run_pass(pl, p, o, nb, s);
        continue;
      }
      double2* A = pl->scratch_a;
      double2* B = pl->scratch_b;
      const int64_t n0 = n;
      const int64_t rows = (d == 3) ? (int64_t)n * n : (int64_t)n;   // last-axis lines per rhs
      const int64_t aper = rows * H;                                  // A per rhs
      // pass 1: real last axis -> half spectrum (k in 0..M/2):  g -> A[r][rows][H]
      BatchOff o1{};
      for (int i = 0; i < nb; ++i) { o1.in[i] = grid_off.in[i]; o1.out[i] = a_off.out[i]; }
      p = LinePass{};
      p.nlines = R * rows; p.inner = rows;
      p.in_o = gs; p.in_q = n; p.in_e = 1; p.in_count = n; p.in_real = 1;
      p.out_o = aper; p.out_q = H; p.out_e = 1; p.out_count = H;
      p.dir = -1; p.in = g; p.out = A; p.mult = pl->mult;
      run_pass(pl, p, o1, nb, s);
      double2* F = A;
      BatchOff fo = a_off;
      int64_t fq = H;   // first-axis lines per rhs (inner)
      if (d == 3) {
        // middle axis forward, keep j in 0..M:  A[r][i0][i1][k] -> B[r][i0][j1][k]
        BatchOff o2{};
        for (int i = 0; i < nb; ++i) { o2.in[i] = a_off.in[i]; o2.out[i] = b_off.out[i]; }
        p = LinePass{};
        p.nlines = R * n0 * H; p.inner = H;
        p.in_o = (int64_t)n * H; p.in_q = 1; p.in_e = H; p.in_count = n;
        p.out_o = (int64_t)K * H; p.out_q = 1; p.out_e = H; p.out_count = K; p.out_sym = 1;
        p.dir = -1; p.in = A; p.out = B; p.mult = pl->mult;
        run_pass(pl, p, o2, nb, s);
        F = B;
        fo = b_off;
        fq = (int64_t)K * H;
      }
      // fused first-axis pass: forward, keep j0 in 0..M, * E, inverse (in place)
      BatchOff o3 = fo;
      for (int i = 0; i < nb; ++i) o3.mult[i] = m_off.mult[i];
      p = LinePass{};
      p.nlines = R * fq; p.inner = fq;
      p.in_o = n0 * fq; p.in_q = 1; p.in_e = fq; p.in_count = n;
      p.out_o = n0 * fq; p.out_q = 1; p.out_e = fq; p.out_count = n;
      p.dir = -1; p.has_mult = 1; p.mult = pl->mult; p.keep_count = K; p.keep_sym = 1;
      p.in = F; p.out = F;
      run_pass(pl, p, o3, nb, s);
      if (d == 3) {
        // middle axis inverse: B[r][i0][j1][k] -> A[r][i0][i1][k]
        BatchOff o4{};
        for (int i = 0; i < nb; ++i) { o4.in[i] = b_off.in[i]; o4.out[i] = a_off.out[i]; }
        p = LinePass{};
        p.nlines = R * n0 * H; p.inner = H;
        p.in_o = (int64_t)K * H; p.in_q = 1; p.in_e = H; p.in_count = K; p.in_sym = 1;
        p.out_o = (int64_t)n * H; p.out_q = 1; p.out_e = H; p.out_count = n;
        p.dir = +1; p.in = B; p.out = A; p.mult = pl->mult;
        run_pass(pl, p, o4, nb, s);
      }
      // last axis: half spectrum -> real grid (the doubling for k>=1 is inside E)
      BatchOff o5{};
      for (int i = 0; i < nb; ++i) { o5.in[i] = a_off.in[i]; o5.out[i] = grid_off.out[i]; }
      p = LinePass{};
      p.nlines = R * rows; p.inner = rows;
      p.in_o = aper; p.in_q = H; p.in_e = 1; p.in_count = H;
      p.out_o = gs; p.out_q = n; p.out_e = 1; p.out_count = n; p.out_real = 1;
      p.dir = +1; p.in = A; p.out = g; p.mult = pl->mult;
      run_pass(pl, p, o5, nb, s);
      (void)none;
    }
  }
  AFS_CUDA(cudaGetLastError());
}

}  // namespace afs
