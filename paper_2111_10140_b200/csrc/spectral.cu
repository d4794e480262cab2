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
constexpr int kMaxLpc = 16;    // lines per CTA (power of two)
constexpr int kLoadBatch = 8;  // global loads in flight per thread in the line loads

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
  // four-step kernel only: 1 = pairs of full real lines in (last-axis forward), 2 = pairs of
  // half spectra in, full real lines out (last-axis inverse); the generic kernel ignores it
  int pack;
  // multiply stored element e of line q by mult[q + e*inner] (forward half of the split
  // spectral stage: the kept bins leave the pass already multiplied by E)
  int mult_out;
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

__device__ __forceinline__ double2 twid(const double2* tw, int idx, int dir) {
  double2 w = tw[idx];
  if (dir > 0) w.y = -w.y;
  return w;
}

// Does team_transform leave its result in t (true) or back in s (false)?
__device__ __forceinline__ bool lands_in_t(int log2n) {
  return log2n < 0 || ((((log2n & 1) + (log2n >> 1)) & 1) != 0);
}

// Transform one line s (natural order in, natural order out); the result lands in t or
// in s as lands_in_t() says, the other buffer is scratch.
// tw: n twiddles e^{-2 pi i k/n}; dir = -1 forward, +1 inverse.
// Power-of-two n: Stockham autosort (no bit reversal), one radix-2 stage when log2 n is
// odd, then radix-4 stages -- ceil(log2 n / 2) barriers instead of log2 n + 1.
// All teams of the CTA call this together (it contains __syncthreads()).
__device__ void team_transform(double2* s, double2* t, const double2* tw, int n, int log2n,
                               int dir, int lane, int T) {
  if (log2n >= 0) {
    double2* src = s;
    double2* dst = t;
    int Ns = 1;
    if (log2n & 1) {
      const int h = n >> 1;
      for (int j = lane; j < h; j += T) {
        const double2 a0 = src[j];
        const double2 a1 = src[j + h];
        dst[2 * j] = make_double2(a0.x + a1.x, a0.y + a1.y);
        dst[2 * j + 1] = make_double2(a0.x - a1.x, a0.y - a1.y);
      }
      __syncthreads();
      double2* x = src; src = dst; dst = x;
      Ns = 2;
    }
    const int q4 = n >> 2;
    for (; Ns < n; Ns <<= 2) {
      const int tstep = n / (4 * Ns);   // twiddle stride: w^{q k/(4Ns)} = tw[q k tstep]
      for (int j = lane; j < q4; j += T) {
        const int k = j & (Ns - 1);
        double2 a0 = src[j], a1 = src[j + q4], a2 = src[j + 2 * q4], a3 = src[j + 3 * q4];
        if (Ns > 1) {
          a1 = cmul(a1, twid(tw, k * tstep, dir));
          a2 = cmul(a2, twid(tw, 2 * k * tstep, dir));
          a3 = cmul(a3, twid(tw, 3 * k * tstep, dir));
        }
        // radix-4 butterfly; forward uses -i, inverse +i
        const double2 b0 = make_double2(a0.x + a2.x, a0.y + a2.y);
        const double2 b1 = make_double2(a0.x - a2.x, a0.y - a2.y);
        const double2 b2 = make_double2(a1.x + a3.x, a1.y + a3.y);
        const double2 d = make_double2(a1.x - a3.x, a1.y - a3.y);
        // b3 = (dir < 0 ? -i : +i) * d
        const double2 b3 = dir < 0 ? make_double2(d.y, -d.x) : make_double2(-d.y, d.x);
        const int o = (j - k) * 4 + k;
        dst[o] = make_double2(b0.x + b2.x, b0.y + b2.y);
        dst[o + Ns] = make_double2(b1.x + b3.x, b1.y + b3.y);
        dst[o + 2 * Ns] = make_double2(b0.x - b2.x, b0.y - b2.y);
        dst[o + 3 * Ns] = make_double2(b1.x - b3.x, b1.y - b3.y);
      }
      __syncthreads();
      double2* x = src; src = dst; dst = x;
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

  // per-line element bases, computed once (one 64-bit division per line, not per element)
  __shared__ int64_t s_inb[kMaxLpc], s_outb[kMaxLpc], s_q[kMaxLpc];
  if (threadIdx.x < lpc) {
    const int64_t l = l0 + threadIdx.x;
    const int64_t outer = l / p.inner, q = l - outer * p.inner;
    const bool ok = l < p.nlines;
    s_inb[threadIdx.x] = ok ? off.in[wb] + outer * p.in_o + q * p.in_q : -1;
    s_outb[threadIdx.x] = ok ? off.out[wb] + outer * p.out_o + q * p.out_q : -1;
    s_q[threadIdx.x] = q;
  }
  for (int i = threadIdx.x; i < lpc * ls; i += blockDim.x) S[i] = make_double2(0.0, 0.0);
  __syncthreads();
  const int lg_lpc = __ffs(lpc) - 1;   // lpc is a power of two
  // cooperative load: contiguous index fastest across threads.  idx -> (line, element) by
  // shift/mask, or by an fp32 reciprocal that is exact here: (idx+0.5)/count < lpc <= 16
  // carries < 2e-6 rounding error while its fraction stays >= 0.5/count away from an
  // integer (count < 2.5e5).
  {
    const int cnt = p.in_count;
    const int tot = lpc * cnt;
    const bool e_fast = p.in_e == 1;
    const float inv = 1.0f / (float)cnt;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
      const int li = e_fast ? (int)(((float)idx + 0.5f) * inv) : (idx & (lpc - 1));
      const int e = e_fast ? idx - li * cnt : (idx >> lg_lpc);
      const int64_t base = s_inb[li];
      if (base < 0) continue;
      const int64_t a = base + e * p.in_e;
      S[li * ls + bin_of(e, p.in_sym, p.half, n)] =
          p.in_real ? make_double2(((const double*)p.in)[a], 0.0) : ((const double2*)p.in)[a];
    }
  }
  __syncthreads();
  const bool swap = lands_in_t(p.log2n);
  double2* R = swap ? Tt : S;                     // buffer holding the result
  team_transform(S + team * ls, Tt + team * ls, tw, n, p.log2n, p.dir, lane, T);

  if (p.has_mult) {
    double2* O = swap ? S : Tt;
    double2* r = R + team * ls;
    double2* o = O + team * ls;
    for (int i = lane; i < n; i += T) o[i] = make_double2(0.0, 0.0);
    __syncthreads();
    if (s_inb[team] >= 0) {
      const int64_t q = s_q[team];
      for (int j = lane; j < p.keep_count; j += T) {
        const int bin = bin_of(j, p.keep_sym, p.half, n);
        const double e = mult[q + (int64_t)j * p.inner];
        const double2 v = r[bin];
        o[bin] = make_double2(v.x * e, v.y * e);
      }
    }
    __syncthreads();
    team_transform(o, r, tw, n, p.log2n, -p.dir, lane, T);
    R = swap ? R : O;
  }

  // cooperative store
  {
    const int cnt = p.out_count;
    const int tot = lpc * cnt;
    const bool e_fast = p.out_e == 1;
    const float inv = 1.0f / (float)cnt;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
      const int li = e_fast ? (int)(((float)idx + 0.5f) * inv) : (idx & (lpc - 1));
      const int e = e_fast ? idx - li * cnt : (idx >> lg_lpc);
      const int64_t base = s_outb[li];
      if (base < 0) continue;
      const int64_t a = base + e * p.out_e;
      double2 v = R[li * ls + bin_of(e, p.out_sym, p.half, n)];
      if (p.mult_out) {
        const double m = mult[s_q[li] + (int64_t)e * p.inner];
        v = make_double2(v.x * m, v.y * m);
      }
      if (p.out_real)
        ((double*)p.out)[a] = v.x;
      else
        ((double2*)p.out)[a] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Four-step line transform for n = N1*N2 (powers of two, 16 <= n <= 1024).
//
//   X[k1 + N1 k2] = sum_t w_N2^{t k2} . w_n^{t k1} . sum_i x[t + N2 i] w_N1^{i k1}
//
// Step A: thread t (< N2) takes column t (x[t + N2 i], i < N1), does the N1-point DFT in
//         registers, applies w_n^{t k1} and writes the column back in place.
// Step B: thread k1 (< N1) takes row k1, does the N2-point DFT in registers -> the bins
//         k1 + N1 k2.  The fused first-axis pass multiplies them by E right there, runs the
//         inverse N2-point DFT (rows and columns swap roles for the inverse four-step),
//         applies w_n^{+k1 k1'} and writes the transposed row; step C (thread k1' < N2)
//         finishes with the inverse N1-point DFT.
// Rows are padded to N2+1 (resp. N1+1) slots so columns, rows and transposes are all
// bank-conflict-free; each thread owns at most one column/row per step (T >= max(N1,N2)).
// ---------------------------------------------------------------------------------------

template <int R>
__device__ __forceinline__ constexpr int brev_ct(int i) {
  return R <= 1 ? 0 : (brev_ct<(R > 1 ? R / 2 : 1)>(i >> 1) | ((i & 1) * (R / 2)));
}

// In-register R-point DFT (radix-2 DIT, bit-reversed input order resolved at compile time).
// w[p] = e^{-2 pi i p/R} for p < R/2; inv conjugates (unnormalised inverse).
template <int R>
__device__ __forceinline__ void dft_reg(double2 (&v)[R], const double2 (&w)[R / 2], bool inv) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int r = brev_ct<R>(i);
    if (r > i) { const double2 x = v[i]; v[i] = v[r]; v[r] = x; }
  }
  constexpr int LOG2R = R <= 1 ? 0 : R <= 2 ? 1 : R <= 4 ? 2 : R <= 8 ? 3 : R <= 16 ? 4 : 5;
#pragma unroll
  for (int st = 0; st < LOG2R; ++st) {
    const int half = 1 << st;
    const int len = half << 1;
#pragma unroll
    for (int bf = 0; bf < R / 2; ++bf) {
      {
        const int g = (bf / half) * len;
        const int q = bf % half;
        const int e = q * (R / len);
        double2 b = v[g + q + half];
        if (e == 0) {
        } else if (4 * e == R) {   // w = -i (forward) / +i (inverse)
          b = inv ? make_double2(-b.y, b.x) : make_double2(b.y, -b.x);
        } else {
          double2 ww = w[e];
          if (inv) ww.y = -ww.y;
          b = cmul(b, ww);
        }
        const double2 a = v[g + q];
        v[g + q] = make_double2(a.x + b.x, a.y + b.y);
        v[g + q + half] = make_double2(a.x - b.x, a.y - b.y);
      }
    }
  }
}

// blocks per SM (register cap): 6 for n <= 128 (no spills; C2 spectral 0.132 -> 0.114 ms),
// 4 for n = 256 (a cap of 6 spills and is slower), 2 from n = 512
template <int N1, int N2>
constexpr int line4s_min_blocks() { return N1 * N2 >= 512 ? 2 : (N1 * N2 >= 256 ? 4 : 6); }

template <int N1, int N2>
__global__ void __launch_bounds__(128, line4s_min_blocks<N1, N2>()) k_line_pass_4s(const LinePass p, const BatchOff off,
                                                      const double2* __restrict__ twg, int lpc,
                                                      int T) {
  constexpr int n = N1 * N2;
  constexpr int NM = N1 > N2 ? N1 : N2;
  constexpr int ls = n + NM + 1;                  // line stride (odd: lines spread on banks)
  extern __shared__ double2 sm[];
  double2* twA = sm;                              // [k1][t]   = w^{t k1}
  double2* twB = sm + n;                          // [k1'][k1] = w^{k1 k1'}
  double2* S = sm + 2 * n;                        // lpc lines
  // memory lines per CTA: lpc, or 2*lpc when pairs of real lines share one complex line
  __shared__ int64_t s_inb[2 * kMaxLpc], s_outb[2 * kMaxLpc], s_q[2 * kMaxLpc];
  const int team = threadIdx.x / T;
  const int lane = threadIdx.x - team * T;
  const int wb = blockIdx.y;
  const double* mult = p.mult + off.mult[wb];
  const int pack = p.pack;
  const int rl = pack ? 2 * lpc : lpc;
  const int64_t l0 = (int64_t)blockIdx.x * rl;
  constexpr int LGN = (n >= 1024) ? 10 : (n >= 512) ? 9 : (n >= 256) ? 8 : (n >= 128) ? 7
                    : (n >= 64) ? 6 : (n >= 32) ? 5 : 4;
  // padded natural layout (load side) and the step-B output layout of bin k
  auto pin = [](int j) { return (j / N2) * (N2 + 1) + (j % N2); };
  auto pnf = [](int k) { return (k % N1) * (N2 + 1) + k / N1; };

  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    twA[i] = twg[((i / N2) * (i % N2)) % n];
    twB[i] = twg[((i / N1) * (i % N1)) % n];
  }
  double2 w1[N1 / 2], w2[N2 / 2];
#pragma unroll
  for (int q = 0; q < N1 / 2; ++q) w1[q] = twg[q * N2];
#pragma unroll
  for (int q = 0; q < N2 / 2; ++q) w2[q] = twg[q * N1];
  if (threadIdx.x < rl) {
    const int64_t l = l0 + threadIdx.x;
    const int64_t outer = l / p.inner, q = l - outer * p.inner;
    const bool ok = l < p.nlines;
    s_inb[threadIdx.x] = ok ? off.in[wb] + outer * p.in_o + q * p.in_q : -1;
    s_outb[threadIdx.x] = ok ? off.out[wb] + outer * p.out_o + q * p.out_q : -1;
    s_q[threadIdx.x] = q;
  }
  if (p.in_count < n)   // bins the input does not cover start at zero
    for (int i = threadIdx.x; i < lpc * ls; i += blockDim.x) S[i] = make_double2(0.0, 0.0);
  __syncthreads();
  const int lg_lpc = __ffs(lpc) - 1;
  const int nthr = blockDim.x;
  if (pack == 1) {
    // real lines 2c, 2c+1 (contiguous, full length n) -> real / imaginary part of line c
    const int tot = rl * n;
    for (int i0 = threadIdx.x; i0 < tot; i0 += kLoadBatch * nthr) {
      double val[kLoadBatch];
      int pos[kLoadBatch];
#pragma unroll
      for (int u = 0; u < kLoadBatch; ++u) {
        const int idx = i0 + u * nthr;
        const int li = idx >> LGN, e = idx & (n - 1);
        const int64_t base = idx < tot ? s_inb[li] : -1;
        pos[u] = idx < tot ? 2 * ((li >> 1) * ls + pin(e)) + (li & 1) : -1;
        val[u] = base >= 0 ? ((const double*)p.in)[base + e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kLoadBatch; ++u)
        if (pos[u] >= 0) ((double*)S)[pos[u]] = val[u];
    }
  } else if (pack == 2) {
    // half spectra C (line 2c), D (line 2c+1), bins 0..cnt-1 with 2(cnt-1) < n:
    // Z = herm(C) + i herm(D), herm(C)[k] = C[k]/2, herm(C)[-k] = conj(C[k])/2, k >= 1
    const int cnt = p.in_count;
    const int tot = lpc * cnt;
    const float inv = 1.0f / (float)cnt;
    constexpr int U = kLoadBatch / 2;
    for (int i0 = threadIdx.x; i0 < tot; i0 += U * nthr) {
      double2 cv[U], dv[U];
      int c_[U], e_[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = i0 + u * nthr;
        const int c = (int)(((float)idx + 0.5f) * inv);
        const int e = idx - c * cnt;
        const bool ok = idx < tot;
        const int64_t bc = ok ? s_inb[2 * c] : -1, bd = ok ? s_inb[2 * c + 1] : -1;
        c_[u] = ok ? c : -1;
        e_[u] = e;
        cv[u] = bc >= 0 ? ((const double2*)p.in)[bc + e] : make_double2(0.0, 0.0);
        dv[u] = bd >= 0 ? ((const double2*)p.in)[bd + e] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c_[u] < 0) continue;
        double2* line = S + c_[u] * ls;
        const double2 C = cv[u], D = dv[u];
        if (e_[u] == 0) {
          line[pin(0)] = make_double2(C.x, D.x);
        } else {
          line[pin(e_[u])] = make_double2(0.5 * (C.x - D.y), 0.5 * (C.y + D.x));
          line[pin(n - e_[u])] = make_double2(0.5 * (C.x + D.y), 0.5 * (D.x - C.y));
        }
      }
    }
  } else {   // cooperative load into the padded natural layout j -> (j / N2)(N2+1) + j % N2;
      // kLoadBatch loads in flight per thread before their shared-memory stores
    const int cnt = p.in_count;
    const int tot = lpc * cnt;
    const bool e_fast = p.in_e == 1;
    const float inv = 1.0f / (float)cnt;
    const int nthr = blockDim.x;
    for (int i0 = threadIdx.x; i0 < tot; i0 += kLoadBatch * nthr) {
      double2 val[kLoadBatch];
      int pos[kLoadBatch];
#pragma unroll
      for (int u = 0; u < kLoadBatch; ++u) {
        const int idx = i0 + u * nthr;
        const int li = e_fast ? (int)(((float)idx + 0.5f) * inv) : (idx & (lpc - 1));
        const int e = e_fast ? idx - li * cnt : (idx >> lg_lpc);
        const int64_t base = idx < tot ? s_inb[li] : -1;
        pos[u] = -1;
        val[u] = make_double2(0.0, 0.0);
        if (base >= 0) {
          const int64_t a = base + e * p.in_e;
          const int j = bin_of(e, p.in_sym, p.half, n);
          pos[u] = li * ls + (j / N2) * (N2 + 1) + (j % N2);
          val[u] = p.in_real ? make_double2(((const double*)p.in)[a], 0.0)
                             : ((const double2*)p.in)[a];
        }
      }
#pragma unroll
      for (int u = 0; u < kLoadBatch; ++u)
        if (pos[u] >= 0) S[pos[u]] = val[u];
    }
  }
  __syncthreads();
  double2* line = S + team * ls;
  const bool inv = p.dir > 0;
  // step A: columns
  if (lane < N2) {
    const int t = lane;
    double2 v[N1];
#pragma unroll
    for (int i = 0; i < N1; ++i) v[i] = line[i * (N2 + 1) + t];
    dft_reg<N1>(v, w1, inv);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) {
      double2 ww = twA[k1 * N2 + t];
      if (inv) ww.y = -ww.y;
      line[k1 * (N2 + 1) + t] = k1 == 0 ? v[0] : cmul(v[k1], ww);
    }
  }
  __syncthreads();
  // step B: rows
  double2 u[N2];
  const int k1 = lane;
  if (k1 < N1) {
#pragma unroll
    for (int t = 0; t < N2; ++t) u[t] = line[k1 * (N2 + 1) + t];
    dft_reg<N2>(u, w2, inv);   // u[k2] = X[k1 + N1 k2]
    if (!p.has_mult) {
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) line[k1 * (N2 + 1) + k2] = u[k2];
    } else {
      const bool keep_line = s_inb[team] >= 0;
      const int64_t q = s_q[team];
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int bin = k1 + N1 * k2;
        int j = bin;
        if (p.keep_sym) { j = bin + p.half; if (j >= n) j -= n; }
        const double e = (keep_line && j < p.keep_count) ? mult[q + (int64_t)j * p.inner] : 0.0;
        u[k2] = make_double2(u[k2].x * e, u[k2].y * e);
      }
      dft_reg<N2>(u, w2, !inv);   // inverse over k2 -> k1'
#pragma unroll
      for (int k1p = 1; k1p < N2; ++k1p) {
        double2 ww = twB[k1p * N1 + k1];
        if (!inv) ww.y = -ww.y;
        u[k1p] = cmul(u[k1p], ww);
      }
    }
  }
  if (p.has_mult) {
    __syncthreads();   // every row read before the transposed write
    if (k1 < N1) {
#pragma unroll
      for (int k1p = 0; k1p < N2; ++k1p) line[k1p * (N1 + 1) + k1] = u[k1p];
    }
    __syncthreads();
    // step C: thread k1' finishes the inverse over k1 -> y[k1' + N2 k2'], own row
    if (lane < N2) {
      const int k1p = lane;
      double2 v[N1];
#pragma unroll
      for (int i = 0; i < N1; ++i) v[i] = line[k1p * (N1 + 1) + i];
      dft_reg<N1>(v, w1, !inv);
#pragma unroll
      for (int k2p = 0; k2p < N1; ++k2p) line[k1p * (N1 + 1) + k2p] = v[k2p];
    }
  }
  __syncthreads();
  if (pack == 1) {
    // separate the two real lines' spectra: X = (Z[k] + conj Z[-k])/2, Y = (Z[k] - conj Z[-k])/2i
    const int cnt = p.out_count;
    const int tot = rl * cnt;
    const float inv_c = 1.0f / (float)cnt;
    for (int idx = threadIdx.x; idx < tot; idx += nthr) {
      const int li = (int)(((float)idx + 0.5f) * inv_c);
      const int e = idx - li * cnt;
      const int64_t base = s_outb[li];
      if (base < 0) continue;
      const double2* line = S + (li >> 1) * ls;
      const double2 A = line[pnf(e)];
      const double2 B = line[pnf((n - e) & (n - 1))];
      const double2 v = (li & 1) ? make_double2(0.5 * (A.y + B.y), 0.5 * (B.x - A.x))
                                 : make_double2(0.5 * (A.x + B.x), 0.5 * (A.y - B.y));
      ((double2*)p.out)[base + e] = v;
    }
  } else if (pack == 2) {
    // full real lines: line 2c is Re, line 2c+1 is Im of the inverse of line c
    const int tot = rl * n;
    for (int idx = threadIdx.x; idx < tot; idx += nthr) {
      const int li = idx >> LGN, e = idx & (n - 1);
      const int64_t base = s_outb[li];
      if (base < 0) continue;
      const double2 v = S[(li >> 1) * ls + pnf(e)];
      ((double*)p.out)[base + e] = (li & 1) ? v.y : v.x;
    }
  } else {   // cooperative store; bin k sits at (k % N1)(N2+1) + k / N1, or after the fused
             // inverse at (k % N2)(N1+1) + k / N2
    const int cnt = p.out_count;
    const int tot = lpc * cnt;
    const bool e_fast = p.out_e == 1;
    const float inv_c = 1.0f / (float)cnt;
    const bool fused = p.has_mult != 0;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
      const int li = e_fast ? (int)(((float)idx + 0.5f) * inv_c) : (idx & (lpc - 1));
      const int e = e_fast ? idx - li * cnt : (idx >> lg_lpc);
      const int64_t base = s_outb[li];
      if (base < 0) continue;
      const int64_t a = base + e * p.out_e;
      const int k = bin_of(e, p.out_sym, p.half, n);
      const int pos = fused ? (k % N2) * (N1 + 1) + k / N2 : (k % N1) * (N2 + 1) + k / N1;
      double2 v = S[li * ls + pos];
      if (p.mult_out) {
        const double m = mult[s_q[li] + (int64_t)e * p.inner];
        v = make_double2(v.x * m, v.y * m);
      }
      if (p.out_real)
        ((double*)p.out)[a] = v.x;
      else
        ((double2*)p.out)[a] = v;
    }
  }
}

template <int N1, int N2>
static void launch_4s(const LinePass& p, const BatchOff& off, int nb, const double2* tw,
                      cudaStream_t s) {
  constexpr int n = N1 * N2;
  constexpr int T = N1 > N2 ? N1 : N2;
  constexpr int ls = n + T + 1;
  int lpc = 128 / T;
  if (lpc > kMaxLpc) lpc = kMaxLpc;
  if (lpc < 1) lpc = 1;
  const size_t smem = sizeof(double2) * (2 * (size_t)n + (size_t)lpc * ls);
  if (smem > 48 * 1024)
    AFS_CUDA(cudaFuncSetAttribute(k_line_pass_4s<N1, N2>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int rl = p.pack ? 2 * lpc : lpc;
  const int64_t blocks = (p.nlines + rl - 1) / rl;
  dim3 grid((unsigned)blocks, (unsigned)nb);
  k_line_pass_4s<N1, N2><<<grid, lpc * T, smem, s>>>(p, off, tw, lpc, T);
}

// four-step variant for this n?  returns false when the generic kernel must run
static bool run_pass_4s(const LinePass& p, const BatchOff& off, int nb, const double2* tw,
                        cudaStream_t s) {
  switch (p.n) {
    case 16: launch_4s<4, 4>(p, off, nb, tw, s); return true;
    case 32: launch_4s<8, 4>(p, off, nb, tw, s); return true;
    case 64: launch_4s<8, 8>(p, off, nb, tw, s); return true;
    case 128: launch_4s<16, 8>(p, off, nb, tw, s); return true;
    case 256: launch_4s<16, 16>(p, off, nb, tw, s); return true;
    case 512: launch_4s<32, 16>(p, off, nb, tw, s); return true;
    case 1024: launch_4s<32, 32>(p, off, nb, tw, s); return true;
    default: return false;
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
  if (pl->fft_mode == 0 && run_pass_4s(p, off, nb, pl->twiddle, s)) return;
  // lines per CTA: enough lines for coalesced strided access, ~64 KB of shared memory
  int lpc = kMaxLpc;
  while (lpc > 1 && (size_t)lpc * 2 * (pl->n + 1) * sizeof(double2) > 72 * 1024) lpc /= 2;
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

// mode 0: grid -> grid (fused first-axis pass).  mode 1: grid -> pruned spectrum E (.) F(g)
// in pl->spec (layout of the multiplier, complex).  mode 2: pruned spectrum -> grid.
// Modes 1 + 2 split the stage so point-sharded ranks can all-reduce the spectrum (linear in
// the nodes) instead of the oversampled grid: K^(d-1)*(M/2+1) instead of n^d values.
static void spectral_subset(afs_plan* pl, int R, cudaStream_t s, int mode,
                            const std::vector<int>* only);

void spectral_all(afs_plan* pl, int R, cudaStream_t s, int mode) {
  spectral_subset(pl, R, s, mode, nullptr);
}

// the fused stage (mode 0) for a subset of the windows (the window pipeline's units)
void spectral_windows(afs_plan* pl, int R, cudaStream_t s, const std::vector<int>& wins) {
  spectral_subset(pl, R, s, 0, &wins);
}

static void spectral_subset(afs_plan* pl, int R, cudaStream_t s, int mode,
                            const std::vector<int>* only) {
  const int n = pl->n, M = pl->M, H = pl->H, K = M + 1;
  const int64_t gs = pl->grid_total;
  const int64_t ss = pl->spec_total;
  for (int d = 1; d <= 3; ++d) {
    std::vector<int> ws;
    if (only) {
      for (int l : *only)
        if (pl->win[l].d == d) ws.push_back(l);
    } else {
      for (int l = 0; l < pl->P; ++l)
        if (pl->win[l].d == d) ws.push_back(l);
    }
    for (size_t b0 = 0; b0 < ws.size(); b0 += kMaxBatch) {
      const int nb = (int)std::min<size_t>(kMaxBatch, ws.size() - b0);
      BatchOff grid_off{}, a_off{}, b_off{}, m_off{}, s_off{};
      for (int i = 0; i < nb; ++i) {
        const Window& w = pl->win[ws[b0 + i]];
        grid_off.in[i] = grid_off.out[i] = w.grid_off;
        a_off.in[i] = a_off.out[i] = w.scratch_a_off;
        b_off.in[i] = b_off.out[i] = w.scratch_b_off;
        m_off.mult[i] = w.mult_off;
        s_off.in[i] = s_off.out[i] = w.mult_off;   // spectrum shares the multiplier layout
      }
      double* g = pl->grids;
      LinePass p{};
      if (d == 1) {
        BatchOff o = grid_off;
        for (int i = 0; i < nb; ++i) o.mult[i] = m_off.mult[i];
        p.nlines = R; p.inner = 1;
        p.mult = pl->mult;
        if (mode == 0) {
          // single fused pass: real line -> keep k in 0..M/2 -> * E -> inverse -> real
          p.in_o = gs; p.in_q = 0; p.in_e = 1; p.in_count = n; p.in_real = 1;
          p.out_o = gs; p.out_q = 0; p.out_e = 1; p.out_count = n; p.out_real = 1;
          p.dir = -1; p.has_mult = 1; p.keep_count = H; p.keep_sym = 0;
          p.in = g; p.out = g;
        } else if (mode == 1) {
          for (int i = 0; i < nb; ++i) o.out[i] = s_off.out[i];
          p.in_o = gs; p.in_q = 0; p.in_e = 1; p.in_count = n; p.in_real = 1;
          p.out_o = ss; p.out_q = 0; p.out_e = 1; p.out_count = H;
          p.dir = -1; p.mult_out = 1;
          p.in = g; p.out = pl->spec;
        } else {
          for (int i = 0; i < nb; ++i) o.in[i] = s_off.in[i];
          p.in_o = ss; p.in_q = 0; p.in_e = 1; p.in_count = H;
          p.out_o = gs; p.out_q = 0; p.out_e = 1; p.out_count = n; p.out_real = 1;
          p.dir = +1;
          p.in = pl->spec; p.out = g;
        }
        run_pass(pl, p, o, nb, s);
        continue;
      }
      double2* A = pl->scratch_a;
      double2* B = pl->scratch_b;
      const int64_t n0 = n;
      const int64_t rows = (d == 3) ? (int64_t)n * n : (int64_t)n;   // last-axis lines per rhs
      const int64_t aper = rows * H;                                  // A per rhs
      // first-axis lines live in F = A (d=2) or B (d=3); fq lines per rhs
      double2* F = d == 3 ? B : A;
      const BatchOff fo = d == 3 ? b_off : a_off;
      const int64_t fq = d == 3 ? (int64_t)K * H : (int64_t)H;
      if (mode != 2) {
        // pass 1: real last axis -> half spectrum (k in 0..M/2):  g -> A[r][rows][H]
        BatchOff o1{};
        for (int i = 0; i < nb; ++i) { o1.in[i] = grid_off.in[i]; o1.out[i] = a_off.out[i]; }
        p = LinePass{};
        p.nlines = R * rows; p.inner = rows;
        p.in_o = gs; p.in_q = n; p.in_e = 1; p.in_count = n; p.in_real = 1;
        p.out_o = aper; p.out_q = H; p.out_e = 1; p.out_count = H;
        p.dir = -1; p.in = g; p.out = A; p.mult = pl->mult;
        p.pack = 1;
        run_pass(pl, p, o1, nb, s);
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
        }
      }
      if (mode == 0) {
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
      } else if (mode == 1) {
        // first axis forward, keep j0 in 0..M, * E -> spectrum [j0][q]
        BatchOff o3{};
        for (int i = 0; i < nb; ++i) {
          o3.in[i] = fo.in[i]; o3.out[i] = s_off.out[i]; o3.mult[i] = m_off.mult[i];
        }
        p = LinePass{};
        p.nlines = R * fq; p.inner = fq;
        p.in_o = n0 * fq; p.in_q = 1; p.in_e = fq; p.in_count = n;
        p.out_o = ss; p.out_q = 1; p.out_e = fq; p.out_count = K; p.out_sym = 1;
        p.dir = -1; p.mult_out = 1; p.mult = pl->mult;
        p.in = F; p.out = pl->spec;
        run_pass(pl, p, o3, nb, s);
        continue;
      } else {
        // spectrum [j0][q] -> first axis inverse (n values) in F
        BatchOff o3{};
        for (int i = 0; i < nb; ++i) { o3.in[i] = s_off.in[i]; o3.out[i] = fo.out[i]; }
        p = LinePass{};
        p.nlines = R * fq; p.inner = fq;
        p.in_o = ss; p.in_q = 1; p.in_e = fq; p.in_count = K; p.in_sym = 1;
        p.out_o = n0 * fq; p.out_q = 1; p.out_e = fq; p.out_count = n;
        p.dir = +1; p.mult = pl->mult;
        p.in = pl->spec; p.out = F;
        run_pass(pl, p, o3, nb, s);
      }
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
      p.pack = (2 * (H - 1) < n) ? 2 : 0;   // Hermitian completion needs k and -k distinct
      run_pass(pl, p, o5, nb, s);
    }
  }
  AFS_CUDA(cudaGetLastError());
}

}  // namespace afs
