/*
 * anovafs.h — C ABI of the B200-native ANOVA fast-summation matvec.
 *
 * Drop-in boundary for the reference's hot path (arXiv 2111.10140, package
 * nfftkrr; paths relative to /root/reference/pkg/src/nfftkrr):
 *
 *   afs_plan_create   replaces the per-window construction in
 *                     AnovaKernelOperator.__init__ (anova.py:146-173), i.e. one
 *                     FastsumOperator per window (fastsum.py:189-232) with its
 *                     NfftPlan geometry (nfft.py:139-177).  Scaling parameters
 *                     (center/scale, fastsum.py:210-217) and the spectral
 *                     multiplier (c_hat * deconv^2, fastsum.py:138-159 +
 *                     nfft.py:158-162) are computed by the host layer and passed in.
 *   afs_apply         replaces AnovaKernelOperator.apply (anova.py:175-183) =
 *                     sum_l eta_l FastsumOperator.apply (fastsum.py:243-256) =
 *                     Re(NfftPlan.forward(c_hat * NfftPlan.adjoint(alpha)))
 *                     (nfft.py:220-250), for nrhs right-hand sides at once.
 *   afs_cg_solve      replaces cg_solve(lambda v: op.apply(v) + beta*v, b, tol,
 *                     maxiter) as called by fit (krr.py:76-110, 162-167), run
 *                     device-resident with the same stopping rule and breakdown
 *                     checks.
 *   afs_last_error    message for the last non-zero status on this thread.
 *
 * Status codes map 1:1 onto the reference's exceptions (errors.py:8-17):
 *   AFS_ERR_SHAPE -> ShapeError, AFS_ERR_VALIDATION -> ValidationError,
 *   AFS_ERR_NUMERICAL -> NumericalError; AFS_ERR_CUDA / AFS_ERR_NOMEM are
 *   device failures (RuntimeError / MemoryError on the Python side).
 *
 * Pointers: bulk arrays (coordinates, alpha, out, b, x) are DEVICE pointers on
 * desc->device; small parameter arrays are HOST pointers.  All arithmetic is
 * IEEE fp64.  A plan's geometry is immutable after creation.  afs_apply is
 * reentrant: the first caller runs on the plan's own workspace,
 * concurrent callers on up to 3 workspace clones (own grids, spectral scratch,
 * streams and graphs; shared sorted nodes and multipliers), so applies from
 * several host threads overlap on the device.  The stage-level entry points,
 * afs_cg_solve and the mode setters use the plan's own workspace and are
 * serialised with each other.
 */
#ifndef ANOVAFS_H
#define ANOVAFS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AFS_ABI_VERSION 3

enum afs_status {
  AFS_OK = 0,
  AFS_ERR_SHAPE = 1,
  AFS_ERR_VALIDATION = 2,
  AFS_ERR_NUMERICAL = 3,
  AFS_ERR_CUDA = 4,
  AFS_ERR_NOMEM = 5
};

typedef struct afs_plan afs_plan;

/* One feature window W_l (anova.py:91-121; fastsum.py:189-232). */
typedef struct afs_window_desc {
  int32_t dims;              /* d_l in 1..3 */
  int32_t features[3];       /* 0-based column indices into the coordinate matrix */
  double center[3];          /* bbox centre of sources (U targets), fastsum.py:217 */
  double scale;              /* ball_radius / bbox diameter, fastsum.py:216 */
  double weight;             /* eta_l; the reference uses 1/P (anova.py:109) */
  /* HOST pointer to the window's real, pruned spectral multiplier E (see
   * DESIGN.md "spectral stage"): layout [j0][j1][k] for d=3, [j0][k] for d=2,
   * [k] for d=1, with j in 0..M (frequency j - M/2) and k in 0..M/2, already
   * symmetrised, scaled by 1/n^(2d) and doubled for k >= 1. */
  const double* multiplier;
} afs_window_desc;

typedef struct afs_plan_desc {
  int32_t device;            /* CUDA ordinal */
  int32_t n_windows;         /* P >= 1 */
  const afs_window_desc* windows;
  int32_t d_total;           /* columns of the coordinate matrices */
  int64_t n_sources;         /* N_x >= 1 */
  const double* sources;     /* device, row-major n_sources x d_total */
  int64_t n_targets;         /* 0 => targets are the sources */
  const double* targets;     /* device, row-major n_targets x d_total, or NULL */
  int32_t bandwidth;         /* M = PeriodizationConfig.coeff_grid (even >= 2) */
  int32_t cutoff;            /* m = AccuracyProfile.cutoff (1..8) */
  int32_t grid;              /* n = max(2m, even(ceil(oversampling*M))), nfft.py:151-153 */
  int32_t max_rhs;           /* largest nrhs passed to afs_apply (>= 1) */
  /* 0: window values from per-offset polynomials (degree 11 at m >= 4, |err| <= 5e-16
   *    of the peak value, below the reference's own 3.5e-15 sinh-argument rounding)
   *    feeding the bin-sorted sliding-window kernels (default, fast);
   * 1: the reference's exact formula sinh(b s)/(pi s) evaluated per node with
   *    numpy's rounding order (slow parity mirror). */
  int32_t window_eval;
} afs_plan_desc;

typedef struct afs_plan_info {
  int64_t device_bytes;      /* bytes of device memory owned by the plan */
  int32_t n_windows;
  int32_t grid;
  int64_t n_sources;
  int64_t n_targets;
  /* kernels one afs_apply launches: counted from its captured CUDA graph once one exists
   * (second apply with the same buffers), a plan-time estimate before */
  int32_t kernel_launches_per_apply;
  /* windows whose (source-side) nodes run on the fp64 tensor-core kernels (ABI 2) */
  int32_t tensor_core_windows;
} afs_plan_info;

int afs_abi_version(void);
const char* afs_last_error(void);

int afs_plan_create(const afs_plan_desc* desc, afs_plan** plan);
int afs_plan_destroy(afs_plan* plan);
int afs_plan_get_info(const afs_plan* plan, afs_plan_info* info);

/* out[r*ld_out + i] = sum_l eta_l (K_l alpha_r)(z_i), r < nrhs.
 * alpha: device, nrhs vectors of n_sources (stride ld_alpha);
 * out:   device, nrhs vectors of n_targets (stride ld_out).
 * stream: a cudaStream_t (NULL = legacy default stream). */
int afs_apply(afs_plan* plan, const double* alpha, int64_t ld_alpha, double* out,
              int64_t ld_out, int32_t nrhs, void* stream);

/* The three stages of afs_apply, for point-sharded multi-GPU use:
 * afs_spread writes every window's oversampled grid (afs_plan_grids: base pointer,
 * doubles per rhs = sum over windows of n^d_l, rhs r at grids + r*stride), the caller
 * may all-reduce the grids across ranks, afs_spectral applies the multipliers in place,
 * afs_gather interpolates into out (same conventions as afs_apply). */
int afs_spread(afs_plan* plan, const double* alpha, int64_t ld_alpha, int32_t nrhs,
               void* stream);
int afs_spectral(afs_plan* plan, int32_t nrhs, void* stream);
int afs_gather(afs_plan* plan, double* out, int64_t ld_out, int32_t nrhs, void* stream);
int afs_plan_grids(afs_plan* plan, double** grids, int64_t* doubles_per_rhs);
/* Let the caller own the grid buffer (e.g. a tensor registered with NCCL): capacity must be
 * >= doubles_per_rhs * max_rhs; the plan stops using (and frees) its own buffer. */
int afs_plan_bind_grids(afs_plan* plan, double* buffer, int64_t capacity_doubles);

/* Split spectral stage for point sharding with a spectrum exchange:
 * afs_spectral_forward turns every window's grid into its pruned spectrum E (.) F(g) --
 * complex, laid out like the window's multiplier ([j0][j1][k], K^(d-1)*(M/2+1) entries) --
 * in the plan's spectrum buffer (afs_plan_spectra: base pointer as doubles, doubles per rhs =
 * 2 * sum of multiplier lengths); the caller may all-reduce it across ranks (the spread and
 * the transform are linear in the nodes); afs_spectral_inverse turns it back into grids
 * for afs_gather.  forward + inverse == afs_spectral up to rounding. */
int afs_spectral_forward(afs_plan* plan, int32_t nrhs, void* stream);
int afs_spectral_inverse(afs_plan* plan, int32_t nrhs, void* stream);
int afs_plan_spectra(afs_plan* plan, double** spectra, int64_t* doubles_per_rhs);
/* caller-owned spectrum buffer (16-byte aligned, >= doubles_per_rhs * max_rhs doubles) */
int afs_plan_bind_spectra(afs_plan* plan, double* buffer, int64_t capacity_doubles);

/* Stage profiling: when enabled, every afs_apply records CUDA events around
 * its spread / spectral / gather stages on the caller's stream, waits for them
 * and accumulates the device milliseconds (this adds one stream sync per
 * apply, so enable it only for a dedicated measurement pass).
 * afs_plan_stage_times writes {spread_ms, spectral_ms, gather_ms, applies}
 * and resets the accumulators when reset != 0. */
int afs_plan_set_profiling(afs_plan* plan, int32_t enable);
int afs_plan_stage_times(afs_plan* plan, double* out4, int32_t reset);
/* Per-window kernel time of the spread and the gather (ms accumulated over profiled
 * applies; arrays of n_windows). */
int afs_plan_window_times(afs_plan* plan, double* spread_ms, double* gather_ms, int32_t reset);

/* Deterministic mode: the spread accumulates each grid cell in exact fixed point -- three
 * limbs of L bits (L = 40 for up to 2^23 source nodes, 36 up to 2^27) added with 64-bit
 * integer reductions -- instead of fp64 atomics, with the scale chosen per apply from
 * max|alpha| so no partial sum can overflow; the limbs are converted back to fp64 once.
 * Plans with more than 2^27 source nodes are rejected (AFS_ERR_VALIDATION: limb headroom);
 * a non-finite alpha yields NaN results.  afs_apply / afs_cg_solve then return bit-identical results run to run
 * for the same plan and inputs (the gather, spectral stage and CG reductions are already
 * fixed-order).  Costs 3x the grid memory for the limbs and ~2 extra passes per apply. */
int afs_plan_set_deterministic(afs_plan* plan, int32_t enable);

/* Solve (K + beta I) x = b by plain CG from x0 = 0 (krr.py:76-110).
 * Requires n_targets == n_sources (no separate targets).  b, x: device.
 * Returns AFS_ERR_NUMERICAL on breakdown with *iterations = failing iteration. */
int afs_cg_solve(afs_plan* plan, const double* b, double* x, double beta, double tol,
                 int32_t maxiter, int32_t* iterations, double* residual,
                 int32_t* converged, void* stream);

/* CG vector kernels on caller-owned device vectors, for CG drivers whose matvec is not one
 * plan -- window-sharded (replicated vectors, Ap all-reduced) and point-sharded (row-sharded
 * vectors, scalars all-reduced) multi-GPU solves.  One iteration of cg_solve
 * (krr.py:86-109) is  Ap = K p  ->  afs_cg_vec_ap  ->  afs_cg_vec_update  ->  host checks on
 * ws[1..3]  ->  afs_cg_vec_direction.  ws: device doubles[AFS_CG_WORKSPACE_DOUBLES]:
 *   ws[0] rs = r.r   ws[1] p.Ap   ws[2] rs_new   ws[3] non-finite flag (> 0: Ap had NaN/Inf)
 * Each kernel writes the LOCAL partial over its n entries; a point-sharded driver sums ws[0]
 * after init, ws[1..3] after ap and ws[2] after update across ranks before the next call.
 *   afs_cg_vec_init:      x = 0, r = p = b, ws[0] = b.b, flags cleared, beta stored
 *   afs_cg_vec_ap:        Ap += beta p (in place), ws[1] = p.Ap, ws[3] |= non-finite(Ap)
 *   afs_cg_vec_update:    x += (ws[0]/ws[1]) p, r -= (ws[0]/ws[1]) Ap, ws[2] = r.r
 *   afs_cg_vec_direction: p = r + (ws[2]/ws[0]) p, then ws[0] = ws[2]
 * Reductions are fixed-order (run-to-run deterministic). */
#define AFS_CG_WORKSPACE_DOUBLES 640
int afs_cg_vec_init(const double* b, double* x, double* r, double* p, int64_t n, double beta,
                    double* ws, void* stream);
int afs_cg_vec_ap(double* ap, const double* p, int64_t n, double* ws, void* stream);
int afs_cg_vec_update(double* x, double* r, const double* p, const double* ap, int64_t n,
                      double* ws, void* stream);
int afs_cg_vec_direction(double* p, const double* r, int64_t n, double* ws, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ANOVAFS_H */
