/* pathtrack_b200.h -- C-ABI of the B200 single-path homotopy tracker.
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json's
 * north_star: track one solution path of h(x,t) = gamma*(1-t)^k g(x) + t^k f(x)
 * in complex double (D), double-double (DD) or quad-double (QD).
 *
 * The reference (/root/reference/proj) ships only the scalar layer; the
 * tracker API exists as SPEC.md signatures.  Each entry point below names the
 * reference interface it replaces:
 *
 *   pt_prec                 PrecisionMode            multiprec.hpp:27
 *   pt_system_desc          PolynomialSystem / Term  SPEC.md:129-136 (canonical form SPEC.md:150)
 *   pt_plan_create          make_homotopy + compile_plan
 *                                                    SPEC.md:165-173, 222-230
 *   pt_step_params          StepControlParams + NewtonParams
 *                                                    SPEC.md:357-359, 448-451, 384, 429, 495
 *   pt_path_stats           TrackOutcome / NewtonOutcome
 *                                                    SPEC.md:361-364, 460-463
 *   pt_trace_event          PathTrace event
 *   pt_track_path           track_path
 *   pt_track_batch          many concurrent trackers SPEC.md:496-497
 *   pt_eval_homotopy        evaluate_homotopy
 *   pt_lstsq                least_squares_solve
 *   pt_default_params       RealTraits<R>::newton_tolerance + SPEC defaults
 *                                                    multiprec.hpp:391,404,418
 *
 * Conventions
 *  - Numbers are binary64 limbs, L = 1 (D), 2 (DD), 4 (QD), limb layout
 *    identical to RealTraits<R>::components (multiprec.hpp:393,406,421).
 *  - Complex vectors of length S are structure-of-arrays: re limb l at
 *    [l*S + i], im limb l at [(L+l)*S + i]  (2*L*S doubles).
 *  - Matrices are column-major complex, S = rows*cols, entry (i,j) at j*rows+i.
 *  - Return codes: 0 ok, negative = error (pt_last_error() has the text).
 *    A path that fails to reach t=1 is NOT an error: see pt_path_stats.status.
 *  - Ownership: the caller owns every host buffer; a plan owns its device
 *    memory and its CUDA stream.  A plan is bound to one device and must not
 *    be used by two host threads at once.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns PT_E_NODEVICE.
 */
#ifndef PATHTRACK_B200_H
#define PATHTRACK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { PT_D = 0, PT_DD = 1, PT_QD = 2 } pt_prec;

enum {
  PT_OK = 0,
  PT_E_INVAL = -1,      /* malformed arguments / system */
  PT_E_CUDA = -2,       /* CUDA runtime error */
  PT_E_RANK = -3,       /* rank-deficient least-squares matrix (pt_lstsq) */
  PT_E_NODEVICE = -4,   /* no usable sm_100 device */
  PT_E_TIMEOUT = -5,    /* device-side watchdog fired (grid barrier stalled) */
  PT_E_NOMEM = -6
};

/* Path status and failure kinds. */
enum { PT_PATH_SUCCESS = 0, PT_PATH_FAIL = 1 };
enum { PT_FAIL_NONE = 0, PT_FAIL_START = 1, PT_FAIL_MAX_STEPS = 2, PT_FAIL_MIN_STEP = 3,
       PT_FAIL_ABORT = 4 /* device watchdog: a barrier or MGS exchange stalled (not a SPEC outcome) */ };

/* pt_path_stats.flags.  PT_STAT_NONFINITE: the path met a non-finite value
 * (max|h|, max|dx| or an MGS diagonal was inf / NaN, or the end point is).
 * DD paths are tracked by kernels whose dd_norm skips the reference's
 * non-finite fix-up (multiprec.hpp:102-107, a select on the critical chain);
 * they are bit-identical to the reference whenever no DD intermediate is
 * inf / NaN, and every path that met one is re-tracked from its start by the
 * exact kernels (same stream, no host round trip), so the reported results
 * always follow the reference's rules. */
enum { PT_STAT_NONFINITE = 1 };

/* One polynomial system in canonical distributed form.
 * Equation i owns terms [eq_ptr[i], eq_ptr[i+1]); term t owns the
 * (var, exp) pairs [term_ptr[t], term_ptr[t+1]) with strictly increasing var
 * and exp >= 1; an empty support is a constant term.  coef is a complex
 * vector of length n_terms in the SoA layout above. */
typedef struct {
  int32_t n_vars, n_eqs, n_terms;
  const int32_t* eq_ptr;
  const int32_t* term_ptr;
  const int32_t* var;
  const int32_t* exp;
  const double* coef;
} pt_system_desc;

/* StepControlParams + NewtonParams.
 * Expansion factor 2, shrink factor 1/2 and the 3-success threshold are the
 * fixed Fig. 3 constants. */
typedef struct {
  double max_step;         /* Delta t_max, also the initial Delta t */
  double min_step;         /* h_min */
  int32_t max_steps;       /* P.max#steps */
  int32_t pred_degree;     /* extrapolation degree, 0..8 */
  int32_t newton_max_iter; /* P.max_iteration */
  int32_t reserved;
  double newton_tol;       /* P.tolerance (residual and update) */
} pt_step_params;

typedef struct {
  int32_t status;          /* PT_PATH_SUCCESS / PT_PATH_FAIL */
  int32_t failure_kind;    /* PT_FAIL_* */
  int32_t steps;           /* m: all predictor-corrector trials */
  int32_t accepted;        /* accepted trials */
  int32_t newton_iters;    /* evaluations, start validation included */
  int32_t start_iters;     /* evaluations of the t=0 start validation */
  int32_t solves;          /* completed least-squares solves (MGS + back substitution) */
  int32_t flags;           /* PT_STAT_NONFINITE: see below */
  double final_residual;   /* last max|h| computed */
  double final_update;     /* last max|dx| computed (-1 if none) */
  double t_end;            /* last accepted t */
} pt_path_stats;

typedef struct {
  double t;                /* trial t */
  int32_t ok;              /* 1 corrected, 0 diverged */
  int32_t iters;           /* Newton evaluations in this trial */
  double residual, update;
} pt_trace_event;

typedef struct pt_plan pt_plan;

/* SPEC defaults for a precision: tol 1e-8/1e-20/1e-44, 6 iterations,
 * Delta t_max 0.1, h_min 1e-6, max steps 500/500/1500, predictor degree 4. */
int pt_default_params(pt_prec prec, pt_step_params* out);

/* Number of usable CUDA devices (0 when none). */
int pt_device_count(void);

/* make_homotopy + compile_plan on `device`.  gamma: 2L limbs (re, im).
 * relax_k >= 1.  g and f must have equal n_vars and n_eqs, n_eqs >= n_vars. */
int pt_plan_create(int device, pt_prec prec, const pt_system_desc* g, const pt_system_desc* f,
                   const double* gamma, int32_t relax_k, pt_plan** out);
void pt_plan_destroy(pt_plan* plan);

/* Query plan facts: 0 n_vars, 1 n_eqs, 2 monomials, 3 contributions,
 * 4 grid CTAs used for one path, 5 precision, 6 batch CTAs resident,
 * 7 monomial workspace entries, 8 single-path engine (0 grid, 1 cluster),
 * 9 cluster size of the cluster engine (0: none schedulable). */
int64_t pt_plan_info(const pt_plan* plan, int32_t what);

/* Force the single-path engine: 0 = cooperative persistent grid (all SMs,
 * grid barriers, L2 flags), 1 = one thread-block cluster (cluster barriers,
 * DSMEM column exchange).  pt_plan_create picks one by problem size; both
 * produce bit-identical results. */
int pt_plan_set_engine(pt_plan* plan, int32_t engine);

/* Arithmetic of a QD plan's tracking kernels.  PT_ARITH_REFERENCE (default):
 * the reference operation sequences (multiprec.hpp), bit-identical to the
 * reference tracker.  PT_ARITH_FAST: tolerance parity -- classic quad-double
 * algorithms (sloppy add, truncated product, long division) and a
 * reciprocal-square-root MGS normalisation (no division on the column chain);
 * end points agree with the reference to ~1e-60 relative (scaled by the
 * conditioning), step / Newton counts agree barring ties at the step-control
 * thresholds.  D and DD plans accept only
 * PT_ARITH_REFERENCE.  Applies to pt_track_path / pt_track_batch /
 * pt_eval_homotopy of this plan. */
enum { PT_ARITH_REFERENCE = 0, PT_ARITH_FAST = 1 };
int pt_plan_set_arith(pt_plan* plan, int32_t arith);

/* Algorithmic work of one unit of the path, counted on the reference
 * algorithms.  kind: 0 one evaluation (h and J),
 * 1 one least-squares solve + update, 2 one prediction of degree `degree`.
 * out[0..4]: real adds, real muls, real divisions, real square roots,
 * binary64 hypots; out[5]: FP64 arithmetic instructions of the reference
 * DD/QD algorithms for those operations in the plan's precision. */
int pt_plan_work(const pt_plan* plan, int32_t kind, int32_t degree, double* out);

/* Measured FP64-pipe peak of `device`: thread-level DFMA instructions per
 * second from an unrolled independent-chain microbenchmark. */
int pt_fp64_peak(int device, double* instr_per_s, double* ms);

/* Latency microbenchmarks used to size the design:
 * what 0: cycles per dependent op, out[0] DADD, [1] DD add, [2] DD mul,
 * [3] QD add, [4] QD mul, [5] complex DD mul, [6] hypot;
 * what 1: out[0] ns per grid barrier (148 CTAs); what 2: out[0] one-way ns of
 * a release/acquire flag between CTA 0 and the last CTA. */
int pt_microbench(int device, int32_t what, double* out);

/* Device phase timers of the single-path kernel (block 0, globaltimer ns,
 * accumulated over launches): out[0] monomials, [1] slot sums + residual,
 * [2] MGS, [3] back substitution + update, [4] predictor, [5] Newton
 * iterations (count); reset != 0 clears them. */
int pt_plan_profile(pt_plan* plan, double* out, int32_t reset);
/* The same timers of batch CTA `slice` (k_track_batch, accumulated over the
 * paths that CTA tracked). */
int pt_plan_batch_profile(pt_plan* plan, int32_t slice, double* out, int32_t reset);

/* MGS timeline of the last single-path launch (debugging aid): for column j,
 * out[3j..3j+2] = globaltimer ns when q_{j-1} reached the owner of column j,
 * after its projection, after q_j was published. */
int pt_plan_mgs_timeline(pt_plan* plan, double* out, int32_t count);

/* Enable a per-trial trace of up to `capacity` events (0 disables). */
int pt_plan_set_trace(pt_plan* plan, int32_t capacity);
/* Copy the trace of the last pt_track_path call; *count = events recorded. */
int pt_plan_get_trace(pt_plan* plan, pt_trace_event* out, int32_t capacity, int32_t* count);

/* track_path: host buffers, host<->device copies included.
 * start, end: complex vectors of length n_vars. */
int pt_track_path(pt_plan* plan, const double* start, const pt_step_params* params, double* end,
                  pt_path_stats* stats);

/* Same with device-resident buffers on `stream` (cudaStream_t, 0 = the
 * plan's stream); stats is a device pointer too.  Asynchronous. */
int pt_track_path_device(pt_plan* plan, const double* d_start, const pt_step_params* params,
                         double* d_end, pt_path_stats* d_stats, void* stream);

/* n_paths independent paths on the plan's device: starts/ends are
 * n_paths consecutive complex vectors (path p at p*2*L*n_vars). */
int pt_track_batch(pt_plan* plan, int32_t n_paths, const double* starts, const pt_step_params* params,
                   double* ends, pt_path_stats* stats);
int pt_track_batch_device(pt_plan* plan, int32_t n_paths, const double* d_starts,
                          const pt_step_params* params, double* d_ends, pt_path_stats* d_stats,
                          void* stream);

/* evaluate_homotopy at (x, t): h (length n_eqs), J (n_eqs x n_vars,
 * column-major), *rmax = max_modulus(h).  Any output may be NULL. */
int pt_eval_homotopy(pt_plan* plan, const double* x, double t, double* h, double* J, double* rmax);

/* run_evalbench: device time of one evaluation and
 * differentiation pass (h and J into the plan's workspace) at (x, t),
 * averaged over `reps` back-to-back launches after one warm-up. */
int pt_eval_bench(pt_plan* plan, const double* x, double t, int32_t reps, double* ms_per_eval);

/* least_squares_solve by MGS on the device: A (N x n, column-major), b (N). */
int pt_lstsq(int device, pt_prec prec, int32_t N, int32_t n, const double* A, const double* b, double* x);

/* Bulk scalar arithmetic on the device (parity tests of the DD/QD kernels):
 * op codes and element layout as documented in DESIGN.md section 3. */
int pt_arith_device(int device, pt_prec prec, int32_t op, int64_t count, const double* a, const double* b,
                    double* out);
/* The same with an explicit arithmetic (PT_ARITH_FAST: the fast QD set). */
int pt_arith_device_mode(int device, pt_prec prec, int32_t arith, int32_t op, int64_t count, const double* a,
                         const double* b, double* out);
/* The same operations through the host build of the device arithmetic. */
int pt_arith_host(pt_prec prec, int32_t op, int64_t count, const double* a, const double* b, double* out);

const char* pt_last_error(void);
const char* pt_version(void);

/* Inputs (synthetic systems, system / solution files, Pieri minors) live in
 * the host-only library declared in pathtrack_inputs.h: building the inputs
 * never loads this library. */

#ifdef __cplusplus
}
#endif

#endif /* PATHTRACK_B200_H */
