/*
 * gato_b200.h -- C ABI of the B200-native batched SQP trajectory-optimisation solve.
 *
 * Drop-in boundary for the reference package's batched-solve path (paths relative to
 * /root/reference/pkg/src/trajbatch/):
 *
 *   gato_create / gato_bind / gato_solve      replace  batch_solve          batch.py:102-124
 *                                             (M x sqp_solve                sqp.py:204-295)
 *   gato_step_many                            replaces dynamics.step_many           dynamics.py:805-816
 *   gato_step_jacobians_many                  replaces dynamics.step_jacobians_many dynamics.py:774-802
 *   gato_pcg_batched / gato_btmv_batched      replace  blocktri.pcg / btmv          blocktri.py:105-173
 *   gato_shift_warm_start                     replaces mpc.shift_warm_start         mpc.py:85-89
 *   gato_merit_candidates                     replaces sqp.merit / merit_many       sqp.py:111-166
 *   gato_best_of_batch                        replaces the best-of-batch argmin     mpc.py:283-298
 *   gato_select_hypothesis                    replaces mpc.select_hypothesis        mpc.py:130-147
 *   gato_solve_host / gato_mpc_advance        one control step of _MpcEngine.advance mpc.py:240-274
 *
 * The reference is pure Python and has no FFI of its own; INTEGRATION.md shows the ctypes
 * stub a maintainer would add to trajbatch/batch.py to call this library.
 *
 * Conventions
 *   - plain C, no torch / C++ types; every pointer in gato_buffers and in the operator
 *     entry points is a DEVICE pointer owned by the caller (the library never frees them);
 *   - all floating point data is IEEE binary64, C-contiguous, packed by solve then knot
 *     (blocktri.py:5-6);
 *   - every call is asynchronous on the given stream (a cudaStream_t passed as void*),
 *     never synchronises the host, and returns 0 or a negative GATO_E_* code; the text of
 *     the last error is kept per handle (gato_last_error) -- nothing is thrown across the ABI;
 *   - a handle is not thread safe: one handle per (device, stream).
 */
#ifndef GATO_B200_H
#define GATO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GATO_ABI_VERSION 1

/* model ids: the reference's analytic models (dynamics.py:145,190,255,388) + iiwa14 */
#define GATO_MODEL_DOUBLE_INTEGRATOR 0 /* params: [dims (1..7), mass]                         */
#define GATO_MODEL_PENDULUM 1          /* params: [mass, length, gravity, damping]             */
#define GATO_MODEL_CARTPOLE 2          /* params: [cart_mass, pole_mass, pole_length, gravity] */
#define GATO_MODEL_TWO_LINK_ARM 3      /* params: [m1, m2, l1, l2, gravity, joint_damping]     */
#define GATO_MODEL_IIWA14 4            /* params: none (table frozen in model_iiwa14.cuh)       */

/* error codes */
#define GATO_OK 0
#define GATO_E_INVALID -1     /* bad argument / unsupported dimension */
#define GATO_E_CUDA -2        /* CUDA runtime error (see gato_last_error) */
#define GATO_E_UNBOUND -3     /* gato_solve before gato_bind */
#define GATO_E_NOMEM -4

/* per-solve status words written to gato_buffers.info[:, GATO_INFO_STATUS] */
#define GATO_STATUS_OK 0
#define GATO_STATUS_FACTORIZATION 1 /* errors.FactorizationError (errors.py:12) */
#define GATO_STATUS_PCG_BREAKDOWN 2 /* errors.PcgBreakdownError  (errors.py:24) */

/* which block failed to factor (info[:, GATO_INFO_FAIL_BLOCK]) */
#define GATO_BLOCK_Q 0 /* "Q_{knot}"                 qpform.py:305-309 */
#define GATO_BLOCK_R 1 /* "R_{knot}"                 qpform.py:310-311 */
#define GATO_BLOCK_S 2 /* "S diagonal block {knot}"  qpform.py:352-353 */

/* layout of the int32 info row of one solve */
#define GATO_INFO_WORDS 8
#define GATO_INFO_N_RECORDS 0  /* number of IterationRecords written (len(trace))       */
#define GATO_INFO_CONVERGED 1  /* SqpResult.converged                                   */
#define GATO_INFO_STATUS 2     /* GATO_STATUS_*                                         */
#define GATO_INFO_FAIL_ITER 3  /* SQP iteration of the failure                          */
#define GATO_INFO_FAIL_KNOT 4  /* FactorizationError.knot                               */
#define GATO_INFO_FAIL_BLOCK 5 /* GATO_BLOCK_*                                          */
#define GATO_INFO_FAIL_AUX 6   /* failing pivot (factorization) / PCG iteration (breakdown) */
#define GATO_INFO_RETRIES 7    /* breakdown count of the failing iteration              */

/* layout of one fp64 trace row == one sqp.IterationRecord (sqp.py:81-92) */
#define GATO_TRACE_WORDS 8
#define GATO_TRACE_MERIT 0
#define GATO_TRACE_CONSTRAINT_L1 1
#define GATO_TRACE_ALPHA 2 /* NaN encodes alpha=None (tolerance exit, sqp.py:261-272) */
#define GATO_TRACE_RHO 3
#define GATO_TRACE_PCG_ITERATIONS 4
#define GATO_TRACE_ACCEPTED 5
#define GATO_TRACE_STEP_INF_NORM 6
#define GATO_TRACE_ITERATION 7

/* gato_config.flags */
#define GATO_FLAG_UNFUSED 1 /* keep form_schur in its own kernel and write the plain stage arrays (Sdiag, Soff, Linv,
                               Lfac, the matrix record) even where the PCG kernel could form the system itself */
#define GATO_FLAG_FUSED 2   /* form the Schur system inside the PCG kernel wherever that kernel supports it, also for
                               batches below the size from which it pays (default: decided by batch x horizon) */

#define GATO_FLAG_UNTIMED 4 /* gato_solve / gato_solve_mpc record no CUDA events around the launch (two event records cost
                               ~5 us of device time per launch: a caller that times the stream itself, or does not
                               time at all, switches them off); gato_last_solve_ms then fails with GATO_E_INVALID */

typedef struct gato_config {
  int32_t abi_version; /* GATO_ABI_VERSION */
  int32_t model_id;
  int32_t batch;       /* M */
  int32_t horizon;     /* N (stage knots); X has N+1 rows */
  int32_t state_dim;   /* n, checked against the model */
  int32_t control_dim; /* m */
  int32_t force_dim;   /* fdim */
  /* sqp.SolverSettings (sqp.py:56-77) */
  int32_t max_sqp_iterations;
  int32_t pcg_max_iterations; /* 0 => 10 * (N+1) * n (blocktri.py:78-81) */
  int32_t num_shrinks;        /* candidates = num_shrinks + 1 (sqp.py:39-52) */
  int32_t regularize_r;
  int32_t pcg_retry_limit;
  int32_t loop_mode; /* 0 auto, 1 CUDA-graph WHILE node, 2 graph of unrolled passes, 3 plain stream launches */
  int32_t flags;     /* GATO_FLAG_* */
  double timestep;
  double pcg_tolerance;
  double mu;
  double beta;
  double rho_min;
  double rho_max;
  double rho_factor;
  double step_tolerance; /* NaN => None: run the fixed budget (sqp.py:65-66) */
  double feasibility_tolerance;
  double model_params[8];
} gato_config;

/* Device buffers of one batch. Inputs are read-only for the library; X, U are in/out. */
typedef struct gato_buffers {
  const double* x_start;  /* [M, n]                                   qpform.py:88   */
  const double* goal;     /* [M, N+1, n] (single goals pre-broadcast) qpform.py:66   */
  const double* Q;        /* [M, n, n]                                qpform.py:45   */
  const double* R;        /* [M, m, m]                                               */
  const double* QN;       /* [M, n, n]                                               */
  const double* force;    /* [M, N, fdim] sampled at k*h              qpform.py:113-123 */
  const double* rho_init; /* [M]                                      batch.py:63-74 */
  double* X;              /* [M, N+1, n] initial guess in, solution out */
  double* U;              /* [M, N, m]                                  */
  double* trace;          /* [M, max_sqp_iterations, GATO_TRACE_WORDS]  */
  int32_t* info;          /* [M, GATO_INFO_WORDS]                       */
} gato_buffers;

typedef struct gato_handle gato_handle;

/* Allocates the per-batch scratch (A, B, e, S, D^-1, gamma, lambda, dX, dU, merits ...)
 * once for (M, N, n, m) on the current device. */
int gato_create(const gato_config* cfg, gato_handle** out);
int gato_bind(gato_handle* h, const gato_buffers* bufs);
/* Runs every solve of the batch to termination, entirely on the device. */
int gato_solve(gato_handle* h, void* stream);
/* gato_solve with the warm-start preparation of a control step folded into the solve's first kernel (no launch of
 * its own; in the graph loop modes the first node's arguments are patched per call):
 *   shift_mode 0  plain gato_solve
 *   shift_mode 1  X, U shifted one knot left with the tail duplicated (gato_shift_warm_start), then the solve
 *   shift_mode 2  gato_mpc_advance(goal_path, path_len, path_stride, step), then the solve
 * One control period of _MpcEngine.advance (mpc.py:240-274) in a single launch. */
int gato_solve_mpc(gato_handle* h, void* stream, int32_t shift_mode, const double* goal_path, int64_t path_len,
                   int64_t path_stride, int64_t step);
/* X <- [X[1:], X[-1]], U <- [U[1:], U[-1]] for every solve, in place (mpc.py:85-89). */
int gato_shift_warm_start(gato_handle* h, void* stream);
/* One control period of a device-resident MPC loop (mpc.py:240-274), in place on the bound buffers:
 * x_start <- X[:, 1] (the predicted next state stands in for the measurement), X and U shifted one knot
 * left with the tail duplicated (mpc.py:85-89), and -- if goal_path is given -- the goal window advanced
 * to goal[k] = goal_path[min(step + k, path_len - 1)], k = 0..N. goal_path: device array [path_len, n]
 * shared by all solves (path_stride = 0) or one path per solve (path_stride = path_len * n doubles).
 * Writes the caller's x_start / goal / X / U buffers. Asynchronous. */
int gato_mpc_advance(gato_handle* h, void* stream, const double* goal_path, int64_t path_len,
                     int64_t path_stride, int64_t step);
/* One control step with HOST buffers in a single call (the MPC caller's inner loop, mpc.py:240-274):
 * copy `in_bytes` from (pinned) host memory to `dev_in`, optionally shift the warm start, run the
 * solve to termination, copy `out_bytes` from `dev_out` back to host memory and synchronise the
 * stream. dev_in / dev_out are caller-owned device addresses (typically spans of the buffers bound
 * with gato_bind); either copy may be skipped with 0 bytes.
 * Up to GATO_ZERO_COPY_MAX bytes per direction (environment, default 1 MiB, 0 = never) and with host buffers
 * that are pinned and device-mapped (cudaHostAlloc / torch pin_memory), no copy engine is involved: the solve's
 * first kernel reads the inputs across PCIe and the last kernel of each pass writes the rows of every finished
 * solve straight into host_out (when dev_out spans result arrays only; a small copy kernel otherwise).
 * Pageable memory and larger spans take cudaMemcpyAsync. Same bytes in host_out on every route. */
int gato_solve_host(gato_handle* h, void* stream, void* dev_in, const void* host_in, int64_t in_bytes,
                    int32_t shift_first, const void* dev_out, void* host_out, int64_t out_bytes);
/* Merit evaluation alone (sqp.py:111-166): for every solve of the bound batch, the L1 merit of the
 * candidates (X + alpha_c dX, U + alpha_c dU), alpha_c = beta^-c, c = 0..num_shrinks, and of the current
 * iterate itself. dX [M, N+1, n], dU [M, N, m]: device arrays (null = zero step). Results in the scratch
 * arrays "merits" / "viols" ([M, num_shrinks + 2]: the candidates, then alpha = 0). Asynchronous. */
int gato_merit_candidates(gato_handle* h, void* stream, const double* dX, const double* dU);
/* Best-of-batch selection on the device (mpc.py:283-298): index of the solve with the lowest final
 * merit among the solves without a failure status, first minimum on ties, -1 if every solve failed;
 * written to the device words *best_index / *best_merit (either may be null). Asynchronous. */
int gato_best_of_batch(gato_handle* h, void* stream, int32_t* best_index, double* best_merit);
/* Loop modes 2/3 enqueue exactly max_sqp_iterations passes; a PCG-breakdown retry (sqp.py:240-248)
 * consumes a pass without advancing its solve. gato_pending synchronises the stream and reports
 * how many solves are still active; gato_resume enqueues further passes. In loop mode 1 (WHILE
 * graph node) the device loops until every solve has terminated and pending is always 0. */
int gato_pending(gato_handle* h, void* stream, int32_t* pending);
int gato_resume(gato_handle* h, void* stream, int32_t passes);
int gato_loop_mode(const gato_handle* h);
/* 1 if this handle forms the Schur system of solves with diagonal weights inside its PCG kernel (no k_schur, no
 * matrix record for them; GATO_FLAG_* and the batch size decide), 0 if every solve goes through k_schur. */
int gato_fused(const gato_handle* h);
/* Device pointer + element count of an internal stage array, for stage-by-stage parity
 * tests: "A","B","e","grad","hinv","Sdiag","Soff","Dinv","gamma","lam","dX","dU","merits",
 * "viols","state","pcg_iters". Valid until gato_destroy. */
int gato_scratch(gato_handle* h, const char* name, void** dev_ptr, int64_t* count);
/* synchronous device->host copy of the first `bytes` bytes of a stage array (tests) */
int gato_read_scratch(gato_handle* h, const char* name, void* host_dst, int64_t bytes);
/* number of kernel launches issued by the last gato_solve (graph nodes count per replay) */
int64_t gato_launch_count(const gato_handle* h);
/* device time of the last gato_solve / gato_solve_mpc in milliseconds, measured with CUDA events on the
 * launching stream; synchronises on the end event. gato_solve_host records no events (its caller times the
 * call); GATO_E_INVALID if the handle has not run a timed solve yet. */
int gato_last_solve_ms(gato_handle* h, float* ms);
/* gato_solve with CUDA events between the kernels of every pass (plain stream launches):
 * ms[0..5] = hessinv, linearize, schur, pcg, linesearch, update totals; ms[6] prologue; ms[7] all. */
int gato_solve_profiled(gato_handle* h, void* stream, float* ms);
/* sustained fp64 FMA throughput of the current GPU in TFLOP/s (roofline denominator R1) */
int gato_measure_fp64_peak(double* tflops);
const char* gato_last_error(const gato_handle* h);
void gato_destroy(gato_handle* h);

/* ---- operator entry points (stateless; same kernels as the solve) ---- */

/* out[r] = one RK4 step of model from (X[r], U[r]) under force F[r], rows independent. */
int gato_step_many(int32_t model_id, const double* model_params, int64_t rows, const double* X,
                   const double* U, const double* F, double timestep, double* out, void* stream);
/* Hypothesis selection (mpc.py:130-147): every candidate force forces[j] (constant over the period)
 * rolls the plant from x_prev with the applied control held for `substeps` RK4 steps of h_plant
 * (simulate_plant, dynamics.py:843-864); *best = index of the candidate whose prediction is closest to
 * x_meas in the 2-norm (positions only if position_only), first minimum on ties; errors[candidates]
 * (optional) receives the distances. Device pointers, asynchronous. */
int gato_select_hypothesis(int32_t model_id, const double* model_params, int32_t candidates,
                           const double* x_prev, const double* u_applied, const double* x_meas,
                           const double* forces, double h_plant, int32_t substeps, int32_t position_only,
                           double* errors, int32_t* best, void* stream);
/* A[r] (n x n), B[r] (n x m): exact Jacobians of the RK4 map at row r. */
int gato_step_jacobians_many(int32_t model_id, const double* model_params, int64_t rows,
                             const double* X, const double* U, const double* F, double timestep,
                             double* A, double* B, void* stream);
/* y = densify(M) v for a batch of symmetric block-tridiagonal matrices stored as diag [nb, bd, bd] +
 * sub-diagonal [nb-1, bd, bd] blocks (blocktri.py:105-120: diagonal, sub-diagonal, super-diagonal term). */
int gato_btmv_batched(int32_t systems, int32_t n_blockrows, int32_t block_dim, const double* diag,
                      const double* off, const double* v, double* y, void* stream);
/* Batched PCG on explicit block-tridiagonal S and preconditioner Phi^-1 (both stored as
 * diag [nb, bd, bd] + sub-diagonal [nb-1, bd, bd] blocks per system). status: 0 ok,
 * 2 breakdown (iters = breakdown iteration). */
int gato_pcg_batched(int32_t systems, int32_t n_blockrows, int32_t block_dim, const double* S_diag,
                     const double* S_off, const double* gamma, const double* P_diag,
                     const double* P_off, double tolerance, int32_t max_iterations, double* lam,
                     int32_t* iterations, int32_t* converged, int32_t* status, double* residual,
                     void* stream);

const char* gato_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GATO_B200_H */
