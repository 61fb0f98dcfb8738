/*
 * cvxreg_b200.h -- C ABI of the B200 pair-sweep solver (libcvxreg_b200.so).
 *
 * Drop-in for the singleton-block dual path of the reference solver
 * (arXiv 1407.7220 `cvxreg`, /root/reference/proj/core). Plain pointers and
 * sizes only; every function returns a cr_status and never throws. The C++
 * shim in include/cvxreg_b200/papg.hpp maps statuses back to the reference's
 * exceptions (std::invalid_argument / std::runtime_error).
 *
 * Reference interfaces replaced (file:line under proj/core/):
 *   cr_papg_*            papg_solve / dual_gradient_ascent      include/cvxreg/papg.hpp:75-82
 *                        (loop: src/papg.cpp:136-283)
 *   cr_sigma_C           estimate_sigma_max(op_C(ops))           src/operators.cpp:302-339, :353-369
 *                        (called from DualDecomposition ctor     src/papg.cpp:68)
 *   cr_get_primal        PapgResult::point                       include/cvxreg/papg.hpp:61
 *   cr_get_theta         PapgResult::dual (DualPoint)            include/cvxreg/types.hpp:50-53
 *   cr_get_rows          DualGradientResult::C_eta               include/cvxreg/papg.hpp:25
 *   cr_gen_instance      gen_instance                            src/testgen.cpp:36-87
 *   cr_prepare_problem   prepare_problem                         src/preprocess.cpp:50-65
 *   cr_certificate       certificate_for_iterate                 src/papg.cpp:298-303
 *   cr_alcc_solve        alcc_solve (standalone ALCC)            include/cvxreg/alcc.hpp:134-136
 *                        (alcc_core src/alcc.cpp:54-191, MAPG src/engines.cpp:57-106)
 *   cr_alcc_multiplier   AlccResult::multiplier                  include/cvxreg/alcc.hpp:110-118
 *   cr_sigma_A           estimate_sigma_max(op_A1 / op_A2)       src/operators.cpp:341-351
 *   cr_set_partition     make_partition + DualDecomposition      src/dataset.cpp:119-130,
 *                        (general-K P-APG(ALCC))                 src/papg.cpp:66-132
 *
 * Threading: a handle is confined to one host thread. Distinct handles may
 * be driven concurrently. Sharded runs use one handle (and one process) per
 * GPU; rank r owns pair rows [row_begin, row_end) of the N x N pair matrix.
 */
#ifndef CVXREG_B200_H
#define CVXREG_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CR_OK = 0,
  CR_EINVAL = 1,      /* shape / precondition (reference: std::invalid_argument) */
  CR_ENOMEM = 2,      /* device or pinned allocation failed */
  CR_ECUDA = 3,       /* CUDA runtime error */
  CR_ENCCL = 4,       /* NCCL error */
  CR_ENONFINITE = 5,  /* "papg: non-finite dual gradient" (papg.cpp:184-185) */
  CR_ESTATE = 6       /* call out of order (e.g. iterate before begin) */
} cr_status;

/* termination reasons, metrics.hpp:41 TermReason */
enum { CR_THRESHOLDS = 0, CR_ITER_BUDGET = 1, CR_TIME_BUDGET = 2, CR_ERROR = 3 };

typedef struct cr_handle cr_handle;

/* PapgConfig (papg.hpp:7-21) minus the inner ALCC settings, which the
   singleton closed form does not use, plus two device knobs. */
typedef struct {
  double gamma;             /* 1e-3 */
  double B_theta;           /* <= 0: adaptive, start at 10 sqrt(N) */
  int32_t adaptive_B_theta; /* 1 */
  int32_t max_restarts;     /* 6 */
  double gap_norm_tol;      /* 1e-6 */
  double infeas_norm_tol;   /* 1e-1 */
  int64_t max_iters;        /* 100000 */
  double max_seconds;       /* 7200 */
  double inner_tol_floor;   /* 1e-6: enters the g* cushion 2 tol K (papg.cpp:198) */
  double final_resolve_tol; /* 1e-10 */
  int32_t record_history;   /* 1 */
  int32_t use_momentum;     /* 1: papg_solve, 0: dual_gradient_ascent */
  double sigma_C;           /* > 0: use this sigma_max(C) instead of estimating it */
  int32_t graph_iters;      /* iterations per CUDA graph launch; <= 0: auto */
  int32_t workers;          /* K-block partition: concurrent block solves; <= 0: 16 */
} cr_papg_config;

/* device history capacity (snapshots) of one solve */
#define CR_HISTORY_CAP 4000000

/* one MetricsSnapshot (metrics.hpp:13-22) */
typedef struct {
  double iter, objective, reg_objective, infeas_raw, infeas_norm, gap_raw, gap_norm, wall_time_s;
} cr_snapshot;

/* PapgResult scalars (papg.hpp:60-69) + SolveReport (metrics.hpp:45-54) */
typedef struct {
  int64_t iters;
  int32_t reason;
  int32_t restarts;
  int32_t saturated;
  int32_t sigma_iters;
  int32_t sigma_converged;
  int32_t history_truncated; /* 1: more than CR_HISTORY_CAP iterations ran; the
                                history holds the first CR_HISTORY_CAP snapshots */
  double g_final;
  double delta_estimate;
  double sigma_C;
  double L_g;
  double B_theta;
  double wall_seconds;     /* device clock, begin -> stop */
  double sigma_seconds;    /* power iteration time (0 if injected) */
  double loop_seconds;     /* dual loop time */
  double last_gap_norm;
  double last_infeas_norm;
} cr_papg_result;

/* ---- handle lifetime ---------------------------------------------------- */
/* Copies X (N x n, row-major) and the SHIFTED observations ybar (N) to the
   device. Rows [row_begin, row_end) of the pair matrix are owned by this
   handle (pass 0, N for a single GPU). gamma > 0. */
cr_status cr_create(const double *X, const double *ybar_shifted, int64_t N, int64_t n,
                    double gamma, int device, int64_t row_begin, int64_t row_end,
                    cr_handle **out);
void cr_destroy(cr_handle *h);
const char *cr_last_error(const cr_handle *h);
const char *cr_status_string(cr_status s);

/* ---- multi-GPU: one handle per rank, NCCL allreduce over NVLink ----------- */
cr_status cr_nccl_unique_id(uint8_t id_out[128]);
cr_status cr_attach_nccl(cr_handle *h, const uint8_t id[128], int rank, int world);
/* Host-exchange seam (tests / emulation): doubles of the per-iteration
   aggregate payload (canonical-block mode: of all D block payloads). */
int64_t cr_exchange_len(const cr_handle *h);
/* GPU-count-invariant sums (results must not depend on the
   worker count; the reference gathers block results in block order,
   papg.cpp:122-129). Rows are cut into D canonical blocks
   [floor(j N / D), floor((j + 1) N / D)); the handle's rows must be a union of
   blocks (world | D with the balanced shards of cr_create's callers). Every
   block is swept by its own launches with its own CTA shares, its payload
   reduced on its own, the payloads of all ranks are allgathered (instead of
   the allreduce) and summed in block order 0..D-1 on every rank. theta, y and
   xi after k iterations are then bitwise the same on 1, 2, 4 ... GPUs for a
   fixed D. D = 0 (default) turns it off. Call before cr_papg_begin;
   singleton blocks only. cr_canonical_blocks reports D, the handle's first
   block and its block count. */
cr_status cr_set_canonical_blocks(cr_handle *h, int32_t D);
cr_status cr_canonical_blocks(const cr_handle *h, int32_t *D, int32_t *first, int32_t *count);

/* ---- sigma_max(C) by power iteration (operators.cpp:302-339) ------------- */
cr_status cr_sigma_C(cr_handle *h, double tol, int32_t max_iters, double *sigma,
                     int32_t *iters, int32_t *converged);

/* ---- the dual loop ------------------------------------------------------ */
/* theta0: canonical [theta_cross (N(N-1)); theta_pos (N)] or NULL (= 0).
   Estimates sigma_C unless cfg->sigma_C > 0. */
cr_status cr_papg_begin(cr_handle *h, const cr_papg_config *cfg, const double *theta0);
/* Runs up to max_steps more iterations (stops early at termination).
   *done = iterations completed so far; *stopped = 1 once terminated. */
cr_status cr_papg_iterate(cr_handle *h, int64_t max_steps, int64_t *done, int32_t *stopped);
/* Same loop, one iteration at a time with the cross-shard exchange done by
   the caller: local phase, then the caller sums the exchange payloads of all
   shards (cr_exchange_get/put), then the finish phase. */
cr_status cr_iter_local(cr_handle *h);
cr_status cr_exchange_get(cr_handle *h, double *buf);
cr_status cr_exchange_put(cr_handle *h, const double *buf);
cr_status cr_iter_finish(cr_handle *h, int32_t *stopped);
/* Final re-solve at theta1 (papg.cpp:265-282): fills res, y (N), xi (N*n) and,
   when history != NULL, res->iters snapshots. */
cr_status cr_papg_finish(cr_handle *h, cr_papg_result *res, double *y, double *xi,
                         cr_snapshot *history);
/* Begin a new solve warm-started from this handle's device-resident theta1
   (papg.cpp:159-164; the gamma continuation of runner.cpp:258-259, 305, 322
   without a host round trip of the N^2 multipliers). */
cr_status cr_papg_begin_resume(cr_handle *h, const cr_papg_config *cfg);
/* Replace the shifted observations (e.g. prepare_problem at the next gamma). */
cr_status cr_set_observations(cr_handle *h, const double *ybar_shifted);
/* begin + iterate to termination + finish */
cr_status cr_papg_solve(cr_handle *h, const cr_papg_config *cfg, const double *theta0,
                        cr_papg_result *res, double *y, double *xi, cr_snapshot *history);

/* theta1 of this shard's rows in canonical order: out receives
   theta_cross[row_begin*(N-1) .. row_end*(N-1)) followed by theta_pos (N). */
cr_status cr_get_theta(cr_handle *h, double *out);
/* C eta of the last loop iteration (the residual rows at eta(theta2)), same
   layout as cr_get_theta. */
cr_status cr_get_rows(cr_handle *h, double *out);
/* The same two exports for global pair rows l1 in [row_begin, row_end) of
   this shard only ((row_end - row_begin) x (N-1) cross entries, canonical
   order, then the N pos rows): spot checks at sizes whose full dual vector
   does not fit the host (BASELINE cfg 5: 80 GB). Singleton blocks only. */
cr_status cr_get_theta_rows(cr_handle *h, int64_t row_begin, int64_t row_end, double *out);
cr_status cr_get_rows_window(cr_handle *h, int64_t row_begin, int64_t row_end, double *out);
/* device timing of the last cr_papg_iterate call and the number of kernel
   launches it issued (for bench.py) */
cr_status cr_last_timing(const cr_handle *h, double *seconds, int64_t *launches,
                         double *sweep_seconds);
/* Durations (s) of the sweep launches the last cr_papg_iterate call bracketed
   with CUDA events (every launch of a call of at most 64 iterations, else every
   8th; CRB_SWEEP_EVENTS=k overrides), in launch order: up to cap into out,
   *count = how many there were. */
cr_status cr_last_sweep_times(const cr_handle *h, double *out, int64_t cap, int64_t *count);
/* Sharded runs: device time of the per-iteration ncclAllReduce in the last
   cr_papg_iterate call, from CUDA events around it in the same iterations whose
   sweeps are bracketed (scaled to all iterations when sampled); 0 otherwise. */
cr_status cr_last_exchange_seconds(const cr_handle *h, double *seconds);
/* sweep kernel variant chosen for this handle: 0 = CUDA-core DFMA,
   1 = FP64 tensor-core DMMA (override with CRB_SWEEP=dfma|mma) */
int32_t cr_sweep_variant(const cr_handle *h);
/* Multipliers written by the P-APG sweeps since the last reset (DMMA sweep:
   a 32-byte sector holding no changed multiplier is not rewritten, a sector
   with a change is written whole), optionally resetting the counter. */
cr_status cr_sweep_store_count(cr_handle *h, uint64_t *count, int32_t reset);
/* Time k sweep-kernel launches alone on the handle's stream with CUDA events
   (the dominant kernel in isolation, for the roofline). */
cr_status cr_time_sweep(cr_handle *h, int32_t k, double *avg_seconds);

/* ---- one-shot metric sweeps on a given point (metrics.cpp) --------------- */
/* |(A1 y + A2 xi)_-|_2 over all N(N-1) rows and its /sqrt(N^2-N) form
   (metrics.cpp:8-15); shift-invariant, so original or shifted y both work. */
cr_status cr_infeasibility(cr_handle *h, const double *y, const double *xi, double out2[2]);
/* theta1 . C eta with the handle's current theta1 (metrics.cpp:17-30). */
cr_status cr_duality_gap(cr_handle *h, const double *y, const double *xi, double out2[2]);
/* max_l y_l + xi_l.(x_q - x_l) for Q query points Xq (Q x n) (metrics.cpp:32-48). */
cr_status cr_evaluate_estimator(cr_handle *h, const double *y, const double *xi,
                                const double *Xq, int64_t Q, double *out);
/* y'_l = estimator(x_l), an exactly feasible point (metrics.cpp:50-56). */
cr_status cr_repair_feasibility(cr_handle *h, const double *y, const double *xi, double *y_out);

/* ---- standalone ALCC (alcc_solve) ------------------ */
/* AlccConfig (alcc.hpp:71-83) plus the solve's inputs that the reference
   takes from ProblemBounds / estimate_sigma_max. */
typedef struct {
  double mu1;              /* 1 */
  double tau1_scale;       /* 1e-2 */
  double alpha1_scale;     /* 1e-3 */
  double c;                /* 5 (> 1) */
  double kappa;            /* 0.5 (> 0) */
  int64_t max_outer;       /* 30 */
  int64_t mapg_cap;        /* 200000 */
  double infeas_norm_tol;  /* 1e-1 */
  double gap_norm_tol;     /* 1e-6 */
  double max_seconds;      /* inf */
  int32_t record_history;  /* 1 */
  int32_t pad_;
  double sigma_A1;         /* > 0: inject sigma_max(A1), else estimated on the device */
  double sigma_A2;         /* > 0: inject sigma_max(A2) */
  double Bbar_y;           /* ball radii (ProblemBounds, preprocess.cpp:9-48) */
  double Bbar_xi;
} cr_alcc_config;

/* AlccResult scalars (alcc.hpp:110-118) + SolveReport */
typedef struct {
  int64_t outer_iters;
  int64_t mapg_iters_total;
  int32_t reason;
  int32_t hit_cap_any;     /* some MAPG call ran to its l_max */
  int32_t sigma_A1_iters;  /* power iterations (0 if injected) */
  int32_t sigma_A2_iters;
  double certified_gap;
  double infeas_raw;
  double gap_raw;
  double objective;
  double wall_seconds;
  double sigma_A1;
  double sigma_A2;
  double sigma_seconds;
  double mapg_seconds;     /* device time of the MAPG loops (CUDA events) */
  int64_t launches;        /* kernels enqueued by the MAPG loops (incl. halted no-ops) */
} cr_alcc_result;

/* sigma_max(A1) (which = 1) or sigma_max(A2) (which = 2) by the reference's
   power method on the full row set (closed-form O(N n^2) steps). */
cr_status cr_sigma_A(cr_handle *h, int32_t which, double tol, int32_t max_iters, double *sigma,
                     int32_t *iters, int32_t *converged);
/* alcc_solve from the warm point (warm_y: N shifted frame, warm_xi: N*n),
   centres (ybar, 0). Unsharded handles only; overwrites any P-APG state on the
   handle. y_out / xi_out / history (max_outer) / mapg_iters (max_outer) may be
   NULL. */
cr_status cr_alcc_solve(cr_handle *h, const cr_alcc_config *cfg, const double *warm_y,
                        const double *warm_xi, double *y_out, double *xi_out,
                        cr_snapshot *history, int64_t *mapg_iters, cr_alcc_result *res);
/* lambda = mu_k (theta_k - R(y, xi))_+ of the last outer step for pair rows
   l1 in [row_begin, row_end), canonical order ((row_end-row_begin) x (N-1)). */
cr_status cr_alcc_multiplier(cr_handle *h, int64_t row_begin, int64_t row_end, double *out);
/* Time k penalty-sweep launches (theta_k at the handle's records, read-only). */
cr_status cr_time_penalty_sweep(cr_handle *h, int32_t k, double *avg_seconds);

/* ---- general-K partition: P-APG(ALCC) ------------- */
/* make_partition (dataset.cpp:119-130) + DualDecomposition (papg.cpp:66-86):
   K blocks of nbar = N/K consecutive points (N % K == 0, nbar >= n+1); every
   block QP is solved by the ALCC (alcc_solve_block, alcc.cpp:222-258) with
   the inner config, warm-started from the previous block minimiser; the block
   balls use the feasible affine point (feas_y: N shifted frame, feas_xi: N*n).
   K == N (or 0) selects the singleton closed form. Call before cr_papg_begin;
   unsharded handles only. theta / C eta then use the general cross ordering
   (indexing.hpp:9-37), N(N-nbar) + N entries. */
cr_status cr_set_partition(cr_handle *h, int64_t K, const double *feas_y, const double *feas_xi,
                           const cr_alcc_config *inner);
/* MAPG iterations and seconds spent in block solves since cr_papg_begin, the
   within-block sigma(A1) and the per-block sigma(A2) (K entries, may be NULL). */
cr_status cr_partition_stats(const cr_handle *h, int64_t *inner_iters, double *inner_seconds,
                             double *sigma_A1, double *sigma_A2);

/* ---- host utilities (no device) ----------------------------------------- */
/* kinds: 0 quadratic, 1 exponential, 2 affine-noiseless, 3 custom-1d
   (testgen.hpp:18-25); 10 sqnorm-uniform, 11 maxaffine-uniform,
   12 lse-uniform (BASELINE.json configs). */
cr_status cr_gen_instance(int32_t kind, int64_t N, int64_t n, double noise, uint64_t seed,
                          int64_t pieces, double *X, double *y);
/* prepare_problem: ys_shifted (N), shift, feasible affine point (shifted
   frame), bounds4 = {B_theta, Bbar_y, Bbar_xi, gamma} */
cr_status cr_prepare_problem(const double *X, const double *y, int64_t N, int64_t n,
                             double gamma, double *ys_shifted, double *shift, double *feas_y,
                             double *feas_xi, double *bounds4);
void cr_certificate(double gamma, double delta, double B_xi_estimate, double sigma_max_C,
                    double out2[2]);
double cr_momentum_next(double t);

#ifdef __cplusplus
}
#endif
#endif
