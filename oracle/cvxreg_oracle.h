/*
 * cvxreg_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference solver path (arXiv 1407.7220, `cvxreg`,
 * /root/reference/proj/core) in the singleton-block closed form. It is the
 * parity checker for the CUDA path and the CPU baseline timed by bench.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product library never links it.
 *
 * Parity status: PINNED to the reference's own code. The reference's proj/core
 * sources compile unmodified into oracle/_ref/libcvxreg_ref.so (oracle/Makefile
 * target `ref`: Eigen calls served by oracle/eigen_shim, alcc.cpp through
 * ref_build/alcc_tu.cpp because of its arity error at alcc.cpp:200-203; the
 * singleton mode that make_partition rejects, dataset.cpp:125-126, is reached
 * with Partition{N, 1} built directly). tests/test_oracle_vs_reference.py
 * compares this restatement with it live and against the committed outputs
 * tests/golden/ref_*.npz (scripts/make_ref_golden.py): operators, generators,
 * PRNG streams and the singleton P-APG trajectory agree bitwise or to 1e-13,
 * sigma_max with identical step counts, general K and ALCC with identical
 * iteration counts. The SPEC.md worked examples and analytic known-answer
 * tests (tests/test_oracle_spec.py) stay as a second pin. See DESIGN.md
 * section "Oracle".
 */
#ifndef CVXREG_ORACLE_H
#define CVXREG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* generator kinds: 0..3 restate testgen.cpp:36-87; 10..12 are the BASELINE.json kinds */
enum {
  CRO_GEN_QUADRATIC = 0,
  CRO_GEN_EXPONENTIAL = 1,
  CRO_GEN_AFFINE_NOISELESS = 2,
  CRO_GEN_CUSTOM_1D = 3,
  CRO_GEN_SQNORM_UNIFORM = 10,    /* cfg 1, 4: y = |x|^2 + eps, x~U[-1,1]^n, eps~U[-a,a] */
  CRO_GEN_MAXAFFINE_UNIFORM = 11, /* cfg 2, 5: y = max_i a_i.x + b_i + eps */
  CRO_GEN_LSE_UNIFORM = 12        /* cfg 3:    y = log sum_k exp(a_k.x) + eps */
};

/* termination reasons, metrics.hpp:41 */
enum { CRO_THRESHOLDS = 0, CRO_ITER_BUDGET = 1, CRO_TIME_BUDGET = 2, CRO_ERROR = 3 };

typedef struct {
  double gamma;            /* papg.hpp:8  */
  double B_theta;          /* <= 0: adaptive 10 sqrt(N) (papg.cpp:149-150) */
  int32_t adaptive_B_theta;
  int32_t max_restarts;
  double gap_norm_tol;
  double infeas_norm_tol;
  int64_t max_iters;
  double max_seconds;
  double inner_tol_floor;
  double final_resolve_tol;
  int32_t record_history;
  int32_t use_momentum;    /* 1: papg_solve, 0: dual_gradient_ascent (papg.cpp:287-296) */
  double sigma_C;          /* > 0: inject sigma_C (skips power iteration) */
  int32_t threads;         /* <= 1: literal single-thread loops; > 1: OpenMP rows */
  int32_t pad_;
} cro_config;

typedef struct {
  /* caller-owned output arrays (may be NULL) */
  double *y;       /* N */
  double *xi;      /* N*n */
  double *theta;   /* N(N-1)+N canonical [theta_cross; theta_pos] */
  double *c_eta;   /* N(N-1)+N: C eta of the LAST loop iteration */
  double *history; /* max_iters * 8: iter, objective, reg_objective, infeas_raw,
                      infeas_norm, gap_raw, gap_norm, wall_time_s */
  /* scalars */
  int64_t iters;
  int32_t reason;
  int32_t restarts;
  int32_t saturated;
  int32_t sigma_iters;
  int32_t sigma_converged;
  int32_t pad_;
  double g_final;
  double delta_estimate;
  double sigma_C;
  double L_g;
  double B_theta;
  double wall_seconds;
} cro_result;

/* PRNG (rng.hpp:7-59) */
uint64_t cro_rng_draws(uint64_t seed, uint64_t tag, int64_t count, int kind, double *out);

/* generators; pieces = number of affine pieces / LSE terms for kinds 11/12.
   returns 0 on success, -1 on invalid arguments, -2 on duplicate rows. */
int cro_gen_instance(int kind, int64_t N, int64_t n, double noise, uint64_t seed,
                     int64_t pieces, double *X /*N*n row-major*/, double *y /*N*/);

/* preprocess.cpp:9-65. bounds4 = {B_theta, Bbar_y, Bbar_xi, gamma}.
   feas_y (N) and feas_xi (N*n) are in the shifted frame. */
int cro_prepare(const double *X, const double *y, int64_t N, int64_t n, double gamma,
                double *ys_shifted, double *shift, double *feas_y, double *feas_xi,
                double *bounds4, double *intercept, double *slope /*n*/);

/* operators.cpp:128-180 in singleton order (K = N, nbar = 1) */
void cro_apply_C(const double *X, int64_t N, int64_t n, const double *y, const double *xi,
                 double *out /*N(N-1)+N*/);
void cro_apply_C_T(const double *X, int64_t N, int64_t n, const double *theta,
                   double *out_y /*N*/, double *out_xi /*N*n*/);

/* operators.cpp:302-339 with op_C (:353-369) */
int cro_sigma_C(const double *X, int64_t N, int64_t n, double tol, int max_iters,
                double *sigma, int *iters, int *converged);

/* papg.cpp:136-283 (singleton closed form). theta0: canonical or NULL. */
int cro_papg(const double *X, const double *ys_shifted, int64_t N, int64_t n,
             const cro_config *cfg, const double *theta0, cro_result *res);

/* Memory-light restatement of cro_papg (zero start): keeps only the
   per-iteration primal and step scalars and recomputes every pair's
   multiplier history on each pass (O(k^2 N^2 n) work, O(k N n) memory), for
   sizes whose N^2 arrays do not fit the host (BASELINE cfg 4, 5). One thread:
   bitwise equal to cro_papg with one thread. theta_rows / c_eta_rows (may be
   NULL) receive theta1 and C eta of the last loop iteration for the cross rows
   of the points l1 = rows[0..nrows) (strictly increasing), each in canonical
   order ((N-1) entries), followed by the N pos rows; res->theta and
   res->c_eta are not used. */
int cro_papg_replay(const double *X, const double *ys_shifted, int64_t N, int64_t n,
                    const cro_config *cfg, const int64_t *rows, int64_t nrows,
                    double *theta_rows, double *c_eta_rows, cro_result *res);

/* metrics.cpp:8-56 (full row set, canonical order) */
void cro_infeasibility(const double *X, int64_t N, int64_t n, const double *y, const double *xi,
                       double out2[2]);
void cro_duality_gap(const double *X, int64_t N, int64_t n, const double *theta, const double *y,
                     const double *xi, double out2[2]);
double cro_evaluate_estimator(const double *X, int64_t N, int64_t n, const double *y,
                              const double *xi, const double *xq);
void cro_repair_feasibility(const double *X, int64_t N, int64_t n, const double *y,
                            const double *xi, double *y_out);

/* projections.hpp:9-13, engines.hpp:11-13, papg.cpp:298-303 */
void cro_project_nonneg_ball(double *v, int64_t len, double radius);
double cro_momentum_next(double t);
void cro_certificate(double gamma, double delta, double B_xi, double sigma, double out2[2]);
int64_t cro_cross_position(int64_t N, int64_t K, int64_t l1, int64_t l2);

/* ---- standalone ALCC (alcc.cpp:54-208, engines.cpp:57-106) ---- */
typedef struct {           /* alcc.hpp:71-83 */
  double mu1, tau1_scale, alpha1_scale, c, kappa;
  int64_t max_outer, mapg_cap;
  double infeas_norm_tol, gap_norm_tol, max_seconds;
  int32_t record_history;
  int32_t threads;         /* <= 1: literal loops; > 1: OpenMP rows */
} cro_alcc_config;

typedef struct {
  double *y, *xi;          /* N, N*n (caller-owned, may be NULL) */
  double *multiplier;      /* N(N-1): lambda = mu (theta - R)_+ of the last outer step */
  double *history;         /* max_outer * 8 */
  int64_t *mapg_iters;     /* max_outer: MAPG iterations per outer step */
  int64_t outer_iters, mapg_iters_total;
  int32_t reason, hit_cap_any;
  double certified_gap, infeas_raw, gap_raw, objective, wall_seconds, sigma_A1, sigma_A2;
} cro_alcc_result;

/* operators.cpp:302-339 on op_A1 (which = 1) / op_A2 (which = 2) */
int cro_sigma_A(const double *X, int64_t N, int64_t n, int which, double tol, int max_iters,
                double *sigma, int *iters, int *converged);
/* alcc_solve (alcc.cpp:193-208, arity fixed) -> alcc_core with centres (ybar, 0).
   sigma_A1/2 <= 0: estimated. returns 0, -1 invalid, -4 non-finite P_1,
   -5 non-finite MAPG gradient. */
int cro_alcc(const double *X, const double *ys, int64_t N, int64_t n, double gamma,
             double Bbar_y, double Bbar_xi, double sigma_A1, double sigma_A2,
             const double *warm_y, const double *warm_xi, const cro_alcc_config *cfg,
             cro_alcc_result *res);

/* ---- general-K P-APG(ALCC) (papg.cpp:66-283 with alcc_solve_block; 8f row f2) ---- */
void cro_apply_C_k(const double *X, int64_t N, int64_t n, int64_t K, const double *y,
                   const double *xi, double *out /* N(N-nbar)+N */);
void cro_apply_C_T_k(const double *X, int64_t N, int64_t n, int64_t K, const double *theta,
                     double *out_y, double *out_xi);
int cro_sigma_C_k(const double *X, int64_t N, int64_t n, int64_t K, double tol, int max_iters,
                  double *sigma, int *iters, int *converged);
/* cfg: the dual loop (cfg->threads > 1: blocks in parallel, deterministic);
   inner: PapgConfig::inner; feas_*: prepare_problem's feasible point (block
   balls and first warm starts). theta/c_eta in res have N(N-nbar)+N entries. */
int cro_papg_k(const double *X, const double *ys, int64_t N, int64_t n, int64_t K,
               const cro_config *cfg, const cro_alcc_config *inner, const double *feas_y,
               const double *feas_xi, const double *theta0, cro_result *res,
               int64_t *inner_iters_out);

#ifdef __cplusplus
}
#endif
#endif
