// TEST INFRASTRUCTURE ONLY -- C entry points over the REFERENCE's own compiled
// code (oracle/_ref/libcvxreg_ref.so; recipe in oracle/Makefile, target `ref`).
// Every function below only marshals plain arrays into the reference's types
// and calls the reference function named in its comment; no algorithm lives
// here. Used by tests/ (to pin oracle/cvxreg_oracle.c and to make the golden
// fixtures of tests/golden/ref_*.npz) and by bench.py's CPU reference legs.
//
// Singleton blocks: the reference's make_partition (dataset.cpp:119-130)
// rejects nbar < n+1, but Partition is a plain aggregate (types.hpp:30-37) and
// ProblemOps only checks part.N() == data.N() (operators.cpp:22-25), so K = N
// is reached here by building Partition{N, 1} directly. Each block solve is
// then alcc_core on an empty row set (alcc.cpp:222-258: sigma = 0 for an empty
// operator, operators.cpp:304-307), whose MAPG lands on the centre
// (ybar + q_y, q_xi / gamma) -- the closed form of SURVEY.md §8 a4 -- to
// rounding.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>

#include "cvxreg/metrics.hpp"
#include "cvxreg/papg.hpp"
#include "cvxreg/projections.hpp"
#include "cvxreg/rng.hpp"
#include "cvxreg/testgen.hpp"

using namespace cvxreg;

namespace {

struct RefConfig {  // same layout as CroConfig (oracle/cvxreg_oracle.h)
  double gamma, B_theta;
  int32_t adaptive_B_theta, max_restarts;
  double gap_norm_tol, infeas_norm_tol;
  int64_t max_iters;
  double max_seconds, inner_tol_floor, final_resolve_tol;
  int32_t record_history, use_momentum;
  double sigma_C;  // ignored: the reference always estimates it (papg.cpp:66)
  int32_t threads, pad_;  // threads -> PapgConfig::workers
};

struct RefAlccConfig {  // same layout as CroAlccConfig
  double mu1, tau1_scale, alpha1_scale, c, kappa;
  int64_t max_outer, mapg_cap;
  double infeas_norm_tol, gap_norm_tol, max_seconds;
  int32_t record_history, threads;
};

struct RefResult {  // same layout as CroResult
  double *y, *xi, *theta, *c_eta, *history;
  int64_t iters;
  int32_t reason, restarts, saturated, sigma_iters, sigma_converged, pad_;
  double g_final, delta_estimate, sigma_C, L_g, B_theta, wall_seconds;
};

struct RefAlccResult {  // same layout as CroAlccResult
  double *y, *xi, *multiplier, *history;
  int64_t* mapg_iters;  // not available from the reference (per-call counts): untouched
  int64_t outer_iters, mapg_iters_total;
  int32_t reason, hit_cap_any;
  double certified_gap, infeas_raw, gap_raw, objective, wall_seconds, sigma_A1, sigma_A2;
};

thread_local char g_error[512];

int fail(const std::exception& e, int code) {
  std::strncpy(g_error, e.what(), sizeof(g_error) - 1);
  g_error[sizeof(g_error) - 1] = 0;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, -1);
  } catch (const std::bad_alloc& e) {
    return fail(e, -2);
  } catch (const std::runtime_error& e) {
    return fail(e, -4);
  } catch (const std::exception& e) {
    return fail(e, -9);
  }
}

Dataset make_dataset(const double* xs_rowmajor, const double* ys, int64_t N, int64_t n) {
  Dataset d;
  d.xs.resize(N, n);
  d.ys.resize(N);
  for (Index l = 0; l < N; ++l) {
    for (Index j = 0; j < n; ++j) d.xs(l, j) = xs_rowmajor[l * n + j];
    d.ys(l) = ys ? ys[l] : 0.0;
  }
  return d;
}

VectorXd make_vector(const double* p, Index n) {
  VectorXd v(n);
  for (Index i = 0; i < n; ++i) v(i) = p[i];
  return v;
}

void put(const VectorXd& v, double* out) {
  if (out) std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(v.size()));
}

Partition partition_for(const Dataset& d, int64_t K) {
  if (K == d.N()) return Partition{d.N(), 1};  // singleton blocks, see the header comment
  return make_partition(d, K);                 // dataset.cpp:119-130
}

void put_history(const std::vector<MetricsSnapshot>& h, double* out) {
  if (!out) return;
  for (size_t k = 0; k < h.size(); ++k) {
    double* r = out + 8 * k;
    r[0] = static_cast<double>(h[k].iter);
    r[1] = h[k].objective;
    r[2] = h[k].reg_objective;
    r[3] = h[k].infeas_raw;
    r[4] = h[k].infeas_norm;
    r[5] = h[k].gap_raw;
    r[6] = h[k].gap_norm;
    r[7] = h[k].wall_time_s;
  }
}

AlccConfig inner_from(const RefAlccConfig* c) {
  AlccConfig a;
  if (!c) return a;
  a.mu1 = c->mu1;
  a.tau1_scale = c->tau1_scale;
  a.alpha1_scale = c->alpha1_scale;
  a.c = c->c;
  a.kappa = c->kappa;
  a.max_outer = c->max_outer;
  a.mapg_cap = c->mapg_cap;
  a.infeas_norm_tol = c->infeas_norm_tol;
  a.gap_norm_tol = c->gap_norm_tol;
  a.max_seconds = c->max_seconds;
  a.record_history = c->record_history != 0;
  return a;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error; }

/// rng.hpp:37-47, 57-59: `count` draws of stream (seed, tag); kind 0 uniform, 1 normal.
int ref_rng_draws(uint64_t seed, uint64_t tag, int64_t count, int kind, double* out) {
  Xoshiro256pp gen = rng_stream(seed, tag);
  for (int64_t i = 0; i < count; ++i) out[i] = kind == 1 ? gen.normal() : gen.uniform();
  return 0;
}

/// testgen.cpp:38-91 gen_instance; kind = GeneratorSpec::Kind (0..3).
int ref_gen_instance(int kind, int64_t N, int64_t n, double noise, uint64_t seed,
                     double* xs_rowmajor, double* ys) {
  return guarded([&] {
    GeneratorSpec spec;
    spec.kind = static_cast<GeneratorSpec::Kind>(kind);
    spec.N = N;
    spec.n = n;
    spec.noise = noise;
    spec.seed = seed;
    Dataset d = gen_instance(spec);
    for (Index l = 0; l < N; ++l) {
      for (Index j = 0; j < n; ++j) xs_rowmajor[l * n + j] = d.xs(l, j);
      ys[l] = d.ys(l);
    }
  });
}

/// dataset.cpp:14-46 validate_dataset.
int ref_validate(const double* xs, const double* ys, int64_t N, int64_t n) {
  return guarded([&] { validate_dataset(make_dataset(xs, ys, N, n)); });
}

/// preprocess.cpp:50-65 prepare_problem. bounds4 = (B_theta, Bbar_y, Bbar_xi, gamma).
int ref_prepare(const double* xs, const double* ys, int64_t N, int64_t n, double gamma,
                double* ys_shifted, double* shift, double* feas_y, double* feas_xi,
                double* bounds4, double* intercept, double* slope) {
  return guarded([&] {
    Dataset d = make_dataset(xs, ys, N, n);
    PreparedProblem prep = prepare_problem(d, gamma);
    AffineFit fit = affine_feasible_point(d, gamma);
    put(prep.data.ys, ys_shifted);
    *shift = prep.shift;
    put(prep.feasible.y, feas_y);
    put(prep.feasible.xi, feas_xi);
    bounds4[0] = prep.bounds.B_theta;
    bounds4[1] = prep.bounds.Bbar_y;
    bounds4[2] = prep.bounds.Bbar_xi;
    bounds4[3] = prep.bounds.gamma;
    *intercept = fit.intercept;
    put(fit.slope, slope);
  });
}

/// operators.cpp:128-153 apply_C with K blocks (K = N: singleton).
int ref_apply_C(const double* xs, int64_t N, int64_t n, int64_t K, const double* y,
                const double* xi, double* out) {
  return guarded([&] {
    Dataset d = make_dataset(xs, nullptr, N, n);
    ProblemOps ops(d, partition_for(d, K));
    VectorXd o;
    ops.apply_C(make_vector(y, N), make_vector(xi, N * n), o);
    put(o, out);
  });
}

/// operators.cpp:155-180 apply_C_T.
int ref_apply_C_T(const double* xs, int64_t N, int64_t n, int64_t K, const double* theta,
                  double* out_y, double* out_xi) {
  return guarded([&] {
    Dataset d = make_dataset(xs, nullptr, N, n);
    ProblemOps ops(d, partition_for(d, K));
    VectorXd oy, oxi;
    ops.apply_C_T(make_vector(theta, ops.indexing().rows_C()), oy, oxi);
    put(oy, out_y);
    put(oxi, out_xi);
  });
}

/// operators.cpp:101-126 apply_rows / rows_adjoint (all N(N-1) rows).
int ref_apply_rows(const double* xs, int64_t N, int64_t n, const double* y, const double* xi,
                   double* out) {
  return guarded([&] {
    Dataset d = make_dataset(xs, nullptr, N, n);
    ProblemOps ops(d, Partition{1, N});
    VectorXd o;
    ops.apply_rows(make_vector(y, N), make_vector(xi, N * n), o);
    put(o, out);
  });
}

int ref_rows_adjoint(const double* xs, int64_t N, int64_t n, const double* z, double* out_y,
                     double* out_xi) {
  return guarded([&] {
    Dataset d = make_dataset(xs, nullptr, N, n);
    ProblemOps ops(d, Partition{1, N});
    VectorXd oy, oxi;
    ops.rows_adjoint(make_vector(z, N * (N - 1)), oy, oxi);
    put(oy, out_y);
    put(oxi, out_xi);
  });
}

/// operators.cpp:302-339 estimate_sigma_max on op_C (which 0, K blocks), op_A1 (1), op_A2 (2).
int ref_sigma(const double* xs, int64_t N, int64_t n, int64_t K, int which, double tol,
              int max_iters, double* sigma, int* iters, int* converged) {
  return guarded([&] {
    Dataset d = make_dataset(xs, nullptr, N, n);
    ProblemOps ops(d, which == 0 ? partition_for(d, K) : Partition{1, N});
    SigmaEstimate e = estimate_sigma_max(
        which == 0 ? op_C(ops) : which == 1 ? op_A1(ops) : op_A2(ops), tol, max_iters);
    *sigma = e.sigma;
    *iters = e.iters;
    *converged = e.converged ? 1 : 0;
  });
}

/// indexing.hpp:30-37 cross_position.
int64_t ref_cross_position(int64_t N, int64_t K, int64_t l1, int64_t l2) {
  try {
    return RowIndexing{N, K, N / K}.cross_position(l1, l2);
  } catch (const std::exception&) {
    return -1;
  }
}

/// projections.hpp:9-13, engines.hpp:11-13, papg.cpp:298-303.
void ref_project_nonneg_ball(double* v, int64_t n, double radius) {
  VectorXd x = make_vector(v, n);
  project_nonneg_ball_inplace(x, radius);
  put(x, v);
}
double ref_momentum_next(double t) { return momentum_next(t); }
void ref_certificate(double gamma, double delta, double B_xi, double sigma, double* out2) {
  auto p = certificate_for_iterate(gamma, delta, B_xi, sigma);
  out2[0] = p.first;
  out2[1] = p.second;
}

/// papg.cpp:287-296 papg_solve / dual_gradient_ascent on prepare_problem(xs, ys_raw)
/// (preprocess.cpp:50-65) with K blocks. `ys_is_shifted` != 0 takes ys as the already
/// shifted observations and (feas_y, feas_xi) as the feasible point instead of calling
/// prepare_problem. C_eta of the last iteration is not part of PapgResult; when c_eta is
/// wanted it is recomputed as apply_C(point) at the final theta1 (papg.cpp:268).
int ref_papg(const double* xs, const double* ys, int64_t N, int64_t n, int64_t K,
             const RefConfig* cfg, const RefAlccConfig* inner, int ys_is_shifted,
             const double* feas_y, const double* feas_xi, const double* theta0,
             RefResult* out) {
  return guarded([&] {
    Dataset d = make_dataset(xs, ys, N, n);
    PreparedProblem prep;
    if (ys_is_shifted) {
      prep.data = d;
      prep.feasible.y = make_vector(feas_y, N);
      prep.feasible.xi = make_vector(feas_xi, N * n);
      prep.bounds.gamma = cfg->gamma;
    } else {
      prep = prepare_problem(d, cfg->gamma);
    }
    ProblemOps ops(prep.data, partition_for(prep.data, K));
    PapgConfig pc;
    pc.gamma = cfg->gamma;
    pc.B_theta = cfg->B_theta;
    pc.adaptive_B_theta = cfg->adaptive_B_theta != 0;
    pc.max_restarts = cfg->max_restarts;
    pc.gap_norm_tol = cfg->gap_norm_tol;
    pc.infeas_norm_tol = cfg->infeas_norm_tol;
    pc.max_iters = cfg->max_iters;
    pc.max_seconds = cfg->max_seconds;
    pc.workers = cfg->threads;
    pc.inner_tol_floor = cfg->inner_tol_floor;
    pc.final_resolve_tol = cfg->final_resolve_tol;
    pc.inner = inner_from(inner);
    pc.record_history = cfg->record_history != 0;
    VectorXd t0;
    if (theta0) t0 = make_vector(theta0, ops.indexing().rows_C());
    PapgResult r = cfg->use_momentum ? papg_solve(ops, prep, pc, theta0 ? &t0 : nullptr)
                                     : dual_gradient_ascent(ops, prep, pc, theta0 ? &t0 : nullptr);
    put(r.point.y, out->y);
    put(r.point.xi, out->xi);
    if (out->theta) {
      put(r.dual.theta_cross, out->theta);
      put(r.dual.theta_pos, out->theta + r.dual.theta_cross.size());
    }
    if (out->c_eta) {
      VectorXd ce;
      ops.apply_C(r.point.y, r.point.xi, ce);
      put(ce, out->c_eta);
    }
    put_history(r.report.history, out->history);
    out->iters = r.report.iters;
    out->reason = static_cast<int32_t>(r.report.reason);
    out->restarts = r.report.restarts;
    out->saturated = r.report.saturated ? 1 : 0;
    out->g_final = r.g_final;
    out->delta_estimate = r.delta_estimate;
    out->sigma_C = r.sigma_C;
    out->L_g = r.L_g;
    out->B_theta = r.B_theta;
    out->wall_seconds = r.report.wall_seconds;
  });
}

/// papg.cpp:89-132 DualDecomposition::dual_gradient at theta (one call on a fresh
/// decomposition): eta, C_eta, g, within-block infeasibility, inner iterations.
int ref_dual_gradient(const double* xs, const double* ys_shifted, int64_t N, int64_t n,
                      int64_t K, const RefConfig* cfg, const RefAlccConfig* inner,
                      const double* feas_y, const double* feas_xi, const double* theta,
                      double inner_tol, double* y, double* xi, double* c_eta, double* scalars3) {
  return guarded([&] {
    PreparedProblem prep;
    prep.data = make_dataset(xs, ys_shifted, N, n);
    prep.feasible.y = make_vector(feas_y, N);
    prep.feasible.xi = make_vector(feas_xi, N * n);
    prep.bounds.gamma = cfg->gamma;
    ProblemOps ops(prep.data, partition_for(prep.data, K));
    PapgConfig pc;
    pc.gamma = cfg->gamma;
    pc.workers = cfg->threads;
    pc.inner = inner_from(inner);
    DualDecomposition decomp(ops, prep, pc);
    DualGradientResult g =
        decomp.dual_gradient(make_vector(theta, ops.indexing().rows_C()), inner_tol);
    put(g.eta.y, y);
    put(g.eta.xi, xi);
    put(g.C_eta, c_eta);
    scalars3[0] = g.g_value;
    scalars3[1] = g.within_infeas_raw;
    scalars3[2] = static_cast<double>(g.inner_iters);
  });
}

/// alcc.cpp:193-208 alcc_solve (standalone ALCC over all N(N-1) rows). The reference
/// estimates sigma(A1), sigma(A2) itself; they are not returned by AlccResult.
int ref_alcc(const double* xs, const double* ys_bar, int64_t N, int64_t n, double gamma,
             double Bbar_y, double Bbar_xi, const double* warm_y, const double* warm_xi,
             const RefAlccConfig* cfg, RefAlccResult* out) {
  return guarded([&] {
    Dataset d = make_dataset(xs, ys_bar, N, n);
    ProblemOps ops(d, Partition{1, N});
    ProblemBounds b;
    b.Bbar_y = Bbar_y;
    b.Bbar_xi = Bbar_xi;
    b.gamma = gamma;
    PrimalPoint warm;
    warm.y = make_vector(warm_y, N);
    warm.xi = make_vector(warm_xi, N * n);
    AlccResult r = alcc_solve(ops, d.ys, gamma, b, inner_from(cfg), warm);
    put(r.point.y, out->y);
    put(r.point.xi, out->xi);
    put(r.multiplier, out->multiplier);
    put_history(r.report.history, out->history);
    out->outer_iters = r.report.iters;
    out->mapg_iters_total = r.mapg_iters_total;
    out->reason = static_cast<int32_t>(r.report.reason);
    out->hit_cap_any = 0;
    out->certified_gap = r.certified_gap;
    out->infeas_raw = r.infeas_raw;
    out->gap_raw = r.report.history.empty() ? 0.0 : r.report.history.back().gap_raw;
    out->objective = r.objective;
    out->wall_seconds = r.report.wall_seconds;
    out->sigma_A1 = 0;
    out->sigma_A2 = 0;
  });
}

/// metrics.cpp:8-15, 17-31, 33-48, 50-56.
int ref_infeasibility(const double* xs, int64_t N, int64_t n, const double* y, const double* xi,
                      double* out2) {
  return guarded([&] {
    Dataset d = make_dataset(xs, nullptr, N, n);
    ProblemOps ops(d, Partition{1, N});
    PrimalPoint p{make_vector(y, N), make_vector(xi, N * n)};
    auto r = infeasibility(ops, p);
    out2[0] = r.first;
    out2[1] = r.second;
  });
}

int ref_duality_gap(const double* xs, int64_t N, int64_t n, const double* theta, const double* y,
                    const double* xi, double* out2) {
  return guarded([&] {
    Dataset d = make_dataset(xs, nullptr, N, n);
    ProblemOps ops(d, Partition{N, 1});
    DualPoint t{make_vector(theta, N * (N - 1)), make_vector(theta + N * (N - 1), N)};
    PrimalPoint p{make_vector(y, N), make_vector(xi, N * n)};
    auto r = duality_gap(ops, t, p);
    out2[0] = r.first;
    out2[1] = r.second;
  });
}

double ref_evaluate_estimator(const double* xs, int64_t N, int64_t n, const double* y,
                              const double* xi, const double* xq) {
  Dataset d = make_dataset(xs, nullptr, N, n);
  PrimalPoint p{make_vector(y, N), make_vector(xi, N * n)};
  return evaluate_estimator(p, d, make_vector(xq, n));
}

int ref_repair_feasibility(const double* xs, int64_t N, int64_t n, const double* y,
                           const double* xi, double* out_y) {
  return guarded([&] {
    Dataset d = make_dataset(xs, nullptr, N, n);
    PrimalPoint p{make_vector(y, N), make_vector(xi, N * n)};
    put(repair_feasibility(p, d).y, out_y);
  });
}

}  // extern "C"
