// papg.hpp -- C++ drop-in for the singleton-block dual solver of the
// reference (proj/core/include/cvxreg/papg.hpp, types.hpp, metrics.hpp,
// preprocess.hpp, testgen.hpp), header-only over the C ABI in
// ../cvxreg_b200.h (link with libcvxreg_b200.so).
//
// Same names, fields, defaults and error behaviour as the reference:
//   papg_solve / dual_gradient_ascent          papg.hpp:75-82
//   certificate_for_iterate                    papg.hpp:85-90
//   prepare_problem                            preprocess.hpp:42
//   gen_instance                               testgen.hpp:27
// CR_EINVAL -> std::invalid_argument, every other failure -> std::runtime_error
// (e.g. "papg: non-finite dual gradient", papg.cpp:184-185). Storage is
// std::vector<double> (row-major xs, flat xi) instead of Eigen.
#pragma once
#include <cstdint>
#include <cstddef>
#include <algorithm>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../cvxreg_b200.h"

namespace cvxreg {
namespace b200 {

using Index = std::ptrdiff_t;

struct Dataset {  // types.hpp:13-19; xs row-major N x n
  std::vector<double> xs;
  std::vector<double> ys;
  Index n_ = 0;
  Index N() const { return static_cast<Index>(ys.size()); }
  Index n() const { return n_; }
};

struct ProblemBounds {  // types.hpp:55-60
  double B_theta = 0, Bbar_y = 0, Bbar_xi = 0, gamma = 0;
};

struct PrimalPoint {  // types.hpp:43-46
  std::vector<double> y;
  std::vector<double> xi;  // xi_l = xi[l*n .. l*n+n)
};

struct DualPoint {  // types.hpp:50-53
  std::vector<double> theta_cross;  // N(N-1), singleton cross order
  std::vector<double> theta_pos;    // N
};

struct PreparedProblem {  // preprocess.hpp:35-40
  Dataset data;
  double shift = 0;
  PrimalPoint feasible;
  ProblemBounds bounds;
};

struct GeneratorSpec {  // testgen.hpp:13-19 (+ pieces for the BASELINE kinds)
  enum class Kind { quadratic = 0, exponential = 1, affine_noiseless = 2, custom_1d = 3,
                    sqnorm_uniform = 10, maxaffine_uniform = 11, lse_uniform = 12 };
  Kind kind = Kind::quadratic;
  Index n = 1;
  Index N = 0;
  double noise = 1.0;
  std::uint64_t seed = 1;
  Index pieces = 0;
};

struct AlccConfig {  // alcc.hpp:71-83
  double mu1 = 1.0;
  double tau1_scale = 1e-2;
  double alpha1_scale = 1e-3;
  double c = 5.0;
  double kappa = 0.5;
  Index max_outer = 30;
  Index mapg_cap = 200000;
  double infeas_norm_tol = 1e-1;
  double gap_norm_tol = 1e-6;
  double max_seconds = std::numeric_limits<double>::infinity();
  bool record_history = true;
  // device knobs: inject the spectral norms instead of estimating them
  double sigma_A1 = 0, sigma_A2 = 0;
};

struct PapgConfig {  // papg.hpp:7-21
  double gamma = 1e-3;
  double B_theta = 0;
  bool adaptive_B_theta = true;
  int max_restarts = 6;
  double gap_norm_tol = 1e-6;
  double infeas_norm_tol = 1e-1;
  Index max_iters = 100000;
  double max_seconds = 7200;
  int workers = 0;  // concurrent block solves of a K-block partition (<= 0: 16)
  double inner_tol_floor = 1e-6;
  double final_resolve_tol = 1e-10;
  AlccConfig inner;  // block QPs of a K < N partition
  bool record_history = true;
  // the partition (make_partition, dataset.cpp:119): 0 or N = singleton blocks
  Index K = 0;
  // device knobs
  int device = 0;
  double sigma_C = 0;   // > 0: inject sigma_max(C)
  int graph_iters = 0;  // 0 auto, > 0 CUDA-graph batch, < 0 direct launches
  // D > 0: sums over D canonical row blocks, bitwise independent of the GPU count
  // (cr_set_canonical_blocks); singleton blocks only
  int canonical_blocks = 0;
};

struct MetricsSnapshot {  // metrics.hpp:13-22
  Index iter = 0;
  double objective = 0, reg_objective = 0, infeas_raw = 0, infeas_norm = 0, gap_raw = 0,
         gap_norm = 0, wall_time_s = 0;
};

enum class TermReason { thresholds, iter_budget, time_budget, error };  // metrics.hpp:41

inline std::string to_string(TermReason r) {
  switch (r) {
    case TermReason::thresholds: return "thresholds";
    case TermReason::iter_budget: return "iter_budget";
    case TermReason::time_budget: return "time_budget";
    case TermReason::error: return "error";
  }
  return "unknown";
}

struct SolveReport {  // metrics.hpp:45-54
  std::vector<MetricsSnapshot> history;
  TermReason reason = TermReason::iter_budget;
  Index iters = 0;
  double wall_seconds = 0;
  double cpu_seconds = 0;
  int restarts = 0;
  bool saturated = false;
  std::string note;
};

struct PapgResult {  // papg.hpp:60-69
  PrimalPoint point;
  DualPoint dual;
  SolveReport report;
  double g_final = 0;
  double delta_estimate = 0;
  double sigma_C = 0;
  double L_g = 0;
  double B_theta = 0;
};

struct AlccResult {  // alcc.hpp:110-118
  PrimalPoint point;
  std::vector<double> multiplier;
  double objective = 0;
  double certified_gap = 0;
  double infeas_raw = 0;
  Index mapg_iters_total = 0;
  SolveReport report;
};

namespace detail {
inline cr_alcc_config to_c(const AlccConfig& a) {
  cr_alcc_config c{};
  c.mu1 = a.mu1;
  c.tau1_scale = a.tau1_scale;
  c.alpha1_scale = a.alpha1_scale;
  c.c = a.c;
  c.kappa = a.kappa;
  c.max_outer = a.max_outer;
  c.mapg_cap = a.mapg_cap;
  c.infeas_norm_tol = a.infeas_norm_tol;
  c.gap_norm_tol = a.gap_norm_tol;
  c.max_seconds = a.max_seconds;
  c.record_history = a.record_history ? 1 : 0;
  c.sigma_A1 = a.sigma_A1;
  c.sigma_A2 = a.sigma_A2;
  return c;
}
inline MetricsSnapshot from_c(const cr_snapshot& s) {
  return {static_cast<Index>(s.iter), s.objective, s.reg_objective, s.infeas_raw,
          s.infeas_norm, s.gap_raw, s.gap_norm, s.wall_time_s};
}
inline void check(cr_status s, const cr_handle* h = nullptr) {
  if (s == CR_OK) return;
  const std::string msg = h ? cr_last_error(h) : cr_status_string(s);
  if (s == CR_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
struct Handle {
  cr_handle* h = nullptr;
  ~Handle() { cr_destroy(h); }
};

inline PapgResult solve(const PreparedProblem& prep, const PapgConfig& cfg,
                        const std::vector<double>* theta0, bool momentum) {
  const Dataset& d = prep.data;
  const Index N = d.N(), n = d.n();
  if (static_cast<Index>(d.xs.size()) != N * n)
    throw std::invalid_argument("papg: xs/ys row count mismatch");
  const Index K = (cfg.K > 0 && cfg.K < N) ? cfg.K : 0;
  const Index cross = K ? N * (N - N / K) : N * (N - 1);
  if (theta0 && static_cast<Index>(theta0->size()) != cross + N)
    throw std::invalid_argument("papg: warm-start theta has wrong size");  // papg.cpp:160-161
  Handle hd;
  check(cr_create(d.xs.data(), d.ys.data(), N, n, cfg.gamma, cfg.device, 0, N, &hd.h), hd.h);
  if (K) {  // P-APG(ALCC) with K blocks (papg.cpp:66-132)
    const cr_alcc_config inner = to_c(cfg.inner);
    check(cr_set_partition(hd.h, K, prep.feasible.y.data(), prep.feasible.xi.data(), &inner),
          hd.h);
  }
  if (cfg.canonical_blocks > 0) check(cr_set_canonical_blocks(hd.h, cfg.canonical_blocks), hd.h);
  cr_papg_config c{};
  c.gamma = cfg.gamma;
  c.B_theta = cfg.B_theta;
  c.adaptive_B_theta = cfg.adaptive_B_theta ? 1 : 0;
  c.max_restarts = cfg.max_restarts;
  c.gap_norm_tol = cfg.gap_norm_tol;
  c.infeas_norm_tol = cfg.infeas_norm_tol;
  c.max_iters = cfg.max_iters;
  c.max_seconds = cfg.max_seconds;
  c.inner_tol_floor = cfg.inner_tol_floor;
  c.final_resolve_tol = cfg.final_resolve_tol;
  c.record_history = cfg.record_history ? 1 : 0;
  c.use_momentum = momentum ? 1 : 0;
  c.sigma_C = cfg.sigma_C;
  c.graph_iters = cfg.graph_iters;
  c.workers = cfg.workers;
  PapgResult out;
  out.point.y.resize(static_cast<size_t>(N));
  out.point.xi.resize(static_cast<size_t>(N * n));
  std::vector<cr_snapshot> hist(
      cfg.record_history ? static_cast<size_t>(std::min<Index>(cfg.max_iters, CR_HISTORY_CAP)) : 0);
  cr_papg_result r{};
  check(cr_papg_solve(hd.h, &c, theta0 ? theta0->data() : nullptr, &r, out.point.y.data(),
                      out.point.xi.data(), hist.empty() ? nullptr : hist.data()),
        hd.h);
  std::vector<double> th(static_cast<size_t>(cross + N));
  check(cr_get_theta(hd.h, th.data()), hd.h);
  out.dual.theta_cross.assign(th.begin(), th.begin() + cross);
  out.dual.theta_pos.assign(th.begin() + cross, th.end());
  out.report.reason = static_cast<TermReason>(r.reason);
  out.report.iters = r.iters;
  out.report.wall_seconds = r.wall_seconds;
  out.report.restarts = r.restarts;
  out.report.saturated = r.saturated != 0;
  for (Index i = 0; i < r.iters && i < static_cast<Index>(hist.size()); ++i)
    out.report.history.push_back(from_c(hist[static_cast<size_t>(i)]));
  out.g_final = r.g_final;
  out.delta_estimate = r.delta_estimate;
  out.sigma_C = r.sigma_C;
  out.L_g = r.L_g;
  out.B_theta = r.B_theta;
  return out;
}
}  // namespace detail

inline Dataset gen_instance(const GeneratorSpec& spec) {  // testgen.cpp:36-87
  Dataset d;
  d.n_ = spec.n;
  d.xs.resize(static_cast<size_t>(spec.N * spec.n));
  d.ys.resize(static_cast<size_t>(spec.N));
  detail::check(cr_gen_instance(static_cast<int32_t>(spec.kind), spec.N, spec.n, spec.noise,
                                spec.seed, spec.pieces, d.xs.data(), d.ys.data()));
  return d;
}

inline PreparedProblem prepare_problem(const Dataset& data, double gamma) {  // preprocess.cpp:50-65
  PreparedProblem p;
  const Index N = data.N(), n = data.n();
  p.data.n_ = n;
  p.data.xs = data.xs;
  p.data.ys.resize(static_cast<size_t>(N));
  p.feasible.y.resize(static_cast<size_t>(N));
  p.feasible.xi.resize(static_cast<size_t>(N * n));
  double b4[4];
  detail::check(cr_prepare_problem(data.xs.data(), data.ys.data(), N, n, gamma, p.data.ys.data(),
                                   &p.shift, p.feasible.y.data(), p.feasible.xi.data(), b4));
  p.bounds = {b4[0], b4[1], b4[2], b4[3]};
  return p;
}

// Fig. 2 P-APG (papg.cpp:287-290) on the device.
inline PapgResult papg_solve(const PreparedProblem& prep, const PapgConfig& cfg,
                             const std::vector<double>* theta0 = nullptr) {
  return detail::solve(prep, cfg, theta0, true);
}

// Projected dual gradient ascent baseline (papg.cpp:292-296).
inline PapgResult dual_gradient_ascent(const PreparedProblem& prep, const PapgConfig& cfg,
                                       const std::vector<double>* theta0 = nullptr) {
  return detail::solve(prep, cfg, theta0, false);
}

// metrics.cpp:8-15 -- (raw, normalised) infeasibility over all N(N-1) rows
inline std::pair<double, double> infeasibility(const Dataset& data, const PrimalPoint& eta,
                                               int device = 0) {
  detail::Handle hd;
  detail::check(cr_create(data.xs.data(), data.ys.data(), data.N(), data.n(), 1e-3, device, 0,
                          data.N(), &hd.h),
                hd.h);
  double out[2];
  detail::check(cr_infeasibility(hd.h, eta.y.data(), eta.xi.data(), out), hd.h);
  return {out[0], out[1]};
}

// metrics.cpp:32-48 -- fhat(x) = max_l y_l + xi_l.(x - x_l) at Q query points (Q x n)
inline std::vector<double> evaluate_estimator(const PrimalPoint& eta, const Dataset& data,
                                              const std::vector<double>& x_query,
                                              int device = 0) {
  detail::Handle hd;
  detail::check(cr_create(data.xs.data(), data.ys.data(), data.N(), data.n(), 1e-3, device, 0,
                          data.N(), &hd.h),
                hd.h);
  const Index Q = static_cast<Index>(x_query.size()) / data.n();
  std::vector<double> out(static_cast<size_t>(Q));
  detail::check(cr_evaluate_estimator(hd.h, eta.y.data(), eta.xi.data(), x_query.data(), Q,
                                      out.data()),
                hd.h);
  return out;
}

// metrics.cpp:50-56 -- y'_l = fhat(x_l)
inline PrimalPoint repair_feasibility(const PrimalPoint& eta, const Dataset& data,
                                      int device = 0) {
  detail::Handle hd;
  detail::check(cr_create(data.xs.data(), data.ys.data(), data.N(), data.n(), 1e-3, device, 0,
                          data.N(), &hd.h),
                hd.h);
  PrimalPoint out = eta;
  detail::check(cr_repair_feasibility(hd.h, eta.y.data(), eta.xi.data(), out.y.data()), hd.h);
  return out;
}

// standalone ALCC (alcc.cpp:193-208): centres (ybar, 0), balls from prep.bounds
inline AlccResult alcc_solve(const PreparedProblem& prep, const AlccConfig& cfg,
                             const PrimalPoint& warm, int device = 0) {
  const Dataset& d = prep.data;
  const Index N = d.N(), n = d.n();
  detail::Handle hd;
  detail::check(cr_create(d.xs.data(), d.ys.data(), N, n, prep.bounds.gamma, device, 0, N,
                          &hd.h),
                hd.h);
  cr_alcc_config c = detail::to_c(cfg);
  c.Bbar_y = prep.bounds.Bbar_y;
  c.Bbar_xi = prep.bounds.Bbar_xi;
  AlccResult out;
  out.point.y.resize(static_cast<size_t>(N));
  out.point.xi.resize(static_cast<size_t>(N * n));
  std::vector<cr_snapshot> hist(static_cast<size_t>(std::max<Index>(cfg.max_outer, 1)));
  cr_alcc_result r{};
  detail::check(cr_alcc_solve(hd.h, &c, warm.y.data(), warm.xi.data(), out.point.y.data(),
                              out.point.xi.data(), hist.data(), nullptr, &r),
                hd.h);
  if (r.outer_iters > 0) {
    out.multiplier.resize(static_cast<size_t>(N * (N - 1)));
    detail::check(cr_alcc_multiplier(hd.h, 0, N, out.multiplier.data()), hd.h);
  }
  out.objective = r.objective;
  out.certified_gap = r.certified_gap;
  out.infeas_raw = r.infeas_raw;
  out.mapg_iters_total = r.mapg_iters_total;
  out.report.reason = static_cast<TermReason>(r.reason);
  out.report.iters = r.outer_iters;
  out.report.wall_seconds = r.wall_seconds;
  if (cfg.record_history)
    for (Index k = 0; k < r.outer_iters; ++k)
      out.report.history.push_back(detail::from_c(hist[static_cast<size_t>(k)]));
  return out;
}

inline std::pair<double, double> certificate_for_iterate(double gamma, double delta,
                                                         double B_xi_estimate,
                                                         double sigma_max_C) {
  double out[2];
  cr_certificate(gamma, delta, B_xi_estimate, sigma_max_C, out);
  return {out[0], out[1]};
}

}  // namespace b200
}  // namespace cvxreg
