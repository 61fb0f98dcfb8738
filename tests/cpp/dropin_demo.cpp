// dropin_demo.cpp -- exercises the C++ drop-in (include/cvxreg_b200/papg.hpp)
// the way a reference caller would (runner.cpp:278-308 calls papg_solve /
// alcc_solve).
// in:  [N, n, iters, sigma_C, K, mode, X (N*n, row-major), ys_shifted (N),
//       feas_y (N), feas_xi (N*n), B_theta, Bbar_y, Bbar_xi, gamma] as float64
//       mode 0: papg_solve with K blocks (0: singleton), iters dual iterations
//       mode 1: alcc_solve from the feasible point, iters outer steps
// out: [iters, y (N), theta (papg) or multiplier (alcc)] as float64
#include <cstdio>
#include <fstream>
#include <iostream>
#include <vector>

#include "cvxreg_b200/papg.hpp"

namespace b2 = cvxreg::b200;

int main(int argc, char** argv) {
  if (argc != 3) {
    std::cerr << "usage: dropin_demo in.bin out.bin\n";
    return 2;
  }
  std::ifstream in(argv[1], std::ios::binary);
  std::vector<double> head(6);
  in.read(reinterpret_cast<char*>(head.data()), 6 * sizeof(double));
  const auto N = static_cast<b2::Index>(head[0]);
  const auto n = static_cast<b2::Index>(head[1]);
  const auto iters = static_cast<b2::Index>(head[2]);
  const auto K = static_cast<b2::Index>(head[4]);
  const int mode = static_cast<int>(head[5]);
  b2::PreparedProblem prep;
  auto rd = [&](std::vector<double>& v, size_t count) {
    v.resize(count);
    in.read(reinterpret_cast<char*>(v.data()), count * sizeof(double));
  };
  prep.data.n_ = n;
  rd(prep.data.xs, static_cast<size_t>(N * n));
  rd(prep.data.ys, static_cast<size_t>(N));
  rd(prep.feasible.y, static_cast<size_t>(N));
  rd(prep.feasible.xi, static_cast<size_t>(N * n));
  std::vector<double> b;
  rd(b, 4);
  prep.bounds = {b[0], b[1], b[2], b[3]};
  try {
    std::ofstream out(argv[2], std::ios::binary);
    auto put = [&](const std::vector<double>& v) {
      out.write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(double));
    };
    if (mode == 0) {
      b2::PapgConfig cfg;
      cfg.max_iters = iters;
      cfg.sigma_C = head[3];
      cfg.gap_norm_tol = -1.0;
      cfg.infeas_norm_tol = -1.0;
      cfg.K = K;
      cfg.inner.max_outer = 6;
      cfg.inner.mapg_cap = 1000;
      const b2::PapgResult r = b2::papg_solve(prep, cfg);
      put({static_cast<double>(r.report.iters)});
      put(r.point.y);
      put(r.dual.theta_cross);
      put(r.dual.theta_pos);
      std::printf("papg_solve (K=%lld): %lld iterations, reason %s\n", static_cast<long long>(K),
                  static_cast<long long>(r.report.iters), b2::to_string(r.report.reason).c_str());
    } else {
      b2::AlccConfig cfg;
      cfg.max_outer = iters;
      cfg.mapg_cap = 1000;
      const b2::AlccResult r = b2::alcc_solve(prep, cfg, prep.feasible);
      put({static_cast<double>(r.report.iters)});
      put(r.point.y);
      put(r.multiplier);
      std::printf("alcc_solve: %lld outer steps, %lld MAPG iterations, reason %s\n",
                  static_cast<long long>(r.report.iters),
                  static_cast<long long>(r.mapg_iters_total),
                  b2::to_string(r.report.reason).c_str());
    }
  } catch (const std::exception& e) {
    std::cerr << "solve failed: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
