// dropin_demo.cpp -- exercises the C++ drop-in (include/cvxreg_b200/papg.hpp)
// the way a reference caller would (runner.cpp:306-308 calls papg_solve).
// in:  [N, n, iters, sigma_C, X (N*n, row-major), ys_shifted (N)] as float64
// out: [iters, y (N), theta (N(N-1)+N)] as float64
#include <cstdio>
#include <fstream>
#include <iostream>
#include <vector>

#include "cvxreg_b200/papg.hpp"

int main(int argc, char** argv) {
  if (argc != 3) {
    std::cerr << "usage: dropin_demo in.bin out.bin\n";
    return 2;
  }
  std::ifstream in(argv[1], std::ios::binary);
  std::vector<double> head(4);
  in.read(reinterpret_cast<char*>(head.data()), 4 * sizeof(double));
  const auto N = static_cast<cvxreg::b200::Index>(head[0]);
  const auto n = static_cast<cvxreg::b200::Index>(head[1]);
  cvxreg::b200::PreparedProblem prep;
  prep.data.n_ = n;
  prep.data.xs.resize(static_cast<size_t>(N * n));
  prep.data.ys.resize(static_cast<size_t>(N));
  in.read(reinterpret_cast<char*>(prep.data.xs.data()), prep.data.xs.size() * sizeof(double));
  in.read(reinterpret_cast<char*>(prep.data.ys.data()), prep.data.ys.size() * sizeof(double));
  cvxreg::b200::PapgConfig cfg;
  cfg.max_iters = static_cast<cvxreg::b200::Index>(head[2]);
  cfg.sigma_C = head[3];
  cfg.gap_norm_tol = -1.0;
  cfg.infeas_norm_tol = -1.0;
  try {
    const cvxreg::b200::PapgResult r = cvxreg::b200::papg_solve(prep, cfg);
    std::ofstream out(argv[2], std::ios::binary);
    const double iters = static_cast<double>(r.report.iters);
    out.write(reinterpret_cast<const char*>(&iters), sizeof(double));
    out.write(reinterpret_cast<const char*>(r.point.y.data()), r.point.y.size() * sizeof(double));
    out.write(reinterpret_cast<const char*>(r.dual.theta_cross.data()),
              r.dual.theta_cross.size() * sizeof(double));
    out.write(reinterpret_cast<const char*>(r.dual.theta_pos.data()),
              r.dual.theta_pos.size() * sizeof(double));
    std::printf("papg_solve: %lld iterations, reason %s\n", static_cast<long long>(r.report.iters),
                cvxreg::b200::to_string(r.report.reason).c_str());
  } catch (const std::exception& e) {
    std::cerr << "papg_solve failed: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
