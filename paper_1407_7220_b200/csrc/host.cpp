// host.cpp -- host utilities of the C ABI: seeded instance generation
// (testgen.cpp:36-87 plus the BASELINE.json kinds), dataset validation
// (dataset.cpp:14-42) and prepare_problem (preprocess.cpp:9-65).
// These run once per solve on the host; the iterative path is on the device.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <thread>
#include <vector>

#include "../../include/cvxreg_b200.h"
#include "host.hpp"

namespace crb {
namespace host {
namespace {

// xoshiro256++ with splitmix64 seeding (rng.hpp:7-55)
class Xoshiro {
 public:
  explicit Xoshiro(uint64_t seed) {
    for (auto& w : s_) w = splitmix(seed);
  }
  static uint64_t splitmix(uint64_t& st) {
    uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint64_t next() {
    const uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return out;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double normal() {  // Box-Muller cosine branch, two uniforms per draw
    double u1 = uniform();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.28318530717958647692528676655900577 * u2);
  }

 private:
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t s_[4];
};

Xoshiro stream(uint64_t seed, uint64_t tag) {  // rng.hpp:57-59
  uint64_t a = seed, b = 0x517cc1b727220a95ULL + tag;
  return Xoshiro(Xoshiro::splitmix(a) ^ Xoshiro::splitmix(b));
}

enum Tag : uint64_t { kLambda = 1, kX = 2, kEps = 3, kP = 4, kAffine = 5, kA = 6, kB = 7 };

std::vector<double> normals(uint64_t seed, uint64_t tag, int64_t count) {
  std::vector<double> v((size_t)count);
  Xoshiro g = stream(seed, tag);
  for (auto& x : v) x = g.normal();
  return v;
}

std::vector<double> uniforms(uint64_t seed, uint64_t tag, int64_t count, double lo, double hi) {
  std::vector<double> v((size_t)count);
  Xoshiro g = stream(seed, tag);
  for (auto& x : v) x = lo + (hi - lo) * g.uniform();
  return v;
}

bool valid_dataset(const double* X, const double* y, int64_t N, int64_t n) {
  if (n < 1 || N < n + 1) return false;
  for (int64_t i = 0; i < N * n; ++i)
    if (!std::isfinite(X[i])) return false;
  for (int64_t i = 0; i < N; ++i)
    if (!std::isfinite(y[i])) return false;
  std::vector<int64_t> order((size_t)N);
  std::iota(order.begin(), order.end(), 0);
  auto less = [&](int64_t a, int64_t b) {
    return std::lexicographical_compare(X + a * n, X + a * n + n, X + b * n, X + b * n + n);
  };
  std::sort(order.begin(), order.end(), less);
  for (size_t k = 1; k < order.size(); ++k)
    if (std::equal(X + order[k - 1] * n, X + order[k - 1] * n + n, X + order[k] * n))
      return false;  // duplicate x rows (dataset.cpp:25-40)
  return true;
}

// OLS fit of y ~ a + b.x by column-pivoted Householder QR on D = [1 X];
// returns false when D is rank deficient (preprocess.cpp:26-40).
bool affine_ls(const double* X, const double* y, int64_t N, int64_t n, std::vector<double>& coef) {
  const int64_t m = n + 1;
  std::vector<std::vector<double>> col((size_t)m, std::vector<double>((size_t)N));
  for (int64_t i = 0; i < N; ++i) {
    col[0][i] = 1.0;
    for (int64_t j = 0; j < n; ++j) col[j + 1][i] = X[i * n + j];
  }
  std::vector<double> rhs(y, y + N), diag((size_t)m);
  std::vector<int64_t> perm((size_t)m);
  std::iota(perm.begin(), perm.end(), 0);
  auto tail_norm2 = [&](const std::vector<double>& c, int64_t from) {
    double s = 0;
    for (int64_t i = from; i < N; ++i) s += c[i] * c[i];
    return s;
  };
  double max_pivot = 0;
  for (int64_t k = 0; k < m; ++k) {
    int64_t best = k;
    double bestn = tail_norm2(col[k], k);
    for (int64_t j = k + 1; j < m; ++j) {
      const double t = tail_norm2(col[j], k);
      if (t > bestn) { bestn = t; best = j; }
    }
    std::swap(col[k], col[best]);
    std::swap(perm[k], perm[best]);
    std::vector<double>& v = col[k];
    const double nrm = std::sqrt(bestn);
    const double alpha = v[k] > 0 ? -nrm : nrm;
    diag[k] = alpha;
    max_pivot = std::max(max_pivot, std::fabs(alpha));
    if (nrm == 0) continue;
    v[k] -= alpha;
    const double vv = tail_norm2(v, k);
    if (vv == 0) continue;
    auto reflect = [&](std::vector<double>& w) {
      double d = 0;
      for (int64_t i = k; i < N; ++i) d += v[i] * w[i];
      const double f = 2.0 * d / vv;
      for (int64_t i = k; i < N; ++i) w[i] -= f * v[i];
    };
    for (int64_t j = k + 1; j < m; ++j) reflect(col[j]);
    reflect(rhs);
  }
  const double thresh = 2.220446049250313e-16 * (double)m * max_pivot;
  for (int64_t k = 0; k < m; ++k)
    if (!(std::fabs(diag[k]) > thresh)) return false;
  std::vector<double> z((size_t)m);
  for (int64_t k = m - 1; k >= 0; --k) {
    double s = rhs[k];
    for (int64_t j = k + 1; j < m; ++j) s -= col[j][k] * z[j];
    z[k] = s / diag[k];
  }
  coef.assign((size_t)m, 0.0);
  for (int64_t k = 0; k < m; ++k) coef[perm[k]] = z[k];
  return true;
}

}  // namespace

// The uniform pairs (u1, u2) of `count` Box-Muller draws, interleaved, in
// stream order: the sequential part of normal_stream (the device applies the
// transform for the sigma start vector).
void uniform_pairs(uint64_t seed, uint64_t tag, int64_t count, double* out2) {
  Xoshiro g = stream(seed, tag);
  for (int64_t i = 0; i < count; ++i) {
    out2[2 * i] = g.uniform();
    out2[2 * i + 1] = g.uniform();
  }
}

// The uniform pairs are drawn sequentially (the stream is sequential); the
// Box-Muller transform, which dominates the cost, runs on several threads.
// Bit-identical to calling Xoshiro::normal() count times.
void normal_stream(uint64_t seed, uint64_t tag, int64_t count, double* out, int max_threads) {
  Xoshiro g = stream(seed, tag);
  std::vector<double> u1((size_t)count), u2((size_t)count);
  for (int64_t i = 0; i < count; ++i) {
    u1[i] = g.uniform();
    u2[i] = g.uniform();
  }
  auto transform = [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      const double a = u1[i] <= 0.0 ? 0x1.0p-53 : u1[i];
      out[i] = std::sqrt(-2.0 * std::log(a)) * std::cos(6.28318530717958647692528676655900577 * u2[i]);
    }
  };
  const unsigned hw = std::thread::hardware_concurrency();
  const int64_t nt = count < 65536 ? 1 : std::max<int64_t>(1, std::min<int64_t>(hw ? hw : 1, max_threads));
  std::vector<std::thread> pool;
  for (int64_t t = 1; t < nt; ++t)
    pool.emplace_back(transform, count * t / nt, count * (t + 1) / nt);
  transform(0, count / nt);
  for (auto& th : pool) th.join();
}

}  // namespace host
}  // namespace crb

using namespace crb::host;

extern "C" {

cr_status cr_gen_instance(int32_t kind, int64_t N, int64_t n, double noise, uint64_t seed,
                          int64_t pieces, double* X, double* y) {
  if (!X || !y || N < n + 1 || n < 1) return CR_EINVAL;
  const size_t Nn = (size_t)(N * n);
  switch (kind) {
    case 0: {  // quadratic: 1/2 x^T L^T L x + noise eps
      const auto L = normals(seed, kLambda, n * n);
      const auto xs = normals(seed, kX, N * n);
      const auto eps = normals(seed, kEps, N);
      std::copy(xs.begin(), xs.end(), X);
      std::vector<double> Q((size_t)(n * n), 0.0);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
          double a = 0;
          for (int64_t k = 0; k < n; ++k) a += L[k * n + i] * L[k * n + j];
          Q[i * n + j] = a;
        }
      for (int64_t l = 0; l < N; ++l) {
        const double* x = X + l * n;
        double quad = 0;
        for (int64_t i = 0; i < n; ++i) {
          double qx = 0;
          for (int64_t j = 0; j < n; ++j) qx += Q[i * n + j] * x[j];
          quad += x[i] * qx;
        }
        y[l] = 0.5 * quad + noise * eps[l];
      }
      break;
    }
    case 1: {  // exponential: exp(p.x) + noise eps, p ~ U[0,1)
      const auto xs = normals(seed, kX, N * n);
      const auto eps = normals(seed, kEps, N);
      std::copy(xs.begin(), xs.end(), X);
      Xoshiro pg = stream(seed, kP);
      std::vector<double> p((size_t)n);
      for (auto& v : p) v = pg.uniform();
      for (int64_t l = 0; l < N; ++l) {
        double d = 0;
        for (int64_t j = 0; j < n; ++j) d += p[j] * X[l * n + j];
        y[l] = std::exp(d) + noise * eps[l];
      }
      break;
    }
    case 2: {  // affine-noiseless: a + b.x
      const auto xs = normals(seed, kX, N * n);
      const auto cf = normals(seed, kAffine, n + 1);
      std::copy(xs.begin(), xs.end(), X);
      for (int64_t l = 0; l < N; ++l) {
        double d = 0;
        for (int64_t j = 0; j < n; ++j) d += X[l * n + j] * cf[1 + j];
        y[l] = cf[0] + d;
      }
      break;
    }
    case 3: {  // custom-1d: x_l = l, y = |x - (N-1)/2| + noise eps
      if (n != 1) return CR_EINVAL;
      const auto eps = normals(seed, kEps, N);
      const double mid = 0.5 * (double)(N - 1);
      for (int64_t l = 0; l < N; ++l) {
        X[l] = (double)l;
        y[l] = std::fabs(X[l] - mid) + noise * eps[l];
      }
      break;
    }
    case 10: {  // BASELINE cfg 1/4: |x|^2 + eps, x ~ U[-1,1]^n, eps ~ U[-a,a]
      const auto xs = uniforms(seed, kX, N * n, -1.0, 1.0);
      const auto eps = uniforms(seed, kEps, N, -noise, noise);
      std::copy(xs.begin(), xs.end(), X);
      for (int64_t l = 0; l < N; ++l) {
        double s = 0;
        for (int64_t j = 0; j < n; ++j) s += X[l * n + j] * X[l * n + j];
        y[l] = s + eps[l];
      }
      break;
    }
    case 11: {  // BASELINE cfg 2/5: max_i (a_i.x + b_i) + eps
      if (pieces < 1) return CR_EINVAL;
      const auto xs = uniforms(seed, kX, N * n, -1.0, 1.0);
      const auto eps = uniforms(seed, kEps, N, -noise, noise);
      const auto A = normals(seed, kA, pieces * n);
      const auto B = normals(seed, kB, pieces);
      std::copy(xs.begin(), xs.end(), X);
      for (int64_t l = 0; l < N; ++l) {
        double best = -INFINITY;
        for (int64_t i = 0; i < pieces; ++i) {
          double d = B[i];
          for (int64_t j = 0; j < n; ++j) d += A[i * n + j] * X[l * n + j];
          best = std::max(best, d);
        }
        y[l] = best + eps[l];
      }
      break;
    }
    case 12: {  // BASELINE cfg 3: log sum_k exp(a_k.x) + eps, a_k ~ N(0, I/20)
      if (pieces < 1) return CR_EINVAL;
      const auto xs = uniforms(seed, kX, N * n, -1.0, 1.0);
      const auto eps = uniforms(seed, kEps, N, -noise, noise);
      auto A = normals(seed, kA, pieces * n);
      const double sc = std::sqrt(1.0 / 20.0);
      for (auto& a : A) a *= sc;
      std::copy(xs.begin(), xs.end(), X);
      for (int64_t l = 0; l < N; ++l) {
        double s = 0;
        for (int64_t k = 0; k < pieces; ++k) {
          double d = 0;
          for (int64_t j = 0; j < n; ++j) d += A[k * n + j] * X[l * n + j];
          s += std::exp(d);
        }
        y[l] = std::log(s) + eps[l];
      }
      break;
    }
    default:
      return CR_EINVAL;
  }
  (void)Nn;
  return valid_dataset(X, y, N, n) ? CR_OK : CR_EINVAL;
}

cr_status cr_prepare_problem(const double* X, const double* y, int64_t N, int64_t n, double gamma,
                             double* ys_shifted, double* shift, double* feas_y, double* feas_xi,
                             double* bounds4) {
  if (!X || !y || !ys_shifted || !shift || !feas_y || !feas_xi || !bounds4) return CR_EINVAL;
  if (!(gamma > 0) || N < n + 1 || n < 1) return CR_EINVAL;
  std::vector<double> coef;
  double a = 0;
  std::vector<double> b((size_t)n, 0.0);
  if (affine_ls(X, y, N, n, coef)) {
    a = coef[0];
    for (int64_t j = 0; j < n; ++j) b[j] = coef[1 + j];
  } else {  // constant fit (preprocess.cpp:36-40)
    double s = 0;
    for (int64_t i = 0; i < N; ++i) s += y[i];
    a = s / (double)N;
  }
  double ry = 0, rxi = 0;
  for (int64_t l = 0; l < N; ++l) {
    double d = 0;
    for (int64_t j = 0; j < n; ++j) d += X[l * n + j] * b[j];
    feas_y[l] = a + d;
    ry += (feas_y[l] - y[l]) * (feas_y[l] - y[l]);
    for (int64_t j = 0; j < n; ++j) feas_xi[l * n + j] = b[j];
  }
  for (int64_t i = 0; i < N * n; ++i) rxi += feas_xi[i] * feas_xi[i];
  const double Bbar = std::max(std::sqrt(ry + gamma * rxi), 1e-8);
  const double ymin = *std::min_element(y, y + N);
  const double s = std::max(0.0, Bbar - ymin);  // preprocess.cpp:43-48
  *shift = s;
  for (int64_t i = 0; i < N; ++i) {
    ys_shifted[i] = y[i] + s;
    feas_y[i] += s;
  }
  bounds4[0] = 10.0 * std::sqrt((double)N);
  bounds4[1] = Bbar;
  bounds4[2] = Bbar / std::sqrt(gamma);
  bounds4[3] = gamma;
  return CR_OK;
}

void cr_certificate(double gamma, double delta, double B_xi_estimate, double sigma_max_C,
                    double out2[2]) {  // papg.cpp:298-303
  const double spread = std::sqrt(2.0 * std::max(delta, 0.0) / gamma) * sigma_max_C;
  out2[0] = B_xi_estimate * std::sqrt(gamma) + spread;
  out2[1] = spread;
}

double cr_momentum_next(double t) { return 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t)); }

}  // extern "C"
