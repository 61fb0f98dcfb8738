/*
 * cvxreg_oracle.c -- TEST INFRASTRUCTURE ONLY (see cvxreg_oracle.h).
 *
 * Literal CPU restatement of the reference's singleton-block P-APG path.
 * Every function cites the reference lines it follows; loops keep the
 * reference's canonical row order and accumulation order. Compiled with
 * -ffp-contract=off so a*b+c stays two roundings, as the reference's default
 * x86-64 build (no -march, so no FMA) computes it.
 */
#include "cvxreg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ PRNG */
/* rng.hpp:7-59 */
static uint64_t splitmix64(uint64_t *state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t mix64(uint64_t x) { return splitmix64(&x); }

typedef struct { uint64_t s[4]; } xo256;

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static void xo_seed(xo256 *g, uint64_t seed) {
  for (int i = 0; i < 4; ++i) g->s[i] = splitmix64(&seed);
}
static uint64_t xo_next(xo256 *g) {
  uint64_t *s = g->s;
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}
static double xo_uniform(xo256 *g) { return (double)(xo_next(g) >> 11) * 0x1.0p-53; }
static double xo_normal(xo256 *g) {
  double u1 = xo_uniform(g);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  const double u2 = xo_uniform(g);
  return sqrt(-2.0 * log(u1)) * cos(6.28318530717958647692528676655900577 * u2);
}
/* rng.hpp:57-59 */
static xo256 rng_stream(uint64_t seed, uint64_t tag) {
  xo256 g;
  xo_seed(&g, mix64(seed) ^ mix64(0x517cc1b727220a95ULL + tag));
  return g;
}

uint64_t cro_rng_draws(uint64_t seed, uint64_t tag, int64_t count, int kind, double *out) {
  xo256 g = rng_stream(seed, tag);
  uint64_t last = 0;
  for (int64_t i = 0; i < count; ++i) {
    if (kind == 0) out[i] = xo_uniform(&g);
    else if (kind == 1) out[i] = xo_normal(&g);
    else { last = xo_next(&g); out[i] = (double)(last >> 11); }
  }
  return last;
}

/* ------------------------------------------------------------ generators */
/* tags: testgen.cpp:12-16; 6/7 are the new BASELINE kinds */
enum { TAG_LAMBDA = 1, TAG_X = 2, TAG_EPS = 3, TAG_P = 4, TAG_AFFINE = 5, TAG_A = 6, TAG_B = 7 };

static void normal_fill(uint64_t seed, uint64_t tag, int64_t count, double *out) {
  xo256 g = rng_stream(seed, tag);
  for (int64_t i = 0; i < count; ++i) out[i] = xo_normal(&g); /* row-major, testgen.cpp:22-23 */
}
static void uniform_fill(uint64_t seed, uint64_t tag, int64_t count, double lo, double hi,
                         double *out) {
  xo256 g = rng_stream(seed, tag);
  for (int64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * xo_uniform(&g);
}

static int row_cmp_n;
static const double *row_cmp_X;
static int row_cmp(const void *a, const void *b) {
  const int64_t ia = *(const int64_t *)a, ib = *(const int64_t *)b;
  for (int j = 0; j < row_cmp_n; ++j) {
    const double xa = row_cmp_X[ia * row_cmp_n + j], xb = row_cmp_X[ib * row_cmp_n + j];
    if (xa != xb) return xa < xb ? -1 : 1;
  }
  return 0;
}

/* dataset.cpp:14-42 */
static int validate_dataset(const double *X, const double *y, int64_t N, int64_t n) {
  if (n < 1 || N < n + 1) return -1;
  for (int64_t i = 0; i < N * n; ++i) if (!isfinite(X[i])) return -1;
  for (int64_t i = 0; i < N; ++i) if (!isfinite(y[i])) return -1;
  int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
  for (int64_t i = 0; i < N; ++i) order[i] = i;
  row_cmp_n = (int)n;
  row_cmp_X = X;
  qsort(order, (size_t)N, sizeof(int64_t), row_cmp);
  int rc = 0;
  for (int64_t k = 1; k < N; ++k)
    if (row_cmp(&order[k - 1], &order[k]) == 0) { rc = -2; break; }
  free(order);
  return rc;
}

/* testgen.cpp:36-87 plus the BASELINE.json kinds */
int cro_gen_instance(int kind, int64_t N, int64_t n, double noise, uint64_t seed,
                     int64_t pieces, double *X, double *y) {
  if (N < n + 1 || n < 1) return -1;
  switch (kind) {
    case CRO_GEN_QUADRATIC: {
      double *Lam = (double *)malloc(sizeof(double) * (size_t)(n * n));
      double *Q = (double *)calloc((size_t)(n * n), sizeof(double));
      double *eps = (double *)malloc(sizeof(double) * (size_t)N);
      normal_fill(seed, TAG_LAMBDA, n * n, Lam);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
          double acc = 0;
          for (int64_t k = 0; k < n; ++k) acc += Lam[k * n + i] * Lam[k * n + j];
          Q[i * n + j] = acc;
        }
      normal_fill(seed, TAG_X, N * n, X);
      normal_fill(seed, TAG_EPS, N, eps);
      for (int64_t l = 0; l < N; ++l) {
        const double *x = X + l * n;
        double quad = 0;
        for (int64_t i = 0; i < n; ++i) {
          double qx = 0;
          for (int64_t j = 0; j < n; ++j) qx += Q[i * n + j] * x[j];
          quad += x[i] * qx;
        }
        y[l] = 0.5 * quad + noise * eps[l];
      }
      free(Lam); free(Q); free(eps);
      break;
    }
    case CRO_GEN_EXPONENTIAL: {
      double *eps = (double *)malloc(sizeof(double) * (size_t)N);
      double *p = (double *)malloc(sizeof(double) * (size_t)n);
      normal_fill(seed, TAG_X, N * n, X);
      normal_fill(seed, TAG_EPS, N, eps);
      xo256 pg = rng_stream(seed, TAG_P);
      for (int64_t j = 0; j < n; ++j) p[j] = xo_uniform(&pg);
      for (int64_t l = 0; l < N; ++l) {
        double d = 0;
        for (int64_t j = 0; j < n; ++j) d += p[j] * X[l * n + j];
        y[l] = exp(d) + noise * eps[l];
      }
      free(eps); free(p);
      break;
    }
    case CRO_GEN_AFFINE_NOISELESS: {
      double *coef = (double *)malloc(sizeof(double) * (size_t)(n + 1));
      normal_fill(seed, TAG_X, N * n, X);
      normal_fill(seed, TAG_AFFINE, n + 1, coef);
      for (int64_t l = 0; l < N; ++l) {
        double d = 0;
        for (int64_t j = 0; j < n; ++j) d += X[l * n + j] * coef[1 + j];
        y[l] = coef[0] + d;
      }
      free(coef);
      break;
    }
    case CRO_GEN_CUSTOM_1D: {
      if (n != 1) return -1;
      double *eps = (double *)malloc(sizeof(double) * (size_t)N);
      for (int64_t l = 0; l < N; ++l) X[l] = (double)l;
      normal_fill(seed, TAG_EPS, N, eps);
      const double mid = 0.5 * (double)(N - 1);
      for (int64_t l = 0; l < N; ++l) y[l] = fabs(X[l] - mid) + noise * eps[l];
      free(eps);
      break;
    }
    case CRO_GEN_SQNORM_UNIFORM: {
      double *eps = (double *)malloc(sizeof(double) * (size_t)N);
      uniform_fill(seed, TAG_X, N * n, -1.0, 1.0, X);
      uniform_fill(seed, TAG_EPS, N, -noise, noise, eps);
      for (int64_t l = 0; l < N; ++l) {
        double s = 0;
        for (int64_t j = 0; j < n; ++j) s += X[l * n + j] * X[l * n + j];
        y[l] = s + eps[l];
      }
      free(eps);
      break;
    }
    case CRO_GEN_MAXAFFINE_UNIFORM: {
      if (pieces < 1) return -1;
      double *eps = (double *)malloc(sizeof(double) * (size_t)N);
      double *A = (double *)malloc(sizeof(double) * (size_t)(pieces * n));
      double *B = (double *)malloc(sizeof(double) * (size_t)pieces);
      uniform_fill(seed, TAG_X, N * n, -1.0, 1.0, X);
      uniform_fill(seed, TAG_EPS, N, -noise, noise, eps);
      normal_fill(seed, TAG_A, pieces * n, A);
      normal_fill(seed, TAG_B, pieces, B);
      for (int64_t l = 0; l < N; ++l) {
        double best = -INFINITY;
        for (int64_t i = 0; i < pieces; ++i) {
          double d = B[i];
          for (int64_t j = 0; j < n; ++j) d += A[i * n + j] * X[l * n + j];
          if (d > best) best = d;
        }
        y[l] = best + eps[l];
      }
      free(eps); free(A); free(B);
      break;
    }
    case CRO_GEN_LSE_UNIFORM: {
      if (pieces < 1) return -1;
      double *eps = (double *)malloc(sizeof(double) * (size_t)N);
      double *A = (double *)malloc(sizeof(double) * (size_t)(pieces * n));
      uniform_fill(seed, TAG_X, N * n, -1.0, 1.0, X);
      uniform_fill(seed, TAG_EPS, N, -noise, noise, eps);
      normal_fill(seed, TAG_A, pieces * n, A);
      const double scale = sqrt(1.0 / 20.0); /* a_k ~ N(0, I/20) (BASELINE cfg 3) */
      for (int64_t i = 0; i < pieces * n; ++i) A[i] *= scale;
      for (int64_t l = 0; l < N; ++l) {
        double s = 0;
        for (int64_t k = 0; k < pieces; ++k) {
          double d = 0;
          for (int64_t j = 0; j < n; ++j) d += A[k * n + j] * X[l * n + j];
          s += exp(d);
        }
        y[l] = log(s) + eps[l];
      }
      free(eps); free(A);
      break;
    }
    default:
      return -1;
  }
  return validate_dataset(X, y, N, n);
}

/* ------------------------------------------------------------ preprocess */
/* Least squares min |D c - y| with D = [1, X] by column-pivoted Householder
   QR; rank test as Eigen's ColPivHouseholderQR default threshold
   (preprocess.cpp:26-36). */
static int lsq_affine(const double *X, const double *y, int64_t N, int64_t n, double *coef) {
  const int64_t m = n + 1;
  double *D = (double *)malloc(sizeof(double) * (size_t)(N * m)); /* column-major */
  double *b = (double *)malloc(sizeof(double) * (size_t)N);
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
  double *cn = (double *)malloc(sizeof(double) * (size_t)m);
  for (int64_t i = 0; i < N; ++i) {
    D[i] = 1.0;
    for (int64_t j = 0; j < n; ++j) D[(j + 1) * N + i] = X[i * n + j];
    b[i] = y[i];
  }
  for (int64_t j = 0; j < m; ++j) {
    perm[j] = j;
    double s = 0;
    for (int64_t i = 0; i < N; ++i) s += D[j * N + i] * D[j * N + i];
    cn[j] = s;
  }
  double maxpivot = 0;
  int64_t rank = 0;
  double *rdiag = (double *)malloc(sizeof(double) * (size_t)m);
  for (int64_t k = 0; k < m; ++k) {
    int64_t best = k;
    for (int64_t j = k + 1; j < m; ++j) if (cn[j] > cn[best]) best = j;
    if (best != k) {
      for (int64_t i = 0; i < N; ++i) {
        double t = D[k * N + i]; D[k * N + i] = D[best * N + i]; D[best * N + i] = t;
      }
      double t = cn[k]; cn[k] = cn[best]; cn[best] = t;
      int64_t tp = perm[k]; perm[k] = perm[best]; perm[best] = tp;
    }
    double *col = D + k * N;
    double norm = 0;
    for (int64_t i = k; i < N; ++i) norm += col[i] * col[i];
    norm = sqrt(norm);
    double alpha = col[k] > 0 ? -norm : norm;
    rdiag[k] = alpha;
    if (fabs(alpha) > maxpivot) maxpivot = fabs(alpha);
    if (norm > 0) {
      col[k] -= alpha;
      double vnorm2 = 0;
      for (int64_t i = k; i < N; ++i) vnorm2 += col[i] * col[i];
      if (vnorm2 > 0) {
        for (int64_t j = k + 1; j < m; ++j) {
          double *cj = D + j * N;
          double d = 0;
          for (int64_t i = k; i < N; ++i) d += col[i] * cj[i];
          const double f = 2.0 * d / vnorm2;
          for (int64_t i = k; i < N; ++i) cj[i] -= f * col[i];
        }
        double d = 0;
        for (int64_t i = k; i < N; ++i) d += col[i] * b[i];
        const double f = 2.0 * d / vnorm2;
        for (int64_t i = k; i < N; ++i) b[i] -= f * col[i];
      }
    }
    for (int64_t j = k + 1; j < m; ++j) {
      double s = 0;
      for (int64_t i = k + 1; i < N; ++i) s += D[j * N + i] * D[j * N + i];
      cn[j] = s;
    }
  }
  const double threshold = 2.220446049250313e-16 * (double)m;
  for (int64_t k = 0; k < m; ++k) if (fabs(rdiag[k]) > threshold * maxpivot) ++rank;
  int ok = rank == m;
  if (ok) {
    double *z = (double *)malloc(sizeof(double) * (size_t)m);
    for (int64_t k = m - 1; k >= 0; --k) {
      double s = b[k];
      for (int64_t j = k + 1; j < m; ++j) s -= D[j * N + k] * z[j];
      z[k] = s / rdiag[k];
    }
    for (int64_t k = 0; k < m; ++k) coef[perm[k]] = z[k];
    free(z);
  }
  free(D); free(b); free(perm); free(cn); free(rdiag);
  return ok;
}

int cro_prepare(const double *X, const double *y, int64_t N, int64_t n, double gamma,
                double *ys_shifted, double *shift, double *feas_y, double *feas_xi,
                double *bounds4, double *intercept, double *slope) {
  if (gamma <= 0 || N < n + 1) return -1;
  double *coef = (double *)malloc(sizeof(double) * (size_t)(n + 1));
  if (lsq_affine(X, y, N, n, coef)) {
    *intercept = coef[0];
    for (int64_t j = 0; j < n; ++j) slope[j] = coef[1 + j];
  } else { /* preprocess.cpp:36-40 constant fallback */
    double s = 0;
    for (int64_t i = 0; i < N; ++i) s += y[i];
    *intercept = s / (double)N;
    for (int64_t j = 0; j < n; ++j) slope[j] = 0;
  }
  free(coef);
  /* preprocess.cpp:42-50 */
  double bsq_y = 0, bsq_xi = 0;
  for (int64_t l = 0; l < N; ++l) {
    double d = 0;
    for (int64_t j = 0; j < n; ++j) d += X[l * n + j] * slope[j];
    feas_y[l] = *intercept + d;
    const double r = feas_y[l] - y[l];
    bsq_y += r * r;
    for (int64_t j = 0; j < n; ++j) feas_xi[l * n + j] = slope[j];
  }
  for (int64_t i = 0; i < N * n; ++i) bsq_xi += feas_xi[i] * feas_xi[i];
  double Bbar = sqrt(bsq_y + gamma * bsq_xi);
  if (Bbar < 1e-8) Bbar = 1e-8;
  /* preprocess.cpp:43-48 shift */
  double ymin = y[0];
  for (int64_t i = 1; i < N; ++i) if (y[i] < ymin) ymin = y[i];
  double s = Bbar - ymin;
  if (s < 0) s = 0;
  *shift = s;
  for (int64_t i = 0; i < N; ++i) { ys_shifted[i] = y[i] + s; feas_y[i] += s; }
  bounds4[0] = 10.0 * sqrt((double)N);
  bounds4[1] = Bbar;
  bounds4[2] = Bbar / sqrt(gamma);
  bounds4[3] = gamma;
  return 0;
}

/* ------------------------------------------------------------- operators */
/* operators.cpp:128-153, singleton partition: cross order == full (l1,l2)
   lexicographic order with the diagonal skipped (indexing.hpp:30-37). */
void cro_apply_C(const double *X, int64_t N, int64_t n, const double *y, const double *xi,
                 double *out) {
  int64_t r = 0;
  for (int64_t l1 = 0; l1 < N; ++l1) {
    const double y1 = y[l1];
    const double *x1 = X + l1 * n;
    for (int64_t l2 = 0; l2 < N; ++l2) {
      if (l1 == l2) continue;
      double acc = y1 - y[l2];
      const double *xi2 = xi + l2 * n;
      const double *x2 = X + l2 * n;
      for (int64_t j = 0; j < n; ++j) acc -= xi2[j] * (x1[j] - x2[j]);
      out[r++] = acc;
    }
  }
  for (int64_t l = 0; l < N; ++l) out[r + l] = y[l]; /* :152 */
}

/* operators.cpp:155-180 */
void cro_apply_C_T(const double *X, int64_t N, int64_t n, const double *theta,
                   double *out_y, double *out_xi) {
  const int64_t rows_cross = N * (N - 1);
  for (int64_t l = 0; l < N; ++l) out_y[l] = theta[rows_cross + l]; /* :161 */
  memset(out_xi, 0, sizeof(double) * (size_t)(N * n));
  int64_t r = 0;
  for (int64_t l1 = 0; l1 < N; ++l1) {
    const double *x1 = X + l1 * n;
    for (int64_t l2 = 0; l2 < N; ++l2) {
      if (l1 == l2) continue;
      const double tr = theta[r++];
      out_y[l1] += tr;
      out_y[l2] -= tr;
      double *o2 = out_xi + l2 * n;
      const double *x2 = X + l2 * n;
      for (int64_t j = 0; j < n; ++j) o2[j] -= tr * (x1[j] - x2[j]);
    }
  }
}

/* Row-parallel variants for the timed multi-core CPU baseline. apply_C is
   embarrassingly parallel by l1; apply_C_T accumulates per-thread partials
   over contiguous l1 ranges and combines them in thread order. */
static void apply_C_omp(const double *X, int64_t N, int64_t n, const double *y,
                        const double *xi, double *out, int threads) {
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t l1 = 0; l1 < N; ++l1) {
    int64_t r = l1 * (N - 1);
    const double y1 = y[l1];
    const double *x1 = X + l1 * n;
    for (int64_t l2 = 0; l2 < N; ++l2) {
      if (l1 == l2) continue;
      double acc = y1 - y[l2];
      const double *xi2 = xi + l2 * n;
      const double *x2 = X + l2 * n;
      for (int64_t j = 0; j < n; ++j) acc -= xi2[j] * (x1[j] - x2[j]);
      out[r++] = acc;
    }
  }
  for (int64_t l = 0; l < N; ++l) out[N * (N - 1) + l] = y[l];
}

static void apply_C_T_omp(const double *X, int64_t N, int64_t n, const double *theta,
                          double *out_y, double *out_xi, int threads) {
  const int64_t rows_cross = N * (N - 1);
  const int64_t w = N * (n + 1);
  double *part = (double *)calloc((size_t)(w * threads), sizeof(double));
#pragma omp parallel num_threads(threads)
  {
    int tid = 0, nt = 1;
#ifdef _OPENMP
    tid = omp_get_thread_num();
    nt = omp_get_num_threads();
#endif
    double *py = part + (int64_t)tid * w;
    double *pxi = py + N;
    const int64_t lo = N * tid / nt, hi = N * (tid + 1) / nt;
    for (int64_t l1 = lo; l1 < hi; ++l1) {
      int64_t r = l1 * (N - 1);
      const double *x1 = X + l1 * n;
      for (int64_t l2 = 0; l2 < N; ++l2) {
        if (l1 == l2) continue;
        const double tr = theta[r++];
        py[l1] += tr;
        py[l2] -= tr;
        double *o2 = pxi + l2 * n;
        const double *x2 = X + l2 * n;
        for (int64_t j = 0; j < n; ++j) o2[j] -= tr * (x1[j] - x2[j]);
      }
    }
  }
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t k = 0; k < w; ++k) {
    double s = k < N ? theta[rows_cross + k] : 0.0;
    for (int t = 0; t < threads; ++t) s += part[(int64_t)t * w + k];
    if (k < N) out_y[k] = s; else out_xi[k - N] = s;
  }
  free(part);
}

static double dot(const double *a, const double *b, int64_t len) {
  double s = 0;
  for (int64_t i = 0; i < len; ++i) s += a[i] * b[i];
  return s;
}
static double dot_omp(const double *a, const double *b, int64_t len, int threads) {
  double s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static) num_threads(threads)
  for (int64_t i = 0; i < len; ++i) s += a[i] * b[i];
  return s;
}

/* --------------------------------------------------------- power method */
/* operators.cpp:302-339 applied to op_C (:353-369) */
int cro_sigma_C(const double *X, int64_t N, int64_t n, double tol, int max_iters,
                double *sigma, int *iters, int *converged) {
  const int64_t cols = N * (n + 1);
  const int64_t rows = N * (N - 1) + N;
  double *v = (double *)malloc(sizeof(double) * (size_t)cols);
  double *u = (double *)malloc(sizeof(double) * (size_t)cols);
  double *w = (double *)malloc(sizeof(double) * (size_t)rows);
  if (!v || !u || !w) { free(v); free(u); free(w); return -1; }
  xo256 g = rng_stream(0x5eedULL, 97);
  for (int64_t k = 0; k < cols; ++k) v[k] = xo_normal(&g);
  double nv = sqrt(dot(v, v, cols));
  for (int64_t k = 0; k < cols; ++k) v[k] /= nv;
  double lambda_prev = 0;
  *converged = 1;
  *iters = 0;
  for (int it = 1; it <= max_iters; ++it) {
    cro_apply_C(X, N, n, v, v + N, w);
    const double lambda = dot(w, w, rows);
    cro_apply_C_T(X, N, n, w, u, u + N);
    const double norm_u = sqrt(dot(u, u, cols));
    if (norm_u == 0 || lambda == 0) {
      *sigma = 0;
      *iters = it;
      free(v); free(u); free(w);
      return 0;
    }
    for (int64_t k = 0; k < cols; ++k) v[k] = u[k] / norm_u;
    *iters = it;
    if (it > 1 && fabs(lambda - lambda_prev) <= tol * lambda) {
      *sigma = sqrt(lambda) * 1.01;
      *converged = 1;
      free(v); free(u); free(w);
      return 0;
    }
    lambda_prev = lambda;
  }
  *sigma = sqrt(lambda_prev) * 1.10;
  *converged = 0;
  free(v); free(u); free(w);
  return 0;
}

/* --------------------------------------------------------------- metrics */
/* metrics.cpp:8-15: apply_rows (operators.cpp:87-105) then |(-r)_+| */
void cro_infeasibility(const double *X, int64_t N, int64_t n, const double *y, const double *xi,
                       double out2[2]) {
  double ss = 0;
  for (int64_t l1 = 0; l1 < N; ++l1) {
    const double *x1 = X + l1 * n;
    for (int64_t l2 = 0; l2 < N; ++l2) {
      if (l1 == l2) continue;
      double acc = y[l1] - y[l2];
      const double *xi2 = xi + l2 * n;
      const double *x2 = X + l2 * n;
      for (int64_t j = 0; j < n; ++j) acc -= xi2[j] * (x1[j] - x2[j]);
      const double m = -acc > 0.0 ? -acc : 0.0;
      ss += m * m;
    }
  }
  out2[0] = sqrt(ss);
  out2[1] = out2[0] / sqrt((double)(N * (N - 1)));
}

/* metrics.cpp:17-30 */
void cro_duality_gap(const double *X, int64_t N, int64_t n, const double *theta, const double *y,
                     const double *xi, double out2[2]) {
  const int64_t dim = N * (N - 1) + N;
  double *ce = (double *)malloc(sizeof(double) * (size_t)dim);
  cro_apply_C(X, N, n, y, xi, ce);
  double a = 0, b = 0;
  for (int64_t i = 0; i < N * (N - 1); ++i) a += theta[i] * ce[i];
  for (int64_t i = 0; i < N; ++i) b += theta[N * (N - 1) + i] * ce[N * (N - 1) + i];
  free(ce);
  out2[0] = a + b;
  out2[1] = out2[0] / (double)(N * (N - 1));
}

/* metrics.cpp:32-48 */
double cro_evaluate_estimator(const double *X, int64_t N, int64_t n, const double *y,
                              const double *xi, const double *xq) {
  double best = -INFINITY;
  for (int64_t l = 0; l < N; ++l) {
    double v = y[l];
    const double *xil = xi + l * n;
    for (int64_t j = 0; j < n; ++j) v += xil[j] * (xq[j] - X[l * n + j]);
    if (v > best) best = v;
  }
  return best;
}

/* metrics.cpp:50-56 */
void cro_repair_feasibility(const double *X, int64_t N, int64_t n, const double *y,
                            const double *xi, double *y_out) {
  for (int64_t l = 0; l < N; ++l) y_out[l] = cro_evaluate_estimator(X, N, n, y, xi, X + l * n);
}

/* ----------------------------------------------------------- small ops */
void cro_project_nonneg_ball(double *v, int64_t len, double radius) { /* projections.hpp:9-13 */
  for (int64_t i = 0; i < len; ++i) v[i] = v[i] > 0.0 ? v[i] : 0.0;
  const double norm = sqrt(dot(v, v, len));
  if (norm > radius) {
    const double s = radius / norm;
    for (int64_t i = 0; i < len; ++i) v[i] *= s;
  }
}
double cro_momentum_next(double t) { return 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t)); }
void cro_certificate(double gamma, double delta, double B_xi, double sigma, double out2[2]) {
  const double spread = sqrt(2.0 * (delta > 0 ? delta : 0.0) / gamma) * sigma; /* papg.cpp:301 */
  out2[0] = B_xi * sqrt(gamma) + spread;
  out2[1] = spread;
}
int64_t cro_cross_position(int64_t N, int64_t K, int64_t l1, int64_t l2) { /* indexing.hpp:30-37 */
  const int64_t nbar = N / K;
  const int64_t i = l1 / nbar, j = l2 / nbar;
  if (i == j) return -1;
  const int64_t pair_rank = i * (K - 1) + j - (j > i ? 1 : 0);
  const int64_t local = (l1 - i * nbar) * nbar + (l2 - j * nbar);
  return pair_rank * nbar * nbar + local;
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------ dual ascent loop */
typedef struct {
  const double *X, *ys;
  int64_t N, n;
  double gamma;
  int threads;
  double *q_y, *q_xi; /* C^T theta */
  double *ey, *exi;   /* eta */
} dg_ctx;

/* papg.cpp:89-132 with the singleton closed-form block minimiser
   (alcc.cpp:233-235 centres; block objective alcc.cpp:254-256). */
static double block_minimisers(dg_ctx *c);
static double dual_gradient(dg_ctx *c, const double *theta, double *C_eta) {
  const int64_t N = c->N, n = c->n;
  if (c->threads > 1) apply_C_T_omp(c->X, N, n, theta, c->q_y, c->q_xi, c->threads);
  else cro_apply_C_T(c->X, N, n, theta, c->q_y, c->q_xi);
  const double g = block_minimisers(c);
  if (c->threads > 1) apply_C_omp(c->X, N, n, c->ey, c->exi, C_eta, c->threads);
  else cro_apply_C(c->X, N, n, c->ey, c->exi, C_eta);
  return g;
}

/* papg.cpp:107-129: K = N singleton block minimisers from q = C^T theta
   (alcc.cpp:233-235 centres, alcc.cpp:254-256 objective), gathered in block order */
static double block_minimisers(dg_ctx *c) {
  const int64_t N = c->N, n = c->n;
  double g = 0;
  for (int64_t i = 0; i < N; ++i) { /* block i = {i}; gathered in block order (:124-128) */
    const double y = c->ys[i] + c->q_y[i];
    c->ey[i] = y;
    double xx = 0, qx = 0;
    for (int64_t j = 0; j < n; ++j) {
      const double xi = c->q_xi[i * n + j] / c->gamma;
      c->exi[i * n + j] = xi;
      xx += xi * xi;
      qx += c->q_xi[i * n + j] * xi;
    }
    const double dy = y - c->ys[i];
    const double obj = 0.5 * (dy * dy) + 0.5 * c->gamma * xx - c->q_y[i] * y - qx;
    g += obj;
  }
  return g;
}

int cro_papg(const double *X, const double *ys, int64_t N, int64_t n, const cro_config *cfg,
             const double *theta0, cro_result *res) {
  const double start = now_seconds();
  if (N < 2 || n < 1 || cfg->gamma <= 0) return -1;
  const int threads = cfg->threads > 1 ? cfg->threads : 1;
  const int64_t rows_total = N * (N - 1); /* papg.cpp:142-145 */
  const int64_t rows_cross = rows_total;  /* singleton: rows_cross = N(N - nbar) = N(N-1) */
  const int64_t dim = rows_cross + N;
  const double infeas_div = sqrt((double)rows_total);
  const double gap_div = (double)rows_total;

  double sigma_C = cfg->sigma_C;
  res->sigma_iters = 0;
  res->sigma_converged = 1;
  if (!(sigma_C > 0)) {
    int it = 0, conv = 0;
    if (cro_sigma_C(X, N, n, 1e-6, 5000, &sigma_C, &it, &conv)) return -2;
    res->sigma_iters = it;
    res->sigma_converged = conv;
  }
  const double L_g = sigma_C * sigma_C / cfg->gamma; /* papg.hpp:43 */
  double B_theta = cfg->B_theta > 0 ? cfg->B_theta : 10.0 * sqrt((double)N);
  res->sigma_C = sigma_C;
  res->L_g = L_g;
  res->reason = CRO_ITER_BUDGET;

  double *theta1 = (double *)calloc((size_t)dim, sizeof(double));
  double *theta1_prev = (double *)malloc(sizeof(double) * (size_t)dim);
  double *theta2 = (double *)malloc(sizeof(double) * (size_t)dim);
  double *C_eta = (double *)malloc(sizeof(double) * (size_t)dim);
  dg_ctx c = {X, ys, N, n, cfg->gamma, threads,
              (double *)malloc(sizeof(double) * (size_t)N),
              (double *)malloc(sizeof(double) * (size_t)(N * n)),
              (double *)malloc(sizeof(double) * (size_t)N),
              (double *)malloc(sizeof(double) * (size_t)(N * n))};
  if (!theta1 || !theta1_prev || !theta2 || !C_eta) return -3;
  if (theta0) { /* papg.cpp:159-164 */
    memcpy(theta1, theta0, sizeof(double) * (size_t)dim);
    cro_project_nonneg_ball(theta1, dim, B_theta);
  }
  memcpy(theta1_prev, theta1, sizeof(double) * (size_t)dim);
  memcpy(theta2, theta1, sizeof(double) * (size_t)dim);
  double t = 1.0;
  double g_star_upper = INFINITY;
  const int64_t K = N; /* singleton partition */
  int64_t ell = 0;
  int restarts = 0;
  int rc = 0;

  while (1) {
    ++ell;
    const double inv3 = 1.0 / ((double)ell * (double)ell * (double)ell);
    const double inner_tol = cfg->inner_tol_floor < inv3 ? cfg->inner_tol_floor : inv3;

    const double g_value = dual_gradient(&c, theta2, C_eta); /* :183 */
    int finite = 1;
    for (int64_t i = 0; i < dim; ++i) if (!isfinite(C_eta[i])) { finite = 0; break; }
    if (!finite) { res->reason = CRO_ERROR; rc = -4; break; } /* :184-185 */

    { double *tmp = theta1_prev; theta1_prev = theta1; theta1 = tmp; } /* :187 */
    if (threads > 1) {
#pragma omp parallel for schedule(static) num_threads(threads)
      for (int64_t i = 0; i < dim; ++i) theta1[i] = theta2[i] - C_eta[i] / L_g; /* :188 */
      double ss = 0;
#pragma omp parallel for reduction(+ : ss) schedule(static) num_threads(threads)
      for (int64_t i = 0; i < dim; ++i) {
        theta1[i] = theta1[i] > 0.0 ? theta1[i] : 0.0;
        ss += theta1[i] * theta1[i];
      }
      const double norm = sqrt(ss);
      if (norm > B_theta) {
        const double s = B_theta / norm;
#pragma omp parallel for schedule(static) num_threads(threads)
        for (int64_t i = 0; i < dim; ++i) theta1[i] *= s;
      }
    } else {
      for (int64_t i = 0; i < dim; ++i) theta1[i] = theta2[i] - C_eta[i] / L_g; /* :188 */
      cro_project_nonneg_ball(theta1, dim, B_theta);                          /* :189 */
    }

    /* :191-199 linearisation bound */
    double cross_sq = 0, all_sq = 0;
    for (int64_t i = 0; i < dim; ++i) {
      const double m = -C_eta[i] > 0.0 ? -C_eta[i] : 0.0;
      if (i < rows_cross) cross_sq += m * m;
      all_sq += m * m;
    }
    const double cross_infeas = rows_cross > 0 ? sqrt(cross_sq) : 0.0;
    const double t2c = threads > 1 ? dot_omp(theta2, C_eta, dim, threads) : dot(theta2, C_eta, dim);
    const double fw = B_theta * sqrt(all_sq) + t2c;
    const double cushion = 2.0 * inner_tol * (double)K;
    const double cand = g_value + fw + cushion;
    if (cand < g_star_upper) g_star_upper = cand;

    /* :201-208 */
    const double gap_raw =
        cfg->use_momentum ? (threads > 1 ? dot_omp(theta1, C_eta, dim, threads) : dot(theta1, C_eta, dim))
                          : t2c;
    const double within = 0.0; /* singleton blocks have no within rows */
    const double infeas_raw = sqrt(within * within + cross_infeas * cross_infeas);
    const double gap_norm = gap_raw / gap_div;
    const double infeas_norm = infeas_raw / infeas_div;

    if (cfg->record_history && res->history) { /* :210-222 */
      double obj = 0, xx = 0;
      for (int64_t i = 0; i < N; ++i) { const double d = c.ey[i] - ys[i]; obj += d * d; }
      for (int64_t i = 0; i < N * n; ++i) xx += c.exi[i] * c.exi[i];
      double *h = res->history + (ell - 1) * 8;
      h[0] = (double)ell;
      h[1] = 0.5 * obj;
      h[2] = 0.5 * obj + 0.5 * cfg->gamma * xx;
      h[3] = infeas_raw;
      h[4] = infeas_norm;
      h[5] = gap_raw;
      h[6] = gap_norm;
      h[7] = now_seconds() - start;
    }
    res->iters = ell;

    int stop = 0; /* :225-236 */
    if (fabs(gap_norm) <= cfg->gap_norm_tol && infeas_norm <= cfg->infeas_norm_tol) {
      res->reason = CRO_THRESHOLDS;
      stop = 1;
    } else if (ell >= cfg->max_iters) {
      res->reason = CRO_ITER_BUDGET;
      stop = 1;
    } else if (now_seconds() - start > cfg->max_seconds) {
      res->reason = CRO_TIME_BUDGET;
      stop = 1;
    }
    if (stop) { /* :238-254 */
      const double n1 = sqrt(threads > 1 ? dot_omp(theta1, theta1, dim, threads) : dot(theta1, theta1, dim));
      const int saturated = n1 > 0.99 * B_theta;
      if (saturated && cfg->adaptive_B_theta && res->reason == CRO_THRESHOLDS &&
          restarts < cfg->max_restarts) {
        B_theta *= 2.0;
        ++restarts;
        memcpy(theta2, theta1, sizeof(double) * (size_t)dim);
        memcpy(theta1_prev, theta1, sizeof(double) * (size_t)dim);
        t = 1.0;
        g_star_upper = INFINITY;
        continue;
      }
      res->saturated = saturated;
      break;
    }
    if (cfg->use_momentum) { /* :256-262 */
      const double t_next = cro_momentum_next(t);
      const double beta = (t - 1.0) / t_next;
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
      for (int64_t i = 0; i < dim; ++i) theta2[i] = theta1[i] + beta * (theta1[i] - theta1_prev[i]);
      t = t_next;
    } else {
      memcpy(theta2, theta1, sizeof(double) * (size_t)dim);
    }
  }

  if (rc == 0) {
    if (res->c_eta) memcpy(res->c_eta, C_eta, sizeof(double) * (size_t)dim);
    /* :265-277 final re-solve at theta1 */
    double ft = 1.0 / pow((double)ell, 3.0);
    if (cfg->inner_tol_floor < ft) ft = cfg->inner_tol_floor;
    if (cfg->final_resolve_tol < ft) ft = cfg->final_resolve_tol;
    const double g_final = dual_gradient(&c, theta1, C_eta);
    res->g_final = g_final;
    const double d = g_star_upper - (g_final - 2.0 * ft * (double)K);
    res->delta_estimate = d > 0 ? d : 0.0;
    if (res->y) memcpy(res->y, c.ey, sizeof(double) * (size_t)N);
    if (res->xi) memcpy(res->xi, c.exi, sizeof(double) * (size_t)(N * n));
    if (res->theta) memcpy(res->theta, theta1, sizeof(double) * (size_t)dim);
    res->B_theta = B_theta;
    res->restarts = restarts;
  }
  res->wall_seconds = now_seconds() - start;
  free(theta1); free(theta1_prev); free(theta2); free(C_eta);
  free(c.q_y); free(c.q_xi); free(c.ey); free(c.exi);
  return rc;
}

/* ============================================ memory-light replay (cfg 4/5) */
/* The same loop as cro_papg (papg.cpp:136-283) without any N^2 array: the
   per-iteration primal eta_k = (y_k, xi_k) (N(n+1) doubles) and the scalars
   of each step (ball scale, momentum beta, restart) are kept, and every pass
   recomputes each pair's multiplier history theta1/theta1_prev/theta2 from
   them with exactly the literal loop's element operations (papg.cpp:188-189,
   projections.hpp:10-12, papg.cpp:244-250, :256-262). Sums run in the literal
   loop's order per thread (one thread: bitwise equal to cro_papg with one
   thread; several: per-thread partials over contiguous l1 ranges combined in
   thread order, as apply_C_T_omp). Two passes per iteration: (A) the new v
   and the sums that fix the ball scale and the metrics; (B) theta1 with its
   scale, the gap, |theta1| and the adjoints C^T theta1 and C^T theta2_next
   (operators.cpp:155-180) for the next dual gradient. O(k^2 N^2 n) work for k
   iterations and O(k N n) memory. */
enum { RP_MOM = 0, RP_COPY = 1, RP_RESTART = 2 };

typedef struct {
  const double *X;
  int64_t N, n;
  double L;
  double **ey, **exi;  /* [1..k] */
  double *scale;       /* [1..k] ball scale (1.0: not scaled) */
  int *kind;           /* [1..k] transition to theta2 of the next iteration */
  double *beta;        /* [1..k] */
} rp_hist;

static inline double rp_resid(const double *X, int64_t n, const double *ey, const double *exi,
                              int64_t l1, int64_t l2) { /* operators.cpp:143-147 */
  double acc = ey[l1] - ey[l2];
  const double *xi2 = exi + l2 * n, *x1 = X + l1 * n, *x2 = X + l2 * n;
  for (int64_t j = 0; j < n; ++j) acc -= xi2[j] * (x1[j] - x2[j]);
  return acc;
}

/* iterations 1..m of one cross pair: theta1, theta1_prev after step m and the
   theta2 that iteration m+1 starts from */
static inline void rp_replay(const rp_hist *h, int64_t m, int64_t l1, int64_t l2, double *th1,
                             double *th1p, double *th2) {
  double a = 0.0, p = 0.0, b = 0.0;
  for (int64_t it = 1; it <= m; ++it) {
    const double row = rp_resid(h->X, h->n, h->ey[it], h->exi[it], l1, l2);
    double u = b - row / h->L;
    u = u > 0.0 ? u : 0.0;
    p = a;
    a = h->scale[it] != 1.0 ? u * h->scale[it] : u;
    if (h->kind[it] == RP_MOM) b = a + h->beta[it] * (a - p);
    else if (h->kind[it] == RP_RESTART) { b = a; p = a; }
    else b = a;
  }
  *th1 = a; *th1p = p; *th2 = b;
}

static int rp_grow(rp_hist *h, int64_t k, int64_t *cap) {
  if (k < *cap) return 0;
  int64_t nc = *cap * 2 + 8;
  double **ey = (double **)realloc(h->ey, sizeof(double *) * (size_t)nc);
  if (ey) h->ey = ey;
  double **exi = (double **)realloc(h->exi, sizeof(double *) * (size_t)nc);
  if (exi) h->exi = exi;
  double *sc = (double *)realloc(h->scale, sizeof(double) * (size_t)nc);
  if (sc) h->scale = sc;
  int *kd = (int *)realloc(h->kind, sizeof(int) * (size_t)nc);
  if (kd) h->kind = kd;
  double *be = (double *)realloc(h->beta, sizeof(double) * (size_t)nc);
  if (be) h->beta = be;
  if (!ey || !exi || !sc || !kd || !be) return -1;
  for (int64_t i = *cap; i < nc; ++i) { h->ey[i] = NULL; h->exi[i] = NULL; }
  *cap = nc;
  return 0;
}

int cro_papg_replay(const double *X, const double *ys, int64_t N, int64_t n,
                    const cro_config *cfg, const int64_t *rows, int64_t nrows,
                    double *theta_rows, double *c_eta_rows, cro_result *res) {
  const double start = now_seconds();
  if (N < 2 || n < 1 || cfg->gamma <= 0 || nrows < 0 || (nrows > 0 && !rows)) return -1;
  for (int64_t i = 0; i < nrows; ++i)
    if (rows[i] < 0 || rows[i] >= N || (i > 0 && rows[i] <= rows[i - 1])) return -1;
  const int T = cfg->threads > 1 ? cfg->threads : 1;
  const int64_t rows_total = N * (N - 1);
  const double infeas_div = sqrt((double)rows_total);
  const double gap_div = (double)rows_total;
  double sigma_C = cfg->sigma_C;
  res->sigma_iters = 0;
  res->sigma_converged = 1;
  if (!(sigma_C > 0)) {
    int it = 0, conv = 0;
    if (cro_sigma_C(X, N, n, 1e-6, 5000, &sigma_C, &it, &conv)) return -2;
    res->sigma_iters = it;
    res->sigma_converged = conv;
  }
  const double L_g = sigma_C * sigma_C / cfg->gamma;
  double B_theta = cfg->B_theta > 0 ? cfg->B_theta : 10.0 * sqrt((double)N);
  res->sigma_C = sigma_C;
  res->L_g = L_g;
  res->reason = CRO_ITER_BUDGET;

  const int64_t w = N * (n + 1);
  rp_hist h = {X, N, n, L_g, NULL, NULL, NULL, NULL, NULL};
  int64_t cap = 0;
  double *th1_pos = (double *)calloc((size_t)N, sizeof(double));
  double *th1p_pos = (double *)calloc((size_t)N, sizeof(double));
  double *th2_pos = (double *)calloc((size_t)N, sizeof(double));
  double *n1_pos = (double *)malloc(sizeof(double) * (size_t)N);  /* theta1_pos of step k */
  double *cand_pos = (double *)malloc(sizeof(double) * (size_t)N);
  double *part = (double *)malloc(sizeof(double) * (size_t)(2 * w * T)); /* [T][th1 | cand] */
  double *scal = (double *)malloc(sizeof(double) * (size_t)(8 * T));
  double *q_th1 = (double *)malloc(sizeof(double) * (size_t)w);
  int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * (size_t)N); /* output row of l1 or -1 */
  if (slot) {
    for (int64_t l = 0; l < N; ++l) slot[l] = -1;
    for (int64_t i = 0; i < nrows; ++i) slot[rows[i]] = i;
  }
  dg_ctx c = {X, ys, N, n, cfg->gamma, T,
              (double *)calloc((size_t)N, sizeof(double)),
              (double *)calloc((size_t)(N * n), sizeof(double)),
              (double *)malloc(sizeof(double) * (size_t)N),
              (double *)malloc(sizeof(double) * (size_t)(N * n))};
  int rc = 0;
  if (!th1_pos || !th1p_pos || !th2_pos || !n1_pos || !cand_pos || !part || !scal || !q_th1 || !slot ||
      !c.q_y || !c.q_xi || !c.ey || !c.exi) { rc = -3; goto done; }
  {
    double t = 1.0;
    double g_star_upper = INFINITY;
    int64_t ell = 0;
    int restarts = 0;
    while (1) {
      ++ell;
      if (rp_grow(&h, ell, &cap)) { rc = -3; break; }
      const double inv3 = 1.0 / ((double)ell * (double)ell * (double)ell);
      const double inner_tol = cfg->inner_tol_floor < inv3 ? cfg->inner_tol_floor : inv3;
      const double g_value = block_minimisers(&c); /* eta of theta2 (q from the last pass B) */
      h.ey[ell] = (double *)malloc(sizeof(double) * (size_t)N);
      h.exi[ell] = (double *)malloc(sizeof(double) * (size_t)(N * n));
      if (!h.ey[ell] || !h.exi[ell]) { rc = -3; break; }
      memcpy(h.ey[ell], c.ey, sizeof(double) * (size_t)N);
      memcpy(h.exi[ell], c.exi, sizeof(double) * (size_t)(N * n));
      h.scale[ell] = 1.0;
      h.kind[ell] = RP_COPY;
      h.beta[ell] = 0.0;

      /* pass A: v_k = max(theta2 - C eta / L, 0) and the sums of :188-199 */
      int finite = 1;
#pragma omp parallel num_threads(T)
      {
        int tid = 0, nt = 1;
#ifdef _OPENMP
        tid = omp_get_thread_num();
        nt = omp_get_num_threads();
#endif
        double ss = 0, csq = 0, t2c = 0;
        int fin = 1;
        const int64_t lo = N * tid / nt, hi = N * (tid + 1) / nt;
        for (int64_t l1 = lo; l1 < hi; ++l1) {
          for (int64_t l2 = 0; l2 < N; ++l2) {
            if (l1 == l2) continue;
            double a, p, b;
            rp_replay(&h, ell - 1, l1, l2, &a, &p, &b);
            const double row = rp_resid(X, n, h.ey[ell], h.exi[ell], l1, l2);
            if (!isfinite(row)) fin = 0;
            double u = b - row / L_g;
            u = u > 0.0 ? u : 0.0;
            ss += u * u;
            const double m = -row > 0.0 ? -row : 0.0;
            csq += m * m;
            t2c += b * row;
          }
        }
        scal[tid * 8 + 0] = ss;
        scal[tid * 8 + 1] = csq;
        scal[tid * 8 + 2] = t2c;
        scal[tid * 8 + 3] = fin;
      }
      double ss = 0, cross_sq = 0, t2c = 0;
      for (int tt = 0; tt < T; ++tt) {
        ss += scal[tt * 8 + 0];
        cross_sq += scal[tt * 8 + 1];
        t2c += scal[tt * 8 + 2];
        if (scal[tt * 8 + 3] == 0) finite = 0;
      }
      double all_sq = cross_sq;
      for (int64_t l = 0; l < N; ++l) { /* the y >= 0 rows, C eta = y (operators.cpp:152) */
        const double row = c.ey[l];
        if (!isfinite(row)) finite = 0;
        double u = th2_pos[l] - row / L_g;
        u = u > 0.0 ? u : 0.0;
        ss += u * u;
        const double m = -row > 0.0 ? -row : 0.0;
        all_sq += m * m;
        t2c += th2_pos[l] * row;
      }
      if (!finite) { res->reason = CRO_ERROR; rc = -4; break; }
      const double norm = sqrt(ss);
      if (norm > B_theta) h.scale[ell] = B_theta / norm; /* projections.hpp:11-12 */
      const double cross_infeas = sqrt(cross_sq);
      const double fw = B_theta * sqrt(all_sq) + t2c;
      const double cushion = 2.0 * inner_tol * (double)N;
      const double cand = g_value + fw + cushion;
      if (cand < g_star_upper) g_star_upper = cand;
      const double t_next = cro_momentum_next(t);
      const double beta = cfg->use_momentum ? (t - 1.0) / t_next : 0.0;

      /* pass B: theta1 = s v, gap, |theta1|, C^T theta1, C^T theta2_next */
      for (int64_t l = 0; l < N; ++l) {
        double u = th2_pos[l] - c.ey[l] / L_g;
        u = u > 0.0 ? u : 0.0;
        n1_pos[l] = h.scale[ell] != 1.0 ? u * h.scale[ell] : u;
        cand_pos[l] = n1_pos[l] + beta * (n1_pos[l] - th1_pos[l]);
      }
#pragma omp parallel num_threads(T)
      {
        int tid = 0, nt = 1;
#ifdef _OPENMP
        tid = omp_get_thread_num();
        nt = omp_get_num_threads();
#endif
        double *p1 = part + (int64_t)tid * 2 * w, *p2 = p1 + w;
        if (nt == 1) { /* literal single-thread apply_C_T: starts from theta_pos */
          memcpy(p1, n1_pos, sizeof(double) * (size_t)N);
          memcpy(p2, cand_pos, sizeof(double) * (size_t)N);
          memset(p1 + N, 0, sizeof(double) * (size_t)(N * n));
          memset(p2 + N, 0, sizeof(double) * (size_t)(N * n));
        } else {
          memset(p1, 0, sizeof(double) * (size_t)(2 * w));
        }
        double gap = 0, nn1 = 0;
        const int64_t lo = N * tid / nt, hi = N * (tid + 1) / nt;
        for (int64_t l1 = lo; l1 < hi; ++l1) {
          const double *x1 = X + l1 * n;
          const int out_row = slot[l1] >= 0;
          int64_t r = slot[l1] * (N - 1);
          for (int64_t l2 = 0; l2 < N; ++l2) {
            if (l1 == l2) continue;
            double a, p, b;
            rp_replay(&h, ell - 1, l1, l2, &a, &p, &b);
            const double row = rp_resid(X, n, h.ey[ell], h.exi[ell], l1, l2);
            double u = b - row / L_g;
            u = u > 0.0 ? u : 0.0;
            p = a;
            a = h.scale[ell] != 1.0 ? u * h.scale[ell] : u;
            gap += a * row;
            nn1 += a * a;
            if (out_row) {
              if (theta_rows) theta_rows[r] = a;
              if (c_eta_rows) c_eta_rows[r] = row;
              ++r;
            }
            const double bn = a + beta * (a - p);
            const double *x2 = X + l2 * n;
            p1[l1] += a;
            p1[l2] -= a;
            p2[l1] += bn;
            p2[l2] -= bn;
            double *o1 = p1 + N + l2 * n, *o2 = p2 + N + l2 * n;
            for (int64_t j = 0; j < n; ++j) {
              const double dx = x1[j] - x2[j];
              o1[j] -= a * dx;
              o2[j] -= bn * dx;
            }
          }
        }
        scal[tid * 8 + 4] = gap;
        scal[tid * 8 + 5] = nn1;
      }
      double gap_m = 0, nsq = 0;
      for (int tt = 0; tt < T; ++tt) { gap_m += scal[tt * 8 + 4]; nsq += scal[tt * 8 + 5]; }
      for (int64_t l = 0; l < N; ++l) {
        gap_m += n1_pos[l] * c.ey[l];
        nsq += n1_pos[l] * n1_pos[l];
      }
      /* combine the adjoints (apply_C_T_omp order) */
      if (T == 1) {
        memcpy(q_th1, part, sizeof(double) * (size_t)w);
        memcpy(c.q_y, part + w, sizeof(double) * (size_t)N);
        memcpy(c.q_xi, part + w + N, sizeof(double) * (size_t)(N * n));
      } else {
#pragma omp parallel for schedule(static) num_threads(T)
        for (int64_t k = 0; k < w; ++k) {
          double s1 = k < N ? n1_pos[k] : 0.0, s2 = k < N ? cand_pos[k] : 0.0;
          for (int tt = 0; tt < T; ++tt) {
            s1 += part[(int64_t)tt * 2 * w + k];
            s2 += part[(int64_t)tt * 2 * w + w + k];
          }
          q_th1[k] = s1;
          if (k < N) c.q_y[k] = s2; else c.q_xi[k - N] = s2;
        }
      }
      for (int64_t l = 0; l < N; ++l) { th1p_pos[l] = th1_pos[l]; th1_pos[l] = n1_pos[l]; }

      const double gap_raw = cfg->use_momentum ? gap_m : t2c; /* :201-208 */
      const double infeas_raw = sqrt(cross_infeas * cross_infeas);
      const double gap_norm = gap_raw / gap_div;
      const double infeas_norm = infeas_raw / infeas_div;
      if (cfg->record_history && res->history) {
        double obj = 0, xx = 0;
        for (int64_t i = 0; i < N; ++i) { const double d = c.ey[i] - ys[i]; obj += d * d; }
        for (int64_t i = 0; i < N * n; ++i) xx += c.exi[i] * c.exi[i];
        double *hh = res->history + (ell - 1) * 8;
        hh[0] = (double)ell;
        hh[1] = 0.5 * obj;
        hh[2] = 0.5 * obj + 0.5 * cfg->gamma * xx;
        hh[3] = infeas_raw;
        hh[4] = infeas_norm;
        hh[5] = gap_raw;
        hh[6] = gap_norm;
        hh[7] = now_seconds() - start;
      }
      res->iters = ell;
      int stop = 0; /* :225-236 */
      if (fabs(gap_norm) <= cfg->gap_norm_tol && infeas_norm <= cfg->infeas_norm_tol) {
        res->reason = CRO_THRESHOLDS;
        stop = 1;
      } else if (ell >= cfg->max_iters) {
        res->reason = CRO_ITER_BUDGET;
        stop = 1;
      } else if (now_seconds() - start > cfg->max_seconds) {
        res->reason = CRO_TIME_BUDGET;
        stop = 1;
      }
      if (stop) { /* :238-254 */
        const int saturated = sqrt(nsq) > 0.99 * B_theta;
        if (saturated && cfg->adaptive_B_theta && res->reason == CRO_THRESHOLDS &&
            restarts < cfg->max_restarts) {
          B_theta *= 2.0;
          ++restarts;
          h.kind[ell] = RP_RESTART;
          for (int64_t l = 0; l < N; ++l) { th2_pos[l] = th1_pos[l]; th1p_pos[l] = th1_pos[l]; }
          memcpy(c.q_y, q_th1, sizeof(double) * (size_t)N);
          memcpy(c.q_xi, q_th1 + N, sizeof(double) * (size_t)(N * n));
          t = 1.0;
          g_star_upper = INFINITY;
          continue;
        }
        res->saturated = saturated;
        /* :265-277 final re-solve at theta1 */
        memcpy(c.q_y, q_th1, sizeof(double) * (size_t)N);
        memcpy(c.q_xi, q_th1 + N, sizeof(double) * (size_t)(N * n));
        double ft = 1.0 / pow((double)ell, 3.0);
        if (cfg->inner_tol_floor < ft) ft = cfg->inner_tol_floor;
        if (cfg->final_resolve_tol < ft) ft = cfg->final_resolve_tol;
        const double g_final = block_minimisers(&c);
        res->g_final = g_final;
        const double d = g_star_upper - (g_final - 2.0 * ft * (double)N);
        res->delta_estimate = d > 0 ? d : 0.0;
        if (res->y) memcpy(res->y, c.ey, sizeof(double) * (size_t)N);
        if (res->xi) memcpy(res->xi, c.exi, sizeof(double) * (size_t)(N * n));
        if (theta_rows) memcpy(theta_rows + nrows * (N - 1), th1_pos, sizeof(double) * (size_t)N);
        if (c_eta_rows) memcpy(c_eta_rows + nrows * (N - 1), h.ey[ell], sizeof(double) * (size_t)N);
        res->B_theta = B_theta;
        res->restarts = restarts;
        break;
      }
      if (cfg->use_momentum) { /* :256-262; q already holds C^T theta2_next */
        h.kind[ell] = RP_MOM;
        h.beta[ell] = beta;
        for (int64_t l = 0; l < N; ++l) th2_pos[l] = cand_pos[l];
        t = t_next;
      } else {
        h.kind[ell] = RP_COPY;
        for (int64_t l = 0; l < N; ++l) th2_pos[l] = th1_pos[l];
      }
    }
  }
done:
  res->wall_seconds = now_seconds() - start;
  for (int64_t i = 0; i < cap; ++i) { free(h.ey ? h.ey[i] : NULL); free(h.exi ? h.exi[i] : NULL); }
  free(h.ey); free(h.exi); free(h.scale); free(h.kind); free(h.beta);
  free(th1_pos); free(th1p_pos); free(th2_pos); free(n1_pos); free(cand_pos); free(part);
  free(scal); free(q_th1); free(slot);
  free(c.q_y); free(c.q_xi); free(c.ey); free(c.exi);
  return rc;
}

/* ================================================= standalone ALCC (f1) */
/* Row set of alcc_solve (alcc.cpp:193-208): all N(N-1) cross rows
   R(y, xi) = A1 y + A2 xi in canonical (l1, l2) order (FullRows,
   alcc.hpp:32-48 -> operators.cpp apply_rows / rows_adjoint). The forward and
   adjoint reuse the op_C restatement: C's pos rows are dropped on the way out
   and fed zeros on the way in. */
typedef struct {
  const double *X;
  int64_t N, n;
  int threads;
  double *rowbuf; /* N(N-1) + N */
  double *zbuf;   /* N(N-1) + N, pos part held at 0 */
} rows_ctx;

static void rows_forward(rows_ctx *r, const double *y, const double *xi, double *out) {
  if (r->threads > 1) apply_C_omp(r->X, r->N, r->n, y, xi, r->rowbuf, r->threads);
  else cro_apply_C(r->X, r->N, r->n, y, xi, r->rowbuf);
  memcpy(out, r->rowbuf, sizeof(double) * (size_t)(r->N * (r->N - 1)));
}
static void rows_adjoint(rows_ctx *r, const double *z, double *out_y, double *out_xi) {
  const int64_t m = r->N * (r->N - 1);
  memcpy(r->zbuf, z, sizeof(double) * (size_t)m);
  memset(r->zbuf + m, 0, sizeof(double) * (size_t)r->N);
  if (r->threads > 1) apply_C_T_omp(r->X, r->N, r->n, r->zbuf, out_y, out_xi, r->threads);
  else cro_apply_C_T(r->X, r->N, r->n, r->zbuf, out_y, out_xi);
}

/* operators.cpp:302-339 on op_A1 (:341-345, cols N) or op_A2 (:347-351, cols N n) */
int cro_sigma_A(const double *X, int64_t N, int64_t n, int which, double tol, int max_iters,
                double *sigma, int *iters, int *converged) {
  if (N < 2 || n < 1 || (which != 1 && which != 2)) return -1;
  const int64_t m = N * (N - 1);
  const int64_t cols = which == 1 ? N : N * n;
  double *v = (double *)malloc(sizeof(double) * (size_t)cols);
  double *u = (double *)malloc(sizeof(double) * (size_t)(N * (n + 1)));
  double *w = (double *)malloc(sizeof(double) * (size_t)m);
  double *zy = (double *)calloc((size_t)N, sizeof(double));
  double *zxi = (double *)calloc((size_t)(N * n), sizeof(double));
  rows_ctx rc = {X, N, n, 1, (double *)malloc(sizeof(double) * (size_t)(m + N)),
                 (double *)malloc(sizeof(double) * (size_t)(m + N))};
  int ret = 0;
  if (!v || !u || !w || !zy || !zxi || !rc.rowbuf || !rc.zbuf) { ret = -2; goto done; }
  {
    xo256 g = rng_stream(0x5eedULL, 97);
    for (int64_t k = 0; k < cols; ++k) v[k] = xo_normal(&g);
    const double nv = sqrt(dot(v, v, cols));
    for (int64_t k = 0; k < cols; ++k) v[k] /= nv;
    double lambda_prev = 0;
    *iters = 0;
    *converged = 1;
    for (int it = 1; it <= max_iters; ++it) {
      /* op.forward: A1 v = R(v, 0) or A2 v = R(0, v) */
      if (which == 1) rows_forward(&rc, v, zxi, w);
      else rows_forward(&rc, zy, v, w);
      const double lambda = dot(w, w, m);
      rows_adjoint(&rc, w, u, u + N); /* A1^T w = u[0..N), A2^T w = u[N..) */
      const double *uu = which == 1 ? u : u + N;
      const double norm_u = sqrt(dot(uu, uu, cols));
      if (norm_u == 0 || lambda == 0) {
        *sigma = 0;
        *iters = it;
        goto done;
      }
      for (int64_t k = 0; k < cols; ++k) v[k] = uu[k] / norm_u;
      *iters = it;
      if (it > 1 && fabs(lambda - lambda_prev) <= tol * lambda) {
        *sigma = sqrt(lambda) * 1.01;
        *converged = 1;
        goto done;
      }
      lambda_prev = lambda;
    }
    *sigma = sqrt(lambda_prev) * 1.10;
    *converged = 0;
  }
done:
  free(v); free(u); free(w); free(zy); free(zxi); free(rc.rowbuf); free(rc.zbuf);
  return ret;
}

/* projections.hpp:22-26 */
static void project_ball_c(double *v, const double *center, int64_t len, double radius) {
  double ss = 0;
  for (int64_t i = 0; i < len; ++i) {
    const double d = v[i] - (center ? center[i] : 0.0);
    ss += d * d;
  }
  const double dist = sqrt(ss);
  if (dist > radius) {
    const double f = radius / dist;
    for (int64_t i = 0; i < len; ++i) {
      const double c = center ? center[i] : 0.0;
      v[i] = c + f * (v[i] - c);
    }
  }
}

/* PenaltyOracle::eval (alcc.cpp:33-47) over a row set with centres (cy, cxi) */
typedef struct {
  rows_ctx *rows;
  const double *cy, *cxi; /* cxi NULL: 0 */
  const double *theta;    /* m */
  double mu, gamma;
  int64_t N, n;           /* points of the row set */
  double *res, *vneg, *ay, *axi; /* scratch */
} pen_ctx;

static void penalty_grad(pen_ctx *p, const double *y, const double *xi, double *gy,
                         double *gxi) {
  const int64_t m = p->N * (p->N - 1);
  rows_forward(p->rows, y, xi, p->res);
  for (int64_t i = 0; i < m; ++i) {
    const double r = p->res[i] - p->theta[i];
    p->vneg[i] = -r > 0.0 ? -r : 0.0;
  }
  rows_adjoint(p->rows, p->vneg, p->ay, p->axi);
  for (int64_t i = 0; i < p->N; ++i) gy[i] = (y[i] - p->cy[i]) / p->mu - p->ay[i];
  const double gm = p->gamma / p->mu;
  for (int64_t i = 0; i < p->N * p->n; ++i)
    gxi[i] = gm * (xi[i] - (p->cxi ? p->cxi[i] : 0.0)) - p->axi[i];
}

/* alcc_core (alcc.cpp:54-191) on the within rows of the nb points Xb (the
   standalone FullRows set is the single block of all N points). target > 0:
   block stop rule (alcc.cpp:153-155), else the standalone thresholds. */
static int alcc_core_c(const double *Xb, int64_t N, int64_t n, const double *cy,
                       const double *cxi, double gamma, double Bbar_y, double Bbar_xi,
                       double sigma_A1, double sigma_A2, const cro_alcc_config *cfg,
                       double target, const double *warm_y, const double *warm_xi,
                       cro_alcc_result *res) {
  const double start = now_seconds();
  if (!(cfg->c > 1) || !(cfg->kappa > 0) || !(cfg->mu1 > 0)) return -1; /* alcc.cpp:59-61 */
  const int threads = cfg->threads > 1 ? cfg->threads : 1;
  const int64_t m = N * (N - 1);
  const int64_t Nn = N * n;
  rows_ctx rc = {Xb, N, n, threads, (double *)malloc(sizeof(double) * (size_t)(m + N)),
                 (double *)malloc(sizeof(double) * (size_t)(m + N))};
  double *theta = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
  double *res_v = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double *vneg = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double *work = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double *rows_center = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  /* point buffers: y, y1, y1_prev, y2, gy, ay | xi, xi1, xi1_prev, xi2, gxi, axi */
  double *pb = (double *)malloc(sizeof(double) * (size_t)(6 * N + 6 * Nn));
  if (!rc.rowbuf || !rc.zbuf || !theta || !res_v || !vneg || !work || !rows_center || !pb)
    return -3;
  double *y = pb, *y1 = pb + N, *y1p = pb + 2 * N, *y2 = pb + 3 * N, *gy = pb + 4 * N,
         *ay = pb + 5 * N;
  double *xi = pb + 6 * N, *xi1 = xi + Nn, *xi1p = xi + 2 * Nn, *xi2 = xi + 3 * Nn,
         *gxi = xi + 4 * Nn, *axi = xi + 5 * Nn;

  double mu = cfg->mu1;
  memcpy(y, warm_y, sizeof(double) * (size_t)N); /* alcc.cpp:68-69 */
  memcpy(xi, warm_xi, sizeof(double) * (size_t)Nn);
  project_ball_c(y, cy, N, Bbar_y);
  project_ball_c(xi, cxi, Nn, Bbar_xi);

  pen_ctx pen = {&rc, cy, cxi, theta, mu, gamma, N, n, work, vneg, ay, axi};
  double tau, alpha_y, alpha_xi;
  int rcode = 0;
  { /* alcc.cpp:75-84: P_1 at the start point */
    penalty_grad(&pen, y, xi, gy, gxi);
    double sy = 0, sx = 0, sv = 0;
    for (int64_t i = 0; i < N; ++i) sy += (y[i] - cy[i]) * (y[i] - cy[i]);
    for (int64_t i = 0; i < Nn; ++i) {
      const double d = xi[i] - (cxi ? cxi[i] : 0.0);
      sx += d * d;
    }
    for (int64_t i = 0; i < m; ++i) sv += vneg[i] * vneg[i];
    const double p1 = sy / (2.0 * mu) + gamma * sx / (2.0 * mu) + 0.5 * sv;
    if (!isfinite(p1)) { rcode = -4; goto out; }
    tau = cfg->tau1_scale * p1;
    if (tau < 1e-16) tau = 1e-16;
    alpha_y = alpha_xi = cfg->alpha1_scale * (Bbar_y + Bbar_xi);
  }
  if (cxi) {
    rows_forward(&rc, cy, cxi, rows_center);
  } else {
    memset(gxi, 0, sizeof(double) * (size_t)Nn);
    rows_forward(&rc, cy, gxi, rows_center);
  }

  res->reason = CRO_ITER_BUDGET;
  res->mapg_iters_total = 0;
  res->outer_iters = 0;
  res->hit_cap_any = 0;
  for (int64_t k = 1; k <= cfg->max_outer; ++k) {
    const double L_y = 1.0 / mu + sigma_A1 * sigma_A1; /* :101-102 */
    const double L_xi = gamma / mu + sigma_A2 * sigma_A2;
    const double lmax_real = 4.0 * sqrt((L_y * Bbar_y * Bbar_y + L_xi * Bbar_xi * Bbar_xi) / tau);
    int64_t lmax = (int64_t)ceil(lmax_real);
    if (lmax < 10) lmax = 10;
    if (lmax > cfg->mapg_cap) lmax = cfg->mapg_cap;
    pen.mu = mu;

    /* mapg (engines.cpp:57-106) from (y, xi) */
    memcpy(y1, y, sizeof(double) * (size_t)N);
    memcpy(y1p, y, sizeof(double) * (size_t)N);
    memcpy(y2, y, sizeof(double) * (size_t)N);
    memcpy(xi1, xi, sizeof(double) * (size_t)Nn);
    memcpy(xi1p, xi, sizeof(double) * (size_t)Nn);
    memcpy(xi2, xi, sizeof(double) * (size_t)Nn);
    double t = 1.0;
    int64_t inner = 0;
    for (int64_t ell = 1; ell <= lmax; ++ell) {
      penalty_grad(&pen, y2, xi2, gy, gxi);
      for (int64_t i = 0; i < N; ++i) if (!isfinite(gy[i])) { rcode = -5; goto out; }
      for (int64_t i = 0; i < Nn; ++i) if (!isfinite(gxi[i])) { rcode = -5; goto out; }
      { double *tmp = y1p; y1p = y1; y1 = tmp; }
      for (int64_t i = 0; i < N; ++i) y1[i] = y2[i] - gy[i] / L_y;
      project_ball_c(y1, cy, N, Bbar_y);
      { double *tmp = xi1p; xi1p = xi1; xi1 = tmp; }
      for (int64_t i = 0; i < Nn; ++i) xi1[i] = xi2[i] - gxi[i] / L_xi;
      project_ball_c(xi1, cxi, Nn, Bbar_xi);
      inner = ell;
      double dy = 0, dx = 0;
      for (int64_t i = 0; i < N; ++i) dy += (y1[i] - y2[i]) * (y1[i] - y2[i]);
      for (int64_t i = 0; i < Nn; ++i) dx += (xi1[i] - xi2[i]) * (xi1[i] - xi2[i]);
      const double disp_y = sqrt(dy), disp_xi = sqrt(dx);
      const double t_next = cro_momentum_next(t);
      const double beta = (t - 1.0) / t_next;
      for (int64_t i = 0; i < N; ++i) y2[i] = y1[i] + beta * (y1[i] - y1p[i]);
      for (int64_t i = 0; i < Nn; ++i) xi2[i] = xi1[i] + beta * (xi1[i] - xi1p[i]);
      t = t_next;
      if (disp_y <= alpha_y && disp_xi <= alpha_xi) break;
      if (ell == lmax) res->hit_cap_any = 1;
    }
    memcpy(y, y1, sizeof(double) * (size_t)N);
    memcpy(xi, xi1, sizeof(double) * (size_t)Nn);
    res->mapg_iters_total += inner;
    if (res->mapg_iters) res->mapg_iters[k - 1] = inner;

    /* :124-160 */
    rows_forward(&rc, y, xi, res_v);
    double nn = 0, gap_raw = 0, lc = 0, ll = 0;
    for (int64_t i = 0; i < m; ++i) {
      const double d = theta[i] - res_v[i];
      vneg[i] = d > 0.0 ? d : 0.0;
      const double lam = mu * vneg[i];
      work[i] = lam;
      const double neg = -res_v[i] > 0.0 ? -res_v[i] : 0.0;
      nn += neg * neg;
      gap_raw += lam * res_v[i];
      lc += lam * rows_center[i];
      ll += lam * lam;
    }
    const double infeas_raw = sqrt(nn);
    rows_adjoint(&rc, work, ay, axi);
    const double dual_value = -0.5 * dot(ay, ay, N) - dot(axi, axi, Nn) / (2.0 * gamma) - lc;
    double sy = 0, sx = 0;
    for (int64_t i = 0; i < N; ++i) sy += (y[i] - cy[i]) * (y[i] - cy[i]);
    for (int64_t i = 0; i < Nn; ++i) {
      const double d = xi[i] - (cxi ? cxi[i] : 0.0);
      sx += d * d;
    }
    const double primal_value = 0.5 * sy + 0.5 * gamma * sx;
    const double certified = primal_value - dual_value;
    res->certified_gap = certified;
    res->infeas_raw = infeas_raw;
    res->gap_raw = gap_raw;
    res->outer_iters = k;
    const double infeas_norm = m > 0 ? infeas_raw / sqrt((double)m) : 0.0;
    const double gap_norm = m > 0 ? gap_raw / (double)m : 0.0;
    if (cfg->record_history && res->history) {
      double *h = res->history + (k - 1) * 8;
      h[0] = (double)k;
      h[1] = 0.5 * sy;
      h[2] = primal_value;
      h[3] = infeas_raw;
      h[4] = infeas_norm;
      h[5] = gap_raw;
      h[6] = gap_norm;
      h[7] = now_seconds() - start;
    }
    if (res->multiplier) memcpy(res->multiplier, work, sizeof(double) * (size_t)m);
    int stop;
    if (target > 0) stop = certified <= target && sqrt(ll) * infeas_raw <= target;
    else stop = infeas_norm <= cfg->infeas_norm_tol && fabs(gap_norm) <= cfg->gap_norm_tol;
    if (stop) {
      res->reason = CRO_THRESHOLDS;
      break;
    }
    if (now_seconds() - start > cfg->max_seconds) {
      res->reason = CRO_TIME_BUDGET;
      break;
    }
    for (int64_t i = 0; i < m; ++i) theta[i] = vneg[i] / cfg->c; /* :176-183 */
    mu *= cfg->c;
    const double decay = pow(cfg->c * pow((double)k, 1.0 + cfg->kappa), 2.0);
    tau /= decay;
    alpha_y /= decay;
    alpha_xi /= decay;
  }
out:
  if (rcode == 0) {
    if (res->y) memcpy(res->y, y, sizeof(double) * (size_t)N);
    if (res->xi) memcpy(res->xi, xi, sizeof(double) * (size_t)Nn);
    double sy = 0;
    for (int64_t i = 0; i < N; ++i) sy += (y[i] - cy[i]) * (y[i] - cy[i]);
    res->objective = 0.5 * sy;
  } else {
    res->reason = CRO_ERROR;
  }
  res->wall_seconds = now_seconds() - start;
  free(rc.rowbuf); free(rc.zbuf); free(theta); free(res_v); free(vneg); free(work); free(pb);
  free(rows_center);
  return rcode;
}

int cro_alcc(const double *X, const double *ys, int64_t N, int64_t n, double gamma,
             double Bbar_y, double Bbar_xi, double sigma_A1, double sigma_A2,
             const double *warm_y, const double *warm_xi, const cro_alcc_config *cfg,
             cro_alcc_result *res) {
  if (N < 2 || n < 1 || !(gamma > 0)) return -1;
  if (!(cfg->c > 1) || !(cfg->kappa > 0) || !(cfg->mu1 > 0)) return -1;
  if (!(sigma_A1 > 0)) {
    int it, cv;
    if (cro_sigma_A(X, N, n, 1, 1e-6, 5000, &sigma_A1, &it, &cv)) return -2;
  }
  if (!(sigma_A2 > 0)) {
    int it, cv;
    if (cro_sigma_A(X, N, n, 2, 1e-6, 5000, &sigma_A2, &it, &cv)) return -2;
  }
  res->sigma_A1 = sigma_A1;
  res->sigma_A2 = sigma_A2;
  /* alcc_solve (alcc.cpp:193-208): FullRows, centres (ybar, 0) */
  return alcc_core_c(X, N, n, ys, NULL, gamma, Bbar_y, Bbar_xi, sigma_A1, sigma_A2, cfg, 0.0,
                     warm_y, warm_xi, res);
}

/* ============================================ general-K P-APG(ALCC) (f2) */
/* operators.cpp:128-153 with K blocks of nbar points: cross rows ordered by
   block pair (i, j), i != j, then (l1, l2) lexicographic (indexing.hpp:9-37). */
void cro_apply_C_k(const double *X, int64_t N, int64_t n, int64_t K, const double *y,
                   const double *xi, double *out) {
  const int64_t nbar = N / K;
  int64_t r = 0;
  for (int64_t i = 0; i < K; ++i)
    for (int64_t j = 0; j < K; ++j) {
      if (i == j) continue;
      for (int64_t l1 = i * nbar; l1 < (i + 1) * nbar; ++l1) {
        const double y1 = y[l1];
        const double *x1 = X + l1 * n;
        for (int64_t l2 = j * nbar; l2 < (j + 1) * nbar; ++l2) {
          double acc = y1 - y[l2];
          const double *xi2 = xi + l2 * n;
          const double *x2 = X + l2 * n;
          for (int64_t jj = 0; jj < n; ++jj) acc -= xi2[jj] * (x1[jj] - x2[jj]);
          out[r++] = acc;
        }
      }
    }
  for (int64_t l = 0; l < N; ++l) out[r + l] = y[l];
}

/* operators.cpp:155-180 */
void cro_apply_C_T_k(const double *X, int64_t N, int64_t n, int64_t K, const double *theta,
                     double *out_y, double *out_xi) {
  const int64_t nbar = N / K;
  const int64_t rows_cross = N * (N - nbar);
  for (int64_t l = 0; l < N; ++l) out_y[l] = theta[rows_cross + l];
  memset(out_xi, 0, sizeof(double) * (size_t)(N * n));
  int64_t r = 0;
  for (int64_t i = 0; i < K; ++i)
    for (int64_t j = 0; j < K; ++j) {
      if (i == j) continue;
      for (int64_t l1 = i * nbar; l1 < (i + 1) * nbar; ++l1) {
        const double *x1 = X + l1 * n;
        for (int64_t l2 = j * nbar; l2 < (j + 1) * nbar; ++l2) {
          const double tr = theta[r++];
          out_y[l1] += tr;
          out_y[l2] -= tr;
          double *o2 = out_xi + l2 * n;
          const double *x2 = X + l2 * n;
          for (int64_t jj = 0; jj < n; ++jj) o2[jj] -= tr * (x1[jj] - x2[jj]);
        }
      }
    }
}

/* operators.cpp:302-339 on op_C (:353-369) with K blocks */
int cro_sigma_C_k(const double *X, int64_t N, int64_t n, int64_t K, double tol, int max_iters,
                  double *sigma, int *iters, int *converged) {
  if (K == N) return cro_sigma_C(X, N, n, tol, max_iters, sigma, iters, converged);
  const int64_t nbar = N / K;
  const int64_t cols = N * (n + 1);
  const int64_t rows = N * (N - nbar) + N;
  double *v = (double *)malloc(sizeof(double) * (size_t)cols);
  double *u = (double *)malloc(sizeof(double) * (size_t)cols);
  double *w = (double *)malloc(sizeof(double) * (size_t)rows);
  if (!v || !u || !w) { free(v); free(u); free(w); return -1; }
  xo256 g = rng_stream(0x5eedULL, 97);
  for (int64_t k = 0; k < cols; ++k) v[k] = xo_normal(&g);
  const double nv = sqrt(dot(v, v, cols));
  for (int64_t k = 0; k < cols; ++k) v[k] /= nv;
  double lambda_prev = 0;
  *converged = 1;
  *iters = 0;
  for (int it = 1; it <= max_iters; ++it) {
    cro_apply_C_k(X, N, n, K, v, v + N, w);
    const double lambda = dot(w, w, rows);
    cro_apply_C_T_k(X, N, n, K, w, u, u + N);
    const double norm_u = sqrt(dot(u, u, cols));
    if (norm_u == 0 || lambda == 0) {
      *sigma = 0;
      *iters = it;
      free(v); free(u); free(w);
      return 0;
    }
    for (int64_t k = 0; k < cols; ++k) v[k] = u[k] / norm_u;
    *iters = it;
    if (it > 1 && fabs(lambda - lambda_prev) <= tol * lambda) {
      *sigma = sqrt(lambda) * 1.01;
      free(v); free(u); free(w);
      return 0;
    }
    lambda_prev = lambda;
  }
  *sigma = sqrt(lambda_prev) * 1.10;
  *converged = 0;
  free(v); free(u); free(w);
  return 0;
}

typedef struct {
  const double *X, *ys, *feas_y, *feas_xi;
  int64_t N, n, K, nbar;
  double gamma;
  int threads;
  const cro_alcc_config *inner;
  double sigma_A1, *sigma_A2;   /* estimate_block_sigmas (alcc.cpp:208-220) */
  double *warm_y, *warm_xi;     /* per-block warm starts (papg.cpp:74-86) */
  double *q_y, *q_xi, *ey, *exi;
  double *blk_obj, *blk_inf2;
  int64_t *blk_iters;
  int err;
} dgk_ctx;

/* alcc_solve_block (alcc.cpp:222-258) */
static void solve_block(dgk_ctx *c, int64_t i, double tol) {
  const int64_t nb = c->nbar, n = c->n, base = i * nb;
  const double gamma = c->gamma;
  double *cy = (double *)malloc(sizeof(double) * (size_t)nb);
  double *cxi = (double *)malloc(sizeof(double) * (size_t)(nb * n));
  for (int64_t a = 0; a < nb; ++a) cy[a] = c->ys[base + a] + c->q_y[base + a];
  for (int64_t a = 0; a < nb * n; ++a) cxi[a] = c->q_xi[base * n + a] / gamma;
  double sy = 0, sx = 0;
  for (int64_t a = 0; a < nb; ++a) {
    const double d = c->feas_y[base + a] - cy[a];
    sy += d * d;
  }
  for (int64_t a = 0; a < nb * n; ++a) {
    const double d = c->feas_xi[base * n + a] - cxi[a];
    sx += d * d;
  }
  const double Bsq = sy + gamma * sx;
  double Bbar = sqrt(Bsq);
  if (Bbar < 1e-8) Bbar = 1e-8;
  cro_alcc_result r;
  memset(&r, 0, sizeof(r));
  r.y = c->ey + base;
  r.xi = c->exi + base * n;
  const int rc = alcc_core_c(c->X + base * n, nb, n, cy, cxi, gamma, Bbar, Bbar / sqrt(gamma),
                             c->sigma_A1, c->sigma_A2[i], c->inner, tol, c->warm_y + base,
                             c->warm_xi + base * n, &r);
  if (rc != 0) c->err = rc;
  /* block objective (alcc.cpp:254-256) */
  double o1 = 0, o2 = 0, o3 = 0, o4 = 0;
  for (int64_t a = 0; a < nb; ++a) {
    const double d = r.y[a] - c->ys[base + a];
    o1 += d * d;
    o3 += c->q_y[base + a] * r.y[a];
  }
  for (int64_t a = 0; a < nb * n; ++a) {
    o2 += r.xi[a] * r.xi[a];
    o4 += c->q_xi[base * n + a] * r.xi[a];
  }
  c->blk_obj[i] = 0.5 * o1 + 0.5 * gamma * o2 - o3 - o4;
  c->blk_inf2[i] = r.infeas_raw * r.infeas_raw;
  c->blk_iters[i] = r.mapg_iters_total;
  memcpy(c->warm_y + base, r.y, sizeof(double) * (size_t)nb);
  memcpy(c->warm_xi + base * n, r.xi, sizeof(double) * (size_t)(nb * n));
  free(cy);
  free(cxi);
}

/* DualDecomposition::dual_gradient (papg.cpp:89-132) */
static double dual_gradient_k(dgk_ctx *c, const double *theta, double tol, double *C_eta,
                              double *within, int64_t *inner_iters) {
  cro_apply_C_T_k(c->X, c->N, c->n, c->K, theta, c->q_y, c->q_xi);
  if (c->threads > 1) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(c->threads)
    for (int64_t i = 0; i < c->K; ++i) solve_block(c, i, tol);
  } else {
    for (int64_t i = 0; i < c->K; ++i) solve_block(c, i, tol);
  }
  double g = 0, inf2 = 0;
  int64_t it = 0;
  for (int64_t i = 0; i < c->K; ++i) { /* gather in block order */
    g += c->blk_obj[i];
    inf2 += c->blk_inf2[i];
    it += c->blk_iters[i];
  }
  *within = sqrt(inf2);
  if (inner_iters) *inner_iters = it;
  cro_apply_C_k(c->X, c->N, c->n, c->K, c->ey, c->exi, C_eta);
  return g;
}

int cro_papg_k(const double *X, const double *ys, int64_t N, int64_t n, int64_t K,
               const cro_config *cfg, const cro_alcc_config *inner, const double *feas_y,
               const double *feas_xi, const double *theta0, cro_result *res,
               int64_t *inner_iters_out) {
  const double start = now_seconds();
  if (N < 2 || n < 1 || cfg->gamma <= 0 || K < 1 || N % K != 0) return -1;
  const int64_t nbar = N / K;
  if (nbar < n + 1) return -1; /* dataset.cpp:127-128 */
  const int threads = cfg->threads > 1 ? cfg->threads : 1;
  const int64_t rows_total = N * (N - 1);
  const int64_t rows_cross = N * (N - nbar);
  const int64_t dim = rows_cross + N;
  const double infeas_div = sqrt((double)rows_total);
  const double gap_div = (double)rows_total;

  dgk_ctx c;
  memset(&c, 0, sizeof(c));
  c.X = X; c.ys = ys; c.feas_y = feas_y; c.feas_xi = feas_xi;
  c.N = N; c.n = n; c.K = K; c.nbar = nbar; c.gamma = cfg->gamma; c.threads = threads;
  c.inner = inner;
  c.sigma_A2 = (double *)malloc(sizeof(double) * (size_t)K);
  { /* estimate_block_sigmas (alcc.cpp:206-220) */
    int it, cv;
    if (cro_sigma_A(X, nbar, n, 1, 1e-6, 5000, &c.sigma_A1, &it, &cv)) return -2;
    for (int64_t i = 0; i < K; ++i)
      if (cro_sigma_A(X + i * nbar * n, nbar, n, 2, 1e-6, 5000, &c.sigma_A2[i], &it, &cv))
        return -2;
  }
  double sigma_C = cfg->sigma_C;
  res->sigma_iters = 0;
  res->sigma_converged = 1;
  if (!(sigma_C > 0)) {
    int it = 0, conv = 0;
    if (cro_sigma_C_k(X, N, n, K, 1e-6, 5000, &sigma_C, &it, &conv)) return -2;
    res->sigma_iters = it;
    res->sigma_converged = conv;
  }
  const double L_g = sigma_C * sigma_C / cfg->gamma;
  double B_theta = cfg->B_theta > 0 ? cfg->B_theta : 10.0 * sqrt((double)N);
  res->sigma_C = sigma_C;
  res->L_g = L_g;
  res->reason = CRO_ITER_BUDGET;

  c.warm_y = (double *)malloc(sizeof(double) * (size_t)N);
  c.warm_xi = (double *)malloc(sizeof(double) * (size_t)(N * n));
  memcpy(c.warm_y, feas_y, sizeof(double) * (size_t)N);
  memcpy(c.warm_xi, feas_xi, sizeof(double) * (size_t)(N * n));
  c.q_y = (double *)malloc(sizeof(double) * (size_t)N);
  c.q_xi = (double *)malloc(sizeof(double) * (size_t)(N * n));
  c.ey = (double *)malloc(sizeof(double) * (size_t)N);
  c.exi = (double *)malloc(sizeof(double) * (size_t)(N * n));
  c.blk_obj = (double *)malloc(sizeof(double) * (size_t)K);
  c.blk_inf2 = (double *)malloc(sizeof(double) * (size_t)K);
  c.blk_iters = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);

  double *theta1 = (double *)calloc((size_t)dim, sizeof(double));
  double *theta1_prev = (double *)malloc(sizeof(double) * (size_t)dim);
  double *theta2 = (double *)malloc(sizeof(double) * (size_t)dim);
  double *C_eta = (double *)malloc(sizeof(double) * (size_t)dim);
  if (theta0) {
    memcpy(theta1, theta0, sizeof(double) * (size_t)dim);
    cro_project_nonneg_ball(theta1, dim, B_theta);
  }
  memcpy(theta1_prev, theta1, sizeof(double) * (size_t)dim);
  memcpy(theta2, theta1, sizeof(double) * (size_t)dim);
  double t = 1.0, g_star_upper = INFINITY;
  int64_t ell = 0, inner_total = 0;
  int restarts = 0, rc = 0;
  while (1) {
    ++ell;
    const double inv3 = 1.0 / ((double)ell * (double)ell * (double)ell);
    const double inner_tol = cfg->inner_tol_floor < inv3 ? cfg->inner_tol_floor : inv3;
    double within = 0;
    int64_t it = 0;
    const double g_value = dual_gradient_k(&c, theta2, inner_tol, C_eta, &within, &it);
    inner_total += it;
    if (c.err) { rc = c.err; res->reason = CRO_ERROR; break; }
    int finite = 1;
    for (int64_t i = 0; i < dim; ++i) if (!isfinite(C_eta[i])) { finite = 0; break; }
    if (!finite) { res->reason = CRO_ERROR; rc = -4; break; }
    { double *tmp = theta1_prev; theta1_prev = theta1; theta1 = tmp; }
    for (int64_t i = 0; i < dim; ++i) theta1[i] = theta2[i] - C_eta[i] / L_g;
    cro_project_nonneg_ball(theta1, dim, B_theta);
    double cross_sq = 0, all_sq = 0;
    for (int64_t i = 0; i < dim; ++i) {
      const double m = -C_eta[i] > 0.0 ? -C_eta[i] : 0.0;
      if (i < rows_cross) cross_sq += m * m;
      all_sq += m * m;
    }
    const double cross_infeas = rows_cross > 0 ? sqrt(cross_sq) : 0.0;
    const double t2c = dot(theta2, C_eta, dim);
    const double fw = B_theta * sqrt(all_sq) + t2c;
    const double cushion = 2.0 * inner_tol * (double)K;
    const double cand = g_value + fw + cushion;
    if (cand < g_star_upper) g_star_upper = cand;
    const double gap_raw = cfg->use_momentum ? dot(theta1, C_eta, dim) : t2c;
    const double infeas_raw = sqrt(within * within + cross_infeas * cross_infeas);
    const double gap_norm = gap_raw / gap_div;
    const double infeas_norm = infeas_raw / infeas_div;
    if (cfg->record_history && res->history) {
      double obj = 0, xx = 0;
      for (int64_t i = 0; i < N; ++i) { const double d = c.ey[i] - ys[i]; obj += d * d; }
      for (int64_t i = 0; i < N * n; ++i) xx += c.exi[i] * c.exi[i];
      double *h = res->history + (ell - 1) * 8;
      h[0] = (double)ell;
      h[1] = 0.5 * obj;
      h[2] = 0.5 * obj + 0.5 * cfg->gamma * xx;
      h[3] = infeas_raw;
      h[4] = infeas_norm;
      h[5] = gap_raw;
      h[6] = gap_norm;
      h[7] = now_seconds() - start;
    }
    res->iters = ell;
    int stop = 0;
    if (fabs(gap_norm) <= cfg->gap_norm_tol && infeas_norm <= cfg->infeas_norm_tol) {
      res->reason = CRO_THRESHOLDS;
      stop = 1;
    } else if (ell >= cfg->max_iters) {
      res->reason = CRO_ITER_BUDGET;
      stop = 1;
    } else if (now_seconds() - start > cfg->max_seconds) {
      res->reason = CRO_TIME_BUDGET;
      stop = 1;
    }
    if (stop) {
      const double n1 = sqrt(dot(theta1, theta1, dim));
      const int saturated = n1 > 0.99 * B_theta;
      if (saturated && cfg->adaptive_B_theta && res->reason == CRO_THRESHOLDS &&
          restarts < cfg->max_restarts) {
        B_theta *= 2.0;
        ++restarts;
        memcpy(theta2, theta1, sizeof(double) * (size_t)dim);
        memcpy(theta1_prev, theta1, sizeof(double) * (size_t)dim);
        t = 1.0;
        g_star_upper = INFINITY;
        continue;
      }
      res->saturated = saturated;
      break;
    }
    if (cfg->use_momentum) {
      const double t_next = cro_momentum_next(t);
      const double beta = (t - 1.0) / t_next;
      for (int64_t i = 0; i < dim; ++i) theta2[i] = theta1[i] + beta * (theta1[i] - theta1_prev[i]);
      t = t_next;
    } else {
      memcpy(theta2, theta1, sizeof(double) * (size_t)dim);
    }
  }
  if (rc == 0) {
    if (res->c_eta) memcpy(res->c_eta, C_eta, sizeof(double) * (size_t)dim);
    double ft = 1.0 / pow((double)ell, 3.0);
    if (cfg->inner_tol_floor < ft) ft = cfg->inner_tol_floor;
    if (cfg->final_resolve_tol < ft) ft = cfg->final_resolve_tol;
    double within = 0;
    int64_t it = 0;
    const double g_final = dual_gradient_k(&c, theta1, ft, C_eta, &within, &it);
    inner_total += it;
    res->g_final = g_final;
    const double d = g_star_upper - (g_final - 2.0 * ft * (double)K);
    res->delta_estimate = d > 0 ? d : 0.0;
    if (res->y) memcpy(res->y, c.ey, sizeof(double) * (size_t)N);
    if (res->xi) memcpy(res->xi, c.exi, sizeof(double) * (size_t)(N * n));
    if (res->theta) memcpy(res->theta, theta1, sizeof(double) * (size_t)dim);
    res->B_theta = B_theta;
    res->restarts = restarts;
  }
  if (inner_iters_out) *inner_iters_out = inner_total;
  res->wall_seconds = now_seconds() - start;
  free(theta1); free(theta1_prev); free(theta2); free(C_eta);
  free(c.q_y); free(c.q_xi); free(c.ey); free(c.exi); free(c.warm_y); free(c.warm_xi);
  free(c.blk_obj); free(c.blk_inf2); free(c.blk_iters); free(c.sigma_A2);
  return rc;
}
