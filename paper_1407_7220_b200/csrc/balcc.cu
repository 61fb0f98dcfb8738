// balcc.cu -- all K block QPs of a P-APG(ALCC) dual gradient in one launch:
// one CTA per block runs alcc_solve_block (alcc.cpp:222-258) -> alcc_core
// (:54-191) with MAPG (engines.cpp:57-106) entirely on chip, for partitions
// with small blocks (nbar <= kMaxBlock). Larger blocks use one sub-problem
// handle per block (general.cu), whose sweeps need the whole GPU.
//
// Per block b (points [b nbar, (b+1) nbar)):
//   theta_k  nbar x nbar in a global workspace (L1/L2-resident, private to
//            the CTA), zero diagonal; updated in place at the outer steps
//   sweep    pass 1, thread per column: v = max(theta - row, 0) and the
//            column aggregates (colsum, V^T X); pass 2, warp per row: the
//            same v recomputed lane-per-column, row sums by a fixed butterfly
//   MAPG     thread per point: gradient step, ball projections, momentum,
//            fixed-order block reductions for the distances and the stop test
//   outer    the scalar logic of alcc_core (P_1, l_max, the certified gap,
//            the target_subopt stop, the decay of tau / alpha), computed
//            redundantly by every thread from the same block sums
// Every reduction has a fixed order: results are deterministic and follow
// the same arithmetic as the per-handle path (alcc.cu) up to summation order.
#include <cuda_runtime.h>
#include <math.h>

#include "device.cuh"
#include "handle.cuh"
#include "pipeline.cuh"
#include "balcc.cuh"

namespace crb {

constexpr int kBT = 256;          // threads per block CTA
constexpr int kMaxBlock = 160;    // largest nbar served here (measured crossover with
                                  // the per-block handles: nbar 100 -> 2.5x faster here,
                                  // nbar 250 -> 2.4x slower)

namespace {

template <int W>
__device__ __forceinline__ void bsum(double (&v)[W]) {  // fixed order, result in every thread
  __shared__ double sh[kBT / 32][W];
  __shared__ double tot[W];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < W; ++w) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[w] += __shfl_xor_sync(0xffffffffu, v[w], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w) sh[warp][w] = v[w];
  }
  __syncthreads();
  if (threadIdx.x < W) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kBT / 32; ++k) t += sh[k][threadIdx.x];
    tot[threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int w = 0; w < W; ++w) v[w] = tot[w];
  __syncthreads();
}

// residual row (l1 = r, l2 = c) at a point: y_r - c_c - x_r . xi_c
template <int NN>
__device__ __forceinline__ double pair_row(const double* xr, double yr, const double* xic,
                                           double ccv) {
  double row = yr - ccv;
#pragma unroll
  for (int j = 0; j < NN; ++j) row = fma(-xr[j], xic[j], row);
  return row;
}

// c_l = y_l - xi_l . x_l of a point
template <int NN>
__device__ __forceinline__ void point_c(const double* X, const double* Y, const double* XI,
                                        double* CC, long long nb) {
  for (long long l = threadIdx.x; l < nb; l += kBT) {
    double cx = 0.0;
#pragma unroll
    for (int j = 0; j < NN; ++j) cx = fma(XI[l * NN + j], X[l * NN + j], cx);
    CC[l] = Y[l] - cx;
  }
}

// One pass over the block's pairs. Warp w owns the 32-column strip w % S and
// the row chunk w / S (S = ceil(nb/32) strips, P = 8 / S chunks), lane = column:
// column aggregates stay in registers, row sums are fixed butterflies per row.
// Partials go to a small per-block scratch (L1-resident) and are combined per
// point in a fixed order. STATS: per-thread (S_nn, S_vr, S_vv); UPDATE: theta
// <- v / c in place (each element is owned by one lane).
struct Tile {
  int S, P;  // strips, row chunks
};
__device__ __forceinline__ Tile tile_of(int nb) {
  Tile t;
  t.S = (nb + 31) / 32;
  t.P = (kBT / 32) / t.S;
  if (t.P < 1) t.P = 1;
  return t;
}

template <int NN, bool STATS, bool UPDATE>
__device__ void block_sweep(const double* X, const double* Y, const double* XI, const double* CC,
                            double* th, int nb, double cdiv, double* CS, double* VX, double* RS,
                            double* colpart /* [P][nb][NN+1] */, double* rspart /* [nb][S] */,
                            double (&sc)[3]) {
  const Tile tl = tile_of(nb);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < tl.S * tl.P) {
    const int strip = warp % tl.S, chunk = warp / tl.S;
    const int rlo = nb * chunk / tl.P, rhi = nb * (chunk + 1) / tl.P;
    const int c = strip * 32 + lane;
    const bool valid = c < nb;
    double xic[NN];
#pragma unroll
    for (int j = 0; j < NN; ++j) xic[j] = valid ? XI[c * NN + j] : 0.0;
    const double ccv = valid ? CC[c] : 0.0;
    double acc[NN + 1];
#pragma unroll
    for (int j = 0; j <= NN; ++j) acc[j] = 0.0;
    const double* xr = X + rlo * NN;
    double* thr = th + rlo * nb + c;
    for (int r = rlo; r < rhi; ++r, xr += NN, thr += nb) {
      double x[NN];
#pragma unroll
      for (int j = 0; j < NN; ++j) x[j] = xr[j];
      double row = pair_row<NN>(x, Y[r], xic, ccv);
      const bool on = valid && r != c;
      if (!on) row = 0.0;
      const double v = on ? keep_if_nonneg(*thr - row) : 0.0;
      acc[0] += v;
#pragma unroll
      for (int j = 0; j < NN; ++j) acc[1 + j] = fma(v, x[j], acc[1 + j]);
      if (STATS) {
        const double m = keep_if_neg(row);
        sc[0] = fma(m, m, sc[0]);
        sc[1] = fma(v, row, sc[1]);
        sc[2] = fma(v, v, sc[2]);
      }
      if (UPDATE && on) *thr = v / cdiv;  // alcc.cpp:176
      double rsum = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
      if (lane == 0) rspart[r * tl.S + strip] = rsum;
    }
    if (valid) {
      double* dst = colpart + (chunk * nb + c) * (NN + 1);
#pragma unroll
      for (int j = 0; j <= NN; ++j) dst[j] = acc[j];
    }
  }
  __syncthreads();
  for (int l = threadIdx.x; l < nb; l += kBT) {  // fixed-order combine per point
    double rs = 0.0;
    for (int st = 0; st < tl.S; ++st) rs += rspart[l * tl.S + st];
    RS[l] = rs;
    double a[NN + 1];
#pragma unroll
    for (int j = 0; j <= NN; ++j) a[j] = 0.0;
    for (int ch = 0; ch < tl.P; ++ch) {
      const double* src = colpart + (ch * nb + l) * (NN + 1);
#pragma unroll
      for (int j = 0; j <= NN; ++j) a[j] += src[j];
    }
    CS[l] = a[0];
#pragma unroll
    for (int j = 0; j < NN; ++j) VX[l * NN + j] = a[1 + j];
  }
  __syncthreads();
}

template <int NN>
__global__ void __launch_bounds__(kBT) balcc_kernel(const BalccArgs A) {
  const int b = blockIdx.x;
  const long long nb = A.nbar, base = (long long)b * nb;
  const double gamma = A.gamma;
  const cr_alcc_config& cfg = A.cfg;
  const double* X = A.X + base * NN;
  const double* cy = A.cy + base;
  const double* cx = A.cxi + base * NN;
  double* y1 = A.ey + base;
  double* x1 = A.exi + base * NN;
  double* y1p = A.y1p + base;
  double* x1p = A.x1p + base * NN;
  double* y2 = A.y2 + base;
  double* x2 = A.x2 + base * NN;
  double* CC = A.cc + base;
  double* RS = A.rs + base;
  double* CS = A.cs + base;
  double* VX = A.vx + base * NN;
  double* th = A.theta + (long long)b * nb * nb;
  double* CP = A.scratch + (long long)b * A.scratch_per_block;  // [P][nb][NN+1] | [nb][S]
  double* RP = CP + (long long)(kBT / 32) * nb * (NN + 1);
  const double sA1 = A.sigma_A1, sA2 = A.sigma_A2[b];
  const long long Nn = nb * NN;

  // block radius (alcc.cpp:238-243)
  double v2[2] = {0.0, 0.0};
  for (long long l = threadIdx.x; l < nb; l += kBT) {
    const double d = A.fy[base + l] - cy[l];
    v2[0] = fma(d, d, v2[0]);
  }
  for (long long i = threadIdx.x; i < Nn; i += kBT) {
    const double d = A.fxi[base * NN + i] - cx[i];
    v2[1] = fma(d, d, v2[1]);
  }
  bsum<2>(v2);
  const double Bbar = fmax(sqrt(v2[0] + gamma * v2[1]), 1e-8);
  const double By = Bbar, Bx = Bbar / sqrt(gamma);
  // project the warm start (alcc.cpp:68-69)
  v2[0] = v2[1] = 0.0;
  for (long long l = threadIdx.x; l < nb; l += kBT) {
    const double d = y1[l] - cy[l];
    v2[0] = fma(d, d, v2[0]);
  }
  for (long long i = threadIdx.x; i < Nn; i += kBT) {
    const double d = x1[i] - cx[i];
    v2[1] = fma(d, d, v2[1]);
  }
  bsum<2>(v2);
  {
    const double dy = sqrt(v2[0]), dx = sqrt(v2[1]);
    if (dy > By) {
      const double f = By / dy;
      for (long long l = threadIdx.x; l < nb; l += kBT) y1[l] = cy[l] + f * (y1[l] - cy[l]);
    }
    if (dx > Bx) {
      const double f = Bx / dx;
      for (long long i = threadIdx.x; i < Nn; i += kBT) x1[i] = cx[i] + f * (x1[i] - cx[i]);
    }
  }
  for (long long i = threadIdx.x; i < nb * nb; i += kBT) th[i] = 0.0;
  __syncthreads();

  // P_1 (alcc.cpp:75-84): penalty at the start point with theta = 0
  double mu = cfg.mu1, tau, alpha_y, alpha_x;
  {
    point_c<NN>(X, y1, x1, CC, nb);
    __syncthreads();
    double sc[3] = {0.0, 0.0, 0.0};
    block_sweep<NN, true, false>(X, y1, x1, CC, th, (int)nb, 1.0, CS, VX, RS, CP, RP, sc);
    double v3[3] = {sc[2], 0.0, 0.0};
    for (long long l = threadIdx.x; l < nb; l += kBT) {
      const double d = y1[l] - cy[l];
      v3[1] = fma(d, d, v3[1]);
    }
    for (long long i = threadIdx.x; i < Nn; i += kBT) {
      const double d = x1[i] - cx[i];
      v3[2] = fma(d, d, v3[2]);
    }
    bsum<3>(v3);
    const double p1 = v3[1] / (2.0 * mu) + gamma * v3[2] / (2.0 * mu) + 0.5 * v3[0];
    if (!isfinite(p1)) {
      if (threadIdx.x == 0) A.status[b] = 5;
      return;
    }
    tau = fmax(cfg.tau1_scale * p1, 1e-16);
    alpha_y = alpha_x = cfg.alpha1_scale * (By + Bx);
  }

  long long total = 0;
  double infeas_raw = 0.0;
  const double m = (double)nb * (double)(nb - 1);
  int status = 0;
  for (long long k = 1; k <= cfg.max_outer; ++k) {
    const double Ly = 1.0 / mu + sA1 * sA1;  // alcc.cpp:101-102
    const double Lx = gamma / mu + sA2 * sA2;
    long long lmax = (long long)ceil(4.0 * sqrt((Ly * By * By + Lx * Bx * Bx) / tau));
    if (lmax < 10) lmax = 10;
    if (lmax > cfg.mapg_cap) lmax = cfg.mapg_cap;
    // MAPG (engines.cpp:65-106) from (y1, x1)
    for (long long l = threadIdx.x; l < nb; l += kBT) y1p[l] = y2[l] = y1[l];
    for (long long i = threadIdx.x; i < Nn; i += kBT) x1p[i] = x2[i] = x1[i];
    __syncthreads();
    point_c<NN>(X, y2, x2, CC, nb);
    __syncthreads();
    double t = 1.0;
    const double gm = gamma / mu;
    long long ell = 0;
    bool bad = false;
    while (ell < lmax) {
      double dummy[3];
      block_sweep<NN, false, false>(X, y2, x2, CC, th, (int)nb, 1.0, CS, VX, RS, CP, RP, dummy);
      double pd[3] = {0.0, 0.0, 0.0};
      for (long long l = threadIdx.x; l < nb; l += kBT) {  // alcc.cpp:38-41, engines.cpp:82-88
        const double csl = CS[l];
        const double gy = (y2[l] - cy[l]) / mu - (RS[l] - csl);
        bool nf = !isfinite(gy);
        const double yn = y2[l] - gy / Ly;
        y1p[l] = y1[l];
        y1[l] = yn;
        const double dy = yn - cy[l];
        pd[0] = fma(dy, dy, pd[0]);
#pragma unroll
        for (int j = 0; j < NN; ++j) {
          const long long q = l * NN + j;
          const double adj = csl * X[q] - VX[q];
          const double g = gm * (x2[q] - cx[q]) - adj;
          nf |= !isfinite(g);
          const double xn = x2[q] - g / Lx;
          x1p[q] = x1[q];
          x1[q] = xn;
          const double dx = xn - cx[q];
          pd[1] = fma(dx, dx, pd[1]);
        }
        if (nf) pd[2] += 1.0;
      }
      bsum<3>(pd);
      bad = pd[2] != 0.0;
      const double dy = sqrt(pd[0]), dx = sqrt(pd[1]);
      const bool sy = dy > By, sx = dx > Bx;
      const double fy = sy ? By / dy : 1.0, fx = sx ? Bx / dx : 1.0;
      const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
      const double beta = (t - 1.0) / t_next;
      double pc[2] = {0.0, 0.0};
      for (long long l = threadIdx.x; l < nb; l += kBT) {
        double yv = y1[l];
        if (sy) {
          yv = cy[l] + fy * (yv - cy[l]);
          y1[l] = yv;
        }
        const double e = yv - y2[l];
        pc[0] = fma(e, e, pc[0]);
        const double y2n = yv + beta * (yv - y1p[l]);
        y2[l] = y2n;
        double cxs = 0.0;
#pragma unroll
        for (int j = 0; j < NN; ++j) {
          const long long q = l * NN + j;
          double xv = x1[q];
          if (sx) {
            xv = cx[q] + fx * (xv - cx[q]);
            x1[q] = xv;
          }
          const double ex = xv - x2[q];
          pc[1] = fma(ex, ex, pc[1]);
          const double x2n = xv + beta * (xv - x1p[q]);
          x2[q] = x2n;
          cxs = fma(x2n, X[q], cxs);
        }
        CC[l] = y2n - cxs;
      }
      bsum<2>(pc);
      t = t_next;
      ++ell;
      if (bad) break;
      if (sqrt(pc[0]) <= alpha_y && sqrt(pc[1]) <= alpha_x) break;
    }
    total += ell;
    if (bad) {
      status = 5;
      break;
    }
    // outer step at y1 (alcc.cpp:124-183): statistics, theta <- v / c in place
    point_c<NN>(X, y1, x1, CC, nb);
    __syncthreads();
    double sc[3] = {0.0, 0.0, 0.0};
    block_sweep<NN, true, true>(X, y1, x1, CC, th, (int)nb, cfg.c, CS, VX, RS, CP, RP, sc);
    double st[8] = {sc[0], sc[1], sc[2], 0.0, 0.0, 0.0, 0.0, 0.0};
    for (long long l = threadIdx.x; l < nb; l += kBT) {
      const double d = y1[l] - cy[l];
      st[3] = fma(d, d, st[3]);
      const double ay = RS[l] - CS[l];
      st[5] = fma(ay, ay, st[5]);
      st[7] = fma(cy[l], ay, st[7]);
#pragma unroll
      for (int j = 0; j < NN; ++j) {
        const long long q = l * NN + j;
        const double dx = x1[q] - cx[q];
        st[4] = fma(dx, dx, st[4]);
        const double ax = CS[l] * X[q] - VX[q];
        st[6] = fma(ax, ax, st[6]);
        st[7] = fma(cx[q], ax, st[7]);
      }
    }
    bsum<8>(st);
    infeas_raw = sqrt(st[0]);
    const double mu2 = mu * mu;
    const double dual = -0.5 * (mu2 * st[5]) - (mu2 * st[6]) / (2.0 * gamma) - mu * st[7];
    const double primal = 0.5 * st[3] + 0.5 * gamma * st[4];
    const double certified = primal - dual;
    bool stop;
    if (A.target > 0)  // alcc.cpp:153-155
      stop = certified <= A.target && (mu * sqrt(st[2])) * infeas_raw <= A.target;
    else
      stop = m > 0 && infeas_raw / sqrt(m) <= cfg.infeas_norm_tol &&
             fabs(mu * st[1] / m) <= cfg.gap_norm_tol;
    if (stop) break;
    mu *= cfg.c;
    const double decay = pow(cfg.c * pow((double)k, 1.0 + cfg.kappa), 2.0);
    tau /= decay;
    alpha_y /= decay;
    alpha_x /= decay;
  }
  if (threadIdx.x == 0) {
    A.infeas[b] = infeas_raw;
    A.iters[b] = total;
    A.status[b] = status;
  }
}

template <int NN>
void launch_n(const BalccArgs& a, cudaStream_t s) {
  balcc_kernel<NN><<<a.K, kBT, 0, s>>>(a);
}
using BalccFn = void (*)(const BalccArgs&, cudaStream_t);

}  // namespace

int balcc_max_block() { return kMaxBlock; }

// [P][nb][n+1] column partials (P <= 8 chunks) and [nb][S] row-sum partials (S <= 8)
long long balcc_scratch_per_block(long long nbar, int n) {
  return (long long)(kBT / 32) * nbar * (n + 1) + nbar * ((nbar + 31) / 32);
}

cudaError_t launch_balcc(const BalccArgs& a, int n, cudaStream_t s) {
  static constexpr BalccFn tab[kMaxN] = {
#define CRB_LAUNCH_N(N) launch_n<N>
      CRB_N_SEQ(CRB_LAUNCH_N)
#undef CRB_LAUNCH_N
};
  if (n < 1 || n > kMaxN || a.nbar > kMaxBlock) return cudaErrorInvalidValue;
  tab[n - 1](a, s);
  return cudaGetLastError();
}

}  // namespace crb
