// alcc.cu -- the standalone augmented-Lagrangian solver:
// alcc_solve (alcc.cpp:193-208) -> alcc_core (alcc.cpp:54-191) with the
// PenaltyOracle (alcc.cpp:33-47) and the MAPG inner loop (engines.cpp:57-106),
// over all N(N-1) pair rows R(y, xi) = A1 y + A2 xi (FullRows, alcc.hpp:32-48).
//
// Device layout: the outer multiplier theta_k is an N x ld pair matrix in
// V[cur] (the P-APG dual buffers are reused; a solve invalidates any P-APG
// state on the handle), theta_{k+1} = v / c is written into V[1-cur] by the
// outer sweep. Points are [y (N) | xi (N n)] vectors: p1 = y1, p1p = y1_prev,
// p2 = y2 of the MAPG recursion.
//
// One MAPG iteration = 4 launches, captured in a CUDA graph and halted on
// the device:
//   K1p  penalty sweep (sweep.cu / sweep_mma.cu, kModePenalty): per pair
//        v = max(theta - row(y2, xi2), 0), aggregates (rowsum, colsum, V^T X)
//        -- 8 B of HBM per pair (theta read once)
//   K3   fixed-order reduce of the sweep partials (kernels.cu)
//   Kg   gradient step: grad = (y2 - ybar)/mu - A1^T v, (gamma/mu) xi2 - A2^T v
//        with A1^T v = rowsum - colsum, (A2^T v)_l = colsum_l x_l - (V^T X)_l;
//        y1 = y2 - grad / L (engines.cpp:83-88); partial ball distances
//   Ks   ball projections (projections.hpp:22-26), displacements, momentum
//        (engines.cpp:97-103), records of y2 for the next sweep; the last
//        block applies the stop test (engines.cpp:104-105) and halts.
// One outer step (alcc.cpp:124-183) = records(y1) + kModePenaltyUpdate sweep
// (stats + theta_{k+1}) + reduce + one stats block; the scalar logic runs on
// the host exactly as in the reference.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "handle.cuh"
#include "host.hpp"
#include "iteration.cuh"
#include "pipeline.cuh"

namespace crb {

struct AlccDev {
  long long ell;   // MAPG iterations of the current outer step
  long long lmax;
  int halt;
  int hit_cap;
  int cur;         // slot of theta_k
  int nonfinite;
  double t;        // momentum
  double mu, gamma, L_y, L_xi, alpha_y, alpha_xi, Bbar_y, Bbar_xi;
  double disp_y, disp_xi;
  // stats block: |y-ybar|^2, |xi|^2, |A1^T v|^2, |A2^T v|^2, ybar.A1^T v, S_vv, S_vr, S_nn
  double stats[8];
};

namespace {

constexpr int kSBlock = 1024;  // single-block kernels

struct AlccArgs {
  AlccDev* d;
  const double* X;
  const double* cy;     // ball / quadratic centre of y (ybar standalone, ybar_i + q_y per block)
  const double* cxi;    // centre of xi (nullptr: 0 standalone, q_xi / gamma per block)
  const double* fy;     // block mode: the feasible affine slice (radius, alcc.cpp:238-243)
  const double* fxi;
  const double* agg;    // [rowsum N | colagg N (n+1) | scalars]
  double *p1, *p1p, *p2;
  double *rowrec, *colrec;
  double *part1, *part2;
  unsigned int* counter;
  long long N;
  int n;
};

// fixed-order block sum of W values (warp butterflies, then warps in order);
// the result is valid in every thread
template <int W, int BS>
__device__ __forceinline__ void block_sum_all(double (&v)[W]) {
  __shared__ double sh[BS / 32][W];
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
    for (int k = 0; k < BS / 32; ++k) t += sh[k][threadIdx.x];
    tot[threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int w = 0; w < W; ++w) v[w] = tot[w];
  __syncthreads();
}

// sum of `count` records part[g][2] in a fixed order, valid in every thread
template <int BS>
__device__ __forceinline__ void records_sum2(const double* part, int count, double (&out)[2]) {
  double v[2] = {0.0, 0.0};
  for (int g = threadIdx.x; g < count; g += BS) {
    v[0] += __ldcg(part + 2 * g);
    v[1] += __ldcg(part + 2 * g + 1);
  }
  block_sum_all<2, BS>(v);
  out[0] = v[0];
  out[1] = v[1];
}

__device__ __forceinline__ double cxi_at(const AlccArgs& a, long long i) {
  return a.cxi != nullptr ? a.cxi[i] : 0.0;
}

template <int NN>
__device__ __forceinline__ void write_records(const AlccArgs& a, long long l, double y,
                                              const double* xi /* NN */) {
  constexpr int RP = rec_pitch(NN);
  double cx = 0.0;
  double* cr = a.colrec + l * RP;
#pragma unroll
  for (int j = 0; j < NN; ++j) {
    cx = fma(xi[j], a.X[l * NN + j], cx);
    cr[j] = -xi[j];
  }
  cr[NN] = -(y - cx);
  cr[NN + 1] = 1.0;
  a.rowrec[l * RP + NN + 1] = y;
}

// project_ball(warm, centre, B) for y and xi (alcc.cpp:68-69); one block
template <int NN>
__global__ void __launch_bounds__(kSBlock) project_start_kernel(const AlccArgs a) {
  const long long N = a.N;
  double v[2] = {0.0, 0.0};
  for (long long l = threadIdx.x; l < N; l += kSBlock) {
    const double d = a.p1[l] - a.cy[l];
    v[0] = fma(d, d, v[0]);
  }
  for (long long i = threadIdx.x; i < N * NN; i += kSBlock) {
    const double d = a.p1[N + i] - cxi_at(a, i);
    v[1] = fma(d, d, v[1]);
  }
  block_sum_all<2, kSBlock>(v);
  const double dy = sqrt(v[0]), dx = sqrt(v[1]);
  const double By = a.d->Bbar_y, Bx = a.d->Bbar_xi;
  if (dy > By) {
    const double f = By / dy;
    for (long long l = threadIdx.x; l < N; l += kSBlock) a.p1[l] = a.cy[l] + f * (a.p1[l] - a.cy[l]);
  }
  if (dx > Bx) {
    const double f = Bx / dx;
    for (long long i = threadIdx.x; i < N * NN; i += kSBlock) {
      const double c = cxi_at(a, i);
      a.p1[N + i] = c + f * (a.p1[N + i] - c);
    }
  }
}

// block radius (alcc.cpp:238-243): Bbar = max(sqrt(|yhat - c_y|^2 + gamma |xihat - c_xi|^2),
// 1e-8); Bbar_y = Bbar, Bbar_xi = Bbar / sqrt(gamma). One block.
template <int NN>
__global__ void __launch_bounds__(kSBlock) block_bounds_kernel(const AlccArgs a) {
  const long long N = a.N;
  double v[2] = {0.0, 0.0};
  for (long long l = threadIdx.x; l < N; l += kSBlock) {
    const double d = a.fy[l] - a.cy[l];
    v[0] = fma(d, d, v[0]);
  }
  for (long long i = threadIdx.x; i < N * NN; i += kSBlock) {
    const double d = a.fxi[i] - cxi_at(a, i);
    v[1] = fma(d, d, v[1]);
  }
  block_sum_all<2, kSBlock>(v);
  if (threadIdx.x == 0) {
    const double gamma = a.d->gamma;
    const double Bsq = v[0] + gamma * v[1];
    const double B = fmax(sqrt(Bsq), 1e-8);
    a.d->Bbar_y = B;
    a.d->Bbar_xi = B / sqrt(gamma);
  }
}

// MAPG start (engines.cpp:65-66): y1_prev = y1 = y2 = y0; records of y2
template <int NN>
__global__ void __launch_bounds__(kPBlock) mapg_reset_kernel(const AlccArgs a) {
  const long long N = a.N;
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock) {
    const double y = a.p1[l];
    a.p1p[l] = y;
    a.p2[l] = y;
    double xi[NN];
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      xi[j] = a.p1[N + l * NN + j];
      a.p1p[N + l * NN + j] = xi[j];
      a.p2[N + l * NN + j] = xi[j];
    }
    write_records<NN>(a, l, y, xi);
  }
}

// records of y1 (the MAPG result) for the outer sweep
template <int NN>
__global__ void __launch_bounds__(kPBlock) point_records_kernel(const AlccArgs a) {
  const long long N = a.N;
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock) {
    double xi[NN];
#pragma unroll
    for (int j = 0; j < NN; ++j) xi[j] = a.p1[N + l * NN + j];
    write_records<NN>(a, l, a.p1[l], xi);
  }
}

// Kg: gradient at y2 (alcc.cpp:38-41), y1 = y2 - g / L (engines.cpp:82-88)
template <int NN>
__global__ void __launch_bounds__(kPBlock) mapg_grad_kernel(const AlccArgs a) {
  AlccDev* d = a.d;
  if (d->halt) return;
  const long long N = a.N;
  const double mu = d->mu, gm = d->gamma / d->mu, Ly = d->L_y, Lx = d->L_xi;
  double acc[2] = {0.0, 0.0};
  bool bad = false;
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock) {
    const double* ca = a.agg + N + l * (NN + 1);
    const double rs = a.agg[l], cs = ca[0];
    const double gy = (a.p2[l] - a.cy[l]) / mu - (rs - cs);
    bad |= !isfinite(gy);
    const double y1 = a.p2[l] - gy / Ly;
    a.p1p[l] = a.p1[l];
    a.p1[l] = y1;
    const double dy = y1 - a.cy[l];
    acc[0] = fma(dy, dy, acc[0]);
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      const long long k = N + l * NN + j;
      const double adj = cs * a.X[l * NN + j] - ca[1 + j];
      const double g = gm * (a.p2[k] - cxi_at(a, l * NN + j)) - adj;
      bad |= !isfinite(g);
      const double x1 = a.p2[k] - g / Lx;
      a.p1p[k] = a.p1[k];
      a.p1[k] = x1;
      const double dx = x1 - cxi_at(a, l * NN + j);
      acc[1] = fma(dx, dx, acc[1]);
    }
  }
  if (bad) d->nonfinite = 1;
  block_sum_all<2, kPBlock>(acc);
  if (threadIdx.x == 0) {
    a.part1[2 * blockIdx.x] = acc[0];
    a.part1[2 * blockIdx.x + 1] = acc[1];
  }
}

// Ks: projections, displacements, momentum, records; last block: stop test
template <int NN>
__global__ void __launch_bounds__(kPBlock) mapg_step_kernel(const AlccArgs a) {
  AlccDev* d = a.d;
  if (d->halt) return;
  const long long N = a.N;
  double dist2[2];
  records_sum2<kPBlock>(a.part1, gridDim.x, dist2);
  const double dy = sqrt(dist2[0]), dx = sqrt(dist2[1]);
  const bool sy = dy > d->Bbar_y, sx = dx > d->Bbar_xi;
  const double fy = sy ? d->Bbar_y / dy : 1.0, fx = sx ? d->Bbar_xi / dx : 1.0;
  const double t = d->t;
  const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));  // engines.hpp:11-13
  const double beta = (t - 1.0) / t_next;
  double acc[2] = {0.0, 0.0};
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock) {
    double y1 = a.p1[l];
    if (sy) {
      y1 = a.cy[l] + fy * (y1 - a.cy[l]);
      a.p1[l] = y1;
    }
    const double e = y1 - a.p2[l];
    acc[0] = fma(e, e, acc[0]);
    const double y2 = y1 + beta * (y1 - a.p1p[l]);
    a.p2[l] = y2;
    double xi2[NN];
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      const long long k = N + l * NN + j;
      double x1 = a.p1[k];
      if (sx) {
        const double c = cxi_at(a, l * NN + j);
        x1 = c + fx * (x1 - c);
        a.p1[k] = x1;
      }
      const double ex = x1 - a.p2[k];
      acc[1] = fma(ex, ex, acc[1]);
      xi2[j] = x1 + beta * (x1 - a.p1p[k]);
      a.p2[k] = xi2[j];
    }
    write_records<NN>(a, l, y2, xi2);
  }
  block_sum_all<2, kPBlock>(acc);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    a.part2[2 * blockIdx.x] = acc[0];
    a.part2[2 * blockIdx.x + 1] = acc[1];
    __threadfence();
    last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double disp2[2];
  records_sum2<kPBlock>(a.part2, gridDim.x, disp2);
  if (threadIdx.x == 0) {
    *a.counter = 0u;
    const double disp_y = sqrt(disp2[0]), disp_x = sqrt(disp2[1]);
    d->disp_y = disp_y;
    d->disp_xi = disp_x;
    d->t = t_next;
    const long long ell = d->ell + 1;
    d->ell = ell;
    const bool stop = disp_y <= d->alpha_y && disp_x <= d->alpha_xi;
    if (!stop && ell == d->lmax) d->hit_cap = 1;
    if (stop || ell >= d->lmax || d->nonfinite) d->halt = 1;
  }
}

// outer-step statistics (alcc.cpp:124-145) from the aggregates of v and y1
template <int NN>
__global__ void __launch_bounds__(kSBlock) alcc_stats_kernel(const AlccArgs a) {
  const long long N = a.N;
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (long long l = threadIdx.x; l < N; l += kSBlock) {
    const double* ca = a.agg + N + l * (NN + 1);
    const double dy = a.p1[l] - a.cy[l];
    v[0] = fma(dy, dy, v[0]);
    const double ay = a.agg[l] - ca[0];
    v[2] = fma(ay, ay, v[2]);
    v[4] = fma(a.cy[l], ay, v[4]);
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      const double c = cxi_at(a, l * NN + j);
      const double dx = a.p1[N + l * NN + j] - c;
      v[1] = fma(dx, dx, v[1]);
      const double ax = ca[0] * a.X[l * NN + j] - ca[1 + j];
      v[3] = fma(ax, ax, v[3]);
      v[4] = fma(c, ax, v[4]);  // lambda . rows_center = (A1^T l).c_y + (A2^T l).c_xi
    }
  }
  block_sum_all<5, kSBlock>(v);
  if (threadIdx.x == 0) {
    AlccDev* d = a.d;
    for (int w = 0; w < 5; ++w) d->stats[w] = v[w];
    const double* sc = a.agg + N + N * (NN + 1);
    d->stats[5] = sc[0];  // S_vv
    d->stats[6] = sc[1];  // S_vr
    d->stats[7] = sc[3];  // S_nn
  }
}

// lambda = mu (theta - row)_+ of rows [ra, rb) in canonical order (alcc.cpp:125-126)
__global__ void multiplier_out_kernel(double* stage, const double* V, double mu,
                                      const double* rowrec, const double* colrec, long long N,
                                      int n, long long ld, long long ra, long long rb) {
  const int RP = rec_pitch(n);
  const long long total = (rb - ra) * (N - 1);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long lr = i / (N - 1), k = i % (N - 1);
    const long long gr = ra + lr;
    const long long c = k + (k >= gr ? 1 : 0);
    const double* xr = rowrec + gr * RP;
    const double* cr = colrec + c * RP;
    double row = xr[n + 1] + cr[n];
    for (int j = 0; j < n; ++j) row = fma(xr[j], cr[j], row);
    const double th = V[gr * ld + c];
    const double vn = th - row > 0.0 ? th - row : 0.0;
    stage[i] = mu * vn;
  }
}

// ---- small sub-problems: the whole MAPG call in one cooperative launch --------
// For N up to a few thousand points (general-K blocks, config 1) an MAPG
// iteration is a few microseconds of work and the 4-launch graph is bound by
// launch latency. Here one launch runs engines.cpp:69-106 to its stop with
// three grid barriers per iteration:
//   A  penalty sweep: warp per (32-column strip, row chunk), v = max(theta -
//      row, 0), column partials [N][n+1][P] and row-sum partials [N][S]
//   B  warp per point: fixed-order partial sums (lanes over partials), the
//      gradient step y1 = y2 - grad / L, block partials of the ball distances
//   C  every block sums the distance partials in the same order (identical
//      projection decisions), projection, displacement, momentum, records
//   D  every block sums the displacement partials -> identical stop decision
namespace cgx = cooperative_groups;
constexpr int kLBlock = 256;

struct LoopArgs {
  AlccArgs a;
  const double* V0;
  const double* V1;
  double* colpart;  // [N][n+1][P]
  double* rowpart;  // [N][S]
  double* partB;    // [G][3]: |y1 - c_y|^2, |xi1 - c_xi|^2, non-finite count
  double* partC;    // [G][2]: displacement^2 (y, xi)
  long long ld;
  int S, P;
};

template <int W>
__device__ __forceinline__ void grid_sum(const double* part, int G, double (&out)[W]) {
  double v[W];
#pragma unroll
  for (int w = 0; w < W; ++w) v[w] = 0.0;
  for (int g = threadIdx.x; g < G; g += kLBlock) {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] += __ldcg(part + (long long)g * W + w);
  }
  block_sum_all<W, kLBlock>(v);
#pragma unroll
  for (int w = 0; w < W; ++w) out[w] = v[w];
}

template <int NN>
__global__ void __launch_bounds__(kLBlock) mapg_loop_kernel(const LoopArgs L) {
  constexpr int RP = rec_pitch(NN);
  cgx::grid_group grid = cgx::this_grid();
  const AlccArgs& a = L.a;
  AlccDev* d = a.d;
  const long long N = a.N;
  const long long tid = (long long)blockIdx.x * kLBlock + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * kLBlock;
  const int lane = threadIdx.x & 31;
  const long long gwarp = tid >> 5, nwarps = nthreads >> 5;
  const int G = gridDim.x;
  const double* th = d->cur ? L.V1 : L.V0;
  const double mu = d->mu, gm = d->gamma / d->mu, Ly = d->L_y, Lx = d->L_xi;
  const double ay = d->alpha_y, ax = d->alpha_xi, By = d->Bbar_y, Bx = d->Bbar_xi;
  const long long lmax = d->lmax;
  double t = d->t;
  long long ell = d->ell;
  bool hit = false, bad = false;
  double disp_y = 0.0, disp_x = 0.0;
  while (ell < lmax) {
    // ---- A: penalty sweep partials
    for (long long w = gwarp; w < (long long)L.S * L.P; w += nwarps) {
      const int strip = (int)(w % L.S);
      const int chunk = (int)(w / L.S);
      const long long rlo = N * chunk / L.P, rhi = N * (chunk + 1) / L.P;
      const long long col = (long long)strip * 32 + lane;
      const bool valid = col < N;
      const double* cr = a.colrec + (valid ? col : 0) * RP;
      double xi[NN], acc[NN + 1];
      const double cc = valid ? __ldcg(cr + NN) : 0.0;
#pragma unroll
      for (int j = 0; j < NN; ++j) xi[j] = valid ? __ldcg(cr + j) : 0.0;
#pragma unroll
      for (int j = 0; j <= NN; ++j) acc[j] = 0.0;
      for (long long r = rlo; r < rhi; ++r) {
        const double* xr = a.rowrec + r * RP;
        double x[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) x[j] = __ldcg(xr + j);
        double row = __ldcg(xr + NN + 1) + cc;
#pragma unroll
        for (int j = 0; j < NN; ++j) row = fma(x[j], xi[j], row);
        if (!valid || col == r) row = 0.0;
        const double tv = valid ? __ldg(th + r * L.ld + col) : 0.0;
        const double v = keep_if_nonneg(tv - row);
        acc[0] += v;
#pragma unroll
        for (int j = 0; j < NN; ++j) acc[1 + j] = fma(v, x[j], acc[1 + j]);
        double rs = v;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
        if (lane == 0) __stcg(L.rowpart + r * L.S + strip, rs);
      }
      if (valid) {
        double* dst = L.colpart + (col * (NN + 1)) * L.P + chunk;
#pragma unroll
        for (int j = 0; j <= NN; ++j) __stcg(dst + (long long)j * L.P, acc[j]);
      }
    }
    grid.sync();
    // ---- B: reduce per point + gradient step
    {
      double pb[3] = {0.0, 0.0, 0.0};
      for (long long l = gwarp; l < N; l += nwarps) {
        double rs = 0.0;
        for (int sidx = lane; sidx < L.S; sidx += 32) rs += __ldcg(L.rowpart + l * L.S + sidx);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
        double ca[NN + 1];
#pragma unroll
        for (int j = 0; j <= NN; ++j) {
          double sj = 0.0;
          const double* src = L.colpart + (l * (NN + 1) + j) * L.P;
          for (int p = lane; p < L.P; p += 32) sj += __ldcg(src + p);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sj += __shfl_xor_sync(0xffffffffu, sj, o);
          ca[j] = sj;
        }
        if (lane == 0) {
          const double cs = ca[0];
          const double y2 = __ldcg(a.p2 + l);
          const double gy = (y2 - a.cy[l]) / mu - (rs - cs);
          bool b = !isfinite(gy);
          const double y1 = y2 - gy / Ly;
          __stcg(a.p1p + l, __ldcg(a.p1 + l));
          __stcg(a.p1 + l, y1);
          const double dy = y1 - a.cy[l];
          pb[0] = fma(dy, dy, pb[0]);
#pragma unroll
          for (int j = 0; j < NN; ++j) {
            const long long k = N + l * NN + j;
            const double adj = cs * a.X[l * NN + j] - ca[1 + j];
            const double c = cxi_at(a, l * NN + j);
            const double g = gm * (__ldcg(a.p2 + k) - c) - adj;
            b |= !isfinite(g);
            const double x1 = __ldcg(a.p2 + k) - g / Lx;
            __stcg(a.p1p + k, __ldcg(a.p1 + k));
            __stcg(a.p1 + k, x1);
            const double dx = x1 - c;
            pb[1] = fma(dx, dx, pb[1]);
          }
          if (b) pb[2] += 1.0;
        }
      }
      block_sum_all<3, kLBlock>(pb);
      if (threadIdx.x == 0) {
        for (int w = 0; w < 3; ++w) __stcg(L.partB + (long long)blockIdx.x * 3 + w, pb[w]);
      }
    }
    grid.sync();
    // ---- C: projections, displacements, momentum, records
    double dist[3];
    grid_sum<3>(L.partB, G, dist);
    bad = dist[2] != 0.0;
    {
      const double dy = sqrt(dist[0]), dx = sqrt(dist[1]);
      const bool sy = dy > By, sx = dx > Bx;
      const double fy = sy ? By / dy : 1.0, fx = sx ? Bx / dx : 1.0;
      const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
      const double beta = (t - 1.0) / t_next;
      double pc[2] = {0.0, 0.0};
      for (long long l = tid; l < N; l += nthreads) {
        double y1 = __ldcg(a.p1 + l);
        if (sy) {
          y1 = a.cy[l] + fy * (y1 - a.cy[l]);
          __stcg(a.p1 + l, y1);
        }
        const double e = y1 - __ldcg(a.p2 + l);
        pc[0] = fma(e, e, pc[0]);
        const double y2n = y1 + beta * (y1 - __ldcg(a.p1p + l));
        __stcg(a.p2 + l, y2n);
        double xi2[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) {
          const long long k = N + l * NN + j;
          double x1 = __ldcg(a.p1 + k);
          if (sx) {
            const double c = cxi_at(a, l * NN + j);
            x1 = c + fx * (x1 - c);
            __stcg(a.p1 + k, x1);
          }
          const double ex = x1 - __ldcg(a.p2 + k);
          pc[1] = fma(ex, ex, pc[1]);
          xi2[j] = x1 + beta * (x1 - __ldcg(a.p1p + k));
          __stcg(a.p2 + k, xi2[j]);
        }
        write_records<NN>(a, l, y2n, xi2);
      }
      block_sum_all<2, kLBlock>(pc);
      if (threadIdx.x == 0) {
        __stcg(L.partC + (long long)blockIdx.x * 2, pc[0]);
        __stcg(L.partC + (long long)blockIdx.x * 2 + 1, pc[1]);
      }
      t = t_next;
    }
    grid.sync();
    // ---- D: identical stop decision in every block (engines.cpp:104-105)
    double disp[2];
    grid_sum<2>(L.partC, G, disp);
    disp_y = sqrt(disp[0]);
    disp_x = sqrt(disp[1]);
    ++ell;
    const bool stop = disp_y <= ay && disp_x <= ax;
    if (!stop && ell == lmax) hit = true;
    if (stop || bad) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    d->ell = ell;
    d->t = t;
    d->hit_cap = hit ? 1 : 0;
    d->nonfinite = bad ? 1 : 0;
    d->disp_y = disp_y;
    d->disp_xi = disp_x;
    d->halt = 1;
  }
}

using AlccKernel = void (*)(const AlccArgs);
template <int NN>
struct AlccTab {
  static constexpr AlccKernel project = project_start_kernel<NN>;
  static constexpr AlccKernel reset = mapg_reset_kernel<NN>;
  static constexpr AlccKernel records = point_records_kernel<NN>;
  static constexpr AlccKernel grad = mapg_grad_kernel<NN>;
  static constexpr AlccKernel step = mapg_step_kernel<NN>;
  static constexpr AlccKernel stats = alcc_stats_kernel<NN>;
  static constexpr AlccKernel bounds = block_bounds_kernel<NN>;
};
struct AlccFns {
  AlccKernel project, reset, records, grad, step, stats, bounds;
};
template <int NN>
constexpr AlccFns fns_for() {
  return {AlccTab<NN>::project, AlccTab<NN>::reset, AlccTab<NN>::records, AlccTab<NN>::grad,
          AlccTab<NN>::step,    AlccTab<NN>::stats, AlccTab<NN>::bounds};
}
template <int NN>
constexpr const void* loop_fn() {
  return (const void*)mapg_loop_kernel<NN>;
}
const void* const kLoopFns[kMaxN] = {
#define CRB_LOOP_FN(N) loop_fn<N>()
    CRB_N_SEQ(CRB_LOOP_FN)
#undef CRB_LOOP_FN
};

constexpr AlccFns kFns[kMaxN] = {
#define CRB_FNS_FOR(N) fns_for<N>()
    CRB_N_SEQ(CRB_FNS_FOR)
#undef CRB_FNS_FOR
};

AlccArgs alcc_args(cr_handle* h) {
  AlccArgs a{};
  a.d = h->alcc.dev;
  a.X = h->X;
  a.cy = h->alcc.cy ? h->alcc.cy : h->ybar;
  a.cxi = h->alcc.cxi;
  a.fy = h->alcc.fy;
  a.fxi = h->alcc.fxi;
  a.agg = h->xbuf;
  a.p1 = h->alcc.p1;
  a.p1p = h->alcc.p1p;
  a.p2 = h->alcc.p2;
  a.rowrec = h->rowrec;
  a.colrec = h->colrec;
  a.part1 = h->alcc.part1;
  a.part2 = h->alcc.part2;
  a.counter = h->alcc.counter;
  a.N = h->N;
  a.n = (int)h->n;
  return a;
}

cudaError_t launch_alcc(AlccKernel k, int grid, int block, const AlccArgs& a, cudaStream_t s) {
  void* args[] = {const_cast<AlccArgs*>(&a)};
  return cudaLaunchKernel((const void*)k, dim3((unsigned)grid), dim3((unsigned)block), args, 0, s);
}

SweepArgs penalty_sweep_args(cr_handle* h, double cdiv) {
  SweepArgs a = sweep_args(h, kModePenalty, false);
  a.cur = &h->alcc.dev->cur;
  a.stopped = nullptr;
  a.coef = h->consts;
  a.invL = 1.0;
  a.cdiv = cdiv;
  return a;
}

cr_status ensure_alcc(cr_handle* h, bool allow_loop) {
  AlccBufs& b = h->alcc;
  if (b.dev) return CR_OK;
  const int64_t P = h->N * (h->n + 1);
  b.blocks = primal_blocks(h->N);
  g_alloc_stream = h->st;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = dalloc(&b.dev, 1);
  if (e == cudaSuccess) e = dalloc(&b.p1, (size_t)P);
  if (e == cudaSuccess) e = dalloc(&b.p1p, (size_t)P);
  if (e == cudaSuccess) e = dalloc(&b.p2, (size_t)P);
  if (e == cudaSuccess) e = dalloc(&b.part1, (size_t)2 * b.blocks);
  if (e == cudaSuccess) e = dalloc(&b.part2, (size_t)2 * b.blocks);
  if (e == cudaSuccess) e = dalloc(&b.counter, 1);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(h, CR_ENOMEM, std::string("alcc allocation failed: ") + cudaGetErrorString(e));
  }
  CUDA_TRY(cudaMallocHost(&b.host, sizeof(AlccDev)));
  std::memset(b.host, 0, sizeof(AlccDev));
  CUDA_TRY(cudaMemsetAsync(b.counter, 0, sizeof(unsigned int), h->st));
  const int pen = kModePenalty, upd = kModePenaltyUpdate;
  b.kpen = sweep_mma_info((int)h->n, pen);
  b.kupd = sweep_mma_info((int)h->n, upd);
  if (!b.kpen.fn || !b.kupd.fn || b.kpen.max_blocks_per_sm < 1 || b.kupd.max_blocks_per_sm < 1)
    return fail(h, CR_EINVAL, "alcc: no penalty sweep kernel for this n");
  // small sub-problems: one cooperative launch per MAPG call (CRB_ALCC_LOOP=0 disables)
  const char* env = std::getenv("CRB_ALCC_LOOP");
  const bool want = allow_loop && h->N <= 2048 && !(env && env[0] == '0');
  if (want) {
    const void* fn = kLoopFns[h->n - 1];
    int bps = 0, sms = 148;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, kLBlock, 0) != cudaSuccess) bps = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    const long long S = (h->N + 31) / 32;
    long long P = std::max<long long>(1, (h->N + 31) / 32);
    long long G = (S * P + 7) / 8;
    const long long Gmax = (long long)bps * sms;
    if (Gmax >= 1) {
      if (G > Gmax) {
        G = Gmax;
        P = std::max<long long>(1, G * 8 / S);
        G = std::min<long long>(Gmax, (S * P + 7) / 8);
      }
      cudaError_t e2 = cudaSuccess;
      if (e2 == cudaSuccess) e2 = dalloc(&b.lcolpart, (size_t)(h->N * (h->n + 1) * P));
      if (e2 == cudaSuccess) e2 = dalloc(&b.lrowpart, (size_t)(h->N * S));
      if (e2 == cudaSuccess) e2 = dalloc(&b.lpartB, (size_t)(3 * G));
      if (e2 == cudaSuccess) e2 = dalloc(&b.lpartC, (size_t)(2 * G));
      if (e2 != cudaSuccess) {
        cudaGetLastError();
        return fail(h, CR_ENOMEM, "alcc: loop buffers");
      }
      b.loop_G = (int)G;
      b.loop_S = (int)S;
      b.loop_P = (int)P;
    }
  }
  return CR_OK;
}

// one MAPG iteration (4 launches)
cr_status enqueue_mapg(cr_handle* h, const AlccFns& f, const AlccArgs& aa, double cdiv) {
  SweepArgs sa = penalty_sweep_args(h, cdiv);
  sa.stopped = &h->alcc.dev->halt;
  CUDA_TRY((cudaError_t)launch_sweep(h->alcc.kpen, sa, h->st));
  const ReduceArgs ra = reduce_args(h, false, &h->alcc.dev->halt, false);
  CUDA_TRY(launch_reduce(ra, h->st));
  CUDA_TRY(launch_alcc(f.grad, h->alcc.blocks, kPBlock, aa, h->st));
  CUDA_TRY(launch_alcc(f.step, h->alcc.blocks, kPBlock, aa, h->st));
  return CR_OK;
}

cr_status build_mapg_graph(cr_handle* h, const AlccFns& f, const AlccArgs& aa, int iters) {
  AlccBufs& b = h->alcc;
  if (b.gexec) {
    cudaGraphExecDestroy(b.gexec);
    b.gexec = nullptr;
  }
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
  cr_status s = CR_OK;
  for (int i = 0; i < iters && s == CR_OK; ++i) s = enqueue_mapg(h, f, aa, 1.0);
  cudaError_t e = cudaStreamEndCapture(h->st, &g);
  if (s != CR_OK) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  CUDA_TRY(e);
  e = cudaGraphInstantiate(&b.gexec, g, 0);
  cudaGraphDestroy(g);
  CUDA_TRY(e);
  b.graph_iters = iters;
  return CR_OK;
}

cr_status push_dev(cr_handle* h) {
  CUDA_TRY(cudaMemcpyAsync(h->alcc.dev, h->alcc.host, sizeof(AlccDev), cudaMemcpyHostToDevice,
                           h->st));
  return CR_OK;
}
cr_status pull_dev(cr_handle* h) {
  CUDA_TRY(cudaMemcpyAsync(h->alcc.host, h->alcc.dev, sizeof(AlccDev), cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

// penalty (or update) sweep over y1 + reduce + stats block; leaves stats in host mirror
cr_status outer_stats(cr_handle* h, const AlccFns& f, const AlccArgs& aa, bool update,
                      double cdiv) {
  CUDA_TRY(launch_alcc(f.records, h->alcc.blocks, kPBlock, aa, h->st));
  SweepArgs sa = penalty_sweep_args(h, cdiv);
  CUDA_TRY((cudaError_t)launch_sweep(update ? h->alcc.kupd : h->alcc.kpen, sa, h->st));
  const ReduceArgs ra = reduce_args(h, false, nullptr, false);
  CUDA_TRY(launch_reduce(ra, h->st));
  CUDA_TRY(launch_alcc(f.stats, 1, kSBlock, aa, h->st));
  return pull_dev(h);
}

}  // namespace

// sub-problem handles of a partition run concurrently: the per-launch path
// (a cooperative launch would serialise them)
cr_status alcc_prepare(cr_handle* h) { return ensure_alcc(h, false); }

void alcc_release(cr_handle* h) {
  AlccBufs& b = h->alcc;
  if (b.gexec) cudaGraphExecDestroy(b.gexec);
  for (double* p : {b.p1, b.p1p, b.p2, b.part1, b.part2, b.lcolpart, b.lrowpart, b.lpartB,
                    b.lpartC})
    dfree(p, h->st);
  dfree(b.counter, h->st);
  dfree(b.dev, h->st);
  if (b.host) {
    if (h->st) cudaStreamSynchronize(h->st);
    cudaFreeHost(b.host);
  }
  b = AlccBufs{};
}
}  // namespace crb

extern "C" {

cr_status cr_sigma_A(cr_handle* h, int32_t which, double tol, int32_t max_iters, double* sigma,
                     int32_t* iters, int32_t* converged) {
  if (!h || !sigma || !iters || !converged || max_iters < 1 || (which != 1 && which != 2))
    return CR_EINVAL;
  CUDA_TRY(cudaSetDevice(h->device));
  const int64_t cols = which == 1 ? h->N : h->N * h->n;
  // fixed seeded start (operators.cpp:309-313)
  std::vector<double> v((size_t)cols);
  host::normal_stream(0x5eedULL, 97, cols, v.data());
  double ss = 0;
  for (double x : v) ss += x * x;
  const double nv = std::sqrt(ss);
  for (double& x : v) x /= nv;
  CUDA_TRY(cudaMemcpyAsync(h->pw_u, v.data(), sizeof(double) * cols, cudaMemcpyHostToDevice,
                           h->st));
  PowerLoopArgs pa{};
  pa.u = h->pw_u;
  pa.v = h->pw_v;
  pa.X = h->X;
  pa.gram = h->gram;
  pa.part = h->ps_part;
  pa.part2 = h->ps_part2;
  pa.state = h->ps_state;
  pa.N = h->N;
  pa.n = (int)h->n;
  pa.max_iters = max_iters;
  pa.tol = tol;
  pa.op = which;
  CUDA_TRY(launch_power_loop(pa, h->power_grid, h->st));
  double st[3];
  CUDA_TRY(cudaMemcpyAsync(st, h->ps_state, sizeof(st), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  *sigma = st[0];
  *iters = (int32_t)st[1];
  *converged = (int32_t)st[2];
  return CR_OK;
}

}  // extern "C"

namespace crb {
// alcc_core (alcc.cpp:54-191) on this handle's row set, starting from the point
// already in alcc.p1. target > 0: block stop rule (alcc.cpp:153-155) and the
// block radius from the feasible slice (alcc.cpp:238-243); else the standalone
// thresholds with cfg's radii. The point stays in alcc.p1.
cr_status alcc_run(cr_handle* h, const cr_alcc_config* cfg, double sA1, double sA2,
                   double target, bool block_mode, cr_snapshot* history, int64_t* mapg_iters,
                   cr_alcc_result* res) {
  const auto t_start = std::chrono::steady_clock::now();
  auto seconds = [&]() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  };
  h->begun = false;  // the dual buffers now hold ALCC multipliers
  AlccBufs& b = h->alcc;
  b.done = false;
  const int64_t N = h->N, n = h->n;
  const double gamma = h->gamma;
  const AlccFns& f = kFns[n - 1];
  const AlccArgs aa = alcc_args(h);
  // theta_1 = 0 in slot 0
  const size_t vbytes = sizeof(double) * (size_t)h->R * (size_t)h->ld;
  CUDA_TRY(cudaMemsetAsync(h->V[0], 0, vbytes, h->st));
  CUDA_TRY(cudaMemsetAsync(h->V[1], 0, vbytes, h->st));
  AlccDev& d = *b.host;
  std::memset(&d, 0, sizeof(d));
  d.cur = 0;
  d.mu = cfg->mu1;
  d.gamma = gamma;
  d.Bbar_y = cfg->Bbar_y;
  d.Bbar_xi = cfg->Bbar_xi;
  d.halt = 1;
  {
    const cr_status s = push_dev(h);
    if (s != CR_OK) return s;
  }
  if (block_mode) {
    CUDA_TRY(launch_alcc(f.bounds, 1, kSBlock, aa, h->st));
    const cr_status s = pull_dev(h);
    if (s != CR_OK) return s;
  }
  const double By = d.Bbar_y, Bx = d.Bbar_xi;
  CUDA_TRY(launch_alcc(f.project, 1, kSBlock, aa, h->st));
  double mapg_ms = 0;
  int64_t launches = 0;

  // P_1 at the start point (alcc.cpp:75-84); the update sweep supplies S_vv and
  // writes v / c into the unused slot (overwritten by the first outer step)
  double mu = cfg->mu1;
  double tau, alpha_y, alpha_xi;
  {
    const cr_status s = outer_stats(h, f, aa, true, cfg->c);
    if (s != CR_OK) return s;
    const double p1 = d.stats[0] / (2.0 * mu) + gamma * d.stats[1] / (2.0 * mu) + 0.5 * d.stats[5];
    if (!std::isfinite(p1)) return fail(h, CR_ENONFINITE, "alcc: non-finite P_1 at the start point");
    tau = std::max(cfg->tau1_scale * p1, 1e-16);
    alpha_y = alpha_xi = cfg->alpha1_scale * (By + Bx);
  }
  const int GI = 16;
  if (b.loop_G == 0 && (!b.gexec || b.graph_iters != GI)) {
    const cr_status s = build_mapg_graph(h, f, aa, GI);
    if (s != CR_OK) return s;
  }

  res->reason = CR_ITER_BUDGET;
  const double m = (double)N * (double)(N - 1);
  for (int64_t k = 1; k <= cfg->max_outer; ++k) {
    const double L_y = 1.0 / mu + sA1 * sA1;  // alcc.cpp:101-102
    const double L_xi = gamma / mu + sA2 * sA2;
    const double lmax_real = 4.0 * std::sqrt((L_y * By * By + L_xi * Bx * Bx) / tau);
    int64_t lmax = (int64_t)std::ceil(lmax_real);
    if (lmax < 10) lmax = 10;
    if (lmax > cfg->mapg_cap) lmax = cfg->mapg_cap;
    d.ell = 0;
    d.lmax = lmax;
    d.halt = 0;
    d.hit_cap = 0;
    d.nonfinite = 0;
    d.t = 1.0;
    d.mu = mu;
    d.L_y = L_y;
    d.L_xi = L_xi;
    d.alpha_y = alpha_y;
    d.alpha_xi = alpha_xi;
    {
      const cr_status s = push_dev(h);
      if (s != CR_OK) return s;
    }
    CUDA_TRY(cudaEventRecord(h->ev_start, h->st));
    CUDA_TRY(launch_alcc(f.reset, b.blocks, kPBlock, aa, h->st));
    launches += 1;
    if (b.loop_G > 0) {  // the whole MAPG call in one cooperative launch
      LoopArgs la{};
      la.a = aa;
      la.V0 = h->V[0];
      la.V1 = h->V[1];
      la.colpart = b.lcolpart;
      la.rowpart = b.lrowpart;
      la.partB = b.lpartB;
      la.partC = b.lpartC;
      la.ld = h->ld;
      la.S = b.loop_S;
      la.P = b.loop_P;
      void* args[] = {&la};
      CUDA_TRY(cudaLaunchCooperativeKernel(kLoopFns[n - 1], dim3((unsigned)b.loop_G),
                                           dim3(kLBlock), args, 0, h->st));
      launches += 1;
      CUDA_TRY(cudaEventRecord(h->ev_end, h->st));
      const cr_status s = pull_dev(h);
      if (s != CR_OK) return s;
    } else {
      for (;;) {
        CUDA_TRY(cudaGraphLaunch(b.gexec, h->st));
        launches += 4 * (int64_t)b.graph_iters;
        CUDA_TRY(cudaEventRecord(h->ev_end, h->st));
        const cr_status s = pull_dev(h);
        if (s != CR_OK) return s;
        if (d.halt) break;
      }
    }
    {
      float ms = 0;
      CUDA_TRY(cudaEventElapsedTime(&ms, h->ev_start, h->ev_end));
      mapg_ms += ms;
    }
    if (d.nonfinite) {
      res->reason = CR_ERROR;
      return fail(h, CR_ENONFINITE, "mapg: non-finite gradient");
    }
    if (mapg_iters) mapg_iters[k - 1] = d.ell;
    res->mapg_iters_total += d.ell;
    if (d.hit_cap) res->hit_cap_any = 1;

    // outer statistics at y1 and theta_{k+1} = v / c into the other slot
    {
      const cr_status s = outer_stats(h, f, aa, true, cfg->c);
      if (s != CR_OK) return s;
    }
    const double sq_y = d.stats[0], sq_xi = d.stats[1];
    const double infeas_raw = std::sqrt(d.stats[7]);
    const double gap_raw = mu * d.stats[6];
    const double mu2 = mu * mu;
    const double dual_value = -0.5 * (mu2 * d.stats[2]) - (mu2 * d.stats[3]) / (2.0 * gamma) -
                              mu * d.stats[4];
    const double primal_value = 0.5 * sq_y + 0.5 * gamma * sq_xi;
    const double certified = primal_value - dual_value;
    res->certified_gap = certified;
    res->infeas_raw = infeas_raw;
    res->gap_raw = gap_raw;
    res->outer_iters = k;
    res->objective = 0.5 * sq_y;
    b.mu = mu;
    b.done = true;
    const double infeas_norm = m > 0 ? infeas_raw / std::sqrt(m) : 0.0;
    const double gap_norm = m > 0 ? gap_raw / m : 0.0;
    if (history) {
      cr_snapshot& sn = history[k - 1];
      sn.iter = (double)k;
      sn.objective = 0.5 * sq_y;
      sn.reg_objective = primal_value;
      sn.infeas_raw = infeas_raw;
      sn.infeas_norm = infeas_norm;
      sn.gap_raw = gap_raw;
      sn.gap_norm = gap_norm;
      sn.wall_time_s = seconds();
    }
    bool stop;
    if (target > 0)  // alcc.cpp:153-155, |lambda| = mu |v|
      stop = certified <= target && (mu * std::sqrt(d.stats[5])) * infeas_raw <= target;
    else
      stop = infeas_norm <= cfg->infeas_norm_tol && std::fabs(gap_norm) <= cfg->gap_norm_tol;
    if (stop) {
      res->reason = CR_THRESHOLDS;
      break;
    }
    if (seconds() > cfg->max_seconds) {
      res->reason = CR_TIME_BUDGET;
      break;
    }
    // alcc.cpp:176-183: theta_{k+1} is already in the other slot
    d.cur = 1 - d.cur;
    mu *= cfg->c;
    const double decay = std::pow(cfg->c * std::pow((double)k, 1.0 + cfg->kappa), 2.0);
    tau /= decay;
    alpha_y /= decay;
    alpha_xi /= decay;
  }
  // the multiplier export reads theta_k of the last outer step: undo a final flip
  if (res->outer_iters > 0 && res->reason == CR_ITER_BUDGET) d.cur = 1 - d.cur;
  {
    const cr_status s = push_dev(h);
    if (s != CR_OK) return s;
  }
  if (res->outer_iters == 0) {  // max_outer = 0: the projected start point
    const cr_status s = outer_stats(h, f, aa, false, cfg->c);
    if (s != CR_OK) return s;
    res->objective = 0.5 * d.stats[0];
  }
  res->mapg_seconds += mapg_ms * 1e-3;
  res->launches += launches;
  res->wall_seconds += seconds();
  return CR_OK;
}
}  // namespace crb

extern "C" {

cr_status cr_alcc_solve(cr_handle* h, const cr_alcc_config* cfg, const double* warm_y,
                        const double* warm_xi, double* y_out, double* xi_out,
                        cr_snapshot* history, int64_t* mapg_iters, cr_alcc_result* res) {
  if (!h || !cfg || !warm_y || !warm_xi || !res) return CR_EINVAL;
  if (!(cfg->c > 1)) return fail(h, CR_EINVAL, "alcc: c must be > 1");          // alcc.cpp:59
  if (!(cfg->kappa > 0)) return fail(h, CR_EINVAL, "alcc: kappa must be > 0");  // :60
  if (!(cfg->mu1 > 0)) return fail(h, CR_EINVAL, "alcc: mu1 must be > 0");      // :61
  if (cfg->max_outer < 0 || cfg->mapg_cap < 1)
    return fail(h, CR_EINVAL, "alcc: bad iteration limits");
  if (h->comm != nullptr || h->R != h->N)
    return fail(h, CR_EINVAL, "alcc: standalone ALCC runs on an unsharded handle");
  CUDA_TRY(cudaSetDevice(h->device));
  const auto t_start = std::chrono::steady_clock::now();
  {
    const cr_status s = ensure_alcc(h, true);
    if (s != CR_OK) return s;
  }
  AlccBufs& b = h->alcc;
  b.cy = nullptr;  // standalone centres (ybar, 0)
  b.cxi = nullptr;
  const int64_t N = h->N, n = h->n, Nn = N * n;
  std::memset(res, 0, sizeof(*res));
  double sA1 = cfg->sigma_A1, sA2 = cfg->sigma_A2;
  if (!(sA1 > 0)) {
    int32_t it = 0, cv = 0;
    const cr_status s = cr_sigma_A(h, 1, 1e-6, 5000, &sA1, &it, &cv);
    if (s != CR_OK) return s;
    res->sigma_A1_iters = it;
  }
  if (!(sA2 > 0)) {
    int32_t it = 0, cv = 0;
    const cr_status s = cr_sigma_A(h, 2, 1e-6, 5000, &sA2, &it, &cv);
    if (s != CR_OK) return s;
    res->sigma_A2_iters = it;
  }
  res->sigma_A1 = sA1;
  res->sigma_A2 = sA2;
  res->sigma_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  CUDA_TRY(cudaMemcpyAsync(b.p1, warm_y, sizeof(double) * N, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(b.p1 + N, warm_xi, sizeof(double) * Nn, cudaMemcpyHostToDevice, h->st));
  {
    const cr_status s = alcc_run(h, cfg, sA1, sA2, 0.0, false, history, mapg_iters, res);
    if (s != CR_OK) return s;
  }
  if (y_out) CUDA_TRY(cudaMemcpyAsync(y_out, b.p1, sizeof(double) * N, cudaMemcpyDeviceToHost, h->st));
  if (xi_out)
    CUDA_TRY(cudaMemcpyAsync(xi_out, b.p1 + N, sizeof(double) * Nn, cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  res->wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return CR_OK;
}

cr_status cr_time_penalty_sweep(cr_handle* h, int32_t k, double* avg_seconds) {
  if (!h || k < 1 || !avg_seconds) return CR_EINVAL;
  if (!h->alcc.done) return fail(h, CR_ESTATE, "alcc: no finished solve on this handle");
  CUDA_TRY(cudaSetDevice(h->device));
  const SweepArgs sa = penalty_sweep_args(h, 1.0);  // read-only on theta
  CUDA_TRY(cudaEventRecord(h->ev_start, h->st));
  for (int i = 0; i < k; ++i) CUDA_TRY((cudaError_t)launch_sweep(h->alcc.kpen, sa, h->st));
  CUDA_TRY(cudaEventRecord(h->ev_end, h->st));
  CUDA_TRY(cudaEventSynchronize(h->ev_end));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, h->ev_start, h->ev_end));
  *avg_seconds = ms * 1e-3 / k;
  return CR_OK;
}

cr_status cr_alcc_multiplier(cr_handle* h, int64_t row_begin, int64_t row_end, double* out) {
  if (!h || !out || row_begin < 0 || row_end > h->N || row_begin > row_end) return CR_EINVAL;
  if (!h->alcc.done) return fail(h, CR_ESTATE, "alcc: no finished solve on this handle");
  CUDA_TRY(cudaSetDevice(h->device));
  const int64_t N = h->N;
  const double* V = h->V[h->alcc.host->cur];
  const int64_t per = std::max<int64_t>(1, h->stage_elems / (N - 1));
  for (int64_t ra = row_begin; ra < row_end; ra += per) {
    const int64_t rb = std::min(row_end, ra + per);
    const long long total = (rb - ra) * (N - 1);
    long long g = (total + 255) / 256;
    if (g > 4096) g = 4096;
    if (g < 1) g = 1;
    multiplier_out_kernel<<<(unsigned)g, 256, 0, h->st>>>(h->stage, V, h->alcc.mu, h->rowrec,
                                                          h->colrec, N, (int)h->n, h->ld, ra, rb);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out + (ra - row_begin) * (N - 1), h->stage,
                             sizeof(double) * (size_t)total, cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  return CR_OK;
}

}  // extern "C"
