// iteration.cuh -- device logic shared by the per-kernel iteration
// (kernels.cu) and the persistent small-N iteration (small.cu): the primal
// closed form of one point (K2), the papg.cpp control step (Kc) and a
// deterministic block reduction.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "device.cuh"
#include "kernels.cuh"

namespace crb {
namespace {

constexpr int kBlock = 256;
constexpr int kPBlock = 64;  // O(N) kernels: small blocks so N = 1e4 still spans every SM

// deterministic block reduction of W values per thread: warp butterflies, then
// the warps' sums in warp order (threads < W write out[w]; callers that read
// out from other threads synchronise first)
template <int W, int BS = kBlock>
__device__ void block_reduce_store(double (&v)[W], double* out /* W values */) {
  constexpr int NW = BS / 32;
  __shared__ double sh[NW][W];
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
  if ((int)threadIdx.x < W) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < NW; ++k) t += sh[k][threadIdx.x];
    out[threadIdx.x] = t;
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// theta2 (or theta1) combination of the two unscaled buffers
__device__ __forceinline__ double combine(double zc, double zp, double s_c, double s_p,
                                          double beta) {
  const double th1 = s_c * zc;
  const double th1p = s_p * zp;
  return fma(beta, th1 - th1p, th1);
}

// One point of K2 (see primal_kernel): primal closed form at theta2 (mode 0)
// or theta1 (mode 1) from the aggregates of the two dual buffers.
template <int NN>
__device__ __forceinline__ void primal_point(const PrimalArgs& a, long long l, double s_c,
                                             double s_p, double beta, const double* vposc,
                                             double* vposp, double (&acc)[kK2Scal]) {
  constexpr int RP = rec_pitch(NN);
  const long long N = a.N;
  const double* rowsum_c = a.aggc;
  const double* colagg_c = a.aggc + N;
  double* rowsum_p = a.aggp;
  double* colagg_p = a.aggp + N;
  const double* x = a.X + l * NN;
  const double* ac = colagg_c + l * (NN + 1);
  double* ap = colagg_p + l * (NN + 1);
  double agc[NN + 1], agp[NN + 1], xv[NN];
#pragma unroll
  for (int j = 0; j <= NN; ++j) {
    agc[j] = ac[j];
    agp[j] = a.mode == 0 ? ap[j] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < NN; ++j) xv[j] = x[j];
  const double rsc = rowsum_c[l];
  const double rsp = a.mode == 0 ? rowsum_p[l] : 0.0;
  const double vpc = vposc[l];
  const double vpp = a.mode == 0 ? vposp[l] : 0.0;
  const double ybar = a.ybar[l];
  if (a.mode == 0) {  // aggregates of V[cur] become those of V[prev] next iteration
    rowsum_p[l] = rsc;
#pragma unroll
    for (int j = 0; j <= NN; ++j) ap[j] = agc[j];
  }
  const double rs = combine(rsc, rsp, s_c, s_p, beta);
  const double cs = combine(agc[0], agp[0], s_c, s_p, beta);
  const double th2pos = combine(vpc, vpp, s_c, s_p, beta);
  const double qy = th2pos + rs - cs;  // operators.cpp:161-172
  const double y = ybar + qy;          // alcc.cpp:234
  double cx = 0.0, xx = 0.0, qx = 0.0;
  double xi[NN];
#pragma unroll
  for (int j = 0; j < NN; ++j) {
    const double vx = combine(agc[1 + j], agp[1 + j], s_c, s_p, beta);
    const double qxi = cs * xv[j] - vx;  // operators.cpp:173-175 summed over l1
    xi[j] = qxi / a.gamma;               // alcc.cpp:235
    cx = fma(xi[j], xv[j], cx);
    xx = fma(xi[j], xi[j], xx);
    qx = fma(qxi, xi[j], qx);
  }
  const double dy = y - ybar;
  if (a.mode == 0) {
    double* crec = a.colrec + l * RP;  // (-xi, -c, 1)
#pragma unroll
    for (int j = 0; j < NN; ++j) crec[j] = -xi[j];
    crec[NN] = -(y - cx);
    crec[NN + 1] = 1.0;
    a.rowrec[l * RP + NN + 1] = y;     // (x, 1, y)
    // y >= 0 rows of C: theta1_pos = max(theta2_pos - y / L, 0) (papg.cpp:188-189)
    const double vnew = fmax(fma(-y, a.invL, th2pos), 0.0);
    vposp[l] = vnew;
    acc[0] = fma(vnew, vnew, acc[0]);
    acc[1] = fma(vnew, y, acc[1]);
    // theta2 . C eta (papg.cpp:191-199): C^T theta2 = (q_y, q_xi) by linearity, so
    // summed over the points the cross pairs' theta2 . row is y (rs - cs) + xi . q_xi
    acc[2] = a.tr_adjoint ? acc[2] + fma(y, qy, qx) : fma(th2pos, y, acc[2]);
  } else {
    a.yout[l] = y;
#pragma unroll
    for (int j = 0; j < NN; ++j) a.xiout[l * NN + j] = xi[j];
  }
  const double m = fmin(y, 0.0);
  acc[3] = fma(m, m, acc[3]);
  // block objective at the closed-form minimiser (alcc.cpp:254-256)
  acc[4] += 0.5 * (dy * dy) + 0.5 * a.gamma * xx - qy * y - qx;
  acc[5] = fma(dy, dy, acc[5]);
  acc[6] += xx;
  acc[7] += isfinite(y) && isfinite(cx) ? 0.0 : 1.0;
}

__device__ __forceinline__ double momentum_next(double t) {  // engines.hpp:11-13
  return 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
}

// Kc: papg.cpp:187-262 on the reduced scalars. One thread.
// wall_in >= 0: the elapsed seconds to test the time budget against (sharded
// runs: one clock for all ranks); < 0: this GPU's own clock
__device__ __forceinline__ void control_logic(DevCtrl* c, const double* scal, const double* k2,
                                              double* hist, double wall_in) {
  const long long ell = c->ell + 1;
  const double S_vv = scal[0] + k2[0];
  const double S_vr = scal[1] + k2[1];
  const double S_tr = scal[2] + k2[2];
  const double S_nn_cross = scal[3];
  const double S_nn_all = scal[3] + k2[3];
  const double g_value = k2[4];
  const double B = c->B_theta;

  // projection scale (projections.hpp:10-12)
  const double norm = sqrt(S_vv);
  const double s_new = norm > B ? B / norm : 1.0;
  // linearisation bound (papg.cpp:191-199)
  const double cross_infeas = sqrt(S_nn_cross);
  const double fw = B * sqrt(S_nn_all) + S_tr;
  const double inv3 = 1.0 / ((double)ell * (double)ell * (double)ell);
  const double inner_tol = fmin(c->inner_tol_floor, inv3);
  const double cushion = 2.0 * inner_tol * c->K;
  c->g_star_upper = fmin(c->g_star_upper, g_value + fw + cushion);
  // gap / infeasibility (papg.cpp:201-208)
  const double gap_raw = c->use_momentum ? s_new * S_vr : S_tr;
  const double within = c->within_raw;  // 0 for singleton blocks
  const double infeas_raw = sqrt(within * within + cross_infeas * cross_infeas);
  const double gap_norm = gap_raw / c->gap_div;
  const double infeas_norm = infeas_raw / c->infeas_div;
  const double wall = wall_in >= 0.0 ? wall_in : (double)(globaltimer() - c->t_start_ns) * 1e-9;
  c->gap_raw = gap_raw;
  c->gap_norm = gap_norm;
  c->infeas_raw = infeas_raw;
  c->infeas_norm = infeas_norm;
  c->g_value = g_value;
  c->fw = fw;
  c->objective = 0.5 * k2[5];
  c->reg_objective = 0.5 * k2[5] + 0.5 * c->gamma * k2[6];
  if (c->record_history && hist != nullptr && ell <= c->hist_cap) {  // papg.cpp:210-222
    double* h = hist + (ell - 1) * 8;
    h[0] = (double)ell;
    h[1] = c->objective;
    h[2] = c->reg_objective;
    h[3] = infeas_raw;
    h[4] = infeas_norm;
    h[5] = gap_raw;
    h[6] = gap_norm;
    h[7] = wall;
  }
  c->ell = ell;
  // theta1 = s_new * V[new]; the new buffer becomes "cur"
  c->s_prev = c->s_cur;
  c->s_cur = s_new;
  c->cur = 1 - c->cur;
  c->theta1_norm = s_new * norm;

  if (!isfinite(S_tr) || !isfinite(S_vv) || k2[7] != 0.0) {  // papg.cpp:184-185
    c->reason = 3;
    c->stopped = 1;
    return;
  }
  bool stop = false;  // papg.cpp:225-236
  if (fabs(gap_norm) <= c->gap_tol && infeas_norm <= c->infeas_tol) {
    c->reason = 0;
    stop = true;
  } else if (ell >= c->max_iters) {
    c->reason = 1;
    stop = true;
  } else if (wall > c->max_seconds) {
    c->reason = 2;
    stop = true;
  }
  if (stop) {  // papg.cpp:238-254
    const bool saturated = c->theta1_norm > 0.99 * B;
    if (saturated && c->adaptive && c->reason == 0 && c->restarts < c->max_restarts) {
      c->B_theta = B * 2.0;
      c->restarts += 1;
      c->t = 1.0;
      c->beta = 0.0;  // theta2 = theta1
      c->g_star_upper = INFINITY;
      return;
    }
    c->saturated = saturated ? 1 : 0;
    c->stopped = 1;
    return;
  }
  if (c->use_momentum) {  // papg.cpp:256-262
    const double t_next = momentum_next(c->t);
    c->beta = (c->t - 1.0) / t_next;
    c->t = t_next;
  } else {
    c->beta = 0.0;
  }
}


// The state block is copied to registers, updated and written back: one round
// trip to memory instead of a chain of dependent field accesses.
__device__ __noinline__ void control_step(DevCtrl* cg, const double* scal_g, const double* k2_g,
                                          double* hist, double wall_in = -1.0) {
  DevCtrl c = *cg;
  double scal[kScal], k2[kK2Scal];
#pragma unroll
  for (int w = 0; w < kScal; ++w) scal[w] = scal_g[w];
#pragma unroll
  for (int w = 0; w < kK2Scal; ++w) k2[w] = k2_g[w];
  control_logic(&c, scal, k2, hist, wall_in);
  c.halt = (c.stopped || c.ell >= c.pause_at) ? 1 : 0;
  *cg = c;
}

}  // namespace
}  // namespace crb
