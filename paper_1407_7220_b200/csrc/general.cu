// general.cu -- P-APG(ALCC) with K blocks of nbar points:
// the reference's default solver (papg.cpp:136-283 with DualDecomposition::
// dual_gradient :89-132 and alcc_solve_block, alcc.cpp:222-258).
//
// The cross-block pair matrix is the singleton path's N x N dual store with
// same-block pairs held at 0 like the diagonal (SweepArgs::nbar masks them in
// the sweep). One dual iteration:
//   Kc   centres: q = C^T theta2 from the two aggregate buffers (operators.cpp:
//        155-180) and the block centres c_y = ybar + q_y, c_xi = q_xi / gamma
//        (alcc.cpp:233-235)
//   ALCC one sub-problem handle per block runs alcc_core on the within-block
//        rows from its warm start (the previous block minimiser, papg.cpp:121-122)
//        with target_subopt = min(floor, 1/l^3) -> eta
//   Ke   eta finish: records of eta for the sweep, the y >= 0 rows of the
//        projected step, block objectives (alcc.cpp:254-256) and metric terms
//   K1   cross sweep (masked) + fixed-order reduce + device control step
// The block sub-problems are the dominant cost (thousands of MAPG sweeps per
// dual iteration); their sweeps use the same pair kernels on nbar x nbar.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "balcc.cuh"
#include "handle.cuh"
#include "iteration.cuh"

namespace crb {
cr_status alcc_run(cr_handle* h, const cr_alcc_config* cfg, double sA1, double sA2,
                   double target, bool block_mode, cr_snapshot* history, int64_t* mapg_iters,
                   cr_alcc_result* res);
cr_status alcc_prepare(cr_handle* h);  // alcc.cu: buffers of a sub-problem handle

namespace {

struct GenArgs {
  const double* X;
  const double* ybar;
  const double* aggc;  // aggregates of V[cur]
  double* aggp;        // aggregates of V[prev]; mode 0 refreshes them with aggc
  double* vpos0;
  double* vpos1;
  const int* cur;
  const double* coef;  // {s_cur, s_prev, beta}
  double *cy, *cxi, *qy, *qxi, *th2pos;
  const double *ey, *exi;
  double *rowrec, *colrec, *k2part, *yout, *xiout;
  double invL, gamma;
  long long N;
  int n;
  int mode;            // 0 iteration (theta2), 1 final re-solve (theta1)
};

// Kc: papg.cpp:99 (apply_C_T at theta2) and the block centres
template <int NN>
__global__ void __launch_bounds__(kPBlock) centres_kernel(const GenArgs a) {
  const long long N = a.N;
  const double s_c = a.coef[0];
  const double s_p = a.mode == 0 ? a.coef[1] : 0.0;
  const double beta = a.mode == 0 ? a.coef[2] : 0.0;
  const int cur = *a.cur;
  const double* vposc = cur ? a.vpos1 : a.vpos0;
  const double* vposp = cur ? a.vpos0 : a.vpos1;
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock) {
    const double* ac = a.aggc + N + l * (NN + 1);
    double* ap = a.aggp + N + l * (NN + 1);
    double agc[NN + 1], agp[NN + 1];
#pragma unroll
    for (int j = 0; j <= NN; ++j) {
      agc[j] = ac[j];
      agp[j] = a.mode == 0 ? ap[j] : 0.0;
    }
    const double rsc = a.aggc[l];
    const double rsp = a.mode == 0 ? a.aggp[l] : 0.0;
    const double vpc = vposc[l];
    const double vpp = a.mode == 0 ? vposp[l] : 0.0;
    if (a.mode == 0) {  // aggregates of V[cur] become those of V[prev] next iteration
      a.aggp[l] = rsc;
#pragma unroll
      for (int j = 0; j <= NN; ++j) ap[j] = agc[j];
    }
    const double rs = combine(rsc, rsp, s_c, s_p, beta);
    const double cs = combine(agc[0], agp[0], s_c, s_p, beta);
    const double th2pos = combine(vpc, vpp, s_c, s_p, beta);
    const double qy = th2pos + rs - cs;  // operators.cpp:161-172
    a.qy[l] = qy;
    a.th2pos[l] = th2pos;
    a.cy[l] = a.ybar[l] + qy;            // alcc.cpp:234
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      const double vx = combine(agc[1 + j], agp[1 + j], s_c, s_p, beta);
      const double qxi = cs * a.X[l * NN + j] - vx;  // operators.cpp:173-175
      a.qxi[l * NN + j] = qxi;
      a.cxi[l * NN + j] = qxi / a.gamma;            // alcc.cpp:235
    }
  }
}

// Ke: eta of the block solves -> records, pos-row step, k2 scalars (as K2)
template <int NN>
__global__ void __launch_bounds__(kPBlock) eta_finish_kernel(const GenArgs a) {
  constexpr int RP = rec_pitch(NN);
  const long long N = a.N;
  const int cur = *a.cur;
  double* vposp = cur ? a.vpos0 : a.vpos1;
  double acc[kK2Scal];
#pragma unroll
  for (int w = 0; w < kK2Scal; ++w) acc[w] = 0.0;
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock) {
    const double y = a.ey[l];
    const double qy = a.qy[l];
    double cx = 0.0, xx = 0.0, qx = 0.0;
    double xi[NN];
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      xi[j] = a.exi[l * NN + j];
      cx = fma(xi[j], a.X[l * NN + j], cx);
      xx = fma(xi[j], xi[j], xx);
      qx = fma(a.qxi[l * NN + j], xi[j], qx);
    }
    const double dy = y - a.ybar[l];
    if (a.mode == 0) {
      double* crec = a.colrec + l * RP;  // (-xi, -c, 1)
#pragma unroll
      for (int j = 0; j < NN; ++j) crec[j] = -xi[j];
      crec[NN] = -(y - cx);
      crec[NN + 1] = 1.0;
      a.rowrec[l * RP + NN + 1] = y;
      const double th2pos = a.th2pos[l];
      const double vnew = fmax(fma(-y, a.invL, th2pos), 0.0);  // papg.cpp:188-189
      vposp[l] = vnew;
      acc[0] = fma(vnew, vnew, acc[0]);
      acc[1] = fma(vnew, y, acc[1]);
      acc[2] = fma(th2pos, y, acc[2]);
    } else {
      a.yout[l] = y;
#pragma unroll
      for (int j = 0; j < NN; ++j) a.xiout[l * NN + j] = xi[j];
    }
    const double m = fmin(y, 0.0);
    acc[3] = fma(m, m, acc[3]);
    acc[4] += 0.5 * (dy * dy) + 0.5 * a.gamma * xx - qy * y - qx;  // alcc.cpp:254-256
    acc[5] = fma(dy, dy, acc[5]);
    acc[6] += xx;
    acc[7] += isfinite(y) && isfinite(cx) ? 0.0 : 1.0;
  }
  block_reduce_store<kK2Scal, kPBlock>(acc, a.k2part + (long long)blockIdx.x * kK2Scal);
}

// canonical cross position (indexing.hpp:30-37) -> (l1, l2)
__device__ __forceinline__ void cross_pair(long long idx, long long K, long long nbar,
                                           long long* l1, long long* l2) {
  const long long nb2 = nbar * nbar;
  const long long pr = idx / nb2, local = idx % nb2;
  const long long i = pr / (K - 1), jj = pr % (K - 1);
  const long long j = jj + (jj >= i ? 1 : 0);
  *l1 = i * nbar + local / nbar;
  *l2 = j * nbar + local % nbar;
}

__global__ void theta_k_out_kernel(double* stage, const double* V, double s, long long K,
                                   long long nbar, long long ld, long long a, long long b) {
  for (long long i = a + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < b;
       i += (long long)gridDim.x * blockDim.x) {
    long long l1, l2;
    cross_pair(i, K, nbar, &l1, &l2);
    stage[i - a] = s * V[l1 * ld + l2];
  }
}

__global__ void theta_k_in_kernel(const double* stage, double* V, long long K, long long nbar,
                                  long long ld, long long a, long long b) {
  for (long long i = a + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < b;
       i += (long long)gridDim.x * blockDim.x) {
    long long l1, l2;
    cross_pair(i, K, nbar, &l1, &l2);
    const double t = stage[i - a];
    V[l1 * ld + l2] = t > 0.0 ? t : 0.0;  // projections.hpp:10 (scale applied separately)
  }
}

__global__ void rows_k_out_kernel(double* stage, const double* rowrec, const double* colrec,
                                  int n, long long K, long long nbar, long long a, long long b) {
  const int RP = rec_pitch(n);
  for (long long i = a + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < b;
       i += (long long)gridDim.x * blockDim.x) {
    long long l1, l2;
    cross_pair(i, K, nbar, &l1, &l2);
    const double* xr = rowrec + l1 * RP;
    const double* cr = colrec + l2 * RP;
    double row = xr[n + 1] + cr[n];
    for (int j = 0; j < n; ++j) row = fma(xr[j], cr[j], row);
    stage[i - a] = row;
  }
}

using GenKernel = void (*)(const GenArgs);
template <int NN>
struct GenTab {
  static constexpr GenKernel centres = centres_kernel<NN>;
  static constexpr GenKernel finish = eta_finish_kernel<NN>;
};
struct GenFns {
  GenKernel centres, finish;
};
template <int NN>
constexpr GenFns gen_for() {
  return {GenTab<NN>::centres, GenTab<NN>::finish};
}
constexpr GenFns kGen[kMaxN] = {
#define CRB_GEN_FOR(N) gen_for<N>()
    CRB_N_SEQ(CRB_GEN_FOR)
#undef CRB_GEN_FOR
};

GenArgs gen_args(cr_handle* h, int mode) {
  Partition& P = h->part;
  GenArgs a{};
  a.X = h->X;
  a.ybar = h->ybar;
  a.aggc = h->xbuf;
  a.aggp = h->aggsave;
  a.vpos0 = h->vpos[0];
  a.vpos1 = h->vpos[1];
  a.cur = &h->ctrl_d->cur;
  a.coef = &h->ctrl_d->s_cur;
  a.cy = P.cy;
  a.cxi = P.cxi;
  a.qy = P.qy;
  a.qxi = P.qxi;
  a.th2pos = P.th2pos;
  a.ey = P.ey;
  a.exi = P.exi;
  a.rowrec = h->rowrec;
  a.colrec = h->colrec;
  a.k2part = h->k2part;
  a.yout = h->yout;
  a.xiout = h->xiout;
  a.invL = 1.0 / h->L;
  a.gamma = h->gamma;
  a.N = h->N;
  a.n = (int)h->n;
  a.mode = mode;
  return a;
}

cudaError_t launch_gen(GenKernel k, const GenArgs& a, cudaStream_t s) {
  void* args[] = {const_cast<GenArgs*>(&a)};
  return cudaLaunchKernel((const void*)k, dim3((unsigned)primal_blocks(a.N)), dim3(kPBlock), args,
                          0, s);
}

unsigned grid_of(long long count) {
  long long g = (count + 255) / 256;
  return (unsigned)std::max<long long>(1, std::min<long long>(g, 4096));
}

// DualDecomposition::dual_gradient's block loop (papg.cpp:107-130): every block
// from its warm start, eta gathered in block order, within infeasibility
cr_status solve_blocks_batched(cr_handle* h, double tol, double* within) {
  Partition& P = h->part;
  const auto t0 = std::chrono::steady_clock::now();
  BalccArgs a{};
  a.X = h->X;
  a.cy = P.cy;
  a.cxi = P.cxi;
  a.fy = P.fy;
  a.fxi = P.fxi;
  a.ey = P.ey;
  a.exi = P.exi;
  a.sigma_A2 = P.d_sigma_A2;
  a.sigma_A1 = P.sigma_A1;
  a.gamma = h->gamma;
  a.target = tol;
  a.cfg = P.inner;
  a.theta = P.w_theta;
  a.y1p = P.w_y1p;
  a.y2 = P.w_y2;
  a.x1p = P.w_x1p;
  a.x2 = P.w_x2;
  a.cc = P.w_cc;
  a.rs = P.w_rs;
  a.cs = P.w_cs;
  a.vx = P.w_vx;
  a.scratch = P.w_scratch;
  a.scratch_per_block = balcc_scratch_per_block(P.nbar, (int)h->n);
  a.infeas = P.w_infeas;
  a.iters = P.w_iters;
  a.status = P.w_status;
  a.nbar = P.nbar;
  a.K = (int)P.K;
  CUDA_TRY(launch_balcc(a, (int)h->n, h->st));
  std::vector<double> inf((size_t)P.K);
  std::vector<long long> its((size_t)P.K);
  std::vector<int> sts((size_t)P.K);
  CUDA_TRY(cudaMemcpyAsync(inf.data(), P.w_infeas, sizeof(double) * P.K, cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaMemcpyAsync(its.data(), P.w_iters, sizeof(long long) * P.K,
                           cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaMemcpyAsync(sts.data(), P.w_status, sizeof(int) * P.K, cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  double sq = 0;
  for (int64_t b = 0; b < P.K; ++b) {  // gathered in block order (papg.cpp:124-128)
    if (sts[(size_t)b] != 0)
      return fail(h, CR_ENONFINITE, "block " + std::to_string(b) + ": mapg: non-finite gradient");
    P.block_infeas[(size_t)b] = inf[(size_t)b];
    sq += inf[(size_t)b] * inf[(size_t)b];
    P.inner_iters += its[(size_t)b];
  }
  P.inner_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *within = std::sqrt(sq);
  return CR_OK;
}

cr_status solve_blocks(cr_handle* h, double tol, double* within) {
  Partition& P = h->part;
  if (P.batched) return solve_blocks_batched(h, tol, within);
  CUDA_TRY(cudaStreamSynchronize(h->st));  // centres ready
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t nb = P.nbar, n = h->n;
  std::vector<cr_status> st((size_t)P.K, CR_OK);
  std::vector<cr_alcc_result> rs((size_t)P.K);
  // one block solve per worker on its own handle/stream (parallel_blocks,
  // papg.cpp:29-58): independent tasks writing their own slots
  auto task = [&](int64_t b) {
    cr_handle* hb = P.blocks[(size_t)b];
    cr_alcc_result& r = rs[(size_t)b];
    std::memset(&r, 0, sizeof(r));
    cudaSetDevice(hb->device);
    cr_status s = alcc_run(hb, &P.inner, P.sigma_A1, P.sigma_A2[(size_t)b], tol, true, nullptr,
                           nullptr, &r);
    if (s == CR_OK) {
      cudaError_t e = cudaMemcpyAsync(P.ey + b * nb, hb->alcc.p1, sizeof(double) * nb,
                                      cudaMemcpyDeviceToDevice, hb->st);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(P.exi + b * nb * n, hb->alcc.p1 + nb, sizeof(double) * nb * n,
                            cudaMemcpyDeviceToDevice, hb->st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(hb->st);
      if (e != cudaSuccess) s = fail(hb, CR_ECUDA, cudaGetErrorString(e));
    }
    st[(size_t)b] = s;
  };
  const int64_t workers = std::min<int64_t>(P.K, P.workers > 0 ? P.workers : 16);
  if (workers <= 1) {
    for (int64_t b = 0; b < P.K; ++b) task(b);
  } else {
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    for (int64_t w = 0; w < workers; ++w)
      pool.emplace_back([&]() {
        for (int64_t b; (b = next.fetch_add(1)) < P.K;) task(b);
      });
    for (auto& t : pool) t.join();
  }
  double sq = 0;
  for (int64_t b = 0; b < P.K; ++b) {  // gathered in block order (papg.cpp:124-128)
    if (st[(size_t)b] != CR_OK)
      return fail(h, st[(size_t)b], "block " + std::to_string(b) + ": " + P.blocks[(size_t)b]->err);
    const cr_alcc_result& r = rs[(size_t)b];
    P.block_infeas[(size_t)b] = r.infeas_raw;
    sq += r.infeas_raw * r.infeas_raw;
    P.inner_iters += r.mapg_iters_total;
  }
  P.inner_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *within = std::sqrt(sq);
  return CR_OK;
}

// the dual sweeps of a partitioned handle mask same-block pairs (blocked
// instantiations); released handles return to the singleton kernels
cr_status select_sweeps(cr_handle* h, bool blocked) {
  const int n = (int)h->n;
  SweepKernelInfo kp, kw;
  kp = sweep_mma_info(n, kModePapg, blocked);
  kw = sweep_mma_info(n, kModePower, blocked);
  if (!kp.fn || !kw.fn || kp.max_blocks_per_sm < 1 || kp.tile_cols != h->kp.tile_cols)
    return fail(h, CR_EINVAL, "partition: no blocked sweep kernel for this n");
  h->kp = kp;
  h->kw = kw;
  return CR_OK;
}

cr_status pull_ctrl(cr_handle* h) {
  CUDA_TRY(cudaMemcpyAsync(h->ctrl_h, h->ctrl_d, sizeof(DevCtrl), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

}  // namespace

// ---- entry points used by capi.cu ------------------------------------------

// papg.cpp:66-86: fresh warm starts (the feasible slices) for a new solve
cr_status general_begin(cr_handle* h) {
  Partition& P = h->part;
  const int64_t nb = P.nbar, n = h->n;
  if (P.batched) {  // the block minimisers live in ey / exi (warm starts in place)
    CUDA_TRY(cudaMemcpyAsync(P.ey, P.fy, sizeof(double) * h->N, cudaMemcpyDeviceToDevice, h->st));
    CUDA_TRY(cudaMemcpyAsync(P.exi, P.fxi, sizeof(double) * h->N * n, cudaMemcpyDeviceToDevice,
                             h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  for (int64_t b = 0; b < P.K; ++b) {
    cr_handle* hb = P.blocks[(size_t)b];
    CUDA_TRY(cudaMemcpyAsync(hb->alcc.p1, P.fy + b * nb, sizeof(double) * nb,
                             cudaMemcpyDeviceToDevice, hb->st));
    CUDA_TRY(cudaMemcpyAsync(hb->alcc.p1 + nb, P.fxi + b * nb * n, sizeof(double) * nb * n,
                             cudaMemcpyDeviceToDevice, hb->st));
    CUDA_TRY(cudaStreamSynchronize(hb->st));
  }
  P.inner_iters = 0;
  P.inner_seconds = 0;
  return CR_OK;
}

// one dual iteration per pass, up to max_steps (papg.cpp:176-263)
cr_status general_iterate(cr_handle* h, int64_t max_steps, int64_t* done, int32_t* stopped,
                          double* sweep_seconds, int64_t* launches) {
  const GenFns& f = kGen[h->n - 1];
  cr_status s = pull_ctrl(h);
  if (s != CR_OK) return s;
  double sw = 0;
  int64_t nl = 0;
  for (int64_t i = 0; i < max_steps && !h->ctrl_h->stopped; ++i) {
    const double ell = (double)(h->ctrl_h->ell + 1);
    const double tol = std::min(h->cfg.inner_tol_floor, 1.0 / (ell * ell * ell));  // :179-182
    CUDA_TRY(launch_gen(f.centres, gen_args(h, 0), h->st));
    double within = 0;
    s = solve_blocks(h, tol, &within);
    if (s != CR_OK) return s;
    CUDA_TRY(cudaMemcpyAsync(&h->ctrl_d->within_raw, &within, sizeof(double),
                             cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(launch_gen(f.finish, gen_args(h, 0), h->st));
    const SweepArgs sa = sweep_args(h, kModePapg, false);
    CUDA_TRY(cudaEventRecord(h->ev_start, h->st));
    CUDA_TRY((cudaError_t)launch_sweep(papg_sweep(h), sa, h->st));
    CUDA_TRY(cudaEventRecord(h->ev_end, h->st));
    const ReduceArgs ra =
        reduce_args(h, true, &h->ctrl_d->halt, true, papg_sweep(h).scal_recs);
    CUDA_TRY(launch_reduce(ra, h->st));
    s = pull_ctrl(h);
    if (s != CR_OK) return s;
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, h->ev_start, h->ev_end));
    sw += ms * 1e-3;
    nl += 4;
  }
  if (done) *done = h->ctrl_h->ell;
  if (stopped) *stopped = h->ctrl_h->stopped;
  if (sweep_seconds) *sweep_seconds = sw;
  if (launches) *launches = nl;
  if (h->ctrl_h->stopped && h->ctrl_h->reason == 3)
    return fail(h, CR_ENONFINITE, "papg: non-finite dual gradient");
  return CR_OK;
}

// final re-solve at theta1 (papg.cpp:265-277): eta into yout/xiout, k2 into k2sum
cr_status general_final(cr_handle* h, double final_tol) {
  const GenFns& f = kGen[h->n - 1];
  CUDA_TRY(launch_gen(f.centres, gen_args(h, 1), h->st));
  double within = 0;
  const cr_status s = solve_blocks(h, final_tol, &within);
  if (s != CR_OK) return s;
  CUDA_TRY(launch_gen(f.finish, gen_args(h, 1), h->st));
  CUDA_TRY(launch_reduce_records(h->k2part, h->k2_blocks, kK2Scal, h->k2sum, h->st));
  return CR_OK;
}

// theta1 / C eta / warm theta0 in the canonical general-K order
cr_status general_get_theta(cr_handle* h, double* out) {
  const Partition& P = h->part;
  const int cur = h->ctrl_h->cur;
  const double sc = h->ctrl_h->s_cur;
  const long long cross = h->N * (h->N - P.nbar);
  for (long long a = 0; a < cross; a += h->stage_elems) {
    const long long b = std::min<long long>(cross, a + h->stage_elems);
    theta_k_out_kernel<<<grid_of(b - a), 256, 0, h->st>>>(
        h->stage, h->V[cur], sc, P.K, P.nbar, h->ld, a, b);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out + a, h->stage, sizeof(double) * (b - a), cudaMemcpyDeviceToHost,
                             h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  CUDA_TRY(launch_scale_copy(h->stage, h->vpos[cur], sc, h->N, h->st));
  CUDA_TRY(cudaMemcpyAsync(out + cross, h->stage, sizeof(double) * h->N, cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

cr_status general_get_rows(cr_handle* h, double* out) {
  const Partition& P = h->part;
  const long long cross = h->N * (h->N - P.nbar);
  for (long long a = 0; a < cross; a += h->stage_elems) {
    const long long b = std::min<long long>(cross, a + h->stage_elems);
    rows_k_out_kernel<<<grid_of(b - a), 256, 0, h->st>>>(h->stage, h->rowrec, h->colrec,
                                                        (int)h->n, P.K, P.nbar, a, b);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out + a, h->stage, sizeof(double) * (b - a), cudaMemcpyDeviceToHost,
                             h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  std::vector<double> rec((size_t)h->N * h->RP);
  CUDA_TRY(cudaMemcpy(rec.data(), h->rowrec, sizeof(double) * rec.size(), cudaMemcpyDeviceToHost));
  for (int64_t l = 0; l < h->N; ++l) out[cross + l] = rec[(size_t)l * h->RP + h->n + 1];
  return CR_OK;
}

cr_status general_theta_in(cr_handle* h, const double* theta0) {
  const Partition& P = h->part;
  const long long cross = h->N * (h->N - P.nbar);
  for (long long a = 0; a < cross; a += h->stage_elems) {
    const long long b = std::min<long long>(cross, a + h->stage_elems);
    CUDA_TRY(cudaMemcpyAsync(h->stage, theta0 + a, sizeof(double) * (b - a),
                             cudaMemcpyHostToDevice, h->st));
    theta_k_in_kernel<<<grid_of(b - a), 256, 0, h->st>>>(h->stage, h->V[0], P.K, P.nbar, h->ld,
                                                        a, b);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  return CR_OK;
}

void general_release(cr_handle* h) {
  Partition& P = h->part;
  if (P.K > 0) select_sweeps(h, false);
  for (cr_handle* hb : P.blocks) cr_destroy(hb);
  P.blocks.clear();
  for (double* b : {P.cy, P.cxi, P.qy, P.qxi, P.th2pos, P.ey, P.exi, P.fy, P.fxi, P.w_theta,
                    P.w_y1p, P.w_y2, P.w_x1p, P.w_x2, P.w_cc, P.w_rs, P.w_cs, P.w_vx,
                    P.w_infeas, P.d_sigma_A2, P.w_scratch})
    dfree(b, h->st);
  dfree(P.w_iters, h->st);
  dfree(P.w_status, h->st);
  P = Partition{};
}

}  // namespace crb

extern "C" {

cr_status cr_set_partition(cr_handle* h, int64_t K, const double* feas_y, const double* feas_xi,
                           const cr_alcc_config* inner) {
  if (!h) return CR_EINVAL;
  CUDA_TRY(cudaSetDevice(h->device));
  h->begun = false;
  if (h->part.K > 0) general_release(h);
  if (K == h->N || K == 0) return CR_OK;  // singleton blocks: the closed-form path
  if (!feas_y || !feas_xi || !inner) return CR_EINVAL;
  if (K < 1 || h->N % K != 0)
    return fail(h, CR_EINVAL, "partition: N = " + std::to_string(h->N) +
                                  " not divisible by K = " + std::to_string(K));
  const int64_t nbar = h->N / K, n = h->n, N = h->N;
  if (nbar < n + 1) return fail(h, CR_EINVAL, "partition: block size must be >= n+1");
  if (!(inner->c > 1) || !(inner->kappa > 0) || !(inner->mu1 > 0) || inner->max_outer < 0 ||
      inner->mapg_cap < 1)
    return fail(h, CR_EINVAL, "partition: bad inner ALCC config");
  if (h->comm != nullptr || h->R != h->N)
    return fail(h, CR_EINVAL, "partition: general K runs on an unsharded handle");
  Partition& P = h->part;
  {
    const cr_status s = select_sweeps(h, true);
    if (s != CR_OK) return s;
  }
  P.K = K;
  P.nbar = nbar;
  P.inner = *inner;
  g_alloc_stream = h->st;
  cudaError_t e = cudaSuccess;
  for (double** b : {&P.cy, &P.qy, &P.th2pos, &P.ey, &P.fy})
    if (e == cudaSuccess) e = dalloc(b, (size_t)N);
  for (double** b : {&P.cxi, &P.qxi, &P.exi, &P.fxi})
    if (e == cudaSuccess) e = dalloc(b, (size_t)(N * n));
  if (e != cudaSuccess) {
    cudaGetLastError();
    general_release(h);
    return fail(h, CR_ENOMEM, "partition buffers");
  }
  CUDA_TRY(cudaMemcpyAsync(P.fy, feas_y, sizeof(double) * N, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(P.fxi, feas_xi, sizeof(double) * N * n, cudaMemcpyHostToDevice, h->st));
  std::vector<double> X((size_t)(N * n)), yb((size_t)N);
  CUDA_TRY(cudaMemcpyAsync(X.data(), h->X, sizeof(double) * N * n, cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaMemcpyAsync(yb.data(), h->ybar, sizeof(double) * N, cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  P.sigma_A2.assign((size_t)K, 0.0);
  P.block_infeas.assign((size_t)K, 0.0);
  for (int64_t b = 0; b < K; ++b) {
    cr_handle* hb = nullptr;
    cr_status s = cr_create(X.data() + b * nbar * n, yb.data() + b * nbar, nbar, n, h->gamma,
                            h->device, 0, nbar, &hb);
    if (s != CR_OK) {
      const std::string why = hb ? hb->err : "cr_create";
      if (hb) cr_destroy(hb);
      general_release(h);
      return fail(h, s, "partition: block handle: " + why);
    }
    P.blocks.push_back(hb);
    s = alcc_prepare(hb);
    if (s != CR_OK) {
      general_release(h);
      return fail(h, s, "partition: block buffers");
    }
    hb->alcc.cy = P.cy + b * nbar;
    hb->alcc.cxi = P.cxi + b * nbar * n;
    hb->alcc.fy = P.fy + b * nbar;
    hb->alcc.fxi = P.fxi + b * nbar * n;
    // estimate_block_sigmas (alcc.cpp:206-220): A1 of block 0 serves every block
    int32_t it = 0, cv = 0;
    if (b == 0) {
      s = cr_sigma_A(hb, 1, 1e-6, 5000, &P.sigma_A1, &it, &cv);
      if (s != CR_OK) return fail(h, s, "partition: sigma(A1)");
    }
    s = cr_sigma_A(hb, 2, 1e-6, 5000, &P.sigma_A2[(size_t)b], &it, &cv);
    if (s != CR_OK) return fail(h, s, "partition: sigma(A2)");
  }
  // small blocks: every block ALCC in one launch (balcc.cu); CRB_BALCC=0 disables
  const char* env = std::getenv("CRB_BALCC");
  if (nbar <= balcc_max_block() && !(env && env[0] == '0')) {
    g_alloc_stream = h->st;
    cudaError_t e2 = cudaSuccess;
    for (double** b : {&P.w_y1p, &P.w_y2, &P.w_cc, &P.w_rs, &P.w_cs})
      if (e2 == cudaSuccess) e2 = dalloc(b, (size_t)N);
    for (double** b : {&P.w_x1p, &P.w_x2, &P.w_vx})
      if (e2 == cudaSuccess) e2 = dalloc(b, (size_t)(N * n));
    if (e2 == cudaSuccess) e2 = dalloc(&P.w_theta, (size_t)(N * nbar));
    if (e2 == cudaSuccess)
      e2 = dalloc(&P.w_scratch, (size_t)(K * balcc_scratch_per_block(nbar, (int)n)));
    if (e2 == cudaSuccess) e2 = dalloc(&P.w_infeas, (size_t)K);
    if (e2 == cudaSuccess) e2 = dalloc(&P.d_sigma_A2, (size_t)K);
    if (e2 == cudaSuccess) e2 = dalloc(&P.w_iters, (size_t)K);
    if (e2 == cudaSuccess) e2 = dalloc(&P.w_status, (size_t)K);
    if (e2 != cudaSuccess) {
      cudaGetLastError();
      general_release(h);
      return fail(h, CR_ENOMEM, "partition: batched block workspaces");
    }
    CUDA_TRY(cudaMemcpyAsync(P.d_sigma_A2, P.sigma_A2.data(), sizeof(double) * K,
                             cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
    P.batched = true;
  }
  return CR_OK;
}

cr_status cr_partition_stats(const cr_handle* h, int64_t* inner_iters, double* inner_seconds,
                             double* sigma_A1, double* sigma_A2 /* K */) {
  if (!h) return CR_EINVAL;
  const Partition& P = h->part;
  if (inner_iters) *inner_iters = P.inner_iters;
  if (inner_seconds) *inner_seconds = P.inner_seconds;
  if (sigma_A1) *sigma_A1 = P.sigma_A1;
  if (sigma_A2)
    for (size_t b = 0; b < P.sigma_A2.size(); ++b) sigma_A2[b] = P.sigma_A2[b];
  return CR_OK;
}

}  // extern "C"
