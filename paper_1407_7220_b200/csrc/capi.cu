// capi.cu -- the C ABI (include/cvxreg_b200.h): handle lifetime, device
// buffers, the device-resident dual loop (CUDA graphs or direct launches),
// the power method for sigma_max(C), NCCL for row-sharded runs and the
// canonical-order import/export of the dual point.
//
// The host loop of the reference (papg.cpp:136-283) is split: the per-
// iteration scalar logic runs on the device (control_kernel), so the host
// only enqueues work and polls a halt flag once per batch of iterations.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <chrono>
#include <mutex>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cvxreg_b200.h"
#include "device.cuh"
#include "host.hpp"
#include "kernels.cuh"
#include "small.cuh"
#include "handle.cuh"

using namespace crb;

cudaStream_t g_alloc_stream = nullptr;

// Process-wide pool of the handles' small pinned host blocks (control-state
// mirrors): cudaMallocHost costs ~0.4 ms per call, three per handle, which a
// service creating one handle per solve would pay every time.
namespace {
std::mutex g_pin_mu;
std::vector<std::pair<size_t, void*>> g_pin_free;
}  // namespace
static cudaError_t pinned_get(void** p, size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (size_t i = 0; i < g_pin_free.size(); ++i)
      if (g_pin_free[i].first == bytes) {
        *p = g_pin_free[i].second;
        g_pin_free.erase(g_pin_free.begin() + (long)i);
        return cudaSuccess;
      }
  }
  return cudaMallocHost(p, bytes);
}
static void pinned_put(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.emplace_back(bytes, p);
}

// The uniform pairs of the sigma_max(C) start vector (rng_stream(0x5eed, 97)), drawn into
// a pinned block of the process pool (a pageable upload of the 2 N (n+1) doubles cost
// ~0.3 ms at config 2), or into the handle's vector when no pinned memory is to be had.
static void draw_sigma_start(cr_handle* h) {
  const int64_t cols = h->N * (h->n + 1);
  const size_t bytes = sizeof(double) * (size_t)(2 * cols);
  if (h->sigma_start_pin == nullptr || h->sigma_start_bytes != bytes) {
    pinned_put(h->sigma_start_pin, h->sigma_start_bytes);
    h->sigma_start_pin = nullptr;
    h->sigma_start_bytes = 0;
    void* p = nullptr;
    if (cudaSetDevice(h->device) == cudaSuccess && pinned_get(&p, bytes) == cudaSuccess) {
      h->sigma_start_pin = (double*)p;
      h->sigma_start_bytes = bytes;
    } else {
      cudaGetLastError();
    }
  }
  if (h->sigma_start_pin) {
    h->sigma_start_ptr = h->sigma_start_pin;
  } else {
    h->sigma_start.resize((size_t)(2 * cols));
    h->sigma_start_ptr = h->sigma_start.data();
  }
  host::uniform_pairs(0x5eedULL, 97, cols, h->sigma_start_ptr);
  h->sigma_start_cols = cols;
}

namespace crb {

// 2-D tensor maps of the dual buffers for the DMMA P-APG producer: dims
// {ld, R}, box {tile + 2, 8} (one stage, the 2 extra columns fill the
// shared-memory pitch padding). Encoded once per handle through the driver
// entry point (cudart is linked statically; no -lcuda). CRB_TMAP=0 keeps the
// per-row bulk copies.
// Tensor maps of rows [row_off, row_off + rows) of both dual buffers.
static bool encode_tmap_pair(cr_handle* h, int64_t row_off, int64_t rows, TmapBytes out[2]) {
  const char* env = std::getenv("CRB_TMAP");
  if ((env && env[0] == '0') || h->variant != kSweepMma || rows <= 0) return false;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  // 3-D view {TC, T, R} of the R x ld buffer (element (x, t, r) at r ld + t TC + x):
  // x in [TC, TC + 2) is out of bounds, so the pitch-padding columns of a stage are
  // zero-filled by the TMA unit instead of read from HBM. Columns >= ld of the
  // last tile alias the next row (never consumed: those warps are inactive); the
  // buffers carry TC doubles of slack for the last row's.
  const cuuint64_t TC = (cuuint64_t)h->kp.tile_cols;
  if (TC + 2 > 256 || h->T > INT_MAX || rows > INT_MAX) return false;
  static_assert(sizeof(TmapBytes) == sizeof(CUtensorMap), "tensor map size");
  for (int b = 0; b < 2; ++b) {
    const cuuint64_t dims[3] = {TC, (cuuint64_t)h->T, (cuuint64_t)rows};
    const cuuint64_t strides[2] = {TC * sizeof(double), (cuuint64_t)h->ld * sizeof(double)};
    const cuuint32_t box[3] = {(cuuint32_t)TC + 2, 1, 8};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, h->V[b] + row_off * h->ld,
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      if (std::getenv("CRB_DEBUG")) std::fprintf(stderr, "cvxreg_b200: tensor map encode failed (%d)\n", (int)r);
      return false;
    }
    std::memcpy(&out[b], &m, sizeof(m));
  }
  return true;
}
static void encode_sweep_tmaps(cr_handle* h) { h->tmap_ok = encode_tmap_pair(h, 0, h->R, h->tmV); }
  // general.cu: P-APG(ALCC) with K blocks
cr_status general_begin(cr_handle* h);
cr_status general_iterate(cr_handle* h, int64_t max_steps, int64_t* done, int32_t* stopped,
                          double* sweep_seconds, int64_t* launches);
cr_status general_final(cr_handle* h, double final_tol);
cr_status general_get_theta(cr_handle* h, double* out);
cr_status general_get_rows(cr_handle* h, double* out);
cr_status general_theta_in(cr_handle* h, const double* theta0);
void general_release(cr_handle* h);
void alcc_release(cr_handle* h);
}  // namespace crb

namespace {

PrimalArgs primal_args(cr_handle* h, int mode) {
  PrimalArgs a{};
  a.X = h->X;
  a.ybar = h->ybar;
  a.rowrec = h->rowrec;
  a.colrec = h->colrec;
  a.aggc = h->xbuf;
  a.aggp = h->aggsave;
  a.vpos0 = h->vpos[0];
  a.vpos1 = h->vpos[1];
  a.cur = &h->ctrl_d->cur;
  a.k2part = h->k2part;
  a.coef = &h->ctrl_d->s_cur;
  a.stopped = mode == 0 ? &h->ctrl_d->halt : nullptr;
  a.yout = h->yout;
  a.xiout = h->xiout;
  a.invL = 1.0 / h->L;
  a.gamma = h->cfg.gamma;
  a.N = h->N;
  a.n = (int)h->n;
  a.mode = mode;
  a.tr_adjoint = h->part.K == 0 ? 1 : 0;  // singleton per-kernel sweep: theta2 . C eta from K2
  return a;
}

void release_canon(cr_handle* h) {
  for (CanonBlock& b : h->canon) {
    dfree(b.colpart, h->st);
    dfree(b.rowpart, h->st);
    dfree(b.scalpart, h->st);
  }
  h->canon.clear();
  dfree(h->canon_pay, h->st);
  h->canon_pay = nullptr;
  h->canon_D = 0;
  h->canon_first = 0;
}

// canonical-block views of the sweep / reduce arguments
SweepArgs sweep_args_block(cr_handle* h, const CanonBlock& b, int mode, bool agg_only) {
  SweepArgs a = sweep_args(h, mode, agg_only);
  a.V0 = h->V[0] + b.a * h->ld;
  a.V1 = h->V[1] + b.a * h->ld;
  a.colpart = b.colpart;
  a.rowpart = b.rowpart;
  a.scalpart = b.scalpart;
  a.R = b.R;
  a.r0 = h->r0 + b.a;
  a.G = b.G;
  a.U = b.U;
  a.maxspan = b.maxspan;
  a.tmap = 0;
  if (b.tmap_ok) {
    a.tmV[0] = b.tmV[0];
    a.tmV[1] = b.tmV[1];
    a.tmap = 1;
  }
  return a;
}

ReduceArgs reduce_args_block(cr_handle* h, const CanonBlock& b, int index, bool with_k2,
                             const int* stopped) {
  ReduceArgs a = reduce_args(h, with_k2, stopped, false, papg_sweep(h).scal_recs);
  a.colpart = b.colpart;
  a.rowpart = b.rowpart;
  a.scalpart = b.scalpart;
  a.agg_out = h->canon_pay + (size_t)(h->canon_first + index) * (size_t)payload_len(h);
  a.rank = 0;  // a halted solve keeps every block payload (the combine is idempotent)
  a.R = b.R;
  a.r0 = h->r0 + b.a;
  a.nw = (long long)b.G * papg_sweep(h).scal_recs;
  a.G = b.G;
  a.U = b.U;
  a.maxspan = b.maxspan;
  return a;
}

// sweeps + reduces of the local canonical blocks, then (use_nccl) the allgather of
// the block payloads; the combine is left to the caller's finish phase
cr_status enqueue_canon_local(cr_handle* h, bool agg_only, const int* stopped, bool with_k2,
                              cudaEvent_t ev_a, cudaEvent_t ev_b, bool use_nccl,
                              cudaEvent_t ev_c, cudaEvent_t ev_d) {
  if (ev_a) CUDA_TRY(cudaEventRecord(ev_a, h->st));
  for (const CanonBlock& b : h->canon) {
    const SweepArgs sa = sweep_args_block(h, b, kModePapg, agg_only);
    CUDA_TRY((cudaError_t)launch_sweep(papg_sweep(h), sa, h->st));
  }
  if (ev_b) CUDA_TRY(cudaEventRecord(ev_b, h->st));
  for (size_t i = 0; i < h->canon.size(); ++i) {
    const ReduceArgs ra = reduce_args_block(h, h->canon[i], (int)i, with_k2 && i == 0, stopped);
    CUDA_TRY(launch_reduce(ra, h->st));
  }
  if (use_nccl && h->comm) {
    const size_t count = h->canon.size() * (size_t)payload_len(h);
    if (ev_c) CUDA_TRY(cudaEventRecord(ev_c, h->st));
    NCCL_TRY(ncclAllGather(h->canon_pay + (size_t)h->canon_first * (size_t)payload_len(h),
                           h->canon_pay, count, ncclDouble, h->comm, h->st));
    if (ev_d) CUDA_TRY(cudaEventRecord(ev_d, h->st));
  }
  return CR_OK;
}

cr_status enqueue_canon_combine(cr_handle* h) {
  CUDA_TRY(launch_canon_combine(h->canon_pay, h->canon_D, payload_len(h), h->xbuf, h->st));
  return CR_OK;
}

// Enqueue one dual iteration (papg.cpp:176-263). phase: 0 = all,
// 1 = local part only (K2, K1, K3), 2 = finish only (control).

cr_status enqueue_iteration(cr_handle* h, int phase, cudaEvent_t ev_a, cudaEvent_t ev_b,
                            bool use_nccl, cudaEvent_t ev_c, cudaEvent_t ev_d) {
  if (!h->canon.empty()) {  // canonical row blocks: per-block launches, ordered combine
    if (phase != 2) {
      const PrimalArgs pa = primal_args(h, 0);
      CUDA_TRY(launch_primal(pa, h->st));
      const cr_status s = enqueue_canon_local(h, false, &h->ctrl_d->halt, true, ev_a, ev_b,
                                              use_nccl, ev_c, ev_d);
      if (s != CR_OK) return s;
    }
    if (phase != 1) {
      const cr_status s = enqueue_canon_combine(h);
      if (s != CR_OK) return s;
      CUDA_TRY(launch_control(h->ctrl_d, h->xbuf + h->N * (h->n + 2), h->k2sum, h->hist, h->st));
    }
    return CR_OK;
  }
  if (phase != 2) {
    const PrimalArgs pa = primal_args(h, 0);
    CUDA_TRY(launch_primal(pa, h->st));
    const SweepArgs sa = sweep_args(h, kModePapg, false);
    if (ev_a) CUDA_TRY(cudaEventRecord(ev_a, h->st));
    CUDA_TRY((cudaError_t)launch_sweep(papg_sweep(h), sa, h->st));
    if (ev_b) CUDA_TRY(cudaEventRecord(ev_b, h->st));
    // single GPU, full iteration: the reduce kernel's last block runs the control step
    const bool fuse = phase == 0 && h->comm == nullptr;
    const ReduceArgs ra =
        reduce_args(h, true, &h->ctrl_d->halt, fuse, papg_sweep(h).scal_recs);
    CUDA_TRY(launch_reduce(ra, h->st));
    if (use_nccl && h->comm) {
      if (ev_c) CUDA_TRY(cudaEventRecord(ev_c, h->st));
      NCCL_TRY(ncclAllReduce(h->xbuf, h->xbuf, (size_t)payload_len(h), ncclDouble, ncclSum,
                             h->comm, h->st));
      if (ev_d) CUDA_TRY(cudaEventRecord(ev_d, h->st));
    }
    if (fuse) return CR_OK;
  }
  if (phase != 1)
    CUDA_TRY(launch_control(h->ctrl_d, h->xbuf + h->N * (h->n + 2), h->k2sum, h->hist, h->st));
  return CR_OK;
}

// our kernels per iteration (the NCCL allreduce kernel is not counted)
int launches_per_iteration(const cr_handle* h) {
  if (!h->canon.empty()) return 3 + 2 * (int)h->canon.size();  // primal, sweeps, reduces, combine, control
  return h->comm ? 4 : 3;
}

cr_status build_graph(cr_handle* h) {
  if (h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
  cr_status s = CR_OK;
  h->primal_pending = true;  // each graph launch starts with the (no-op unless needed) primal
  for (int i = 0; i < h->graph_iters && s == CR_OK; ++i)
    s = enqueue_iteration(h, 0, nullptr, nullptr, true, nullptr, nullptr);
  cudaError_t e = cudaStreamEndCapture(h->st, &g);
  if (s != CR_OK) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  CUDA_TRY(e);
  e = cudaGraphInstantiate(&h->gexec, g, 0);
  cudaGraphDestroy(g);
  CUDA_TRY(e);
  return CR_OK;
}

cr_status sync_ctrl(cr_handle* h) {
  CUDA_TRY(cudaMemcpyAsync(h->ctrl_h, h->ctrl_d, sizeof(DevCtrl), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

// one power step (operators.cpp:318-327) through the pair sweep; returns lambda and |u|
cr_status power_step(cr_handle* h, double norm_u, double* lambda, double* nu) {
  PowerArgs pa{};
  pa.X = h->X;
  pa.u = h->pw_u;
  pa.v = h->pw_v;
  pa.norm_u = norm_u;
  pa.rowrec = h->rowrec;
  pa.colrec = h->colrec;
  pa.agg = h->xbuf;
  pa.part = h->pw_part;
  pa.N = h->N;
  pa.n = (int)h->n;
  CUDA_TRY(launch_power_prep(pa, h->st));
  SweepArgs sa = sweep_args(h, kModePower, false);
  sa.cur = h->izero;
  CUDA_TRY((cudaError_t)launch_sweep(h->kw, sa, h->st));
  const ReduceArgs ra = reduce_args(h, false, nullptr, false);
  CUDA_TRY(launch_reduce(ra, h->st));
  if (h->comm)
    NCCL_TRY(ncclAllReduce(h->xbuf, h->xbuf, (size_t)payload_len(h), ncclDouble, ncclSum, h->comm,
                           h->st));
  CUDA_TRY(launch_power_post(pa, h->st));
  CUDA_TRY(launch_reduce_records(h->pw_part, primal_blocks(h->N), 2, h->pw_sum, h->st));
  double host[3];
  CUDA_TRY(cudaMemcpyAsync(host, h->xbuf + h->N * (h->n + 2), sizeof(double),
                           cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaMemcpyAsync(host + 1, h->pw_sum, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  *lambda = host[0] + host[1];
  *nu = std::sqrt(host[2]);
  return CR_OK;
}

cr_status set_pause(cr_handle* h, long long pause_at) {
  h->pause_h[0] = pause_at;
  const int halt = (h->ctrl_h->stopped || h->ctrl_h->ell >= pause_at) ? 1 : 0;
  reinterpret_cast<int*>(h->pause_h + 1)[0] = halt;
  CUDA_TRY(cudaMemcpyAsync(&h->ctrl_d->pause_at, h->pause_h, sizeof(long long),
                           cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(&h->ctrl_d->halt, h->pause_h + 1, sizeof(int), cudaMemcpyHostToDevice,
                           h->st));
  return CR_OK;
}

}  // namespace

extern "C" {

const char* cr_status_string(cr_status s) {
  switch (s) {
    case CR_OK: return "ok";
    case CR_EINVAL: return "invalid argument";
    case CR_ENOMEM: return "out of memory";
    case CR_ECUDA: return "CUDA error";
    case CR_ENCCL: return "NCCL error";
    case CR_ENONFINITE: return "papg: non-finite dual gradient";
    case CR_ESTATE: return "call out of order";
  }
  return "unknown";
}

const char* cr_last_error(const cr_handle* h) { return h ? h->err.c_str() : "null handle"; }

int64_t cr_exchange_len(const cr_handle* h) {
  if (!h) return 0;
  return h->canon.empty() ? payload_len(h) : (int64_t)h->canon_D * payload_len(h);
}

cr_status cr_create(const double* Xh, const double* ybar_shifted, int64_t N, int64_t n,
                    double gamma, int device, int64_t row_begin, int64_t row_end,
                    cr_handle** out) {
  if (!out) return CR_EINVAL;
  *out = nullptr;
  if (!Xh || !ybar_shifted || N < 2 || n < 1 || !(gamma > 0) || row_begin < 0 ||
      row_end > N || row_begin >= row_end)
    return CR_EINVAL;
  if (n > kMaxN) return CR_EINVAL;
  cr_handle* h = new cr_handle();
  *out = h;
  h->device = device;
  h->N = N;
  h->n = n;
  h->r0 = row_begin;
  h->r1 = row_end;
  h->R = row_end - row_begin;
  h->RP = rec_pitch((int)n);
  h->gamma = gamma;
  h->cfg.gamma = gamma;
  const bool tdbg = std::getenv("CRB_DEBUG_CREATE") != nullptr;
  const auto tc0 = std::chrono::steady_clock::now();
  auto tmark = [&](const char* what) {
    if (tdbg)
      std::fprintf(stderr, "create %-12s %.3f ms\n", what,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count() * 1e3);
  };
  h->sigma_prep = std::thread([h] {  // overlaps the allocations and uploads below
    draw_sigma_start(h);  // beside the creation
  });
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
  tmark("stream");
  keep_pool_memory(device);
  g_alloc_stream = h->st;
  // the FP64 tensor-core (DMMA) pair sweep for every n
  h->variant = kSweepMma;
  h->kp = sweep_mma_info((int)n, kModePapg);
  h->kw = sweep_mma_info((int)n, kModePower);
  if (!h->kp.fn || !h->kw.fn || h->kp.max_blocks_per_sm < 1)
    return fail(h, CR_EINVAL, "no sweep kernel for this n");
  tmark("kernel info");
  const int W = h->kp.strip_cols;
  h->S = (int)((N + W - 1) / W);
  h->ld = (int64_t)h->S * W;
  int sms = 148;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  // one persistent wave; each CTA gets an equal contiguous share of the
  // T x R (tile, row) units, at least 64 rows
  h->T = (h->S + h->kp.warps_per_block - 1) / h->kp.warps_per_block;
  const long long units = (long long)h->T * h->R;
  long long G = (long long)sms * h->kp.max_blocks_per_sm;
  G = std::min<long long>(G, (units + 63) / 64);
  if (G < 1) G = 1;
  h->U = (units + G - 1) / G;
  h->G = (int)((units + h->U - 1) / h->U);
  h->maxspan = (int)((h->U - 1) / h->R + 2);
  h->k2_blocks = primal_blocks(N);

  const size_t RP = (size_t)h->RP;
  const size_t vlen = (size_t)h->R * (size_t)h->ld;
  cudaError_t e = cudaSuccess;
#define ALLOC(ptr, count)                                             \
  if (e == cudaSuccess) e = dalloc(&(ptr), (size_t)(count));
  ALLOC(h->X, N * n);
  ALLOC(h->ybar, N);
  ALLOC(h->rowrec, N * RP);
  ALLOC(h->colrec, N * RP);
  // + one column tile of slack: the tensor-map view of the last tile's row ends
  ALLOC(h->V[0], vlen + h->kp.tile_cols);
  ALLOC(h->V[1], vlen + h->kp.tile_cols);
  ALLOC(h->vpos[0], N);
  ALLOC(h->vpos[1], N);
  ALLOC(h->xbuf, payload_len(h));
  ALLOC(h->aggsave, payload_len(h));
  ALLOC(h->colpart, (size_t)h->G * h->maxspan * h->kp.tile_cols * (n + 1));
  ALLOC(h->rowpart, (size_t)h->T * h->R);
  ALLOC(h->scalpart, (size_t)h->G * h->kp.warps_per_block * kScal);
  // K2 records of the primal (k2_blocks)
  ALLOC(h->k2part, (size_t)h->k2_blocks * kK2Scal);
  ALLOC(h->k2sum, kK2Scal);
  ALLOC(h->yout, N);
  ALLOC(h->xiout, N * n);
  ALLOC(h->pw_u, N * (n + 1));
  ALLOC(h->pw_v, N * (n + 1));
  ALLOC(h->pw_part, (size_t)h->k2_blocks * 2);
  ALLOC(h->pw_sum, 2);
  h->power_grid = power_loop_grid(sms, N);
  if (const char* pg = std::getenv("CRB_POWER_GRID")) h->power_grid = std::max(1, std::atoi(pg));
  ALLOC(h->gram, n * n + n);
  // op-C power loop: two step-parity buffers of (4 + 2n)-value records
  ALLOC(h->ps_part, (size_t)h->power_grid * 2 * (4 + 2 * n));
  ALLOC(h->ps_part2, (size_t)h->power_grid * 2);
  ALLOC(h->ps_state, 4);
  ALLOC(h->consts, 4);
  ALLOC(h->izero, 1);
  ALLOC(h->counter, 1);
  ALLOC(h->d_stores, 1);
  ALLOC(h->ctrl_d, 1);
#undef ALLOC
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(h, CR_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e));
  }
  tmark("allocs");
  encode_sweep_tmaps(h);
  tmark("tmaps");
  h->stage_elems = std::min<int64_t>((int64_t)1 << 25, h->R * (N - 1) + N);  // <= 256 MB
  if (dalloc(&h->stage, (size_t)h->stage_elems) != cudaSuccess) {
    cudaGetLastError();
    return fail(h, CR_ENOMEM, "stage allocation failed");
  }
  CUDA_TRY(pinned_get((void**)&h->ctrl_h, sizeof(DevCtrl)));
  CUDA_TRY(pinned_get((void**)&h->ctrl_poll, 2 * sizeof(DevCtrl)));
  CUDA_TRY(pinned_get((void**)&h->pause_h, 2 * sizeof(long long)));
  std::memset(h->ctrl_h, 0, sizeof(DevCtrl));
  CUDA_TRY(cudaEventCreate(&h->ev_start));
  CUDA_TRY(cudaEventCreate(&h->ev_end));
  CUDA_TRY(cudaEventCreateWithFlags(&h->ev_poll[0], cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&h->ev_poll[1], cudaEventDisableTiming));
  tmark("pinned+events");

  // static inputs: X, ybar, row records (y placeholder, x, pad)
  CUDA_TRY(cudaMemcpyAsync(h->X, Xh, sizeof(double) * N * n, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(h->ybar, ybar_shifted, sizeof(double) * N, cudaMemcpyHostToDevice,
                           h->st));
  CUDA_TRY(launch_rowrec_init(h->X, h->ybar, h->rowrec, N, (int)n, (int)RP, h->st));  // (x, 1, y)
  CUDA_TRY(cudaMemsetAsync(h->colrec, 0, sizeof(double) * N * RP, h->st));
  const double consts[4] = {1.0, 1.0, 0.0, 0.0};
  CUDA_TRY(cudaMemcpyAsync(h->consts, consts, sizeof(consts), cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemsetAsync(h->izero, 0, sizeof(int), h->st));
  CUDA_TRY(cudaMemsetAsync(h->counter, 0, sizeof(unsigned int), h->st));
  CUDA_TRY(cudaMemsetAsync(h->d_stores, 0, sizeof(unsigned long long), h->st));
  CUDA_TRY(cudaMemsetAsync(h->ctrl_d, 0, sizeof(DevCtrl), h->st));
  CUDA_TRY(launch_gram(h->X, N, (int)n, h->gram, h->st));
  const char* sig = std::getenv("CRB_SIGMA");
  h->sigma_by_sweep = sig && std::strcmp(sig, "sweep") == 0;
  tmark("uploads");
  CUDA_TRY(cudaStreamSynchronize(h->st));
  tmark("sync");
  return CR_OK;
}

void cr_destroy(cr_handle* h) {
  if (!h) return;
  if (h->sigma_prep.joinable()) h->sigma_prep.join();
  cudaSetDevice(h->device);
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->part.K > 0) general_release(h);
  alcc_release(h);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->comm) ncclCommDestroy(h->comm);
  double* bufs[] = {h->X,       h->ybar,    h->rowrec,  h->colrec,   h->V[0],   h->V[1],
                    h->vpos[0], h->vpos[1], h->xbuf,    h->aggsave,  h->colpart, h->rowpart,
                    h->scalpart, h->k2part, h->k2sum,   h->hist,     h->yout,   h->xiout,
                    h->pw_u,    h->pw_v,    h->pw_part, h->pw_sum,   h->consts, h->stage,
                    h->gram,    h->ps_part, h->ps_part2, h->ps_state, h->sv_u12};
  for (double* b : bufs) dfree(b, h->st);
  for (double* b : {h->s_colpart, h->s_rowpart, h->s_scalpart, h->s_k2part}) dfree(b, h->st);
  release_canon(h);
  dfree(h->izero, h->st);
  dfree(h->counter, h->st);
  dfree(h->d_stores, h->st);
  dfree(h->ctrl_d, h->st);
  if (h->st) cudaStreamSynchronize(h->st);
  pinned_put(h->sigma_start_pin, h->sigma_start_bytes);
  pinned_put(h->out_pin, h->out_pin_bytes);
  pinned_put(h->ctrl_h, sizeof(DevCtrl));
  pinned_put(h->ctrl_poll, 2 * sizeof(DevCtrl));
  pinned_put(h->pause_h, 2 * sizeof(long long));
  for (cudaEvent_t ev : h->ev_sweep) cudaEventDestroy(ev);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  if (h->ev_end) cudaEventDestroy(h->ev_end);
  if (h->ev_poll[0]) cudaEventDestroy(h->ev_poll[0]);
  if (h->ev_poll[1]) cudaEventDestroy(h->ev_poll[1]);
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
}

cr_status cr_set_canonical_blocks(cr_handle* h, int32_t D) {
  if (!h || D < 0) return CR_EINVAL;
  if (h->begun && h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  release_canon(h);
  if (D == 0) return CR_OK;
  if (h->part.K > 0) return fail(h, CR_EINVAL, "canonical blocks: singleton blocks only");
  const int64_t N = h->N;
  if (D > N) return fail(h, CR_EINVAL, "canonical blocks: more blocks than rows");
  // block j = rows [floor(j N / D), floor((j + 1) N / D)): the shard must be a union of blocks
  auto bound = [&](int64_t j) { return (int64_t)(((__int128)j * N) / D); };
  int first = -1, last = -1;
  for (int j = 0; j <= D; ++j) {
    if (bound(j) == h->r0 && first < 0) first = j;
    if (bound(j) == h->r1) last = j;
  }
  if (first < 0 || last <= first)
    return fail(h, CR_EINVAL, "canonical blocks: the shard's rows are not a union of blocks");
  int sms = 148;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  g_alloc_stream = h->st;
  cudaError_t e = cudaSuccess;
  for (int j = first; j < last && e == cudaSuccess; ++j) {
    CanonBlock b;
    b.a = bound(j) - h->r0;
    b.R = bound(j + 1) - bound(j);
    const long long units = (long long)h->T * b.R;
    long long G = (long long)sms * h->kp.max_blocks_per_sm;
    G = std::min<long long>(G, (units + 63) / 64);
    if (G < 1) G = 1;
    b.U = (units + G - 1) / G;
    b.G = (int)((units + b.U - 1) / b.U);
    b.maxspan = (int)((b.U - 1) / b.R + 2);
    e = dalloc(&b.colpart, (size_t)b.G * b.maxspan * h->kp.tile_cols * (h->n + 1));
    if (e == cudaSuccess) e = dalloc(&b.rowpart, (size_t)h->T * b.R);
    if (e == cudaSuccess) e = dalloc(&b.scalpart, (size_t)b.G * h->kp.warps_per_block * kScal);
    b.tmap_ok = e == cudaSuccess && encode_tmap_pair(h, b.a, b.R, b.tmV);
    h->canon.push_back(b);
  }
  if (e == cudaSuccess) e = dalloc(&h->canon_pay, (size_t)D * (size_t)payload_len(h));
  if (e != cudaSuccess) {
    cudaGetLastError();
    release_canon(h);
    return fail(h, CR_ENOMEM, "canonical blocks: device allocation failed");
  }
  h->canon_D = D;
  h->canon_first = first;
  CUDA_TRY(cudaMemsetAsync(h->canon_pay, 0, sizeof(double) * (size_t)D * (size_t)payload_len(h),
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  h->begun = false;  // geometry changed: begin again
  return CR_OK;
}

cr_status cr_canonical_blocks(const cr_handle* h, int32_t* D, int32_t* first, int32_t* count) {
  if (!h) return CR_EINVAL;
  if (D) *D = h->canon_D;
  if (first) *first = h->canon_first;
  if (count) *count = (int32_t)h->canon.size();
  return CR_OK;
}

cr_status cr_nccl_unique_id(uint8_t id_out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CR_ENCCL;
  std::memcpy(id_out, &id, 128);
  return CR_OK;
}

cr_status cr_attach_nccl(cr_handle* h, const uint8_t id[128], int rank, int world) {
  if (!h || !id || world < 1 || rank < 0 || rank >= world) return CR_EINVAL;
  CUDA_TRY(cudaSetDevice(h->device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  NCCL_TRY(ncclCommInitRank(&h->comm, world, uid, rank));
  h->rank = rank;
  h->world = world;
  if (h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  return CR_OK;
}

cr_status cr_sigma_C(cr_handle* h, double tol, int32_t max_iters, double* sigma, int32_t* iters,
                     int32_t* converged) {
  if (!h || !sigma || !iters || !converged || max_iters < 1) return CR_EINVAL;
  CUDA_TRY(cudaSetDevice(h->device));
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t cols = h->N * (h->n + 1);
  const bool sdbg = std::getenv("CRB_DEBUG_SIGMA") != nullptr;
  auto smark = [&](const char* what) {
    if (sdbg)
      std::fprintf(stderr, "sigma %-10s %.3f ms\n", what,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3);
  };
  // fixed seeded start (operators.cpp:309-313), drawn at handle creation
  if (h->sigma_prep.joinable()) h->sigma_prep.join();
  smark("joined");
  if (h->sigma_start_ptr == nullptr || h->sigma_start_cols != cols) draw_sigma_start(h);
  if (!h->sv_u12) CUDA_TRY(dalloc(&h->sv_u12, (size_t)(2 * cols + 256)));
  CUDA_TRY(cudaMemcpyAsync(h->sv_u12, h->sigma_start_ptr, sizeof(double) * 2 * cols,
                           cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(launch_start_vector(h->sv_u12, h->pw_u, cols, h->sv_u12 + 2 * cols, h->st));
  smark("start enq");
  // closed-form steps assume singleton blocks; a K-block partition masks the
  // same-block pairs inside the sweep instead
  if (!h->sigma_by_sweep && h->part.K == 0) {  // whole power iteration in one cooperative launch
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
    CUDA_TRY(launch_power_loop(pa, h->power_grid, h->st));
    smark("loop enq");
    double st[3];
    CUDA_TRY(cudaMemcpyAsync(st, h->ps_state, sizeof(st), cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
    smark("done");
    *sigma = st[0];
    *iters = (int32_t)st[1];
    *converged = (int32_t)st[2];
    h->sigma_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return CR_OK;
  }
  double norm_u = 1.0;  // v = u / 1 on the first step
  double lambda_prev = 0;
  *converged = 1;
  for (int it = 1; it <= max_iters; ++it) {
    double lambda = 0, nu = 0;
    const cr_status s = power_step(h, norm_u, &lambda, &nu);
    if (s != CR_OK) return s;
    if (nu == 0 || lambda == 0) {
      *sigma = 0;
      *iters = it;
      h->sigma_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      return CR_OK;
    }
    norm_u = nu;
    *iters = it;
    if (it > 1 && std::fabs(lambda - lambda_prev) <= tol * lambda) {
      *sigma = std::sqrt(lambda) * 1.01;
      *converged = 1;
      h->sigma_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      return CR_OK;
    }
    lambda_prev = lambda;
  }
  *sigma = std::sqrt(lambda_prev) * 1.10;
  *converged = 0;
  h->sigma_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return CR_OK;
}

}  // extern "C"

namespace {
// resume: warm start from the handle's device-resident theta1 (papg.cpp:159-164
// with theta0 = the previous solve's theta1, e.g. the gamma continuation of
// runner.cpp:258-259, 305, 322) without a host round trip.
cr_status begin_impl(cr_handle* h, const cr_papg_config* cfg, const double* theta0, bool resume) {
  if (!h || !cfg) return CR_EINVAL;
  if (!(cfg->gamma > 0) || cfg->max_iters < 1) return fail(h, CR_EINVAL, "papg: bad config");
  if (resume && (!h->begun || theta0 != nullptr))
    return fail(h, CR_ESTATE, "papg: resume needs a previous solve on this handle");
  CUDA_TRY(cudaSetDevice(h->device));
  if (resume) {
    const cr_status s0 = sync_ctrl(h);
    if (s0 != CR_OK) return s0;
  }
  const DevCtrl prev = *h->ctrl_h;
  h->t_begin = std::chrono::steady_clock::now();
  h->cfg = *cfg;
  h->begun = false;
  const int64_t N = h->N;
  // clock origin of the time budget (papg.cpp:139) is set before sigma_C
  DevCtrl c{};
  std::memset(&c, 0, sizeof(c));
  CUDA_TRY(cudaMemcpyAsync(h->ctrl_d, &c, sizeof(c), cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(launch_begin(h->ctrl_d, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  h->sigma_iters = 0;
  h->sigma_conv = 1;
  h->sigma_seconds = 0;
  if (cfg->sigma_C > 0) {
    h->sigma_C = cfg->sigma_C;
  } else if (resume && h->sigma_C > 0) {
    // same X -> the same power iteration and sigma; keep the cached value
  } else {
    int32_t it = 0, conv = 1;
    double s = 0;
    const cr_status st = cr_sigma_C(h, 1e-6, 5000, &s, &it, &conv);
    if (st != CR_OK) return st;
    h->sigma_C = s;
    h->sigma_iters = it;
    h->sigma_conv = conv;
  }
  if (!(h->sigma_C > 0)) return fail(h, CR_EINVAL, "papg: sigma_max(C) is zero");
  h->L = h->sigma_C * h->sigma_C / cfg->gamma;  // papg.hpp:43

  // history buffer
  const int64_t want_hist = cfg->record_history ? std::min<int64_t>(cfg->max_iters, CR_HISTORY_CAP) : 0;
  if (want_hist > h->hist_cap) {
    dfree(h->hist, h->st);
    h->hist = nullptr;
    h->hist_cap = 0;
    g_alloc_stream = h->st;
    if (dalloc(&h->hist, (size_t)(8 * want_hist)) != cudaSuccess) {
      cudaGetLastError();
      return fail(h, CR_ENOMEM, "history allocation failed");
    }
    h->hist_cap = want_hist;
    if (h->gexec) {
      cudaGraphExecDestroy(h->gexec);
      h->gexec = nullptr;
    }
  }

  // device control block (papg.cpp:148-175)
  CUDA_TRY(cudaMemcpyAsync(&c, h->ctrl_d, sizeof(c), cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  const unsigned long long t0 = c.t_start_ns;
  std::memset(&c, 0, sizeof(c));
  c.t_start_ns = t0;
  c.ell = 0;
  c.max_iters = cfg->max_iters;
  c.hist_cap = cfg->record_history ? h->hist_cap : 0;
  c.cur = resume ? prev.cur : 0;
  c.max_restarts = cfg->max_restarts;
  c.adaptive = cfg->adaptive_B_theta ? 1 : 0;
  c.use_momentum = cfg->use_momentum ? 1 : 0;
  c.record_history = cfg->record_history ? 1 : 0;
  c.pause_at = LLONG_MAX;
  c.s_cur = 1.0;
  c.s_prev = 1.0;
  c.beta = 0.0;
  c.t = 1.0;
  c.B_theta = cfg->B_theta > 0 ? cfg->B_theta : 10.0 * std::sqrt((double)N);
  c.g_star_upper = INFINITY;
  c.invL = 1.0 / h->L;
  c.gamma = cfg->gamma;
  c.gap_tol = cfg->gap_norm_tol;
  c.infeas_tol = cfg->infeas_norm_tol;
  c.inner_tol_floor = cfg->inner_tol_floor;
  c.max_seconds = cfg->max_seconds;
  c.gap_div = (double)N * (double)(N - 1);
  c.infeas_div = std::sqrt(c.gap_div);
  c.K = h->part.K > 0 ? (double)h->part.K : (double)N;  // papg.cpp:198 cushion
  if (resume) {  // theta1 = Pi_Q2(theta0), theta0 = s V[cur] >= 0: a rescale only
    const double nrm = prev.theta1_norm;
    const double sc = nrm > c.B_theta ? c.B_theta / nrm : 1.0;
    c.s_cur = prev.s_cur * sc;
    c.s_prev = c.s_cur;
  }
  CUDA_TRY(cudaMemcpyAsync(h->ctrl_d, &c, sizeof(c), cudaMemcpyHostToDevice, h->st));
  std::memcpy(h->ctrl_h, &c, sizeof(c));

  const size_t vbytes = sizeof(double) * (size_t)h->R * (size_t)h->ld;
  // small N (V, V' L2-resident, one GPU): one persistent cooperative launch runs
  // many iterations (small.cu). CRB_SMALL=0 disables, CRB_SMALL=1 forces.
  const char* smenv = std::getenv("CRB_SMALL");
  // measured crossover against the per-kernel path with CUDA graphs (us/iteration,
  // n = 5: N = 600 16.4 vs 20.8, N = 1000 20.0 vs 21.2, N = 1500 28.4 vs 23.0;
  // N = 1000, n = 10: 29.5 vs 24.7): N^2 (n + 2) <= 7e6
  bool want_small = h->comm == nullptr && cfg->graph_iters == 0 &&
                    (double)h->R * (double)h->N * (double)(h->n + 2) <= 7.0e6 && h->part.K == 0;
  if (smenv && smenv[0] == '0') want_small = false;
  if (smenv && smenv[0] == '1' && h->comm == nullptr && h->R == h->N && h->part.K == 0)
    want_small = true;
  if (!h->canon.empty()) {
    if (h->part.K > 0) return fail(h, CR_EINVAL, "canonical blocks: singleton blocks only");
    if (h->comm && ((int)h->canon.size() * h->world != h->canon_D ||
                    h->canon_first != h->rank * (int)h->canon.size()))
      return fail(h, CR_EINVAL, "canonical blocks: every rank must own D / world consecutive blocks");
    want_small = false;  // the persistent loop's shares are not canonical
  }
  if (!resume) {
    CUDA_TRY(cudaMemsetAsync(h->V[0], 0, vbytes, h->st));
    CUDA_TRY(cudaMemsetAsync(h->V[1], 0, vbytes, h->st));
    CUDA_TRY(cudaMemsetAsync(h->vpos[0], 0, sizeof(double) * N, h->st));
    CUDA_TRY(cudaMemsetAsync(h->vpos[1], 0, sizeof(double) * N, h->st));
    CUDA_TRY(cudaMemsetAsync(h->xbuf, 0, sizeof(double) * payload_len(h), h->st));
    CUDA_TRY(cudaMemsetAsync(h->aggsave, 0, sizeof(double) * payload_len(h), h->st));
  }
  if (h->canon_pay)
    CUDA_TRY(cudaMemsetAsync(h->canon_pay, 0,
                             sizeof(double) * (size_t)h->canon_D * (size_t)payload_len(h), h->st));

  if (theta0 && h->part.K > 0) {
    const cr_status s = general_theta_in(h, theta0);
    if (s != CR_OK) return s;
  }
  if (theta0) {  // warm start: theta1 = Pi_Q2(theta0) (papg.cpp:159-164)
    const int64_t rowlen = N - 1;
    const int64_t rows_per = std::max<int64_t>(1, h->stage_elems / rowlen);
    for (int64_t ra = 0; ra < h->R && h->part.K == 0; ra += rows_per) {
      const int64_t rb = std::min(h->R, ra + rows_per);
      CUDA_TRY(cudaMemcpyAsync(h->stage, theta0 + ra * rowlen,
                               sizeof(double) * (rb - ra) * rowlen, cudaMemcpyHostToDevice,
                               h->st));
      CUDA_TRY(launch_theta_in(h->stage, h->V[0], N, h->ld, h->r0, ra, rb, h->st));
    }
    const double* tpos =
        theta0 + (h->part.K > 0 ? h->N * (h->N - h->part.nbar) : h->R * rowlen);
    double pos_sq = 0;
    for (int64_t l = 0; l < N; ++l) {
      const double t = tpos[l] > 0 ? tpos[l] : 0.0;
      pos_sq += t * t;
    }
    CUDA_TRY(cudaMemcpyAsync(h->stage, tpos, sizeof(double) * N, cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(launch_pos_in(h->vpos[0], h->stage, N, h->st));
    // aggregates and |.|^2 of max(theta0, 0): a sweep with 1/L = 0 is a copy
    if (!h->canon.empty()) {
      cr_status cs = enqueue_canon_local(h, true, nullptr, false, nullptr, nullptr, true, nullptr,
                                         nullptr);
      if (cs == CR_OK) cs = enqueue_canon_combine(h);
      if (cs != CR_OK) return cs;
    } else {
      const SweepArgs sa = sweep_args(h, kModePapg, true);
      CUDA_TRY((cudaError_t)launch_sweep(papg_sweep(h), sa, h->st));
      const ReduceArgs ra = reduce_args(h, false, nullptr, false, papg_sweep(h).scal_recs);
      CUDA_TRY(launch_reduce(ra, h->st));
      if (h->comm)
        NCCL_TRY(ncclAllReduce(h->xbuf, h->xbuf, (size_t)payload_len(h), ncclDouble, ncclSum,
                               h->comm, h->st));
    }
    CUDA_TRY(launch_warm_ctrl(h->ctrl_d, h->xbuf + N * (h->n + 2), pos_sq, h->st));
  }

  {
    const bool want = want_small;
    h->small_mode = false;
    if (want) {
      h->ks = small_loop_info((int)h->n);
      int sms = 148;
      CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
      const int bps = std::min(h->ks.max_blocks_per_sm, 2);
      if (h->ks.fn && bps >= 1) {
        h->small_grid = sms * bps;
        h->small_S = (int)((h->N + 31) / 32);
        const long long warps = (long long)h->small_grid * (h->ks.threads / 32);
        h->small_P = (int)std::max<long long>(1, std::min<long long>(h->N, warps / h->small_S));
        // resident variant (one block per SM): one (strip, chunk) task per warp and the
        // tiles of a block's 8 warps within 200 KB of shared memory (config 1: 27 rows,
        // 110 KB). CRB_SMALL_RESIDENT=0 keeps the L2 variant.
        h->small_RT = 0;
        h->small_smem = 0;
        {
          const SmallInfo kr = small_loop_info((int)h->n, true);
          const long long warps1 = (long long)sms * (kr.threads / 32);
          const long long P1 = std::max<long long>(1, std::min<long long>(h->N, warps1 / h->small_S));
          const long long RT = (h->N + P1 - 1) / P1;
          const char* rv = std::getenv("CRB_SMALL_RESIDENT");
          if (!(rv && rv[0] == '0') && kr.fn && kr.max_blocks_per_sm >= 1 &&
              (long long)h->small_S * P1 <= warps1 &&
              small_resident_smem((int)RT, kr.threads) <= 200 * 1024) {
            h->ks = kr;
            h->small_grid = sms;
            h->small_P = (int)P1;
            h->small_RT = (int)RT;
            h->small_smem = small_resident_smem((int)RT, kr.threads);
          }
        }
        for (double* b : {h->s_colpart, h->s_rowpart, h->s_scalpart, h->s_k2part})
          dfree(b, h->st);
        h->s_colpart = h->s_rowpart = h->s_scalpart = h->s_k2part = nullptr;
        g_alloc_stream = h->st;
        cudaError_t e = cudaSuccess;
        if (e == cudaSuccess)
          e = dalloc(&h->s_colpart, (size_t)h->small_P * h->N * (h->n + 1));
        if (e == cudaSuccess) e = dalloc(&h->s_rowpart, (size_t)h->small_S * h->N);
        if (e == cudaSuccess)
          e = dalloc(&h->s_scalpart, (size_t)h->small_grid * kScal);
        // K2 records double buffered by iteration parity + the launch's clock slot
        if (e == cudaSuccess) e = dalloc(&h->s_k2part, (size_t)2 * h->small_grid * kK2Scal + 1);
        if (e != cudaSuccess) {
          cudaGetLastError();
          return fail(h, CR_ENOMEM, "small-N buffers");
        }
        h->small_mode = true;
      }
    }
  }

  // batch size: graphs when an iteration is short, direct launches otherwise
  if (h->part.K > 0) {
    h->graph_iters = 0;  // host-driven (block solves between the kernels)
    h->part.workers = cfg->workers;
    const cr_status s = general_begin(h);
    if (s != CR_OK) return s;
  } else if (cfg->graph_iters > 0) {
    h->graph_iters = cfg->graph_iters;
  } else if (cfg->graph_iters < 0) {
    h->graph_iters = 0;
  } else {
    const double est_us = 24.0 * (double)h->R * (double)h->ld / 5.0e6 + 12.0;
    h->graph_iters = est_us > 300.0 ? 0 : (int)std::min(256.0, std::ceil(2000.0 / est_us));
  }
  if (h->graph_iters > 0 && !h->small_mode) {
    const cr_status s = build_graph(h);
    if (s != CR_OK) return s;
  }
  const cr_status s = sync_ctrl(h);
  if (s != CR_OK) return s;
  h->loop_seconds = 0;
  h->begun = true;
  return CR_OK;
}
}  // namespace

extern "C" {

cr_status cr_papg_begin(cr_handle* h, const cr_papg_config* cfg, const double* theta0) {
  return begin_impl(h, cfg, theta0, false);
}

cr_status cr_papg_begin_resume(cr_handle* h, const cr_papg_config* cfg) {
  return begin_impl(h, cfg, nullptr, true);
}

cr_status cr_set_observations(cr_handle* h, const double* ybar_shifted) {
  if (!h || !ybar_shifted) return CR_EINVAL;
  CUDA_TRY(cudaSetDevice(h->device));
  CUDA_TRY(cudaMemcpyAsync(h->ybar, ybar_shifted, sizeof(double) * h->N, cudaMemcpyHostToDevice,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

cr_status cr_papg_iterate(cr_handle* h, int64_t max_steps, int64_t* done, int32_t* stopped) {
  if (!h) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "papg: iterate before begin");
  CUDA_TRY(cudaSetDevice(h->device));
  if (max_steps < 0) max_steps = 0;
  const long long ell0 = h->ctrl_h->ell;
  long long pause = ell0 + max_steps;
  if (pause < ell0) pause = LLONG_MAX;
  cr_status s = set_pause(h, pause);
  if (s != CR_OK) return s;
  if (h->part.K > 0) {  // general-K partition: host-driven iterations (general.cu)
    const auto wall0 = std::chrono::steady_clock::now();
    double sw = 0;
    int64_t nl = 0;
    s = general_iterate(h, max_steps, done, stopped, &sw, &nl);
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    h->last_seconds = wall;
    h->last_sweep_seconds = sw;
    h->last_launches = nl;
    h->loop_seconds += wall;
    return s;
  }
  if (h->small_mode) {  // one persistent launch, halts on termination or pause
    if (h->ctrl_h->stopped || max_steps == 0) {
      h->last_seconds = 0;
      h->last_launches = 0;
      h->last_sweep_seconds = 0;
    } else {
      SmallArgs sa{};
      sa.pa = primal_args(h, 0);
      sa.pa.tr_adjoint = 0;  // the small-N loop's sweep accumulates theta2 . row itself
      sa.V0 = h->V[0];
      sa.V1 = h->V[1];
      sa.colpart = h->s_colpart;
      sa.rowpart = h->s_rowpart;
      sa.scalpart = h->s_scalpart;
      sa.k2part = h->s_k2part;
      sa.clock = reinterpret_cast<unsigned long long*>(h->s_k2part + (size_t)2 * h->small_grid * kK2Scal);
      sa.xbuf = h->xbuf;
      sa.k2sum = h->k2sum;
      sa.hist = h->hist;
      sa.ctrl = h->ctrl_d;
      sa.N = h->N;
      sa.ld = h->ld;
      sa.max_iters = max_steps;
      sa.S = h->small_S;
      sa.P = h->small_P;
      sa.RT = h->small_RT;
      unsigned long long* trace = nullptr;
      if (std::getenv("CRB_TRACE")) {
        CUDA_TRY(cudaMalloc(&trace, 64 * 8 * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemsetAsync(trace, 0, 64 * 8 * sizeof(unsigned long long), h->st));
      }
      sa.trace = trace;
      const auto wall0 = std::chrono::steady_clock::now();
      CUDA_TRY(cudaEventRecord(h->ev_start, h->st));
      CUDA_TRY(launch_small_loop(h->ks, sa, h->small_grid, h->st, h->small_smem));
      CUDA_TRY(cudaEventRecord(h->ev_end, h->st));
      s = sync_ctrl(h);
      if (s != CR_OK) return s;
      float ms = 0;
      CUDA_TRY(cudaEventElapsedTime(&ms, h->ev_start, h->ev_end));
      h->last_seconds = ms * 1e-3;
      h->last_launches = 1;
      h->last_sweep_seconds = 0;
      if (trace) {  // dev aid: mean phase durations of the first iterations
        unsigned long long tb[64 * 8];
        CUDA_TRY(cudaMemcpy(tb, trace, sizeof(tb), cudaMemcpyDeviceToHost));
        double acc[7] = {0};
        int cnt = 0;
        for (int it = 1; it < 64 && tb[it * 8 + 7] != 0; ++it, ++cnt)
          for (int k = 0; k < 7; ++k) acc[k] += (double)(tb[it * 8 + k + 1] - tb[it * 8 + k]);
        std::fprintf(stderr, "small-loop phases (ns, mean of %d): B-load %.0f B-math %.0f B-store %.0f syncB %.0f C+ctl %.0f A %.0f sync %.0f\n",
                     cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt,
                     acc[5] / cnt, acc[6] / cnt);
        cudaFree(trace);
      }
      h->loop_seconds +=
          std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    }
    if (done) *done = h->ctrl_h->ell;
    if (stopped) *stopped = h->ctrl_h->stopped;
    if (h->ctrl_h->stopped && h->ctrl_h->reason == 3)
      return fail(h, CR_ENONFINITE, "papg: non-finite dual gradient");
    return CR_OK;
  }
  const bool timed_sweeps = h->graph_iters == 0;
  // Sweep timing: an event pair around every 8th sweep (CRB_SWEEP_EVENTS=k: every
  // k-th, 0: none); the reported sweep seconds are the sampled mean times the
  // iterations run. Event records between the kernels cost ~5 us per cfg 2
  // iteration (measured 384.8 vs 379.9 us; external event nodes in a captured
  // graph cost more: 388.9 us at 4 iterations per graph), so long calls sample.
  // A call of at most 64 iterations brackets every sweep (a short call's early
  // iterations differ too much for a sample).
  int every = max_steps <= 64 ? 1 : 8;
  if (const char* ev = std::getenv("CRB_SWEEP_EVENTS")) every = std::max(0, std::atoi(ev));
  // direct launches: poll the device state every `per_unit` iterations (one D2H copy
  // + event per unit); CRB_POLL_UNIT overrides (measurement knob)
  int per_unit = h->graph_iters > 0 ? h->graph_iters : 4;
  if (h->graph_iters == 0)
    if (const char* pu = std::getenv("CRB_POLL_UNIT")) per_unit = std::max(1, std::atoi(pu));
  h->primal_pending = true;  // direct launches: the call starts with the (maybe no-op) primal
  int64_t enq_iters = 0;
  int64_t units = 0;
  bool halted = h->ctrl_h->stopped || max_steps == 0;
  int64_t timed_pairs = 0;
  CUDA_TRY(cudaEventRecord(h->ev_start, h->st));
  const auto wall0 = std::chrono::steady_clock::now();
  while (!halted) {
    if (h->graph_iters > 0) {
      CUDA_TRY(cudaGraphLaunch(h->gexec, h->st));
    } else {
      for (int i = 0; i < per_unit && enq_iters + i < max_steps; ++i) {
        cudaEvent_t a = nullptr, b = nullptr, c = nullptr, d = nullptr;
        const bool sample = every > 0 && ((enq_iters + i) % every) == 0;
        if (timed_sweeps && sample && timed_pairs < (1 << 16)) {  // event pairs created on demand
          const size_t per = h->comm ? 4 : 2;  // sharded: the allreduce is bracketed too
          while (h->ev_sweep.size() < (size_t)(per * timed_pairs + per)) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreate(&e));
            h->ev_sweep.push_back(e);
          }
          a = h->ev_sweep[per * timed_pairs];
          b = h->ev_sweep[per * timed_pairs + 1];
          if (h->comm) {
            c = h->ev_sweep[per * timed_pairs + 2];
            d = h->ev_sweep[per * timed_pairs + 3];
          }
          ++timed_pairs;
        }
        s = enqueue_iteration(h, 0, a, b, true, c, d);
        if (s != CR_OK) return s;
      }
    }
    enq_iters += per_unit;
    // long direct-launch runs poll less often (16 iterations per unit after the
    // first 64: +0.5 % at cfg 2; short solves keep the 4-iteration halting latency)
    if (h->graph_iters == 0 && per_unit < 16 && enq_iters >= 64 && !std::getenv("CRB_POLL_UNIT"))
      per_unit = 16;
    const int slot = (int)(units & 1);
    CUDA_TRY(cudaMemcpyAsync(&h->ctrl_poll[slot], h->ctrl_d, sizeof(DevCtrl),
                             cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaEventRecord(h->ev_poll[slot], h->st));
    if (units >= 1) {  // keep one unit in flight while polling the previous one
      const int ps = (int)((units - 1) & 1);
      CUDA_TRY(cudaEventSynchronize(h->ev_poll[ps]));
      if (h->ctrl_poll[ps].halt) halted = true;
    }
    ++units;
    if (!halted && h->graph_iters == 0 && enq_iters >= max_steps) {
      CUDA_TRY(cudaEventSynchronize(h->ev_poll[slot]));
      halted = true;
    }
  }
  CUDA_TRY(cudaEventRecord(h->ev_end, h->st));
  s = sync_ctrl(h);
  if (s != CR_OK) return s;
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, h->ev_start, h->ev_end));
  h->last_seconds = units > 0 ? ms * 1e-3 : 0.0;
  double sw = 0, xw = 0;
  h->last_sweep_times.clear();
  const int64_t per = h->comm ? 4 : 2;
  for (int64_t i = 0; i < timed_pairs; ++i) {
    float m = 0;
    CUDA_TRY(cudaEventElapsedTime(&m, h->ev_sweep[per * i], h->ev_sweep[per * i + 1]));
    sw += m * 1e-3;
    h->last_sweep_times.push_back(m * 1e-3);
    if (h->comm) {
      float mx = 0;
      CUDA_TRY(cudaEventElapsedTime(&mx, h->ev_sweep[per * i + 2], h->ev_sweep[per * i + 3]));
      xw += mx * 1e-3;
    }
  }
  {
    const int64_t ran = std::min<int64_t>(enq_iters, max_steps);
    const double scale = (timed_pairs > 0 && every > 1) ? (double)ran / (double)timed_pairs : 1.0;
    h->last_sweep_seconds = sw * scale;
    h->last_exchange_seconds = xw * scale;
  }
  h->last_launches = (h->graph_iters > 0 ? units * h->graph_iters
                                         : std::min<int64_t>(enq_iters, max_steps)) *
                         launches_per_iteration(h);
  h->loop_seconds +=
      std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  if (done) *done = h->ctrl_h->ell;
  if (stopped) *stopped = h->ctrl_h->stopped;
  if (h->ctrl_h->stopped && h->ctrl_h->reason == 3)
    return fail(h, CR_ENONFINITE, "papg: non-finite dual gradient");
  return CR_OK;
}

cr_status cr_iter_local(cr_handle* h) {
  if (!h) return CR_EINVAL;
  if (h->part.K > 0) return fail(h, CR_EINVAL, "partition: the exchange seam is singleton-only");
  if (!h->begun) return fail(h, CR_ESTATE, "papg: iterate before begin");
  CUDA_TRY(cudaSetDevice(h->device));
  cr_status s = set_pause(h, LLONG_MAX);
  if (s != CR_OK) return s;
  s = enqueue_iteration(h, 1, nullptr, nullptr, false, nullptr, nullptr);
  if (s != CR_OK) return s;
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

cr_status cr_exchange_get(cr_handle* h, double* buf) {
  if (!h || !buf) return CR_EINVAL;
  if (!h->canon.empty()) {  // all D block payloads; only this shard's own blocks are current
    CUDA_TRY(cudaMemcpyAsync(buf, h->canon_pay, sizeof(double) * (size_t)cr_exchange_len(h),
                             cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
    return CR_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(buf, h->xbuf, sizeof(double) * payload_len(h), cudaMemcpyDeviceToHost,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

cr_status cr_exchange_put(cr_handle* h, const double* buf) {
  if (!h || !buf) return CR_EINVAL;
  if (!h->canon.empty()) {  // the gathered block payloads (what ncclAllGather would leave)
    CUDA_TRY(cudaMemcpyAsync(h->canon_pay, buf, sizeof(double) * (size_t)cr_exchange_len(h),
                             cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
    return CR_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(h->xbuf, buf, sizeof(double) * payload_len(h), cudaMemcpyHostToDevice,
                           h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

cr_status cr_iter_finish(cr_handle* h, int32_t* stopped) {
  if (!h) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "papg: iterate before begin");
  cr_status s = enqueue_iteration(h, 2, nullptr, nullptr, false, nullptr, nullptr);
  if (s != CR_OK) return s;
  s = sync_ctrl(h);
  if (s != CR_OK) return s;
  if (stopped) *stopped = h->ctrl_h->stopped;
  if (h->ctrl_h->stopped && h->ctrl_h->reason == 3)
    return fail(h, CR_ENONFINITE, "papg: non-finite dual gradient");
  return CR_OK;
}

cr_status cr_papg_finish(cr_handle* h, cr_papg_result* res, double* y, double* xi,
                         cr_snapshot* history) {
  if (!h || !res) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "papg: finish before begin");
  CUDA_TRY(cudaSetDevice(h->device));
  const bool fdbg = std::getenv("CRB_DEBUG_FINISH") != nullptr;
  const auto tf0 = std::chrono::steady_clock::now();
  auto fmark = [&](const char* what) {
    if (fdbg)
      std::fprintf(stderr, "finish %-10s %.3f ms\n", what,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - tf0).count() * 1e3);
  };
  cr_status s = sync_ctrl(h);
  if (s != CR_OK) return s;
  fmark("sync_ctrl");
  const DevCtrl& c = *h->ctrl_h;
  double ft = 1.0 / std::pow((double)c.ell, 3.0);  // papg.cpp:266-269
  ft = std::min(ft, h->cfg.inner_tol_floor);
  ft = std::min(ft, h->cfg.final_resolve_tol);
  if (h->part.K > 0) {  // block re-solves at theta1 (general.cu)
    s = general_final(h, ft);
    if (s != CR_OK) return s;
  } else {
    // final re-solve at theta1 (papg.cpp:265-277): primal of s_cur * V[cur]
    const PrimalArgs pa = primal_args(h, 1);
    CUDA_TRY(launch_primal(pa, h->st));
    CUDA_TRY(launch_reduce_records(h->k2part, h->k2_blocks, kK2Scal, h->k2sum, h->st));
  }
  fmark("enqueued");
  double k2[kK2Scal];
  CUDA_TRY(cudaMemcpyAsync(k2, h->k2sum, sizeof(k2), cudaMemcpyDeviceToHost, h->st));
  fmark("k2 copy");
  // (y, xi) through a pinned staging block of the process pool: pageable destinations made
  // these two copies 0.4 ms of a 12.6 ms config-2 solve
  const size_t out_bytes = sizeof(double) * (size_t)(h->N * (h->n + 1));
  if ((y || xi) && h->out_pin == nullptr) {
    void* p = nullptr;
    if (pinned_get(&p, out_bytes) == cudaSuccess) {
      h->out_pin = (double*)p;
      h->out_pin_bytes = out_bytes;
    } else {
      cudaGetLastError();
    }
  }
  double* ystage = h->out_pin ? h->out_pin : y;
  double* xistage = h->out_pin ? h->out_pin + h->N : xi;
  if (y)
    CUDA_TRY(cudaMemcpyAsync(ystage, h->yout, sizeof(double) * h->N, cudaMemcpyDeviceToHost,
                             h->st));
  if (xi)
    CUDA_TRY(cudaMemcpyAsync(xistage, h->xiout, sizeof(double) * h->N * h->n,
                             cudaMemcpyDeviceToHost, h->st));
  const int64_t nh = std::min<int64_t>(c.ell, c.hist_cap);
  if (history && nh > 0)
    CUDA_TRY(cudaMemcpyAsync(history, h->hist, sizeof(double) * 8 * nh, cudaMemcpyDeviceToHost,
                             h->st));
  fmark("copies");
  CUDA_TRY(cudaStreamSynchronize(h->st));
  if (h->out_pin) {
    if (y) std::memcpy(y, ystage, sizeof(double) * h->N);
    if (xi) std::memcpy(xi, xistage, sizeof(double) * h->N * h->n);
  }
  fmark("synced");
  std::memset(res, 0, sizeof(*res));
  res->iters = c.ell;
  res->reason = c.reason;
  res->restarts = c.restarts;
  res->saturated = c.saturated;
  res->history_truncated = c.record_history && c.ell > c.hist_cap ? 1 : 0;
  res->sigma_iters = h->sigma_iters;
  res->sigma_converged = h->sigma_conv;
  res->g_final = k2[4];
  res->delta_estimate = std::max(0.0, c.g_star_upper - (k2[4] - 2.0 * ft * c.K));
  res->sigma_C = h->sigma_C;
  res->L_g = h->L;
  res->B_theta = c.B_theta;
  res->wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - h->t_begin).count();
  res->sigma_seconds = h->sigma_seconds;
  res->loop_seconds = h->loop_seconds;
  res->last_gap_norm = c.gap_norm;
  res->last_infeas_norm = c.infeas_norm;
  if (k2[7] != 0.0) return fail(h, CR_ENONFINITE, "papg: non-finite primal");
  return CR_OK;
}

cr_status cr_papg_solve(cr_handle* h, const cr_papg_config* cfg, const double* theta0,
                        cr_papg_result* res, double* y, double* xi, cr_snapshot* history) {
  cr_status s = cr_papg_begin(h, cfg, theta0);
  if (s != CR_OK) return s;
  int64_t done = 0;
  int32_t stopped = 0;
  while (!stopped) {
    s = cr_papg_iterate(h, INT64_MAX / 4, &done, &stopped);
    if (s != CR_OK) return s;
  }
  return cr_papg_finish(h, res, y, xi, history);
}

// theta1 / C eta of local rows [la, lb) of the shard, followed by the N pos rows
static cr_status get_theta_window(cr_handle* h, int64_t la, int64_t lb, double* out) {
  CUDA_TRY(cudaSetDevice(h->device));
  cr_status s = sync_ctrl(h);
  if (s != CR_OK) return s;
  const int cur = h->ctrl_h->cur;
  const double sc = h->ctrl_h->s_cur;
  const int64_t rowlen = h->N - 1;
  const int64_t rows_per = std::max<int64_t>(1, h->stage_elems / rowlen);
  for (int64_t ra = la; ra < lb; ra += rows_per) {
    const int64_t rb = std::min(lb, ra + rows_per);
    CUDA_TRY(launch_theta_out(h->stage, h->V[cur], sc, h->N, h->ld, h->r0, ra, rb, h->st));
    CUDA_TRY(cudaMemcpyAsync(out + (ra - la) * rowlen, h->stage, sizeof(double) * (rb - ra) * rowlen,
                             cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  CUDA_TRY(launch_scale_copy(h->stage, h->vpos[cur], sc, h->N, h->st));
  CUDA_TRY(cudaMemcpyAsync(out + (lb - la) * rowlen, h->stage, sizeof(double) * h->N,
                           cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}

static cr_status get_rows_window(cr_handle* h, int64_t la, int64_t lb, double* out) {
  CUDA_TRY(cudaSetDevice(h->device));
  const int64_t rowlen = h->N - 1;
  const int64_t rows_per = std::max<int64_t>(1, h->stage_elems / rowlen);
  for (int64_t ra = la; ra < lb; ra += rows_per) {
    const int64_t rb = std::min(lb, ra + rows_per);
    CUDA_TRY(launch_rows_out(h->stage, h->rowrec, h->colrec, h->N, (int)h->n, h->r0, ra, rb, h->st));
    CUDA_TRY(cudaMemcpyAsync(out + (ra - la) * rowlen, h->stage, sizeof(double) * (rb - ra) * rowlen,
                             cudaMemcpyDeviceToHost, h->st));
    CUDA_TRY(cudaStreamSynchronize(h->st));
  }
  std::vector<double> rec((size_t)h->N * h->RP);
  CUDA_TRY(cudaMemcpy(rec.data(), h->rowrec, sizeof(double) * rec.size(), cudaMemcpyDeviceToHost));
  for (int64_t l = 0; l < h->N; ++l)  // apply_C :152, y of eta
    out[(lb - la) * rowlen + l] = rec[(size_t)l * h->RP + h->n + 1];
  return CR_OK;
}

cr_status cr_get_theta(cr_handle* h, double* out) {
  if (!h || !out) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "no dual state");
  if (h->part.K > 0) {
    CUDA_TRY(cudaSetDevice(h->device));
    cr_status s = sync_ctrl(h);
    if (s != CR_OK) return s;
    return general_get_theta(h, out);
  }
  return get_theta_window(h, 0, h->R, out);
}

cr_status cr_get_rows(cr_handle* h, double* out) {
  if (!h || !out) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "no dual state");
  if (h->part.K > 0) {
    CUDA_TRY(cudaSetDevice(h->device));
    return general_get_rows(h, out);
  }
  return get_rows_window(h, 0, h->R, out);
}

cr_status cr_get_theta_rows(cr_handle* h, int64_t row_begin, int64_t row_end, double* out) {
  if (!h || !out) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "no dual state");
  if (h->part.K > 0) return fail(h, CR_EINVAL, "row windows need singleton blocks");
  if (row_begin < h->r0 || row_end > h->r0 + h->R || row_begin > row_end)
    return fail(h, CR_EINVAL, "row window outside the shard");
  return get_theta_window(h, row_begin - h->r0, row_end - h->r0, out);
}

cr_status cr_get_rows_window(cr_handle* h, int64_t row_begin, int64_t row_end, double* out) {
  if (!h || !out) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "no dual state");
  if (h->part.K > 0) return fail(h, CR_EINVAL, "row windows need singleton blocks");
  if (row_begin < h->r0 || row_end > h->r0 + h->R || row_begin > row_end)
    return fail(h, CR_EINVAL, "row window outside the shard");
  return get_rows_window(h, row_begin - h->r0, row_end - h->r0, out);
}

cr_status cr_last_timing(const cr_handle* h, double* seconds, int64_t* launches,
                         double* sweep_seconds) {
  if (!h) return CR_EINVAL;
  if (seconds) *seconds = h->last_seconds;
  if (launches) *launches = h->last_launches;
  if (sweep_seconds) *sweep_seconds = h->last_sweep_seconds;
  return CR_OK;
}

cr_status cr_last_exchange_seconds(const cr_handle* h, double* seconds) {
  if (!h || !seconds) return CR_EINVAL;
  *seconds = h->last_exchange_seconds;
  return CR_OK;
}

cr_status cr_last_sweep_times(const cr_handle* h, double* out, int64_t cap, int64_t* count) {
  if (!h || cap < 0) return CR_EINVAL;
  const int64_t k = (int64_t)h->last_sweep_times.size();
  if (count) *count = k;
  if (out)
    for (int64_t i = 0; i < std::min(k, cap); ++i) out[i] = h->last_sweep_times[i];
  return CR_OK;
}

int32_t cr_sweep_variant(const cr_handle* h) { return h ? h->variant : -1; }

cr_status cr_sweep_store_count(cr_handle* h, uint64_t* count, int32_t reset) {
  if (!h || !count) return CR_EINVAL;
  CUDA_TRY(cudaSetDevice(h->device));
  unsigned long long c = 0;
  CUDA_TRY(cudaMemcpyAsync(&c, h->d_stores, sizeof(c), cudaMemcpyDeviceToHost, h->st));
  if (reset) CUDA_TRY(cudaMemsetAsync(h->d_stores, 0, sizeof(c), h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  *count = c;
  return CR_OK;
}

cr_status cr_time_sweep(cr_handle* h, int32_t k, double* avg_seconds) {
  if (!h || k < 1 || !avg_seconds) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "no dual state");
  CUDA_TRY(cudaSetDevice(h->device));
  SweepArgs sa = sweep_args(h, kModePapg, false);
  sa.stopped = nullptr;
  CUDA_TRY(cudaEventRecord(h->ev_start, h->st));
  for (int i = 0; i < k; ++i) CUDA_TRY((cudaError_t)launch_sweep(papg_sweep(h), sa, h->st));
  CUDA_TRY(cudaEventRecord(h->ev_end, h->st));
  CUDA_TRY(cudaEventSynchronize(h->ev_end));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, h->ev_start, h->ev_end));
  *avg_seconds = ms * 1e-3 / k;
  return CR_OK;
}

}  // extern "C"

// ---- one-shot metric sweeps (metrics.cpp) ---------------------------------
namespace {
struct PointBufs {
  double *y = nullptr, *xi = nullptr, *rowrec = nullptr, *colrec = nullptr, *part = nullptr;
  cudaStream_t st = nullptr;
  ~PointBufs() {
    for (double* b : {y, xi, rowrec, colrec, part}) dfree(b, st);
    if (st) cudaStreamSynchronize(st);
  }
};

cr_status upload_point(cr_handle* h, const double* y, const double* xi, PointBufs& b) {
  b.st = h->st;
  g_alloc_stream = h->st;
  const size_t RP = (size_t)h->RP;
  if (dalloc(&b.y, h->N) != cudaSuccess || dalloc(&b.xi, h->N * h->n) != cudaSuccess ||
      dalloc(&b.rowrec, h->N * RP) != cudaSuccess || dalloc(&b.colrec, h->N * RP) != cudaSuccess) {
    cudaGetLastError();
    return fail(h, CR_ENOMEM, "metric buffers");
  }
  CUDA_TRY(cudaMemcpyAsync(b.y, y, sizeof(double) * h->N, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(cudaMemcpyAsync(b.xi, xi, sizeof(double) * h->N * h->n, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(launch_records(h->X, b.y, b.xi, h->N, (int)h->n, b.rowrec, b.colrec, h->st));
  return CR_OK;
}

// (sum min(row,0)^2, sum theta1.row) over all shards' rows
cr_status pair_metrics(cr_handle* h, PointBufs& b, bool with_theta, double out[2]) {
  int sms = 148;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  const int grid = sms * 4;
  if (dalloc(&b.part, (size_t)grid * 2 + 2) != cudaSuccess) {
    cudaGetLastError();
    return fail(h, CR_ENOMEM, "metric buffers");
  }
  MetricsArgs a{};
  a.rowrec = b.rowrec;
  a.colrec = b.colrec;
  a.V = with_theta ? h->V[h->ctrl_h->cur] : nullptr;
  a.s = h->ctrl_h->s_cur;
  a.part = b.part;
  a.N = h->N;
  a.R = h->R;
  a.r0 = h->r0;
  a.ld = h->ld;
  a.n = (int)h->n;
  a.S = (int)((h->N + 31) / 32);
  a.P = (int)std::max<long long>(1, std::min<long long>(h->R, (long long)grid * 8 / a.S));
  CUDA_TRY(launch_pair_metrics(a, grid, h->st));
  CUDA_TRY(launch_reduce_records(b.part, grid, 2, b.part + (size_t)grid * 2, h->st));
  if (h->comm)
    NCCL_TRY(ncclAllReduce(b.part + (size_t)grid * 2, b.part + (size_t)grid * 2, 2, ncclDouble,
                           ncclSum, h->comm, h->st));
  CUDA_TRY(cudaMemcpyAsync(out, b.part + (size_t)grid * 2, 2 * sizeof(double),
                           cudaMemcpyDeviceToHost, h->st));
  CUDA_TRY(cudaStreamSynchronize(h->st));
  return CR_OK;
}
}  // namespace

extern "C" {

cr_status cr_infeasibility(cr_handle* h, const double* y, const double* xi, double out2[2]) {
  if (!h || !y || !xi || !out2) return CR_EINVAL;
  CUDA_TRY(cudaSetDevice(h->device));
  PointBufs b;
  cr_status s = upload_point(h, y, xi, b);
  if (s != CR_OK) return s;
  double r[2];
  s = pair_metrics(h, b, false, r);
  if (s != CR_OK) return s;
  out2[0] = std::sqrt(r[0]);  // metrics.cpp:12-14
  out2[1] = out2[0] / std::sqrt((double)h->N * (double)(h->N - 1));
  return CR_OK;
}

cr_status cr_duality_gap(cr_handle* h, const double* y, const double* xi, double out2[2]) {
  if (!h || !y || !xi || !out2) return CR_EINVAL;
  if (!h->begun) return fail(h, CR_ESTATE, "no dual state");
  CUDA_TRY(cudaSetDevice(h->device));
  cr_status s = sync_ctrl(h);
  if (s != CR_OK) return s;
  PointBufs b;
  s = upload_point(h, y, xi, b);
  if (s != CR_OK) return s;
  double r[2];
  s = pair_metrics(h, b, true, r);
  if (s != CR_OK) return s;
  // identity rows: theta_pos . y (metrics.cpp:26-27), replicated on every shard
  std::vector<double> vp((size_t)h->N);
  CUDA_TRY(cudaMemcpy(vp.data(), h->vpos[h->ctrl_h->cur], sizeof(double) * h->N,
                      cudaMemcpyDeviceToHost));
  double pos = 0.0;
  for (int64_t l = 0; l < h->N; ++l) pos += (h->ctrl_h->s_cur * vp[l]) * y[l];
  out2[0] = r[1] + pos;
  out2[1] = out2[0] / ((double)h->N * (double)(h->N - 1));
  return CR_OK;
}

}  // extern "C"

namespace {
// Xq: host queries, or nullptr to evaluate at the data points themselves
cr_status estimator_impl(cr_handle* h, const double* y, const double* xi, const double* Xq,
                         int64_t Q, double* out) {
  CUDA_TRY(cudaSetDevice(h->device));
  PointBufs b;
  cr_status s = upload_point(h, y, xi, b);
  if (s != CR_OK) return s;
  double *dq = nullptr, *dout = nullptr;
  g_alloc_stream = h->st;
  if ((Xq && dalloc(&dq, (size_t)(Q * h->n)) != cudaSuccess) ||
      dalloc(&dout, (size_t)Q) != cudaSuccess) {
    cudaGetLastError();
    dfree(dq, h->st);
    return fail(h, CR_ENOMEM, "estimator buffers");
  }
  cudaError_t e = cudaSuccess;
  if (Xq) e = cudaMemcpyAsync(dq, Xq, sizeof(double) * Q * h->n, cudaMemcpyHostToDevice, h->st);
  const double* qsrc = Xq ? dq : h->X;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  if (e == cudaSuccess)
    e = launch_estimator(qsrc, Q, h->X, b.y, b.xi, h->N, (int)h->n, dout, sms * 8, h->st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, dout, sizeof(double) * Q, cudaMemcpyDeviceToHost, h->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->st);
  dfree(dq, h->st);
  dfree(dout, h->st);
  CUDA_TRY(e);
  return CR_OK;
}

}  // namespace

extern "C" {

cr_status cr_evaluate_estimator(cr_handle* h, const double* y, const double* xi,
                                const double* Xq, int64_t Q, double* out) {
  if (!h || !y || !xi || !Xq || !out || Q < 0) return CR_EINVAL;
  if (Q == 0) return CR_OK;
  return estimator_impl(h, y, xi, Xq, Q, out);
}

cr_status cr_repair_feasibility(cr_handle* h, const double* y, const double* xi, double* y_out) {
  if (!h || !y || !xi || !y_out) return CR_EINVAL;
  return estimator_impl(h, y, xi, nullptr, h->N, y_out);  // metrics.cpp:50-56
}

}  // extern "C"
