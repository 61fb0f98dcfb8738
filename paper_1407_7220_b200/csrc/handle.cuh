// handle.cuh -- the C-ABI handle (include/cvxreg_b200.h: cr_handle) shared by
// capi.cu (P-APG, metrics, sharding) and alcc.cu (standalone ALCC), plus the
// small helpers both use (error capture, pooled allocation, sweep/reduce args).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cvxreg_b200.h"
#include "device.cuh"
#include "kernels.cuh"
#include "small.cuh"

namespace crb {
struct AlccDev;  // alcc.cu
struct AlccBufs {
  AlccDev* dev = nullptr;       // device-resident MAPG / outer state
  AlccDev* host = nullptr;      // pinned mirror
  double *p1 = nullptr, *p1p = nullptr, *p2 = nullptr;  // [y | xi] points (N (n+1))
  // block mode (general-K P-APG sub-problem): centres and the feasible slice;
  // cy == nullptr means the standalone centres (ybar, 0)
  double *cy = nullptr, *cxi = nullptr, *fy = nullptr, *fxi = nullptr;
  double *part1 = nullptr, *part2 = nullptr;            // per-block partials
  unsigned int* counter = nullptr;
  SweepKernelInfo kpen{}, kupd{};
  cudaGraphExec_t gexec = nullptr;
  int graph_iters = 0;
  int blocks = 0;
  // small sub-problems: cooperative MAPG loop (grid, strips, row chunks, partials)
  int loop_G = 0, loop_S = 0, loop_P = 0;
  double *lcolpart = nullptr, *lrowpart = nullptr, *lpartB = nullptr, *lpartC = nullptr;
  bool done = false;            // a finished solve is on the handle (multiplier export)
  double mu = 0;                // mu of the last outer step
};
// general-K P-APG(ALCC) state (general.cu): K blocks of nbar points, one ALCC
// sub-problem handle per block (alcc_solve_block, alcc.cpp:222-258)
struct Partition {
  int64_t K = 0, nbar = 1;
  std::vector<cr_handle*> blocks;
  cr_alcc_config inner{};
  double sigma_A1 = 0;                 // within A1 (the same in every block)
  std::vector<double> sigma_A2;        // within A2 per block
  std::vector<double> block_infeas;    // last ALCC infeasibility per block
  double *cy = nullptr, *cxi = nullptr;      // block centres ybar + q_y, q_xi / gamma
  double *qy = nullptr, *qxi = nullptr;      // C^T theta2 (objective terms)
  double *th2pos = nullptr;                  // theta2 of the y >= 0 rows
  double *ey = nullptr, *exi = nullptr;      // eta (block minimisers)
  double *fy = nullptr, *fxi = nullptr;      // feasible affine point (prepare_problem)
  int64_t inner_iters = 0;
  double inner_seconds = 0;
  int workers = 0;                     // concurrent block solves (PapgConfig::workers); 0: 16
  // small blocks: all block ALCCs in one launch, one CTA per block (balcc.cu)
  bool batched = false;
  double *w_theta = nullptr, *w_y1p = nullptr, *w_y2 = nullptr, *w_x1p = nullptr,
         *w_x2 = nullptr, *w_cc = nullptr, *w_rs = nullptr, *w_cs = nullptr, *w_vx = nullptr,
         *w_infeas = nullptr;
  long long* w_iters = nullptr;
  int* w_status = nullptr;
  double* d_sigma_A2 = nullptr;        // device copy of sigma_A2
  double* w_scratch = nullptr;         // batched sweep partials
};
}  // namespace crb

using namespace crb;  // the ABI translation units all work in crb

// One canonical row block of the shard (cr_set_canonical_blocks): rows
// [a, a + R) of the local buffers swept by their own launch, with their own
// CTA shares and partial slots, so its payload does not depend on which GPU
// holds the block or on how many blocks share that GPU.
struct CanonBlock {
  int64_t a = 0, R = 0;
  long long U = 0;
  int G = 0, maxspan = 0;
  double *colpart = nullptr, *rowpart = nullptr, *scalpart = nullptr;
  TmapBytes tmV[2] = {};
  bool tmap_ok = false;
};

struct cr_handle {
  int device = 0;
  cudaStream_t st = nullptr;
  int64_t N = 0, n = 0, r0 = 0, r1 = 0, R = 0, ld = 0;
  int RP = 0;
  double gamma = 1e-3;
  SweepKernelInfo kp{}, kw{};
  int S = 0;            // column strips
  int T = 0;            // sweep CTA column tiles = row-sum slices
  int variant = kSweepMma;
  // persistent small-N loop (small.cu)
  bool small_mode = false;
  SmallInfo ks{};
  int small_grid = 0, small_S = 0, small_P = 0;
  int small_RT = 0;          // > 0: resident variant (V, V' tiles in shared memory), tile rows
  size_t small_smem = 0;     // its dynamic shared memory per block
  double *s_colpart = nullptr, *s_rowpart = nullptr, *s_scalpart = nullptr, *s_k2part = nullptr;
  int G = 0;            // sweep CTAs (one persistent wave)
  int maxspan = 0;      // tiles one CTA's unit range can touch
  long long U = 0;      // (tile, row) units per CTA
  int k2_blocks = 0;
  unsigned int* counter = nullptr;
  unsigned long long* d_stores = nullptr;  // multipliers written by the P-APG sweeps
  TmapBytes tmV[2] = {};    // tensor maps of V[0], V[1] for the DMMA P-APG producer
  bool tmap_ok = false;
  bool primal_pending = true; // enqueue the (possibly no-op) standalone primal next
  // device buffers
  double *X = nullptr, *ybar = nullptr, *rowrec = nullptr, *colrec = nullptr;
  double *V[2] = {nullptr, nullptr}, *vpos[2] = {nullptr, nullptr};
  double *xbuf = nullptr, *aggsave = nullptr;
  double *colpart = nullptr, *rowpart = nullptr, *scalpart = nullptr;
  double *k2part = nullptr, *k2sum = nullptr, *hist = nullptr;
  double *yout = nullptr, *xiout = nullptr;
  double *pw_u = nullptr, *pw_v = nullptr, *pw_part = nullptr, *pw_sum = nullptr;
  double *gram = nullptr, *ps_part = nullptr, *ps_part2 = nullptr, *ps_state = nullptr;
  int power_grid = 0;  // closed-form power iteration (power.cu)
  bool sigma_by_sweep = false;  // CRB_SIGMA=sweep: O(N^2 n) power steps through the sweep
  double *consts = nullptr;  // {1, 1, 0}
  int *izero = nullptr;      // constant 0 (slot index / never halted)
  double *stage = nullptr;
  int64_t stage_elems = 0;
  int64_t hist_cap = 0;
  DevCtrl* ctrl_d = nullptr;
  DevCtrl* ctrl_h = nullptr;     // pinned mirror (latest copy)
  DevCtrl* ctrl_poll = nullptr;  // pinned, 2 polling slots
  long long* pause_h = nullptr;  // pinned {pause_at, halt}
  // canonical row blocks (GPU-count-invariant sums); empty: off
  std::vector<CanonBlock> canon;
  int canon_D = 0, canon_first = 0;
  double* canon_pay = nullptr;  // [canon_D][payload_len]: every block's payload
  // NCCL
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // loop state
  cr_papg_config cfg{};
  bool begun = false;
  int graph_iters = 0;  // 0: direct launches
  cudaGraphExec_t gexec = nullptr;
  double sigma_C = 0, L = 0, sigma_seconds = 0;
  int sigma_iters = 0, sigma_conv = 1;
  std::chrono::steady_clock::time_point t_begin;
  double loop_seconds = 0;
  // timing
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_poll[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> ev_sweep;  // pairs
  // sigma_max(C) start vector (rng_stream(0x5eed, 97), normalised), drawn on a
  // host thread while the handle's device state is set up
  std::thread sigma_prep;
  std::vector<double> sigma_start;  // uniform pairs of the sigma start vector (host drawn):
  double* sigma_start_pin = nullptr;  // pinned block from the process pool when available,
  size_t sigma_start_bytes = 0;       // else the vector; sigma_start_ptr points at the one in use
  double* sigma_start_ptr = nullptr;
  int64_t sigma_start_cols = 0;
  double* out_pin = nullptr;          // pinned staging of (y, xi) for cr_papg_finish
  size_t out_pin_bytes = 0;
  double* sv_u12 = nullptr;          // their device copy + 256 doubles of block partials
  double last_seconds = 0, last_sweep_seconds = 0;
  std::vector<double> last_sweep_times;  // per bracketed sweep launch of the last call (s)
  double last_exchange_seconds = 0;      // sharded: allreduce time of the last call (s)
  int64_t last_launches = 0;
  // standalone ALCC (alcc.cu)
  crb::AlccBufs alcc{};
  // general-K partition (general.cu); K == 0: singleton blocks
  crb::Partition part{};
  std::string err;
};

inline cr_status fail(cr_handle* h, cr_status s, const std::string& what) {
  if (h) h->err = what;
  return s;
}

#define CUDA_TRY(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(h, CR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

#define NCCL_TRY(call)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      return fail(h, CR_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));      \
  } while (0)

// Device buffers come from the device's stream-ordered memory pool, which is
// told to keep freed memory: a service that creates a handle per solve reuses
// the mapping instead of paying cudaMalloc/cudaFree of gigabytes each time.
extern cudaStream_t g_alloc_stream;  // stream of the handle being created (capi.cu)
// On failure the pool's retained (freed) memory is returned to the device and
// the allocation retried once: a 160 GB handle after a 40 GB one in the same
// process must not fail on memory the pool only keeps for reuse.
template <typename T>
inline cudaError_t dalloc(T** p, size_t count) {
  const size_t bytes = (count ? count : 1) * sizeof(T);
  cudaError_t e = cudaMallocAsync((void**)p, bytes, g_alloc_stream);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess &&
        cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaMemPoolTrimTo(pool, 0);
      e = cudaMallocAsync((void**)p, bytes, g_alloc_stream);
    }
  }
  return e;
}
inline void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}
inline void keep_pool_memory(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

// [row sums N | colagg N(n+1) | kScal sweep scalars | clock]: the clock slot
// carries the elapsed seconds of the shard that owns row 0 (0 elsewhere), so
// the summed payload gives every rank the same time-budget decision
inline int64_t payload_len(const cr_handle* h) { return h->N * (h->n + 2) + kScal + 1; }

inline SweepArgs sweep_args(cr_handle* h, int mode, bool agg_only) {
  SweepArgs a{};
  a.V0 = h->V[0];
  a.V1 = h->V[1];
  a.cur = &h->ctrl_d->cur;
  a.rowrec = h->rowrec;
  a.colrec = h->colrec;
  a.colpart = h->colpart;
  a.rowpart = h->rowpart;
  a.scalpart = h->scalpart;
  a.coef = agg_only ? h->consts : &h->ctrl_d->s_cur;
  a.stopped = (mode == kModePapg && !agg_only) ? &h->ctrl_d->halt : nullptr;
  a.invL = agg_only ? 0.0 : 1.0 / h->L;
  a.N = h->N;
  a.R = h->R;
  a.r0 = h->r0;
  a.ld = h->ld;
  a.S = h->S;
  a.T = h->T;
  a.G = h->G;
  a.U = h->U;
  a.maxspan = h->maxspan;
  a.nbar = h->part.K > 0 ? h->part.nbar : 1;
  a.stores = h->d_stores;
  if ((mode == kModePapg || mode == kModePenalty || mode == kModePenaltyUpdate) && h->tmap_ok) {
    a.tmV[0] = h->tmV[0];
    a.tmV[1] = h->tmV[1];
    a.tmap = 1;
  }
  return a;
}
// the P-APG sweep of this solve
inline const SweepKernelInfo& papg_sweep(const cr_handle* h) { return h->kp; }

inline ReduceArgs reduce_args(cr_handle* h, bool with_k2, const int* stopped, bool fuse_control,
                              int sweep_warps = 0 /* scalar records per sweep CTA */) {
  ReduceArgs a{};
  a.colpart = h->colpart;
  a.rowpart = h->rowpart;
  a.scalpart = h->scalpart;
  a.k2part = h->k2part;
  a.agg_out = h->xbuf;
  a.k2sum = with_k2 ? h->k2sum : nullptr;
  a.stopped = stopped;
  a.rank = h->rank;
  a.ctrl = fuse_control ? h->ctrl_d : nullptr;
  a.clk = with_k2 ? h->ctrl_d : nullptr;
  a.hist = h->hist;
  a.counter = h->counter;
  a.N = h->N;
  a.ld = h->ld;
  a.R = h->R;
  a.r0 = h->r0;
  a.nw = (long long)h->G * (sweep_warps > 0 ? sweep_warps : h->kp.scal_recs);
  a.nk2 = with_k2 ? h->k2_blocks : 0;
  a.n1 = (int)h->n + 1;
  a.S = h->T;
  a.TC = h->kp.tile_cols;
  a.G = h->G;
  a.U = h->U;
  a.maxspan = h->maxspan;
  return a;
}
