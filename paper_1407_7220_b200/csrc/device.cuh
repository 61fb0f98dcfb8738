// device.cuh -- device-side data layout and launch interfaces of the
// singleton-block P-APG pair sweep (arXiv 1407.7220 reference:
// proj/core/src/papg.cpp:136-283, operators.cpp:128-180).
//
// HBM layout (one shard = global rows [r0, r0+R) of the N x N pair matrix):
//   V[2]      : R x ld fp64, row-major, ld = N rounded up to the strip width.
//               Unscaled projected multipliers v (theta1 = s * v, appendix A.3
//               of SURVEY.md). Diagonal and pad columns are held at exactly 0.
//   vpos[2]   : N fp64, the y >= 0 multipliers (replicated on every shard).
//   xbuf      : [rowsum N | colagg N x (n+1) | sweep scalars 4] fp64 -- the
//               aggregates of the newest V (linear, so aggregates of theta2
//               are the same combination of xbuf and aggsave). xbuf is the
//               NCCL allreduce payload of sharded runs.
//   aggsave   : the same aggregates for the previous V.
//   rowrec    : N x RQ  (x_l[0..n-1], 1, y_l, 0...)
//   colrec    : N x RQ  (-xi_l[0..n-1], -c_l, 1, 0...)   c_l = y_l - xi_l . x_l
//               so that (C eta)_{l1 l2} = colrec[l2] . rowrec[l1] (the MMA
//               residual), RQ = max(round_up(n+2, 4), round_up(n+1, 8)) + 2.
#pragma once
#include <cstdint>

namespace crb {

constexpr int kMaxN = 32;    // templated register path covers n = 1..kMaxN
// every per-n kernel table is generated from these two lists (keep them = 1..kMaxN)
#ifndef CRB_N_LIST  // (-DCRB_N_LIST=10: one-n builds for SASS inspection only)
#define CRB_N_LIST                                                                           \
  1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23, 24, 25, \
      26, 27, 28, 29, 30, 31, 32
#endif
#define CRB_N_SEQ(F)                                                                         \
  F(1), F(2), F(3), F(4), F(5), F(6), F(7), F(8), F(9), F(10), F(11), F(12), F(13), F(14),   \
      F(15), F(16), F(17), F(18), F(19), F(20), F(21), F(22), F(23), F(24), F(25), F(26),    \
      F(27), F(28), F(29), F(30), F(31), F(32)

// max(round_up(n+2, 4), round_up(n+1, 8)) + 2: the +2 makes the row pitch an odd
// multiple of 16 B, so the MMA aggregation fragment reads (8 lanes per row, 4 rows)
// are bank-conflict free and the residual fragment reads at most 2-way.
__host__ __device__ constexpr int rec_pitch(int n) {
  return (((n + 5) & ~3) > ((n + 8) & ~7) ? ((n + 5) & ~3) : ((n + 8) & ~7)) + 2;
}
constexpr int kScal = 4;     // sweep scalars: S_vv, S_vr, S_tr, S_nn
constexpr int kK2Scal = 8;   // primal scalars, see primal_kernel

// Device-resident solver state: papg.cpp:148-175 locals plus the deferred
// ball scale (theta1 = s_cur * V[cur]).
struct DevCtrl {
  long long ell;        // completed iterations
  long long max_iters;
  long long hist_cap;
  int cur;              // slot holding V_k
  int stopped;
  int reason;           // 0 thresholds, 1 iter budget, 2 time budget, 3 error
  int restarts;
  int max_restarts;
  int adaptive;
  int use_momentum;
  int record_history;
  int saturated;
  int halt;             // stopped || ell >= pause_at: kernels become no-ops
  long long pause_at;   // host-set iteration limit of the current iterate call
  // coefficients of theta2 = th1 + beta (th1 - th1p), th1 = s_cur V[cur],
  // th1p = s_prev V[1-cur]; read by the primal and sweep kernels
  double s_cur, s_prev, beta;
  double t;
  double B_theta;
  double g_star_upper;
  double invL;
  double gamma;
  double gap_tol, infeas_tol, inner_tol_floor, max_seconds;
  double gap_div, infeas_div, K;
  unsigned long long t_start_ns;
  // metrics of the last completed iteration (papg.cpp:191-208)
  double gap_raw, gap_norm, infeas_raw, infeas_norm, g_value, fw, theta1_norm;
  double objective, reg_objective;
  // general-K partition: |within-block infeasibility| of the current eta
  // (dual_gradient's within_infeas_raw, papg.cpp:128), host-set per iteration
  double within_raw;
};

// opaque CUtensorMap (cuda.h): 128 bytes, 64-byte aligned; encoded on the host
// (tmap.cu), read by the TMA unit from the kernel's parameter space
struct alignas(64) TmapBytes {
  unsigned long long w[16];
};

struct SweepArgs {
  // tensor maps of V[0], V[1] (3-D view {TC, T, R}; box = one 8-row stage x
  // (TC + 2) columns, the 2 out-of-bounds columns zero-filled into the
  // shared-memory row pitch of the DMMA sweep); used by its P-APG producer when
  // tmap != 0 -- one TMA per buffer and stage instead of one bulk copy per row
  TmapBytes tmV[2];
  int tmap;
  double* V0;             // V[0]; V[cur] is read, V[1-cur] is read (theta1_prev)
  double* V1;             // and then overwritten by v_{k+1}
  const int* cur;         // device slot index (DevCtrl::cur)
  const double* rowrec;   // N x RP
  const double* colrec;   // N x RP
  double* colpart;        // [G*maxspan][TC][n+1]: one slot per (CTA, segment)
  double* rowpart;        // [T][R]: one row-sum slice per column tile
  double* scalpart;       // [G*CW][kScal]
  const double* coef;     // {s_cur, s_prev, beta} (DevCtrl fields or constants)
  const int* stopped;     // nullptr: always run
  double invL;            // 1 / L_g (0 turns the step into a pure copy + aggregate)
  double cdiv;            // kModePenaltyUpdate: theta_{k+1} = v / cdiv (alcc.cpp:176)
  long long N, R, r0, ld;
  long long U;            // rows of the (tile, row) unit space per CTA
  int S;                  // column strips (32*C columns each)
  int T;                  // column tiles (CW strips each)
  int G;                  // CTAs (persistent, one wave)
  int maxspan;            // max segments (tiles) one CTA can touch
  long long nbar;         // block size of the partition: pairs inside one block are
                          // masked like the diagonal (1: singleton blocks)
  unsigned long long* stores;  // optional: multipliers written by the P-APG sweep
};

// same block of the partition. BLK = false: singleton blocks (the diagonal);
// the blocked test is a separate instantiation so the singleton kernels carry
// no 64-bit division code (it cost 17% of the cfg2 sweep, measured).
template <bool BLK>
__host__ __device__ __forceinline__ bool same_block(long long a, long long b, long long nbar) {
  if constexpr (BLK) return a / nbar == b / nbar;
  else return a == b;
}
// the row range [r0, r0 + nr) and column range [c0, c0 + nc) share no block
template <bool BLK>
__host__ __device__ __forceinline__ bool blocks_disjoint(long long r0, long long nr, long long c0,
                                                         long long nc, long long nbar) {
  if constexpr (BLK) return (r0 + nr - 1) / nbar < c0 / nbar || r0 / nbar > (c0 + nc - 1) / nbar;
  else return r0 + nr <= c0 || r0 >= c0 + nc;
}

// kModePapg:   the P-APG step above (reads V, V'; writes V')
// kModePower:  aggregates of the residual itself (sigma_max(C) by sweeps)
// kModePenalty / kModePenaltyUpdate: the ALCC penalty oracle (alcc.cpp:33-47,
//   :124-127): v = max(theta - row, 0) with theta = V[cur]; aggregates of v.
//   The update variant (outer step) also accumulates the scalars (S_vv, S_vr,
//   -, S_nn) and writes v / cdiv into V[1-cur] (the next multiplier, alcc.cpp:176).
enum SweepMode { kModePapg = 0, kModePower = 1, kModePenalty = 2, kModePenaltyUpdate = 3 };

// returns the kernel attribute table entry for (n, mode); host side helpers
struct SweepKernelInfo {
  const void* fn;
  int strip_cols;         // columns per consumer warp (W)
  int warps_per_block;    // consumer warps
  int max_blocks_per_sm;
  int tile_cols;          // TC = warps_per_block * strip_cols
  int scal_recs;          // sweep scalar records per CTA (scalpart [G * scal_recs][kScal])
  int threads;
  int smem_bytes;
};
enum SweepVariant { kSweepMma = 1 };  // the FP64 tensor-core sweep (the DFMA one was removed)
// blocked = true: same-block pairs of a K-block partition masked (kModePapg /
// kModePower only)
SweepKernelInfo sweep_mma_info(int n, int mode, bool blocked = false);   // sweep_mma.cu (DMMA)
int launch_sweep(const SweepKernelInfo& info, const SweepArgs& a, void* stream);

}  // namespace crb
