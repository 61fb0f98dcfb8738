// sweep.cu -- K1, the fused pair sweep: one HBM pass over the lambda stream
// per dual iteration.
//
// Replaces, for the singleton-block closed form, the reference's per-iteration
// passes: apply_C (operators.cpp:128-153), the projected step
// (papg.cpp:187-189, projections.hpp:9-13), the metric reductions
// (papg.cpp:191-208) and apply_C_T of the next iterate (operators.cpp:155-180).
//
// Per pair (l1 = row, l2 = column), with theta1 = s V, theta1_prev = s' V':
//   row   = y_l1 - c_l2 - x_l1 . xi_l2               (= (C eta)_{l1 l2})
//   th2   = th1 + beta (th1 - th1p)                   (papg.cpp:256-259)
//   v     = max(th2 - row / L, 0)                     (unscaled projection)
//   S_vv += v^2, S_vr += v row, S_tr += th2 row, S_nn += min(row,0)^2
//   colagg[l2] += (v, v x_l1), rowsum[l1] += v
// HBM traffic: 8 B read V, 8 B read V', 8 B write v -> 24 B per pair.
//
// CTA organisation (sm_100a): 8 consumer warps (4 for n > 10) + 1 producer
// warp. The CTA
// owns a tile of 8 adjacent column strips (32*C columns each, one per
// consumer warp) and a contiguous chunk of rows. The producer streams the
// chunk through an NS-stage shared-memory ring with cp.async.bulk (TMA bulk
// copies completing on mbarriers): per stage, TR rows of V and V' for the
// whole tile plus the TR row records (y, x). Consumers keep their columns'
// state (c, xi, colsum, V^T X) in registers for the whole chunk, read V/V'
// with conflict-free 16-byte shared loads, write v with 16-byte streaming
// global stores, and reduce row sums through a 32-row shared transpose.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "pipeline.cuh"

namespace crb {

namespace {

constexpr int kNS = 4;       // pipeline stages

template <int NN>
__host__ __device__ constexpr int cols_per_lane() { return NN <= 10 ? 2 : 1; }
// consumer warps per CTA: fewer for wide n so each thread may hold 255 registers
template <int NN>
__host__ __device__ constexpr int consumer_warps() { return NN <= 10 ? 8 : 4; }
template <int NN>
__host__ __device__ constexpr int threads_per_cta() { return (consumer_warps<NN>() + 1) * 32; }
template <int NN>
__host__ __device__ constexpr int rows_per_stage() { return cols_per_lane<NN>() == 2 ? 4 : 8; }
template <int NN>
__host__ __device__ constexpr int tile_cols() {
  return consumer_warps<NN>() * 32 * cols_per_lane<NN>();
}
// doubles per stage: V and V' rows for the tile + row records
template <int NN>
__host__ __device__ constexpr int stage_doubles() {
  return 2 * rows_per_stage<NN>() * tile_cols<NN>() + rows_per_stage<NN>() * rec_pitch(NN);
}
constexpr int kRsPitch = 17;  // per-warp row-sum transpose: 32 rows x 16 lanes (+1 pad)
template <int NN>
__host__ __device__ constexpr int smem_bytes() {
  return kNS * stage_doubles<NN>() * 8 + consumer_warps<NN>() * 32 * kRsPitch * 8 +
         2 * consumer_warps<NN>() * 32 * 8 + 2 * kNS * 8;
}

template <int C> struct VecT;
template <> struct VecT<1> { using T = double; };
template <> struct VecT<2> { using T = double2; };

__device__ __forceinline__ double vget(const double& v, int) { return v; }
__device__ __forceinline__ double vget(const double2& v, int k) { return k == 0 ? v.x : v.y; }
__device__ __forceinline__ void vset(double& v, int, double x) { v = x; }
__device__ __forceinline__ void vset(double2& v, int k, double x) {
  if (k == 0) v.x = x; else v.y = x;
}

// ---- consumer building blocks ---------------------------------------------
template <int NN, int C>
struct ColState {       // registers of one lane's C columns
  double cc[C];         // c_l2 = y_l2 - xi_l2 . x_l2
  double xi[C][NN];
  double acc[C][NN + 1];  // colsum, (V^T X)_l2
  bool valid[C];
};
struct Coef {
  double s_c, s_p, beta, invL, cdiv;
};
struct Scal {
  double vv, vr, tr, nn;
};
struct StageView {
  const double* vc;   // smem V   row 0 at this lane's columns (row stride TC)
  const double* vp;   // smem V'  row 0
  const double* rec;  // smem row records (stride RP)
  double* gout;       // global V' row 0 at this lane's columns (row stride ld)
  long long ld;
  long long col0;     // global column of this lane's first column
  long long g0;       // global row of stage row 0
  double* srs;        // row-sum transpose slot of stage row 0
  long long nbar;     // partition block size (same-block pairs masked)
};

template <int NN, int MODE, int TR, int TC, bool MASK, bool UNIT, bool BLK>
__device__ __forceinline__ void run_stage(const StageView& sv, int nr, int lane,
                                          ColState<NN, cols_per_lane<NN>()>& cs, const Coef& cf,
                                          Scal& sc) {
  constexpr int C = cols_per_lane<NN>();
  constexpr int RP = rec_pitch(NN);
  using VT = typename VecT<C>::T;
#pragma unroll
  for (int q = 0; q < TR; ++q) {
    if (q < nr) {
      const double* xr = sv.rec + q * RP;  // (x, 1, y)
      double x[NN];
      const double y1 = xr[NN + 1];
#pragma unroll
      for (int j = 0; j < NN; ++j) x[j] = xr[j];
      VT vc, vp, out;
      if (MODE == kModePapg) {
        vc = *reinterpret_cast<const VT*>(sv.vc + q * TC);
        vp = *reinterpret_cast<const VT*>(sv.vp + q * TC);
      } else if (MODE == kModePenalty || MODE == kModePenaltyUpdate) {
        vc = *reinterpret_cast<const VT*>(sv.vc + q * TC);
      }
      double rs = 0.0;
#pragma unroll
      for (int k = 0; k < C; ++k) {
        // colrec holds (-xi, -c): row = y1 - c - x.xi, two FMA chains for ILP
        double ra = y1 + cs.cc[k], rb = 0.0;
#pragma unroll
        for (int j = 0; j < NN; j += 2) {
          ra = fma(x[j], cs.xi[k][j], ra);
          if (j + 1 < NN) rb = fma(x[j + 1], cs.xi[k][j + 1], rb);
        }
        double row = ra + rb;
        if (MASK && (!cs.valid[k] || same_block<BLK>(sv.col0 + k, sv.g0 + q, sv.nbar))) row = 0.0;
        double v;
        if (MODE == kModePapg) {
          double th2;
          if (UNIT) {
            const double c1 = vget(vc, k);
            th2 = fma(cf.beta, c1 - vget(vp, k), c1);
          } else {
            const double th1 = cf.s_c * vget(vc, k);
            th2 = fma(cf.beta, th1 - cf.s_p * vget(vp, k), th1);
          }
          v = keep_if_nonneg(fma(-row, cf.invL, th2));
          vset(out, k, v);
          sc.vv = fma(v, v, sc.vv);
          sc.vr = fma(v, row, sc.vr);
          sc.tr = fma(th2, row, sc.tr);
          const double m = keep_if_neg(row);
          sc.nn = fma(m, m, sc.nn);
        } else if (MODE == kModePenalty || MODE == kModePenaltyUpdate) {
          v = keep_if_nonneg(vget(vc, k) - row);
          if (MODE == kModePenaltyUpdate) {  // outer step: statistics + theta_{k+1}
            vset(out, k, v / cf.cdiv);
            sc.vv = fma(v, v, sc.vv);
            sc.vr = fma(v, row, sc.vr);
            const double m = keep_if_neg(row);
            sc.nn = fma(m, m, sc.nn);
          }
        } else {
          v = row;
          sc.vv = fma(row, row, sc.vv);
        }
        cs.acc[k][0] += v;
#pragma unroll
        for (int j = 0; j < NN; ++j) cs.acc[k][1 + j] = fma(v, x[j], cs.acc[k][1 + j]);
        rs += v;
      }
      if (MODE == kModePenaltyUpdate) st_stream(reinterpret_cast<VT*>(sv.gout + q * sv.ld), out);
      if (MODE == kModePapg) {
        // v goes into the buffer that holds vp (theta1_prev): skip unchanged values
        bool changed = false;
#pragma unroll
        for (int k = 0; k < C; ++k)
          changed |= __double_as_longlong(vget(out, k)) != __double_as_longlong(vget(vp, k));
        if (changed) st_stream(reinterpret_cast<VT*>(sv.gout + q * sv.ld), out);
      }
      rs += __shfl_xor_sync(0xffffffffu, rs, 16);
      if (lane < 16) sv.srs[q * kRsPitch + lane] = rs;
    }
  }
}

template <int NN, int MODE, bool BLK>
__global__ void __launch_bounds__(threads_per_cta<NN>()) sweep_kernel(const SweepArgs a) {
  constexpr int kCW = consumer_warps<NN>();
  constexpr int C = cols_per_lane<NN>();
  constexpr int W = 32 * C;
  constexpr int RP = rec_pitch(NN);
  constexpr int TR = rows_per_stage<NN>();
  constexpr int TC = tile_cols<NN>();
  constexpr int SD = stage_doubles<NN>();
  extern __shared__ __align__(128) double smem[];
  double* stages = smem;
  double* srs_all = smem + kNS * SD;
  double* rowacc = srs_all + kCW * 32 * kRsPitch;  // [2][kCW][32] CTA row-sum combine
  uint64_t* full = reinterpret_cast<uint64_t*>(rowacc + 2 * kCW * 32);
  uint64_t* empty = full + kNS;

  if (a.stopped != nullptr && *a.stopped) return;
  const int cur = (MODE != kModePower) ? *a.cur : 0;
  constexpr bool kPen = MODE == kModePenalty || MODE == kModePenaltyUpdate;
  const double* Vc = cur ? a.V1 : a.V0;
  double* Vp = cur ? a.V0 : a.V1;

  // Persistent balanced split: the (tile, row) unit space of T * R rows is
  // cut into G equal contiguous ranges, one per CTA; a range covers one or a
  // few "segments" (a row range of one column tile).
  const long long units = (long long)a.T * a.R;
  const long long u0 = (long long)blockIdx.x * a.U;
  const long long u1 = min(u0 + a.U, units);
  if (u0 >= u1) return;
  const int t_first = (int)(u0 / a.R);
  const int t_last = (int)((u1 - 1) / a.R);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCW) {  // ------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      int i = 0;  // global stage counter
      for (int t = t_first; t <= t_last; ++t) {
        const long long rlo = max(u0, (long long)t * a.R) - (long long)t * a.R;
        const long long rhi = min(u1, (long long)(t + 1) * a.R) - (long long)t * a.R;
        const long long c0 = (long long)t * TC;
        const uint32_t vbytes = (uint32_t)min((long long)TC, a.ld - c0) * 8u;
        for (long long r = rlo; r < rhi; r += TR, ++i) {
          const int s = i % kNS;
          if (i >= kNS) mbar_wait(&empty[s], (uint32_t)(((i / kNS) - 1) & 1));
          const int nr = (int)min((long long)TR, rhi - r);
          double* st = stages + s * SD;
          const uint32_t bytes = (MODE == kModePapg ? 2u * nr * vbytes : 0u) +
                                 (kPen ? (uint32_t)nr * vbytes : 0u) + (uint32_t)nr * RP * 8u;
          mbar_arrive_expect_tx(&full[s], bytes);
          if (MODE == kModePapg) {
            for (int q = 0; q < nr; ++q) {
              const long long off = (r + q) * a.ld + c0;
              bulk_g2s(st + q * TC, Vc + off, vbytes, &full[s], pol_stream);
              bulk_g2s(st + (TR + q) * TC, Vp + off, vbytes, &full[s], pol_stream);
            }
          } else if (kPen) {
            for (int q = 0; q < nr; ++q)
              bulk_g2s(st + q * TC, Vc + (r + q) * a.ld + c0, vbytes, &full[s], pol_stream);
          }
          bulk_g2s(st + 2 * TR * TC, a.rowrec + (a.r0 + r) * RP, (uint32_t)nr * RP * 8u,
                   &full[s], pol_keep);
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  double* srs = srs_all + warp * 32 * kRsPitch;
  const int lane_off = warp * W + lane * C;
  Coef cf{1.0, 0.0, 0.0, a.invL, a.cdiv};
  if (MODE == kModePapg) {
    cf.s_c = a.coef[0];
    cf.s_p = a.coef[1];
    cf.beta = a.coef[2];
  }
  const bool unit_scale = (cf.s_c == 1.0) && (cf.s_p == 1.0);
  Scal sc{0.0, 0.0, 0.0, 0.0};
  int i = 0;        // global stage counter (matches the producer)
  int flushes = 0;  // row-sum combine buffer parity

  for (int t = t_first; t <= t_last; ++t) {
    const long long rlo = max(u0, (long long)t * a.R) - (long long)t * a.R;
    const long long rhi = min(u1, (long long)(t + 1) * a.R) - (long long)t * a.R;
    const long long c0 = (long long)t * TC;
    const int strip = t * kCW + warp;
    const bool active = strip < a.S;
    const long long col0 = c0 + warp * W + lane * C;  // first column of this lane

    ColState<NN, C> cs;
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const long long col = col0 + k;
      cs.valid[k] = active && col < a.N;
      const double* rec = a.colrec + (cs.valid[k] ? col : 0) * RP;  // (-xi, -c, 1)
      cs.cc[k] = cs.valid[k] ? __ldg(rec + NN) : 0.0;
#pragma unroll
      for (int j = 0; j < NN; ++j) cs.xi[k][j] = cs.valid[k] ? __ldg(rec + j) : 0.0;
#pragma unroll
      for (int j = 0; j <= NN; ++j) cs.acc[k][j] = 0.0;
    }
    // warp-uniform: every column of the strip is a real column
    const bool strip_full = active && (c0 + (long long)(warp + 1) * W <= a.N);
    const long long strip_lo = c0 + (long long)warp * W;
    int win = 0;               // rows held in the row-sum transpose window
    long long win_base = rlo;  // local row of window slot 0

    for (long long r = rlo; r < rhi; r += TR, ++i) {
      const int s = i % kNS;
      mbar_wait(&full[s], (uint32_t)((i / kNS) & 1));
      const int nr = (int)min((long long)TR, rhi - r);
      if (active) {
        const double* st = stages + s * SD;
        StageView sv{st + lane_off, st + TR * TC + lane_off, st + 2 * TR * TC,
                     Vp + r * a.ld + col0, a.ld, col0, a.r0 + r, srs + win * kRsPitch,
                     a.nbar};
        // the diagonal (a same-block pair) or a pad column touches this stage:
        // per-pair masks
        const bool clean = strip_full && blocks_disjoint<BLK>(sv.g0, nr, strip_lo, W, a.nbar);
        if (clean) {
          if (unit_scale) run_stage<NN, MODE, TR, TC, false, true, BLK>(sv, nr, lane, cs, cf, sc);
          else run_stage<NN, MODE, TR, TC, false, false, BLK>(sv, nr, lane, cs, cf, sc);
        } else {
          if (unit_scale) run_stage<NN, MODE, TR, TC, true, true, BLK>(sv, nr, lane, cs, cf, sc);
          else run_stage<NN, MODE, TR, TC, true, false, BLK>(sv, nr, lane, cs, cf, sc);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      win += nr;
      if (win == 32 || r + TR >= rhi) {
        // per-warp row sums of the window (lane i <-> row i), then a
        // fixed-order sum over the CTA's warps into the tile's row-sum slice
        double tsum = 0.0;
        if (active && lane < win) {
#pragma unroll
          for (int l = 0; l < 16; ++l) tsum += srs[lane * kRsPitch + l];
        }
        double* ra = rowacc + (flushes & 1) * kCW * 32;
        ra[warp * 32 + lane] = tsum;
        asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");
        if (warp == 0 && lane < win) {
          double u = 0.0;
#pragma unroll
          for (int w = 0; w < kCW; ++w) u += ra[w * 32 + lane];
          a.rowpart[(long long)t * a.R + win_base + lane] = u;
        }
        __syncwarp();
        win_base += win;
        win = 0;
        ++flushes;
      }
    }
    // column partials of this segment: slot (CTA, segment index)
    if (active) {
      const long long slot = (long long)blockIdx.x * a.maxspan + (t - t_first);
#pragma unroll
      for (int k = 0; k < C; ++k) {
        double* dst = a.colpart + (slot * TC + warp * W + lane * C + k) * (NN + 1);
#pragma unroll
        for (int j = 0; j <= NN; ++j) dst[j] = cs.acc[k][j];
      }
    }
  }

  double vv = sc.vv, vr = sc.vr, tr = sc.tr, nn = sc.nn;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {  // fixed butterfly: deterministic
    vv += __shfl_xor_sync(0xffffffffu, vv, off);
    vr += __shfl_xor_sync(0xffffffffu, vr, off);
    tr += __shfl_xor_sync(0xffffffffu, tr, off);
    nn += __shfl_xor_sync(0xffffffffu, nn, off);
  }
  if (lane == 0) {
    double* sp = a.scalpart + ((long long)blockIdx.x * kCW + warp) * kScal;
    sp[0] = vv;
    sp[1] = vr;
    sp[2] = tr;
    sp[3] = nn;
  }
}

template <int NN>
SweepKernelInfo info_for(int mode, bool blocked) {
  SweepKernelInfo inf{};
  if (blocked) {
    inf.fn = mode == kModePapg    ? (const void*)sweep_kernel<NN, kModePapg, true>
             : mode == kModePower ? (const void*)sweep_kernel<NN, kModePower, true>
                                  : nullptr;
    if (!inf.fn) return inf;
  } else {
    inf.fn = mode == kModePapg      ? (const void*)sweep_kernel<NN, kModePapg, false>
             : mode == kModePower   ? (const void*)sweep_kernel<NN, kModePower, false>
             : mode == kModePenalty ? (const void*)sweep_kernel<NN, kModePenalty, false>
                                    : (const void*)sweep_kernel<NN, kModePenaltyUpdate, false>;
  }
  inf.strip_cols = 32 * cols_per_lane<NN>();
  inf.warps_per_block = consumer_warps<NN>();
  inf.scal_recs = consumer_warps<NN>();
  inf.tile_cols = tile_cols<NN>();
  inf.threads = threads_per_cta<NN>();
  inf.smem_bytes = smem_bytes<NN>();
  cudaFuncSetAttribute(inf.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, inf.smem_bytes);
  int bps = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, inf.fn, inf.threads, inf.smem_bytes) !=
      cudaSuccess)
    bps = 0;
  inf.max_blocks_per_sm = bps;
  return inf;
}

template <int... Ns> struct Table;
template <int N0, int... Ns> struct Table<N0, Ns...> {
  static SweepKernelInfo info(int n, int mode, bool blocked) {
    return n == N0 ? info_for<N0>(mode, blocked) : Table<Ns...>::info(n, mode, blocked);
  }
};
template <> struct Table<> {
  static SweepKernelInfo info(int, int, bool) { return SweepKernelInfo{}; }
};
using AllN = Table<CRB_N_LIST>;

}  // namespace

SweepKernelInfo sweep_dfma_info(int n, int mode, bool blocked) {
  return AllN::info(n, mode, blocked);
}

int launch_sweep(const SweepKernelInfo& info, const SweepArgs& a, void* stream) {
  void* args[] = {const_cast<SweepArgs*>(&a)};
  return (int)cudaLaunchKernel(info.fn, dim3((unsigned)a.G), dim3(info.threads), args,
                               info.smem_bytes, (cudaStream_t)stream);
}

}  // namespace crb
