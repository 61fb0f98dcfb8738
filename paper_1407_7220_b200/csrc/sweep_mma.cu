// sweep_mma.cu -- K1 on the FP64 tensor cores (mma.sync m8n8k4 f64 -> DMMA).
//
// Same contract as sweep.cu (one HBM pass per dual iteration, 24 B per pair;
// reference: operators.cpp:128-180, papg.cpp:187-208) but the two rank-n
// contractions of the pair sweep run as 8x8x4 fp64 MMAs:
//
//   residual     row^T (8 cols x 8 rows) = Xi'(8 x K) . X'^T(K x 8)
//                with Xi'_l = (-xi_l, -c_l, 1), X'_l = (x_l, 1, y_l), K = n+2 -> mult. of 4
//   aggregation  (V^T [X 1])^T (F x 8 cols) += [X 1]^T(F x 4 rows) . V(4 rows x 8 cols)
//
// The residual's accumulator fragment puts (col = lane/4, rows 2(lane%4)+{0,1})
// in each thread. Splitting the 8 rows of a tile into the k-steps {0,2,4,6}
// and {1,3,5,7} makes exactly those two values the B fragments of the two
// aggregation MMAs (B[k=lane%4][n=lane/4]), so v never moves between lanes.
//
// CTA: 15 consumer warps x (2 tiles of 8 columns) = 240 columns, 1 producer
// warp streaming 8-row stages of V, V' and the row records through a 4-deep
// cp.async.bulk / mbarrier ring (row pitch padded by 16 B: conflict-free
// column-fragment reads). Work split, partial layouts and row-sum combine are
// identical to sweep.cu.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "device.cuh"
#include "mma_geo.cuh"
#include "pipeline.cuh"

// producer back-off while a slot drains (ns)
#ifndef CRB_PROD_SLEEP
#define CRB_PROD_SLEEP 64
#endif
// measurement probe only (wrong results): consumers skip the P-APG stage work,
// leaving the TMA ring, barriers and row-sum flushes (the memory-side floor)
#ifndef CRB_PROBE_MEMONLY
#define CRB_PROBE_MEMONLY 0
#endif
#ifndef CRB_LEAN_ORDER  // 1: a tile's aggregation MMAs issued before its stores and sums
#define CRB_LEAN_ORDER 1
#endif
// 1: the singleton sweep leaves theta2 . row to K2 (PrimalArgs::tr_adjoint);
// must agree with primal_args() in capi.cu
#ifndef CRB_TR_ADJOINT
#define CRB_TR_ADJOINT 1
#endif
#ifndef CRB_PROBE_NOWAIT  // probe: producer fills the ring once, consumers never wait (compute only)
#define CRB_PROBE_NOWAIT 0
#endif
#ifndef CRB_RS_SMEM  // lean P-APG loop: row sums through a 32-row shared window, no shuffles
#define CRB_RS_SMEM 1
#endif
#ifndef CRB_PROBE_SKIP  // measurement probe (wrong results): 1 residual, 2 aggregation, 4 sums, 8 row-sum shuffles
#define CRB_PROBE_SKIP 0
#endif
#ifndef CRB_PROBE_TIMING  // measurement probe: clock64 wait accounting, printf from 2 CTAs
#define CRB_PROBE_TIMING 0
#endif

namespace crb {

namespace {

// P-APG aggregation of one tile's v (fragment rows 2q, 2q+1 of column c8):
// the DMMA feature blocks, then the DFMA remainder (agg_split: the last x
// features and the column sum, accumulated per lane and reduced over q at the
// end of the segment).
template <int NN>
__device__ __forceinline__ void papg_agg(const double (&Ag)[2][max1(agg_fbd<NN>())],
                                         const double (&xr)[2][max1(agg_rx<NN>())], const double (&v)[2],
                                         double (&D)[max1(agg_fbd<NN>())][2], double (&E)[max1(agg_re<NN>())]) {
  constexpr int FBD = agg_fbd<NN>();
  constexpr int RX = agg_rx<NN>();
#pragma unroll
  for (int fb = 0; fb < FBD; ++fb) {
    dmma(D[fb][0], D[fb][1], Ag[0][fb], v[0]);
    dmma(D[fb][0], D[fb][1], Ag[1][fb], v[1]);
  }
  if constexpr (agg_re<NN>() > 0) {
#pragma unroll
    for (int r = 0; r < RX; ++r) E[r] = fma(xr[1][r], v[1], fma(xr[0][r], v[0], E[r]));
    E[RX] = (E[RX] + v[0]) + v[1];
  }
}

// Residual tiles of one stage for one warp: row^T (8 cols x 8 rows) per tile as
// KS chained k-steps, the kCT tiles' chains interleaved.
template <int NN>
__device__ __forceinline__ void stage_residual(const double* __restrict__ srec, int lane,
                                               const double (&A)[mma_ct<NN>()][ksteps<NN>()],
                                               double (&d)[mma_ct<NN>()][2]) {
  constexpr int kCT = mma_ct<NN>();
  constexpr int KS = ksteps<NN>();
  constexpr int RQ = rec_pitch(NN);
  const int q = lane & 3;
  const int c8 = lane >> 2;
  double B[KS];  // residual B fragments: X'[row c8][k]
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) B[ks] = srec[c8 * RQ + ks * 4 + q];
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) d[ct][0] = d[ct][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
    for (int ct = 0; ct < kCT; ++ct) dmma(d[ct][0], d[ct][1], A[ct][ks], B[ks]);
  }
}

// Lean P-APG stage for a clean stage (no diagonal in the warp's columns, all 8
// rows present, no pad column), one warp: the residuals of all kCT tiles first
// (independent DMMA chains interleaved), then per tile theta2, v, the store of a
// changed multiplier, the scalar sums and the aggregation.
// TEST: per-tile cold test on the inputs -- with theta1 = theta1_prev = 0 and
// row >= 0 everywhere in a tile (late in a solve almost every tile) theta2 = 0
// and v = 0 = theta1_prev: no store, and every scalar, row-sum and aggregate
// update adds an exact zero, so the warp skips the tile after one vote; a tile
// whose v are all zero skips its aggregation. !TEST: no tests at all (the
// dense early iterations, where no tile is cold). Both variants evaluate the
// same expressions for a hot tile, so results are bitwise identical. Returns
// the number of cold tiles (TEST).
template <int NN, bool UNIT, bool TEST>
__device__ __forceinline__ int papg_clean(const double* __restrict__ sv, const double* __restrict__ svp,
                                          const double* __restrict__ srec, double* g0, double* g1,
                                          int lane, const double (&d)[mma_ct<NN>()][2],
                                          double (&D)[mma_ct<NN>()][max1(agg_fbd<NN>())][2],
                                          double (&E)[mma_ct<NN>()][max1(agg_re<NN>())],
                                          const double (&Cc)[mma_ct<NN>()], const MCoef& cf, MScal& sc,
                                          double (&rs)[2], int& nst) {
  CRB_GEO(NN)
  constexpr int KS = ksteps<NN>();
  constexpr int FBD = agg_fbd<NN>();
  constexpr int RX = agg_rx<NN>();
  constexpr int RQ = rec_pitch(NN);
  constexpr bool SPLIT = split_yc<NN>();
  const int q = lane & 3;
  const int c8 = lane >> 2;
  const double* r0 = srec + (2 * q) * RQ;  // records of rows 2q, 2q+1
  const double* r1 = r0 + RQ;
  double yr[2] = {0.0, 0.0};  // y of rows 2q, 2q+1 (split form)
  if (SPLIT) {
    yr[0] = r0[NN + 1];
    yr[1] = r1[NN + 1];
  }
  // aggregation A fragments ([X 1][row 2q+j][feature fb*8 + c8]) and the DFMA
  // remainder's x of rows 2q, 2q+1, shared by the stage's tiles
  double Ag[2][max1(FBD)];
  double xr[2][max1(RX)];
#pragma unroll
  for (int fb = 0; fb < FBD; ++fb) {
    Ag[0][fb] = r0[fb * 8 + c8];
    Ag[1][fb] = r1[fb * 8 + c8];
  }
#pragma unroll
  for (int r = 0; r < RX; ++r) {
    xr[0][r] = r0[8 * FBD + r];
    xr[1][r] = r1[8 * FBD + r];
  }
  int cold = 0;
  rs[0] = 0.0;
  rs[1] = 0.0;
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) {
    const int cl = ct * 8 + c8;  // column within the warp's strip
    double row[2], c1[2], p1[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int rr = 2 * q + j;
      row[j] = d[ct][j];
      if (SPLIT) row[j] += yr[j] + Cc[ct];  // y_l1 - c_l2 (Cc holds -c_l2)
      c1[j] = sv[rr * kTCP + cl];
      p1[j] = svp[rr * kTCP + cl];
    }
    if (TEST) {
      // stored multipliers are v >= +0 (never -0), so "both zero" is one OR of the bits
      const unsigned long long bits =
          (unsigned long long)__double_as_longlong(c1[0]) | (unsigned long long)__double_as_longlong(c1[1]) |
          (unsigned long long)__double_as_longlong(p1[0]) | (unsigned long long)__double_as_longlong(p1[1]);
      const bool hot = bits != 0ull || (__double2hiint(row[0]) | __double2hiint(row[1])) < 0;
      if (!__any_sync(0xffffffffu, hot)) {
        ++cold;
        continue;
      }
    }
    double v[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double th2;
      if (UNIT) {
        th2 = fma(cf.beta, c1[j] - p1[j], c1[j]);
      } else {
        const double th1 = cf.s_c * c1[j];
        th2 = fma(cf.beta, th1 - cf.s_p * p1[j], th1);
      }
      v[j] = keep_if_nonneg(fma(-row[j], cf.invL, th2));
      // v goes into the buffer that holds p1 (theta1_prev): an unchanged value
      // needs no store
      store_changed_sector((j ? g1 : g0) + ct * 8, v[j], p1[j], true, lane, nst);
      sc.vv = fma(v[j], v[j], sc.vv);
      sc.vr = fma(v[j], row[j], sc.vr);
      sc.tr = fma(th2, row[j], sc.tr);
      acc_neg_sq(sc.nn, row[j]);  // min(row, 0)^2
      if (!TEST && ct == 0)
        rs[j] = v[j];  // = 0 + v exactly
      else
        rs[j] += v[j];
    }
    // a tile whose v are all zero adds exact zeros to the aggregates
    if (!TEST || __any_sync(0xffffffffu, v[0] != 0.0 || v[1] != 0.0))
      papg_agg<NN>(Ag, xr, v, D[ct], E[ct]);
  }
  return cold;
}

// Residual of one stage from the lane's B-fragment pointer (lb: X'[row c8][q]).
template <int NN>
__device__ __forceinline__ void lean_residual(const double* __restrict__ lb,
                                              const double (&A)[mma_ct<NN>()][ksteps<NN>()],
                                              double (&d)[mma_ct<NN>()][2]) {
  constexpr int kCT = mma_ct<NN>();
  constexpr int KS = ksteps<NN>();
  double B[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) B[ks] = lb[ks * 4];
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) d[ct][0] = d[ct][1] = 0.0;
  if (CRB_PROBE_SKIP & 1) {  // probe: one DFMA instead of the residual DMMAs
#pragma unroll
    for (int ct = 0; ct < kCT; ++ct) {
      d[ct][0] = A[ct][0] * B[0];
      d[ct][1] = A[ct][1] * B[0];
    }
  } else {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
      for (int ct = 0; ct < kCT; ++ct) dmma(d[ct][0], d[ct][1], A[ct][ks], B[ks]);
    }
  }
}

// Lean-loop form of papg_clean: the stage's lane-dependent smem addresses come
// in precomputed (lv: theta1 of row 2q, tile 0, column c8 of the warp; lb: the
// residual B fragment X'[row c8][q]; lr: the record of row 2q; la: lr + c8), the output rows
// 2q, 2q+1 are o0, o0 + ld, and the residual is computed here. Same expressions
// as papg_clean (bitwise-equal results).
template <int NN, bool UNIT, bool TEST>
__device__ __forceinline__ int papg_lean(const double* __restrict__ lv, const double* __restrict__ lb,
                                         const double* __restrict__ lr, const double* __restrict__ la,
                                         double* o0, long long ld, int lane,
                                         const double (&A)[mma_ct<NN>()][ksteps<NN>()],
                                         double (&D)[mma_ct<NN>()][max1(agg_fbd<NN>())][2],
                                         double (&E)[mma_ct<NN>()][max1(agg_re<NN>())],
                                         const double (&Cc)[mma_ct<NN>()], const MCoef& cf, MScal& sc,
                                         double (&rs)[2], int& nst) {
  CRB_GEO(NN)
  constexpr int KS = ksteps<NN>();
  constexpr int FBD = agg_fbd<NN>();
  constexpr int RX = agg_rx<NN>();
  constexpr int RQ = rec_pitch(NN);
  constexpr bool SPLIT = split_yc<NN>();
  double d[kCT][2];
  lean_residual<NN>(lb, A, d);
  double Ag[2][max1(FBD)];
  double xr[2][max1(RX)];
#pragma unroll
  for (int fb = 0; fb < FBD; ++fb) {
    Ag[0][fb] = la[fb * 8];
    Ag[1][fb] = la[RQ + fb * 8];
  }
#pragma unroll
  for (int r = 0; r < RX; ++r) {  // x of rows 2q, 2q+1 for the DFMA remainder
    xr[0][r] = lr[8 * FBD + r];
    xr[1][r] = lr[RQ + 8 * FBD + r];
  }
  double yr[2] = {0.0, 0.0};  // y of rows 2q, 2q+1 (split form)
  if (SPLIT) {
    yr[0] = lr[NN + 1];
    yr[1] = lr[RQ + NN + 1];
  }
  int cold = 0;
  rs[0] = 0.0;
  rs[1] = 0.0;
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) {
    double row[2], c1[2], p1[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      row[j] = d[ct][j];
      if (SPLIT) row[j] += yr[j] + Cc[ct];
      c1[j] = lv[j * kTCP + ct * 8];
      p1[j] = lv[(kTR + j) * kTCP + ct * 8];
    }
    if (TEST) {
      const unsigned long long bits =
          (unsigned long long)__double_as_longlong(c1[0]) | (unsigned long long)__double_as_longlong(c1[1]) |
          (unsigned long long)__double_as_longlong(p1[0]) | (unsigned long long)__double_as_longlong(p1[1]);
      const bool hot = bits != 0ull || (__double2hiint(row[0]) | __double2hiint(row[1])) < 0;
      if (!__any_sync(0xffffffffu, hot)) {
        ++cold;
        continue;
      }
    }
    double v[2], th2[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (UNIT) {
        th2[j] = fma(cf.beta, c1[j] - p1[j], c1[j]);
      } else {
        const double th1 = cf.s_c * c1[j];
        th2[j] = fma(cf.beta, th1 - cf.s_p * p1[j], th1);
      }
      v[j] = keep_if_nonneg(fma(-row[j], cf.invL, th2[j]));
    }
    // the aggregation MMAs go first (long latency, 16 pipe cycles each); the
    // stores and the scalar sums fill behind them (CRB_LEAN_ORDER = 0: old order)
    const bool agg = !(CRB_PROBE_SKIP & 2) &&
                     (!TEST || __any_sync(0xffffffffu, v[0] != 0.0 || v[1] != 0.0));
    if (CRB_LEAN_ORDER == 1 && agg) papg_agg<NN>(Ag, xr, v, D[ct], E[ct]);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      store_changed_sector(o0 + (j ? ld : 0) + ct * 8, v[j], p1[j], true, lane, nst);
      if (!(CRB_PROBE_SKIP & 4)) {
        sc.vv = fma(v[j], v[j], sc.vv);
        sc.vr = fma(v[j], row[j], sc.vr);
        if (!CRB_TR_ADJOINT) sc.tr = fma(th2[j], row[j], sc.tr);
        acc_neg_sq(sc.nn, row[j]);
      }
      if (!TEST && ct == 0)
        rs[j] = v[j];
      else
        rs[j] += v[j];
    }
    if (CRB_LEAN_ORDER == 0 && agg) papg_agg<NN>(Ag, xr, v, D[ct], E[ct]);
  }
  return cold;
}

// Lean-loop stage of the ALCC penalty sweep (kModePenalty, alcc.cpp:33-47):
// v = max(theta_k - row, 0) over a clean stage, its row sums and column
// aggregates; theta_k = V[cur] is the stage's first buffer. TEST: the same
// per-tile cold test as the P-APG stage (theta = 0 and row >= 0: v = 0 exactly).
template <int NN, bool TEST>
__device__ __forceinline__ int pen_lean(const double* __restrict__ lv, const double* __restrict__ lb,
                                        const double* __restrict__ lr, const double* __restrict__ la,
                                        const double (&A)[mma_ct<NN>()][ksteps<NN>()],
                                        double (&D)[mma_ct<NN>()][max1(agg_fbd<NN>())][2],
                                        double (&E)[mma_ct<NN>()][max1(agg_re<NN>())],
                                        const double (&Cc)[mma_ct<NN>()], double (&rs)[2]) {
  CRB_GEO(NN)
  constexpr int FBD = agg_fbd<NN>();
  constexpr int RX = agg_rx<NN>();
  constexpr int RQ = rec_pitch(NN);
  constexpr bool SPLIT = split_yc<NN>();
  double d[kCT][2];
  lean_residual<NN>(lb, A, d);
  double Ag[2][max1(FBD)];
  double xr[2][max1(RX)];
#pragma unroll
  for (int fb = 0; fb < FBD; ++fb) {
    Ag[0][fb] = la[fb * 8];
    Ag[1][fb] = la[RQ + fb * 8];
  }
#pragma unroll
  for (int r = 0; r < RX; ++r) {
    xr[0][r] = lr[8 * FBD + r];
    xr[1][r] = lr[RQ + 8 * FBD + r];
  }
  double yr[2] = {0.0, 0.0};
  if (SPLIT) {
    yr[0] = lr[NN + 1];
    yr[1] = lr[RQ + NN + 1];
  }
  int cold = 0;
  rs[0] = 0.0;
  rs[1] = 0.0;
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) {
    double row[2], th[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      row[j] = d[ct][j];
      if (SPLIT) row[j] += yr[j] + Cc[ct];
      th[j] = lv[j * kTCP + ct * 8];
    }
    if (TEST) {
      const unsigned long long bits =
          (unsigned long long)__double_as_longlong(th[0]) | (unsigned long long)__double_as_longlong(th[1]);
      const bool hot = bits != 0ull || (__double2hiint(row[0]) | __double2hiint(row[1])) < 0;
      if (!__any_sync(0xffffffffu, hot)) {
        ++cold;
        continue;
      }
    }
    double v[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      v[j] = keep_if_nonneg(th[j] - row[j]);
      rs[j] += v[j];
    }
    if (!TEST || __any_sync(0xffffffffu, v[0] != 0.0 || v[1] != 0.0)) papg_agg<NN>(Ag, xr, v, D[ct], E[ct]);
  }
  return cold;
}

// P-APG stage with masking (diagonal, partial stage, pad columns), one warp.
template <int NN, bool UNIT, bool BLK, bool TR = true>
__device__ __forceinline__ void papg_masked(const double* __restrict__ sv, const double* __restrict__ svp,
                                            const double* __restrict__ srec, double* gout,
                                            long long ld, long long gcol0, long long grow0, int nr,
                                            long long ncols, long long nbar,
                                            int lane, const double (&d)[mma_ct<NN>()][2],
                                            double (&D)[mma_ct<NN>()][max1(agg_fbd<NN>())][2],
                                            double (&E)[mma_ct<NN>()][max1(agg_re<NN>())],
                                            const double (&Cc)[mma_ct<NN>()], const MCoef& cf,
                                            MScal& sc, double (&rs)[2], int& nst) {
  CRB_GEO(NN)
  constexpr int KS = ksteps<NN>();
  constexpr int FBD = agg_fbd<NN>();
  constexpr int RX = agg_rx<NN>();
  constexpr int RQ = rec_pitch(NN);
  constexpr bool SPLIT = split_yc<NN>();
  const int q = lane & 3;
  const int c8 = lane >> 2;
  double yr[2] = {0.0, 0.0};
  if (SPLIT) {
    yr[0] = srec[(2 * q) * RQ + NN + 1];
    yr[1] = srec[(2 * q + 1) * RQ + NN + 1];
  }
  double Ag[2][max1(FBD)];
  double xr[2][max1(RX)];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool rv = 2 * q + j < nr;
#pragma unroll
    for (int fb = 0; fb < FBD; ++fb) Ag[j][fb] = rv ? srec[(2 * q + j) * RQ + fb * 8 + c8] : 0.0;
#pragma unroll
    for (int r = 0; r < RX; ++r) xr[j][r] = rv ? srec[(2 * q + j) * RQ + 8 * FBD + r] : 0.0;
  }
  double* g0 = gout + (long long)(2 * q) * ld + c8;
  rs[0] = 0.0;
  rs[1] = 0.0;
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) {
    const int cl = ct * 8 + c8;
    double v[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int rr = 2 * q + j;
      const bool rv = rr < nr;  // row present in this (partial) stage
      double row = d[ct][j];
      if (SPLIT) row += yr[j] + Cc[ct];
      // diagonal, rows past a partial stage, pad columns (with y - c split out
      // of the MMA a pad column's zero fragments no longer zero its row)
      if (same_block<BLK>(gcol0 + cl, grow0 + rr, nbar) || !rv || gcol0 + cl >= ncols) row = 0.0;
      const double c1 = sv[rr * kTCP + cl];
      const double p1 = svp[rr * kTCP + cl];
      double th2;
      if (UNIT) {
        th2 = fma(cf.beta, c1 - p1, c1);
      } else {
        const double th1 = cf.s_c * c1;
        th2 = fma(cf.beta, th1 - cf.s_p * p1, th1);
      }
      if (!rv) th2 = 0.0;
      v[j] = keep_if_nonneg(fma(-row, cf.invL, th2));
      store_changed_sector(g0 + (long long)j * ld + ct * 8, v[j], p1, rv, lane, nst);
      sc.vv = fma(v[j], v[j], sc.vv);
      sc.vr = fma(v[j], row, sc.vr);
      if (TR) sc.tr = fma(th2, row, sc.tr);
      acc_neg_sq(sc.nn, row);
      rs[j] += v[j];
    }
    if (__any_sync(0xffffffffu, v[0] != 0.0 || v[1] != 0.0)) papg_agg<NN>(Ag, xr, v, D[ct], E[ct]);
  }
}

// DMMA feature blocks of the column aggregates per mode: the P-APG and ALCC
// penalty sweeps use the split aggregation (agg_split), the power step all blocks
template <int NN, int MODE>
__host__ __device__ constexpr int mode_fbk() {
  return MODE == kModePower ? fblocks<NN>() : max1(agg_fbd<NN>());
}

// One 8-row stage for one warp, the other modes (power, penalty). MASK:
// diagonal / partial-stage masking.
template <int NN, int MODE, bool MASK, bool BLK>
__device__ __forceinline__ void mma_stage(const double* __restrict__ sv,
                                          const double* __restrict__ srec, double* gout,
                                          long long ld, long long gcol0, long long grow0, int nr,
                                          long long ncols, long long nbar,
                                          int lane, const double (&A)[mma_ct<NN>()][ksteps<NN>()],
                                          double (&D)[mma_ct<NN>()][mode_fbk<NN, MODE>()][2],
                                          double (&E)[mma_ct<NN>()][max1(agg_re<NN>())],
                                          const double (&Cc)[mma_ct<NN>()], const MCoef& cf,
                                          MScal& sc, double (&rs)[2]) {
  CRB_GEO(NN)
  constexpr int KS = ksteps<NN>();
  constexpr bool kPen = MODE != kModePower;  // split aggregation (papg_agg)
  constexpr int FB = kPen ? agg_fbd<NN>() : fblocks<NN>();
  constexpr int RX = agg_rx<NN>();
  constexpr int RQ = rec_pitch(NN);
  constexpr bool SPLIT = split_yc<NN>();
  const int q = lane & 3;
  const int c8 = lane >> 2;
  double yr[2] = {0.0, 0.0};  // y of rows 2q, 2q+1 (split form)
  if (SPLIT) {
    yr[0] = srec[(2 * q) * RQ + NN + 1];
    yr[1] = srec[(2 * q + 1) * RQ + NN + 1];
  }
  // residual B fragments: X'[row c8][k]
  double B[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) B[ks] = srec[c8 * RQ + ks * 4 + q];
  // aggregation A fragments: [X 1][row 2q+j][feature fb*8 + c8] (+ the split's x)
  double Ag[2][max1(FB)];
  double xr[2][max1(RX)];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool rv = !MASK || (2 * q + j < nr);
#pragma unroll
    for (int fb = 0; fb < FB; ++fb) Ag[j][fb] = rv ? srec[(2 * q + j) * RQ + fb * 8 + c8] : 0.0;
#pragma unroll
    for (int r = 0; r < RX; ++r) xr[j][r] = (kPen && rv) ? srec[(2 * q + j) * RQ + 8 * FB + r] : 0.0;
  }
  rs[0] = 0.0;
  rs[1] = 0.0;
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) {
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) dmma(d0, d1, A[ct][ks], B[ks]);
    const int cl = ct * 8 + c8;  // column within the warp's strip
    double v[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int rr = 2 * q + j;
      const bool rv = !MASK || rr < nr;  // row present in this (partial) stage
      double row = j == 0 ? d0 : d1;
      if (SPLIT) row += yr[j] + Cc[ct];  // y_l1 - c_l2 (Cc holds -c_l2)
      if (MASK && (same_block<BLK>(gcol0 + cl, grow0 + rr, nbar) || !rv || gcol0 + cl >= ncols))
        row = 0.0;
      if (MODE == kModePenalty || MODE == kModePenaltyUpdate) {
        const double th = (MASK && !rv) ? 0.0 : sv[rr * kTCP + cl];
        v[j] = keep_if_nonneg(th - row);
        if (MODE == kModePenaltyUpdate) {  // outer step: statistics + theta_{k+1}
          sc.vv = fma(v[j], v[j], sc.vv);
          sc.vr = fma(v[j], row, sc.vr);
          const double m = keep_if_neg(row);
          sc.nn = fma(m, m, sc.nn);
          if (rv) st_stream(gout + rr * ld + cl, v[j] / cf.cdiv);
        }
      } else {
        v[j] = row;
        sc.vv = fma(row, row, sc.vv);
      }
      rs[j] += v[j];
    }
    // a tile whose v are all zero adds exact zeros to the aggregates (the power
    // mode's v is the residual itself, rarely zero)
    if (MODE == kModePower || __any_sync(0xffffffffu, v[0] != 0.0 || v[1] != 0.0)) {
      if constexpr (kPen) {
        papg_agg<NN>(Ag, xr, v, D[ct], E[ct]);
      } else {
#pragma unroll
        for (int fb = 0; fb < FB; ++fb) {
          dmma(D[ct][fb][0], D[ct][fb][1], Ag[0][fb], v[0]);
          dmma(D[ct][fb][0], D[ct][fb][1], Ag[1][fb], v[1]);
        }
      }
    }
  }
}

template <int NN, int MODE, bool BLK>
__global__ void __launch_bounds__(mma_threads<NN>(), mma_ctas<NN>()) sweep_mma_kernel(const __grid_constant__ SweepArgs a) {
  constexpr int kNS = mma_ns<NN>();
  CRB_GEO(NN)
  constexpr int KS = ksteps<NN>();
  constexpr int FB = fblocks<NN>();
  constexpr int RQ = rec_pitch(NN);
  constexpr int SD = stage_doubles<NN>();
  extern __shared__ __align__(128) double smem[];
  double* stages = smem;
  double* rowacc = smem + kNS * SD;  // [2][kCW][kWinM]
  uint64_t* full = reinterpret_cast<uint64_t*>(rowacc + 2 * kCW * kWinM);
  uint64_t* empty = full + kNS;
  double* afrag = reinterpret_cast<double*>(empty + kNS);  // [kCW][kCT][KS][32] (CRB_A_SMEM)

  if (a.stopped != nullptr && *a.stopped) return;
  const int cur = (MODE != kModePower) ? *a.cur : 0;
  constexpr bool kPen = MODE == kModePenalty || MODE == kModePenaltyUpdate;
  const double* Vc = cur ? a.V1 : a.V0;
  double* Vp = cur ? a.V0 : a.V1;

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
      int i = 0;
#if CRB_PROBE_TIMING
      const long long pt0 = clock64();
      long long pw = 0;
#endif
      for (int t = t_first; t <= t_last; ++t) {
        const long long rlo = max(u0, (long long)t * a.R) - (long long)t * a.R;
        const long long rhi = min(u1, (long long)(t + 1) * a.R) - (long long)t * a.R;
        const long long c0 = (long long)t * kTC;
        const uint32_t vbytes = (uint32_t)min((long long)kTC, a.ld - c0) * 8u;
        for (long long r = rlo; r < rhi; r += kTR, ++i) {
          const int s = i % kNS;
          // short back-off: the spin otherwise takes ~3 % of the SM's issue slots
#if CRB_PROBE_TIMING
          const long long tp0 = clock64();
#endif
          if (CRB_PROBE_NOWAIT && i >= kNS) break;
          if (i >= kNS) mbar_wait_sleep<CRB_PROD_SLEEP>(&empty[s], (uint32_t)(((i / kNS) - 1) & 1));
#if CRB_PROBE_TIMING
          pw += clock64() - tp0;
#endif
          const int nr = (int)min((long long)kTR, rhi - r);
          double* st = stages + s * SD;
          const uint32_t bytes = (MODE == kModePapg ? 2u * nr * vbytes : 0u) +
                                 (kPen ? (uint32_t)nr * vbytes : 0u) + (uint32_t)nr * RQ * 8u;
          if ((MODE == kModePapg || kPen) && a.tmap) {
            // one tensor TMA per buffer: 8 rows x kTCP columns (the 2 pitch-padding
            // columns and rows past the shard are zero-filled, not read); the
            // penalty modes read theta = V[cur] only
            constexpr uint32_t nbuf = MODE == kModePapg ? 2u : 1u;
            mbar_arrive_expect_tx(&full[s], nbuf * kTR * kTCP * 8u + (uint32_t)nr * RQ * 8u);
            tma_g2s_3d(st, &a.tmV[cur], 0, t, (int)r, &full[s], pol_stream);
            if (MODE == kModePapg)
              tma_g2s_3d(st + kTR * kTCP, &a.tmV[1 - cur], 0, t, (int)r, &full[s], pol_stream);
            bulk_g2s(st + 2 * kTR * kTCP, a.rowrec + (a.r0 + r) * RQ, (uint32_t)nr * RQ * 8u,
                     &full[s], pol_keep);
            continue;
          }
          mbar_arrive_expect_tx(&full[s], bytes);
          if (MODE == kModePapg) {
            for (int qq = 0; qq < nr; ++qq) {
              const long long off = (r + qq) * a.ld + c0;
              bulk_g2s(st + qq * kTCP, Vc + off, vbytes, &full[s], pol_stream);
              bulk_g2s(st + (kTR + qq) * kTCP, Vp + off, vbytes, &full[s], pol_stream);
            }
          } else if (kPen) {
            for (int qq = 0; qq < nr; ++qq)
              bulk_g2s(st + qq * kTCP, Vc + (r + qq) * a.ld + c0, vbytes, &full[s], pol_stream);
          }
          bulk_g2s(st + 2 * kTR * kTCP, a.rowrec + (a.r0 + r) * RQ, (uint32_t)nr * RQ * 8u,
                   &full[s], pol_keep);
        }
      }
#if CRB_PROBE_TIMING
      if ((blockIdx.x == 0 || blockIdx.x == 77) && MODE == kModePapg)
        printf("probe cta %d producer total %lld wait_empty %lld stages %d\n", (int)blockIdx.x,
               clock64() - pt0, pw, i);
#endif
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
#if CRB_PROBE_TIMING
  const long long p_t0 = clock64();
  long long p_wait = 0, p_bar = 0;
#endif
  const int q = lane & 3;
  const int c8 = lane >> 2;
  MCoef cf{1.0, 0.0, 0.0, a.invL, a.cdiv};
  if (MODE == kModePapg) {
    cf.s_c = a.coef[0];
    cf.s_p = a.coef[1];
    cf.beta = a.coef[2];
  }
  const bool unit_scale = (cf.s_c == 1.0) && (cf.s_p == 1.0);
  MScal sc{0.0, 0.0, 0.0, 0.0};
  int nst = 0;  // stores issued by this thread (P-APG mode)
  int probe = 0, pstage = 0;  // adaptive cold test (P-APG mode)
  int i = 0;
  int flushes = 0;

  for (int t = t_first; t <= t_last; ++t) {
    const long long rlo = max(u0, (long long)t * a.R) - (long long)t * a.R;
    const long long rhi = min(u1, (long long)(t + 1) * a.R) - (long long)t * a.R;
    const long long gcol0 = (long long)t * kTC + warp * kW;  // first column of the warp
    const bool active = gcol0 < a.N;
    // residual A fragments: Xi'[col][k] (zero for pad columns -> row = 0 there)
    double A[kCT][KS];
    // column aggregates: DMMA fragments (P-APG: agg_fbd blocks) and the P-APG
    // DFMA remainder
    constexpr int FBK = mode_fbk<NN, MODE>();
    constexpr int RE = agg_re<NN>();
    double D[kCT][FBK][2];
    double E[kCT][max1(RE)];
    double Cc[kCT];
#pragma unroll
    for (int ct = 0; ct < kCT; ++ct) {
      const long long col = gcol0 + ct * 8 + c8;
      const bool cv = active && col < a.N;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int k = ks * 4 + q;
        A[ct][ks] = (cv && (!split_yc<NN>() || k < NN)) ? __ldg(a.colrec + col * RQ + k) : 0.0;
      }
      Cc[ct] = cv ? __ldg(a.colrec + col * RQ + NN) : 0.0;
#pragma unroll
      for (int fb = 0; fb < FBK; ++fb) D[ct][fb][0] = D[ct][fb][1] = 0.0;
#pragma unroll
      for (int r = 0; r < max1(RE); ++r) E[ct][r] = 0.0;
    }
    if constexpr ((MODE == kModePapg || MODE == kModePenalty) && !BLK) {
      // lean stage loop of the singleton P-APG and ALCC penalty sweeps: 32-bit stage counters, the
      // ring slot and phase advanced incrementally, lane addresses precomputed,
      // the stages that meet the diagonal precomputed per segment
      const int nrows = (int)(rhi - rlo);
      const int nstage = (nrows + kTR - 1) / kTR;
      const long long base = a.r0 + rlo;  // global row of the segment's first stage
      // stage s (rows base + 8s .. +8) meets the warp's columns [gcol0, gcol0 + kW)
      // iff s in [s_dlo, s_dhi)
      const long long dlo = gcol0 - kTR - base, dhi = gcol0 + kW - 1 - base;
      const int s_dlo = (int)max(0ll, (dlo >= 0 ? dlo / kTR : -((-dlo + kTR - 1) / kTR)) + 1);
      const int s_dhi = (int)max(0ll, min((long long)nstage, (dhi >= 0 ? dhi / kTR : -((-dhi + kTR - 1) / kTR)) + 1));
      // stages below s_clean_end can be clean (not the partial last stage, none
      // when the warp holds a pad column)
      const int s_clean_end = (gcol0 + kW <= a.N) ? ((nrows % kTR) ? nstage - 1 : nstage) : 0;
      double* gout = Vp + rlo * a.ld + gcol0;  // the warp's output block of stage 0
      const long long gstep = (long long)kTR * a.ld;
      const long long lane_out = (long long)(2 * q) * a.ld + c8;
      // lane offsets inside a stage (doubles)
      const int off_v = (2 * q) * kTCP + warp * kW + c8;
      const int off_b = 2 * kTR * kTCP + c8 * RQ + q;
      const int off_r = 2 * kTR * kTCP + (2 * q) * RQ;
      const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty);
      uint32_t slot = (uint32_t)i % kNS, phase = ((uint32_t)i / kNS) & 1u;
      const double* const aw = afrag + warp * kCT * KS * 32 + lane;
      if (CRB_A_SMEM) {
        double* w = afrag + warp * kCT * KS * 32 + lane;
#pragma unroll
        for (int ct = 0; ct < kCT; ++ct)
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) w[(ct * KS + ks) * 32] = A[ct][ks];
        __syncwarp();
      }
      double* const rowacc_lane = rowacc + warp * kWinM + 2 * (lane & 3) + ((lane >> 2) & 1);
#if CRB_RS_SMEM
      // row-sum window of kRsW rows: per buffer [kRsW/2 row pairs][kCW warps][8 column lanes][2]
      constexpr int kRsW = 32;
      constexpr int kRsBuf = kRsW / 2 * kCW * 16;
      static_assert(kRsBuf <= kCW * kWinM, "row-sum window must fit the rowacc buffers");
      double* const rs_lane = rowacc + (q * kCW + warp) * 16 + c8 * 2;
#endif
      int win = 0, win_base = 0;
      for (int st8 = 0; st8 < nstage; ++st8, gout += gstep) {
        if (!CRB_PROBE_NOWAIT || i + st8 < kNS) mbar_wait_u32(full_u + 8u * slot, phase);
        double rsj[2] = {0.0, 0.0};
        bool hot_stage = true;
        if (active && !CRB_PROBE_MEMONLY) {
          double Al[kCT][KS];
#pragma unroll
          for (int ct = 0; ct < kCT; ++ct)
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) Al[ct][ks] = CRB_A_SMEM ? aw[(ct * KS + ks) * 32] : A[ct][ks];
          const double* stg = stages + slot * SD;
          const double* lv = stg + off_v;
          const double* lb = stg + off_b;
          const double* lr = stg + off_r;
          const double* la = lr + c8;
          if ((st8 < s_dlo || st8 >= s_dhi) && st8 < s_clean_end) {
            double* o0 = gout + lane_out;
            // per-warp adaptive cold test: a tested stage that finds a cold tile
            // keeps the test on for the next 8 stages; otherwise every 8th stage
            // probes and the others run without any test
            if constexpr (MODE == kModePenalty) {
              (void)o0;
              if (probe > 0 || (pstage & 7) == 0) {
                const int cold = pen_lean<NN, true>(lv, lb, lr, la, Al, D, E, Cc, rsj);
                probe = cold ? 8 : (probe > 0 ? probe - 1 : 0);
                hot_stage = cold < kCT;
              } else {
                pen_lean<NN, false>(lv, lb, lr, la, Al, D, E, Cc, rsj);
              }
            } else if (probe > 0 || (pstage & 7) == 0) {
              const int cold = unit_scale
                  ? papg_lean<NN, true, true>(lv, lb, lr, la, o0, a.ld, lane, Al, D, E, Cc, cf, sc, rsj, nst)
                  : papg_lean<NN, false, true>(lv, lb, lr, la, o0, a.ld, lane, Al, D, E, Cc, cf, sc, rsj, nst);
              probe = cold ? 8 : (probe > 0 ? probe - 1 : 0);
              hot_stage = cold < kCT;
            } else if (unit_scale) {
              papg_lean<NN, true, false>(lv, lb, lr, la, o0, a.ld, lane, Al, D, E, Cc, cf, sc, rsj, nst);
            } else {
              papg_lean<NN, false, false>(lv, lb, lr, la, o0, a.ld, lane, Al, D, E, Cc, cf, sc, rsj, nst);
            }
            ++pstage;
          } else {
            const int nr = min(kTR, nrows - st8 * kTR);
            const long long grow0 = base + (long long)st8 * kTR;
            const double* sv = stg + warp * kW;
            const double* svp = sv + kTR * kTCP;
            const double* srec = stg + 2 * kTR * kTCP;
            if constexpr (MODE == kModePenalty) {
              (void)svp;
              mma_stage<NN, MODE, true, false>(sv, srec, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar, lane,
                                               Al, D, E, Cc, cf, sc, rsj);
            } else {
              double dres[kCT][2];
              stage_residual<NN>(srec, lane, Al, dres);
              if (unit_scale)
                papg_masked<NN, true, false, false>(sv, svp, srec, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar,
                                                    lane, dres, D, E, Cc, cf, sc, rsj, nst);
              else
                papg_masked<NN, false, false, false>(sv, svp, srec, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar,
                                                     lane, dres, D, E, Cc, cf, sc, rsj, nst);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(empty_u + 8u * slot);
        if (++slot == (uint32_t)kNS) {
          slot = 0;
          phase ^= 1u;
        }
#if CRB_RS_SMEM
        // row sums without shuffles: every lane parks its two rows' partials over
        // its 2 tiles in the window; the flush sums the 8 column lanes x kCW warps
        // of a row in a fixed order (every kRsW rows, one CTA barrier)
        (void)hot_stage;
        *reinterpret_cast<double2*>(rs_lane + (flushes & 1) * kRsBuf + (win >> 1) * kCW * 16) =
            make_double2(rsj[0], rsj[1]);
        win += kTR;
        if (win == kRsW || st8 == nstage - 1) {
          asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");
          const int valid_rows = min(win, nrows - win_base);
          const int tid = warp * 32 + lane;
          if (tid < kRsW * 8) {  // 8 threads per row: column lane g, then a 3-step butterfly
            const int r = tid >> 3, g = tid & 7;
            const double* rb = rowacc + (flushes & 1) * kRsBuf + ((r >> 1) * kCW * 8 + g) * 2 + (r & 1);
            double u = 0.0;
#pragma unroll
            for (int w = 0; w < kCW; ++w) u += rb[w * 16];
            u += __shfl_xor_sync(0xffffffffu, u, 1);
            u += __shfl_xor_sync(0xffffffffu, u, 2);
            u += __shfl_xor_sync(0xffffffffu, u, 4);
            if (g == 0 && r < valid_rows) a.rowpart[(long long)t * a.R + rlo + win_base + r] = u;
          }
          win_base += win;
          win = 0;
          ++flushes;
        }
        continue;
#endif
        double rsum = 0.0;  // row sums, as in the generic loop below
        if (CRB_PROBE_SKIP & 8) {
          rsum = rsj[0] + rsj[1];
        } else if (hot_stage) {
          const bool b2 = (lane & 4) != 0;
          const double send = b2 ? rsj[0] : rsj[1];
          rsum = b2 ? rsj[1] : rsj[0];
          rsum += __shfl_xor_sync(0xffffffffu, send, 4);
          rsum += __shfl_xor_sync(0xffffffffu, rsum, 8);
          rsum += __shfl_xor_sync(0xffffffffu, rsum, 16);
        }
        if (lane < 8) rowacc_lane[(flushes & 1) * kCW * kWinM + win] = rsum;
        win += kTR;
        if (win == kWinM || st8 == nstage - 1) {
#if CRB_PROBE_TIMING
          const long long tb0 = clock64();
#endif
          asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");
#if CRB_PROBE_TIMING
          p_bar += clock64() - tb0;
#endif
          const int valid_rows = min(win, nrows - win_base);
          const int wr = warp * 32 + lane;
          if (warp < kWinM / 32 && wr < valid_rows) {
            const double* rb = rowacc + (flushes & 1) * kCW * kWinM;
            double u = 0.0;
#pragma unroll
            for (int w = 0; w < kCW; ++w) u += rb[w * kWinM + wr];
            a.rowpart[(long long)t * a.R + rlo + win_base + wr] = u;
          }
          win_base += win;
          win = 0;
          ++flushes;
        }
      }
      i += nstage;
    } else {
  int win = 0;
      long long win_base = rlo;
      for (long long r = rlo; r < rhi; r += kTR, ++i) {
      const int s = i % kNS;
      mbar_wait(&full[s], (uint32_t)((i / kNS) & 1));
      const int nr = (int)min((long long)kTR, rhi - r);
      double rsj[2] = {0.0, 0.0};
      bool hot_stage = true;  // P-APG: false when every tile of the stage was cold
      if (active) {
        const double* st = stages + s * SD;
        const double* sv = st + warp * kW;
        const double* svp = st + kTR * kTCP + warp * kW;
        const double* srec = st + 2 * kTR * kTCP;
        double* gout = Vp + r * a.ld + gcol0;
        double* o0 = gout + (long long)(2 * q) * a.ld + c8;
        double* o1 = o0 + a.ld;
        const long long grow0 = a.r0 + r;
        // warp-uniform: no diagonal in this 8-row block of the warp's columns, full
        // stage, no pad column
        const bool clean = nr == kTR && gcol0 + kW <= a.N &&
                           blocks_disjoint<BLK>(grow0, kTR, gcol0, kW, a.nbar);
        if constexpr (MODE == kModePapg) {
          double dc[kCT][2];
          stage_residual<NN>(srec, lane, A, dc);
          if (clean) {
            // per-warp adaptive cold test: a tested stage that finds a cold tile
            // keeps the test on for the next 8 stages; otherwise every 8th stage
            // probes and the others run without any test
            const bool test = probe > 0 || (pstage & 7) == 0;
            ++pstage;
            if (test) {
              const int cold = unit_scale
                  ? papg_clean<NN, true, true>(sv, svp, srec, o0, o1, lane, dc, D, E, Cc, cf, sc, rsj, nst)
                  : papg_clean<NN, false, true>(sv, svp, srec, o0, o1, lane, dc, D, E, Cc, cf, sc, rsj, nst);
              probe = cold ? 8 : (probe > 0 ? probe - 1 : 0);
              hot_stage = cold < kCT;
            } else if (unit_scale) {
              papg_clean<NN, true, false>(sv, svp, srec, o0, o1, lane, dc, D, E, Cc, cf, sc, rsj, nst);
            } else {
              papg_clean<NN, false, false>(sv, svp, srec, o0, o1, lane, dc, D, E, Cc, cf, sc, rsj, nst);
            }
          } else {
            if (unit_scale)
              papg_masked<NN, true, BLK>(sv, svp, srec, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar,
                                         lane, dc, D, E, Cc, cf, sc, rsj, nst);
            else
              papg_masked<NN, false, BLK>(sv, svp, srec, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar,
                                          lane, dc, D, E, Cc, cf, sc, rsj, nst);
          }
        } else if (clean) {
          mma_stage<NN, MODE, false, BLK>(sv, srec, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar, lane, A, D,
                                          E, Cc, cf, sc, rsj);
        } else {
          mma_stage<NN, MODE, true, BLK>(sv, srec, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar, lane, A, D,
                                         E, Cc, cf, sc, rsj);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      // row sums over the warp's columns: lanes sharing q hold the same rows
      // 2q, 2q+1; the first exchange leaves each lane one of the two (row 2q +
      // bit 2 of the lane), then two butterflies; lane b*4 + q ends with row
      // 2q + b (a cold stage's sums are exact zeros already)
      double rsum = 0.0;
      if (hot_stage) {
        const bool b2 = (lane & 4) != 0;
        const double send = b2 ? rsj[0] : rsj[1];
        rsum = b2 ? rsj[1] : rsj[0];
        rsum += __shfl_xor_sync(0xffffffffu, send, 4);
        rsum += __shfl_xor_sync(0xffffffffu, rsum, 8);
        rsum += __shfl_xor_sync(0xffffffffu, rsum, 16);
      }
      double* ra = rowacc + (flushes & 1) * kCW * kWinM + warp * kWinM;
      if (lane < 8) ra[win + 2 * (lane & 3) + ((lane >> 2) & 1)] = rsum;
      win += kTR;
      if (win == kWinM || r + kTR >= rhi) {
        // fixed-order sum over the CTA's warps into the tile's row-sum slice
        // (warp k sums window rows 32k .. 32k + 31)
        asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");
        const int valid_rows = (int)min((long long)win, rhi - win_base);
        const int wr = warp * 32 + lane;
        if (warp < kWinM / 32 && wr < valid_rows) {
          const double* rb = rowacc + (flushes & 1) * kCW * kWinM;
          double u = 0.0;
#pragma unroll
          for (int w = 0; w < kCW; ++w) u += rb[w * kWinM + wr];
          a.rowpart[(long long)t * a.R + win_base + wr] = u;
        }
        win_base += win;
        win = 0;
        ++flushes;
      }
    }
    }
    if (active) {  // column partials: thread holds (feature fb*8+c8, cols 2q+{0,1})
      const long long slot = (long long)blockIdx.x * a.maxspan + (t - t_first);
      constexpr int FBW = MODE == kModePower ? FB : agg_fbd<NN>();  // DMMA blocks in use
#pragma unroll
      for (int ct = 0; ct < kCT; ++ct) {
#pragma unroll
        for (int fb = 0; fb < FBW; ++fb) {
          const int f = fb * 8 + c8;
          if (f <= NN) {
            const int slotf = (f == NN) ? 0 : 1 + f;  // colagg = (colsum, V^T X)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const long long coff = (long long)warp * kW + ct * 8 + 2 * q + j;
              a.colpart[(slot * kTC + coff) * (NN + 1) + slotf] = D[ct][fb][j];
            }
          }
        }
        if constexpr (MODE != kModePower && RE > 0) {
          // DFMA remainder: lanes 4 c8 + q hold rows 2q, 2q+1 of column c8; sum over q
          const long long coff = (long long)warp * kW + ct * 8 + c8;
#pragma unroll
          for (int r = 0; r < RE; ++r) {
            double e = E[ct][r];
            e += __shfl_xor_sync(0xffffffffu, e, 1);
            e += __shfl_xor_sync(0xffffffffu, e, 2);
            const int f = 8 * agg_fbd<NN>() + r;  // feature; r == RE - 1: the column sum
            const int slotf = (r == RE - 1) ? 0 : 1 + f;
            if (q == 0) a.colpart[(slot * kTC + coff) * (NN + 1) + slotf] = e;
          }
        }
      }
    }
  }

#if CRB_PROBE_TIMING
  if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77) && MODE == kModePapg)
    printf("probe cta %d warp %d total %lld wait_full %lld bar %lld\n", (int)blockIdx.x, warp,
           clock64() - p_t0, p_wait, p_bar);
#endif
  double vv = sc.vv, vr = sc.vr, tr = sc.tr, nn = sc.nn;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    vv += __shfl_xor_sync(0xffffffffu, vv, off);
    vr += __shfl_xor_sync(0xffffffffu, vr, off);
    tr += __shfl_xor_sync(0xffffffffu, tr, off);
    nn += __shfl_xor_sync(0xffffffffu, nn, off);
  }
  // one scalar record per CTA: the consumer warps' sums combined in warp order
  // (in the row-sum window buffer the last flush did not use)
  double* wsc = rowacc + (flushes & 1) * kCW * kWinM;
  if (lane == 0) {
    wsc[warp * kScal + 0] = vv;
    wsc[warp * kScal + 1] = vr;
    wsc[warp * kScal + 2] = tr;
    wsc[warp * kScal + 3] = nn;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");
  if (warp == 0 && lane < kScal) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kCW; ++w) t += wsc[w * kScal + lane];
    a.scalpart[(long long)blockIdx.x * kScal + lane] = t;
  }
  if (MODE == kModePapg && a.stores != nullptr) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nst += __shfl_xor_sync(0xffffffffu, nst, off);
    if (lane == 0 && nst) atomicAdd(a.stores, (unsigned long long)nst);
  }
}

template <int NN>
SweepKernelInfo info_for(int mode, bool blocked) {
  CRB_GEO(NN)
  SweepKernelInfo inf{};
  if (blocked) {
    inf.fn = mode == kModePapg    ? (const void*)sweep_mma_kernel<NN, kModePapg, true>
             : mode == kModePower ? (const void*)sweep_mma_kernel<NN, kModePower, true>
                                  : nullptr;
    if (!inf.fn) return inf;
  } else {
    inf.fn = mode == kModePapg      ? (const void*)sweep_mma_kernel<NN, kModePapg, false>
             : mode == kModePower   ? (const void*)sweep_mma_kernel<NN, kModePower, false>
             : mode == kModePenalty ? (const void*)sweep_mma_kernel<NN, kModePenalty, false>
                                    : (const void*)sweep_mma_kernel<NN, kModePenaltyUpdate, false>;
  }
  inf.strip_cols = kW;
  inf.warps_per_block = kCW;
  inf.scal_recs = 1;
  inf.tile_cols = kTC;
  inf.threads = kThreads;
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

SweepKernelInfo sweep_mma_info(int n, int mode, bool blocked) {
  return AllN::info(n, mode, blocked);
}

int launch_sweep(const SweepKernelInfo& info, const SweepArgs& a, void* stream) {
  void* args[] = {const_cast<SweepArgs*>(&a)};
  return (int)cudaLaunchKernel(info.fn, dim3((unsigned)a.G), dim3(info.threads), args,
                               info.smem_bytes, (cudaStream_t)stream);
}

}  // namespace crb
