// sweep_sparse.cu -- K1 over a masked dual store (the P-APG step of sweep_mma.cu
// with HBM traffic proportional to the nonzero multipliers).
//
// After a few dozen iterations almost every pair multiplier is exactly zero
// (cfg 2: 16 % nonzero at iteration 20, 3 % at 100, 0.2 % at 2000; the
// projection max(., 0) keeps inactive constraints at 0). The dense sweep still
// streams 24 B per pair. Here the dual store keeps its dense value layout plus
// one 32-bit live word per 8x8 MMA tile in the fragments' ballot order (bit =
// lane: a live test is one shift, the new word is one ballot), stored per CTA
// and stage of the static work split (device.cuh MaskGeo), so a stage's words
// are one contiguous TMA copy and no word is shared by two CTAs. Per pair the residual is
// still evaluated on the tensor cores (every constraint is checked every
// iteration); values move only where live:
//   producer   TMA ring (8 deep, small): row records + the two mask blocks
//   consumers  two stages ahead, each warp reads the masks of its own columns
//              and gathers the live V / V' values into its private slot of a
//              3-deep value ring (one 8-byte cp.async per live bit); a stage
//              is computed as in the dense kernel with non-live values
//              selected as 0; v > 0 is stored, the new masks are assembled
//              from ballots; aggregation MMAs of an all-zero 8x8 tile are
//              skipped.
// Results are bitwise identical to the dense kernel: zero entries contribute
// exact zeros to every sum.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "mma_geo.cuh"
#include "pipeline.cuh"

namespace crb {

namespace {

constexpr int kLook = 2;        // value gathers are issued this many stages ahead
constexpr int kNA = 8;          // TMA ring (row records + masks): deep, it is small
constexpr int kNB = kLook + 1;  // value ring (per-warp columns, filled by cp.async)
#ifndef CRB_SP_CW
#define CRB_SP_CW 7             // consumer warps for n <= 12 (7 x 4 tiles or 14 x 2)
#endif

// Geometry: the dense kernel's column tiles (224 columns for n <= 12, 240
// above) split over twice as many warps, 2 MMA tiles each -- without the HBM
// stream the sweep is latency bound and needs the warps (measured: 7 consumer
// warps x 4 tiles leave 28 % issue utilisation).
template <int NN>
__host__ __device__ constexpr int sp_cw() { return mma_wide<NN>() ? 15 : CRB_SP_CW; }
template <int NN>
__host__ __device__ constexpr int sp_ct() { return mma_wide<NN>() ? 2 : 28 / CRB_SP_CW; }
template <int NN>
__host__ __device__ constexpr int sp_threads() { return (sp_cw<NN>() + 1) * 32; }
#define SP_GEO(NN)                               \
  constexpr int kCW = sp_cw<NN>();               \
  constexpr int kCT = sp_ct<NN>();               \
  constexpr int kW = 8 * kCT;                    \
  constexpr int kTC = kCW * kW;                  \
  constexpr int kTCP = kTC + 2;                  \
  constexpr int kThreads = (kCW + 1) * 32;       \
  (void)kThreads;                                \
  static_assert(kTC == mma_cw<NN>() * 8 * mma_ct<NN>(), "same column tiles as the dense sweep");

template <int NN>
__host__ __device__ constexpr int ringA_doubles() {  // row records + live words of V, V'
  return kTR * rec_pitch(NN) + 2 * (mma_cw<NN>() * mma_ct<NN>() * 2) / 2;
}
template <int NN>
__host__ __device__ constexpr int ringB_doubles() {  // V, V' values of a stage
  return 2 * kTR * (mma_cw<NN>() * 8 * mma_ct<NN>() + 2);
}
template <int NN>
__host__ __device__ constexpr int sp_smem_bytes() {
  return (kNA * ringA_doubles<NN>() + kNB * ringB_doubles<NN>()) * 8 +
         2 * sp_cw<NN>() * kWin * 8 + 2 * kNA * 8;
}

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// stage enumeration shared by producer and consumers: segment (tile t, rows
// [rlo, rhi)) after segment, 8 rows at a time
struct StageIt {
  long long u0, u1, R;
  int t, t_last;
  long long r, rhi;
  __device__ void init(long long u0_, long long u1_, long long R_) {
    u0 = u0_;
    u1 = u1_;
    R = R_;
    t = (int)(u0 / R);
    t_last = (int)((u1 - 1) / R);
    r = u0 - (long long)t * R;
    rhi = min(u1, (long long)(t + 1) * R) - (long long)t * R;
  }
  __device__ bool valid() const { return t <= t_last; }
  __device__ int nr() const { return (int)min((long long)kTR, rhi - r); }
  __device__ void next() {
    r += kTR;
    if (r >= rhi) {
      ++t;
      r = max(u0, (long long)t * R) - (long long)t * R;
      rhi = min(u1, (long long)(t + 1) * R) - (long long)t * R;
    }
  }
};

template <int NN, bool MASK, bool UNIT, bool BLK>
__device__ __forceinline__ void sp_stage(const double* __restrict__ sv, const double* __restrict__ svp,
                                         const double* __restrict__ srec, double* gout, long long ld,
                                         long long gcol0, long long grow0, int nr, long long ncols,
                                         long long nbar, int lane,
                                         const double (&A)[sp_ct<NN>()][ksteps<NN>()],
                                         double (&D)[sp_ct<NN>()][fblocks<NN>()][2],
                                         const double (&Cc)[sp_ct<NN>()], const MCoef& cf,
                                         MScal& sc, double (&rs)[2],
                                         uint32_t (&mw)[2 * sp_ct<NN>()],
                                         const uint32_t (&wc)[2 * sp_ct<NN>()],
                                         const uint32_t (&wp)[2 * sp_ct<NN>()]) {
  SP_GEO(NN)
  constexpr int KS = ksteps<NN>();
  constexpr int FB = fblocks<NN>();
  constexpr int RQ = rec_pitch(NN);
  constexpr bool SPLIT = split_yc<NN>();
  const int q = lane & 3;
  const int c8 = lane >> 2;
  double B[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) B[ks] = srec[c8 * RQ + ks * 4 + q];
  rs[0] = rs[1] = 0.0;
  // residuals of every tile first: independent DMMA chains interleave
  double dd[kCT][2];
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) dd[ct][0] = dd[ct][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
    for (int ct = 0; ct < kCT; ++ct) dmma(dd[ct][0], dd[ct][1], A[ct][ks], B[ks]);
  }
  double yr[2] = {0.0, 0.0};
  if (SPLIT) {
    yr[0] = srec[(2 * q) * RQ + NN + 1];
    yr[1] = srec[(2 * q + 1) * RQ + NN + 1];
  }
  // whole warp-stage cold (no live multiplier, no violated constraint): every
  // contribution is an exact zero
  {
    bool any = false;
#pragma unroll
    for (int ct = 0; ct < kCT; ++ct) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double row = dd[ct][j];
        if (SPLIT) row += yr[j] + Cc[ct];
        any |= row < 0.0 || (((wc[2 * ct + j] | wp[2 * ct + j]) >> lane) & 1u);
      }
    }
    if (!__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int k = 0; k < 2 * kCT; ++k) mw[k] = 0u;
      return;
    }
  }
  double Ag[2][FB];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool rv = !MASK || (2 * q + j < nr);
#pragma unroll
    for (int fb = 0; fb < FB; ++fb) Ag[j][fb] = rv ? srec[(2 * q + j) * RQ + fb * 8 + c8] : 0.0;
  }
#pragma unroll
  for (int ct = 0; ct < kCT; ++ct) {
    const int cl = ct * 8 + c8;
    double rows[2];
    bool hot = false;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int rr = 2 * q + j;
      const bool rv = !MASK || rr < nr;
      double row = dd[ct][j];
      if (SPLIT) row += yr[j] + Cc[ct];
      if (MASK && (same_block<BLK>(gcol0 + cl, grow0 + rr, nbar) || !rv || gcol0 + cl >= ncols))
        row = 0.0;
      rows[j] = row;
      hot |= row < 0.0 || (((wc[2 * ct + j] | wp[2 * ct + j]) >> lane) & 1u);
    }
    // a tile with no live multiplier and no violated constraint has v = 0 and
    // contributes exact zeros to every sum: nothing to do
    if (!__any_sync(0xffffffffu, hot)) {
      mw[2 * ct] = mw[2 * ct + 1] = 0u;
      continue;
    }
    double v[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int rr = 2 * q + j;
      const bool rv = !MASK || rr < nr;
      const double row = rows[j];
      // live bits of this lane's element (clear: exactly 0)
      const double c1 = ((wc[2 * ct + j] >> lane) & 1u) ? sv[rr * kTCP + cl] : 0.0;
      const double p1 = ((wp[2 * ct + j] >> lane) & 1u) ? svp[rr * kTCP + cl] : 0.0;
      double th2;
      if (UNIT) {
        th2 = fma(cf.beta, c1 - p1, c1);
      } else {
        const double th1 = cf.s_c * c1;
        th2 = fma(cf.beta, th1 - cf.s_p * p1, th1);
      }
      if (MASK && !rv) th2 = 0.0;
      v[j] = keep_if_nonneg(fma(-row, cf.invL, th2));
      sc.vv = fma(v[j], v[j], sc.vv);
      sc.vr = fma(v[j], row, sc.vr);
      sc.tr = fma(th2, row, sc.tr);
      const double m = keep_if_neg(row);
      sc.nn = fma(m, m, sc.nn);
      const bool live = v[j] > 0.0;
      if (rv && live) st_stream(gout + rr * ld + cl, v[j]);
      mw[2 * ct + j] = __ballot_sync(0xffffffffu, live);
      rs[j] += v[j];
    }
    // an all-zero 8x8 tile adds nothing to the aggregates
    if (__any_sync(0xffffffffu, v[0] != 0.0 || v[1] != 0.0)) {
#pragma unroll
      for (int fb = 0; fb < FB; ++fb) {
        dmma(D[ct][fb][0], D[ct][fb][1], Ag[0][fb], v[0]);
        dmma(D[ct][fb][0], D[ct][fb][1], Ag[1][fb], v[1]);
      }
    }
  }
}

template <int NN, bool BLK>
__global__ void __launch_bounds__(sp_threads<NN>(), 1) sweep_sparse_kernel(const SweepArgs a) {
  SP_GEO(NN)
  constexpr int FB = fblocks<NN>();
  constexpr int KS = ksteps<NN>();
  constexpr int RQ = rec_pitch(NN);
  constexpr int SA = ringA_doubles<NN>();
  constexpr int SB = ringB_doubles<NN>();
  static_assert((2 * kCT) % 4 == 0 && (kTC / 4) % 4 == 0, "16-byte word groups");
  extern __shared__ __align__(128) double smem[];
  double* ringA = smem;                      // [kNA][records | masks]
  double* ringB = ringA + kNA * SA;          // [kNB][V | V']
  double* rowacc = ringB + kNB * SB;
  uint64_t* full = reinterpret_cast<uint64_t*>(rowacc + 2 * kCW * kWin);
  uint64_t* empty = full + kNA;

  if (a.stopped != nullptr && *a.stopped) return;
  const int cur = *a.cur;
  const double* Vc = cur ? a.V1 : a.V0;
  double* Vp = cur ? a.V0 : a.V1;
  const uint32_t* Mc = cur ? a.M1 : a.M0;
  uint32_t* Mp = cur ? a.M0 : a.M1;

  const long long units = (long long)a.T * a.R;
  const long long u0 = (long long)blockIdx.x * a.U;
  const long long u1 = min(u0 + a.U, units);
  if (u0 >= u1) return;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNA; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCW) {  // ------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_keep = policy_evict_last();
      const uint64_t pol_stream = policy_evict_first();
      StageIt it;
      it.init(u0, u1, a.R);
      for (int i = 0; it.valid(); it.next(), ++i) {
        const int s = i % kNA;
        if (i >= kNA) mbar_wait_sleep(&empty[s], (uint32_t)(((i / kNA) - 1) & 1));
        const int nr = it.nr();
        double* st = ringA + s * SA;
        const uint32_t mbytes = (uint32_t)kTC;  // kTC / 4 words
        mbar_arrive_expect_tx(&full[s], (uint32_t)nr * RQ * 8u + 2u * mbytes);
        bulk_g2s(st, a.rowrec + (a.r0 + it.r) * RQ, (uint32_t)nr * RQ * 8u, &full[s], pol_keep);
        const long long mo = ((long long)blockIdx.x * a.mstages + i) * (kTC / 4);
        uint32_t* sm = reinterpret_cast<uint32_t*>(st + kTR * RQ);
        bulk_g2s(sm, Mc + mo, mbytes, &full[s], pol_stream);
        bulk_g2s(sm + kTC / 4, Mp + mo, mbytes, &full[s], pol_stream);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  const int q = lane & 3;
  const int c8 = lane >> 2;
  MCoef cf{a.coef[0], a.coef[1], a.coef[2], a.invL, 0.0};
  const bool unit_scale = (cf.s_c == 1.0) && (cf.s_p == 1.0);
  MScal sc{0.0, 0.0, 0.0, 0.0};

  // gather the live values of stage j (this warp's columns) into value slot j % kNB:
  // one lane per live word (buffer, tile, j), one cp.async per set bit
  const int wbase = warp * kCT * 2;  // this warp's first word of a stage
  auto issue = [&](int j, const StageIt& jt) {
    const int s = j % kNA;
    mbar_wait(&full[s], (uint32_t)((j / kNA) & 1));
    const uint32_t* sm = reinterpret_cast<const uint32_t*>(ringA + s * SA + kTR * RQ);
    double* vb = ringB + (j % kNB) * SB;
    const long long gcol0 = (long long)jt.t * kTC + warp * kW;
    if (lane < 4 * kCT) {
      const int buf = lane / (2 * kCT), rem = lane % (2 * kCT);
      const int ct = rem >> 1, jj = rem & 1;
      uint32_t word = sm[buf * (kTC / 4) + wbase + rem];
      const double* src = (buf == 0 ? Vc : Vp) + (jt.r + jj) * a.ld + gcol0 + ct * 8;
      double* dst = vb + buf * kTR * kTCP + jj * kTCP + warp * kW + ct * 8;
      while (word) {
        const int b = __ffs(word) - 1;
        word &= word - 1;
        const int qq = b & 3, cc = b >> 2;  // row 2 qq + jj, column cc of the tile
        cp_async8(dst + 2 * qq * kTCP + cc, src + 2 * qq * a.ld + cc);
      }
    }
    cp_async_commit();
  };

  StageIt it, la;
  it.init(u0, u1, a.R);
  la = it;
  int jla = 0;
  for (; jla < kLook && la.valid(); ++jla, la.next()) issue(jla, la);

  int i = 0;
  int flushes = 0;
  int cur_t = -1;
  int win = 0;
  long long win_base = 0;
  double A[kCT][KS];
  double D[kCT][FB][2];
  double Cc[kCT];
  bool active = false;
  long long gcol0 = 0;
  for (; it.valid(); ++i) {
    const int t = it.t;
    if (t != cur_t) {  // segment prologue: column fragments of this tile
      cur_t = t;
      gcol0 = (long long)t * kTC + warp * kW;
      active = gcol0 < a.N;
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
        for (int fb = 0; fb < FB; ++fb) D[ct][fb][0] = D[ct][fb][1] = 0.0;
      }
      win = 0;
      win_base = max(u0, (long long)t * a.R) - (long long)t * a.R;
    }
    // keep kLook stages of gathers in flight
    if (la.valid()) {
      issue(jla, la);
      ++jla;
      la.next();
    } else {
      cp_async_commit();  // empty group: uniform wait_group accounting
    }
    cp_async_wait<kLook>();
    __syncwarp();
    const int s = i % kNA;
    const int nr = it.nr();
    const long long r = it.r;
    double rsj[2] = {0.0, 0.0};
    uint32_t mw[2] = {0u, 0u};
    if (active) {
      const double* sa = ringA + s * SA;
      const uint32_t* sm = reinterpret_cast<const uint32_t*>(sa + kTR * RQ);
      const double* vb = ringB + (i % kNB) * SB;
      const double* sv = vb + warp * kW;
      const double* svp = vb + kTR * kTCP + warp * kW;
      uint32_t wc[2 * kCT], wp[2 * kCT], mw[2 * kCT];
#pragma unroll
      for (int k = 0; k < 2 * kCT; k += 4) {  // 16-byte words groups (broadcast)
        const uint4 c4 = *reinterpret_cast<const uint4*>(sm + wbase + k);
        const uint4 p4 = *reinterpret_cast<const uint4*>(sm + kTC / 4 + wbase + k);
        wc[k] = c4.x, wc[k + 1] = c4.y, wc[k + 2] = c4.z, wc[k + 3] = c4.w;
        wp[k] = p4.x, wp[k + 1] = p4.y, wp[k + 2] = p4.z, wp[k + 3] = p4.w;
      }
      double* gout = Vp + r * a.ld + gcol0;
      const long long grow0 = a.r0 + r;
      const bool clean = nr == kTR && gcol0 + kW <= a.N &&
                         blocks_disjoint<BLK>(grow0, kTR, gcol0, kW, a.nbar);
      if (clean) {
        if (unit_scale)
          sp_stage<NN, false, true, BLK>(sv, svp, sa, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar,
                                         lane, A, D, Cc, cf, sc, rsj, mw, wc, wp);
        else
          sp_stage<NN, false, false, BLK>(sv, svp, sa, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar,
                                          lane, A, D, Cc, cf, sc, rsj, mw, wc, wp);
      } else {
        if (unit_scale)
          sp_stage<NN, true, true, BLK>(sv, svp, sa, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar,
                                        lane, A, D, Cc, cf, sc, rsj, mw, wc, wp);
        else
          sp_stage<NN, true, false, BLK>(sv, svp, sa, gout, a.ld, gcol0, grow0, nr, a.N, a.nbar,
                                         lane, A, D, Cc, cf, sc, rsj, mw, wc, wp);
      }
      // the stage's new live words of this warp (one ballot per tile and row parity)
      if (lane == 0) {
        uint32_t* dst = Mp + ((long long)blockIdx.x * a.mstages + i) * (kTC / 4) + wbase;
#pragma unroll
        for (int k = 0; k < 2 * kCT; k += 4)
          *reinterpret_cast<uint4*>(dst + k) = make_uint4(mw[k], mw[k + 1], mw[k + 2], mw[k + 3]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      rsj[j] += __shfl_xor_sync(0xffffffffu, rsj[j], 4);
      rsj[j] += __shfl_xor_sync(0xffffffffu, rsj[j], 8);
      rsj[j] += __shfl_xor_sync(0xffffffffu, rsj[j], 16);
    }
    double* ra = rowacc + (flushes & 1) * kCW * kWin + warp * kWin;
    if (c8 == 0) {
      ra[win + 2 * q] = rsj[0];
      ra[win + 2 * q + 1] = rsj[1];
    }
    win += kTR;
    const bool seg_end = r + kTR >= it.rhi;
    if (win == kWin || seg_end) {
      asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");
      const int valid_rows = (int)min((long long)win, it.rhi - win_base);
      if (warp == 0 && lane < valid_rows) {
        const double* rb = rowacc + (flushes & 1) * kCW * kWin;
        double u = 0.0;
#pragma unroll
        for (int w = 0; w < kCW; ++w) u += rb[w * kWin + lane];
        a.rowpart[(long long)t * a.R + win_base + lane] = u;
      }
      win_base += win;
      win = 0;
      ++flushes;
    }
    if (seg_end && active) {  // column partials of this segment
      const int t_first = (int)(u0 / a.R);
      const long long slot = (long long)blockIdx.x * a.maxspan + (t - t_first);
#pragma unroll
      for (int ct = 0; ct < kCT; ++ct) {
#pragma unroll
        for (int fb = 0; fb < FB; ++fb) {
          const int f = fb * 8 + c8;
          if (f <= NN) {
            const int slotf = (f == NN) ? 0 : 1 + f;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const long long coff = (long long)warp * kW + ct * 8 + 2 * q + j;
              a.colpart[(slot * kTC + coff) * (NN + 1) + slotf] = D[ct][fb][j];
            }
          }
        }
      }
    }
    it.next();
  }
  cp_async_wait<0>();

  double vv = sc.vv, vr = sc.vr, tr = sc.tr, nn = sc.nn;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
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
SweepKernelInfo sp_info_for(bool blocked) {
  SP_GEO(NN)
  SweepKernelInfo inf{};
  inf.fn = blocked ? (const void*)sweep_sparse_kernel<NN, true>
                   : (const void*)sweep_sparse_kernel<NN, false>;
  inf.strip_cols = kW;
  inf.warps_per_block = kCW;
  inf.scal_recs = kCW;
  inf.tile_cols = kTC;
  inf.threads = kThreads;
  inf.smem_bytes = sp_smem_bytes<NN>();
  cudaFuncSetAttribute(inf.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, inf.smem_bytes);
  int bps = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, inf.fn, inf.threads, inf.smem_bytes) !=
      cudaSuccess)
    bps = 0;
  inf.max_blocks_per_sm = bps;
  return inf;
}

template <int... Ns> struct SpTable;
template <int N0, int... Ns> struct SpTable<N0, Ns...> {
  static SweepKernelInfo info(int n, bool blocked) {
    return n == N0 ? sp_info_for<N0>(blocked) : SpTable<Ns...>::info(n, blocked);
  }
};
template <> struct SpTable<> {
  static SweepKernelInfo info(int, bool) { return SweepKernelInfo{}; }
};
using SpAll = SpTable<CRB_N_LIST>;

}  // namespace

SweepKernelInfo sweep_sparse_info(int n, bool blocked) { return SpAll::info(n, blocked); }

}  // namespace crb
