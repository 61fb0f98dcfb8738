// mma_geo.cuh -- geometry and primitives of the DMMA pair sweeps (sweep_mma.cu).
#pragma once
#include <cstdint>

#include "device.cuh"

namespace crb {

// CTA geometry per n, measured on B200: 11 or 15 consumer
// warps x 2 tiles at one CTA per SM (mma_cw) since the P-APG producer loads a
// stage with one tensor TMA per buffer. CRB_WIDE_ABOVE = 14 restores the narrow
// geometry (7 warps x 4 tiles, two CTAs per SM) for n <= 14.
#ifndef CRB_WIDE_ABOVE
#define CRB_WIDE_ABOVE 0
#endif
template <int NN>
__host__ __device__ constexpr bool mma_wide() { return NN > CRB_WIDE_ABOVE; }
#ifndef CRB_CW  // geometry overrides of the wide layout (measurement builds; 0: per n)
#define CRB_CW 0
#endif
#ifndef CRB_CT
#define CRB_CT 2
#endif
// consumer warps per CTA (x 2 tiles): 15 for 9 <= n <= 14, else 11 -- measured at
// N = 1e4, iterations 6-25, us per sweep with 15 / 11 warps: n = 1 394 / 390, 3
// 388 / 378, 5 383 / 373, 8 372 / 367, 10 365 / 381, 12 370 / 386, 16 431 / 411,
// 20 (N = 2e4) 2074 / 1909, 24 601 / 523, 32 837 / 632 (profiles/r2_experiments.md)
template <int NN>
__host__ __device__ constexpr int mma_cw() {
  return !mma_wide<NN>() ? 7 : (CRB_CW > 0 ? CRB_CW : ((NN >= 9 && NN <= 14) ? 15 : 11));
}
template <int NN>
__host__ __device__ constexpr int mma_ct() { return mma_wide<NN>() ? CRB_CT : 4; }   // 8-col tiles / warp
template <int NN>
__host__ __device__ constexpr int mma_threads() { return (mma_cw<NN>() + 1) * 32; }
// kW columns per warp, kTC per CTA tile, kTCP smem row pitch (+16 B: conflict-free)
#define CRB_GEO(NN)                              \
  constexpr int kCW = mma_cw<NN>();              \
  constexpr int kCT = mma_ct<NN>();              \
  constexpr int kW = 8 * kCT;                    \
  constexpr int kTC = kCW * kW;                  \
  constexpr int kTCP = kTC + 2;                  \
  constexpr int kThreads = (kCW + 1) * 32;       \
  (void)kThreads;
constexpr int kTR = 8;                 // rows per stage (one MMA row block)
#ifndef CRB_MMA_CTAS_PER_SM
#define CRB_MMA_CTAS_PER_SM 0  // 0: per n (mma_ctas)
#endif
// CTAs per SM: the narrow geometry runs two CTAs, the wide one (16 warps
// already) one (two wide CTAs do not fit the register file).
template <int NN>
__host__ __device__ constexpr int mma_ctas() {
  return CRB_MMA_CTAS_PER_SM > 0 ? CRB_MMA_CTAS_PER_SM : (mma_wide<NN>() ? 1 : 2);
}
#ifndef CRB_MMA_NS
#define CRB_MMA_NS 0  // 0: per geometry (mma_ns)
#endif
template <int NN>
__host__ __device__ constexpr int mma_ns() {  // ring stages
  return CRB_MMA_NS > 0 ? CRB_MMA_NS : (mma_ctas<NN>() == 2 ? 3 : 4);
}
#ifndef CRB_MMA_WIN
#define CRB_MMA_WIN 256
#endif
// row-sum window of the dense DMMA sweep (multiple of 32): one CTA barrier per
// 32 stages; measured 32 / 64 / 128 / 256 rows: n = 10 iterations 50-300 344 /
// 331 / 325 / 321 us, n = 20 late 321 / 308 / 303 / 296 us
constexpr int kWinM = CRB_MMA_WIN;

// Residual K: the n features plus (1, y) with (-c, 1) folded in -- unless
// dropping those two columns saves a k-step, then y - c is added with DADDs.
template <int NN>
__host__ __device__ constexpr bool split_yc() { return (NN + 3) / 4 < (NN + 5) / 4; }
template <int NN>
__host__ __device__ constexpr int ksteps() { return split_yc<NN>() ? (NN + 3) / 4 : (NN + 5) / 4; }
template <int NN>
__host__ __device__ constexpr int fblocks() { return ((NN + 1) + 7) / 8; }
// P-APG aggregation split: the DMMA aggregation runs whole 8-feature blocks of
// [X 1]; a short remainder of R = (n+1) mod 8 features (the last x columns and
// the column sum) runs on DFMA/DADD in the lanes that hold v instead of a
// padded DMMA block (2R fp64 warp instructions per tile, 4R pipe cycles, vs 32
// for the block's two DMMAs). n = 10: 1 block + x8, x9 and the column sum.
// Remainders above 3 features (n = 5, 20) keep the padded block: the extra
// per-lane accumulators spill at 128 registers.
#ifndef CRB_AGG_REM_MAX
#define CRB_AGG_REM_MAX 3
#endif
template <int NN>
__host__ __device__ constexpr bool agg_split() {
  return (NN + 1) % 8 > 0 && (NN + 1) % 8 <= CRB_AGG_REM_MAX;
}
// DMMA feature blocks of the P-APG aggregation
template <int NN>
__host__ __device__ constexpr int agg_fbd() { return agg_split<NN>() ? (NN + 1) / 8 : fblocks<NN>(); }
// x features on DFMA, and those plus the column sum
template <int NN>
__host__ __device__ constexpr int agg_rx() { return agg_split<NN>() ? NN - 8 * ((NN + 1) / 8) : 0; }
template <int NN>
__host__ __device__ constexpr int agg_re() { return agg_split<NN>() ? agg_rx<NN>() + 1 : 0; }
__host__ __device__ constexpr int max1(int x) { return x > 0 ? x : 1; }

template <int NN>
__host__ __device__ constexpr int stage_doubles() {
  return 2 * kTR * (mma_cw<NN>() * 8 * mma_ct<NN>() + 2) + kTR * rec_pitch(NN);
}
// P-APG lean loop: the residual A fragments of each warp's columns live in
// shared memory (reloaded per stage) instead of 2 x ksteps registers per lane
#ifndef CRB_A_SMEM
#define CRB_A_SMEM 0
#endif
template <int NN>
__host__ __device__ constexpr int afrag_doubles() {
  return CRB_A_SMEM ? mma_cw<NN>() * mma_ct<NN>() * ksteps<NN>() * 32 : 0;
}
template <int NN>
__host__ __device__ constexpr int smem_bytes() {
  return mma_ns<NN>() * stage_doubles<NN>() * 8 + 2 * mma_cw<NN>() * kWinM * 8 +
         2 * mma_ns<NN>() * 8 + afrag_doubles<NN>() * 8;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct MCoef {
  double s_c, s_p, beta, invL, cdiv;
};
struct MScal {
  double vv, vr, tr, nn;
};

}  // namespace crb
