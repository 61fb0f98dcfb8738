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
__host__ __device__ constexpr int rec_pitch() { return (NN + 2) & ~1; }
template <int NN>
__host__ __device__ constexpr int rows_per_stage() { return cols_per_lane<NN>() == 2 ? 4 : 8; }
template <int NN>
__host__ __device__ constexpr int tile_cols() {
  return consumer_warps<NN>() * 32 * cols_per_lane<NN>();
}
// doubles per stage: V and V' rows for the tile + row records
template <int NN>
__host__ __device__ constexpr int stage_doubles() {
  return 2 * rows_per_stage<NN>() * tile_cols<NN>() + rows_per_stage<NN>() * rec_pitch<NN>();
}
constexpr int kRsPitch = 17;  // per-warp row-sum transpose: 32 rows x 16 lanes (+1 pad)
template <int NN>
__host__ __device__ constexpr int smem_bytes() {
  return kNS * stage_doubles<NN>() * 8 + consumer_warps<NN>() * 32 * kRsPitch * 8 + 2 * kNS * 8;
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

__device__ __forceinline__ void st_stream(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
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
  double s_c, s_p, beta, invL;
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
};

// max(u, 0) and min(r, 0) on the sign bit: three integer ops, no FSEL chains
__device__ __forceinline__ double keep_if_nonneg(double u) {
  const int hi = __double2hiint(u), lo = __double2loint(u);
  const int m = ~(hi >> 31);
  return __hiloint2double(hi & m, lo & m);
}
__device__ __forceinline__ double keep_if_neg(double r) {
  const int hi = __double2hiint(r), lo = __double2loint(r);
  const int m = hi >> 31;
  return __hiloint2double(hi & m, lo & m);
}

template <int NN, int MODE, int TR, int TC, bool MASK, bool UNIT>
__device__ __forceinline__ void run_stage(const StageView& sv, int nr, int lane,
                                          ColState<NN, cols_per_lane<NN>()>& cs, const Coef& cf,
                                          Scal& sc) {
  constexpr int C = cols_per_lane<NN>();
  constexpr int RP = rec_pitch<NN>();
  using VT = typename VecT<C>::T;
#pragma unroll
  for (int q = 0; q < TR; ++q) {
    if (q < nr) {
      const double* xr = sv.rec + q * RP;
      double x[NN];
      const double y1 = xr[0];
#pragma unroll
      for (int j = 0; j < NN; ++j) x[j] = xr[1 + j];
      VT vc, vp, out;
      if (MODE == kModePapg) {
        vc = *reinterpret_cast<const VT*>(sv.vc + q * TC);
        vp = *reinterpret_cast<const VT*>(sv.vp + q * TC);
      }
      double rs = 0.0;
#pragma unroll
      for (int k = 0; k < C; ++k) {
        double ra = y1 - cs.cc[k], rb = 0.0;  // two FMA chains for ILP
#pragma unroll
        for (int j = 0; j < NN; j += 2) {
          ra = fma(-x[j], cs.xi[k][j], ra);
          if (j + 1 < NN) rb = fma(-x[j + 1], cs.xi[k][j + 1], rb);
        }
        double row = ra + rb;
        if (MASK && (!cs.valid[k] || sv.col0 + k == sv.g0 + q)) row = 0.0;
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
        } else {
          v = row;
          sc.vv = fma(row, row, sc.vv);
        }
        cs.acc[k][0] += v;
#pragma unroll
        for (int j = 0; j < NN; ++j) cs.acc[k][1 + j] = fma(v, x[j], cs.acc[k][1 + j]);
        rs += v;
      }
      if (MODE == kModePapg) st_stream(reinterpret_cast<VT*>(sv.gout + q * sv.ld), out);
      rs += __shfl_xor_sync(0xffffffffu, rs, 16);
      if (lane < 16) sv.srs[q * kRsPitch + lane] = rs;
    }
  }
}

template <int NN, int MODE>
__global__ void __launch_bounds__(threads_per_cta<NN>()) sweep_kernel(const SweepArgs a) {
  constexpr int kCW = consumer_warps<NN>();
  constexpr int C = cols_per_lane<NN>();
  constexpr int W = 32 * C;
  constexpr int RP = rec_pitch<NN>();
  constexpr int TR = rows_per_stage<NN>();
  constexpr int TC = tile_cols<NN>();
  constexpr int SD = stage_doubles<NN>();
  using VT = typename VecT<C>::T;
  extern __shared__ __align__(128) double smem[];
  double* stages = smem;
  double* srs_all = smem + kNS * SD;
  uint64_t* full = reinterpret_cast<uint64_t*>(srs_all + kCW * 32 * kRsPitch);
  uint64_t* empty = full + kNS;

  if (a.stopped != nullptr && *a.stopped) return;
  const int cur = (MODE == kModePapg) ? *a.cur : 0;
  const double* Vc = cur ? a.V1 : a.V0;
  double* Vp = cur ? a.V0 : a.V1;

  const int T = (a.S + kCW - 1) / kCW;  // column tiles
  const int ct = blockIdx.x % T;
  const int chunk = blockIdx.x / T;
  const long long rlo = a.R * chunk / a.P;
  const long long rhi = a.R * (chunk + 1) / a.P;
  const int nstage = (int)((rhi - rlo + TR - 1) / TR);
  const long long c0 = (long long)ct * TC;
  const int tile_w = (int)min((long long)TC, a.ld - c0);  // columns actually present

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
      const uint32_t vbytes = (uint32_t)tile_w * 8u;
      for (int i = 0; i < nstage; ++i) {
        const int s = i % kNS;
        if (i >= kNS) mbar_wait(&empty[s], (uint32_t)(((i / kNS) - 1) & 1));
        const long long r = rlo + (long long)i * TR;
        const int nr = (int)min((long long)TR, rhi - r);
        double* st = stages + s * SD;
        const uint32_t bytes =
            (MODE == kModePapg ? 2u * nr * vbytes : 0u) + (uint32_t)nr * RP * 8u;
        mbar_arrive_expect_tx(&full[s], bytes);
        if (MODE == kModePapg) {
          for (int q = 0; q < nr; ++q) {
            const long long off = (r + q) * a.ld + c0;
            bulk_g2s(st + q * TC, Vc + off, vbytes, &full[s], pol_stream);
            bulk_g2s(st + (TR + q) * TC, Vp + off, vbytes, &full[s], pol_stream);
          }
        }
        bulk_g2s(st + 2 * TR * TC, a.rowrec + (a.r0 + r) * RP, (uint32_t)nr * RP * 8u, &full[s],
                 pol_keep);
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  const int strip = ct * kCW + warp;
  const bool active = strip < a.S;
  const long long col0 = c0 + warp * W + lane * C;  // first column of this lane
  double* srs = srs_all + warp * 32 * kRsPitch;

  ColState<NN, C> cs;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const long long col = col0 + k;
    cs.valid[k] = active && col < a.N;
    const double* rec = a.colrec + (cs.valid[k] ? col : 0) * RP;
    cs.cc[k] = cs.valid[k] ? __ldg(rec) : 0.0;
#pragma unroll
    for (int j = 0; j < NN; ++j) cs.xi[k][j] = cs.valid[k] ? __ldg(rec + 1 + j) : 0.0;
#pragma unroll
    for (int j = 0; j <= NN; ++j) cs.acc[k][j] = 0.0;
  }
  // warp-uniform: every column of the strip is a real column
  const bool strip_full = active && (c0 + (long long)(warp + 1) * W <= a.N);
  const long long strip_lo = c0 + (long long)warp * W;
  Coef cf{1.0, 0.0, 0.0, a.invL};
  if (MODE == kModePapg) {
    cf.s_c = a.coef[0];
    cf.s_p = a.coef[1];
    cf.beta = a.coef[2];
  }
  const bool unit_scale = (cf.s_c == 1.0) && (cf.s_p == 1.0);
  Scal sc{0.0, 0.0, 0.0, 0.0};
  int win = 0;               // rows held in the row-sum transpose window
  long long win_base = rlo;  // local row of window slot 0
  const int lane_off = warp * W + lane * C;

  for (int i = 0; i < nstage; ++i) {
    const int s = i % kNS;
    mbar_wait(&full[s], (uint32_t)((i / kNS) & 1));
    const long long r = rlo + (long long)i * TR;
    const int nr = (int)min((long long)TR, rhi - r);
    if (active) {
      const double* st = stages + s * SD;
      StageView sv{st + lane_off, st + TR * TC + lane_off, st + 2 * TR * TC,
                   Vp + r * a.ld + col0, a.ld, col0, a.r0 + r, srs + win * kRsPitch};
      // the diagonal or a pad column touches this stage: per-pair masks
      const bool clean =
          strip_full && (sv.g0 + nr <= strip_lo || sv.g0 >= strip_lo + W);
      if (clean) {
        if (unit_scale) run_stage<NN, MODE, TR, TC, false, true>(sv, nr, lane, cs, cf, sc);
        else run_stage<NN, MODE, TR, TC, false, false>(sv, nr, lane, cs, cf, sc);
      } else {
        if (unit_scale) run_stage<NN, MODE, TR, TC, true, true>(sv, nr, lane, cs, cf, sc);
        else run_stage<NN, MODE, TR, TC, true, false>(sv, nr, lane, cs, cf, sc);
      }
      win += nr;
      if (win == 32 || i == nstage - 1) {  // fixed-order row reduction of the window
        __syncwarp();
        if (lane < win) {
          double t = 0.0;
#pragma unroll
          for (int l = 0; l < 16; ++l) t += srs[lane * kRsPitch + l];
          a.rowpart[(long long)strip * a.R + win_base + lane] = t;
        }
        __syncwarp();
        win_base += win;
        win = 0;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (!active) return;

#pragma unroll
  for (int k = 0; k < C; ++k) {
    double* dst = a.colpart + ((long long)chunk * a.ld + col0 + k) * (NN + 1);
#pragma unroll
    for (int j = 0; j <= NN; ++j) dst[j] = cs.acc[k][j];
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
    double* sp = a.scalpart + ((long long)chunk * a.S + strip) * kScal;
    sp[0] = vv;
    sp[1] = vr;
    sp[2] = tr;
    sp[3] = nn;
  }
}

template <int NN>
SweepKernelInfo info_for(int mode) {
  SweepKernelInfo inf;
  inf.fn = mode == kModePapg ? (const void*)sweep_kernel<NN, kModePapg>
                             : (const void*)sweep_kernel<NN, kModePower>;
  inf.C = cols_per_lane<NN>();
  inf.warps_per_block = consumer_warps<NN>();
  const int smem = smem_bytes<NN>();
  cudaFuncSetAttribute(inf.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bps = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, inf.fn, threads_per_cta<NN>(), smem) !=
      cudaSuccess)
    bps = 0;
  inf.max_blocks_per_sm = bps;
  return inf;
}

template <int NN>
int launch_for(const SweepKernelInfo& info, const SweepArgs& a, cudaStream_t s) {
  constexpr int kCW = consumer_warps<NN>();
  const int T = (a.S + kCW - 1) / kCW;
  const unsigned grid = (unsigned)((long long)T * a.P);
  void* args[] = {const_cast<SweepArgs*>(&a)};
  return (int)cudaLaunchKernel(info.fn, dim3(grid), dim3(threads_per_cta<NN>()), args,
                               smem_bytes<NN>(), s);
}

template <int... Ns> struct Table;
template <int N0, int... Ns> struct Table<N0, Ns...> {
  static SweepKernelInfo info(int n, int mode) {
    return n == N0 ? info_for<N0>(mode) : Table<Ns...>::info(n, mode);
  }
  static int launch(int n, const SweepKernelInfo& i, const SweepArgs& a, cudaStream_t s) {
    return n == N0 ? launch_for<N0>(i, a, s) : Table<Ns...>::launch(n, i, a, s);
  }
};
template <> struct Table<> {
  static SweepKernelInfo info(int, int) { return SweepKernelInfo{nullptr, 0, 0, 0}; }
  static int launch(int, const SweepKernelInfo&, const SweepArgs&, cudaStream_t) {
    return (int)cudaErrorInvalidValue;
  }
};
using AllN = Table<1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22,
                   23, 24>;

}  // namespace

SweepKernelInfo sweep_kernel_info(int n, int mode) { return AllN::info(n, mode); }

int launch_sweep(const SweepKernelInfo& info, const SweepArgs& a, int n, void* stream) {
  return AllN::launch(n, info, a, (cudaStream_t)stream);
}

}  // namespace crb
