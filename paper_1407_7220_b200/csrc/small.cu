// small.cu -- persistent cooperative dual loop for small N (V, V' L2-resident).
//
// For N ~ 1e3 (BASELINE config 1: 24 MB per iteration, L2-resident) a dual
// iteration is a few microseconds of work and the per-kernel path is bound by
// launch and pipeline-fill latency. Here one cooperative launch runs many
// iterations of papg.cpp:176-263; grid-wide barriers separate the phases:
//   A  primal closed form of every point (K2, iteration.cuh)
//   B  pair sweep: a warp owns 32 columns (one per lane) and a chunk of rows
//   C  fixed-order reduction of the partials; block 0 also reduces the
//      scalars and runs the control step (papg.cpp:187-262)
// Data produced inside the launch is read with L2-coherent loads (ld.cg).
// Same math, same partial layout and same fixed-order sums as the per-kernel
// path; results are deterministic.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "device.cuh"
#include "iteration.cuh"
#include "kernels.cuh"
#include "small.cuh"

namespace cg = cooperative_groups;

namespace crb {

namespace {

constexpr int kSBlock = 256;
// Threads per block of a variant. 512-thread blocks for the resident variant (16 warps per
// SM on half the rows each) were measured at config 1: the sweep's math halves (3.9 -> 2.4 us)
// but twice the column partials make its stores and the reduce slower (0.8 -> 2.3 us,
// 3.5 -> 4.4 us): 16.9 vs 15.4 us per iteration, so every variant runs 256 threads.
template <int NN, bool SV>
__host__ __device__ constexpr int small_threads() {
  return kSBlock;
}

// Row sums of U rows over a warp's 32 columns (lane = column) with a
// transpose-reduce: log2(U) halving exchanges (xor 16, 8, ...) leave each lane
// one row's partial, then a butterfly over the remaining lane bits. U - 1 + (5 -
// log2 U) shuffles instead of 5 U; fixed order, so deterministic. Returns the
// row index (within the U) whose sum lanes with (lane & (32/U - 1)) == 0 hold.
template <int U>
__device__ __forceinline__ int rows_transpose_sum(double (&t)[U], int lane, double& out) {
  int row = 0;
  int width = U;
  int bit = 16;
#pragma unroll
  for (int lvl = 0; (1 << lvl) < U; ++lvl) {
    const bool upper = (lane & bit) != 0;
    const int half = width >> 1;
#pragma unroll
    for (int i = 0; i < U / 2; ++i) {
      if (i < half) {
        const double send = upper ? t[i] : t[i + half];
        const double keep = upper ? t[i + half] : t[i];
        t[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
      }
    }
    if (upper) row += half;
    width = half;
    bit >>= 1;
  }
  double v = t[0];
#pragma unroll
  for (int o = bit; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  out = v;
  return row;
}

#ifndef CRB_SMALL_MINB
#define CRB_SMALL_MINB 1
#endif
// SV: every warp owns one (strip, chunk) task for the whole launch and keeps its V / V' tile
// (rows x 32 columns x 2 buffers) in shared memory: loaded once at the start of the launch,
// written back at its end, so an iteration moves no multiplier through L2 (at config 1 the
// 16 MB of V, V' streamed through L2 every iteration were ~3 us of the sweep).
template <int NN, bool SV>
__global__ void __launch_bounds__(small_threads<NN, SV>(), CRB_SMALL_MINB)
    small_loop_kernel(const SmallArgs a) {
  constexpr int kSB = small_threads<NN, SV>();
  constexpr int RP = rec_pitch(NN);
  cg::grid_group grid = cg::this_grid();
  const long long tid = (long long)blockIdx.x * kSB + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * kSB;
  const int lane = threadIdx.x & 31;
  const long long gwarp = tid >> 5;
  const long long nwarps = nthreads >> 5;
  const long long N = a.N;
  DevCtrl* c = a.ctrl;
  // every block keeps the control state in shared memory (loaded once per
  // launch) and runs the control step itself on the same fixed-order sums, so
  // all blocks take identical decisions without a broadcast; block 0 writes the
  // history and the final state
  __shared__ DevCtrl sctrl;
  // sweep: the records (x, 1, y) of the RB rows a warp is working on
  constexpr int RB = kSB == 512 ? 16 : (NN <= 8 ? 32 : (NN <= 16 ? 16 : (NN <= 24 ? 8 : 4)));
  __shared__ double srec[kSB / 32][RB * RP];
  extern __shared__ double vtile[];  // SV: [warp][buffer][RT][32]
  double* tile0 = vtile + (size_t)(threadIdx.x >> 5) * 2 * a.RT * 32;
  double* tile1 = tile0 + (size_t)a.RT * 32;
  // SV: the warp's task (fixed for the launch) and its tile, loaded from the dual buffers
  const long long tw_rlo = SV && gwarp < (long long)a.S * a.P ? N * (gwarp / a.S) / a.P : 0;
  const long long tw_rhi = SV && gwarp < (long long)a.S * a.P ? N * (gwarp / a.S + 1) / a.P : 0;
  const long long tw_col = SV ? (gwarp % a.S) * 32 + lane : 0;
  if constexpr (SV) {
    for (long long i = 0; i < tw_rhi - tw_rlo; ++i) {
      const bool ok = tw_col < N;
      tile0[i * 32 + lane] = ok ? __ldcg(a.V0 + (tw_rlo + i) * a.ld + tw_col) : 0.0;
      tile1[i * 32 + lane] = ok ? __ldcg(a.V1 + (tw_rlo + i) * a.ld + tw_col) : 0.0;
    }
  }
  if (threadIdx.x < (int)(sizeof(DevCtrl) / 8))
    reinterpret_cast<unsigned long long*>(&sctrl)[threadIdx.x] =
        __ldcg(reinterpret_cast<const unsigned long long*>(c) + threadIdx.x);
  const bool tr0 = a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  auto stamp = [&](long long it, int k) {
    if (tr0 && it < 64) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[it * 8 + k] = t;
    }
  };
  // the block's points (contiguous) for the reduction and the primal closed form
  const long long ppb = (N + gridDim.x - 1) / gridDim.x;
  const long long pl0 = (long long)blockIdx.x * ppb;
  const long long pl1 = min(N, pl0 + ppb);
  const long long nk2 = gridDim.x;
  // K2 of the next iteration for the block's points -> k2part[parity][block]
  auto primal_phase = [&]() {
    const int cur = sctrl.cur;
    const double* vposc = cur ? a.pa.vpos1 : a.pa.vpos0;
    double* vposp = cur ? a.pa.vpos0 : a.pa.vpos1;
    double acc[kK2Scal];
#pragma unroll
    for (int w = 0; w < kK2Scal; ++w) acc[w] = 0.0;
    for (long long l = pl0 + threadIdx.x; l < pl1; l += kSB)
      primal_point<NN>(a.pa, l, sctrl.s_cur, sctrl.s_prev, sctrl.beta, vposc, vposp, acc);
    block_reduce_store<kK2Scal, kSB>(
        acc, a.k2part + (((sctrl.ell + 1) & 1) * nk2 + blockIdx.x) * kK2Scal);
  };
  __syncthreads();
  if (!sctrl.halt) primal_phase();  // the first iteration's primal
  grid.sync();

  for (long long it = 0; it < a.max_iters; ++it) {
    stamp(it, 0);
    if (sctrl.halt) break;  // identical in every block
    const int cur = sctrl.cur;
    const double s_c = sctrl.s_cur, s_p = sctrl.s_prev, beta = sctrl.beta;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // one clock for the time budget of every block
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      __stcg(&a.clock[0], t);
    }

    // ---- B: pair sweep
    {
      const double* Vc = cur ? a.V1 : a.V0;
      double* Vp = cur ? a.V0 : a.V1;
      const double* tc = cur ? tile1 : tile0;  // SV: the same two buffers, resident
      double* tp = cur ? tile0 : tile1;
      const double invL = a.pa.invL;
      const bool unit = (s_c == 1.0) && (s_p == 1.0);
      double wsc[kScal] = {0.0, 0.0, 0.0, 0.0};
      for (long long w = gwarp; w < (long long)a.S * a.P; w += nwarps) {
        const int strip = (int)(w % a.S);
        const int chunk = (int)(w / a.S);
        const long long rlo = N * chunk / a.P, rhi = N * (chunk + 1) / a.P;
        const long long col = (long long)strip * 32 + lane;
        const bool valid = col < N;
        const double* rec = a.pa.colrec + (valid ? col : 0) * RP;  // (-xi, -c, 1)
        double xi[NN], acc[NN + 1];
        const double cc = valid ? __ldcg(rec + NN) : 0.0;
#pragma unroll
        for (int j = 0; j < NN; ++j) xi[j] = valid ? __ldcg(rec + j) : 0.0;
#pragma unroll
        for (int j = 0; j <= NN; ++j) acc[j] = 0.0;
        double vv = 0.0, vr = 0.0, tr = 0.0, nn = 0.0;
        // One L2 round trip per RB rows: the V / V' values of all RB rows are loaded up
        // front (2 RB registers) and the rows' records (x, 1, y) go to the warp's shared
        // slab in the same round trip; the math then runs from registers and shared
        // memory (per-batch record loads into registers made every 8-row batch a
        // dependent L2 round trip: cfg 1 sweep 9.0 -> 8.0 us). Phases of the sweep at
        // config 1 (CRB_TRACE): loads 3.0 us (16 MB through L2), math 4.1, stores 1.1.
#ifndef CRB_SMALL_U5
#define CRB_SMALL_U5 8
#endif
        constexpr int U = NN <= 5 ? CRB_SMALL_U5 : ((NN + 3) <= 8 ? 4 : ((NN + 3) <= 16 ? 2 : 1));
        double* slab = &srec[threadIdx.x >> 5][0];
        for (long long rb0 = rlo; rb0 < rhi; rb0 += RB) {
          const int nrows = (int)min((long long)RB, rhi - rb0);
          double cb[SV ? 1 : RB], pb[SV ? 1 : RB];
          if constexpr (!SV) {
#pragma unroll
            for (int u = 0; u < RB; ++u) {
              const long long r = u < nrows ? rb0 + u : rhi - 1;
              // the V pitch ld comes from the TMA kernels' strip width and may be
              // narrower than this kernel's 32-column strips: touch real columns only
              cb[u] = valid ? __ldcg(Vc + r * a.ld + col) : 0.0;
              pb[u] = valid ? __ldcg(Vp + r * a.ld + col) : 0.0;
            }
          }
          __syncwarp();  // the previous slab's readers are done
          for (int k = lane; k < nrows * RP; k += 32) slab[k] = __ldcg(a.pa.rowrec + rb0 * RP + k);
          __syncwarp();
          if (rb0 == rlo) stamp(it, 1);  // trace: the first rows' records have arrived
          auto group = [&](const int g0) {
            const long long r0 = rb0 + g0;
            double vrow[U];  // this lane's v of the batch's rows (0 when cold / absent)
            bool any_hot = false;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              vrow[u] = 0.0;
              const long long r = r0 + u;
              if (g0 + u >= nrows) continue;
              const double* xr = slab + (g0 + u) * RP;  // (x, 1, y)
              double row = xr[NN + 1] + cc;
#pragma unroll
              for (int j = 0; j < NN; ++j) row = fma(xr[j], xi[j], row);
              if (!valid || col == r) row = 0.0;
              double c1, p1;
              if constexpr (SV) {  // the lane's column of the warp's resident tile
                c1 = tc[(r - rlo) * 32 + lane];
                p1 = tp[(r - rlo) * 32 + lane];
              } else {
                c1 = cb[g0 + u];
                p1 = pb[g0 + u];
              }
              // cold: theta1 = theta1_prev = 0 (stored multipliers are never -0) and
              // row >= 0 -> theta2 = 0, v = 0 = p1: no store, every update below adds
              // an exact zero (late in a solve almost every row of a strip)
              const bool hot = ((unsigned long long)__double_as_longlong(c1) |
                                (unsigned long long)__double_as_longlong(p1)) != 0ull ||
                               __double2hiint(row) < 0;
              if (!__any_sync(0xffffffffu, hot)) continue;
              any_hot = true;
              double th2;
              if (unit) {
                th2 = fma(beta, c1 - p1, c1);
              } else {
                const double th1 = s_c * c1;
                th2 = fma(beta, th1 - s_p * p1, th1);
              }
              const double uu = fma(-row, invL, th2);
              const double v = uu > 0.0 ? uu : 0.0;
              if (valid && __double_as_longlong(v) != __double_as_longlong(p1)) {  // unchanged: no store
                if constexpr (SV) tp[(r - rlo) * 32 + lane] = v;
                else __stcg(Vp + r * a.ld + col, v);
              }
              vv = fma(v, v, vv);
              vr = fma(v, row, vr);
              tr = fma(th2, row, tr);
              const double m = row < 0.0 ? row : 0.0;
              nn = fma(m, m, nn);
              acc[0] += v;
#pragma unroll
              for (int j = 0; j < NN; ++j) acc[1 + j] = fma(v, xr[j], acc[1 + j]);
              vrow[u] = v;
            }
            // row sums of the batch over the strip's 32 columns -> rowpart [N][S]
            double rs = 0.0;
            int ru = lane / (32 / U);  // all-cold batch: zero sums, no shuffles
            if (any_hot) ru = rows_transpose_sum<U>(vrow, lane, rs);
            if ((lane & (32 / U - 1)) == 0 && g0 + ru < nrows)
              __stcg(a.rowpart + (r0 + ru) * a.S + strip, rs);
          };
          if constexpr (SV) {
            // nothing indexed by g0 lives in registers: a real loop keeps the sweep's code
            // within the instruction cache (32 unrolled rows were ~60 KB of SASS)
#pragma unroll 1
            for (int g0 = 0; g0 < nrows; g0 += U) group(g0);
          } else {
#pragma unroll
            for (int g0 = 0; g0 < RB; g0 += U) {
              if (g0 >= nrows) break;  // warp-uniform
              group(g0);
            }
          }
        }
        stamp(it, 2);  // trace: the task's math is done
        // [N][n+1][P]: the P partials of one column entry are contiguous
        if (valid) {
          double* dst = a.colpart + (col * (NN + 1)) * a.P + chunk;
#pragma unroll
          for (int j = 0; j <= NN; ++j) __stcg(dst + (long long)j * a.P, acc[j]);
        }
        wsc[0] += vv;
        wsc[1] += vr;
        wsc[2] += tr;
        wsc[3] += nn;
      }
      // scalars: lanes, then the block's warps, in a fixed order -> one record per block
#pragma unroll
      for (int k = 0; k < kScal; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wsc[k] += __shfl_xor_sync(0xffffffffu, wsc[k], o);
      }
      __shared__ double bsc[kSB / 32][kScal];
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < kScal; ++k) bsc[threadIdx.x >> 5][k] = wsc[k];
      }
      __syncthreads();
      if (threadIdx.x < kScal) {
        double t = 0.0;
#pragma unroll
        for (int w8 = 0; w8 < kSB / 32; ++w8) t += bsc[w8][threadIdx.x];
        __stcg(a.scalpart + (long long)blockIdx.x * kScal + threadIdx.x, t);
      }
    }
    stamp(it, 3);
    grid.sync();
    stamp(it, 4);

    // ---- C + control + the next iteration's primal, in every block:
    // warps 0-3 reduce the scalar records (sweep + K2, fixed order) and thread 0
    // runs the control step; warps 4-7 reduce the block's points' aggregates
    // (8 lanes per element over its contiguous partials); then the primal
    {
      const long long ncol = N * (NN + 1);
      const int w = threadIdx.x >> 5;
      if (w < 4) {
        constexpr int W = kScal + kK2Scal;
        const long long par = ((sctrl.ell + 1) & 1) * nk2;
        double v[W];
#pragma unroll
        for (int k = 0; k < W; ++k) v[k] = 0.0;
        for (long long i = threadIdx.x; i < gridDim.x; i += 128) {
#pragma unroll
          for (int k = 0; k < kScal; ++k) v[k] += __ldcg(a.scalpart + i * kScal + k);
#pragma unroll
          for (int k = 0; k < kK2Scal; ++k) v[kScal + k] += __ldcg(a.k2part + (par + i) * kK2Scal + k);
        }
#pragma unroll
        for (int k = 0; k < W; ++k) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        }
        __shared__ double sh[4][W];
        __shared__ double out[W];
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < W; ++k) sh[w][k] = v[k];
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (threadIdx.x < W) out[threadIdx.x] = ((sh[0][threadIdx.x] + sh[1][threadIdx.x]) + sh[2][threadIdx.x]) +
                                                sh[3][threadIdx.x];
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (threadIdx.x == 0) {
          if (blockIdx.x == 0) {
            double* scal = a.xbuf + N + ncol;
            for (int k = 0; k < kScal; ++k) scal[k] = out[k];
            for (int k = 0; k < kK2Scal; ++k) a.k2sum[k] = out[kScal + k];
          }
          if (!sctrl.halt) {
            const double wall = (double)(__ldcg(&a.clock[0]) - sctrl.t_start_ns) * 1e-9;
            control_step(&sctrl, out, out + kScal, blockIdx.x == 0 ? a.hist : nullptr, wall);
          }
        }
      } else {
        const int t4 = threadIdx.x - 128;
        const int g = lane & 7;
        const long long nel = (pl1 - pl0) * (NN + 2);  // (n+1) column values + the row sum per point
        // warp-uniform loop (4 elements per warp) so the group shuffles see every lane
        for (long long eb = (t4 >> 5) * 4; eb < nel; eb += (kSB / 32 - 4) * 4) {
          const long long e = eb + (lane >> 3);
          const bool ok = e < nel;
          const long long l = pl0 + (ok ? e / (NN + 2) : 0);
          const int j = ok ? (int)(e % (NN + 2)) : 0;
          const bool colp = j <= NN;
          const double* src = colp ? a.colpart + (l * (NN + 1) + j) * a.P : a.rowpart + l * a.S;
          const int cnt = ok ? (colp ? a.P : a.S) : 0;
          const int per = (cnt + 7) >> 3;
          const int lo = g * per, hi = min(cnt, lo + per);
          double sum = 0.0;
          for (int p0 = lo; p0 < hi; p0 += 8) {
            double vv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) vv[u] = p0 + u < hi ? __ldcg(src + p0 + u) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (p0 + u < hi) sum += vv[u];
          }
          sum += __shfl_xor_sync(0xffffffffu, sum, 1);
          sum += __shfl_xor_sync(0xffffffffu, sum, 2);
          sum += __shfl_xor_sync(0xffffffffu, sum, 4);
          if (g == 0 && ok) __stcg(a.xbuf + (colp ? N + l * (NN + 1) + j : l), sum);
        }
      }
      __syncthreads();
      stamp(it, 5);
      if (!sctrl.halt) primal_phase();  // identical decision in every block
    }
    stamp(it, 6);
    grid.sync();
    stamp(it, 7);
  }
  if constexpr (SV) {  // the resident tiles go back to the dual buffers (a lane owns its column)
    if (tw_col < N) {
      for (long long i = 0; i < tw_rhi - tw_rlo; ++i) {
        __stcg(a.V0 + (tw_rlo + i) * a.ld + tw_col, tile0[i * 32 + lane]);
        __stcg(a.V1 + (tw_rlo + i) * a.ld + tw_col, tile1[i * 32 + lane]);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *c = sctrl;  // full state for the host
}

constexpr size_t kResidentSmemMax = 200 * 1024;

template <int NN, bool SV>
SmallInfo small_info_for() {
  SmallInfo inf{};
  inf.fn = (const void*)small_loop_kernel<NN, SV>;
  inf.threads = small_threads<NN, SV>();
  if (SV && cudaFuncSetAttribute(inf.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kResidentSmemMax) != cudaSuccess) {
    cudaGetLastError();
    inf.fn = nullptr;
    return inf;
  }
  int bps = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, inf.fn, inf.threads,
                                                    SV ? kResidentSmemMax : 0) != cudaSuccess)
    bps = 0;
  inf.max_blocks_per_sm = bps;
  return inf;
}

template <int... Ns> struct STable;
template <int N0, int... Ns> struct STable<N0, Ns...> {
  static SmallInfo info(int n, bool sv) {
    if (n != N0) return STable<Ns...>::info(n, sv);
    return sv ? small_info_for<N0, true>() : small_info_for<N0, false>();
  }
};
template <> struct STable<> {
  static SmallInfo info(int, bool) { return SmallInfo{}; }
};
using AllS = STable<CRB_N_LIST>;

}  // namespace

SmallInfo small_loop_info(int n, bool resident) { return AllS::info(n, resident); }

size_t small_resident_smem(int RT, int threads) {
  return (size_t)(threads / 32) * 2 * (size_t)RT * 32 * sizeof(double);
}

cudaError_t launch_small_loop(const SmallInfo& info, const SmallArgs& a, int grid,
                              cudaStream_t s, size_t dyn_smem) {
  void* args[] = {const_cast<SmallArgs*>(&a)};
  return cudaLaunchCooperativeKernel(info.fn, dim3((unsigned)grid), dim3(info.threads), args,
                                     dyn_smem, s);
}

}  // namespace crb
