// sweep.cu -- K1, the fused pair sweep (one HBM pass over the lambda stream
// per dual iteration).
//
// Replaces, for the singleton-block closed form, the reference's per-iteration
// passes: apply_C (operators.cpp:128-153), the projected step
// (papg.cpp:187-189, projections.hpp:9-13), the metric reductions
// (papg.cpp:191-208) and apply_C_T of the next iterate (operators.cpp:155-180).
//
// Work decomposition: a warp owns a strip of 32*C adjacent columns (l2) and a
// contiguous chunk of rows (l1). Column state -- c_l2, xi_l2 and the column
// aggregates (colsum, V^T X) -- lives in registers for the whole chunk, so the
// column reductions need no communication. Row records (y_l1, x_l1) are staged
// per 32-row tile in shared memory and read as warp broadcasts. Row sums go
// through a 32x33 shared transpose so each lane reduces one row. Per pair:
//   row   = y_l1 - c_l2 - x_l1 . xi_l2                    (= C eta entry)
//   th2   = th1 + beta (th1 - th1p), th1 = s V, th1p = s' V'
//   v     = max(th2 - row / L, 0)                         (unscaled projection)
//   S_vv += v^2, S_vr += v row, S_tr += th2 row, S_nn += min(row,0)^2
//   colagg[l2] += (v, v x_l1), rowsum[l1] += v
// HBM traffic: 8 B read V, 8 B read V', 8 B write v -> 24 B per pair.
#include <cuda_runtime.h>

#include "device.cuh"

namespace crb {

namespace {

constexpr int kWarpsPerBlock = 4;

template <int C> struct VecT;
template <> struct VecT<1> { using T = double; };
template <> struct VecT<2> { using T = double2; };

__device__ __forceinline__ double vget(const double& v, int) { return v; }
__device__ __forceinline__ double vget(const double2& v, int k) { return k == 0 ? v.x : v.y; }
__device__ __forceinline__ void vset(double& v, int, double x) { v = x; }
__device__ __forceinline__ void vset(double2& v, int k, double x) {
  if (k == 0) v.x = x; else v.y = x;
}

// streaming loads/stores: lambda is touched once per iteration, keep it out of L1
__device__ __forceinline__ double ld_stream(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
// V' is read and then overwritten by the same thread: a plain (coherent) load
__device__ __forceinline__ double ld_rw(const double* p) {
  double r;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_rw(const double2* p) {
  double2 r;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(double* p, double v) {
  asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y)
               : "memory");
}

template <int NN>
__host__ __device__ constexpr int rec_pitch() { return (NN + 2) & ~1; }

template <int NN, int C>
__host__ __device__ constexpr int smem_doubles_per_warp() { return 32 * rec_pitch<NN>() + 32 * 33; }

template <int NN, int C, int MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
sweep_kernel(const SweepArgs a) {
  using VT = typename VecT<C>::T;
  constexpr int RP = rec_pitch<NN>();
  constexpr int U = (C == 2) ? 4 : 8;  // rows of V in flight per batch
  extern __shared__ __align__(16) double smem[];

  if (a.stopped != nullptr && *a.stopped) return;
  const int cur = (MODE == kModePapg) ? *a.cur : 0;
  const double* Vc = cur ? a.V1 : a.V0;
  double* Vp = cur ? a.V0 : a.V1;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long gw = (long long)blockIdx.x * kWarpsPerBlock + wib;
  if (gw >= (long long)a.S * a.P) return;
  const int strip = (int)(gw % a.S);
  const int chunk = (int)(gw / a.S);
  const long long rlo = a.R * chunk / a.P;
  const long long rhi = a.R * (chunk + 1) / a.P;
  const long long col0 = (long long)strip * (32 * C) + lane * C;
  double* srow = smem + wib * smem_doubles_per_warp<NN, C>();
  double* srs = srow + 32 * RP;

  // column state for this lane's C columns
  double cc[C], xi[C][NN], acc[C][NN + 1];
  bool cvalid[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const long long col = col0 + k;
    cvalid[k] = col < a.N;
    const double* rec = a.colrec + (cvalid[k] ? col : 0) * RP;
    cc[k] = cvalid[k] ? __ldg(rec) : 0.0;
#pragma unroll
    for (int j = 0; j < NN; ++j) xi[k][j] = cvalid[k] ? __ldg(rec + 1 + j) : 0.0;
#pragma unroll
    for (int j = 0; j <= NN; ++j) acc[k][j] = 0.0;
  }
  double s_c = 1.0, s_p = 0.0, beta = 0.0;
  if (MODE == kModePapg) {
    s_c = a.coef[0];
    s_p = a.coef[1];
    beta = a.coef[2];
  }
  const double invL = a.invL;
  double vv = 0.0, vr = 0.0, tr = 0.0, nn = 0.0;

  for (long long rt = rlo; rt < rhi; rt += 32) {
    const int nrows = (int)min(32LL, rhi - rt);
    {  // stage the row records of this tile (contiguous, RP even -> double2)
      const double2* src = reinterpret_cast<const double2*>(a.rowrec + (a.r0 + rt) * RP);
      double2* dst = reinterpret_cast<double2*>(srow);
      for (int i = lane; i < nrows * (RP / 2); i += 32) dst[i] = __ldg(src + i);
    }
    __syncwarp();
    for (int rb = 0; rb < nrows; rb += U) {
      VT vc[U], vp[U];
      if (MODE == kModePapg) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (rb + u < nrows) {
            const long long off = (rt + rb + u) * a.ld + col0;
            vc[u] = ld_stream(reinterpret_cast<const VT*>(Vc + off));
            vp[u] = ld_rw(reinterpret_cast<const VT*>(Vp + off));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rr = rb + u;
        if (rr < nrows) {
          const long long gr = a.r0 + rt + rr;
          const double* xr = srow + rr * RP;
          double x[NN];
          const double y1 = xr[0];
#pragma unroll
          for (int j = 0; j < NN; ++j) x[j] = xr[1 + j];
          double rs = 0.0;
          VT out;
#pragma unroll
          for (int k = 0; k < C; ++k) {
            double row = y1 - cc[k];
#pragma unroll
            for (int j = 0; j < NN; ++j) row = fma(-x[j], xi[k][j], row);
            if (!cvalid[k] || col0 + k == gr) row = 0.0;
            double v;
            if (MODE == kModePapg) {
              const double th1 = s_c * vget(vc[u], k);
              const double th1p = s_p * vget(vp[u], k);
              const double th2 = fma(beta, th1 - th1p, th1);
              v = fmax(fma(-row, invL, th2), 0.0);
              vset(out, k, v);
              vv = fma(v, v, vv);
              vr = fma(v, row, vr);
              tr = fma(th2, row, tr);
              const double m = fmin(row, 0.0);
              nn = fma(m, m, nn);
            } else {
              v = row;
              vv = fma(row, row, vv);
            }
            acc[k][0] += v;
#pragma unroll
            for (int j = 0; j < NN; ++j) acc[k][1 + j] = fma(v, x[j], acc[k][1 + j]);
            rs += v;
          }
          if (MODE == kModePapg)
            st_stream(reinterpret_cast<VT*>(Vp + (rt + rr) * a.ld + col0), out);
          srs[rr * 33 + lane] = rs;
        }
      }
    }
    __syncwarp();
    if (lane < nrows) {  // fixed-order row reduction of the tile
      double s = 0.0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) s += srs[lane * 33 + l];
      a.rowpart[(long long)strip * a.R + rt + lane] = s;
    }
    __syncwarp();
  }

  // column partials of this (strip, chunk)
#pragma unroll
  for (int k = 0; k < C; ++k) {
    double* dst = a.colpart + ((long long)chunk * a.ld + col0 + k) * (NN + 1);
#pragma unroll
    for (int j = 0; j <= NN; ++j) dst[j] = acc[k][j];
  }
  // scalar partials: fixed butterfly -> deterministic
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    vv += __shfl_xor_sync(0xffffffffu, vv, off);
    vr += __shfl_xor_sync(0xffffffffu, vr, off);
    tr += __shfl_xor_sync(0xffffffffu, tr, off);
    nn += __shfl_xor_sync(0xffffffffu, nn, off);
  }
  if (lane == 0) {
    double* sp = a.scalpart + gw * kScal;
    sp[0] = vv;
    sp[1] = vr;
    sp[2] = tr;
    sp[3] = nn;
  }
}

template <int NN>
__host__ __device__ constexpr int cols_per_lane() { return NN <= 12 ? 2 : 1; }

template <int NN>
SweepKernelInfo info_for(int mode) {
  constexpr int C = cols_per_lane<NN>();
  SweepKernelInfo inf;
  inf.fn = mode == kModePapg ? (const void*)sweep_kernel<NN, C, kModePapg>
                             : (const void*)sweep_kernel<NN, C, kModePower>;
  inf.C = C;
  inf.warps_per_block = kWarpsPerBlock;
  const int smem = kWarpsPerBlock * smem_doubles_per_warp<NN, C>() * 8;
  cudaFuncSetAttribute(inf.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bps = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, inf.fn, kWarpsPerBlock * 32, smem) !=
      cudaSuccess)
    bps = 0;
  inf.max_blocks_per_sm = bps;
  return inf;
}

template <int NN>
int launch_for(const SweepKernelInfo& info, const SweepArgs& a, cudaStream_t s) {
  constexpr int C = cols_per_lane<NN>();
  const int smem = kWarpsPerBlock * smem_doubles_per_warp<NN, C>() * 8;
  const long long warps = (long long)a.S * a.P;
  const unsigned grid = (unsigned)((warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
  void* args[] = {const_cast<SweepArgs*>(&a)};
  return (int)cudaLaunchKernel(info.fn, dim3(grid), dim3(kWarpsPerBlock * 32), args, smem, s);
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
