// metrics.cu -- one-shot O(N^2 n) sweeps over a given primal point
// (reference: metrics.cpp, runner.cpp:296-343):
//   infeasibility   |(A1 y + A2 xi)_-|_2 over all N(N-1) rows   metrics.cpp:8-15
//   duality gap     theta . C eta with the handle's theta1       metrics.cpp:17-30, runner.cpp:315-319
//   estimator       max_l y_l + xi_l.(x - x_l) for Q queries    metrics.cpp:32-48
//   repair          y'_l = estimator(x_l)                         metrics.cpp:50-56
// The pair sweep reads point records built by records_kernel (same layout as
// the solver's rowrec/colrec) and, for the gap, the device-resident V.
#include <cuda_runtime.h>
#include <math.h>

#include "device.cuh"
#include "kernels.cuh"

namespace crb {

namespace {

constexpr int kMBlock = 256;

// rowrec = (x, 1, y), colrec = (-xi, -(y - xi.x), 1) of a given point
__global__ void records_kernel(const double* X, const double* y, const double* xi, long long N,
                               int n, double* rowrec, double* colrec) {
  const int RQ = rec_pitch(n);
  for (long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x; l < N;
       l += (long long)gridDim.x * blockDim.x) {
    double* rr = rowrec + l * RQ;
    double* cr = colrec + l * RQ;
    double cx = 0.0;
    for (int j = 0; j < n; ++j) {
      const double x = X[l * n + j], g = xi[l * n + j];
      rr[j] = x;
      cr[j] = -g;
      cx = fma(g, x, cx);
    }
    rr[n] = 1.0;
    rr[n + 1] = y[l];
    cr[n] = -(y[l] - cx);
    cr[n + 1] = 1.0;
    for (int j = n + 2; j < RQ; ++j) rr[j] = cr[j] = 0.0;
  }
}

// per block: (sum min(row,0)^2, sum theta.row) over rows [0, R) of this shard
template <int NN>
__global__ void __launch_bounds__(kMBlock) pair_metrics_kernel(const MetricsArgs a) {
  constexpr int RQ = rec_pitch(NN);
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * kMBlock + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * kMBlock) >> 5;
  const long long N = a.N;
  double nn = 0.0, gap = 0.0;
  for (long long w = gwarp; w < (long long)a.S * a.P; w += nwarps) {
    const int strip = (int)(w % a.S);
    const int chunk = (int)(w / a.S);
    const long long rlo = a.R * chunk / a.P, rhi = a.R * (chunk + 1) / a.P;
    const long long col = (long long)strip * 32 + lane;
    const bool valid = col < N;
    const double* cr = a.colrec + (valid ? col : 0) * RQ;
    double cc = valid ? cr[NN] : 0.0, xi[NN];
#pragma unroll
    for (int j = 0; j < NN; ++j) xi[j] = valid ? cr[j] : 0.0;
    for (long long r = rlo; r < rhi; ++r) {
      const long long g = a.r0 + r;
      const double* xr = a.rowrec + g * RQ;
      double row = xr[NN + 1] + cc;
#pragma unroll
      for (int j = 0; j < NN; ++j) row = fma(xr[j], xi[j], row);
      if (!valid || col == g) row = 0.0;
      const double m = row < 0.0 ? row : 0.0;
      nn = fma(m, m, nn);
      if (a.V != nullptr && valid)
        gap = fma(a.s * a.V[r * a.ld + col], row, gap);
    }
  }
  // fixed-order block reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nn += __shfl_xor_sync(0xffffffffu, nn, o);
    gap += __shfl_xor_sync(0xffffffffu, gap, o);
  }
  __shared__ double sh[kMBlock / 32][2];
  if (lane == 0) {
    sh[threadIdx.x >> 5][0] = nn;
    sh[threadIdx.x >> 5][1] = gap;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int k = 0; k < kMBlock / 32; ++k) t += sh[k][threadIdx.x];
    a.part[(long long)blockIdx.x * 2 + threadIdx.x] = t;
  }
}

// one warp per query: max over points of y_l + xi_l.(x_q - x_l) (metrics.cpp:41-46)
template <int NN>
__global__ void __launch_bounds__(kMBlock) estimator_kernel(const double* Xq, long long Q,
                                                            const double* X, const double* y,
                                                            const double* xi, long long N,
                                                            double* out) {
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * kMBlock + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * kMBlock) >> 5;
  for (long long q = gwarp; q < Q; q += nwarps) {
    double xq[NN];
#pragma unroll
    for (int j = 0; j < NN; ++j) xq[j] = Xq[q * NN + j];
    double best = -INFINITY;
    for (long long l = lane; l < N; l += 32) {
      double v = y[l];
#pragma unroll
      for (int j = 0; j < NN; ++j) v += xi[l * NN + j] * (xq[j] - X[l * NN + j]);
      best = fmax(best, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) out[q] = best;
  }
}

template <int NN>
void metrics_n(const MetricsArgs& a, int grid, cudaStream_t s) {
  pair_metrics_kernel<NN><<<grid, kMBlock, 0, s>>>(a);
}
template <int NN>
void estimator_n(const double* Xq, long long Q, const double* X, const double* y,
                 const double* xi, long long N, double* out, int grid, cudaStream_t s) {
  estimator_kernel<NN><<<grid, kMBlock, 0, s>>>(Xq, Q, X, y, xi, N, out);
}
using MetricsFn = void (*)(const MetricsArgs&, int, cudaStream_t);
using EstimatorFn = void (*)(const double*, long long, const double*, const double*,
                             const double*, long long, double*, int, cudaStream_t);

#define CRB_MET(N) metrics_n<N>
#define CRB_EST(N) estimator_n<N>

}  // namespace

cudaError_t launch_records(const double* X, const double* y, const double* xi, long long N, int n,
                           double* rowrec, double* colrec, cudaStream_t s) {
  long long g = (N + 255) / 256;
  if (g > 4096) g = 4096;
  records_kernel<<<(unsigned)g, 256, 0, s>>>(X, y, xi, N, n, rowrec, colrec);
  return cudaGetLastError();
}

cudaError_t launch_pair_metrics(const MetricsArgs& a, int grid, cudaStream_t s) {
  static constexpr MetricsFn tab[kMaxN] = {CRB_N_SEQ(CRB_MET)};
  if (a.n < 1 || a.n > kMaxN) return cudaErrorInvalidValue;
  tab[a.n - 1](a, grid, s);
  return cudaGetLastError();
}

cudaError_t launch_estimator(const double* Xq, long long Q, const double* X, const double* y,
                             const double* xi, long long N, int n, double* out, int grid,
                             cudaStream_t s) {
  static constexpr EstimatorFn tab[kMaxN] = {CRB_N_SEQ(CRB_EST)};
  if (n < 1 || n > kMaxN) return cudaErrorInvalidValue;
  tab[n - 1](Xq, Q, X, y, xi, N, out, grid, s);
  return cudaGetLastError();
}

}  // namespace crb
