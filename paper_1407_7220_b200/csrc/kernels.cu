// kernels.cu -- the O(N n) kernels around the pair sweep:
//   K2 primal closed form   (apply_C_T aggregation + block centres,
//                            operators.cpp:155-180, alcc.cpp:233-235, :254-256)
//   K3 fixed-order reduce   (deterministic second stage of the sweep partials)
//   Kc control              (papg.cpp:187-262 scalar logic, one thread)
//   K4 power-method helpers (operators.cpp:302-339 on op_C)
//   K5 layout conversion    (canonical DualPoint order, indexing.hpp:30-37)
#include <cuda_runtime.h>
#include <math.h>

#include "device.cuh"
#include "iteration.cuh"
#include "kernels.cuh"

namespace crb {

namespace {

// K2. mode 0: iteration (primal at theta2, pos-row step, records);
//     mode 1: final (primal at theta1 = s_cur V[cur], outputs y/xi, no writes
//     to the dual state). NN = n is a template parameter so every load of a
//     point is issued up front.
template <int NN>
__global__ void __launch_bounds__(kPBlock) primal_kernel(const PrimalArgs a) {
  const long long N = a.N;
  // the halt flag, coefficients and slot index are independent loads: issue them
  // together (one L2 round trip before the point loads, not two), and start
  // pulling the block's first points' aggregate rows into L1 meanwhile
  {
    const long long l = (long long)blockIdx.x * kPBlock + threadIdx.x;
    if (l < N) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(a.aggc + N + l * (NN + 1)));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(a.aggp + N + l * (NN + 1)));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(a.X + l * NN));
    }
  }
  const int stop = a.stopped != nullptr ? *a.stopped : 0;
  const double s_c = a.coef[0];
  const double s_p = a.mode == 0 ? a.coef[1] : 0.0;
  const double beta = a.mode == 0 ? a.coef[2] : 0.0;
  const int cur = *a.cur;
  if (stop) return;
  const double* vposc = cur ? a.vpos1 : a.vpos0;
  double* vposp = cur ? a.vpos0 : a.vpos1;
  double acc[kK2Scal];
#pragma unroll
  for (int w = 0; w < kK2Scal; ++w) acc[w] = 0.0;
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock)
    primal_point<NN>(a, l, s_c, s_p, beta, vposc, vposp, acc);
  block_reduce_store<kK2Scal, kPBlock>(acc, a.k2part + (long long)blockIdx.x * kK2Scal);
}

// sharded / phased iterations: scal[kScal] is the payload's clock slot (the
// elapsed time of the shard owning row 0), so every rank takes the same
// time-budget decision (papg.cpp:233-236)
__global__ void control_kernel(DevCtrl* c, const double* scal /* kScal + clock, allreduced */,
                               const double* k2 /* kK2Scal, replicated */, double* hist) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (c->halt) return;
  control_step(c, scal, k2, hist, scal[kScal]);
}

// fixed-order sum of the sweep scalar records and the K2 records (one block):
// per thread in record order (2 records per batch), warp butterflies, then the
// 8 warps in order -- small shared memory and registers, so the reduce kernel's
// column / row blocks run in a single wave
__device__ __forceinline__ void scalar_records(const ReduceArgs& a, long long scal_at,
                                               long long nk2) {
  constexpr int W = kScal + kK2Scal;
  double v[W];
#pragma unroll
  for (int w = 0; w < W; ++w) v[w] = 0.0;
  for (long long i0 = threadIdx.x; i0 < a.nw; i0 += 2 * kBlock) {
    double r2[2][kScal];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long i = i0 + (long long)u * kBlock;
#pragma unroll
      for (int w = 0; w < kScal; ++w) r2[u][w] = i < a.nw ? a.scalpart[i * kScal + w] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int w = 0; w < kScal; ++w) v[w] += r2[u][w];
    }
  }
  for (long long i = threadIdx.x; i < nk2; i += kBlock) {
#pragma unroll
    for (int w = 0; w < kK2Scal; ++w) v[kScal + w] += __ldcg(a.k2part + i * kK2Scal + w);
  }
  __shared__ double sh[kBlock / 32][W];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < W; ++w) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[w] += __shfl_xor_sync(0xffffffffu, v[w], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w) sh[warp][w] = v[w];
  }
  __syncthreads();
  if (threadIdx.x < W) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kBlock / 32; ++k) t += sh[k][threadIdx.x];
    if (threadIdx.x < kScal) a.agg_out[scal_at + threadIdx.x] = t;
    else if (a.k2sum != nullptr) a.k2sum[threadIdx.x - kScal] = t;
  }
  if (threadIdx.x == 0 && a.clk != nullptr)
    a.agg_out[scal_at + kScal] = a.r0 == 0 ? (double)(globaltimer() - a.clk->t_start_ns) * 1e-9 : 0.0;
}

// K3: fixed-order reduction of the sweep partials. On a single GPU block 0
// also runs the control step (no separate launch); sharded runs call
// control_kernel after the allreduce instead.
__global__ void __launch_bounds__(kBlock, 6) reduce_kernel(const ReduceArgs a) {
  const long long N = a.N;
  const int n1 = a.n1;
  const long long ncol = N * n1;
  // With the control step fused (single GPU) only block 0 looks at the halt flag:
  // it is the block that may set it, and a halted solve's sweep did not run, so
  // re-reducing its unchanged partials rewrites identical aggregates.
  if (a.ctrl == nullptr && a.stopped != nullptr && *a.stopped) {
    // halted: keep the (already reduced) payload on rank 0, zero it elsewhere,
    // so a trailing in-place allreduce leaves it unchanged on every rank
    if (a.rank != 0) {
      const long long total = N + ncol + kScal + 1;
      for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < total;
           i += (long long)gridDim.x * kBlock)
        a.agg_out[i] = 0.0;
    }
    return;
  }
  // column aggregates: one block per (column tile, chunk of its TC x n1 values);
  // the tile's values of one (CTA, segment) slot are contiguous, so a block sums
  // a few contiguous slot arrays in CTA order (no per-element index division)
  const long long per_tile = (long long)a.TC * n1;
  const long long chunks = (per_tile + kBlock - 1) / kBlock;
  const long long T = (N + a.TC - 1) / a.TC;
  const long long nb_col = T * chunks;
  const long long nb_row = (N + 31) / 32;
  // block 0: the scalar records (the longest chain, so it is dispatched first)
  const long long b = (long long)blockIdx.x - 1;
  if (b < 0) {
    // scalars first, then (single GPU) the control step right away: it needs
    // only the scalars, so it runs while the other blocks reduce the aggregates
    if (a.ctrl != nullptr && a.ctrl->halt) return;
    scalar_records(a, N + ncol, a.nk2);
    if (a.ctrl != nullptr) {
      __syncthreads();
      if (threadIdx.x == 0) control_step(a.ctrl, a.agg_out + N + ncol, a.k2sum, a.hist);
    }
  } else if (b < nb_col) {
    // column tile t was swept by CTAs g_lo..g_hi (contiguous unit ranges)
    const long long t = b / chunks;
    const long long e = (b - t * chunks) * kBlock + threadIdx.x;
    const long long g_lo = (t * a.R) / a.U;
    long long g_hi = ((t + 1) * a.R - 1) / a.U;
    if (g_hi > a.G - 1) g_hi = a.G - 1;
    __shared__ long long slot_off[64];
    const long long nslot = g_hi - g_lo + 1;
    for (long long k = threadIdx.x; k < nslot && k < 64; k += kBlock) {
      const long long g = g_lo + k;
      slot_off[k] = (g * a.maxspan + (t - (g * a.U) / a.R)) * per_tile;
    }
    __syncthreads();
    if (e < per_tile && e < (N - t * a.TC) * n1) {
      // slot values loaded in batches of 4 (independent loads), summed in CTA order
      double s = 0.0;
      for (long long k0 = 0; k0 < nslot; k0 += 4) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long long k = k0 + u;
          const long long off =
              k < 64 ? slot_off[k < 64 ? k : 0]
                     : ((g_lo + k) * a.maxspan + (t - ((g_lo + k) * a.U) / a.R)) * per_tile;
          v[u] = k < nslot ? a.colpart[off + e] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (k0 + u < nslot) s += v[u];
      }
      a.agg_out[N + t * per_tile + e] = s;
    }
  } else if (b < nb_col + nb_row) {
    // row sums: 32 rows x 8 slice groups per block (lane = row, warp = group of
    // column-tile slices st = w, w + 8, ...), then a fixed-order combine
    __shared__ double part[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long r = (b - nb_col) * 32 + lane;
    const long long lr = r - a.r0;
    const bool own = r < N && lr >= 0 && lr < a.R;
    double s = 0.0;
    if (own) {
      for (int st0 = w; st0 < a.S; st0 += 8 * 4) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int st = st0 + 8 * u;
          v[u] = st < a.S ? a.rowpart[(long long)st * a.R + lr] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) s += v[u];
      }
    }
    part[w][lane] = s;
    __syncthreads();
    if (w == 0 && r < N) {
      double u = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) u += part[k][lane];
      a.agg_out[r] = u;
    }
  }
}


__global__ void rowrec_init_kernel(const double* X, const double* ybar, double* rowrec, long long N,
                                   int n, int RP) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N * RP) return;
  const long long l = k / RP;
  const int j = (int)(k - l * RP);
  rowrec[k] = j < n ? X[l * n + j] : (j == n ? 1.0 : (j == n + 1 ? ybar[l] : 0.0));
}

__global__ void begin_kernel(DevCtrl* c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) c->t_start_ns = globaltimer();
}

__global__ void stamp_kernel(unsigned long long* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = globaltimer();
}

// K4a: v = u / norm_u (operators.cpp:327) and the records of eta = v
__global__ void __launch_bounds__(kPBlock) power_prep_kernel(const PowerArgs a) {
  const long long N = a.N;
  const int n = a.n;
  const int RP = rec_pitch(n);
  double acc[1] = {0.0};
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock) {
    const double vy = a.u[l] / a.norm_u;
    a.v[l] = vy;
    double cx = 0.0;
    const double* x = a.X + l * n;
    double* crec = a.colrec + l * RP;
    for (int j = 0; j < n; ++j) {
      const double vxi = a.u[N + l * n + j] / a.norm_u;
      a.v[N + l * n + j] = vxi;
      cx = fma(vxi, x[j], cx);
      crec[j] = -vxi;
    }
    crec[n] = -(vy - cx);
    crec[n + 1] = 1.0;
    a.rowrec[l * RP + n + 1] = vy;
    acc[0] = fma(vy, vy, acc[0]);  // pos rows of C v = v_y
  }
  block_reduce_store<1, kPBlock>(acc, a.part + (long long)blockIdx.x * 2);
}

// K4b: u = C^T w from the reduced aggregates (operators.cpp:161-178)
__global__ void __launch_bounds__(kPBlock) power_post_kernel(const PowerArgs a) {
  const long long N = a.N;
  const int n = a.n;
  double acc[1] = {0.0};
  for (long long l = (long long)blockIdx.x * kPBlock + threadIdx.x; l < N;
       l += (long long)gridDim.x * kPBlock) {
    const double rs = a.agg[l];
    const double cs = a.agg[N + l * (n + 1)];
    const double uy = a.v[l] + rs - cs;
    a.u[l] = uy;
    double s = uy * uy;
    const double* x = a.X + l * n;
    for (int j = 0; j < n; ++j) {
      const double ux = cs * x[j] - a.agg[N + l * (n + 1) + 1 + j];
      a.u[N + l * n + j] = ux;
      s = fma(ux, ux, s);
    }
    acc[0] += s;
  }
  block_reduce_store<1, kPBlock>(acc, a.part + (long long)blockIdx.x * 2 + 1);
}

// fixed-order sum of `count` records of width `width` -> out[width]
__global__ void __launch_bounds__(kBlock) reduce_records_kernel(const double* part,
                                                                long long count, int width,
                                                                double* out) {
  double v[kK2Scal];
#pragma unroll
  for (int w = 0; w < kK2Scal; ++w) v[w] = 0.0;
  for (long long i = threadIdx.x; i < count; i += kBlock)
#pragma unroll
    for (int w = 0; w < kK2Scal; ++w)
      if (w < width) v[w] += part[i * width + w];
  __shared__ double o[kK2Scal];
  block_reduce_store<kK2Scal>(v, o);
  __syncthreads();
  if ((int)threadIdx.x < width && threadIdx.x < kK2Scal) out[threadIdx.x] = o[threadIdx.x];
}

// K5: canonical theta rows [a, b) (local) <-> device V
__global__ void theta_in_kernel(const double* stage, double* V, long long N, long long ld,
                                long long r0, long long ra, long long rb) {
  const long long total = (rb - ra) * ld;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long lr = i / ld, c = i % ld;
    const long long r = ra + lr, gr = r0 + r;
    double v = 0.0;
    if (c < N && c != gr) {
      const double t = stage[lr * (N - 1) + c - (c > gr ? 1 : 0)];
      v = t > 0.0 ? t : 0.0;  // projections.hpp:10 (scale applied separately)
    }
    V[r * ld + c] = v;
  }
}

__global__ void theta_out_kernel(double* stage, const double* V, double s, long long N,
                                 long long ld, long long r0, long long ra, long long rb) {
  const long long total = (rb - ra) * (N - 1);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long lr = i / (N - 1), k = i % (N - 1);
    const long long gr = r0 + ra + lr;
    const long long c = k + (k >= gr ? 1 : 0);
    stage[i] = s * V[(ra + lr) * ld + c];
  }
}

__global__ void rows_out_kernel(double* stage, const double* rowrec, const double* colrec,
                                long long N, int n, long long r0, long long ra, long long rb) {
  const int RP = rec_pitch(n);
  const long long total = (rb - ra) * (N - 1);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long lr = i / (N - 1), k = i % (N - 1);
    const long long gr = r0 + ra + lr;
    const long long c = k + (k >= gr ? 1 : 0);
    const double* xr = rowrec + gr * RP;
    const double* cr = colrec + c * RP;
    double row = xr[n + 1] + cr[n];  // y_l1 - c_l2 - x_l1 . xi_l2
    for (int j = 0; j < n; ++j) row = fma(xr[j], cr[j], row);
    stage[i] = row;
  }
}

__global__ void scale_copy_kernel(double* dst, const double* src, double s, long long len) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = s * src[i];
}

__global__ void pos_in_kernel(double* vpos, const double* src, long long N) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    vpos[i] = src[i] > 0.0 ? src[i] : 0.0;
}

// warm start: s = min(1, B / |max(theta0, 0)|) (papg.cpp:163), coefficient
// state for iteration 1 (theta1 = theta1_prev = theta2, t = 1)
__global__ void warm_ctrl_kernel(DevCtrl* c, const double* scal_cross, double pos_sq) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double ss = scal_cross[0] + pos_sq;
  const double norm = sqrt(ss);
  const double s = norm > c->B_theta ? c->B_theta / norm : 1.0;
  c->s_cur = s;
  c->s_prev = s;
  c->beta = 0.0;
}

unsigned grid_for(long long n, int block, int cap) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

}  // namespace

int primal_blocks(long long N) { return (int)grid_for(N, kPBlock, 4736); }

template <int NN>
void launch_primal_n(const PrimalArgs& a, cudaStream_t s) {
  primal_kernel<NN><<<primal_blocks(a.N), kPBlock, 0, s>>>(a);
}
using PrimalLauncher = void (*)(const PrimalArgs&, cudaStream_t);
cudaError_t launch_primal(const PrimalArgs& a, cudaStream_t s) {
  static constexpr PrimalLauncher tab[kMaxN] = {
#define CRB_LP(N) launch_primal_n<N>
      CRB_N_SEQ(CRB_LP)
#undef CRB_LP
};
  if (a.n < 1 || a.n > kMaxN) return cudaErrorInvalidValue;
  tab[a.n - 1](a, s);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const ReduceArgs& a, cudaStream_t s) {
  const long long chunks = ((long long)a.TC * a.n1 + kBlock - 1) / kBlock;
  const long long nb = (a.N + a.TC - 1) / a.TC * chunks + (a.N + 31) / 32 + 1;
  reduce_kernel<<<(unsigned)nb, kBlock, 0, s>>>(a);
  return cudaGetLastError();
}

// canonical-block mode: the payload is the sum of the D block payloads in block
// order (left to right), whatever GPU produced each of them
__global__ void canon_combine_kernel(const double* __restrict__ pay, int D, long long len,
                                     double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  double s = pay[i];
  for (int j = 1; j < D; ++j) s += pay[(long long)j * len + i];
  out[i] = s;
}

cudaError_t launch_canon_combine(const double* pay, int D, long long len, double* out,
                                 cudaStream_t s) {
  canon_combine_kernel<<<(unsigned)((len + 255) / 256), 256, 0, s>>>(pay, D, len, out);
  return cudaGetLastError();
}

cudaError_t launch_control(DevCtrl* c, const double* scal, const double* k2, double* hist,
                           cudaStream_t s) {
  control_kernel<<<1, 32, 0, s>>>(c, scal, k2, hist);
  return cudaGetLastError();
}

cudaError_t launch_begin(DevCtrl* c, cudaStream_t s) {
  begin_kernel<<<1, 32, 0, s>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_stamp(unsigned long long* out, cudaStream_t s) {
  stamp_kernel<<<1, 32, 0, s>>>(out);
  return cudaGetLastError();
}

cudaError_t launch_rowrec_init(const double* X, const double* ybar, double* rowrec, long long N, int n,
                               int RP, cudaStream_t s) {
  const long long tot = N * RP;
  rowrec_init_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(X, ybar, rowrec, N, n, RP);
  return cudaGetLastError();
}

cudaError_t launch_power_prep(const PowerArgs& a, cudaStream_t s) {
  power_prep_kernel<<<primal_blocks(a.N), kPBlock, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_power_post(const PowerArgs& a, cudaStream_t s) {
  power_post_kernel<<<primal_blocks(a.N), kPBlock, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_reduce_records(const double* part, long long count, int width, double* out,
                                  cudaStream_t s) {
  reduce_records_kernel<<<1, kBlock, 0, s>>>(part, count, width, out);
  return cudaGetLastError();
}

cudaError_t launch_theta_in(const double* stage, double* V, long long N, long long ld,
                            long long r0, long long ra, long long rb, cudaStream_t s) {
  theta_in_kernel<<<grid_for((rb - ra) * ld, 256, 4096), 256, 0, s>>>(stage, V, N, ld, r0, ra,
                                                                       rb);
  return cudaGetLastError();
}

cudaError_t launch_theta_out(double* stage, const double* V, double sc, long long N,
                             long long ld, long long r0, long long ra, long long rb,
                             cudaStream_t s) {
  theta_out_kernel<<<grid_for((rb - ra) * (N - 1), 256, 4096), 256, 0, s>>>(stage, V, sc, N, ld,
                                                                            r0, ra, rb);
  return cudaGetLastError();
}


cudaError_t launch_rows_out(double* stage, const double* rowrec, const double* colrec,
                            long long N, int n, long long r0, long long ra, long long rb,
                            cudaStream_t s) {
  rows_out_kernel<<<grid_for((rb - ra) * (N - 1), 256, 4096), 256, 0, s>>>(stage, rowrec, colrec,
                                                                           N, n, r0, ra, rb);
  return cudaGetLastError();
}

cudaError_t launch_scale_copy(double* dst, const double* src, double sc, long long len,
                              cudaStream_t s) {
  scale_copy_kernel<<<grid_for(len, 256, 1024), 256, 0, s>>>(dst, src, sc, len);
  return cudaGetLastError();
}

cudaError_t launch_pos_in(double* vpos, const double* src, long long N, cudaStream_t s) {
  pos_in_kernel<<<grid_for(N, 256, 1024), 256, 0, s>>>(vpos, src, N);
  return cudaGetLastError();
}

cudaError_t launch_warm_ctrl(DevCtrl* c, const double* scal_cross, double pos_sq,
                             cudaStream_t s) {
  warm_ctrl_kernel<<<1, 32, 0, s>>>(c, scal_cross, pos_sq);
  return cudaGetLastError();
}

}  // namespace crb
