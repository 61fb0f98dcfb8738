// fp64 throughput microbenchmark on B200: DMMA shapes (mma.sync f64) and DFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_tput scripts/micro/fp64_tput.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_m8n8k4(double* out, int iters) {
  double d[CH][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void k_m16n8k4(double* out, int iters) {
  double d[CH][4];
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void k_m16n8k8(double* out, int iters) {
  double d[CH][4];
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0 + threadIdx.x * 1e-4, b1 = b0 + 1;
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void k_m16n8k16(double* out, int iters) {
  double d[CH][4];
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 + threadIdx.x * 1e-4 + j;
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void k_dfma(double* out, int iters) {
  double d[CH];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
  for (int c = 0; c < CH; ++c) d[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c] = fma(d[c], b, a);
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DMMA chains interleaved with DFMA chains: if the two share the fp64
// datapath, the mixed rate is the harmonic combination, else close to the sum
template <int CH, int RATIO>
__global__ void k_mixed(double* out, int iters) {
  double d[CH][2];
  double f[CH * RATIO];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = c;
  for (int c = 0; c < CH * RATIO; ++c) f[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int r = 0; r < RATIO; ++r) f[c * RATIO + r] = fma(f[c * RATIO + r], b, a);
    }
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  for (int c = 0; c < CH * RATIO; ++c) s += f[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
void run(const char* name, F kern, int warps_per_block, int iters, double flop_per_warp_iter) {
  int sms = 148;
  double* out;
  int threads = warps_per_block * 32;
  int blocks = sms * 1;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  kern<<<blocks, threads>>>(out, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double flops = flop_per_warp_iter * iters * (double)blocks * warps_per_block;
  printf("%-28s warps/SM %2d  %8.3f ms  %7.2f TFLOP/s  (%s)\n", name, warps_per_block, ms,
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  const int it = 20000;
  for (int w : {4, 8, 16, 32}) {
    run("m8n8k4 x8 chains", k_m8n8k4<8>, w, it, 8 * 512.0);
    run("m16n8k4 x8 chains", k_m16n8k4<8>, w, it, 8 * 1024.0);
    run("m16n8k8 x8 chains", k_m16n8k8<8>, w, it, 8 * 2048.0);
    run("m16n8k16 x4 chains", k_m16n8k16<4>, w, it / 2, 4 * 4096.0);
    run("dfma x8 chains", k_dfma<8>, w, it, 8 * 64.0);
  }
  for (int w : {8, 16}) {
    run("mixed 1 DMMA : 4 DFMA", k_mixed<4, 4>, w, it, 4 * (512.0 + 4 * 64.0));
    run("mixed 1 DMMA : 8 DFMA", k_mixed<4, 8>, w, it, 4 * (512.0 + 8 * 64.0));
  }
  run("m8n8k4 x1 chain (latency)", k_m8n8k4<1>, 1, it, 512.0);
  run("m16n8k8 x1 chain (latency)", k_m16n8k8<1>, 1, it, 2048.0);
  run("dfma x1 chain (latency)", k_dfma<1>, 1, it, 64.0);
  return 0;
}
