// small.cuh -- persistent cooperative dual loop for small N (small.cu)
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"
#include "kernels.cuh"

namespace crb {

struct SmallArgs {
  PrimalArgs pa;       // K2 arguments (mode 0): records, aggregates, vpos, k2part
  double* V0;
  double* V1;
  double* colpart;     // [N][n+1][P]
  double* rowpart;     // [N][S]
  double* scalpart;    // [grid][kScal]
  double* k2part;      // [grid][kK2Scal]
  double* xbuf;        // aggregates of the newest V (also read by K2 as aggc)
  double* k2sum;
  double* hist;
  DevCtrl* ctrl;
  long long N, ld;
  long long max_iters; // iterations this launch may run (halts earlier on termination)
  int S, P;            // 32-column strips, row chunks
  int RT;              // resident variant: rows of a warp's V / V' tile (>= ceil(N / P))
  unsigned long long* trace;  // optional: block 0 phase timestamps (CRB_TRACE), 8 per iteration
  unsigned long long* clock;  // one timestamp per iteration (block 0): every block's time budget
};

struct SmallInfo {
  const void* fn;
  int threads;
  int max_blocks_per_sm;
};

// resident = true: the variant that keeps every warp's V / V' tile in shared memory for the
// whole launch (one (strip, chunk) task per warp; needs small_resident_smem(RT) bytes of
// dynamic shared memory per block)
SmallInfo small_loop_info(int n, bool resident = false);
size_t small_resident_smem(int RT, int threads);
cudaError_t launch_small_loop(const SmallInfo& info, const SmallArgs& a, int grid,
                              cudaStream_t s, size_t dyn_smem = 0);

}  // namespace crb
