// balcc.cuh -- launch interface of the batched block ALCC (balcc.cu)
#pragma once
#include <cuda_runtime.h>

#include "../../include/cvxreg_b200.h"

namespace crb {

struct BalccArgs {
  const double* X;       // N x n
  const double* cy;      // centres ybar_i + q_y  (N)
  const double* cxi;     // q_xi / gamma          (N n)
  const double* fy;      // feasible slice (N), (N n): block radii
  const double* fxi;
  double* ey;            // in: warm start (previous block minimisers), out: eta
  double* exi;
  const double* sigma_A2;  // K
  double sigma_A1;
  double gamma;
  double target;           // target_subopt (inner tolerance)
  cr_alcc_config cfg;
  // workspaces (global point indexing)
  double *theta;           // K nbar^2
  double *y1p, *y2, *x1p, *x2, *cc, *rs, *cs, *vx;
  double* scratch;         // K x scratch_per_block: sweep partials
  long long scratch_per_block;
  double *infeas;          // K out
  long long *iters;        // K out
  int *status;             // K out: 0 ok, 5 non-finite
  long long nbar;
  int K;
};

int balcc_max_block();
long long balcc_scratch_per_block(long long nbar, int n);
cudaError_t launch_balcc(const BalccArgs& a, int n, cudaStream_t s);

}  // namespace crb
