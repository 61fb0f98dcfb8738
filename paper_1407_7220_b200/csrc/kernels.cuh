// kernels.cuh -- argument blocks and launchers of the O(N n) kernels (kernels.cu)
#pragma once
#include <cuda_runtime.h>

#include "device.cuh"

namespace crb {

struct PrimalArgs {
  const double* X;       // N x n
  const double* ybar;    // N (shifted observations)
  double* rowrec;        // N x RP (y written, x static)
  double* colrec;        // N x RP
  const double* aggc;    // aggregates of V[cur] (xbuf)
  double* aggp;          // aggregates of V[prev] (aggsave); mode 0 refreshes it with aggc
  double* vpos0;         // vpos[cur] is read, vpos[1-cur] is read and then
  double* vpos1;         // overwritten with the new pos multipliers
  const int* cur;
  double* k2part;        // [blocks][kK2Scal]
  const double* coef;    // {s_cur, s_prev, beta}
  const int* stopped;
  double* yout;          // mode 1
  double* xiout;         // mode 1
  double invL, gamma;
  long long N;
  int n;
  int mode;              // 0 iteration, 1 final
  // 1: the k2 record's theta2.C eta slot carries all of it through the adjoint,
  // sum_l y_l q_y_l + xi_l . q_xi_l (the singleton per-kernel sweep does not
  // accumulate theta2 . row); 0: only the y >= 0 rows' theta2_pos y
  int tr_adjoint;
};

struct ReduceArgs {
  const double* colpart;  // [G*maxspan][TC][n1] (sweep CTA, segment) slots
  const double* rowpart;  // [S][R], S = number of row-sum slices (CTA column tiles)
  const double* scalpart; // [nw][kScal]
  const double* k2part;   // [nk2][kK2Scal]
  double* agg_out;        // [N | N n1 | kScal]
  double* k2sum;          // kK2Scal (may be null)
  const int* stopped;     // halted: rank 0 keeps agg_out, other ranks zero it
  DevCtrl* ctrl;          // non-null: the last block runs the control step
  const DevCtrl* clk;     // non-null: write the payload's clock slot (elapsed seconds
                          // since clk->t_start_ns on the shard with r0 == 0, else 0)
  double* hist;
  unsigned int* counter;  // (unused by the reduce kernel; kept for the ABI of ReduceArgs users)
  int rank;
  long long N, ld, R, r0, nw, nk2, U;
  int n1, S, TC, G, maxspan;
};

struct PowerArgs {
  const double* X;
  double* u;       // N (n+1): [u_y | u_xi]
  double* v;       // N (n+1)
  double norm_u;
  double* rowrec;
  double* colrec;
  const double* agg;
  double* part;    // [blocks][2]
  long long N;
  int n;
};

// closed-form power iteration for sigma_max(C) in one cooperative launch (power.cu)
struct PowerLoopArgs {
  double* u;            // N (n+1): in = normalised start vector, scratch afterwards
  double* v;            // N (n+1) scratch
  const double* X;
  const double* gram;   // [S (n x n) | s (n)]
  double* part;         // op 0: [2][grid][4 + 2n]; ops 1, 2: [grid][2 + 2n]
  double* part2;        // [grid][2]
  double* state;        // out: sigma, iterations, converged
  long long N;
  int n;
  int max_iters;
  double tol;
  int op;               // 0: C (cols N(n+1)), 1: A1 (cols N), 2: A2 (cols N n)
};

// one-shot metric sweeps over a given point (metrics.cu)
struct MetricsArgs {
  const double* rowrec;  // N x RQ records of the point (x, 1, y)
  const double* colrec;  // N x RQ (-xi, -c, 1)
  const double* V;       // optional: theta1 = s V (local rows) for the duality gap
  double s;
  double* part;          // [grid][2]: (sum min(row,0)^2, sum theta.row)
  long long N, R, r0, ld;
  int n, S, P;
};
cudaError_t launch_records(const double* X, const double* y, const double* xi, long long N, int n,
                           double* rowrec, double* colrec, cudaStream_t s);
cudaError_t launch_pair_metrics(const MetricsArgs& a, int grid, cudaStream_t s);
cudaError_t launch_estimator(const double* Xq, long long Q, const double* X, const double* y,
                             const double* xi, long long N, int n, double* out, int grid,
                             cudaStream_t s);

int primal_blocks(long long N);
// row records (x, 1, ybar, 0 ...) of every point, pitch RP (handle creation)
cudaError_t launch_rowrec_init(const double* X, const double* ybar, double* rowrec, long long N, int n,
                               int RP, cudaStream_t s);
// sigma start vector from host-drawn uniform pairs (power.cu); part: 148 doubles
cudaError_t launch_start_vector(const double* u12, double* v, long long cols, double* part,
                                cudaStream_t s);
cudaError_t launch_gram(const double* X, long long N, int n, double* out, cudaStream_t s);
int power_loop_grid(int sms, long long N);
cudaError_t launch_power_loop(const PowerLoopArgs& a, int grid, cudaStream_t s);
cudaError_t launch_primal(const PrimalArgs& a, cudaStream_t s);
cudaError_t launch_reduce(const ReduceArgs& a, cudaStream_t s);
cudaError_t launch_control(DevCtrl* c, const double* scal, const double* k2, double* hist,
                           cudaStream_t s);
cudaError_t launch_canon_combine(const double* pay, int D, long long len, double* out,
                                 cudaStream_t s);
cudaError_t launch_begin(DevCtrl* c, cudaStream_t s);
cudaError_t launch_stamp(unsigned long long* out, cudaStream_t s);
cudaError_t launch_power_prep(const PowerArgs& a, cudaStream_t s);
cudaError_t launch_power_post(const PowerArgs& a, cudaStream_t s);
cudaError_t launch_reduce_records(const double* part, long long count, int width, double* out,
                                  cudaStream_t s);
cudaError_t launch_theta_in(const double* stage, double* V, long long N, long long ld,
                            long long r0, long long ra, long long rb, cudaStream_t s);
cudaError_t launch_theta_out(double* stage, const double* V, double sc, long long N,
                             long long ld, long long r0, long long ra, long long rb,
                             cudaStream_t s);
cudaError_t launch_rows_out(double* stage, const double* rowrec, const double* colrec,
                            long long N, int n, long long r0, long long ra, long long rb,
                            cudaStream_t s);
cudaError_t launch_scale_copy(double* dst, const double* src, double sc, long long len,
                              cudaStream_t s);
cudaError_t launch_pos_in(double* vpos, const double* src, long long N, cudaStream_t s);
cudaError_t launch_warm_ctrl(DevCtrl* c, const double* scal_cross, double pos_sq,
                             cudaStream_t s);

}  // namespace crb
