"""Row-sharded multi-GPU solve: one process per GPU, torch.distributed for the
plumbing (rendezvous, broadcast of the NCCL unique id), NCCL inside
libcvxreg_b200.so for the per-iteration exchange.

Rank r owns pair rows [r0, r1) of the N x N multiplier matrix (both
momentum buffers). Every iteration each rank sweeps its rows and the ranks
allreduce one payload of N(n+2)+4 doubles: row sums (owned rows, zeros
elsewhere), column sums + V^T X (partial over rows) and the four sweep
scalars. The O(N n) primal update is replicated, so y, xi and every control
decision are identical on all ranks. With
PapgConfig.canonical_blocks = D the ranks allgather D per-block payloads
instead and sum them in block order, which makes the iterates bitwise
independent of the GPU count (world | D). The reference has no
distributed mode; this is the B200 scale-out of its
single-process dual state (types.hpp:50-53).
"""
from __future__ import annotations

import numpy as np

from .papg import DualPoint, MetricsSnapshot, PapgConfig, PapgResult, PrimalPoint, \
    PreparedProblem, SolveReport, TermReason, DualSolver


def shard_rows(N: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous row block of rank `rank` (sizes differ by <= 1)."""
    if not (0 <= rank < world) or world < 1 or N < world:
        raise ValueError("shard_rows: need 0 <= rank < world <= N")
    return N * rank // world, N * (rank + 1) // world


def canonical_bounds(N: int, D: int) -> list[int]:
    """Row boundaries of the D canonical blocks of cr_set_canonical_blocks: block j covers
    rows [floor(j N / D), floor((j + 1) N / D)). shard_rows(N, world, r) falls on these
    boundaries whenever world divides D."""
    if D < 1 or D > N:
        raise ValueError("canonical_bounds: need 1 <= D <= N")
    return [j * N // D for j in range(D + 1)]


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank receives it (any backend)."""
    import torch.distributed as dist

    obj = [DualSolver.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def sharded_solver(xs, ys_shifted, gamma=1e-3, device=None, group=None) -> DualSolver:
    """DualSolver over this rank's row block, attached to an NCCL communicator
    spanning the process group."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    N = xs.shape[0]
    r0, r1 = shard_rows(N, world, rank)
    if device is None:
        import torch

        device = torch.cuda.current_device()
    uid = broadcast_nccl_id(group)
    s = DualSolver(xs, ys_shifted, gamma, device=device, row_begin=r0, row_end=r1)
    if world > 1:
        s.attach_nccl(uid, rank, world)
    return s


def papg_solve_sharded(prep: PreparedProblem, cfg: PapgConfig | None = None, momentum=True,
                       group=None) -> PapgResult:
    """papg_solve over all ranks of `group`; the returned point is replicated,
    `dual` holds this rank's rows of theta_cross and the (replicated) theta_pos."""
    cfg = cfg or PapgConfig()
    with sharded_solver(prep.data.xs, prep.data.ys, cfg.gamma, group=group) as s:
        if cfg.canonical_blocks > 0:  # bitwise the same iterates on every world | D
            s.set_canonical_blocks(cfg.canonical_blocks)
        s.begin(cfg, momentum)
        stopped = False
        while not stopped:
            _, stopped = s.iterate(1 << 40)
        res, y, xi, hist = s.finish()
        th = s.theta()
        N = prep.data.N
        rows = s.row_end - s.row_begin
        dual = DualPoint(th[: rows * (N - 1)], th[rows * (N - 1):])
    history = [MetricsSnapshot(int(h[0]), *map(float, h[1:])) for h in hist]
    rep = SolveReport(history=history, reason=TermReason(res.reason), iters=int(res.iters),
                      wall_seconds=res.wall_seconds, restarts=res.restarts,
                      saturated=bool(res.saturated), history_array=hist)
    return PapgResult(PrimalPoint(y, xi), dual, rep, res.g_final, res.delta_estimate, res.sigma_C,
                      res.L_g, res.B_theta, res.sigma_iters, res.sigma_seconds, res.loop_seconds)


def local_payload(theta_rows: np.ndarray, theta_pos: np.ndarray, xs: np.ndarray, r0: int, r1: int):
    """Host restatement of one rank's exchange payload for canonical theta rows
    [r0, r1): [row sums (owned rows, 0 elsewhere) | (colsum, Theta^T X) per
    column]. Summing it over ranks gives the full-matrix aggregates that drive
    the primal closed form (operators.cpp:155-180). Used by the CPU tests of the
    sharding arithmetic."""
    N, n = xs.shape
    blk = np.zeros((r1 - r0, N))
    for i, r in enumerate(range(r0, r1)):
        row = theta_rows[i * (N - 1):(i + 1) * (N - 1)]
        blk[i, :r] = row[:r]
        blk[i, r + 1:] = row[r:]
    rowsum = np.zeros(N)
    rowsum[r0:r1] = blk.sum(1)
    colagg = np.zeros((N, n + 1))
    colagg[:, 0] = blk.sum(0)
    colagg[:, 1:] = blk.T @ xs[r0:r1]
    return np.concatenate([rowsum, colagg.reshape(-1)])
