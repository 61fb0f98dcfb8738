"""Multi-process (gloo, world_size 2) CPU tests of the row-sharded path:
shard layout, NCCL-id broadcast over torch.distributed, and the exchange
arithmetic (per-rank payloads summed over ranks == full aggregates, primal
closed form identical on every rank). The GPU kernels themselves are covered
by the 1-GPU sharded emulation in test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest

from paper_1407_7220_b200.dist import canonical_bounds, local_payload, shard_rows


def test_shard_rows_cover_and_balance():
    for N in (2, 7, 1000, 10001):
        for world in (1, 2, 3, 8):
            if world > N:
                continue
            blocks = [shard_rows(N, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, N, n, out_dir):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1407_7220_b200.dist import broadcast_nccl_id

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    uid = broadcast_nccl_id()
    X, y = O.gen_instance("maxaffine-uniform", N, n, 0.1, 5, 6)
    p = O.prepare(X, y)
    r = O.papg(X, p.ys, max_iters=7, gap_norm_tol=-1, infeas_norm_tol=-1)
    theta = r.theta
    r0, r1 = shard_rows(N, world, rank)
    mine = theta[r0 * (N - 1): r1 * (N - 1)]
    pay = torch.from_numpy(local_payload(mine, theta[N * (N - 1):], X, r0, r1))
    dist.all_reduce(pay)  # the NCCL payload, summed over ranks
    total = pay.numpy()
    # primal closed form from the reduced payload (alcc.cpp:233-235)
    rowsum, colagg = total[:N], total[N:].reshape(N, n + 1)
    qy = theta[N * (N - 1):] + rowsum - colagg[:, 0]
    y_rank = p.ys + qy
    xi_rank = (colagg[:, :1] * X - colagg[:, 1:]) / 1e-3
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), uid=np.frombuffer(uid, np.uint8), y=y_rank,
             xi=xi_rank, ref_y=r.y, ref_xi=r.xi)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_exchange_matches_unsharded(tmp_path, world):
    import torch.multiprocessing as mp

    N, n = 37, 4
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, N, n, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    assert all(np.array_equal(res[0]["uid"], r["uid"]) for r in res)  # same NCCL id
    for r in res:
        assert np.allclose(r["y"], r["ref_y"], rtol=1e-12, atol=1e-12)
        assert np.allclose(r["xi"], r["ref_xi"], rtol=1e-9, atol=1e-9)
    assert np.array_equal(res[0]["y"], res[1]["y"])  # replicated primal is bitwise equal


def test_canonical_bounds_contain_every_balanced_shard():
    for N in (8, 37, 1000, 10001):
        b = canonical_bounds(N, 8)
        assert b[0] == 0 and b[-1] == N and all(x < y for x, y in zip(b, b[1:]))
        for world in (1, 2, 4, 8):
            for r in range(world):
                r0, r1 = shard_rows(N, world, r)
                assert r0 in b and r1 in b
    with pytest.raises(ValueError):
        canonical_bounds(4, 5)


def _block_payloads(theta, X, D, lo, hi):
    """Payloads of canonical blocks lo..hi-1 (host restatement of what each block's sweep +
    reduce produces)."""
    N = X.shape[0]
    b = canonical_bounds(N, D)
    return np.stack([local_payload(theta[b[j] * (N - 1): b[j + 1] * (N - 1)], theta[N * (N - 1):],
                                   X, b[j], b[j + 1]) for j in range(lo, hi)])


def _canon_worker(rank, world, port, N, n, D, out_dir):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, y = O.gen_instance("maxaffine-uniform", N, n, 0.1, 5, 6)
    p = O.prepare(X, y)
    theta = O.papg(X, p.ys, max_iters=7, gap_norm_tol=-1, infeas_norm_tol=-1).theta
    per = D // world
    mine = torch.from_numpy(_block_payloads(theta, X, D, rank * per, (rank + 1) * per))
    every = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(every, mine)  # the canonical-block exchange: gather, do not reduce
    blocks = torch.cat(every).numpy()
    total = blocks[0].copy()
    for j in range(1, D):  # block order, on every rank
        total += blocks[j]
    np.save(os.path.join(out_dir, f"c{rank}.npy"), total)
    dist.destroy_process_group()


def test_gloo_canonical_block_exchange_is_world_size_invariant(tmp_path):
    """The allgather + block-order sum gives bitwise the payload of a single process
    (SPEC.md:382, 619), unlike a sum over per-rank partial sums."""
    import torch.multiprocessing as mp

    from oracle import oracle as O

    N, n, D, world = 41, 3, 4, 2
    port = _free_port()
    mp.start_processes(_canon_worker, args=(world, port, N, n, D, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    got = [np.load(tmp_path / f"c{r}.npy") for r in range(world)]
    X, y = O.gen_instance("maxaffine-uniform", N, n, 0.1, 5, 6)
    p = O.prepare(X, y)
    theta = O.papg(X, p.ys, max_iters=7, gap_norm_tol=-1, infeas_norm_tol=-1).theta
    blocks = _block_payloads(theta, X, D, 0, D)
    single = blocks[0].copy()
    for j in range(1, D):
        single += blocks[j]
    assert np.array_equal(got[0], single) and np.array_equal(got[1], single)
    whole = local_payload(theta[: N * (N - 1)], theta[N * (N - 1):], X, 0, N)
    assert np.allclose(single, whole, rtol=1e-12, atol=1e-13)
