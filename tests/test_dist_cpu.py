"""Multi-process (gloo, world_size 2) CPU tests of the row-sharded path:
shard layout, NCCL-id broadcast over torch.distributed, and the exchange
arithmetic (per-rank payloads summed over ranks == full aggregates, primal
closed form identical on every rank). The GPU kernels themselves are covered
by the 1-GPU sharded emulation in test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest

from paper_1407_7220_b200.dist import local_payload, shard_rows


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
