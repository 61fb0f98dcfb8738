"""GPU-count-invariant determinism (cr_set_canonical_blocks).

SPEC.md:382, 619 ask for results that do not depend on the worker count, and the
reference gathers block results in block order (papg.cpp:122-129). With D
canonical row blocks every block is swept and reduced on its own and the block
payloads are summed in block order, so theta, y, xi and the history after k
iterations are BITWISE the same whether the D blocks live on 1, 2, 4 or 8
handles. One GPU is available: the shards are separate handles on the same
device and the allgather is done on the host (cr_exchange_get/put), exactly
the data ncclAllGather would leave in every rank's buffer.
"""
import numpy as np
import pytest

import paper_1407_7220_b200 as crb

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def instance(O, kind, N, n, noise, seed, pieces=0):
    X, y = O.gen_instance(kind, N, n, noise, seed, pieces)
    return X, O.prepare(X, y).ys


def run_shards(X, ys, cfg, p, D, iters):
    """p shard handles, D canonical blocks, host-emulated allgather per iteration."""
    N = X.shape[0]
    shards = [crb.DualSolver(X, ys, row_begin=N * r // p, row_end=N * (r + 1) // p)
              for r in range(p)]
    try:
        for d in shards:
            d.set_canonical_blocks(D)
            d.begin(cfg)
        plen = shards[0].exchange_len // D
        for _ in range(iters):
            for d in shards:
                d.iter_local()
            allp = np.zeros((D, plen))
            covered = np.zeros(D, bool)
            for d in shards:
                Dq, first, cnt = d.canonical_blocks()
                assert Dq == D and cnt == D // p
                allp[first:first + cnt] = d.exchange_get().reshape(D, plen)[first:first + cnt]
                covered[first:first + cnt] = True
            assert covered.all()
            for d in shards:
                d.exchange_put(allp)
            stops = [d.iter_finish() for d in shards]
            assert len(set(stops)) == 1
        th = [d.theta() for d in shards]
        theta = np.concatenate([t[:-N] for t in th] + [th[0][-N:]])
        fin = [d.finish() for d in shards]
        for f in fin[1:]:  # replicated primal and history: identical on every shard
            assert np.array_equal(f[1], fin[0][1]) and np.array_equal(f[2], fin[0][2])
            assert np.array_equal(f[3][:, :7], fin[0][3][:, :7])
        return dict(theta=theta, y=fin[0][1], xi=fin[0][2], hist=fin[0][3][:, :7], res=fin[0][0])
    finally:
        for d in shards:
            d.close()


@pytest.mark.parametrize("kind,N,n,pieces,iters", [
    ("maxaffine-uniform", 424, 10, 20, 25),   # N divisible by 8
    ("sqnorm-uniform", 603, 5, 0, 20),        # ragged blocks: floor(j N / 8)
    ("lse-uniform", 330, 20, 50, 12),
])
def test_iterates_do_not_depend_on_the_shard_count(oracle, kind, N, n, pieces, iters):
    X, ys = instance(oracle, kind, N, n, 0.1, 17 + n, pieces)
    s, _, _ = oracle.sigma_C(X)
    cfg = crb.PapgConfig(max_iters=iters, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    D = 8
    runs = {p: run_shards(X, ys, cfg, p, D, iters) for p in (1, 2, 4, 8)}
    base = runs[1]
    assert np.linalg.norm(base["theta"]) > 0
    for p in (2, 4, 8):
        for key in ("theta", "y", "xi", "hist"):
            assert np.array_equal(runs[p][key], base[key]), (p, key)
    o = oracle.papg(X, ys, max_iters=iters, sigma_C=s, gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
    assert rel(base["theta"], o.theta) <= 1e-12 and rel(base["y"], o.y) <= 1e-8


def test_public_solve_with_canonical_blocks_matches_the_sharded_runs(oracle):
    """papg_solve(cfg.canonical_blocks = D) on one handle (graph / direct launch loop) gives
    the bits of the emulated multi-handle runs; to tolerance against the default path."""
    X, y = oracle.gen_instance("maxaffine-uniform", 512, 10, 0.1, 5, 20)
    P = oracle.prepare(X, y)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=30, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    prep = crb.PreparedProblem(crb.Dataset(X, P.ys), P.shift, crb.PrimalPoint(P.feas_y, P.feas_xi),
                               crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma))
    r = crb.papg_solve(prep, crb.PapgConfig(canonical_blocks=8, **kw))
    e = run_shards(X, P.ys, crb.PapgConfig(**kw), 4, 8, 30)
    th = np.concatenate([r.dual.theta_cross, r.dual.theta_pos])
    assert np.array_equal(th, e["theta"]) and np.array_equal(r.point.y, e["y"])
    d = crb.papg_solve(prep, crb.PapgConfig(**kw))
    assert rel(th, np.concatenate([d.dual.theta_cross, d.dual.theta_pos])) <= 1e-12
    assert r.report.iters == d.report.iters == 30


def test_canonical_blocks_thresholds_and_warm_start(oracle):
    X, ys = instance(oracle, "sqnorm-uniform", 400, 5, 0.1, 9)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(sigma_C=s)  # default tolerances: stops on thresholds
    o = oracle.papg(X, ys, **kw)
    with crb.DualSolver(X, ys) as d:
        d.set_canonical_blocks(8)
        d.begin(crb.PapgConfig(**kw))
        stopped = False
        while not stopped:
            _, stopped = d.iterate(1 << 40)
        res, y, xi, hist = d.finish()
        th = d.theta()
        assert (res.iters, res.reason) == (o.iters, 0)
        assert rel(th, o.theta) <= 1e-12 and rel(y, o.y) <= 1e-8
        # warm start from a clipped multiple of the solution (papg.cpp:158-164)
        theta0 = o.theta * 3e4
        kw2 = dict(max_iters=15, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s, B_theta=20.0)
        d.begin(crb.PapgConfig(**kw2), True, theta0)
        d.iterate(100)
        res2, y2, _, _ = d.finish()
        o2 = oracle.papg(X, ys, theta0=theta0, **kw2)
        assert rel(d.theta(), o2.theta) <= 1e-12 and rel(y2, o2.y) <= 1e-8
        # switching the mode off restores the default path on the same handle
        d.set_canonical_blocks(0)
        d.begin(crb.PapgConfig(**kw2), True, theta0)
        d.iterate(100)
        assert rel(d.theta(), o2.theta) <= 1e-12


def test_canonical_blocks_errors(oracle):
    X, ys = instance(oracle, "sqnorm-uniform", 120, 3, 0.1, 3)
    with crb.DualSolver(X, ys, row_begin=0, row_end=50) as d:  # 50 is not a block boundary
        with pytest.raises(Exception, match="union of blocks"):
            d.set_canonical_blocks(8)
    with crb.DualSolver(X, ys) as d:
        with pytest.raises(Exception):
            d.set_canonical_blocks(121)  # more blocks than rows
        d.set_canonical_blocks(8)
        assert d.canonical_blocks() == (8, 0, 8)
        assert d.exchange_len == 8 * (120 * 5 + 5)
        # the mode is for singleton blocks: a K-block partition on top of it is refused at begin
        P = oracle.prepare(*oracle.gen_instance("sqnorm-uniform", 120, 3, 0.1, 3))
        d.set_partition(4, crb.PrimalPoint(P.feas_y, P.feas_xi))
        with pytest.raises(Exception, match="singleton"):
            d.begin(crb.PapgConfig(max_iters=2, sigma_C=10.0, K=4))
    with crb.DualSolver(X, ys) as d:
        P = oracle.prepare(*oracle.gen_instance("sqnorm-uniform", 120, 3, 0.1, 3))
        d.set_partition(4, crb.PrimalPoint(P.feas_y, P.feas_xi))
        with pytest.raises(Exception, match="singleton"):
            d.set_canonical_blocks(8)


def test_canonical_blocks_nccl_allgather_single_rank(oracle):
    """The NCCL path of the mode (in-place ncclAllGather of the block payloads, captured in the
    iteration graph or launched directly) on a one-rank communicator: the bits of the
    communicator-free run."""
    X, ys = instance(oracle, "maxaffine-uniform", 320, 7, 0.1, 31, 9)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=30, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    base = run_shards(X, ys, crb.PapgConfig(**kw), 1, 8, 30)
    for graph_iters in (6, -1):
        with crb.DualSolver(X, ys) as d:
            d.attach_nccl(crb.DualSolver.nccl_unique_id(), 0, 1)
            d.set_canonical_blocks(8)
            d.begin(crb.PapgConfig(graph_iters=graph_iters, **kw))
            done, stopped = d.iterate(1 << 30)
            assert done == 30 and stopped
            res, y, xi, hist = d.finish()
            assert np.array_equal(d.theta(), base["theta"]) and np.array_equal(y, base["y"])
