"""End-to-end run() on the GPU solvers (runner.cpp:226-366, SURVEY.md 8f row
f4): every solver, gamma continuation, the report / history files, and the
final metrics re-derived with the oracle from the reported solution."""
import json

import numpy as np
import pytest

from paper_1407_7220_b200 import papg as P
from paper_1407_7220_b200 import runner as R

pytestmark = pytest.mark.gpu


def check_final(O, data, rep, gamma):
    y, xi = rep.solution.y, rep.solution.xi
    assert rep.final.objective == pytest.approx(0.5 * np.sum((y - data.ys) ** 2), rel=1e-12)
    raw, norm = O.infeasibility(data.xs, y, xi)
    assert rep.final.infeas_raw == pytest.approx(raw, rel=1e-9, abs=1e-14)
    assert rep.final.infeas_norm == pytest.approx(norm, rel=1e-9, abs=1e-16)
    N = len(y)
    assert rep.final.gap_norm == pytest.approx(rep.final.gap_raw / (N * (N - 1)), rel=1e-15)
    sub, inf = O.certificate(gamma, rep.certificates.delta_estimate,
                             rep.certificates.B_xi_estimate, rep.certificates.sigma_C)
    assert rep.certificates.subopt_bound == pytest.approx(sub, rel=1e-15)
    assert rep.certificates.infeas_bound == pytest.approx(inf, rel=1e-15)
    assert rep.exit_code == {"thresholds": 0, "error": 1}.get(rep.final.reason, 2)


def test_run_papg_singleton_matches_oracle(oracle, tmp_path):
    """solver papg-alcc with K = N: the closed-form dual path end to end"""
    spec = P.GeneratorSpec("sqnorm-uniform", 2, 60, 0.1, 4)
    out, hist = tmp_path / "r.json", tmp_path / "h.csv"
    cfg = R.RunConfig(generate=spec, K=60, out_json=str(out), out_history_csv=str(hist))
    rep = R.run(cfg)
    data = P.gen_instance(spec)
    check_final(oracle, data, rep, 1e-3)
    # the same solve on the oracle (shifted frame), then unshifted
    pr = oracle.prepare(data.xs, data.ys, 1e-3)
    o = oracle.papg(data.xs, pr.ys)
    assert len(rep.history) == o.iters
    assert rep.final.reason == {"thresholds": "thresholds", "iter_budget": "iter-budget"}[o.reason]
    assert np.linalg.norm(rep.solution.y - (o.y - pr.shift)) <= 1e-8 * np.linalg.norm(o.y)
    back = R.report_from_json(out.read_text())
    assert np.array_equal(back.solution.y, rep.solution.y)
    assert back.final == rep.final
    assert hist.read_text().count("\n") == len(rep.history) + 1


def test_run_dga_and_continuation(oracle):
    spec = P.GeneratorSpec("sqnorm-uniform", 2, 50, 0.1, 5)
    rep = R.run(R.RunConfig(generate=spec, K=50, solver="dga", max_iters=40, continuation=True))
    data = P.gen_instance(spec)
    check_final(oracle, data, rep, 1e-4)
    assert rep.final.reason in ("thresholds", "iter-budget")


def test_run_alcc_standalone(oracle):
    spec = P.GeneratorSpec("sqnorm-uniform", 2, 40, 0.1, 6)
    rep = R.run(R.RunConfig(generate=spec, K=40, solver="alcc", max_iters=6))
    data = P.gen_instance(spec)
    check_final(oracle, data, rep, 1e-3)
    # sigma_C of the run's partition (runner.cpp:292)
    assert rep.certificates.sigma_C == pytest.approx(oracle.sigma_C(data.xs)[0], rel=1e-10)


def test_run_general_k_from_csv(oracle, tmp_path):
    """the reference default solver (papg-alcc, K = 2) from a dataset file"""
    spec = P.GeneratorSpec("sqnorm-uniform", 2, 40, 0.1, 7)
    data = P.gen_instance(spec)
    csv = tmp_path / "d.csv"
    R.save_csv(data, str(csv))
    cfg = R.RunConfig(input_csv=str(csv), K=2, max_iters=3,
                      inner=P.AlccConfig(max_outer=6, mapg_cap=1000))
    rep = R.run(cfg)
    check_final(oracle, data, rep, 1e-3)
    N = 40
    assert rep.certificates.sigma_C == pytest.approx(oracle.sigma_C_k(data.xs, 2)[0], rel=1e-10)
    assert len(rep.solution.y) == N


def test_bench_csv():
    batch = R.batch_from_json(json.dumps([
        {"generate": {"kind": "sqnorm-uniform", "n": 2, "N": 40, "noise": 0.1}, "K": 40,
         "seed": 3},
        {"generate": {"kind": "sqnorm-uniform", "n": 2, "N": 40, "noise": 0.1}, "K": 40,
         "max_iters": 1, "gap_tol": 1e-12, "seed": 4},
        {"generate": {"kind": "sqnorm-uniform", "n": 2, "N": 40}, "K": 3},
    ]))
    lines = R.bench(batch).splitlines()
    assert lines[0] == "N,solver,seed,cpu_min,wall_min,objective,gap_norm,infeas_norm,reason"
    assert lines[1].startswith("40,papg-alcc,3,") and lines[1].endswith(",thresholds")
    assert lines[2] == "40,papg-alcc,4,N/A,N/A,N/A,N/A,N/A,iter-budget"
    assert "error: partition: N = 40 not divisible by K = 3" in lines[3]
