"""Wire/disk formats of the run driver: dataset CSV
(dataset.cpp:44-117), config / report JSON (runner.cpp:64-202) and history
CSV (runner.cpp:204-216). CPU only (no solver calls)."""
import json
import re

import numpy as np
import pytest

from paper_1407_7220_b200 import papg as P
from paper_1407_7220_b200 import runner as R


def test_dataset_csv_round_trip_is_exact(tmp_path):
    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (25, 3)) * np.array([1e-300, 1.0, 1e300])
    y = rng.standard_normal(25) / 3.0
    p = tmp_path / "d.csv"
    R.save_csv(P.Dataset(X, y), str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "x1,x2,x3,y"
    assert lines[1].split(",")[0] == "%.17g" % X[0, 0]
    d = R.load_csv(str(p))
    assert np.array_equal(d.xs, X) and np.array_equal(d.ys, y)


@pytest.mark.parametrize("text,msg", [
    ("", "empty dataset file"),
    ("a,b\n1,2\n", "header must be x1,...,xn,y"),
    ("x1,x3,y\n1,2,3\n", "header must be x1,...,xn,y"),
    ("x1,y\n1,abc\n2,3\n", "bad numeric field 'abc'"),
    ("x1,y\n1,2,3\n2,3\n", "row with 3 fields, expected 2"),
    ("x1,y\n1,2\n", "need N >= n+1"),
    ("x1,y\n1,2\n1,3\n", "duplicate x rows (observations 0 and 1)"),
    ("x1,y\n1,nan\n2,3\n", "non-finite entry"),
])
def test_dataset_csv_errors(tmp_path, text, msg):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(ValueError, match=re.escape(msg)):
        R.load_csv(str(p))


def test_dataset_csv_missing_file(tmp_path):
    with pytest.raises(ValueError, match="cannot open dataset"):
        R.load_csv(str(tmp_path / "none.csv"))


def test_config_json_defaults_and_round_trip():
    cfg = R.config_from_json("{}")
    assert (cfg.gamma, cfg.K, cfg.solver, cfg.gap_tol, cfg.infeas_tol, cfg.max_iters,
            cfg.max_seconds, cfg.seed) == (1e-3, 2, "papg-alcc", 1e-6, 1e-1, 100000, 7200.0, 1)
    cfg = R.RunConfig(generate=P.GeneratorSpec("quadratic", 3, 60, 0.5, 9), K=3, solver="dga",
                      gap_tol=1e-5, continuation=True, out_json="r.json")
    text = R.config_to_json(cfg)
    j = json.loads(text)
    assert list(j) == sorted(j)  # keys sorted like nlohmann::json
    assert j["generate"] == {"kind": "quadratic", "n": 3, "N": 60, "noise": 0.5, "seed": 9}
    back = R.config_from_json(text)
    assert back.generate.kind == "quadratic" and back.generate.N == 60
    assert (back.K, back.solver, back.gap_tol, back.continuation, back.out_json) == \
        (3, "dga", 1e-5, True, "r.json")
    with pytest.raises(ValueError, match="unknown generator kind"):
        R.config_from_json('{"generate": {"kind": "cubic", "n": 1, "N": 5}}')


def test_report_json_round_trip_and_history_csv():
    hist = [P.MetricsSnapshot(1, 0.5, 0.6, 1e-3, 1e-5, -2e-4, -3e-8, 0.01),
            P.MetricsSnapshot(2, 0.25, 0.26, 1e-4, 1e-6, 1.0 / 3.0, 2e-9, 0.02)]
    r = R.RunReport(config=R.RunConfig(), history=hist,
                    final=R.Final(1.0, 1.1, 2e-3, 1e-9, 0.5, 0.01, 0.1, 0.2, "thresholds"),
                    certificates=R.Certificates(1e-3, 2e-3, 3e-3, 4.5, 6.0, True),
                    solution=P.PrimalPoint(np.array([1.0, 2.0 / 3.0]), np.array([0.1, -0.2])),
                    shift=0.7, environment="test", exit_code=0)
    back = R.report_from_json(R.report_to_json(r))
    assert back.history == hist
    assert back.final == r.final and back.certificates == r.certificates
    assert np.array_equal(back.solution.y, r.solution.y) and back.shift == 0.7
    csv = R.history_to_csv(hist).splitlines()
    assert csv[0] == "iter,objective,reg_objective,infeas_raw,infeas_norm,gap_raw,gap_norm,wall_time_s"
    assert csv[2].split(",")[5] == "%.17g" % (1.0 / 3.0)
    assert csv[1].startswith("1,0.5,")


def test_batch_and_run_validation():
    with pytest.raises(ValueError, match="JSON array"):
        R.batch_from_json("{}")
    assert len(R.batch_from_json('[{"solver": "dga"}, {}]')) == 2
    with pytest.raises(ValueError, match="unknown solver"):
        R.run(R.RunConfig(solver="sgd"))
    with pytest.raises(ValueError, match="gamma"):
        R.run(R.RunConfig(gamma=0.0))
    with pytest.raises(ValueError, match="no input"):
        R.run(R.RunConfig())
