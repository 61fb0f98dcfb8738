"""End-to-end run driver and its wire/disk formats,
mirroring the reference's runner (proj/core/src/runner.cpp) and dataset I/O
(proj/core/src/dataset.cpp:44-117) on top of the B200 solvers:

  RunConfig / config_to_json / config_from_json   runner.cpp:64-119, :139-145
  RunReport / report_to_json / report_from_json   runner.cpp:147-202
  history_to_csv                                  runner.cpp:204-216
  run(cfg)                                        runner.cpp:226-366
  batch_from_json / bench                         runner.cpp:368-407
  load_csv / save_csv / validate_dataset          dataset.cpp:14-117
  format_double ("%.17g")                         runner.cpp:21-25

The solvers are the GPU ones: "papg-alcc" (singleton blocks when K == N, the
P-APG(ALCC) block path otherwise), "dga" and the standalone "alcc". JSON keys
are written sorted with two-space indentation, as nlohmann::json::dump(2)
does; doubles round-trip exactly.
"""
from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

import numpy as np

from . import papg as P

SOLVERS = ("papg-alcc", "alcc", "dga")
REASON_NAMES = {P.TermReason.thresholds: "thresholds", P.TermReason.iter_budget: "iter-budget",
                P.TermReason.time_budget: "time-budget", P.TermReason.error: "error"}  # metrics.cpp:58-66


def format_double(v: float) -> str:
    return "%.17g" % v


# ---- datasets (dataset.cpp) ----------------------------------------------------
def validate_dataset(data: P.Dataset) -> None:
    """dataset.cpp:14-42: shapes, finiteness, N >= n+1, no duplicate x rows."""
    X, y = np.asarray(data.xs), np.asarray(data.ys)
    if X.ndim != 2 or y.shape != (X.shape[0],):
        raise ValueError("dataset: xs/ys row count mismatch")
    N, n = X.shape
    if n < 1:
        raise ValueError("dataset: need at least one feature")
    if N < n + 1:
        raise ValueError("dataset: need N >= n+1 observations")
    if not (np.isfinite(X).all() and np.isfinite(y).all()):
        raise ValueError("dataset: non-finite entry")
    order = np.lexsort(X.T[::-1])
    Xs = X[order]
    dup = np.nonzero((Xs[1:] == Xs[:-1]).all(axis=1))[0]
    if dup.size:
        a, b = sorted((int(order[dup[0]]), int(order[dup[0] + 1])))
        raise ValueError(f"dataset: duplicate x rows (observations {a} and {b})")


def load_csv(path: str) -> P.Dataset:
    """dataset.cpp:44-100: header x1,...,xn,y then N rows of n+1 numbers."""
    try:
        f = open(path)
    except OSError:
        raise ValueError(f"cannot open dataset: {path}") from None
    with f:
        header = f.readline()
        if not header:
            raise ValueError(f"empty dataset file: {path}")
        names = header.rstrip("\n").split(",")
        n = len(names) - 1
        if len(names) < 2 or names[-1] != "y" or names[:-1] != [f"x{j + 1}" for j in range(n)]:
            raise ValueError("dataset header must be x1,...,xn,y")
        rows = []
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            toks = line.split(",")
            vals = []
            for t in toks:
                try:
                    vals.append(float(t))
                except ValueError:
                    raise ValueError(f"bad numeric field '{t}' in {path}") from None
            if len(vals) != n + 1:
                raise ValueError(f"row with {len(vals)} fields, expected {n + 1}")
            rows.append(vals)
    A = np.array(rows, np.float64).reshape(-1, n + 1)
    data = P.Dataset(np.ascontiguousarray(A[:, :n]), np.ascontiguousarray(A[:, n]))
    validate_dataset(data)
    return data


def save_csv(data: P.Dataset, path: str) -> None:
    """dataset.cpp:102-117 (%.17g: exact round trip)."""
    X, y = np.asarray(data.xs), np.asarray(data.ys)
    try:
        f = open(path, "w")
    except OSError:
        raise ValueError(f"cannot write dataset: {path}") from None
    with f:
        f.write(",".join(f"x{j + 1}" for j in range(X.shape[1])) + ",y\n")
        for i in range(X.shape[0]):
            f.write(",".join(format_double(v) for v in X[i]) + "," + format_double(y[i]) + "\n")


# ---- configuration and report (runner.hpp:12-56) ----------------------------------
@dataclass
class RunConfig:
    input_csv: str = ""
    generate: P.GeneratorSpec | None = None
    gamma: float = 1e-3
    K: int = 2
    solver: str = "papg-alcc"
    gap_tol: float = 1e-6
    infeas_tol: float = 1e-1
    max_iters: int = 100000
    max_seconds: float = 7200.0
    workers: int = 0
    seed: int = 1
    continuation: bool = False
    repair: bool = False
    out_json: str = ""
    out_history_csv: str = ""
    # device knob: inner ALCC settings of the block path (PapgConfig::inner)
    inner: P.AlccConfig | None = None


@dataclass
class Final:
    objective: float = 0.0
    reg_objective: float = 0.0
    gap_raw: float = 0.0
    gap_norm: float = 0.0
    infeas_raw: float = 0.0
    infeas_norm: float = 0.0
    cpu_min: float = 0.0
    wall_min: float = 0.0
    reason: str = ""


@dataclass
class Certificates:
    delta_estimate: float = 0.0
    subopt_bound: float = 0.0
    infeas_bound: float = 0.0
    sigma_C: float = 0.0
    B_xi_estimate: float = 0.0
    estimated: bool = True


@dataclass
class RunReport:
    config: RunConfig = field(default_factory=RunConfig)
    history: list = field(default_factory=list)
    final: Final = field(default_factory=Final)
    certificates: Certificates = field(default_factory=Certificates)
    solution: P.PrimalPoint | None = None
    shift: float = 0.0
    environment: str = ""
    exit_code: int = 0


def _dump(obj) -> str:
    return json.dumps(obj, indent=2, sort_keys=True)


def config_to_obj(cfg: RunConfig) -> dict:
    """runner.cpp:64-91"""
    j = {"input": cfg.input_csv, "gamma": cfg.gamma, "K": cfg.K, "solver": cfg.solver,
         "gap_tol": cfg.gap_tol, "infeas_tol": cfg.infeas_tol, "max_iters": cfg.max_iters,
         "max_seconds": cfg.max_seconds, "workers": cfg.workers, "seed": cfg.seed,
         "continuation": cfg.continuation, "repair": cfg.repair, "out": cfg.out_json,
         "history_out": cfg.out_history_csv}
    if cfg.generate is not None:
        g = cfg.generate
        j["generate"] = {"kind": g.kind, "n": g.n, "N": g.N, "noise": g.noise, "seed": g.seed}
    return j


def config_from_obj(j: dict) -> RunConfig:
    """runner.cpp:93-119 (defaults as the reference)"""
    cfg = RunConfig()
    cfg.input_csv = j.get("input", "")
    g = j.get("generate")
    if g is not None:
        if g["kind"] not in P.GEN_KINDS:
            raise ValueError(f"unknown generator kind: {g['kind']}")
        cfg.generate = P.GeneratorSpec(g["kind"], int(g["n"]), int(g["N"]),
                                       float(g.get("noise", 1.0)), int(g.get("seed", 0)))
    cfg.gamma = float(j.get("gamma", 1e-3))
    cfg.K = int(j.get("K", 2))
    cfg.solver = j.get("solver", "papg-alcc")
    cfg.gap_tol = float(j.get("gap_tol", 1e-6))
    cfg.infeas_tol = float(j.get("infeas_tol", 1e-1))
    cfg.max_iters = int(j.get("max_iters", 100000))
    cfg.max_seconds = float(j.get("max_seconds", 7200.0))
    cfg.workers = int(j.get("workers", 0))
    cfg.seed = int(j.get("seed", 1))
    cfg.continuation = bool(j.get("continuation", False))
    cfg.repair = bool(j.get("repair", False))
    cfg.out_json = j.get("out", "")
    cfg.out_history_csv = j.get("history_out", "")
    return cfg


def config_to_json(cfg: RunConfig) -> str:
    return _dump(config_to_obj(cfg))


def config_from_json(text: str) -> RunConfig:
    return config_from_obj(json.loads(text))


_SNAP = ("iter", "objective", "reg_objective", "infeas_raw", "infeas_norm", "gap_raw",
         "gap_norm", "wall_time_s")


def report_to_json(r: RunReport) -> str:
    """runner.cpp:147-175"""
    f, c = r.final, r.certificates
    j = {
        "config": config_to_obj(r.config),
        "history": [{k: (int(getattr(s, k)) if k == "iter" else float(getattr(s, k)))
                     for k in _SNAP} for s in r.history],
        "final": {"objective": f.objective, "reg_objective": f.reg_objective,
                  "gap_raw": f.gap_raw, "gap_norm": f.gap_norm, "infeas_raw": f.infeas_raw,
                  "infeas_norm": f.infeas_norm, "cpu_min": f.cpu_min, "wall_min": f.wall_min,
                  "reason": f.reason},
        "certificates": {"delta_estimate": c.delta_estimate, "subopt_bound": c.subopt_bound,
                         "infeas_bound": c.infeas_bound, "sigma_C": c.sigma_C,
                         "B_xi_estimate": c.B_xi_estimate, "estimated": c.estimated},
        "solution": {"y": [float(v) for v in r.solution.y],
                     "xi": [float(v) for v in np.asarray(r.solution.xi).reshape(-1)],
                     "shift": r.shift},
        "environment": r.environment,
        "exit_code": r.exit_code,
    }
    return _dump(j)


def report_from_json(text: str) -> RunReport:
    """runner.cpp:177-202"""
    j = json.loads(text)
    r = RunReport()
    r.config = config_from_obj(j["config"])
    r.history = [P.MetricsSnapshot(int(s["iter"]), *(float(s[k]) for k in _SNAP[1:]))
                 for s in j["history"]]
    f = j["final"]
    r.final = Final(*(float(f[k]) for k in ("objective", "reg_objective", "gap_raw", "gap_norm",
                                            "infeas_raw", "infeas_norm", "cpu_min",
                                            "wall_min")), str(f["reason"]))
    c = j["certificates"]
    r.certificates = Certificates(float(c["delta_estimate"]), float(c["subopt_bound"]),
                                  float(c["infeas_bound"]), float(c["sigma_C"]),
                                  float(c["B_xi_estimate"]), bool(c["estimated"]))
    s = j["solution"]
    r.solution = P.PrimalPoint(np.array(s["y"], np.float64), np.array(s["xi"], np.float64))
    r.shift = float(s["shift"])
    r.environment = str(j["environment"])
    r.exit_code = int(j["exit_code"])
    return r


def history_to_csv(history) -> str:
    """runner.cpp:204-216"""
    lines = ["iter,objective,reg_objective,infeas_raw,infeas_norm,gap_raw,gap_norm,wall_time_s"]
    for s in history:
        lines.append(",".join([str(int(s.iter))] +
                              [format_double(float(getattr(s, k))) for k in _SNAP[1:]]))
    return "\n".join(lines) + "\n"


# ---- run (runner.cpp:226-366) ------------------------------------------------------
def _environment(device: int) -> str:
    """runner.cpp:29-44 (our build's facts instead of compiler / Eigen versions)"""
    return (f"device=cuda:{device} (sm_100a); solver=libcvxreg_b200 fp64 pair sweeps; "
            f"rng=xoshiro256++ (per-array streams, Box-Muller cosine branch)")


def run(cfg: RunConfig, device: int = 0) -> RunReport:
    if cfg.solver not in SOLVERS:
        raise ValueError(f"unknown solver: {cfg.solver}")
    if cfg.gamma <= 0:
        raise ValueError("gamma must be > 0")
    if cfg.max_iters <= 0 or cfg.max_seconds <= 0:
        raise ValueError("budgets must be positive")
    if cfg.input_csv:
        data = load_csv(cfg.input_csv)
    elif cfg.generate is not None:
        spec = cfg.generate
        if spec.seed == 0:
            spec = P.GeneratorSpec(spec.kind, spec.n, spec.N, spec.noise, cfg.seed, spec.pieces)
        data = P.gen_instance(spec)
    else:
        raise ValueError("no input: set a CSV path or a generator")
    N, n = data.xs.shape
    if cfg.K < 1 or N % cfg.K != 0:  # make_partition (dataset.cpp:119-130)
        raise ValueError(f"partition: N = {N} not divisible by K = {cfg.K}")
    # K == N (singleton blocks) is the closed-form north-star path of this
    # build; the reference's make_partition rejects it (dataset.cpp:127-128)
    if cfg.K != N and N // cfg.K < n + 1:
        raise ValueError("partition: block size must be >= n+1")
    K = cfg.K if cfg.K < N else 0

    report = RunReport(config=cfg, environment=_environment(device))
    wall0 = time.perf_counter()
    cpu0 = time.process_time()
    gammas = [cfg.gamma] + ([cfg.gamma / 10.0] if cfg.continuation else [])
    reason = P.TermReason.error
    solution = None
    shift = sigma_C = delta = B_xi = gap_raw = 0.0
    theta_warm = None
    primal_warm = None
    for gamma in gammas:
        prep = P.prepare_problem(data, gamma)
        B_xi = prep.bounds.Bbar_xi
        if cfg.solver == "alcc":
            acfg = P.AlccConfig(max_outer=cfg.max_iters, max_seconds=cfg.max_seconds,
                                infeas_norm_tol=cfg.infeas_tol, gap_norm_tol=cfg.gap_tol)
            warm = primal_warm or prep.feasible
            with P.DualSolver(prep.data.xs, prep.data.ys, gamma, device) as s:
                res, y, xi, hist, mi = s.alcc(acfg, prep.bounds, warm)
                if K:
                    s.set_partition(K, prep.feasible, cfg.inner)
                sigma_C = s.sigma_C()[0]  # runner.cpp:292 (op_C of the run's partition)
            report.history = [P.MetricsSnapshot(int(h[0]), *map(float, h[1:])) for h in hist]
            reason = P.TermReason(res.reason)
            solution = P.PrimalPoint(y, xi)
            shift = prep.shift
            delta = max(res.certified_gap, 0.0)
            gap_raw = res.gap_raw  # multiplier . rows(solution), runner.cpp:293-295
            primal_warm = solution
        else:
            pcfg = P.PapgConfig(gamma=gamma, gap_norm_tol=cfg.gap_tol,
                                infeas_norm_tol=cfg.infeas_tol, max_iters=cfg.max_iters,
                                max_seconds=cfg.max_seconds, workers=cfg.workers, K=K,
                                inner=cfg.inner, device=device)
            with P.DualSolver(prep.data.xs, prep.data.ys, gamma, device) as s:
                if K:
                    s.set_partition(K, prep.feasible, cfg.inner)
                s.begin(pcfg, cfg.solver == "papg-alcc", theta_warm)
                stopped = False
                while not stopped:
                    _, stopped = s.iterate(1 << 40)
                res, y, xi, hist = s.finish()
                theta_warm = s.theta()
                gap_raw = s.duality_gap(y, xi)[0]  # theta . C eta (runner.cpp:317-321)
            report.history = [P.MetricsSnapshot(int(h[0]), *map(float, h[1:])) for h in hist]
            reason = P.TermReason(res.reason)
            solution = P.PrimalPoint(y, xi)
            shift = prep.shift
            delta = res.delta_estimate
            sigma_C = res.sigma_C
    # final metrics against the original observations (runner.cpp:327-343)
    y = np.asarray(solution.y) - shift
    xi = np.asarray(solution.xi).reshape(-1)
    report.solution = P.PrimalPoint(y, xi)
    report.shift = shift
    with P.DualSolver(data.xs, data.ys, gammas[-1], device) as s:
        infeas_raw, infeas_norm = s.infeasibility(y, xi)
    rows = float(N) * float(N - 1)
    f = report.final
    f.objective = 0.5 * float(np.sum((y - data.ys) ** 2))
    f.reg_objective = f.objective + 0.5 * gammas[-1] * float(np.dot(xi, xi))
    f.infeas_raw, f.infeas_norm = infeas_raw, infeas_norm
    f.gap_raw = gap_raw
    f.gap_norm = gap_raw / rows
    f.reason = REASON_NAMES[reason]
    f.wall_min = (time.perf_counter() - wall0) / 60.0
    f.cpu_min = (time.process_time() - cpu0) / 60.0
    c = report.certificates
    c.delta_estimate, c.sigma_C, c.B_xi_estimate = delta, sigma_C, B_xi
    c.subopt_bound, c.infeas_bound = P.certificate_for_iterate(gammas[-1], delta, B_xi, sigma_C)
    report.exit_code = {P.TermReason.thresholds: 0, P.TermReason.error: 1}.get(reason, 2)
    if cfg.out_json:
        try:
            with open(cfg.out_json, "w") as out:
                out.write(report_to_json(report) + "\n")
        except OSError:
            raise RuntimeError(f"cannot write report: {cfg.out_json}") from None
    if cfg.out_history_csv:
        try:
            with open(cfg.out_history_csv, "w") as out:
                out.write(history_to_csv(report.history))
        except OSError:
            raise RuntimeError(f"cannot write history: {cfg.out_history_csv}") from None
    return report


def batch_from_json(text: str) -> list:
    j = json.loads(text)
    if not isinstance(j, list):
        raise ValueError("batch file must be a JSON array")
    return [config_from_obj(item) for item in j]


def bench(batch, device: int = 0) -> str:
    """runner.cpp:376-405: one CSV row per run, N/A in the value columns on budget stops."""
    lines = ["N,solver,seed,cpu_min,wall_min,objective,gap_norm,infeas_norm,reason"]
    for cfg in batch:
        N = cfg.generate.N if cfg.generate is not None else 0
        try:
            r = run(cfg, device)
            N = len(r.solution.y)
            head = f"{N},{cfg.solver},{cfg.seed},"
            if r.exit_code == 0:
                vals = ",".join(format_double(v) for v in (r.final.cpu_min, r.final.wall_min,
                                                           r.final.objective, r.final.gap_norm,
                                                           r.final.infeas_norm))
            else:
                vals = "N/A,N/A,N/A,N/A,N/A"
            lines.append(head + vals + "," + r.final.reason)
        except Exception as err:  # noqa: BLE001 - the reference reports and continues
            lines.append(f"{N},{cfg.solver},{cfg.seed},N/A,N/A,N/A,N/A,N/A,error: {err}")
    return "\n".join(lines) + "\n"
