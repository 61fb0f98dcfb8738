"""Python mirror of the reference solver interface for the singleton-block
dual path (proj/core/include/cvxreg/papg.hpp, types.hpp, metrics.hpp,
preprocess.hpp, testgen.hpp), backed by libcvxreg_b200.so.

Names, argument meaning and error behaviour follow the reference:
  papg_solve(prep, cfg, theta0=None)            papg.hpp:75-76
  dual_gradient_ascent(prep, cfg, theta0=None)  papg.hpp:79-82
  certificate_for_iterate(...)                  papg.hpp:85-90
  prepare_problem(data, gamma)                  preprocess.hpp:42
  gen_instance(spec)                            testgen.hpp:27
  alcc_solve(prep, cfg, warm=None)              alcc.hpp:134-136 (standalone ALCC)
Shape / precondition errors raise ValueError (std::invalid_argument);
numerical failures raise RuntimeError (std::runtime_error), e.g.
"papg: non-finite dual gradient" (papg.cpp:184-185).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat

GEN_KINDS = {
    "quadratic": 0, "exponential": 1, "affine-noiseless": 2, "custom-1d": 3,
    "sqnorm-uniform": 10, "maxaffine-uniform": 11, "lse-uniform": 12,
}


class TermReason(enum.IntEnum):  # metrics.hpp:41
    thresholds = 0
    iter_budget = 1
    time_budget = 2
    error = 3


@dataclass
class Dataset:  # types.hpp:13-19 (xs row l = x_l)
    xs: np.ndarray
    ys: np.ndarray

    @property
    def N(self):
        return self.xs.shape[0]

    @property
    def n(self):
        return self.xs.shape[1]


@dataclass
class ProblemBounds:  # types.hpp:55-60
    B_theta: float
    Bbar_y: float
    Bbar_xi: float
    gamma: float


@dataclass
class PrimalPoint:  # types.hpp:43-46 (xi flat: xi_l = xi[l*n:(l+1)*n])
    y: np.ndarray
    xi: np.ndarray


@dataclass
class DualPoint:  # types.hpp:50-53
    theta_cross: np.ndarray
    theta_pos: np.ndarray


@dataclass
class PreparedProblem:  # preprocess.hpp:35-40
    data: Dataset
    shift: float
    feasible: PrimalPoint
    bounds: ProblemBounds


@dataclass
class GeneratorSpec:  # testgen.hpp:13-19 (+ pieces for the BASELINE kinds)
    kind: str = "quadratic"
    n: int = 1
    N: int = 0
    noise: float = 1.0
    seed: int = 1
    pieces: int = 0


@dataclass
class PapgConfig:  # papg.hpp:7-21 (+ the partition size K of make_partition)
    gamma: float = 1e-3
    B_theta: float = 0.0
    adaptive_B_theta: bool = True
    max_restarts: int = 6
    gap_norm_tol: float = 1e-6
    infeas_norm_tol: float = 1e-1
    max_iters: int = 100000
    max_seconds: float = 7200.0
    workers: int = 0
    inner_tol_floor: float = 1e-6
    final_resolve_tol: float = 1e-10
    record_history: bool = True
    inner: "AlccConfig | None" = None  # block ALCC settings (papg.hpp:19), K < N only
    K: int = 0                 # blocks (make_partition, dataset.cpp:119); 0 or N: singleton
    # device knobs (not in the reference)
    sigma_C: float = 0.0       # > 0: inject sigma_max(C)
    graph_iters: int = 0       # 0 auto, > 0 graph batch, < 0 direct launches
    device: int = 0
    canonical_blocks: int = 0  # D > 0: GPU-count-invariant sums over D row blocks

    def to_c(self, use_momentum: bool) -> nat.PapgConfigC:
        return nat.PapgConfigC(self.gamma, self.B_theta, int(self.adaptive_B_theta),
                               self.max_restarts, self.gap_norm_tol, self.infeas_norm_tol,
                               int(self.max_iters), self.max_seconds, self.inner_tol_floor,
                               self.final_resolve_tol, int(self.record_history),
                               int(use_momentum), self.sigma_C, self.graph_iters,
                               int(self.workers))


@dataclass
class MetricsSnapshot:  # metrics.hpp:13-22
    iter: int
    objective: float
    reg_objective: float
    infeas_raw: float
    infeas_norm: float
    gap_raw: float
    gap_norm: float
    wall_time_s: float


@dataclass
class SolveReport:  # metrics.hpp:45-54
    history: list = field(default_factory=list)
    reason: TermReason = TermReason.iter_budget
    iters: int = 0
    wall_seconds: float = 0.0
    cpu_seconds: float = 0.0
    restarts: int = 0
    saturated: bool = False
    note: str = ""
    history_array: np.ndarray | None = None
    history_truncated: bool = False  # more than CR_HISTORY_CAP iterations: first ones kept


@dataclass
class PapgResult:  # papg.hpp:60-69
    point: PrimalPoint
    dual: DualPoint | None
    report: SolveReport
    g_final: float
    delta_estimate: float
    sigma_C: float
    L_g: float
    B_theta: float
    sigma_iters: int = 0
    sigma_seconds: float = 0.0
    loop_seconds: float = 0.0


def _f64(a):
    return np.ascontiguousarray(a, np.float64).reshape(-1)


def _raise(status, handle=None, what=""):
    if status == 0:
        return
    L = nat.load()
    msg = L.cr_last_error(handle).decode() if handle else L.cr_status_string(status).decode()
    if status == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def gen_instance(spec: GeneratorSpec) -> Dataset:
    """testgen.cpp:36-87 (+ BASELINE kinds sqnorm-/maxaffine-/lse-uniform)."""
    if spec.kind not in GEN_KINDS:
        raise ValueError(f"unknown generator kind: {spec.kind}")
    X = np.empty((spec.N, spec.n), np.float64)
    y = np.empty(spec.N, np.float64)
    st = nat.load().cr_gen_instance(GEN_KINDS[spec.kind], spec.N, spec.n, spec.noise, spec.seed,
                                    spec.pieces, nat.ptr(X), nat.ptr(y))
    if st != 0:
        raise ValueError("generator: invalid spec or duplicate rows")
    return Dataset(X, y)


def prepare_problem(data: Dataset, gamma: float = 1e-3) -> PreparedProblem:
    """preprocess.cpp:50-65: affine feasible point, bounds, shifted ys."""
    X = np.ascontiguousarray(data.xs, np.float64)
    y = np.ascontiguousarray(data.ys, np.float64)
    N, n = X.shape
    ys = np.empty(N)
    shift = np.zeros(1)
    fy = np.empty(N)
    fxi = np.empty(N * n)
    b4 = np.empty(4)
    st = nat.load().cr_prepare_problem(nat.ptr(X), nat.ptr(y), N, n, gamma, nat.ptr(ys),
                                       nat.ptr(shift), nat.ptr(fy), nat.ptr(fxi), nat.ptr(b4))
    if st != 0:
        raise ValueError("prepare_problem: invalid dataset or gamma")
    return PreparedProblem(Dataset(X, ys), float(shift[0]), PrimalPoint(fy, fxi),
                           ProblemBounds(*map(float, b4)))


def momentum_next(t: float) -> float:  # engines.hpp:11-13
    return nat.load().cr_momentum_next(t)


def certificate_for_iterate(gamma, delta, B_xi_estimate, sigma_max_C):  # papg.cpp:298-303
    out = np.empty(2)
    nat.load().cr_certificate(gamma, delta, B_xi_estimate, sigma_max_C, nat.ptr(out))
    return float(out[0]), float(out[1])


@dataclass
class AlccConfig:  # alcc.hpp:71-83
    mu1: float = 1.0
    tau1_scale: float = 1e-2
    alpha1_scale: float = 1e-3
    c: float = 5.0
    kappa: float = 0.5
    max_outer: int = 30
    mapg_cap: int = 200000
    infeas_norm_tol: float = 1e-1
    gap_norm_tol: float = 1e-6
    max_seconds: float = float("inf")
    record_history: bool = True
    # device knobs: inject spectral norms instead of estimating them
    sigma_A1: float = 0.0
    sigma_A2: float = 0.0

    def to_c(self, bounds: "ProblemBounds") -> nat.AlccConfigC:
        return nat.AlccConfigC(self.mu1, self.tau1_scale, self.alpha1_scale, self.c, self.kappa,
                               self.max_outer, self.mapg_cap, self.infeas_norm_tol,
                               self.gap_norm_tol, self.max_seconds, int(self.record_history), 0,
                               self.sigma_A1, self.sigma_A2, bounds.Bbar_y, bounds.Bbar_xi)


@dataclass
class AlccResult:  # alcc.hpp:110-118
    point: PrimalPoint
    multiplier: np.ndarray | None
    objective: float
    certified_gap: float
    infeas_raw: float
    mapg_iters_total: int
    report: SolveReport
    gap_raw: float = 0.0
    mapg_iters: np.ndarray | None = None
    hit_cap: bool = False
    sigma_A1: float = 0.0
    sigma_A2: float = 0.0


class DualSolver:
    """One device handle over pair rows [row_begin, row_end) of an N x N
    problem (the whole matrix on one GPU by default). Owns the device-resident
    dual state between calls, like DualDecomposition (papg.hpp:33-58)."""

    def __init__(self, xs, ys_shifted, gamma=1e-3, device=0, row_begin=0, row_end=None):
        self.xs = np.ascontiguousarray(xs, np.float64)
        self.ys = np.ascontiguousarray(ys_shifted, np.float64)
        if self.xs.ndim != 2:
            raise ValueError("xs must be N x n")
        self.N, self.n = self.xs.shape
        if self.ys.shape != (self.N,):  # operators.cpp:12-14 shape checks
            raise ValueError(f"ys has shape {self.ys.shape}, expected ({self.N},)")
        self.row_begin = row_begin
        self.row_end = self.N if row_end is None else row_end
        self._L = nat.load()
        h = C.c_void_p()
        st = self._L.cr_create(nat.ptr(self.xs), nat.ptr(self.ys), self.N, self.n, gamma, device,
                               self.row_begin, self.row_end, C.byref(h))
        if st != 0:
            msg = self._L.cr_last_error(h).decode() if h.value else "cr_create failed"
            if h.value:
                self._L.cr_destroy(h)
            if st == 1:
                raise ValueError(msg)
            raise RuntimeError(msg)
        self.h = h
        self.cfg = None
        self.K = 0

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self._L.cr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- multi-GPU ------------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _raise(nat.load().cr_nccl_unique_id(buf))
        return buf.raw

    def attach_nccl(self, uid: bytes, rank: int, world: int):
        _raise(self._L.cr_attach_nccl(self.h, uid, rank, world), self.h)

    @property
    def sweep_variant(self) -> str:
        return {0: "dfma", 1: "mma"}.get(int(self._L.cr_sweep_variant(self.h)), "?")

    @property
    def exchange_len(self):
        return int(self._L.cr_exchange_len(self.h))

    # -- sigma_max(C) -------------------------------------------------------------
    def sigma_C(self, tol=1e-6, max_iters=5000):
        s = C.c_double(0)
        it = C.c_int32(0)
        cv = C.c_int32(0)
        _raise(self._L.cr_sigma_C(self.h, tol, max_iters, C.byref(s), C.byref(it), C.byref(cv)),
               self.h)
        return s.value, it.value, bool(cv.value)

    # -- loop -------------------------------------------------------------------
    def begin(self, cfg: PapgConfig, use_momentum=True, theta0=None):
        self.cfg = cfg
        c = cfg.to_c(use_momentum)
        t0 = None if theta0 is None else np.ascontiguousarray(theta0, np.float64).reshape(-1)
        if t0 is not None and t0.size != self._dual_len():  # papg.cpp:160-161
            raise ValueError("papg: warm-start theta has wrong size")
        _raise(self._L.cr_papg_begin(self.h, C.byref(c), nat.ptr(t0)), self.h)

    def iterate(self, max_steps):
        done = C.c_int64(0)
        stopped = C.c_int32(0)
        _raise(self._L.cr_papg_iterate(self.h, int(max_steps), C.byref(done), C.byref(stopped)),
               self.h)
        return done.value, bool(stopped.value)

    def set_canonical_blocks(self, D: int):
        """GPU-count-invariant sums (cr_set_canonical_blocks): D canonical row blocks, every
        block swept and reduced on its own, block payloads summed in block order."""
        _raise(self._L.cr_set_canonical_blocks(self.h, int(D)), self.h)

    def canonical_blocks(self):
        """(D, first block of this handle, blocks of this handle)."""
        D, first, count = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        _raise(self._L.cr_canonical_blocks(self.h, C.byref(D), C.byref(first), C.byref(count)),
               self.h)
        return D.value, first.value, count.value

    def iter_local(self):
        _raise(self._L.cr_iter_local(self.h), self.h)

    def exchange_get(self):
        buf = np.empty(self.exchange_len)
        _raise(self._L.cr_exchange_get(self.h, nat.ptr(buf)), self.h)
        return buf

    def exchange_put(self, buf):
        buf = np.ascontiguousarray(buf, np.float64)
        _raise(self._L.cr_exchange_put(self.h, nat.ptr(buf)), self.h)

    def iter_finish(self):
        stopped = C.c_int32(0)
        _raise(self._L.cr_iter_finish(self.h, C.byref(stopped)), self.h)
        return bool(stopped.value)

    def finish(self, want_history=True):
        res = nat.PapgResultC()
        y = np.empty(self.N)
        xi = np.empty(self.N * self.n)
        cap = 0
        if want_history and self.cfg is not None and self.cfg.record_history:
            cap = int(min(self.cfg.max_iters, nat.HISTORY_CAP))
        hist = np.zeros((max(cap, 1), 8))
        _raise(self._L.cr_papg_finish(self.h, C.byref(res), nat.ptr(y), nat.ptr(xi),
                                      nat.ptr(hist) if cap else None), self.h)
        return res, y, xi, hist[: min(res.iters, cap)] if cap else np.zeros((0, 8))

    def begin_resume(self, cfg: PapgConfig, use_momentum=True):
        """Warm start from this handle's theta1 (device-resident), e.g. the next
        gamma stage of a continuation (runner.cpp:258-259, 305, 322)."""
        self.cfg = cfg
        c = cfg.to_c(use_momentum)
        _raise(self._L.cr_papg_begin_resume(self.h, C.byref(c)), self.h)

    def set_observations(self, ys_shifted):
        self.ys = np.ascontiguousarray(ys_shifted, np.float64)
        _raise(self._L.cr_set_observations(self.h, nat.ptr(self.ys)), self.h)

    # -- one-shot metric sweeps (metrics.cpp) --------------------------------
    def infeasibility(self, y, xi):
        out = np.empty(2)
        _raise(self._L.cr_infeasibility(self.h, nat.ptr(_f64(y)), nat.ptr(_f64(xi)),
                                        nat.ptr(out)), self.h)
        return float(out[0]), float(out[1])

    def duality_gap(self, y, xi):
        """theta1 . C eta with this handle's current theta1 (metrics.cpp:17-30)."""
        out = np.empty(2)
        _raise(self._L.cr_duality_gap(self.h, nat.ptr(_f64(y)), nat.ptr(_f64(xi)), nat.ptr(out)),
               self.h)
        return float(out[0]), float(out[1])

    def evaluate_estimator(self, y, xi, Xq):
        Xq = _f64(Xq).reshape(-1, self.n)
        out = np.empty(Xq.shape[0])
        _raise(self._L.cr_evaluate_estimator(self.h, nat.ptr(_f64(y)), nat.ptr(_f64(xi)),
                                             nat.ptr(Xq), Xq.shape[0], nat.ptr(out)), self.h)
        return out

    def repair_feasibility(self, y, xi):
        out = np.empty(self.N)
        _raise(self._L.cr_repair_feasibility(self.h, nat.ptr(_f64(y)), nat.ptr(_f64(xi)),
                                             nat.ptr(out)), self.h)
        return out

    def _dual_len(self):
        K = getattr(self, "K", 0)
        if K:
            return self.N * (self.N - self.N // K) + self.N
        return (self.row_end - self.row_begin) * (self.N - 1) + self.N

    def theta(self):
        out = np.empty(self._dual_len())
        _raise(self._L.cr_get_theta(self.h, nat.ptr(out)), self.h)
        return out

    def rows(self):
        out = np.empty(self._dual_len())
        _raise(self._L.cr_get_rows(self.h, nat.ptr(out)), self.h)
        return out

    def theta_rows(self, row_begin, row_end):
        """theta1 of global pair rows [row_begin, row_end) (canonical order) + the N pos rows."""
        out = np.empty((row_end - row_begin) * (self.N - 1) + self.N)
        _raise(self._L.cr_get_theta_rows(self.h, row_begin, row_end, nat.ptr(out)), self.h)
        return out

    def rows_window(self, row_begin, row_end):
        """C eta of the last iteration for pair rows [row_begin, row_end) + the N pos rows."""
        out = np.empty((row_end - row_begin) * (self.N - 1) + self.N)
        _raise(self._L.cr_get_rows_window(self.h, row_begin, row_end, nat.ptr(out)), self.h)
        return out

    def last_timing(self):
        s = C.c_double(0)
        k = C.c_int64(0)
        sw = C.c_double(0)
        _raise(self._L.cr_last_timing(self.h, C.byref(s), C.byref(k), C.byref(sw)), self.h)
        return s.value, k.value, sw.value

    def last_exchange_seconds(self):
        """Sharded runs: allreduce device time of the last iterate call (s)."""
        x = C.c_double(0)
        _raise(self._L.cr_last_exchange_seconds(self.h, C.byref(x)), self.h)
        return x.value

    def last_sweep_times(self):
        """Durations (s) of the sweep launches the last iterate call bracketed with
        CUDA events, in launch order (every launch of a call of <= 64 iterations)."""
        k = C.c_int64(0)
        _raise(self._L.cr_last_sweep_times(self.h, None, 0, C.byref(k)), self.h)
        out = np.zeros(k.value)
        _raise(self._L.cr_last_sweep_times(self.h, nat.ptr(out), k.value, C.byref(k)), self.h)
        return out

    def sweep_store_count(self, reset=False):
        """Multipliers written by the P-APG sweeps since the last reset (whole
        32-byte sectors: those with a changed multiplier)."""
        c = C.c_uint64(0)
        _raise(self._L.cr_sweep_store_count(self.h, C.byref(c), int(reset)), self.h)
        return c.value

    def time_sweep(self, k=10):
        """Times k sweep launches alone; clobbers the previous dual iterate."""
        s = C.c_double(0)
        _raise(self._L.cr_time_sweep(self.h, k, C.byref(s)), self.h)
        return s.value


    # ---- general-K partition (P-APG(ALCC), papg.cpp:66-132)
    def set_partition(self, K, feasible: PrimalPoint, inner: "AlccConfig | None" = None):
        """K blocks of N/K consecutive points; K = N (or 0) selects singleton blocks."""
        inner = inner or AlccConfig()
        c = inner.to_c(ProblemBounds(0.0, 0.0, 0.0, 0.0))
        _raise(self._L.cr_set_partition(self.h, K, nat.ptr(_f64(feasible.y)),
                                        nat.ptr(_f64(feasible.xi)), C.byref(c)), self.h)
        self.K = K if 0 < K < self.N else 0

    def partition_stats(self):
        K = getattr(self, "K", 0)
        it = C.c_int64(0)
        sec = C.c_double(0)
        s1 = C.c_double(0)
        s2 = np.zeros(max(K, 1))
        _raise(self._L.cr_partition_stats(self.h, C.byref(it), C.byref(sec), C.byref(s1),
                                          nat.ptr(s2)), self.h)
        return dict(inner_iters=it.value, inner_seconds=sec.value, sigma_A1=s1.value,
                    sigma_A2=s2[:K].copy())

    # ---- standalone ALCC (alcc.cpp:193-208) on this handle's device buffers
    def sigma_A(self, which, tol=1e-6, max_iters=5000):
        """estimate_sigma_max(op_A1) (which=1) / (op_A2) (which=2), operators.cpp:302-351."""
        s = C.c_double(0)
        it = C.c_int32(0)
        cv = C.c_int32(0)
        _raise(self._L.cr_sigma_A(self.h, which, tol, max_iters, C.byref(s), C.byref(it),
                                  C.byref(cv)), self.h)
        return s.value, it.value, bool(cv.value)

    def alcc(self, cfg: "AlccConfig", bounds: ProblemBounds, warm: PrimalPoint):
        c = cfg.to_c(bounds)
        N, n = self.N, self.n
        y = np.empty(N)
        xi = np.empty(N * n)
        K = max(int(cfg.max_outer), 0)
        hist = np.zeros((max(K, 1), 8))
        mi = np.zeros(max(K, 1), np.int64)
        res = nat.AlccResultC()
        _raise(self._L.cr_alcc_solve(self.h, C.byref(c), nat.ptr(_f64(warm.y)),
                                     nat.ptr(_f64(warm.xi)), nat.ptr(y), nat.ptr(xi),
                                     nat.ptr(hist) if cfg.record_history else None,
                                     mi.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(res)),
               self.h)
        k = int(res.outer_iters)
        return res, y, xi, hist[:k] if cfg.record_history else hist[:0], mi[:k]

    def time_penalty_sweep(self, k=10):
        """Times k penalty-sweep launches on the last ALCC state (read-only)."""
        s = C.c_double(0)
        _raise(self._L.cr_time_penalty_sweep(self.h, k, C.byref(s)), self.h)
        return s.value

    def alcc_multiplier(self, row_begin=0, row_end=None):
        row_end = self.N if row_end is None else row_end
        out = np.empty((row_end - row_begin) * (self.N - 1))
        _raise(self._L.cr_alcc_multiplier(self.h, row_begin, row_end, nat.ptr(out)), self.h)
        return out


def alcc_solve(prep: PreparedProblem, cfg: AlccConfig | None = None,
               warm: PrimalPoint | None = None, device=0, want_multiplier=True) -> AlccResult:
    """Standalone Fig-3 augmented Lagrangian (alcc.cpp:193-208 -> alcc_core
    :54-191), centres (ybar, 0), balls from prep.bounds, warm start = the
    exactly feasible affine point unless given (runner.cpp:278-286)."""
    cfg = cfg or AlccConfig()
    warm = warm or prep.feasible
    data = prep.data
    with DualSolver(data.xs, data.ys, prep.bounds.gamma, device) as s:
        res, y, xi, hist, mi = s.alcc(cfg, prep.bounds, warm)
        mult = s.alcc_multiplier() if (want_multiplier and res.outer_iters > 0) else None
    history = [MetricsSnapshot(int(h[0]), *map(float, h[1:])) for h in hist]
    rep = SolveReport(history=history, reason=TermReason(res.reason), iters=int(res.outer_iters),
                      wall_seconds=res.wall_seconds, history_array=hist)
    return AlccResult(PrimalPoint(y, xi), mult, res.objective, res.certified_gap, res.infeas_raw,
                      int(res.mapg_iters_total), rep, res.gap_raw, mi, bool(res.hit_cap_any),
                      res.sigma_A1, res.sigma_A2)


def _solve(prep: PreparedProblem, cfg: PapgConfig, theta0, use_momentum, want_dual=True):
    data = prep.data
    N = data.N
    with DualSolver(data.xs, data.ys, cfg.gamma, cfg.device) as s:
        K = cfg.K if 0 < cfg.K < N else 0
        if K:
            s.set_partition(K, prep.feasible, cfg.inner)
        if cfg.canonical_blocks > 0:
            s.set_canonical_blocks(cfg.canonical_blocks)
        s.begin(cfg, use_momentum, theta0)
        stopped = False
        while not stopped:
            _, stopped = s.iterate(1 << 40)
        res, y, xi, hist = s.finish()
        dual = None
        if want_dual:
            th = s.theta()
            cross = N * (N - (N // K if K else 1))
            dual = DualPoint(th[:cross], th[cross:])
    history = [MetricsSnapshot(int(h[0]), *map(float, h[1:])) for h in hist]
    rep = SolveReport(history=history, reason=TermReason(res.reason), iters=int(res.iters),
                      wall_seconds=res.wall_seconds, restarts=res.restarts,
                      saturated=bool(res.saturated), history_array=hist,
                      history_truncated=bool(res.history_truncated))
    return PapgResult(PrimalPoint(y, xi), dual, rep, res.g_final, res.delta_estimate, res.sigma_C,
                      res.L_g, res.B_theta, res.sigma_iters, res.sigma_seconds, res.loop_seconds)


def papg_solve(prep: PreparedProblem, cfg: PapgConfig | None = None, theta0=None,
               want_dual=True) -> PapgResult:
    """Fig. 2 P-APG on the regularised dual, singleton blocks (papg.cpp:287-290)."""
    return _solve(prep, cfg or PapgConfig(), theta0, True, want_dual)


def dual_gradient_ascent(prep: PreparedProblem, cfg: PapgConfig | None = None, theta0=None,
                         want_dual=True) -> PapgResult:
    """Projected dual gradient ascent baseline (papg.cpp:292-296)."""
    return _solve(prep, cfg or PapgConfig(), theta0, False, want_dual)


def infeasibility(data: Dataset, eta: PrimalPoint, device=0):
    """(raw, normalised) |(A1 y + A2 xi)_-| over all N(N-1) rows (metrics.cpp:8-15)."""
    with DualSolver(data.xs, data.ys, device=device) as s:
        return s.infeasibility(eta.y, eta.xi)


def evaluate_estimator(eta: PrimalPoint, data: Dataset, x_query, device=0):
    """max_l y_l + xi_l.(x - x_l) (metrics.cpp:32-48); x_query (n,) or (Q, n)."""
    xq = np.asarray(x_query, np.float64)
    with DualSolver(data.xs, data.ys, device=device) as s:
        out = s.evaluate_estimator(eta.y, eta.xi, xq)
    return float(out[0]) if xq.ndim == 1 else out


def repair_feasibility(eta: PrimalPoint, data: Dataset, device=0) -> PrimalPoint:
    """y'_l = estimator(x_l): an exactly feasible point (metrics.cpp:50-56)."""
    with DualSolver(data.xs, data.ys, device=device) as s:
        return PrimalPoint(s.repair_feasibility(eta.y, eta.xi), np.array(eta.xi, copy=True))
