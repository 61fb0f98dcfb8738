"""B200-native singleton-block P-APG pair sweep for least-squares convex
regression (arXiv 1407.7220, reference `cvxreg` proj/core)."""
from .papg import (AlccConfig, AlccResult, Dataset, DualPoint, DualSolver, GeneratorSpec,  # noqa: F401
                   MetricsSnapshot, PapgConfig, PapgResult, PreparedProblem, PrimalPoint,
                   ProblemBounds, SolveReport, TermReason, certificate_for_iterate,
                   dual_gradient_ascent, evaluate_estimator, gen_instance, infeasibility,
                   momentum_next, papg_solve, alcc_solve, prepare_problem, repair_feasibility)
