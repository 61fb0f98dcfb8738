"""CPU-side checks of the product library (no GPU compute):
  * libcvxreg_b200.so loads and exports every symbol include/cvxreg_b200.h declares,
  * its host utilities (generators, prepare_problem, certificate) agree with the oracle,
  * the device entry points fail loudly without a GPU (no CPU fallback).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1407_7220_b200 as crb
from paper_1407_7220_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "cvxreg_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cr_[A-Za-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = nat.load()
    declared = _declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(nat.EXPORTS) == declared


def test_cpp_header_mirrors_c_abi():
    hpp = open(os.path.join(ROOT, "include", "cvxreg_b200", "papg.hpp")).read()
    for name in ["papg_solve", "dual_gradient_ascent", "prepare_problem", "gen_instance",
                 "certificate_for_iterate", "PapgConfig", "PapgResult", "SolveReport",
                 "MetricsSnapshot", "TermReason"]:
        assert name in hpp


KINDS = [("quadratic", 50, 3, 1.0, 0), ("exponential", 40, 2, 0.5, 0),
         ("affine-noiseless", 30, 4, 0.0, 0), ("custom-1d", 25, 1, 0.3, 0),
         ("sqnorm-uniform", 100, 5, 0.1, 0), ("maxaffine-uniform", 90, 10, 0.1, 20),
         ("lse-uniform", 70, 20, 0.05, 50)]


@pytest.mark.parametrize("kind,N,n,noise,pieces", KINDS)
def test_generators_bit_identical_to_oracle(oracle, kind, N, n, noise, pieces):
    d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, noise, 11, pieces))
    X, y = oracle.gen_instance(kind, N, n, noise, 11, pieces)
    assert np.array_equal(d.xs, X) and np.array_equal(d.ys, y)


def test_generator_rejects_bad_specs():
    with pytest.raises(ValueError):
        crb.gen_instance(crb.GeneratorSpec("quadratic", 3, 3))  # N < n + 1
    with pytest.raises(ValueError):
        crb.gen_instance(crb.GeneratorSpec("custom-1d", 2, 10))
    with pytest.raises(ValueError):
        crb.gen_instance(crb.GeneratorSpec("nope", 2, 10))


@pytest.mark.parametrize("kind,N,n,noise,pieces", KINDS)
def test_prepare_problem_matches_oracle(oracle, kind, N, n, noise, pieces):
    d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, noise, 3, pieces))
    p = crb.prepare_problem(d, 1e-3)
    o = oracle.prepare(d.xs, d.ys, 1e-3)
    assert abs(p.shift - o.shift) <= 1e-12 * max(1.0, abs(o.shift))
    assert np.allclose(p.data.ys, o.ys, rtol=1e-13, atol=1e-13)
    assert np.allclose(p.feasible.y, o.feas_y, rtol=1e-12, atol=1e-12)
    assert np.allclose(p.feasible.xi, o.feas_xi, rtol=1e-10, atol=1e-12)
    assert p.bounds.B_theta == pytest.approx(o.B_theta)
    assert p.bounds.Bbar_y == pytest.approx(o.Bbar_y, rel=1e-12)


def test_prepare_rejects_bad_gamma():
    d = crb.gen_instance(crb.GeneratorSpec("quadratic", 2, 10))
    with pytest.raises(ValueError):
        crb.prepare_problem(d, 0.0)


def test_certificate_and_momentum():
    a, b = crb.certificate_for_iterate(0.04, 1e-4, 1.0, 2.0)
    assert abs(a - 0.3414) < 1e-4 and abs(b - 0.1414) < 1e-4
    assert crb.momentum_next(1.0) == pytest.approx((1 + 5 ** 0.5) / 2)


def _have_gpu():
    try:
        cudart = ctypes.CDLL("libcuda.so.1")
        return cudart.cuInit(0) == 0
    except OSError:
        return False


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure path")
def test_device_path_fails_loudly_without_gpu():
    d = crb.gen_instance(crb.GeneratorSpec("sqnorm-uniform", 3, 20, 0.1))
    p = crb.prepare_problem(d)
    with pytest.raises(RuntimeError):
        crb.papg_solve(p, crb.PapgConfig(max_iters=2))
    with pytest.raises(RuntimeError):
        crb.DualSolver(p.data.xs, p.data.ys)


def test_create_rejects_invalid_shapes():
    X = np.zeros((40, 33))
    with pytest.raises(ValueError):
        crb.DualSolver(X, np.zeros(40))  # n > 32 (kMaxN) is not supported
    with pytest.raises(ValueError):
        crb.DualSolver(np.zeros((1, 2)), np.zeros(1))
    with pytest.raises(ValueError):
        crb.DualSolver(np.zeros((40, 3)), np.zeros(39))  # ys must have N entries


def test_host_side_generators_and_prepare_match_the_compiled_reference():
    """The drop-in's own host code (csrc/host.cpp: gen_instance, prepare_problem) against the
    reference's testgen.cpp / preprocess.cpp compiled in oracle/_ref, when that is present."""
    from oracle import ref as R

    if not R.available():
        pytest.skip("oracle/_ref not built")
    for kind, n in (("quadratic", 3), ("exponential", 4), ("affine-noiseless", 2),
                    ("custom-1d", 1)):
        d = crb.gen_instance(crb.GeneratorSpec(kind, n, 40, 0.3, 9))
        Xr, yr = R.gen_instance(kind, 40, n, 0.3, 9)
        assert np.array_equal(d.xs, Xr)
        assert np.allclose(d.ys, yr, rtol=1e-13, atol=1e-14)
    d = crb.gen_instance(crb.GeneratorSpec("quadratic", 4, 90, 0.5, 2))
    p = crb.prepare_problem(d, 1e-3)
    r = R.prepare(d.xs, d.ys, 1e-3)
    assert np.allclose(p.data.ys, r.ys, rtol=1e-13)
    assert p.shift == pytest.approx(r.shift, rel=1e-13)
    assert np.allclose(p.feasible.y, r.feas_y, rtol=1e-11, atol=1e-12)
    assert np.allclose(p.feasible.xi, r.feas_xi, rtol=1e-10, atol=1e-12)
    b = p.bounds
    assert (b.B_theta, b.gamma) == (r.B_theta, r.gamma)
    assert b.Bbar_y == pytest.approx(r.Bbar_y, rel=1e-12)
    assert b.Bbar_xi == pytest.approx(r.Bbar_xi, rel=1e-12)
    assert crb.momentum_next(1.0) == R.momentum_next(1.0)
    assert np.allclose(crb.certificate_for_iterate(1e-3, 0.02, 3.0, 40.0),
                       R.certificate(1e-3, 0.02, 3.0, 40.0), rtol=1e-15)
