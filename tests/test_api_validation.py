"""Reference-facing API validation on the host (no GPU): the checks run before any
engine is created, with the reference's exception types (`errors.py:4-57`)."""

import numpy as np
import pytest

from paper_2004_00546_b200 import (RK4Config, baseline, descend, direct_adjoint_loop, scaled, solve_adjoint_linear,
                                   solve_direct_linear, solve_hybrid)
from paper_2004_00546_b200.errors import ConfigError
from paper_2004_00546_b200.optimization import ALGORITHMS


def test_algorithms_match_reference_names():
    assert set(ALGORITHMS) == {"serial", "linear", "nonlinear", "hybrid"}


def test_loop_rejects_bad_arguments():
    c = baseline(1)
    u0, ut, ctrl = c.inputs()
    rk = RK4Config(c.dt)
    with pytest.raises(ValueError):
        direct_adjoint_loop(c.system, ctrl, ut, "linear", N=c.P, rk=rk, backend="thread")
    with pytest.raises(ValueError):
        direct_adjoint_loop(c.system, ctrl, ut, "chebyshev", N=c.P, rk=rk)
    with pytest.raises(ValueError):   # Burgers algorithms on the linear testbed
        direct_adjoint_loop(c.system, ctrl, ut, "hybrid", N=c.P, rk=rk)
    with pytest.raises(ConfigError):  # fixed-step RK4 needs its dt
        direct_adjoint_loop(c.system, ctrl, ut, "linear", N=c.P)
    with pytest.raises(ValueError):   # control coefficients of the wrong length
        direct_adjoint_loop(c.system, np.zeros(c.K + 1), ut, "linear", N=c.P, rk=rk)
    b = baseline(3)
    with pytest.raises(ValueError):   # linear algorithm on Burgers
        direct_adjoint_loop(b.system, b.inputs()[2], b.inputs()[1], "linear", N=b.P, rk=RK4Config(b.dt))
    with pytest.raises(ValueError):
        descend(c.system, ctrl, ut, steps=1, lr=0.0, N=c.P, rk=rk)
    brk = RK4Config(b.dt)
    with pytest.raises(ValueError):   # unknown Burgers adjoint form
        direct_adjoint_loop(b.system, b.inputs()[2], b.inputs()[1], "hybrid", N=b.P, rk=brk, hybrid_adjoint="x")
    with pytest.raises(ValueError):   # the frozen-span adjoint is solve_hybrid's (the hybrid algorithm)
        direct_adjoint_loop(b.system, b.inputs()[2], b.inputs()[1], "nonlinear", N=b.P, rk=brk,
                            hybrid_adjoint="frozen_span")


def test_solver_level_rejects_wrong_testbed():
    c = baseline(1)
    b = baseline(3)
    rk = RK4Config(c.dt)
    with pytest.raises(ValueError):
        solve_direct_linear(b.system, b.inputs()[0], b.inputs()[2], b.P, RK4Config(b.dt))
    with pytest.raises(ValueError):
        solve_adjoint_linear(b.system, np.zeros(b.n), b.P, RK4Config(b.dt))
    with pytest.raises(ValueError):
        solve_hybrid(c.system, c.inputs()[0], c.inputs()[2], None, c.P, rk)
    with pytest.raises(ConfigError):
        solve_direct_linear(c.system, c.inputs()[0], c.inputs()[2], c.P, None)


def test_unstable_step_is_a_config_error():
    """An RK4 step outside the stability region is refused before any GPU work."""
    from paper_2004_00546_b200.engine import check_rk4_stability
    c = scaled(baseline(5), nx=640, P=4, steps_per_slice=10, K=16)
    with pytest.raises(ConfigError):
        check_rk4_stability(c.system.region(), c.dt)


def test_planner_failure_is_propagation_failure():
    """An exp-action that no admissible Chebyshev plan can deliver raises the reference's
    PropagationFailure (`errors.py:18-19`) on the host, before any GPU work."""
    from paper_2004_00546_b200 import ChebyshevConfig
    from paper_2004_00546_b200.errors import PropagationFailure
    from paper_2004_00546_b200.expaction import plan_chebyshev
    c = baseline(2)
    with pytest.raises(PropagationFailure):
        plan_chebyshev(c.system.region(), 50.0 * c.spec.T, ChebyshevConfig(tol=1e-14, max_degree=8))
