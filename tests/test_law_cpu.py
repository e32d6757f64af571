"""The forcing time law and the field control on the CPU: the oracle restatement
(oracle.config_mode.linear_gradient_law) against the time-constant oracle and finite
differences, the planner's law series, and the host-side API validation."""

import numpy as np
import pytest

from tests.conftest import rel_l2


def _case():
    from paper_2004_00546_b200 import baseline
    from paper_2004_00546_b200.expaction import ChebyshevConfig, plan_chebyshev
    c = baseline(1)
    s = c.system
    u0, ut, ctrl = c.inputs()
    pl = plan_chebyshev(s.region(), c.spec.T / c.P, ChebyshevConfig(tol=1e-13), omega=3.0)
    args = (s.grid.nx, s.grid.ny, s.A.as_tuple(), s.basis, c.spec.T, c.P, c.nsteps, u0, ut)
    return c, args, ctrl, pl


def test_constant_law_is_the_time_constant_path():
    from oracle.config_mode import linear_gradient, linear_gradient_law
    c, args, ctrl, pl = _case()
    r1 = linear_gradient_law(*args, ctrl, (1.0, 0.0, 0.0, 0.0), pl)
    r0 = linear_gradient(*args, ctrl, pl)
    assert np.allclose(r1.J, r0.J, rtol=1e-14, atol=0)
    assert rel_l2(r1.grad, r0.grad) <= 1e-13 and rel_l2(r1.G, r0.G) <= 1e-13


def test_law_gradient_vs_finite_differences():
    """J is quadratic in the controls and the discrete adjoint is exact up to the exp-action
    truncation: central differences agree to ~1e-10."""
    from oracle.config_mode import linear_gradient_law
    c, args, ctrl, pl = _case()
    law = (0.2, 1.0, 0.3, 3.0)
    r = linear_gradient_law(*args, ctrl, law, pl)
    d = np.random.default_rng(0).standard_normal(ctrl.shape)
    eps = 1e-5
    fd = (linear_gradient_law(*args, ctrl + eps * d, law, pl).J - linear_gradient_law(*args, ctrl - eps * d, law, pl).J) / (2 * eps)
    assert abs(fd[0] - np.sum(r.grad * d)) <= 1e-8 * abs(fd[0])


def test_law_series_in_the_slice_plan():
    _, _, _, pl = _case()
    assert pl.omega == 3.0 and pl.coef_gc is not None and len(pl.coef_gs) == pl.degree + 1


def test_field_basis_is_the_identity():
    from paper_2004_00546_b200 import ADVECTION_DIFFUSION, Grid, ProblemSpec
    from paper_2004_00546_b200.systems import build_field_system
    fs = build_field_system(Grid(16, 8), ProblemSpec(ADVECTION_DIFFUSION, (1.0, 0.5), 0.01, 1.0))
    x = np.random.default_rng(1).standard_normal((2, 128))
    assert fs.basis.K == fs.n == 128 and np.array_equal(fs.basis.field(x), x) and np.array_equal(fs.basis.project(x), x)
    with pytest.raises(ValueError):
        from paper_2004_00546_b200 import BURGERS
        build_field_system(Grid(16), ProblemSpec(BURGERS, (0.0, 0.0), 0.01, 1.0))


def test_time_law_api_validation():
    from paper_2004_00546_b200 import ConfigError, RK4Config, TimeLaw, baseline, direct_adjoint_loop
    c3 = baseline(3)
    with pytest.raises(ConfigError):   # Burgers with the terminal objective: no law
        direct_adjoint_loop(c3.system, np.zeros(c3.system.basis.K), np.zeros(c3.system.n), "hybrid",
                            rk=RK4Config(c3.dt), time_law=TimeLaw.sine(1.0))
