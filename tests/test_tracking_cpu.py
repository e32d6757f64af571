"""The linear testbed's tracking objective (the reference's linear loop, `optimization.py:154-231`)
on the CPU: the oracle restatement (oracle.config_mode.linear_tracking_gradient) pinned to the
reference's own loop (tests/golden/reference_linear_tracking.npz, made by
oracle/gen_golden_linear_tracking.py) and checked against finite differences of its own J."""

import os

import numpy as np

from tests.conftest import rel_l2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _golden_problem(steps):
    from oracle.config_mode import rk4_full_law, stencil_apply
    from paper_2004_00546_b200 import ChebyshevConfig, TimeLaw
    from paper_2004_00546_b200.expaction import plan_chebyshev
    from paper_2004_00546_b200.problems import ADVECTION_DIFFUSION, Grid, ProblemSpec
    from paper_2004_00546_b200.systems import build_field_system
    g = np.load(os.path.join(ROOT, "tests", "golden", "reference_linear_tracking.npz"))
    nx, ny, T, N = int(g["nx"]), int(g["ny"]), float(g["T"]), int(g["N"])
    fs = build_field_system(Grid(nx, ny), ProblemSpec(ADVECTION_DIFFUSION, (float(g["a"]),) * 2, float(g["D"]), T))
    law = TimeLaw.sine(float(g["omega"]))
    S = N * steps
    A = fs.A.as_tuple()
    # q_true: the serial RK4 trajectory of f_true (the reference synthesises it by DOPRI5)
    target = rk4_full_law(lambda u: stencil_apply(A, u, nx, ny), np.zeros((1, fs.n)), g["f_true"][None, :],
                          law.as_tuple(), 0.0, T / S, S)[:, 0]
    pl = plan_chebyshev(fs.region(), T / N, ChebyshevConfig(tol=1e-13), omega=law.omega)
    return g, fs, law, target, pl


def test_oracle_vs_the_reference_linear_loop():
    """J, ∂L/∂f, q†(0) and u(T) of the reference's linear loop (DOPRI5 + Leja, probe-grid
    trapezoids) against the restatement (classical RK4, Chebyshev carries, node trapezoid):
    agreement at the discretisations' level, improving with the step."""
    from oracle.config_mode import linear_tracking_gradient
    errs = []
    for steps in (100, 200):
        g, fs, law, target, pl = _golden_problem(steps)
        o = linear_tracking_gradient(int(g["nx"]), int(g["ny"]), fs.A.as_tuple(), fs.basis, float(g["T"]), int(g["N"]),
                                     steps, np.zeros(fs.n), g["f"], law.as_tuple(), target, pl)
        errs.append((abs(o.J[0] - g["J"]) / g["J"], rel_l2(o.grad[0], g["grad"]), rel_l2(o.qdag0[0], g["qdag0"])))
        assert rel_l2(o.uT[0], g["uT"]) <= 2e-12
    assert errs[1][0] <= 2e-5 and errs[1][1] <= 5e-6 and errs[1][2] <= 5e-6
    assert all(b < 0.5 * a for a, b in zip(errs[0], errs[1]))   # second order in the step


def test_oracle_gradient_vs_finite_differences():
    """The continuous adjoint's gradient against central differences of the oracle's own J,
    converging at second order (trapezoid cost, linearly interpolated source)."""
    from oracle.config_mode import linear_tracking_gradient
    from paper_2004_00546_b200 import ChebyshevConfig, TimeLaw, baseline, scaled
    from paper_2004_00546_b200.expaction import plan_chebyshev
    from paper_2004_00546_b200.systems import build_field_system
    rel = []
    for ns in (5, 10):
        c = scaled(baseline(5), nx=16, P=4, steps_per_slice=ns, K=4)
        fs = build_field_system(c.system.grid, c.system.spec)
        law = TimeLaw.sine(5.0)
        pl = plan_chebyshev(fs.region(), c.spec.T / c.P, ChebyshevConfig(tol=1e-13), omega=law.omega)
        rng = np.random.default_rng(0)
        u0, f, d = 0.1 * rng.standard_normal(fs.n), rng.standard_normal(fs.n), rng.standard_normal(fs.n)
        S = c.P * c.nsteps
        tg = np.sin(3.0 * np.linspace(0.0, 1.0, S + 1))[:, None] * (0.1 * rng.standard_normal(fs.n))[None, :]
        args = (fs.grid.nx, fs.grid.ny, fs.A.as_tuple(), fs.basis, c.spec.T, c.P, c.nsteps, u0)
        o = linear_tracking_gradient(*args, f, law.as_tuple(), tg, pl)
        eps = 1e-5
        Jp = linear_tracking_gradient(*args, f + eps * d, law.as_tuple(), tg, pl).J[0]
        Jm = linear_tracking_gradient(*args, f - eps * d, law.as_tuple(), tg, pl).J[0]
        fd = (Jp - Jm) / (2 * eps)
        rel.append(abs(fd - o.grad[0] @ d) / abs(fd))
    assert rel[0] <= 2e-2 and rel[1] <= 0.3 * rel[0]
