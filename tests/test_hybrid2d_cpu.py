"""CPU tests of the reference's hybrid loop on its 2D two-field Burgers testbed: the config-mode
restatement (oracle.config_mode.burgers_tracking_hybrid with ``ny``) pinned to the reference's own
loop (tests/golden/reference_hybrid2d_tracking.npz from oracle/gen_golden_hybrid2d.py), the FOV
box of the frozen two-field operator, and the gradient against finite differences."""

import os

import numpy as np

from paper_2004_00546_b200.expaction import ChebyshevConfig, plan_family
from paper_2004_00546_b200.hybrid import TimeLaw, make_hybrid_plan, slice_offsets
from paper_2004_00546_b200.problems import Grid, frozen_bounds, frozen_bounds_2d, frozen_region_from_bounds

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_hybrid2d_tracking.npz")


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _plans_for(grid, D, offs, h, w, tol=1e-12):
    cfg = ChebyshevConfig(tol=tol)

    def plans_for(ubar):
        reg = frozen_region_from_bounds(*frozen_bounds_2d(ubar, grid, D))
        return plan_family(reg, [(offs[p + 1] - offs[p]) * h for p in range(len(offs) - 1)], cfg, omega=w)

    return plans_for


def _golden_case(dt):
    from oracle.config_mode import burgers_direct_law, burgers_ops, burgers_tracking_hybrid
    gd = np.load(GOLDEN)
    nx, ny, T, D, w = int(gd["nx"]), int(gd["ny"]), float(gd["T"]), float(gd["D"]), float(gd["omega"])
    law = TimeLaw.sine(w).as_tuple()
    grid = Grid(nx, ny)
    offs = slice_offsets(make_hybrid_plan(T, int(gd["N"]), float(gd["k"])).partition, dt)
    S = int(offs[-1])
    h = T / S
    rhs, _, n2 = burgers_ops(nx, D, ny)
    tgt = burgers_direct_law(np.zeros((1, n2)), gd["f_true"][None, :], law, D, grid.hx, h, S, rhs=rhs)[:, 0, :]
    return gd, burgers_tracking_hybrid(nx, D, T, offs, np.zeros(n2), gd["f"], law, tgt,
                                       _plans_for(grid, D, offs, h, w), ny=ny)


def test_oracle_2d_tracking_hybrid_pinned_to_the_reference_loop():
    """Classical RK4 / Chebyshev frozen actions / node trapezoid against the reference's own
    hybrid loop on a genuinely two-dimensional two-field problem (DOPRI5 at rtol 1e-10, Leja,
    4001 probe nodes): agreement at the discretisations' level."""
    gd, r = _golden_case(1e-3)
    assert abs(r.J[0] - gd["J"]) <= 1e-6 * abs(gd["J"])
    assert rel_l2(r.grad[0], gd["grad"]) <= 1e-5
    assert rel_l2(r.qdag0[0], gd["qdag0"]) <= 1e-6
    assert rel_l2(r.uT[0], gd["uT"]) <= 1e-9
    n = int(gd["nx"]) * int(gd["ny"])
    assert np.linalg.norm(r.grad[0][n:]) > 1e-2 * np.linalg.norm(r.grad[0])  # the V block is active


def test_frozen_bounds_2d_enclose_the_field_of_values_and_reduce_to_1d():
    from oracle.config_mode import burgers2d_adjoint_apply
    rng = np.random.default_rng(5)
    nx, ny, D = 9, 7, 0.03
    g = Grid(nx, ny)
    n = nx * ny
    q = rng.normal(size=2 * n)
    lo, hi, im = frozen_bounds_2d(q, g, D)
    M = np.stack([burgers2d_adjoint_apply(q, e, D, g.hx, g.hy, nx, ny) for e in np.eye(2 * n)], axis=1)
    ev_h = np.linalg.eigvalsh(0.5 * (M + M.T))
    ev_s = np.linalg.eigvals(0.5 * (M - M.T)).imag
    assert lo <= ev_h.min() and ev_h.max() <= hi and np.abs(ev_s).max() <= im
    # y-invariant U, V ≡ 0: the 1D box
    u = rng.normal(size=nx)
    q1 = np.concatenate([np.tile(u, ny), np.zeros(n)])
    b2 = frozen_bounds_2d(q1, g, D)
    b1 = frozen_bounds(u, Grid(nx), D)
    dy = 2.0 * D / g.hy**2
    assert abs(b2[0] - (b1[0] - 2 * dy)) <= 1e-12 * abs(b2[0]) and abs(b2[2] - b1[2]) <= 1e-12 * b1[2]


def test_oracle_2d_gradient_vs_finite_differences():
    """∂L/∂f of the serial one-slice loop (exact discrete-adjoint structure up to O(h²)) against
    central differences of the oracle's own J, in both components."""
    from oracle.config_mode import burgers_direct_law, burgers_ops, burgers_tracking_hybrid
    nx, ny, D, T, S, w = 8, 6, 0.08, 0.3, 300, 3.0
    g = Grid(nx, ny)
    n = nx * ny
    law = TimeLaw.sine(w).as_tuple()
    X, Y = g.coordinates()
    f = np.concatenate([0.3 * np.sin(X) * np.cos(Y), 0.2 * np.cos(X + Y)])
    ft = np.concatenate([0.5 * np.sin(X) * np.sin(Y), 0.3 * np.sin(Y)])
    rhs, _, n2 = burgers_ops(nx, D, ny)
    u0 = np.concatenate([0.2 * np.cos(X), 0.1 * np.sin(X - Y)])
    tgt = burgers_direct_law(u0[None, :], ft[None, :], law, D, g.hx, T / S, S, rhs=rhs)[:, 0, :]
    run = lambda ff: burgers_tracking_hybrid(nx, D, T, [0, S], u0, ff, law, tgt, lambda ub: [], ny=ny)
    r = run(f)
    rng = np.random.default_rng(1)
    d = rng.normal(size=2 * n)
    eps = 1e-5
    fd = (run(f + eps * d).J[0] - run(f - eps * d).J[0]) / (2 * eps)
    # the gradient w.r.t. a field on the grid: L's derivative in direction d is ⟨grad, d⟩
    assert abs(fd - float(r.grad[0] @ d)) <= 2e-4 * abs(fd)


def _nl_plans(grid, D, delta, h, w, tol=1e-12):
    from paper_2004_00546_b200.expaction import plan_chebyshev
    cfg = ChebyshevConfig(tol=tol)

    def plans_nl(qbar):
        reg = frozen_region_from_bounds(*frozen_bounds_2d(qbar, grid, D))
        return plan_chebyshev(reg, delta, cfg), plan_chebyshev(reg, h, cfg)

    return plans_nl


def test_oracle_2d_nonlinear_loop_pinned_to_the_reference_loop():
    """The reference's loop with algorithm "nonlinear" (Algorithm 2 + `solve_adjoint_varying`,
    eps = 1e-9, DOPRI5 at rtol 1e-10, Leja) against the restatement (RK4 with the iterate linearly
    interpolated, Chebyshev actions, node trapezoid): agreement at the discretisations' level, and
    the iterated trajectory converges to the serial sweep's (Algorithm 2's fixed point)."""
    from oracle.config_mode import burgers2d_nonlinear_tracking, burgers_direct_law, burgers_ops
    gd = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_nonlinear2d_tracking.npz"))
    nx, ny, T, D, w, P = int(gd["nx"]), int(gd["ny"]), float(gd["T"]), float(gd["D"]), float(gd["omega"]), int(gd["N"])
    law = TimeLaw.sine(w).as_tuple()
    grid = Grid(nx, ny)
    nsteps = 125
    S = P * nsteps
    h = T / S
    offs = np.arange(P + 1) * nsteps
    rhs, _, n2 = burgers_ops(nx, D, ny)
    tgt = burgers_direct_law(np.zeros((1, n2)), gd["f_true"][None, :], law, D, grid.hx, h, S, rhs=rhs)[:, 0, :]
    r = burgers2d_nonlinear_tracking(nx, ny, D, T, P, nsteps, np.zeros(n2), gd["f"], law, tgt,
                                     _nl_plans(grid, D, T / P, h, w), _plans_for(grid, D, offs, h, w), eps=1e-10)
    assert abs(r.J[0] - gd["J"]) <= 2e-6 * abs(gd["J"])
    assert rel_l2(r.grad[0], gd["grad"]) <= 1e-5
    assert rel_l2(r.qdag0[0], gd["qdag0"]) <= 1e-5
    assert rel_l2(r.uT[0], gd["uT"]) <= 1e-6
    assert 2 <= r.extras["sweeps"] <= 12 and r.extras["history"][-1] < 1e-10
    serial = burgers_direct_law(np.zeros((1, n2)), gd["f"][None, :], law, D, grid.hx, h, S, rhs=rhs)
    assert rel_l2(r.extras["traj"][-1], serial[-1]) <= 1e-6   # second order in h (interpolated iterate)
