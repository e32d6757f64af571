"""GPU parity of the reference's hybrid loop on its own 2D two-field Burgers testbed
(px_hybrid_* with desc.ny > 1, csrc/hybrid2d.cu) against the oracle restatement (pinned to the
reference's loop by tests/test_hybrid2d_cpu.py) and against the reference's golden numbers."""

import os

import numpy as np
import pytest

from tests.conftest import ROOT, rel_l2

pytestmark = pytest.mark.gpu


def _case(nx=48, ny=40, T=0.4, D=0.02, dt=1e-3, B=2, law=None, seed=3):
    from paper_2004_00546_b200 import ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system
    from paper_2004_00546_b200.problems import BURGERS
    law = law or TimeLaw.sine(2 * np.pi)
    sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), D, T))
    X, Y = sysm.grid.coordinates()
    rng = np.random.default_rng(seed)
    u0 = np.concatenate([0.4 * np.sin(X) * np.cos(Y) + 0.05 * np.cos(3 * X), 0.3 * np.cos(X) * np.sin(Y)])
    f = np.stack([np.concatenate([0.3 * np.cos((b + 1) * X) * np.sin(Y) + 0.2 * np.sin(2 * X),
                                  0.25 * np.sin(X) * np.sin((b + 1) * Y) - 0.1 * np.cos(X + Y)])
                  + 0.02 * rng.standard_normal(2 * nx * ny) for b in range(B)])
    f_true = np.concatenate([0.5 * np.sin(X) * np.sin(Y) + 0.1 * np.cos(2 * X), 0.3 * np.sin(X) * np.sin(Y)])
    return sysm, u0, f, f_true, RK4Config(dt), ChebyshevConfig(tol=1e-12), law


def _oracle(sysm, u0, f, target, offs, law, cfg, qdag_T=None):
    from oracle.config_mode import burgers_tracking_hybrid
    from paper_2004_00546_b200.expaction import plan_family
    from paper_2004_00546_b200.problems import frozen_bounds_2d, frozen_region_from_bounds
    T = sysm.spec.T
    h = T / offs[-1]

    def plans_for(ubar):
        reg = frozen_region_from_bounds(*frozen_bounds_2d(ubar, sysm.grid, sysm.spec.D))
        return plan_family(reg, [(offs[p + 1] - offs[p]) * h for p in range(len(offs) - 1)], cfg, omega=law.omega)

    return burgers_tracking_hybrid(sysm.grid.nx, sysm.spec.D, T, offs, u0, f, law.as_tuple(), target, plans_for,
                                   qdag_T=qdag_T, ny=sysm.grid.ny)


@pytest.fixture
def per_stage_launches(monkeypatch):
    """Force the per-stage-launch kernels on a small grid (handles read PX_HYB2D_ONCHIP at create)."""
    from paper_2004_00546_b200.tracking import release_tracking_engines
    release_tracking_engines()
    monkeypatch.setenv("PX_HYB2D_ONCHIP", "0")
    yield
    release_tracking_engines()


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("grid", [(48, 40), (64, 48)])   # on-chip kernels (≤ 2048 points) / per-stage launches
def test_hybrid2d_tracking_vs_oracle(cuda_ok, overlap, grid):
    """Geometric partition (6 slices), sine law, two members, both fields active: J, ∂L/∂f,
    q†(0), u(T), the slice means and the slice adjoint ends against the oracle."""
    from paper_2004_00546_b200 import make_hybrid_plan, solve_hybrid_tracking, synthesize_trajectory
    from paper_2004_00546_b200 import _native as N
    from paper_2004_00546_b200.tracking import get_tracking_engine
    sysm, u0, f, f_true, rk, cfg, law = _case(nx=grid[0], ny=grid[1])
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    plan = make_hybrid_plan(sysm.spec.T, 6, 1.5)
    r = solve_hybrid_tracking(sysm, u0, f, target, plan, rk=rk, expaction=cfg, law=law, overlap=overlap)
    o = _oracle(sysm, u0, f, target, r.offsets, law, cfg)
    assert np.max(np.abs(r.J - o.J) / np.abs(o.J)) <= 1e-10
    assert rel_l2(r.final_state, o.uT) <= 1e-10
    for b in range(2):
        assert rel_l2(r.grad[b], o.grad[b]) <= 1e-8
        assert rel_l2(r.qdag0[b], o.qdag0[b]) <= 1e-10
    assert r.timing["overlapped"] == overlap
    eng = get_tracking_engine(sysm, r.offsets, law, 2, False)
    P, n2 = len(r.offsets) - 1, sysm.n
    assert rel_l2(eng.get(N.PX_HFIELD_UBAR, (P, 2, n2)), o.extras["ubar"]) <= 1e-12
    assert rel_l2(eng.get(N.PX_HFIELD_AEND, (2, P, n2)), np.swapaxes(o.extras["a_end"], 0, 1)) <= 1e-10
    n = sysm.grid.npoints
    assert np.linalg.norm(r.grad[0][n:]) > 1e-2 * np.linalg.norm(r.grad[0])  # the V block is active


def test_hybrid2d_terminal_data_mixed_law_per_member_target(cuda_ok):
    """Non-zero q†_T (the final span, hybrid.py:232-233), a mixed law α + β sin + γ cos,
    equidistant slices, a per-member target, a non-square grid with odd sizes."""
    from paper_2004_00546_b200 import TimeLaw, solve_hybrid_tracking, synthesize_trajectory
    law = TimeLaw(0.4, 0.7, -0.3, 3.0)
    sysm, u0, f, f_true, rk, cfg, _ = _case(nx=33, ny=21, law=law)
    tg = synthesize_trajectory(sysm, np.stack([f_true, 0.5 * f_true]), rk, law)   # (S+1, 2, 2n)
    X, Y = sysm.grid.coordinates()
    qT = 0.1 * np.stack([np.concatenate([np.sin(X), np.cos(Y)]), np.concatenate([np.cos(2 * X) * np.sin(Y), np.sin(X + Y)])])
    r = solve_hybrid_tracking(sysm, u0, f, tg, None, N=5, rk=rk, expaction=cfg, law=law, qdag_T=qT)
    o = _oracle(sysm, u0, f, tg, r.offsets, law, cfg, qdag_T=qT)
    assert np.max(np.abs(r.J - o.J) / np.abs(o.J)) <= 1e-10
    assert rel_l2(r.grad, o.grad) <= 1e-8
    assert rel_l2(r.qdag0, o.qdag0) <= 1e-10


def test_hybrid2d_reduces_to_the_1d_path(cuda_ok):
    """A y-invariant U with V ≡ 0 on the 2D two-field path equals the 1D path's numbers (the
    reference's embedding of 1D Burgers): J per row, the gradient rows, V-gradient zero."""
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system, build_system,
        make_hybrid_plan, solve_hybrid_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.problems import BURGERS
    nx, ny, T, D = 64, 5, 0.3, 0.02
    law, rk, cfg = TimeLaw.sine(5.0), RK4Config(1e-3), ChebyshevConfig(tol=1e-12)
    spec = ProblemSpec(BURGERS, (0.0, 0.0), D, T)
    s1, s2 = build_system(Grid(nx), spec, 2), build_burgers2d_system(Grid(nx, ny), spec)
    x = s1.grid.x1()
    emb = lambda u: np.concatenate([np.tile(u, ny), np.zeros(nx * ny)])
    u0, f, ft = 0.5 * np.sin(x), 0.3 * np.cos(2 * x) + 0.2 * np.sin(x), 0.4 * np.sin(x) + 0.1 * np.cos(3 * x)
    plan = make_hybrid_plan(T, 4, 2.0)
    t1 = synthesize_trajectory(s1, ft, rk, law)[:, 0, :]
    t2 = synthesize_trajectory(s2, emb(ft), rk, law)[:, 0, :]
    assert rel_l2(t2[:, :nx], t1) <= 1e-12 and np.all(t2[:, nx * ny:] == 0.0)
    r1 = solve_hybrid_tracking(s1, u0, f, t1, plan, rk=rk, expaction=cfg, law=law)
    r2 = solve_hybrid_tracking(s2, emb(u0), emb(f), t2, plan, rk=rk, expaction=cfg, law=law)
    assert abs(r2.J[0] - ny * r1.J[0]) <= 1e-11 * abs(r2.J[0])
    assert rel_l2(r2.grad[0][: nx * ny].reshape(ny, nx), np.tile(r1.grad[0], (ny, 1))) <= 1e-9
    assert np.max(np.abs(r2.grad[0][nx * ny:])) <= 1e-13
    assert rel_l2(r2.qdag0[0][:nx], r1.qdag0[0]) <= 1e-9


def test_hybrid2d_against_the_reference_golden_and_binding(cuda_ok):
    """The reference's own 2D two-field hybrid-loop case (tests/golden/reference_hybrid2d_tracking
    .npz) on the GPU, directly and through the reference-side binding driven with stand-ins shaped
    like the reference's objects (the reference itself is not on the GPU box)."""
    from types import SimpleNamespace

    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system, make_hybrid_plan,
        solve_hybrid_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.integration import direct_adjoint_loop
    from paper_2004_00546_b200.problems import BURGERS
    gd = np.load(os.path.join(ROOT, "tests", "golden", "reference_hybrid2d_tracking.npz"))
    nx, ny, T, D, w = int(gd["nx"]), int(gd["ny"]), float(gd["T"]), float(gd["D"]), float(gd["omega"])
    sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), D, T))
    law, rk = TimeLaw.sine(w), RK4Config(1e-3)
    target = synthesize_trajectory(sysm, gd["f_true"], rk, law)[:, 0, :]
    r = solve_hybrid_tracking(sysm, np.zeros(sysm.n), gd["f"], target,
                              make_hybrid_plan(T, int(gd["N"]), float(gd["k"])), rk=rk,
                              expaction=ChebyshevConfig(tol=1e-12), law=law)
    assert abs(r.J[0] - gd["J"]) <= 1e-6 * abs(gd["J"])
    assert rel_l2(r.grad[0], gd["grad"]) <= 1e-5
    assert rel_l2(r.qdag0[0], gd["qdag0"]) <= 1e-6
    assert rel_l2(r.final_state[0], gd["uT"]) <= 1e-9

    def ref_system(f):
        spec = SimpleNamespace(kind="burgers", a=0.0, D=D, omega=w, T=T, f_spatial=f)
        return SimpleNamespace(grid=SimpleNamespace(nx=nx, ny=ny), spec=spec,
                               with_forcing_field=lambda g: ref_system(np.asarray(g)))

    nodes = np.linspace(0.0, T, target.shape[0])
    q_true = SimpleNamespace(eval_many=lambda ts: np.stack(
        [np.array([np.interp(t, nodes, target[:, i]) for i in range(sysm.n)]) for t in ts]))
    plan = SimpleNamespace(N=int(gd["N"]), k=float(gd["k"]))
    rb = direct_adjoint_loop(ref_system(np.zeros(sysm.n)), gd["f"], q_true, "hybrid", N=3, plan=plan, dt=1e-3)
    assert abs(rb.J - gd["J"]) <= 1e-6 * abs(gd["J"]) and rb.grad.shape == (sysm.n,)
    assert rel_l2(rb.grad, gd["grad"]) <= 1e-5
    # the same binding with the reference's algorithm "nonlinear" (its golden numbers: the nonlinear loop's)
    gn = np.load(os.path.join(ROOT, "tests", "golden", "reference_nonlinear2d_tracking.npz"))
    rn = direct_adjoint_loop(ref_system(np.zeros(sysm.n)), gn["f"], q_true, "nonlinear", N=int(gn["N"]), eps=1e-9, dt=1e-3)
    assert abs(rn.J - gn["J"]) <= 2e-6 * abs(gn["J"]) and rel_l2(rn.grad, gn["grad"]) <= 1e-5
    assert rn.cuda.iterations == int(gn["iterations"])


def test_hybrid2d_reference_config_size_and_overlap(cuda_ok):
    """The reference's `configs/burgers_hybrid.json` shape (32×32, D = 1, ω = 1, T = 1, forcing
    sin x·sin y on both fields from f_init = ones) on 16 geometric slices: the stream-level overlap
    gives the same numbers as the sequential run, the loop API returns them, NaN input is refused."""
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system, direct_adjoint_loop,
        make_hybrid_plan, solve_hybrid_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.errors import IntegrationFailure
    from paper_2004_00546_b200.problems import BURGERS
    nx = ny = 32
    sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), 1.0, 1.0))
    X, Y = sysm.grid.coordinates()
    f_true = np.concatenate([np.sin(X) * np.sin(Y)] * 2)
    f = np.ones(sysm.n)
    law, rk, cfg = TimeLaw.sine(1.0), RK4Config(1e-3), ChebyshevConfig(tol=1e-12)
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    plan = make_hybrid_plan(1.0, 16, 3.0)
    seq = solve_hybrid_tracking(sysm, np.zeros(sysm.n), f, target, plan, rk=rk, expaction=cfg, law=law, overlap=False)
    ovl = solve_hybrid_tracking(sysm, np.zeros(sysm.n), f, target, plan, rk=rk, expaction=cfg, law=law, overlap=True)
    assert ovl.timing["overlapped"] and not seq.timing["overlapped"]
    assert np.array_equal(seq.grad, ovl.grad) and np.array_equal(seq.J, ovl.J) and np.array_equal(seq.qdag0, ovl.qdag0)
    o = _oracle(sysm, np.zeros(sysm.n), f[None, :], target, ovl.offsets, law, cfg)
    assert abs(ovl.J[0] - o.J[0]) <= 1e-10 * abs(o.J[0]) and rel_l2(ovl.grad, o.grad) <= 1e-8
    loop = direct_adjoint_loop(sysm, f, target, "hybrid", rk=rk, expaction=cfg, objective="tracking", plan=plan,
                               time_law=law)
    assert loop.J == pytest.approx(float(ovl.J[0]), rel=1e-14) and np.array_equal(loop.grad, ovl.grad[0])
    bad = f.copy()
    bad[7] = np.nan
    with pytest.raises((IntegrationFailure, FloatingPointError, ValueError)):
        solve_hybrid_tracking(sysm, np.zeros(sysm.n), bad, target, plan, rk=rk, expaction=cfg, law=law)


def test_hybrid2d_on_chip_equals_per_stage_launches(cuda_ok, per_stage_launches):
    """The same small case through the per-stage-launch kernels (PX_HYB2D_ONCHIP=0) against the
    oracle, with terminal data and a mixed law (the on-chip run of it is the test above)."""
    from paper_2004_00546_b200 import TimeLaw, make_hybrid_plan, solve_hybrid_tracking, synthesize_trajectory
    law = TimeLaw(0.4, 0.7, -0.3, 3.0)
    sysm, u0, f, f_true, rk, cfg, _ = _case(nx=33, ny=21, law=law)
    tg = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    X, Y = sysm.grid.coordinates()
    qT = 0.1 * np.concatenate([np.sin(X), np.cos(Y)])
    for ov in (False, True):
        r = solve_hybrid_tracking(sysm, u0, f, tg, make_hybrid_plan(sysm.spec.T, 5, 2.0), rk=rk, expaction=cfg, law=law,
                                  qdag_T=qT, overlap=ov)
        assert r.timing["overlapped"] == ov
        o = _oracle(sysm, u0, f, tg, r.offsets, law, cfg, qdag_T=qT)
        assert np.max(np.abs(r.J - o.J) / np.abs(o.J)) <= 1e-10
        assert rel_l2(r.grad, o.grad) <= 1e-8 and rel_l2(r.qdag0, o.qdag0) <= 1e-10


def _nl_oracle(sysm, u0, f, target, P, nsteps, law, cfg, eps):
    from oracle.config_mode import burgers2d_nonlinear_tracking
    from paper_2004_00546_b200.expaction import plan_chebyshev, plan_family
    from paper_2004_00546_b200.problems import frozen_bounds_2d, frozen_region_from_bounds
    T, D, g = sysm.spec.T, sysm.spec.D, sysm.grid
    h = T / (P * nsteps)

    def plans_nl(qbar):
        reg = frozen_region_from_bounds(*frozen_bounds_2d(qbar, g, D))
        return plan_chebyshev(reg, T / P, cfg), plan_chebyshev(reg, h, cfg)

    def plans_adj(ubar):
        reg = frozen_region_from_bounds(*frozen_bounds_2d(ubar, g, D))
        return plan_family(reg, [T / P] * P, cfg, omega=law.omega)

    return burgers2d_nonlinear_tracking(g.nx, g.ny, D, T, P, nsteps, u0, f, law.as_tuple(), target, plans_nl, plans_adj,
                                        eps)


def test_nonlinear2d_loop_vs_oracle(cuda_ok):
    """Algorithm 2 on the two-field testbed (px_hybrid_nl_*) + the zero-terminal adjoint: sweeps, error
    history, J, ∂L/∂f, q†(0), u(T) against the oracle; two members; through the loop API."""
    from paper_2004_00546_b200 import direct_adjoint_loop, solve_nonlinear_tracking, synthesize_trajectory
    sysm, u0, f, f_true, rk, cfg, law = _case(nx=24, ny=20, T=0.3, dt=1.5e-3)
    P, nsteps = 4, 50
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    r = solve_nonlinear_tracking(sysm, u0, f, target, N=P, rk=rk, expaction=cfg, law=law, eps=1e-10)
    o = _nl_oracle(sysm, u0, f, target, P, nsteps, law, cfg, 1e-10)
    hist = r.timing["history"]
    assert len(hist) == o.extras["sweeps"]
    for a, b in zip(hist[:-1], o.extras["history"][:-1]):
        assert abs(a - b) <= 1e-6 * abs(b)
    assert np.max(np.abs(r.J - o.J) / np.abs(o.J)) <= 1e-10
    assert rel_l2(r.final_state, o.uT) <= 1e-10
    assert rel_l2(r.grad, o.grad) <= 1e-8 and rel_l2(r.qdag0, o.qdag0) <= 1e-10
    loop = direct_adjoint_loop(sysm, f[0], target, "nonlinear", N=P, rk=rk, expaction=cfg, u0=u0,
                               objective="tracking", time_law=law, eps=1e-10)
    assert loop.iterations == len(hist) and loop.J == pytest.approx(float(r.J[0]), rel=1e-13)
    assert rel_l2(loop.grad, r.grad[0]) <= 1e-12 and len(loop.error_history) == loop.iterations


def test_nonlinear2d_against_the_reference_golden_and_limits(cuda_ok):
    """The reference's own nonlinear-loop case (tests/golden/reference_nonlinear2d_tracking.npz) on the
    GPU; a loose eps stops early; too few sweeps allowed raises IterationDivergence."""
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system, solve_nonlinear_tracking,
        synthesize_trajectory)
    from paper_2004_00546_b200.errors import IterationDivergence
    from paper_2004_00546_b200.problems import BURGERS
    gd = np.load(os.path.join(ROOT, "tests", "golden", "reference_nonlinear2d_tracking.npz"))
    nx, ny, T, D, w, P = int(gd["nx"]), int(gd["ny"]), float(gd["T"]), float(gd["D"]), float(gd["omega"]), int(gd["N"])
    sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), D, T))
    law, rk, cfg = TimeLaw.sine(w), RK4Config(T / (P * 125)), ChebyshevConfig(tol=1e-12)
    target = synthesize_trajectory(sysm, gd["f_true"], rk, law)[:, 0, :]
    r = solve_nonlinear_tracking(sysm, np.zeros(sysm.n), gd["f"], target, N=P, rk=rk, expaction=cfg, law=law, eps=1e-10)
    assert abs(r.J[0] - gd["J"]) <= 2e-6 * abs(gd["J"])
    assert rel_l2(r.grad[0], gd["grad"]) <= 1e-5
    assert rel_l2(r.qdag0[0], gd["qdag0"]) <= 1e-5
    assert len(r.timing["history"]) == int(gd["iterations"])   # the reference needed the same number of sweeps
    loose = solve_nonlinear_tracking(sysm, np.zeros(sysm.n), gd["f"], target, N=P, rk=rk, expaction=cfg, law=law, eps=1e-2)
    assert len(loose.timing["history"]) < len(r.timing["history"])
    with pytest.raises(IterationDivergence):
        solve_nonlinear_tracking(sysm, np.zeros(sysm.n), gd["f"], target, N=P, rk=rk, expaction=cfg, law=law,
                                 eps=1e-12, max_iter=2)


@pytest.mark.parametrize("grid", [(24, 20), (64, 48)])
def test_nonlinear2d_per_stage_launches_vs_oracle(cuda_ok, per_stage_launches, grid):
    """Algorithm 2 through the per-stage-launch kernels (forced on a small grid, and a grid above the
    on-chip limit): the same sweeps and numbers as the oracle."""
    from paper_2004_00546_b200 import solve_nonlinear_tracking, synthesize_trajectory
    sysm, u0, f, f_true, rk, cfg, law = _case(nx=grid[0], ny=grid[1], T=0.24, dt=1.5e-3, B=2 if grid[0] < 32 else 1)
    P, nsteps = 4, 40
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    r = solve_nonlinear_tracking(sysm, u0, f, target, N=P, rk=rk, expaction=cfg, law=law, eps=1e-10)
    o = _nl_oracle(sysm, u0, f, target, P, nsteps, law, cfg, 1e-10)
    assert len(r.timing["history"]) == o.extras["sweeps"]
    assert np.max(np.abs(r.J - o.J) / np.abs(o.J)) <= 1e-10
    assert rel_l2(r.final_state, o.uT) <= 1e-10
    assert rel_l2(r.grad, o.grad) <= 1e-8 and rel_l2(r.qdag0, o.qdag0) <= 1e-10


@pytest.mark.parametrize("two_d", [False, True])
def test_checkpointed_hybrid_tracking_equals_the_plain_loop(cuda_ok, two_d):
    """`run_checkpointed_tracking` (the reference's checkpointed loop, hybrid algorithm): M = 0 is the
    plain loop; M = 1 with N equal slices per segment equals the plain hybrid loop on 2N equal slices
    (same serial sweep from the checkpoint, same frozen operators and carries; the terminal data of the
    first segment is the second's q†) up to the exp-action truncation; memory peaks at one segment."""
    from paper_2004_00546_b200 import (
        CheckpointSchedule, ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system,
        build_system, run_checkpointed_tracking, solve_hybrid_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.problems import BURGERS
    T, D, S, N = 0.4, 0.02, 400, 3
    law, rk, cfg = TimeLaw(0.2, 0.8, -0.3, 4.0), RK4Config(T / S), ChebyshevConfig(tol=1e-13)
    spec = ProblemSpec(BURGERS, (0.0, 0.0), D, T)
    if two_d:
        sysm = build_burgers2d_system(Grid(20, 18), spec)
        X, Y = sysm.grid.coordinates()
        f = np.concatenate([0.3 * np.cos(X) * np.sin(Y), 0.2 * np.sin(X + Y)])
        ft = np.concatenate([0.5 * np.sin(X) * np.sin(Y), 0.1 * np.cos(Y)])
        u0 = np.concatenate([0.2 * np.sin(X), 0.1 * np.cos(X - Y)])
    else:
        sysm = build_system(Grid(128), spec, 2)
        x = sysm.grid.x1()
        f, ft, u0 = 0.3 * np.cos(2 * x) + 0.2 * np.sin(x), 0.4 * np.sin(x) + 0.1 * np.cos(3 * x), 0.5 * np.sin(x)
    target = synthesize_trajectory(sysm, ft, rk, law, u0=u0)[:, 0, :]
    plain = solve_hybrid_tracking(sysm, u0, f, target, None, N=2 * N, rk=rk, expaction=cfg, law=law)
    c0 = run_checkpointed_tracking(sysm, f, target, CheckpointSchedule(T, 0), N=2 * N, rk=rk, expaction=cfg, law=law, u0=u0)
    assert c0.cost == pytest.approx(float(plain.J[0]), rel=1e-13) and rel_l2(c0.gradient, plain.grad[0]) <= 1e-13
    c1 = run_checkpointed_tracking(sysm, f, target, CheckpointSchedule(T, 1), N=N, rk=rk, expaction=cfg, law=law, u0=u0)
    assert c1.cost == pytest.approx(float(plain.J[0]), rel=1e-12)
    assert rel_l2(c1.final_state, plain.final_state[0]) <= 1e-13
    assert rel_l2(c1.gradient, plain.grad[0]) <= 1e-9 and rel_l2(c1.qdag0, plain.qdag0[0]) <= 1e-9
    assert c1.memory.peak == S // 2 + 1 and len(c1.checkpoint_states) == 2
    assert rel_l2(c1.checkpoint_states[1], target[0] * 0 + synthesize_trajectory(sysm, f, rk, law, u0=u0)[S // 2, 0]) <= 1e-13


def test_serial2d_gradient_vs_finite_differences_on_the_device(cuda_ok):
    """Independent of the oracle: the serial (one-slice) loop's ∂L/∂f on the 2D testbed against central
    differences of the device's own J in a random direction of both components (second order in h)."""
    from paper_2004_00546_b200 import direct_adjoint_loop, synthesize_trajectory
    sysm, u0, f, f_true, rk, cfg, law = _case(nx=32, ny=32, T=0.3, dt=1e-3, B=1)
    target = synthesize_trajectory(sysm, f_true, rk, law, u0=u0)[:, 0, :]
    run = lambda ff: direct_adjoint_loop(sysm, ff, target, "serial", rk=rk, expaction=cfg, u0=u0, objective="tracking",
                                         time_law=law)
    r = run(f[0])
    d = np.random.default_rng(11).standard_normal(sysm.n)
    eps = 1e-5
    fd = (run(f[0] + eps * d).J - run(f[0] - eps * d).J) / (2 * eps)
    assert abs(fd - float(r.grad @ d)) <= 2e-4 * abs(fd)
