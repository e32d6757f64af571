"""GPU parity of the reference's hybrid with its tracking objective (px_hybrid_*, SURVEY §8(f)
rank 2) against the oracle restatement (pinned to the reference's own loop by
tests/test_hybrid_cpu.py) and, on the golden case, against the reference's numbers directly."""

import os

import numpy as np
import pytest

from tests.conftest import ROOT, rel_l2

pytestmark = pytest.mark.gpu


def _case(nx=256, T=0.5, D=0.01, dt=1e-3, P=8, k=1.5, B=2, law=None, batched_target=False, seed=5):
    from paper_2004_00546_b200 import ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_system
    from paper_2004_00546_b200.problems import BURGERS
    law = law or TimeLaw.sine(2 * np.pi)
    sysm = build_system(Grid(nx), ProblemSpec(BURGERS, (0.0, 0.0), D, T), 8)
    x = sysm.grid.x1()
    rng = np.random.default_rng(seed)
    u0 = 0.5 * np.sin(x) + 0.05 * np.cos(3 * x)
    f = np.stack([0.3 * np.cos((b + 2) * x) + 0.2 * np.sin(3 * x) + 0.02 * rng.standard_normal(nx)
                  for b in range(B)])
    f_true = 0.5 * np.sin(x) + 0.1 * np.cos(2 * x)
    return sysm, u0, f, f_true, RK4Config(dt), ChebyshevConfig(tol=1e-12), law


def _oracle(sysm, u0, f, target, offs, law, cfg, qdag_T=None):
    from oracle.config_mode import burgers_tracking_hybrid
    from paper_2004_00546_b200.expaction import plan_family
    from paper_2004_00546_b200.problems import frozen_bounds, frozen_region_from_bounds
    T = sysm.spec.T
    h = T / offs[-1]

    def plans_for(ubar):
        reg = frozen_region_from_bounds(*frozen_bounds(ubar, sysm.grid, sysm.spec.D))
        return plan_family(reg, [(offs[p + 1] - offs[p]) * h for p in range(len(offs) - 1)], cfg, omega=law.omega)

    return burgers_tracking_hybrid(sysm.grid.nx, sysm.spec.D, T, offs, u0, f, law.as_tuple(), target, plans_for,
                                   qdag_T=qdag_T)


@pytest.mark.parametrize("overlap", [True, False])
def test_hybrid_tracking_vs_oracle(cuda_ok, overlap):
    """Geometric partition (8 slices), sine law, two members: J, ∂L/∂f, q†(0), u(T) vs the oracle."""
    from paper_2004_00546_b200 import make_hybrid_plan, solve_hybrid_tracking, synthesize_trajectory
    sysm, u0, f, f_true, rk, cfg, law = _case()
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    plan = make_hybrid_plan(sysm.spec.T, 8, 1.5)
    r = solve_hybrid_tracking(sysm, u0, f, target, plan, rk=rk, expaction=cfg, law=law, overlap=overlap)
    o = _oracle(sysm, u0, f, target, r.offsets, law, cfg)
    assert np.max(np.abs(r.J - o.J) / np.abs(o.J)) <= 1e-10
    assert rel_l2(r.final_state, o.uT) <= 1e-10
    for b in range(2):
        assert rel_l2(r.grad[b], o.grad[b]) <= 1e-8
        assert rel_l2(r.qdag0[b], o.qdag0[b]) <= 1e-10
    assert r.timing["overlapped"] == overlap


def test_hybrid_tracking_terminal_data_and_cosine_law(cuda_ok):
    """Non-zero q†_T (the final span, hybrid.py:232-233), a mixed law α + β sin + γ cos,
    equidistant slices and a per-member target."""
    from paper_2004_00546_b200 import TimeLaw, solve_hybrid_tracking, synthesize_trajectory
    law = TimeLaw(0.4, 0.7, -0.3, 3.0)
    sysm, u0, f, f_true, rk, cfg, _ = _case(nx=128, P=5, law=law)
    tg = synthesize_trajectory(sysm, np.stack([f_true, 0.5 * f_true]), rk, law)   # (S+1, 2, n)
    qT = 0.1 * np.stack([np.sin(sysm.grid.x1()), np.cos(2 * sysm.grid.x1())])
    r = solve_hybrid_tracking(sysm, u0, f, tg, None, N=5, rk=rk, expaction=cfg, law=law, qdag_T=qT)
    o = _oracle(sysm, u0, f, tg, r.offsets, law, cfg, qdag_T=qT)
    assert np.max(np.abs(r.J - o.J) / np.abs(o.J)) <= 1e-10
    assert rel_l2(r.grad, o.grad) <= 1e-8
    assert rel_l2(r.qdag0, o.qdag0) <= 1e-10


def test_hybrid_tracking_against_the_reference_golden(cuda_ok):
    """The GPU path on the reference's own hybrid-loop case (tests/golden/reference_hybrid_tracking
    .npz): J and the gradient within the two discretisations' difference (the oracle is held to
    the same numbers on the CPU)."""
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_system, make_hybrid_plan,
        solve_hybrid_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.problems import BURGERS
    gd = np.load(os.path.join(ROOT, "tests", "golden", "reference_hybrid_tracking.npz"))
    nx, T, D, w = int(gd["nx"]), float(gd["T"]), float(gd["D"]), float(gd["omega"])
    sysm = build_system(Grid(nx), ProblemSpec(BURGERS, (0.0, 0.0), D, T), 4)
    law, rk = TimeLaw.sine(w), RK4Config(1e-3)
    target = synthesize_trajectory(sysm, gd["f_true"], rk, law)[:, 0, :]
    r = solve_hybrid_tracking(sysm, np.zeros(nx), gd["f"], target, make_hybrid_plan(T, int(gd["N"]), float(gd["k"])),
                              rk=rk, expaction=ChebyshevConfig(tol=1e-12), law=law)
    assert abs(r.J[0] - gd["J"] / 3) <= 1e-6 * abs(gd["J"] / 3)
    assert rel_l2(r.grad[0], gd["grad_rows"][0]) <= 1e-5
    assert rel_l2(r.qdag0[0], gd["qdag0"]) <= 1e-6


def test_hybrid_overlap_full_config3_size(cuda_ok):
    """Config 3's grid and steps (2048 points, 2000 steps) on a 64-slice geometric partition: the
    slice solves run during the serial sweep (only a tail remains after it), and the overlapped
    and sequential runs are bitwise identical."""
    from paper_2004_00546_b200 import (
        ChebyshevConfig, make_hybrid_plan, solve_hybrid_tracking, synthesize_trajectory)
    sysm, u0, f, f_true, rk, cfg, law = _case(nx=2048, T=1.0, D=0.005, dt=5e-4, B=1)
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    plan = make_hybrid_plan(1.0, 64, 20.0)
    runs = {}
    for ov in (False, True, True):
        runs[ov] = solve_hybrid_tracking(sysm, u0, f, target, plan, rk=rk, expaction=cfg, law=law, overlap=ov)
    seq, ovl = runs[False], runs[True]
    assert ovl.timing["overlapped"] and not seq.timing["overlapped"]
    assert np.array_equal(seq.grad, ovl.grad) and np.array_equal(seq.J, ovl.J)
    assert np.array_equal(seq.qdag0, ovl.qdag0)
    # the overlap hides the slice solves behind the serial sweep: what remains after it ends is
    # less than the sequential run's slice solves
    assert ovl.timing["tail_ms"] < 0.8 * seq.timing["slices_ms"]
    assert ovl.timing["total_ms"] < seq.timing["total_ms"]
    assert np.all(np.isfinite(ovl.grad))
    # one oracle comparison at full size (J and the gradient)
    o = _oracle(sysm, u0, f, target, ovl.offsets, law, cfg)
    assert abs(ovl.J[0] - o.J[0]) <= 1e-10 * abs(o.J[0])
    assert rel_l2(ovl.grad, o.grad) <= 1e-8


def test_tracking_loop_api_and_estimate_k(cuda_ok):
    """direct_adjoint_loop(objective="tracking") with mode coefficients and with a field; the
    serial algorithm is the one-slice case; estimate_k times the device pilot."""
    from paper_2004_00546_b200 import (
        direct_adjoint_loop, estimate_k, make_hybrid_plan, solve_hybrid_tracking, synthesize_trajectory)
    sysm, u0, f, f_true, rk, cfg, law = _case(nx=128, B=1)
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    plan = make_hybrid_plan(sysm.spec.T, 6, 2.0)
    loop = direct_adjoint_loop(sysm, f[0], target, "hybrid", rk=rk, expaction=cfg, u0=u0, objective="tracking",
                               plan=plan, time_law=law)
    ref = solve_hybrid_tracking(sysm, u0, f[0], target, plan, rk=rk, expaction=cfg, law=law)
    assert loop.J == pytest.approx(float(ref.J[0]), rel=1e-14) and np.allclose(loop.grad, ref.grad[0], rtol=0, atol=0)
    c = np.random.default_rng(1).standard_normal(sysm.basis.K) * 0.1
    lc = direct_adjoint_loop(sysm, c, target, "hybrid", rk=rk, expaction=cfg, u0=u0, objective="tracking",
                             plan=plan, time_law=law)
    lf = direct_adjoint_loop(sysm, sysm.basis.field(c[None, :])[0], target, "hybrid", rk=rk, expaction=cfg, u0=u0,
                             objective="tracking", plan=plan, time_law=law)
    assert lc.J == pytest.approx(lf.J, rel=1e-13)
    assert rel_l2(lc.grad, sysm.basis.project(lf.grad[None, :])[0]) <= 1e-12
    ser = direct_adjoint_loop(sysm, f[0], target, "serial", rk=rk, u0=u0, objective="tracking", time_law=law)
    o = _oracle(sysm, u0, f[:1], target, np.array([0, int(round(sysm.spec.T / rk.dt))]), law, cfg)
    assert ser.J == pytest.approx(float(o.J[0]), rel=1e-10) and rel_l2(ser.grad, o.grad[0]) <= 1e-8
    k = estimate_k(sysm, 0.1, rk, repeats=2, law=law)
    assert k > 1.0   # the adjoint slice step costs more than a direct step (test_hybrid.py:102-105)


def test_reference_binding_on_the_gpu(cuda_ok):
    """integration.direct_adjoint_loop — the call a reference maintainer wires behind
    backend="cuda" — driven with stand-ins shaped like the reference's objects (Grid2D,
    ProblemSpec, System.with_forcing_field, PiecewiseSolution.eval_many, HybridPlan; the reference
    itself is not on the GPU box) on the golden case: J and the embedded gradient equal the
    reference's own loop's numbers to the discretisations' difference."""
    from types import SimpleNamespace

    from paper_2004_00546_b200 import RK4Config, TimeLaw, synthesize_trajectory
    from paper_2004_00546_b200.integration import direct_adjoint_loop, system_from_reference
    gd = np.load(os.path.join(ROOT, "tests", "golden", "reference_hybrid_tracking.npz"))
    nx, T, D, w = int(gd["nx"]), float(gd["T"]), float(gd["D"]), float(gd["omega"])
    emb = lambda u: np.concatenate([np.tile(u, 3), np.zeros(3 * nx)])

    def ref_system(f):
        spec = SimpleNamespace(kind="burgers", a=0.0, D=D, omega=w, T=T, f_spatial=f)
        return SimpleNamespace(grid=SimpleNamespace(nx=nx, ny=3), spec=spec,
                               with_forcing_field=lambda g: ref_system(np.asarray(g)))

    sysm, _, _, _ = system_from_reference(ref_system(emb(np.zeros(nx))))
    traj = synthesize_trajectory(sysm, gd["f_true"], RK4Config(1e-3), TimeLaw.sine(w))[:, 0, :]
    nodes = np.linspace(0.0, T, traj.shape[0])
    q_true = SimpleNamespace(eval_many=lambda ts: np.stack(
        [emb(np.array([np.interp(t, nodes, traj[:, i]) for i in range(nx)])) for t in ts]))
    plan = SimpleNamespace(N=int(gd["N"]), k=float(gd["k"]))
    r = direct_adjoint_loop(ref_system(emb(np.zeros(nx))), emb(gd["f"]), q_true, "hybrid", N=3, plan=plan, dt=1e-3)
    assert abs(r.J - gd["J"]) <= 1e-6 * abs(gd["J"])
    assert r.grad.shape == (6 * nx,)
    assert rel_l2(r.grad[: 3 * nx].reshape(3, nx), gd["grad_rows"]) <= 1e-5
    assert np.all(r.grad[3 * nx:] == 0.0)


def test_hybrid_fallbacks_and_limits(cuda_ok):
    """More slice CTAs than SMs: the overlap is declined (a waiting CTA must never block the
    sweep) and the slices run after it, with the same numbers; a grid that fits neither the
    cluster nor the run layout is refused."""
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, TimeLaw, build_system, make_hybrid_plan, solve_hybrid_tracking,
        synthesize_trajectory)
    from paper_2004_00546_b200.problems import BURGERS
    sysm, u0, f, f_true, rk, cfg, law = _case(nx=96, P=64, B=3)
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    plan = make_hybrid_plan(sysm.spec.T, 64, 4.0)
    r = solve_hybrid_tracking(sysm, u0, f, target, plan, rk=rk, expaction=cfg, law=law, overlap=True)
    assert not r.timing["overlapped"]   # 3·64 slice CTAs + 3 sweep CTAs > 148 SMs
    o = _oracle(sysm, u0, f, target, r.offsets, law, cfg)
    assert np.max(np.abs(r.J - o.J) / np.abs(o.J)) <= 1e-10
    assert rel_l2(r.grad, o.grad) <= 1e-8 and rel_l2(r.qdag0, o.qdag0) <= 1e-10
    bad = build_system(Grid(3000), ProblemSpec(BURGERS, (0.0, 0.0), 0.01, 0.1), 2)
    with pytest.raises(ValueError):
        solve_hybrid_tracking(bad, np.zeros(3000), np.zeros(3000), np.zeros((101, 3000)), None, N=2,
                              rk=rk, law=TimeLaw.constant())
