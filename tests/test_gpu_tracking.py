"""GPU parity of the linear testbed's tracking objective — the reference's linear loop
(`optimization.py:154-231`, algorithm "linear": J = (1/T)∫‖u − u_t‖² dt, the adjoint source
2(u − u_t), q†(T) = 0, ∂L/∂f = (1/T)∫θ·q† dt) through `px_set_tracking_target` — against the
oracle (oracle.config_mode.linear_tracking_gradient) and the reference's own numbers
(tests/golden/reference_linear_tracking.npz)."""

import os

import numpy as np
import pytest

from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle(system, c, u0, ctrl, law, target, tol=1e-13):
    from oracle.config_mode import linear_tracking_gradient
    from paper_2004_00546_b200.expaction import ChebyshevConfig, plan_chebyshev
    pl = plan_chebyshev(system.region(), c.spec.T / c.P, ChebyshevConfig(tol=tol), omega=law.omega) \
        if c.P > 1 else None   # one slice: no carries
    return linear_tracking_gradient(system.grid.nx, system.grid.ny, system.A.as_tuple(), system.basis, c.spec.T, c.P,
                                    c.nsteps, u0, ctrl, law.as_tuple(), target, pl)


def _target(n, S, B=None, seed=3):
    rng = np.random.default_rng(seed)
    t = np.linspace(0.0, 1.0, S + 1)
    shape = (S + 1, n) if B is None else (S + 1, B, n)
    base = 0.2 * rng.standard_normal(shape[1:])
    return np.sin(2.5 * t).reshape((S + 1,) + (1,) * (len(shape) - 1)) * base + 0.01 * rng.standard_normal(shape)


def _check(r, o, j_tol=1e-10, tol=1e-9):
    J = np.atleast_1d(r.J)
    assert np.max(np.abs(J - o.J) / np.abs(o.J)) <= j_tol
    assert rel_l2(np.atleast_2d(r.grad), o.grad) <= tol
    assert rel_l2(np.atleast_2d(np.asarray(r.direct.final_state)), o.uT) <= tol
    assert rel_l2(np.atleast_2d(np.asarray(r.adjoint.initial_state)), o.qdag0) <= tol
    assert rel_l2(np.atleast_2d(np.asarray(r.adjoint.integral)), o.G) <= tol


def test_tracking_2d_field_control_sine_law(cuda_ok):
    """A full forcing field with the reference's f·sin(ωt): recording sweep from the Paraexp edge
    states, node trapezoid cost, adjoint lanes with the tracking source, Chebyshev carries with the
    per-carry law series; the recorded trajectory is the oracle's."""
    from paper_2004_00546_b200 import ChebyshevConfig, RK4Config, TimeLaw, baseline, direct_adjoint_loop, scaled
    from paper_2004_00546_b200.systems import build_field_system
    c = scaled(baseline(5), nx=32, P=6, steps_per_slice=5, K=8)
    fs = build_field_system(c.system.grid, c.system.spec)
    rng = np.random.default_rng(1)
    u0, f = 0.1 * rng.standard_normal(fs.n), rng.standard_normal(fs.n)
    law = TimeLaw.sine(5.0)
    tg = _target(fs.n, c.P * c.nsteps)
    r = direct_adjoint_loop(fs, f, tg, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0,
                            expaction=ChebyshevConfig(tol=1e-13), objective="tracking", time_law=law)
    o = _oracle(fs, c, u0, f, law, tg)
    _check(r, o)
    assert rel_l2(r.stats["trajectory"].numpy(), o.extras["traj"]) <= 1e-12
    assert rel_l2(np.asarray(r.direct.boundary_states), np.swapaxes(o.extras["edges"], 0, 1)) <= 1e-12


@pytest.mark.parametrize("law_kind", ["constant", "mixed"])
def test_tracking_2d_modes_batch_per_member_target(cuda_ok, law_kind):
    """Mode coefficients (the configs' basis), two members with their own targets, a constant and
    a mixed α + β sin + γ cos law; the constant law's carries take the summed-input φ₁ action."""
    from paper_2004_00546_b200 import ChebyshevConfig, RK4Config, TimeLaw, baseline, direct_adjoint_loop, scaled
    c = scaled(baseline(5), nx=48, P=8, steps_per_slice=4, K=16, batch=2)
    u0, _, ctrl = c.inputs()
    law = TimeLaw.constant() if law_kind == "constant" else TimeLaw(0.3, 1.0, -0.5, 7.0)
    tg = _target(c.system.n, c.P * c.nsteps, B=2)
    r = direct_adjoint_loop(c.system, ctrl, tg, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0,
                            expaction=ChebyshevConfig(tol=1e-13), objective="tracking", time_law=law)
    _check(r, _oracle(c.system, c, u0, ctrl, law, tg))


def test_tracking_1d_and_serial(cuda_ok):
    """The 1D testbed (config 1's grid, the generic carries) and the serial algorithm (one slice:
    the recording sweep from u0 is the serial RK4 trajectory)."""
    from paper_2004_00546_b200 import ChebyshevConfig, RK4Config, TimeLaw, baseline, direct_adjoint_loop, scaled
    c = scaled(baseline(1), P=8, steps_per_slice=10)
    u0, _, ctrl = c.inputs()
    law = TimeLaw.sine(3.0 * np.pi / c.spec.T)
    tg = _target(c.system.n, c.P * c.nsteps)
    cfg = ChebyshevConfig(tol=1e-13)
    r = direct_adjoint_loop(c.system, ctrl, tg, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0, expaction=cfg,
                            objective="tracking", time_law=law)
    _check(r, _oracle(c.system, c, u0, ctrl, law, tg))
    c1 = scaled(c, P=1, steps_per_slice=c.P * c.nsteps)
    s = direct_adjoint_loop(c.system, ctrl, tg, "serial", rk=RK4Config(c.dt), u0=u0, expaction=cfg,
                            objective="tracking", time_law=law)
    o1 = _oracle(c1.system, c1, u0, ctrl, law, tg)
    _check(s, o1)
    # the same problem on 8 slices and on one: the slices' edge states come from exact (Chebyshev)
    # propagation, the one-slice sweep's from RK4 — the gradients differ by that RK4 error only
    assert rel_l2(np.atleast_2d(r.grad), np.atleast_2d(s.grad)) <= 1e-6


def test_tracking_krylov_carries(cuda_ok):
    """Krylov (Arnoldi) carries with the time-constant law against the Chebyshev oracle."""
    from paper_2004_00546_b200 import KrylovConfig, RK4Config, TimeLaw, baseline, direct_adjoint_loop, scaled
    c = scaled(baseline(5), nx=32, P=4, steps_per_slice=5, K=8)
    u0, _, ctrl = c.inputs()
    tg = _target(c.system.n, c.P * c.nsteps)
    r = direct_adjoint_loop(c.system, ctrl, tg, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0,
                            expaction=KrylovConfig(m=30, tol=1e-13), objective="tracking")
    _check(r, _oracle(c.system, c, u0, ctrl, TimeLaw.constant(), tg), j_tol=1e-9, tol=1e-8)


def test_tracking_against_the_reference_golden(cuda_ok):
    """The GPU path on the reference's own linear-loop case (DOPRI5 + Leja, probe-grid
    trapezoids): the target is the GPU's own serial recording of f_true; J, the gradient and
    q†(0) within the discretisations' difference (the oracle meets the same bounds on the CPU)."""
    from paper_2004_00546_b200 import ChebyshevConfig, RK4Config, TimeLaw, direct_adjoint_loop, synthesize_trajectory
    from paper_2004_00546_b200.problems import ADVECTION_DIFFUSION, Grid, ProblemSpec
    from paper_2004_00546_b200.systems import build_field_system
    g = np.load(os.path.join(ROOT, "tests", "golden", "reference_linear_tracking.npz"))
    nx, ny, T, N = int(g["nx"]), int(g["ny"]), float(g["T"]), int(g["N"])
    fs = build_field_system(Grid(nx, ny), ProblemSpec(ADVECTION_DIFFUSION, (float(g["a"]),) * 2, float(g["D"]), T))
    law, rk = TimeLaw.sine(float(g["omega"])), RK4Config(T / 400)
    target = synthesize_trajectory(fs, g["f_true"], rk, law)[:, 0, :]
    r = direct_adjoint_loop(fs, g["f"], target, "linear", N=N, rk=rk, expaction=ChebyshevConfig(tol=1e-13),
                            objective="tracking", time_law=law)
    assert abs(r.J - g["J"]) <= 2e-5 * g["J"]
    assert rel_l2(r.grad, g["grad"]) <= 5e-6
    assert rel_l2(np.asarray(r.adjoint.initial_state), g["qdag0"]) <= 5e-6
    assert rel_l2(np.asarray(r.direct.final_state), g["uT"]) <= 2e-12


def test_reference_linear_binding_on_the_gpu(cuda_ok):
    """integration.direct_adjoint_loop on the linear testbed with stand-ins shaped like the
    reference's objects (Grid2D, ProblemSpec, System.with_forcing_field, PiecewiseSolution.
    eval_many): the reference's own loop's numbers (golden) to the discretisations' difference."""
    from types import SimpleNamespace

    from paper_2004_00546_b200 import RK4Config, TimeLaw, synthesize_trajectory
    from paper_2004_00546_b200.integration import direct_adjoint_loop, system_from_reference
    g = np.load(os.path.join(ROOT, "tests", "golden", "reference_linear_tracking.npz"))
    nx, ny, T, N, w = int(g["nx"]), int(g["ny"]), float(g["T"]), int(g["N"]), float(g["omega"])

    def ref_system(f):
        spec = SimpleNamespace(kind="advection_diffusion", a=float(g["a"]), D=float(g["D"]), omega=w, T=T,
                               f_spatial=f)
        return SimpleNamespace(grid=SimpleNamespace(nx=nx, ny=ny), spec=spec,
                               with_forcing_field=lambda v: ref_system(np.asarray(v)))

    sysm, _, _, _ = system_from_reference(ref_system(np.zeros(nx * ny)))
    traj = synthesize_trajectory(sysm, g["f_true"], RK4Config(T / 800), TimeLaw.sine(w))[:, 0, :]
    nodes = np.linspace(0.0, T, traj.shape[0])
    q_true = SimpleNamespace(eval_many=lambda ts: np.stack([[np.interp(t, nodes, traj[:, i]) for i in range(nx * ny)]
                                                            for t in ts]))
    r = direct_adjoint_loop(ref_system(np.zeros(nx * ny)), g["f"], q_true, "linear", N=N, dt=T / 400)
    assert abs(r.J - g["J"]) <= 2e-5 * g["J"]
    assert r.grad.shape == (nx * ny,) and rel_l2(r.grad, g["grad"]) <= 5e-6


def test_objective_switching_and_validation(cuda_ok):
    """A cached engine returns to the terminal objective after a tracking loop (bitwise the same
    terminal result); wrong target shapes and the hybrid plan are refused; the device-resident
    target gives the host target's numbers."""
    import torch

    from paper_2004_00546_b200 import (
        ChebyshevConfig, ConfigError, RK4Config, baseline, direct_adjoint_loop, make_hybrid_plan, scaled)
    from paper_2004_00546_b200.optimization import get_engine
    c = scaled(baseline(5), nx=32, P=4, steps_per_slice=5, K=8)
    u0, ut, ctrl = c.inputs()
    cfg = ChebyshevConfig(tol=1e-12)
    kw = dict(N=c.P, rk=RK4Config(c.dt), u0=u0, expaction=cfg)
    t0 = direct_adjoint_loop(c.system, ctrl, ut, "linear", **kw)
    tg = _target(c.system.n, c.P * c.nsteps)
    tr = direct_adjoint_loop(c.system, ctrl, tg, "linear", objective="tracking", **kw)
    t1 = direct_adjoint_loop(c.system, ctrl, ut, "linear", **kw)
    assert np.array_equal(np.asarray(t0.grad), np.asarray(t1.grad)) and np.array_equal(t0.J, t1.J)
    assert not np.allclose(np.asarray(tr.grad), np.asarray(t0.grad))
    with pytest.raises(ValueError):
        direct_adjoint_loop(c.system, ctrl, tg[:-1], "linear", objective="tracking", **kw)
    with pytest.raises(ConfigError):
        direct_adjoint_loop(c.system, ctrl, tg, "linear", objective="tracking", plan=make_hybrid_plan(1.0, 4, 2.0), **kw)
    with pytest.raises(ValueError):
        direct_adjoint_loop(c.system, ctrl, tg, "hybrid", objective="tracking", **kw)
    eng = get_engine(c.system, c.P, RK4Config(c.dt), cfg, 1, tracking=True)
    eng.set_inputs(u0, ut, ctrl)
    eng.set_tracking_target(torch.as_tensor(tg, device="cuda").contiguous())
    eng.gradient()
    rd = eng.results(fields=False)
    assert np.array_equal(rd["grad"][0], np.atleast_2d(tr.grad)[0]) and rd["J"][0] == pytest.approx(tr.J, rel=0)
    with pytest.raises(ValueError):
        eng.set_tracking_target(np.zeros((3, c.system.n)))
    eng.set_tracking_target(None)
