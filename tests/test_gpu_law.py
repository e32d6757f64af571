"""GPU parity of the linear testbed with a forcing time law θ(t) (the reference's f·sin(ωt),
`problems.py:155-162`) and with a full-field control (PX_FLAG_FIELD_CONTROL), against the oracle
(oracle.config_mode.linear_gradient_law / linear_gradient)."""

import numpy as np
import pytest

from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu


def _check(J, grad, uT, qdag0, G, o, grad_tol=1e-8, state_tol=1e-10):
    assert np.max(np.abs(np.atleast_1d(J) - o.J) / np.abs(o.J)) <= 1e-10
    assert rel_l2(np.atleast_2d(grad), o.grad) <= grad_tol
    assert rel_l2(uT, o.uT) <= state_tol
    assert rel_l2(qdag0, o.qdag0) <= state_tol
    assert rel_l2(G, o.G) <= state_tol


def _check_loop(r, o, **kw):
    _check(r.J, r.grad, r.direct.final_state, r.adjoint.initial_state, r.adjoint.integral, o, **kw)


def _oracle(c, law, system=None, ctrl=None, tol=1e-12):
    from oracle.config_mode import linear_gradient_law
    from paper_2004_00546_b200.expaction import ChebyshevConfig, plan_chebyshev
    s = system or c.system
    u0, ut, cc = c.inputs()
    pl = plan_chebyshev(s.region(), c.spec.T / c.P, ChebyshevConfig(tol=tol), omega=law.omega)
    return linear_gradient_law(s.grid.nx, s.grid.ny, s.A.as_tuple(), s.basis, c.spec.T, c.P, c.nsteps, u0, ut,
                               cc if ctrl is None else ctrl, law.as_tuple(), pl)


@pytest.mark.parametrize("index", [1, 2])
def test_time_law_1d_vs_oracle(cuda_ok, index):
    """1D on-chip lanes with θ at every stage, θ-weighted lane integrals, the generic Chebyshev
    carries with per-carry law series (config 1 at full size, config 2 scaled, batch 2)."""
    from paper_2004_00546_b200 import ChebyshevConfig, RK4Config, TimeLaw, baseline, direct_adjoint_loop, scaled
    c = baseline(1) if index == 1 else scaled(baseline(2), nx=512, P=8, steps_per_slice=25, batch=2, T=0.5)
    law = TimeLaw.sine(3.0 * np.pi / c.spec.T)
    u0, ut, ctrl = c.inputs()
    r = direct_adjoint_loop(c.system, ctrl, ut, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0,
                            expaction=ChebyshevConfig(tol=1e-12), time_law=law)
    _check_loop(r, _oracle(c, law))


def test_time_law_2d_vs_oracle(cuda_ok):
    """2D one-step march with the law stream (direct) and the θ-weighted ∫ (adjoint lanes), the
    2D Chebyshev passes with per-carry law series; a mixed α + β sin + γ cos law."""
    from paper_2004_00546_b200 import ChebyshevConfig, RK4Config, TimeLaw, baseline, direct_adjoint_loop, scaled
    c = scaled(baseline(5), nx=64, P=8, steps_per_slice=6, K=16)
    law = TimeLaw(0.3, 1.0, -0.5, 7.0)
    u0, ut, ctrl = c.inputs()
    r = direct_adjoint_loop(c.system, ctrl, ut, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0,
                            expaction=ChebyshevConfig(tol=1e-12), time_law=law)
    _check_loop(r, _oracle(c, law))


def test_field_control_and_law_2d(cuda_ok):
    """A full spatial control field (the reference's f_spatial) with and without the law: the
    gradient is the field ∫θ·q† dt; the constant law is the time-constant path."""
    from oracle.config_mode import linear_gradient
    from paper_2004_00546_b200 import ChebyshevConfig, RK4Config, TimeLaw, baseline, direct_adjoint_loop, scaled
    from paper_2004_00546_b200.expaction import plan_chebyshev
    from paper_2004_00546_b200.systems import build_field_system
    c = scaled(baseline(5), nx=64, P=6, steps_per_slice=5, K=16)
    fs = build_field_system(c.system.grid, c.system.spec)
    u0, ut, cc = c.inputs()
    f = c.system.basis.field(cc) + 0.01 * np.random.default_rng(2).standard_normal((1, fs.n))
    cfg = ChebyshevConfig(tol=1e-12)
    r0 = direct_adjoint_loop(fs, f, ut, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0, expaction=cfg)
    pl = plan_chebyshev(fs.region(), c.spec.T / c.P, cfg)
    o0 = linear_gradient(fs.grid.nx, fs.grid.ny, fs.A.as_tuple(), fs.basis, c.spec.T, c.P, c.nsteps, u0, ut, f, pl)
    _check_loop(r0, o0)
    assert np.asarray(r0.grad).shape[-1] == fs.n
    # the field gradient projected on the modes is the mode gradient of the same forcing
    rm = direct_adjoint_loop(c.system, cc, ut, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0, expaction=cfg)
    r0m = direct_adjoint_loop(fs, c.system.basis.field(cc), ut, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0,
                              expaction=cfg)
    assert rel_l2(c.system.basis.project(np.atleast_2d(r0m.grad)), np.atleast_2d(rm.grad)) <= 1e-12
    law = TimeLaw.sine(5.0)
    r1 = direct_adjoint_loop(fs, f, ut, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0, expaction=cfg, time_law=law)
    _check_loop(r1, _oracle(c, law, system=fs, ctrl=f))


def test_time_law_local_blocks_and_ranks_emulated(cuda_ok):
    """The law through the block-scan: local blocks (each block's law series from its own top
    time) and two emulated ranks (the long adjoint span from the rank's lower edge) agree with the
    oracle's single-rank scan to the truncation level (tol 1e-13)."""
    import torch
    from paper_2004_00546_b200 import ChebyshevConfig, TimeLaw, baseline, scaled
    from paper_2004_00546_b200.engine import EngineSpec, ParaexpEngine
    c = scaled(baseline(5), nx=64, P=8, steps_per_slice=5, K=16)
    law = TimeLaw(0.2, 1.0, 0.4, 6.0)
    cfg = ChebyshevConfig(tol=1e-13)
    u0, ut, ctrl = c.inputs()
    ref = _oracle(c, law, tol=1e-13)
    eng = ParaexpEngine(EngineSpec(c.system, c.P, c.dt, cfg, 1, local_blocks=2, law=law.as_tuple()))
    assert eng.local_blocks == 2
    eng.set_inputs(u0, ut, ctrl)
    eng.gradient()
    r = eng.results()
    _check(r["J"], r["grad"], r["uT"], r["qdag0"], r["G"], ref, grad_tol=1e-9, state_tol=1e-9)
    eng.close()
    engs = [ParaexpEngine(EngineSpec(c.system, c.P, c.dt, cfg, 1, rank=k, world=2, law=law.as_tuple()))
            for k in range(2)]

    def allreduce(fields):
        for f in fields:
            views = [e.device_view(f) for e in engs]
            total = torch.stack(views).sum(0)
            for v in views:
                v.copy_(total)

    for e in engs:
        e.set_inputs(u0, ut, ctrl)
        e.direct_partial()
    allreduce(engs[0].direct_reduce_fields())
    for e in engs:
        e.finish_direct()
        e.adjoint_partial()
    allreduce(engs[0].adjoint_reduce_fields(True))
    for e in engs:
        e.finish_adjoint()
    for e in engs:
        r = e.results()
        _check(r["J"], r["grad"], r["uT"], r["qdag0"], r["G"], ref, grad_tol=1e-9, state_tol=1e-9)
        e.close()


def test_time_law_solver_level_and_validation(cuda_ok):
    """solve_direct_linear / solve_adjoint_linear with the law (the reference's solver entry
    points take a forcing callable), and a Krylov plan with a law is refused."""
    from paper_2004_00546_b200 import (
        ChebyshevConfig, ConfigError, KrylovConfig, RK4Config, TimeLaw, baseline, direct_adjoint_loop, scaled,
        solve_adjoint_linear, solve_direct_linear)
    c = scaled(baseline(5), nx=64, P=8, steps_per_slice=6, K=16)
    law = TimeLaw.sine(4.0)
    u0, ut, ctrl = c.inputs()
    cfg = ChebyshevConfig(tol=1e-12)
    o = _oracle(c, law)
    d = solve_direct_linear(c.system, u0, ctrl, c.P, RK4Config(c.dt), cfg, time_law=law)
    assert rel_l2(d.final_state, o.uT) <= 1e-10
    a = solve_adjoint_linear(c.system, o.uT - ut, c.P, RK4Config(c.dt), cfg, time_law=law)
    assert rel_l2(a.initial_state, o.qdag0) <= 1e-10 and rel_l2(a.integral, o.G) <= 1e-10
    with pytest.raises(ConfigError):
        direct_adjoint_loop(c.system, ctrl, ut, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0,
                            expaction=KrylovConfig(m=10), time_law=law)
