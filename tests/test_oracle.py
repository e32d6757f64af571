"""CPU oracle (config mode) validated independently of the GPU.

* exp-actions vs FFT-exact circulant propagators (the linear operators are
  circulant, so exp(τA) and τφ₁(τA) are exact in Fourier space);
* RK4 slice solves vs the exact variation-of-constants solution (the reference's
  `harmonic_oracle` technique, `test_paraexp.py:28-37`, with FFT instead of expm);
* gradient vs central finite differences of the same discrete pipeline
  (`test_optimization.py:124-146`);
* formulation equivalence: reference neighbour chains ≡ summed-chain scan ≡
  blockscan(G) (`paraexp.py:207-217` by linearity);
* Burgers: adjoint operator identity and FD gradient up to the frozen-slice
  model error.
"""

import numpy as np
import pytest

from oracle.config_mode import (
    burgers_adjoint_apply,
    burgers_gradient,
    burgers_rhs,
    cheb_action,
    krylov_action,
    linear_gradient,
    rk4_linear,
    stencil_apply,
)
from paper_2004_00546_b200.expaction import ChebyshevConfig, KrylovConfig, phi1, plan_chebyshev, plan_krylov
from paper_2004_00546_b200.problems import (
    ADVECTION_DIFFUSION,
    BURGERS,
    Grid,
    ProblemSpec,
    advdiff_region,
    advdiff_stencil,
    burgers_frozen_region,
)
from paper_2004_00546_b200.systems import build_system
from tests.conftest import rel_l2


def fft_apply(st, nx, ny, fn):
    cc, ce, cw, cn, cs = st
    th = 2 * np.pi * np.arange(nx) / nx
    lam = cc + ce * np.exp(1j * th) + cw * np.exp(-1j * th)
    if ny > 1:
        ty = 2 * np.pi * np.arange(ny) / ny
        lam = lam[None, :] + cn * np.exp(1j * ty)[:, None] + cs * np.exp(-1j * ty)[:, None]

    def apply(v):
        V = np.fft.fftn(v.reshape(ny, nx) if ny > 1 else v)
        return np.real(np.fft.ifftn(fn(lam) * V)).ravel()
    return apply, lam


CASES = {
    "c1": (Grid(256), (1.0, 0.0), 0.01, 0.25, 1e-12),
    "c2": (Grid(1024), (1.0, 0.0), 0.005, 2 / 64, 1e-12),
    "c4": (Grid(64, 64), (1.0, 0.5), 1e-3, 1 / 128, 1e-10),
    "c5": (Grid(96, 96), (1.0, 0.5), 5e-4, 1 / 512, 1e-10),
    "long": (Grid(64, 64), (1.0, 0.5), 5e-4, 0.5, 1e-10),
}


def test_spectrum_enclosure_contains_eigenvalues():
    for g, a, D, _, _ in CASES.values():
        st = advdiff_stencil(g, a, D).as_tuple()
        _, lam = fft_apply(st, g.nx, g.ny, lambda l: l)
        lo, hi, im = advdiff_region(g, a, D).box()
        lam = np.ravel(lam)
        assert np.all(lam.real >= lo - 1e-9) and np.all(lam.real <= hi + 1e-9)
        assert np.all(np.abs(lam.imag) <= im + 1e-9)


@pytest.mark.parametrize("name", list(CASES))
def test_chebyshev_action_vs_fft_exact(name):
    g, a, D, span, tol = CASES[name]
    st = advdiff_stencil(g, a, D).as_tuple()
    plan = plan_chebyshev(advdiff_region(g, a, D), span, ChebyshevConfig(tol=tol))
    v = np.random.default_rng(1).standard_normal(g.npoints)
    phi = np.zeros_like(v)
    got = cheb_action(lambda u: stencil_apply(st, u, g.nx, g.ny), plan, v, phi)
    ex, _ = fft_apply(st, g.nx, g.ny, lambda l: np.exp(span * l))
    exp_phi, _ = fft_apply(st, g.nx, g.ny, lambda l: span * phi1(span * l))
    assert np.linalg.norm(got - ex(v)) <= 10 * tol * np.linalg.norm(v)
    assert np.linalg.norm(phi - exp_phi(v)) <= 10 * tol * span * np.linalg.norm(v)


def test_krylov_action_vs_fft_exact():
    g, a, D, span, tol = CASES["c4"]
    st = advdiff_stencil(g, a, D).as_tuple()
    plan = plan_krylov(advdiff_region(g, a, D), span, KrylovConfig(m=30, tol=tol))
    v = np.random.default_rng(2).standard_normal(g.npoints)
    phi = np.zeros_like(v)
    got = krylov_action(lambda u: stencil_apply(st, u, g.nx, g.ny), plan, v, phi)
    ex, _ = fft_apply(st, g.nx, g.ny, lambda l: np.exp(span * l))
    exp_phi, _ = fft_apply(st, g.nx, g.ny, lambda l: span * phi1(span * l))
    assert np.linalg.norm(got - ex(v)) <= 10 * tol * np.linalg.norm(v)
    assert np.linalg.norm(phi - exp_phi(v)) <= 10 * tol * span * np.linalg.norm(v)


def test_planner_is_deterministic_and_cheap_at_slice_width():
    g, a, D, span, tol = CASES["c5"]
    r = advdiff_region(g, a, D)
    p1 = plan_chebyshev(r, span, ChebyshevConfig(tol=tol))
    p2 = plan_chebyshev(r, span, ChebyshevConfig(tol=tol))
    assert p1 is p2 or (np.array_equal(p1.coef_exp, p2.coef_exp) and p1.degree == p2.degree)
    assert p1.terms <= 40


def test_rk4_slice_vs_exact_variation_of_constants():
    g = Grid(128)
    st = advdiff_stencil(g, (1.0, 0.0), 0.02).as_tuple()
    gsrc = np.random.default_rng(3).standard_normal(g.npoints)
    T, n = 0.1, 200
    y, z = rk4_linear(lambda u: stencil_apply(st, u, g.nx, 1), gsrc, T / n, n, want_z=True)
    ex, _ = fft_apply(st, g.nx, 1, lambda l: T * phi1(T * l))
    # z = ∫ y = ∫_0^T s φ1(sA) g ds = T² φ2(TA) g
    def phi2(zz):
        with np.errstate(all="ignore"):
            return np.where(np.abs(zz) < 1e-3, 0.5 + zz / 6 + zz * zz / 24, (np.exp(zz) - 1 - zz) / (zz * zz))
    ez, _ = fft_apply(st, g.nx, 1, lambda l: T * T * phi2(T * l))
    assert rel_l2(y, ex(gsrc)) < 1e-8
    assert rel_l2(z, ez(gsrc)) < 1e-8


def _small_linear(nx=48, ny=1, P=4, nsteps=40, B=2, K=6, T=1.0):
    g = Grid(nx, ny)
    spec = ProblemSpec(ADVECTION_DIFFUSION, (1.0, 0.5), 0.05, T)
    sysm = build_system(g, spec, K)
    rng = np.random.default_rng(11)
    x, y = g.coordinates()
    u0 = np.exp(-((x - np.pi) ** 2 + (y - np.pi) ** 2) / 0.3)
    ut = 0.1 * np.sin(2 * x + y)
    ctrl = rng.normal(0, 0.1, (B, K))
    cfg = ChebyshevConfig(tol=1e-13)
    r = sysm.region()
    plan = plan_chebyshev(r, T / P, cfg)
    longp = lambda span: plan_chebyshev(r, span, cfg)
    return sysm, u0, ut, ctrl, plan, longp, P, nsteps, T


@pytest.mark.parametrize("ny", [1, 12])
def test_gradient_vs_central_fd(ny):
    sysm, u0, ut, ctrl, plan, _, P, nsteps, T = _small_linear(nx=24 if ny > 1 else 48, ny=ny, K=4 if ny > 1 else 6)
    g = sysm.grid
    A = sysm.A.as_tuple()
    base = linear_gradient(g.nx, g.ny, A, sysm.basis, T, P, nsteps, u0, ut, ctrl[:1], plan)
    eps = 1e-5
    fd = np.zeros(sysm.basis.K)
    for k in range(sysm.basis.K):
        cp, cm = ctrl[:1].copy(), ctrl[:1].copy()
        cp[0, k] += eps
        cm[0, k] -= eps
        Jp = linear_gradient(g.nx, g.ny, A, sysm.basis, T, P, nsteps, u0, ut, cp, plan).J[0]
        Jm = linear_gradient(g.nx, g.ny, A, sysm.basis, T, P, nsteps, u0, ut, cm, plan).J[0]
        fd[k] = (Jp - Jm) / (2 * eps)
    assert rel_l2(base.grad[0], fd) < 1e-8


def test_formulations_agree():
    sysm, u0, ut, ctrl, plan, longp, P, nsteps, T = _small_linear(P=6)
    g = sysm.grid
    A = sysm.A.as_tuple()
    scan = linear_gradient(g.nx, g.ny, A, sysm.basis, T, P, nsteps, u0, ut, ctrl, plan, want_boundary=True)
    chains = linear_gradient(g.nx, g.ny, A, sysm.basis, T, P, nsteps, u0, ut, ctrl, plan, formulation="chains")
    assert rel_l2(chains.uT, scan.uT) < 1e-13
    assert rel_l2(chains.qdag0, scan.qdag0) < 1e-13
    assert rel_l2(chains.grad, scan.grad) < 1e-13
    for world in (2, 3, 6):
        bs = linear_gradient(g.nx, g.ny, A, sysm.basis, T, P, nsteps, u0, ut, ctrl, plan, longp, longp,
                             formulation="blockscan", world=world)
        assert rel_l2(bs.uT, scan.uT) < 1e-11
        assert rel_l2(bs.qdag0, scan.qdag0) < 1e-11
        assert rel_l2(bs.grad, scan.grad) < 1e-11
    assert np.allclose(scan.u_bnd[:, -1], scan.uT)
    assert np.allclose(scan.u_bnd[:, 0], u0)


def test_adjoint_initial_state_matches_exact_backward_propagation():
    """q†(0) = exp(T·Aᵀ)q†_T exactly for the terminal objective (no adjoint source)."""
    sysm, u0, ut, ctrl, plan, _, P, nsteps, T = _small_linear(P=4)
    g = sysm.grid
    res = linear_gradient(g.nx, g.ny, sysm.A.as_tuple(), sysm.basis, T, P, nsteps, u0, ut, ctrl[:1], plan)
    qT = res.uT - ut
    ex, _ = fft_apply(sysm.A.transpose().as_tuple(), g.nx, g.ny, lambda l: np.exp(T * l))
    assert rel_l2(res.qdag0[0], ex(qT[0])) < 1e-9


def test_burgers_operators():
    g = Grid(64)
    rng = np.random.default_rng(5)
    u = 0.4 * rng.standard_normal(g.nx)
    x = rng.standard_normal(g.nx)
    y = rng.standard_normal(g.nx)
    D, h = 0.1, g.hx
    # Jᵀ is the transpose of the directional derivative of the rhs (FD Jacobian check)
    eps = 1e-6
    Jx = (burgers_rhs(u + eps * x, 0.0, D, h) - burgers_rhs(u - eps * x, 0.0, D, h)) / (2 * eps)
    lhs = y @ Jx
    rhs = burgers_adjoint_apply(u, y, D, h) @ x
    assert abs(lhs - rhs) <= 1e-6 * np.linalg.norm(x) * np.linalg.norm(y)


def test_burgers_region_contains_frozen_spectrum():
    g = Grid(64)
    rng = np.random.default_rng(6)
    ub = 0.5 * np.sin(g.x1()) + 0.1 * rng.standard_normal(g.nx)
    D = 0.05
    M = np.stack([burgers_adjoint_apply(ub, e, D, g.hx) for e in np.eye(g.nx)], axis=1)
    reg = burgers_frozen_region(ub, g, D)
    lo, hi, im = reg.rect
    # field of values ⊂ box: Rayleigh quotients of random complex vectors
    for _ in range(50):
        v = rng.standard_normal(g.nx) + 1j * rng.standard_normal(g.nx)
        r = np.vdot(v, M @ v) / np.vdot(v, v)
        assert lo - 1e-9 <= r.real <= hi + 1e-9 and abs(r.imag) <= im + 1e-9
    ev = np.linalg.eigvals(M)
    assert np.all(ev.real >= lo - 1e-9) and np.all(ev.real <= hi + 1e-9)


def test_burgers_gradient_vs_fd_within_frozen_model_error():
    g = Grid(96)
    spec = ProblemSpec(BURGERS, (0, 0), 0.05, 1.0)
    sysm = build_system(g, spec, 4)
    x = g.x1()
    u0 = 0.5 * np.sin(x)
    ut = 0.3 * np.sin(x + 0.5)
    ctrl = np.random.default_rng(1).normal(0, 0.1, (1, 4))
    cfg = ChebyshevConfig(tol=1e-12)
    planf = lambda region, span: plan_chebyshev(region, span, cfg)
    regf = lambda ub: burgers_frozen_region(ub, g, spec.D)
    P, ns = 6, 24
    res = burgers_gradient(g.nx, spec.D, sysm.basis, 1.0, P, ns, u0, ut, ctrl, planf, regf)
    eps = 1e-6
    fd = np.zeros(4)
    for k in range(4):
        cp, cm = ctrl.copy(), ctrl.copy()
        cp[0, k] += eps
        cm[0, k] -= eps
        fd[k] = (burgers_gradient(g.nx, spec.D, sysm.basis, 1.0, P, ns, u0, ut, cp, planf, regf).J[0]
                 - burgers_gradient(g.nx, spec.D, sysm.basis, 1.0, P, ns, u0, ut, cm, planf, regf).J[0]) / (2 * eps)
    # piecewise-frozen homogeneous parts carry a model error (~6.5e-5 on q†(0))
    assert rel_l2(res.grad[0], fd) < 2e-3
    rb = burgers_gradient(g.nx, spec.D, sysm.basis, 1.0, P, ns, u0, ut, ctrl, planf, regf, world=2)
    assert rel_l2(rb.grad, res.grad) < 1e-13


def test_unstable_rk4_step_is_rejected_before_any_gpu_work():
    from paper_2004_00546_b200 import ConfigError, baseline, scaled
    from paper_2004_00546_b200.engine import EngineSpec, ParaexpEngine
    c = scaled(baseline(5), nx=640, P=4, steps_per_slice=3, K=16)  # h·ρ ≈ 13
    with pytest.raises(ConfigError):
        ParaexpEngine(EngineSpec(c.system, c.P, c.dt, c.expaction))
