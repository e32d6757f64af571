"""The reference's hybrid with its tracking objective: host logic and the
oracle restatement, on the CPU. The restatement is pinned to the reference's own
`direct_adjoint_loop(..., "hybrid", plan=make_hybrid_plan(...))` through
tests/golden/reference_hybrid_tracking.npz (oracle/gen_golden_hybrid.py)."""

import os

import numpy as np
import pytest

from tests.conftest import ROOT, rel_l2

from paper_2004_00546_b200.errors import ConfigError
from paper_2004_00546_b200.expaction import ChebyshevConfig, plan_chebyshev, plan_family
from paper_2004_00546_b200.hybrid import HybridPlan, TimeLaw, make_hybrid_plan, partition_geometric, slice_offsets
from paper_2004_00546_b200.problems import Grid, frozen_bounds, frozen_region_from_bounds

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_hybrid_tracking.npz")


def test_geometric_partition_follows_the_ratio():
    """T_n = T(1 − rⁿ)/(1 − r^N), r = k/(k+1) (`hybrid.py:35-55`); widths shrink by r."""
    part = partition_geometric(2.0, 5, 3.0)
    r = 0.75
    expect = 2.0 * (1 - r ** np.arange(6)) / (1 - r ** 5)
    np.testing.assert_allclose(part.boundaries, expect, rtol=0, atol=1e-15)
    w = part.widths()
    np.testing.assert_allclose(w[1:] / w[:-1], r, rtol=1e-12)
    assert part.kind == "geometric" and part.ratio == 3.0
    plan = make_hybrid_plan(2.0, 5, 3.0)
    assert plan.N == 5 and plan.k == 3.0
    with pytest.raises(ValueError):
        HybridPlan(partition_geometric(1.0, 4, 1.0), 2.0)      # widths do not follow k
    with pytest.raises(ValueError):
        make_hybrid_plan(1.0, 6, 0.5, h_min=0.01)             # last width below 2·h_min
    with pytest.raises(ValueError):
        partition_geometric(1.0, 0, 1.0)
    with pytest.raises(ValueError):
        partition_geometric(1.0, 3, -1.0)


def test_slice_offsets_on_the_node_grid():
    part = partition_geometric(1.0, 64, 20.0)
    o = slice_offsets(part, 5e-4)
    assert o[0] == 0 and o[-1] == 2000 and np.all(np.diff(o) >= 1)
    np.testing.assert_allclose(o * 5e-4, part.boundaries, rtol=0, atol=0.5 * 5e-4 + 1e-12)
    # widths below one step: every slice still gets a step, the last edges stay in range
    o2 = slice_offsets(partition_geometric(1.0, 64, 2.0), 5e-4)
    assert o2[-1] == 2000 and np.all(np.diff(o2) >= 1)
    with pytest.raises(ConfigError):
        slice_offsets(partition_geometric(1.0, 8, 1.0), 0.25)   # 4 steps cannot hold 8 slices
    eq = slice_offsets(partition_geometric(1.0, 1, 1.0), 1e-3)
    assert list(eq) == [0, 1000]


def test_time_law():
    law = TimeLaw.sine(3.0)
    t = np.linspace(0, 1, 7)
    np.testing.assert_allclose(law(t), np.sin(3.0 * t))
    np.testing.assert_allclose(TimeLaw(0.5, 0.0, 2.0, 1.0)(t), 0.5 + 2.0 * np.cos(t))
    assert TimeLaw.constant()(0.7) == 1.0
    with pytest.raises(ValueError):
        TimeLaw(omega=-1.0)


def test_law_series_vs_dense_quadrature():
    """exp(τM)v and ∫₀^span θ(t_top − σ)·e^{σM}v dσ from the planned series (several substeps)
    against a dense exponential and Gauss–Legendre quadrature, on a frozen J(ū)ᵀ."""
    from scipy.linalg import expm

    from oracle.config_mode import burgers_adjoint_apply, cheb_law_action
    nx, D = 48, 0.05
    g = Grid(nx)
    x = g.x1()
    ub = 0.6 * np.sin(x) + 0.2
    M = np.stack([burgers_adjoint_apply(ub, e, D, g.hx) for e in np.eye(nx)], axis=1)
    region = frozen_region_from_bounds(*frozen_bounds(ub[None, :], g, D))
    law = TimeLaw(0.3, 1.0, -0.5, 5.0)
    span, t_top = 0.07, 0.4
    pl = plan_chebyshev(region, span, ChebyshevConfig(tol=1e-13), omega=law.omega)
    v = np.cos(2 * x) + 0.1 * np.sin(5 * x)
    Gs = np.zeros(nx)
    out = cheb_law_action(lambda y: M @ y, pl, v.copy(), Gs, law.as_tuple(), t_top)
    np.testing.assert_allclose(out, expm(span * M) @ v, rtol=0, atol=1e-11 * np.linalg.norm(v))
    s, w = np.polynomial.legendre.leggauss(60)
    ref = np.zeros(nx)
    for si, wi in zip(0.5 * span * (s + 1), 0.5 * span * w):
        ref += wi * law(t_top - si) * (expm(si * M) @ v)
    assert rel_l2(Gs, ref) <= 1e-11


def test_plan_family_meets_the_bound_on_every_span():
    region = frozen_region_from_bounds(-400.0, 0.0, 60.0)
    spans = [0.02 * 0.7 ** p for p in range(6)]
    plans = plan_family(region, spans, ChebyshevConfig(tol=1e-12), omega=4.0)
    assert [p.span for p in plans] == spans
    for p in plans:
        assert p.coef_gc is not None and len(p.coef_gc) == p.degree + 1 and p.err_bound <= 1e-12 / p.substeps
    assert plans[-1].substeps * plans[-1].degree <= plans[0].substeps * plans[0].degree


def _golden_case(dt):
    from oracle.config_mode import burgers_direct_law, burgers_tracking_hybrid
    gd = np.load(GOLDEN)
    nx, T, D, w = int(gd["nx"]), float(gd["T"]), float(gd["D"]), float(gd["omega"])
    law = TimeLaw.sine(w).as_tuple()
    grid = Grid(nx)
    offs = slice_offsets(make_hybrid_plan(T, int(gd["N"]), float(gd["k"])).partition, dt)
    S = int(offs[-1])
    h = T / S
    tgt = burgers_direct_law(np.zeros((1, nx)), gd["f_true"][None, :], law, D, grid.hx, h, S)[:, 0, :]
    cfg = ChebyshevConfig(tol=1e-12)

    def plans_for(ubar):
        reg = frozen_region_from_bounds(*frozen_bounds(ubar, grid, D))
        return plan_family(reg, [(offs[p + 1] - offs[p]) * h for p in range(len(offs) - 1)], cfg, omega=w)

    return gd, burgers_tracking_hybrid(nx, D, T, offs, np.zeros(nx), gd["f"], law, tgt, plans_for)


def test_oracle_tracking_hybrid_pinned_to_the_reference_loop():
    """The restatement (classical RK4, Chebyshev frozen actions, node trapezoid) against the
    reference's own hybrid loop (DOPRI5 at rtol 1e-10, Leja, 4001 probe nodes): the embedded
    1D problem's J is a third of the reference's (three identical rows), the gradient of one row
    is the 1D gradient. Agreement at the discretisations' level; a wrong sign, factor, phase of
    the law or the absorbed (Option A) adjoint instead of `solve_hybrid`'s would be ≥ 1e-4 off."""
    gd, r = _golden_case(1e-3)
    assert abs(r.J[0] - gd["J"] / 3) <= 1e-6 * abs(gd["J"] / 3)
    assert rel_l2(r.grad[0], gd["grad_rows"][0]) <= 1e-5
    assert rel_l2(r.qdag0[0], gd["qdag0"]) <= 1e-6
    assert rel_l2(r.uT[0], gd["uT"]) <= 1e-10
    assert float(gd["v_grad_max"]) <= 1e-15  # V ≡ 0 in the reference too (rounding only)


def test_oracle_tracking_gradient_vs_finite_differences_serial():
    """One slice (the reference's serial loop): the adjoint gradient is the continuous adjoint,
    so it matches central differences of J to O(h²)."""
    from oracle.config_mode import burgers_direct_law, burgers_tracking_hybrid
    nx, D, T, S = 32, 0.05, 0.3, 150
    g = Grid(nx)
    x = g.x1()
    law = TimeLaw.sine(2 * np.pi).as_tuple()
    u0 = 0.5 * np.sin(x)
    f = (0.3 * np.cos(2 * x) + 0.2 * np.sin(3 * x))[None, :]
    tgt = burgers_direct_law(u0[None, :], 0.5 * np.sin(x)[None, :], law, D, g.hx, T / S, S)[:, 0, :]
    run = lambda ff: burgers_tracking_hybrid(nx, D, T, [0, S], u0, ff, law, tgt, lambda ub: [])
    r = run(f)
    d = np.random.default_rng(3).standard_normal(nx)[None, :]
    eps = 1e-4
    fd = (run(f + eps * d).J[0] - run(f - eps * d).J[0]) / (2 * eps)
    assert abs(fd - np.sum(r.grad * d)) <= 1e-4 * abs(fd)


def test_tracking_loop_validation():
    from paper_2004_00546_b200 import RK4Config, baseline, direct_adjoint_loop
    c1, c3 = baseline(1), baseline(3)
    rk = RK4Config(1e-3)
    with pytest.raises(ValueError):   # linear testbed
        direct_adjoint_loop(c1.system, np.zeros(c1.system.n), np.zeros((1001, c1.system.n)), "hybrid", rk=rk,
                            objective="tracking")
    with pytest.raises(ValueError):   # algorithm
        direct_adjoint_loop(c3.system, np.zeros(c3.system.n), None, "nonlinear", rk=rk, objective="tracking")
    with pytest.raises(ValueError):
        direct_adjoint_loop(c3.system, np.zeros(c3.system.n), None, "hybrid", rk=rk, objective="bogus")
    with pytest.raises(ConfigError):  # plan / law belong to the tracking objective
        direct_adjoint_loop(c3.system, np.zeros(c3.system.basis.K), np.zeros(c3.system.n), "hybrid", rk=rk,
                            time_law=TimeLaw.sine(1.0))


# --- the reference's own partition / pilot tests (`tests/test_hybrid.py:25-110`), mirrored ----


def test_geometric_single_interval_and_decreasing_widths():
    assert partition_geometric(5.0, 1, 2.0).boundaries.tolist() == [0.0, 5.0]
    part = partition_geometric(3.0, 6, 1.7)
    assert part.boundaries[0] == 0.0 and part.boundaries[-1] == 3.0
    assert np.all(np.diff(part.widths()) < 0)


def test_geometric_boundaries_high_precision():
    """The reference's pinned k = 2.11 boundaries 0.4676 / 0.7848 (`test_hybrid.py:36-47`),
    against the closed form at 50 digits."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 50
    k = mp.mpf("2.11")
    r = k / (k + 1)
    want = [float((1 - r ** n) / (1 - r ** 3)) for n in (0, 1, 2, 3)]
    part = partition_geometric(1.0, 3, 2.11)
    assert part.boundaries == pytest.approx(want, abs=1e-12)
    assert part.boundaries[1] == pytest.approx(0.4676, abs=5e-5)
    assert part.boundaries[2] == pytest.approx(0.7848, abs=5e-5)
    assert make_hybrid_plan(1.0, 8, 2.11).partition.widths()[1:] / make_hybrid_plan(1.0, 8, 2.11).partition.widths()[:-1] \
        == pytest.approx(2.11 / 3.11, rel=1e-10)


def test_plan_rejects_an_equidistant_partition():
    from paper_2004_00546_b200.partition import partition_equidistant
    with pytest.raises(ValueError):
        HybridPlan(partition_equidistant(1.0, 4), 2.11)
    with pytest.raises(ValueError):
        make_hybrid_plan(1.0, 8, 2.11, h_min=0.05)


def _burgers16():
    from paper_2004_00546_b200 import BURGERS, Grid, ProblemSpec, build_system
    return build_system(Grid(16), ProblemSpec(BURGERS, (0.0, 0.0), 1.0, 1.0), 2)


def test_estimate_k_with_synthetic_pilot_costs(monkeypatch):
    """k = τ_adjoint/τ_direct: symmetric costs give 1, doubling the adjoint's doubles k
    (`test_hybrid.py:71-100`, the pilot patched with synthetic times)."""
    import paper_2004_00546_b200.hybrid as H
    from paper_2004_00546_b200 import RK4Config, estimate_k
    sysm = _burgers16()
    monkeypatch.setattr(H, "_pilot_times", lambda *a, **kw: (0.1, 0.1))
    assert estimate_k(sysm, 0.05, RK4Config(1e-3)) == pytest.approx(1.0, rel=0.2)
    monkeypatch.setattr(H, "_pilot_times", lambda *a, **kw: (0.1, 0.25))
    base = estimate_k(sysm, 0.05, RK4Config(1e-3))
    monkeypatch.setattr(H, "_pilot_times", lambda *a, **kw: (0.1, 0.5))
    assert estimate_k(sysm, 0.05, RK4Config(1e-3)) == pytest.approx(2.0 * base, rel=1e-12)


def test_estimate_k_validation():
    from paper_2004_00546_b200 import PilotTooShort, RK4Config, estimate_k
    sysm = _burgers16()
    with pytest.raises(ValueError):
        estimate_k(sysm, 0.5, RK4Config(1e-3))
    with pytest.raises(PilotTooShort):
        estimate_k(sysm, 0.001, RK4Config(1e-3))
