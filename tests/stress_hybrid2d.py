"""Randomised GPU-vs-oracle sweep of the 2D two-field Burgers path (not a pytest module; run
`python tests/stress_hybrid2d.py [count] [seed]` on a GPU box): random grid shapes (odd sizes, both kernel
families), members, slice counts and partitions, laws, terminal data, hybrid and nonlinear loops."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def run(count: int, seed: int) -> dict:
    from oracle.config_mode import burgers2d_nonlinear_tracking, burgers_tracking_hybrid
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system, make_hybrid_plan,
        solve_hybrid_tracking, solve_nonlinear_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.expaction import plan_chebyshev, plan_family
    from paper_2004_00546_b200.problems import BURGERS, frozen_bounds_2d, frozen_region_from_bounds
    from paper_2004_00546_b200.tracking import release_tracking_engines
    rng = np.random.default_rng(seed)
    worst = {"J": 0.0, "grad": 0.0, "qdag0": 0.0, "uT": 0.0}
    for case in range(count):
        big = rng.random() < 0.3
        nx, ny = (int(rng.integers(46, 70)), int(rng.integers(46, 70))) if big else (int(rng.integers(5, 45)), int(rng.integers(5, 45)))
        B = int(rng.integers(1, 4))
        P = int(rng.integers(1, 7))
        T, D = float(rng.uniform(0.1, 0.4)), float(rng.uniform(0.01, 0.2))
        lam = 4 * D * ((nx / (2 * np.pi)) ** 2 + (ny / (2 * np.pi)) ** 2)
        steps = int(np.ceil(T / min(2e-3, 1.0 / lam) / P)) * P
        rk, cfg = RK4Config(T / steps), ChebyshevConfig(tol=1e-12)
        law = TimeLaw(*rng.uniform(-1, 1, 3), float(rng.uniform(0.5, 6.0))) if rng.random() < 0.7 else TimeLaw.constant()
        sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), D, T))
        X, Y = sysm.grid.coordinates()
        mk = lambda: np.concatenate([rng.uniform(-.4, .4) * np.sin(X) * np.cos(Y) + rng.uniform(-.3, .3) * np.cos(2 * X + Y),
                                     rng.uniform(-.4, .4) * np.cos(X) * np.sin(Y) + rng.uniform(-.3, .3) * np.sin(X - 2 * Y)])
        u0, f, ft = mk(), np.stack([mk() for _ in range(B)]), mk()
        target = synthesize_trajectory(sysm, ft, rk, law, u0=u0)[:, 0, :]
        nonlinear = P > 1 and rng.random() < 0.35
        reg = lambda q: frozen_region_from_bounds(*frozen_bounds_2d(q, sysm.grid, D))
        h = T / steps
        if nonlinear:
            r = solve_nonlinear_tracking(sysm, u0, f, target, N=P, rk=rk, expaction=cfg, law=law, eps=1e-10)
            o = burgers2d_nonlinear_tracking(nx, ny, D, T, P, steps // P, u0, f, law.as_tuple(), target,
                                             lambda q: (plan_chebyshev(reg(q), T / P, cfg), plan_chebyshev(reg(q), h, cfg)),
                                             lambda q: plan_family(reg(q), [T / P] * P, cfg, omega=law.omega), 1e-10)
            kind = f"nonlinear sweeps {len(r.timing['history'])}/{o.extras['sweeps']}"
        else:
            plan = make_hybrid_plan(T, P, float(rng.uniform(0.5, 6.0))) if P > 1 and rng.random() < 0.6 else None
            qT = 0.1 * np.stack([mk() for _ in range(B)]) if rng.random() < 0.4 else None
            ov = bool(rng.random() < 0.5)
            r = solve_hybrid_tracking(sysm, u0, f, target, plan, N=P, rk=rk, expaction=cfg, law=law, qdag_T=qT, overlap=ov)
            offs = r.offsets
            o = burgers_tracking_hybrid(nx, D, T, offs, u0, f, law.as_tuple(), target,
                                        lambda q: plan_family(reg(q), [(offs[p + 1] - offs[p]) * h for p in range(P)], cfg,
                                                              omega=law.omega), qdag_T=qT, ny=ny)
            kind = f"hybrid {'geometric' if plan else 'equal'} qT={qT is not None} overlap={ov}"
        e = {"J": float(np.max(np.abs(r.J - o.J) / np.abs(o.J))), "grad": rel(r.grad, o.grad), "qdag0": rel(r.qdag0, o.qdag0),
             "uT": rel(r.final_state, o.uT)}
        ok = e["J"] <= 1e-10 and e["grad"] <= 1e-8 and e["qdag0"] <= 1e-9 and e["uT"] <= 1e-10
        for k in worst:
            worst[k] = max(worst[k], e[k])
        print(f"case {case}: {nx}x{ny} B={B} P={P} S={steps} {kind}: " + " ".join(f"{k}={v:.1e}" for k, v in e.items()) +
              ("" if ok else "  <-- FAIL"), flush=True)
        release_tracking_engines()
        if not ok:
            raise AssertionError(f"case {case} exceeds the parity bounds: {e}")
    print("worst", worst)
    return worst


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 12, int(sys.argv[2]) if len(sys.argv) > 2 else 7)
