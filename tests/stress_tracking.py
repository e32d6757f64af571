"""Randomised GPU-vs-oracle sweep of the linear testbed's tracking loop (the reference's linear loop:
`px_set_tracking_target`) and of the terminal objective with a time law: 1D and non-square 2D grids, field
and mode controls, members with shared / own targets, constant / sine / mixed laws, slices and steps.
Not a pytest module; run `python tests/stress_tracking.py [count] [seed]` on a GPU box."""

import os
import sys
from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def run(count: int, seed: int) -> dict:
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, RK4Config, TimeLaw, baseline, direct_adjoint_loop, release_engines, scaled)
    from paper_2004_00546_b200.systems import build_field_system
    from tests.test_gpu_tracking import _oracle, _target
    rng = np.random.default_rng(seed)
    worst = {}
    for case in range(count):
        two_d = rng.random() < 0.6
        P = int(rng.integers(1, 9))
        steps = int(rng.integers(2, 8))
        B = int(rng.integers(1, 4))
        field = rng.random() < 0.5
        if two_d:
            nx, ny = 2 * int(rng.integers(6, 60)), int(rng.integers(6, 90))
            c = scaled(baseline(5), nx=nx, P=P, steps_per_slice=steps, K=int(rng.choice([4, 16])), batch=B,
                       T=float(rng.uniform(0.02, 0.2)))
            c = replace(c, grid=Grid(nx, ny))
        else:
            nx, ny = int(rng.choice([64, 128, 256, 512, 1024])), 1
            h = float(rng.uniform(0.5, 1.0)) / (4 * 0.01 * (nx / (2 * np.pi)) ** 2 + nx / (2 * np.pi))
            c = scaled(baseline(1), nx=nx, P=P, steps_per_slice=steps, K=2 * int(rng.integers(1, 6)), batch=B,
                       T=P * steps * min(h, 0.3 / (P * steps)))
        sysm = build_field_system(c.system.grid, c.system.spec) if field else c.system
        n = sysm.n
        u0 = 0.1 * rng.standard_normal(n)
        ctrl = rng.standard_normal((B, n)) if field else c.inputs()[2]
        kind = rng.random()
        law = TimeLaw.constant() if kind < 0.25 else (TimeLaw.sine(float(rng.uniform(1, 9))) if kind < 0.6 else
                                                      TimeLaw(*rng.uniform(-1, 1, 3), float(rng.uniform(1, 9))))
        own = B > 1 and rng.random() < 0.5
        tg = _target(n, c.P * c.nsteps, B=B if own else None, seed=int(rng.integers(1 << 30)))
        r = direct_adjoint_loop(sysm, ctrl, tg, "linear", N=c.P, rk=RK4Config(c.dt), u0=u0,
                                expaction=ChebyshevConfig(tol=1e-13), objective="tracking", time_law=law)
        o = _oracle(sysm, c, u0, ctrl, law, tg)
        e = {"J": float(np.max(np.abs(np.atleast_1d(r.J) - o.J) / np.abs(o.J))), "grad": rel(np.atleast_2d(r.grad), o.grad),
             "uT": rel(np.atleast_2d(np.asarray(r.direct.final_state)), o.uT),
             "qdag0": rel(np.atleast_2d(np.asarray(r.adjoint.initial_state)), o.qdag0)}
        ok = e["J"] <= 1e-10 and max(e["grad"], e["uT"], e["qdag0"]) <= 1e-9
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
        print(f"case {case}: {nx}x{ny} P={P} steps={steps} B={B} {'field' if field else 'modes'} law={law.as_tuple()[3]:.2f} "
              f"own_target={own}: " + " ".join(f"{k}={v:.1e}" for k, v in e.items()) + ("" if ok else "  <-- FAIL"), flush=True)
        release_engines()
        if not ok:
            raise AssertionError(f"case {case} exceeds the parity bounds: {e}")
    print("worst", worst)
    return worst


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 12, int(sys.argv[2]) if len(sys.argv) > 2 else 7)
