"""Randomised GPU-vs-oracle sweep of the 1D hybrid tracking loop (px_hybrid_*, csrc/hybrid.cuh): grid
sizes incl. the cluster sweep (≥ 2048 points), members, slices, equal / geometric partitions, laws,
terminal data, overlap on / off. Not a pytest module; run `python tests/stress_hybrid1d.py [count] [seed]`."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def run(count: int, seed: int) -> dict:
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_system, make_hybrid_plan,
        solve_hybrid_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.errors import PropagationFailure
    from paper_2004_00546_b200.problems import BURGERS
    from paper_2004_00546_b200.tracking import release_tracking_engines
    from tests.test_gpu_hybrid import _oracle
    rng = np.random.default_rng(seed)
    worst = {}
    for case in range(count):
        nx = int(rng.choice([48, 64, 96, 128, 192, 256, 320, 512, 1024, 2048, 4096]))
        B = int(rng.integers(1, 4))
        P = int(rng.integers(1, 13))
        D = float(rng.uniform(0.005, 0.05))
        T = float(rng.uniform(0.1, 0.4))
        lam = 4 * D * (nx / (2 * np.pi)) ** 2 + nx / (2 * np.pi)
        S = max(P, int(np.ceil(T / min(2e-3, 1.0 / lam))))
        rk, cfg = RK4Config(T / S), ChebyshevConfig(tol=1e-12)
        kind = rng.random()
        law = TimeLaw.constant() if kind < 0.25 else (TimeLaw.sine(float(rng.uniform(1, 9))) if kind < 0.6 else
                                                      TimeLaw(*rng.uniform(-1, 1, 3), float(rng.uniform(1, 9))))
        sysm = build_system(Grid(nx), ProblemSpec(BURGERS, (0.0, 0.0), D, T), 4)
        x = sysm.grid.x1()
        mk = lambda: sum(rng.uniform(-.3, .3) * np.sin((m + 1) * x + rng.uniform(0, 6)) for m in range(3))
        u0, f, ft = 0.5 * np.sin(x) + 0.2 * mk(), np.stack([mk() for _ in range(B)]), mk()
        target = synthesize_trajectory(sysm, ft, rk, law, u0=u0)[:, 0, :]
        plan = make_hybrid_plan(T, P, float(rng.uniform(0.5, 8.0))) if P > 1 and rng.random() < 0.6 else None
        qT = 0.1 * np.stack([mk() for _ in range(B)]) if rng.random() < 0.4 else None
        ov = bool(rng.random() < 0.5)
        try:
            r = solve_hybrid_tracking(sysm, u0, f, target, plan, N=P, rk=rk, expaction=cfg, law=law, qdag_T=qT, overlap=ov)
        except (ValueError, PropagationFailure) as err:   # a slice narrower than one step after snapping to the
            # node grid; or a frozen action too stiff for the planner's fp64 rounding budget at tol 1e-12
            print(f"case {case}: nx={nx} P={P} S={S}: skipped ({err})", flush=True)
            release_tracking_engines()
            continue
        o = _oracle(sysm, u0, f, target, r.offsets, law, cfg, qdag_T=qT)
        e = {"J": float(np.max(np.abs(r.J - o.J) / np.abs(o.J))), "grad": rel(r.grad, o.grad), "qdag0": rel(r.qdag0, o.qdag0),
             "uT": rel(r.final_state, o.uT)}
        ok = e["J"] <= 1e-10 and e["grad"] <= 1e-8 and e["qdag0"] <= 1e-9 and e["uT"] <= 1e-10
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
        print(f"case {case}: nx={nx} B={B} P={P} S={S} {'geometric' if plan else 'equal'} qT={qT is not None} overlap={ov}"
              f"/{r.timing['overlapped']}: " + " ".join(f"{k}={v:.1e}" for k, v in e.items()) + ("" if ok else "  <-- FAIL"), flush=True)
        release_tracking_engines()
        if not ok:
            raise AssertionError(f"case {case} exceeds the parity bounds: {e}")
    print("worst", worst)
    return worst


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 12, int(sys.argv[2]) if len(sys.argv) > 2 else 7)
