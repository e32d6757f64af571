"""Device timing of the hybrid tracking path on the reference's own 2D two-field Burgers testbed
(csrc/hybrid2d.cu): the reference's `configs/burgers_hybrid.json` shape (32×32, D = 1, ω = 1,
T = 1) and larger grids; sequential vs stream-overlapped slice solves; whole-gradient time with
events around the public solve. Prints one JSON line per variant. (The CPU oracle's time for the
same gradients: tests/time_hybrid2d_vs_oracle.py — only tests/ may run the oracle.)"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(nx, ny, D, T, dt, P, k, with_oracle=False):
    import torch

    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system, make_hybrid_plan,
        solve_hybrid_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.problems import BURGERS
    sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), D, T))
    X, Y = sysm.grid.coordinates()
    rk, cfg, law = RK4Config(dt), ChebyshevConfig(tol=1e-12), TimeLaw.sine(1.0)
    f_true = np.concatenate([np.sin(X) * np.sin(Y)] * 2)
    f = np.ones(sysm.n)
    u0 = np.zeros(sysm.n)
    target_host = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    target = torch.as_tensor(target_host, device="cuda")
    plan = make_hybrid_plan(T, P, k)
    for ov in (False, True):
        for _ in range(2):
            solve_hybrid_tracking(sysm, u0, f, target, plan, rk=rk, expaction=cfg, law=law, overlap=ov)
        reps = []
        for _ in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a.record()
            r = solve_hybrid_tracking(sysm, u0, f, target, plan, rk=rk, expaction=cfg, law=law, overlap=ov)
            b.record()
            torch.cuda.synchronize()
            reps.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3, r.timing))
        best = min(reps, key=lambda z: z[0])
        S = int(r.offsets[-1])
        terms = sum(p.substeps * p.degree for p in r.plans[:-1])
        print(json.dumps({"grid": [nx, ny], "steps": S, "slices": P, "k": k, "overlap": ov,
                          "gradient_ms_events": best[0], "gradient_ms_wall": best[1], **best[2],
                          "frozen_terms": terms, "J": float(r.J[0])}), flush=True)
    return sysm, u0, f, law, cfg, target_host, r


def run_nonlinear(nx, ny, D, T, dt, P, eps, with_oracle=False):
    """The reference's `configs/burgers_iterative.json` shape: Algorithm 2 + the zero-terminal adjoint."""
    import torch

    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system, solve_nonlinear_tracking,
        synthesize_trajectory)
    from paper_2004_00546_b200.problems import BURGERS
    sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), D, T))
    X, Y = sysm.grid.coordinates()
    rk, cfg, law = RK4Config(dt), ChebyshevConfig(tol=1e-12), TimeLaw.sine(1.0)
    f_true = np.concatenate([np.sin(X) * np.sin(Y)] * 2)
    f = np.ones(sysm.n)
    u0 = np.zeros(sysm.n)
    target = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    for _ in range(2):
        solve_nonlinear_tracking(sysm, u0, f, target, N=P, rk=rk, expaction=cfg, law=law, eps=eps)
    reps = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = solve_nonlinear_tracking(sysm, u0, f, target, N=P, rk=rk, expaction=cfg, law=law, eps=eps)
        torch.cuda.synchronize()
        reps.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps({"grid": [nx, ny], "algorithm": "nonlinear", "slices": P, "steps": int(r.offsets[-1]), "eps": eps,
                      "sweeps": len(r.timing["history"]), "gradient_ms_wall": min(reps), "J": float(r.J[0])}), flush=True)
    return sysm, u0, f, law, cfg, target, r


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "large":   # the 512×512 per-stage-launch case only (ncu captures)
        run(512, 512, 0.01, 0.2, 1e-3, 8, 3.0)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "small":   # the 32×32 hybrid case only (ncu captures)
        run(32, 32, 1.0, 1.0, 1e-3, 16, 3.0, False)
        sys.exit(0)
    run_nonlinear(32, 32, 1.0, 1.0, 1e-3, 8, 1e-3)   # the reference's burgers_iterative.json shape
    run(32, 32, 1.0, 1.0, 1e-3, 16, 3.0)      # the reference's burgers_hybrid.json shape
    run(128, 128, 0.05, 0.5, 1e-3, 16, 3.0, False)
    run(512, 512, 0.01, 0.2, 1e-3, 8, 3.0, False)
