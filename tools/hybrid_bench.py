"""Device timing of the hybrid tracking path at config 3's size (1D Burgers, 2048 points,
2000 RK4 steps, 64 slices): the serial direct kernel, the slice solves, what the overlap leaves
after the sweep, the adjoint carry — equidistant vs geometric partitions, overlapped vs
sequential. Prints one JSON line per variant (CUDA events via px_hybrid_get_timing; the
whole-gradient time with events around the public solve on the current stream)."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_system, estimate_k, make_hybrid_plan,
        solve_hybrid_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.problems import BURGERS
    sysm = build_system(Grid(2048), ProblemSpec(BURGERS, (0.0, 0.0), 0.005, 1.0), 16)
    x = sysm.grid.x1()
    rk, cfg, law = RK4Config(5e-4), ChebyshevConfig(tol=1e-12), TimeLaw.sine(2 * np.pi)
    u0 = 0.5 * np.sin(x) + 0.05 * np.cos(3 * x)
    f = 0.3 * np.cos(2 * x) + 0.2 * np.sin(3 * x)
    target_host = synthesize_trajectory(sysm, 0.5 * np.sin(x) + 0.1 * np.cos(2 * x), rk, law)[:, 0, :]
    target = torch.as_tensor(target_host, device="cuda")   # resident target: the timed solve moves no 33 MB H2D
    k = estimate_k(sysm, 0.05, rk, repeats=3, law=law)
    print(json.dumps({"estimate_k": k}), flush=True)
    for name, plan in (("equidistant", None), ("geometric_k", make_hybrid_plan(1.0, 64, max(k, 0.5) * 40.0)),
                       ("geometric_20", make_hybrid_plan(1.0, 64, 20.0))):
        for ov in (False, True):
            for _ in range(2):
                solve_hybrid_tracking(sysm, u0, f, target, plan, N=64, rk=rk, expaction=cfg, law=law, overlap=ov)
            reps = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                a.record()
                r = solve_hybrid_tracking(sysm, u0, f, target, plan, N=64, rk=rk, expaction=cfg, law=law, overlap=ov)
                b.record()
                torch.cuda.synchronize()
                reps.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3, r.timing))
            best = min(reps, key=lambda z: z[0])
            print(json.dumps({"partition": name, "overlap": ov, "gradient_ms_events": best[0],
                              "gradient_ms_wall": best[1], **best[2],
                              "slice_steps": np.diff(r.offsets).tolist()[:4] + ["…"] + np.diff(r.offsets).tolist()[-2:]}),
                  flush=True)


if __name__ == "__main__":
    main()
