"""GPU vs CPU-oracle wall time of one gradient on the reference's 32×32 two-field Burgers configs
(`configs/burgers_hybrid.json`, `configs/burgers_iterative.json` shapes) — the numbers quoted in
DESIGN.md §3.5. Not a pytest module (the oracle is test infrastructure: only tests/ may run it);
run with `python tests/time_hybrid2d_vs_oracle.py` on a GPU box."""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import hybrid2d_bench as hb
    from oracle.config_mode import burgers2d_nonlinear_tracking, burgers_tracking_hybrid
    from paper_2004_00546_b200.expaction import plan_chebyshev, plan_family
    from paper_2004_00546_b200.problems import frozen_bounds_2d, frozen_region_from_bounds
    nx = ny = 32
    D, T = 1.0, 1.0
    sysm, u0, f, law, cfg, target, r = hb.run(nx, ny, D, T, 1e-3, 16, 3.0, False)
    offs = r.offsets
    P = len(offs) - 1
    h = T / offs[-1]
    reg = lambda q: frozen_region_from_bounds(*frozen_bounds_2d(q, sysm.grid, D))
    t0 = time.perf_counter()
    o = burgers_tracking_hybrid(nx, D, T, offs, u0, f[None, :], law.as_tuple(), target,
                                lambda q: plan_family(reg(q), [(offs[p + 1] - offs[p]) * h for p in range(P)], cfg,
                                                      omega=law.omega), ny=ny)
    print(json.dumps({"algorithm": "hybrid", "cpu_oracle_s": time.perf_counter() - t0, "cores": 1,
                      "J_rel": abs(o.J[0] - r.J[0]) / abs(o.J[0]),
                      "grad_rel": float(np.linalg.norm(o.grad - r.grad) / np.linalg.norm(o.grad))}), flush=True)
    sysm, u0, f, law, cfg, target, r = hb.run_nonlinear(nx, ny, D, T, 1e-3, 8, 1e-3, False)
    P, nsteps = 8, int(r.offsets[1])
    h = T / (P * nsteps)
    t0 = time.perf_counter()
    o = burgers2d_nonlinear_tracking(nx, ny, D, T, P, nsteps, u0, f[None, :], law.as_tuple(), target,
                                     lambda q: (plan_chebyshev(reg(q), T / P, cfg), plan_chebyshev(reg(q), h, cfg)),
                                     lambda q: plan_family(reg(q), [T / P] * P, cfg, omega=law.omega), 1e-3)
    print(json.dumps({"algorithm": "nonlinear", "cpu_oracle_s": time.perf_counter() - t0, "cores": 1,
                      "sweeps": o.extras["sweeps"], "J_rel": abs(o.J[0] - r.J[0]) / abs(o.J[0]),
                      "grad_rel": float(np.linalg.norm(o.grad - r.grad) / np.linalg.norm(o.grad))}), flush=True)


if __name__ == "__main__":
    main()
