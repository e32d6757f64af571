"""Randomised GPU-vs-oracle sweep of the 1D paths (configs 1–3 shapes): the linear gradient (on-chip RK4
lanes, Chebyshev scans incl. the 8-CTA cluster scan) and the Burgers gradient (serial sweep incl. the
cluster sweep, time-varying adjoint, frozen carry) over grid sizes, slices, steps, members and modes.
Not a pytest module; run `python tests/stress_1d.py [count] [seed]` on a GPU box."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def run(count: int, seed: int) -> dict:
    from oracle.config_mode import burgers_gradient
    from paper_2004_00546_b200 import RK4Config, baseline, direct_adjoint_loop, release_engines, scaled
    from paper_2004_00546_b200.expaction import plan_chebyshev
    from paper_2004_00546_b200.problems import burgers_frozen_region
    from tests.test_gpu_parity import _gpu_linear, _oracle_linear
    rng = np.random.default_rng(seed)
    worst = {}
    for case in range(count):
        burgers = rng.random() < 0.45
        nx = int(rng.choice([64, 96, 128, 160, 256, 384, 512, 768, 1024, 2048, 3072, 4096]))
        P = int(rng.integers(2, 17))
        steps = int(rng.integers(3, 12))
        K = 2 * int(rng.integers(1, 9))
        B = int(rng.integers(1, 5))
        # a stable RK4 step for the finest grid's diffusion + advection scale
        h = float(rng.uniform(0.5, 1.0)) / (4 * 0.01 * (nx / (2 * np.pi)) ** 2 + nx / (2 * np.pi))
        T = P * steps * min(h, 0.3 / (P * steps))   # (and a horizon ≤ 0.3: the forced Burgers flow stays smooth)
        if burgers:
            c = scaled(baseline(3), nx=nx, P=P, steps_per_slice=steps, K=K, batch=B, T=T)
            u0, ut, ctrl = c.inputs()
            loop = direct_adjoint_loop(c.system, ctrl, ut, "hybrid", N=c.P, rk=RK4Config(c.dt), expaction=c.expaction, u0=u0)
            ref = burgers_gradient(c.grid.nx, c.spec.D, c.system.basis, c.spec.T, c.P, c.nsteps, u0, ut, ctrl,
                                   lambda region, span: plan_chebyshev(region, span, c.expaction),
                                   lambda ub: burgers_frozen_region(ub, c.grid, c.spec.D))
        else:
            c = scaled(baseline(int(rng.choice([1, 2]))), nx=nx, P=P, steps_per_slice=steps, K=K, batch=B, T=T)
            loop, ref = _gpu_linear(c), _oracle_linear(c)
        Bn = np.atleast_2d(loop.grad).shape[0]
        e = {"uT": rel(loop.direct.final_state, ref.uT), "qdag0": rel(loop.adjoint.initial_state, ref.qdag0),
             "G": rel(loop.adjoint.integral, ref.G), "grad": rel(np.reshape(loop.grad, (Bn, -1)), ref.grad),
             "J": float(np.max(np.abs(np.ravel(loop.J) - ref.J) / np.abs(ref.J)))}
        ok = e["uT"] <= 1e-10 and e["qdag0"] <= 1e-10 and e["G"] <= 1e-10 and e["grad"] <= 1e-8 and e["J"] <= 1e-10
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
        print(f"case {case}: {'burgers' if burgers else 'linear'} nx={nx} P={P} steps={steps} K={K} B={B}: " +
              " ".join(f"{k}={v:.1e}" for k, v in e.items()) + ("" if ok else "  <-- FAIL"), flush=True)
        release_engines()
        if not ok:
            raise AssertionError(f"case {case} exceeds the parity bounds: {e}")
    print("worst", worst)
    return worst


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 12, int(sys.argv[2]) if len(sys.argv) > 2 else 7)
