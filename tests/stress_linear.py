"""Randomised GPU-vs-oracle sweep of the linear Paraexp gradient (the BASELINE path) over non-square
grids, slice / step counts, batch sizes, mode counts and kernel variants (one- / two-step march, 2 or 3
columns per thread, Chebyshev terms per pass, Chebyshev / Krylov). Not a pytest module; run
`python tests/stress_linear.py [count] [seed]` on a GPU box."""

import os
import sys
from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def run(count: int, seed: int) -> dict:
    from paper_2004_00546_b200 import Grid, RK4Config, baseline, release_engines, scaled
    from paper_2004_00546_b200.optimization import get_engine
    from tests.test_gpu_parity import _gpu_linear, _oracle_linear
    rng = np.random.default_rng(seed)
    worst = {}
    for case in range(count):
        krylov = rng.random() < 0.25
        base = baseline(4 if krylov else 5)
        nx = 2 * int(rng.integers(8, 330 if not krylov else 100))
        ny = int(rng.integers(8, 300 if not krylov else 100))
        P = int(rng.integers(2, 10))
        steps = int(rng.integers(3, 10))
        K = int(rng.choice([4, 16, 36]))
        B = int(rng.integers(1, 4))
        c = scaled(base, nx=nx, P=P, steps_per_slice=steps, K=K, batch=B, T=float(rng.uniform(0.02, 0.2)))
        c = replace(c, grid=Grid(nx, ny))
        var = {"march2": int(rng.choice([0, 2])), "march_cols": int(rng.choice([2, 3])),
               "cheb_terms": int(rng.integers(1, 8)), "cheb_terms_phi": int(rng.integers(1, 6))}
        eng = get_engine(c.system, c.P, RK4Config(c.dt), c.expaction, c.batch)
        for k, v in var.items():
            eng.set_variant(k, v)
        loop, ref = _gpu_linear(c), _oracle_linear(c)
        Bn = np.atleast_2d(loop.grad).shape[0]
        e = {"uT": rel(loop.direct.final_state, ref.uT), "qdag0": rel(loop.adjoint.initial_state, ref.qdag0),
             "G": rel(loop.adjoint.integral, ref.G), "grad": rel(np.reshape(loop.grad, (Bn, -1)), ref.grad),
             "J": float(np.max(np.abs(np.ravel(loop.J) - ref.J) / np.abs(ref.J)))}
        ok = e["uT"] <= 1e-10 and e["qdag0"] <= 1e-10 and e["G"] <= 1e-10 and e["grad"] <= 1e-8 and e["J"] <= 1e-10
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
        print(f"case {case}: {'krylov' if krylov else 'cheb'} {nx}x{ny} P={P} steps={steps} K={c.K} B={B} {var}: " +
              " ".join(f"{k}={v:.1e}" for k, v in e.items()) + ("" if ok else "  <-- FAIL"), flush=True)
        release_engines()
        if not ok:
            raise AssertionError(f"case {case} exceeds the parity bounds: {e}")
    print("worst", worst)
    return worst


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 12, int(sys.argv[2]) if len(sys.argv) > 2 else 7)
