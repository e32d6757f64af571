"""Golden vectors of the reference's hybrid loop on its 2D two-field Burgers testbed — TEST
INFRASTRUCTURE ONLY.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_hybrid2d.py

Runs the reference, unmodified, through `direct_adjoint_loop(system, f, q_true, "hybrid", N, rk,
leja, plan=make_hybrid_plan(...))` (`optimization.py:154-231`) on `ProblemSpec("burgers", …)` with
genuinely two-dimensional fields (U and V both active, forcing on both components,
`problems.py:177-186`): tracking objective, forcing f·sin(ωt), serial direct sweep, geometric
partition, the `solve_hybrid` adjoint with the source 2(q − q_true) and its frozen spans
(`hybrid.py:185-237`). Writes ``tests/golden/reference_hybrid2d_tracking.npz``; the CPU test
(`tests/test_hybrid2d_cpu.py`) holds the config-mode restatement
(oracle.config_mode.burgers_tracking_hybrid with ``ny``) to it at the level of the two
discretisations; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "reference_hybrid2d_tracking.npz")

NX, NY, T, D, OMEGA, N, K_RATIO = 10, 8, 0.5, 0.05, 2.0 * np.pi, 3, 1.5


def fields(nx, ny):
    x = np.arange(nx) * (2.0 * np.pi / nx)
    y = np.arange(ny) * (2.0 * np.pi / ny)
    X, Y = np.meshgrid(x, y, indexing="xy")  # (ny, nx), x fastest
    fu = 0.3 * np.cos(2.0 * X) * np.sin(Y) + 0.4 * np.sin(X) + 0.1 * np.cos(Y)
    fv = 0.25 * np.sin(X) * np.sin(Y) - 0.2 * np.cos(X + Y)
    tu = 0.5 * np.sin(X) * np.sin(Y) + 0.2 * np.cos(X)
    tv = 0.3 * np.sin(X) * np.sin(Y) + 0.1 * np.sin(2.0 * Y)
    return np.concatenate([fu.ravel(), fv.ravel()]), np.concatenate([tu.ravel(), tv.ravel()])


def main():
    try:
        import paradjoint as R  # the reference
    except ImportError:
        sys.exit("reference not importable: PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_hybrid2d.py")
    grid = R.Grid2D(NX, NY)
    f, f_true = fields(NX, NY)
    spec = R.ProblemSpec("burgers", 0.0, D, OMEGA, T, np.zeros(2 * NX * NY))
    system = R.build_system(grid, spec)
    rk = R.RKConfig(rtol=1e-10, atol=1e-13)
    leja = R.LejaConfig(tol=1e-12)
    q_true = R.synthesize_truth(system, f_true, R.RKConfig(rtol=1e-10, atol=1e-13, h_max=2.5e-4),
                                algorithm="serial")
    plan = R.make_hybrid_plan(T, N, K_RATIO)
    res = R.direct_adjoint_loop(system, f, q_true, "hybrid", N=N, rk=rk, leja=leja, plan=plan, probe_nodes=4001)
    np.savez_compressed(OUT, nx=NX, ny=NY, T=T, D=D, omega=OMEGA, N=N, k=K_RATIO, f=f, f_true=f_true,
                        boundaries=plan.partition.boundaries, J=res.J, grad=np.asarray(res.grad),
                        qdag0=np.asarray(res.adjoint.eval(0.0)), uT=np.asarray(res.direct.eval(T)),
                        probe_nodes=4001, rtol=1e-10)
    print("J", res.J, "|grad|", np.linalg.norm(res.grad), "->", OUT)


if __name__ == "__main__":
    main()
