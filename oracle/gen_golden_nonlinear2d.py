"""Golden vectors of the reference's loop with algorithm "nonlinear" (the iterative nonlinear
direct, Algorithm 2, + `solve_adjoint_varying`) on its 2D two-field Burgers testbed — TEST
INFRASTRUCTURE ONLY.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_nonlinear2d.py

Runs the reference, unmodified: `direct_adjoint_loop(system, f, q_true, "nonlinear", N, rk, leja,
eps)` (`optimization.py:154-231`, `nonlinear.py:69-194`) with the same fields as
gen_golden_hybrid2d.py. Writes ``tests/golden/reference_nonlinear2d_tracking.npz``; the CPU test
(`tests/test_hybrid2d_cpu.py`) holds oracle.config_mode.burgers2d_nonlinear_tracking to it at the
level of the two discretisations; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "reference_nonlinear2d_tracking.npz")


def main():
    from gen_golden_hybrid2d import D, NX, NY, OMEGA, T, fields
    try:
        import paradjoint as R  # the reference
    except ImportError:
        sys.exit("reference not importable: PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_nonlinear2d.py")
    N, EPS = 4, 1e-9
    grid = R.Grid2D(NX, NY)
    f, f_true = fields(NX, NY)
    spec = R.ProblemSpec("burgers", 0.0, D, OMEGA, T, np.zeros(2 * NX * NY))
    system = R.build_system(grid, spec)
    rk = R.RKConfig(rtol=1e-10, atol=1e-13)
    leja = R.LejaConfig(tol=1e-12)
    q_true = R.synthesize_truth(system, f_true, R.RKConfig(rtol=1e-10, atol=1e-13, h_max=2.5e-4),
                                algorithm="serial")
    res = R.direct_adjoint_loop(system, f, q_true, "nonlinear", N=N, rk=rk, leja=leja, eps=EPS, probe_nodes=4001)
    np.savez_compressed(OUT, nx=NX, ny=NY, T=T, D=D, omega=OMEGA, N=N, eps=EPS, f=f, f_true=f_true, J=res.J,
                        grad=np.asarray(res.grad), qdag0=np.asarray(res.adjoint.eval(0.0)),
                        uT=np.asarray(res.direct.eval(T)), iterations=res.iterations,
                        history=np.asarray(res.error_history), probe_nodes=4001, rtol=1e-10)
    print("J", res.J, "|grad|", np.linalg.norm(res.grad), "sweeps", res.iterations, "->", OUT)


if __name__ == "__main__":
    main()
