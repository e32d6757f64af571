"""Golden vectors of the reference's own LINEAR loop — TEST INFRASTRUCTURE ONLY.

Run in the development container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_linear_tracking.py

Runs the reference, unmodified, through its public loop `direct_adjoint_loop(system, f, q_true,
"linear", N, rk, leja)` (`optimization.py:154-231`) on its advection–diffusion testbed: Paraexp
direct with the forcing f·sin(ωt) from q(0) = 0, the tracking objective (1/T)∫‖q − q_true‖² dt,
`solve_adjoint_linear` with the source 2(q − q_true) and q†(T) = 0, the gradient
(1/T)∫q†·sin(ωt) dt (probe-grid trapezoids). q_true is the reference's `synthesize_truth` of a
second forcing field. Writes ``tests/golden/reference_linear_tracking.npz``; the CPU test
(`tests/test_tracking_cpu.py`) holds the config-mode restatement (oracle.config_mode.
linear_tracking_gradient: classical RK4, Chebyshev carries, node trapezoid) to it at the level of
the two discretisations, the GPU test (`tests/test_gpu_tracking.py`) the device path; nothing at
test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "reference_linear_tracking.npz")

NX, NY, A, D, OMEGA, T, N = 12, 10, 0.7, 0.05, 3.0, 0.4, 2
PROBE = 4001


def fields(nx, ny):
    x = np.arange(nx) * (2.0 * np.pi / nx)
    y = np.arange(ny) * (2.0 * np.pi / ny)
    X, Y = np.meshgrid(x, y)   # x fastest (row-major ny × nx)
    f = (0.6 * np.sin(X) * np.cos(Y) + 0.3 * np.cos(2.0 * X) + 0.2 * np.sin(Y)).ravel()
    f_true = (0.5 * np.cos(X) * np.sin(Y) + 0.4 * np.sin(X + Y)).ravel()
    return f, f_true


def main():
    try:
        import paradjoint as R  # the reference
    except ImportError:
        sys.exit("reference not importable: PYTHONPATH=/root/reference/pkg/src python "
                 "oracle/gen_golden_linear_tracking.py")
    grid = R.Grid2D(NX, NY)
    f, f_true = fields(NX, NY)
    spec = R.ProblemSpec("advection_diffusion", A, D, OMEGA, T, np.zeros(grid.npoints))
    system = R.build_system(grid, spec)
    rk = R.RKConfig(rtol=1e-11, atol=1e-14)
    leja = R.LejaConfig(tol=1e-13)
    # the target is evaluated by linear interpolation between its nodes (timestepping.py:64-75):
    # cap the truth's steps so that interpolation stays below the comparison's resolution
    q_true = R.synthesize_truth(system, f_true, R.RKConfig(rtol=1e-11, atol=1e-14, h_max=2.5e-4),
                                leja=leja, algorithm="serial")
    res = R.direct_adjoint_loop(system, f, q_true, "linear", N=N, rk=rk, leja=leja, probe_nodes=PROBE)
    np.savez_compressed(OUT, nx=NX, ny=NY, a=A, D=D, omega=OMEGA, T=T, N=N, f=f, f_true=f_true, J=res.J,
                        grad=np.asarray(res.grad), qdag0=np.asarray(res.adjoint.eval(0.0)),
                        uT=np.asarray(res.direct.eval(T)), probe_nodes=PROBE, rtol=1e-11)
    print("J", res.J, "|grad|", np.linalg.norm(res.grad), "->", OUT)


if __name__ == "__main__":
    main()
