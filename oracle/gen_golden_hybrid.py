"""Golden vectors of the reference's own hybrid loop — TEST INFRASTRUCTURE ONLY.

Run in the development container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_hybrid.py

Runs the reference, unmodified, through its public loop `direct_adjoint_loop(system, f, q_true,
"hybrid", N, rk, leja, plan=make_hybrid_plan(...))` (`optimization.py:154-231`): tracking
objective (1/T)∫‖q − q_true‖² dt, forcing f·sin(ωt), serial direct sweep, the geometric
partition, the `solve_hybrid` adjoint with the source 2(q − q_true) and its frozen spans, the
gradient (1/T)∫q†·sin(ωt) dt. 1D Burgers is the reference's 2D system on an nx×3 grid with a
y-invariant U and V ≡ 0. Writes ``tests/golden/reference_hybrid_tracking.npz``; the CPU test
(`tests/test_hybrid_cpu.py`) holds the config-mode restatement (oracle.config_mode.
burgers_tracking_hybrid: classical RK4, Chebyshev frozen actions, node trapezoid) to it at the
level of the two discretisations (≤ 1e-4); nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "reference_hybrid_tracking.npz")

NX, T, D, OMEGA, N, K_RATIO = 16, 0.5, 0.05, 2.0 * np.pi, 3, 1.5


def fields(nx):
    x = np.arange(nx) * (2.0 * np.pi / nx)
    f = 0.3 * np.cos(2.0 * x) + 0.2 * np.sin(3.0 * x) + 0.4 * np.sin(x)
    f_true = 0.5 * np.sin(x) + 0.2 * np.cos(x)
    return f, f_true


def main():
    try:
        import paradjoint as R  # the reference
    except ImportError:
        sys.exit("reference not importable: PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_hybrid.py")
    grid = R.Grid2D(NX, 3)
    f1, ft1 = fields(NX)
    emb = lambda u: np.concatenate([np.tile(u, 3), np.zeros(3 * NX)])  # (U y-invariant, V ≡ 0)
    spec = R.ProblemSpec("burgers", 0.0, D, OMEGA, T, emb(np.zeros(NX)))
    system = R.build_system(grid, spec)
    rk = R.RKConfig(rtol=1e-10, atol=1e-13)
    leja = R.LejaConfig(tol=1e-12)
    # the target is evaluated by linear interpolation between its nodes (timestepping.py:64-75):
    # cap the truth's steps so that interpolation stays below the comparison's resolution
    q_true = R.synthesize_truth(system, emb(ft1), R.RKConfig(rtol=1e-10, atol=1e-13, h_max=2.5e-4),
                                algorithm="serial")
    plan = R.make_hybrid_plan(T, N, K_RATIO)
    res = R.direct_adjoint_loop(system, emb(f1), q_true, "hybrid", N=N, rk=rk, leja=leja, plan=plan,
                                probe_nodes=4001)
    g = np.asarray(res.grad)
    gU = g[: 3 * NX].reshape(3, NX)
    qd0 = np.asarray(res.adjoint.eval(0.0))[: 3 * NX].reshape(3, NX)
    uT = np.asarray(res.direct.eval(T))[: 3 * NX].reshape(3, NX)
    np.savez_compressed(OUT, nx=NX, T=T, D=D, omega=OMEGA, N=N, k=K_RATIO, f=f1, f_true=ft1,
                        boundaries=plan.partition.boundaries, J=res.J,
                        # the embedded gradient of a y-invariant control sums the three rows
                        grad_rows=gU, grad=gU.sum(axis=0), qdag0=qd0[0], uT=uT[0],
                        v_grad_max=float(np.max(np.abs(g[3 * NX:]))), probe_nodes=4001, rtol=1e-10)
    print("J", res.J, "|grad|", np.linalg.norm(gU.sum(axis=0)), "->", OUT)


if __name__ == "__main__":
    main()
