"""Generate golden vectors from the REFERENCE implementation — TEST INFRASTRUCTURE ONLY.

Run in the development container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

It imports ``paradjoint`` (the reference, unmodified), runs its own functions on
small seeded inputs and writes ``tests/golden/reference_*.npz``. The CPU tests
(`tests/test_reference_pin.py`) then check the oracle's restatements against
these files; nothing at test time reads /root/reference. The fixtures pin:

* the stencil operators: `build_advdiff_operator` apply / transpose-apply
  (`problems.py:149-152`, `linalg.py:70-74`), including the 1D embedding nx×3;
* Burgers: `burgers_rhs`, `burgers_adjoint_apply`, `average_jacobian`
  (`problems.py:177-185,316-366`) on y-invariant states with V ≡ 0;
* `rk45_integrate` nodes/states with waypoints (`timestepping.py:128-203`);
* `leja_points`, `spectral_interval`, `relpm_propagate(record=m)` (`:235-423`);
* `solve_direct_linear` / `solve_adjoint_linear` pieces for N ∈ {1, 2, 3}
  (`paraexp.py:221-326`) — the Paraexp superposition structure;
* `Trajectory.eval_many` linear interpolation (`timestepping.py:64-75`);
* `solve_hybrid` with a final condition and no adjoint source (`hybrid.py:194-237`):
  q† at the slice edges of a geometric partition, with the slices' trapezoid means ū_p.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def main():
    try:
        import paradjoint as R  # the reference
    except ImportError:
        sys.exit("reference not importable: PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py")
    from paradjoint.problems import grid_operators  # noqa: F401
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20040546)

    # 1. stencil operators -------------------------------------------------------
    g2 = R.Grid2D(8, 6)
    A2 = R.build_advdiff_operator(g2, 0.7, 0.3)
    x2 = rng.standard_normal(g2.npoints)
    g1 = R.Grid2D(16, 3)
    A1 = R.build_advdiff_operator(g1, 1.3, 0.05)
    x1 = np.tile(rng.standard_normal(16), 3)  # y-invariant
    np.savez_compressed(os.path.join(OUT, "reference_stencil.npz"),
             nx2=8, ny2=6, a2=0.7, D2=0.3, x2=x2, Ax2=A2.apply(x2), ATx2=A2.transpose_apply(x2),
             nx1=16, a1=1.3, D1=0.05, x1=x1[:16], Ax1=A1.apply(x1)[:16], ATx1=A1.transpose_apply(x1)[:16])

    # 2. Burgers (1D embedded as nx×3, V ≡ 0) ------------------------------------
    nb = 12
    gb = R.Grid2D(nb, 3)
    U = 0.4 * rng.standard_normal(nb)
    fU = 0.2 * rng.standard_normal(nb)
    yb = rng.standard_normal(nb)
    n3 = gb.npoints
    f_sp = np.concatenate([np.tile(fU, 3), np.zeros(n3)])
    spec = R.ProblemSpec(R.BURGERS, a=1.0, D=0.2, omega=1.0, T=1.0, f_spatial=f_sp)
    q = np.concatenate([np.tile(U, 3), np.zeros(n3)])
    rhs = R.burgers_rhs(gb, spec, q, np.pi / 2)  # sin(ωt) = 1
    yv = np.concatenate([np.tile(yb, 3), np.zeros(n3)])
    adj = R.burgers_adjoint_apply(gb, spec, q, yv)
    tnodes = np.sort(rng.uniform(0.0, 1.0, 5))
    tstates1d = 0.4 * rng.standard_normal((5, nb))
    traj = R.Trajectory(tnodes, np.stack([np.concatenate([np.tile(s, 3), np.zeros(n3)]) for s in tstates1d]))
    avgJT_y = R.average_jacobian(traj, gb, spec).transpose().apply(yv)
    diffT_y = R.burgers_nonlinear_split(gb, spec)[0].transpose().apply(yv)
    mids = 0.5 * (tnodes[:-1] + tnodes[1:])
    np.savez_compressed(os.path.join(OUT, "reference_burgers.npz"),
             nx=nb, D=0.2, U=U, f=fU, y=yb, rhs=rhs[:nb], rhs_V=rhs[n3:n3 + nb], adj=adj[:nb],
             adj_b=adj[n3:n3 + nb], tnodes=tnodes, tstates=tstates1d, frozenT_y=(avgJT_y + diffT_y)[:nb],
             mids=mids, interp=traj.eval_many(mids)[:, :nb])

    # 3. DOPRI5 with waypoints ---------------------------------------------------
    g4 = R.Grid2D(4, 4)
    A4 = R.build_advdiff_operator(g4, 1.0, 0.5)
    f4 = rng.standard_normal(16)
    y0 = rng.standard_normal(16)
    rk = R.RKConfig(rtol=1e-6)
    wps = np.linspace(0.0, 0.7, 6)[1:-1]
    tr = R.rk45_integrate(lambda t, y: A4.matrix @ y + f4 * np.sin(1.3 * t), y0, 0.0, 0.7, rk, waypoints=wps)
    np.savez_compressed(os.path.join(OUT, "reference_dopri5.npz"), f=f4, y0=y0, wps=wps, nodes=tr.nodes, states=tr.states,
             rtol=1e-6)

    # 4. Leja / ReLPM --------------------------------------------------------------
    g6 = R.Grid2D(6, 6)
    A6 = R.build_advdiff_operator(g6, 1.0, 1.0)
    v6 = rng.standard_normal(36)
    lc = R.LejaConfig(tol=1e-8)
    end, rec = R.relpm_propagate(A6, v6, 0.3, lc, record=3)
    np.savez_compressed(os.path.join(OUT, "reference_leja.npz"), leja12=R.leja_points(12),
             interval=np.array(R.spectral_interval(A6)), v=v6, end=end, rec=rec, tol=1e-8, dt=0.3)

    # 5. Paraexp direct / adjoint pieces -----------------------------------------
    q0 = rng.standard_normal(36)
    f0 = rng.standard_normal(36)
    qT = rng.standard_normal(36)
    s0 = rng.standard_normal(36)
    out = {"q0": q0, "f0": f0, "qT": qT, "s0": s0, "rtol": 1e-4, "tol": 1e-6, "T": 2.0, "omega": 1.3}
    for N in (1, 2, 3):
        part = R.partition_equidistant(2.0, N)
        d = R.solve_direct_linear(A6, q0, lambda t: f0 * np.sin(1.3 * t), part, R.RKConfig(rtol=1e-4),
                                  R.LejaConfig(tol=1e-6))
        a = R.solve_adjoint_linear(A6, qT, lambda t: s0 * np.cos(2.0 * t), part, R.RKConfig(rtol=1e-4),
                                   R.LejaConfig(tol=1e-6))
        for p in range(N):
            out[f"d{N}_{p}_nodes"] = d.pieces[p].nodes
            out[f"d{N}_{p}_states"] = d.pieces[p].states
            out[f"a{N}_{p}_nodes"] = a.pieces[p].nodes
            out[f"a{N}_{p}_states"] = a.pieces[p].states
    np.savez_compressed(os.path.join(OUT, "reference_paraexp.npz"), **out)

    # 6. solve_hybrid with a final condition and no adjoint source (hybrid.py:194-237) --
    # the terminal objective's case: the inhomogeneous adjoint solves vanish and q† is
    # q†_T carried back through the frozen interval operators (`propagate_span`)
    nh = 12
    gh = R.Grid2D(nh, 3)
    n3h = gh.npoints
    xh = 2.0 * np.pi * np.arange(nh) / nh
    f_h = np.concatenate([np.tile(0.3 * np.sin(2.0 * xh), 3), np.zeros(n3h)])
    spec_h = R.ProblemSpec(R.BURGERS, a=1.0, D=0.2, omega=1.0, T=1.0, f_spatial=f_h)
    sys_h = R.build_system(gh, spec_h)
    q0_h = np.concatenate([np.tile(0.5 * np.sin(xh), 3), np.zeros(n3h)])
    qT1 = rng.standard_normal(nh)
    qT_h = np.concatenate([np.tile(qT1, 3), np.zeros(n3h)])
    plan_h = R.make_hybrid_plan(1.0, 3, 1.5)
    res = R.solve_hybrid(sys_h, q0_h, qT_h, lambda t, q: np.zeros_like(q), plan_h,
                         R.RKConfig(rtol=1e-10), R.LejaConfig(tol=1e-12))
    bnd = plan_h.partition.boundaries
    ubar = []
    for piece in res.direct.pieces:  # the trapezoid mean of each slice (average_jacobian's weights)
        w = np.zeros(len(piece.nodes))
        gaps = np.diff(piece.nodes)
        w[:-1] += 0.5 * gaps
        w[1:] += 0.5 * gaps
        ubar.append((w @ piece.states)[:nh] / (piece.nodes[-1] - piece.nodes[0]))
    qstart = np.stack([pc.states[0][:nh] for pc in res.adjoint.pieces])   # q†(T_m)
    qend = np.stack([pc.states[-1][:nh] for pc in res.adjoint.pieces])    # q†(T_{m+1}⁻)
    vmax = max(float(np.max(np.abs(pc.states[:, n3h:]))) for pc in res.adjoint.pieces)
    np.savez_compressed(os.path.join(OUT, "reference_hybrid.npz"), nx=nh, D=0.2, boundaries=bnd,
                        ubar=np.stack(ubar), qT=qT1, qstart=qstart, qend=qend, vmax=vmax)
    print("wrote", sorted(f for f in os.listdir(OUT) if f.startswith("reference_")))


if __name__ == "__main__":
    main()
