"""The CPU reference path for bench.py — TEST INFRASTRUCTURE ONLY (the baseline, never the product).

A full-work CPU gradient with the oracle's arithmetic (``oracle.config_mode``: classical RK4
``rk4_linear``, the planned Chebyshev / Krylov actions ``exp_action``), parallelised like the
reference's time-slice workers (`workers.py:298-346`): W host processes, each owning a
contiguous block of slices. Unlike ``config_mode.linear_gradient`` — which solves the one
slice problem the BASELINE configs' identical slices share and reuses it — every worker
solves EVERY one of its slice problems, as Paraexp does (`paraexp.py:187-218`): the work
timed here is the work the GPU does. Workers combine their slices by the block-scan (each
block's summed-chain carry, then one long span to the horizon), the partials
are summed in the parent.

Two uses:

* ``full_gradient(case, W)``: one complete gradient (J, ∂J/∂c, u(T), q†(0), ∫q†) — configs 1–3
  in ``bench.py --impl reference`` (seconds each), and the offline validation run
  ``oracle/time_fullsize_cpu.py`` for configs 4/5 (tens of minutes on a host);
* ``sampled_rate(case, W)``: the bounded per-step sample for configs 4/5 — every worker times
  a few units of each kind (an RK4 step of a direct lane, of an adjoint lane with its ∫, one
  slice action with and without the φ₁ accumulator) on the full-size field, concurrently;
  one gradient's time is the slowest worker's Σ units × unit time, the units counted
  exactly from the worker's slice block and plans.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import platform
import time

import numpy as np

from oracle.config_mode import exp_action, rk4_linear, stencil_apply


def _limit_threads():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"


def field_separable(basis, ctrl) -> np.ndarray:
    """f = Σ_k c_k φ_k from the separable factor tables (no K×n matrix): (B, K) → (B, n)."""
    ctrl = np.atleast_2d(ctrl)
    tx, ty, ix, iy = basis.tx, basis.ty, basis.ix, basis.iy
    out = np.empty((ctrl.shape[0], ty.shape[1] * tx.shape[1]))
    for b in range(ctrl.shape[0]):
        F = (ty[iy].T * ctrl[b][None, :]) @ tx[ix]          # (ny, K)·(K, nx)
        out[b] = F.ravel()
    return out


def project_separable(basis, G) -> np.ndarray:
    """⟨φ_k, G⟩ for (B, n) → (B, K) from the factor tables."""
    G = np.atleast_2d(G)
    tx, ty, ix, iy = basis.tx, basis.ty, basis.ix, basis.iy
    ny, nx = ty.shape[1], tx.shape[1]
    out = np.empty((G.shape[0], basis.K))
    for b in range(G.shape[0]):
        R = G[b].reshape(ny, nx) @ tx.T                     # (ny, rows_x)
        out[b] = np.einsum("kj,jk->k", ty[iy], R[:, ix])
    return out


def _plans(case):
    from paper_2004_00546_b200.expaction import plan_for
    region = case.system.region()
    delta = case.spec.T / case.P
    return plan_for(region, delta, case.expaction), (lambda span: plan_for(region, span, case.expaction,
                                                                            base_span=delta))


def _ops(case):
    A = case.system.A.as_tuple()
    AT = tuple(np.asarray(A)[[0, 2, 1, 4, 3]])
    nx, ny = case.grid.nx, case.grid.ny
    return (lambda u: stencil_apply(A, u, nx, ny)), (lambda u: stencil_apply(AT, u, nx, ny))


def _direct_block(args):
    """Worker w: RK4 every slice of its block (lane p from zero data), summed-chain carry
    D ← exp(ΔA)D + v_p interleaved, then the long span to T. Returns the partial of u(T) − u0."""
    _limit_threads()
    case, rank, world, sp, lng = args
    from paper_2004_00546_b200.partition import rank_block
    u0, ut, ctrl = case.inputs()
    applyA, _ = _ops(case)
    p0, p1 = rank_block(case.P, rank, world)
    h = case.spec.T / case.P / case.nsteps
    g = applyA(np.broadcast_to(u0, (ctrl.shape[0], u0.size))) + field_separable(case.system.basis, ctrl)
    D = None
    for p in range(p0, p1):
        v, _ = rk4_linear(applyA, g, h, case.nsteps)
        D = v if D is None else exp_action(applyA, sp, D) + v
    if lng is not None:
        D = exp_action(applyA, lng, D)
    return D


def _adjoint_block(args):
    """Worker w: adjoint RK4 of every slice (absorbed q†_T, reflected time, ∫ accumulated
    RK4-consistently), backward carry with the φ₁ accumulator, long span to 0."""
    _limit_threads()
    case, rank, world, qT, sp, lng = args
    from paper_2004_00546_b200.partition import rank_block
    _, applyAT = _ops(case)
    p0, p1 = rank_block(case.P, rank, world)
    h = case.spec.T / case.P / case.nsteps
    gadj = applyAT(qT)
    C = None
    Gp = np.zeros_like(qT)
    for p in range(p1 - 1, p0 - 1, -1):
        w, z = rk4_linear(applyAT, gadj, h, case.nsteps, want_z=True)
        Gp += z
        C = w if C is None else exp_action(applyAT, sp, C, Gp) + w
    if lng is not None:
        C = exp_action(applyAT, lng, C, Gp)
    return C, Gp


def full_gradient(case, workers: int):
    """One complete CPU gradient of the linear testbed with W worker processes."""
    from paper_2004_00546_b200.partition import rank_block
    workers = max(1, min(workers, case.P))
    u0, ut, ctrl = case.inputs()
    sp, lp = _plans(case)
    delta = case.spec.T / case.P
    blocks = [rank_block(case.P, r, workers) for r in range(workers)]
    ldir = [lp((case.P - p1) * delta) if p1 < case.P else None for p0, p1 in blocks]
    ladj = [lp(p0 * delta) if p0 > 0 else None for p0, p1 in blocks]
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        parts = pool.map(_direct_block, [(case, r, workers, sp, ldir[r]) for r in range(workers)])
        uT = u0[None, :] + sum(parts)
        qT = uT - ut[None, :]
        J = 0.5 * np.sum(qT * qT, axis=1)
        adj = pool.map(_adjoint_block, [(case, r, workers, qT, sp, ladj[r]) for r in range(workers)])
    qdag0 = qT + sum(a[0] for a in adj)
    G = case.spec.T * qT + sum(a[1] for a in adj)
    grad = project_separable(case.system.basis, G)
    return {"J": J, "grad": grad, "uT": uT, "qdag0": qdag0, "G": G}


# ---------------------------------------------------------------------------
# Bounded sample (configs 4 and 5)
# ---------------------------------------------------------------------------


def _sample_units(args):
    """Time a few units of every kind on the full-size field (all workers run concurrently)."""
    _limit_threads()
    case, reps, sp = args
    u0, ut, ctrl = case.inputs()
    applyA, applyAT = _ops(case)
    h = case.spec.T / case.P / case.nsteps
    rng = np.random.default_rng(0)
    g = rng.standard_normal((ctrl.shape[0], u0.size))
    v = rng.standard_normal((ctrl.shape[0], u0.size))
    out = {}
    rk4_linear(applyA, g, h, 1)  # untimed warm-up (first-touch of the temporaries)
    t = time.perf_counter()
    rk4_linear(applyA, g, h, reps)
    out["rk4_direct_step"] = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    rk4_linear(applyAT, g, h, reps, want_z=True)
    out["rk4_adjoint_step"] = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    exp_action(applyA, sp, v)
    out["slice_action"] = time.perf_counter() - t
    acc = np.zeros_like(v)
    t = time.perf_counter()
    exp_action(applyAT, sp, v, acc)
    out["slice_action_phi"] = time.perf_counter() - t
    out["slice_terms"] = sp.terms
    return out


def gradient_units(case, rank: int, world: int) -> dict:
    """Units of work of one worker in one gradient (block-scan over `world` workers)."""
    from paper_2004_00546_b200.partition import rank_block
    sp, lp = _plans(case)
    p0, p1 = rank_block(case.P, rank, world)
    Pl = p1 - p0
    delta = case.spec.T / case.P
    return {"rk4_direct_step": Pl * case.nsteps, "rk4_adjoint_step": Pl * case.nsteps,
            "slice_actions": Pl - 1, "slice_actions_phi": Pl - 1,
            "long_terms": lp((case.P - p1) * delta).terms if p1 < case.P else 0,
            "long_terms_phi": lp(p0 * delta).terms if p0 > 0 else 0}


def predict_gradient_seconds(case, world: int, u: dict) -> float:
    """Slowest worker's Σ units × measured unit cost (long-span terms at the slice action's
    per-term cost)."""
    worst = 0.0
    t_term, t_term_phi = u["slice_action"] / u["slice_terms"], u["slice_action_phi"] / u["slice_terms"]
    for r in range(world):
        n = gradient_units(case, r, world)
        t = (n["rk4_direct_step"] * u["rk4_direct_step"] + n["rk4_adjoint_step"] * u["rk4_adjoint_step"]
             + n["slice_actions"] * u["slice_action"] + n["slice_actions_phi"] * u["slice_action_phi"]
             + n["long_terms"] * t_term + n["long_terms_phi"] * t_term_phi)
        worst = max(worst, t)
    return worst


def sampled_rate(case, workers: int, reps: int = 1):
    """One bounded sample: W concurrent workers time their units; returns (evals/s predicted,
    sample wall seconds, per-unit costs (slowest worker), fraction of a gradient the sample is)."""
    workers = max(1, min(workers, case.P))
    sp, _ = _plans(case)
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        pool.map(_limit_threads_noop, range(workers))  # spawn the workers before timing
        t0 = time.perf_counter()
        res = pool.map(_sample_units, [(case, reps, sp)] * workers)
        wall = time.perf_counter() - t0
    u = {k: float(np.mean([r[k] for r in res])) for k in res[0]}  # contended unit cost, mean over workers
    tg = predict_gradient_seconds(case, workers, u)
    return case.batch / tg, wall, u, wall / tg


def _limit_threads_noop(_):
    _limit_threads()
    return 0


def host_info() -> dict:
    import scipy
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu": model, "logical_cpus": os.cpu_count(), "numpy": np.__version__, "scipy": scipy.__version__}
