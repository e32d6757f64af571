"""Run files in the reference's JSON layout (`config.py:28-175`, `configs/*.json`) on the GPU.

A reference user's run file — ``{"problem": {"kind", "nx", "ny", "a", "D", "omega", "T", "f_true",
"f_init"}, "algorithm", "workers", "repeats", "pilot_fraction", "descent": {"steps", "lr"}, …}`` —
is read as it is and run through this package's loop (`python -m paper_2004_00546_b200 run
--config file.json`, the counterpart of `paradjoint run`, `cli.py:106-262`): the truth is
synthesised with ``f_true``, the serial loop and the parallel-in-time loop for every N of
``workers`` are timed from ``f_init`` with the reference's tracking objective and forcing
f·sin(ωt), and ``results.csv`` / ``summary.json`` (and ``descent.csv``) are written.

The reference's adaptive tolerances (``rtol``, ``leja_tol``) have no fixed-step counterpart: the
RK4 step is ``dt`` (default: min(T/200, 1/λ) with λ the diffusion part's spectral radius) and the
exponential actions are planned to 1e-12. ``checkpoints`` run with the hybrid algorithm
(`checkpointing.run_checkpointed_tracking`); the Gantt / PNG outputs are not part of this path. Field shapes: "sin_product", "ones", "zeros" or a flat list."""

from __future__ import annotations

import csv
import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError
from .problems import ADVECTION_DIFFUSION, BURGERS, Grid, ProblemSpec

ALGORITHMS = ("linear", "nonlinear", "hybrid")
_MISSING = object()


@dataclass(frozen=True)
class RunFile:
    kind: str
    nx: int
    ny: int
    a: float
    D: float
    omega: float
    T: float
    f_true: np.ndarray = field(repr=False)
    f_init: np.ndarray = field(repr=False)
    algorithm: str = "linear"
    workers: tuple = (1, 2, 4, 8, 16)
    checkpoints: int = 0
    repeats: int = 3
    pilot_fraction: float = 0.05
    output: str = "results"
    descent_steps: int = 0
    descent_lr: float = 0.5
    eps: float = 1e-3


def _take(obj: dict, where: str, key: str, types, default=_MISSING):
    name = f"{where}.{key}" if where else key
    if key not in obj:
        if default is _MISSING:
            raise ConfigError(f"{name}: this field is required")
        return default
    v = obj[key]
    if isinstance(v, bool) or not isinstance(v, types):
        raise ConfigError(f"{name}: expected {' or '.join(t.__name__ for t in np.atleast_1d(types))}")
    return v


def _shape(value, grid: Grid, fields: int, name: str) -> np.ndarray:
    n = fields * grid.npoints
    if isinstance(value, str):
        if value == "sin_product":   # sin x · sin y on every field (`problems.py:86-90`)
            X, Y = grid.coordinates()
            return np.tile(np.sin(X) * np.sin(Y), fields)
        if value in ("ones", "zeros"):
            return np.full(n, 1.0 if value == "ones" else 0.0)
        raise ConfigError(f"{name}: no field shape called {value!r} (sin_product, ones, zeros)")
    if isinstance(value, list):
        arr = np.asarray(value, dtype=np.float64)
        if arr.shape != (n,):
            raise ConfigError(f"{name}: expected {n} values, got {arr.size}")
        return arr
    raise ConfigError(f"{name}: a shape name (sin_product, ones, zeros) or a flat list of values")


def parse_run_file(data: dict) -> RunFile:
    if not isinstance(data, dict):
        raise ConfigError("a run file is a JSON object (problem, algorithm, workers, …)")
    prob = _take(data, "", "problem", dict)
    kind = _take(prob, "problem", "kind", str)
    if kind not in (ADVECTION_DIFFUSION, BURGERS):
        raise ConfigError(f"problem.kind: one of '{ADVECTION_DIFFUSION}', '{BURGERS}'")
    nx, ny = _take(prob, "problem", "nx", int, 32), _take(prob, "problem", "ny", int, 32)
    if nx < 3 or ny < 3:
        raise ConfigError("problem.nx/ny: the periodic stencil needs at least 3 points per direction")
    num = (int, float)
    a = float(_take(prob, "problem", "a", num, 1.0))
    D = float(_take(prob, "problem", "D", num))
    omega = float(_take(prob, "problem", "omega", num, 1.0))
    T = float(_take(prob, "problem", "T", num))
    if D <= 0 or T <= 0:
        raise ConfigError("problem.D / problem.T: must be positive")
    grid = Grid(nx, ny)
    fields = 2 if kind == BURGERS else 1
    f_true = _shape(prob.get("f_true", "sin_product"), grid, fields, "problem.f_true")
    f_init = _shape(prob.get("f_init", "ones"), grid, fields, "problem.f_init")
    algorithm = _take(data, "", "algorithm", str)
    if algorithm not in ALGORITHMS:
        raise ConfigError(f"algorithm: expected one of {ALGORITHMS}")
    if algorithm == "linear" and kind == BURGERS:
        raise ConfigError("algorithm: 'linear' is for the advection–diffusion (linear) problem")
    workers = data.get("workers", [1, 2, 4, 8, 16])
    if isinstance(workers, int) and not isinstance(workers, bool):
        workers = [workers]
    if not isinstance(workers, list) or not workers or not all(
            isinstance(w, int) and not isinstance(w, bool) and w >= 1 for w in workers):
        raise ConfigError("workers: a slice count ≥ 1 or a non-empty list of such counts")
    checkpoints = _take(data, "", "checkpoints", int, 0)
    repeats = _take(data, "", "repeats", int, 3)
    if repeats < 1:
        raise ConfigError("repeats: at least one timed repetition is needed")
    pilot = float(_take(data, "", "pilot_fraction", num, 0.05))
    if not 0.0 < pilot <= 0.1:
        raise ConfigError("pilot_fraction: a fraction of the horizon in (0, 0.1]")
    descent = data.get("descent", {})
    if not isinstance(descent, dict):
        raise ConfigError("descent: an object {steps, lr}")
    steps = _take(descent, "descent", "steps", int, 0)
    lr = float(_take(descent, "descent", "lr", num, 0.5))
    if steps < 0 or (steps and lr <= 0):
        raise ConfigError("descent: steps cannot be negative and lr must be positive")
    eps = float(_take(data, "", "eps", num, 1e-3))
    if eps <= 0:
        raise ConfigError("eps: must be positive")
    return RunFile(kind, nx, ny, a, D, omega, T, f_true, f_init, algorithm, tuple(workers), checkpoints, repeats,
                   pilot, _take(data, "", "output", str, "results"), steps, lr, eps)


def load_run_file(path: str) -> RunFile:
    try:
        with open(path) as fh:
            return parse_run_file(json.load(fh))
    except (OSError, json.JSONDecodeError) as e:
        raise ConfigError(f"{path}: {e}")


def default_dt(rf: RunFile) -> float:
    """min(T/200, 1/λ), λ = 4D(1/hx² + 1/hy²) (classical RK4 is stable up to 2.78/λ)."""
    g = Grid(rf.nx, rf.ny)
    lam = 4.0 * rf.D * (1.0 / g.hx**2 + 1.0 / g.hy**2)
    return min(rf.T / 200.0, 1.0 / lam)


def run_file(rf: RunFile, output: str | None = None, dt: float | None = None, repeats: int | None = None) -> dict:
    """Time the serial loop and the parallel-in-time loop for every N of ``workers``; returns
    (and writes) the summary. Raises ConfigError for what this path does not run."""
    from .expaction import ChebyshevConfig
    from .hybrid import TimeLaw, estimate_k, make_hybrid_plan
    from .optimization import descend, direct_adjoint_loop
    from .partition import RK4Config
    from .systems import build_burgers2d_system, build_field_system
    from .tracking import synthesize_trajectory
    if rf.checkpoints and rf.algorithm != "hybrid":
        raise ConfigError("checkpoints: checkpointed run files run the hybrid algorithm here (run_checkpointed_tracking)")
    if rf.algorithm in ("hybrid", "nonlinear") and rf.kind != BURGERS:
        raise ConfigError(f"algorithm: the {rf.algorithm} algorithm is for the Burgers testbed")
    out = output or rf.output
    reps = repeats or rf.repeats
    grid = Grid(rf.nx, rf.ny)
    law = TimeLaw.sine(rf.omega)
    cfg = ChebyshevConfig(tol=1e-12)
    dt0 = dt or default_dt(rf)
    linear = rf.kind == ADVECTION_DIFFUSION
    if linear:
        system = build_field_system(grid, ProblemSpec(ADVECTION_DIFFUSION, (rf.a, rf.a), rf.D, rf.T))
    else:
        system = build_burgers2d_system(grid, ProblemSpec(BURGERS, (0.0, 0.0), rf.D, rf.T))
    targets: dict = {}

    def target_for(S: int):
        if S not in targets:
            targets[S] = synthesize_trajectory(system, rf.f_true, RK4Config(rf.T / S), law)[:, 0, :]
        return targets[S]

    def steps_for(N: int) -> int:
        if linear or rf.algorithm == "nonlinear":   # whole steps per (equal) slice
            return N * max(1, int(np.ceil(rf.T / (N * dt0) - 1e-9)))
        return max(1, int(np.ceil(rf.T / dt0 - 1e-9)))

    def timed_checkpointed(N, k):
        """`checkpoints` > 0 (`cli.py:155-162`): the hybrid loop segment by segment."""
        from .checkpointing import CheckpointSchedule, run_checkpointed_tracking
        M1 = rf.checkpoints + 1
        S = M1 * max(1, int(np.ceil(rf.T / (M1 * dt0) - 1e-9)))
        kw = dict(N=N, rk=RK4Config(rf.T / S), expaction=cfg, law=law, k_ratio=k)
        sched = CheckpointSchedule(rf.T, rf.checkpoints)
        tgt = target_for(S)
        run = run_checkpointed_tracking(system, rf.f_init, tgt, sched, **kw)
        tick = time.perf_counter()
        for _ in range(reps):
            run = run_checkpointed_tracking(system, rf.f_init, tgt, sched, **kw)
        return (time.perf_counter() - tick) / reps, run

    def timed(algorithm, N, plan=None):
        S = steps_for(N)
        kw = dict(N=N, rk=RK4Config(rf.T / S), expaction=cfg, objective="tracking", time_law=law)
        if algorithm == "nonlinear":
            kw["eps"] = rf.eps
        if plan is not None:
            kw["plan"] = plan
        tgt = target_for(S)
        loop = direct_adjoint_loop(system, rf.f_init, tgt, algorithm, **kw)   # warm-up: plans, allocation
        tick = time.perf_counter()
        for _ in range(reps):
            loop = direct_adjoint_loop(system, rf.f_init, tgt, algorithm, **kw)
        return (time.perf_counter() - tick) / reps, loop, kw, tgt

    t_serial, serial, _, _ = timed("serial", 1)
    k = None
    if rf.algorithm == "hybrid":
        k = estimate_k(system, rf.pilot_fraction, RK4Config(rf.T / steps_for(1)), repeats=reps, law=law)
    rows = []
    last = None
    for N in rf.workers:
        if rf.checkpoints:
            t_par, run = timed_checkpointed(N, k)
            rows.append([rf.algorithm, N, rf.D, reps, 1, f"{t_serial:.6f}", f"{t_par:.6f}", f"{t_serial / t_par:.6f}",
                         f"{run.cost:.12e}", f"{np.linalg.norm(run.gradient):.12e}"])
            continue
        plan = make_hybrid_plan(rf.T, N, k) if rf.algorithm == "hybrid" else None
        t_par, loop, kw, tgt = timed(rf.algorithm, N, plan)
        last = (N, kw, tgt)
        rows.append([rf.algorithm, N, rf.D, reps, loop.iterations, f"{t_serial:.6f}", f"{t_par:.6f}",
                     f"{t_serial / t_par:.6f}", f"{float(loop.J):.12e}", f"{np.linalg.norm(loop.grad):.12e}"])
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "results.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["algorithm", "N", "D", "repeats", "K", "t_serial_s", "t_parallel_s", "s_measured", "J", "grad_norm"])
        w.writerows(rows)
    summary = {"algorithm": rf.algorithm, "workers": list(rf.workers), "checkpoints": rf.checkpoints, "D": rf.D, "T": rf.T,
               "grid": [rf.nx, rf.ny], "backend": "cuda", "dt": rf.T / steps_for(1), "k": k,
               "t_serial_s": t_serial, "J_serial": float(serial.J),
               "J": {str(r[1]): float(r[8]) for r in rows}}
    if rf.descent_steps > 0 and last is not None:
        N, kw, tgt = last
        res = descend(system, rf.f_init, tgt, rf.descent_steps, rf.descent_lr, algorithm=rf.algorithm, **kw)
        with open(os.path.join(out, "descent.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["step", "J", "grad_norm", "wallclock_s"])
            for i, (J, g, s) in enumerate(zip(res.J_history, res.grad_norms, res.step_seconds)):
                w.writerow([i, f"{float(J):.9e}", f"{float(np.ravel(g)[0]):.9e}", f"{s:.6f}"])
        np.save(os.path.join(out, "f_final.npy"), res.f_final)
        summary["descent"] = {"steps": rf.descent_steps, "lr": rf.descent_lr, "N": N,
                              "J_first": float(res.J_history[0]), "J_last": float(res.J_history[-1])}
    with open(os.path.join(out, "summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    return summary
