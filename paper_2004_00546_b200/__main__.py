"""Command line (mirror of the reference's `paradjoint run|predict`, `cli.py:352-403`,
for the BASELINE configs with ``backend="cuda"``).

    python -m paper_2004_00546_b200 run --config 5 --repeats 3 --output results/c5
    python -m paper_2004_00546_b200 run --config 3 --checkpoints 3
    python -m paper_2004_00546_b200 predict --config 5 --gpus 1 2 4 8
    python -m paper_2004_00546_b200 run --config burgers_hybrid.json      # a reference run file (runfile.py)

``run`` times `direct_adjoint_loop` (or config 2's 20-step `descend`) on this
GPU and writes ``results.csv`` and ``summary.json`` (timing columns separate,
as `reporting.py:22-55`); ``predict`` measures the per-unit kernel times with one
gradient and prints the block-scan strong-scaling model (`scaling.py` here).
Exit codes as the reference: 0 ok, 1 usage/config error, 2 solver failure.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

import numpy as np


def _case(index: int):
    from .configs import baseline
    return baseline(index)


def _run_file(args) -> int:
    """`run --config file.json`: a run file in the reference's own layout (`config.py:28-175`)."""
    from .runfile import load_run_file, run_file
    rf = load_run_file(args.config)
    out = args.output if args.output != "results" else rf.output
    summary = run_file(rf, out, dt=args.dt, repeats=args.repeats if args.repeats != 3 else None)
    print(json.dumps(summary))
    return 0


def cmd_run(args) -> int:
    from .optimization import descend, direct_adjoint_loop
    from .partition import RK4Config
    if not str(args.config).isdigit():
        return _run_file(args)
    args.config = int(args.config)
    c = _case(args.config)
    u0, ut, ctrl = c.inputs()
    algo = "linear" if c.system.is_linear else ("nonlinear" if args.nonlinear else "hybrid")
    if args.algorithm:
        algo = args.algorithm
    rk = RK4Config(c.dt)
    rows, t = [], []
    if args.checkpoints:
        return _run_checkpointed(args, c, u0, ut, ctrl, rk)
    extra = {"hybrid_adjoint": args.hybrid_adjoint} if algo == "hybrid" else {}
    # warm-up outside the timed region: plans, HBM allocation, graph capture
    direct_adjoint_loop(c.system, ctrl, ut, algo, N=c.P, rk=rk, expaction=c.expaction, u0=u0, **extra)
    if c.descent_steps and not args.single:
        tick = time.perf_counter()
        res = descend(c.system, ctrl, ut, steps=c.descent_steps, lr=c.lr, algorithm=algo, N=c.P, rk=rk,
                      expaction=c.expaction, u0=u0)
        t.append(time.perf_counter() - tick)
        for i, (J, g) in enumerate(zip(res.J_history, res.grad_norms)):
            for b, (Jb, gb) in enumerate(zip(np.ravel(J), np.ravel(g))):
                rows.append([i, b, f"{Jb:.17g}", f"{gb:.17g}"])
        evals = c.descent_steps * c.batch
    else:
        for rep in range(args.repeats):
            tick = time.perf_counter()
            loop = direct_adjoint_loop(c.system, ctrl, ut, algo, N=c.P, rk=rk, expaction=c.expaction, u0=u0,
                                       **extra)
            t.append(time.perf_counter() - tick)
        for b, (Jb, gb) in enumerate(zip(np.ravel(loop.J), np.atleast_2d(loop.grad))):
            rows.append([0, b, f"{Jb:.17g}", f"{np.linalg.norm(gb):.17g}"])
        evals = c.batch
    os.makedirs(args.output, exist_ok=True)
    with open(os.path.join(args.output, "results.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["iteration", "member", "J", "grad_norm"])
        w.writerows(rows)
    summary = {"config": c.name, "algorithm": algo, **extra, "backend": "cuda", "grid": [c.grid.nx, c.grid.ny],
               "P": c.P, "steps_per_slice": c.nsteps, "batch": c.batch,
               "timing": {"seconds_median": float(np.median(t)), "repeats": len(t),
                          "gradient_evals_per_s": evals / float(np.median(t))}}
    with open(os.path.join(args.output, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary))
    return 0


def _run_checkpointed(args, c, u0, ut, ctrl, rk) -> int:
    """`run --checkpoints M` (the reference's `run_checkpointed_loop` branch, `cli.py:155-162`):
    M equispaced checkpoints, P/(M+1) slices per segment; one gradient per repeat."""
    from .checkpointing import CheckpointSchedule, run_checkpointed_loop
    M = args.checkpoints
    if c.P % (M + 1):
        raise ValueError(f"P = {c.P} slices do not split into {M + 1} equal segments")
    if c.batch != 1:
        raise ValueError("checkpointed runs take one control (batch 1)")
    algo = "linear" if c.system.is_linear else "hybrid"
    sched = CheckpointSchedule(c.spec.T, M)
    kw = dict(N=c.P // (M + 1), rk=rk, expaction=c.expaction, u0=u0)
    run_checkpointed_loop(c.system, ctrl[0], ut, sched, algo, **kw)   # warm-up
    t = []
    for _ in range(args.repeats):
        tick = time.perf_counter()
        run = run_checkpointed_loop(c.system, ctrl[0], ut, sched, algo, **kw)
        t.append(time.perf_counter() - tick)
    os.makedirs(args.output, exist_ok=True)
    with open(os.path.join(args.output, "results.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["iteration", "member", "J", "grad_norm"])
        w.writerow([0, 0, f"{float(run.cost[0]):.17g}", f"{np.linalg.norm(run.gradient):.17g}"])
    summary = {"config": c.name, "algorithm": algo, "backend": "cuda", "checkpoints": M,
               "segments": sched.segment_bounds, "slices_per_segment": c.P // (M + 1),
               "peak_trajectory_nodes": run.memory.peak,
               "timing": {"seconds_median": float(np.median(t)), "repeats": len(t),
                          "gradient_evals_per_s": 1.0 / float(np.median(t))}}
    with open(os.path.join(args.output, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary))
    return 0


def cmd_predict(args) -> int:
    from .engine import EngineSpec, ParaexpEngine
    from .scaling import profile_from_timing, scaling_table
    c = _case(args.config)
    u0, ut, ctrl = c.inputs()
    eng = ParaexpEngine(EngineSpec(c.system, c.P, c.dt, c.expaction, c.batch, local_blocks=1))  # per-unit costs
    eng.set_inputs(u0, ut, ctrl)
    eng.gradient()
    eng.get(0)
    eng.set_timing(True)
    eng.timing()
    for _ in range(args.repeats):
        eng.gradient()
    eng.get(0)
    prof = profile_from_timing(c, eng.timing(), {}, args.repeats)
    out = {"config": c.name, "profile": json.loads(prof.to_json()),
           "prediction": [{"gpus": p.G, "seconds": p.seconds, "speedup": p.speedup, "efficiency": p.efficiency,
                           "critical_rank": p.critical_rank, "breakdown": p.breakdown}
                          for p in scaling_table(c, prof, tuple(args.gpus))]}
    print(json.dumps(out, indent=1))
    eng.close()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2004_00546_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="time the direct-adjoint loop of a BASELINE config on this GPU")
    r.add_argument("--config", default="5",
                   help="a BASELINE config number, or a run file in the reference's JSON layout (configs/*.json)")
    r.add_argument("--dt", type=float, default=None, help="run files: the fixed RK4 step (default min(T/200, 1/λ))")
    r.add_argument("--repeats", type=int, default=3)
    r.add_argument("--output", default="results")
    r.add_argument("--single", action="store_true", help="one gradient even for descent configs")
    r.add_argument("--nonlinear", action="store_true", help="Burgers: Algorithm 2 direct instead of serial")
    r.add_argument("--algorithm", choices=["serial", "linear", "nonlinear", "hybrid"], default=None,
                   help="override the config's algorithm (serial = the reference loop, no Paraexp)")
    r.add_argument("--hybrid-adjoint", choices=["absorbed", "frozen_span"], default="absorbed",
                   help="Burgers hybrid: config 3's absorbed adjoint or the reference solve_hybrid's frozen span")
    r.add_argument("--checkpoints", type=int, default=0,
                   help="M equispaced checkpoints (run_checkpointed_loop; P/(M+1) slices per segment)")
    p = sub.add_parser("predict", help="measure per-unit kernel times, print the multi-GPU scaling model")
    p.add_argument("--config", type=int, default=5)
    p.add_argument("--repeats", type=int, default=2)
    p.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    args = ap.parse_args(argv)
    try:
        return cmd_run(args) if args.cmd == "run" else cmd_predict(args)
    except (ValueError, KeyError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except RuntimeError as e:
        print(f"solver failure: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
