#!/usr/bin/env python
"""Benchmark: Paraexp direct-adjoint gradient evaluations per second on B200.

One *step* = one full direct-adjoint gradient evaluation (direct Paraexp sweep, objective,
adjoint Paraexp sweep, gradient projection) of BASELINE config 5 (2D advection–diffusion 2048²,
P = 512 slices, Chebyshev, tol 1e-10 as the sweep's error budget; the largest config and the one
BASELINE names for 1/2/4/8 GPUs). Multi-GPU (torchrun): the P slices are sharded in contiguous
blocks, partials allreduced over NCCL (strong scaling: total work fixed). ``--config k`` benches
another config.

Line fields (see the task contract):

* ``value`` — gradient evals/s with inputs resident in HBM (CUDA events on the work stream,
  max over ranks);
* ``e2e`` — the same metric through the public API ``direct_adjoint_loop`` with host numpy
  inputs/outputs (H2D/D2H inside the timed region, host wall clock);
* ``roofline`` — the dominant kernel (the fused two-step RK4 march, ≈ 75% of a gradient):
  ``achieved`` = its algorithmic bytes per launch (each distinct operand once: y in and y out per
  lane, the source b per member) ÷ its average launch time, measured in this run
  with CUDA events around every launch; ``traffic`` = the DRAM bytes ncu measured per launch
  (profiles/ncu_traffic.json); ``model_frac`` = the SURVEY per-step model (24n per lane and RK4
  step, two steps per launch) for comparison; ``fp64`` = DFMA rate against the measured fp64
  peak (profiles/r02_fp64_peak.json); ``binding`` = the limiter from the ncu capture;
* ``cpu_baseline`` — the CPU reference path (oracle/cpu_reference.py: the oracle's arithmetic,
  every slice solved, W host processes) on this host: full gradients for configs 1–3, a bounded
  sample for configs 4/5 (every worker times each unit kind on the full-size field; one gradient
  = the slowest worker's units × unit times), validated offline against a full CPU gradient
  (profiles/r02_cpu_reference_c*.json);
* ``--impl reference`` prints the CPU arm alone (rank 0; other ranks exit).
* ``--testbed hybrid|nonlinear`` benches the reference's own 2D two-field Burgers run-file shapes
  (32×32; widening rows) with the same line: value, e2e, roofline (the on-chip serial
  sweep: fp64 fraction of its one SM), cpu_baseline (the oracle's same gradient, one core).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Paraexp direct-adjoint gradient evals/s"
UNIT = "gradient evals/s"
FP64_FALLBACK_TFLOPS = 37.0  # B200 datasheet order of magnitude; used only without the measured file


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        hbm, src = float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    q = os.path.join(ROOT, "profiles", "r02_fp64_peak.json")
    if os.path.exists(q):
        with open(q) as f:
            fp = json.load(f)
        fp64, fsrc = float(fp["fp64_tflops_avg"]), "measured (profiles/r02_fp64_peak.json, tools/mb/fp64_peak.cu)"
    else:
        fp64, fsrc = FP64_FALLBACK_TFLOPS, "fallback (datasheet order)"
    return hbm, src, fp64, fsrc


def load_profile(config: int) -> dict:
    """The committed ncu summary (per-launch DRAM bytes, limiter) of the dominant kernel."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f).get(f"c{config}", {})


class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (the recipe's clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU reference path (oracle port, host cores)
# ---------------------------------------------------------------------------


def cpu_workers() -> int:
    return max(1, os.cpu_count() or 1)


def cpu_reference(index: int, workers: int) -> dict:
    """One CPU measurement of the config: a full gradient (configs 1–3) or one bounded sample
    (configs 4, 5). Returns the rate, the seconds this step took and what it was."""
    from oracle.cpu_reference import full_gradient, host_info, sampled_rate
    from paper_2004_00546_b200 import baseline
    c = baseline(index)
    if index in (4, 5):
        rate, wall, units, frac = sampled_rate(c, workers)
        w = max(1, min(workers, c.P))
        sample = (f"bounded sample: each of {w} concurrent worker processes (slice block of a {w}-way "
                  f"block-scan) times 1 direct and 1 adjoint RK4 step (after a warm-up step), one slice action with and one "
                  f"without the φ₁ accumulator on the full {c.grid.nx}x{c.grid.ny} field; one gradient = "
                  f"the slowest worker's unit counts × unit times ({frac:.4f} of a gradient per step)")
        return {"value": rate, "seconds": wall, "cores": w, "sample": sample, "gradient_fraction": frac,
                "unit_seconds": units, "host": host_info()}
    t0 = time.perf_counter()
    if index == 3:
        from oracle.config_mode import burgers_gradient
        from paper_2004_00546_b200.expaction import plan_chebyshev
        from paper_2004_00546_b200.problems import burgers_frozen_region
        u0, ut, ctrl = c.inputs()
        burgers_gradient(c.grid.nx, c.spec.D, c.system.basis, c.spec.T, c.P, c.nsteps, u0, ut, ctrl,
                         lambda region, span: plan_chebyshev(region, span, c.expaction),
                         lambda ub: burgers_frozen_region(ub, c.grid, c.spec.D))
        w = 1
        what = "one full gradient (serial direct sweep + every adjoint slice), one process"
    else:
        w = max(1, min(workers, c.P))
        full_gradient(c, w)
        what = f"one full gradient, every slice solved, {w}-process block-scan"
    wall = time.perf_counter() - t0
    return {"value": c.batch / wall, "seconds": wall, "cores": w, "sample": what, "gradient_fraction": 1.0,
            "host": host_info()}


def load_cpu_validation(index: int):
    p = os.path.join(ROOT, "profiles", f"r02_cpu_reference_c{index}.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    W = cpu_workers()
    runs = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference(args.config, W)
        if i >= args.warmup:
            runs.append(r)
    v = statistics.median(r["value"] for r in runs)
    last = runs[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(r["seconds"] for r in runs),
        "gradient_fraction_per_step": last["gradient_fraction"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, paper_2004_00546_b200/configs.py)", "config": config_block(args.config, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": last["cores"], "kind": "port", "sample": last["sample"],
                         "host": last["host"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    val = load_cpu_validation(args.config)
    if val:
        line["cpu_baseline"]["validation"] = val
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_block(index, world):
    from paper_2004_00546_b200 import baseline
    c = baseline(index)
    return {"workload": c.name, "grid": [c.grid.nx, c.grid.ny], "P": c.P, "steps_per_slice": c.nsteps,
            "T": c.spec.T, "dt": c.spec.T / c.P / c.nsteps, "batch": c.batch, "K": c.K,
            "expaction": type(c.expaction).__name__, "tol": c.expaction.tol,
            "tol_horizon": c.expaction.horizon or None,
            "parallelism": f"slices{world}" if world > 1 else "single",
            "l2": "inputs larger than L2 (lane buffers of P×n fp64)" if c.n * c.P * 8 > 126e6 else
                  "working set fits L2 (not flushed)"}


def roofline_2d(eng, c, peak, peak_src, fp64_peak, fp64_src, prof, world):
    """The fused two-step RK4 march: bytes and DFMA per launch over its measured launch time."""
    import torch
    from paper_2004_00546_b200 import _native as N
    s = int(torch.cuda.current_stream().cuda_stream)
    eng.kernel_timing(N.PX_KCLASS_MARCH2)
    eng.kernel_timing(N.PX_KCLASS_CHEB)
    eng.set_timing(True, kernels=True)
    for _ in range(2):
        eng.gradient(s, want_fields=False)
    torch.cuda.synchronize()
    eng.set_timing(False)
    eng.timing()
    ms, cnt = eng.kernel_timing(N.PX_KCLASS_MARCH2)
    cms, ccnt = eng.kernel_timing(N.PX_KCLASS_CHEB)
    if cnt == 0:
        return None
    t = ms / cnt / 1e3
    n, L, B = c.n, eng.B * (eng.p1 - eng.p0), eng.B
    alg = 16.0 * n * L + 8.0 * n * B      # y in + y out per lane, b per member: distinct operands once
    model = 2 * 24.0 * n * L              # 24n per lane and RK4 step, two steps
    dfma = 2 * 21.0 * n * L               # 4 Horner stages × 5 stencil FMAs + the source add, per step
    pr = prof.get("rk4_direct", {})
    traffic = pr.get("dram_bytes_per_launch")
    out = {"bound": "hbm", "kernel": "k_rk4_marchc<3,64,3,4,br> (two RK4 steps per launch)",
           "achieved": alg / t / 1e9, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
           "frac": alg / t / 1e9 / peak, "traffic": traffic,
           "algorithmic_bytes_per_launch": alg, "avg_launch_ms": t * 1e3, "launches_timed": cnt,
           "model_bytes_per_launch": model, "model_frac": model / t / 1e9 / peak,
           "fp64": {"dfma_per_launch": dfma, "achieved_tflops": 2 * dfma / t / 1e12, "peak_tflops": fp64_peak,
                    "peak_source": fp64_src, "frac": 2 * dfma / t / 1e12 / fp64_peak}}
    if traffic:
        out["dram_achieved"] = traffic / t / 1e9
        out["dram_frac"] = traffic / t / 1e9 / peak
        out["traffic_source"] = pr.get("source")
    if pr.get("limiter"):
        out["binding"] = pr["limiter"]
    if ccnt:
        out["chebyshev_pass_avg_ms"] = cms / ccnt
    return out


# ---------------------------------------------------------------------------
# The reference's own 2D two-field Burgers configs (widening rows)
# ---------------------------------------------------------------------------


def run_testbed(args):
    """`--testbed hybrid|nonlinear`: the reference's `configs/burgers_hybrid.json` /
    `burgers_iterative.json` shapes (32×32 two-field Burgers, D = 1, ω = 1, T = 1, 1000 RK4 steps;
    16 geometric slices / 8 equal slices with eps 1e-3) — one step = one tracking-objective
    gradient through `solve_hybrid_tracking` / `solve_nonlinear_tracking`. ``value``: target
    resident on the device (events on the work stream; the host planning between the sweeps is
    part of a gradient); ``e2e``: host arrays each step (target included); ``roofline``: the serial
    sweep kernel — on chip, so the HBM figure (the trajectory it streams out) is small by design and
    ``fp64`` (its DFMA count over its measured time against one SM's share of the measured peak) is
    the meaningful fraction; ``cpu_baseline``: the oracle's same gradient timed here on one core."""
    import torch
    from paper_2004_00546_b200 import (
        ChebyshevConfig, Grid, ProblemSpec, RK4Config, TimeLaw, build_burgers2d_system, make_hybrid_plan,
        solve_hybrid_tracking, solve_nonlinear_tracking, synthesize_trajectory)
    from paper_2004_00546_b200.problems import BURGERS
    torch.cuda.set_device(0)
    nx = ny = 32
    D = T = 1.0
    S, P = 1000, (16 if args.testbed == "hybrid" else 8)
    sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), D, T))
    X, Y = sysm.grid.coordinates()
    rk, cfg, law = RK4Config(T / S), ChebyshevConfig(tol=1e-12), TimeLaw.sine(1.0)
    f_true = np.concatenate([np.sin(X) * np.sin(Y)] * 2)
    f, u0 = np.ones(sysm.n), np.zeros(sysm.n)
    target_host = synthesize_trajectory(sysm, f_true, rk, law)[:, 0, :]
    target_dev = torch.as_tensor(target_host, device="cuda")
    plan = make_hybrid_plan(T, P, 3.0)

    def solve(target):
        if args.testbed == "hybrid":
            return solve_hybrid_tracking(sysm, u0, f, target, plan, rk=rk, expaction=cfg, law=law, overlap=True)
        return solve_nonlinear_tracking(sysm, u0, f, np.asarray(target_host), N=P, rk=rk, expaction=cfg, law=law, eps=1e-3)

    resident = target_dev if args.testbed == "hybrid" else target_host
    for _ in range(args.warmup):
        r = solve(resident)
    torch.cuda.synchronize()
    if args.profile_only:
        for _ in range(args.steps):
            solve(resident)
        torch.cuda.synchronize()
        return 0
    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sweep_ms = []
    with ClockSampler(0) as clk:
        a.record(stream)
        for _ in range(args.steps):
            r = solve(resident)
            sweep_ms.append(r.timing["direct_ms"])
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):   # (inside the clock sampler: the timed loop alone lasts < 200 ms)
            r = solve(target_host)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        while time.perf_counter() - t0 < 0.7:   # a few more gradients so that nvidia-smi gets samples under load
            solve(resident)
    value = args.steps / (ms / 1e3)
    e2e = {"value": args.e2e_steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(target_host.nbytes + 2 * sysm.n * 8), "d2h_bytes_per_step": int((1 + 3 * sysm.n) * 8),
           "api": "solve_hybrid_tracking / solve_nonlinear_tracking with host numpy arrays (J, grad, u(T), q†(0) read back)"}
    peak, peak_src, fp64_peak, fp64_src = load_peaks()
    n = nx * ny
    roofline = None
    if args.testbed == "hybrid":
        t = statistics.median(sweep_ms) / 1e3       # the serial sweep kernel (CUDA events, px_hybrid_get_timing)
        alg = 16.0 * n * (S + 1)                     # every node of (U, V) streamed to HBM once
        dfma = 4.0 * S * n * 2 * 16                  # 4 stages × 2 fields × ≈ 16 fp64 pipe instructions per point
        sm_peak = fp64_peak / 148.0                  # one CTA per member: one SM's share of the measured peak
        roofline = {"bound": "hbm", "kernel": "k_b2s_direct<2> (the whole serial sweep, one CTA on one SM)",
                    "achieved": alg / t / 1e9, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                    "frac": alg / t / 1e9 / peak, "traffic": None, "algorithmic_bytes_per_launch": alg,
                    "avg_launch_ms": t * 1e3,
                    "fp64": {"instr_per_launch": dfma, "achieved_tflops": 2 * dfma / t / 1e12,
                             "peak_tflops_one_sm": sm_peak, "frac_of_one_sm": 2 * dfma / t / 1e12 / sm_peak,
                             "peak_source": fp64_src},
                    "note": "on-chip kernel: the state never leaves shared memory / registers, only the trajectory "
                            "nodes go to HBM; the serial sweep is bound by the fp64 pipe of the single SM it runs on "
                            "(profiles/r02b_prof_hybrid2d_raw.csv: 45% fp64 pipe, 25% warps active)",
                    "share_of_step": t / (ms / 1e3 / args.steps)}
    cpu = None
    if not args.no_cpu_baseline:
        from oracle.config_mode import burgers2d_nonlinear_tracking, burgers_tracking_hybrid
        from paper_2004_00546_b200.expaction import plan_chebyshev, plan_family
        from paper_2004_00546_b200.problems import frozen_bounds_2d, frozen_region_from_bounds
        reg = lambda q: frozen_region_from_bounds(*frozen_bounds_2d(q, sysm.grid, D))
        offs = r.offsets
        h = T / S
        t0 = time.perf_counter()
        if args.testbed == "hybrid":
            o = burgers_tracking_hybrid(nx, D, T, offs, u0, f[None, :], law.as_tuple(), target_host,
                                        lambda q: plan_family(reg(q), [(offs[p + 1] - offs[p]) * h for p in range(P)],
                                                              cfg, omega=law.omega), ny=ny)
        else:
            o = burgers2d_nonlinear_tracking(nx, ny, D, T, P, S // P, u0, f[None, :], law.as_tuple(), target_host,
                                             lambda q: (plan_chebyshev(reg(q), T / P, cfg), plan_chebyshev(reg(q), h, cfg)),
                                             lambda q: plan_family(reg(q), [T / P] * P, cfg, omega=law.omega), 1e-3)
        sec = time.perf_counter() - t0
        cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": "one complete gradient of the same problem by the oracle restatement (numpy, one core)",
               "agreement": {"J_rel": float(abs(o.J[0] - r.J[0]) / abs(o.J[0])),
                             "grad_rel": float(np.linalg.norm(o.grad - r.grad) / np.linalg.norm(o.grad))}}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (the reference's run-file shapes: f_true = sin x·sin y, f_init = ones)",
            "config": {"workload": f"reference_burgers2d_{args.testbed}_32x32", "grid": [nx, ny], "P": P, "steps": S,
                       "T": T, "D": D, "omega": 1.0, "objective": "tracking", "batch": 1,
                       "partition": "geometric k=3" if args.testbed == "hybrid" else "equidistant, eps 1e-3",
                       "sweeps": len(r.timing.get("history", [])) or None,
                       "l2": "working set fits L2 (not flushed): an on-chip latency-bound path"},
            "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "clocks": clk.summary(),
            # on-chip kernels per gradient: sweep, slice lanes, cost (2), means, bounds, frozen carry; Algorithm 2:
            # (means, bounds, lanes, carry, node parts, error) per sweep + the seven above without the serial sweep
            "gpu_launches": args.steps * (7 if args.testbed == "hybrid" else 6 * len(r.timing.get("history", [])) + 6),
            "timing": {k: v for k, v in r.timing.items() if k != "history"}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--testbed", choices=["hybrid", "nonlinear"], default=None,
                    help="bench the reference's own 2D two-field Burgers config instead of a BASELINE config")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="warmup+steps only (for ncu); no extras")
    args = ap.parse_args()
    if args.warmup < 3 and not args.profile_only and args.impl != "reference":
        args.warmup = 3

    if args.impl == "reference":
        return run_reference(args)
    if args.testbed:
        return run_testbed(args)

    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    dev_index = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_index)
    if world > 1:
        # PX_BENCH_DIST_BACKEND=gloo: host-mediated collectives, for exercising the multi-rank
        # path with fewer GPUs than ranks (no kernel waits on another rank); default NCCL
        backend = os.environ.get("PX_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    from paper_2004_00546_b200 import RK4Config, baseline, direct_adjoint_loop
    from paper_2004_00546_b200.engine import EngineSpec, ParaexpEngine

    c = baseline(args.config)
    u0, ut, ctrl = c.inputs()
    eng = ParaexpEngine(EngineSpec(c.system, c.P, c.dt, c.expaction, c.batch, rank, world))
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (u0, ut, ctrl)]
    eng.set_inputs(*dev)
    stream = torch.cuda.current_stream()
    s = int(stream.cuda_stream)

    def step():
        eng.gradient(s, want_fields=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if args.profile_only:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        return 0
    eng.reset_stats()
    eng.timing()
    eng.set_timing(True)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_index) as clk:
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    eng.set_timing(False)
    ms = start.elapsed_time(end)
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    J = eng.get(0)
    assert np.all(np.isfinite(J)), "non-finite objective"
    phases = eng.timing()
    stats = eng.stats()
    launches = int(stats["kernel_launches"])
    value = args.steps * c.batch / (ms_max / 1e3)

    peak, peak_src, fp64_peak, fp64_src = load_peaks()
    prof = load_profile(args.config)
    roofline = None
    if c.grid.dim == 2 and c.system.is_linear:
        roofline = roofline_2d(eng, c, peak, peak_src, fp64_peak, fp64_src, prof, world)
    if roofline is None:
        # on-chip configs (1D lanes and scans, Burgers): phase-level algorithmic bytes
        dom = max(phases, key=lambda k: phases[k]["ms"])
        ph = phases[dom]
        tl = (ph["ms"] / 1e3) / max(ph["launches"], 1)
        bpl = ph["bytes"] / max(ph["launches"], 1)
        roofline = {"bound": "hbm", "phase": dom, "achieved": bpl / tl / 1e9 if tl > 0 else 0.0, "peak": peak,
                    "peak_source": peak_src, "unit": "GB/s", "frac": (bpl / tl / 1e9 / peak) if tl > 0 else 0.0,
                    "traffic": None, "bytes_per_launch": bpl, "avg_launch_ms": tl * 1e3,
                    "note": "on-chip kernels (state in shared memory / registers across steps or terms): "
                            "the SURVEY §8(d) per-unit model counts bytes these kernels never move; the "
                            "binding resources are the fp64 pipe and barrier latency"}
    roofline["share_of_step"] = None
    total_ms = sum(p["ms"] for p in phases.values())
    if total_ms > 0:
        roofline["share_of_step"] = (phases["rk4_direct"]["ms"] + phases["rk4_adjoint"]["ms"]) / total_ms
    phase_ms = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                    "algorithmic_GB/s": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None}
                for k, v in phases.items()}

    eng.close()  # the public-API leg below owns its own engine (HBM scratch)
    del dev
    torch.cuda.empty_cache()
    # e2e: public API with host inputs/outputs, host wall clock
    e2e = None
    if args.e2e_steps > 0:
        rk = RK4Config(c.dt)
        algo = "linear" if c.system.is_linear else "hybrid"
        direct_adjoint_loop(c.system, ctrl, ut, algo, N=c.P, rk=rk, expaction=c.expaction, u0=u0)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            direct_adjoint_loop(c.system, ctrl, ut, algo, N=c.P, rk=rk, expaction=c.expaction, u0=u0)
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        el = float(el.item())
        e2e = {"value": args.e2e_steps * c.batch / el, "unit": UNIT,
               "h2d_bytes_per_step": (2 * c.n + c.batch * c.K) * 8,
               "d2h_bytes_per_step": (c.batch + c.batch * c.K) * 8,
               "api": "direct_adjoint_loop(numpy host arrays); J and dJ/dc read to the host each step, "
                      "u(T) / q†(0) / ∫q† kept as device snapshots copied on first access"}
        # the same with every n-sized result field read to the host each step (u(T), q†(0), ∫q† dt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            lp = direct_adjoint_loop(c.system, ctrl, ut, algo, N=c.P, rk=rk, expaction=c.expaction, u0=u0)
            fields = (lp.direct.final_state, lp.adjoint.initial_state, lp.adjoint.integral)
        torch.cuda.synchronize()
        el2 = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(el2, op=dist.ReduceOp.MAX)
        e2e["with_result_fields"] = {"value": args.e2e_steps * c.batch / float(el2.item()), "unit": UNIT,
                                     "d2h_bytes_per_step": (c.batch + c.batch * c.K) * 8 + sum(int(f.nbytes) for f in fields)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference(args.config, cpu_workers())
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port", "sample": r["sample"],
               "host": r["host"]}
        if "unit_seconds" in r:
            cpu["unit_seconds"] = r["unit_seconds"]
        val = load_cpu_validation(args.config)
        if val:
            cpu["validation"] = val

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded inputs, paper_2004_00546_b200/configs.py)",
            "config": config_block(args.config, world),
            "roofline": roofline, "phases": phase_ms,
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": launches,
            "J": float(J[0]),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
