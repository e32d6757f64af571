#!/usr/bin/env python
"""Benchmark: Paraexp direct-adjoint gradient evaluations per second on B200.

One *step* = one full direct-adjoint gradient evaluation (direct Paraexp sweep,
objective, adjoint Paraexp sweep, gradient projection) of BASELINE config 5
(2D advection–diffusion 2048², P = 512 slices, Chebyshev tol 1e-10; the largest
config and the one BASELINE names for 1/2/4/8 GPUs). Multi-GPU (torchrun): the
P slices are sharded in contiguous blocks, partials allreduced over NCCL
(strong scaling: total work fixed). ``--config k`` benches another config.

Line fields (see the task contract): ``value`` = gradient evals/s with inputs
resident in HBM (device-timed with CUDA events, max over ranks); ``e2e`` = the
same metric through the public API ``direct_adjoint_loop`` with host numpy
inputs/outputs (H2D/D2H inside the timed region, host wall clock);
``roofline`` = the dominant kernel class's algorithmic bytes per launch (SURVEY §8(d)
per-unit bytes × the units a launch processes: 24n per lane and RK4 step) ÷ its
average launch duration (CUDA events around the phase on the work stream) vs the
measured HBM peak — above 1 for kernels that fuse two steps per launch, with the DRAM
they actually move (committed ncu capture) beside it; ``cpu_baseline`` = the numpy oracle port on this host's cores
(bounded sample, extrapolated); ``--impl reference`` prints the CPU arm alone.
"""

from __future__ import annotations

import argparse
import json
import math
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


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_profile(phase_kernel: str, config: int) -> dict:
    """The committed ncu summary (per-launch DRAM bytes, limiter) for the dominant kernel."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        d = json.load(f)
    return d.get(f"c{config}", {}).get(phase_kernel) or {}


def load_traffic(phase_kernel: str, config: int):
    """ncu dram bytes per launch for the dominant kernel, from the committed profile summary."""
    return load_profile(phase_kernel, config).get("dram_bytes_per_launch")


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
# CPU baseline: the numpy oracle port on the host cores (bounded sample)
# ---------------------------------------------------------------------------


def _cpu_worker(args):
    """Time per-unit oracle costs on the full-size field: RK4 step (direct, adjoint
    with ∫), Chebyshev term with and without the φ₁ accumulator."""
    cfg_index, reps = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle.config_mode import stencil_apply
    from paper_2004_00546_b200 import baseline
    c = baseline(cfg_index)
    st = c.system.A.as_tuple()
    nx, ny = c.grid.nx, c.grid.ny
    n = c.n
    rng = np.random.default_rng(0)
    y = rng.standard_normal(n)
    g = rng.standard_normal(n)
    z = np.zeros(n)
    apply = lambda u: stencil_apply(st, u, nx, ny)
    h = 1e-5

    def rk4(y, z, want_z):
        k1 = apply(y) + g
        Y2 = y + (0.5 * h) * k1
        k2 = apply(Y2) + g
        Y3 = y + (0.5 * h) * k2
        k3 = apply(Y3) + g
        Y4 = y + h * k3
        k4 = apply(Y4) + g
        if want_z:
            z = z + (h / 6.0) * (y + 2.0 * Y2 + 2.0 * Y3 + Y4)
        return y + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4), z

    out = {}
    t = time.perf_counter()
    for _ in range(reps):
        y, _ = rk4(y, z, False)
    out["rk4_direct"] = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    for _ in range(reps):
        y, z = rk4(y, z, True)
    out["rk4_adjoint"] = (time.perf_counter() - t) / reps
    up, uc, acc, pac = rng.standard_normal(n), rng.standard_normal(n), np.zeros(n), np.zeros(n)
    t = time.perf_counter()
    for _ in range(2 * reps):
        un = 2e-3 * (apply(uc) - 1.0 * uc) + up
        up, uc = uc, un
        acc = acc + 0.1 * uc
    out["term"] = (time.perf_counter() - t) / (2 * reps)
    t = time.perf_counter()
    for _ in range(2 * reps):
        un = 2e-3 * (apply(uc) - 1.0 * uc) + up
        up, uc = uc, un
        acc = acc + 0.1 * uc
        pac = pac + 0.1 * uc
    out["term_phi"] = (time.perf_counter() - t) / (2 * reps)
    return out


def cpu_reference_rate(cfg_index: int, reps: int = 1, workers: int | None = None):
    """Gradient evals/s of the oracle port with W host processes, each owning a
    contiguous slice block (the GPU decomposition); per-unit costs
    measured concurrently on the full-size field, then the block-scan critical
    path (own slices + long span) extrapolated from the planner's term counts."""
    import multiprocessing as mp
    from paper_2004_00546_b200 import baseline
    from paper_2004_00546_b200.expaction import KrylovPlan, plan_for
    from paper_2004_00546_b200.partition import rank_block
    c = baseline(cfg_index)
    W = workers or os.cpu_count() or 1
    W = max(1, min(W, c.P))
    t0 = time.perf_counter()
    ctx = mp.get_context("spawn")
    with ctx.Pool(W) as pool:
        res = pool.map(_cpu_worker, [(cfg_index, reps)] * W)
    wall = time.perf_counter() - t0
    u = {k: max(r[k] for r in res) for k in res[0]}  # contended per-unit cost (slowest worker)
    region = c.system.region() if c.system.is_linear else None
    delta = c.spec.T / c.P
    worst = 0.0
    for r in range(W):
        p0, p1 = rank_block(c.P, r, W)
        Pl = p1 - p0
        t = Pl * c.nsteps * (u["rk4_direct"] + u["rk4_adjoint"])
        if region is not None:
            sp = plan_for(region, delta, c.expaction)
            per = sp.terms if not isinstance(sp, KrylovPlan) else sp.terms * 4  # Arnoldi ≈ 4 vector passes/step
            t += (Pl - 1) * per * (u["term"] + u["term_phi"])
            if p1 < c.P:
                t += plan_for(region, (c.P - p1) * delta, c.expaction, base_span=delta).terms * u["term"]
            if p0 > 0:
                t += plan_for(region, p0 * delta, c.expaction, base_span=delta).terms * u["term_phi"]
        worst = max(worst, t)
    rate = c.batch / worst
    sample = (f"per-unit oracle costs timed on the full {c.grid.nx}x{c.grid.ny} field by {W} concurrent "
              f"numpy processes ({reps} RK4 steps direct+adjoint, {4 * reps} Chebyshev terms each; "
              f"{wall:.1f}s wall), extrapolated to one gradient = max over workers of own-slice RK4 "
              f"({c.nsteps} steps/slice) + block scan + long span (blockscan over W workers)")
    return rate, W, sample, u


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    rates = []
    for i in range(args.warmup + args.steps):
        rate, W, sample, _ = cpu_reference_rate(args.config, reps=args.cpu_reps)
        if i >= args.warmup:
            rates.append(rate)
    v = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, configs.py)",
        "config": config_block(args.config, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": W, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_block(index, world):
    from paper_2004_00546_b200 import baseline
    c = baseline(index)
    return {"workload": c.name, "grid": [c.grid.nx, c.grid.ny], "P": c.P, "steps_per_slice": c.nsteps,
            "T": c.spec.T, "dt": c.spec.T / c.P / c.nsteps, "batch": c.batch, "K": c.K,
            "expaction": type(c.expaction).__name__, "tol": c.expaction.tol,
            "parallelism": f"slices{world}" if world > 1 else "single",
            "l2": "inputs larger than L2 (lane buffers of P×n fp64)" if c.n * c.P * 8 > 126e6 else
                  "working set fits L2 (not flushed)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-reps", type=int, default=3, help="oracle unit repetitions per CPU worker (~3 s each)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="warmup+steps only (for ncu); no extras")
    args = ap.parse_args()
    if args.warmup < 3 and not args.profile_only and args.impl != "reference":
        args.warmup = 3

    if args.impl == "reference":
        return run_reference(args)

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
    gpu_evals = args.steps * c.batch
    value = gpu_evals / (ms_max / 1e3)

    # dominant kernel class: the phase with the largest device time
    dom = max(phases, key=lambda k: phases[k]["ms"])
    ph = phases[dom]
    peak, peak_src = load_peaks()
    avg_launch_s = (ph["ms"] / 1e3) / max(ph["launches"], 1)
    bytes_per_launch = ph["bytes"] / max(ph["launches"], 1)
    achieved = bytes_per_launch / avg_launch_s / 1e9 if avg_launch_s > 0 else 0.0
    two_d = c.grid.dim == 2
    # two RK4 steps per launch (k_rk4_march2) when the phase launched fewer kernels than steps
    fused = two_d and ph["launches"] / args.steps < (c.nsteps - 1) * 0.75
    # (the library's default variant: three columns per thread, 64-thread CTAs, in strip
    # mode; PX_M2_COLS=2 selects the two-column k_rk4_march2)
    cols = int(os.environ.get("PX_M2_COLS", "3"))
    m2 = "k_rk4_marchc<3,64,3,4,br>" if cols == 3 and c.grid.nx > 192 else "k_rk4_march2<false,128,3,3,tma>"
    kernel_name = {"rk4_direct": (m2 if fused else "k_rk4_march<false>") if two_d
                   else "k_rk4_lane1d<false>",
                   # 2D adjoint lanes run the direct kernel: their ∫ is recovered in closed form
                   # (one cuFFT solve, `z_closed_form`) instead of a per-lane accumulator
                   "rk4_adjoint": (m2 + " (adjoint lanes)" if fused else "k_rk4_march<false>")
                   if two_d else "k_rk4_lane1d<true>",
                   "exp_direct": "k_cheb_march<M>" if two_d else "k_scan1d",
                   "exp_adjoint": "k_cheb_march<M>+phi" if two_d else "k_scan1d+phi",
                   "other": "reductions/projection"}[dom]
    if type(c.expaction).__name__ == "KrylovConfig" and dom.startswith("exp"):
        kernel_name = "Arnoldi CGS2 (k_kr_spmv_dots/k_kr_update/k_kr_expm/k_kr_combine)"
    if not c.system.is_linear:
        kernel_name = {"rk4_direct": "k_burgers_direct", "rk4_adjoint": "k_burgers_adjoint_rk4+k_burgers_scan"}.get(
            dom, kernel_name)
    roofline = {"bound": "hbm", "kernel": kernel_name, "phase": dom, "achieved": achieved, "peak": peak,
                "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_launch_s * 1e3,
                "share_of_step": ph["ms"] / sum(p["ms"] for p in phases.values()),
                "traffic": load_traffic(dom, args.config)}
    prof = load_profile(dom, args.config)
    if prof.get("limiter"):
        roofline["limiter"] = prof["limiter"]
    if prof.get("dram_bytes_per_launch") and prof.get("duration_ms"):
        # what the kernel actually moves, from the committed ncu capture (its own clock)
        dgbs = prof["dram_bytes_per_launch"] / (prof["duration_ms"] / 1e3) / 1e9
        roofline["dram_achieved_ncu"] = dgbs
        roofline["dram_frac_ncu"] = dgbs / peak
    if roofline["frac"] > 1.0 and fused and dom.startswith("rk4"):
        roofline["note"] = ("temporal blocking: each launch advances two RK4 steps and streams y, b and y_out "
                            "once (24n per lane per launch, half the SURVEY §8(d) model of 24n per lane-step), "
                            "so frac on the model exceeds 1; the DRAM actually moved is `traffic` "
                            "(dram_frac_ncu), and the binding resource is the shared-memory data pipe (limiter)")
    elif roofline["frac"] > 1.0:
        roofline["note"] = ("on-chip kernel (state resident in shared memory / registers across steps or "
                            "terms): the per-unit HBM model of SURVEY §8(d) counts bytes this kernel never "
                            "moves, so frac > 1; its binding resources are the fp64 pipe and barrier latency")
    phase_gbs = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                     "GB/s": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None}
                 for k, v in phases.items()}
    whole = stats["algorithmic_bytes"] / (ms_max / 1e3) / 1e9

    eng.close()  # the public-API leg below owns its own engine (HBM scratch)
    del dev
    torch.cuda.empty_cache()
    # e2e: public API with host inputs/outputs, host wall clock
    e2e = None
    if args.e2e_steps > 0:
        rk = RK4Config(c.dt)
        direct_adjoint_loop(c.system, ctrl, ut, "linear" if c.system.is_linear else "hybrid", N=c.P, rk=rk,
                            expaction=c.expaction, u0=u0)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            direct_adjoint_loop(c.system, ctrl, ut, "linear" if c.system.is_linear else "hybrid", N=c.P,
                                rk=rk, expaction=c.expaction, u0=u0)
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

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, W, sample, units = cpu_reference_rate(args.config, reps=args.cpu_reps)
        cpu = {"value": rate, "unit": UNIT, "cores": W, "kind": "port", "sample": sample,
               "unit_seconds": units}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded inputs, paper_2004_00546_b200/configs.py)",
            "config": config_block(args.config, world),
            "roofline": roofline, "whole_step_algorithmic_GBps": whole, "phases": phase_gbs,
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": launches,
            "J": float(J[0]),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
