"""GPU timing profile and multi-GPU strong-scaling model (§8(f) rank 4).

The reference's `scaling.py` measures per-time-unit kernel costs τ_I, τ_H on CPU
workers and predicts Paraexp speedups in closed form (`scaling.py:29-110`).
Here the same idea is applied to the GPU decomposition: the
per-unit device times of the kernel classes are measured on ONE GPU with the
engine's CUDA-event phase timing, and the block-scan schedule on G GPUs is
costed exactly from the planner's term counts:

    rank g (slices [p0, p1)):  RK4 lanes (p1−p0)·n_s·(τ_rk4 + τ_rk4†)
                             + own carry (p1−p0−1)·terms(Δ)·(τ_term + τ_term†)
                             + long spans terms((P−p1)Δ)·τ_term  [g < G−1]
                                       + terms(p0Δ)·τ_term†       [g > 0]
    plus two NCCL allreduces (u(T): B·n doubles; gradient: B·K doubles),
    ring bus time 2(G−1)/G · bytes / bw (bw defaults to the measured 725 GB/s).

The predicted time per gradient is the slowest rank's; speedup = t(1)/t(G).
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass

from .configs import BaselineCase
from .expaction import KrylovPlan, plan_for
from .partition import rank_block

NCCL_BUS_BW = 725e9  # B/s, 8-rank all-reduce bus bandwidth measured on this pool (B200_PROFILING.md)


@dataclass(frozen=True)
class GpuProfile:
    """Seconds per unit on one B200 (lane-step: one RK4 step of one n-field lane;
    term: one Chebyshev term, or one Arnoldi step for Krylov, on one vector)."""

    rk4_direct: float
    rk4_adjoint: float
    term_direct: float
    term_adjoint: float
    fixed: float = 0.0          # per-gradient constant (sources, reductions, projections)
    bus_bw: float = NCCL_BUS_BW

    def to_json(self) -> str:
        return json.dumps(asdict(self))


def profile_from_timing(case: BaselineCase, timing: dict, stats_terms: dict, gradients: int) -> GpuProfile:
    """Per-unit times from `ParaexpEngine.timing()` accumulated over ``gradients``
    single-GPU evaluations; ``stats_terms`` = {"rk4_lane_steps_direct", ...} counts."""
    g = max(gradients, 1)
    lane_steps = case.batch * case.P * max(case.nsteps - (0 if case.grid.dim == 1 else 1), 1)
    region = case.system.region()
    sp = plan_for(region, case.spec.T / case.P, case.expaction)
    terms = (case.P - 1) * sp.terms * case.batch
    ms = lambda k: timing[k]["ms"] / 1e3 / g
    return GpuProfile(
        rk4_direct=ms("rk4_direct") / lane_steps,
        rk4_adjoint=ms("rk4_adjoint") / lane_steps,
        term_direct=ms("exp_direct") / max(terms, 1),
        term_adjoint=ms("exp_adjoint") / max(terms, 1),
        fixed=ms("other"),
    )


@dataclass(frozen=True)
class ScalingPrediction:
    G: int
    seconds: float
    speedup: float
    efficiency: float
    critical_rank: int
    breakdown: dict


def predict_blockscan(case: BaselineCase, G: int, prof: GpuProfile) -> ScalingPrediction:
    if not case.system.is_linear:
        raise ValueError("the block-scan model covers the linear testbed")
    region = case.system.region()
    delta = case.spec.T / case.P
    slice_terms = plan_for(region, delta, case.expaction).terms
    steps = max(case.nsteps - (0 if case.grid.dim == 1 else 1), 1)

    def rank_time(p0, p1):
        Pl = p1 - p0
        rk4 = Pl * steps * case.batch * (prof.rk4_direct + prof.rk4_adjoint)
        scan = (Pl - 1) * slice_terms * case.batch * (prof.term_direct + prof.term_adjoint)
        long_d = long_a = 0.0
        if p1 < case.P:
            long_d = plan_for(region, (case.P - p1) * delta, case.expaction, base_span=delta).terms \
                * case.batch * prof.term_direct
        if p0 > 0:
            long_a = plan_for(region, p0 * delta, case.expaction, base_span=delta).terms \
                * case.batch * prof.term_adjoint
        return rk4, scan, long_d, long_a

    def total(G):
        worst, who, parts = 0.0, 0, {}
        for r in range(G):
            p0, p1 = rank_block(case.P, r, G)
            rk4, scan, ld, la = rank_time(p0, p1)
            t = rk4 + scan + ld + la + prof.fixed
            if t > worst:
                worst, who, parts = t, r, {"rk4": rk4, "scan": scan, "long_direct": ld, "long_adjoint": la}
        comm = 0.0
        if G > 1:
            nbytes = 8.0 * case.batch * (case.n + case.K)
            comm = 2.0 * (G - 1) / G * nbytes / prof.bus_bw
        parts["allreduce"] = comm
        parts["fixed"] = prof.fixed
        return worst + comm, who, parts

    t1, _, _ = total(1)
    tg, who, parts = total(G)
    return ScalingPrediction(G, tg, t1 / tg, t1 / tg / G, who, parts)


def scaling_table(case: BaselineCase, prof: GpuProfile, gpus=(1, 2, 4, 8)) -> list[ScalingPrediction]:
    return [predict_blockscan(case, G, prof) for G in gpus if G <= case.P]
