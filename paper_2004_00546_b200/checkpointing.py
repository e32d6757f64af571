"""Equispaced checkpointing on the GPU path.

Mirror of `pkg/src/paradjoint/checkpointing.py:34-267` (`CheckpointSchedule`,
`MemoryCounter`, `run_checkpointed_loop`) for the BASELINE objective
J = ½‖u(T) − u_target‖² and time-constant controls:

* phase 1 (`checkpointing.py:161-181`): a rough forward sweep over the M+1 segments
  keeps only the M+1 segment-start states (the direct solve of each segment runs on
  the device; only its final state is read back);
* phase 2 (`checkpointing.py:192-251`): segments are walked backward; each segment's
  direct solution is recomputed from its checkpoint (the Burgers dense trajectory of
  that segment only is resident), its Paraexp adjoint is seeded with the carried
  q† (`px_set_adjoint_terminal`), and the gradient, ∫q† dt and q†(t_m) accumulate.

Each segment is a fresh [0, T/(M+1)] problem with ``N`` slices (the reference's
`seg_partition`), so one engine (one set of HBM buffers sized for a segment) serves
every segment: device memory for the Burgers trajectory falls from P·n_s + 1 to
N·n_s + 1 nodes and, for the linear testbed, the lane buffers from P to N lanes.
The forward sweep is the same step sequence as the unsegmented sweep (bitwise for
the serial Burgers direct); the adjoint's Paraexp decomposition is per segment, so
for M > 0 it differs from the unsegmented one by the Paraexp approximation
(exp-action truncation; frozen-operator error for Burgers), and for M = 0 it is the
plain loop.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import _native as NV
from .errors import ConfigError
from .optimization import HYBRID, LINEAR, _default_expaction, get_engine
from .partition import RK4Config
from .systems import System


@dataclass(frozen=True)
class CheckpointSchedule:
    """Equispaced checkpoint times inside (0, T) (API of `checkpointing.py:34-59`).

    ``checkpoints`` = M interior checkpoints split [0, T] into M + 1 equal segments;
    the edges are ``T·i/(M+1)``, i = 0 … M+1.
    """

    T: float
    checkpoints: int

    def __post_init__(self):
        if not self.T > 0:
            raise ValueError("T must be positive")
        if self.checkpoints < 0:
            raise ValueError("checkpoint count cannot be negative")

    def _edges(self) -> np.ndarray:
        return np.linspace(0.0, 1.0, self.checkpoints + 2) * self.T

    @property
    def segment_count(self) -> int:
        return self.checkpoints + 1

    @property
    def times(self) -> np.ndarray:
        """The M interior checkpoint times."""
        return self._edges()[1:-1]

    @property
    def segment_bounds(self) -> list[tuple[float, float]]:
        e = [float(x) for x in self._edges()]
        e[-1] = float(self.T)
        return list(zip(e[:-1], e[1:]))


@dataclass
class MemoryCounter:
    """Dense-trajectory node bookkeeping (API of `checkpointing.py:62-76`).

    ``current`` nodes resident now, ``peak`` the high-water mark, ``total_allocated``
    every node ever acquired.
    """

    current: int = 0
    peak: int = 0
    total_allocated: int = 0

    def acquire(self, nodes: int) -> None:
        self.total_allocated += nodes
        self.current += nodes
        if self.current > self.peak:
            self.peak = self.current

    def release(self, nodes: int) -> None:
        self.current -= nodes


@dataclass
class CheckpointRun:
    """Result of `run_checkpointed_loop` (`checkpointing.py:79-91`, GPU fields)."""

    gradient: np.ndarray            # (B, K) ∂J/∂c
    qdag0: np.ndarray               # (B, n) q†(0)
    cost: np.ndarray                # (B,) J
    integral: np.ndarray            # (B, n) ∫₀ᵀ q† dt
    final_state: np.ndarray         # (B, n) u(T)
    segment_bounds: list[tuple[float, float]]
    checkpoint_states: list[np.ndarray]           # u(t_m), m = 0 … M
    adjoint_checkpoint_states: list[np.ndarray]   # q†(t_m), m = 0 … M
    memory: MemoryCounter
    segment_grads: list[np.ndarray] = field(default_factory=list)


def segment_system(system: System, T_seg: float) -> System:
    """The system on a segment in local time τ = t − t0 (the controls are time-constant,
    so only the horizon changes; `checkpointing.py:94-101`)."""
    return dataclasses.replace(system, spec=dataclasses.replace(system.spec, T=T_seg))


def run_checkpointed_loop(
    system: System,
    f: np.ndarray,
    q_true: np.ndarray,
    sched: CheckpointSchedule,
    algorithm: str | None = None,
    N: int = 1,
    rk: RK4Config | None = None,
    expaction=None,
    u0: np.ndarray | None = None,
    backend: str = "cuda",
) -> CheckpointRun:
    """Direct-adjoint loop under equispaced checkpointing (`checkpointing.py:119-267`).

    ``N`` is the number of Paraexp slices per segment (as the reference's
    `seg_partition`); ``algorithm`` is "linear" (advection–diffusion) or "hybrid"
    (Burgers: serial direct recomputed per segment + frozen-operator Paraexp adjoint).
    """
    if backend != "cuda":
        raise ValueError(f"unknown backend {backend!r}; the B200 path provides ('cuda',)")
    if rk is None:
        raise ConfigError("rk: an RK4Config(dt) is required (fixed-step RK4)")
    if abs(sched.T - system.spec.T) > 1e-12 * system.spec.T:
        raise ValueError("schedule horizon differs from the system's T")
    algorithm = algorithm or (LINEAR if system.is_linear else HYBRID)
    if algorithm not in (LINEAR, HYBRID):
        raise ValueError(f"checkpointed runs support 'linear' and 'hybrid', not {algorithm!r}")
    if (algorithm == LINEAR) != system.is_linear:
        raise ValueError(f"the {algorithm} algorithm does not match the testbed")
    expaction = expaction or _default_expaction(system)
    ctrl = np.atleast_2d(np.asarray(f, dtype=np.float64))
    B = ctrl.shape[0]
    if ctrl.shape[1] != system.basis.K:
        raise ValueError("control coefficient count does not match the basis")
    if B != 1:
        # segment start states differ per control member; the handle takes one u0
        raise ConfigError("checkpointed runs take one control (batch 1)")
    n = system.n
    u0 = np.zeros(n) if u0 is None else np.asarray(u0, dtype=np.float64).reshape(-1)
    ut = np.asarray(q_true, dtype=np.float64).reshape(-1)

    bounds = sched.segment_bounds
    M1 = sched.segment_count
    T_seg = sched.T / M1
    seg = segment_system(system, T_seg)
    eng = get_engine(seg, N, rk, expaction, B)
    nodes_per_segment = N * eng.spec.nsteps + 1 if not system.is_linear else 0
    memory = MemoryCounter()

    # ---- phase 1: rough sweep, checkpoint states only ----------------------
    states = [u0.reshape(1, n).copy()]
    for m in range(M1 - 1):
        eng.set_inputs(states[-1][0], ut, ctrl)
        eng.direct_partial()
        if system.is_linear:
            eng.finish_direct()          # u(t_{m+1}) = u(t_m) + carries
        states.append(eng.get(NV.PX_FIELD_UT).reshape(1, n))
        # Burgers: this segment's dense trajectory is overwritten by the next one

    # ---- phase 2: backward sweep with recompute ----------------------------
    grad = np.zeros((1, system.basis.K))
    integral = np.zeros((1, n))
    qdag = None
    cost = None
    uT = None
    adj_states: list[np.ndarray] = []
    seg_grads: list[np.ndarray] = []
    for m in range(M1 - 1, -1, -1):
        eng.set_inputs(states[m][0], ut, ctrl)
        last = qdag is None
        if last or not system.is_linear:
            # Burgers: recompute the segment's dense trajectory (the adjoint's Jᵀ(u(t)) and
            # frozen operators need it); linear: only the last segment's u(T) is needed
            eng.direct_partial()
            memory.acquire(nodes_per_segment)
        if last:   # q†(T) = u(T) − u_target, J
            eng.finish_direct()
            cost = eng.get(NV.PX_FIELD_J)
            uT = eng.get(NV.PX_FIELD_UT).reshape(1, n)
        else:
            eng.set_adjoint_terminal(qdag)
        eng.adjoint_partial()
        eng.finish_adjoint()
        g = eng.get(NV.PX_FIELD_GRAD).reshape(1, system.basis.K)
        grad += g
        seg_grads.append(g)
        integral += eng.get(NV.PX_FIELD_G).reshape(1, n)
        qdag = eng.get(NV.PX_FIELD_QDAG0).reshape(1, n)
        adj_states.append(qdag.copy())
        if last or not system.is_linear:
            memory.release(nodes_per_segment)
    return CheckpointRun(
        gradient=grad, qdag0=qdag, cost=cost, integral=integral, final_state=uT,
        segment_bounds=bounds, checkpoint_states=states, adjoint_checkpoint_states=adj_states[::-1],
        memory=memory, segment_grads=seg_grads[::-1],
    )


@dataclass
class CheckpointTrackingRun:
    """Result of `run_checkpointed_tracking` (the reference's `CheckpointRun`, `checkpointing.py:79-91`)."""

    gradient: np.ndarray            # (n,) ∂L/∂f
    qdag0: np.ndarray               # (n,) q†(0)
    cost: float                     # J = (1/T)∫‖q − q_t‖² dt
    final_state: np.ndarray         # (n,) q(T)
    segment_bounds: list[tuple[float, float]]
    checkpoint_states: list[np.ndarray]
    adjoint_checkpoint_states: list[np.ndarray]
    memory: MemoryCounter


def run_checkpointed_tracking(system: System, f, target, sched: CheckpointSchedule, N: int = 1,
                              rk: RK4Config | None = None, expaction=None, law=None, k_ratio: float | None = None,
                              u0=None, overlap: bool = True) -> CheckpointTrackingRun:
    """The reference's checkpointed loop with its own objective on the Burgers testbed, algorithm
    "hybrid" (`checkpointing.py:119-267`): phase one sweeps the segments forward keeping only the
    checkpoint states; phase two walks them backward — each segment is one hybrid solve
    (`tracking.solve_hybrid_tracking`) from its checkpoint with the forcing law and the target in
    the segment's local time, seeded with the carried adjoint state as terminal data (the final
    span, `hybrid.py:232-233`), its cost and gradient shares (T_seg/T of the segment's own
    (1/T_seg)∫) accumulated. ``N`` slices per segment: geometric with ``k_ratio``, else equal.
    ``target`` on the RK4 nodes of the whole horizon, (S+1, n); S a multiple of the segment count.
    With equal slices the result equals the plain hybrid loop on (M+1)·N slices up to the
    exp-action truncation (the same frozen operators and carries)."""
    from .hybrid import TimeLaw, make_hybrid_plan
    from .tracking import get_tracking_engine, solve_hybrid_tracking, _offsets_for
    if rk is None:
        raise ConfigError("rk: an RK4Config(dt) is required (fixed-step RK4)")
    if system.is_linear:
        raise ConfigError("run_checkpointed_tracking: the Burgers testbed (hybrid algorithm)")
    if abs(sched.T - system.spec.T) > 1e-12 * system.spec.T:
        raise ValueError("schedule horizon differs from the system's T")
    law = law or TimeLaw.constant()
    n = system.n
    f = np.asarray(f, dtype=np.float64).reshape(n)
    target = np.asarray(target, dtype=np.float64)
    M1 = sched.segment_count
    S = target.shape[0] - 1
    if target.shape != (S + 1, n) or S % M1:
        raise ValueError(f"target: (S+1, n) on the RK4 nodes with S a multiple of the {M1} segments")
    if abs(system.spec.T / S - rk.dt) > 1e-12 * rk.dt:
        raise ConfigError("rk.dt must be the node spacing T/S of the target")
    S_seg = S // M1
    T_seg = sched.T / M1
    seg = segment_system(system, T_seg)
    plan = make_hybrid_plan(T_seg, N, k_ratio) if k_ratio is not None else None
    u0 = np.zeros(n) if u0 is None else np.asarray(u0, dtype=np.float64).reshape(n)
    memory = MemoryCounter()
    offs, _ = _offsets_for(seg, plan, N, rk)
    # ---- phase 1: rough sweep, checkpoint states only ----------------------
    states = [u0.copy()]
    zeros = np.zeros((S_seg + 1, n))
    for m in range(M1 - 1):
        eng = get_tracking_engine(seg, offs, law.shifted(m * T_seg), 1, False)
        eng.set_inputs(states[-1], f, zeros)
        eng.direct(overlap=False)
        states.append(eng.get(NV.PX_HFIELD_UT, (1, n))[0])
    # ---- phase 2: backward sweep with recompute ----------------------------
    grad = np.zeros(n)
    cost = 0.0
    qdag = None
    uT = None
    adj_states = []
    share = T_seg / sched.T
    for m in range(M1 - 1, -1, -1):
        memory.acquire(S_seg + 1)
        r = solve_hybrid_tracking(seg, states[m], f, target[m * S_seg:(m + 1) * S_seg + 1], plan, N, rk, expaction,
                                  law.shifted(m * T_seg), qdag, overlap)
        if uT is None:
            uT = r.final_state[0]
        cost += float(r.J[0]) * share
        grad += r.grad[0] * share
        qdag = r.qdag0[0]
        adj_states.append(qdag.copy())
        memory.release(S_seg + 1)
    return CheckpointTrackingRun(gradient=grad, qdag0=qdag, cost=cost, final_state=uT,
                                 segment_bounds=sched.segment_bounds, checkpoint_states=states,
                                 adjoint_checkpoint_states=adj_states[::-1], memory=memory)
