"""The reference's hybrid algorithm on the GPU (`hybrid.py:1-290`).

The reference sweeps the direct equation serially across its workers and, as soon as a worker
has its chunk, starts that chunk's adjoint inhomogeneous solve (zero terminal data, driven by
the adjoint source of the tracking objective) so that it overlaps the rest of the direct sweep;
the geometric partition makes all those solves finish together; afterwards the homogeneous
adjoint problems run over the full spans with frozen operators.

On the B200 the serial direct sweep occupies one CTA per batch member; the adjoint slice solves
are one CTA each on the other SMs and start the moment the direct kernel publishes that their
slice is complete (a per-slice progress flag in HBM, release/acquire), so they run *during* the
serial sweep instead of after it. The frozen-operator carry then walks the slices down. This
module holds the host side of that path:

* `partition_geometric`, `HybridPlan`, `make_hybrid_plan` (`hybrid.py:35-97`) — the same
  boundaries T_n = T(1 − rⁿ)/(1 − r^N), r = k/(k+1); `slice_offsets` snaps them to the RK4 node
  grid (every slice a whole number of the sweep's uniform steps, at least one);
* `estimate_k` (`hybrid.py:100-154`): the cost ratio k = τ_adjoint/τ_direct per unit of
  simulated time, measured on the device (CUDA events) on a pilot span;
* `TimeLaw`: the forcing's time law θ(t) = α + β·sin(ωt) + γ·cos(ωt) (the reference's
  f·sin(ωt), `problems.py:155-162`, is ``TimeLaw.sine(ω)``).

`direct_adjoint_loop(..., algorithm="hybrid", plan=HybridPlan, objective="tracking")`
(optimization.py) runs the loop; `solve_hybrid_tracking` is the solver-level entry.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, PilotTooShort
from .partition import GEOMETRIC, TimePartition


@dataclass(frozen=True)
class TimeLaw:
    """θ(t) = alpha + beta·sin(omega·t) + gamma·cos(omega·t) multiplying the forcing field."""

    alpha: float = 1.0
    beta: float = 0.0
    gamma: float = 0.0
    omega: float = 0.0

    def __post_init__(self):
        if self.omega < 0:
            raise ValueError("omega must be non-negative")
        for v in (self.alpha, self.beta, self.gamma, self.omega):
            if not math.isfinite(v):
                raise ValueError("time law coefficients must be finite")

    @staticmethod
    def constant() -> "TimeLaw":
        return TimeLaw(1.0, 0.0, 0.0, 0.0)

    @staticmethod
    def sine(omega: float) -> "TimeLaw":
        """The reference's forcing law sin(ωt) (`problems.py:155-162`, `systems.py:56-60`)."""
        return TimeLaw(0.0, 1.0, 0.0, float(omega))

    def as_tuple(self) -> tuple[float, float, float, float]:
        return (self.alpha, self.beta, self.gamma, self.omega)

    def __call__(self, t):
        return self.alpha + self.beta * np.sin(self.omega * t) + self.gamma * np.cos(self.omega * t)

    def shifted(self, t0: float) -> "TimeLaw":
        """The law in local time τ = t − t0: θ(t0 + τ) as α + β′ sin ωτ + γ′ cos ωτ (a segment of a
        checkpointed run, the reference's `_shifted_system`, `checkpointing.py:94-101`)."""
        c, s = math.cos(self.omega * t0), math.sin(self.omega * t0)
        return TimeLaw(self.alpha, self.beta * c - self.gamma * s, self.beta * s + self.gamma * c, self.omega)


def partition_geometric(T: float, N: int, k: float) -> TimePartition:
    """Boundaries T_n = T·(1 − rⁿ)/(1 − r^N), r = k/(k+1) (`hybrid.py:35-55`): later slices
    shrink by r so that the serial direct sweep plus each slice's adjoint solve end together."""
    if N < 1:
        raise ValueError("need at least one interval")
    if T <= 0 or k <= 0:
        raise ValueError("need positive T and k")
    r = k / (k + 1.0)
    b = T * (1.0 - r ** np.arange(N + 1, dtype=np.float64)) / (1.0 - r ** N)
    b[0], b[-1] = 0.0, T
    if np.any(np.diff(b) <= 0):
        raise ValueError(f"geometric partition degenerates for k={k:.3g}, N={N}: "
                         "the last widths underflow; reduce N")
    return TimePartition(b, kind=GEOMETRIC, ratio=float(k))


@dataclass(frozen=True)
class HybridPlan:
    """Geometric partition plus the measured cost ratio behind it (`hybrid.py:58-82`)."""

    partition: TimePartition
    k: float

    def __post_init__(self):
        w = self.partition.widths()
        r = self.k / (self.k + 1.0)
        if len(w) > 1 and np.max(np.abs(w[1:] - r * w[:-1])) > 1e-10 * np.max(w):
            raise ValueError("partition widths do not follow the k/(k+1) ratio")

    @property
    def N(self) -> int:
        return self.partition.N


def make_hybrid_plan(T: float, N: int, k: float, h_min: float = 0.0) -> HybridPlan:
    """The geometric plan; rejects partitions finer than the stepper (`hybrid.py:85-97`)."""
    part = partition_geometric(T, N, k)
    if h_min > 0.0 and float(np.min(part.widths())) < 2.0 * h_min:
        raise ValueError("smallest partition width is below twice the minimum step size; "
                         "reduce N or the cost ratio")
    return HybridPlan(part, float(k))


def slice_offsets(part: TimePartition, dt: float) -> np.ndarray:
    """Snap a partition to the uniform RK4 node grid of the serial sweep: S = ⌈T/dt⌉ steps of
    h = T/S; slice p covers nodes [o_p, o_{p+1}] with o_p the nearest node to T_p, every slice
    at least one step (the GPU sweeps and the oracle use these offsets)."""
    T = part.T
    S = max(1, int(math.ceil(T / dt - 1e-9)))
    N = part.N
    if S < N:
        raise ConfigError(f"dt: {S} steps cannot hold {N} slices")
    o = np.rint(part.boundaries / T * S).astype(np.int64)
    o[0], o[-1] = 0, S
    for p in range(1, N):
        # room for the slices on both sides, then at least one step after the previous edge
        o[p] = max(min(o[p], S - (N - p)), o[p - 1] + 1)
    return o


def aligned_partition(offsets: np.ndarray, T: float, ratio: float | None = None) -> TimePartition:
    """The partition the sweeps actually use: boundaries on the node grid (``slice_offsets``)."""
    S = int(offsets[-1])
    b = offsets.astype(np.float64) * (T / S)
    b[-1] = T
    if len(set(np.diff(offsets).tolist())) == 1:
        return TimePartition(b)
    return TimePartition(b, kind="node-aligned", ratio=ratio)


def estimate_k(system, pilot_fraction: float, rk, repeats: int = 3, law: TimeLaw | None = None) -> float:
    """k = τ_adjoint/τ_direct per unit of simulated time (`hybrid.py:100-154`), measured on the
    device: a pilot span of ``pilot_fraction``·T is swept by the serial direct kernel and by one
    adjoint slice kernel (tracking source, CUDA events, median of ``repeats``)."""
    if not 0.0 < pilot_fraction <= 0.1:
        raise ValueError("pilot_fraction must lie in (0, 0.1]")
    span = pilot_fraction * system.spec.T
    steps = int(round(span / rk.dt))
    if steps < 2:
        raise PilotTooShort("pilot resolved fewer than 2 steps; widen pilot_fraction")
    t_dir, t_adj = _pilot_times(system, steps, rk, repeats, law or TimeLaw.constant())
    return t_adj / t_dir


def _pilot_times(system, steps: int, rk, repeats: int, law: TimeLaw) -> tuple[float, float]:
    """Device seconds per unit time of the direct sweep and of one slice's adjoint solve
    (`hybrid.py:100-129`; the tests patch it with synthetic costs, as the reference's do)."""
    from .tracking import pilot_times
    return pilot_times(system, steps, rk, repeats, law)
