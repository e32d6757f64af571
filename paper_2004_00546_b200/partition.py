"""Time partition, slice rule and rank blocks (host logic).

`TimePartition` / `partition_equidistant` / `worker_plans` mirror
`pkg/src/paradjoint/paraexp.py:31-97`. The fixed-step slice rule and the
contiguous per-rank slice blocks are this path's additions (SURVEY.md §7.2-3,
§8(e)).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

EQUIDISTANT = "equidistant"
GEOMETRIC = "geometric"


@dataclass(frozen=True)
class TimePartition:
    """Ordered boundaries 0 = T_0 < T_1 < … < T_N = T (`paraexp.py:31-69`)."""

    boundaries: np.ndarray
    kind: str = EQUIDISTANT
    ratio: float | None = None  # the hybrid's cost ratio k of a geometric partition (`paraexp.py:31-69`)

    def __post_init__(self):
        b = np.asarray(self.boundaries, dtype=np.float64)
        object.__setattr__(self, "boundaries", b)
        if b.ndim != 1 or len(b) < 2:
            raise ValueError("partition needs at least two boundaries")
        if b[0] != 0.0:
            raise ValueError("partition must start at 0")
        if not np.all(np.diff(b) > 0):
            raise ValueError("partition boundaries must be strictly increasing")
        if self.kind == EQUIDISTANT:
            widths = np.diff(b)
            if np.max(np.abs(widths - widths[0])) > 1e-12 * b[-1]:
                raise ValueError("equidistant partition has unequal widths")

    @property
    def N(self) -> int:
        return len(self.boundaries) - 1

    @property
    def T(self) -> float:
        return float(self.boundaries[-1])

    def width(self, p: int) -> float:
        return float(self.boundaries[p + 1] - self.boundaries[p])

    def widths(self) -> np.ndarray:
        return np.diff(self.boundaries)


def partition_equidistant(T: float, N: int) -> TimePartition:
    """Split [0, T] into N equal intervals (`paraexp.py:72-78`)."""
    if N < 1:
        raise ValueError("need at least one interval")
    if T <= 0:
        raise ValueError("T must be positive")
    return TimePartition(T * np.arange(N + 1) / N, kind=EQUIDISTANT)


@dataclass(frozen=True)
class WorkerPlan:
    p: int
    t_start: float
    t_end: float
    direct_homogeneous: int
    adjoint_homogeneous: int


def worker_plans(part: TimePartition) -> list[WorkerPlan]:
    """Chain counts of the reference's neighbour form (`paraexp.py:92-97`).

    The GPU path replaces the P(P−1)/2 chains by one summed-chain carry per
    sweep (P−1 slice-width actions); the counts are kept for reporting.
    """
    return [WorkerPlan(p, part.boundaries[p], part.boundaries[p + 1], p, part.N - 1 - p)
            for p in range(part.N)]


@dataclass(frozen=True)
class RK4Config:
    """Classical fixed-step RK4 (BASELINE's stepper; replaces the reference's
    adaptive DOPRI5 `RKConfig`, `timestepping.py:86-104`)."""

    dt: float

    def __post_init__(self):
        if not self.dt > 0:
            raise ValueError("dt must be positive")


def slice_steps(width: float, dt: float) -> int:
    """Slice rule: n_p = ⌈Δ_p/dt⌉ uniform steps of Δ_p/n_p.

    A relative slack of 1e-9 keeps exact multiples (Δ/dt = 250 up to rounding)
    from rounding up to an extra step.
    """
    return max(1, int(math.ceil(width / dt - 1e-9)))


def rank_block(P: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice block [p0, p1) of ``rank``.

    Blocks differ in size by at most one slice; earlier ranks get the extra.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if world > P:
        raise ValueError(f"cannot shard {P} slices over {world} ranks")
    base, extra = divmod(P, world)
    p0 = rank * base + min(rank, extra)
    p1 = p0 + base + (1 if rank < extra else 0)
    return p0, p1


def balanced_blocks(P: int, G: int, rho: float) -> list[int]:
    """Sizes of G contiguous slice blocks whose block-scan critical paths are balanced: block g
    runs s_g carries and then one long span over the later blocks costing ρ carries per slice
    spanned, so s_g + ρ·Σ_{k>g} s_k is (as nearly as integers allow) the same for every block
    (`px_set_local_block_sizes`; the adjoint sweep uses the mirrored partition)."""
    if G < 1 or G > P:
        raise ValueError("need 1 ≤ G ≤ P blocks")
    if G == 1:
        return [P]

    def sizes_for(C):
        out = [0.0] * G
        acc = 0.0
        for g in range(G - 1, -1, -1):
            out[g] = max(C - rho * acc, 1.0)
            acc += out[g]
        return out

    lo, hi = 1.0, float(P)
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if sum(sizes_for(mid)) < P:
            lo = mid
        else:
            hi = mid
    real = sizes_for(hi)
    ints = [max(1, int(math.floor(x))) for x in real]
    # distribute the remainder to the blocks with the largest fractional parts (later blocks first)
    rem = P - sum(ints)
    order = sorted(range(G), key=lambda g: (-(real[g] - math.floor(real[g])), -g))
    i = 0
    while rem > 0:
        ints[order[i % G]] += 1
        rem -= 1
        i += 1
    while rem < 0:
        g = max(range(G), key=lambda k: ints[k])
        ints[g] -= 1
        rem += 1
    return ints
