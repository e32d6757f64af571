"""Iterative nonlinear Paraexp direct solve (Algorithm 2) — reference-facing API.

Mirrors `pkg/src/paradjoint/nonlinear.py:149-194` (`solve_direct_nonlinear`,
`NonlinearResult`) for the Burgers testbed with the configs' numerics: each
sweep freezes the slice-averaged Jacobian J(ū_p) of the current iterate, solves
the Jacobian-augmented linear problem per slice (fixed-step RK4 lanes), carries
the homogeneous parts with planned Chebyshev actions, and stops when the
max-over-slices relative change is below ``eps`` after at least ``min_iter``
sweeps (`IterationDivergence` after ``max_iter``). Runs on one GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import ConfigError
from .expaction import ChebyshevConfig
from .optimization import get_engine
from .partition import RK4Config, TimePartition, partition_equidistant
from .systems import System


@dataclass
class NonlinearResult:
    partition: TimePartition
    trajectory: np.ndarray          # (P·n_p + 1, B, n): the converged iterate at every RK4 node
    iterations: int
    error_history: list[float] = field(default_factory=list)

    @property
    def final_state(self) -> np.ndarray:
        return self.trajectory[-1]


def solve_direct_nonlinear(system: System, u0: np.ndarray, f: np.ndarray, N_slices: int, rk: RK4Config,
                           expaction: ChebyshevConfig | None = None, eps: float = 1e-3, max_iter: int = 25,
                           min_iter: int = 2, backend: str = "cuda") -> NonlinearResult:
    if backend != "cuda":
        raise ValueError(f"unknown backend {backend!r}; the B200 path provides ('cuda',)")
    if system.is_linear:
        raise ConfigError("Algorithm 2 is for the nonlinear (Burgers) testbed")
    if eps <= 0:
        raise ValueError("eps must be positive")
    ctrl = np.atleast_2d(np.asarray(f, dtype=np.float64))
    eng = get_engine(system, N_slices, rk, expaction or ChebyshevConfig(tol=1e-12), ctrl.shape[0],
                     direct="iterative", eps=eps, max_iter=max_iter, min_iter=min_iter)
    u0 = np.asarray(u0, dtype=np.float64)
    eng.set_inputs(u0, np.zeros_like(u0), ctrl)
    eng.direct_partial()
    traj = eng.get(N.PX_FIELD_TRAJ).reshape(-1, ctrl.shape[0], system.n)
    return NonlinearResult(partition_equidistant(system.spec.T, N_slices), traj, len(eng.nl_history),
                           list(eng.nl_history))
