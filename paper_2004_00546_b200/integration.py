"""The reference-side binding: what a maintainer of the reference (`paradjoint`) calls when its
backend selector is given ``"cuda"`` (the selector: `config.py:44,154-156`,
`optimization.py:154-169`).

The reference describes a problem with `Grid2D`, `ProblemSpec(kind, a, D, omega, T, f_spatial)`
and a `System` of CSR operators and closures (`problems.py:25-83`, `systems.py:27-117`); its
forcing is f_spatial·sin(ωt) (`problems.py:155-162`) and its loop's objective is tracking
(`optimization.py:84-112`). This module converts those objects to this path's structured
description — stencil coefficients, a full-field control with the time law sin(ωt), the
tracking target on the RK4 node grid — runs the GPU path and returns the results in the
reference's own layouts:

* `system_from_reference(ref_system)` → (System, f, TimeLaw, embedding);
* `direct_adjoint_loop(ref_system, f, q_true, algorithm, N, rk, leja, plan=…, dt=…)` — the
  reference's loop signature with its tracking objective; advection–diffusion with "linear" or
  "serial" runs the Paraexp linear loop (`px_set_tracking_target`: the trajectory recorded from
  the slice edge states, the adjoint with the source 2(q − q_true)); Burgers with "hybrid" or
  "serial" runs the hybrid tracking loop on the GPU (`tracking.py`): the reference's 1D-embedded
  Burgers (y-invariant U on an nx×ny grid, V ≡ 0) maps onto the 1D path, J and ∂L/∂f are
  returned on the embedded grid; a genuinely two-dimensional forcing (U and V) runs the
  two-field 2D path (`csrc/hybrid2d.cu`) in the reference's own state layout, with "hybrid",
  "serial" or "nonlinear" (Algorithm 2, ``eps`` / ``min_iter`` / ``max_iter`` as the reference's);
* `solve_direct_linear` / `solve_adjoint_linear` (`paraexp.py:221-326`) for the linear
  testbed with the reference's forcing f·sin(ωt) and a terminal adjoint condition.

The reference's adaptive DOPRI5/Leja numerics are replaced by fixed-step RK4 (``dt``) and
planned Chebyshev actions; the results agree with the reference to the discretisations'
difference (tests/test_integration_cpu.py against the reference itself, tests/test_gpu_hybrid.py
against its golden numbers).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError
from .expaction import ChebyshevConfig
from .hybrid import TimeLaw, make_hybrid_plan
from .partition import RK4Config
from .problems import ADVECTION_DIFFUSION, BURGERS, Grid, ProblemSpec
from .systems import System, build_burgers2d_system, build_field_system, build_system


@dataclass(frozen=True)
class Embedding:
    """How a converted state maps back onto the reference's state vector."""

    kind: str           # "field" (advection–diffusion, identity) or "burgers1d"
    nx: int
    ny: int

    def to_reference(self, v: np.ndarray) -> np.ndarray:
        """A 1D field (…, nx) → the reference's (…, 2·nx·ny) Burgers state (U rows, V ≡ 0)."""
        v = np.asarray(v, dtype=np.float64)
        if self.kind == "field":
            return v
        U = np.tile(v, self.ny)
        return np.concatenate([U, np.zeros_like(U)], axis=-1)


def system_from_reference(ref_system):
    """(System, f, TimeLaw, Embedding) for a reference `System` (`systems.py:27-117`)."""
    grid, spec = ref_system.grid, ref_system.spec
    nx, ny = int(grid.nx), int(grid.ny)
    f = np.asarray(spec.f_spatial, dtype=np.float64)
    law = TimeLaw.sine(float(spec.omega))
    if spec.kind == ADVECTION_DIFFUSION:
        sysm = build_field_system(Grid(nx, ny), ProblemSpec(ADVECTION_DIFFUSION, (float(spec.a), float(spec.a)),
                                                            float(spec.D), float(spec.T)))
        return sysm, f, law, Embedding("field", nx, ny)
    if spec.kind == BURGERS:
        n = nx * ny
        U, V = f[:n].reshape(ny, nx), f[n:]
        if np.any(V != 0.0) or np.any(U != U[0]):
            # genuinely two-dimensional: the two-field path (hybrid2d.cu), the reference's own layout
            sysm = build_burgers2d_system(Grid(nx, ny), ProblemSpec(BURGERS, (0.0, 0.0), float(spec.D), float(spec.T)))
            return sysm, f.copy(), law, Embedding("field", nx, ny)
        sysm = build_system(Grid(nx), ProblemSpec(BURGERS, (0.0, 0.0), float(spec.D), float(spec.T)), 2)
        return sysm, U[0].copy(), law, Embedding("burgers1d", nx, ny)
    raise ConfigError(f"unknown problem kind {spec.kind!r}")


def _node_trajectory(q_true, emb: Embedding, T: float, S: int) -> np.ndarray:
    """The reference's target `PiecewiseSolution` on the RK4 nodes, as 1D fields (S+1, nx)."""
    ts = np.linspace(0.0, T, S + 1)
    vals = np.asarray(q_true.eval_many(ts), dtype=np.float64)
    if emb.kind == "burgers1d":
        vals = vals[:, : emb.nx]   # the first row of U (y-invariant)
    return vals


@dataclass
class ReferenceLoopResult:
    """The reference's `LoopResult` fields (J, grad on the reference's state layout) plus the
    GPU loop's own result."""

    J: float
    grad: np.ndarray
    seconds: float
    cuda: object = field(repr=False, default=None)


def direct_adjoint_loop(ref_system, f, q_true, algorithm: str, N: int = 1, rk=None, leja=None, eps: float = 1e-3,
                        min_iter: int = 2, max_iter: int = 25, plan=None,
                        backend: str = "cuda", probe_nodes: int | None = None, *, dt: float,
                        expaction: ChebyshevConfig | None = None, overlap: bool = True) -> ReferenceLoopResult:
    """`paradjoint.direct_adjoint_loop` with backend="cuda" (`optimization.py:154-231`).

    ``dt`` is the fixed RK4 step replacing the reference's adaptive ``rk``; ``leja`` and
    ``probe_nodes`` are not used (planned Chebyshev actions, node-grid quadrature)."""
    from .optimization import direct_adjoint_loop as loop
    if backend != "cuda":
        raise ValueError("this binding is the cuda backend")
    forced = ref_system.with_forcing_field(np.asarray(f, dtype=np.float64)) \
        if hasattr(ref_system, "with_forcing_field") else ref_system
    sysm, f1, law, emb = system_from_reference(forced)
    T = sysm.spec.T
    if sysm.is_linear or algorithm == "nonlinear":
        # equal slices (the linear loop; the iterative nonlinear direct): whole steps per slice
        steps = max(1, int(math.ceil(T / (N * dt) - 1e-9)))
        S = N * steps
        gplan = None
    else:
        S = max(1, int(math.ceil(T / dt - 1e-9)))
        gplan = make_hybrid_plan(T, plan.N, float(plan.k)) if plan is not None else None
    target = _node_trajectory(q_true, emb, T, S)
    r = loop(sysm, f1, target, algorithm, N=N, rk=RK4Config(T / S), expaction=expaction, u0=np.zeros(sysm.n),
             objective="tracking", plan=gplan, time_law=law, overlap=overlap, eps=eps, min_iter=min_iter,
             max_iter=max_iter)
    rows = emb.ny if emb.kind == "burgers1d" else 1
    return ReferenceLoopResult(J=float(r.J) * rows, grad=emb.to_reference(np.asarray(r.grad)), seconds=r.seconds,
                               cuda=r)


def solve_direct_linear(ref_system, q0, N: int, *, dt: float, expaction: ChebyshevConfig | None = None):
    """u(T) of the reference's linear system with its forcing f·sin(ωt) (`paraexp.py:221-248`)."""
    from .solvers import solve_direct_linear as sdl
    sysm, f, law, _ = system_from_reference(ref_system)
    if not sysm.is_linear:
        raise ValueError("solve_direct_linear requires a linear testbed")
    T = sysm.spec.T
    steps = max(1, int(math.ceil(T / (N * dt) - 1e-9)))
    return sdl(sysm, q0, f[None, :], N, RK4Config(T / (N * steps)), expaction or ChebyshevConfig(tol=1e-12),
               time_law=law).final_state[0]


def solve_adjoint_linear(ref_system, qdag_T, N: int, *, dt: float, expaction: ChebyshevConfig | None = None):
    """(q†(0), ∫₀ᵀ sin(ωt)·q† dt) for the terminal condition q†(T) = ``qdag_T`` and no adjoint source
    (`paraexp.py:298-326`; the reference's `gradient_wrt_forcing` is the second value over T)."""
    from .solvers import solve_adjoint_linear as sal
    sysm, _, law, _ = system_from_reference(ref_system)
    T = sysm.spec.T
    steps = max(1, int(math.ceil(T / (N * dt) - 1e-9)))
    a = sal(sysm, qdag_T, N, RK4Config(T / (N * steps)), expaction or ChebyshevConfig(tol=1e-12), time_law=law)
    return a.initial_state[0], a.integral[0]
