"""Solver-level mirrors of the reference's Paraexp entry points, ``backend="cuda"``.

The reference exposes the direct and adjoint solves separately below the loop
(`paraexp.py:221-248` `solve_direct_linear`, `:298-326` `solve_adjoint_linear`,
`:329-353` `solve_adjoint_varying`, `hybrid.py:240-290` `solve_hybrid`). These
functions run the same GPU sweeps as `direct_adjoint_loop` through one engine,
for callers that compose their own loops:

* `solve_direct_linear(system, u0, f, N, rk, …)` → `DirectSolution` (u(T), and the
  slice-boundary states u(T_p) when ``boundary_states``);
* `solve_adjoint_linear(system, qdag_T, N, rk, …)` → `AdjointSolution` (q†(0) and
  ∫₀ᵀ q† dt for the terminal condition q†(T) = ``qdag_T``; the BASELINE objective has
  no adjoint source);
* `solve_hybrid(system, u0, f, qdag_T, N, rk, …, adjoint="frozen_span")` → (`DirectSolution`,
  `AdjointSolution`) for Burgers: serial direct sweep (trajectory in HBM), then the
  Paraexp adjoint driven by it — the reference's frozen-span form by default, config 3's
  absorbed form (Option A) with ``adjoint="absorbed"``. ``qdag_T=None`` uses u(T) − ``u_target``.

Differences from the reference, as for the loop: time-constant Fourier-mode controls
``f`` (coefficients), fixed-step RK4 (`RK4Config`), planned Chebyshev/Krylov actions,
and results materialised at the slice boundaries rather than as dense
`PiecewiseSolution`s (a dense config-5 solution would be 20 480 × 33.5 MB).
"""

from __future__ import annotations

import numpy as np

from . import _native as NV
from .errors import ConfigError
from .optimization import AdjointSolution, DirectSolution, _default_expaction, get_engine
from .partition import RK4Config, partition_equidistant
from .systems import System


def _prepare(system: System, f, rk, expaction):
    if rk is None:
        raise ConfigError("rk: an RK4Config(dt) is required (fixed-step RK4)")
    ctrl = np.atleast_2d(np.asarray(f, dtype=np.float64))
    if ctrl.shape[1] != system.basis.K:
        raise ValueError("control coefficient count does not match the basis")
    return ctrl, expaction or _default_expaction(system)


def _law(time_law):
    return tuple(float(v) for v in time_law.as_tuple()) if time_law is not None else (1.0, 0.0, 0.0, 0.0)


def solve_direct_linear(system: System, u0, f, N: int, rk: RK4Config, expaction=None,
                        boundary_states: bool = False, time_law=None) -> DirectSolution:
    """u(T) of u' = A u + f·θ(t), u(0) = u0, by Paraexp over N slices (`paraexp.py:221-248`);
    f = Σ c_k φ_k (or the field itself with a field system), θ ≡ 1 unless ``time_law``."""
    if not system.is_linear:
        raise ValueError("solve_direct_linear requires a linear testbed")
    ctrl, expaction = _prepare(system, f, rk, expaction)
    B = ctrl.shape[0]
    eng = get_engine(system, N, rk, expaction, B, boundary_states=boundary_states, law=_law(time_law))
    u0 = np.asarray(u0, dtype=np.float64).reshape(-1)
    eng.set_inputs(u0, np.zeros(system.n), ctrl)
    eng.direct_partial()
    eng.finish_direct()
    uT = eng.get(NV.PX_FIELD_UT).reshape(B, system.n)
    bnd = eng.get(NV.PX_FIELD_UBND).reshape(B, N + 1, system.n) if boundary_states else None
    return DirectSolution(partition_equidistant(system.spec.T, N), uT, bnd)


def solve_adjoint_linear(system: System, qdag_T, N: int, rk: RK4Config, expaction=None,
                         batch: int = 1, time_law=None) -> AdjointSolution:
    """q†(0) and ∫₀ᵀ θ(t)·q† dt (θ ≡ 1 unless ``time_law``) of −q†' = Aᵀ q†, q†(T) = ``qdag_T``
    by Paraexp over N slices in reflected time (`paraexp.py:298-326`, absorbed final condition)."""
    if not system.is_linear:
        raise ValueError("solve_adjoint_linear requires a linear testbed (Burgers: solve_hybrid)")
    ctrl, expaction = _prepare(system, np.zeros((batch, system.basis.K)), rk, expaction)
    q = np.broadcast_to(np.asarray(qdag_T, dtype=np.float64).reshape(-1, system.n), (batch, system.n))
    eng = get_engine(system, N, rk, expaction, batch, law=_law(time_law))
    eng.set_inputs(np.zeros(system.n), np.zeros(system.n), ctrl)
    eng.set_adjoint_terminal(np.ascontiguousarray(q))
    eng.adjoint_partial()
    eng.finish_adjoint()
    return AdjointSolution(partition_equidistant(system.spec.T, N),
                           eng.get(NV.PX_FIELD_QDAG0).reshape(batch, system.n),
                           eng.get(NV.PX_FIELD_G).reshape(batch, system.n))


def solve_hybrid(system: System, u0, f, qdag_T, N: int, rk: RK4Config, expaction=None,
                 u_target=None, adjoint: str = "frozen_span") -> tuple[DirectSolution, AdjointSolution]:
    """Burgers: serial direct sweep keeping the trajectory (`hybrid.py:185-191`), then the
    Paraexp adjoint driven by it. ``qdag_T=None`` takes q†(T) = u(T) − ``u_target``.

    ``adjoint="frozen_span"`` (default, the reference's `solve_hybrid`, `hybrid.py:194-237`):
    the inhomogeneous solves start from zero terminal data and, without an adjoint source,
    vanish; q†_T is propagated over [T, 0] through the frozen J(ū_p)ᵀ. ``"absorbed"``:
    config 3's Option A — exact Jᵀ(u(t)) lanes with the final condition absorbed and the
    frozen-operator carry (`solve_adjoint_varying`, `paraexp.py:329-353`)."""
    if system.is_linear:
        raise ValueError("solve_hybrid is the Burgers testbed's")
    ctrl, expaction = _prepare(system, f, rk, expaction)
    B = ctrl.shape[0]
    if qdag_T is None and u_target is None:
        raise ValueError("give qdag_T or u_target")
    eng = get_engine(system, N, rk, expaction, B)
    eng.set_adjoint_mode(adjoint)
    try:
        ut = np.zeros(system.n) if u_target is None else np.asarray(u_target, dtype=np.float64).reshape(-1)
        eng.set_inputs(np.asarray(u0, dtype=np.float64).reshape(-1), ut, ctrl)
        eng.direct_partial()
        if qdag_T is None:
            eng.finish_direct()
        else:
            q = np.broadcast_to(np.asarray(qdag_T, dtype=np.float64).reshape(-1, system.n), (B, system.n))
            eng.set_adjoint_terminal(np.ascontiguousarray(q))
        eng.adjoint_partial()
        eng.finish_adjoint()
        part = partition_equidistant(system.spec.T, N)
        direct = DirectSolution(part, eng.get(NV.PX_FIELD_UT).reshape(B, system.n))
        adjoint_sol = AdjointSolution(part, eng.get(NV.PX_FIELD_QDAG0).reshape(B, system.n),
                                      eng.get(NV.PX_FIELD_G).reshape(B, system.n))
    finally:
        eng.set_adjoint_mode("absorbed")  # cached engines default to the absorbed form
    return direct, adjoint_sol


def synthesize_truth(system: System, f_true, rk: RK4Config, algorithm: str = "serial", N: int = 1,
                     expaction=None, u0=None) -> DirectSolution:
    """Evolve the system under the control ``f_true`` to produce the target
    (`optimization.py:66-80`); for the terminal objective the target is its u(T)
    (``final_state``). ``algorithm`` "serial" is one sweep; otherwise Paraexp over N slices."""
    u0 = np.zeros(system.n) if u0 is None else np.asarray(u0, dtype=np.float64).reshape(-1)
    if algorithm == "serial":
        N = 1
    if system.is_linear:
        return solve_direct_linear(system, u0, f_true, N, rk, expaction)
    ctrl, expaction = _prepare(system, f_true, rk, expaction)
    eng = get_engine(system, N, rk, expaction, ctrl.shape[0])
    eng.set_inputs(u0, np.zeros(system.n), ctrl)
    eng.direct_partial()
    return DirectSolution(partition_equidistant(system.spec.T, N),
                          eng.get(NV.PX_FIELD_UT).reshape(ctrl.shape[0], system.n))
