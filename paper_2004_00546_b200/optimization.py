"""Reference-facing optimisation API with ``backend="cuda"``.

Mirrors `pkg/src/paradjoint/optimization.py`: ``direct_adjoint_loop``
(`:154-231`) runs one direct solve plus one adjoint solve and returns
``LoopResult(J, grad, direct, adjoint, …)``; ``descend`` (`:242-281`) is the
fixed-step steepest-descent driver with the same non-finite check.

Differences forced by the BASELINE configs: the
control is a time-constant Fourier-mode field f = Σ c_k φ_k (``f`` holds the
coefficients, batched as (B, K)); the objective is terminal,
J = ½‖u(T) − u_target‖² (``q_true`` is u_target); ∂J/∂c_k = ⟨φ_k, ∫q† dt⟩; the
initial state ``u0`` is passed through (the reference hard-wires q0 = 0,
`optimization.py:179`). ``algorithm`` is "linear" (Paraexp direct + adjoint,
advection–diffusion), "hybrid" (serial direct sweep + Paraexp adjoint with
frozen linearisation, Burgers) or "nonlinear" (Algorithm 2: iterative
Jacobian-augmented Paraexp direct, then the same frozen-linearisation adjoint,
Burgers; ``eps``/``min_iter``/``max_iter`` as `optimization.py:162-164`) or "serial"
(`optimization.py:197-203`: one RK4 sweep over the whole horizon for the direct and one for
the adjoint, no exponential actions — the one-slice case of the same kernels; ``N`` is
ignored). The only backend is "cuda": there is no CPU fallback.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .engine import EngineSpec, ParaexpEngine
from .errors import ConfigError
from .expaction import ChebyshevConfig, KrylovConfig
from .partition import RK4Config, TimePartition, partition_equidistant
from .systems import System

SERIAL = "serial"
LINEAR = "linear"
NONLINEAR = "nonlinear"
HYBRID = "hybrid"
ALGORITHMS = (SERIAL, LINEAR, NONLINEAR, HYBRID)
BACKENDS = ("cuda",)


@dataclass
class DeviceField:
    """A result field kept on the device (a snapshot of the native buffer, so later
    gradients cannot overwrite it) and copied to the host on first use. The loop's
    scalar outputs (J, ∂J/∂c) are read eagerly; the n-sized fields only when asked
    for, like the reference's lazily evaluated `PiecewiseSolution`s."""

    def __init__(self, tensor, shape, live: bool = False):
        self._t = tensor        # a view of the engine's buffer while `live`, else a private copy
        self._shape = shape
        self._host = None
        self._live = live

    def detach(self) -> None:
        """Copy-on-write: the engine calls this before new work overwrites the buffer."""
        if self._live and self._t is not None:
            self._t = self._t.clone()
        self._live = False

    def numpy(self) -> np.ndarray:
        if self._host is None:
            self._host = _to_host(self._t).reshape(self._shape)
            self._t = None
            self._live = False
        return self._host


_PINNED: dict = {}


def _to_host(t) -> np.ndarray:
    """Device tensor → a fresh numpy array through a cached pinned staging buffer (large fields: the
    D2H copy runs at the link rate instead of the pageable-memory rate)."""
    import torch
    if not t.is_cuda or t.numel() < (1 << 16):
        return t.cpu().numpy()
    key = (t.numel(), t.dtype)
    buf = _PINNED.get(key)
    if buf is None:
        if len(_PINNED) >= 4:
            _PINNED.clear()
        buf = _PINNED[key] = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
    buf.copy_(t.reshape(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return buf.numpy().copy()


def _host(v):
    return v.numpy() if isinstance(v, DeviceField) else v


@dataclass
class DirectSolution:
    """u(T) (and, when requested, the boundary states u(T_p))."""

    partition: TimePartition
    _final: object
    boundary_states: np.ndarray | None = None

    @property
    def final_state(self) -> np.ndarray:
        self._final = _host(self._final)
        return self._final


@dataclass
class AdjointSolution:
    """q†(0) and G = ∫₀ᵀ q† dt (the gradient with respect to a full control field)."""

    partition: TimePartition
    _initial: object
    _integral: object

    @property
    def initial_state(self) -> np.ndarray:
        self._initial = _host(self._initial)
        return self._initial

    @property
    def integral(self) -> np.ndarray:
        self._integral = _host(self._integral)
        return self._integral


@dataclass
class LoopResult:
    J: np.ndarray | float
    grad: np.ndarray
    direct: DirectSolution
    adjoint: AdjointSolution
    iterations: int = 1
    seconds: float = 0.0
    error_history: list[float] = field(default_factory=list)
    stats: dict = field(default_factory=dict)


@dataclass
class DescentResult:
    f_final: np.ndarray
    J_history: list
    grad_norms: list
    step_seconds: list[float]


def cost(u_T: np.ndarray, u_target: np.ndarray) -> np.ndarray:
    """J = ½‖u(T) − u_target‖² (unweighted discrete norm, `PAPER.md:149-155`)."""
    d = np.atleast_2d(u_T) - np.asarray(u_target)
    return 0.5 * np.sum(d * d, axis=-1)


def initial_condition_gradient(adjoint: AdjointSolution) -> np.ndarray:
    """∂J/∂u0 = q†(0) (`optimization.py:115-117`)."""
    return adjoint.initial_state


_ENGINES: dict = {}


def _default_expaction(system: System):
    return ChebyshevConfig(tol=1e-12)


def get_engine(system: System, N: int, rk: RK4Config, expaction, batch: int, rank: int = 0, world: int = 1,
               boundary_states: bool = False, direct: str = "serial", eps: float = 1e-3, max_iter: int = 25,
               min_iter: int = 2, law: tuple = (1.0, 0.0, 0.0, 0.0), tracking: bool = False) -> ParaexpEngine:
    """Cached engine per (problem, partition, numerics, rank): handles own HBM scratch. A cached
    engine left in the tracking objective is switched back unless ``tracking``."""
    key = (system.grid, system.spec, type(system.basis).__name__, system.basis.K, N, rk.dt, expaction, batch, rank,
           world, boundary_states, direct, eps, max_iter, min_iter, tuple(law))
    eng = _ENGINES.get(key)
    if eng is None:
        eng = ParaexpEngine(EngineSpec(system, N, rk.dt, expaction, batch, rank, world, boundary_states,
                                       direct, eps, max_iter, min_iter, law=tuple(law)))
        _ENGINES[key] = eng
    if eng.tracking and not tracking:
        eng.set_tracking_target(None)
    return eng


def release_engines() -> None:
    for e in _ENGINES.values():
        e.close()
    _ENGINES.clear()


def _dist_rank_world():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return 0, 1


def direct_adjoint_loop(
    system: System,
    f: np.ndarray,
    q_true: np.ndarray,
    algorithm: str = LINEAR,
    N: int = 1,
    rk: RK4Config | None = None,
    expaction: ChebyshevConfig | KrylovConfig | None = None,
    u0: np.ndarray | None = None,
    backend: str = "cuda",
    boundary_states: bool = False,
    distributed: bool = True,
    eps: float = 1e-3,
    min_iter: int = 2,
    max_iter: int = 25,
    hybrid_adjoint: str = "absorbed",
    objective: str = "terminal",
    plan=None,
    time_law=None,
    overlap: bool = True,
) -> LoopResult:
    """One direct solve plus one adjoint solve, yielding J and ∂J/∂c (`optimization.py:154-231`).

    ``f``: control coefficients (K,) or (B, K); ``q_true``: u_target (n,);
    ``N``: number of time slices; with ``torch.distributed`` initialised the
    slices are sharded over the ranks (contiguous blocks) unless
    ``distributed=False``. ``hybrid_adjoint`` (Burgers, ``algorithm="hybrid"``):
    "absorbed" — config 3's Option A (`solve_adjoint_varying` driven by the serial
    trajectory); "frozen_span" — the reference's `solve_hybrid` adjoint
    (`hybrid.py:194-237`: q†_T through the frozen J(ū_p)ᵀ; one rank).

    ``time_law`` (`hybrid.TimeLaw`, linear testbed, terminal objective): the control acts as
    f·θ(t) — the reference's f·sin(ωt) is ``TimeLaw.sine(ω)`` — and ∂J/∂f = ∫θ·q† dt. With a
    field system (`systems.build_field_system`) ``f`` is the forcing field and ``grad`` its field
    gradient.

    ``objective="tracking"`` runs the reference's own loop (`optimization.py:172-189`) for
    Burgers with ``algorithm`` "hybrid" or "serial": J = (1/T)∫‖u − u_t‖² dt against the target
    trajectory ``q_true`` given on the serial sweep's nodes ((S+1, n) or (S+1, B, n), e.g. from
    `tracking.synthesize_trajectory`), the forcing ``f``·θ(t) with ``time_law`` (`hybrid.TimeLaw`;
    the reference's sin(ωt) is ``TimeLaw.sine(ω)``), ``f`` a field (n,) / (B, n) or mode
    coefficients, the adjoint of the reference's `solve_hybrid` with the source 2(u − u_t) on the
    geometric partition of ``plan`` (a `HybridPlan`; None: ``N`` equal slices), each slice's
    adjoint solve overlapping the serial sweep (``overlap``), and ∂L/∂f = (1/T)∫θ·q† dt.
    """
    if objective not in ("terminal", "tracking"):
        raise ValueError(f"objective must be 'terminal' or 'tracking', not {objective!r}")
    if getattr(system, "is_burgers2d", False) and objective != "tracking":
        raise ConfigError("the two-field 2D Burgers testbed runs the reference's own loop: objective='tracking' "
                          "with algorithm 'hybrid' or 'serial'")
    if objective == "tracking":
        return _tracking_loop(system, f, q_true, algorithm, N, rk, expaction, u0, backend, plan, time_law, overlap,
                              eps, max_iter, min_iter)
    if plan is not None:
        raise ConfigError("plan: the geometric partition belongs to the hybrid tracking loop (objective='tracking')")
    law = tuple(float(v) for v in time_law.as_tuple()) if time_law is not None else (1.0, 0.0, 0.0, 0.0)
    if law[:3] != (1.0, 0.0, 0.0) and not system.is_linear:
        raise ConfigError("time_law with the terminal objective: the linear testbed (Burgers: objective='tracking')")
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; the B200 path provides {BACKENDS}")
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    if algorithm == LINEAR and not system.is_linear:
        raise ValueError("linear algorithm requires a linear testbed")
    if algorithm == SERIAL:
        # serial reference loop: a single "slice" spanning [0, T] (no exp-actions); for Burgers
        # the serial direct sweep and one time-varying adjoint lane over the whole horizon
        N = 1
    if algorithm in (HYBRID, NONLINEAR) and system.is_linear:
        raise ValueError(f"the {algorithm} path is the Burgers testbed's")
    if hybrid_adjoint not in ("absorbed", "frozen_span"):
        raise ValueError(f"hybrid_adjoint must be 'absorbed' or 'frozen_span', not {hybrid_adjoint!r}")
    if hybrid_adjoint == "frozen_span" and algorithm != HYBRID:
        raise ValueError("the frozen-span adjoint is the hybrid algorithm's (solve_hybrid)")
    if rk is None:
        raise ConfigError("rk: an RK4Config(dt) is required (fixed-step RK4)")
    expaction = expaction or _default_expaction(system)
    ctrl = np.atleast_2d(np.asarray(f, dtype=np.float64))
    B = ctrl.shape[0]
    if ctrl.shape[1] != system.basis.K:
        raise ValueError("control coefficient count does not match the basis")
    u0 = np.zeros(system.n) if u0 is None else np.asarray(u0, dtype=np.float64)
    rank, world = _dist_rank_world() if distributed else (0, 1)
    if algorithm in (NONLINEAR, SERIAL) or hybrid_adjoint == "frozen_span":
        rank, world = 0, 1  # one rank (every rank computes it identically): nothing to shard
    eng = get_engine(system, N, rk, expaction, B, rank, world, boundary_states and world == 1,
                     "iterative" if algorithm == NONLINEAR else "serial", eps, max_iter, min_iter, law)
    tick = time.perf_counter()
    eng.set_inputs(u0, np.asarray(q_true, dtype=np.float64), ctrl)
    if hybrid_adjoint != "absorbed":
        eng.set_adjoint_mode(hybrid_adjoint)
        try:
            eng.gradient()
        finally:
            eng.set_adjoint_mode("absorbed")  # cached engines default to the absorbed form
    else:
        eng.gradient()
    from . import _native as NN
    res = eng.results(fields=False)  # J and ∂J/∂c to the host; the n-sized fields stay on the device
    part = partition_equidistant(system.spec.T, N)
    bnd = None
    if boundary_states and world == 1:
        bnd = eng.get(NN.PX_FIELD_UBND).reshape(B, N + 1, system.n)
    J = res["J"] if B > 1 or np.ndim(f) > 1 else float(res["J"][0])
    grad = res["grad"] if B > 1 or np.ndim(f) > 1 else res["grad"][0]
    fields = {k: eng.snapshot(fld, (B, system.n))
              for k, fld in (("uT", NN.PX_FIELD_UT), ("qdag0", NN.PX_FIELD_QDAG0), ("G", NN.PX_FIELD_G))}
    return LoopResult(
        J, grad,
        DirectSolution(part, fields["uT"], bnd),
        AdjointSolution(part, fields["qdag0"], fields["G"]),
        iterations=len(eng.nl_history) if algorithm == NONLINEAR else 1,
        seconds=time.perf_counter() - tick,
        error_history=list(eng.nl_history) if algorithm == NONLINEAR else [],
        stats=eng.stats(),
    )


def _nonlinear_tracking_loop(system, f, q_true, N, rk, expaction, u0, time_law, eps, max_iter, min_iter):
    """The reference's loop with algorithm "nonlinear" on the two-field 2D Burgers testbed
    (`optimization.py:206-231`): Algorithm 2 direct + the zero-terminal adjoint with the tracking source."""
    from .hybrid import TimeLaw
    from .tracking import solve_nonlinear_tracking
    fa = np.asarray(f, dtype=np.float64)
    tick = time.perf_counter()
    r = solve_nonlinear_tracking(system, np.zeros(system.n) if u0 is None else u0, np.atleast_2d(fa), q_true, N, rk,
                                 expaction or ChebyshevConfig(tol=1e-12), time_law or TimeLaw.constant(), eps,
                                 max_iter, min_iter)
    single = fa.ndim == 1
    hist = list(r.timing.get("history", []))
    return LoopResult(
        float(r.J[0]) if single else r.J, r.grad[0] if single else r.grad,
        DirectSolution(r.partition, r.final_state[0] if single else r.final_state),
        AdjointSolution(r.partition, r.qdag0[0] if single else r.qdag0, r.grad[0] if single else r.grad),
        iterations=len(hist), seconds=time.perf_counter() - tick, error_history=hist,
        stats={"timing": r.timing, "offsets": r.offsets})


def _tracking_loop(system, f, q_true, algorithm, N, rk, expaction, u0, backend, plan, time_law, overlap,
                   eps=1e-3, max_iter=25, min_iter=2):
    from .hybrid import HybridPlan, TimeLaw
    from .tracking import solve_hybrid_tracking
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; the B200 path provides {BACKENDS}")
    if system.is_linear:
        return _linear_tracking_loop(system, f, q_true, algorithm, N, rk, expaction, u0, plan, time_law)
    if algorithm == NONLINEAR and getattr(system, "is_burgers2d", False):
        return _nonlinear_tracking_loop(system, f, q_true, N, rk, expaction, u0, time_law, eps, max_iter, min_iter)
    if algorithm not in (HYBRID, SERIAL):
        raise ValueError("the tracking objective runs with algorithm 'hybrid' or 'serial' "
                         "(and 'nonlinear' on the two-field 2D testbed)")
    if rk is None:
        raise ConfigError("rk: an RK4Config(dt) is required (fixed-step RK4)")
    if algorithm == SERIAL:
        plan, N = None, 1
    if plan is not None and not isinstance(plan, HybridPlan):
        raise ConfigError("plan: a HybridPlan (make_hybrid_plan)")
    law = time_law or TimeLaw.constant()
    fa = np.asarray(f, dtype=np.float64)
    n = system.n
    coeffs = fa.shape[-1] == system.basis.K and fa.shape[-1] != n
    if not coeffs and fa.shape[-1] != n:
        raise ValueError("f: a forcing field of n points or K mode coefficients")
    field_f = system.basis.field(np.atleast_2d(fa)) if coeffs else np.atleast_2d(fa)
    tick = time.perf_counter()
    r = solve_hybrid_tracking(system, np.zeros(n) if u0 is None else u0, field_f, q_true, plan, N, rk,
                              expaction or ChebyshevConfig(tol=1e-12), law, None, overlap)
    grad = system.basis.project(r.grad) if coeffs else r.grad
    single = fa.ndim == 1
    return LoopResult(
        float(r.J[0]) if single else r.J, grad[0] if single else grad,
        DirectSolution(r.partition, r.final_state[0] if single else r.final_state),
        AdjointSolution(r.partition, r.qdag0[0] if single else r.qdag0, r.grad[0] if single else r.grad),
        iterations=1, seconds=time.perf_counter() - tick, stats={"timing": r.timing, "offsets": r.offsets})


def _linear_tracking_loop(system, f, q_true, algorithm, N, rk, expaction, u0, plan, time_law):
    """The reference's linear loop with its own objective (`optimization.py:154-231`, algorithm
    "linear"): the Paraexp direct with the forcing f·θ(t), the trajectory recorded from the slice
    edge states, J = (1/T)∫‖u − u_t‖² dt, the adjoint with the source 2(u − u_t) and zero terminal
    data, ∂L/∂f = (1/T)∫θ·q† dt (`px_set_tracking_target`). One rank."""
    if algorithm not in (LINEAR, SERIAL):
        raise ValueError("the linear testbed's tracking loop runs with algorithm 'linear' or 'serial'")
    if plan is not None:
        raise ConfigError("plan: the geometric partition belongs to the Burgers hybrid")
    if rk is None:
        raise ConfigError("rk: an RK4Config(dt) is required (fixed-step RK4)")
    if algorithm == SERIAL:
        N = 1
    law = tuple(float(v) for v in time_law.as_tuple()) if time_law is not None else (1.0, 0.0, 0.0, 0.0)
    ctrl = np.atleast_2d(np.asarray(f, dtype=np.float64))
    B = ctrl.shape[0]
    if ctrl.shape[1] != system.basis.K:
        raise ValueError("f: K control values per member (a field system takes the forcing field)")
    u0 = np.zeros(system.n) if u0 is None else np.asarray(u0, dtype=np.float64)
    eng = get_engine(system, N, rk, expaction or _default_expaction(system), B, 0, 1, False, "serial", law=law,
                     tracking=True)
    S = N * eng.spec.nsteps
    torch = _torch_or_none()
    tgt = q_true if torch is not None and isinstance(q_true, torch.Tensor) else np.asarray(q_true, dtype=np.float64)
    if tuple(tgt.shape[:1]) != (S + 1,):
        raise ValueError(f"q_true: the target trajectory on the {S + 1} RK4 nodes ((S+1, n) or (S+1, B, n))")
    from . import _native as _N
    tick = time.perf_counter()
    eng.set_inputs(u0, np.zeros(system.n), ctrl)
    eng.set_tracking_target(tgt)  # get_engine restores the terminal objective for the other loops
    eng.gradient()
    res = eng.results(fields=False)
    fields = {k: eng.snapshot(fld, (B, system.n))
              for k, fld in (("uT", _N.PX_FIELD_UT), ("qdag0", _N.PX_FIELD_QDAG0), ("G", _N.PX_FIELD_G))}
    fields["traj"] = eng.snapshot(_N.PX_FIELD_TRAJ, (S + 1, B, system.n))
    bnd = eng.get(_N.PX_FIELD_UBND).reshape(B, N + 1, system.n)
    single = np.ndim(f) == 1
    part = partition_equidistant(system.spec.T, N)
    return LoopResult(
        float(res["J"][0]) if single else res["J"], res["grad"][0] if single else res["grad"],
        DirectSolution(part, fields["uT"], bnd),
        AdjointSolution(part, fields["qdag0"], fields["G"]),
        iterations=1, seconds=time.perf_counter() - tick, stats={**eng.stats(), "trajectory": fields["traj"]})


def _torch_or_none():
    try:
        import torch
        return torch
    except ImportError:  # pragma: no cover
        return None


def descend(
    system: System,
    f_init: np.ndarray,
    q_true: np.ndarray,
    steps: int,
    lr: float,
    algorithm: str = SERIAL,
    N: int = 1,
    rk: RK4Config | None = None,
    expaction=None,
    u0: np.ndarray | None = None,
    backend: str = "cuda",
    **loop_options,
) -> DescentResult:
    """Fixed-step gradient descent on the control coefficients (`optimization.py:242-281`).
    ``loop_options`` go to `direct_adjoint_loop` (objective, time_law, plan, overlap, …)."""
    if lr <= 0:
        raise ValueError("learning rate must be positive")
    f = np.array(f_init, dtype=np.float64)
    J_history, grad_norms, step_seconds = [], [], []
    for _ in range(steps):
        loop = direct_adjoint_loop(system, f, q_true, algorithm, N=N, rk=rk, expaction=expaction, u0=u0,
                                   backend=backend, **loop_options)
        if not np.all(np.isfinite(loop.J)):
            raise FloatingPointError("cost became non-finite during descent")
        J_history.append(loop.J)
        grad_norms.append(np.linalg.norm(np.atleast_2d(loop.grad), axis=-1))
        step_seconds.append(loop.seconds)
        f = f - lr * loop.grad
    return DescentResult(f, J_history, grad_norms, step_seconds)
